// aifmm.cu — libaifmm host orchestrator and C-ABI (include/aifmm.h).
//
// The host plans; every floating-point step runs in the batched sm_100a kernels of
// dense_kernels.cu / tree_kernels.cu / nnca_kernels.cu.  The host only handles integers:
// tree metadata, lists, colours, ranks (read back after the kernels that decide them),
// block offsets and task lists.
//
//   build  : G1 tree, G2 lists + colours, G3/G4 NNCA
//   factor : per level L..2 (Alg. 3): setup / level transition,
//            orthonormalisation (R13), per colour: compression + redirection of the pending
//            far fill-ins (§3.2.1-3.2.3), batched pivot inverses and Schur updates (P:724-729,
//            Table 4); top dense solve
//   solve  : Algorithm 4 replaying the records on nrhs columns.
#include <nvtx3/nvToolsExt.h>
#include <chrono>
#include <functional>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <numeric>

#include "runtime.cuh"
#include "dist.cuh"

namespace aifmm {

long long g_launches = 0;
void (*g_before_launch)() = nullptr;

// tree launchers
void tree_minmax(const double* pts, long long n, int d, double* part, int nparts, int* nonfinite, double* root, cudaStream_t s);
void tree_coords(const double* pts, long long n, int d, const double* root, int* kc, cudaStream_t s);
void tree_keys(const int* kc, long long n, int d, int l, int* key, cudaStream_t s);
void tree_hist(const int* key, long long n, int* cnt, cudaStream_t s);
void tree_max(const int* a, int n, int* out, cudaStream_t s);
void tree_scan(const int* cnt, int nb, long long* off, cudaStream_t s);
void tree_scatter(const int* key, long long n, const long long* off, int* cursor, int* perm, cudaStream_t s);
void tree_segsort(const long long* off, int nb, int maxlen, int* perm, cudaStream_t s);
void tree_gather(const double* pts, const int* perm, long long n, int d, double* sorted, cudaStream_t s);
void tree_level_offsets(const long long* offL, int shift, int nb_l, long long* offl, cudaStream_t s);
void tree_lists(const long long* offl, int l, int d, int ncap, int icap, int* ncnt, int* nidx, int* icnt, int* iidx, cudaStream_t s);
void tree_colour(const long long* offl, int nb, int ncap, const int* ncnt, const int* nidx, int* col, cudaStream_t s);

struct AcaTask {
  const int* R;
  const int* frange;
  const int* fidx;
  int nR, nfr, nF, kmax;
  double* Uw;
  double* Vw;
  unsigned char* rused;
  unsigned char* cused;
  int* rank;
  int* rpiv;
  int* cpiv;
};
void launch_aca(const AcaTask* t, int ntasks, const double* pts, KernelParams kp, double eps, cudaStream_t s);
void launch_aca_cluster(const AcaTask* t, int ntasks, int kmax, const double* pts, KernelParams kp, double eps,
                        cudaStream_t s);
struct KmvTarget { const int* rows; int row0, nr; double* y; int ldy; int src_begin, src_end; };
struct KmvSource { const int* cols; int col0, nc; const double* x; int ldx; int pad; };
void launch_kmv(const KmvTarget* t, const KmvSource* s, int ntargets, const double* pts, KernelParams kp, int nrhs,
                int accumulate, cudaStream_t st);
void vec_dot(const double* a, const double* b, long long n, double* part, double* out, int sqrt_mode, cudaStream_t s);
void vec_axpy(double* y, const double* x, long long n, const double* alpha, double sign, double beta, cudaStream_t s);
void vec_scale_div(double* y, const double* x, long long n, const double* den, cudaStream_t s);
void gm_givens(double* H, int ldh, double* cs, double* sn, double* g, int j, double* res, cudaStream_t s);
void gm_backsub(const double* H, int ldh, const double* g, double* y, int k, cudaStream_t s);
void gm_gemv(const double* V, long long ldv, const double* y, int k, long long n, double* out, cudaStream_t s);
void set_scalar(double* dst, const double* src, double value, cudaStream_t s);
void resid_finish(const double* part, int nchunks, long long nrows, int nrhs, const double* B, long long ldb,
                  const int* rows_user, double* out, cudaStream_t s);

// small integer kernels
__global__ void iota_kernel(int* dst, long long n, int base) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    dst[i] = base + (int)i;
}
__global__ void icopy_kernel(const int* src, int* dst, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    dst[i] = src[i];
}
// batched integer copies: task t copies n[t] ints from src[t] (or base[t] + i if src is null)
struct ICopyTask { const int* src; int* dst; int n, base; };
__global__ void icopy_tasks_kernel(const ICopyTask* __restrict__ t) {
  const ICopyTask k = t[blockIdx.x];
  for (int i = threadIdx.x; i < k.n; i += blockDim.x) k.dst[i] = k.src ? k.src[i] : k.base + i;
}
// rows permutation of an N x nrhs column-major matrix: dst[j,:] = src[perm[j],:] (gather) or
// dst[perm[j],:] = src[j,:] (scatter)
__global__ void permute_rows_kernel(const double* src, double* dst, const int* perm, long long n, int nrhs, int scatter) {
  const long long tot = n * nrhs;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.x * blockDim.x) {
    const long long j = e % n, c = e / n;
    if (scatter) dst[c * n + perm[j]] = src[c * n + j];
    else dst[c * n + j] = src[c * n + perm[j]];
  }
}
// deterministic pseudo-random fill (counter-based: splitmix64 of (seed, row, column)), uniform
// in [-1, 1): the test matrix Omega of the null-space pivot formation (R31)
struct HashFillTask { double* dst; int ld, rows, cols; unsigned long long seed; };
__device__ __forceinline__ unsigned long long splitmix64(unsigned long long x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__global__ void hash_fill_kernel(const HashFillTask* __restrict__ t) {
  const HashFillTask k = t[blockIdx.x];
  const long long tot = (long long)k.rows * k.cols;
  for (long long e = threadIdx.x; e < tot; e += blockDim.x) {
    const int i = (int)(e % k.rows), j = (int)(e / k.rows);
    const unsigned long long h = splitmix64(k.seed ^ splitmix64(((unsigned long long)i << 32) | (unsigned)j));
    k.dst[(size_t)j * k.ld + i] = (double)(h >> 11) * (2.0 / 9007199254740992.0) - 1.0;
  }
}
__global__ void finite_kernel(const double* a, long long n, int* flag) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    if (!isfinite(a[i])) *flag = 1;
}
static int gsz(long long n) { return (int)std::min<long long>(std::max<long long>((n + 255) / 256, 1), 148 * 8); }

// ------------------------------------------------------------------------------------ context
struct Rec {
  double* G = nullptr;
  int m = 0, k = 0;
  std::vector<std::pair<int, Blk>> R, C;   // (partner, block) as they were at elimination
  std::vector<char> Rkind_y, Ckind_z;      // R: column was y_q (q eliminated); C: row was Z_p
};

struct NLevel {        // NNCA per level
  std::vector<int> k, nR;              // by box id
  std::vector<long long> Roff, Uoff, skoff;
  int* dR = nullptr;                   // candidate rows (concatenated)
  int* dsk = nullptr;                  // skeletons (concatenated, by skoff)
  int* dfp = nullptr;                  // far pivots
  double* dU = nullptr;                // compact U (nR x k, ld nR) at Uoff
};

// Blocks of one level keyed by (row box p, column box q) with q in a per-box list of p (the near
// list N(p) or the interaction list IL(p); fixed capacity per box, sorted by Morton id): flat
// storage over the list slots, binary-search lookup, no hashing.
struct BlkTable {
  int nb = 0, cap = 0;
  const int* cnt = nullptr;   // list length per box
  const int* idx = nullptr;   // nb x cap list entries
  std::vector<Blk> v;
  std::vector<char> has;
  void init(int nb_, int cap_, const int* cnt_, const int* idx_) {
    nb = nb_;
    cap = cap_;
    cnt = cnt_;
    idx = idx_;
    v.assign((size_t)nb * cap, Blk{});
    has.assign((size_t)nb * cap, 0);
  }
  void clear() {
    v.clear();
    has.clear();
    nb = 0;
  }
  long long slot(long long key) const {
    if (!nb) return -1;
    const int p = (int)(key / nb), q = (int)(key % nb);
    const int* L = idx + (size_t)p * cap;
    const int* e = L + cnt[p];
    const int* it = std::lower_bound(L, e, q);
    return (it != e && *it == q) ? (long long)p * cap + (it - L) : -1;
  }
  Blk& operator[](long long key) {
    const long long s = slot(key);
    AIFMM_REQUIRE(s >= 0, AIFMM_ESINGULAR_PIVOT, "block outside the near/interaction lists");
    has[s] = 1;
    return v[s];
  }
  Blk& at(long long key) {
    const long long s = slot(key);
    AIFMM_REQUIRE(s >= 0 && has[s], AIFMM_ESINGULAR_PIVOT, "missing block");
    return v[s];
  }
  Blk* get(long long key) {
    const long long s = slot(key);
    return (s >= 0 && has[s]) ? &v[s] : nullptr;
  }
  // entry t of box p's list (no search)
  Blk& put_at(int p, int t) {
    const size_t s = (size_t)p * cap + t;
    has[s] = 1;
    return v[s];
  }
  Blk& at_slot(int p, int t) { return v[(size_t)p * cap + t]; }
};

struct FLevel {
  int l = 0, nb = 0;
  std::vector<int> boxes;
  std::vector<int> m, k, kP;           // kP: columns of Ud (parent NNCA rank)
  std::vector<int> kcap;               // rank capacity of the far (M2L) blocks of a box
  int* dinfo = nullptr;                // per-box pivot-inverse status (checked at level end)
  std::vector<double*> U, V, Ud, Vd;   // capacity: U,V m x m; Ud,Vd m x kP (ld m)
  std::vector<char> E;
  BlkTable nearb;      // current version of near blocks (over N(p))
  BlkTable A, F;       // far M2L (cap kcap_p x kcap_q), far fill m_p x m_q (distance 2); over IL(p)
  std::set<std::pair<int, int>> pending;
  // far fill-in slots live from their first Schur update to their compression (lazy_fill()):
  // free slots by capacity (doubles), capacity of each F table slot
  std::multimap<size_t, double*> ffree;
  std::vector<size_t> fcap;
  std::vector<Rec> rec;
  std::vector<int> xoff;               // row offset of child c (level l+1 id) inside its parent's x
  std::vector<long long> xrow, zrow;   // solve layout
  long long Xtot = 0, Ztot = 0;
  long long key(int p, int q) const { return (long long)p * nb + q; }
};

struct Ctx {
  cudaStream_t s = nullptr;
  bool inited = false;       // stream, uploader and flag allocated (s may legitimately be 0)
  bool own_stream = false;
  Uploader up;
  // persist: build outputs and the factor records the solve replays (pivot inverses, near-block
  // versions); scratch0/1: per-level state that dies with the next level's setup (bases, M2L,
  // far fill-ins, final near blocks), alternating by level parity; work: per-phase temporaries
  DevPool persist{(size_t)512 << 20}, work{(size_t)256 << 20}, buildp{(size_t)256 << 20};
  DevPool scratch0{(size_t)256 << 20}, scratch1{(size_t)256 << 20};
  DevPool& scr(int l) { return (l & 1) ? scratch1 : scratch0; }
  // H2 matvec (row a8): a second NNCA at the matvec tolerance on the same tree
  std::vector<NLevel> hnn;
  bool h2_built = false;
  double h2_tol = 0;
  DevPool h2pool, h2work, gmpool;
  // leaf block-diagonal inverses (GMRES precond 2, row f3)
  DevPool bdpool;
  bool bd_ready = false;
  double* bdinv = nullptr;
  std::vector<long long> bdoff;
  int d = 0, kid = 0, leaf = 0, L = 0;
  long long n = 0;
  KernelParams kp{};
  double tol = 0, tol_c = -1, tol_c_user = -1;
  int algorithm = 3;                       // 3: Alg. 3; 2: Alg. 2 (R29)
  double* pts = nullptr;                   // sorted points (device)
  int* perm = nullptr;                     // device int32
  int* dflag = nullptr;                    // device int error flag
  std::vector<std::vector<long long>> off; // host, per level
  std::vector<std::vector<int>> ncnt, nidx, icnt, iidx, col;
  int ncap = 0, icap = 0;
  std::vector<NLevel> nn;
  std::vector<FLevel> fl;
  double* topinv = nullptr;
  int topn = 0;
  std::vector<long long> topoff;
  bool built = false, factored = false;
  double stats[AIFMM_NSTATS] = {0};
  FlopCounter fc_all, fc_schur;
  bool timing = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;
  // per-phase device time (CUDA events bracketing the phase's launches on c.s) and algorithmic
  // work, for the bench's roofline entries: PH_PIVOT pivot factorisations, PH_TRI Householder
  // first stage of the RRQR, PH_PQR truncated pivoted QR, PH_REDIR redirection GEMMs
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> evp[8];
  FlopCounter fcp[8];
  // workspace budget of one batch of ACA tasks / compressions: larger batches mean fewer,
  // fuller launches (config 3: 6 -> 48 GB gave factor 4.01 -> 3.59 s, build 0.72 -> 0.63 s);
  // 26% of the device memory, between 6 and 48 GB (set_ws_budget)
  double ws_budget = 6e9;
  // ownership of the boxes of every level (-1: redundant level)
  Comm comm;
  int lp_user = -1, lp = -1;
  std::vector<std::vector<int>> owner;
  bool dist_level(int l) const { return comm.on() && l > lp && l < (int)owner.size(); }
  // debug toggle AIFMM_DIST_PHASES: bit 0 compression, 1 pivots, 2 Schur (others redundant)
  int dist_phases = getenv("AIFMM_DIST_PHASES") ? atoi(getenv("AIFMM_DIST_PHASES")) : 7;
  bool dist_ph(int l, int bit) const { return dist_level(l) && (dist_phases & bit); }
  bool mine(int l, int b, int bit = 7) const { return !dist_ph(l, bit) || owner[l][b] == comm.rank; }
  int own(int l, int b) const { return dist_level(l) ? owner[l][b] : -1; }
  // accessors
  bool nonempty(int l, int b) const { return off[l][b + 1] > off[l][b]; }
  int count(int l, int b) const { return (int)(off[l][b + 1] - off[l][b]); }
  const int* nlist(int l, int b, int* cnt) const { *cnt = ncnt[l][b]; return &nidx[l][(size_t)b * ncap]; }
  const int* ilist(int l, int b, int* cnt) const { *cnt = icnt[l][b]; return &iidx[l][(size_t)b * icap]; }
  int cheb(int l, int a, int b) const {
    int r = 0;
    for (int ax = 0; ax < d; ++ax) {
      int ca = 0, cb = 0;
      for (int bit = 0; bit < l; ++bit) {
        ca |= ((a >> (bit * d + ax)) & 1) << bit;
        cb |= ((b >> (bit * d + ax)) & 1) << bit;
      }
      r = std::max(r, std::abs(ca - cb));
    }
    return r;
  }
};



static Ctx* g_ctx = nullptr;
static std::string g_err;
// Reading R32 (symmetric records): with V = U (R27) and a symmetric kernel
// the column multipliers of an elimination are the transposes of its row multipliers
// (C_p = R_p^T), so the solve replays C_p through R_p^T and the blocks that would only serve
// as C records live in the per-level scratch pool instead of the persistent record pool
// (about half the near-block record memory).  AIFMM_FULL_RECORDS=1 keeps both (debug toggle).
// Far fill-in slots (m_p x m_q, distance-2 pairs) are allocated when a Schur update first creates
// the fill-in and recycled once it is compressed and redirected, instead of for every
// distance-2 pair at the level start (AIFMM_EAGER_FILL=1 restores the latter).  Same arithmetic:
// the creating update writes with beta = 0 where the eager slot held zeros.
static bool lazy_fill() {
  static const bool v = getenv("AIFMM_EAGER_FILL") == nullptr;
  return v;
}
static bool half_records() {
  static const bool v = getenv("AIFMM_FULL_RECORDS") == nullptr;
  return v;
}
enum { PH_PIVOT = 0, PH_TRI = 1, PH_PQR = 2, PH_REDIR = 3, PH_MULT = 4, PH_PROJ = 5, PH_FRESH = 6, PH_ORTH = 7, NPH = 8 };
// records an event pair around a phase's launches when timing is on
struct PhaseTimer {
  Ctx& c;
  int ph;
  cudaEvent_t e0 = nullptr;
  PhaseTimer(Ctx& c_, int ph_) : c(c_), ph(ph_) {
    if (!c.timing) return;
    AIFMM_CUDA(cudaEventCreate(&e0));
    AIFMM_CUDA(cudaEventRecord(e0, c.s));
  }
  ~PhaseTimer() {
    if (!e0) return;
    cudaEvent_t e1 = nullptr;
    if (cudaEventCreate(&e1) == cudaSuccess && cudaEventRecord(e1, c.s) == cudaSuccess) c.evp[ph].push_back({e0, e1});
  }
};

static Ctx& ctx() {
  if (!g_ctx) g_ctx = new Ctx();
  if (!g_ctx->inited) {
    // a blocking stream: it is ordered after work on the legacy default stream (torch's default)
    AIFMM_CUDA(cudaStreamCreate(&g_ctx->s));
    g_ctx->inited = true;
    g_ctx->own_stream = true;
    g_ctx->up.init(g_ctx->s);
    g_before_launch = [] {
      g_expose.launching();
      if (g_ctx) g_ctx->up.flush();
    };
    AIFMM_CUDA(cudaMalloc(&g_ctx->dflag, 64));
  }
  return *g_ctx;
}

static void check_flag(Ctx& c, int code, const char* msg) {
  int h = 0;
  AIFMM_CUDA(cudaMemcpyAsync(&h, c.dflag, sizeof(int), cudaMemcpyDeviceToHost, c.s));
  c.up.sync();
  if (h) {
    AIFMM_CUDA(cudaMemsetAsync(c.dflag, 0, sizeof(int), c.s));
    throw Error(code, msg);
  }
}

template <class T>
static std::vector<T> d2h(Ctx& c, const T* d, size_t n) {
  std::vector<T> h(n);
  if (n) AIFMM_CUDA(cudaMemcpyAsync(h.data(), d, n * sizeof(T), cudaMemcpyDeviceToHost, c.s));
  c.up.sync();
  return h;
}

// ------------------------------------------------------------------------------------ build
static void build_tree(Ctx& c, const double* user_pts) {
  const long long n = c.n;
  const int d = c.d;
  DevPool& P = c.buildp;
  double* part = P.d(6 * 148);
  double* root = P.d(4);
  int* kc = P.i((size_t)n * d);
  int* key = P.i(n);
  AIFMM_CUDA(cudaMemsetAsync(c.dflag, 0, 64, c.s));
  tree_minmax(user_pts, n, d, part, 148, c.dflag, root, c.s);
  check_flag(c, AIFMM_ENONFINITE, "non-finite point coordinates");
  tree_coords(user_pts, n, d, root, kc, c.s);
  int* dmax = P.i(1);
  int L = -1;
  for (int l = 2; l <= 20; ++l) {
    AIFMM_REQUIRE(d * l <= 24, AIFMM_ECOINCIDENT,
                  "cannot subdivide: more than leaf_size coincident points (tree deeper than 2^24 boxes per level)");
    const int nb = 1 << (d * l);
    int* cnt = c.work.i(nb);
    AIFMM_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int) * nb, c.s));
    AIFMM_CUDA(cudaMemsetAsync(dmax, 0, sizeof(int), c.s));
    tree_keys(kc, n, d, l, key, c.s);
    tree_hist(key, n, cnt, c.s);
    tree_max(cnt, nb, dmax, c.s);
    int mx = d2h(c, dmax, 1)[0];
    c.work.reset();
    if (mx <= c.leaf) { L = l; break; }
  }
  c.L = L;
  const int nbL = 1 << (d * L);
  int* cnt = P.i(nbL);
  int* cursor = P.i(nbL);
  long long* offL = static_cast<long long*>(P.alloc(sizeof(long long) * (nbL + 1)));
  AIFMM_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int) * nbL, c.s));
  AIFMM_CUDA(cudaMemsetAsync(cursor, 0, sizeof(int) * nbL, c.s));
  tree_keys(kc, n, d, L, key, c.s);
  tree_hist(key, n, cnt, c.s);
  tree_scan(cnt, nbL, offL, c.s);
  c.perm = static_cast<int*>(c.persist.alloc(sizeof(int) * n));
  tree_scatter(key, n, offL, cursor, c.perm, c.s);
  tree_segsort(offL, nbL, c.leaf, c.perm, c.s);
  c.pts = c.persist.d((size_t)n * d);
  tree_gather(user_pts, c.perm, n, d, c.pts, c.s);
  // offsets per level + lists + colours
  c.off.assign(L + 1, {});
  c.ncnt.assign(L + 1, {});
  c.nidx.assign(L + 1, {});
  c.icnt.assign(L + 1, {});
  c.iidx.assign(L + 1, {});
  c.col.assign(L + 1, {});
  c.ncap = (d == 2) ? 9 : 27;
  c.icap = (d == 2) ? 27 : 189;
  for (int l = 0; l <= L; ++l) {
    const int nb = 1 << (d * l);
    long long* offl = static_cast<long long*>(P.alloc(sizeof(long long) * (nb + 1)));
    tree_level_offsets(offL, d * (L - l), nb, offl, c.s);
    if (l >= 2) {
      int* ncnt = P.i(nb);
      int* nidx = P.i((size_t)nb * c.ncap);
      int* icnt = P.i(nb);
      int* iidx = P.i((size_t)nb * c.icap);
      int* col = P.i(nb);
      tree_lists(offl, l, d, c.ncap, c.icap, ncnt, nidx, icnt, iidx, c.s);
      tree_colour(offl, nb, c.ncap, ncnt, nidx, col, c.s);
      c.ncnt[l] = d2h(c, ncnt, nb);
      c.nidx[l] = d2h(c, nidx, (size_t)nb * c.ncap);
      c.icnt[l] = d2h(c, icnt, nb);
      c.iidx[l] = d2h(c, iidx, (size_t)nb * c.icap);
      c.col[l] = d2h(c, col, nb);
    }
    c.off[l] = d2h(c, offl, nb + 1);
  }
}

// NNCA operators of every level into `nnv` (device arrays from `pool`), ACA tolerance eps.
static void build_nnca(Ctx& c, std::vector<NLevel>& nnv, double eps, DevPool& pool) {
  const int L = c.L;
  nnv.assign(L + 1, NLevel{});
  for (int l = L; l >= 2; --l) {
    NLevel& nl = nnv[l];
    const int nb = 1 << (c.d * l);
    nl.k.assign(nb, 0);
    nl.nR.assign(nb, 0);
    nl.Roff.assign(nb + 1, 0);
    std::vector<int> boxes;
    for (int b = 0; b < nb; ++b)
      if (c.nonempty(l, b)) boxes.push_back(b);
    // candidate rows
    for (int b = 0; b < nb; ++b) {
      int r = 0;
      if (c.nonempty(l, b)) {
        if (l == L) r = c.count(l, b);
        else
          for (int ch = 0; ch < (1 << c.d); ++ch) r += nnv[l + 1].k[(b << c.d) | ch];
      }
      nl.nR[b] = r;
      nl.Roff[b + 1] = nl.Roff[b] + r;
    }
    nl.dR = pool.i(std::max<long long>(nl.Roff[nb], 1));
    {
      // leaf rows are point ranges; above, the children's skeletons (children have consecutive
      // ids, so their sk arrays are one contiguous run per parent)
      std::vector<ICopyTask> ic;
      for (int b : boxes) {
        if (!nl.nR[b]) continue;
        if (l == L) ic.push_back(ICopyTask{nullptr, nl.dR + nl.Roff[b], nl.nR[b], (int)c.off[l][b]});
        else ic.push_back(ICopyTask{nnv[l + 1].dsk + nnv[l + 1].skoff[(size_t)b << c.d], nl.dR + nl.Roff[b], nl.nR[b], 0});
      }
      if (!ic.empty()) { const ICopyTask* dic = c.up.put(ic); LAUNCH(icopy_tasks_kernel, (int)ic.size(), 128, 0, c.s, dic); }
    }
    // far sources per box (R11b): IL boxes' points at the leaf level, their children's
    // skeletons above.  Both are ranges of one index array: the identity at the leaves, the
    // level-(l+1) skeleton array above (whose box-ordered runs are exactly the R_D of level l).
    const int* fidx = (l == L) ? nullptr : nnv[l + 1].dsk;
    auto src_range = [&](int la, int D, int* a, int* e) {
      if (l == L) { *a = (int)c.off[la][D]; *e = (int)c.off[la][D + 1]; return; }
      const int sh = c.d * (l + 1 - la);
      *a = (int)nnv[l + 1].skoff[(size_t)D << sh];
      *e = (int)nnv[l + 1].skoff[(size_t)(D + 1) << sh];
    };
    std::vector<int> fr;
    std::vector<long long> froff(nb + 1, 0);
    std::vector<int> nF(nb, 0);
    for (int b = 0; b < nb; ++b) {
      froff[b + 1] = froff[b];
      if (!c.nonempty(l, b)) continue;
      int ni;
      const int* il = c.ilist(l, b, &ni);
      for (int t = 0; t < ni; ++t) {
        int a, e;
        src_range(l, il[t], &a, &e);
        if (e <= a) continue;
        if (froff[b + 1] > froff[b] && fr.back() == a) fr.back() = e;   // merge adjacent runs
        else { fr.push_back(a); fr.push_back(e); froff[b + 1] += 1; }
        nF[b] += e - a;
      }
      // R20: sparse neighbourhoods -> append the ancestors' interaction lists
      int la = l, ab = b;
      while (nF[b] < nl.nR[b] && la > 2) {
        --la;
        ab >>= c.d;
        const int* ila = c.ilist(la, ab, &ni);
        for (int t = 0; t < ni; ++t) {
          int a, e;
          src_range(la, ila[t], &a, &e);
          if (e <= a) continue;
          if (froff[b + 1] > froff[b] && fr.back() == a) fr.back() = e;
          else { fr.push_back(a); fr.push_back(e); froff[b + 1] += 1; }
          nF[b] += e - a;
        }
      }
    }
    // far ranges in level-lifetime device memory (not the staging arena: the chunk loop below
    // synchronises, which rewinds the arena while later chunks still read the ranges)
    int* dfr = nullptr;
    if (!fr.empty()) {
      dfr = pool.i(fr.size());
      AIFMM_CUDA(cudaMemcpyAsync(dfr, fr.data(), sizeof(int) * fr.size(), cudaMemcpyHostToDevice, c.s));
    }
    // ACA in chunks bounded by workspace
    int* drank = pool.i(nb);
    AIFMM_CUDA(cudaMemsetAsync(drank, 0, sizeof(int) * nb, c.s));
    std::vector<long long> kmaxv(nb, 0);
    long long pivtot = 0;
    std::vector<long long> pivoff(nb + 1, 0);
    for (int b = 0; b < nb; ++b) {
      kmaxv[b] = std::min<long long>(nl.nR[b], nF[b]);
      pivoff[b + 1] = pivoff[b] + kmaxv[b];
    }
    pivtot = pivoff[nb];
    int* drp = pool.i(std::max<long long>(pivtot, 1));
    int* dcp = pool.i(std::max<long long>(pivtot, 1));
    const size_t budget = getenv("AIFMM_ACA_BUDGET_GB") ? (size_t)(atof(getenv("AIFMM_ACA_BUDGET_GB")) * 1e9)
                                                        : (size_t)c.ws_budget;
    size_t i0 = 0;
    while (i0 < boxes.size()) {
      std::vector<AcaTask> tasks;
      size_t ws = 0;
      size_t i1 = i0;
      c.work.reset();
      while (i1 < boxes.size()) {
        int b = boxes[i1];
        size_t need = (size_t)kmaxv[b] * (nl.nR[b] + nF[b]) * 8 + nl.nR[b] + nF[b] + 1024;
        if (!tasks.empty() && ws + need > budget) break;
        ws += need;
        if (kmaxv[b] > 0 && c.mine(l, b)) {   // §8(e): a rank runs the ACA of its own boxes
          AcaTask t{};
          t.R = nl.dR + nl.Roff[b];
          t.frange = dfr + 2 * froff[b];
          t.fidx = fidx;
          t.nR = nl.nR[b];
          t.nfr = (int)(froff[b + 1] - froff[b]);
          AIFMM_REQUIRE(t.nfr <= 256, AIFMM_EINVALID_ARG, "too many far ranges");
          t.nF = nF[b];
          t.kmax = (int)kmaxv[b];
          t.Uw = c.work.d((size_t)t.nR * t.kmax);
          t.Vw = c.work.d((size_t)t.nF * t.kmax);
          t.rused = static_cast<unsigned char*>(c.work.alloc(t.nR));
          t.cused = static_cast<unsigned char*>(c.work.alloc(t.nF));
          t.rank = drank + b;
          t.rpiv = drp + pivoff[b];
          t.cpiv = dcp + pivoff[b];
          tasks.push_back(t);
        }
        ++i1;
      }
      // long far sets on few boxes (upper levels, 3D) go to the 8-CTA cluster kernel
      std::vector<AcaTask> small, big;
      int kbig = 1;
      // AIFMM_ACA_CLUSTER_NF (experiment): far sets at least this long go to the cluster kernel at
      // any box count (its 8 slices of a box's cross history stay L2-resident).  Measured on
      // config 3: thresholds 8192 / 4096 / 2048 neutral, 1024 +45% build time; default off
      static const int aca_cl_nf = getenv("AIFMM_ACA_CLUSTER_NF") ? atoi(getenv("AIFMM_ACA_CLUSTER_NF")) : (1 << 30);
      for (const AcaTask& t : tasks) {
        if (t.nF >= 16384 || t.nF >= aca_cl_nf || (boxes.size() < 512 && t.nF >= 1024)) {
          big.push_back(t);
          kbig = std::max(kbig, t.kmax);
        } else {
          small.push_back(t);
        }
      }
      if (!small.empty()) launch_aca(c.up.put(small), (int)small.size(), c.pts, c.kp, eps, c.s);
      if (!big.empty()) launch_aca_cluster(c.up.put(big), (int)big.size(), kbig, c.pts, c.kp, eps, c.s);
      c.up.sync();
      i0 = i1;
    }
    c.work.reset();
    nl.k = d2h(c, drank, nb);
    if (c.dist_level(l)) {   // §8(e): the owners' ranks and pivots (non-owners hold zeros)
      c.comm.allreduce_int(nl.k.data(), nb, c.s);
      for (int w = 0; w < 2; ++w) {
        int* dp = w ? dcp : drp;
        std::vector<int> h = d2h(c, dp, (size_t)std::max<long long>(pivtot, 1));
        for (int b = 0; b < nb; ++b)
          for (long long q = pivoff[b] + (c.mine(l, b) ? nl.k[b] : 0); q < pivoff[b + 1]; ++q) h[q] = 0;
        c.comm.allreduce_int(h.data(), (int)h.size(), c.s);
        AIFMM_CUDA(cudaMemcpyAsync(dp, h.data(), sizeof(int) * h.size(), cudaMemcpyHostToDevice, c.s));
        c.up.sync();
      }
    }
    // skeleton / far-pivot arrays compacted by box
    nl.skoff.assign(nb + 1, 0);
    for (int b = 0; b < nb; ++b) nl.skoff[b + 1] = nl.skoff[b] + nl.k[b];
    nl.dsk = pool.i(std::max<long long>(nl.skoff[nb], 1));
    nl.dfp = pool.i(std::max<long long>(nl.skoff[nb], 1));
    {
      std::vector<ICopyTask> ic;
      for (int b : boxes) {
        if (!nl.k[b]) continue;
        ic.push_back(ICopyTask{drp + pivoff[b], nl.dsk + nl.skoff[b], nl.k[b], 0});
        ic.push_back(ICopyTask{dcp + pivoff[b], nl.dfp + nl.skoff[b], nl.k[b], 0});
      }
      if (!ic.empty()) { const ICopyTask* dic = c.up.put(ic); LAUNCH(icopy_tasks_kernel, (int)ic.size(), 128, 0, c.s, dic); }
    }
    // operators: [A(fp,sk) | A(fp,R)] -> [I | X] by Gauss-Jordan (a solve, not an explicit
    // inverse: A(fp,sk) can be ill-conditioned), U = X^T (R10: V = U)
    nl.Uoff.assign(nb + 1, 0);
    for (int b = 0; b < nb; ++b) nl.Uoff[b + 1] = nl.Uoff[b] + (long long)nl.nR[b] * nl.k[b];
    nl.dU = pool.d(std::max<long long>(nl.Uoff[nb], 1));
    std::vector<KEvalTask> kt;
    std::vector<GJTask> gs, gg;
    long long smem_s = 0;
    int nmax_g = 1;
    CopyBatch cb;
    int* dinfo = c.work.i(nb);
    AIFMM_CUDA(cudaMemsetAsync(dinfo, 0, sizeof(int) * nb, c.s));
    AIFMM_CUDA(cudaMemsetAsync(c.dflag, 0, sizeof(int), c.s));
    for (int b : boxes) {
      const int k = nl.k[b], nr = nl.nR[b];
      if (!k || !c.mine(l, b)) continue;
      double* aug = c.work.d((size_t)k * (k + nr));
      kt.push_back(KEvalTask{aug, k, k, k, nl.dfp + nl.skoff[b], nl.dsk + nl.skoff[b], 0, 0});
      kt.push_back(KEvalTask{aug + (size_t)k * k, k, k, nr, nl.dfp + nl.skoff[b], nl.dR + nl.Roff[b], 0, 0});
      const long long need = (long long)k * (k + nr) + k + k / 2 + 2;
      if (need * 8 <= 160 * 1024) {
        gs.push_back(GJTask{aug, k, k, k + nr, 0, dinfo + b});
        smem_s = std::max(smem_s, need);
      } else {
        gg.push_back(GJTask{aug, k, k, k + nr, 0, dinfo + b});
        nmax_g = std::max(nmax_g, k);
      }
      cb.copy(aug + (size_t)k * k, k, nl.dU + nl.Uoff[b], nr, nr, k, 1.0, /*trans=*/1);
    }
    if (!kt.empty()) {
      launch_keval(c.up.put(kt), (int)kt.size(), 4, c.pts, c.kp, c.dflag, c.s);
      if (!gs.empty()) launch_gj(c.up.put(gs), (int)gs.size(), (int)smem_s, 0, c.s);
      if (!gg.empty()) launch_gj(c.up.put(gg), (int)gg.size(), -nmax_g, 0, c.s);
      cb.run(c.up, c.s);
    }
    if (c.dist_level(l)) {   // §8(e): the owners' operators U_B
      std::vector<std::vector<Region>> reg(c.comm.world);
      for (int b : boxes)
        if (nl.k[b] && nl.nR[b]) reg[c.own(l, b)].push_back(Region{nl.dU + nl.Uoff[b], nl.nR[b], nl.nR[b], nl.k[b]});
      c.comm.exchange(reg, c.up, c.s);
    }
    check_flag(c, AIFMM_ECOINCIDENT, "coincident points with a singular kernel");
    std::vector<int> info = d2h(c, dinfo, nb);
    for (int b : boxes)
      if (nl.k[b] && info[b])
        throw Error(AIFMM_ESINGULAR_SKELETON, "NNCA skeleton block singular at level " + std::to_string(l) +
                                                  " box " + std::to_string(b));
    c.work.reset();
  }
}

static void build_nnca(Ctx& c) { build_nnca(c, c.nn, c.tol / 100.0, c.persist); }   // reading R18

// ------------------------------------------------------------------------------------ factor
static inline int live(const FLevel& f, int b) { return f.E[b] ? f.k[b] : f.m[b]; }

static void setup_level(Ctx& c, int l) {
  g_expose.set("setup");
  g_prof.hstart();
  FLevel& f = c.fl[l];
  const int d = c.d, nb = 1 << (d * l);
  f.l = l;
  f.nb = nb;
  f.boxes.clear();
  for (int b = 0; b < nb; ++b)
    if (c.nonempty(l, b)) f.boxes.push_back(b);
  f.m.assign(nb, 0);
  f.k.assign(nb, 0);
  f.kP.assign(nb, 0);
  f.U.assign(nb, nullptr);
  f.V.assign(nb, nullptr);
  f.Ud.assign(nb, nullptr);
  f.Vd.assign(nb, nullptr);
  f.E.assign(nb, 0);
  f.kcap.assign(nb, 0);
  f.rec.assign(nb, Rec{});
  DevPool& S = c.scr(l);
  S.reset();   // held level l+2 (stream order makes the reuse safe)
  f.nearb.init(nb, c.ncap, c.ncnt[l].data(), c.nidx[l].data());
  f.A.init(nb, c.icap, c.icnt[l].data(), c.iidx[l].data());
  f.F.init(nb, c.icap, c.icnt[l].data(), c.iidx[l].data());
  f.pending.clear();
  f.ffree.clear();
  f.fcap.assign((size_t)nb * c.icap, 0);
  const NLevel& nl = c.nn[l];
  FLevel* prev = (l < c.L) ? &c.fl[l + 1] : nullptr;
  if (prev) prev->xoff.assign(1 << (d * (l + 1)), 0);
  for (int b : f.boxes) {
    if (l == c.L) f.m[b] = c.count(l, b);
    else {
      int o = 0;
      for (int ch = 0; ch < (1 << d); ++ch) {
        int cb = (b << d) | ch;
        if (!c.nonempty(l + 1, cb)) continue;
        prev->xoff[cb] = o;
        o += prev->k[cb];
      }
      f.m[b] = o;
    }
    f.k[b] = nl.k[b];
    f.kP[b] = (l > 2) ? c.nn[l - 1].k[b >> d] : 0;
    // compression grows ranks by ~1-1.5x the NNCA rank (measured); regrow() handles the rest
    f.kcap[b] = std::min(f.m[b], 2 * f.k[b] + 16);
  }
  f.dinfo = c.persist.i(2 * nb);   // checked once at the end of the factorisation (no level-end sync)
  AIFMM_CUDA(cudaMemsetAsync(f.dinfo, 0, sizeof(int) * 2 * nb, c.s));   // [nb, 2nb): R31 CholeskyQR
  // zero-initialised capacity storage: U, V, Ud, Vd, far A, far F
  // zero-initialised blocks are carved from the level pool; consecutive carvings are
  // contiguous within a chunk, so the memset runs over few ranges
  auto rnd = [](size_t x) { return (std::max<size_t>(x * 8, 1) + 255) & ~(size_t)255; };
  std::vector<std::pair<char*, size_t>> zr;
  size_t zchunk = (size_t)-1;
  auto carve = [&](size_t nel) {
    char* p = static_cast<char*>(S.alloc(rnd(nel)));
    // merge only within one chunk (separate allocations may be adjacent in address space)
    if (!zr.empty() && S.nchunks() == zchunk && zr.back().first + zr.back().second == p) zr.back().second += rnd(nel);
    else zr.push_back({p, rnd(nel)});
    zchunk = S.nchunks();
    return reinterpret_cast<double*>(p);
  };
  for (int b : f.boxes) {
    f.U[b] = carve((size_t)f.m[b] * f.m[b]);
    f.V[b] = carve((size_t)f.m[b] * f.m[b]);
    f.Ud[b] = carve((size_t)f.m[b] * f.kP[b]);
    f.Vd[b] = carve((size_t)f.m[b] * f.kP[b]);
    int ni;
    const int* il = c.ilist(l, b, &ni);
    for (int t = 0; t < ni; ++t) {
      int q = il[t];
      f.A.put_at(b, t) = Blk{carve((size_t)f.kcap[b] * f.kcap[q]), std::max(f.kcap[b], 1), f.k[b], f.k[q]};
      if (c.cheb(l, b, q) == 2)
        f.F.put_at(b, t) = Blk{lazy_fill() ? nullptr : carve((size_t)f.m[b] * f.m[q]), std::max(f.m[b], 1), 0, 0};
    }
  }
  for (auto& r : zr) AIFMM_CUDA(cudaMemsetAsync(r.first, 0, r.second, c.s));
  g_prof.hlap("setup.carve");
  // near blocks: allocated serially (the pools are not thread-safe) ...
  for (int b : f.boxes) {
    const int m = f.m[b];
    int nn_;
    const int* nbl = c.nlist(l, b, &nn_);
    for (int t = 0; t < nn_; ++t) {
      const int q = nbl[t];
      // the diagonal block is consumed by the pivot; off-diagonal ones are solve records: (b, q)
      // is an R record of b if b is eliminated first, else only a C record of q (R32: scratch)
      DevPool& bp = (q == b || (half_records() && c.col[l][q] < c.col[l][b])) ? S : c.persist;
      f.nearb.put_at(b, t) = Blk{bp.d(std::max<size_t>((size_t)m * f.m[q], 1)), std::max(m, 1), m, f.m[q]};
    }
  }
  g_prof.hlap("setup.nearalloc");
  // ... the fill tasks are planned on several threads (box chunks, merged in box order)
  std::vector<CopyBatch> cbt(8);
  std::vector<std::vector<KEvalTask>> ktt(8);
  const int nthr = parallel_chunks((int)f.boxes.size(), 256, [&](int lo, int hi, int th) {
    CopyBatch& cb = cbt[th];
    std::vector<KEvalTask>& kt = ktt[th];
    for (int bi = lo; bi < hi; ++bi) {
      const int b = f.boxes[bi];
      const int m = f.m[b], k = f.k[b];
      if (l == c.L) {
        cb.copy(nl.dU + nl.Uoff[b], nl.nR[b], f.U[b], m, m, k);
        cb.copy(nl.dU + nl.Uoff[b], nl.nR[b], f.V[b], m, m, k);
      } else {
        for (int ch = 0; ch < (1 << d); ++ch) {
          int cbx = (b << d) | ch;
          if (!c.nonempty(l + 1, cbx)) continue;
          cb.copy(prev->Ud[cbx], std::max(prev->m[cbx], 1), f.U[b] + prev->xoff[cbx], m, prev->k[cbx], k);
          cb.copy(prev->Vd[cbx], std::max(prev->m[cbx], 1), f.V[b] + prev->xoff[cbx], m, prev->k[cbx], k);
        }
      }
      if (l > 2) {
        // L2L / M2M: rows of the parent's NNCA operator belonging to b
        const int P = b >> d;
        const NLevel& pl = c.nn[l - 1];
        int r0 = 0;
        for (int ch = 0; ch < (b & ((1 << d) - 1)); ++ch) r0 += nl.k[(P << d) | ch];
        cb.copy(pl.dU + pl.Uoff[P] + r0, pl.nR[P], f.Ud[b], std::max(m, 1), k, f.kP[b]);
        cb.copy(pl.dU + pl.Uoff[P] + r0, pl.nR[P], f.Vd[b], std::max(m, 1), k, f.kP[b]);
      }
      // near blocks (current version = X_p x x_q)
      int nn_;
      const int* nbl = c.nlist(l, b, &nn_);
      for (int t = 0; t < nn_; ++t) {
        const int q = nbl[t];
        const Blk& blk = f.nearb.at_slot(b, t);
        if (l == c.L) {
          // evaluated from the block table below (keval_table_kernel, mode 1)
        } else {
          for (int ch = 0; ch < (1 << d); ++ch) {
            int c1 = (b << d) | ch;
            if (!c.nonempty(l + 1, c1)) continue;
            for (int ch2 = 0; ch2 < (1 << d); ++ch2) {
              int c2 = (q << d) | ch2;
              if (!c.nonempty(l + 1, c2)) continue;
              const Blk* it = prev->nearb.get(prev->key(c1, c2));
              const Blk& src = it ? *it : prev->A.at(prev->key(c1, c2));
              cb.copy(src.p, src.ld, blk.p + (size_t)prev->xoff[c2] * blk.ld + prev->xoff[c1], blk.ld,
                      prev->k[c1], prev->k[c2]);
            }
          }
        }
      }
      // M2L A(sk b, sk q): evaluated from the block table below (mode 0)
    }
  });
  g_prof.hlap("setup.par");
  CopyBatch cb;
  std::vector<KEvalTask> kt;
  for (int t = 0; t < nthr; ++t) {
    cb.append(cbt[t]);
    kt.insert(kt.end(), ktt[t].begin(), ktt[t].end());
  }
  g_prof.hlap("setup.plan");
  cb.run(c.up, c.s);
  if (!kt.empty()) launch_keval(c.up.put(kt), (int)kt.size(), 4, c.pts, c.kp, c.dflag, c.s);
  {
    // kernel-entry blocks straight from the block tables: M2L A(sk b, sk q) at every
    // level, the near blocks at the leaf level (one upload of the tables, no task lists)
    static_assert(sizeof(Blk) == sizeof(BlkDev), "Blk / BlkDev layout");
    const void* dA = c.up.put(f.A.v);
    const int* dicnt = c.up.put(c.icnt[l]);
    const int* diidx = c.up.put(c.iidx[l]);
    const long long* dsko = c.up.put(nl.skoff);
    launch_keval_table(dA, dicnt, diidx, nb, c.icap, 0, nl.dsk, dsko, c.pts, c.kp, c.dflag, c.s);
    if (l == c.L) {
      const void* dN = c.up.put(f.nearb.v);
      const int* dncnt = c.up.put(c.ncnt[l]);
      const int* dnidx = c.up.put(c.nidx[l]);
      const long long* doff = c.up.put(c.off[l]);
      launch_keval_table(dN, dncnt, dnidx, nb, c.ncap, 1, nullptr, doff, c.pts, c.kp, c.dflag, c.s);
    }
  }
  g_prof.hlap("setup.launch");
  // level l+1's per-level state is dead once copied: mark its pool free (reused by level l-1,
  // or given back by an out-of-memory trim)
  if (prev) c.scr(l + 1).reset();
}

// R13: U_b = Q T, V_b = Q' T'; rows of Z_b <- T (.), columns of y_b <- (.) T'^T
// CholeskyQR2 (two passes of G = B^T B, G = R^T R, B <- B R^{-1}) for every box's U and V at
// once: DMMA GEMMs plus one batched Cholesky; T = R2 R1 so that B_old = Q T.  Returns false if
// a Gram matrix is not numerically positive definite (then the pivoted-QR path runs instead).
static bool bases_cholqr2(Ctx& c, FLevel& f, std::vector<double*>& T, std::vector<double*>& T2) {
  // V_b = U_b bitwise at every level start (R27: V's new columns are copies of U's; R10 at the
  // leaves; the same operations on Ud and Vd above), so only U is factored: V <- Q, T' = T
  std::vector<int> bx;
  int kmax = 0;
  for (int b : f.boxes)
    if (f.k[b]) { bx.push_back(b); kmax = std::max(kmax, f.k[b]); }
  if (bx.empty()) return true;
  const int nt = (int)bx.size();
  int* dinfo = c.work.i(2 * nt);
  AIFMM_CUDA(cudaMemsetAsync(dinfo, 0, sizeof(int) * 2 * nt, c.s));
  std::vector<double*> B(nt), Q1(nt), G(nt), R1(nt), R1i(nt), R2(nt), R2i(nt);
  for (int t = 0; t < nt; ++t) {
    const int b = bx[t], m = f.m[b], k = f.k[b];
    B[t] = f.U[b];
    Q1[t] = c.work.d((size_t)m * k);
    G[t] = c.work.d((size_t)k * k);
    R1[t] = c.work.d((size_t)k * k);
    R1i[t] = c.work.d((size_t)k * k);
    R2[t] = c.work.d((size_t)k * k);
    R2i[t] = c.work.d((size_t)k * k);
  }
  auto pass = [&](std::vector<double*>& src, std::vector<double*>& R, std::vector<double*>& Ri, int info0) {
    GemmBatch g;
    for (int t = 0; t < nt; ++t) {
      const int b = bx[t], m = f.m[b], k = f.k[b];
      g.task(G[t], k, k, k, 0.0);
      g.term(1.0, src[t], m, 1, src[t], m, 0, m);
    }
    g.run(c.up, c.s, &c.fc_all);
    std::vector<CholTask> ct(nt);
    for (int t = 0; t < nt; ++t) ct[t] = CholTask{G[t], R[t], Ri[t], f.k[bx[t]], 0, dinfo + info0 + t};
    launch_chol_inv(c.up.put(ct), nt, kmax, c.s);
  };
  pass(B, R1, R1i, 0);
  {
    GemmBatch g;
    for (int t = 0; t < nt; ++t) {
      const int b = bx[t], m = f.m[b], k = f.k[b];
      g.task(Q1[t], m, m, k, 0.0);
      g.term(1.0, B[t], m, 0, R1i[t], k, 0, k);
    }
    g.run(c.up, c.s, &c.fc_all);
  }
  pass(Q1, R2, R2i, nt);
  std::vector<int> info = d2h(c, dinfo, 2 * nt);
  for (int v : info)
    if (v) return false;
  GemmBatch g;
  for (int t = 0; t < nt; ++t) {
    const int b = bx[t], m = f.m[b], k = f.k[b];
    double* Tt = c.work.d((size_t)k * k);
    T[b] = T2[b] = Tt;
    g.task(B[t], m, m, k, 0.0);                 // Q = Q1 R2^{-1}
    g.term(1.0, Q1[t], m, 0, R2i[t], k, 0, k);
    g.task(Tt, k, k, k, 0.0);                   // T = R2 R1
    g.term(1.0, R2[t], k, 0, R1[t], k, 0, k);
  }
  g.run(c.up, c.s, &c.fc_all);
  CopyBatch vc;
  for (int b : bx) vc.copy(f.U[b], f.m[b], f.V[b], f.m[b], f.m[b], f.k[b]);
  vc.run(c.up, c.s);
  return true;
}

// pivoted Gram-Schmidt variant (fallback): Q by the RRQR kernel with tmin = tmax = k, T = Q^T B
static void bases_pqr(Ctx& c, FLevel& f, std::vector<double*>& T, std::vector<double*>& T2) {
  std::vector<double*> Uold(f.nb, nullptr), Vold(f.nb, nullptr);
  CopyBatch cb;
  std::vector<PqrTask> pq;
  for (int b : f.boxes) {
    const int m = f.m[b], k = f.k[b];
    if (!k) continue;
    Uold[b] = c.work.d((size_t)m * k);
    Vold[b] = c.work.d((size_t)m * k);
    double* wu = c.work.d((size_t)m * k);
    double* wv = c.work.d((size_t)m * k);
    cb.copy(f.U[b], m, Uold[b], m, m, k);
    cb.copy(f.U[b], m, wu, m, m, k);
    cb.copy(f.V[b], m, Vold[b], m, m, k);
    cb.copy(f.V[b], m, wv, m, m, k);
    pq.push_back(PqrTask{wu, f.U[b], m, m, m, k, 0, k, k, 0, nullptr, 0.0, nullptr, nullptr});
    pq.push_back(PqrTask{wv, f.V[b], m, m, m, k, 0, k, k, 0, nullptr, 0.0, nullptr, nullptr});
  }
  cb.run(c.up, c.s);
  if (!pq.empty()) run_pqr(pq, c.up, c.s);
  GemmBatch g;
  for (int b : f.boxes) {
    const int m = f.m[b], k = f.k[b];
    if (!k) continue;
    T[b] = c.work.d((size_t)k * k);
    T2[b] = c.work.d((size_t)k * k);
    g.task(T[b], k, k, k, 0.0);
    g.term(1.0, f.U[b], m, 1, Uold[b], m, 0, m);
    g.task(T2[b], k, k, k, 0.0);
    g.term(1.0, f.V[b], m, 1, Vold[b], m, 0, m);
  }
  g.run(c.up, c.s, &c.fc_all);
}

static void orthonormalise(Ctx& c, FLevel& f) {
  g_expose.set("orth");
  const int l = f.l;
  std::vector<double*> T(f.nb, nullptr), T2(f.nb, nullptr);
  g_prof.begin(c.s);
  static const bool orth_pqr = getenv("AIFMM_ORTH_PQR") != nullptr;   // debug toggle
  if (orth_pqr || !bases_cholqr2(c, f, T, T2)) {
    c.work.reset();
    bases_pqr(c, f, T, T2);
    c.stats[AIFMM_STAT_HOST_SYNCS] += 0;   // (fallback taken: pivoted Gram-Schmidt bases)
    g_prof.end("orth.pqr_fallback");
  } else {
    g_prof.end("orth.cholqr2");
  }
  CopyBatch cb;
  GemmBatch g;
  // Ud <- T Ud, Vd <- T' Vd ; A_pq <- T_p A_pq T'_q^T
  std::vector<double*> udc(f.nb, nullptr), vdc(f.nb, nullptr);
  std::vector<double*> tmpA((size_t)f.nb * c.icap, nullptr);   // by IL slot of (b, q)
  for (int b : f.boxes) {
    const int m = f.m[b], k = f.k[b];
    if (!k) continue;
    if (f.kP[b]) {
      udc[b] = c.work.d((size_t)k * f.kP[b]);
      vdc[b] = c.work.d((size_t)k * f.kP[b]);
      cb.copy(f.Ud[b], m, udc[b], k, k, f.kP[b]);
      cb.copy(f.Vd[b], m, vdc[b], k, k, f.kP[b]);
    }
    int ni;
    const int* il = c.ilist(l, b, &ni);
    for (int t = 0; t < ni; ++t) {
      int q = il[t];
      if (!f.k[q]) continue;
      if (k <= ORTH_SW_KMAX && f.k[q] <= ORTH_SW_KMAX) continue;   // orth_sandwich_kernel below
      double* tp = c.work.d((size_t)k * f.k[q]);
      tmpA[(size_t)b * c.icap + t] = tp;
      const Blk& a = f.A.at_slot(b, t);
      g.task(tp, k, k, f.k[q], 0.0);
      g.term(1.0, a.p, a.ld, 0, T2[q], f.k[q], 1, f.k[q]);
    }
  }
  cb.run(c.up, c.s);
  g.run(c.up, c.s, &c.fc_all);
  for (int b : f.boxes) {
    const int m = f.m[b], k = f.k[b];
    if (!k) continue;
    if (f.kP[b]) {
      g.task(f.Ud[b], m, k, f.kP[b], 0.0);
      g.term(1.0, T[b], k, 0, udc[b], k, 0, k);
      g.task(f.Vd[b], m, k, f.kP[b], 0.0);
      g.term(1.0, T2[b], k, 0, vdc[b], k, 0, k);
    }
    int ni;
    const int* il = c.ilist(l, b, &ni);
    for (int t = 0; t < ni; ++t) {
      int q = il[t];
      if (!f.k[q]) continue;
      if (k <= ORTH_SW_KMAX && f.k[q] <= ORTH_SW_KMAX) continue;
      const Blk& a = f.A.at_slot(b, t);
      g.task(a.p, a.ld, k, f.k[q], 0.0);
      g.term(1.0, T[b], k, 0, tmpA[(size_t)b * c.icap + t], k, 0, k);
    }
  }
  g.run(c.up, c.s, &c.fc_all);
  // the small far blocks: one fused T_b A T'_q^T per block table slot
  const void* dA = c.up.put(f.A.v);
  const int* dicnt = c.up.put(c.icnt[l]);
  const int* diidx = c.up.put(c.iidx[l]);
  double* const* dT = c.up.put(T);
  double* const* dT2 = c.up.put(T2);
  launch_orth_sandwich(dA, dicnt, diidx, f.nb, c.icap, dT, dT2, c.s);
  c.work.reset();   // stream order: later writes to these temporaries follow the reads
}

// Far (M2L) blocks are stored with a per-box rank capacity kcap; when compression grows a box's
// rank past it, every block in that box's Z row and y column moves to larger zero-padded storage.
static void regrow(Ctx& c, FLevel& f, const std::vector<int>& grown) {
  if (grown.empty()) return;
  std::vector<int> ncap = f.kcap;
  for (int b : grown) ncap[b] = std::min(f.m[b], std::max(f.k[b], f.kcap[b] + f.kcap[b] / 2 + 8));
  std::set<long long> keys;
  for (int b : grown) {
    int ni;
    const int* il = c.ilist(f.l, b, &ni);
    for (int t = 0; t < ni; ++t) {
      keys.insert(f.key(b, il[t]));
      keys.insert(f.key(il[t], b));
    }
  }
  DevPool& S = c.scr(f.l);
  CopyBatch zero, mv;
  for (long long key : keys) {
    const int p = (int)(key / f.nb), q = (int)(key % f.nb);
    Blk& A = f.A.at(key);
    Blk nb_{S.d(std::max<size_t>((size_t)ncap[p] * ncap[q], 1)), std::max(ncap[p], 1), A.rows, A.cols};
    zero.fill(nb_.p, nb_.ld, ncap[p], ncap[q], 0.0);
    mv.copy(A.p, A.ld, nb_.p, nb_.ld, f.kcap[p], f.kcap[q]);
    A = nb_;
  }
  zero.run(c.up, c.s);
  mv.run(c.up, c.s);
  f.kcap = ncap;
}

// Phase 1 of the compression for a group of affected boxes: new basis columns (written into
// U_b after column k_b, copied into V_b: reading R27) and the rank growth tgt (R8, R8b).  The
// group's temporaries live in c.work; the rank read-back at the end synchronises the stream.
static void compress_boxes(Ctx& c, FLevel& f, const std::vector<int>& aff, std::map<int, std::vector<int>>& part,
                           std::vector<int>& tgt) {
  const int na = (int)aff.size();
  if (g_prof.on) g_prof.begin(c.s);
  // candidates stored transposed (rows = fill-in columns): WT = [F_bq^T ...] (row X_b, R27: the
  // column-side fill-ins are their transposes, so one side is compressed)
  struct Side { double* WT; int n; double* M; int r; };
  std::vector<Side> su(na);
  double* dnorm = c.work.d(2 * na);
  int* dt = c.work.i(4 * na);
  CopyBatch cb;
  std::vector<NormTask> nt;
  AIFMM_CUDA(cudaMemsetAsync(dt, 0, sizeof(int) * 4 * na, c.s));
  std::vector<char> full(na, 0);
  g_expose.set("cmp.gather");
  g_prof.hstart();
  for (int a = 0; a < na; ++a) {
    int b = aff[a];
    const int m = f.m[b];
    if (f.k[b] >= m) {            // basis already spans R^m: nothing to add (t = 0)
      full[a] = 1;
      su[a] = Side{nullptr, 0, nullptr, 0};
      continue;
    }
    int nu = 0;
    for (int q : part[b]) nu += live(f, q);
    su[a].n = nu;
    su[a].WT = c.work.d((size_t)std::max(nu, 1) * m);
    su[a].r = std::min(nu, m);
    su[a].M = c.work.d((size_t)m * std::max(su[a].r, 1));
    int o = 0;
    for (int q : part[b]) {
      const Blk& fb = f.F.at(f.key(b, q));   // row X_b, column of q: m x live_q -> transposed
      if (fb.p) cb.copy(fb.p, fb.ld, su[a].WT + o, nu, live(f, q), m, 1.0, /*trans=*/1);
      else cb.fill(su[a].WT + o, nu, live(f, q), m, 0.0);   // never created (a zero-size update)
      o += live(f, q);
    }
    nt.push_back(NormTask{su[a].WT, std::max(nu, 1), nu, m, dnorm + 2 * a});
  }
  g_prof.hlap("cmp.gather");
  cb.run(c.up, c.s);
  launch_norm(c.up.put(nt), (int)nt.size(), c.s);
  if (g_prof.on) { g_prof.end("cmp.gather"); g_prof.begin(c.s); }
  // projection W <- (I - B B^T) W, i.e. WT <- WT - (WT B) B^T
  g_expose.set("cmp.proj");
  GemmBatch g;
  {
    PhaseTimer pt(c, PH_PROJ);
    std::vector<double*> tu(na);
    for (int a = 0; a < na; ++a) {
      int b = aff[a];
      const int m = f.m[b], k = f.k[b], nu = su[a].n;
      if (!k || !nu) continue;
      tu[a] = c.work.d((size_t)nu * k);
      g.task(tu[a], nu, nu, k, 0.0);
      g.term(1.0, su[a].WT, nu, 0, f.U[b], m, 0, m);
    }
    {
      FlopCounter fp;
      g.run(c.up, c.s, &fp);
      c.fc_all.flops += fp.flops;
      c.fcp[PH_PROJ].flops += fp.flops;
      c.fcp[PH_PROJ].bytes += fp.bytes;
    }
    for (int a = 0; a < na; ++a) {
      int b = aff[a];
      const int m = f.m[b], k = f.k[b], nu = su[a].n;
      if (!k || !nu) continue;
      g.task(su[a].WT, nu, nu, m, 1.0);
      g.term(-1.0, tu[a], nu, 0, f.U[b], m, 1, k);
    }
    FlopCounter fp;
    g.run(c.up, c.s, &fp);
    c.fc_all.flops += fp.flops;
    c.fcp[PH_PROJ].flops += fp.flops;
    c.fcp[PH_PROJ].bytes += fp.bytes;
  }
  // two-stage RRQR (R8b): M = R^T with WT = Q R
  std::vector<TriRootReq> tr;
  for (int a = 0; a < na; ++a) {
    int b = aff[a];
    const int m = f.m[b], nu = su[a].n;
    if (!nu || !m) continue;
    tr.push_back(TriRootReq{su[a].WT, nu, nu, m, su[a].M, m});
  }
  g_expose.set("cmp.tri");
  {
    PhaseTimer pt(c, PH_TRI);
    FlopCounter fp;
    batched_tri_root(tr, c.work, c.up, c.s, &fp);
    c.fc_all.flops += fp.flops;
    c.fcp[PH_TRI].flops += fp.flops;
    // algorithmic: read each candidate matrix once, write its triangular root once
    for (const TriRootReq& q : tr) c.fcp[PH_TRI].bytes += 8.0 * ((double)q.n * q.m + (double)q.m * std::min(q.n, q.m));
  }
  g_expose.set("cmp.pqr");
  if (g_prof.on) { g_prof.end("cmp.proj+triroot"); g_prof.begin(c.s); }
  // truncated pivoted QR (R8): tmin = 0, so the columns taken are exactly the t_trunc of R8
  std::vector<PqrTask> pq;
  for (int a = 0; a < na; ++a) {
    int b = aff[a];
    const int m = f.m[b], k = f.k[b];
    if (full[a]) continue;
    pq.push_back(PqrTask{su[a].M, f.U[b], m, m, m, su[a].r, k, 0, m - k, 0, dnorm + 2 * a, c.tol_c, dt + 4 * a, dt + 4 * a + 1});
  }
  if (!pq.empty()) {
    PhaseTimer pt(c, PH_PQR);
    run_pqr(pq, c.up, c.s);
    // algorithmic: read each m x r candidate matrix once and write the new basis columns (the
    // number taken is decided on the device; counted as the read only)
    for (const PqrTask& t : pq) c.fcp[PH_PQR].bytes += 8.0 * (double)t.m * t.ncols;
  }
  std::vector<int> th = d2h(c, dt, 4 * na);
  g_expose.set("cmp.post");
  if (g_prof.on) { g_prof.end("cmp.pqrA"); g_prof.begin(c.s); }
  tgt.assign(na, 0);
  // R27: V_b's new columns are U_b's
  CopyBatch vb;
  for (int a = 0; a < na; ++a) {
    int b = aff[a];
    const int m = f.m[b], k = f.k[b];
    if (full[a]) continue;
    tgt[a] = std::min(th[4 * a + 1], m - k);
    vb.copy(f.U[b] + (size_t)k * m, m, f.V[b] + (size_t)k * m, m, m, tgt[a]);
  }
  vb.run(c.up, c.s);
  if (g_prof.on) { g_prof.end("cmp.pqrB"); g_prof.begin(c.s); }
}

// Alg. 3 lines P:1118-1129 for the pending pairs S (colour-batched, R12; R14, R15)
// after_ranks runs as soon as the new ranks are known (before the regrow / redirection
// planning): the caller launches the colour's pivot inverses there, which need only the final
// bases, so the GPU works on them while the host plans the redirection.
static void compress(Ctx& c, FLevel& f, const std::vector<std::pair<int, int>>& S,
                     const std::function<void()>& after_ranks) {
  g_expose.set("cmp.pre");
  std::map<int, std::vector<int>> part;
  for (auto& pr : S) {
    part[pr.first].push_back(pr.second);
    part[pr.second].push_back(pr.first);
  }
  std::vector<int> aff;
  for (auto& kv : part) {
    std::sort(kv.second.begin(), kv.second.end());
    if (!f.E[kv.first]) aff.push_back(kv.first);
  }
  const int na = (int)aff.size();
  if (!na) {
    after_ranks();
    return;
  }
  if (g_prof.on) g_prof.begin(c.s);
  // phase 1 in groups whose temporaries stay under a workspace budget
  std::vector<int> tgt(na, 0);
  {
    const double budget = getenv("AIFMM_CMP_BUDGET_GB") ? atof(getenv("AIFMM_CMP_BUDGET_GB")) * 1e9 : c.ws_budget;
    size_t a0 = 0;
    while (a0 < aff.size()) {
      double ws = 0.0;
      size_t a1 = a0;
      while (a1 < aff.size()) {
        const int b = aff[a1], m = f.m[b];
        int nu = 0;
        for (int q : part[b]) nu += live(f, q);
        const double need = 8.0 * (4.0 * nu * m + 2.0 * m * m + 2.0 * nu * 32 + 4.0 * 32 * m) + 4096.0;
        if (a1 > a0 && ws + need > budget) break;
        ws += need;
        ++a1;
      }
      std::vector<int> grp(aff.begin() + a0, aff.begin() + a1), tg;
      if (c.dist_ph(f.l, 1)) {   // §8(e): a rank compresses its own boxes only
        std::vector<int> pos_;
        std::vector<int> mine_;
        for (size_t t = 0; t < grp.size(); ++t)
          if (c.mine(f.l, grp[t])) { pos_.push_back((int)t); mine_.push_back(grp[t]); }
        if (!mine_.empty()) compress_boxes(c, f, mine_, part, tg);
        for (size_t t = 0; t < pos_.size(); ++t) tgt[a0 + pos_[t]] = tg[t];
      } else {
        compress_boxes(c, f, grp, part, tg);
        for (size_t t = 0; t < grp.size(); ++t) tgt[a0 + t] = tg[t];
      }
      c.work.reset();
      a0 = a1;
    }
  }
  if (c.dist_ph(f.l, 1)) {
    // the owners' new ranks, then their new basis columns U_b[:, k:k+t] (and V_b's, R27)
    c.comm.allreduce_int(tgt.data(), na, c.s);
    std::vector<std::vector<Region>> reg(c.comm.world);
    for (int a = 0; a < na; ++a) {
      const int b = aff[a], m = f.m[b], k = f.k[b];
      if (!tgt[a]) continue;
      auto& R = reg[c.own(f.l, b)];
      R.push_back(Region{f.U[b] + (size_t)k * m, m, m, tgt[a]});
      R.push_back(Region{f.V[b] + (size_t)k * m, m, m, tgt[a]});
    }
    c.comm.exchange(reg, c.up, c.s);
  }
  // new ranks
  std::vector<int> grown;
  for (int a = 0; a < na; ++a) {
    int b = aff[a];
    f.k[b] += tgt[a];
    if (f.k[b] > f.kcap[b]) grown.push_back(b);
    c.stats[AIFMM_STAT_COMPRESSIONS] += 1;
  }
  after_ranks();
  g_expose.set("cmp.redirect");
  regrow(c, f, grown);
  for (int b : aff) {   // only the compressed boxes' ranks changed
    int ni;
    const int* il = c.ilist(f.l, b, &ni);
    for (int t = 0; t < ni; ++t) {
      f.A.at_slot(b, t).rows = f.k[b];
      f.A.at(f.key(il[t], b)).cols = f.k[b];
    }
  }
  // redirection: A_xy += U~_x^* F_xy V~_y  (P2P) | F V~ (P2L) | U~^* F (M2P)
  g_prof.hstart();
  GemmBatch g;
  CopyBatch cb;
  std::vector<std::pair<std::pair<int, int>, double*>> p2p;
  for (auto& pr : S)
    for (int dir = 0; dir < 2; ++dir) {
      int x = dir ? pr.second : pr.first, y = dir ? pr.first : pr.second;
      const Blk& F = f.F.at(f.key(x, y));
      if (!f.E[x] && !f.E[y]) {
        double* tp = c.work.d((size_t)f.m[x] * std::max(f.k[y], 1));
        g.task(tp, f.m[x], f.m[x], f.k[y], 0.0);
        if (F.p) g.term(1.0, F.p, F.ld, 0, f.V[y], f.m[y], 0, f.m[y]);
        p2p.push_back({{x, y}, tp});
      }
    }
  g.run(c.up, c.s, &c.fc_all);
  size_t pi_ = 0;
  for (auto& pr : S)
    for (int dir = 0; dir < 2; ++dir) {
      int x = dir ? pr.second : pr.first, y = dir ? pr.first : pr.second;
      const Blk& F = f.F.at(f.key(x, y));
      const Blk& A = f.A.at(f.key(x, y));
      if (!f.E[x] && !f.E[y]) {
        double* tp = p2p[pi_++].second;
        g.task(A.p, A.ld, f.k[x], f.k[y], 1.0);
        g.term(1.0, f.U[x], f.m[x], 1, tp, f.m[x], 0, f.m[x]);
      } else if (f.E[x] && !f.E[y]) {
        g.task(A.p, A.ld, f.k[x], f.k[y], 1.0);
        if (F.p) g.term(1.0, F.p, F.ld, 0, f.V[y], f.m[y], 0, f.m[y]);
      } else {
        g.task(A.p, A.ld, f.k[x], f.k[y], 1.0);
        if (F.p) g.term(1.0, f.U[x], f.m[x], 1, F.p, F.ld, 0, f.m[x]);
      }
      if (!lazy_fill()) cb.fill(F.p, F.ld, live(f, x), live(f, y), 0.0);
    }
  g_prof.hlap("cmp.redirect");
  {
    PhaseTimer pt(c, PH_REDIR);
    FlopCounter fp;
    g.run(c.up, c.s, &fp);
    c.fc_all.flops += fp.flops;
    c.fcp[PH_REDIR].flops += fp.flops;
    c.fcp[PH_REDIR].bytes += fp.bytes;
  }
  cb.run(c.up, c.s);
  for (auto& pr : S) f.pending.erase(pr);
  if (lazy_fill()) {
    // the compressed pairs' slots are free for later fill-ins: their next writer is planned
    // after this point, so in stream order it follows these reads
    for (auto& pr : S)
      for (int dir = 0; dir < 2; ++dir) {
        const int x = dir ? pr.second : pr.first, y = dir ? pr.first : pr.second;
        const long long sl = f.F.slot(f.key(x, y));
        Blk& F = f.F.v[sl];
        if (!F.p) continue;
        f.ffree.insert({f.fcap[sl], F.p});
        F.p = nullptr;
      }
  }
  if (g_prof.on) g_prof.end("cmp.redirect");
}

// Host plan of a colour's Schur updates (Table 4, Alg. 3), built BEFORE
// the colour's compression so that it overlaps the GPU work still queued for the previous colour.
// Nothing in it depends on the ranks the compression decides: targets are neighbours of the
// colour's boxes (live sizes fixed), block pointers do not move (regrow() only touches blocks of
// boxes that are not eliminated), and the operand W_i = G[:, 0:m] R_i is referenced by column
// offset and patched once n_i = m_i + k_i is known.
struct SchurPlan {
  GemmBatch g;
  struct Fix { size_t term; int a, off, pidx; };
  std::vector<Fix> fix;
  std::vector<std::vector<int>> nbs;
  std::vector<std::vector<std::pair<int, int>>> wcol;   // (q, column offset in W_i)
  std::vector<int> tot;
  std::vector<std::pair<int, int>> new_pending;
  std::vector<double*> W;   // W_i = G[:, 0:m] R_i (eliminate_invert -> eliminate_update)
  // reading R30 (symmetric Schur): for p < q the update
  // T_pq = sum_i C_p^(i) W_q^(i)[0:m] is formed once into a temporary (task `task`, C patched in
  // eliminate_update) and applied as (p,q) -= T_pq and (q,p) -= T_pq^T
  struct Mirror { size_t task; Blk pq, qp; int M, N; };
  std::vector<Mirror> mir;
  // R31 low-rank Schur terms of the null-space boxes: G11 = N Y1 (Y1 = D^{-1} N^T), so
  // C_p G11 R_q = (C_p N)(Y1 R_q) with inner dimension m - k instead of m
  std::vector<int> pdim;                    // m - k of a null-space box, 0 otherwise
  std::vector<double*> Nb, Y1b, Rh;         // N (m x p), Y1 (p x m), Rh = Y1 [R_q ...] (p x tot)
  std::vector<std::vector<double*>> Ch;     // C_p N (live_p x p) per neighbour p (order of nbs[a])
  // §8(e): per task of g, the owner of its target row box and the target block
  std::vector<int> towner;
  std::vector<Blk> tblk;
};
static int wcol_of(const std::vector<std::pair<int, int>>& w, int q) {
  for (auto& e : w)
    if (e.first == q) return e.second;
  return -1;
}
static void plan_schur(Ctx& c, FLevel& f, const std::vector<int>& cs, SchurPlan& P) {
  g_expose.set("plan");
  const int l = f.l;
  g_prof.hstart();
  P.nbs.assign(cs.size(), {});
  P.wcol.assign(cs.size(), {});
  P.tot.assign(cs.size(), 0);
  for (size_t a = 0; a < cs.size(); ++a) {
    const int i = cs[a];
    int nn_;
    const int* nl = c.nlist(l, i, &nn_);
    int tot = 0;
    for (int t = 0; t < nn_; ++t)
      if (nl[t] != i) { P.nbs[a].push_back(nl[t]); P.wcol[a].push_back({nl[t], tot}); tot += live(f, nl[t]); }
    P.tot[a] = tot;
  }
  // targets (p, q) in ascending (p, q) order, each with its eliminated boxes a in ascending
  // order (fixed summation order): p runs over the boxes next to the colour, a over the colour's
  // boxes in N(p), q over N(cs[a]) \ cs[a]
  std::vector<int> pos(f.nb, -1);
  std::vector<char> isp(f.nb, 0);
  for (size_t a = 0; a < cs.size(); ++a) pos[cs[a]] = (int)a;
  for (size_t a = 0; a < cs.size(); ++a)
    for (int p : P.nbs[a]) isp[p] = 1;
  g_prof.hlap("tg.sort");
  std::vector<std::pair<int, int>> qa;   // (q, a) of one target row p
  std::vector<int> grp_a;
  // R30 is opt-in (AIFMM_SYM_SCHUR=1): half the Schur flops, but measured slower end to end on
  // configs 2 and 3 (the factorisation then takes larger ranks)
  static const bool no_sym_env = getenv("AIFMM_SYM_SCHUR") == nullptr;
  const bool no_sym = no_sym_env || c.comm.on();   // R30 is not used while distributed
  for (int p = 0; p < f.nb; ++p) {
    if (!isp[p]) continue;
    qa.clear();
    int npn;
    const int* pn = c.nlist(l, p, &npn);
    for (int t = 0; t < npn; ++t) {
      const int a = pos[pn[t]];
      if (a < 0) continue;
      for (int q : P.nbs[a]) qa.push_back({q, a});
    }
    std::sort(qa.begin(), qa.end());
    for (size_t t0 = 0; t0 < qa.size();) {
      size_t t1 = t0;
      grp_a.clear();
      while (t1 < qa.size() && qa[t1].first == qa[t0].first) {
        const int a = qa[t1++].second;
        // R28: a box whose basis spans R^m (k = m) when its colour begins (this plan precedes
        // the colour's compression) has G11 = 0 -- no Schur term, no fill-in
        static const bool no_r28 = getenv("AIFMM_NO_R28") != nullptr;   // debug toggle
        // (a box with m = 0 contributes nothing but, as in the oracle, still makes its far
        // neighbour pairs pending; its zero-size terms are dropped below)
        if (!f.m[cs[a]] || no_r28 || f.k[cs[a]] < f.m[cs[a]]) grp_a.push_back(a);
      }
      const int q = qa[t0].first;
      t0 = t1;
      if (grp_a.empty()) continue;
      const int M = live(f, p), N = live(f, q);
      // a far pair touched by the colour becomes pending even when one of its live sizes is 0
      // (as in the oracle: its compression then adds nothing, but it is counted)
      if (!f.nearb.get(f.key(p, q)) && !(f.E[p] && f.E[q]) && p < q)
        P.new_pending.push_back({p, q});
      if (!M || !N) continue;
      // R30: the (p, q) and (q, p) updates are transposes (symmetric kernel, V = U, R27); the
      // pair is planned once, at p < q (the contributing boxes are the same for both)
      if (p > q && !no_sym) continue;
      bool fresh = false;   // a fill-in slot allocated by this update (written with beta = 0)
      auto target = [&](int x, int y) {
        Blk T;
        if (const Blk* it = f.nearb.get(f.key(x, y))) T = *it;
        else if (f.E[x] && f.E[y]) T = f.A.at(f.key(x, y));
        else {
          AIFMM_REQUIRE(c.cheb(l, x, y) == 2, AIFMM_ESINGULAR_PIVOT, "fill-in outside N and IL");
          const long long sl = f.F.slot(f.key(x, y));
          AIFMM_REQUIRE(sl >= 0 && f.F.has[sl], AIFMM_ESINGULAR_PIVOT, "missing fill-in slot");
          Blk& Fb = f.F.v[sl];
          if (!Fb.p) {
            const size_t need = std::max<size_t>((size_t)Fb.ld * f.m[y], 1);
            auto it = f.ffree.lower_bound(need);
            if (it != f.ffree.end() && it->first <= need + need / 4 + 1024) {
              Fb.p = it->second;
              f.fcap[sl] = it->first;
              f.ffree.erase(it);
            } else {
              Fb.p = c.scr(l).d(need);
              f.fcap[sl] = need;
            }
            fresh = true;
            // R30 adds its mirrored temporaries onto the slots: those need zeros (stream order: the
            // slot's previous readers were enqueued before this memset)
            if (!no_sym) AIFMM_CUDA(cudaMemsetAsync(Fb.p, 0, sizeof(double) * need, c.s));
          }
          T = Fb;
        }
        return T;
      };
      Blk T = target(p, q);
      if (p < q && !no_sym) {
        P.mir.push_back({P.g.size(), T, target(q, p), M, N});
        P.g.task(nullptr, M, M, N, 0.0);   // temporary T_pq, allocated in eliminate_update
      } else {
        P.g.task(T.p, T.ld, M, N, fresh ? 0.0 : 1.0);
        P.towner.push_back(c.own(l, p));
        P.tblk.push_back(Blk{T.p, T.ld, M, N});
      }
      for (int a : grp_a) {
        const int i = cs[a];
        if (!f.m[i]) continue;
        const Blk& C = f.nearb.at(f.key(p, i));
        int pidx = 0;
        while (P.nbs[a][pidx] != p) ++pidx;
        P.fix.push_back({P.g.nterms(), a, wcol_of(P.wcol[a], q), pidx});
        P.g.term(-1.0, C.p, C.ld, 0, nullptr, 0, 0, f.m[i]);   // B patched in eliminate_colour
      }
    }
  }
  g_prof.hlap("tg.tasks");
}

// Reading R31 (null-space formation of the pivot inverse).  For P = [[K, U], [U^T, 0]] with
// orthonormal U (m x k, R13; V = U, R27) and N any well-conditioned basis of the orthogonal
// complement of range(U) (m x (m-k)), block elimination in the basis [U, N] gives, with
// D = N^T K N:
//   G11 = N D^{-1} N^T,   G12 = U - G11 K U,   G21 = U^T - U^T K G11,
//   G22 = -U^T K U + U^T K G11 K U
// (exact; independent of the choice of N).  The only inverses are D and the triangular factor
// below, of size m - k instead of m + k; everything else is a DMMA GEMM.  N = Y R^{-1} with
// Y = (I - U U^T) Omega (Omega a fixed counter-based pseudo-random m x (m-k) matrix) and Y = Q R
// (Householder), re-projected against U once.  G is written into the record r.G exactly
// where the explicit inverse went, so the multipliers, new blocks and the solve are unchanged.
static void nullspace_pivots(Ctx& c, FLevel& f, const std::vector<int>& cs, const std::vector<int>& ns, FlopCounter& fp,
                             SchurPlan& P) {
  const size_t nb = ns.size();
  struct NS { double *Y, *t1, *R1, *N, *t4, *KN, *KU, *D, *Y1, *t, *t3; int m, k, p, n; const double* U; Blk K; double* G; };
  std::vector<NS> v(nb);
  std::vector<HashFillTask> hf;
  for (size_t x = 0; x < nb; ++x) {
    const int i = cs[ns[x]];
    NS& e = v[x];
    e.m = f.m[i];
    e.k = f.k[i];
    e.p = e.m - e.k;
    e.n = e.m + e.k;
    e.U = f.U[i];
    e.K = f.nearb.at(f.key(i, i));
    e.G = f.rec[i].G;
    const size_t mp = (size_t)e.m * e.p, pp = (size_t)e.p * e.p;
    e.Y = c.work.d(mp);
    e.t1 = c.work.d((size_t)e.k * e.p);
    e.R1 = c.work.d(pp);
    e.N = c.work.d(mp);
    e.t4 = c.work.d((size_t)e.k * e.p);
    e.KN = c.work.d(mp);
    e.KU = c.work.d((size_t)e.m * e.k);
    e.D = c.work.d(pp);
    e.Y1 = c.work.d(mp);
    e.t = c.work.d((size_t)e.p * e.k);
    e.t3 = c.work.d((size_t)e.k * e.p);
    hf.push_back(HashFillTask{e.Y, e.m, e.m, e.p, 0x5EEDull * 0x100000001ull + (unsigned long long)e.m * 7919ull + e.p});
  }
  {
    const HashFillTask* dh = c.up.put(hf);
    LAUNCH(hash_fill_kernel, (int)nb, 256, 0, c.s, dh);
  }
  GemmBatch g;
  // Y = Omega - U (U^T Omega)
  for (auto& e : v) { g.task(e.t1, e.k, e.k, e.p, 0.0); g.term(1.0, e.U, e.m, 1, e.Y, e.m, 0, e.m); }
  g.run(c.up, c.s, &fp);
  for (auto& e : v) { g.task(e.Y, e.m, e.m, e.p, 1.0); g.term(-1.0, e.U, e.m, 0, e.t1, e.k, 0, e.k); }
  g.run(c.up, c.s, &fp);
  // N = Y R^{-1} with Y = Q R (Householder on a copy of Y: the batched panels of the RRQR's first
  // stage, R8b machinery; then the triangular factor inverted by the batched Gauss-Jordan),
  // then N -= U (U^T N).  (A CholeskyQR pass measured 22% of the config-3 run: its one-CTA
  // Cholesky of the (m-k)^2 Gram matrices is latency-bound.)
  {
    CopyBatch yc;
    std::vector<TriRootReq> tr;
    for (auto& e : v) {
      yc.copy(e.Y, e.m, e.N, e.m, e.m, e.p);   // N's storage holds the destroyed copy
      tr.push_back(TriRootReq{e.N, e.m, e.m, e.p, e.R1, e.p});   // R1 <- R^T (p x p, lower)
    }
    yc.run(c.up, c.s);
    batched_tri_root(tr, c.work, c.up, c.s, &fp, 0);
    std::vector<InvReq> inv;
    for (size_t x = 0; x < nb; ++x) inv.push_back(InvReq{v[x].R1, v[x].p, v[x].p, f.dinfo + f.nb + cs[ns[x]]});
    batched_inverse(inv, c.work, c.up, c.s, &fp);   // R1 <- R^{-T}
  }
  for (auto& e : v) { g.task(e.N, e.m, e.m, e.p, 0.0); g.term(1.0, e.Y, e.m, 0, e.R1, e.p, 1, e.p); }
  g.run(c.up, c.s, &fp);
  for (auto& e : v) { g.task(e.t4, e.k, e.k, e.p, 0.0); g.term(1.0, e.U, e.m, 1, e.N, e.m, 0, e.m); }
  g.run(c.up, c.s, &fp);
  for (auto& e : v) { g.task(e.N, e.m, e.m, e.p, 1.0); g.term(-1.0, e.U, e.m, 0, e.t4, e.k, 0, e.k); }
  g.run(c.up, c.s, &fp);
  // K N, K U
  for (auto& e : v) {
    g.task(e.KN, e.m, e.m, e.p, 0.0);
    g.term(1.0, e.K.p, e.K.ld, 0, e.N, e.m, 0, e.m);
    g.task(e.KU, e.m, e.m, e.k, 0.0);
    g.term(1.0, e.K.p, e.K.ld, 0, e.U, e.m, 0, e.m);
  }
  g.run(c.up, c.s, &fp);
  // D = N^T K N; t3 = U^T K N; G22 <- -U^T K U (completed below)
  for (auto& e : v) {
    g.task(e.D, e.p, e.p, e.p, 0.0);
    g.term(1.0, e.N, e.m, 1, e.KN, e.m, 0, e.m);
    g.task(e.t3, e.k, e.k, e.p, 0.0);
    g.term(1.0, e.U, e.m, 1, e.KN, e.m, 0, e.m);
  }
  g.run(c.up, c.s, &fp);
  {
    std::vector<InvReq> inv;
    for (size_t x = 0; x < nb; ++x) inv.push_back(InvReq{v[x].D, v[x].p, v[x].p, f.dinfo + cs[ns[x]]});
    batched_inverse(inv, c.work, c.up, c.s, &fp);
  }
  // Y1 = D^{-1} N^T
  for (auto& e : v) { g.task(e.Y1, e.p, e.p, e.m, 0.0); g.term(1.0, e.D, e.p, 0, e.N, e.m, 1, e.p); }
  g.run(c.up, c.s, &fp);
  // G11 = N Y1 (into G[0:m, 0:m]); t = Y1 K U
  for (auto& e : v) {
    g.task(e.G, e.n, e.m, e.m, 0.0);
    g.term(1.0, e.N, e.m, 0, e.Y1, e.p, 0, e.p);
    g.task(e.t, e.p, e.p, e.k, 0.0);
    g.term(1.0, e.Y1, e.p, 0, e.KU, e.m, 0, e.m);
  }
  g.run(c.up, c.s, &fp);
  // G12 = U - N t;  G21 = U^T - t3 Y1;  G22 = -U^T K U + t3 t
  for (auto& e : v) {
    g.task(e.G + (size_t)e.m * e.n, e.n, e.m, e.k, 0.0);
    g.add(1.0, e.U, e.m, 0);
    g.term(-1.0, e.N, e.m, 0, e.t, e.p, 0, e.p);
    g.task(e.G + e.m, e.n, e.k, e.m, 0.0);
    g.add(1.0, e.U, e.m, 1);
    g.term(-1.0, e.t3, e.k, 0, e.Y1, e.p, 0, e.p);
    g.task(e.G + (size_t)e.m * e.n + e.m, e.n, e.k, e.k, 0.0);
    g.term(-1.0, e.U, e.m, 1, e.KU, e.m, 0, e.m);
    g.term(1.0, e.t3, e.k, 0, e.t, e.p, 0, e.p);
  }
  g.run(c.up, c.s, &fp);
  for (auto& e : v) c.fcp[PH_PIVOT].bytes += 8.0 * ((double)e.m * e.m + (double)e.m * e.k + (double)e.n * e.n);
  for (size_t x = 0; x < nb; ++x) {
    P.pdim[ns[x]] = v[x].p;
    P.Nb[ns[x]] = v[x].N;
    P.Y1b[ns[x]] = v[x].Y1;
  }
}

// Steps 1-2 of a colour's elimination: pivot inverses and W_i = G[:, 0:m] R_i.  They need only
// the colour's final bases and near blocks (no far M2L block), so they are launched before the
// redirection of the colour's compression is planned.
static void eliminate_invert(Ctx& c, FLevel& f, const std::vector<int>& cs, SchurPlan& P) {
  g_expose.set("elim.inv");
  const int l = f.l;
  if (g_prof.on) g_prof.begin(c.s);
  // 1. G_i = P_i^{-1}, P_i = [[K_ii, U_i],[V_i^T, 0]] (R16).  Boxes with 0 < k < m: null-space
  //    formation (R31, below); the others (k = 0: P = K; k = m, R28): assembled and inverted.
  CopyBatch cb;
  std::vector<InvReq> inv;
  std::vector<int> ns;   // colour positions a of the null-space boxes
  // R31 by default (mode 2) for the boxes whose complement is small, m - k <= 64
  // (AIFMM_NULLSPACE_PMAX): there the inverse shrinks most (size m - k instead of m + k) and the
  // Schur terms get inner dimension m - k; measured -1.8% factor time on configs 2 and 3 (all
  // boxes: -2% / +15%).  AIFMM_NULLSPACE=0 off, 1 every box with 0 < k < m,
  // -1 boxes with m >= AIFMM_NULLSPACE_MMIN.
  static const int ns_env = getenv("AIFMM_NULLSPACE") ? atoi(getenv("AIFMM_NULLSPACE")) : 2;
  static const int ns_mmin = getenv("AIFMM_NULLSPACE_MMIN") ? atoi(getenv("AIFMM_NULLSPACE_MMIN")) : 400;
  static const int ns_pmax = getenv("AIFMM_NULLSPACE_PMAX") ? atoi(getenv("AIFMM_NULLSPACE_PMAX")) : 64;
  const int ns_min = ns_env == 0 || ns_env == 2 ? (1 << 30) : (ns_env == 1 ? 0 : ns_mmin);
  for (size_t a = 0; a < cs.size(); ++a) {
    int i = cs[a];
    const int m = f.m[i], k = f.k[i], n = m + k;
    Rec& r = f.rec[i];
    r.m = m;
    r.k = k;
    r.G = c.persist.d(std::max<size_t>((size_t)n * n, 1));
    if (!n) continue;
    const bool nsbox = k > 0 && k < m && (m >= ns_min || (ns_env == 2 && m - k <= ns_pmax));
    // §8(e): G_i arrives from owner(i); the R31 boxes are formed by every rank (their Schur
    // operands C_p N and Y1 R_q are temporaries; by default their inverses are of size <= 64)
    if (!nsbox && !c.mine(l, i, 2)) continue;
    if (nsbox) {
      ns.push_back((int)a);
      continue;
    }
    const Blk& K = f.nearb.at(f.key(i, i));
    cb.copy(K.p, K.ld, r.G, n, m, m);
    cb.copy(f.U[i], m, r.G + (size_t)m * n, n, m, k);
    cb.copy(f.V[i], m, r.G + m, n, k, m, 1.0, 1);
    cb.fill(r.G + (size_t)m * n + m, n, k, k, 0.0);
    inv.push_back(InvReq{r.G, n, n, f.dinfo + i});
  }
  cb.run(c.up, c.s);
  {
    PhaseTimer pt(c, PH_PIVOT);
    FlopCounter fp;
    batched_inverse(inv, c.work, c.up, c.s, &fp);
    for (const InvReq& r : inv) c.fcp[PH_PIVOT].bytes += 16.0 * r.n * r.n;   // read + write each pivot once
    P.pdim.assign(cs.size(), 0);
    P.Nb.assign(cs.size(), nullptr);
    P.Y1b.assign(cs.size(), nullptr);
    if (!ns.empty()) nullspace_pivots(c, f, cs, ns, fp, P);
    c.fc_all.flops += fp.flops;
    c.fcp[PH_PIVOT].flops += fp.flops;
  }
  static const bool dbg_g11 = getenv("AIFMM_DEBUG_G11") != nullptr;   // debug: |G11| of full boxes (R28)
  if (dbg_g11) {
    for (int i : cs) {
      const int m = f.m[i], k = f.k[i], n = m + k;
      if (!m || k < m) continue;
      std::vector<double> h = d2h(c, f.rec[i].G, (size_t)n * n);
      double a = 0.0, g = 0.0;
      for (int cc = 0; cc < m; ++cc)
        for (int r = 0; r < m; ++r) a = std::max(a, std::fabs(h[(size_t)cc * n + r]));
      for (double v : h) g = std::max(g, std::fabs(v));
      fprintf(stderr, "[aifmm g11] level %d box %d m %d k %d max|G11| %.3e max|G| %.3e\n", l, i, m, k, a, g);
    }
  }
  static const bool dbg_piv = getenv("AIFMM_DEBUG_PIVOTS") != nullptr;   // debug: largest |P_i^-1| entries
  if (dbg_piv) {
    std::vector<std::pair<double, int>> mx;
    for (int i : cs) {
      const int n = f.m[i] + f.k[i];
      if (!n) continue;
      std::vector<double> h = d2h(c, f.rec[i].G, (size_t)n * n);
      double a = 0.0;
      for (double v : h) a = std::max(a, std::fabs(v));
      mx.push_back({a, i});
    }
    std::sort(mx.rbegin(), mx.rend());
    for (size_t t = 0; t < std::min<size_t>(3, mx.size()); ++t)
      fprintf(stderr, "[aifmm pivots] level %d colour-first-box %d box %d m %d k %d max|G| %.3e\n", l, cs[0], mx[t].second,
              f.m[mx[t].second], f.k[mx[t].second], mx[t].first);
  }
  if (g_prof.on) { g_prof.end("elim.inverse"); g_prof.begin(c.s); }
  // 2. W_i = G[:, 0:m] * R_i (row X_i blocks), columns ordered as N(i) \ i.  Null-space boxes
  //    (R31): only W_z = G[m:, 0:m] R_i (the new (Z_i, x_q) blocks); their Schur terms use
  //    Rh = Y1 R_i and Ch_p = C_p N instead of W[0:m]
  std::vector<double*> W(cs.size());
  P.Rh.assign(cs.size(), nullptr);
  P.Ch.assign(cs.size(), {});
  GemmBatch g;
  for (size_t a = 0; a < cs.size(); ++a) {
    int i = cs[a];
    const int m = f.m[i], k = f.k[i], n = m + k, pd = P.pdim[a];
    W[a] = c.work.d(std::max<size_t>((size_t)n * P.tot[a], 1));
    if (!n || (!pd && !c.mine(l, i, 2))) continue;
    if (pd) P.Rh[a] = c.work.d(std::max<size_t>((size_t)pd * P.tot[a], 1));
    for (auto& wq : P.wcol[a]) {
      const int q = wq.first;
      const Blk& R = f.nearb.at(f.key(i, q));
      if (!live(f, q)) continue;
      if (!pd) {
        g.task(W[a] + (size_t)wq.second * n, n, n, live(f, q), 0.0);
        g.term(1.0, f.rec[i].G, n, 0, R.p, R.ld, 0, m);
      } else {
        g.task(W[a] + (size_t)wq.second * n + m, n, k, live(f, q), 0.0);
        g.term(1.0, f.rec[i].G + m, n, 0, R.p, R.ld, 0, m);
        g.task(P.Rh[a] + (size_t)wq.second * pd, pd, pd, live(f, q), 0.0);
        g.term(1.0, P.Y1b[a], pd, 0, R.p, R.ld, 0, m);
      }
    }
    if (pd) {
      for (int p : P.nbs[a]) {
        const Blk& C = f.nearb.at(f.key(p, i));
        double* ch = c.work.d(std::max<size_t>((size_t)live(f, p) * pd, 1));
        P.Ch[a].push_back(ch);
        if (!live(f, p)) continue;
        g.task(ch, live(f, p), live(f, p), pd, 0.0);
        g.term(1.0, C.p, C.ld, 0, P.Nb[a], m, 0, m);
      }
    }
  }
  {
    PhaseTimer pt(c, PH_MULT);
    FlopCounter fp;
    g.run(c.up, c.s, &fp);
    c.fc_all.flops += fp.flops;
    c.fcp[PH_MULT].flops += fp.flops;
    c.fcp[PH_MULT].bytes += fp.bytes;
  }
  if (c.dist_ph(l, 2)) {   // §8(e): G_i and W_i from their owners
    std::vector<std::vector<Region>> reg(c.comm.world);
    for (size_t a = 0; a < cs.size(); ++a) {
      const int i = cs[a], n = f.m[i] + f.k[i];
      if (!n || P.pdim[a]) continue;   // R31 boxes: formed by every rank
      auto& R = reg[c.own(l, i)];
      R.push_back(Region{f.rec[i].G, n, n, n});
      if (P.tot[a]) R.push_back(Region{W[a], n, n, P.tot[a]});
    }
    c.comm.exchange(reg, c.up, c.s);
  }
  P.W = std::move(W);
  if (g_prof.on) g_prof.end("elim.W");
}

// debug (AIFMM_DEBUG_SYM=1): largest |B_pq - B_qp^T| / max|B_pq| over the near, M2L and pending
// fill-in blocks of the level (the symmetric system keeps every pair transposed, R27 / R30)
// debug (AIFMM_DEBUG_DIST=1, distributed runs): FNV digest of the level state (bases, near /
// M2L / fill-in blocks, records) printed per rank, to find a block an exchange missed
static void dbg_digest(Ctx& c, FLevel& f, const char* where) {
  unsigned long long h[5] = {1469598103934665603ull, 1469598103934665603ull, 1469598103934665603ull,
                             1469598103934665603ull, 1469598103934665603ull};
  auto eat = [&](int w, const double* p, int ld, int rows, int cols) {
    if (!p || rows <= 0 || cols <= 0) return;
    std::vector<double> hb((size_t)ld * (cols - 1) + rows);
    AIFMM_CUDA(cudaMemcpyAsync(hb.data(), p, sizeof(double) * hb.size(), cudaMemcpyDeviceToHost, c.s));
    c.up.sync();
    for (int j = 0; j < cols; ++j)
      for (int i = 0; i < rows; ++i) {
        unsigned long long x;
        std::memcpy(&x, &hb[(size_t)j * ld + i], 8);
        h[w] = (h[w] ^ x) * 1099511628211ull;
      }
  };
  for (int b : f.boxes) eat(0, f.U[b], f.m[b], f.m[b], f.k[b]);
  static const bool per_box = getenv("AIFMM_DEBUG_DIST") && atoi(getenv("AIFMM_DEBUG_DIST")) == 2;
  if (per_box && strstr(where, "compressed"))
    for (int b : f.boxes) {
      const int m = f.m[b], k = f.k[b];
      std::vector<double> hb((size_t)m * std::max(k, 1));
      if (k) AIFMM_CUDA(cudaMemcpyAsync(hb.data(), f.U[b], sizeof(double) * (size_t)m * k, cudaMemcpyDeviceToHost, c.s));
      c.up.sync();
      double n2 = 0, colsum = 0;
      for (int j = 0; j < k; ++j) {
        double cn = 0;
        for (int i = 0; i < m; ++i) cn += hb[(size_t)j * m + i] * hb[(size_t)j * m + i];
        n2 += cn;
        colsum += std::fabs(cn - 1.0);
      }
      fprintf(stderr, "[dist %d] box L%d %s b=%d m=%d k=%d own=%d |U|^2=%.12e dev_from_unit=%.3e\n", c.comm.rank, f.l, where, b, m, k,
              c.own(f.l, b), n2, colsum);
    }
  BlkTable* T[3] = {&f.nearb, &f.A, &f.F};
  for (int w = 0; w < 3; ++w)
    for (size_t s = 0; s < T[w]->v.size(); ++s)
      if (T[w]->has[s]) eat(1 + w, T[w]->v[s].p, T[w]->v[s].ld, T[w]->v[s].rows, T[w]->v[s].cols);
  for (int b : f.boxes)
    if (f.E[b] && f.rec[b].G) eat(4, f.rec[b].G, f.m[b] + f.k[b], f.rec[b].m + f.rec[b].k, f.rec[b].m + f.rec[b].k);
  fprintf(stderr, "[dist %d] level %d %s: U %016llx near %016llx M2L %016llx fill %016llx G %016llx\n", c.comm.rank, f.l,
          where, h[0], h[1], h[2], h[3], h[4]);
}

static void dbg_symmetry(Ctx& c, FLevel& f, const char* where) {
  double worst[3] = {0, 0, 0};
  int wp[3] = {-1, -1, -1}, wq[3] = {-1, -1, -1};
  for (int p : f.boxes)
    for (int kind = 0; kind < 3; ++kind) {
      int ni;
      const int* li = kind == 0 ? c.nlist(f.l, p, &ni) : c.ilist(f.l, p, &ni);
      for (int t = 0; t < ni; ++t) {
        const int q = li[t];
        if (q <= p) continue;
        BlkTable& T = kind == 0 ? f.nearb : (kind == 1 ? f.A : f.F);
        const Blk* a = T.get(f.key(p, q));
        const Blk* b = T.get(f.key(q, p));
        if (!a || !b || !a->p || !b->p) continue;
        if (kind == 2 && !f.pending.count({p, q})) continue;
        const int M = kind == 1 ? f.k[p] : live(f, p), N = kind == 1 ? f.k[q] : live(f, q);
        if (!M || !N) continue;
        std::vector<double> ha((size_t)a->ld * N), hb((size_t)b->ld * M);
        AIFMM_CUDA(cudaMemcpyAsync(ha.data(), a->p, sizeof(double) * ha.size(), cudaMemcpyDeviceToHost, c.s));
        AIFMM_CUDA(cudaMemcpyAsync(hb.data(), b->p, sizeof(double) * hb.size(), cudaMemcpyDeviceToHost, c.s));
        c.up.sync();
        double mx = 0, df = 0;
        for (int j = 0; j < N; ++j)
          for (int i = 0; i < M; ++i) {
            const double x = ha[(size_t)j * a->ld + i], y = hb[(size_t)i * b->ld + j];
            mx = std::max(mx, std::fabs(x));
            df = std::max(df, std::fabs(x - y));
          }
        const double r = mx > 0 ? df / mx : df;
        if (r > worst[kind]) { worst[kind] = r; wp[kind] = p; wq[kind] = q; }
      }
    }
  fprintf(stderr, "[aifmm sym] level %d %s: near %.2e (%d,%d)  M2L %.2e (%d,%d)  fill %.2e (%d,%d)\n", f.l, where, worst[0], wp[0],
          wq[0], worst[1], wp[1], wq[1], worst[2], wp[2], wq[2]);
}

static void eliminate_update(Ctx& c, FLevel& f, const std::vector<int>& cs, SchurPlan& P) {
  g_expose.set("elim.upd");
  const int l = f.l;
  const std::vector<double*>& W = P.W;
  CopyBatch cb;
  if (g_prof.on) g_prof.begin(c.s);
  // 3. Schur updates (planned) are launched first; the new blocks (p,i) = C G12,
  //    (i,q) = G21 R = W_z, (i,i) = -G22 (R17) are planned while they run (they touch no
  //    Schur target: (p,i) with i in the colour is never a target of the colour, whose boxes
  //    are not neighbours)
  for (const auto& fx : P.fix) {
    const int i = cs[fx.a];
    const int n = f.m[i] + f.k[i];
    GemmTerm& t = P.g.term_ref(fx.term);
    const int pd = P.pdim.empty() ? 0 : P.pdim[fx.a];
    if (pd) {   // R31: (C_p N)(Y1 R_q)
      const int p = P.nbs[fx.a][fx.pidx];
      t.A = P.Ch[fx.a][fx.pidx];
      t.lda = std::max(live(f, p), 1);
      t.B = P.Rh[fx.a] + (size_t)fx.off * pd;
      t.ldb = pd;
      t.K = pd;
    } else {
      t.B = W[fx.a] + (size_t)fx.off * n;
      t.ldb = n;
    }
  }
  for (auto& pr : P.new_pending) f.pending.insert(pr);
  // R30 temporaries (the work pool is not reset between here and the end of the colour)
  std::vector<double*> mtmp(P.mir.size());
  GemmBatch gm;
  for (size_t t = 0; t < P.mir.size(); ++t) {
    const SchurPlan::Mirror& mr = P.mir[t];
    mtmp[t] = c.work.d((size_t)mr.M * mr.N);
    GemmTask& tk = P.g.task_ref(mr.task);
    tk.C = mtmp[t];
    tk.ldc = mr.M;
    // the temporary already holds -T_pq (the planned terms carry alpha = -1)
    gm.task(mr.pq.p, mr.pq.ld, mr.M, mr.N, 1.0);
    gm.add(1.0, mtmp[t], mr.M, 0);
    gm.task(mr.qp.p, mr.qp.ld, mr.N, mr.M, 1.0);
    gm.add(1.0, mtmp[t], mr.M, 1);
  }
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (c.timing) {
    AIFMM_CUDA(cudaEventCreate(&e0));
    AIFMM_CUDA(cudaEventCreate(&e1));
    AIFMM_CUDA(cudaEventRecord(e0, c.s));
  }
  long long l0 = g_launches;
  nvtxRangePushA("schur");   // lets `ncu --nvtx --nvtx-include schur/` capture exactly these launches
  if (c.dist_ph(l, 4)) {   // §8(e): the targets of my row boxes, then everyone's targets
    std::vector<char> keep(P.g.size(), 0);
    std::vector<std::vector<Region>> reg(c.comm.world);
    for (size_t t = 0; t < P.g.size(); ++t) {
      keep[t] = P.towner[t] == c.comm.rank;
      const Blk& T = P.tblk[t];
      reg[P.towner[t]].push_back(Region{T.p, T.ld, T.rows, T.cols});
    }
    GemmBatch mine_ = P.g.filtered(keep);
    mine_.run(c.up, c.s, &c.fc_schur);
    c.comm.exchange(reg, c.up, c.s);
  } else {
    P.g.run(c.up, c.s, &c.fc_schur);
  }
  gm.run(c.up, c.s, &c.fc_schur);
  nvtxRangePop();
  c.stats[AIFMM_STAT_SCHUR_LAUNCHES] += (double)(g_launches - l0);
  if (c.timing) {
    AIFMM_CUDA(cudaEventRecord(e1, c.s));
    c.ev.push_back({e0, e1});
  }
  if (g_prof.on) { g_prof.end("elim.schur"); g_prof.begin(c.s); }
  g_prof.hstart();
  GemmBatch gf;
  std::vector<std::pair<long long, Blk>> fresh;
  {
    size_t nf = 0;
    for (size_t a = 0; a < cs.size(); ++a) nf += P.nbs[a].size() + P.wcol[a].size() + 1;
    fresh.reserve(nf);
  }
  for (size_t a = 0; a < cs.size(); ++a) {
    int i = cs[a];
    const int m = f.m[i], k = f.k[i], n = m + k;
    Rec& r = f.rec[i];
    r.C.reserve(P.nbs[a].size());
    r.Ckind_z.reserve(P.nbs[a].size());
    r.R.reserve(P.wcol[a].size());
    r.Rkind_y.reserve(P.wcol[a].size());
    for (int p : P.nbs[a]) {
      const Blk& C = f.nearb.at(f.key(p, i));
      r.C.push_back({p, C});
      r.Ckind_z.push_back(f.E[p]);
      // (X_p, y_i) is replayed by the solve when p is eliminated; (Z_p, y_i) is final
      DevPool& bp = f.E[p] ? c.scr(l) : c.persist;
      Blk nb_{bp.d(std::max<size_t>((size_t)live(f, p) * k, 1)), std::max(live(f, p), 1), live(f, p), k};
      if (live(f, p) && k) {
        gf.task(nb_.p, nb_.ld, live(f, p), k, 0.0);
        if (m) gf.term(1.0, C.p, C.ld, 0, r.G + (size_t)m * n, n, 0, m);
      }
      fresh.push_back({f.key(p, i), nb_});
    }
    for (auto& wq : P.wcol[a]) {
      const int q = wq.first;
      const Blk& R = f.nearb.at(f.key(i, q));
      r.R.push_back({q, R});
      r.Rkind_y.push_back(f.E[q]);
      // (Z_i, x_q | y_q): final if q is eliminated, else a C record of q (R32: scratch)
      DevPool& bp = (f.E[q] || half_records()) ? c.scr(l) : c.persist;
      Blk nb_{bp.d(std::max<size_t>((size_t)k * live(f, q), 1)), std::max(k, 1), k, live(f, q)};
      cb.copy(W[a] + (size_t)wq.second * n + m, n, nb_.p, nb_.ld, k, live(f, q));
      fresh.push_back({f.key(i, q), nb_});
    }
    Blk nb_{c.scr(l).d(std::max<size_t>((size_t)k * k, 1)), std::max(k, 1), k, k};
    cb.copy(r.G + (size_t)m * n + m, n, nb_.p, nb_.ld, k, k, -1.0);
    fresh.push_back({f.key(i, i), nb_});
  }
  g_prof.hlap("fresh");
  {
    PhaseTimer pt(c, PH_FRESH);
    FlopCounter fp;
    gf.run(c.up, c.s, &fp);
    cb.run(c.up, c.s);
    c.fc_all.flops += fp.flops;
    c.fcp[PH_FRESH].flops += fp.flops;
    c.fcp[PH_FRESH].bytes += fp.bytes;
  }
  if (g_prof.on) { g_prof.end("elim.fresh"); g_prof.begin(c.s); }
  for (auto& fr : fresh) f.nearb[fr.first] = fr.second;
  for (int i : cs) f.E[i] = 1;
  c.work.reset();   // stream order: the next colour's temporaries are written after these reads
  if (g_prof.on) g_prof.end("elim.tail");
}

// The kernels record coincident points (near-field kernel blocks) and singular box pivots in
// sticky device flags; they are read once, at the end of the factorisation or when another error
// interrupts it (so that the root cause is the one reported), instead of synchronising the
// stream at every level.
static void deferred_checks(Ctx& c) {
  check_flag(c, AIFMM_ECOINCIDENT, "coincident points with a singular kernel");
  for (int l = c.L; l >= 2 && l < (int)c.fl.size(); --l) {
    const FLevel& fl = c.fl[l];
    if (!fl.dinfo) continue;
    std::vector<int> info = d2h(c, fl.dinfo, 2 * (size_t)fl.nb);
    if (c.dist_level(l)) c.comm.allreduce_int(info.data(), (int)info.size(), c.s);   // owners' flags
    for (int b : fl.boxes)
      if (info[b] || info[fl.nb + b])
        throw Error(AIFMM_ESINGULAR_PIVOT, std::string(info[b] ? "singular pivot" : "null-space basis (R31) not of full rank") +
                                               " at level " + std::to_string(l) + " box " + std::to_string(b));
  }
}

// §8(e): the points (in tree order) are cut into world contiguous ranges of equal size; a box
// belongs to the rank whose range holds its median point.  At the fine levels this is a split
// into contiguous Morton ranges of subtrees; at the coarse levels, where a subtree split would
// leave ranks idle, every box still has one owner.  Any ownership that all ranks agree on gives
// the same factorisation (each phase exchanges every block it wrote); this one balances the
// work level by level.  Levels <= l_p (default 1: none) are computed redundantly.
static void plan_ownership(Ctx& c) {
  c.owner.assign(c.L + 1, {});
  c.lp = -1;
  if (!c.comm.on()) return;
  const int W = c.comm.world;
  c.lp = c.lp_user >= 1 ? std::min(c.lp_user, c.L - 1) : 1;
  for (int l = c.lp + 1; l <= c.L; ++l) {
    c.owner[l].assign((size_t)1 << (c.d * l), 0);
    for (size_t b = 0; b < c.owner[l].size(); ++b) {
      const long long mid = c.off[l][b] + (c.off[l][b + 1] - c.off[l][b]) / 2;
      c.owner[l][b] = (int)std::min<long long>(W - 1, mid * W / c.n);
    }
  }
}

// a quarter of the device memory, at most 48 GB (a function of the device only, so that repeated
// factorisations batch, and therefore round, identically)
static void set_ws_budget(Ctx& c) {
  size_t fr = 0, tot = 0;
  if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) tot = 0;
  c.ws_budget = std::max(6e9, std::min(48e9, 0.26 * (double)tot));
}

static void factor_levels(Ctx& c);
static void factor_all(Ctx& c) {
  g_expose.set("factor.start");
  set_ws_budget(c);
  plan_ownership(c);
  c.comm.bytes_in = 0.0;
  c.comm.exchanges = 0;
  c.fl.assign(c.L + 1, FLevel{});
  AIFMM_CUDA(cudaMemsetAsync(c.dflag, 0, sizeof(int), c.s));
  try {
    factor_levels(c);
  } catch (const Error&) {
    deferred_checks(c);
    throw;
  }
}

static void factor_levels(Ctx& c) {
  const int L = c.L;
  for (int l = L; l >= 2; --l) {
    g_prof.begin(c.s);
    setup_level(c, l);
    // the near-field kernel blocks are evaluated at the leaf level only (upper levels assemble
    // theirs from the children's blocks): one check there
    if (l == L) check_flag(c, AIFMM_ECOINCIDENT, "coincident points with a singular kernel");
    FLevel& f = c.fl[l];
    g_prof.end("setup");
    g_prof.begin(c.s);
    {
      PhaseTimer pt(c, PH_ORTH);
      orthonormalise(c, f);
    }
    g_prof.end("orth");
    if (getenv("AIFMM_DEBUG_SYM")) dbg_symmetry(c, f, "after setup");
    int ncol = 0;
    for (int b : f.boxes) ncol = std::max(ncol, c.col[l][b] + 1);
    for (int col = 0; col < ncol; ++col) {
      std::vector<int> cs;
      for (int b : f.boxes)
        if (c.col[l][b] == col) cs.push_back(b);
      std::vector<std::pair<int, int>> S;
      for (auto& pr : f.pending)
        if (c.col[l][pr.first] == col || c.col[l][pr.second] == col) S.push_back(pr);
      SchurPlan plan;
      plan_schur(c, f, cs, plan);   // host work, overlaps the previous colour's kernels
      g_prof.begin(c.s);
      static const bool dbg_dist = getenv("AIFMM_DEBUG_DIST") != nullptr;
      if (dbg_dist) dbg_digest(c, f, ("colour " + std::to_string(col) + " start").c_str());
      if (!S.empty()) compress(c, f, S, [&] {
          if (dbg_dist) dbg_digest(c, f, ("colour " + std::to_string(col) + " compressed").c_str());
          eliminate_invert(c, f, cs, plan);
        });
      else eliminate_invert(c, f, cs, plan);
      if (dbg_dist) dbg_digest(c, f, ("colour " + std::to_string(col) + " inverted+redirected").c_str());
      g_prof.end(("compress.L" + std::to_string(l)).c_str());
      g_prof.begin(c.s);
      eliminate_update(c, f, cs, plan);
      g_prof.end(("eliminate.L" + std::to_string(l)).c_str());
      static const bool dbg_sym = getenv("AIFMM_DEBUG_SYM") != nullptr;
      if (dbg_sym) dbg_symmetry(c, f, ("after colour " + std::to_string(col)).c_str());
      if (dbg_dist) dbg_digest(c, f, ("colour " + std::to_string(col) + " eliminated").c_str());
      if (c.algorithm == 2 && !f.pending.empty()) {   // Alg. 2: compress on creation (R29)
        std::vector<std::pair<int, int>> all(f.pending.begin(), f.pending.end());
        compress(c, f, all, [] {});
      }
    }
    AIFMM_REQUIRE(f.pending.empty(), AIFMM_ESINGULAR_PIVOT, "pending far fill-ins at level end");
    if (g_prof.on) {
      double ms = 0, mx = 0, ks = 0, kx = 0, k0s = 0;
      for (int b : f.boxes) { ms += f.m[b]; mx = std::max(mx, (double)f.m[b]); ks += f.k[b]; kx = std::max(kx, (double)f.k[b]); k0s += c.nn[l].k[b]; }
      double nbx = (double)f.boxes.size();
      fprintf(stderr, "[aifmm profile] level %d boxes %d m avg %.1f max %.0f | k nnca avg %.1f final avg %.1f max %.0f"
              " | GB persist %.2f (all %.2f) scratch %.2f+%.2f work %.2f\n",
              l, (int)nbx, ms / nbx, mx, k0s / nbx, ks / nbx, kx, c.persist.total() / 1e9, chunk_cache().total() / 1e9,
              c.scratch0.total() / 1e9, c.scratch1.total() / 1e9, c.work.total() / 1e9);
    }
    for (int b : f.boxes) c.stats[AIFMM_STAT_MAX_RANK] = std::max(c.stats[AIFMM_STAT_MAX_RANK], (double)f.k[b]);
    // solve layout
    f.xrow.assign(f.nb + 1, 0);
    f.zrow.assign(f.nb + 1, 0);
    for (int b = 0; b < f.nb; ++b) {
      f.xrow[b + 1] = f.xrow[b] + f.m[b];
      f.zrow[b + 1] = f.zrow[b] + f.k[b];
    }
    f.Xtot = f.xrow[f.nb];
    f.Ztot = f.zrow[f.nb];
  }
  g_expose.set("top");
  // top: M = (Z_p, y_q) over level-2 boxes; inverted in place (R19 dense GJ)
  g_prof.begin(c.s);
  FLevel& f = c.fl[2];
  c.topn = (int)f.Ztot;
  c.topoff = f.zrow;
  c.topinv = c.persist.d(std::max<size_t>((size_t)c.topn * c.topn, 1));
  CopyBatch cb;
  for (int p : f.boxes)
    for (int q : f.boxes) {
      if (!f.k[p] || !f.k[q]) continue;
      const Blk* it = f.nearb.get(f.key(p, q));
      const Blk& B = it ? *it : f.A.at(f.key(p, q));
      cb.copy(B.p, B.ld, c.topinv + (size_t)f.zrow[q] * c.topn + f.zrow[p], c.topn, f.k[p], f.k[q]);
    }
  cb.run(c.up, c.s);
  if (c.topn) {
    int* dinfo = c.work.i(1);
    AIFMM_CUDA(cudaMemsetAsync(dinfo, 0, sizeof(int), c.s));
    batched_inverse(std::vector<InvReq>{InvReq{c.topinv, c.topn, c.topn, dinfo}}, c.work, c.up, c.s, &c.fc_all);
    int info = d2h(c, dinfo, 1)[0];
    if (info) throw Error(AIFMM_ESINGULAR_PIVOT, "singular top-level system");
  }
  // deferred checks (the kernels set sticky device flags; reading them once here keeps the
  // level loop free of stream synchronisations): coincident points in the near-field kernel
  // blocks, singular box pivots
  deferred_checks(c);
  c.stats[AIFMM_STAT_TOP_SIZE] = c.topn;
  c.work.reset();
  g_prof.end("top");
  g_prof.dump("factor");
  g_expose.set("after");
  g_expose.dump();
}

// ------------------------------------------------------------------------------------ solve
static void solve_dev(Ctx& c, double* B, int nrhs) {
  const int L = c.L;
  const long long n = c.n;
  DevPool& W = c.work;
  W.reset();
  double* Bs = W.d((size_t)n * nrhs);
  LAUNCH(permute_rows_kernel, gsz(n * nrhs), 256, 0, c.s, B, Bs, c.perm, n, nrhs, 0);
  std::vector<double*> RZ(L + 2, nullptr), SX(L + 1, nullptr);
  for (int l = 2; l <= L; ++l) {
    RZ[l] = W.d(std::max<long long>(c.fl[l].Ztot * nrhs, 1));
    AIFMM_CUDA(cudaMemsetAsync(RZ[l], 0, sizeof(double) * c.fl[l].Ztot * nrhs, c.s));
    SX[l] = (l == L) ? W.d((size_t)n * nrhs) : W.d(std::max<long long>(c.fl[l].Xtot * nrhs, 1));
  }
  auto RXp = [&](int l, int b, int* ld) -> double* {
    if (l == L) { *ld = (int)n; return Bs + c.off[L][b]; }
    *ld = (int)c.fl[l + 1].Ztot;
    return RZ[l + 1] + c.fl[l].xrow[b];
  };
  // forward (Alg. 4 replays the eliminations on the rhs; T_As includes it)
  for (int l = L; l >= 2; --l) {
    FLevel& f = c.fl[l];
    int ncol = 0;
    for (int b : f.boxes) ncol = std::max(ncol, c.col[l][b] + 1);
    const int ldz = (int)f.Ztot;
    for (int col = 0; col < ncol; ++col) {
      std::vector<int> cs;
      for (int b : f.boxes)
        if (c.col[l][b] == col) cs.push_back(b);
      GemmBatch g;
      std::vector<double*> w(cs.size());
      for (size_t a = 0; a < cs.size(); ++a) {
        const Rec& r = f.rec[cs[a]];
        const int nn = r.m + r.k;
        w[a] = W.d(std::max<size_t>((size_t)nn * nrhs, 1));
        if (!nn || !r.m) {
          if (nn) { CopyBatch z; z.fill(w[a], nn, nn, nrhs, 0.0); z.run(c.up, c.s); }
          continue;
        }
        int ld;
        double* rx = RXp(l, cs[a], &ld);
        g.task(w[a], nn, nn, nrhs, 0.0);
        g.term(1.0, r.G, nn, 0, rx, ld, 0, r.m);
      }
      g.run(c.up, c.s, &c.fc_all);
      // targets: (p, row-kind) -> contributions
      std::map<std::pair<int, int>, std::vector<std::pair<int, int>>> tg;   // -> (a, idx in C)
      for (size_t a = 0; a < cs.size(); ++a) {
        const Rec& r = f.rec[cs[a]];
        for (size_t t = 0; t < r.C.size(); ++t) tg[{r.C[t].first, (int)r.Ckind_z[t]}].push_back({(int)a, (int)t});
        tg[{cs[a], 2}].push_back({(int)a, -1});
      }
      for (auto& kv : tg) {
        const int p = kv.first.first, kind = kv.first.second;
        double* C;
        int ldc, M;
        if (kind == 0) { C = RXp(l, p, &ldc); M = f.m[p]; }
        else { C = RZ[l] + f.zrow[p]; ldc = ldz; M = f.k[p]; }
        if (!M) continue;
        g.task(C, ldc, M, nrhs, 1.0);
        for (auto& at : kv.second) {
          const Rec& r = f.rec[cs[at.first]];
          const int nn = r.m + r.k;
          if (at.second < 0) {
            if (r.k) g.add(1.0, w[at.first] + r.m, nn, 0);
          } else if (half_records()) {   // R32: C_p = R_p^T (same partner order in R and C)
            const Blk& Rb = r.R[at.second].second;
            if (r.m) g.term(-1.0, Rb.p, Rb.ld, 1, w[at.first], nn, 0, r.m);
          } else {
            const Blk& Cb = r.C[at.second].second;
            if (r.m) g.term(-1.0, Cb.p, Cb.ld, 0, w[at.first], nn, 0, r.m);
          }
        }
      }
      g.run(c.up, c.s, &c.fc_all);
    }
  }
  // top: y2 = M^{-1} b_Z
  double* y2 = W.d(std::max<long long>((long long)c.topn * nrhs, 1));
  {
    GemmBatch g;
    if (c.topn) {
      g.task(y2, c.topn, c.topn, nrhs, 0.0);
      g.term(1.0, c.topinv, c.topn, 0, RZ[2], c.topn, 0, c.topn);
    }
    g.run(c.up, c.s, &c.fc_all);
  }
  // backward
  for (int l = 2; l <= L; ++l) {
    FLevel& f = c.fl[l];
    double* Y = (l == 2) ? y2 : SX[l - 1];
    const int ldy = (int)f.Ztot;
    double* X = SX[l];
    const int ldx = (l == L) ? (int)n : (int)f.Xtot;
    auto xrow = [&](int b) -> long long { return (l == L) ? c.off[L][b] : f.xrow[b]; };
    int ncol = 0;
    for (int b : f.boxes) ncol = std::max(ncol, c.col[l][b] + 1);
    for (int col = ncol - 1; col >= 0; --col) {
      std::vector<int> cs;
      for (int b : f.boxes)
        if (c.col[l][b] == col) cs.push_back(b);
      CopyBatch cb;
      GemmBatch g;
      std::vector<double*> tmp(cs.size());
      for (size_t a = 0; a < cs.size(); ++a) {
        const int i = cs[a];
        const Rec& r = f.rec[i];
        const int nn = r.m + r.k;
        tmp[a] = W.d(std::max<size_t>((size_t)nn * nrhs, 1));
        int ld;
        double* rx = RXp(l, i, &ld);
        cb.copy(rx, ld, tmp[a], nn, r.m, nrhs);
        cb.copy(Y + f.zrow[i], ldy, tmp[a] + r.m, nn, r.k, nrhs);
      }
      cb.run(c.up, c.s);
      for (size_t a = 0; a < cs.size(); ++a) {
        const int i = cs[a];
        const Rec& r = f.rec[i];
        const int nn = r.m + r.k;
        if (!r.m) continue;
        g.task(tmp[a], nn, r.m, nrhs, 1.0);
        for (size_t t = 0; t < r.R.size(); ++t) {
          const int q = r.R[t].first;
          const Blk& Rb = r.R[t].second;
          if (r.Rkind_y[t]) {
            if (f.k[q]) g.term(-1.0, Rb.p, Rb.ld, 0, Y + f.zrow[q], ldy, 0, f.k[q]);
          } else {
            if (f.m[q]) g.term(-1.0, Rb.p, Rb.ld, 0, X + xrow(q), ldx, 0, f.m[q]);
          }
        }
      }
      g.run(c.up, c.s, &c.fc_all);
      for (size_t a = 0; a < cs.size(); ++a) {
        const int i = cs[a];
        const Rec& r = f.rec[i];
        const int nn = r.m + r.k;
        if (!r.m) continue;
        g.task(X + xrow(i), ldx, r.m, nrhs, 0.0);
        g.term(1.0, r.G, nn, 0, tmp[a], nn, 0, nn);
      }
      g.run(c.up, c.s, &c.fc_all);
    }
  }
  LAUNCH(permute_rows_kernel, gsz(n * nrhs), 256, 0, c.s, SX[L], B, c.perm, n, nrhs, 1);
  c.up.sync();
  W.reset();
}

// ------------------------------------------------------------------------------------ H2 matvec
// Y = A_H2 X (user order, N x nrhs column-major, device), row a8 (oracle/h2.py): upward
// P2M/M2M as DMMA GEMMs with the NNCA operators (V = U, R10), M2L and near field as fused
// kernel-evaluation sums (kmv_kernel), downward L2L and L2P as GEMMs.  Multipoles and locals
// of a level are stored box-ordered (skoff), so a box's children are one contiguous run.
static void matvec_dev(Ctx& c, const double* X, double* Y, int nrhs) {
  const int L = c.L, d = c.d;
  const long long n = c.n;
  DevPool& W = c.h2work;
  W.reset();
  double* Xs = W.d((size_t)n * nrhs);
  double* Ys = W.d((size_t)n * nrhs);
  LAUNCH(permute_rows_kernel, gsz(n * nrhs), 256, 0, c.s, X, Xs, c.perm, n, nrhs, 0);
  std::vector<double*> q(L + 1, nullptr), lc(L + 1, nullptr);
  std::vector<int> kt(L + 1, 0);
  for (int l = 2; l <= L; ++l) {
    const NLevel& nl = c.hnn[l];
    kt[l] = (int)nl.skoff[(size_t)1 << (d * l)];
    q[l] = W.d(std::max<size_t>((size_t)kt[l] * nrhs, 1));
    lc[l] = W.d(std::max<size_t>((size_t)kt[l] * nrhs, 1));
  }
  auto boxes = [&](int l) {
    std::vector<int> v;
    for (int b = 0; b < (1 << (d * l)); ++b)
      if (c.nonempty(l, b)) v.push_back(b);
    return v;
  };
  // upward
  for (int l = L; l >= 2; --l) {
    const NLevel& nl = c.hnn[l];
    GemmBatch g;
    for (int b : boxes(l)) {
      const int k = nl.k[b], nR = nl.nR[b];
      if (!k) continue;
      g.task(q[l] + nl.skoff[b], std::max(kt[l], 1), k, nrhs, 0.0);
      if (!nR) continue;
      const double* src = (l == L) ? Xs + c.off[L][b] : q[l + 1] + c.hnn[l + 1].skoff[(size_t)b << d];
      const int lds = (l == L) ? (int)n : std::max(kt[l + 1], 1);
      g.term(1.0, nl.dU + nl.Uoff[b], nR, 1, src, lds, 0, nR);
    }
    g.run(c.up, c.s);
  }
  // M2L (all levels in one launch): l_B = sum_{D in IL(B)} A(sk_B, sk_D) q_D
  {
    std::vector<KmvTarget> tg;
    std::vector<KmvSource> sr;
    for (int l = 2; l <= L; ++l) {
      const NLevel& nl = c.hnn[l];
      for (int b : boxes(l)) {
        if (!nl.k[b]) continue;
        KmvTarget t{nl.dsk + nl.skoff[b], 0, nl.k[b], lc[l] + nl.skoff[b], std::max(kt[l], 1), (int)sr.size(), 0};
        int ni;
        const int* il = c.ilist(l, b, &ni);
        for (int s = 0; s < ni; ++s) {
          const int D = il[s];
          if (!nl.k[D]) continue;
          sr.push_back(KmvSource{nl.dsk + nl.skoff[D], 0, nl.k[D], q[l] + nl.skoff[D], std::max(kt[l], 1), 0});
        }
        t.src_end = (int)sr.size();
        tg.push_back(t);
      }
    }
    if (!tg.empty()) {
      const KmvSource* ds = sr.empty() ? nullptr : c.up.put(sr);
      launch_kmv(c.up.put(tg), ds, (int)tg.size(), c.pts, c.kp, nrhs, 0, c.s);
    }
  }
  // downward: l_c += U_P[rows of c] l_P
  for (int l = 2; l < L; ++l) {
    const NLevel& nl = c.hnn[l];
    GemmBatch g;
    for (int b : boxes(l)) {
      const int k = nl.k[b], nR = nl.nR[b];
      if (!k || !nR) continue;
      g.task(lc[l + 1] + c.hnn[l + 1].skoff[(size_t)b << d], std::max(kt[l + 1], 1), nR, nrhs, 1.0);
      g.term(1.0, nl.dU + nl.Uoff[b], nR, 0, lc[l] + nl.skoff[b], std::max(kt[l], 1), 0, k);
    }
    g.run(c.up, c.s);
  }
  // leaf: L2P, then the near field
  AIFMM_CUDA(cudaMemsetAsync(Ys, 0, sizeof(double) * n * nrhs, c.s));
  {
    const NLevel& nl = c.hnn[L];
    GemmBatch g;
    std::vector<KmvTarget> tg;
    std::vector<KmvSource> sr;
    for (int b : boxes(L)) {
      const int k = nl.k[b], m = c.count(L, b);
      if (k) {
        g.task(Ys + c.off[L][b], (int)n, m, nrhs, 1.0);
        g.term(1.0, nl.dU + nl.Uoff[b], m, 0, lc[L] + nl.skoff[b], std::max(kt[L], 1), 0, k);
      }
      KmvTarget t{nullptr, (int)c.off[L][b], m, Ys + c.off[L][b], (int)n, (int)sr.size(), 0};
      int nn_;
      const int* nbl = c.nlist(L, b, &nn_);
      for (int s = 0; s < nn_; ++s)
        sr.push_back(KmvSource{nullptr, (int)c.off[L][nbl[s]], c.count(L, nbl[s]), Xs + c.off[L][nbl[s]], (int)n, 0});
      t.src_end = (int)sr.size();
      tg.push_back(t);
    }
    g.run(c.up, c.s);
    if (!tg.empty()) launch_kmv(c.up.put(tg), c.up.put(sr), (int)tg.size(), c.pts, c.kp, nrhs, 1, c.s);
  }
  LAUNCH(permute_rows_kernel, gsz(n * nrhs), 256, 0, c.s, Ys, Y, c.perm, n, nrhs, 1);
  c.up.sync();
}

// Block-diagonal preconditioner (the paper's I_BD column, P:1628-1629,
// table): M = blockdiag(A(points(b), points(b))) over the leaves b, each block
// evaluated exactly and inverted once (batched Gauss-Jordan, R16); stored in c.bdpool.
static void bd_prepare(Ctx& c) {
  if (c.bd_ready) return;
  const int L = c.L;
  const int nb = 1 << (c.d * L);
  c.bdpool.reset();
  c.bdoff.assign(nb + 1, 0);
  for (int b = 0; b < nb; ++b) c.bdoff[b + 1] = c.bdoff[b] + (long long)c.count(L, b) * c.count(L, b);
  c.bdinv = c.bdpool.d(std::max<long long>(c.bdoff[nb], 1));
  std::vector<KEvalTask> kt;
  std::vector<InvReq> inv;
  int* dinfo = c.bdpool.i(nb);
  AIFMM_CUDA(cudaMemsetAsync(dinfo, 0, sizeof(int) * nb, c.s));
  AIFMM_CUDA(cudaMemsetAsync(c.dflag, 0, sizeof(int), c.s));
  for (int b = 0; b < nb; ++b) {
    const int m = c.count(L, b);
    if (!m) continue;
    const int r0 = (int)c.off[L][b];
    kt.push_back(KEvalTask{c.bdinv + c.bdoff[b], m, m, m, nullptr, nullptr, r0, r0});
    inv.push_back(InvReq{c.bdinv + c.bdoff[b], m, m, dinfo + b});
  }
  if (!kt.empty()) launch_keval(c.up.put(kt), (int)kt.size(), 4, c.pts, c.kp, c.dflag, c.s);
  batched_inverse(inv, c.work, c.up, c.s, &c.fc_all);
  check_flag(c, AIFMM_ECOINCIDENT, "coincident points with a singular kernel");
  std::vector<int> info = d2h(c, dinfo, nb);
  for (int b = 0; b < nb; ++b)
    if (info[b]) throw Error(AIFMM_ESINGULAR_PIVOT, "singular leaf block " + std::to_string(b));
  c.work.reset();
  c.bd_ready = true;
}
// v <- M^{-1} v (user order, one column): gather to tree order, one GEMM per leaf, scatter back
static void bd_apply(Ctx& c, double* v, double* tmp) {
  const int L = c.L;
  const long long n = c.n;
  LAUNCH(permute_rows_kernel, gsz(n), 256, 0, c.s, v, tmp, c.perm, n, 1, 0);
  GemmBatch g;
  for (int b = 0; b < (1 << (c.d * L)); ++b) {
    const int m = c.count(L, b);
    if (!m) continue;
    g.task(tmp + n + c.off[L][b], m, m, 1, 0.0);
    g.term(1.0, c.bdinv + c.bdoff[b], m, 0, tmp + c.off[L][b], m, 0, m);
  }
  g.run(c.up, c.s, &c.fc_all);
  LAUNCH(permute_rows_kernel, gsz(n), 256, 0, c.s, tmp + n, v, c.perm, n, 1, 1);
}

// Right-preconditioned GMRES(restart) with MGS Arnoldi (oracle/h2.py: gmres); A = the H2
// matvec, M^{-1} = the AIFMM solve (precond 1), the leaf block-diagonal inverse (precond 2) or
// none (precond 0).  b, x: device, user order, N x 1.
static void gmres_dev(Ctx& c, const double* b, double* x, int restart, double rtol, int maxit, int precond,
                      int* iters, double* relres) {
  const long long n = c.n;
  DevPool& P = c.gmpool;
  P.reset();
  const int ldh = restart + 1;
  double* V = P.d((size_t)n * (restart + 1));
  double* w = P.d(n);
  double* t = P.d(n);
  double* r = P.d(n);
  double* H = P.d((size_t)ldh * restart);
  double* cs = P.d(restart);
  double* sn = P.d(restart);
  double* g = P.d(restart + 1);
  double* y = P.d(restart);
  double* part = P.d(512);
  double* sc = P.d(8);   // 0: ||b||, 1: beta, 2: residual estimate
  double* bdt = precond == 2 ? P.d((size_t)2 * n) : nullptr;
  if (precond == 2) bd_prepare(c);
  auto apply_precond = [&](double* v) {
    if (precond == 1) solve_dev(c, v, 1);
    else if (precond == 2) bd_apply(c, v, bdt);
  };
  auto rd = [&](double* dp) {
    double h = 0;
    AIFMM_CUDA(cudaMemcpyAsync(&h, dp, sizeof(double), cudaMemcpyDeviceToHost, c.s));
    AIFMM_CUDA(cudaStreamSynchronize(c.s));
    return h;
  };
  AIFMM_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * n, c.s));
  vec_dot(b, b, n, part, sc + 0, 1, c.s);
  const double bnorm = rd(sc + 0);
  int it = 0;
  if (bnorm == 0.0) { *iters = 0; *relres = 0.0; return; }
  vec_axpy(r, b, n, nullptr, 1.0, 0.0, c.s);   // r = b - A 0
  vec_dot(r, r, n, part, sc + 1, 1, c.s);
  double beta = rd(sc + 1);
  while (it < maxit && beta > rtol * bnorm) {
    AIFMM_CUDA(cudaMemsetAsync(H, 0, sizeof(double) * ldh * restart, c.s));
    AIFMM_CUDA(cudaMemsetAsync(g, 0, sizeof(double) * (restart + 1), c.s));
    set_scalar(g, sc + 1, 0.0, c.s);
    vec_scale_div(V, r, n, sc + 1, c.s);
    int j = 0;
    while (j < restart && it < maxit) {
      double* vj = V + (size_t)j * n;
      const double* op = vj;
      if (precond) {
        vec_axpy(t, vj, n, nullptr, 1.0, 0.0, c.s);
        apply_precond(t);
        op = t;
      }
      matvec_dev(c, op, w, 1);
      for (int i = 0; i <= j; ++i) {                   // modified Gram-Schmidt
        double* hij = H + (size_t)j * ldh + i;
        vec_dot(w, V + (size_t)i * n, n, part, hij, 0, c.s);
        vec_axpy(w, V + (size_t)i * n, n, hij, -1.0, 1.0, c.s);
      }
      double* hj1 = H + (size_t)j * ldh + j + 1;
      vec_dot(w, w, n, part, hj1, 1, c.s);
      vec_scale_div(V + (size_t)(j + 1) * n, w, n, hj1, c.s);
      gm_givens(H, ldh, cs, sn, g, j, sc + 2, c.s);
      ++j;
      ++it;
      if (rd(sc + 2) <= rtol * bnorm) break;
    }
    gm_backsub(H, ldh, g, y, j, c.s);
    gm_gemv(V, n, y, j, n, t, c.s);
    if (precond) apply_precond(t);
    vec_axpy(x, t, n, nullptr, 1.0, 1.0, c.s);
    matvec_dev(c, x, w, 1);                            // true residual at the restart
    vec_axpy(r, b, n, nullptr, 1.0, 0.0, c.s);
    vec_axpy(r, w, n, nullptr, -1.0, 1.0, c.s);
    vec_dot(r, r, n, part, sc + 1, 1, c.s);
    beta = rd(sc + 1);
  }
  *iters = it;
  *relres = beta / bnorm;
}

// ------------------------------------------------------------------------------------ residual
// Row a9 (verification, not timed): ||A X - B||_F / ||B||_F over the sampled rows by exact direct
// sum (A_ij = K(x_i, x_j), A_ii = diag).  X, B: device, user order, n x nrhs
// column-major.  The rows are split into blocks of 128 (one thread per row) and the sources
// into chunks; each (row block, chunk) pair writes its own partial product (kmv_kernel), and
// the partials are summed in chunk order (deterministic).
static double residual_dev(Ctx& c, const double* X, const double* B, int nrhs, const int64_t* rows, long long nrows) {
  const long long n = c.n;
  c.work.reset();
  std::vector<int> permh = d2h(c, c.perm, (size_t)n);
  std::vector<int> inv((size_t)n);
  for (long long j = 0; j < n; ++j) inv[permh[j]] = (int)j;
  std::vector<int> rt((size_t)nrows), ru((size_t)nrows);
  for (long long i = 0; i < nrows; ++i) {
    const long long u = rows ? rows[i] : i;
    AIFMM_REQUIRE(u >= 0 && u < n, AIFMM_EINVALID_ARG, "residual row out of range");
    ru[i] = (int)u;
    rt[i] = inv[u];
  }
  int* drt = c.work.i(nrows);
  int* dru = c.work.i(nrows);
  AIFMM_CUDA(cudaMemcpyAsync(drt, rt.data(), sizeof(int) * nrows, cudaMemcpyHostToDevice, c.s));
  AIFMM_CUDA(cudaMemcpyAsync(dru, ru.data(), sizeof(int) * nrows, cudaMemcpyHostToDevice, c.s));
  double* Xt = c.work.d((size_t)n * nrhs);
  LAUNCH(permute_rows_kernel, gsz(n * nrhs), 256, 0, c.s, X, Xt, c.perm, n, nrhs, 0);
  const long long nblk = (nrows + 127) / 128;
  const int S = (int)std::max<long long>(1, std::min<long long>(std::max<long long>(1, 2048 / nblk), (n + 1023) / 1024));
  const long long cs = (n + S - 1) / S;
  double* part = c.work.d((size_t)S * nrows * nrhs);
  std::vector<KmvTarget> tg;
  std::vector<KmvSource> src;
  for (int s = 0; s < S; ++s) {
    const long long c0 = s * cs, nc = std::max<long long>(0, std::min(cs, n - c0));
    src.push_back(KmvSource{nullptr, (int)c0, (int)nc, Xt + c0, (int)n, 0});
  }
  for (long long rb = 0; rb < nblk; ++rb)
    for (int s = 0; s < S; ++s) {
      const long long r0 = rb * 128;
      tg.push_back(KmvTarget{drt + r0, 0, (int)std::min<long long>(128, nrows - r0), part + (size_t)s * nrows * nrhs + r0,
                             (int)nrows, s, s + 1});
    }
  const KmvTarget* dtg = c.up.put(tg);
  const KmvSource* dsrc = c.up.put(src);
  launch_kmv(dtg, dsrc, (int)tg.size(), c.pts, c.kp, nrhs, 0, c.s);
  double* dout = c.work.d(2);
  resid_finish(part, S, nrows, nrhs, B, n, dru, dout, c.s);
  std::vector<double> o = d2h(c, dout, 2);
  c.work.reset();
  return o[1] > 0.0 ? std::sqrt(o[0] / o[1]) : std::sqrt(o[0]);
}

}  // namespace aifmm

// ====================================================================================== C-ABI
using namespace aifmm;

#define CAPI_BEGIN try {
#define CAPI_END                                      \
  }                                                   \
  catch (const aifmm::Error& e) {                     \
    g_err = e.what();                                 \
    return e.code;                                    \
  }                                                   \
  catch (const std::exception& e) {                   \
    g_err = e.what();                                 \
    return AIFMM_ECUDA;                               \
  }                                                   \
  g_err.clear();                                      \
  return AIFMM_OK;

static double ms_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

extern "C" {

int aifmm_build(const double* points, int64_t n, int d, int kernel_id, const double* kparams, int leaf_size,
                double tol) {
  CAPI_BEGIN
  AIFMM_REQUIRE(points && kparams, AIFMM_EINVALID_ARG, "null pointer");
  AIFMM_REQUIRE(n >= 1 && n < (1ll << 31), AIFMM_EINVALID_ARG, "n out of range");
  AIFMM_REQUIRE(d == 2 || d == 3, AIFMM_EINVALID_ARG, "d must be 2 or 3");
  AIFMM_REQUIRE(kernel_id >= 0 && kernel_id <= 2, AIFMM_EINVALID_ARG, "unknown kernel id");
  AIFMM_REQUIRE(leaf_size >= 1 && leaf_size <= 4096, AIFMM_EINVALID_ARG, "leaf_size out of range");
  AIFMM_REQUIRE(tol > 0.0 && tol < 1.0, AIFMM_EINVALID_ARG, "tol must lie in (0,1)");
  Ctx& c = ctx();
  auto t0 = std::chrono::steady_clock::now();
  c.persist.recycle();
  c.buildp.recycle();
  c.scratch0.recycle();
  c.scratch1.recycle();
  c.work.reset();
  c.fl.clear();
  c.nn.clear();
  c.hnn.clear();
  c.h2_built = false;
  c.bd_ready = false;
  c.bdpool.reset();
  c.h2pool.reset();
  c.built = c.factored = false;
  c.n = n;
  c.d = d;
  c.kid = kernel_id;
  c.leaf = leaf_size;
  c.tol = tol;
  c.kp = KernelParams{kernel_id, d, kparams[0], kparams[1]};
  if (kernel_id == 1) AIFMM_REQUIRE(kparams[1] > 0.0, AIFMM_EINVALID_ARG, "ell must be > 0");
  g_prof.on = getenv("AIFMM_PROFILE") != nullptr;
  g_prof.begin(c.s);
  build_tree(c, points);
  g_prof.end("tree");
  plan_ownership(c);   // §8(e): the build's NNCA is split by subtree as well
  set_ws_budget(c);
  g_prof.begin(c.s);
  build_nnca(c);
  g_prof.end("nnca");
  g_prof.dump("build");
  c.buildp.recycle();
  c.built = true;
  c.stats[AIFMM_STAT_LEVELS] = c.L;
  c.stats[AIFMM_STAT_BUILD_MS] = ms_since(t0);
  CAPI_END
}

int aifmm_set_compression_tol(double tol_c) {
  CAPI_BEGIN
  AIFMM_REQUIRE(tol_c >= 0.0 && tol_c < 1.0, AIFMM_EINVALID_ARG, "tol_c must lie in [0,1)");
  ctx().tol_c_user = tol_c;
  CAPI_END
}

int aifmm_set_algorithm(int alg) {
  CAPI_BEGIN
  AIFMM_REQUIRE(alg == 2 || alg == 3, AIFMM_EINVALID_ARG, "algorithm must be 2 or 3");
  ctx().algorithm = alg;
  CAPI_END
}

int aifmm_factor(void) {
  CAPI_BEGIN
  Ctx& c = ctx();
  AIFMM_REQUIRE(c.built, AIFMM_ESTATE, "factor before build");
  auto t0 = std::chrono::steady_clock::now();
  if (c.factored) {
    // re-factor from the same build: drop the previous factor storage but keep NNCA
    throw Error(AIFMM_ESTATE, "already factored: call aifmm_build again");
  }
  c.tol_c = (c.tol_c_user >= 0) ? c.tol_c_user : c.tol;
  for (auto& e : c.ev) { cudaEventDestroy(e.first); cudaEventDestroy(e.second); }
  c.ev.clear();
  for (auto& v : c.evp) {
    for (auto& e : v) { cudaEventDestroy(e.first); cudaEventDestroy(e.second); }
    v.clear();
  }
  factor_all(c);
  c.up.sync();
  double sch = 0.0;
  for (auto& e : c.ev) {
    float ms = 0.f;
    AIFMM_CUDA(cudaEventElapsedTime(&ms, e.first, e.second));
    sch += ms;
    cudaEventDestroy(e.first);
    cudaEventDestroy(e.second);
  }
  c.ev.clear();
  for (int ph = 0; ph < NPH; ++ph) {
    double t = 0.0;
    for (auto& e : c.evp[ph]) {
      float ms = 0.f;
      AIFMM_CUDA(cudaEventElapsedTime(&ms, e.first, e.second));
      t += ms;
      cudaEventDestroy(e.first);
      cudaEventDestroy(e.second);
    }
    c.evp[ph].clear();
    c.stats[AIFMM_STAT_PIVOT_MS + 3 * ph] += t;
    c.stats[AIFMM_STAT_PIVOT_FLOPS + 3 * ph] = c.fcp[ph].flops;
    c.stats[AIFMM_STAT_PIVOT_BYTES + 3 * ph] = c.fcp[ph].bytes;
  }
  c.stats[AIFMM_STAT_SCHUR_MS] += sch;
  c.stats[AIFMM_STAT_SCHUR_FLOPS] = c.fc_schur.flops;
  c.stats[AIFMM_STAT_SCHUR_BYTES] = c.fc_schur.bytes;
  c.stats[AIFMM_STAT_FACTOR_FLOPS] = c.fc_all.flops + c.fc_schur.flops;
  c.factored = true;
  c.stats[AIFMM_STAT_DIST_BYTES] = c.comm.bytes_in;
  c.stats[AIFMM_STAT_DIST_EXCHANGES] = (double)c.comm.exchanges;
  c.stats[AIFMM_STAT_FACTOR_MS] = ms_since(t0);
  c.stats[AIFMM_STAT_DEVICE_BYTES] =
      (double)chunk_cache().total();
  CAPI_END
}

int aifmm_solve(double* B, int nrhs) {
  CAPI_BEGIN
  Ctx& c = ctx();
  AIFMM_REQUIRE(c.factored, AIFMM_ESTATE, "solve before factor");
  AIFMM_REQUIRE(B && nrhs >= 1, AIFMM_EINVALID_ARG, "bad right-hand side");
  auto t0 = std::chrono::steady_clock::now();
  AIFMM_CUDA(cudaMemsetAsync(c.dflag, 0, sizeof(int), c.s));
  LAUNCH(finite_kernel, gsz(c.n * nrhs), 256, 0, c.s, B, c.n * nrhs, c.dflag);
  check_flag(c, AIFMM_ENONFINITE, "non-finite right-hand side");
  solve_dev(c, B, nrhs);
  c.stats[AIFMM_STAT_SOLVE_MS] = ms_since(t0);
  CAPI_END
}

int aifmm_solve_host(double* B, int nrhs) {
  CAPI_BEGIN
  Ctx& c = ctx();
  AIFMM_REQUIRE(c.factored, AIFMM_ESTATE, "solve before factor");
  AIFMM_REQUIRE(B && nrhs >= 1, AIFMM_EINVALID_ARG, "bad right-hand side");
  double* dB = nullptr;
  size_t bytes = sizeof(double) * c.n * nrhs;
  AIFMM_CUDA(cudaMalloc(&dB, bytes));
  try {
    AIFMM_CUDA(cudaMemcpyAsync(dB, B, bytes, cudaMemcpyHostToDevice, c.s));
    int rc = aifmm_solve(dB, nrhs);
    if (rc) throw Error(rc, g_err);
    AIFMM_CUDA(cudaMemcpyAsync(B, dB, bytes, cudaMemcpyDeviceToHost, c.s));
    AIFMM_CUDA(cudaStreamSynchronize(c.s));
  } catch (...) {
    cudaFree(dB);
    throw;
  }
  cudaFree(dB);
  CAPI_END
}

void aifmm_free(void) {
  if (!g_ctx) return;
  Ctx& c = *g_ctx;
  if (c.inited) cudaStreamSynchronize(c.s);
  c.fl.clear();
  c.nn.clear();
  c.hnn.clear();
  c.h2_built = false;
  c.bd_ready = false;
  c.bdpool.reset();
  c.h2pool.reset();
  c.h2work.reset();
  c.gmpool.reset();
  // device memory stays cached in the chunk cache (released at process exit or under pressure)
  c.persist.recycle();
  c.scratch0.recycle();
  c.scratch1.recycle();
  c.work.reset();
  c.buildp.recycle();
  c.built = c.factored = false;
  c.tol_c_user = -1;
}

const char* aifmm_last_error(void) { return g_err.c_str(); }

int aifmm_set_stream(void* stream) {
  CAPI_BEGIN
  Ctx& c = ctx();
  cudaStream_t ns = static_cast<cudaStream_t>(stream);
  if (ns == c.s) return 0;
  c.up.set_stream(ns);               // flushes and completes everything queued on the old stream
  AIFMM_CUDA(cudaStreamSynchronize(c.s));
  if (c.own_stream) cudaStreamDestroy(c.s);
  c.s = ns;
  c.own_stream = false;
  CAPI_END
}

int aifmm_get_tree(int64_t* perm, int* L) {
  CAPI_BEGIN
  Ctx& c = ctx();
  AIFMM_REQUIRE(c.built, AIFMM_ESTATE, "no build");
  if (L) *L = c.L;
  if (perm) {
    std::vector<int> p = d2h(c, c.perm, c.n);
    for (long long i = 0; i < c.n; ++i) perm[i] = p[i];
  }
  CAPI_END
}

int aifmm_get_level_offsets(int level, int64_t* off) {
  CAPI_BEGIN
  Ctx& c = ctx();
  AIFMM_REQUIRE(c.built && level >= 0 && level <= c.L && off, AIFMM_EINVALID_ARG, "bad level");
  for (size_t i = 0; i < c.off[level].size(); ++i) off[i] = c.off[level][i];
  CAPI_END
}

int aifmm_get_lists(int level, int32_t* n_ptr, int32_t* n_idx, int32_t* il_ptr, int32_t* il_idx) {
  CAPI_BEGIN
  Ctx& c = ctx();
  AIFMM_REQUIRE(c.built && level >= 2 && level <= c.L && n_ptr && il_ptr, AIFMM_EINVALID_ARG, "bad level");
  const int nb = 1 << (c.d * level);
  n_ptr[0] = il_ptr[0] = 0;
  for (int b = 0; b < nb; ++b) {
    n_ptr[b + 1] = n_ptr[b] + c.ncnt[level][b];
    il_ptr[b + 1] = il_ptr[b] + c.icnt[level][b];
    if (n_idx)
      for (int t = 0; t < c.ncnt[level][b]; ++t) n_idx[n_ptr[b] + t] = c.nidx[level][(size_t)b * c.ncap + t];
    if (il_idx)
      for (int t = 0; t < c.icnt[level][b]; ++t) il_idx[il_ptr[b] + t] = c.iidx[level][(size_t)b * c.icap + t];
  }
  CAPI_END
}

int aifmm_get_colours(int level, int32_t* colour) {
  CAPI_BEGIN
  Ctx& c = ctx();
  AIFMM_REQUIRE(c.built && level >= 2 && level <= c.L && colour, AIFMM_EINVALID_ARG, "bad level");
  for (size_t b = 0; b < c.col[level].size(); ++b) colour[b] = c.col[level][b];
  CAPI_END
}

int aifmm_get_ranks(int level, int which, int32_t* ranks) {
  CAPI_BEGIN
  Ctx& c = ctx();
  AIFMM_REQUIRE(c.built && level >= 2 && level <= c.L && ranks, AIFMM_EINVALID_ARG, "bad level");
  const int nb = 1 << (c.d * level);
  for (int b = 0; b < nb; ++b) {
    if (which == 0) ranks[b] = c.nn[level].k[b];
    else {
      AIFMM_REQUIRE(c.factored, AIFMM_ESTATE, "not factored");
      ranks[b] = c.fl[level].k[b];
    }
  }
  CAPI_END
}

int aifmm_get_skeletons(int level, int32_t* sk_ptr, int32_t* sk_idx, int32_t* fp_idx) {
  CAPI_BEGIN
  Ctx& c = ctx();
  AIFMM_REQUIRE(c.built && level >= 2 && level <= c.L && sk_ptr, AIFMM_EINVALID_ARG, "bad level");
  const NLevel& nl = c.nn[level];
  const int nb = 1 << (c.d * level);
  for (int b = 0; b <= nb; ++b) sk_ptr[b] = (int32_t)nl.skoff[b];
  const size_t tot = (size_t)nl.skoff[nb];
  if (tot && sk_idx) {
    std::vector<int> h = d2h(c, nl.dsk, tot);
    std::copy(h.begin(), h.end(), sk_idx);
  }
  if (tot && fp_idx) {
    std::vector<int> h = d2h(c, nl.dfp, tot);
    std::copy(h.begin(), h.end(), fp_idx);
  }
  CAPI_END
}

int aifmm_stats(double* out) {
  CAPI_BEGIN
  Ctx& c = ctx();
  c.stats[AIFMM_STAT_LAUNCHES] = (double)g_launches;
  c.stats[AIFMM_STAT_HOST_SYNCS] = (double)c.up.syncs;
  for (int i = 0; i < AIFMM_NSTATS; ++i) out[i] = c.stats[i];
  CAPI_END
}

int aifmm_reset_counters(void) {
  CAPI_BEGIN
  Ctx& c = ctx();
  g_launches = 0;
  c.up.syncs = 0;
  c.fc_all = FlopCounter{};
  c.fc_schur = FlopCounter{};
  for (auto& f : c.fcp) f = FlopCounter{};
  for (int i = AIFMM_STAT_PIVOT_MS; i < AIFMM_NSTATS; ++i) c.stats[i] = 0;
  c.stats[AIFMM_STAT_SCHUR_MS] = 0;
  c.stats[AIFMM_STAT_SCHUR_LAUNCHES] = 0;
  c.stats[AIFMM_STAT_COMPRESSIONS] = 0;
  c.stats[AIFMM_STAT_MAX_RANK] = 0;
  CAPI_END
}

int aifmm_debug_inverse(double* A, int n, int lda) {
  CAPI_BEGIN
  Ctx& c = ctx();
  int* dinfo = c.work.i(1);
  AIFMM_CUDA(cudaMemsetAsync(dinfo, 0, sizeof(int), c.s));
  batched_inverse(std::vector<InvReq>{InvReq{A, lda, n, dinfo}}, c.work, c.up, c.s);
  int info = d2h(c, dinfo, 1)[0];
  c.work.reset();
  if (info) throw Error(AIFMM_ESINGULAR_PIVOT, "singular matrix");
  CAPI_END
}

int aifmm_debug_inverse_batch(double* A, int n, int batch, int path) {
  CAPI_BEGIN
  AIFMM_REQUIRE(A && n >= 1 && batch >= 1 && path >= 0 && path <= 2, AIFMM_EINVALID_ARG, "bad arguments");
  Ctx& c = ctx();
  std::vector<InvReq> reqs;
  int* dinfo = c.work.i(batch);
  AIFMM_CUDA(cudaMemsetAsync(dinfo, 0, sizeof(int) * batch, c.s));
  for (int b = 0; b < batch; ++b) reqs.push_back(InvReq{A + (size_t)b * n * n, n, n, dinfo + b});
  g_gj_force = path;
  try {
    batched_inverse(reqs, c.work, c.up, c.s);
  } catch (...) {
    g_gj_force = 0;
    throw;
  }
  g_gj_force = 0;
  std::vector<int> info = d2h(c, dinfo, batch);
  c.work.reset();
  for (int b = 0; b < batch; ++b)
    if (info[b]) throw Error(AIFMM_ESINGULAR_PIVOT, "singular matrix " + std::to_string(b));
  CAPI_END
}

int aifmm_debug_tri_root(double* A, int n, int m, int batch, double* M) {
  CAPI_BEGIN
  Ctx& c = ctx();
  AIFMM_REQUIRE(A && M && n >= 1 && m >= 1 && batch >= 1, AIFMM_EINVALID_ARG, "bad tri_root arguments");
  const int r = std::min(n, m);
  std::vector<TriRootReq> reqs;
  for (int b = 0; b < batch; ++b)
    reqs.push_back(TriRootReq{A + (size_t)b * n * m, n, n, m, M + (size_t)b * m * r, m});
  batched_tri_root(reqs, c.work, c.up, c.s, nullptr, 1 << 30);   // every route, TSQR included
  c.up.sync();
  c.work.reset();
  CAPI_END
}

int aifmm_matvec_build(double tol) {
  CAPI_BEGIN
  Ctx& c = ctx();
  AIFMM_REQUIRE(c.built, AIFMM_ESTATE, "matvec_build before build");
  AIFMM_REQUIRE(tol > 0.0 && tol < 1.0, AIFMM_EINVALID_ARG, "tol must lie in (0,1)");
  c.h2_built = false;
  c.bd_ready = false;
  c.bdpool.reset();
  c.h2pool.reset();
  build_nnca(c, c.hnn, tol / 100.0, c.h2pool);   // reading R18: eps_ACA = tol / 100
  c.h2_tol = tol;
  c.h2_built = true;
  CAPI_END
}

int aifmm_matvec(const double* X, double* Y, int nrhs) {
  CAPI_BEGIN
  Ctx& c = ctx();
  AIFMM_REQUIRE(c.h2_built, AIFMM_ESTATE, "matvec before matvec_build");
  AIFMM_REQUIRE(X && Y && nrhs >= 1, AIFMM_EINVALID_ARG, "bad matvec arguments");
  matvec_dev(c, X, Y, nrhs);
  CAPI_END
}

int aifmm_gmres(const double* b, double* x, int restart, double rtol, int maxit, int precond, int* iters,
                double* relres) {
  CAPI_BEGIN
  Ctx& c = ctx();
  AIFMM_REQUIRE(c.h2_built, AIFMM_ESTATE, "gmres before matvec_build");
  AIFMM_REQUIRE(precond >= 0 && precond <= 2, AIFMM_EINVALID_ARG, "precond must be 0, 1 or 2");
  AIFMM_REQUIRE(precond != 1 || c.factored, AIFMM_ESTATE, "AIFMM-preconditioned gmres before factor");
  AIFMM_REQUIRE(b && x && iters && relres && restart >= 1 && maxit >= 1 && rtol > 0.0, AIFMM_EINVALID_ARG,
                "bad gmres arguments");
  AIFMM_CUDA(cudaMemsetAsync(c.dflag, 0, sizeof(int), c.s));
  LAUNCH(finite_kernel, gsz(c.n), 256, 0, c.s, b, c.n, c.dflag);
  check_flag(c, AIFMM_ENONFINITE, "non-finite right-hand side");
  gmres_dev(c, b, x, restart, rtol, maxit, precond, iters, relres);
  CAPI_END
}

int aifmm_residual(const double* X, const double* B, int nrhs, const int64_t* rows, int64_t nrows, double* rel) {
  CAPI_BEGIN
  Ctx& c = ctx();
  AIFMM_REQUIRE(c.built, AIFMM_ESTATE, "residual before build");
  AIFMM_REQUIRE(X && B && rel && nrhs >= 1, AIFMM_EINVALID_ARG, "residual: null pointer or nrhs < 1");
  const long long nr = rows ? (long long)nrows : c.n;
  AIFMM_REQUIRE(nr >= 1, AIFMM_EINVALID_ARG, "residual: no rows");
  *rel = residual_dev(c, X, B, nrhs, rows, nr);
  CAPI_END
}

int aifmm_set_timing(int on) {
  CAPI_BEGIN
  ctx().timing = on != 0;
  CAPI_END
}

// ------------------------------------------------------------------ SURVEY §8(e) (dist.cuh)
int aifmm_dist_unique_id(void* out) {
  CAPI_BEGIN
  AIFMM_REQUIRE(out, AIFMM_EINVALID_ARG, "null pointer");
  Comm::unique_id(out);
  CAPI_END
}

int aifmm_dist_init(int rank, int world, const void* unique_id, int level_p) {
  CAPI_BEGIN
  AIFMM_REQUIRE(world >= 1 && rank >= 0 && rank < world && unique_id, AIFMM_EINVALID_ARG, "bad rank/world/unique id");
  Ctx& c = ctx();
  c.lp_user = level_p;
  if (world == 1 && !getenv("AIFMM_DIST_FORCE")) c.comm.finalize();
  else c.comm.init_nccl(rank, world, unique_id, c.s);
  CAPI_END
}

int aifmm_dist_init_local(int rank, int world, void* shared, int level_p) {
  CAPI_BEGIN
  Ctx& c = ctx();
  c.lp_user = level_p;
  c.comm.init_local(rank, world, shared);
  CAPI_END
}

int aifmm_dist_finalize(void) {
  CAPI_BEGIN
  ctx().comm.finalize();
  CAPI_END
}

int aifmm_get_owners(int level, int32_t* owner) {
  CAPI_BEGIN
  Ctx& c = ctx();
  AIFMM_REQUIRE(c.built, AIFMM_ESTATE, "owners before build");
  AIFMM_REQUIRE(owner && level >= 0 && level <= c.L, AIFMM_EINVALID_ARG, "bad level");
  const size_t nb = (size_t)1 << (c.d * level);
  const bool have = level < (int)c.owner.size() && c.owner[level].size() == nb && c.dist_level(level);
  for (size_t b = 0; b < nb; ++b) owner[b] = have ? c.owner[level][b] : -1;
  CAPI_END
}

}  // extern "C"
