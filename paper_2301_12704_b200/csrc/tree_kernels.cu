// tree_kernels.cu — G1/G2: uniform 2^d tree, Morton order, lists N(i)/IL(i), colouring (sm_100a).
//
// P:121-123 (§2.1) root hypercube and uniform refinement until leaves hold <= n_max points;
// P:198-230 (§2.2) strong admissibility with eta = sqrt(d) == Chebyshev index distance >= 2
// (reading R5); N(i) = same-level non-admissible boxes, IL(i) = children of N(P(i)) not in N(i).
// Integer outputs are bit-exact with oracle/tree.py (readings R1-R6 in DESIGN.md).
#include "common.cuh"

namespace aifmm {

constexpr int LMAX = 20;  // integer coordinates at level 20 (R3)

__device__ __forceinline__ long long morton_encode(const int* c, int d, int bits) {
  long long key = 0;
  for (int b = 0; b < bits; ++b)
    for (int a = 0; a < d; ++a) key |= (long long)((c[a] >> b) & 1) << (b * d + a);
  return key;
}
__device__ __forceinline__ void morton_decode(long long key, int d, int bits, int* c) {
  for (int a = 0; a < d; ++a) c[a] = 0;
  for (int b = 0; b < bits; ++b)
    for (int a = 0; a < d; ++a) c[a] |= (int)((key >> (b * d + a)) & 1) << b;
}

// ---- root box: per-axis min/max (two-stage), then g = c - h, two_h = 2h (R2)
__global__ void minmax_partial_kernel(const double* __restrict__ pts, long long n, int d,
                                      double* __restrict__ part, int* __restrict__ nonfinite) {
  __shared__ double slo[3][256], shi[3][256];
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    for (int a = 0; a < d; ++a) {
      double v = pts[i * d + a];
      if (!isfinite(v)) *nonfinite = 1;
      lo[a] = fmin(lo[a], v);
      hi[a] = fmax(hi[a], v);
    }
  }
  for (int a = 0; a < 3; ++a) { slo[a][threadIdx.x] = lo[a]; shi[a][threadIdx.x] = hi[a]; }
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s)
      for (int a = 0; a < 3; ++a) {
        slo[a][threadIdx.x] = fmin(slo[a][threadIdx.x], slo[a][threadIdx.x + s]);
        shi[a][threadIdx.x] = fmax(shi[a][threadIdx.x], shi[a][threadIdx.x + s]);
      }
    __syncthreads();
  }
  if (threadIdx.x == 0)
    for (int a = 0; a < 3; ++a) { part[blockIdx.x * 6 + a] = slo[a][0]; part[blockIdx.x * 6 + 3 + a] = shi[a][0]; }
}

// root[0..2] = g, root[3] = two_h
__global__ void root_kernel(const double* __restrict__ part, int nparts, int d, double* __restrict__ root) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double lo[3], hi[3];
  for (int a = 0; a < 3; ++a) { lo[a] = INFINITY; hi[a] = -INFINITY; }
  for (int p = 0; p < nparts; ++p)
    for (int a = 0; a < d; ++a) { lo[a] = fmin(lo[a], part[p * 6 + a]); hi[a] = fmax(hi[a], part[p * 6 + 3 + a]); }
  double h = 0.0;
  for (int a = 0; a < d; ++a) h = fmax(h, __dsub_rn(hi[a], lo[a]));
  h = h / 2.0;
  if (!(h > 0.0)) h = 9.5367431640625e-07;  // 2^-20, degenerate cloud
  for (int a = 0; a < d; ++a) {
    double c = __dadd_rn(lo[a], hi[a]) / 2.0;
    root[a] = __dsub_rn(c, h);
  }
  root[3] = 2.0 * h;
}

// integer coordinates at LMAX: k = clamp(floor(((p - g) / (2h)) * 2^LMAX)) (R3, IEEE RN, no FMA)
__global__ void coords_kernel(const double* __restrict__ pts, long long n, int d, const double* __restrict__ root,
                              int* __restrict__ kc) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    for (int a = 0; a < d; ++a) {
      double t = __ddiv_rn(__dsub_rn(pts[i * d + a], root[a]), root[3]);
      t = __dmul_rn(t, (double)(1 << LMAX));
      double f = floor(t);
      long long k = (long long)f;
      if (!(f >= 0.0)) k = 0;
      if (k > (1 << LMAX) - 1) k = (1 << LMAX) - 1;
      kc[i * d + a] = (int)k;
    }
  }
}

// leaf Morton id at level l
__global__ void keys_kernel(const int* __restrict__ kc, long long n, int d, int l, int* __restrict__ key) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    int c[3];
    for (int a = 0; a < d; ++a) c[a] = kc[i * d + a] >> (LMAX - l);
    key[i] = (int)morton_encode(c, d, l);
  }
}

__global__ void histogram_kernel(const int* __restrict__ key, long long n, int* __restrict__ cnt) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    atomicAdd(&cnt[key[i]], 1);
}

__global__ void max_int_kernel(const int* __restrict__ a, int n, int* __restrict__ out) {
  int v = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) v = max(v, a[i]);
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, v);
}

// exclusive scan of cnt[0..nb) into off[0..nb] (single CTA, chunked)
__global__ void scan_kernel(const int* __restrict__ cnt, int nb, long long* __restrict__ off) {
  __shared__ long long part[1024];
  const int t = threadIdx.x, nt = blockDim.x;
  const int chunk = (nb + nt - 1) / nt;
  const int b0 = min(nb, t * chunk), b1 = min(nb, b0 + chunk);
  long long s = 0;
  for (int b = b0; b < b1; ++b) s += cnt[b];
  part[t] = s;
  __syncthreads();
  if (t == 0) {
    long long acc = 0;
    for (int i = 0; i < nt; ++i) { long long v = part[i]; part[i] = acc; acc += v; }
    off[nb] = acc;
  }
  __syncthreads();
  long long acc = part[t];
  for (int b = b0; b < b1; ++b) { off[b] = acc; acc += cnt[b]; }
}

__global__ void scatter_kernel(const int* __restrict__ key, long long n, const long long* __restrict__ off,
                               int* __restrict__ cursor, int* __restrict__ perm) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    int k = key[i];
    int pos = atomicAdd(&cursor[k], 1);
    perm[off[k] + pos] = (int)i;
  }
}

// stable order inside each leaf: sort the leaf's segment of perm ascending (segments <= n_max)
__global__ void segsort_kernel(const long long* __restrict__ off, int nb, int* __restrict__ perm) {
  extern __shared__ int seg[];
  for (int b = blockIdx.x; b < nb; b += gridDim.x) {
    const long long a0 = off[b], a1 = off[b + 1];
    const int len = (int)(a1 - a0);
    if (len <= 1) continue;
    int p2 = 1;
    while (p2 < len) p2 <<= 1;
    for (int i = threadIdx.x; i < p2; i += blockDim.x) seg[i] = (i < len) ? perm[a0 + i] : 0x7fffffff;
    __syncthreads();
    for (int k = 2; k <= p2; k <<= 1)
      for (int j = k >> 1; j > 0; j >>= 1) {
        for (int i = threadIdx.x; i < p2; i += blockDim.x) {
          int ixj = i ^ j;
          if (ixj > i) {
            bool up = ((i & k) == 0);
            int a = seg[i], c = seg[ixj];
            if ((a > c) == up) { seg[i] = c; seg[ixj] = a; }
          }
        }
        __syncthreads();
      }
    for (int i = threadIdx.x; i < len; i += blockDim.x) perm[a0 + i] = seg[i];
    __syncthreads();
  }
}

__global__ void gather_points_kernel(const double* __restrict__ pts, const int* __restrict__ perm, long long n, int d,
                                     double* __restrict__ sorted) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    for (int a = 0; a < d; ++a) sorted[i * d + a] = pts[(long long)perm[i] * d + a];
}

// level-l offsets from leaf offsets: off_l[b] = off_L[b << (d (L - l))]
__global__ void level_offsets_kernel(const long long* __restrict__ offL, int shift, int nb_l,
                                     long long* __restrict__ offl) {
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b <= nb_l; b += gridDim.x * blockDim.x)
    offl[b] = offL[(long long)b << shift];
}

// lists at level l: near (cap 3^d) and IL (cap 6^d - 3^d), Morton-sorted, for non-empty boxes
__global__ void lists_kernel(const long long* __restrict__ offl, int l, int d, int ncap, int icap,
                             int* __restrict__ ncnt, int* __restrict__ nidx, int* __restrict__ icnt,
                             int* __restrict__ iidx) {
  const int nb = 1 << (d * l);
  const int side = 1 << l;
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += gridDim.x * blockDim.x) {
    int nn = 0, ni = 0;
    if (offl[b + 1] > offl[b]) {
      int c[3] = {0, 0, 0};
      morton_decode(b, d, l, c);
      int* N = nidx + (size_t)b * ncap;
      int* I = iidx + (size_t)b * icap;
      const int n3 = (d == 2) ? 9 : 27;
      for (int o = 0; o < n3; ++o) {
        int cc[3] = {0, 0, 0};
        bool in = true;
        int oo = o;
        for (int a = 0; a < d; ++a) { cc[a] = c[a] + (oo % 3) - 1; oo /= 3; in = in && cc[a] >= 0 && cc[a] < side; }
        if (!in) continue;
        int j = (int)morton_encode(cc, d, l);
        if (offl[j + 1] > offl[j]) N[nn++] = j;
      }
      int pc[3] = {c[0] >> 1, c[1] >> 1, c[2] >> 1};
      for (int o = 0; o < n3; ++o) {
        int pp[3] = {0, 0, 0};
        bool in = true;
        int oo = o;
        for (int a = 0; a < d; ++a) { pp[a] = pc[a] + (oo % 3) - 1; oo /= 3; in = in && pp[a] >= 0 && pp[a] < (side >> 1); }
        if (!in) continue;
        int pb = (int)morton_encode(pp, d, l - 1);
        for (int ch = 0; ch < (1 << d); ++ch) {
          int cb = (pb << d) | ch;
          if (!(offl[cb + 1] > offl[cb])) continue;
          int cq[3] = {0, 0, 0};
          morton_decode(cb, d, l, cq);
          int cheb = 0;
          for (int a = 0; a < d; ++a) cheb = max(cheb, abs(cq[a] - c[a]));
          if (cheb >= 2) I[ni++] = cb;
        }
      }
      // insertion sorts (Morton order)
      for (int i = 1; i < nn; ++i) { int v = N[i], j = i - 1; while (j >= 0 && N[j] > v) { N[j + 1] = N[j]; --j; } N[j + 1] = v; }
      for (int i = 1; i < ni; ++i) { int v = I[i], j = i - 1; while (j >= 0 && I[j] > v) { I[j + 1] = I[j]; --j; } I[j + 1] = v; }
    }
    ncnt[b] = nn;
    icnt[b] = ni;
  }
}

// greedy first-fit colouring in Morton order, conflict = N(i) \ {i} (R6); one thread per level
// greedy first-fit in Morton order (R6) is sequential by definition: one thread walks the boxes,
// the colours live in shared memory (byte per box) when they fit
__global__ void colour_kernel(const long long* __restrict__ offl, int nb, int ncap, const int* __restrict__ ncnt,
                              const int* __restrict__ nidx, int* __restrict__ col, int use_smem) {
  extern __shared__ signed char cs[];
  for (int b = threadIdx.x; b < nb; b += blockDim.x) {
    col[b] = -1;
    if (use_smem) cs[b] = -1;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  for (int b = 0; b < nb; ++b) {
    if (!(offl[b + 1] > offl[b])) continue;
    unsigned long long used = 0;
    for (int t = 0; t < ncnt[b]; ++t) {
      int j = nidx[(size_t)b * ncap + t];
      const int cj = use_smem ? cs[j] : col[j];
      if (j != b && cj >= 0 && cj < 64) used |= 1ull << cj;
    }
    int c = 0;
    while (used & (1ull << c)) ++c;
    if (use_smem) cs[b] = (signed char)c;
    col[b] = c;
  }
}

// ------------------------------------------------------------------------------ launchers
static int grid_for(long long n) { long long g = (n + 255) / 256; return (int)std::min<long long>(std::max<long long>(g, 1), 148 * 8); }

void tree_minmax(const double* pts, long long n, int d, double* part, int nparts, int* nonfinite, double* root,
                 cudaStream_t s) {
  LAUNCH(minmax_partial_kernel, nparts, 256, 0, s, pts, n, d, part, nonfinite);
  LAUNCH(root_kernel, 1, 1, 0, s, part, nparts, d, root);
}
void tree_coords(const double* pts, long long n, int d, const double* root, int* kc, cudaStream_t s) {
  LAUNCH(coords_kernel, grid_for(n), 256, 0, s, pts, n, d, root, kc);
}
void tree_keys(const int* kc, long long n, int d, int l, int* key, cudaStream_t s) {
  LAUNCH(keys_kernel, grid_for(n), 256, 0, s, kc, n, d, l, key);
}
void tree_hist(const int* key, long long n, int* cnt, cudaStream_t s) {
  LAUNCH(histogram_kernel, grid_for(n), 256, 0, s, key, n, cnt);
}
void tree_max(const int* a, int n, int* out, cudaStream_t s) {
  LAUNCH(max_int_kernel, grid_for(n), 256, 0, s, a, n, out);
}
void tree_scan(const int* cnt, int nb, long long* off, cudaStream_t s) { LAUNCH(scan_kernel, 1, 1024, 0, s, cnt, nb, off); }
void tree_scatter(const int* key, long long n, const long long* off, int* cursor, int* perm, cudaStream_t s) {
  LAUNCH(scatter_kernel, grid_for(n), 256, 0, s, key, n, off, cursor, perm);
}
void tree_segsort(const long long* off, int nb, int maxlen, int* perm, cudaStream_t s) {
  int p2 = 1;
  while (p2 < maxlen) p2 <<= 1;
  size_t smem = (size_t)p2 * sizeof(int);
  ensure_dyn_smem(segsort_kernel, smem);
  LAUNCH(segsort_kernel, std::min(nb, 148 * 16), 256, smem, s, off, nb, perm);
}
void tree_gather(const double* pts, const int* perm, long long n, int d, double* sorted, cudaStream_t s) {
  LAUNCH(gather_points_kernel, grid_for(n), 256, 0, s, pts, perm, n, d, sorted);
}
void tree_level_offsets(const long long* offL, int shift, int nb_l, long long* offl, cudaStream_t s) {
  LAUNCH(level_offsets_kernel, grid_for(nb_l + 1), 256, 0, s, offL, shift, nb_l, offl);
}
void tree_lists(const long long* offl, int l, int d, int ncap, int icap, int* ncnt, int* nidx, int* icnt, int* iidx,
                cudaStream_t s) {
  LAUNCH(lists_kernel, grid_for(1 << (d * l)), 256, 0, s, offl, l, d, ncap, icap, ncnt, nidx, icnt, iidx);
}
void tree_colour(const long long* offl, int nb, int ncap, const int* ncnt, const int* nidx, int* col, cudaStream_t s) {
  const int use_smem = nb <= 200 * 1024;
  if (use_smem) ensure_dyn_smem(colour_kernel, (size_t)nb);
  LAUNCH(colour_kernel, 1, 256, use_smem ? (size_t)nb : 0, s, offl, nb, ncap, ncnt, nidx, col, use_smem);
}

}  // namespace aifmm
