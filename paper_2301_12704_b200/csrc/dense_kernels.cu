// dense_kernels.cu — batched variable-size dense FP64 kernels of the AIFMM hot path (sm_100a).
//
//   gemm_tasks_kernel  : C = beta C + sum_t alpha_t op(A_t) op(B_t) on FP64 tensor cores
//                        (mma.sync m8n8k4 f64 -> SASS DMMA; tcgen05 has no f64 kind on sm_100a).
//                        Used for the Schur-complement updates (Table 4),
//                        the multipliers W = P_i^{-1} R_i, projections / redirections
//                         and the solve (Alg. 4).
//   gj_tasks_kernel    : Gauss-Jordan with partial pivoting (pivot inverse G = P_i^{-1}, the
//                        NNCA skeleton solve A(fp,sk)^{-1} A(fp,R) of P:361/P:365, top solve).
//   pqr_tasks_kernel   : column-pivoted Gram-Schmidt with truncation (the paper's RRQR).
//   keval_tasks_kernel : kernel-entry blocks A(rows, cols).
//   copy/norm kernels  : block assembly, level transition gathers, Frobenius norms.
#include <cooperative_groups.h>
#include <algorithm>
#include <cstdio>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace aifmm {

// ------------------------------------------------------------------------------ DMMA GEMM
__device__ __forceinline__ void dmma_884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool pred) {
  const unsigned saddr = (unsigned)__cvta_generic_to_shared(smem);
  const int sz = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(saddr), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Batched variable-size GEMM on FP64 tensor cores.  One CTA = one BM x BN tile of one task;
// the K loop runs over all terms of the task (deterministic order), operand tiles are staged
// global -> shared by cp.async through a GEMM_ST-stage ring (dynamic shared memory), each warp
// owns a 32 x 32 sub-tile (4 x 4 DMMA 8x8x4 fragments), alpha is applied to the A fragments.
constexpr int GEMM_ST = 2, GEMM_BK = 16;   // measured: 2 stages beat 3 and 4 (occupancy: 118 registers)
template <int BM, int BN>
constexpr size_t gemm_smem() { return sizeof(double) * (size_t)GEMM_ST * GEMM_BK * ((BM + 4) + (BN + 4)); }

template <int BM, int BN, int MINB = 1>
__global__ void __launch_bounds__(BM * BN / 32, MINB)
gemm_tasks_kernel(const GemmTask* __restrict__ tasks, const GemmTerm* __restrict__ terms,
                  const GemmTile* __restrict__ tiles) {
  constexpr int BK = GEMM_BK, ST = GEMM_ST;
  constexpr int NT = BM * BN / 32;
  constexpr int LDS_A = BM + 4;              // (BM+4) % 16 == 4 -> conflict-free fragment loads
  constexpr int LDS_B = BN + 4;
  extern __shared__ __align__(16) double gsm[];
  double* sA = gsm;                          // [ST][BK][LDS_A]
  double* sB = gsm + (size_t)ST * BK * LDS_A; // [ST][BK][LDS_B]
  __shared__ double s_alpha[ST];

  const GemmTile tile = tiles[blockIdx.x];
  const GemmTask tk = tasks[tile.task];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int WARPS_M = BM / 32;
  const int wm = (warp % WARPS_M) * 32, wn = (warp / WARPS_M) * 32;
  const int m0 = tile.m0, n0 = tile.n0;

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  auto next_term = [&](int t) {
    while (t < tk.term_end && terms[t].A == nullptr) ++t;
    return t;
  };
  int nk = 0;                                // number of (term, k0) tiles of this task
  bool has_add = false;                      // addition terms (A == nullptr: C += alpha B)
  for (int t = tk.term_begin; t < tk.term_end; ++t) {
    const GemmTerm tm = terms[t];
    if (tm.A) nk += (tm.K + BK - 1) / BK;
    else has_add = true;
  }
  int lt = next_term(tk.term_begin), lk = 0; // next tile to load
  auto load_next = [&](int st) {
    if (lt < tk.term_end) {
      const GemmTerm tm = terms[lt];
      double* a_s = sA + (size_t)st * BK * LDS_A;
      double* b_s = sB + (size_t)st * BK * LDS_B;
      for (int e = tid; e < BM * BK; e += NT) {
        int mm, kk;
        if (!tm.transA) { mm = e % BM; kk = e / BM; } else { kk = e % BK; mm = e / BK; }
        const int gm = m0 + mm, gk = lk + kk;
        const bool ok = gm < tk.M && gk < tm.K;
        const double* src = ok ? (tm.transA ? tm.A + (size_t)gm * tm.lda + gk : tm.A + (size_t)gk * tm.lda + gm) : tm.A;
        cp_async8(a_s + kk * LDS_A + mm, src, ok);
      }
      for (int e = tid; e < BN * BK; e += NT) {
        int nn, kk;
        if (!tm.transB) { kk = e % BK; nn = e / BK; } else { nn = e % BN; kk = e / BN; }
        const int gn = n0 + nn, gk = lk + kk;
        const bool ok = gn < tk.N && gk < tm.K;
        const double* src = ok ? (tm.transB ? tm.B + (size_t)gk * tm.ldb + gn : tm.B + (size_t)gn * tm.ldb + gk) : tm.B;
        cp_async8(b_s + kk * LDS_B + nn, src, ok);
      }
      if (tid == 0) s_alpha[st] = tm.alpha;
      lk += BK;
      if (lk >= tm.K) { lt = next_term(lt + 1); lk = 0; }
    }
    cp_async_commit();
  };
#pragma unroll
  for (int s = 0; s < ST - 1; ++s) load_next(s);
  for (int it = 0; it < nk; ++it) {
    load_next((it + ST - 1) % ST);
    cp_async_wait<ST - 1>();
    __syncthreads();
    const int st = it % ST;
    const double alpha = s_alpha[st];
    const double* a_s = sA + (size_t)st * BK * LDS_A;
    const double* b_s = sB + (size_t)st * BK * LDS_B;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = alpha * a_s[(kk + (lane & 3)) * LDS_A + wm + i * 8 + (lane >> 2)];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = b_s[(kk + (lane & 3)) * LDS_B + wn + j * 8 + (lane >> 2)];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma_884(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
    __syncthreads();
  }
  cp_async_wait<0>();
  // epilogue: C = beta*C + (acc + sum(addition terms)).  Every load (C, addition terms) is
  // issued before the first store: the compiler cannot prove that a store to C does not alias a
  // later load, and would otherwise expose one memory latency per element.
  // Done per 8-row group i (8 elements per thread) to bound the registers.
  const bool has_beta = tk.beta != 0.0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gm = m0 + wm + i * 8 + (lane >> 2);
    const bool okm = gm < tk.M;
    double cv[4][2];
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int gn = n0 + wn + j * 8 + (lane & 3) * 2 + e;
        cv[j][e] = (has_beta && okm && gn < tk.N) ? tk.C[(size_t)gn * tk.ldc + gm] : 0.0;
      }
    if (has_add) {
      for (int t = tk.term_begin; t < tk.term_end; ++t) {
        const GemmTerm tm = terms[t];
        if (tm.A != nullptr) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int gn = n0 + wn + j * 8 + (lane & 3) * 2 + e;
            if (okm && gn < tk.N)
              acc[i][j][e] += tm.alpha * (tm.transB ? tm.B[(size_t)gm * tm.ldb + gn] : tm.B[(size_t)gn * tm.ldb + gm]);
          }
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int gn = n0 + wn + j * 8 + (lane & 3) * 2 + e;
        if (okm && gn < tk.N)
          tk.C[(size_t)gn * tk.ldc + gm] = has_beta ? tk.beta * cv[j][e] + acc[i][j][e] : acc[i][j][e];
      }
  }
}

template __global__ void gemm_tasks_kernel<64, 64>(const GemmTask*, const GemmTerm*, const GemmTile*);
template __global__ void gemm_tasks_kernel<64, 64, 5>(const GemmTask*, const GemmTerm*, const GemmTile*);
template __global__ void gemm_tasks_kernel<64, 128, 2>(const GemmTask*, const GemmTerm*, const GemmTile*);
template __global__ void gemm_tasks_kernel<64, 64, 6>(const GemmTask*, const GemmTerm*, const GemmTile*);
template __global__ void gemm_tasks_kernel<32, 32>(const GemmTask*, const GemmTerm*, const GemmTile*);
template __global__ void gemm_tasks_kernel<64, 32>(const GemmTask*, const GemmTerm*, const GemmTile*);
template __global__ void gemm_tasks_kernel<32, 64>(const GemmTask*, const GemmTerm*, const GemmTile*);

// ------------------------------------------------------------------------------ block reductions
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    v = (lane < NT / 32) ? red[lane] : 0.0;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[0] = v;
  }
  __syncthreads();
  double r = red[0];
  __syncthreads();
  return r;
}

template <int NT>
__device__ __forceinline__ double block_max(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    v = (lane < NT / 32) ? red[lane] : -1.0;
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane == 0) red[0] = v;
  }
  __syncthreads();
  double r = red[0];
  __syncthreads();
  return r;
}

template <int NT>
__device__ __forceinline__ int block_min_int(int v, int* red) {
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    v = (lane < NT / 32) ? red[lane] : 0x7fffffff;
    for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane == 0) red[0] = v;
  }
  __syncthreads();
  int r = red[0];
  __syncthreads();
  return r;
}

// (sum, max) over the block in one shared-memory round
template <int NT>
__device__ __forceinline__ void block_sum_max(double s, double m, double* red, double* so, double* mo) {
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) { red[w] = s; red[16 + w] = m; }
  __syncthreads();
  double ts = 0.0, tm = -1.0;
  for (int q = 0; q < NT / 32; ++q) { ts += red[q]; tm = fmax(tm, red[16 + q]); }
  *so = ts;
  *mo = tm;
}

// (max |x|, lowest index attaining it) over the block in one shared-memory round
template <int NT>
__device__ __forceinline__ void block_argmax(double v, int idx, double* redv, int* redi, double* mx, int* at) {
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, v, o);
    const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
    if (ov > v || (ov == v && oi < idx)) { v = ov; idx = oi; }
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) { redv[w] = v; redi[w] = idx; }
  __syncthreads();
  double bv = redv[0];
  int bi = redi[0];
  for (int q = 1; q < NT / 32; ++q)
    if (redv[q] > bv || (redv[q] == bv && redi[q] < bi)) { bv = redv[q]; bi = redi[q]; }
  *mx = bv;
  *at = bi;
}

// ------------------------------------------------------------------------------ Gauss-Jordan
// Unblocked Gauss-Jordan with partial pivoting on an n x ncols column-major matrix M (ld).
// mode 0: [A | B] -> [I | A^{-1} B];  mode 1: in-place inverse of A (n x n).
// Returns the failing step + 1 (exact zero pivot) or 0.
constexpr int GJ_NT = 256;
__device__ int gj_device(double* M, int ld, int n, int nc, int mode, double* f, int* piv, double* red, int* redi) {
  const int tid = threadIdx.x;
  for (int k = 0; k < n; ++k) {
    double v = -1.0;
    for (int i = k + tid; i < n; i += GJ_NT) v = fmax(v, fabs(M[(size_t)k * ld + i]));
    const double mx = block_max<GJ_NT>(v, red);
    int cand = 0x7fffffff;
    for (int i = k + tid; i < n; i += GJ_NT)
      if (fabs(M[(size_t)k * ld + i]) == mx) { cand = i; break; }
    const int p = block_min_int<GJ_NT>(cand, redi);
    if (!(mx > 0.0)) return k + 1;
    if (tid == 0) piv[k] = p;
    const int jlo = (mode == 1) ? 0 : k;
    const int jhi = (mode == 1) ? n : nc;
    if (p != k)
      for (int j = jlo + tid; j < jhi; j += GJ_NT) {
        double a = M[(size_t)j * ld + k], b = M[(size_t)j * ld + p];
        M[(size_t)j * ld + k] = b;
        M[(size_t)j * ld + p] = a;
      }
    __syncthreads();
    const double d = 1.0 / M[(size_t)k * ld + k];
    for (int i = tid; i < n; i += GJ_NT) f[i] = M[(size_t)k * ld + i];
    __syncthreads();
    for (int j = jlo + tid; j < jhi; j += GJ_NT) {
      if (j == k) M[(size_t)j * ld + k] = (mode == 1) ? d : 1.0;
      else M[(size_t)j * ld + k] *= d;
    }
    __syncthreads();
    // rank-1 update, one warp per column (rows contiguous: no integer division per element)
    const int lane = tid & 31, warp = tid >> 5;
    for (int j = jlo + warp; j < jhi; j += GJ_NT / 32) {
      double* col = M + (size_t)j * ld;
      if (j == k) {
        for (int i = lane; i < n; i += 32)
          if (i != k) col[i] = (mode == 1) ? -f[i] * d : 0.0;
      } else {
        const double mk = col[k];
        for (int i = lane; i < n; i += 32)
          if (i != k) col[i] -= f[i] * mk;
      }
    }
    __syncthreads();
  }
  if (mode == 1) {
    for (int k = n - 1; k >= 0; --k) {
      const int p = piv[k];
      if (p != k)
        for (int i = tid; i < n; i += GJ_NT) {
          double a = M[(size_t)k * ld + i], b = M[(size_t)p * ld + i];
          M[(size_t)k * ld + i] = b;
          M[(size_t)p * ld + i] = a;
        }
      __syncthreads();
    }
  }
  return 0;
}

// small matrices: staged in shared memory (fast); smem = n*ncols + n doubles + n ints
__global__ void __launch_bounds__(GJ_NT) gj_small_kernel(const GJTask* __restrict__ tasks, int mode) {
  extern __shared__ double gsm[];
  __shared__ double red[32];
  __shared__ int redi[32];
  const GJTask tk = tasks[blockIdx.x];
  const int n = tk.n, nc = (mode == 1) ? n : tk.ncols;
  if (n == 0) { if (threadIdx.x == 0 && tk.info) *tk.info = 0; return; }
  double* M = gsm;
  double* f = M + (size_t)n * nc;
  int* piv = reinterpret_cast<int*>(f + n);
  for (int e = threadIdx.x; e < n * nc; e += GJ_NT) M[e] = tk.A[(size_t)(e / n) * tk.lda + (e % n)];
  __syncthreads();
  const int info = gj_device(M, n, n, nc, mode, f, piv, red, redi);
  if (info) { if (threadIdx.x == 0 && tk.info) *tk.info = info; return; }
  for (int e = threadIdx.x; e < n * nc; e += GJ_NT) tk.A[(size_t)(e / n) * tk.lda + (e % n)] = M[e];
  if (threadIdx.x == 0 && tk.info) *tk.info = 0;
}

// large augmented solves in global memory (NNCA skeleton solves that do not fit in smem)
__global__ void __launch_bounds__(GJ_NT) gj_global_kernel(const GJTask* __restrict__ tasks, int mode) {
  extern __shared__ double gsm[];
  __shared__ double red[32];
  __shared__ int redi[32];
  const GJTask tk = tasks[blockIdx.x];
  const int n = tk.n;
  double* f = gsm;
  int* piv = reinterpret_cast<int*>(f + n);
  const int info = gj_device(tk.A, tk.lda, n, (mode == 1) ? n : tk.ncols, mode, f, piv, red, redi);
  if (threadIdx.x == 0 && tk.info) *tk.info = info;
}

// ---- blocked in-place Gauss-Jordan inverse for larger matrices (pivot inverses at upper
// levels, the top system).  Per panel J = [j, j+nbw): panel LU with partial pivoting picks
// the pivots (identical to GJ's), rows are swapped, D = A[J,J] is inverted from its LU,
// A[J,:] <- D^{-1} A[J,:], A[R,J] <- 0, B = old A[R,J]; then a DMMA GEMM does A[R,:] -= B A[J,:].
constexpr int GJB = 32;
constexpr int GJ_CPW = 4;   // columns per warp in flight in the row-interchange / D^{-1} pass
struct GJBTask {
  double* A;
  int lda, n;
  double* PW;    // workspace n x GJB
  double* Bws;   // workspace n x GJB (ld n)
  int* piv;      // n
  int* info;
};

// One panel step of the blocked Gauss-Jordan inverse for one matrix (the whole CTA); returns
// false (info set) on an exactly singular panel.  Used by gj_panel_kernel (one launch per panel,
// DMMA update by a separate GEMM launch) and gj_fused_kernel (all panels and their updates in
// one CTA).
__device__ __forceinline__ bool gj_panel_dev(const GJBTask& tk, int j, double* gj_pw_smem, int smem_elems) {
  const int n = tk.n;
  const int nbw = min(GJB, n - j), rows = n - j, ld = tk.lda;
  double* A = tk.A;
  double* PW = (rows * nbw <= smem_elems) ? gj_pw_smem : tk.PW;   // panel LU in smem when it fits
  __shared__ double red[32];
  __shared__ int redi[32];
  __shared__ double Li[GJB][GJB + 1], Ui[GJB][GJB + 1], Di[GJB][GJB + 1];
  __shared__ double ycol[GJ_NT / 32][GJB];
  __shared__ int prow_dst[2 * GJB], prow_src[2 * GJB];
  __shared__ int prow_cnt;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int c = warp; c < nbw; c += GJ_NT / 32)
    for (int r = lane; r < rows; r += 32) PW[(size_t)c * rows + r] = A[(size_t)(j + c) * ld + j + r];
  __syncthreads();
  for (int c = 0; c < nbw; ++c) {
    // pivot: largest |entry|, lowest row among equal ones (same rule as before, one reduction)
    double v = -1.0;
    int vi = 0x7fffffff;
    for (int r = c + tid; r < rows; r += GJ_NT) {
      const double a = fabs(PW[(size_t)c * rows + r]);
      if (a > v) { v = a; vi = r; }
    }
    double mx;
    int p;
    block_argmax<GJ_NT>(v, vi, red, redi, &mx, &p);
    if (!(mx > 0.0)) {
      if (tid == 0) *tk.info = j + c + 1;
      return false;
    }
    if (tid == 0) tk.piv[j + c] = j + p;
    if (p != c)
      for (int cc = tid; cc < nbw; cc += GJ_NT) {
        double a = PW[(size_t)cc * rows + c], b = PW[(size_t)cc * rows + p];
        PW[(size_t)cc * rows + c] = b;
        PW[(size_t)cc * rows + p] = a;
      }
    __syncthreads();
    const double dinv = 1.0 / PW[(size_t)c * rows + c];
    for (int r = c + 1 + tid; r < rows; r += GJ_NT) PW[(size_t)c * rows + r] *= dinv;
    __syncthreads();
    // rank-1 update of the panel: one warp per column, rows coalesced
    for (int cc = c + 1 + warp; cc < nbw; cc += GJ_NT / 32) {
      double* y = PW + (size_t)cc * rows;
      const double f = y[c];
      const double* x = PW + (size_t)c * rows;
      for (int r = c + 1 + lane; r < rows; r += 32) y[r] -= x[r] * f;
    }
    __syncthreads();
  }
  __syncthreads();
  __shared__ int pv[GJB];
  if (tid < nbw) pv[tid] = tk.piv[j + tid];
  // D^{-1} = U11^{-1} L11^{-1} from the panel LU (unit lower L11, upper U11)
  for (int e = tid; e < GJB * GJB; e += GJ_NT) {
    const int r = e % GJB, c = e / GJB;
    Li[r][c] = 0.0;
    Ui[r][c] = 0.0;
  }
  __syncthreads();
  if (warp == 0) {
    // column `lane` of L^{-1}: forward substitution
    if (lane < nbw) {
      for (int r = 0; r < nbw; ++r) {
        double s = (r == lane) ? 1.0 : 0.0;
        for (int t = lane; t < r; ++t) s -= PW[(size_t)t * rows + r] * Li[t][lane];
        Li[r][lane] = (r < lane) ? 0.0 : s;
      }
    }
  } else if (warp == 1) {
    // column `lane` of U^{-1}: back substitution
    if (lane < nbw) {
      for (int r = nbw - 1; r >= 0; --r) {
        double s = (r == lane) ? 1.0 : 0.0;
        for (int t = r + 1; t <= lane; ++t) s -= PW[(size_t)t * rows + r] * Ui[t][lane];
        Ui[r][lane] = (r > lane) ? 0.0 : s / PW[(size_t)r * rows + r];
      }
    }
  } else if (warp == 2 && lane == 0) {
    // the panel's row interchanges (j + c <-> pv[c], in order) as one permutation of the affected
    // rows: rows J first (dst j + t), then the pivot rows outside J; src = the old row that ends
    // up in dst
    int cnt = nbw;
    for (int t = 0; t < nbw; ++t) { prow_dst[t] = j + t; prow_src[t] = j + t; }
    for (int c = 0; c < nbw; ++c) {
      const int p = pv[c];
      if (p == j + c) continue;
      int ip = -1;
      for (int q = 0; q < cnt; ++q)
        if (prow_dst[q] == p) { ip = q; break; }
      if (ip < 0) { ip = cnt++; prow_dst[ip] = p; prow_src[ip] = p; }
      const int tmp = prow_src[c];
      prow_src[c] = prow_src[ip];
      prow_src[ip] = tmp;
    }
    prow_cnt = cnt;
  }
  __syncthreads();
  for (int e = tid; e < nbw * nbw; e += GJ_NT) {
    const int r = e % nbw, c = e / nbw;
    double s = 0.0;
    for (int t = 0; t < nbw; ++t) s += Ui[r][t] * Li[t][c];
    Di[r][c] = s;
  }
  __syncthreads();
  // every column: the interchanges in one gather / scatter of the affected rows (one memory round
  // trip instead of one per interchange); outside J also A[J, c] <- D^{-1} A[J, c].  A warp takes
  // GJ_CPW columns at a time (their loads in flight together).
  const int pc = prow_cnt;
  const int sA0 = (lane < pc) ? prow_src[lane] : 0, dA0 = (lane < pc) ? prow_dst[lane] : 0;
  const int sA1 = (lane + 32 < pc) ? prow_src[lane + 32] : 0, dA1 = (lane + 32 < pc) ? prow_dst[lane + 32] : 0;
  for (int col0 = warp * GJ_CPW; col0 < n; col0 += GJ_NT / 32 * GJ_CPW) {
    double v0[GJ_CPW], v1[GJ_CPW];
#pragma unroll
    for (int u = 0; u < GJ_CPW; ++u) {
      const int col = col0 + u;
      v0[u] = (col < n && lane < pc) ? A[(size_t)col * ld + sA0] : 0.0;
      v1[u] = (col < n && lane + 32 < pc) ? A[(size_t)col * ld + sA1] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < GJ_CPW; ++u) {
      const int col = col0 + u;
      if (col >= n) break;
      double* ac = A + (size_t)col * ld;
      // entries 0..nbw-1 (lanes < nbw of v0) land in rows J; the rest are outside pivot rows
      if (lane >= nbw && lane < pc) ac[dA0] = v0[u];
      if (lane + 32 < pc) ac[dA1] = v1[u];
      if (col >= j && col < j + nbw) {
        if (lane < nbw) ac[j + lane] = v0[u];
      } else {
        if (lane < nbw) ycol[warp][lane] = v0[u];
        __syncwarp();
        if (lane < nbw) {
          double s = 0.0;
          for (int t = 0; t < nbw; ++t) s += Di[lane][t] * ycol[warp][t];
          ac[j + lane] = s;
        }
        __syncwarp();
      }
    }
  }
  __syncthreads();
  // B = A[:, J] with rows J zeroed, A[R, J] = 0, A[J, J] = D^{-1}
  for (int c = warp; c < nbw; c += GJ_NT / 32)
    for (int r = lane; r < n; r += 32) {
      const bool inJ = (r >= j && r < j + nbw);
      tk.Bws[(size_t)c * n + r] = inJ ? 0.0 : A[(size_t)(j + c) * ld + r];
      A[(size_t)(j + c) * ld + r] = inJ ? Di[r - j][c] : 0.0;
    }
  return true;
}

__global__ void __launch_bounds__(GJ_NT) gj_panel_kernel(const GJBTask* __restrict__ tasks, int j, int smem_elems) {
  extern __shared__ double gj_pw_smem[];
  const GJBTask tk = tasks[blockIdx.x];
  if (j >= tk.n) return;
  if (*tk.info) return;
  gj_panel_dev(tk, j, gj_pw_smem, smem_elems);
}

// Fused blocked Gauss-Jordan inverse: one CTA per matrix runs every panel step and its rank-nbw
// update A <- A - B A[J, :] (B = Bws: the panel's old column block with rows J zeroed) on the FP64
// tensor cores (DMMA 8x8x4), then the column unscrambling -- one launch for the whole batch
// instead of 2 launches per 32 columns.  The update covers every row: rows J of B are exact
// zeros, so those rows are rewritten with their own values (C + (+-0) = C) and the arithmetic of
// every other entry is the separate GEMM launch's (same DMMA k order, C + acc with beta = 1):
// the result is bitwise that of the gj_panel_kernel + gemm_tasks_kernel path.
constexpr int GJF_TM = 64, GJF_TN = 128, GJF_LA = GJF_TM + 4, GJF_LB = GJF_TN + 4;
constexpr int GJF_TILE_DOUBLES = GJB * (GJF_LA + GJF_LB);
__device__ __forceinline__ void gj_fused_update(const GJBTask& tk, int j, int nbw, double* sm) {
  const int n = tk.n, lda = tk.lda;
  double* A = tk.A;
  const double* Bw = tk.Bws;
  double* sA = sm;                       // [GJB][GJF_LA]: sA[k][m] = -B[m0 + m][k]
  double* sB = sm + GJB * GJF_LA;        // [GJB][GJF_LB]: sB[k][c] = A[j + k][n0 + c]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 32;
  for (int m0 = 0; m0 < n; m0 += GJF_TM) {
    for (int e = tid; e < GJB * GJF_TM; e += GJ_NT) {
      const int mm = e % GJF_TM, kk = e / GJF_TM;
      const int gm = m0 + mm;
      sA[kk * GJF_LA + mm] = (gm < n && kk < nbw) ? -Bw[(size_t)kk * n + gm] : 0.0;
    }
    for (int n0 = 0; n0 < n; n0 += GJF_TN) {
      for (int e = tid; e < GJB * GJF_TN; e += GJ_NT) {
        const int kk = e % GJB, nn = e / GJB;
        const int gn = n0 + nn;
        sB[kk * GJF_LB + nn] = (gn < n && kk < nbw) ? A[(size_t)gn * lda + j + kk] : 0.0;
      }
      __syncthreads();
      double acc[4][4][2];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[i][q][0] = acc[i][q][1] = 0.0;
#pragma unroll
      for (int kk = 0; kk < GJB; kk += 4) {
        double a[4], b[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = sA[(kk + (lane & 3)) * GJF_LA + wm + i * 8 + (lane >> 2)];
#pragma unroll
        for (int q = 0; q < 4; ++q) b[q] = sB[(kk + (lane & 3)) * GJF_LB + wn + q * 8 + (lane >> 2)];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int q = 0; q < 4; ++q) dmma_884(acc[i][q][0], acc[i][q][1], a[i], b[q]);
      }
      // epilogue C = 1.0 * C + acc, loads issued before stores per 8-row group
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int gm = m0 + wm + i * 8 + (lane >> 2);
        const bool okm = gm < n;
        double cv[4][2];
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int gn = n0 + wn + q * 8 + (lane & 3) * 2 + e;
            cv[q][e] = (okm && gn < n) ? A[(size_t)gn * lda + gm] : 0.0;
          }
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int gn = n0 + wn + q * 8 + (lane & 3) * 2 + e;
            if (okm && gn < n) A[(size_t)gn * lda + gm] = 1.0 * cv[q][e] + acc[i][q][e];
          }
      }
      __syncthreads();
    }
  }
}

__global__ void __launch_bounds__(GJ_NT, 2) gj_fused_kernel(const GJBTask* __restrict__ tasks, int smem_elems) {
  extern __shared__ __align__(16) double gjf_smem[];
  const GJBTask tk = tasks[blockIdx.x];
  const int n = tk.n;
  if (*tk.info) return;
  for (int j = 0; j < n; j += GJB) {
    if (!gj_panel_dev(tk, j, gjf_smem, smem_elems)) return;
    __syncthreads();
    gj_fused_update(tk, j, min(GJB, n - j), gjf_smem);
  }
  // column interchanges in reverse pivot order (each thread owns rows)
  __syncthreads();
  double* A = tk.A;
  for (int i = threadIdx.x; i < n; i += GJ_NT)
    for (int k = n - 1; k >= 0; --k) {
      const int p = tk.piv[k];
      if (p != k) {
        const double a = A[(size_t)k * tk.lda + i];
        A[(size_t)k * tk.lda + i] = A[(size_t)p * tk.lda + i];
        A[(size_t)p * tk.lda + i] = a;
      }
    }
}

// Cluster variant of the Gauss-Jordan panel for few large matrices (the top system, upper-level
// pivots): the GJC CTAs of a cluster own contiguous row slices of the panel in shared memory.
// Per column one cluster barrier: every CTA publishes its local pivot candidate (value, row and
// the whole candidate row) and, if it owns row c, row c; afterwards every CTA knows the pivot row
// and the owner of the pivot row swaps in the old row c.  Same pivot rule as gj_panel_kernel
// (largest |entry|, lowest row on ties).  The interchanges of the full rows, D^{-1} and the
// B / A[J, :] writes are split over the cluster as well.
struct GjcShared {
  double v[2];
  int idx[2];
  double cand[2][GJB];   // the candidate row of this CTA
  double rowc[2][GJB];   // row c, if this CTA owns it
  double D[GJB][GJB + 1];
};
template <int GJC>
__global__ void __cluster_dims__(GJC, 1, 1) __launch_bounds__(GJ_NT)
gj_panel_cluster_kernel(const GJBTask* __restrict__ tasks, int j, int cap_rows) {
  extern __shared__ double gjc_p[];      // own panel rows: cnt x GJB, row-major (ld GJB + 1)
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  const GJBTask tk = tasks[blockIdx.x / GJC];
  const int n = tk.n;
  if (j >= n) return;                    // uniform over the cluster
  if (*tk.info) return;
  const int nbw = min(GJB, n - j), rows = n - j, ld = tk.lda;
  const int chunk = (rows + GJC - 1) / GJC;
  const int lo = min(rows, rank * chunk), hi = min(rows, lo + chunk), cnt = hi - lo;
  constexpr int LP = GJB + 1;
  double* P = gjc_p;
  __shared__ GjcShared sh;
  __shared__ double red[32];
  __shared__ int redi[32];
  __shared__ double prow[GJB];
  __shared__ double s_gm;
  __shared__ int s_gp;
  __shared__ double Li[GJB][GJB + 1], Ui[GJB][GJB + 1];
  __shared__ int pv[GJB];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* A = tk.A;
  for (int c = warp; c < nbw; c += GJ_NT / 32)
    for (int r = lane; r < cnt; r += 32) P[r * LP + c] = A[(size_t)(j + c) * ld + j + lo + r];
  __syncthreads();
  int ph = 0;
  for (int c = 0; c < nbw; ++c) {
    // local candidate: largest |P[r][c]| over own rows r >= c, lowest row on ties
    double v = -1.0;
    int vi = 0x7fffffff;
    for (int r = max(c - lo, 0) + tid; r < cnt; r += GJ_NT) {
      const double a = fabs(P[r * LP + c]);
      if (a > v) { v = a; vi = lo + r; }
    }
    double mx;
    int p;
    block_argmax<GJ_NT>(v, vi, red, redi, &mx, &p);
    if (tid == 0) { sh.v[ph] = mx; sh.idx[ph] = p; }
    if (p >= lo && p < hi)
      for (int cc = tid; cc < nbw; cc += GJ_NT) sh.cand[ph][cc] = P[(p - lo) * LP + cc];
    if (c >= lo && c < hi)
      for (int cc = tid; cc < nbw; cc += GJ_NT) sh.rowc[ph][cc] = P[(c - lo) * LP + cc];
    cl.sync();
    // global pivot: lanes 0..GJC-1 of warp 0 read the CTAs' candidates in parallel (one round
    // of DSMEM loads), a shuffle argmax picks (largest, lowest row), warp 0 fetches the pivot row
    if (warp == 0) {
      double ov = -1.0;
      int oi = 0x7fffffff;
      if (lane < GJC) {
        const GjcShared* o = cl.map_shared_rank(&sh, lane);
        ov = o->v[ph];
        oi = o->idx[ph];
      }
      int oq = lane;
      for (int off = GJC / 2; off > 0; off >>= 1) {   // GJC lanes
        const double v2 = __shfl_xor_sync(0xffffffffu, ov, off);
        const int i2 = __shfl_xor_sync(0xffffffffu, oi, off);
        const int q2 = __shfl_xor_sync(0xffffffffu, oq, off);
        if (v2 > ov || (v2 == ov && i2 < oi)) { ov = v2; oi = i2; oq = q2; }
      }
      ov = __shfl_sync(0xffffffffu, ov, 0);
      oi = __shfl_sync(0xffffffffu, oi, 0);
      oq = __shfl_sync(0xffffffffu, oq, 0);
      if (lane == 0) { s_gm = ov; s_gp = oi; }
      if (ov > 0.0 && lane < nbw) prow[lane] = cl.map_shared_rank(&sh, oq)->cand[ph][lane];
    }
    __syncthreads();
    const double gm = s_gm;
    const int gp = s_gp;
    if (!(gm > 0.0)) {
      if (rank == 0 && tid == 0) *tk.info = j + c + 1;
      cl.sync();
      return;
    }
    const int oc = min(GJC - 1, c / chunk);   // owner of row c
    if (rank == 0 && tid == 0) tk.piv[j + c] = j + gp;
    // the owner of the pivot row receives old row c
    if (gp != c && gp >= lo && gp < hi) {
      const GjcShared* co = cl.map_shared_rank(&sh, oc);
      for (int cc = tid; cc < nbw; cc += GJ_NT) P[(gp - lo) * LP + cc] = co->rowc[ph][cc];
    }
    __syncthreads();
    if (c >= lo && c < hi)
      for (int cc = tid; cc < nbw; cc += GJ_NT) P[(c - lo) * LP + cc] = prow[cc];
    // scale the column below the diagonal and update the trailing panel columns (own rows)
    const double dinv = 1.0 / prow[c];
    for (int r = max(c + 1 - lo, 0) + tid; r < cnt; r += GJ_NT) {
      double* pr = P + r * LP;
      const double l = pr[c] * dinv;
      pr[c] = l;
      for (int cc = c + 1; cc < nbw; ++cc) pr[cc] -= l * prow[cc];
    }
    __syncthreads();
    ph ^= 1;
  }
  // panel LU back to PW (rows relative to j, ld rows) for D
  for (int c = warp; c < nbw; c += GJ_NT / 32)
    for (int r = lane; r < cnt; r += 32) tk.PW[(size_t)c * rows + lo + r] = P[r * LP + c];
  cl.sync();
  if (tid < nbw) pv[tid] = tk.piv[j + tid];
  // interchanges of the full rows: columns split over the cluster
  const int cw = (n + GJC - 1) / GJC, c0 = min(n, rank * cw), c1 = min(n, c0 + cw);
  __syncthreads();
  for (int col = c0 + tid; col < c1; col += GJ_NT) {
    double* ac = A + (size_t)col * ld;
    for (int c = 0; c < nbw; ++c) {
      const int p = pv[c];
      if (p != j + c) {
        const double a = ac[j + c];
        ac[j + c] = ac[p];
        ac[p] = a;
      }
    }
  }
  // D^{-1} = U11^{-1} L11^{-1} (rank 0), shared through DSMEM
  const double* PW = tk.PW;
  if (rank == 0) {
    for (int e = tid; e < GJB * GJB; e += GJ_NT) { Li[e % GJB][e / GJB] = 0.0; Ui[e % GJB][e / GJB] = 0.0; }
    __syncthreads();
    if (warp == 0) {
      if (lane < nbw)
        for (int r = 0; r < nbw; ++r) {
          double s = (r == lane) ? 1.0 : 0.0;
          for (int t = lane; t < r; ++t) s -= PW[(size_t)t * rows + r] * Li[t][lane];
          Li[r][lane] = (r < lane) ? 0.0 : s;
        }
    } else if (warp == 1) {
      if (lane < nbw)
        for (int r = nbw - 1; r >= 0; --r) {
          double s = (r == lane) ? 1.0 : 0.0;
          for (int t = r + 1; t <= lane; ++t) s -= PW[(size_t)t * rows + r] * Ui[t][lane];
          Ui[r][lane] = (r > lane) ? 0.0 : s / PW[(size_t)r * rows + r];
        }
    }
    __syncthreads();
    for (int e = tid; e < nbw * nbw; e += GJ_NT) {
      const int r = e % nbw, c = e / nbw;
      double s = 0.0;
      for (int t = 0; t < nbw; ++t) s += Ui[r][t] * Li[t][c];
      sh.D[r][c] = s;
    }
  }
  cl.sync();   // row interchanges done everywhere, D published
  const GjcShared* d0 = cl.map_shared_rank(&sh, 0);
  for (int e = tid; e < nbw * nbw; e += GJ_NT) Li[e % nbw][e / nbw] = d0->D[e % nbw][e / nbw];   // Li := D
  __syncthreads();
  // B = A[:, J] with rows J zeroed, A[R, J] = 0, A[J, J] = D^{-1}: rows split over the cluster
  const int rw2 = (n + GJC - 1) / GJC, r0 = min(n, rank * rw2), r1 = min(n, r0 + rw2);
  for (int c = warp; c < nbw; c += GJ_NT / 32)
    for (int r = r0 + lane; r < r1; r += 32) {
      const bool inJ = (r >= j && r < j + nbw);
      tk.Bws[(size_t)c * n + r] = inJ ? 0.0 : A[(size_t)(j + c) * ld + r];
      A[(size_t)(j + c) * ld + r] = inJ ? Li[r - j][c] : 0.0;
    }
  // A[J, col] <- D^{-1} A[J, col] for columns outside J: columns split over the cluster
  __shared__ double ycol[GJ_NT / 32][GJB];
  for (int col = c0 + warp; col < c1; col += GJ_NT / 32) {
    if (col >= j && col < j + nbw) continue;
    if (lane < nbw) ycol[warp][lane] = A[(size_t)col * ld + j + lane];
    __syncwarp();
    if (lane < nbw) {
      double s = 0.0;
      for (int t = 0; t < nbw; ++t) s += Li[lane][t] * ycol[warp][t];
      A[(size_t)col * ld + j + lane] = s;
    }
    __syncwarp();
  }
  cl.sync();   // keep the cluster's shared memory alive until every CTA has read rank 0's D
}

// column interchanges in reverse pivot order; each thread owns one row (accesses over the
// threads of a warp are consecutive rows: coalesced), blockIdx.y splits the rows
__global__ void gj_unscramble_kernel(const GJBTask* __restrict__ tasks) {
  const GJBTask tk = tasks[blockIdx.x];
  if (*tk.info) return;
  const int i = blockIdx.y * blockDim.x + threadIdx.x;
  if (i >= tk.n) return;
  double* A = tk.A;
  for (int k = tk.n - 1; k >= 0; --k) {
    const int p = tk.piv[k];
    if (p != k) {
      const double a = A[(size_t)k * tk.lda + i];
      A[(size_t)k * tk.lda + i] = A[(size_t)p * tk.lda + i];
      A[(size_t)p * tk.lda + i] = a;
    }
  }
}

// ------------------------------------------------------------------------------ Cholesky
// Batched Cholesky G = R^T R (R upper) and the triangular inverse R^{-1}, for CholeskyQR2
// orthonormalisation of the NNCA bases (reading R13: any orthonormal basis of the same range
// gives the same exact change of variables).  One CTA per matrix, in shared memory up to
// CHOL_SMEM_MAX, else in global memory (in place).  info = 1 + step of a non-positive pivot.
constexpr int CHOL_NT = 256;
// Lower Cholesky G = L L^T in place (column-major, ld), column oriented: column j is scaled,
// then every trailing column c > j is updated along its contiguous rows i >= c (one warp per
// column, lanes over rows: coalesced).  Returns 0 or 1 + the step of a non-positive pivot.
__device__ int chol_lower_device(double* S, int ld, int k) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int j = 0; j < k; ++j) {
    const double piv = S[(size_t)j * ld + j];
    if (!(piv > 0.0)) return j + 1;                 // uniform: every thread read the same value
    const double d = sqrt(piv);
    double* cj = S + (size_t)j * ld;
    __syncthreads();
    for (int i = j + 1 + tid; i < k; i += CHOL_NT) cj[i] /= d;
    if (tid == 0) cj[j] = d;
    __syncthreads();
    for (int c = j + 1 + warp; c < k; c += CHOL_NT / 32) {
      const double lc = cj[c];
      double* cc = S + (size_t)c * ld;
      for (int i = c + lane; i < k; i += 32) cc[i] -= cj[i] * lc;
    }
    __syncthreads();
  }
  return 0;
}
// In-place inverse X = L^{-1} of a lower-triangular L (column-major), dtrti2 order: for
// j = k-1 .. 0, X(j+1:, j) = -X(j,j) X(j+1:, j+1:) L(j+1:, j); threads over the rows i read
// X(i, l) for consecutive i at fixed l (coalesced).  tmp: k doubles.
__device__ void trtri_lower_device(double* S, int ld, int k, double* tmp) {
  const int tid = threadIdx.x;
  for (int j = k - 1; j >= 0; --j) {
    const double ajj = 1.0 / S[(size_t)j * ld + j];
    for (int l = j + 1 + tid; l < k; l += CHOL_NT) tmp[l] = S[(size_t)j * ld + l];
    __syncthreads();
    for (int i = j + 1 + tid; i < k; i += CHOL_NT) {
      double acc = 0.0;
      for (int l = j + 1; l <= i; ++l) acc += S[(size_t)l * ld + i] * tmp[l];
      S[(size_t)j * ld + i] = -ajj * acc;
    }
    __syncthreads();
    if (tid == 0) S[(size_t)j * ld + j] = ajj;
    __syncthreads();
  }
}
// Batched Cholesky G = R^T R (R = L^T upper) and R^{-1} = (L^{-1})^T, for CholeskyQR2 of the
// NNCA bases (reading R13) and the null-space basis of R31.  One CTA per matrix, in shared
// memory up to CHOL_SMEM_MAX, else in global memory (Rinv's storage, in place).
constexpr int CHOL_SMEM_MAX = 160;
__global__ void __launch_bounds__(CHOL_NT) chol_inv_kernel(const CholTask* __restrict__ tasks, int smem_doubles) {
  extern __shared__ double csm[];
  const CholTask tk = tasks[blockIdx.x];
  const int k = tk.k;
  if (k == 0) { if (threadIdx.x == 0) *tk.info = 0; return; }
  const bool smem = (long long)k * (k + 1) <= smem_doubles;
  double* S = smem ? csm : tk.Rinv;
  double* tmp = smem ? csm + (size_t)k * k : csm;     // k doubles
  for (int c = 0; c < k; ++c)
    for (int r = threadIdx.x; r < k; r += CHOL_NT) S[(size_t)c * k + r] = tk.G[(size_t)c * k + r];
  __syncthreads();
  const int info = chol_lower_device(S, k, k);
  if (threadIdx.x == 0) *tk.info = info;
  if (info) return;
  // R = L^T (upper; zero below the diagonal)
  for (int c = 0; c < k; ++c)
    for (int r = threadIdx.x; r < k; r += CHOL_NT) tk.R[(size_t)c * k + r] = (r <= c) ? S[(size_t)r * k + c] : 0.0;
  __syncthreads();
  trtri_lower_device(S, k, k, tmp);
  // R^{-1} = X^T (upper)
  if (smem) {
    for (int c = 0; c < k; ++c)
      for (int r = threadIdx.x; r < k; r += CHOL_NT) tk.Rinv[(size_t)c * k + r] = (r <= c) ? S[(size_t)r * k + c] : 0.0;
  } else {
    // in place: the strict upper part is written from the lower part (disjoint), then zeroed below
    for (int c = 1; c < k; ++c)
      for (int r = threadIdx.x; r < c; r += CHOL_NT) S[(size_t)c * k + r] = S[(size_t)r * k + c];
    __syncthreads();
    for (int c = 0; c < k; ++c)
      for (int r = c + 1 + threadIdx.x; r < k; r += CHOL_NT) S[(size_t)c * k + r] = 0.0;
  }
}
void launch_chol_inv(const CholTask* t, int ntasks, int kmax, cudaStream_t s) {
  const int kk = std::min(kmax, CHOL_SMEM_MAX);
  const int nd = std::max(kk * (kk + 1), kmax);   // global-path tasks need k doubles of smem temp
  ensure_dyn_smem(chol_inv_kernel, (size_t)nd * sizeof(double));
  LAUNCH(chol_inv_kernel, ntasks, CHOL_NT, (size_t)nd * sizeof(double), s, t, nd);
}

// ------------------------------------------------------------------------------ pivoted QR
constexpr int PQR_NT = 256;
constexpr double TIE = 1e-10;  // reading R7 (same rule as oracle/linalg.py: pick)

__global__ void __launch_bounds__(PQR_NT) pqr_tasks_kernel(const PqrTask* __restrict__ tasks) {
  extern __shared__ double pq_smem[];
  const PqrTask tk = tasks[blockIdx.x];
  const int m = tk.m, nc = tk.ncols, ldw = tk.ldw, ldq = tk.ldq;
  double* norms = pq_smem;          // nc
  double* w = norms + nc;           // m
  double* coef = w + m;             // k0 + tmax
  __shared__ double red[32];
  __shared__ int redi[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = PQR_NT / 32;
  const double tau = tk.tol * (tk.fnorm ? *tk.fnorm : 1.0);
  double* W = tk.W;
  double* Q = tk.Q;

  for (int c = warp; c < nc; c += NW) {
    double s = 0.0;
    for (int r = lane; r < m; r += 32) { double x = W[(size_t)c * ldw + r]; s += x * x; }
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) norms[c] = s;
  }
  __syncthreads();
  int t = 0, t_trunc = -1;
  while (true) {
    // residual ||W||_F^2 and the largest column norm in one reduction
    double part = 0.0, v = -1.0;
    for (int c = tid; c < nc; c += PQR_NT) { part += norms[c]; v = fmax(v, sqrt(norms[c])); }
    double res2, mx;
    block_sum_max<PQR_NT>(part, v, red, &res2, &mx);
    const bool ok = !(sqrt(res2) > tau);
    if (ok && t_trunc < 0) t_trunc = t;
    if (t >= tk.tmin && ok) break;
    if (t >= tk.tmax) break;
    if (!(mx > 0.0)) break;
    const double thr = mx * (1.0 - TIE);
    int cand = 0x7fffffff;
    for (int c = tid; c < nc; c += PQR_NT)
      if (sqrt(norms[c]) >= thr) { cand = c; break; }
    const int j = block_min_int<PQR_NT>(cand, redi);
    for (int r = tid; r < m; r += PQR_NT) w[r] = W[(size_t)j * ldw + r];
    __syncthreads();
    const int kb = tk.k0 + t;
    // re-orthogonalisation (R8): two passes, a third if the second cancelled more than
    // half; a column still collapsing lies in span(Q) numerically and is discarded
    double nprev = 0.0, nw = 0.0;
    for (int pass = 0; pass < 3; ++pass) {
      for (int s = warp; s < kb; s += NW) {
        double a = 0.0;
        for (int r = lane; r < m; r += 32) a += Q[(size_t)s * ldq + r] * w[r];
        for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
        if (lane == 0) coef[s] = a;
      }
      __syncthreads();
      double p2 = 0.0;
      for (int r = tid; r < m; r += PQR_NT) {
        double a = w[r];
        for (int s = 0; s < kb; ++s) a -= Q[(size_t)s * ldq + r] * coef[s];
        w[r] = a;
        p2 += a * a;
      }
      nw = sqrt(block_sum<PQR_NT>(p2, red));
      if (pass == 1 && nw > 0.5 * nprev) break;
      if (pass == 2 && !(nw > 0.5 * nprev)) nw = 0.0;
      nprev = nw;
    }
    for (int r = tid; r < m; r += PQR_NT) {
      const double q = w[r] / nw;
      w[r] = q;
      Q[(size_t)kb * ldq + r] = q;
    }
    __syncthreads();
    // W <- W - q (q^T W); recompute column norms; W[:, j] = 0
    for (int c = warp; c < nc; c += NW) {
      double* col = W + (size_t)c * ldw;
      if (c == j) {
        for (int r = lane; r < m; r += 32) col[r] = 0.0;
        if (lane == 0) norms[c] = 0.0;
        continue;
      }
      double s = 0.0, n2 = 0.0;
      if (m <= 32 * 16) {
        // column cached in registers between the dot product and the update (one read, one
        // write per step; same arithmetic order)
        double cr[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const int r = lane + 32 * u;
          cr[u] = (r < m) ? col[r] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const int r = lane + 32 * u;
          if (r < m) s += w[r] * cr[u];
        }
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const int r = lane + 32 * u;
          if (r < m) {
            const double x = cr[u] - s * w[r];
            col[r] = x;
            n2 += x * x;
          }
        }
      } else {
        for (int r = lane; r < m; r += 32) s += w[r] * col[r];
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        for (int r = lane; r < m; r += 32) {
          const double x = col[r] - s * w[r];
          col[r] = x;
          n2 += x * x;
        }
      }
      for (int o = 16; o > 0; o >>= 1) n2 += __shfl_xor_sync(0xffffffffu, n2, o);
      if (lane == 0) norms[c] = n2;
    }
    __syncthreads();
    ++t;
  }
  if (tid == 0) {
    if (t_trunc < 0) t_trunc = t;
    if (tk.t_trunc) *tk.t_trunc = t_trunc;
    if (tk.t_taken) *tk.t_taken = t;
  }
}

// Cluster variant of the pivoted QR (same decision rule and arithmetic order per column as
// pqr_tasks_kernel): the 8 CTAs of a cluster own contiguous column slices of W (staged in
// shared memory when they fit), the pivot search / residual sums / re-orthogonalisation
// coefficients are combined through DSMEM, and the re-orthogonalisation is row-split.
constexpr int PQC = 8;
constexpr int PQR_RC = 32;   // column cached in registers (32 per lane) for m <= 1024
__global__ void __cluster_dims__(PQC, 1, 1) __launch_bounds__(PQR_NT)
pqr_cluster_kernel(const PqrTask* __restrict__ tasks, int smem_cap) {
  extern __shared__ double pqs[];
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  const PqrTask tk = tasks[blockIdx.x / PQC];
  const int m = tk.m, nc = tk.ncols, ldq = tk.ldq;
  const int cw = (nc + PQC - 1) / PQC;
  const int c0 = min(nc, rank * cw), c1 = min(nc, c0 + cw), ncl = c1 - c0;
  const int kmax = tk.k0 + tk.tmax;
  // shared layout: w[m] | coef[kmax] | norms[cw] | Wl[m*cw] (if staged)
  double* w = pqs;
  double* coef = w + m;
  double* norms = coef + kmax;
  double* Wst = norms + cw;
  const bool staged = (size_t)(m + kmax + cw) + (size_t)m * cw <= (size_t)smem_cap;
  double* Wl = staged ? Wst : tk.W + (size_t)c0 * tk.ldw;
  const int ldl = staged ? m : tk.ldw;
  __shared__ double red[32];
  __shared__ int redi[32];
  __shared__ double s_part, s_max;
  __shared__ int s_idx;
  __shared__ double s_bc[3];
  __shared__ int s_bci;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = PQR_NT / 32;
  const double tau = tk.tol * (tk.fnorm ? *tk.fnorm : 1.0);
  double* Q = tk.Q;
  if (staged)
    for (int e = tid; e < m * ncl; e += PQR_NT) Wl[(size_t)(e / m) * ldl + e % m] = tk.W[(size_t)(c0 + e / m) * tk.ldw + e % m];
  __syncthreads();
  for (int c = warp; c < ncl; c += NW) {
    double sacc = 0.0;
    for (int r = lane; r < m; r += 32) { const double x = Wl[(size_t)c * ldl + r]; sacc += x * x; }
    for (int o = 16; o > 0; o >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, o);
    if (lane == 0) norms[c] = sacc;
  }
  __syncthreads();
  // row slice for the re-orthogonalisation
  const int rw = (m + PQC - 1) / PQC;
  const int r0 = min(m, rank * rw), r1 = min(m, r0 + rw);
  int t = 0, t_trunc = -1;
  while (true) {
    // residual and largest column norm: one block reduction, one cluster barrier
    double part = 0.0, v = -1.0;
    for (int c = tid; c < ncl; c += PQR_NT) { part += norms[c]; v = fmax(v, sqrt(norms[c])); }
    block_sum_max<PQR_NT>(part, v, red, &part, &v);
    if (tid == 0) { s_part = part; s_max = v; }
    cl.sync();
    // warp 0 fetches the PQC partials in one parallel round of DSMEM loads
    if (warp == 0) {
      double a2 = 0.0, b2 = -1.0;
      if (lane < PQC) { a2 = *cl.map_shared_rank(&s_part, lane); b2 = *cl.map_shared_rank(&s_max, lane); }
      for (int o = 4; o > 0; o >>= 1) {
        a2 += __shfl_xor_sync(0xffffffffu, a2, o);
        b2 = fmax(b2, __shfl_xor_sync(0xffffffffu, b2, o));
      }
      if (lane == 0) { s_bc[0] = a2; s_bc[1] = b2; }
    }
    __syncthreads();
    const double res2 = s_bc[0], mx = s_bc[1];
    const bool ok = !(sqrt(res2) > tau);
    if (ok && t_trunc < 0) t_trunc = t;
    if ((t >= tk.tmin && ok) || t >= tk.tmax) break;
    if (!(mx > 0.0)) break;
    const double thr = mx * (1.0 - TIE);
    int cand = 0x7fffffff;
    for (int c = tid; c < ncl; c += PQR_NT)
      if (sqrt(norms[c]) >= thr) { cand = c0 + c; break; }
    cand = block_min_int<PQR_NT>(cand, redi);
    if (tid == 0) s_idx = cand;
    cl.sync();
    if (warp == 0) {
      int jj = (lane < PQC) ? *cl.map_shared_rank(&s_idx, lane) : 0x7fffffff;
      for (int o = 4; o > 0; o >>= 1) jj = min(jj, __shfl_xor_sync(0xffffffffu, jj, o));
      if (lane == 0) s_bci = jj;
    }
    __syncthreads();
    const int j = s_bci;
    const int jo = min(PQC - 1, j / cw);       // owner rank of column j
    // fetch column j (owner's slice) into w
    {
      const double* src = (staged ? cl.map_shared_rank(Wst, jo) : tk.W + (size_t)(jo * cw) * tk.ldw);
      const int lds = staged ? m : tk.ldw;
      const int lj = j - jo * cw;
      for (int r = tid; r < m; r += PQR_NT) w[r] = src[(size_t)lj * lds + r];
    }
    __syncthreads();
    const int kb = tk.k0 + t;
    double nprev = 0.0, nw = 0.0;
    for (int pass = 0; pass < 3; ++pass) {
      // coefficients for basis vectors s in this rank's slice of [0, kb)
      const int sw = (kb + PQC - 1) / PQC;
      const int s0 = min(kb, rank * sw), s1 = min(kb, s0 + sw);
      for (int sidx = s0 + warp; sidx < s1; sidx += NW) {
        double acc = 0.0;
        for (int r = lane; r < m; r += 32) acc += Q[(size_t)sidx * ldq + r] * w[r];
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) coef[sidx] = acc;
      }
      cl.sync();
      // gather all coefficients
      for (int sidx = tid; sidx < kb; sidx += PQR_NT) {
        const int own = min(PQC - 1, sidx / max(sw, 1));
        if (own != rank) coef[sidx] = cl.map_shared_rank(coef, own)[sidx];
      }
      cl.sync();
      // own row slice of w -= Q coef
      double p2 = 0.0;
      for (int r = r0 + tid; r < r1; r += PQR_NT) {
        double acc = w[r];
        for (int sidx = 0; sidx < kb; ++sidx) acc -= Q[(size_t)sidx * ldq + r] * coef[sidx];
        w[r] = acc;
        p2 += acc * acc;
      }
      p2 = block_sum<PQR_NT>(p2, red);
      if (tid == 0) s_part = p2;
      cl.sync();
      if (warp == 0) {
        double a2 = (lane < PQC) ? *cl.map_shared_rank(&s_part, lane) : 0.0;
        for (int o = 4; o > 0; o >>= 1) a2 += __shfl_xor_sync(0xffffffffu, a2, o);
        if (lane == 0) s_bc[2] = a2;
      }
      __syncthreads();
      const double n2 = s_bc[2];
      // gather the full w from the row owners
      for (int r = tid; r < m; r += PQR_NT) {
        const int own = min(PQC - 1, r / max(rw, 1));
        if (own != rank) w[r] = cl.map_shared_rank(w, own)[r];
      }
      cl.sync();
      nw = sqrt(n2);
      if (pass == 1 && nw > 0.5 * nprev) break;
      if (pass == 2 && !(nw > 0.5 * nprev)) nw = 0.0;
      nprev = nw;
    }
    if (!(nw > 0.0)) {
      if (j >= c0 && j < c1) {
        for (int r = tid; r < m; r += PQR_NT) Wl[(size_t)(j - c0) * ldl + r] = 0.0;
        if (tid == 0) norms[j - c0] = 0.0;
      }
      __syncthreads();
      cl.sync();
      continue;
    }
    for (int r = tid; r < m; r += PQR_NT) {
      const double qv = w[r] / nw;
      w[r] = qv;
      if (rank == 0) Q[(size_t)kb * ldq + r] = qv;
    }
    __syncthreads();
    for (int c = warp; c < ncl; c += NW) {
      double* col = Wl + (size_t)c * ldl;
      if (c0 + c == j) {
        for (int r = lane; r < m; r += 32) col[r] = 0.0;
        if (lane == 0) norms[c] = 0.0;
        continue;
      }
      double sacc = 0.0, n2 = 0.0;
      if (m <= 32 * PQR_RC) {
        // the column stays in registers between the dot product and the update: one read and
        // one write of it per step instead of two reads and a write (same arithmetic order)
        double cr[PQR_RC];
#pragma unroll
        for (int u = 0; u < PQR_RC; ++u) {
          const int r = lane + 32 * u;
          cr[u] = (r < m) ? col[r] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < PQR_RC; ++u) {
          const int r = lane + 32 * u;
          if (r < m) sacc += w[r] * cr[u];
        }
        for (int o = 16; o > 0; o >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, o);
#pragma unroll
        for (int u = 0; u < PQR_RC; ++u) {
          const int r = lane + 32 * u;
          if (r < m) {
            const double x = cr[u] - sacc * w[r];
            col[r] = x;
            n2 += x * x;
          }
        }
      } else {
        for (int r = lane; r < m; r += 32) sacc += w[r] * col[r];
        for (int o = 16; o > 0; o >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, o);
        for (int r = lane; r < m; r += 32) {
          const double x = col[r] - sacc * w[r];
          col[r] = x;
          n2 += x * x;
        }
      }
      for (int o = 16; o > 0; o >>= 1) n2 += __shfl_xor_sync(0xffffffffu, n2, o);
      if (lane == 0) norms[c] = n2;
    }
    __syncthreads();
    cl.sync();
    ++t;
  }
  if (staged)
    for (int e = tid; e < m * ncl; e += PQR_NT) tk.W[(size_t)(c0 + e / m) * tk.ldw + e % m] = Wl[(size_t)(e / m) * ldl + e % m];
  if (rank == 0 && tid == 0) {
    if (t_trunc < 0) t_trunc = t;
    if (tk.t_trunc) *tk.t_trunc = t_trunc;
    if (tk.t_taken) *tk.t_taken = t;
  }
  cl.sync();
}

// ------------------------------------------------------------------------------ Householder QR
// Blocked Householder QR of a batch of tall n x m matrices A (column-major, lda), used for the
// first stage of the two-stage RRQR (reading R8b): W^T = Q R, then pivoted QR of R^T.
// Panel kernel: unblocked Householder (LAPACK dlarfg convention) on columns [j, j+nbw) and
// rows [j, n), explicit V (unit diagonal) and the compact-WY factor T (dlarft, forward);
// the trailing update (I - V T^T V^T) C is three DMMA GEMM launches issued by the host.
constexpr int HHB = 32;
struct HHTask {
  double* A;
  int lda, n, m;
  double* V;     // workspace n x HHB (ld n)
  double* T;     // workspace HHB x HHB (ld HHB)
};

// One CTA (512 threads) per task, panel read from global memory / L2: used when the batch
// has enough tasks to fill the GPU (the cluster variants below spread one task over 8 SMs).
constexpr int HHP_NT = 512;
__global__ void __launch_bounds__(HHP_NT) hh_panel_kernel(const HHTask* __restrict__ tasks, int j) {
  const HHTask tk = tasks[blockIdx.x];
  const int r = min(tk.n, tk.m);
  if (j >= r) return;
  const int nbw = min(HHB, r - j), rows = tk.n - j, ld = tk.lda;
  double* A = tk.A + j + (size_t)j * ld;   // panel origin
  __shared__ double red[32];
  __shared__ double tau_s[HHB];
  __shared__ double G[HHB][HHB + 1];
  __shared__ double Ts[HHB][HHB + 1];
  constexpr int NW = HHP_NT / 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int c = 0; c < nbw; ++c) {
    double* x = A + (size_t)c * ld + c;     // column c, from the diagonal down
    const int len = rows - c;
    double p = 0.0;
    for (int i = 1 + tid; i < len; i += HHP_NT) p += x[i] * x[i];
    const double sigma = block_sum<HHP_NT>(p, red);
    const double alpha = x[0];
    double tau = 0.0, beta = alpha, scal = 0.0;
    if (sigma > 0.0) {
      const double nrm = sqrt(alpha * alpha + sigma);
      beta = (alpha >= 0.0) ? -nrm : nrm;
      tau = (beta - alpha) / beta;
      scal = 1.0 / (alpha - beta);
    }
    // v = [1; x[1:] * scal], A[c][c] = beta
    if (sigma > 0.0)
      for (int i = 1 + tid; i < len; i += HHP_NT) x[i] *= scal;
    __syncthreads();
    if (tid == 0) { x[0] = beta; tau_s[c] = tau; }
    // apply H = I - tau v v^T to the remaining panel columns (one warp per column)
    for (int cc = c + 1 + warp; cc < nbw; cc += NW) {
      double* y = A + (size_t)cc * ld + c;
      double w = (lane == 0) ? y[0] : 0.0;
      for (int i = 1 + lane; i < len; i += 32) w += x[i] * y[i];
      for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
      w *= tau;
      if (lane == 0) y[0] -= w;
      for (int i = 1 + lane; i < len; i += 32) y[i] -= w * x[i];
    }
    __syncthreads();
  }
  // explicit V (rows j..n of the full matrix, ld n): unit diagonal, zeros above
  for (int c = warp; c < nbw; c += NW) {
    const double* src = A + (size_t)c * ld;
    double* dst = tk.V + (size_t)c * tk.n;
    for (int i = lane; i < rows; i += 32) dst[i] = (i < c) ? 0.0 : (i == c ? 1.0 : src[i]);
  }
  __syncthreads();
  // Gram V^T V (a < b), one warp per entry
  for (int e = warp; e < nbw * nbw; e += NW) {
    const int a = e % nbw, b = e / nbw;
    if (a >= b) continue;
    const double* va = tk.V + (size_t)a * tk.n;
    const double* vb = tk.V + (size_t)b * tk.n;
    double s = 0.0;
    for (int i = b + lane; i < rows; i += 32) s += va[i] * vb[i];   // v_b is zero above row b
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) G[a][b] = s;
  }
  for (int e = tid; e < HHB * HHB; e += HHP_NT) Ts[e % HHB][e / HHB] = 0.0;
  __syncthreads();
  // dlarft (forward, columnwise): T[0:i, i] = -tau_i T[0:i, 0:i] (V^T v_i), rows in parallel
  for (int i = 0; i < nbw; ++i) {
    const double ti = tau_s[i];
    if (tid < i) {
      double s = 0.0;
      for (int b = tid; b < i; ++b) s += Ts[tid][b] * G[b][i];
      Ts[tid][i] = -ti * s;
    } else if (tid == i) {
      Ts[i][i] = ti;
    }
    __syncthreads();
  }
  for (int e = tid; e < HHB * HHB; e += HHP_NT) tk.T[e] = Ts[e % HHB][e / HHB];
}

// One CTA (512 threads) per task with the whole panel (rows <= HHS_ROWS, 32 columns) staged in
// shared memory: one load, 32 column steps at shared-memory speed, one store.  Used for the row
// chunks of the TSQR stage (batched_tri_root), whose chunk height is chosen to fit.  Same
// arithmetic (thread partition, reduction order) as hh_panel_kernel.
constexpr int HHS_ROWS = 768;
__global__ void __launch_bounds__(HHP_NT) hh_panel_smem_kernel(const HHTask* __restrict__ tasks, int j) {
  extern __shared__ __align__(16) double hps[];   // rows x nbw, ld = rows
  const HHTask tk = tasks[blockIdx.x];
  const int r = min(tk.n, tk.m);
  if (j >= r) return;
  const int nbw = min(HHB, r - j), rows = tk.n - j, ld = tk.lda;
  double* A = tk.A + j + (size_t)j * ld;
  double* P = hps;
  __shared__ double red[32];
  __shared__ double tau_s[HHB];
  __shared__ double G[HHB][HHB + 1];
  __shared__ double Ts[HHB][HHB + 1];
  constexpr int NW = HHP_NT / 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < rows * nbw; e += HHP_NT) {
    const int i = e % rows, c = e / rows;
    P[(size_t)c * rows + i] = A[(size_t)c * ld + i];
  }
  __syncthreads();
  for (int c = 0; c < nbw; ++c) {
    double* x = P + (size_t)c * rows + c;
    const int len = rows - c;
    double p = 0.0;
    for (int i = 1 + tid; i < len; i += HHP_NT) p += x[i] * x[i];
    const double sigma = block_sum<HHP_NT>(p, red);
    const double alpha = x[0];
    double tau = 0.0, beta = alpha, scal = 0.0;
    if (sigma > 0.0) {
      const double nrm = sqrt(alpha * alpha + sigma);
      beta = (alpha >= 0.0) ? -nrm : nrm;
      tau = (beta - alpha) / beta;
      scal = 1.0 / (alpha - beta);
    }
    if (sigma > 0.0)
      for (int i = 1 + tid; i < len; i += HHP_NT) x[i] *= scal;
    __syncthreads();
    if (tid == 0) { x[0] = beta; tau_s[c] = tau; }
    for (int cc = c + 1 + warp; cc < nbw; cc += NW) {
      double* y = P + (size_t)cc * rows + c;
      double w = (lane == 0) ? y[0] : 0.0;
      for (int i = 1 + lane; i < len; i += 32) w += x[i] * y[i];
      for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
      w *= tau;
      if (lane == 0) y[0] -= w;
      for (int i = 1 + lane; i < len; i += 32) y[i] -= w * x[i];
    }
    __syncthreads();
  }
  // write back, explicit V (ld n, unit diagonal, zeros above)
  for (int e = tid; e < rows * nbw; e += HHP_NT) {
    const int i = e % rows, c = e / rows;
    const double v = P[(size_t)c * rows + i];
    A[(size_t)c * ld + i] = v;
    tk.V[(size_t)c * tk.n + i] = (i < c) ? 0.0 : (i == c ? 1.0 : v);
  }
  // Gram V^T V (a < b) from shared memory, one warp per entry
  for (int e = warp; e < nbw * nbw; e += NW) {
    const int a = e % nbw, b = e / nbw;
    if (a >= b) continue;
    const double* va = P + (size_t)a * rows;
    const double* vb = P + (size_t)b * rows;
    double s = 0.0;
    for (int i = b + lane; i < rows; i += 32) s += (i == a ? 1.0 : va[i]) * (i == b ? 1.0 : vb[i]);
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) G[a][b] = s;
  }
  for (int e = tid; e < HHB * HHB; e += HHP_NT) Ts[e % HHB][e / HHB] = 0.0;
  __syncthreads();
  for (int i = 0; i < nbw; ++i) {
    const double ti = tau_s[i];
    if (tid < i) {
      double s = 0.0;
      for (int b = tid; b < i; ++b) s += Ts[tid][b] * G[b][i];
      Ts[tid][i] = -ti * s;
    } else if (tid == i) {
      Ts[i][i] = ti;
    }
    __syncthreads();
  }
  for (int e = tid; e < HHB * HHB; e += HHP_NT) tk.T[e] = Ts[e % HHB][e / HHB];
}

// Register-resident panel: 256 threads, thread t owns rows t + 256 q (q < RPT) of the 32-column
// panel in registers (rows <= 256 RPT).  Column step c needs ONE 32-value block reduction:
//   tot[k] = sum_{i>c} a_i[c] a_i[k]   (k = c: sigma; k > c: dots with the trailing columns;
//                                       k < c: V^T v_c for the compact-WY factor T)
// with row c broadcast through shared memory; then v_i = a_i[c] / (alpha - beta),
// v^T y_k = a_c[k] + scal tot[k], and the rank-1 update is local to each thread.  Same
// Householder convention (dlarfg / dlarft forward) as hh_panel_kernel; the summation order of
// the reductions differs (butterfly within warps, then across the 8 warps).
constexpr int HHR_NT = 256;
constexpr int HHC_REG = 8;   // CTAs per cluster of hh_panel_reg_cluster_kernel
__device__ __forceinline__ void warp_transpose_reduce32(double (&p)[HHB], int lane) {
  // after it, lane l holds (in p[0]) the warp sum of value l: 16 + 8 + 4 + 2 + 1 shuffles
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    const bool upper = (lane & off) != 0;
#pragma unroll
    for (int t = 0; t < off; ++t) {
      const double send = upper ? p[t] : p[t + off];
      const double keep = upper ? p[t + off] : p[t];
      p[t] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
}
template <int RPT>
__global__ void __launch_bounds__(HHR_NT) hh_panel_reg_kernel(const HHTask* __restrict__ tasks, int j) {
  const HHTask tk = tasks[blockIdx.x];
  const int r = min(tk.n, tk.m);
  if (j >= r) return;
  const int nbw = min(HHB, r - j), rows = tk.n - j, ld = tk.lda;
  double* A = tk.A + j + (size_t)j * ld;
  __shared__ double red[2][HHR_NT / 32][HHB];
  __shared__ double tot[2][HHB];
  __shared__ double rowc[2][HHB];
  __shared__ double Ts[HHB][HHB + 1];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double a[RPT][HHB];
#pragma unroll
  for (int q = 0; q < RPT; ++q) {
    const int i = tid + HHR_NT * q;
#pragma unroll
    for (int k = 0; k < HHB; ++k) a[q][k] = (i < rows && k < nbw) ? A[(size_t)k * ld + i] : 0.0;
  }
  for (int e = tid; e < HHB * (HHB + 1); e += HHR_NT) (&Ts[0][0])[e] = 0.0;
#pragma unroll
  for (int c = 0; c < HHB; ++c) {
    if (c < nbw) {
      const int ph = c & 1;
      if (tid == c) {
#pragma unroll
        for (int k = 0; k < HHB; ++k) rowc[ph][k] = a[0][k];
      }
      double p[HHB];
#pragma unroll
      for (int k = 0; k < HHB; ++k) p[k] = 0.0;
#pragma unroll
      for (int q = 0; q < RPT; ++q) {
        const int i = tid + HHR_NT * q;
        const double x = (i > c && i < rows) ? a[q][c] : 0.0;
#pragma unroll
        for (int k = 0; k < HHB; ++k) p[k] = fma(x, a[q][k], p[k]);
      }
      warp_transpose_reduce32(p, lane);
      red[ph][warp][lane] = p[0];
      __syncthreads();
      if (tid < HHB) {
        double t = 0.0;
#pragma unroll
        for (int w = 0; w < HHR_NT / 32; ++w) t += red[ph][w][tid];
        tot[ph][tid] = t;
      }
      __syncthreads();
      const double sigma = tot[ph][c], alpha = rowc[ph][c];
      double tau = 0.0, beta = alpha, scal = 0.0;
      if (sigma > 0.0) {
        const double nrm = sqrt(alpha * alpha + sigma);
        beta = (alpha >= 0.0) ? -nrm : nrm;
        tau = (beta - alpha) / beta;
        scal = 1.0 / (alpha - beta);
      }
      double tw[HHB];   // tau * v^T y_k for the trailing columns
#pragma unroll
      for (int k = 0; k < HHB; ++k) tw[k] = (k > c) ? tau * (rowc[ph][k] + scal * tot[ph][k]) : 0.0;
#pragma unroll
      for (int q = 0; q < RPT; ++q) {
        const int i = tid + HHR_NT * q;
        const double v = (i > c) ? a[q][c] * scal : (i == c ? 1.0 : 0.0);
#pragma unroll
        for (int k = c + 1; k < HHB; ++k) a[q][k] = fma(-tw[k], v, a[q][k]);
        if (i > c) a[q][c] = v;
        else if (i == c) a[q][c] = beta;
      }
      // T[0:c, c] = -tau T[0:c, 0:c] (V^T v_c),  (V^T v_c)_b = a_c[b] + scal tot[b]
      if (tid < c) {
        double t = 0.0;
        for (int b = tid; b < c; ++b) t += Ts[tid][b] * (rowc[ph][b] + scal * tot[ph][b]);
        Ts[tid][c] = -tau * t;
      } else if (tid == c) {
        Ts[c][c] = tau;
      }
    }
  }
#pragma unroll
  for (int q = 0; q < RPT; ++q) {
    const int i = tid + HHR_NT * q;
    if (i < rows) {
#pragma unroll
      for (int k = 0; k < HHB; ++k)
        if (k < nbw) {
          A[(size_t)k * ld + i] = a[q][k];
          tk.V[(size_t)k * tk.n + i] = (i < k) ? 0.0 : (i == k ? 1.0 : a[q][k]);
        }
    }
  }
  __syncthreads();
  for (int e = tid; e < HHB * HHB; e += HHR_NT) tk.T[e] = Ts[e % HHB][e / HHB];
}

// Cluster variant of the panel: the 8 CTAs of a cluster split the panel rows and combine
// their partial norms / dot products through distributed shared memory (DSMEM), so the long
// panels of the upper levels (n up to several thousand rows) are not serialised on one SM.
constexpr int HHC = 8;
__global__ void __cluster_dims__(HHC, 1, 1) __launch_bounds__(256)
hh_panel_cluster_kernel(const HHTask* __restrict__ tasks, int j) {
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  const HHTask tk = tasks[blockIdx.x / HHC];
  const int r = min(tk.n, tk.m);
  if (j >= r) return;                       // uniform across the cluster (same task)
  const int nbw = min(HHB, r - j), rows = tk.n - j, ld = tk.lda;
  const int chunk = (rows + HHC - 1) / HHC;
  const int lo = min(rows, rank * chunk), hi = min(rows, lo + chunk);
  double* A = tk.A + j + (size_t)j * ld;
  __shared__ double red[32];
  __shared__ double s_sig;
  __shared__ double s_dot[HHB];
  __shared__ double wloc[HHB];
  __shared__ double tau_s[HHB];
  __shared__ double gram[HHB][HHB + 1];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int c = 0; c < nbw; ++c) {
    double* x = A + (size_t)c * ld;
    const double alpha = x[c];
    double p = 0.0;
    for (int i = max(lo, c + 1) + tid; i < hi; i += 256) p += x[i] * x[i];
    p = block_sum<256>(p, red);
    if (tid == 0) s_sig = p;
    cl.sync();
    double sigma = 0.0;
    for (int q = 0; q < HHC; ++q) sigma += *cl.map_shared_rank(&s_sig, q);
    double tau = 0.0, beta = alpha, scal = 0.0;
    if (sigma > 0.0) {
      const double nrm = sqrt(alpha * alpha + sigma);
      beta = (alpha >= 0.0) ? -nrm : nrm;
      tau = (beta - alpha) / beta;
      scal = 1.0 / (alpha - beta);
      for (int i = max(lo, c + 1) + tid; i < hi; i += 256) x[i] *= scal;
    }
    const bool owner = (c >= lo && c < hi);
    if (tid == 0) tau_s[c] = tau;
    __syncthreads();
    for (int cc = c + 1 + warp; cc < nbw; cc += 8) {
      const double* y = A + (size_t)cc * ld;
      double w = (owner && lane == 0) ? y[c] : 0.0;
      for (int i = max(lo, c + 1) + lane; i < hi; i += 32) w += x[i] * y[i];
      for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
      if (lane == 0) s_dot[cc] = w;
    }
    cl.sync();
    for (int cc = c + 1 + tid; cc < nbw; cc += 256) {
      double w = 0.0;
      for (int q = 0; q < HHC; ++q) w += cl.map_shared_rank(s_dot, q)[cc];
      wloc[cc] = w * tau;
    }
    __syncthreads();
    for (int cc = c + 1 + warp; cc < nbw; cc += 8) {
      double* y = A + (size_t)cc * ld;
      const double w = wloc[cc];
      if (owner && lane == 0) y[c] -= w;
      for (int i = max(lo, c + 1) + lane; i < hi; i += 32) y[i] -= w * x[i];
    }
    if (owner && tid == 0) x[c] = beta;
    cl.sync();
  }
  // explicit V for own rows, partial Gram V^T V over own rows
  for (int e = tid; e < (hi - lo) * nbw; e += 256) {
    const int i = lo + e % (hi - lo), c = e / (hi - lo);
    const double v = (i < c) ? 0.0 : (i == c ? 1.0 : A[(size_t)c * ld + i]);
    tk.V[(size_t)c * tk.n + i] = v;
  }
  __syncthreads();
  for (int e = warp; e < nbw * nbw; e += 8) {
    const int a = e % nbw, b = e / nbw;
    if (a >= b) continue;
    double sacc = 0.0;
    for (int i = lo + lane; i < hi; i += 32) sacc += tk.V[(size_t)a * tk.n + i] * tk.V[(size_t)b * tk.n + i];
    for (int o = 16; o > 0; o >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, o);
    if (lane == 0) gram[a][b] = sacc;
  }
  cl.sync();
  __shared__ double gsum[HHB][HHB + 1];
  if (rank == 0) {
    for (int e = tid; e < nbw * nbw; e += 256) {
      const int a = e % nbw, b = e / nbw;
      double g = 0.0;
      if (a < b)
        for (int q = 0; q < HHC; ++q) g += cl.map_shared_rank(&gram[0][0], q)[a * (HHB + 1) + b];
      gsum[a][b] = g;
    }
  }
  __syncthreads();
  if (rank == 0 && tid == 0) {
    double* T = tk.T;
    for (int e = 0; e < HHB * HHB; ++e) T[e] = 0.0;
    for (int i = 0; i < nbw; ++i) {
      const double ti = tau_s[i];
      T[i + i * HHB] = ti;
      for (int a2 = 0; a2 < i; ++a2) {
        double sacc = 0.0;
        for (int b2 = a2; b2 < i; ++b2) sacc += T[a2 + b2 * HHB] * gsum[b2][i];
    T[a2 + i * HHB] = -ti * sacc;
      }
    }
  }
  cl.sync();
}

// Register-resident panel on an 8-CTA cluster: CTA r of the cluster owns the contiguous row
// slice [r*chunk, (r+1)*chunk) of the panel (chunk <= 256 RPT), one row per thread and slot, in
// registers.  Per column: the 32-value reduction of hh_panel_reg_kernel inside each CTA, one
// cluster barrier, then every CTA sums the 8 partial vectors and reads row c from its owner
// through distributed shared memory (double-buffered by column parity, so one barrier per
// column suffices).  Panels of up to 8 x 256 RPT rows.
template <int RPT, int CL>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(HHR_NT)
hh_panel_reg_cluster_kernel(const HHTask* __restrict__ tasks, int j) {
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  const HHTask tk = tasks[blockIdx.x / CL];
  const int r = min(tk.n, tk.m);
  if (j >= r) return;                       // uniform over the cluster
  const int nbw = min(HHB, r - j), rows = tk.n - j, ld = tk.lda;
  const int chunk = (rows + CL - 1) / CL;
  const int lo = min(rows, rank * chunk), hi = min(rows, lo + chunk);
  double* A = tk.A + j + (size_t)j * ld;
  __shared__ double red[2][HHR_NT / 32][HHB];
  __shared__ double part[2][HHB];          // this CTA's partial sums (read remotely)
  __shared__ double rowc[2][HHB];          // row c, if this CTA owns it (read remotely)
  __shared__ double tot[2][HHB];
  __shared__ double rc[2][HHB];
  __shared__ double Ts[HHB][HHB + 1];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double a[RPT][HHB];
#pragma unroll
  for (int q = 0; q < RPT; ++q) {
    const int i = lo + tid + HHR_NT * q;
#pragma unroll
    for (int k = 0; k < HHB; ++k) a[q][k] = (i < hi && k < nbw) ? A[(size_t)k * ld + i] : 0.0;
  }
  for (int e = tid; e < HHB * (HHB + 1); e += HHR_NT) (&Ts[0][0])[e] = 0.0;
#pragma unroll
  for (int c = 0; c < HHB; ++c) {
    if (c < nbw) {
      const int ph = c & 1;
      const int oc = min(CL - 1, c / max(chunk, 1));   // owner CTA of row c
#pragma unroll
      for (int q = 0; q < RPT; ++q)
        if (lo + tid + HHR_NT * q == c) {
#pragma unroll
          for (int k = 0; k < HHB; ++k) rowc[ph][k] = a[q][k];
        }
      double p[HHB];
#pragma unroll
      for (int k = 0; k < HHB; ++k) p[k] = 0.0;
#pragma unroll
      for (int q = 0; q < RPT; ++q) {
        const int i = lo + tid + HHR_NT * q;
        const double x = (i > c && i < hi) ? a[q][c] : 0.0;
#pragma unroll
        for (int k = 0; k < HHB; ++k) p[k] = fma(x, a[q][k], p[k]);
      }
      warp_transpose_reduce32(p, lane);
      red[ph][warp][lane] = p[0];
      __syncthreads();
      if (tid < HHB) {
        double t = 0.0;
#pragma unroll
        for (int w = 0; w < HHR_NT / 32; ++w) t += red[ph][w][tid];
        part[ph][tid] = t;
      }
      cl.sync();
      if (tid < HHB) {
        double t = 0.0;
#pragma unroll
        for (int qq = 0; qq < CL; ++qq) t += cl.map_shared_rank(&part[0][0], qq)[ph * HHB + tid];
        tot[ph][tid] = t;
        rc[ph][tid] = cl.map_shared_rank(&rowc[0][0], oc)[ph * HHB + tid];
      }
      __syncthreads();
      const double sigma = tot[ph][c], alpha = rc[ph][c];
      double tau = 0.0, beta = alpha, scal = 0.0;
      if (sigma > 0.0) {
        const double nrm = sqrt(alpha * alpha + sigma);
        beta = (alpha >= 0.0) ? -nrm : nrm;
        tau = (beta - alpha) / beta;
        scal = 1.0 / (alpha - beta);
      }
      double tw[HHB];
#pragma unroll
      for (int k = 0; k < HHB; ++k) tw[k] = (k > c) ? tau * (rc[ph][k] + scal * tot[ph][k]) : 0.0;
#pragma unroll
      for (int q = 0; q < RPT; ++q) {
        const int i = lo + tid + HHR_NT * q;
        const double v = (i > c) ? a[q][c] * scal : (i == c ? 1.0 : 0.0);
#pragma unroll
        for (int k = c + 1; k < HHB; ++k) a[q][k] = fma(-tw[k], v, a[q][k]);
        if (i > c) a[q][c] = v;
        else if (i == c) a[q][c] = beta;
      }
      if (tid < c) {
        double t = 0.0;
        for (int b = tid; b < c; ++b) t += Ts[tid][b] * (rc[ph][b] + scal * tot[ph][b]);
        Ts[tid][c] = -tau * t;
      } else if (tid == c) {
        Ts[c][c] = tau;
      }
    }
  }
#pragma unroll
  for (int q = 0; q < RPT; ++q) {
    const int i = lo + tid + HHR_NT * q;
    if (i < hi) {
#pragma unroll
      for (int k = 0; k < HHB; ++k)
        if (k < nbw) {
          A[(size_t)k * ld + i] = a[q][k];
          tk.V[(size_t)k * tk.n + i] = (i < k) ? 0.0 : (i == k ? 1.0 : a[q][k]);
        }
    }
  }
  __syncthreads();
  if (rank == 0)
    for (int e = tid; e < HHB * HHB; e += HHR_NT) tk.T[e] = Ts[e % HHB][e / HHB];
  cl.sync();   // remote shared memory stays alive until every CTA has read it
}

// Same cluster panel with the panel rows of every CTA staged in shared memory (one load,
// one store); used when (rows/8) x 32 doubles fit.  Same arithmetic order as the global one.
__global__ void __cluster_dims__(HHC, 1, 1) __launch_bounds__(256)
hh_panel_cluster_smem_kernel(const HHTask* __restrict__ tasks, int j, int cap_rows) {
  extern __shared__ double P[];          // chunk x nbw, ld = cap_rows
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  const HHTask tk = tasks[blockIdx.x / HHC];
  const int r = min(tk.n, tk.m);
  if (j >= r) return;
  const int nbw = min(HHB, r - j), rows = tk.n - j, ld = tk.lda;
  const int chunk = (rows + HHC - 1) / HHC;
  const int lo = min(rows, rank * chunk), hi = min(rows, lo + chunk);
  const int cnt = hi - lo;
  double* A = tk.A + j + (size_t)j * ld;
  __shared__ double red[32];
  __shared__ double s_sig[2], s_alpha[2];   // double-buffered by column parity: no trailing
  __shared__ double s_dot[2][HHB];           // cluster barrier per column (WAR is ordered by the next column's barriers)
  __shared__ double wloc[HHB];
  __shared__ double tau_s[HHB];
  __shared__ double gram[HHB][HHB + 1];
  __shared__ double gsum[HHB][HHB + 1];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < cnt * nbw; e += 256) {
    const int i = e % cnt, c = e / cnt;
    P[(size_t)c * cap_rows + i] = A[(size_t)c * ld + lo + i];
  }
  __syncthreads();
  for (int c = 0; c < nbw; ++c) {
    double* x = P + (size_t)c * cap_rows;          // local rows
    const bool owner = (c >= lo && c < hi);
    const int i0 = max(lo, c + 1) - lo;               // first local row below the diagonal
    double p = 0.0;
    for (int i = i0 + tid; i < cnt; i += 256) p += x[i] * x[i];
    p = block_sum<256>(p, red);
    const int ph = c & 1;
    if (tid == 0) { s_sig[ph] = p; if (owner) s_alpha[ph] = x[c - lo]; }
    cl.sync();
    double sigma = 0.0;
    for (int q = 0; q < HHC; ++q) sigma += cl.map_shared_rank(s_sig, q)[ph];
    const int orank = min(HHC - 1, c / chunk);
    const double alpha = cl.map_shared_rank(s_alpha, orank)[ph];
    double tau = 0.0, beta = alpha, scal = 0.0;
    if (sigma > 0.0) {
      const double nrm = sqrt(alpha * alpha + sigma);
      beta = (alpha >= 0.0) ? -nrm : nrm;
      tau = (beta - alpha) / beta;
      scal = 1.0 / (alpha - beta);
      for (int i = i0 + tid; i < cnt; i += 256) x[i] *= scal;
    }
    if (tid == 0) tau_s[c] = tau;
    __syncthreads();
    for (int cc = c + 1 + warp; cc < nbw; cc += 8) {
      const double* y = P + (size_t)cc * cap_rows;
      double w = (owner && lane == 0) ? y[c - lo] : 0.0;
      for (int i = i0 + lane; i < cnt; i += 32) w += x[i] * y[i];
      for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
      if (lane == 0) s_dot[ph][cc] = w;
    }
    cl.sync();
    for (int cc = c + 1 + tid; cc < nbw; cc += 256) {
      double w = 0.0;
      for (int q = 0; q < HHC; ++q) w += cl.map_shared_rank(&s_dot[0][0], q)[ph * HHB + cc];
      wloc[cc] = w * tau;
    }
    __syncthreads();
    for (int cc = c + 1 + warp; cc < nbw; cc += 8) {
      double* y = P + (size_t)cc * cap_rows;
      const double w = wloc[cc];
      if (owner && lane == 0) y[c - lo] -= w;
      for (int i = i0 + lane; i < cnt; i += 32) y[i] -= w * x[i];
    }
    if (owner && tid == 0) x[c - lo] = beta;
    __syncthreads();
  }
  cl.sync();
  // write back, explicit V, partial Gram
  for (int e = tid; e < cnt * nbw; e += 256) {
    const int i = e % cnt, c = e / cnt, gi = lo + i;
    const double val = P[(size_t)c * cap_rows + i];
    A[(size_t)c * ld + gi] = val;
    tk.V[(size_t)c * tk.n + gi] = (gi < c) ? 0.0 : (gi == c ? 1.0 : val);
  }
  for (int e = warp; e < nbw * nbw; e += 8) {
    const int a = e % nbw, b = e / nbw;
    if (a >= b) continue;
    double sacc = 0.0;
    for (int i = lane; i < cnt; i += 32) {
      const int gi = lo + i;
      const double va = (gi < a) ? 0.0 : (gi == a ? 1.0 : P[(size_t)a * cap_rows + i]);
      const double vb = (gi < b) ? 0.0 : (gi == b ? 1.0 : P[(size_t)b * cap_rows + i]);
      sacc += va * vb;
    }
    for (int o = 16; o > 0; o >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, o);
    if (lane == 0) gram[a][b] = sacc;
  }
  cl.sync();
  if (rank == 0) {
    for (int e = tid; e < nbw * nbw; e += 256) {
      const int a = e % nbw, b = e / nbw;
      double g = 0.0;
      if (a < b)
        for (int q = 0; q < HHC; ++q) g += cl.map_shared_rank(&gram[0][0], q)[a * (HHB + 1) + b];
      gsum[a][b] = g;
    }
  }
  __syncthreads();
  if (rank == 0 && tid == 0) {
    double* T = tk.T;
    for (int e = 0; e < HHB * HHB; ++e) T[e] = 0.0;
    for (int i = 0; i < nbw; ++i) {
      const double ti = tau_s[i];
      T[i + i * HHB] = ti;
      for (int a2 = 0; a2 < i; ++a2) {
        double sacc = 0.0;
        for (int b2 = a2; b2 < i; ++b2) sacc += T[a2 + b2 * HHB] * gsum[b2][i];
        T[a2 + i * HHB] = -ti * sacc;
      }
    }
  }
  cl.sync();
}

// Fused trailing update of one Householder panel (compact WY, forward): for a 64-column block
// C of the trailing matrix (rows j..n, all of them), C <- (I - V T V^T)^T C = C - V (T^T (V^T C)).
// One CTA per (task, column block); both passes over C stream rows in 32-row chunks staged in
// shared memory, the products run on DMMA (mma.sync m8n8k4 f64).  Fixed summation order.
struct HHUTile { int task, n0; };
constexpr int HHU_NT = 256;
constexpr int HHU_BN = 64;   // column block (row chunk HHU_RK and pipeline stages: template)
constexpr int HHU_LV = HHB + 4, HHU_LC = HHU_BN + 4;  // padded rows (stride = 4 mod 16: no bank conflicts)
// (pass 1 alone keeps Z in the stage buffers, which are idle once its K loop has drained)
template <int HHU_ST, int HHU_RK = 32, int PH = 0>
constexpr size_t hhu_smem() {
  return sizeof(double) * ((size_t)HHU_ST * HHU_RK * (HHU_LV + HHU_LC) + (PH == 1 ? 0 : (size_t)HHB * HHU_LC));
}
// PH = 0: both passes in one CTA.  PH = 1: pass 1 only, Z2 = T^T V^T C written to zg (one
// HHB x HHU_BN slot per tile).  PH = 2: pass 2 only, for the rows [blockIdx.y * seg, +seg) of the
// tile, Z2 read from zg.  Every element of Z2 and of C sees the same operations in the same order
// in the three variants (pass 2 has no reduction across rows), so the split is bitwise neutral;
// it lets a panel with few column blocks spread its row-parallel pass over many CTAs.
template <int HHU_ST, int HHU_RK = 32, int PH = 0>
__global__ void __launch_bounds__(HHU_NT) hh_update_kernel(const HHTask* __restrict__ tasks,
                                                           const HHUTile* __restrict__ tiles, int j,
                                                           double* __restrict__ zg = nullptr, int seg = 0) {
  extern __shared__ __align__(16) double hhu_smem[];
  const HHUTile tl = tiles[blockIdx.x];
  const HHTask tk = tasks[tl.task];
  const int r = min(tk.n, tk.m);
  const int nbw = min(HHB, r - j), rows = tk.n - j, ld = tk.lda;
  const int nc = tk.m - j - nbw;
  const int n0 = tl.n0, ncb = min(HHU_BN, nc - n0);
  double* C = tk.A + j + (size_t)(j + nbw + n0) * ld;
  const double* V = tk.V;
  double* Vs = hhu_smem;                                  // [ST][RK][LV]
  double* Cs = Vs + (size_t)HHU_ST * HHU_RK * HHU_LV;     // [ST][RK][LC]
  double* Zs = PH == 1 ? hhu_smem : Cs + (size_t)HHU_ST * HHU_RK * HHU_LC;   // [HHB][LC]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp & 1) * 16, wn = (warp >> 1) * 16;   // 2 x 4 warps over 32 x 64
  const double* __restrict__ Tg = tk.T;                     // HHB x HHB, ld HHB (L1-resident)
  const int nch_all = (rows + HHU_RK - 1) / HHU_RK;
  const int ch0 = PH == 2 ? (int)blockIdx.y * (seg / HHU_RK) : 0;
  if (PH == 2 && ch0 >= nch_all) return;
  const int nch = PH == 2 ? min(nch_all, ch0 + seg / HHU_RK) : nch_all;
  auto issue = [&](int ch) {
    if (ch < nch) {
      const int st = ch % HHU_ST, r0 = ch * HHU_RK;
      double* vs = Vs + (size_t)st * HHU_RK * HHU_LV;
      double* cs = Cs + (size_t)st * HHU_RK * HHU_LC;
      for (int e = tid; e < HHU_RK * HHB; e += HHU_NT) {
        const int rr = e % HHU_RK, c = e / HHU_RK, gr = r0 + rr;
        const bool ok = gr < rows && c < nbw;
        cp_async8(vs + rr * HHU_LV + c, ok ? V + (size_t)c * tk.n + gr : V, ok);
      }
      for (int e = tid; e < HHU_RK * HHU_BN; e += HHU_NT) {
        const int rr = e % HHU_RK, c = e / HHU_RK, gr = r0 + rr;
        const bool ok = gr < rows && c < ncb;
        cp_async8(cs + rr * HHU_LC + c, ok ? C + (size_t)c * ld + gr : C, ok);
      }
    }
    cp_async_commit();
  };
  if (PH != 2) {
  // pass 1: Z = V^T C  (32 x 64, K = rows), 3-stage cp.async pipeline
  double acc[2][2][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int q = 0; q < 2; ++q) acc[i][q][0] = acc[i][q][1] = 0.0;
  for (int s = 0; s < HHU_ST - 1; ++s) issue(s);
  for (int ch = 0; ch < nch; ++ch) {
    issue(ch + HHU_ST - 1);
    cp_async_wait<HHU_ST - 1>();
    __syncthreads();
    const double* vs = Vs + (size_t)(ch % HHU_ST) * HHU_RK * HHU_LV;
    const double* cs = Cs + (size_t)(ch % HHU_ST) * HHU_RK * HHU_LC;
#pragma unroll
    for (int kk = 0; kk < HHU_RK; kk += 4) {
      double a[2], b[2];
#pragma unroll
      for (int i = 0; i < 2; ++i) a[i] = vs[(kk + (lane & 3)) * HHU_LV + wm + i * 8 + (lane >> 2)];
#pragma unroll
      for (int q = 0; q < 2; ++q) b[q] = cs[(kk + (lane & 3)) * HHU_LC + wn + q * 8 + (lane >> 2)];
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int q = 0; q < 2; ++q) dmma_884(acc[i][q][0], acc[i][q][1], a[i], b[q]);
    }
    __syncthreads();
  }
  cp_async_wait<0>();
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
      for (int e = 0; e < 2; ++e) Zs[(wm + i * 8 + (lane >> 2)) * HHU_LC + wn + q * 8 + (lane & 3) * 2 + e] = acc[i][q][e];
  __syncthreads();
  // Z2 = T^T Z (rows >= nbw vanish because T is zero there)
  double z2[HHB * HHU_BN / HHU_NT];
#pragma unroll
  for (int t = 0; t < HHB * HHU_BN / HHU_NT; ++t) {
    const int e = tid + t * HHU_NT, i = e % HHB, c = e / HHB;
    double s = 0.0;
    for (int a2 = 0; a2 <= i; ++a2) s += __ldg(Tg + a2 + i * HHB) * Zs[a2 * HHU_LC + c];   // T upper triangular
    z2[t] = s;
  }
  __syncthreads();
  if (PH == 1) {
    double* zt = zg + (size_t)blockIdx.x * HHB * HHU_BN;
#pragma unroll
    for (int t = 0; t < HHB * HHU_BN / HHU_NT; ++t) zt[tid + t * HHU_NT] = z2[t];
    return;
  }
#pragma unroll
  for (int t = 0; t < HHB * HHU_BN / HHU_NT; ++t) {
    const int e = tid + t * HHU_NT, i = e % HHB, c = e / HHB;
    Zs[i * HHU_LC + c] = z2[t];
  }
  } else {   // PH == 2: Z2 of this tile from pass 1
    const double* zt = zg + (size_t)blockIdx.x * HHB * HHU_BN;
#pragma unroll
    for (int t = 0; t < HHB * HHU_BN / HHU_NT; ++t) {
      const int e = tid + t * HHU_NT, i = e % HHB, c = e / HHB;
      Zs[i * HHU_LC + c] = zt[e];
    }
  }
  __syncthreads();
  // pass 2: C -= V Z2, chunk by chunk (same pipeline), results stored from shared memory
  for (int s = 0; s < HHU_ST - 1; ++s) issue(ch0 + s);
  for (int ch = ch0; ch < nch; ++ch) {
    issue(ch + HHU_ST - 1);
    cp_async_wait<HHU_ST - 1>();
    __syncthreads();
    const double* vs0 = Vs + (size_t)(ch % HHU_ST) * HHU_RK * HHU_LV;
    double* cs0 = Cs + (size_t)(ch % HHU_ST) * HHU_RK * HHU_LC;
#pragma unroll
    for (int rb = 0; rb < HHU_RK; rb += 32) {   // 32-row sub-blocks (2 x 4 warps over 32 x 64)
    const double* vs = vs0 + (size_t)rb * HHU_LV;
    double* cs = cs0 + (size_t)rb * HHU_LC;
    double o[2][2][2];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int q = 0; q < 2; ++q) o[i][q][0] = o[i][q][1] = 0.0;
#pragma unroll
    for (int kk = 0; kk < HHB; kk += 4) {
      double a[2], b[2];
#pragma unroll
      for (int i = 0; i < 2; ++i) a[i] = vs[(wm + i * 8 + (lane >> 2)) * HHU_LV + kk + (lane & 3)];
#pragma unroll
      for (int q = 0; q < 2; ++q) b[q] = Zs[(kk + (lane & 3)) * HHU_LC + wn + q * 8 + (lane >> 2)];
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int q = 0; q < 2; ++q) dmma_884(o[i][q][0], o[i][q][1], a[i], b[q]);
    }
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int q = 0; q < 2; ++q)
#pragma unroll
        for (int e = 0; e < 2; ++e) cs[(wm + i * 8 + (lane >> 2)) * HHU_LC + wn + q * 8 + (lane & 3) * 2 + e] -= o[i][q][e];
    }
    const double* cs = cs0;
    __syncthreads();
    const int r0 = ch * HHU_RK;
    for (int e = tid; e < HHU_RK * HHU_BN; e += HHU_NT) {
      const int rr = e % HHU_RK, c = e / HHU_RK, gr = r0 + rr;
      if (gr < rows && c < ncb) C[(size_t)c * ld + gr] = cs[rr * HHU_LC + c];
    }
    __syncthreads();
  }
  cp_async_wait<0>();
}
// one pass of the split trailing update (look-ahead schedule: pass 2 of the next panel's
// column tile runs first, the other tiles' pass 2 on a second stream under the next panel)
void launch_hh_update_pass(const void* tasks, const void* tiles, int ntiles, int j, cudaStream_t s,
                           double* zbuf, int seg, int nseg, int pass) {
  if (ntiles <= 0) return;
  const HHTask* tk = static_cast<const HHTask*>(tasks);
  const HHUTile* tt = static_cast<const HHUTile*>(tiles);
  if (pass == 1) {
    ensure_dyn_smem(hh_update_kernel<3, 32, 1>, hhu_smem<3, 32, 1>());
    LAUNCH((hh_update_kernel<3, 32, 1>), ntiles, HHU_NT, (hhu_smem<3, 32, 1>()), s, tk, tt, j, zbuf, 0);
  } else {
    ensure_dyn_smem(hh_update_kernel<3, 32, 2>, hhu_smem<3, 32, 2>());
    if (g_before_launch) g_before_launch();
    hh_update_kernel<3, 32, 2><<<dim3(ntiles, nseg), HHU_NT, hhu_smem<3, 32, 2>(), s>>>(tk, tt, j, zbuf, seg);
    AIFMM_CUDA(cudaGetLastError());
    ++g_launches;
  }
}
void launch_hh_update(const void* tasks, const void* tiles, int ntiles, int j, cudaStream_t s,
                      double* zbuf, int seg, int nseg) {
  static const int st = getenv("AIFMM_HHU_ST") ? atoi(getenv("AIFMM_HHU_ST")) : 3;   // experiment toggle
  if (zbuf && nseg > 1) {    // split: pass 1 per tile, then pass 2 over (tile, row segment)
    // pipeline variants (same arithmetic order; shared memory sets the CTAs per SM)
    static const int p1 = getenv("AIFMM_HHU_P1") ? atoi(getenv("AIFMM_HHU_P1")) : 3;
    static const int p2 = getenv("AIFMM_HHU_P2") ? atoi(getenv("AIFMM_HHU_P2")) : 3;
    const HHTask* tk = static_cast<const HHTask*>(tasks);
    const HHUTile* tt = static_cast<const HHUTile*>(tiles);
    if (p1 == 2) {
      ensure_dyn_smem(hh_update_kernel<2, 32, 1>, hhu_smem<2, 32, 1>());
      LAUNCH((hh_update_kernel<2, 32, 1>), ntiles, HHU_NT, (hhu_smem<2, 32, 1>()), s, tk, tt, j, zbuf, 0);
    } else if (p1 == 4) {
      ensure_dyn_smem(hh_update_kernel<4, 16, 1>, hhu_smem<4, 16, 1>());
      LAUNCH((hh_update_kernel<4, 16, 1>), ntiles, HHU_NT, (hhu_smem<4, 16, 1>()), s, tk, tt, j, zbuf, 0);
    } else {
      ensure_dyn_smem(hh_update_kernel<3, 32, 1>, hhu_smem<3, 32, 1>());
      LAUNCH((hh_update_kernel<3, 32, 1>), ntiles, HHU_NT, (hhu_smem<3, 32, 1>()), s, tk, tt, j, zbuf, 0);
    }
    if (g_before_launch) g_before_launch();
    if (p2 == 2) {
      ensure_dyn_smem(hh_update_kernel<2, 32, 2>, hhu_smem<2, 32, 2>());
      hh_update_kernel<2, 32, 2><<<dim3(ntiles, nseg), HHU_NT, hhu_smem<2, 32, 2>(), s>>>(tk, tt, j, zbuf, seg);
    } else {
      ensure_dyn_smem(hh_update_kernel<3, 32, 2>, hhu_smem<3, 32, 2>());
      hh_update_kernel<3, 32, 2><<<dim3(ntiles, nseg), HHU_NT, hhu_smem<3, 32, 2>(), s>>>(tk, tt, j, zbuf, seg);
    }
    AIFMM_CUDA(cudaGetLastError());
    ++g_launches;
  } else if (st == 64) {            // 64-row chunks, 2 stages (experiment)
    ensure_dyn_smem(hh_update_kernel<2, 64>, hhu_smem<2, 64>());
    LAUNCH((hh_update_kernel<2, 64>), ntiles, HHU_NT, (hhu_smem<2, 64>()), s, static_cast<const HHTask*>(tasks), static_cast<const HHUTile*>(tiles), j);
  } else if (st == 2) {
    ensure_dyn_smem(hh_update_kernel<2>, hhu_smem<2>());
    LAUNCH(hh_update_kernel<2>, ntiles, HHU_NT, hhu_smem<2>(), s, static_cast<const HHTask*>(tasks), static_cast<const HHUTile*>(tiles), j);
  } else {
    ensure_dyn_smem(hh_update_kernel<3>, hhu_smem<3>());
    LAUNCH(hh_update_kernel<3>, ntiles, HHU_NT, hhu_smem<3>(), s, static_cast<const HHTask*>(tasks), static_cast<const HHUTile*>(tiles), j);
  }
}

// M = R^T (m x r) from the upper triangle of the factored A (n x m, lda)
__global__ void hh_extract_rt_kernel(const HHTask* __restrict__ tasks, double* const* __restrict__ out, const int* ldo) {
  const HHTask tk = tasks[blockIdx.x];
  const int r = min(tk.n, tk.m);
  double* M = out[blockIdx.x];
  const int ldm = ldo[blockIdx.x];
  if (ldm > 0) {
    for (int e = threadIdx.x; e < tk.m * r; e += blockDim.x) {
      const int jj = e % tk.m, i = e / tk.m;   // M[jj, i] = R[i, jj]
      M[(size_t)i * ldm + jj] = (i <= jj) ? tk.A[(size_t)jj * tk.lda + i] : 0.0;
    }
  } else {                                     // ldm < 0: R itself (r x m, ld -ldm), TSQR stacking
    for (int e = threadIdx.x; e < tk.m * r; e += blockDim.x) {
      const int i = e % r, jj = e / r;
      M[(size_t)jj * (-ldm) + i] = (i <= jj) ? tk.A[(size_t)jj * tk.lda + i] : 0.0;
    }
  }
}

// ------------------------------------------------------------------------------ kernel entries
__global__ void keval_tasks_kernel(const KEvalTask* __restrict__ tasks, const double* __restrict__ pts,
                                   KernelParams kp, int* __restrict__ flag) {
  const KEvalTask tk = tasks[blockIdx.x];
  const int tot = tk.nr * tk.nc;
  for (int e = threadIdx.x + blockIdx.y * blockDim.x; e < tot; e += blockDim.x * gridDim.y) {
    const int i = e % tk.nr, j = e / tk.nr;
    const int gi = tk.rows ? tk.rows[i] : tk.row0 + i;
    const int gj = tk.cols ? tk.cols[j] : tk.col0 + j;
    const double v = kernel_entry(kp, pts, gi, gj);
    if (!isfinite(v)) *flag = 1;
    tk.out[(size_t)j * tk.ld + i] = v;
  }
}

// Kernel-entry blocks straight from a level's block table (no per-block task list): CTA s
// handles slot s = b * cap + t of box b's list (N(b) or IL(b), entry q = idx[s]):
//   mode 0 (M2L): A(sk_b, sk_q) with the skeleton index lists sk + skoff[.];
//   mode 1 (leaf near blocks): A(points(b), points(q)) with point ranges off[.].
// The block sizes are the table entry's rows / cols; empty slots and empty blocks exit.
__global__ void keval_table_kernel(const BlkDev* __restrict__ v, const int* __restrict__ cnt,
                                   const int* __restrict__ idx, int cap, int mode,
                                   const int* __restrict__ sk, const long long* __restrict__ base,
                                   const double* __restrict__ pts, KernelParams kp, int* __restrict__ flag) {
  const long long slot = blockIdx.x;
  const int b = (int)(slot / cap), t = (int)(slot % cap);
  if (t >= cnt[b]) return;
  const BlkDev blk = v[slot];
  const int nr = blk.rows, nc = blk.cols;
  if (nr <= 0 || nc <= 0 || blk.p == nullptr) return;
  const int q = idx[slot];
  const long long rb = base[b], cb = base[q];
  for (int e = threadIdx.x; e < nr * nc; e += blockDim.x) {
    const int i = e % nr, j = e / nr;
    const int gi = mode == 0 ? sk[rb + i] : (int)(rb + i);
    const int gj = mode == 0 ? sk[cb + j] : (int)(cb + j);
    const double val = kernel_entry(kp, pts, gi, gj);
    if (!isfinite(val)) *flag = 1;
    blk.p[(size_t)j * blk.ld + i] = val;
  }
}

void launch_keval_table(const void* v, const int* cnt, const int* idx, int nb, int cap, int mode, const int* sk,
                        const long long* base, const double* pts, KernelParams kp, int* flag, cudaStream_t s) {
  LAUNCH(keval_table_kernel, nb * cap, 128, 0, s, static_cast<const BlkDev*>(v), cnt, idx, cap, mode, sk, base, pts, kp, flag);
}

// Level-start change of variables on the far blocks (reading R13): A_bq <- T_b A_bq T'_q^T for
// every IL slot of the level's block table with k_b, k_q <= SW_KMAX, one CTA per slot, the
// intermediate in shared memory, fixed summation order (the larger blocks go
// through the DMMA GEMM).  T, T2: per-box k x k factors (ld k) of U_b = Q T, V_b = Q' T'.
constexpr int SW_KMAX = 64;
__global__ void __launch_bounds__(256) orth_sandwich_kernel(const BlkDev* __restrict__ v, const int* __restrict__ cnt,
                                                            const int* __restrict__ idx, int cap,
                                                            const double* const* __restrict__ T,
                                                            const double* const* __restrict__ T2) {
  __shared__ double sX[SW_KMAX * SW_KMAX];
  const long long slot = blockIdx.x;
  const int b = (int)(slot / cap), t = (int)(slot % cap);
  if (t >= cnt[b]) return;
  const BlkDev blk = v[slot];
  const int kb = blk.rows, kq = blk.cols;
  if (kb <= 0 || kq <= 0 || kb > SW_KMAX || kq > SW_KMAX || blk.p == nullptr) return;
  const int q = idx[slot];
  const double* Tb = T[b];
  const double* Tq = T2[q];
  // X = A T'_q^T  (kb x kq): X[i][j] = sum_l A[i][l] T'_q[j][l]  (A read from global / L1)
  for (int e = threadIdx.x; e < kb * kq; e += blockDim.x) {
    const int i = e % kb, j = e / kb;
    double acc = 0.0;
    for (int l2 = 0; l2 < kq; ++l2) acc = fma(blk.p[(size_t)l2 * blk.ld + i], Tq[(size_t)l2 * kq + j], acc);
    sX[j * kb + i] = acc;
  }
  __syncthreads();
  // A = T_b X: A[i][j] = sum_l T_b[i][l] X[l][j]
  for (int e = threadIdx.x; e < kb * kq; e += blockDim.x) {
    const int i = e % kb, j = e / kb;
    double acc = 0.0;
    for (int l2 = 0; l2 < kb; ++l2) acc = fma(Tb[(size_t)l2 * kb + i], sX[j * kb + l2], acc);
    blk.p[(size_t)j * blk.ld + i] = acc;
  }
}

void launch_orth_sandwich(const void* v, const int* cnt, const int* idx, int nb, int cap, const double* const* T,
                          const double* const* T2, cudaStream_t s) {
  LAUNCH(orth_sandwich_kernel, nb * cap, 256, 0, s, static_cast<const BlkDev*>(v), cnt, idx, cap, T, T2);
}

// ------------------------------------------------------------------------------ copies, norms
__global__ void copy_tasks_kernel(const CopyTask* __restrict__ tasks) {
  const CopyTask tk = tasks[blockIdx.x];
  if (tk.src && tk.trans) {
    // transposed copy through a 32 x 32 shared-memory tile: src reads and dst writes both
    // coalesced (same per-element arithmetic as below: alpha * src, then store / accumulate)
    __shared__ double tile[32][33];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 8 rows of 32
    const int tr = (tk.rows + 31) / 32, tcn = (tk.cols + 31) / 32;
    for (int t = blockIdx.y; t < tr * tcn; t += gridDim.y) {
      const int r0 = (t % tr) * 32, c0 = (t / tr) * 32;
#pragma unroll
      for (int i = 0; i < 4; ++i) {   // dst(r, c) = alpha * src[r * lds + c]: read along c
        const int r = r0 + ty + 8 * i, c = c0 + tx;
        if (r < tk.rows && c < tk.cols) tile[ty + 8 * i][tx] = tk.alpha * tk.src[(size_t)r * tk.lds + c];
      }
      __syncthreads();
#pragma unroll
      for (int i = 0; i < 4; ++i) {   // write along r
        const int r = r0 + tx, c = c0 + ty + 8 * i;
        if (r < tk.rows && c < tk.cols) {
          double* d = tk.dst + (size_t)c * tk.ldd + r;
          const double v = tile[tx][ty + 8 * i];
          *d = tk.accumulate ? *d + v : v;
        }
      }
      __syncthreads();
    }
    return;
  }
  const int tot = tk.rows * tk.cols;
  for (int e = threadIdx.x + blockIdx.y * blockDim.x; e < tot; e += blockDim.x * gridDim.y) {
    const int r = e % tk.rows, c = e / tk.rows;
    double v = tk.alpha;
    if (tk.src) v *= tk.trans ? tk.src[(size_t)r * tk.lds + c] : tk.src[(size_t)c * tk.lds + r];
    double* d = tk.dst + (size_t)c * tk.ldd + r;
    *d = tk.accumulate ? *d + v : v;
  }
}

__global__ void norm_tasks_kernel(const NormTask* __restrict__ tasks) {
  const NormTask tk = tasks[blockIdx.x];
  __shared__ double red[32];
  double s = 0.0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int c = warp; c < tk.cols; c += 8) {          // warp per column, rows coalesced
    const double* col = tk.A + (size_t)c * tk.lda;
    for (int r = lane; r < tk.rows; r += 32) s += col[r] * col[r];
  }
  s = block_sum<256>(s, red);
  if (threadIdx.x == 0) *tk.out = sqrt(s);
}

// ------------------------------------------------------------------------------ host launchers
void launch_gemm(int tileclass, const GemmTask* t, const GemmTerm* tm, const GemmTile* tiles, int ntiles,
                 cudaStream_t s) {
  static bool init = false;
  if (!init) {
    ensure_dyn_smem(gemm_tasks_kernel<32, 32>, gemm_smem<32, 32>());
    ensure_dyn_smem(gemm_tasks_kernel<64, 32>, gemm_smem<64, 32>());
    ensure_dyn_smem(gemm_tasks_kernel<32, 64>, gemm_smem<32, 64>());
    ensure_dyn_smem(gemm_tasks_kernel<64, 64>, gemm_smem<64, 64>());
    init = true;
  }
  switch (tileclass) {
    case 4:   // 64 x 128 tiles, 8 warps (same per-element accumulation order as 64 x 64)
      ensure_dyn_smem(gemm_tasks_kernel<64, 128, 2>, gemm_smem<64, 128>());
      LAUNCH((gemm_tasks_kernel<64, 128, 2>), ntiles, 256, (gemm_smem<64, 128>()), s, t, tm, tiles);
      break;
    case 0: LAUNCH((gemm_tasks_kernel<32, 32>), ntiles, 32, (gemm_smem<32, 32>()), s, t, tm, tiles); break;
    case 1: LAUNCH((gemm_tasks_kernel<64, 32>), ntiles, 64, (gemm_smem<64, 32>()), s, t, tm, tiles); break;
    case 2: LAUNCH((gemm_tasks_kernel<32, 64>), ntiles, 64, (gemm_smem<32, 64>()), s, t, tm, tiles); break;
    default: {
      // 5 CTAs per SM (96 registers, a few spilled) measured ~2% faster on config 3 than 4 CTAs
      // (128 registers); same arithmetic.  AIFMM_GEMM_MINB=1 / 6: the other variants
      static const int minb = getenv("AIFMM_GEMM_MINB") ? atoi(getenv("AIFMM_GEMM_MINB")) : 5;
      if (minb == 5) {
        ensure_dyn_smem(gemm_tasks_kernel<64, 64, 5>, gemm_smem<64, 64>());
        LAUNCH((gemm_tasks_kernel<64, 64, 5>), ntiles, 128, (gemm_smem<64, 64>()), s, t, tm, tiles);
      } else if (minb == 6) {
        ensure_dyn_smem(gemm_tasks_kernel<64, 64, 6>, gemm_smem<64, 64>());
        LAUNCH((gemm_tasks_kernel<64, 64, 6>), ntiles, 128, (gemm_smem<64, 64>()), s, t, tm, tiles);
      } else {
        LAUNCH((gemm_tasks_kernel<64, 64>), ntiles, 128, (gemm_smem<64, 64>()), s, t, tm, tiles);
      }
      break;
    }
  }
}

void launch_gj(const GJTask* t, int ntasks, int nmax, int mode, cudaStream_t s) {
  // nmax here is the largest n*ncols (small kernel) or n (global kernel, negative)
  if (nmax >= 0) {
    size_t smem = (size_t)nmax * sizeof(double) + 0;  // caller passes n*nc + n + n/2 doubles
    ensure_dyn_smem(gj_small_kernel, smem);
    LAUNCH(gj_small_kernel, ntasks, GJ_NT, smem, s, t, mode);
  } else {
    size_t smem = (size_t)(-nmax) * (sizeof(double) + sizeof(int));
    ensure_dyn_smem(gj_global_kernel, smem);
    LAUNCH(gj_global_kernel, ntasks, GJ_NT, smem, s, t, mode);
  }
}

template <int CL>
static void launch_gj_panel_cluster_cl(const void* t, int ntasks, int j, int nmax, cudaStream_t s) {
  const int cap = (std::max(nmax - j, 1) + CL - 1) / CL;
  const size_t smem = (size_t)cap * (GJB + 1) * sizeof(double);
  ensure_dyn_smem(gj_panel_cluster_kernel<CL>, smem);
  LAUNCH(gj_panel_cluster_kernel<CL>, ntasks * CL, GJ_NT, smem, s, static_cast<const GJBTask*>(t), j, cap);
}
// cluster size by batch: 8 CTAs per matrix for a few matrices, fewer when 8 x the batch would
// take several waves of the 148 SMs (the row slices must still fit shared memory)
void launch_gj_panel_cluster(const void* t, int ntasks, int j, int nmax, cudaStream_t s) {
  static const int force = getenv("AIFMM_GJ_CL") ? atoi(getenv("AIFMM_GJ_CL")) : 0;   // debug toggle
  const auto fits = [&](int cl) { return (size_t)((nmax + cl - 1) / cl) * (GJB + 1) * sizeof(double) <= 200 * 1024; };
  int cl = 8;
  if (force) cl = force;
  else if (ntasks * 8 > 2 * 148 && fits(4)) cl = (ntasks * 4 > 2 * 148 && fits(2)) ? 2 : 4;
  if (cl == 2) launch_gj_panel_cluster_cl<2>(t, ntasks, j, nmax, s);
  else if (cl == 4) launch_gj_panel_cluster_cl<4>(t, ntasks, j, nmax, s);
  else launch_gj_panel_cluster_cl<8>(t, ntasks, j, nmax, s);
}
void launch_gj_panel(const void* t, int ntasks, int j, cudaStream_t s) {
  const int elems = (160 * 1024) / 8;
  ensure_dyn_smem(gj_panel_kernel, (size_t)elems * 8);
  LAUNCH(gj_panel_kernel, ntasks, GJ_NT, (size_t)elems * 8, s, static_cast<const GJBTask*>(t), j, elems);
}
void launch_gj_fused(const void* t, int ntasks, int nmax, cudaStream_t s) {
  // the panel LU is staged in shared memory when it fits next to nothing else (it is dead by the
  // time the update tiles use the same buffer); capped so that two CTAs fit on an SM
  const int elems = std::max(GJF_TILE_DOUBLES, std::min(nmax * GJB, (72 * 1024) / 8));
  ensure_dyn_smem(gj_fused_kernel, (size_t)elems * 8);
  LAUNCH(gj_fused_kernel, ntasks, GJ_NT, (size_t)elems * 8, s, static_cast<const GJBTask*>(t), elems);
}
void launch_gj_unscramble(const void* t, int ntasks, int nmax, cudaStream_t s) {
  if (ntasks <= 0) return;
  dim3 grid(ntasks, (nmax + 127) / 128);
  if (g_before_launch) g_before_launch();
  gj_unscramble_kernel<<<grid, 128, 0, s>>>(static_cast<const GJBTask*>(t));
  AIFMM_CUDA(cudaGetLastError());
  ++g_launches;
}
size_t gjb_task_size() { return sizeof(GJBTask); }
void gjb_make(void* out, double* A, int lda, int n, double* PW, double* Bws, int* piv, int* info) {
  GJBTask* t = static_cast<GJBTask*>(out);
  *t = GJBTask{A, lda, n, PW, Bws, piv, info};
}

void launch_pqr_cluster(const PqrTask* t, int ntasks, cudaStream_t s) {
  const int cap = (200 * 1024) / 8;
  ensure_dyn_smem(pqr_cluster_kernel, (size_t)cap * 8);
  LAUNCH(pqr_cluster_kernel, ntasks * PQC, PQR_NT, (size_t)cap * 8, s, t, cap);
}

void launch_pqr(const PqrTask* t, int ntasks, size_t smem_doubles, cudaStream_t s) {
  size_t smem = smem_doubles * sizeof(double);
  AIFMM_REQUIRE(smem <= 227 * 1024, AIFMM_EOOM, "pivoted QR candidate matrix too wide for shared memory");
  ensure_dyn_smem(pqr_tasks_kernel, smem);
  LAUNCH(pqr_tasks_kernel, ntasks, PQR_NT, smem, s, t);
}

void launch_keval(const KEvalTask* t, int ntasks, int ysplit, const double* pts, KernelParams kp, int* flag,
                  cudaStream_t s) {
  if (ntasks <= 0) return;
  dim3 g(ntasks, ysplit);
  if (g_before_launch) g_before_launch();
  keval_tasks_kernel<<<g, 256, 0, s>>>(t, pts, kp, flag);
  AIFMM_CUDA(cudaGetLastError());
  ++g_launches;
}

void launch_copy(const CopyTask* t, int ntasks, int ysplit, cudaStream_t s) {
  if (ntasks <= 0) return;
  dim3 g(ntasks, ysplit);
  if (g_before_launch) g_before_launch();
  copy_tasks_kernel<<<g, 256, 0, s>>>(t);
  AIFMM_CUDA(cudaGetLastError());
  ++g_launches;
}

void launch_norm(const NormTask* t, int ntasks, cudaStream_t s) { LAUNCH(norm_tasks_kernel, ntasks, 256, 0, s, t); }

size_t hh_task_size() { return sizeof(HHTask); }
void hh_make(void* out, double* A, int lda, int n, int m, double* V, double* T) {
  *static_cast<HHTask*>(out) = HHTask{A, lda, n, m, V, T};
}
void launch_hh_panel(const void* t, int ntasks, int j, cudaStream_t s, int mode, int nmax) {
  // mode 0: one CTA; mode 1: 8-CTA cluster (global memory); mode 2: cluster, smem-staged;
  // mode 3: one CTA, smem-staged (rows <= HHS_ROWS)
  if (mode == 2) {
    const int cap_rows = (std::max(nmax - j, 1) + HHC - 1) / HHC;
    const size_t smem = (size_t)cap_rows * HHB * sizeof(double);
    ensure_dyn_smem(hh_panel_cluster_smem_kernel, smem);
    if (g_before_launch) g_before_launch();
    hh_panel_cluster_smem_kernel<<<ntasks * HHC, 256, smem, s>>>(static_cast<const HHTask*>(t), j, cap_rows);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      cudaFuncAttributes fa{};
      cudaFuncGetAttributes(&fa, hh_panel_cluster_smem_kernel);
      fprintf(stderr, "hh smem launch failed: %s smem=%zu static=%zu maxdyn=%d ntasks=%d j=%d nmax=%d\n", cudaGetErrorString(e),
              smem, fa.sharedSizeBytes, fa.maxDynamicSharedSizeBytes, ntasks, j, nmax);
      AIFMM_CUDA(e);
    }
    ++g_launches;
  } else if (mode == 5) {
    // register-resident panel on 8-CTA clusters (rows - j <= 8 x 256 RPT)
    const int chunk = (std::max(nmax - j, 1) + HHC_REG - 1) / HHC_REG;
    if (chunk <= HHR_NT) LAUNCH((hh_panel_reg_cluster_kernel<1, HHC_REG>), ntasks * HHC_REG, HHR_NT, 0, s, static_cast<const HHTask*>(t), j);
    else LAUNCH((hh_panel_reg_cluster_kernel<2, HHC_REG>), ntasks * HHC_REG, HHR_NT, 0, s, static_cast<const HHTask*>(t), j);
  } else if (mode == 6) {
    // register-resident panel on 2-CTA clusters (rows - j <= 2 x 512)
    LAUNCH((hh_panel_reg_cluster_kernel<2, 2>), ntasks * 2, HHR_NT, 0, s, static_cast<const HHTask*>(t), j);
  } else if (mode == 4) {
    // register-resident panel (rows - j <= 256 RPT); nmax = max rows of the batch
    if (nmax - j <= HHR_NT) LAUNCH(hh_panel_reg_kernel<1>, ntasks, HHR_NT, 0, s, static_cast<const HHTask*>(t), j);
    else LAUNCH(hh_panel_reg_kernel<2>, ntasks, HHR_NT, 0, s, static_cast<const HHTask*>(t), j);
  } else if (mode == 3) {
    // one CTA, panel in shared memory (rows - j <= HHS_ROWS)
    const size_t smem = (size_t)std::max(std::min(nmax - j, HHS_ROWS), 1) * HHB * sizeof(double);
    ensure_dyn_smem(hh_panel_smem_kernel, (size_t)HHS_ROWS * HHB * sizeof(double));
    LAUNCH(hh_panel_smem_kernel, ntasks, HHP_NT, smem, s, static_cast<const HHTask*>(t), j);
  } else if (mode == 1) {
    LAUNCH(hh_panel_cluster_kernel, ntasks * HHC, 256, 0, s, static_cast<const HHTask*>(t), j);
  } else {
    LAUNCH(hh_panel_kernel, ntasks, HHP_NT, 0, s, static_cast<const HHTask*>(t), j);
  }
}
void launch_hh_extract(const void* t, int ntasks, double* const* out, const int* ldo, cudaStream_t s) {
  LAUNCH(hh_extract_rt_kernel, ntasks, 256, 0, s, static_cast<const HHTask*>(t), out, ldo);
}

}  // namespace aifmm
