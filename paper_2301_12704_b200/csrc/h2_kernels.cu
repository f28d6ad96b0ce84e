// h2_kernels.cu — SURVEY §8(a) row a8: the NNCA (H2) matrix-vector product and the vector
// kernels of restarted GMRES (BASELINE config 5: AIFMM-preconditioned GMRES, §5
// Exp. 5 P:1628-1707).
//
//   kmv_kernel   : y_t (+)= sum_s K(rows_t, cols_s) x_s with the kernel entries evaluated on the
//                  fly (never stored): the M2L A(sk_B, sk_D) q_D sums and the near-field
//                  K_BX x_X sums.  One CTA per target block, sources staged through
//                  shared memory, fixed source order (deterministic).  FP64-ALU bound.
//   dot / axpy / scale / Givens / back substitution / gemv: GMRES(m) with modified
//                  Gram-Schmidt (the scalars stay on the device; the host reads one residual
//                  estimate per iteration for the stopping test).
#include <algorithm>

#include "common.cuh"

namespace aifmm {

struct KmvTarget {
  const int* rows;   // global tree-order point index per row, or nullptr: row0 + i
  int row0, nr;
  double* y;
  int ldy;
  int src_begin, src_end;
};
struct KmvSource {
  const int* cols;   // or nullptr: col0 + j
  int col0, nc;
  const double* x;
  int ldx;
  int pad;
};

constexpr int KMV_NT = 128;
constexpr int KMV_CH = 128;   // source columns staged per chunk
constexpr int KMV_R = 4;      // right-hand sides per register pass

__global__ void __launch_bounds__(KMV_NT) kmv_kernel(const KmvTarget* __restrict__ T, const KmvSource* __restrict__ S,
                                                     const double* __restrict__ pts, KernelParams kp, int nrhs,
                                                     int accumulate) {
  const KmvTarget tg = T[blockIdx.x];
  __shared__ double sc[KMV_CH * 3];
  __shared__ int sg[KMV_CH];
  __shared__ double sx[KMV_R][KMV_CH];
  const int d = kp.d;
  for (int r0 = 0; r0 < nrhs; r0 += KMV_R) {
    const int nr_r = min(KMV_R, nrhs - r0);
    for (int ib = 0; ib < tg.nr; ib += KMV_NT) {
      const int i = ib + threadIdx.x;
      const bool act = i < tg.nr;
      const int gi = act ? (tg.rows ? tg.rows[i] : tg.row0 + i) : 0;
      double xi[3] = {0.0, 0.0, 0.0};
      if (act)
        for (int a = 0; a < d; ++a) xi[a] = pts[(size_t)gi * d + a];
      double acc[KMV_R] = {0.0, 0.0, 0.0, 0.0};
      for (int s = tg.src_begin; s < tg.src_end; ++s) {
        const KmvSource src = S[s];
        for (int j0 = 0; j0 < src.nc; j0 += KMV_CH) {
          const int nj = min(KMV_CH, src.nc - j0);
          __syncthreads();
          for (int j = threadIdx.x; j < nj; j += KMV_NT) {
            const int gj = src.cols ? src.cols[j0 + j] : src.col0 + j0 + j;
            sg[j] = gj;
            for (int a = 0; a < d; ++a) sc[j * 3 + a] = pts[(size_t)gj * d + a];
            for (int r = 0; r < nr_r; ++r) sx[r][j] = src.x[(size_t)(r0 + r) * src.ldx + j0 + j];
          }
          __syncthreads();
          if (act) {
            for (int j = 0; j < nj; ++j) {
              double v;
              if (sg[j] == gi) {
                v = kp.diag;
              } else {
                // r^2 left to right without FMA contraction (same rounding as kernel_entry)
                double dx = __dsub_rn(xi[0], sc[j * 3]);
                double s2 = __dmul_rn(dx, dx);
                for (int a = 1; a < d; ++a) {
                  const double dt = __dsub_rn(xi[a], sc[j * 3 + a]);
                  s2 = __dadd_rn(s2, __dmul_rn(dt, dt));
                }
                const double rr = sqrt(s2);
                v = (kp.id == 0) ? log(rr) : (kp.id == 1) ? exp(-rr / kp.ell) : 1.0 / rr;
              }
#pragma unroll
              for (int r = 0; r < KMV_R; ++r)
                if (r < nr_r) acc[r] += v * sx[r][j];
            }
          }
        }
      }
      if (act)
        for (int r = 0; r < nr_r; ++r) {
          double* yp = tg.y + (size_t)(r0 + r) * tg.ldy + i;
          *yp = accumulate ? *yp + acc[r] : acc[r];
        }
    }
  }
}

void launch_kmv(const KmvTarget* t, const KmvSource* s, int ntargets, const double* pts, KernelParams kp, int nrhs,
                int accumulate, cudaStream_t st) {
  LAUNCH(kmv_kernel, ntargets, KMV_NT, 0, st, t, s, pts, kp, nrhs, accumulate);
}

// ------------------------------------------------------------------------------ GMRES vectors
constexpr int VEC_NT = 256;
constexpr int DOT_BLOCKS = 296;   // 2 x 148 SMs; fixed so the reduction order is fixed

__global__ void __launch_bounds__(VEC_NT) dot_partial_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                                             long long n, double* __restrict__ part) {
  __shared__ double red[VEC_NT / 32];
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)VEC_NT + threadIdx.x; i < n; i += (long long)DOT_BLOCKS * VEC_NT)
    s += a[i] * b[i];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < VEC_NT / 32; ++w) t += red[w];
    part[blockIdx.x] = t;
  }
}
// out = sum(part) (mode 0) or sqrt(sum(part)) (mode 1)
__global__ void dot_final_kernel(const double* __restrict__ part, double* __restrict__ out, int mode) {
  __shared__ double red[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < DOT_BLOCKS; i += 32) s += part[i];
  red[threadIdx.x] = s;
  __syncwarp();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 32; ++w) t += red[w];
    *out = mode ? sqrt(t) : t;
  }
}
// y = beta * y + sign * (*alpha or 1) * x
__global__ void axpy_kernel(double* __restrict__ y, const double* __restrict__ x, long long n, const double* alpha,
                            double sign, double beta) {
  const double a = sign * (alpha ? *alpha : 1.0);
  for (long long i = blockIdx.x * (long long)VEC_NT + threadIdx.x; i < n; i += (long long)gridDim.x * VEC_NT)
    y[i] = (beta == 0.0 ? 0.0 : beta * y[i]) + a * x[i];
}
// y = x / (*den)  (den == 0: y = 0)
__global__ void scale_div_kernel(double* __restrict__ y, const double* __restrict__ x, long long n, const double* den) {
  const double dv = *den;
  for (long long i = blockIdx.x * (long long)VEC_NT + threadIdx.x; i < n; i += (long long)gridDim.x * VEC_NT)
    y[i] = (dv != 0.0) ? x[i] / dv : 0.0;
}
// H[i, j] = dots[i] written by the MGS loop; apply the previous rotations to column j, form the
// new rotation, update g; res = |g[j+1]|
__global__ void givens_kernel(double* H, int ldh, double* cs, double* sn, double* g, int j, double* res) {
  if (threadIdx.x != 0) return;
  double* h = H + (size_t)j * ldh;
  for (int i = 0; i < j; ++i) {
    const double h0 = h[i], h1 = h[i + 1];
    h[i] = cs[i] * h0 + sn[i] * h1;
    h[i + 1] = -sn[i] * h0 + cs[i] * h1;
  }
  const double den = hypot(h[j], h[j + 1]);
  const double c = (den == 0.0) ? 1.0 : h[j] / den, s = (den == 0.0) ? 0.0 : h[j + 1] / den;
  cs[j] = c;
  sn[j] = s;
  h[j] = c * h[j] + s * h[j + 1];
  h[j + 1] = 0.0;
  g[j + 1] = -s * g[j];
  g[j] = c * g[j];
  *res = fabs(g[j + 1]);
}
// H[0:k,0:k] y = g[0:k] (upper triangular)
__global__ void backsub_kernel(const double* H, int ldh, const double* g, double* y, int k) {
  if (threadIdx.x != 0) return;
  for (int i = k - 1; i >= 0; --i) {
    double s = g[i];
    for (int c = i + 1; c < k; ++c) s -= H[(size_t)c * ldh + i] * y[c];
    y[i] = s / H[(size_t)i * ldh + i];
  }
}
// out[i] = sum_c V[i + c ldv] y[c]
__global__ void gemv_kernel(const double* __restrict__ V, long long ldv, const double* __restrict__ y, int k, long long n,
                            double* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)VEC_NT + threadIdx.x; i < n; i += (long long)gridDim.x * VEC_NT) {
    double s = 0.0;
    for (int c = 0; c < k; ++c) s += V[i + c * ldv] * y[c];
    out[i] = s;
  }
}
__global__ void set_scalar_kernel(double* dst, const double* src, double value) {
  if (threadIdx.x == 0) *dst = src ? *src : value;
}

// Direct-sum residual (verification only): part[s] holds the partial
// products A(rows, chunk_s) X of source chunk s (kmv_kernel); this sums them in chunk order and
// accumulates sum (y - b)^2 and sum b^2 over the sampled rows in a fixed order (one CTA).
constexpr int RES_NT = 1024;
__global__ void __launch_bounds__(RES_NT) resid_finish_kernel(const double* __restrict__ part, int nchunks, long long nrows,
                                                              int nrhs, const double* __restrict__ B, long long ldb,
                                                              const int* __restrict__ rows_user, double* __restrict__ out) {
  __shared__ double r1[RES_NT / 32], r2[RES_NT / 32];
  double a = 0.0, bb = 0.0;
  const long long tot = nrows * nrhs;
  for (long long e = threadIdx.x; e < tot; e += RES_NT) {
    const long long i = e % nrows, c = e / nrows;
    double y = 0.0;
    for (int s = 0; s < nchunks; ++s) y += part[(size_t)s * tot + e];
    const double b = B[(size_t)c * ldb + rows_user[i]];
    a += (y - b) * (y - b);
    bb += b * b;
  }
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    bb += __shfl_xor_sync(0xffffffffu, bb, o);
  }
  if ((threadIdx.x & 31) == 0) { r1[threadIdx.x >> 5] = a; r2[threadIdx.x >> 5] = bb; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t1 = 0.0, t2 = 0.0;
    for (int w = 0; w < RES_NT / 32; ++w) { t1 += r1[w]; t2 += r2[w]; }
    out[0] = t1;
    out[1] = t2;
  }
}
void resid_finish(const double* part, int nchunks, long long nrows, int nrhs, const double* B, long long ldb,
                  const int* rows_user, double* out, cudaStream_t s) {
  LAUNCH(resid_finish_kernel, 1, RES_NT, 0, s, part, nchunks, nrows, nrhs, B, ldb, rows_user, out);
}

static int vgrid(long long n) { return (int)std::min<long long>(std::max<long long>((n + VEC_NT - 1) / VEC_NT, 1), 148 * 8); }
void vec_dot(const double* a, const double* b, long long n, double* part, double* out, int sqrt_mode, cudaStream_t s) {
  LAUNCH(dot_partial_kernel, DOT_BLOCKS, VEC_NT, 0, s, a, b, n, part);
  LAUNCH(dot_final_kernel, 1, 32, 0, s, part, out, sqrt_mode);
}
void vec_axpy(double* y, const double* x, long long n, const double* alpha, double sign, double beta, cudaStream_t s) {
  LAUNCH(axpy_kernel, vgrid(n), VEC_NT, 0, s, y, x, n, alpha, sign, beta);
}
void vec_scale_div(double* y, const double* x, long long n, const double* den, cudaStream_t s) {
  LAUNCH(scale_div_kernel, vgrid(n), VEC_NT, 0, s, y, x, n, den);
}
void gm_givens(double* H, int ldh, double* cs, double* sn, double* g, int j, double* res, cudaStream_t s) {
  LAUNCH(givens_kernel, 1, 32, 0, s, H, ldh, cs, sn, g, j, res);
}
void gm_backsub(const double* H, int ldh, const double* g, double* y, int k, cudaStream_t s) {
  LAUNCH(backsub_kernel, 1, 32, 0, s, H, ldh, g, y, k);
}
void gm_gemv(const double* V, long long ldv, const double* y, int k, long long n, double* out, cudaStream_t s) {
  LAUNCH(gemv_kernel, vgrid(n), VEC_NT, 0, s, V, ldv, y, k, n, out);
}
void set_scalar(double* dst, const double* src, double value, cudaStream_t s) {
  LAUNCH(set_scalar_kernel, 1, 32, 0, s, dst, src, value);
}

}  // namespace aifmm
