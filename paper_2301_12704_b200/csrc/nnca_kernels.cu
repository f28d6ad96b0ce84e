// nnca_kernels.cu — G3: NNCA pivot selection by ACA with partial pivoting, one CTA per box.
//
// Eq. NCA: row pivots t^{B,i} from the candidate rows R_B (points of B at the leaf,
// stacked child skeletons above, Eq. P:414-416), far pivots s^{B,i} from F_B = points of IL(B)
// (Eq. Fj).  The pivot rule is deferred by the paper; reading R9:
// ACA with partial pivoting, tie-window argmax (R7), stop when ||u_k|| ||v_k|| <= eps ||S_k||_F,
// reject a cross whose pivot is below GUARD * max|previous pivots|.  Same rule as oracle/nnca.py.
#include "common.cuh"

namespace aifmm {

struct AcaTask {
  const int* R;        // candidate rows: global (tree-order) point indices, nR
  const int* frange;   // far ranges: [2*i] = start, [2*i+1] = end (tree-order indices)
  int nR, nfr, nF, kmax;
  double* Uw;          // nR x kmax (ld nR)
  double* Vw;          // nF x kmax (ld nF)
  unsigned char* rused;
  unsigned char* cused;
  int* rank;           // out
  int* rpiv;           // out: global point index of row pivots (kmax)
  int* cpiv;           // out: global point index of column pivots (kmax)
};

constexpr int ACA_NT = 256;
constexpr double ACA_TIE = 1e-10;
constexpr double ACA_GUARD = 1e-13;
constexpr int ACA_MAXR = 256;   // far ranges per box held in shared memory

template <int NT>
__device__ __forceinline__ double bsum(double v, double* red) {
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
__device__ __forceinline__ double bmax(double v, double* red) {
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
__device__ __forceinline__ int bmin_int(int v, int* red) {
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

// tie-window argmax of |x| over entries with used[i] == 0; returns -1 if max == 0 (R7)
template <int NT>
__device__ int pick_tw(const double* x, const unsigned char* used, int n, double* red, int* redi) {
  double v = -1.0;
  for (int i = threadIdx.x; i < n; i += NT)
    if (!used[i]) v = fmax(v, fabs(x[i]));
  const double mx = bmax<NT>(v, red);
  if (!(mx > 0.0)) return -1;
  const double thr = mx * (1.0 - ACA_TIE);
  int cand = 0x7fffffff;
  for (int i = threadIdx.x; i < n; i += NT)
    if (!used[i] && fabs(x[i]) >= thr) { cand = i; break; }
  return bmin_int<NT>(cand, redi);
}

__device__ __forceinline__ int far_point(const int* pre, const int* st, int nfr, int j) {
  int lo = 0, hi = nfr - 1;
  while (lo < hi) {  // last range with pre[r] <= j
    int mid = (lo + hi + 1) >> 1;
    if (pre[mid] <= j) lo = mid; else hi = mid - 1;
  }
  return st[lo] + (j - pre[lo]);
}

__global__ void __launch_bounds__(ACA_NT) aca_kernel(const AcaTask* __restrict__ tasks, const double* __restrict__ pts,
                                                     KernelParams kp, double eps) {
  const AcaTask tk = tasks[blockIdx.x];
  __shared__ int pre[ACA_MAXR], st[ACA_MAXR];
  __shared__ double red[32];
  __shared__ int redi[32];
  __shared__ double sdot[2 * 512];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = ACA_NT / 32;
  const int nR = tk.nR, nF = tk.nF, nfr = tk.nfr;
  if (tid == 0) {
    int acc = 0;
    for (int r = 0; r < nfr; ++r) { pre[r] = acc; st[r] = tk.frange[2 * r]; acc += tk.frange[2 * r + 1] - tk.frange[2 * r]; }
  }
  for (int i = tid; i < nR; i += ACA_NT) tk.rused[i] = 0;
  for (int j = tid; j < nF; j += ACA_NT) tk.cused[j] = 0;
  __syncthreads();
  int k = 0, i = 0;
  double norm2 = 0.0, first = -1.0;
  const int kmax = tk.kmax;
  while (k < kmax) {
    if (tid == 0) tk.rused[i] = 1;
    const int gi = tk.R[i];
    double* v = tk.Vw + (size_t)k * nF;
    double* u = tk.Uw + (size_t)k * nR;
    // residual row r_j = A(R_i, F_j) - sum_t u_t[i] v_t[j]
    for (int j = tid; j < nF; j += ACA_NT) {
      double r = kernel_entry(kp, pts, gi, far_point(pre, st, nfr, j));
      for (int t = 0; t < k; ++t) r -= tk.Uw[(size_t)t * nR + i] * tk.Vw[(size_t)t * nF + j];
      v[j] = r;
    }
    __syncthreads();
    const int j = pick_tw<ACA_NT>(v, tk.cused, nF, red, redi);
    if (j < 0) {
      int cand = 0x7fffffff;
      for (int q = tid; q < nR; q += ACA_NT)
        if (!tk.rused[q]) { cand = q; break; }
      const int nxt = bmin_int<ACA_NT>(cand, redi);
      if (nxt == 0x7fffffff) break;
      i = nxt;
      continue;
    }
    const double delta = v[j];
    if (first >= 0.0 && fabs(delta) <= ACA_GUARD * first) break;
    first = (first < 0.0) ? fabs(delta) : fmax(first, fabs(delta));
    __syncthreads();
    for (int q = tid; q < nF; q += ACA_NT) v[q] = v[q] / delta;
    const int gj = far_point(pre, st, nfr, j);
    __syncthreads();
    for (int q = tid; q < nR; q += ACA_NT) {
      double c = kernel_entry(kp, pts, tk.R[q], gj);
      for (int t = 0; t < k; ++t) c -= tk.Vw[(size_t)t * nF + j] * tk.Uw[(size_t)t * nR + q];
      u[q] = c;
    }
    if (tid == 0) tk.cused[j] = 1;
    __syncthreads();
    // norms and cross terms
    double pu = 0.0, pv = 0.0;
    for (int q = tid; q < nR; q += ACA_NT) pu += u[q] * u[q];
    for (int q = tid; q < nF; q += ACA_NT) pv += v[q] * v[q];
    const double uu = bsum<ACA_NT>(pu, red);
    const double vv = bsum<ACA_NT>(pv, red);
    for (int t0 = 0; t0 < k; t0 += 512) {
      const int tn = min(512, k - t0);
      for (int t = warp; t < tn; t += NW) {
        const double* ut = tk.Uw + (size_t)(t0 + t) * nR;
        const double* vt = tk.Vw + (size_t)(t0 + t) * nF;
        double a = 0.0, b = 0.0;
        for (int q = lane; q < nR; q += 32) a += ut[q] * u[q];
        for (int q = lane; q < nF; q += 32) b += vt[q] * v[q];
        for (int o = 16; o > 0; o >>= 1) { a += __shfl_xor_sync(0xffffffffu, a, o); b += __shfl_xor_sync(0xffffffffu, b, o); }
        if (lane == 0) { sdot[2 * t] = a; sdot[2 * t + 1] = b; }
      }
      __syncthreads();
      if (tid == 0) {
        double cr = 0.0;
        for (int t = 0; t < tn; ++t) cr += sdot[2 * t] * sdot[2 * t + 1];
        red[31] = cr;
      }
      __syncthreads();
      norm2 += 2.0 * red[31];
      __syncthreads();
    }
    norm2 += uu * vv;
    if (tid == 0) { tk.rpiv[k] = gi; tk.cpiv[k] = gj; }
    ++k;
    if (sqrt(uu * vv) <= eps * sqrt(fmax(norm2, 0.0))) break;
    int nxt = pick_tw<ACA_NT>(u, tk.rused, nR, red, redi);
    if (nxt < 0) {
      int cand = 0x7fffffff;
      for (int q = tid; q < nR; q += ACA_NT)
        if (!tk.rused[q]) { cand = q; break; }
      nxt = bmin_int<ACA_NT>(cand, redi);
      if (nxt == 0x7fffffff) break;
    }
    i = nxt;
    __syncthreads();
  }
  if (tid == 0) *tk.rank = k;
}

void launch_aca(const AcaTask* t, int ntasks, const double* pts, KernelParams kp, double eps, cudaStream_t s) {
  LAUNCH(aca_kernel, ntasks, ACA_NT, 0, s, t, pts, kp, eps);
}

}  // namespace aifmm
