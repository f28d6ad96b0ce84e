// nnca_kernels.cu — G3: NNCA pivot selection by ACA with partial pivoting, one CTA per box.
//
// Eq. NCA: row pivots t^{B,i} from the candidate rows R_B (points of B at the leaf,
// stacked child skeletons above, Eq. P:414-416), far pivots s^{B,i} from F_B = sources of IL(B)
// (Eq. Fj; reading R11b: IL points at the leaf level, the IL boxes' children's skeletons above).  The pivot rule is deferred by the paper; reading R9:
// ACA with partial pivoting, tie-window argmax (R7), stop when ||u_k|| ||v_k|| <= eps ||S_k||_F,
// reject a cross whose pivot is below GUARD * max|previous pivots|.  Same rule as oracle/nnca.py.
#include <algorithm>
#include <cooperative_groups.h>

#include "common.cuh"

namespace aifmm {

struct AcaTask {
  const int* R;        // candidate rows: global (tree-order) point indices, nR
  const int* frange;   // far ranges: [2*i] = start, [2*i+1] = end (positions in fidx)
  const int* fidx;     // far source index array (nullptr: identity = tree-order point index)
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
#ifndef ACA_JB_DEF
#define ACA_JB_DEF 4
#endif
constexpr int ACA_JB = ACA_JB_DEF;   // residual-row columns per thread in flight

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

__device__ __forceinline__ int far_point(const int* pre, const int* st, int nfr, int j, const int* fidx) {
  int lo = 0, hi = nfr - 1;
  while (lo < hi) {  // last range with pre[r] <= j
    int mid = (lo + hi + 1) >> 1;
    if (pre[mid] <= j) lo = mid; else hi = mid - 1;
  }
  const int pos = st[lo] + (j - pre[lo]);
  return fidx ? fidx[pos] : pos;
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
    // residual row r_j = A(R_i, F_j) - sum_t u_t[i] v_t[j]; ACA_JB columns per thread in flight
    // (independent chains: more loads of the cross history outstanding; each r_j still
    // subtracts its terms in ascending t)
    for (int j0 = tid; j0 < nF; j0 += ACA_NT * ACA_JB) {
      double r[ACA_JB];
#pragma unroll
      for (int b = 0; b < ACA_JB; ++b) {
        const int jj = j0 + b * ACA_NT;
        r[b] = jj < nF ? kernel_entry(kp, pts, gi, far_point(pre, st, nfr, jj, tk.fidx)) : 0.0;
      }
      const double* Ui = tk.Uw + i;
      for (int t = 0; t < k; ++t) {
        const double ut = Ui[(size_t)t * nR];
        const double* Vt = tk.Vw + (size_t)t * nF;
#pragma unroll
        for (int b = 0; b < ACA_JB; ++b)
          if (j0 + b * ACA_NT < nF) r[b] -= ut * Vt[j0 + b * ACA_NT];
      }
#pragma unroll
      for (int b = 0; b < ACA_JB; ++b)
        if (j0 + b * ACA_NT < nF) v[j0 + b * ACA_NT] = r[b];
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
    const int gj = far_point(pre, st, nfr, j, tk.fidx);
    __syncthreads();
    // residual column, two rows per thread in flight (each c_q in ascending t)
    for (int q0 = tid; q0 < nR; q0 += 2 * ACA_NT) {
      const int q1 = q0 + ACA_NT;
      double c0 = kernel_entry(kp, pts, tk.R[q0], gj);
      double c1 = q1 < nR ? kernel_entry(kp, pts, tk.R[q1], gj) : 0.0;
      const double* Vj = tk.Vw + j;
      for (int t = 0; t < k; ++t) {
        const double vt = Vj[(size_t)t * nF];
        const double* Ut = tk.Uw + (size_t)t * nR;
        c0 -= vt * Ut[q0];
        if (q1 < nR) c1 -= vt * Ut[q1];
      }
      u[q0] = c0;
      if (q1 < nR) u[q1] = c1;
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

// Cluster variant for boxes with a long far set (upper levels, 3D): the ACA_C CTAs of a cluster
// own contiguous slices of the far columns F and of the candidate rows R; residual rows/columns,
// norms and cross terms are computed slice-wise and combined through distributed shared memory.
// Same decision rule as aca_kernel (tie-window argmax R7, guard, stopping test); only the
// summation order of the norms differs (rank-ordered partial sums, identical on every CTA).
constexpr int ACA_C = 8;
constexpr int ACA_CH = 256;   // cross-term chunk
struct AcaShared {
  double dv[2][4];            // per-phase published scalars
  int iv[2][2];
  double av[2][ACA_CH], bv[2][ACA_CH];
};

__global__ void __cluster_dims__(ACA_C, 1, 1) __launch_bounds__(ACA_NT)
aca_cluster_kernel(const AcaTask* __restrict__ tasks, const double* __restrict__ pts, KernelParams kp, double eps) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  const AcaTask tk = tasks[blockIdx.x / ACA_C];
  __shared__ int pre[ACA_MAXR], st[ACA_MAXR];
  __shared__ double red[32];
  __shared__ int redi[32];
  __shared__ AcaShared sh;
  extern __shared__ double aca_dyn[];   // ucol[kmax] | vrow[kmax]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = ACA_NT / 32;
  const int nR = tk.nR, nF = tk.nF, nfr = tk.nfr, kmax = tk.kmax;
  double* urow = aca_dyn;          // Uw[i, 0:k]  (row i of U)
  double* vcol = aca_dyn + kmax;   // Vw[j, 0:k]
  const int fw = (nF + ACA_C - 1) / ACA_C, f0 = min(nF, rank * fw), f1 = min(nF, f0 + fw);
  const int rw = (nR + ACA_C - 1) / ACA_C, r0 = min(nR, rank * rw), r1 = min(nR, r0 + rw);
  if (tid == 0) {
    int acc = 0;
    for (int r = 0; r < nfr; ++r) { pre[r] = acc; st[r] = tk.frange[2 * r]; acc += tk.frange[2 * r + 1] - tk.frange[2 * r]; }
  }
  for (int i = r0 + tid; i < r1; i += ACA_NT) tk.rused[i] = 0;
  for (int j = f0 + tid; j < f1; j += ACA_NT) tk.cused[j] = 0;
  int ph = 0;
  // cluster reductions (double-buffered by phase: one cluster barrier each)
  auto cl_max = [&](double v) {
    v = bmax<ACA_NT>(v, red);
    if (tid == 0) sh.dv[ph][0] = v;
    cl.sync();
    double m = -1.0;
    for (int q = 0; q < ACA_C; ++q) m = fmax(m, cl.map_shared_rank(&sh, q)->dv[ph][0]);
    ph ^= 1;
    return m;
  };
  auto cl_min_int = [&](int v) {
    v = bmin_int<ACA_NT>(v, redi);
    if (tid == 0) sh.iv[ph][0] = v;
    cl.sync();
    int m = 0x7fffffff;
    for (int q = 0; q < ACA_C; ++q) m = min(m, cl.map_shared_rank(&sh, q)->iv[ph][0]);
    ph ^= 1;
    return m;
  };
  // tie-window argmax over a sliced vector (global positions [a0, a1) local to this CTA); the
  // winner's value travels with its index (no CTA reads another CTA's slice of x)
  auto cl_pick = [&](const double* x, const unsigned char* used, int a0, int a1, double* val) {
    double v = -1.0;
    for (int i = a0 + tid; i < a1; i += ACA_NT)
      if (!used[i]) v = fmax(v, fabs(x[i]));
    const double mx = cl_max(v);
    if (!(mx > 0.0)) return -1;
    const double thr = mx * (1.0 - ACA_TIE);
    int cand = 0x7fffffff;
    for (int i = a0 + tid; i < a1; i += ACA_NT)
      if (!used[i] && fabs(x[i]) >= thr) { cand = i; break; }
    cand = bmin_int<ACA_NT>(cand, redi);
    if (tid == 0) {
      sh.iv[ph][0] = cand;
      sh.dv[ph][3] = (cand != 0x7fffffff) ? x[cand] : 0.0;
    }
    cl.sync();
    int best = 0x7fffffff;
    double bv = 0.0;
    for (int q = 0; q < ACA_C; ++q) {
      const AcaShared* o = cl.map_shared_rank(&sh, q);
      if (o->iv[ph][0] < best) { best = o->iv[ph][0]; bv = o->dv[ph][3]; }
    }
    ph ^= 1;
    *val = bv;
    return best;
  };
  auto first_free_row = [&]() {
    int cand = 0x7fffffff;
    for (int q = r0 + tid; q < r1; q += ACA_NT)
      if (!tk.rused[q]) { cand = q; break; }
    return cl_min_int(cand);
  };
  __syncthreads();
  cl.sync();
  int k = 0, i = 0;
  double norm2 = 0.0, first = -1.0;
  while (k < kmax) {
    if (i >= r0 && i < r1 && tid == 0) tk.rused[i] = 1;
    const int gi = tk.R[i];
    double* v = tk.Vw + (size_t)k * nF;
    double* u = tk.Uw + (size_t)k * nR;
    // row i / column j may belong to another CTA's slice: read around L1 (__ldcg)
    for (int t = tid; t < k; t += ACA_NT) urow[t] = __ldcg(tk.Uw + (size_t)t * nR + i);
    __syncthreads();
    for (int j = f0 + tid; j < f1; j += ACA_NT) {
      double r = kernel_entry(kp, pts, gi, far_point(pre, st, nfr, j, tk.fidx));
      for (int t = 0; t < k; ++t) r -= urow[t] * tk.Vw[(size_t)t * nF + j];
      v[j] = r;
    }
    __syncthreads();
    double delta = 0.0;
    const int j = cl_pick(v, tk.cused, f0, f1, &delta);
    if (j < 0) {
      const int nxt = first_free_row();
      if (nxt == 0x7fffffff) break;
      i = nxt;
      continue;
    }
    if (first >= 0.0 && fabs(delta) <= ACA_GUARD * first) break;
    first = (first < 0.0) ? fabs(delta) : fmax(first, fabs(delta));
    for (int t = tid; t < k; t += ACA_NT) vcol[t] = __ldcg(tk.Vw + (size_t)t * nF + j);
    __syncthreads();
    const int gj = far_point(pre, st, nfr, j, tk.fidx);
    double pv = 0.0;
    for (int q = f0 + tid; q < f1; q += ACA_NT) {
      const double x = v[q] / delta;
      v[q] = x;
      pv += x * x;
    }
    double pu = 0.0;
    for (int q = r0 + tid; q < r1; q += ACA_NT) {
      double cc = kernel_entry(kp, pts, tk.R[q], gj);
      for (int t = 0; t < k; ++t) cc -= vcol[t] * tk.Uw[(size_t)t * nR + q];
      u[q] = cc;
      pu += cc * cc;
    }
    if (j >= f0 && j < f1 && tid == 0) tk.cused[j] = 1;
    pu = bsum<ACA_NT>(pu, red);
    pv = bsum<ACA_NT>(pv, red);
    // cross terms sum_t (U_t . u)(V_t . v) over slices, chunked
    double cross = 0.0;
    for (int t0 = 0; t0 < k || t0 == 0; t0 += ACA_CH) {
      const int tn = min(ACA_CH, k - t0);
      for (int t = warp; t < tn; t += NW) {
        const double* ut = tk.Uw + (size_t)(t0 + t) * nR;
        const double* vt = tk.Vw + (size_t)(t0 + t) * nF;
        double a = 0.0, b = 0.0;
        for (int q = r0 + lane; q < r1; q += 32) a += ut[q] * u[q];
        for (int q = f0 + lane; q < f1; q += 32) b += vt[q] * v[q];
        for (int o = 16; o > 0; o >>= 1) { a += __shfl_xor_sync(0xffffffffu, a, o); b += __shfl_xor_sync(0xffffffffu, b, o); }
        if (lane == 0) { sh.av[ph][t] = a; sh.bv[ph][t] = b; }
      }
      if (tid == 0) { sh.dv[ph][1] = pu; sh.dv[ph][2] = pv; }
      __syncthreads();
      cl.sync();   // publishes u, v slices, partial dots and norms
      if (tid == 0) {
        double cr = 0.0;
        for (int t = 0; t < tn; ++t) {
          double a = 0.0, b = 0.0;
          for (int q = 0; q < ACA_C; ++q) {
            const AcaShared* o = cl.map_shared_rank(&sh, q);
            a += o->av[ph][t];
            b += o->bv[ph][t];
          }
          cr += a * b;
        }
        if (t0 == 0) {
          double uu = 0.0, vv = 0.0;
          for (int q = 0; q < ACA_C; ++q) {
            const AcaShared* o = cl.map_shared_rank(&sh, q);
            uu += o->dv[ph][1];
            vv += o->dv[ph][2];
          }
          red[30] = uu;
          red[29] = vv;
        }
        red[31] = cr;
      }
      __syncthreads();
      cross += red[31];
      ph ^= 1;
      if (tn <= 0) break;
    }
    const double uu = red[30], vv = red[29];
    __syncthreads();
    norm2 += 2.0 * cross;
    norm2 += uu * vv;
    if (rank == 0 && tid == 0) { tk.rpiv[k] = gi; tk.cpiv[k] = gj; }
    ++k;
    if (sqrt(uu * vv) <= eps * sqrt(fmax(norm2, 0.0))) break;
    double unused_val;
    int nxt = cl_pick(u, tk.rused, r0, r1, &unused_val);
    if (nxt < 0) {
      nxt = first_free_row();
      if (nxt == 0x7fffffff) break;
    }
    i = nxt;
  }
  if (rank == 0 && tid == 0) *tk.rank = k;
  cl.sync();
}

void launch_aca(const AcaTask* t, int ntasks, const double* pts, KernelParams kp, double eps, cudaStream_t s) {
  // experiment toggle: unused dynamic shared memory (KB) per CTA to cap the number of resident
  // boxes, so that their cross histories (V: k x nF each) stay in L2
  static const int pad_kb = getenv("AIFMM_ACA_SMEM_KB") ? atoi(getenv("AIFMM_ACA_SMEM_KB")) : 0;
  const size_t smem = (size_t)pad_kb * 1024;
  if (smem) ensure_dyn_smem(aca_kernel, smem);
  LAUNCH(aca_kernel, ntasks, ACA_NT, smem, s, t, pts, kp, eps);
}
void launch_aca_cluster(const AcaTask* t, int ntasks, int kmax, const double* pts, KernelParams kp, double eps,
                        cudaStream_t s) {
  const size_t smem = (size_t)2 * std::max(kmax, 1) * sizeof(double);
  ensure_dyn_smem(aca_cluster_kernel, smem);
  LAUNCH(aca_cluster_kernel, ntasks * ACA_C, ACA_NT, smem, s, t, pts, kp, eps);
}

}  // namespace aifmm
