// common.cuh — shared device/host utilities of libaifmm (B200, sm_100a).
#pragma once
#include <unordered_map>
#include <cuda_runtime.h>
#include <stdint.h>
#include <string>
#include <vector>
#include <stdexcept>

#include "../../include/aifmm.h"

namespace aifmm {

struct Error : public std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define AIFMM_CUDA(call)                                                              \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess) {                                                          \
      if (e_ == cudaErrorMemoryAllocation)                                            \
        throw ::aifmm::Error(AIFMM_EOOM, std::string("out of device memory at ") +    \
                                            __FILE__ + ":" + std::to_string(__LINE__)); \
      throw ::aifmm::Error(AIFMM_ECUDA, std::string(cudaGetErrorString(e_)) + " at " + \
                                            __FILE__ + ":" + std::to_string(__LINE__)); \
    }                                                                                 \
  } while (0)

#define AIFMM_REQUIRE(cond, code, msg) \
  do { if (!(cond)) throw ::aifmm::Error((code), (msg)); } while (0)

// Launch bookkeeping: every kernel launch of the library goes through LAUNCH so that
// aifmm_stats can report how many of OUR kernels ran (bench "gpu_launches").
extern long long g_launches;
// Called before every kernel launch: uploads task lists staged since the previous launch in one
// host-to-device copy (Uploader::flush in the library context).  LAUNCH calls it before its
// arguments are evaluated, so a launch argument must never stage an upload itself.
extern void (*g_before_launch)();
#define LAUNCH(kernel, grid, block, smem, stream, ...)                \
  do {                                                                \
    if ((grid) > 0) {                                                 \
      if (::aifmm::g_before_launch) ::aifmm::g_before_launch();       \
      kernel<<<(grid), (block), (smem), (stream)>>>(__VA_ARGS__);     \
      AIFMM_CUDA(cudaGetLastError());                                 \
      ++::aifmm::g_launches;                                          \
    }                                                                 \
  } while (0)

// Raise a kernel's dynamic shared-memory limit when a launch needs more than it allows
// (the default allowance is 48 KB minus the kernel's static shared memory).
template <class F>
inline void ensure_dyn_smem(F* func, size_t bytes) {
  // the allowance already granted per kernel is cached (no driver query per launch)
  static thread_local std::unordered_map<const void*, int> granted;
  auto it = granted.find(reinterpret_cast<const void*>(func));
  if (it != granted.end() && (int)bytes <= it->second) return;
  cudaFuncAttributes fa{};
  AIFMM_CUDA(cudaFuncGetAttributes(&fa, func));
  int have = fa.maxDynamicSharedSizeBytes;
  if ((int)bytes > have) {
    AIFMM_CUDA(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    have = (int)bytes;
  }
  granted[reinterpret_cast<const void*>(func)] = have;
}

// ---------------------------------------------------------------------------------------
// Task records (built on the host by the planner, uploaded, consumed by batched kernels).
// All matrices are column-major; "ld" is the leading dimension.
// ---------------------------------------------------------------------------------------

// C[MxN] = beta*C + sum_t alpha_t * op(A_t)[MxK_t] * op(B_t)[K_txN]
// A term with A == nullptr is an addition  C += alpha_t * op(B_t) (B_t is M x N).
struct GemmTask {
  double* C;
  int ldc, M, N;
  double beta;
  int term_begin, term_end;
};
struct GemmTerm {
  const double* A;
  const double* B;
  int lda, ldb, K;
  int transA, transB;
  double alpha;
};
// One tile of one GEMM task (host-expanded so that a CTA finds its work in O(1)).
struct GemmTile {
  int task, m0, n0, pad;
};

// 2-D copy: dst[r,c] (+)= alpha * src[r,c]  (or src[c,r] if trans); src == nullptr writes alpha.
struct CopyTask {
  const double* src;
  double* dst;
  int lds, ldd, rows, cols;
  int trans, accumulate;
  double alpha;
};

// Gauss-Jordan with partial pivoting on an n x ncols column-major matrix (ncols >= n):
// [A | B] -> [I | A^{-1} B].  info: 0 ok, k+1 if the k-th pivot is exactly zero.
struct GJTask {
  double* A;
  int lda, n, ncols, pad;
  int* info;
};

// Kernel-entry block: out[i,j] = K(x_{rows[i]}, x_{cols[j]}) (diag value when equal).
// rows/cols == nullptr means the contiguous range row0 + i / col0 + j.
// Device view of the host planner's per-level block table entry (aifmm.cu Blk: same layout).
struct BlkDev {
  double* p;
  int ld, rows, cols;
};

struct KEvalTask {
  double* out;
  int ld, nr, nc;
  const int* rows;
  const int* cols;
  int row0, col0;
};

// Pivoted Gram-Schmidt extension (RRQR, reading R8 / R15): W (m x ncols) is the candidate
// matrix already projected against the basis Q[:, 0:k0]; new orthonormal columns are written
// to Q[:, k0 + t].  Takes pivots while t < tmin or ||W_t||_F > tau, never more than tmax.
struct PqrTask {
  double* W;
  double* Q;
  int ldw, ldq, m, ncols;
  int k0, tmin, tmax, pad;
  const double* fnorm;  // tau = tol * (*fnorm)  (fnorm may be nullptr -> tau = tol)
  double tol;
  int* t_trunc;         // first t at which ||W_t|| <= tau held (or taken count)
  int* t_taken;         // columns appended
};

// Cholesky G = R^T R of a k x k SPD block (ld k) and R^{-1}; info = 1 + failing step or 0.
struct CholTask {
  const double* G;
  double* R;
  double* Rinv;
  int k, pad;
  int* info;
};

// Frobenius norm of a column-major block (written to *out).
struct NormTask {
  const double* A;
  int lda, rows, cols;
  double* out;
};

// Kernel parameters shared by all entry evaluations.
struct KernelParams {
  int id, d;
  double diag, ell;
};

// Device-side helpers --------------------------------------------------------------------
__device__ __forceinline__ double kernel_entry(const KernelParams& kp, const double* __restrict__ pts,
                                               int i, int j) {
  if (i == j) return kp.diag;
  const double* a = pts + (size_t)i * kp.d;
  const double* b = pts + (size_t)j * kp.d;
  // r^2 evaluated left to right without FMA contraction (same rounding as the oracle)
  double dx = __dsub_rn(a[0], b[0]);
  double s = __dmul_rn(dx, dx);
  for (int t = 1; t < kp.d; ++t) {
    double dt = __dsub_rn(a[t], b[t]);
    s = __dadd_rn(s, __dmul_rn(dt, dt));
  }
  double r = sqrt(s);
  if (kp.id == 0) return log(r);
  if (kp.id == 1) return exp(-r / kp.ell);
  return 1.0 / r;
}

}  // namespace aifmm
