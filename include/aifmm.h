/*
 * aifmm.h — C-ABI of libaifmm.so, the B200 (sm_100a) AIFMM hot path.
 *
 * The operation (PAPER.md, cited as P:<line>):
 *   Solve A x = b for dense N-body matrices A_ij = K(x_i, x_j) (problem statement
 *   P:105-111; targets = sources) with the Algebraic Inverse Fast Multipole
 *   Method: a 2^d tree (§2.1), strong admissibility / interaction lists
 *   (§2.2), NNCA far-field operators (§2.3 Eq. NCA), the extended
 *   sparse system (§3.1), level-by-level elimination with deferred (Alg. 3,
 *   P:1107-1164) compression and redirection of far fill-ins (§3.2.1-3.2.3),
 *   and back substitution (Alg. 4).  The factorization is independent of b
 *   (Remark P:1186-1188): build + factor once, solve many times.
 *
 * Conventions
 *   - One implicit context per process (one process per GPU), one CUDA stream.  Calls are
 *     serialised by the caller, including solves of one factorization from several host
 *     threads (they share the context's workspace); there is no internal locking.  The Python
 *     binding runs every call on torch's current stream (aifmm_set_stream).
 *   - "device" pointers are CUDA device pointers on the current device; "host" pointers
 *     are ordinary (pageable or pinned) host memory.
 *   - Matrices are column-major.  Points are N x d row-major (point i at points[i*d]).
 *   - Every function returns 0 on success or a negative AIFMM_E* code; the message is
 *     available from aifmm_last_error().  No C++ exception crosses this boundary.
 *   - Floating point is IEEE binary64 throughout (the paper's double / BASELINE FP64).
 */
#ifndef AIFMM_H
#define AIFMM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Error codes. */
#define AIFMM_OK                   0
#define AIFMM_EINVALID_ARG        -1  /* n < 1, d not 2|3, leaf_size < 1, tol not in (0,1), nrhs < 1, NULL */
#define AIFMM_ENONFINITE          -2  /* NaN/Inf in points or B                                         */
#define AIFMM_ECOINCIDENT         -3  /* two coincident points with a singular kernel (log r, 1/r)      */
#define AIFMM_ESINGULAR_SKELETON  -4  /* NNCA skeleton block A(fp, sk) singular                          */
#define AIFMM_ESINGULAR_PIVOT     -5  /* a box pivot [[K, U],[V^*, 0]] or the top system is singular     */
#define AIFMM_ESTATE              -6  /* factor before build, solve before factor                        */
#define AIFMM_ECUDA               -7  /* CUDA runtime error                                              */
#define AIFMM_ENCCL               -8  /* NCCL error (multi-GPU)                                          */
#define AIFMM_EOOM                -9  /* device memory exhausted                                         */

/* Kernel ids (BASELINE.json configs; kparams = {diag, ell}):
 *   0  log r         A_ii = diag            (configs 1, 2)
 *   1  exp(-r/ell)   A_ii = diag (1+nugget) (config 3, Matern-1/2)
 *   2  1/r           A_ii = diag            (configs 4, 5; paper Exp. 3 with diag sqrt(1000N)) */

/* aifmm_build — tree, lists, colouring and NNCA operators (the paper's assembly, T_Aa).
 *   points    device, n x d row-major float64, user order.  Copied; the caller may free it
 *             after the call returns.
 *   n, d      number of points (>= 1), dimension (2 or 3).
 *   kernel_id 0|1|2 (above).  kparams: host, 2 doubles {diag, ell}.
 *   leaf_size n_max: leaves hold no more than n_max points, depth L >= 2.
 *   tol       eps_A in (0,1): NNCA (ACA at tol/100, reading R18) and RRQR truncation tol.
 * Discards any previous build/factorization.  Errors: EINVALID_ARG, ENONFINITE,
 * ECOINCIDENT, ESINGULAR_SKELETON, ECUDA, EOOM. */
int aifmm_build(const double* points, int64_t n, int d, int kernel_id,
                const double* kparams, int leaf_size, double tol);

/* aifmm_set_compression_tol — optional, before aifmm_factor: the fill-in truncation
 * tolerance tol_c (default = tol).  tol_c = 0 keeps every fill-in direction (exact
 * redirection; used by the tests to separate NNCA error from compression error). */
int aifmm_set_compression_tol(double tol_c);

/* aifmm_set_algorithm — optional, before aifmm_factor (default 3, kept across builds):
 *   3  Algorithm 3: far fill-ins accumulated and compressed / redirected once,
 *      just before one of their boxes is eliminated (the paper's efficient variant);
 *   2  Algorithm 2: fill-ins compressed as soon as they are created or updated,
 *      here right after the colour whose eliminations created them (the
 *      ablation of P:1090-1096).  Same results up to O(tol); more compressions.
 * Errors: EINVALID_ARG. */
int aifmm_set_algorithm(int alg);

/* aifmm_factor — elimination with colour-batched Algorithm 3 (T_Af).
 * Needs a successful build.  Errors: ESTATE, ESINGULAR_PIVOT, ECUDA, EOOM. */
int aifmm_factor(void);

/* aifmm_solve — Algorithm 4 for nrhs right-hand sides (T_As).
 *   B     device, n x nrhs column-major (ld = n), user order; overwritten by X.
 *   nrhs  >= 1.
 * Errors: ESTATE, EINVALID_ARG, ENONFINITE, ECUDA, EOOM. */
int aifmm_solve(double* B, int nrhs);

/* aifmm_solve_host — the same through host buffers: B (host, n x nrhs column-major) is
 * copied to the device, solved and copied back (end-to-end path used by bench.py e2e). */
int aifmm_solve_host(double* B, int nrhs);

/* aifmm_free — release every device buffer of the context. */
void aifmm_free(void);

/* aifmm_last_error — message of the last failing call ("" if none). Owned by the library. */
const char* aifmm_last_error(void);

/* aifmm_set_stream — optional: run on the given cudaStream_t (default: a library stream). */
int aifmm_set_stream(void* stream);

/* Introspection for parity tests (integer outputs are bit-exact with the oracle). */
/* aifmm_get_tree — perm: host int64[n] (perm[j] = user index of the j-th point in tree
 * order); L: host int*; either may be NULL. */
int aifmm_get_tree(int64_t* perm, int* L);
/* aifmm_get_level_offsets — host int64[2^(d*level)+1]: point offsets of every box. */
int aifmm_get_level_offsets(int level, int64_t* off);
/* aifmm_get_lists — CSR over the 2^(d*level) boxes (empty boxes have empty lists):
 * n_ptr/il_ptr host int32[2^(d*level)+1]; n_idx/il_idx host int32 of size n_ptr[last] /
 * il_ptr[last] (query sizes first by passing NULL idx arrays).  Lists are Morton-sorted. */
int aifmm_get_lists(int level, int32_t* n_ptr, int32_t* n_idx, int32_t* il_ptr, int32_t* il_idx);
/* aifmm_get_colours — host int32[2^(d*level)]: colour of each box (-1 for empty boxes). */
int aifmm_get_colours(int level, int32_t* colour);
/* aifmm_get_ranks — host int32[2^(d*level)]: NNCA rank (which = 0) or final rank after
 * factorization (which = 1) of every box (0 for empty boxes). */
int aifmm_get_ranks(int level, int which, int32_t* ranks);

/* aifmm_get_skeletons — the NNCA skeletons sk(B) = t^{B,i} (row pivots, R10) and
 * far pivots fp(B) = s^{B,i} of every box at `level`, as tree-order point indices, in pivot
 * order: CSR with sk_ptr host int32[2^(d*level)+1] (sk_ptr[b+1]-sk_ptr[b] = NNCA rank of b);
 * sk_idx / fp_idx host int32[sk_ptr[last]] or NULL (query the sizes first). */
int aifmm_get_skeletons(int level, int32_t* sk_ptr, int32_t* sk_idx, int32_t* fp_idx);

/* ---- Row a8 (BASELINE config 5): H2 matvec and AIFMM-preconditioned GMRES --------------
 * aifmm_matvec_build — build a second NNCA (ACA tolerance tol/100, reading R18) on the tree of
 *   the last aifmm_build, for the H2 matrix-vector product (Eq. NCA P:347-367 with the nested
 *   operators of Table; §5 Exp. 5 uses an FMM matvec inside GMRES,
 *   P:1628-1707).  Requires aifmm_build.  Owned by the library until the next build / free.
 * aifmm_matvec — Y = A_H2 X.  X, Y: device, N x nrhs column-major (ld N), user point order;
 *   X is read, Y is overwritten; they must not alias.  Near field and M2L kernel entries are
 *   evaluated on the fly (never stored).  AIFMM_ESTATE before aifmm_matvec_build.
 * aifmm_gmres — solve A x = b by restarted GMRES(restart) (modified Gram-Schmidt, Givens),
 *   matrix = the H2 matvec, right preconditioner: precond = 1 the AIFMM factorization
 *   (aifmm_solve; requires aifmm_factor), precond = 2 the leaf block-diagonal inverse
 *   blockdiag(A(points(b), points(b)))^-1 (the paper's block-diagonal comparison, P:1628-1629,
 *   table; blocks evaluated exactly and inverted on the first use), precond = 0
 *   none; stopping when ||b - A x|| / ||b|| <= rtol (Arnoldi
 *   estimate inside a cycle, true residual at each restart) or after maxit iterations.
 *   b (read) and x (written): device, N doubles, user order.  iters / relres: host out.
 *   AIFMM_ENONFINITE for a non-finite b. */
int aifmm_matvec_build(double tol);
int aifmm_matvec(const double* X, double* Y, int nrhs);
int aifmm_gmres(const double* b, double* x, int restart, double rtol, int maxit, int precond,
                int* iters, double* relres);

/* aifmm_residual — row a9 (verification; not part of the timed path): the relative residual
 *   ||A X - B||_F / ||B||_F of a solution X over the sampled rows, with A_ij = K(x_i, x_j) and
 *   A_ii = diag evaluated exactly by direct sum (the problem statement P:105-111; the paper's
 *   accuracy metric is a relative error in the 2-norm).
 *   X, B   device, n x nrhs column-major (ld n), user point order; read only.
 *   rows   host int64[nrows] user row indices (NULL: every row, nrows ignored).
 *   rel    host out.  Deterministic (fixed reduction order).
 * Requires aifmm_build.  Errors: ESTATE, EINVALID_ARG (NULL pointer, nrhs < 1, row out of
 * range), ECUDA, EOOM.  Cost: nrows x n kernel evaluations per right-hand side group of 4. */
int aifmm_residual(const double* X, const double* B, int nrhs, const int64_t* rows, int64_t nrows, double* rel);

/* aifmm_stats — host double[AIFMM_NSTATS], see the AIFMM_STAT_* indices. */
#define AIFMM_NSTATS 42
#define AIFMM_STAT_BUILD_MS        0
#define AIFMM_STAT_FACTOR_MS       1
#define AIFMM_STAT_SOLVE_MS        2
#define AIFMM_STAT_LEVELS          3
#define AIFMM_STAT_TOP_SIZE        4
#define AIFMM_STAT_FACTOR_FLOPS    5   /* algorithmic FLOPs of the factorization (model) */
#define AIFMM_STAT_SCHUR_FLOPS     6   /* FLOPs of the Schur-update GEMM launches                        */
#define AIFMM_STAT_SCHUR_MS        7   /* device time of the Schur-update GEMM launches (CUDA events)    */
#define AIFMM_STAT_LAUNCHES        8   /* kernels launched by the library since the last reset           */
#define AIFMM_STAT_COMPRESSIONS    9
#define AIFMM_STAT_MAX_RANK       10
#define AIFMM_STAT_DEVICE_BYTES   11
#define AIFMM_STAT_SCHUR_BYTES    12   /* algorithmic bytes of the Schur-update launches                */
#define AIFMM_STAT_SCHUR_LAUNCHES 13
#define AIFMM_STAT_SOLVE_BYTES    14
#define AIFMM_STAT_HOST_SYNCS     15
/* per-phase device time (CUDA events around the phase's launches, recorded when
 * aifmm_set_timing(1)) and algorithmic FLOPs / bytes of the last factorization:
 * pivot factorisations (P_i of P:753), Householder first stage and truncated pivoted QR of the
 * RRQR, redirection GEMMs */
#define AIFMM_STAT_PIVOT_MS       16
#define AIFMM_STAT_PIVOT_FLOPS    17
#define AIFMM_STAT_PIVOT_BYTES    18
#define AIFMM_STAT_TRI_MS         19
#define AIFMM_STAT_TRI_FLOPS      20
#define AIFMM_STAT_TRI_BYTES      21
#define AIFMM_STAT_PQR_MS         22
#define AIFMM_STAT_PQR_FLOPS      23
#define AIFMM_STAT_PQR_BYTES      24
#define AIFMM_STAT_REDIR_MS       25
#define AIFMM_STAT_REDIR_FLOPS    26
#define AIFMM_STAT_REDIR_BYTES    27
/* multipliers W_i = G_i[:, 0:m] R_i, compression projections (I - U U^T) F, the new blocks
 * of an elimination (C_p G12, G21 R_q, -G22), the level-start orthonormalisation (R13)
 * (device time includes host planning gaps inside the phase) */
#define AIFMM_STAT_MULT_MS        28
#define AIFMM_STAT_MULT_FLOPS     29
#define AIFMM_STAT_MULT_BYTES     30
#define AIFMM_STAT_PROJ_MS        31
#define AIFMM_STAT_PROJ_FLOPS     32
#define AIFMM_STAT_PROJ_BYTES     33
#define AIFMM_STAT_FRESH_MS       34
#define AIFMM_STAT_FRESH_FLOPS    35
#define AIFMM_STAT_FRESH_BYTES    36
#define AIFMM_STAT_ORTH_MS        37
#define AIFMM_STAT_ORTH_FLOPS     38
#define AIFMM_STAT_ORTH_BYTES     39
/* multi-GPU (aifmm_dist_init): bytes this rank received in ownership exchanges during the
 * last factorization, and the number of exchanges */
#define AIFMM_STAT_DIST_BYTES     40
#define AIFMM_STAT_DIST_EXCHANGES 41
int aifmm_stats(double* out);
/* aifmm_reset_counters — zero the launch / FLOP / time counters. */
int aifmm_reset_counters(void);
/* aifmm_set_timing — 1: record CUDA events around the Schur launches (for bench roofline). */
int aifmm_set_timing(int on);

/* ---- the factorization split across ranks (one process per GPU) ------------
 * The paper's per-level loop (Alg. 3) runs colour by colour; the boxes of one
 * colour are independent (Remark P:402-404), so their work is split by subtree: the points (in
 * tree order) are cut into `world` contiguous ranges of equal size and a box belongs to the rank
 * holding its median point -- contiguous Morton ranges of subtrees at the fine levels, one owner
 * per box at the coarse ones.
 * Owner computes, state replicated: every rank builds the same tree / lists / NNCA and holds
 * every block; in each colour of a split level a rank compresses (RRQR) only
 * its own boxes, inverts only its own pivots and forms their multipliers, and
 * performs only the Schur updates (Table 4) of target blocks whose row box it owns;
 * each of these three phases ends with an exchange that gives every rank the blocks the others
 * wrote (new basis columns with their ranks, G_i and W_i, updated targets).  The NNCA build is
 * split the same way (ACA and skeleton solves per owned box).  Levels <= level_p, the level
 * set-up, orthonormalisation, redirection, new blocks, top and solve run
 * redundantly.  Every rank ends with the same factorization and solves locally.  The pivots
 * of the R31 (null-space) boxes are formed by every rank (their Schur operands are per-rank
 * temporaries; their inverses are small); the opt-in R30 is not used while distributed.
 *
 * aifmm_dist_unique_id — host out[128]: a fresh NCCL unique id (call on one rank, send it to
 *   the others, e.g. with torch.distributed.broadcast_object_list).  Errors: ENCCL.
 * aifmm_dist_init — join an NCCL communicator of `world` ranks as `rank` (one GPU per rank;
 *   the current CUDA device must be this rank's).  unique_id: host, 128 bytes from
 *   aifmm_dist_unique_id.  level_p: levels <= level_p are computed redundantly by every rank
 *   (-1: none, every level from 2 down is split; at most L - 1).  Collective: every
 *   rank calls it, then every rank calls build / factor with the SAME arguments.  A world of 1
 *   is the single-GPU path.  Errors: EINVALID_ARG, ENCCL.
 * aifmm_dist_init_local — the same over an in-process transport, for validation on one GPU:
 *   `world` copies of this library loaded in one process, each driven by its own host thread
 *   and stream, meet through `shared` (host memory of at least 4096 bytes, zeroed before the
 *   first init, the same pointer for every rank) and exchange by device-to-device copies.
 * aifmm_dist_finalize — leave the communicator (back to the single-GPU path).
 * aifmm_get_owners — host int32[2^(d*level)]: owning rank of every box at `level` of the last
 *   factorization's partition (-1: computed redundantly, level <= level_p or not distributed).
 *   Errors: ESTATE before a build.
 * A rank that raises inside a distributed factorization leaves the others waiting in the next
 * exchange: errors are fatal for the job (as with any collective). */
int aifmm_dist_unique_id(void* out);
int aifmm_dist_init(int rank, int world, const void* unique_id, int level_p);
int aifmm_dist_init_local(int rank, int world, void* shared, int level_p);
int aifmm_dist_finalize(void);
int aifmm_get_owners(int level, int32_t* owner);

/* Test hook: in-place inverse of one n x n column-major device matrix with the library's
 * batched Gauss-Jordan (R16; the kernel behind pivot inverses and the top solve). */
int aifmm_debug_inverse(double* A, int n, int lda);
/* Test hook: in-place inverses of `batch` n x n column-major device matrices stored back to back
 * (ld n) by the batched Gauss-Jordan; path 0 = the library's routing, 1 = one panel launch +
 * one DMMA GEMM launch per 32 columns, 2 = the fused one-CTA-per-matrix kernel (n > 160).
 * Errors: EINVALID_ARG, ESINGULAR_PIVOT. */
int aifmm_debug_inverse_batch(double* A, int n, int batch, int path);
/* Test hook: first stage of the two-stage RRQR (reading R8b) on `batch` device matrices A_b
 * (n x m column-major, ld n, stored back to back; destroyed): M_b = R_b^T (m x min(n,m), ld m,
 * back to back), where A_b = Q_b R_b (Householder; TSQR row chunks when n > 768 and m <= 384).
 * R_b is unique up to the signs of its rows. */
int aifmm_debug_tri_root(double* A, int n, int m, int batch, double* M);

#ifdef __cplusplus
}
#endif
#endif /* AIFMM_H */
