// aifmm_oracle.cpp — ORACLE (test infrastructure, NOT the product path).
//
// A plain serial C++ implementation of the AIFMM of PAPER.md (arXiv 2301.12704, cited as
// P:<line>) with plain dense loops (no BLAS, no LAPACK), written step by step after the paper
// and the readings of DESIGN.md (R<n>).  It is the north_star's "plain serial CPU C++" oracle
// and follows oracle/*.py (the numpy oracle) function by function, so the two can be checked
// against each other; it shares no code, header, table or helper with the CUDA path
// (paper_2301_12704_b200/csrc), and neither includes the other.  Only tests/, bench.py's
// cpu_baseline leg and the golden-writing tools may load it (ctypes, oracle/cpp.py).
//
//   tree      §2.1 P:121-123 (R1-R4)                      -> oracle/tree.py
//   lists     §2.2, Remark P:402-404 (R5)        -> oracle/tree.py
//   colours   R6                                            -> oracle/tree.py
//   kernels   P:105-111                                     -> oracle/kernels.py
//   NNCA      Eq. NCA, operators P:360-367 (R9, R10, R11, R11b, R18, R20) -> oracle/nnca.py
//   factor    §3.1, Alg. 3, §3.2.1-3.2.3, Table 4
//             (R8, R8b, R12-R17, R21-R23, R27, R28)    -> oracle/factor.py
//   solve     Alg. 4 P:1169-1184                            -> oracle/factor.py
//
// Threads: `threads > 1` runs loops over independent boxes / blocks with OpenMP; every
// floating-point operation happens in the same order as with one thread (per-target Schur
// contributions are applied in ascending eliminated-box order, the level-start change of
// variables applies its two factors in the serial order), so the result is bit-identical
// for every thread count (tested).
//
// Build: g++ -O2 -fopenmp -ffp-contract=off -shared -fPIC (oracle/cpp.py: build()).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <set>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <utility>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

// ----------------------------------------------------------------------------- dense matrices
// column-major, r x c
struct Mat {
  int r = 0, c = 0;
  std::vector<double> a;
  Mat() {}
  Mat(int r_, int c_) : r(r_), c(c_), a((size_t)r_ * c_, 0.0) {}
  double& operator()(int i, int j) { return a[(size_t)j * r + i]; }
  double operator()(int i, int j) const { return a[(size_t)j * r + i]; }
  double* col(int j) { return a.data() + (size_t)j * r; }
  const double* col(int j) const { return a.data() + (size_t)j * r; }
};

struct OracleError : std::runtime_error {
  int code;
  OracleError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

// fixed-order dot product (4 interleaved partial sums, combined in a fixed order)
static double dot(const double* x, const double* y, int n) {
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  int i = 0;
  for (; i + 4 <= n; i += 4) {
    s0 += x[i] * y[i];
    s1 += x[i + 1] * y[i + 1];
    s2 += x[i + 2] * y[i + 2];
    s3 += x[i + 3] * y[i + 3];
  }
  for (; i < n; ++i) s0 += x[i] * y[i];
  return (s0 + s1) + (s2 + s3);
}
static double nrm2sq(const double* x, int n) { return dot(x, x, n); }
static double fro(const Mat& A) { return std::sqrt(nrm2sq(A.a.data(), (int)A.a.size())); }

// C = op(A) op(B) (+ C if acc), op = identity or transpose
static void gemm(const Mat& A, bool ta, const Mat& B, bool tb, Mat& C, double alpha = 1.0, bool acc = false) {
  const int m = ta ? A.c : A.r, k = ta ? A.r : A.c, n = tb ? B.r : B.c;
  if ((tb ? B.c : B.r) != k) throw OracleError(-1, "gemm shape");
  if (!acc) C = Mat(m, n);
  if (C.r != m || C.c != n) throw OracleError(-1, "gemm out shape");
  if (!ta) {
    // C[:, j] += alpha A[:, p] B(p, j): column axpys (contiguous)
    for (int j = 0; j < n; ++j) {
      double* cj = C.col(j);
      for (int p = 0; p < k; ++p) {
        const double b = alpha * (tb ? B(j, p) : B(p, j));
        if (b == 0.0) continue;
        const double* ap = A.col(p);
        for (int i = 0; i < m; ++i) cj[i] += ap[i] * b;
      }
    }
  } else {
    // C(i, j) += alpha A[:, i] . op(B)[:, j]
    std::vector<double> bj(k);
    for (int j = 0; j < n; ++j) {
      if (tb)
        for (int p = 0; p < k; ++p) bj[p] = B(j, p);
      else
        std::memcpy(bj.data(), B.col(j), sizeof(double) * k);
      for (int i = 0; i < m; ++i) C(i, j) += alpha * dot(A.col(i), bj.data(), k);
    }
  }
}
static Mat mul(const Mat& A, bool ta, const Mat& B, bool tb) {
  Mat C;
  gemm(A, ta, B, tb, C);
  return C;
}
static Mat sub(const Mat& A, int r0, int r1, int c0, int c1) {
  Mat S(r1 - r0, c1 - c0);
  for (int j = c0; j < c1; ++j)
    for (int i = r0; i < r1; ++i) S(i - r0, j - c0) = A(i, j);
  return S;
}
static Mat hcat(const std::vector<const Mat*>& v, int rows) {
  int c = 0;
  for (auto* m : v) c += m->c;
  Mat out(rows, c);
  int o = 0;
  for (auto* m : v) {
    if (m->r != rows) throw OracleError(-1, "hcat rows");
    std::memcpy(out.col(o), m->a.data(), sizeof(double) * m->a.size());
    o += m->c;
  }
  return out;
}
static Mat vcat(const std::vector<const Mat*>& v, int cols) {
  int r = 0;
  for (auto* m : v) r += m->r;
  Mat out(r, cols);
  int o = 0;
  for (auto* m : v) {
    for (int j = 0; j < cols; ++j)
      for (int i = 0; i < m->r; ++i) out(o + i, j) = (*m)(i, j);
    o += m->r;
  }
  return out;
}
static Mat pad(const Mat& M, int r, int c) {
  Mat out(r, c);
  for (int j = 0; j < M.c; ++j)
    for (int i = 0; i < M.r; ++i) out(i, j) = M(i, j);
  return out;
}

// LU with partial pivoting (R16, R19, R20): P A = L U in place; piv[j] = row swapped with j.
// Pivot = largest |entry| in the column, lowest row on ties.  Returns false if singular.
static bool lu(Mat& A, std::vector<int>& piv) {
  const int n = A.r;
  piv.assign(n, 0);
  for (int j = 0; j < n; ++j) {
    int p = j;
    double mx = std::fabs(A(j, j));
    for (int i = j + 1; i < n; ++i)
      if (std::fabs(A(i, j)) > mx) { mx = std::fabs(A(i, j)); p = i; }
    piv[j] = p;
    if (!(mx > 0.0)) return false;
    if (p != j)
      for (int c = 0; c < n; ++c) std::swap(A(j, c), A(p, c));
    const double d = A(j, j);
    double* cj = A.col(j);
    for (int i = j + 1; i < n; ++i) cj[i] /= d;
    for (int c = j + 1; c < n; ++c) {
      double* cc = A.col(c);
      const double a = cc[j];
      if (a == 0.0) continue;
      for (int i = j + 1; i < n; ++i) cc[i] -= cj[i] * a;
    }
  }
  return true;
}
// solve (LU) X = B in place (B: n x nrhs)
static void lu_solve(const Mat& LU, const std::vector<int>& piv, Mat& B) {
  const int n = LU.r;
  for (int c = 0; c < B.c; ++c) {
    double* b = B.col(c);
    for (int j = 0; j < n; ++j)
      if (piv[j] != j) std::swap(b[j], b[piv[j]]);
    for (int j = 0; j < n; ++j) {          // L y = b (unit lower), column oriented
      const double v = b[j];
      if (v == 0.0) continue;
      const double* lj = LU.col(j);
      for (int i = j + 1; i < n; ++i) b[i] -= lj[i] * v;
    }
    for (int j = n - 1; j >= 0; --j) {     // U x = y
      b[j] /= LU(j, j);
      const double v = b[j];
      if (v == 0.0) continue;
      const double* uj = LU.col(j);
      for (int i = 0; i < j; ++i) b[i] -= uj[i] * v;
    }
  }
}
static bool solve(const Mat& A, Mat& B) {
  Mat LU = A;
  std::vector<int> piv;
  if (!lu(LU, piv)) return false;
  lu_solve(LU, piv, B);
  return true;
}
static bool inverse(const Mat& A, Mat& G) {
  const int n = A.r;
  G = Mat(n, n);
  for (int i = 0; i < n; ++i) G(i, i) = 1.0;
  return n == 0 || solve(A, G);
}

// Householder QR of A (m x n, m >= n when Q is wanted): R (min(m,n) x n, upper) and, if Q is
// non-null, the thin Q (m x min(m,n)).  Reflectors H = I - tau v v^T with v(0) = 1.
static void householder(const Mat& A, Mat* Q, Mat& R) {
  const int m = A.r, n = A.c, r = std::min(m, n);
  Mat W = A;
  std::vector<double> tau(r, 0.0);
  for (int j = 0; j < r; ++j) {
    double* x = W.col(j) + j;
    const int len = m - j;
    const double sig = (len > 1) ? nrm2sq(x + 1, len - 1) : 0.0;
    const double alpha = x[0];
    if (sig == 0.0) {
      tau[j] = 0.0;
      continue;
    }
    const double nrm = std::sqrt(alpha * alpha + sig);
    const double beta = (alpha <= 0.0) ? nrm : -nrm;     // R(j,j) = beta
    const double v0 = alpha - beta;
    for (int i = 1; i < len; ++i) x[i] /= v0;
    tau[j] = (beta - alpha) / beta;
    x[0] = beta;
    // apply to the trailing columns: c -= tau v (v^T c)
    for (int c = j + 1; c < n; ++c) {
      double* y = W.col(c) + j;
      double s = y[0] + dot(x + 1, y + 1, len - 1);
      s *= tau[j];
      y[0] -= s;
      for (int i = 1; i < len; ++i) y[i] -= s * x[i];
    }
  }
  R = Mat(r, n);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i <= std::min(j, r - 1); ++i) R(i, j) = W(i, j);
  if (!Q) return;
  Mat& q = *Q;
  q = Mat(m, r);
  for (int i = 0; i < r; ++i) q(i, i) = 1.0;
  for (int j = r - 1; j >= 0; --j) {       // Q = H_0 H_1 ... H_{r-1} [I; 0]
    const double* v = W.col(j) + j;
    const int len = m - j;
    for (int c = j; c < r; ++c) {
      double* y = q.col(c) + j;
      double s = y[0] + dot(v + 1, y + 1, len - 1);
      s *= tau[j];
      y[0] -= s;
      for (int i = 1; i < len; ++i) y[i] -= s * v[i];
    }
  }
}

// first error raised inside an OpenMP loop (rethrown after the loop)
struct ErrSlot {
  int code = 0;
  std::string msg;
  void set(const OracleError& e) {
#pragma omp critical(oracle_err)
    {
      if (!code) { code = e.code; msg = e.what(); }
    }
  }
  void rethrow() const {
    if (code) throw OracleError(code, msg);
  }
};

// ----------------------------------------------------------------------------- decision rules
constexpr double TIE = 1e-10;      // R7
// R7: lowest index with |v| >= (1 - TIE) max|v| over unused entries; -1 if max is 0
static int pick(const std::vector<double>& v, const std::vector<char>* used) {
  double mx = -1.0;
  for (size_t i = 0; i < v.size(); ++i) {
    const double a = (used && (*used)[i]) ? -1.0 : std::fabs(v[i]);
    if (a > mx) mx = a;
  }
  if (!(mx > 0.0)) return -1;
  const double thr = mx * (1.0 - TIE);
  for (size_t i = 0; i < v.size(); ++i) {
    const double a = (used && (*used)[i]) ? -1.0 : std::fabs(v[i]);
    if (a >= thr) return (int)i;
  }
  return -1;
}

// R8: pivoted Gram-Schmidt on the columns of W (already projected against B), taking pivots
// while t < tmin or ||W_t||_F > tau, never more than tmax; re-orthogonalisation (two passes, a
// third if the second cancelled more than half; a column still collapsing is discarded).
// Returns the new orthonormal columns; *t_trunc = columns taken when the tau test first held.
static Mat pivoted_qr_extend(Mat W, const Mat& Bin, double tau, int tmin, int tmax, int* t_trunc_out) {
  const int m = W.r, nc = W.c;
  std::vector<std::vector<double>> B;
  for (int j = 0; j < Bin.c; ++j) B.emplace_back(Bin.col(j), Bin.col(j) + m);
  const int kb0 = (int)B.size();
  int t_trunc = -1;
  std::vector<double> norms(nc), w(m);
  auto reorth = [&](std::vector<double>& x) {
    // w = w - B (B^T w): coefficients first, then the update (the order of oracle/linalg.py)
    std::vector<double> coef(B.size());
    for (size_t s = 0; s < B.size(); ++s) coef[s] = dot(B[s].data(), x.data(), m);
    for (int i = 0; i < m; ++i) {
      double a = 0.0;
      for (size_t s = 0; s < B.size(); ++s) a += B[s][i] * coef[s];
      x[i] -= a;
    }
    return std::sqrt(nrm2sq(x.data(), m));
  };
  while ((int)B.size() - kb0 < tmax) {
    double res2 = 0.0;
    for (int c = 0; c < nc; ++c) {
      norms[c] = nrm2sq(W.col(c), m);
      res2 += norms[c];
    }
    const double res = std::sqrt(res2);
    const int taken = (int)B.size() - kb0;
    if (t_trunc < 0 && !(res > tau)) t_trunc = taken;
    if (taken >= tmin && !(res > tau)) break;
    std::vector<double> sn(nc);
    for (int c = 0; c < nc; ++c) sn[c] = std::sqrt(norms[c]);
    const int j = pick(sn, nullptr);
    if (j < 0) break;
    std::memcpy(w.data(), W.col(j), sizeof(double) * m);
    const double n1 = reorth(w);
    double nw = reorth(w);
    if (!(nw > 0.5 * n1)) {
      const double n2 = nw;
      nw = reorth(w);
      if (!(nw > 0.5 * n2)) nw = 0.0;
    }
    if (!(nw > 0.0)) {
      std::fill(W.col(j), W.col(j) + m, 0.0);
      continue;
    }
    for (int i = 0; i < m; ++i) w[i] /= nw;
    B.push_back(w);
    const std::vector<double>& q = B.back();
    for (int c = 0; c < nc; ++c) {      // W <- W - q (q^T W)
      double* col = W.col(c);
      const double s = dot(q.data(), col, m);
      for (int i = 0; i < m; ++i) col[i] -= q[i] * s;
    }
    std::fill(W.col(j), W.col(j) + m, 0.0);
  }
  const int taken = (int)B.size() - kb0;
  if (t_trunc < 0) t_trunc = taken;
  *t_trunc_out = t_trunc;
  Mat Q(m, taken);
  for (int t = 0; t < taken; ++t) std::memcpy(Q.col(t), B[kb0 + t].data(), sizeof(double) * m);
  return Q;
}

// ----------------------------------------------------------------------------- kernels
struct Kern {
  int id, d;
  double diag, ell;
};
// A_ij = K(x_i, x_j); the diagonal (same global index) is `diag`
static double entry(const Kern& K, const double* P, long long i, long long j) {
  if (i == j) return K.diag;
  const double* x = P + i * K.d;
  const double* y = P + j * K.d;
  double s = 0.0;
  for (int a = 0; a < K.d; ++a) {
    const double t = x[a] - y[a];
    s += t * t;
  }
  const double r = std::sqrt(s);
  double v;
  if (K.id == 0) v = std::log(r);
  else if (K.id == 1) v = std::exp(-r / K.ell);
  else v = 1.0 / r;
  if (!std::isfinite(v)) throw OracleError(-3, "coincident points with a singular kernel");
  return v;
}
static Mat kblock(const Kern& K, const double* P, const std::vector<long long>& rows, const std::vector<long long>& cols) {
  Mat M((int)rows.size(), (int)cols.size());
  for (size_t j = 0; j < cols.size(); ++j)
    for (size_t i = 0; i < rows.size(); ++i) M((int)i, (int)j) = entry(K, P, rows[i], cols[j]);
  return M;
}
static std::vector<long long> range(long long a, long long b) {
  std::vector<long long> v;
  for (long long i = a; i < b; ++i) v.push_back(i);
  return v;
}

// ----------------------------------------------------------------------------- tree (§2.1)
constexpr int LMAX = 20;   // R3
struct Tree {
  int d = 0, L = 0, nmax = 0;
  long long n = 0;
  std::vector<long long> perm;            // perm[j] = user index of tree-order point j
  std::vector<double> pts;                // tree order, n x d
  std::vector<std::vector<long long>> off;
  int nboxes(int l) const { return 1 << (d * l); }
  long long count(int l, int b) const { return off[l][b + 1] - off[l][b]; }
  std::vector<int> coords(int l, int b) const {
    std::vector<int> c(d, 0);
    for (int bit = 0; bit < l; ++bit)
      for (int a = 0; a < d; ++a) c[a] |= ((b >> (bit * d + a)) & 1) << bit;
    return c;
  }
  int box_id(const std::vector<int>& c, int l) const {
    int b = 0;
    for (int bit = 0; bit < l; ++bit)
      for (int a = 0; a < d; ++a) b |= ((c[a] >> bit) & 1) << (bit * d + a);
    return b;
  }
  std::vector<int> children(int l, int b) const {
    std::vector<int> out;
    for (int j = 0; j < (1 << d); ++j) {
      const int c = (b << d) | j;
      if (count(l + 1, c) > 0) out.push_back(c);
    }
    return out;
  }
};

static long long morton(const long long* kc, int d, int bits) {
  long long key = 0;
  for (int b = 0; b < bits; ++b)
    for (int a = 0; a < d; ++a) key |= ((kc[a] >> b) & 1LL) << (b * d + a);
  return key;
}

static void build_tree(Tree& t, const double* P, long long n, int d, int nmax) {
  if (n < 1) throw OracleError(-1, "empty input");
  if (d != 2 && d != 3) throw OracleError(-1, "d must be 2 or 3");
  t.d = d;
  t.n = n;
  t.nmax = nmax;
  // P:122 smallest hypercube containing the points (R2)
  std::vector<double> lo(d), hi(d), g(d);
  for (int a = 0; a < d; ++a) lo[a] = hi[a] = P[a];
  for (long long i = 0; i < n; ++i)
    for (int a = 0; a < d; ++a) {
      const double v = P[i * d + a];
      if (!std::isfinite(v)) throw OracleError(-2, "non-finite point coordinates");
      lo[a] = std::min(lo[a], v);
      hi[a] = std::max(hi[a], v);
    }
  double h = 0.0;
  for (int a = 0; a < d; ++a) h = std::max(h, hi[a] - lo[a]);
  h /= 2.0;
  if (!(h > 0.0)) h = std::ldexp(1.0, -20);
  for (int a = 0; a < d; ++a) g[a] = (lo[a] + hi[a]) / 2.0 - h;
  const double two_h = 2.0 * h;
  // R3: k_a = clamp(floor(((p - g) / (2h)) 2^LMAX)), each step rounded (no FMA contraction)
  std::vector<long long> kc((size_t)n * d);
  const long long top = (1LL << LMAX) - 1;
  for (long long i = 0; i < n; ++i)
    for (int a = 0; a < d; ++a) {
      volatile double t1 = P[i * d + a] - g[a];
      volatile double t2 = t1 / two_h;
      volatile double t3 = t2 * (double)(1LL << LMAX);
      long long k = (long long)std::floor((double)t3);
      kc[i * d + a] = std::min(std::max(k, 0LL), top);
    }
  // R1: smallest L >= 2 with every box holding <= n_max points
  int L = -1;
  std::vector<long long> key(n), tmp(d);
  for (int l = 2; l <= LMAX; ++l) {
    std::unordered_map<long long, long long> cnt;
    long long mx = 0;
    for (long long i = 0; i < n; ++i) {
      for (int a = 0; a < d; ++a) tmp[a] = kc[i * d + a] >> (LMAX - l);
      mx = std::max(mx, ++cnt[morton(tmp.data(), d, l)]);
    }
    if (mx <= nmax) { L = l; break; }
    if (d * l > 24) break;
  }
  if (L < 0) throw OracleError(-3, "cannot subdivide: coincident points or too deep a tree");
  t.L = L;
  for (long long i = 0; i < n; ++i) {
    for (int a = 0; a < d; ++a) tmp[a] = kc[i * d + a] >> (LMAX - L);
    key[i] = morton(tmp.data(), d, L);
  }
  t.perm.resize(n);
  for (long long i = 0; i < n; ++i) t.perm[i] = i;
  std::stable_sort(t.perm.begin(), t.perm.end(), [&](long long a, long long b) { return key[a] < key[b]; });
  t.pts.resize((size_t)n * d);
  std::vector<long long> sk(n);
  for (long long j = 0; j < n; ++j) {
    for (int a = 0; a < d; ++a) t.pts[j * d + a] = P[t.perm[j] * d + a];
    sk[j] = key[t.perm[j]];
  }
  t.off.assign(L + 1, {});
  for (int l = 0; l <= L; ++l) {
    const int nb = 1 << (d * l);
    std::vector<long long>& o = t.off[l];
    o.assign(nb + 1, 0);
    long long j = 0;
    for (int b = 0; b <= nb; ++b) {
      while (j < n && (sk[j] >> (d * (L - l))) < b) ++j;
      o[b] = j;
    }
  }
}

// N(i), IL(i) per level >= 2 (Table, R5: Chebyshev distance >= 2), sorted by Morton id
struct Lists {
  std::vector<std::map<int, std::vector<int>>> nearl, il;   // [level][box]
};
static void build_lists(const Tree& t, Lists& ls) {
  ls.nearl.assign(t.L + 1, {});
  ls.il.assign(t.L + 1, {});
  const int d = t.d;
  const int n3 = (d == 2) ? 9 : 27;
  for (int l = 2; l <= t.L; ++l) {
    const int side = 1 << l;
    for (int b = 0; b < t.nboxes(l); ++b) {
      if (t.count(l, b) == 0) continue;
      const std::vector<int> c = t.coords(l, b);
      std::vector<int> nb, cand;
      for (int o = 0; o < n3; ++o) {
        std::vector<int> cc(d);
        bool ok = true;
        int oo = o;
        for (int a = 0; a < d; ++a) {
          cc[a] = c[a] + (oo % 3) - 1;
          oo /= 3;
          ok = ok && cc[a] >= 0 && cc[a] < side;
        }
        if (!ok) continue;
        const int j = t.box_id(cc, l);
        if (t.count(l, j) > 0) nb.push_back(j);
      }
      std::vector<int> pc(d);
      for (int a = 0; a < d; ++a) pc[a] = c[a] >> 1;
      for (int o = 0; o < n3; ++o) {
        std::vector<int> pp(d);
        bool ok = true;
        int oo = o;
        for (int a = 0; a < d; ++a) {
          pp[a] = pc[a] + (oo % 3) - 1;
          oo /= 3;
          ok = ok && pp[a] >= 0 && pp[a] < (side >> 1);
        }
        if (!ok) continue;
        const int pb = t.box_id(pp, l - 1);
        for (int j = 0; j < (1 << d); ++j) {
          const int ch = (pb << d) | j;
          if (t.count(l, ch) == 0) continue;
          const std::vector<int> c2 = t.coords(l, ch);
          int cheb = 0;
          for (int a = 0; a < d; ++a) cheb = std::max(cheb, std::abs(c2[a] - c[a]));
          if (cheb >= 2) cand.push_back(ch);
        }
      }
      std::sort(nb.begin(), nb.end());
      std::sort(cand.begin(), cand.end());
      ls.nearl[l][b] = nb;
      ls.il[l][b] = cand;
    }
  }
}
// R6: greedy first-fit in Morton order; conflict = N(i) minus i
static std::map<int, int> greedy_colours(const std::map<int, std::vector<int>>& nearl) {
  std::map<int, int> col;
  for (auto& kv : nearl) {
    std::set<int> used;
    for (int j : kv.second) {
      auto it = col.find(j);
      if (it != col.end()) used.insert(it->second);
    }
    int c = 0;
    while (used.count(c)) ++c;
    col[kv.first] = c;
  }
  return col;
}

// ----------------------------------------------------------------------------- NNCA (§2.3)
constexpr double GUARD = 1e-13;   // R9

// ACA with partial pivoting on A(R, F) (R9); returns (row pivots, column pivots)
static void aca(const Kern& K, const double* P, const std::vector<long long>& R, const std::vector<long long>& F,
                double eps, std::vector<int>& rp, std::vector<int>& cp) {
  const int nR = (int)R.size(), nF = (int)F.size();
  std::vector<std::vector<double>> us, vs;
  std::vector<char> rows_used(nR, 0), cols_used(nF, 0);
  const int kmax = std::min(nR, nF);
  int i = 0;
  double norm2 = 0.0, first = -1.0;
  auto first_free = [&]() {
    for (int r = 0; r < nR; ++r)
      if (!rows_used[r]) return r;
    return -1;
  };
  while ((int)us.size() < kmax) {
    rows_used[i] = 1;
    std::vector<double> r(nF);
    for (int j = 0; j < nF; ++j) r[j] = entry(K, P, R[i], F[j]);
    for (size_t s = 0; s < us.size(); ++s) {          // residual row, crosses in order
      const double ui = us[s][i];
      for (int j = 0; j < nF; ++j) r[j] = r[j] - ui * vs[s][j];
    }
    const int j = pick(r, &cols_used);
    if (j < 0) {
      const int f = first_free();
      if (f < 0) break;
      i = f;
      continue;
    }
    const double delta = r[j];
    if (first >= 0.0 && std::fabs(delta) <= GUARD * first) break;
    first = (first < 0.0) ? std::fabs(delta) : std::max(first, std::fabs(delta));
    std::vector<double> v(nF);
    for (int q = 0; q < nF; ++q) v[q] = r[q] / delta;
    std::vector<double> u(nR);
    for (int q = 0; q < nR; ++q) u[q] = entry(K, P, R[q], F[j]);
    for (size_t s = 0; s < us.size(); ++s) {
      const double vj = vs[s][j];
      for (int q = 0; q < nR; ++q) u[q] = u[q] - vj * us[s][q];
    }
    cols_used[j] = 1;
    const double uu = dot(u.data(), u.data(), nR);
    const double vv2 = dot(v.data(), v.data(), nF);
    double cross = 0.0;
    for (size_t s = 0; s < us.size(); ++s) cross += dot(us[s].data(), u.data(), nR) * dot(vs[s].data(), v.data(), nF);
    norm2 = norm2 + 2.0 * cross + uu * vv2;
    us.push_back(u);
    vs.push_back(v);
    rp.push_back(i);
    cp.push_back(j);
    if (std::sqrt(uu * vv2) <= eps * std::sqrt(std::max(norm2, 0.0))) break;
    int nxt = pick(u, &rows_used);
    if (nxt < 0) {
      nxt = first_free();
      if (nxt < 0) break;
    }
    i = nxt;
  }
}

struct NNCALevel {
  std::map<int, std::vector<long long>> R, sk, fp;
  std::map<int, Mat> U;   // |R| x k: A(R, fp) A(sk, fp)^-1 (V = U, R10)
};

static void build_nnca(const Tree& t, const Lists& ls, const Kern& K, double eps, std::vector<NNCALevel>& nn, int threads) {
  nn.assign(t.L + 1, {});
  const double* P = t.pts.data();
  for (int l = t.L; l >= 2; --l) {
    NNCALevel& nl = nn[l];
    std::vector<int> boxes;
    for (auto& kv : ls.nearl[l]) boxes.push_back(kv.first);
    for (int B : boxes) {
      if (l == t.L) {
        nl.R[B] = range(t.off[l][B], t.off[l][B + 1]);
      } else {
        std::vector<long long> r;
        for (int c : t.children(l, B)) r.insert(r.end(), nn[l + 1].sk.at(c).begin(), nn[l + 1].sk.at(c).end());
        nl.R[B] = r;
      }
      nl.sk[B];
      nl.fp[B];
      nl.U[B];
    }
    std::string err;
    int ecode = 0;
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads)
    for (int bi = 0; bi < (int)boxes.size(); ++bi) {
      try {
        const int B = boxes[bi];
        const std::vector<long long>& R = nl.R.at(B);
        // R11b: sources of an IL box = its x-variables (points at the leaf, children's skeletons above)
        std::vector<long long> F;
        for (int D : ls.il[l].at(B)) F.insert(F.end(), nl.R.at(D).begin(), nl.R.at(D).end());
        // R20: ancestors' interaction lists while IL(B) holds fewer sources than R_B
        int la = l, A_ = B;
        while ((long long)F.size() < (long long)R.size() && la > 2) {
          --la;
          A_ >>= t.d;
          for (int D : ls.il[la].at(A_)) {
            if (l == t.L) {
              for (long long p = t.off[la][D]; p < t.off[la][D + 1]; ++p) F.push_back(p);
            } else {
              const int sh = t.d * (l + 1 - la);
              for (int c = D << sh; c < ((D + 1) << sh); ++c) {
                auto it = nn[l + 1].sk.find(c);
                if (it != nn[l + 1].sk.end()) F.insert(F.end(), it->second.begin(), it->second.end());
              }
            }
          }
        }
        std::vector<int> ri, ci;
        if (!R.empty() && !F.empty()) aca(K, P, R, F, eps, ri, ci);
        std::vector<long long> sk, fp;
        for (int q : ri) sk.push_back(R[q]);
        for (int q : ci) fp.push_back(F[q]);
        Mat U((int)R.size(), (int)sk.size());
        if (!sk.empty()) {
          // V^* = A(fp, sk)^-1 A(fp, R); U = V (R10)
          Mat Afs = kblock(K, P, fp, sk);
          Mat X = kblock(K, P, fp, R);
          if (!solve(Afs, X)) throw OracleError(-4, "NNCA skeleton block singular");
          for (int j = 0; j < X.c; ++j)
            for (int i = 0; i < X.r; ++i) U(j, i) = X(i, j);
        }
        nl.sk.at(B) = sk;
        nl.fp.at(B) = fp;
        nl.U.at(B) = std::move(U);
      } catch (const OracleError& e) {
#pragma omp critical
        {
          if (!ecode) { ecode = e.code; err = e.what(); }
        }
      }
    }
    if (ecode) throw OracleError(ecode, err);
  }
}

// ----------------------------------------------------------------------------- factor (§3)
struct Rec {
  Mat G;
  int m = 0, k = 0;
  std::vector<std::pair<int, std::pair<Mat, bool>>> R, C;   // (partner, (block, E flag)), ascending partner
};

struct Level {
  int l = 0;
  std::vector<int> boxes;
  std::unordered_map<int, int> m, k;
  std::unordered_map<int, Mat> U, V, Ud, Vd;
  std::unordered_map<int, char> E;
  std::unordered_map<long long, Mat> nearb, A, F;
  std::set<std::pair<int, int>> pending;
  std::unordered_map<int, Rec> rec;
  std::map<std::pair<int, int>, std::pair<int, int>> xoff;   // (parent, child) -> rows of child in x_parent
};

struct Oracle {
  Tree t;
  Lists ls;
  std::vector<std::map<int, int>> colour;
  Kern K{};
  double tol = 0, tol_c = 0;
  int threads = 1;
  int algorithm = 3;         // 3: Alg. 3 (deferred); 2: Alg. 2 (on creation; R29)
  std::vector<NNCALevel> nn;
  std::vector<Level> lv;     // by level
  Mat top;
  std::map<int, std::pair<int, int>> top_offs;
  std::vector<int> top_piv;
  bool factored = false;
  long long compressions = 0;
  double t_build = 0, t_factor = 0, t_solve = 0;

  long long key(int p, int q) const { return (long long)p * t.nboxes(t.L) + q; }   // unique per level
  bool in_near(int l, int p, int q) const {
    const auto& v = ls.nearl[l].at(p);
    return std::binary_search(v.begin(), v.end(), q);
  }
  bool in_il(int l, int p, int q) const {
    const auto& v = ls.il[l].at(p);
    return std::binary_search(v.begin(), v.end(), q);
  }
  int cheb(int l, int a, int b) const {
    auto ca = t.coords(l, a), cb = t.coords(l, b);
    int r = 0;
    for (int x = 0; x < t.d; ++x) r = std::max(r, std::abs(ca[x] - cb[x]));
    return r;
  }
  int live(const Level& L_, int b) const { return L_.E.at(b) ? L_.k.at(b) : L_.m.at(b); }

  // level setup / level transition and the M2L blocks
  void setup_level(int l) {
    Level& L_ = lv[l];
    const Level* prev = (l < t.L) ? &lv[l + 1] : nullptr;
    L_.l = l;
    for (auto& kv : ls.nearl[l]) L_.boxes.push_back(kv.first);
    for (int b : L_.boxes) {
      if (l == t.L) {
        L_.m[b] = (int)t.count(l, b);
        L_.U[b] = nn[l].U.at(b);
        L_.V[b] = nn[l].U.at(b);
      } else {
        std::vector<int> ch = t.children(l, b);
        int o = 0;
        std::vector<const Mat*> us, vs;
        for (int c : ch) {
          L_.xoff[{b, c}] = {o, o + prev->k.at(c)};
          o += prev->k.at(c);
          us.push_back(&prev->Ud.at(c));
          vs.push_back(&prev->Vd.at(c));
        }
        L_.m[b] = o;
        const int kb = (int)nn[l].sk.at(b).size();
        L_.U[b] = vcat(us, kb);
        L_.V[b] = vcat(vs, kb);
      }
      L_.k[b] = (int)nn[l].sk.at(b).size();
      if (l > 2) {
        const int P = b >> t.d;
        int r0 = 0;
        for (int c : t.children(l - 1, P)) {
          if (c == b) break;
          r0 += (int)nn[l].sk.at(c).size();
        }
        const Mat& UP = nn[l - 1].U.at(P);
        L_.Ud[b] = sub(UP, r0, r0 + L_.k[b], 0, UP.c);   // L2L U_b^dag
        L_.Vd[b] = L_.Ud[b];                             // M2M = L2L (R10)
      } else {
        L_.Ud[b] = Mat(L_.k[b], 0);
        L_.Vd[b] = Mat(L_.k[b], 0);
      }
      L_.E[b] = 0;
    }
    // blocks: create the keys serially, fill in parallel
    std::vector<std::pair<long long, std::pair<int, int>>> nk, ak;
    for (int p : L_.boxes) {
      for (int q : ls.nearl[l].at(p)) { nk.push_back({key(p, q), {p, q}}); L_.nearb[key(p, q)]; }
      for (int q : ls.il[l].at(p)) { ak.push_back({key(p, q), {p, q}}); L_.A[key(p, q)]; }
    }
    const double* P = t.pts.data();
    ErrSlot es;
#pragma omp parallel for schedule(dynamic, 16) num_threads(threads)
    for (size_t e = 0; e < nk.size(); ++e) {
      try {
      const int p = nk[e].second.first, q = nk[e].second.second;
      Mat& M = L_.nearb.at(nk[e].first);
      if (l == t.L) {
        M = kblock(K, P, range(t.off[l][p], t.off[l][p + 1]), range(t.off[l][q], t.off[l][q + 1]));
      } else {
        M = Mat(L_.m.at(p), L_.m.at(q));
        for (int c : t.children(l, p)) {
          auto ro = L_.xoff.at({p, c});
          for (int c2 : t.children(l, q)) {
            auto so = L_.xoff.at({q, c2});
            const Mat& blk = in_near(l + 1, c, c2) ? prev->nearb.at(key(c, c2)) : prev->A.at(key(c, c2));
            for (int j = 0; j < blk.c; ++j)
              for (int i = 0; i < blk.r; ++i) M(ro.first + i, so.first + j) = blk(i, j);
          }
        }
      }
      } catch (const OracleError& ex) {
        es.set(ex);
      }
    }
    es.rethrow();
#pragma omp parallel for schedule(dynamic, 16) num_threads(threads)
    for (size_t e = 0; e < ak.size(); ++e) {
      try {
        const int p = ak[e].second.first, q = ak[e].second.second;
        L_.A.at(ak[e].first) = kblock(K, P, nn[l].sk.at(p), nn[l].sk.at(q));
      } catch (const OracleError& ex) {
        es.set(ex);
      }
    }
    es.rethrow();
    orthonormalise(L_);
  }

  // R13: U_b = Q T, z~_b = T z_b: U_b <- Q, rows of Z_b (U^dag, A_bc) <- T (.);
  // V_b = Q' T', y_b = T'^T y~_b: columns of y_b (A_db, V^dag*) <- (.) T'^T
  void orthonormalise(Level& L_) {
    const int l = L_.l;
    std::unordered_map<int, Mat> T, T2;
    for (int b : L_.boxes) { T[b]; T2[b]; }
#pragma omp parallel for schedule(dynamic, 4) num_threads(threads)
    for (size_t bi = 0; bi < L_.boxes.size(); ++bi) {
      const int b = L_.boxes[bi];
      if (L_.k.at(b) == 0) continue;
      Mat Q, R;
      householder(L_.U.at(b), &Q, R);
      L_.U.at(b) = Q;
      L_.Ud.at(b) = mul(R, false, L_.Ud.at(b), false);
      T.at(b) = R;
      Mat Q2, R2;
      householder(L_.V.at(b), &Q2, R2);
      L_.V.at(b) = Q2;
      L_.Vd.at(b) = mul(R2, false, L_.Vd.at(b), false);
      T2.at(b) = R2;
    }
    // block (p, q), q in IL(p): left factor T_p (applied at b = p), right factor T'_q^T (at
    // b = q), in the order of the serial loop over ascending b
    std::vector<std::pair<int, int>> blocks;
    for (int p : L_.boxes)
      for (int q : ls.il[l].at(p)) blocks.push_back({p, q});
#pragma omp parallel for schedule(dynamic, 16) num_threads(threads)
    for (size_t e = 0; e < blocks.size(); ++e) {
      const int p = blocks[e].first, q = blocks[e].second;
      Mat& A = L_.A.at(key(p, q));
      const bool left = L_.k.at(p) > 0, right = L_.k.at(q) > 0;
      if (p < q) {
        if (left) A = mul(T.at(p), false, A, false);
        if (right) A = mul(A, false, T2.at(q), true);
      } else {
        if (right) A = mul(A, false, T2.at(q), true);
        if (left) A = mul(T.at(p), false, A, false);
      }
    }
  }

  // R8b: W^T = Q R (Householder); returns R^T (m x min(m, n))
  static Mat tri_root(const Mat& W) {
    if (W.c == 0) return W;
    Mat WT(W.c, W.r);
    for (int j = 0; j < W.c; ++j)
      for (int i = 0; i < W.r; ++i) WT(j, i) = W(i, j);
    Mat R;
    householder(WT, nullptr, R);
    Mat RT(R.c, R.r);
    for (int j = 0; j < R.c; ++j)
      for (int i = 0; i < R.r; ++i) RT(j, i) = R(i, j);
    return RT;
  }

  // Alg. 3 lines P:1118-1129 for the pending pairs S (R12, R14; R27: one side)
  void compress(Level& L_, const std::vector<std::pair<int, int>>& S) {
    const int l = L_.l;
    std::map<int, std::vector<int>> part;
    for (auto& pr : S) {
      part[pr.first].push_back(pr.second);
      part[pr.second].push_back(pr.first);
    }
    std::vector<int> affected;
    for (auto& kv : part)
      if (!L_.E.at(kv.first)) affected.push_back(kv.first);
    std::vector<Mat> newU(affected.size());
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads)
    for (size_t a = 0; a < affected.size(); ++a) {
      const int b = affected[a];
      std::vector<int> ps = part.at(b);
      std::sort(ps.begin(), ps.end());
      const int m = L_.m.at(b), k = L_.k.at(b);
      std::vector<const Mat*> fs;
      for (int q : ps) fs.push_back(&L_.F.at(key(b, q)));
      Mat FU = hcat(fs, m);                                   // row X_b
      const double nU = fro(FU);
      const Mat& Ub = L_.U.at(b);
      Mat UtF = mul(Ub, true, FU, false);
      gemm(Ub, false, UtF, false, FU, -1.0, true);           // (I - U U^T) F
      Mat WU = tri_root(FU);                                  // R8b
      int tU = 0;
      Mat QU = pivoted_qr_extend(WU, Ub, tol_c * nU, 0, m - k, &tU);
      // tmin = 0: the columns taken are exactly the t_trunc of R8 (R27: V_b's new columns = U_b's)
      Mat nu(m, k + QU.c);
      std::memcpy(nu.a.data(), Ub.a.data(), sizeof(double) * Ub.a.size());
      std::memcpy(nu.col(k), QU.a.data(), sizeof(double) * QU.a.size());
      newU[a] = std::move(nu);
    }
    // zero-pad Z_b rows / y_b columns (other M2L, M2M, L2L updates)
    for (size_t a = 0; a < affected.size(); ++a) {
      const int b = affected[a];
      const int k1 = newU[a].c;
      ++compressions;
      if (k1 != L_.k.at(b)) {
        Mat& Ud = L_.Ud.at(b);
        Ud = pad(Ud, k1, Ud.c);
        Mat& Vd = L_.Vd.at(b);
        Vd = pad(Vd, k1, Vd.c);
        for (int c : ls.il[l].at(b)) {
          Mat& A1 = L_.A.at(key(b, c));
          A1 = pad(A1, k1, A1.c);
          Mat& A2 = L_.A.at(key(c, b));
          A2 = pad(A2, A2.r, k1);
        }
        L_.k.at(b) = k1;
      }
    }
    for (size_t a = 0; a < affected.size(); ++a) {
      L_.U.at(affected[a]) = newU[a];
      L_.V.at(affected[a]) = std::move(newU[a]);
    }
    // redirect the fill-ins (Galerkin projection onto the new bases)
    std::vector<std::pair<int, int>> dirs;
    for (auto& pr : S) {
      dirs.push_back({pr.first, pr.second});
      dirs.push_back({pr.second, pr.first});
    }
#pragma omp parallel for schedule(dynamic, 4) num_threads(threads)
    for (size_t e = 0; e < dirs.size(); ++e) {
      const int x = dirs[e].first, y = dirs[e].second;
      const Mat& Fxy = L_.F.at(key(x, y));
      Mat& A = L_.A.at(key(x, y));
      const bool Ex = L_.E.at(x), Ey = L_.E.at(y);
      if (!Ex && !Ey) {                                         // P2P
        Mat T1 = mul(L_.U.at(x), true, Fxy, false);
        gemm(T1, false, L_.V.at(y), false, A, 1.0, true);
      } else if (Ex && !Ey) {                                   // P2L
        gemm(Fxy, false, L_.V.at(y), false, A, 1.0, true);
      } else if (!Ex && Ey) {                                   // M2P
        gemm(L_.U.at(x), true, Fxy, false, A, 1.0, true);
      }
    }
    for (auto& pr : S) {
      L_.F.erase(key(pr.first, pr.second));
      L_.F.erase(key(pr.second, pr.first));
      L_.pending.erase(pr);
    }
  }

  // where a Schur update of (p, q) lands (O7(ii)): near block, M2L block, or far fill-in slot
  Mat* target(Level& L_, int p, int q) {
    const int l = L_.l;
    if (in_near(l, p, q)) return &L_.nearb.at(key(p, q));
    if (L_.E.at(p) && L_.E.at(q)) return &L_.A.at(key(p, q));
    if (!(in_il(l, p, q) && cheb(l, p, q) == 2)) throw OracleError(-5, "fill-in outside distance-2 far pairs");
    auto it = L_.F.find(key(p, q));
    if (it == L_.F.end()) it = L_.F.emplace(key(p, q), Mat(live(L_, p), live(L_, q))).first;
    L_.pending.insert({std::min(p, q), std::max(p, q)});
    return &it->second;
  }

  // elimination of the boxes of one colour (Table 4)
  void eliminate_colour(Level& L_, const std::vector<int>& cs, const std::set<int>& full) {
    const int l = L_.l;
    struct Work {
      Mat G;
      std::vector<int> nb;
      std::vector<Mat> W;   // G[:, :m] R_q per q in nb
    };
    std::vector<Work> wk(cs.size());
    std::string err;
    int ecode = 0;
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads)
    for (size_t a = 0; a < cs.size(); ++a) {
      const int i = cs[a];
      const int m = L_.m.at(i), k = L_.k.at(i);
      Mat P(m + k, m + k);
      const Mat& Kii = L_.nearb.at(key(i, i));
      const Mat& U = L_.U.at(i);
      const Mat& V = L_.V.at(i);
      for (int j = 0; j < m; ++j)
        for (int r = 0; r < m; ++r) P(r, j) = Kii(r, j);
      for (int j = 0; j < k; ++j)
        for (int r = 0; r < m; ++r) {
          P(r, m + j) = U(r, j);
          P(m + j, r) = V(r, j);
        }
      Work& w = wk[a];
      if (!inverse(P, w.G)) {
#pragma omp critical
        {
          if (!ecode) { ecode = -5; err = "singular box pivot at level " + std::to_string(l) + " box " + std::to_string(i); }
        }
        continue;
      }
      for (int q : ls.nearl[l].at(i))
        if (q != i) w.nb.push_back(q);
      const Mat G1 = sub(w.G, 0, m + k, 0, m);
      for (int q : w.nb) w.W.push_back(mul(G1, false, L_.nearb.at(key(i, q)), false));
    }
    if (ecode) throw OracleError(ecode, err);
    // Schur updates: targets created serially; each target then receives its contributions in
    // ascending order of the eliminated box (the serial loop order), targets in parallel
    struct Contrib {
      int a, pi, qi;
    };
    std::vector<Mat*> tptr;
    std::vector<std::vector<Contrib>> tc;
    std::unordered_map<Mat*, int> tix;
    for (size_t a = 0; a < cs.size(); ++a) {
      if (full.count(cs[a])) continue;              // R28: G11 = 0, no Schur update
      const Work& w = wk[a];
      for (size_t pi = 0; pi < w.nb.size(); ++pi)
        for (size_t qi = 0; qi < w.nb.size(); ++qi) {
          Mat* T = target(L_, w.nb[pi], w.nb[qi]);
          auto it = tix.find(T);
          if (it == tix.end()) {
            it = tix.emplace(T, (int)tptr.size()).first;
            tptr.push_back(T);
            tc.emplace_back();
          }
          tc[it->second].push_back(Contrib{(int)a, (int)pi, (int)qi});
        }
    }
#pragma omp parallel for schedule(dynamic, 8) num_threads(threads)
    for (size_t e = 0; e < tptr.size(); ++e) {
      for (const Contrib& ct : tc[e]) {
        const int i = cs[ct.a];
        const int m = L_.m.at(i);
        const Work& w = wk[ct.a];
        const Mat& Cp = L_.nearb.at(key(w.nb[ct.pi], i));
        const Mat Wq = sub(w.W[ct.qi], 0, m, 0, w.W[ct.qi].c);
        Mat upd = mul(Cp, false, Wq, false);
        Mat& T = *tptr[e];
        for (size_t z = 0; z < T.a.size(); ++z) T.a[z] = T.a[z] - upd.a[z];
      }
    }
    // records (snapshots of the multiplier blocks) and the new blocks
    for (size_t a = 0; a < cs.size(); ++a) {
      const int i = cs[a];
      const int m = L_.m.at(i), k = L_.k.at(i);
      Work& w = wk[a];
      Rec r;
      r.m = m;
      r.k = k;
      for (size_t qi = 0; qi < w.nb.size(); ++qi) {
        const int q = w.nb[qi];
        r.R.push_back({q, {std::move(L_.nearb.at(key(i, q))), (bool)L_.E.at(q)}});
        r.C.push_back({q, {std::move(L_.nearb.at(key(q, i))), (bool)L_.E.at(q)}});
      }
      const Mat G12 = sub(w.G, 0, m, m, m + k);
      for (size_t pi = 0; pi < w.nb.size(); ++pi)     // (X_p | Z_p, y_i) = C G12
        L_.nearb.at(key(w.nb[pi], i)) = mul(r.C[pi].second.first, false, G12, false);
      for (size_t qi = 0; qi < w.nb.size(); ++qi)     // (Z_i, x_q | y_q) = G21 R
        L_.nearb.at(key(i, w.nb[qi])) = sub(w.W[qi], m, m + k, 0, w.W[qi].c);
      Mat G22 = sub(w.G, m, m + k, m, m + k);
      for (double& v : G22.a) v = -v;
      L_.nearb.at(key(i, i)) = std::move(G22);        // (Z_i, y_i) = -G22 (R17)
      r.G = std::move(w.G);
      L_.rec[i] = std::move(r);
    }
  }

  void factor() {
    auto t0 = std::chrono::steady_clock::now();
    lv.assign(t.L + 1, Level{});
    for (int l = t.L; l >= 2; --l) {
      setup_level(l);
      if (l < t.L) {                                   // level l+1's blocks are no longer needed
        Level& pv = lv[l + 1];
        pv.nearb.clear();
        pv.A.clear();
        pv.U.clear();
        pv.V.clear();
        pv.Ud.clear();
        pv.Vd.clear();
      }
      Level& L_ = lv[l];
      int ncol = 0;
      for (auto& kv : colour[l]) ncol = std::max(ncol, kv.second + 1);
      for (int c = 0; c < ncol; ++c) {
        std::vector<int> cs;
        for (int b : L_.boxes)
          if (colour[l].at(b) == c) cs.push_back(b);
        std::set<int> cset(cs.begin(), cs.end());
        std::vector<std::pair<int, int>> S;
        for (auto& pr : L_.pending)
          if (cset.count(pr.first) || cset.count(pr.second)) S.push_back(pr);
        std::set<int> full;   // R28, decided when the colour begins
        for (int i : cs)
          if (L_.m.at(i) > 0 && L_.k.at(i) >= L_.m.at(i)) full.insert(i);
        if (!S.empty()) compress(L_, S);
        eliminate_colour(L_, cs, full);
        for (int i : cs) L_.E.at(i) = 1;
        if (algorithm == 2 && !L_.pending.empty()) {   // Alg. 2: compress on creation (R29)
          std::vector<std::pair<int, int>> all(L_.pending.begin(), L_.pending.end());
          compress(L_, all);
        }
      }
      if (!L_.pending.empty() || !L_.F.empty()) throw OracleError(-5, "pending far fill-ins at level end");
    }
    // top: (Z_p, y_q) over the level-2 boxes
    Level& L2 = lv[2];
    int o = 0;
    for (int b : L2.boxes) {
      top_offs[b] = {o, o + L2.k.at(b)};
      o += L2.k.at(b);
    }
    top = Mat(o, o);
    for (int p : L2.boxes)
      for (int q : L2.boxes) {
        const Mat& blk = in_near(2, p, q) ? L2.nearb.at(key(p, q)) : L2.A.at(key(p, q));
        for (int j = 0; j < blk.c; ++j)
          for (int i = 0; i < blk.r; ++i) top(top_offs[p].first + i, top_offs[q].first + j) = blk(i, j);
      }
    if (o > 0 && !lu(top, top_piv)) throw OracleError(-5, "singular top system");
    L2.nearb.clear();
    L2.A.clear();
    factored = true;
    t_factor = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }

  // Algorithm 4; B, X: n x nrhs column-major, user order
  void solve(const double* Bu, int nrhs, double* Xu) {
    if (!factored) throw OracleError(-6, "solve before factor");
    auto t0 = std::chrono::steady_clock::now();
    const long long n = t.n;
    Mat Bs((int)n, nrhs);
    for (int c = 0; c < nrhs; ++c)
      for (long long j = 0; j < n; ++j) {
        const double v = Bu[(size_t)c * n + t.perm[j]];
        if (!std::isfinite(v)) throw OracleError(-2, "non-finite right-hand side");
        Bs((int)j, c) = v;
      }
    std::vector<std::unordered_map<int, Mat>> bX(t.L + 1), bZ(t.L + 1);
    for (int l = t.L; l >= 2; --l) {
      Level& L_ = lv[l];
      for (int b : L_.boxes) {
        if (l == t.L) {
          bX[l][b] = sub(Bs, (int)t.off[l][b], (int)t.off[l][b + 1], 0, nrhs);
        } else {
          std::vector<const Mat*> v;
          for (int c : t.children(l, b)) v.push_back(&bZ[l + 1].at(c));
          bX[l][b] = vcat(v, nrhs);
        }
        bZ[l][b] = Mat(L_.k.at(b), nrhs);
      }
      int ncol = 0;
      for (auto& kv : colour[l]) ncol = std::max(ncol, kv.second + 1);
      for (int c = 0; c < ncol; ++c)
        for (int i : L_.boxes) {
          if (colour[l].at(i) != c) continue;
          const Rec& r = L_.rec.at(i);
          const int m = r.m;
          const Mat w = mul(sub(r.G, 0, r.G.r, 0, m), false, bX[l].at(i), false);
          const Mat wx = sub(w, 0, m, 0, nrhs);
          for (auto& pc : r.C) {
            Mat& tgt = pc.second.second ? bZ[l].at(pc.first) : bX[l].at(pc.first);
            gemm(pc.second.first, false, wx, false, tgt, -1.0, true);
          }
          Mat& z = bZ[l].at(i);
          for (int cc = 0; cc < nrhs; ++cc)
            for (int q = 0; q < r.k; ++q) z(q, cc) += w(m + q, cc);
        }
    }
    Level& L2 = lv[2];
    std::vector<const Mat*> v;
    for (int b : L2.boxes) v.push_back(&bZ[2].at(b));
    Mat rhs = vcat(v, nrhs);
    if (rhs.r) lu_solve(top, top_piv, rhs);
    std::vector<std::unordered_map<int, Mat>> y(t.L + 2), x(t.L + 1);
    for (int b : L2.boxes) y[2][b] = sub(rhs, top_offs[b].first, top_offs[b].second, 0, nrhs);
    for (int l = 2; l <= t.L; ++l) {
      Level& L_ = lv[l];
      int ncol = 0;
      for (auto& kv : colour[l]) ncol = std::max(ncol, kv.second + 1);
      for (int c = ncol - 1; c >= 0; --c)
        for (auto it = L_.boxes.rbegin(); it != L_.boxes.rend(); ++it) {
          const int i = *it;
          if (colour[l].at(i) != c) continue;
          const Rec& r = L_.rec.at(i);
          const int m = r.m;
          Mat rr = bX[l].at(i);
          for (auto& pr : r.R) gemm(pr.second.first, false, pr.second.second ? y[l].at(pr.first) : x[l].at(pr.first), false, rr, -1.0, true);
          std::vector<const Mat*> st{&rr, &y[l].at(i)};
          Mat xz = mul(r.G, false, vcat(st, nrhs), false);
          x[l][i] = sub(xz, 0, m, 0, nrhs);
        }
      if (l < t.L)
        for (int b : L_.boxes)
          for (int c : t.children(l, b)) {
            auto ro = L_.xoff.at({b, c});
            y[l + 1][c] = sub(x[l].at(b), ro.first, ro.second, 0, nrhs);
          }
    }
    for (int b : lv[t.L].boxes) {
      const Mat& xb = x[t.L].at(b);
      for (int c = 0; c < nrhs; ++c)
        for (long long j = t.off[t.L][b]; j < t.off[t.L][b + 1]; ++j)
          Xu[(size_t)c * n + t.perm[j]] = xb((int)(j - t.off[t.L][b]), c);
    }
    t_solve = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
};

thread_local std::string g_err;

}  // namespace

// ============================================================================== C interface
extern "C" {

const char* oc_last_error() { return g_err.c_str(); }

// build: tree, lists, colours, NNCA (ACA at eps = tol / 100, R18).  Returns a handle or NULL.
void* oc_build(const double* pts, long long n, int d, int kid, const double* kparams, int leaf, double tol,
               double tol_c, int threads, int* err) {
  try {
    auto t0 = std::chrono::steady_clock::now();
    Oracle* o = new Oracle();
    o->K = Kern{kid, d, kparams[0], kparams[1]};
    o->tol = tol;
    o->tol_c = tol_c < 0 ? tol : tol_c;
    o->threads = std::max(1, threads);
    try {
      build_tree(o->t, pts, n, d, leaf);
      build_lists(o->t, o->ls);
      o->colour.assign(o->t.L + 1, {});
      for (int l = 2; l <= o->t.L; ++l) o->colour[l] = greedy_colours(o->ls.nearl[l]);
      build_nnca(o->t, o->ls, o->K, tol / 100.0, o->nn, o->threads);
    } catch (...) {
      delete o;
      throw;
    }
    o->t_build = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *err = 0;
    return o;
  } catch (const OracleError& e) {
    g_err = e.what();
    *err = e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    *err = -9;
  }
  return nullptr;
}

int oc_factor(void* h) {
  try {
    static_cast<Oracle*>(h)->factor();
    return 0;
  } catch (const OracleError& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -9;
  }
}

int oc_solve(void* h, const double* B, int nrhs, double* X) {
  try {
    static_cast<Oracle*>(h)->solve(B, nrhs, X);
    return 0;
  } catch (const OracleError& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -9;
  }
}

void oc_free(void* h) { delete static_cast<Oracle*>(h); }
// before oc_factor: 3 = Algorithm 3 (default), 2 = Algorithm 2
int oc_set_algorithm(void* h, int alg) {
  if (alg != 2 && alg != 3) return -1;
  static_cast<Oracle*>(h)->algorithm = alg;
  return 0;
}

int oc_depth(void* h) { return static_cast<Oracle*>(h)->t.L; }
void oc_perm(void* h, long long* perm) {
  auto& t = static_cast<Oracle*>(h)->t;
  std::memcpy(perm, t.perm.data(), sizeof(long long) * t.n);
}
void oc_offsets(void* h, int l, long long* off) {
  auto& t = static_cast<Oracle*>(h)->t;
  std::memcpy(off, t.off[l].data(), sizeof(long long) * t.off[l].size());
}
// CSR over all 2^(d l) boxes (empty boxes: empty lists); idx arrays may be NULL (sizes only)
void oc_lists(void* h, int l, int* nptr, int* nidx, int* iptr, int* iidx) {
  Oracle* o = static_cast<Oracle*>(h);
  const int nb = o->t.nboxes(l);
  nptr[0] = iptr[0] = 0;
  for (int b = 0; b < nb; ++b) {
    auto it = o->ls.nearl[l].find(b);
    const std::vector<int>* nv = (it != o->ls.nearl[l].end()) ? &it->second : nullptr;
    const std::vector<int>* iv = nv ? &o->ls.il[l].at(b) : nullptr;
    nptr[b + 1] = nptr[b] + (nv ? (int)nv->size() : 0);
    iptr[b + 1] = iptr[b] + (iv ? (int)iv->size() : 0);
    if (nidx && nv) std::copy(nv->begin(), nv->end(), nidx + nptr[b]);
    if (iidx && iv) std::copy(iv->begin(), iv->end(), iidx + iptr[b]);
  }
}
void oc_colours(void* h, int l, int* col) {
  Oracle* o = static_cast<Oracle*>(h);
  for (int b = 0; b < o->t.nboxes(l); ++b) {
    auto it = o->colour[l].find(b);
    col[b] = (it == o->colour[l].end()) ? -1 : it->second;
  }
}
// which = 0: NNCA rank; 1: final rank after factor (0 for empty boxes)
void oc_ranks(void* h, int l, int which, int* r) {
  Oracle* o = static_cast<Oracle*>(h);
  for (int b = 0; b < o->t.nboxes(l); ++b) {
    r[b] = 0;
    auto it = o->nn[l].sk.find(b);
    if (it == o->nn[l].sk.end()) continue;
    r[b] = which ? o->lv[l].k.at(b) : (int)it->second.size();
  }
}
// skeleton of box b at level l (tree-order point indices); returns the count (out may be NULL)
int oc_skeleton(void* h, int l, int b, long long* out) {
  Oracle* o = static_cast<Oracle*>(h);
  auto it = o->nn[l].sk.find(b);
  if (it == o->nn[l].sk.end()) return 0;
  if (out) std::copy(it->second.begin(), it->second.end(), out);
  return (int)it->second.size();
}
// {build_s, factor_s, solve_s, compressions, top_size}
void oc_stats(void* h, double* out) {
  Oracle* o = static_cast<Oracle*>(h);
  out[0] = o->t_build;
  out[1] = o->t_factor;
  out[2] = o->t_solve;
  out[3] = (double)o->compressions;
  out[4] = (double)o->top.r;
}

}  // extern "C"
