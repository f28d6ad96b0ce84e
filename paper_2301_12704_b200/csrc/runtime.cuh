// runtime.cuh — host-side runtime pieces of libaifmm: device pools, task upload arena, batch builders.
#pragma once
#include <exception>
#include <thread>
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <string>
#include <cstring>
#include <cstdlib>
#include <map>
#include <set>
#include <unordered_map>
#include <vector>

#include "common.cuh"

namespace aifmm {

// launchers (dense_kernels.cu, tree_kernels.cu, nnca_kernels.cu)
void launch_gemm(int tileclass, const GemmTask* t, const GemmTerm* tm, const GemmTile* tiles, int ntiles, cudaStream_t s);
void launch_gj(const GJTask* t, int ntasks, int nmax, int mode, cudaStream_t s);
void launch_pqr(const PqrTask* t, int ntasks, size_t smem_doubles, cudaStream_t s);
void launch_pqr_cluster(const PqrTask* t, int ntasks, cudaStream_t s);
void launch_keval(const KEvalTask* t, int ntasks, int ysplit, const double* pts, KernelParams kp, int* flag, cudaStream_t s);
constexpr int ORTH_SW_KMAX = 64;   // = SW_KMAX of orth_sandwich_kernel
void launch_orth_sandwich(const void* v, const int* cnt, const int* idx, int nb, int cap, const double* const* T,
                          const double* const* T2, cudaStream_t s);
void launch_keval_table(const void* v, const int* cnt, const int* idx, int nb, int cap, int mode, const int* sk,
                        const long long* base, const double* pts, KernelParams kp, int* flag, cudaStream_t s);
void launch_copy(const CopyTask* t, int ntasks, int ysplit, cudaStream_t s);
void launch_norm(const NormTask* t, int ntasks, cudaStream_t s);
void launch_chol_inv(const CholTask* t, int ntasks, int kmax, cudaStream_t s);
void launch_gj_panel(const void* t, int ntasks, int j, cudaStream_t s);
void launch_gj_panel_cluster(const void* t, int ntasks, int j, int nmax, cudaStream_t s);
void launch_gj_unscramble(const void* t, int ntasks, int nmax, cudaStream_t s);
void launch_gj_fused(const void* t, int ntasks, int nmax, cudaStream_t s);
size_t gjb_task_size();
void gjb_make(void* out, double* A, int lda, int n, double* PW, double* Bws, int* piv, int* info);
size_t hh_task_size();
void hh_make(void* out, double* A, int lda, int n, int m, double* V, double* T);
void launch_hh_panel(const void* t, int ntasks, int j, cudaStream_t s, int mode, int nmax);
void launch_hh_extract(const void* t, int ntasks, double* const* out, const int* ldo, cudaStream_t s);
void launch_hh_update(const void* tasks, const void* tiles, int ntiles, int j, cudaStream_t s,
                      double* zbuf = nullptr, int seg = 0, int nseg = 0);
void launch_hh_update_pass(const void* tasks, const void* tiles, int ntiles, int j, cudaStream_t s,
                           double* zbuf, int seg, int nseg, int pass);
constexpr int HH_PANEL = 32;
constexpr int GJ_SMALL_MAX = 160;  // in-place inverses up to this size run in shared memory (<= 206 KB)
constexpr int GJ_PANEL = 32;

// Batches with >= 296 independent tasks, or >= this many moderate-size ones, run one CTA per
// task (they fill the GPU); smaller batches of long tasks spread each task over an 8-CTA
// cluster (measured on configs 2 and 3).  AIFMM_MANY overrides.
inline int many_threshold() {
  static const int v = [] {
    const char* e = getenv("AIFMM_MANY");
    return e ? atoi(e) : 96;
  }();
  return v;
}

// Optional phase profile (AIFMM_PROFILE=1): synchronises at phase boundaries and prints a
// breakdown to stderr at the end of factor / solve.  Off by default (no extra syncs).
struct Prof {
  bool on = false;
  std::map<std::string, double> ms;
  std::chrono::steady_clock::time_point t0;
  cudaStream_t s = nullptr;
  void begin(cudaStream_t st) { if (!on) return; s = st; cudaStreamSynchronize(s); t0 = std::chrono::steady_clock::now(); }
  void end(const char* name) {
    if (!on) return;
    cudaStreamSynchronize(s);
    ms[name] += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  }
  // host-only lap timer (no stream synchronisation): accumulates under "h.<name>"
  std::chrono::steady_clock::time_point hl;
  void hstart() { if (on) hl = std::chrono::steady_clock::now(); }
  void hlap(const char* name) {
    if (!on) return;
    auto t = std::chrono::steady_clock::now();
    ms[std::string("h.") + name] += std::chrono::duration<double, std::milli>(t - hl).count();
    hl = t;
  }
  void dump(const char* title) {
    if (!on) return;
    fprintf(stderr, "[aifmm profile] %s:", title);
    for (auto& kv : ms) fprintf(stderr, " %s=%.2fms", kv.first.c_str(), kv.second);
    fprintf(stderr, "\n");
    ms.clear();
  }
};
inline Prof g_prof;

// Exposed host time (AIFMM_EXPOSE=1): wall time from a stream synchronisation returning to the
// next kernel launch -- the GPU is idle for all of it -- accumulated under the current phase.
struct Exposure {
  bool on = getenv("AIFMM_EXPOSE") != nullptr;
  const char* phase = "?";
  bool pending = false;
  std::chrono::steady_clock::time_point t;
  std::map<std::string, std::pair<double, int>> ms;
  std::map<std::string, double> wall;   // host wall time per phase (incl. waits)
  double wait_ms = 0.0;                 // host blocked in stream synchronisations
  std::chrono::steady_clock::time_point tw, tph;
  void set(const char* p) {
    if (!on) { phase = p; return; }
    auto n = std::chrono::steady_clock::now();
    wall[phase] += std::chrono::duration<double, std::milli>(n - tph).count();
    tph = n;
    phase = p;
  }
  void wait_begin() { if (on) tw = std::chrono::steady_clock::now(); }
  void synced() {
    if (on) {
      pending = true;
      t = std::chrono::steady_clock::now();
      wait_ms += std::chrono::duration<double, std::milli>(t - tw).count();
    }
  }
  void launching() {
    if (!on || !pending) return;
    auto& e = ms[phase];
    e.first += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t).count();
    e.second += 1;
    pending = false;
  }
  void dump() {
    if (!on) return;
    fprintf(stderr, "[aifmm exposed host ms]");
    for (auto& kv : ms) fprintf(stderr, " %s=%.2f(%d)", kv.first.c_str(), kv.second.first, kv.second.second);
    fprintf(stderr, " | sync wait %.2f | wall:", wait_ms);
    for (auto& kv : wall) fprintf(stderr, " %s=%.2f", kv.first.c_str(), kv.second);
    fprintf(stderr, "\n");
    ms.clear();
    wall.clear();
    wait_ms = 0.0;
  }
};
inline Exposure g_expose;

// ---------------------------------------------------------------------------------- pools
// Device memory: one process-wide cache of fixed-size chunks (oversize requests get a
// dedicated chunk) shared by every pool, so the per-level pools hand chunks to each other
// instead of going through cudaMalloc/cudaFree; under memory pressure the cache gives its
// idle chunks back and the allocation is retried once.  All work runs on one stream, so a
// chunk returned by reset() can be handed out again at once (stream order).
class ChunkCache {
 public:
  static constexpr size_t CH = (size_t)512 << 20;
  void* get(size_t bytes, size_t* got) {
    if (bytes <= CH) {
      *got = CH;
      if (!free_.empty()) {
        void* p = free_.back();
        free_.pop_back();
        return p;
      }
      return fresh(CH);
    }
    // oversize: best fit among the idle oversize chunks
    size_t best = (size_t)-1;
    for (size_t i = 0; i < big_.size(); ++i)
      if (big_[i].second >= bytes && (best == (size_t)-1 || big_[i].second < big_[best].second)) best = i;
    if (best != (size_t)-1 && big_[best].second <= 2 * bytes) {
      auto r = big_[best];
      big_.erase(big_.begin() + best);
      *got = r.second;
      return r.first;
    }
    const size_t sz = (bytes + CH - 1) / CH * CH;
    *got = sz;
    return fresh(sz);
  }
  void put(void* p, size_t sz) {
    if (sz == CH) free_.push_back(p);
    else big_.push_back({p, sz});
  }
  // give every idle chunk back to the driver
  void trim() {
    if (free_.empty() && big_.empty()) return;
    cudaDeviceSynchronize();
    for (void* p : free_) { cudaFree(p); total_ -= CH; }
    for (auto& b : big_) { cudaFree(b.first); total_ -= b.second; }
    free_.clear();
    big_.clear();
  }
  size_t total() const { return total_; }
  size_t idle() const {
    size_t t = free_.size() * CH;
    for (auto& b : big_) t += b.second;
    return t;
  }

 private:
  void* fresh(size_t sz) {
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, sz);
    if (e == cudaErrorMemoryAllocation) {
      cudaGetLastError();
      trim();
      e = cudaMalloc(&p, sz);
    }
    AIFMM_CUDA(e);
    total_ += sz;
    return p;
  }
  std::vector<void*> free_;
  std::vector<std::pair<void*, size_t>> big_;
  size_t total_ = 0;
};
inline ChunkCache& chunk_cache() {
  static ChunkCache* c = new ChunkCache();   // never destroyed: chunks die with the context
  return *c;
}

// Bump allocator over chunks of the cache.  Blocks live until reset() returns the chunks.
class DevPool {
 public:
  explicit DevPool(size_t = 0) {}
  ~DevPool() { reset(); }
  DevPool(const DevPool&) = delete;
  DevPool& operator=(const DevPool&) = delete;
  void* alloc(size_t bytes) {
    bytes = (bytes + 255) & ~(size_t)255;
    if (bytes == 0) bytes = 256;
    if (!chunks_.empty() && used_ + bytes <= chunks_.back().second) {
      void* p = static_cast<char*>(chunks_.back().first) + used_;
      used_ += bytes;
      return p;
    }
    size_t got = 0;
    void* p = chunk_cache().get(bytes, &got);
    chunks_.push_back({p, got});
    held_ += got;
    used_ = bytes;
    return p;
  }
  double* d(size_t n) { return static_cast<double*>(alloc(n * sizeof(double))); }
  int* i(size_t n) { return static_cast<int*>(alloc(n * sizeof(int))); }
  // return every chunk to the cache (the blocks are dead; stream order makes reuse safe)
  void reset() {
    for (auto& c : chunks_) chunk_cache().put(c.first, c.second);
    chunks_.clear();
    used_ = 0;
    held_ = 0;
  }
  void recycle() { reset(); }
  size_t total() const { return held_; }
  size_t nchunks() const { return chunks_.size(); }

 private:
  std::vector<std::pair<void*, size_t>> chunks_;
  size_t used_ = 0, held_ = 0;
};

// Pinned host staging + device mirror for task arrays.  Appends are copied H2D by the next
// flush(); the region is reused only after sync() (stream synchronised), which bumps gen():
// a device pointer returned by put() is valid only while gen() is unchanged, so a caller that
// keeps one across calls that may sync (reserve / put / GemmBatch::run) must re-put its data
// when gen() moved (see batched_inverse, batched_tri_root).
class Uploader {
 public:
  void init(cudaStream_t s, size_t cap = (size_t)256 << 20) {
    s_ = s;
    grow(cap);
  }
  // switch to another stream: everything staged so far is flushed and completed on the old one
  void set_stream(cudaStream_t s) {
    if (h_) sync();
    s_ = s;
  }
  unsigned long long gen() const { return gen_; }
  ~Uploader() { free_all(); }
  void free_all() {
    if (h_) cudaFreeHost(h_);
    if (d_) cudaFree(d_);
    h_ = nullptr;
    d_ = nullptr;
    cap_ = used_ = flushed_ = 0;
  }
  template <class T>
  T* put(const T* src, size_t n) {
    size_t bytes = n * sizeof(T);
    size_t need = (bytes + 255) & ~(size_t)255;
    if (need == 0) return nullptr;
    if (used_ + need > cap_) {
      sync();
      if (need > cap_) grow(std::max(need, cap_ * 2));
    }
    std::memcpy(h_ + used_, src, bytes);
    T* out = reinterpret_cast<T*>(d_ + used_);
    used_ += need;
    return out;   // copied to the device by the next flush() (before the next kernel launch)
  }
  // one host-to-device copy of everything staged since the last flush
  void flush() {
    if (used_ > flushed_) {
      AIFMM_CUDA(cudaMemcpyAsync(d_ + flushed_, h_ + flushed_, used_ - flushed_, cudaMemcpyHostToDevice, s_));
      flushed_ = used_;
    }
  }
  template <class T>
  T* put(const std::vector<T>& v) { return put(v.data(), v.size()); }
  // make room for `bytes` of consecutive puts (so a batch never straddles a reset)
  void reserve(size_t bytes) {
    bytes += 4096;
    if (used_ + bytes <= cap_) return;
    sync();
    if (bytes > cap_) grow(std::max(bytes, cap_ * 2));
  }
  void sync() {
    flush();
    g_expose.wait_begin();
    AIFMM_CUDA(cudaStreamSynchronize(s_));
    used_ = flushed_ = 0;
    ++syncs;
    ++gen_;
    g_expose.synced();
  }
  long long syncs = 0;

 private:
  void grow(size_t cap) {
    if (h_) { flush(); AIFMM_CUDA(cudaStreamSynchronize(s_)); cudaFreeHost(h_); cudaFree(d_); }
    AIFMM_CUDA(cudaMallocHost(&h_, cap));
    AIFMM_CUDA(cudaMalloc(&d_, cap));
    cap_ = cap;
    used_ = flushed_ = 0;
    ++gen_;
  }
  unsigned long long gen_ = 0;
  cudaStream_t s_ = 0;
  char* h_ = nullptr;
  char* d_ = nullptr;
  size_t cap_ = 0, used_ = 0, flushed_ = 0;
};

// ---------------------------------------------------------------------------------- batches
struct Blk {
  double* p = nullptr;
  int ld = 0, rows = 0, cols = 0;
  double* at(int r, int c) const { return p + (size_t)c * ld + r; }
};

struct FlopCounter {
  double flops = 0.0, bytes = 0.0;
};

class GemmBatch {
 public:
  int task(double* C, int ldc, int M, int N, double beta) {
    GemmTask t{C, ldc, M, N, beta, (int)terms_.size(), (int)terms_.size()};
    tasks_.push_back(t);
    return (int)tasks_.size() - 1;
  }
  // term on the LAST task
  void term(double alpha, const double* A, int lda, int transA, const double* B, int ldb, int transB, int K) {
    GemmTerm tm{A, B, lda, ldb, K, transA, transB, alpha};
    terms_.push_back(tm);
    tasks_.back().term_end = (int)terms_.size();
  }
  void add(double alpha, const double* B, int ldb, int transB) { term(alpha, nullptr, 0, 0, B, ldb, transB, 0); }
  bool empty() const { return tasks_.empty(); }
  size_t size() const { return tasks_.size(); }
  size_t nterms() const { return terms_.size(); }
  // o's tasks after this batch's (term indices shifted; order preserved)
  void append(const GemmBatch& o) {
    const int off = (int)terms_.size();
    for (GemmTask t : o.tasks_) {
      t.term_begin += off;
      t.term_end += off;
      tasks_.push_back(t);
    }
    terms_.insert(terms_.end(), o.terms_.begin(), o.terms_.end());
  }
  GemmTerm& term_ref(size_t i) { return terms_[i]; }
  // the tasks with keep[t] != 0, with their terms, in the same order (a rank runs
  // the tasks it owns; each task's arithmetic is unchanged)
  GemmBatch filtered(const std::vector<char>& keep) const {
    GemmBatch o;
    o.splitk_ = splitk_;
    for (size_t t = 0; t < tasks_.size(); ++t) {
      if (!keep[t]) continue;
      GemmTask k = tasks_[t];
      const int b = (int)o.terms_.size();
      o.terms_.insert(o.terms_.end(), terms_.begin() + k.term_begin, terms_.begin() + k.term_end);
      k.term_begin = b;
      k.term_end = (int)o.terms_.size();
      o.tasks_.push_back(k);
    }
    return o;
  }
  GemmTask& task_ref(size_t i) { return tasks_[i]; }
  // Deterministic split-K: single-term tasks with a long K and few output tiles are split into
  // S partial GEMMs into workspace slices, then reduced in a fixed order by a second launch.
  void set_splitk_pool(DevPool* p) { splitk_ = p; }
  void run(Uploader& up, cudaStream_t s, FlopCounter* fc = nullptr) {
    if (tasks_.empty()) return;
    std::vector<GemmTask> red_tasks;
    std::vector<GemmTerm> red_terms;
    if (splitk_) {
      const size_t nt0 = tasks_.size();
      for (size_t t = 0; t < nt0; ++t) {
        GemmTask k = tasks_[t];
        if (k.term_end - k.term_begin != 1) continue;
        GemmTerm tm = terms_[k.term_begin];
        if (!tm.A || k.M <= 0 || k.N <= 0) continue;
        const long long tiles = (long long)((k.M + 63) / 64) * ((k.N + 63) / 64);
        if (tm.K < 1024 || tiles >= 64) continue;
        int S = (int)std::min<long long>(32, std::max<long long>(2, tm.K / 384));
        const int kc = (tm.K + S - 1) / S;
        S = (tm.K + kc - 1) / kc;
        double* ws = splitk_->d((size_t)S * k.M * k.N);
        GemmTask r{k.C, k.ldc, k.M, k.N, k.beta, (int)red_terms.size(), (int)red_terms.size()};
        for (int q = 0; q < S; ++q) {
          const int k0 = q * kc, kl = std::min(kc, tm.K - k0);
          double* P = ws + (size_t)q * k.M * k.N;
          GemmTerm part = tm;
          part.K = kl;
          part.A = tm.transA ? tm.A + k0 : tm.A + (size_t)k0 * tm.lda;
          part.B = tm.transB ? tm.B + (size_t)k0 * tm.ldb : tm.B + k0;
          if (q == 0) {
            tasks_[t] = GemmTask{P, k.M, k.M, k.N, 0.0, k.term_begin, k.term_end};
            terms_[k.term_begin] = part;
          } else {
            tasks_.push_back(GemmTask{P, k.M, k.M, k.N, 0.0, (int)terms_.size(), (int)terms_.size() + 1});
            terms_.push_back(part);
          }
          red_terms.push_back(GemmTerm{nullptr, P, 0, k.M, 0, 0, 0, 1.0});
        }
        r.term_end = (int)red_terms.size();
        red_tasks.push_back(r);
      }
    }
    std::vector<GemmTile> tl[5];
    static const bool wide = getenv("AIFMM_GEMM_WIDE") != nullptr;   // experiment toggle
    for (size_t t = 0; t < tasks_.size(); ++t) {
      const GemmTask& k = tasks_[t];
      if (k.M <= 0 || k.N <= 0) continue;
      int cls = (k.M <= 32 ? 0 : 1) + (k.N <= 32 ? 0 : 2);
      // class ids: 0 -> 32x32, 1 -> 64x32, 2 -> 32x64, 3 -> 64x64, 4 -> 64x128
      if (wide && cls == 3 && k.N > 64) cls = 4;
      int bm = (cls & 1) || cls == 4 ? 64 : 32, bn = cls == 4 ? 128 : ((cls & 2) ? 64 : 32);
      for (int m0 = 0; m0 < k.M; m0 += bm)
        for (int n0 = 0; n0 < k.N; n0 += bn) tl[cls].push_back(GemmTile{(int)t, m0, n0, 0});
      if (fc) {
        fc->bytes += 8.0 * k.M * k.N * (k.beta != 0.0 ? 2.0 : 1.0);
        for (int q = k.term_begin; q < k.term_end; ++q) {
          const GemmTerm& tm = terms_[q];
          if (tm.A) {
            fc->flops += 2.0 * k.M * k.N * tm.K;
            fc->bytes += 8.0 * ((double)k.M * tm.K + (double)tm.K * k.N);
          } else {
            fc->flops += (double)k.M * k.N;
            fc->bytes += 8.0 * k.M * k.N;
          }
        }
      }
    }
    size_t need = tasks_.size() * sizeof(GemmTask) + terms_.size() * sizeof(GemmTerm) + 4 * 256;
    for (int c = 0; c < 5; ++c) need += tl[c].size() * sizeof(GemmTile);
    up.reserve(need);
    GemmTask* dt = up.put(tasks_);
    GemmTerm* dm = terms_.empty() ? nullptr : up.put(terms_);
    for (int c = 0; c < 5; ++c) {
      if (tl[c].empty()) continue;
      GemmTile* dtl = up.put(tl[c]);
      launch_gemm(c, dt, dm, dtl, (int)tl[c].size(), s);
    }
    tasks_.clear();
    terms_.clear();
    if (!red_tasks.empty()) {
      tasks_ = std::move(red_tasks);
      terms_ = std::move(red_terms);
      DevPool* keep = splitk_;
      splitk_ = nullptr;
      run(up, s, nullptr);
      splitk_ = keep;
    }
  }

 private:
  std::vector<GemmTask> tasks_;
  std::vector<GemmTerm> terms_;
  DevPool* splitk_ = nullptr;
};

// Host planning loops over boxes: contiguous chunks on up to 8 threads (serial for small n).
// fn(lo, hi, t) must only write thread-private outputs (merged by the caller in chunk order).
template <class F>
inline int parallel_chunks(int n, int min_per_thread, F&& fn) {
  const int hw = (int)std::max(1u, std::thread::hardware_concurrency());
  const int T = std::max(1, std::min({8, hw, n / std::max(min_per_thread, 1)}));
  if (T == 1) {
    fn(0, n, 0);
    return 1;
  }
  std::vector<std::thread> th;
  std::vector<std::exception_ptr> err(T);
  for (int t = 0; t < T; ++t)
    th.emplace_back([&, t] {
      try {
        fn((int)((long long)n * t / T), (int)((long long)n * (t + 1) / T), t);
      } catch (...) {
        err[t] = std::current_exception();
      }
    });
  for (auto& x : th) x.join();
  for (auto& e : err)
    if (e) std::rethrow_exception(e);   // the first failing chunk's error, on the calling thread
  return T;
}

class CopyBatch {
 public:
  void copy(const double* src, int lds, double* dst, int ldd, int rows, int cols, double alpha = 1.0, int trans = 0,
            int accumulate = 0) {
    if (rows <= 0 || cols <= 0) return;
    v_.push_back(CopyTask{src, dst, lds, ldd, rows, cols, trans, accumulate, alpha});
    maxel_ = std::max(maxel_, (long long)rows * cols);
  }
  void fill(double* dst, int ldd, int rows, int cols, double value) { copy(nullptr, 0, dst, ldd, rows, cols, value); }
  bool empty() const { return v_.empty(); }
  void append(const CopyBatch& o) {   // o's tasks after this batch's (order preserved)
    v_.insert(v_.end(), o.v_.begin(), o.v_.end());
    maxel_ = std::max(maxel_, o.maxel_);
  }
  void run(Uploader& up, cudaStream_t s) {
    if (v_.empty()) return;
    int ys = (int)std::min<long long>(64, std::max<long long>(1, maxel_ / 4096));
    launch_copy(up.put(v_), (int)v_.size(), ys, s);
    v_.clear();
    maxel_ = 0;
  }

 private:
  std::vector<CopyTask> v_;
  long long maxel_ = 0;
};


// Batched in-place matrix inverse (Gauss-Jordan, partial pivoting; reading R16).
// Small matrices: one CTA each in shared memory.  Larger: blocked GJ, one panel kernel per
// 32 columns plus one DMMA GEMM launch for the rank-32 update, batched across matrices.
struct InvReq {
  double* A;
  int lda, n;
  int* info;
};
// test hook (aifmm_debug_inverse_batch): 0 automatic routing, 1 panel + GEMM launches, 2 fused
inline int g_gj_force = 0;
template <class Pool>
inline void batched_inverse_impl(const std::vector<InvReq>& reqs, Pool& work, Uploader& up, cudaStream_t s,
                                 FlopCounter* fc);
// debug (AIFMM_DEBUG_INV=1): per call, the batch shape and its device time (synchronising)
template <class Pool>
inline void batched_inverse(const std::vector<InvReq>& reqs, Pool& work, Uploader& up, cudaStream_t s,
                            FlopCounter* fc = nullptr) {
  static const bool dbg = getenv("AIFMM_DEBUG_INV") != nullptr;
  if (!dbg) return batched_inverse_impl(reqs, work, up, s, fc);
  int cnt = 0, nmin = 1 << 30, nmax = 0;
  double fl = 0;
  for (const InvReq& r : reqs)
    if (r.n > 0) { ++cnt; nmin = std::min(nmin, r.n); nmax = std::max(nmax, r.n); fl += 2.0 * r.n * (double)r.n * r.n; }
  up.sync();
  auto t0 = std::chrono::steady_clock::now();
  batched_inverse_impl(reqs, work, up, s, fc);
  up.sync();
  const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  fprintf(stderr, "[aifmm inv] count %d n %d..%d  %.3f ms  %.2f TF/s\n", cnt, cnt ? nmin : 0, nmax, ms, fl / ms / 1e9);
}
template <class Pool>
inline void batched_inverse_impl(const std::vector<InvReq>& reqs, Pool& work, Uploader& up, cudaStream_t s,
                                 FlopCounter* fc) {
  std::vector<GJTask> small;
  int nsm = 0;
  std::vector<InvReq> big;
  for (const InvReq& r : reqs) {
    if (r.n <= 0) continue;
    if (r.n <= GJ_SMALL_MAX) {
      small.push_back(GJTask{r.A, r.lda, r.n, r.n, 0, r.info});
      nsm = std::max(nsm, r.n);
    } else {
      big.push_back(r);
    }
    if (fc) fc->flops += 2.0 * (double)r.n * r.n * r.n;
  }
  if (!small.empty()) {
    long long smem_d = (long long)nsm * nsm + nsm + nsm / 2 + 2;
    launch_gj(up.put(small), (int)small.size(), (int)smem_d, 1, s);
  }
  if (big.empty()) return;
  const size_t tsz = gjb_task_size();
  std::vector<char> tb(tsz * big.size());
  std::vector<double*> Bw(big.size());
  int nmax = 0;
  for (size_t i = 0; i < big.size(); ++i) {
    const InvReq& r = big[i];
    double* PW = work.d((size_t)r.n * GJ_PANEL);
    Bw[i] = work.d((size_t)r.n * GJ_PANEL);
    int* piv = work.i(r.n);
    gjb_make(tb.data() + i * tsz, r.A, r.lda, r.n, PW, Bw[i], piv, r.info);
    nmax = std::max(nmax, r.n);
  }
  const void* dt = up.put(tb.data(), tb.size());
  unsigned long long dgen = up.gen();
  // opt-in (AIFMM_GJ_FUSED_MIN = batch size from which it is used): one CTA per matrix runs all
  // panels and their DMMA updates in one launch.  Measured slower on config 3 (pivot inverses
  // 464 vs 398 ms: the rank-32 update is memory-bound either way and one CTA per matrix
  // serialises each matrix's panel latency with its update), so off by default
  static const int fused_min = getenv("AIFMM_GJ_FUSED_MIN") ? atoi(getenv("AIFMM_GJ_FUSED_MIN")) : 0;
  const bool fused = g_gj_force == 2 || (g_gj_force == 0 && fused_min > 0 && (int)big.size() >= fused_min);
  if (fused) {
    launch_gj_fused(dt, (int)big.size(), nmax, s);
    return;
  }
  // few matrices: 8-CTA clusters per matrix (row slices in shared memory); many: one CTA each
  static const bool gj_single = getenv("AIFMM_GJ_SINGLE") != nullptr;   // debug toggle
  static const int cl_max = getenv("AIFMM_GJ_CLUSTER_MAX") ? atoi(getenv("AIFMM_GJ_CLUSTER_MAX")) : 148;
  const bool cluster = !gj_single && (int)big.size() <= cl_max && nmax <= 8 * 700;
  for (int j = 0; j < nmax; j += GJ_PANEL) {
    if (up.gen() != dgen) { dt = up.put(tb.data(), tb.size()); dgen = up.gen(); }   // staging rewound
    if (cluster) launch_gj_panel_cluster(dt, (int)big.size(), j, nmax, s);
    else launch_gj_panel(dt, (int)big.size(), j, s);
    GemmBatch g;
    for (size_t i = 0; i < big.size(); ++i) {
      const InvReq& r = big[i];
      if (j >= r.n) continue;
      const int nbw = std::min(GJ_PANEL, r.n - j);
      if (j > 0) {
        g.task(r.A, r.lda, j, r.n, 1.0);
        g.term(-1.0, Bw[i], r.n, 0, r.A + j, r.lda, 0, nbw);
      }
      if (j + nbw < r.n) {
        g.task(r.A + j + nbw, r.lda, r.n - j - nbw, r.n, 1.0);
        g.term(-1.0, Bw[i] + j + nbw, r.n, 0, r.A + j, r.lda, 0, nbw);
      }
    }
    g.run(up, s);
  }
  if (up.gen() != dgen) dt = up.put(tb.data(), tb.size());
  launch_gj_unscramble(dt, (int)big.size(), nmax, s);
}


// Batched two-stage RRQR, first stage (reading R8b): for each tall A (n x m, lda) compute the
// Householder factor R and write M = R^T (m x min(n,m), ld ldm) to out.  A is destroyed.
struct TriRootReq {
  double* A;
  int lda, n, m;
  double* out;
  int ldm;
};
constexpr int HH_SMEM_ROWS = 768;   // = HHS_ROWS of hh_panel_smem_kernel
constexpr int HH_REG_ROWS = 512;    // = 256 threads x 2 rows of hh_panel_reg_kernel<2>
constexpr int HH_REGCL_ROWS = 4096; // = 8 CTAs x 256 threads x 2 rows of hh_panel_reg_cluster_kernel<2>
template <class Pool>
inline void batched_tri_root(const std::vector<TriRootReq>& reqs_in, Pool& work, Uploader& up, cudaStream_t s,
                             FlopCounter* fc = nullptr, int tsqr_m = -1) {
  if (reqs_in.empty()) return;
  // TSQR: a tall request (n > HH_REG_ROWS rows) is split into balanced row chunks of at most
  // HH_REG_ROWS rows.  Each chunk's R (min(n_c, m) x m upper trapezoid) goes into a stacked
  // buffer, rows in chunk order, and the stack is factored in turn (recursively; a split is only
  // made when the stack has <= 0.8 n rows): R([A_1; A_2; ...]) = R([R_1; R_2; ...]) up to the
  // signs of its rows, which the pivoted QR of the second stage (on R^T's columns) does not see.
  // Every chunk panel then lives in registers (hh_panel_reg_kernel).
  static const bool no_tsqr = getenv("AIFMM_NO_TSQR") != nullptr;   // debug toggle
  // the test hook aifmm_debug_tri_root forces chunks of HH_REG_ROWS rows for every request
  // Default (measured on config 3: factor -11%, config 2 neutral; chunks of 1024 / 2048 rows
  // were slower): requests taller than HH_REGCL_ROWS are split into balanced chunks of at most
  // HH_REGCL_ROWS rows, so every chunk panel lives in registers of an 8-CTA cluster instead of
  // running the global-memory cluster panel.  AIFMM_TSQR_{MMAX,ROWS,NMIN} override (experiments).
  static const int tsqr_env = getenv("AIFMM_TSQR_MMAX") ? atoi(getenv("AIFMM_TSQR_MMAX")) : (1 << 30);
  static const int tsqr_rows = getenv("AIFMM_TSQR_ROWS") ? atoi(getenv("AIFMM_TSQR_ROWS")) : HH_REGCL_ROWS;
  static const int tsqr_nmin = getenv("AIFMM_TSQR_NMIN") ? atoi(getenv("AIFMM_TSQR_NMIN")) : HH_REGCL_ROWS;
  const int tsqr_mmax = tsqr_m >= 0 ? tsqr_m : tsqr_env;
  const int CHR = tsqr_m >= 0 ? HH_REG_ROWS : tsqr_rows;
  const int NMIN = tsqr_m >= 0 ? 0 : tsqr_nmin;
  std::vector<TriRootReq> reqs, stacks;
  for (const TriRootReq& q : reqs_in) {
    bool split = !no_tsqr && q.m >= 1 && q.m <= tsqr_mmax && q.n > CHR && q.n > NMIN;
    int nch = 0, S = 0;
    if (split) {
      nch = (q.n + CHR - 1) / CHR;
      for (int c = 0; c < nch; ++c) S += std::min(q.n / nch + (c < q.n % nch ? 1 : 0), q.m);
      split = 5LL * S <= 4LL * q.n;
    }
    if (!split) {
      reqs.push_back(q);
      continue;
    }
    double* st = work.d((size_t)S * q.m);
    int row0 = 0, srow = 0;
    for (int c = 0; c < nch; ++c) {
      const int nc = q.n / nch + (c < q.n % nch ? 1 : 0);
      reqs.push_back(TriRootReq{q.A + row0, q.lda, nc, q.m, st + srow, -S});
      row0 += nc;
      srow += std::min(nc, q.m);
    }
    stacks.push_back(TriRootReq{st, S, S, q.m, q.out, q.ldm});
  }
  const size_t tsz = hh_task_size();
  // long panels (n >= 512 rows) go to the 8-CTA cluster kernel, short ones to one CTA
  // three classes: short panels (one CTA), long panels staged in the smem of an 8-CTA cluster,
  // very long panels (cluster, global memory)
  const int SM_ROWS = 8 * ((176 * 1024) / (HH_PANEL * 8));
  std::vector<TriRootReq> sorted_reqs;
  // enough tasks to fill the GPU with one CTA each: no clusters (their 8x more CTAs only add
  // waves of latency-bound panel steps)
  static const bool hh_cluster = getenv("AIFMM_HH_CLUSTER") != nullptr;   // debug toggle
  int nmax_rows = 0;
  for (const auto& q : reqs) nmax_rows = std::max(nmax_rows, q.n);
  const bool many = !hh_cluster && ((int)reqs.size() >= 2 * 148 ||
                                    ((int)reqs.size() >= many_threshold() && nmax_rows <= 4096));
  // classes: panels that fit one CTA's shared memory; other short or many panels (one CTA,
  // global memory); long panels staged in the smem of an 8-CTA cluster; very long (cluster, global)
  int nmax_rg = 0, nmax_sm = 0;
  for (const auto& q : reqs) if (q.n <= HH_REG_ROWS) { sorted_reqs.push_back(q); nmax_rg = std::max(nmax_rg, q.n); }
  const size_t nrg = sorted_reqs.size();
  // 512 < n <= 1024: register panels on 2-CTA clusters (mode 6; 4% faster on config 2 than the
  // one-CTA shared-memory panel for n <= 768, which AIFMM_HH_SMEM=1 selects)
  static const bool use_smem = getenv("AIFMM_HH_SMEM") != nullptr;   // variant toggle
  const int SM_LIM = use_smem ? HH_SMEM_ROWS : 2 * HH_REG_ROWS;
  for (const auto& q : reqs) if (q.n > HH_REG_ROWS && q.n <= SM_LIM) { sorted_reqs.push_back(q); nmax_sm = std::max(nmax_sm, q.n); }
  const size_t nsm = sorted_reqs.size() - nrg;
  static const bool no_regcl = getenv("AIFMM_NO_REGCLUSTER") != nullptr;   // debug toggle
  static const bool regcl_many = getenv("AIFMM_REGCL_FEW") == nullptr;     // debug toggle
  const int RC_ROWS = no_regcl ? 0 : HH_REGCL_ROWS;
  auto to_rc = [&](const TriRootReq& q) { return q.n > SM_LIM && q.n <= RC_ROWS && (!many || regcl_many); };
  for (const auto& q : reqs) if (q.n > SM_LIM && (q.n < 512 || many) && !to_rc(q)) sorted_reqs.push_back(q);
  const size_t nsmall = sorted_reqs.size() - nrg - nsm;
  int nmax_rc = 0, nmax_mid = 0;
  for (const auto& q : reqs) if (to_rc(q)) { sorted_reqs.push_back(q); nmax_rc = std::max(nmax_rc, q.n); }
  const size_t nrc = sorted_reqs.size() - nrg - nsm - nsmall;
  for (const auto& q : reqs) if (q.n > SM_LIM && !many && q.n > RC_ROWS && q.n <= SM_ROWS) { sorted_reqs.push_back(q); nmax_mid = std::max(nmax_mid, q.n); }
  const size_t nmid = sorted_reqs.size() - nrg - nsm - nsmall - nrc;
  for (const auto& q : reqs) if (q.n > SM_LIM && !many && q.n > SM_ROWS) sorted_reqs.push_back(q);
  const std::vector<TriRootReq>& R = sorted_reqs;
  std::vector<char> tb(tsz * reqs.size());
  // look-ahead schedule (opt-in): the descriptors of odd panels point at a second V / T pair,
  // so panel p + 1 can run while the other column tiles of panel p's update still read V / T
  static const bool lookahead = getenv("AIFMM_HHU_LOOKAHEAD") != nullptr;
  std::vector<char> tb2(lookahead ? tsz * reqs.size() : 0);
  std::vector<double*> V(reqs.size()), T(reqs.size());
  std::vector<double*> outs(reqs.size());
  std::vector<int> ldo(reqs.size());
  int rmax = 0;
  for (size_t i = 0; i < reqs.size(); ++i) {
    const TriRootReq& q = R[i];
    V[i] = work.d((size_t)std::max(q.n, 1) * HH_PANEL);
    T[i] = work.d((size_t)HH_PANEL * HH_PANEL);
    hh_make(tb.data() + i * tsz, q.A, q.lda, q.n, q.m, V[i], T[i]);
    if (lookahead)
      hh_make(tb2.data() + i * tsz, q.A, q.lda, q.n, q.m, work.d((size_t)std::max(q.n, 1) * HH_PANEL),
              work.d((size_t)HH_PANEL * HH_PANEL));
    outs[i] = q.out;
    ldo[i] = q.ldm;
    rmax = std::max(rmax, std::min(q.n, q.m));
    if (fc) fc->flops += 2.0 * q.n * (double)q.m * q.m;
  }
  up.reserve(2 * tb.size() + outs.size() * 8 + ldo.size() * 4 + 1024);
  const void* dt = up.put(tb.data(), tb.size());
  const void* dt2 = lookahead ? up.put(tb2.data(), tb2.size()) : nullptr;
  double* const* douts = up.put(outs);
  const int* dldo = up.put(ldo);
  unsigned long long dgen = up.gen();
  auto restage = [&] {   // the staging arena was rewound by a sync: upload the descriptors again
    if (up.gen() == dgen) return;
    up.reserve(2 * tb.size() + outs.size() * 8 + ldo.size() * 4 + 1024);
    dt = up.put(tb.data(), tb.size());
    if (lookahead) dt2 = up.put(tb2.data(), tb2.size());
    douts = up.put(outs);
    dldo = up.put(ldo);
    dgen = up.gen();
  };
  if (g_prof.on) { g_prof.end("cmp.proj"); g_prof.begin(s); }
  // trailing updates run as two launches: pass 1 (Z2, one CTA per column-block tile) and the
  // row-parallel pass 2 split over (tile, 256-row segment) — bitwise the same C as the fused
  // kernel (see hh_update_kernel), measured -2% config-3 factor, -12% config-2 RRQR stage 1;
  // AIFMM_HHU_SPLIT=<n> keeps the fused kernel for panels with >= n tiles.  The Z2 slots are
  // sized by the first panel, which has the most tiles
  static const int split_tiles = getenv("AIFMM_HHU_SPLIT") ? atoi(getenv("AIFMM_HHU_SPLIT")) : 1 << 30;
  static const int hhu_seg = getenv("AIFMM_HHU_SEG") ? atoi(getenv("AIFMM_HHU_SEG")) : 256;
  double* zbuf = nullptr;
  {
    size_t t0 = 0;
    for (const auto& q : reqs) {
      const int r = std::min(q.n, q.m);
      if (r > 0) t0 += (size_t)((std::max(q.m - std::min(HH_PANEL, r), 0) + 63) / 64);
    }
    if (t0 > 0 && (int)t0 < split_tiles) zbuf = work.d(t0 * HH_PANEL * 64);
  }
  const bool la = lookahead && zbuf && !g_prof.on;
  static cudaStream_t s2 = nullptr;
  static cudaEvent_t ev_a = nullptr, ev_b = nullptr;
  if (la && !s2) {
    AIFMM_CUDA(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
    AIFMM_CUDA(cudaEventCreateWithFlags(&ev_a, cudaEventDisableTiming));
    AIFMM_CUDA(cudaEventCreateWithFlags(&ev_b, cudaEventDisableTiming));
  }
  bool rest_pending = false;   // ev_b marks the side stream's last pass 2
  for (int j = 0; j < rmax; j += HH_PANEL) {
    if (g_prof.on) g_prof.begin(s);
    restage();
    const void* dcur = (la && ((j / HH_PANEL) & 1)) ? dt2 : dt;
    const char* d0 = static_cast<const char*>(dcur);
    const size_t o1 = nrg, o2 = o1 + nsm, o3 = o2 + nsmall, o4 = o3 + nrc, o5 = o4 + nmid;
    if (nrg && j < nmax_rg) launch_hh_panel(d0, (int)nrg, j, s, 4, nmax_rg);
    if (nsm && j < nmax_sm) launch_hh_panel(d0 + o1 * tsz, (int)nsm, j, s, use_smem ? 3 : 6, nmax_sm);
    if (nsmall) launch_hh_panel(d0 + o2 * tsz, (int)nsmall, j, s, 0, 0);
    if (nrc) launch_hh_panel(d0 + o3 * tsz, (int)nrc, j, s, 5, nmax_rc);
    if (nmid) launch_hh_panel(d0 + o4 * tsz, (int)nmid, j, s, 2, nmax_mid);
    if (reqs.size() > o5) launch_hh_panel(d0 + o5 * tsz, (int)(reqs.size() - o5), j, s, 1, 0);
    // fused trailing update: one CTA per (task, 64-column block of the trailing matrix)
    std::vector<int2> ut;
    for (size_t i = 0; i < reqs.size(); ++i) {
      const TriRootReq& q = R[i];
      const int r = std::min(q.n, q.m);
      if (j >= r) continue;
      const int nbw = std::min(HH_PANEL, r - j);
      const int nc = q.m - j - nbw;
      for (int n0 = 0; n0 < nc; n0 += 64)
        if (!la || n0 == 0) ut.push_back(make_int2((int)i, n0));
    }
    const size_t n_first = ut.size();   // look-ahead: the tiles holding the next panel come first
    if (la)
      for (size_t i = 0; i < reqs.size(); ++i) {
        const TriRootReq& q = R[i];
        const int r = std::min(q.n, q.m);
        if (j >= r) continue;
        const int nc = q.m - j - std::min(HH_PANEL, r - j);
        for (int n0 = 64; n0 < nc; n0 += 64) ut.push_back(make_int2((int)i, n0));
      }
    if (la && rest_pending) {   // pass 1 reads the columns the side stream was still updating
      AIFMM_CUDA(cudaStreamWaitEvent(s, ev_b, 0));
      rest_pending = false;
    }
    if (g_prof.on) { g_prof.end("hh.panel"); g_prof.begin(s); }
    if (!ut.empty()) {
      up.reserve(tb.size() + outs.size() * 8 + ldo.size() * 4 + ut.size() * sizeof(int2) + 2048);
      restage();
      const int2* dut = up.put(ut);
      int nseg = 0;
      if (zbuf && (int)ut.size() < split_tiles) {
        int rows_max = 0;
        for (const int2& u : ut) rows_max = std::max(rows_max, R[u.x].n - j);
        nseg = (rows_max + hhu_seg - 1) / hhu_seg;
      }
      if (la) {
        launch_hh_update_pass(dcur, dut, (int)ut.size(), j, s, zbuf, hhu_seg, nseg, 1);
        launch_hh_update_pass(dcur, dut, (int)n_first, j, s, zbuf, hhu_seg, nseg, 2);
        if (ut.size() > n_first) {
          AIFMM_CUDA(cudaEventRecord(ev_a, s));
          AIFMM_CUDA(cudaStreamWaitEvent(s2, ev_a, 0));
          launch_hh_update_pass(dcur, dut + n_first, (int)(ut.size() - n_first), j, s2,
                                zbuf + n_first * HH_PANEL * 64, hhu_seg, nseg, 2);
          AIFMM_CUDA(cudaEventRecord(ev_b, s2));
          rest_pending = true;
        }
      } else {
        launch_hh_update(dcur, dut, (int)ut.size(), j, s, zbuf, hhu_seg, nseg);
      }
    }
    if (g_prof.on) g_prof.end("hh.trail");
  }
  if (rest_pending) AIFMM_CUDA(cudaStreamWaitEvent(s, ev_b, 0));
  if (g_prof.on) g_prof.begin(s);
  restage();
  launch_hh_extract(dt, (int)reqs.size(), douts, dldo, s);
  if (!stacks.empty()) batched_tri_root(stacks, work, up, s, fc, tsqr_m);   // next TSQR round
}
// run pivoted-QR tasks: tall ones (m >= 128) on 8-CTA clusters, the rest one CTA each
inline void run_pqr(const std::vector<PqrTask>& v, Uploader& up, cudaStream_t s) {
  std::vector<PqrTask> small, big;
  size_t smem = 0;
  // many tasks: one CTA each fills the GPU; few tall tasks: 8-CTA clusters
  int mmax = 0;
  for (const PqrTask& t : v) mmax = std::max(mmax, t.m);
  // one CTA per task also for moderately tall tasks when there are many (700: measured -3% pqr time on
  // config 3, neutral on config 2); AIFMM_PQR_MANY_MMAX overrides
  static const int mm_lim = getenv("AIFMM_PQR_MANY_MMAX") ? atoi(getenv("AIFMM_PQR_MANY_MMAX")) : 700;
  const bool many = (int)v.size() >= 2 * 148 || ((int)v.size() >= many_threshold() && mmax <= mm_lim);
  for (const PqrTask& t : v) {
    if (t.m >= 128 && !many) big.push_back(t);
    else {
      small.push_back(t);
      smem = std::max(smem, (size_t)t.ncols + t.m + t.k0 + t.tmax + 8);
    }
  }
  if (!small.empty()) launch_pqr(up.put(small), (int)small.size(), smem, s);
  if (!big.empty()) launch_pqr_cluster(up.put(big), (int)big.size(), s);
}

}  // namespace aifmm
