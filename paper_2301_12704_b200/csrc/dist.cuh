// dist.cuh — SURVEY §8(e): the subtree split of the factorisation across ranks (one process
// per GPU), DESIGN.md §8.
//
// Model: owner computes, replicated state.  Every rank builds the same tree, lists and colours
// and holds every block of the factorisation.  The points (tree order) are cut into `world`
// contiguous ranges of equal size and a box belongs to the rank holding its median point
// (contiguous Morton ranges of subtrees at the fine levels, one owner per box at the coarse
// ones).  Within each colour phase of a split level the expensive batched work is split by
// ownership:
//   * NNCA pivot search (ACA) and skeleton solve of a box b     -> owner(b)   (build)
//   * compression (RRQR stages 1 and 2) of a box b              -> owner(b)
//   * pivot inverse G_i = P_i^-1 and multipliers W_i             -> owner(i)   (R31 boxes: all)
//   * Schur update of a target block (p, q)                      -> owner(p)
// and each phase ends with an exchange that hands every rank the blocks the others wrote (the
// skeletons and operators, the new basis columns and their ranks, G_i and W_i, the updated Schur
// targets).  Every block has exactly one writer per phase and every reader runs after the
// exchange, so all ranks hold bit-identical state after every phase; the cheap phases (level
// set-up, orthonormalisation, redirection, new blocks, top level, solve) and the levels
// <= level_p (default: none) run redundantly on every rank.
//
// Two transports: NCCL (production: grouped in-place ncclBroadcast from each owner over
// NVLink/NVSwitch, ncclAllReduce for the integer ranks), and an in-process transport for
// validation on one GPU: `world` copies of the library loaded in one process (one host thread
// each, one stream each) exchange through a shared host rendezvous block and device-to-device
// copies.  No kernel ever waits on another rank's kernel: ranks meet on the host only.
#pragma once
#include <dlfcn.h>
#include <nccl.h>

#include <atomic>
#include <cstring>
#include <thread>
#include <vector>

namespace aifmm {

struct Region {   // a column-major double block (local pointer; same shape on every rank)
  double* p;
  int ld, rows, cols;
};

// shared host block of the in-process transport (allocated zeroed by the caller, >= 4 KB)
struct LocalShared {
  std::atomic<int> arrived;
  std::atomic<int> sense;
  int pad[14];
  void* ptr[16];
};

class Comm {
 public:
  int rank = 0, world = 1, lp = -1;
  int kind = 0;   // 0 off, 1 NCCL, 2 in-process
  // force1 (AIFMM_DIST_FORCE=1, test hook): a world of one still runs the distributed code path
  // (ownership, filtered batches, NCCL calls on a one-rank communicator)
  bool force1 = false;
  bool on() const { return kind != 0 && (world > 1 || force1); }

  ~Comm() { finalize(); }

  void init_nccl(int r, int w, const void* uid, cudaStream_t s) {
    finalize();
    load_nccl();
    ncclUniqueId id;
    std::memcpy(&id, uid, sizeof(id));
    AIFMM_CUDA(cudaStreamSynchronize(s));
    nccl_check(p_init(&comm_, w, id, r), "ncclCommInitRank");
    force1 = getenv("AIFMM_DIST_FORCE") != nullptr;
    rank = r;
    world = w;
    kind = 1;
  }
  void init_local(int r, int w, void* shared) {
    finalize();
    AIFMM_REQUIRE(w >= 1 && w <= 16 && r >= 0 && r < w && shared, AIFMM_EINVALID_ARG, "bad in-process rank/world");
    sh_ = static_cast<LocalShared*>(shared);
    rank = r;
    world = w;
    kind = 2;
    force1 = getenv("AIFMM_DIST_FORCE") != nullptr;
    my_sense_ = sh_->sense.load();   // every rank joins while no barrier is in flight
  }
  void finalize() {
    if (kind == 1 && comm_) p_destroy(comm_);
    comm_ = nullptr;
    if (buf_) cudaFree(buf_);
    if (ibuf_) cudaFree(ibuf_);
    buf_ = nullptr;
    ibuf_ = nullptr;
    cap_ = icap_ = 0;
    kind = 0;
    world = 1;
    rank = 0;
    force1 = false;
  }
  static void unique_id(void* out) {
    load_nccl();
    ncclUniqueId id;
    nccl_check(p_getid(&id), "ncclGetUniqueId");
    std::memcpy(out, &id, sizeof(id));
  }

  // host int array: element-wise sum over ranks (the owners' values; others contribute 0)
  void allreduce_int(int* v, int n, cudaStream_t s) {
    if (!on() || n <= 0) return;
    if (kind == 1) {
      ensure_ibuf((size_t)n);
      AIFMM_CUDA(cudaMemcpyAsync(ibuf_, v, sizeof(int) * n, cudaMemcpyHostToDevice, s));
      nccl_check(p_allreduce(ibuf_, ibuf_, (size_t)n, ncclInt32, ncclSum, comm_, s), "ncclAllReduce");
      AIFMM_CUDA(cudaMemcpyAsync(v, ibuf_, sizeof(int) * n, cudaMemcpyDeviceToHost, s));
      AIFMM_CUDA(cudaStreamSynchronize(s));
    } else {
      std::vector<int> mine(v, v + n);
      sh_->ptr[rank] = mine.data();
      barrier();
      for (int i = 0; i < n; ++i) {
        int acc = 0;
        for (int r = 0; r < world; ++r) acc += static_cast<const int*>(sh_->ptr[r])[i];
        v[i] = acc;
      }
      barrier();
    }
  }

  // by_owner[r]: the regions rank r wrote (identical shapes and order on every rank, local
  // pointers).  Afterwards every rank holds rank r's values in by_owner[r] for every r.
  template <class Up>
  void exchange(const std::vector<std::vector<Region>>& by_owner, Up& up, cudaStream_t s) {
    if (!on()) return;
    std::vector<size_t> off(world + 1, 0);
    for (int r = 0; r < world; ++r) {
      size_t n = 0;
      for (const Region& g : by_owner[r]) n += (size_t)g.rows * g.cols;
      off[r + 1] = off[r] + n;
    }
    if (off[world] == 0) return;
    ensure_buf(off[world]);
    // pack my regions into my segment
    CopyBatch pk;
    size_t o = off[rank];
    for (const Region& g : by_owner[rank]) {
      pk.copy(g.p, g.ld, buf_ + o, std::max(g.rows, 1), g.rows, g.cols);
      o += (size_t)g.rows * g.cols;
    }
    pk.run(up, s);
    if (kind == 1) {
      nccl_check(p_gstart(), "ncclGroupStart");
      for (int r = 0; r < world; ++r)
        if (off[r + 1] > off[r])
          nccl_check(p_bcast(buf_ + off[r], buf_ + off[r], off[r + 1] - off[r], ncclFloat64, r, comm_, s), "ncclBroadcast");
      nccl_check(p_gend(), "ncclGroupEnd");
    } else {
      up.flush();
      AIFMM_CUDA(cudaStreamSynchronize(s));
      sh_->ptr[rank] = buf_;
      barrier();
      for (int r = 0; r < world; ++r)
        if (r != rank && off[r + 1] > off[r])
          AIFMM_CUDA(cudaMemcpyAsync(buf_ + off[r], static_cast<double*>(sh_->ptr[r]) + off[r],
                                     sizeof(double) * (off[r + 1] - off[r]), cudaMemcpyDeviceToDevice, s));
      AIFMM_CUDA(cudaStreamSynchronize(s));
      barrier();
    }
    bytes_in += 8.0 * (double)(off[world] - (off[rank + 1] - off[rank]));
    ++exchanges;
    // unpack the others' segments
    CopyBatch uk;
    for (int r = 0; r < world; ++r) {
      if (r == rank) continue;
      size_t q = off[r];
      for (const Region& g : by_owner[r]) {
        uk.copy(buf_ + q, std::max(g.rows, 1), g.p, g.ld, g.rows, g.cols);
        q += (size_t)g.rows * g.cols;
      }
    }
    uk.run(up, s);
    static const bool dsync = getenv("AIFMM_DIST_SYNC") != nullptr;   // debug toggle
    if (dsync) AIFMM_CUDA(cudaStreamSynchronize(s));
  }
  double bytes_in = 0.0;
  long long exchanges = 0;

 private:
  void barrier() {   // sense-reversing barrier over the shared block (in-process transport)
    my_sense_ ^= 1;
    if (sh_->arrived.fetch_add(1) + 1 == world) {
      sh_->arrived.store(0);
      sh_->sense.store(my_sense_);
    } else {
      while (sh_->sense.load() != my_sense_) std::this_thread::yield();
    }
  }
  void ensure_buf(size_t n) {
    if (n <= cap_) return;
    if (buf_) { cudaDeviceSynchronize(); cudaFree(buf_); }
    cap_ = std::max(n, cap_ * 2);
    AIFMM_CUDA(cudaMalloc(&buf_, sizeof(double) * cap_));
  }
  void ensure_ibuf(size_t n) {
    if (n <= icap_) return;
    if (ibuf_) { cudaDeviceSynchronize(); cudaFree(ibuf_); }
    icap_ = std::max(n, icap_ * 2);
    AIFMM_CUDA(cudaMalloc(&ibuf_, sizeof(int) * icap_));
  }
  static void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
      throw Error(AIFMM_ENCCL, std::string(what) + ": " + std::string(p_err ? p_err(r) : "NCCL error"));
  }
  static void load_nccl() {
    if (p_init) return;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);   // torch's NCCL if already loaded
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) throw Error(AIFMM_ENCCL, "libnccl.so.2 not found");
    p_getid = reinterpret_cast<decltype(p_getid)>(dlsym(h, "ncclGetUniqueId"));
    p_destroy = reinterpret_cast<decltype(p_destroy)>(dlsym(h, "ncclCommDestroy"));
    p_bcast = reinterpret_cast<decltype(p_bcast)>(dlsym(h, "ncclBroadcast"));
    p_allreduce = reinterpret_cast<decltype(p_allreduce)>(dlsym(h, "ncclAllReduce"));
    p_gstart = reinterpret_cast<decltype(p_gstart)>(dlsym(h, "ncclGroupStart"));
    p_gend = reinterpret_cast<decltype(p_gend)>(dlsym(h, "ncclGroupEnd"));
    p_err = reinterpret_cast<decltype(p_err)>(dlsym(h, "ncclGetErrorString"));
    auto init = reinterpret_cast<decltype(p_init)>(dlsym(h, "ncclCommInitRank"));
    if (!p_getid || !p_destroy || !p_bcast || !p_allreduce || !p_gstart || !p_gend || !init)
      throw Error(AIFMM_ENCCL, "libnccl.so.2 lacks a required symbol");
    p_init = init;
  }
  static inline ncclResult_t (*p_init)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  static inline ncclResult_t (*p_getid)(ncclUniqueId*) = nullptr;
  static inline ncclResult_t (*p_destroy)(ncclComm_t) = nullptr;
  static inline ncclResult_t (*p_bcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  static inline ncclResult_t (*p_allreduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                            cudaStream_t) = nullptr;
  static inline ncclResult_t (*p_gstart)() = nullptr;
  static inline ncclResult_t (*p_gend)() = nullptr;
  static inline const char* (*p_err)(ncclResult_t) = nullptr;

  ncclComm_t comm_ = nullptr;
  LocalShared* sh_ = nullptr;
  int my_sense_ = 0;
  double* buf_ = nullptr;
  int* ibuf_ = nullptr;
  size_t cap_ = 0, icap_ = 0;
};

}  // namespace aifmm
