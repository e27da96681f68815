// context.h -- per-GPU context: stream, stream-ordered memory pool, launch
// accounting, optional NCCL communicator.
#pragma once
#include <cstdlib>
#include <cstdio>
#include <chrono>

#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <memory>
#include <utility>
#include <vector>

#include "../../include/bfly_b200.h"
#include "common.cuh"

struct ncclComm;

namespace bfly {

struct Ctx;
// host-staged transport (bfly_ctx_set_host_comm): the caller's collectives +
// pinned staging buffers + the point-to-point group being assembled
struct HostComm {
  bfly_host_comm fns{};
  unsigned char* buf[2] = {nullptr, nullptr};
  size_t cap[2] = {0, 0};
  struct Xfer {
    bool send;
    int peer;
    void* dev;
    size_t bytes;
  };
  std::vector<Xfer> pending;
  bool grouped = false;
  unsigned char* stage(Ctx* c, int slot, size_t bytes);
  ~HostComm();
};

// Per-kernel device timing (CUDA events on the library stream) for the
// roofline numbers; off unless requested, resolved lazily.
struct KRecord {
  const char* name;
  cudaEvent_t start, stop;
  double flops, bytes;
};
struct KStat {
  int64_t launches = 0;
  double ms = 0, flops = 0, bytes = 0;
};

struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaMemPool_t pool = nullptr;
  int64_t launches = 0;
  int sm_count = 148;
  bool profiling = false;
  std::vector<KRecord> records;
  std::vector<std::pair<std::string, KStat>> stats;
  void resolve_records();  // fold finished records into stats
  // multi-GPU (rank-sharded probes + NCCL all-gather of each level)
  int rank = 0, world = 1;
  ncclComm* comm = nullptr;
  std::unique_ptr<HostComm> host;  // host-staged transport (instead of NCCL)

  explicit Ctx(int dev);
  ~Ctx();
  void* alloc(size_t bytes);
  void release(void* p);
  void sync();
  // host -> device upload on the library stream that never blocks the host:
  // the bytes are staged in a pinned ring (a region is reused only after
  // the copy that read it has executed), so planning of the next launches
  // overlaps the running kernels; oversized uploads fall back to a pageable
  // copy.  Not for use during graph capture.
  void upload(void* dst, const void* src, size_t bytes);
  struct StageUse {
    size_t begin, end;
    cudaEvent_t done;
  };
  unsigned char* stage_p = nullptr;
  size_t stage_n = 0, stage_off = 0;
  std::vector<StageUse> stage_uses;
  // K2 int8-slice path range flag (k_matvec_oz.cu).  oz_deferred: launches OR
  // into one persistent device flag that is checked once per factorization
  // (no per-launch host sync); force_fp64: recompute on the FP64 DMMA path.
  bool oz_deferred = false, force_fp64 = false;
  int* oz_flag = nullptr;
  int* oz_flag_dev();
  bool take_oz_overflow();  // all ranks agree; resets the flag
  void clear_oz_flag();     // drop a stale flag (start of a factorization / error path)
  // pool sizing: a factorization reserves one contiguous chunk sized to the
  // previous one's peak (see reserve_pool)
  size_t pool_reserved = 0, pool_hint = 0, pool_used_start = 0;
  void reserve_pool(size_t bytes);
  // device bytes this context could hold in its pool: free device memory plus
  // the pool's reservation, sampled on first use and after the pool is
  // resized (the memory guard's denominator; cudaMemGetInfo is not called per level)
  double budget = -1;
  double device_budget();
  void mark_pool_start();
  void note_pool_peak();
};

// The context kernels are currently being launched for (set by the C ABI
// entry points; the library is used from one host thread per context).
Ctx* current_ctx();
void set_current_ctx(Ctx* c);

// RAII: brackets one kernel launch with events when profiling is on.
// host-side timeline (BFLY_HOST_TRACE=1): milliseconds since the first call
inline bool host_trace_on() {
  static const bool on = std::getenv("BFLY_HOST_TRACE") != nullptr;
  return on;
}
inline double host_ms() {
  static const auto t0 = std::chrono::steady_clock::now();
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}
#define BFLY_HOST_TRACE(...)                                     \
  do {                                                           \
    if (::bfly::host_trace_on()) {                               \
      fprintf(stderr, "[host %9.3f ms] ", ::bfly::host_ms());    \
      fprintf(stderr, __VA_ARGS__);                              \
      fputc('\n', stderr);                                       \
    }                                                            \
  } while (0)

struct KTimer {
  Ctx* c;
  KRecord rec{};
  bool on;
  KTimer(Ctx* ctx, const char* name, double flops, double bytes) : c(ctx), on(ctx && ctx->profiling) {
    if (!on) return;
    rec.name = name;
    rec.flops = flops;
    rec.bytes = bytes;
    cudaEventCreate(&rec.start);
    cudaEventCreate(&rec.stop);
    cudaEventRecord(rec.start, c->stream);
  }
  ~KTimer() {
    if (!on) return;
    cudaEventRecord(rec.stop, c->stream);
    c->records.push_back(rec);
  }
};

struct CtxScope {
  Ctx* prev;
  explicit CtxScope(Ctx* c) : prev(current_ctx()) {
    set_current_ctx(c);
    if (c) BFLY_CUDA(cudaSetDevice(c->device));
  }
  ~CtxScope() { set_current_ctx(prev); }
};

// RAII device buffer on the context's stream-ordered pool.
template <typename T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  Ctx* ctx = nullptr;

  DBuf() = default;
  DBuf(Ctx* c, size_t count) { reset(c, count); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), n(o.n), ctx(o.ctx) { o.p = nullptr; o.n = 0; }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) {
      free();
      p = o.p; n = o.n; ctx = o.ctx;
      o.p = nullptr; o.n = 0;
    }
    return *this;
  }
  ~DBuf() { free(); }

  void reset(Ctx* c, size_t count) {
    free();
    ctx = c;
    n = count;
    p = count ? static_cast<T*>(c->alloc(count * sizeof(T))) : nullptr;
  }
  void zero() {
    if (n) BFLY_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), ctx->stream));
  }
  void free() {
    if (p && ctx) ctx->release(p);
    p = nullptr;
    n = 0;
  }
  void upload(const T* host, size_t count) {
    if (count) ctx->upload(p, host, count * sizeof(T));
  }
  void upload(const std::vector<T>& v) {
    if (v.size() > n) reset(ctx, v.size());
    upload(v.data(), v.size());
  }
  void download(T* host, size_t count) const {
    if (count) BFLY_CUDA(cudaMemcpyAsync(host, p, count * sizeof(T), cudaMemcpyDeviceToHost, ctx->stream));
  }
  size_t bytes() const { return n * sizeof(T); }
};

template <typename T>
DBuf<T> to_device(Ctx* c, const std::vector<T>& v) {
  DBuf<T> d(c, v.size());
  d.upload(v.data(), v.size());
  return d;
}

}  // namespace bfly
