// context.cu -- per-GPU context implementation.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "context.h"
#include "comm.h"

namespace bfly {

static thread_local Ctx* g_current = nullptr;
Ctx* current_ctx() { return g_current; }
void set_current_ctx(Ctx* c) { g_current = c; }

void note_launch(const char*) {
  if (g_current) ++g_current->launches;
}

Ctx::Ctx(int dev) : device(dev) {
  BFLY_CUDA(cudaSetDevice(dev));
  BFLY_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
  // the library's own stream-ordered pool (isolated from other users of the
  // device's default pool); freed blocks stay cached: level buffers are
  // re-allocated every phase and must not go back to the driver each time.
  cudaMemPoolProps props = {};
  props.allocType = cudaMemAllocationTypePinned;
  props.handleTypes = cudaMemHandleTypeNone;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = dev;
  BFLY_CUDA(cudaMemPoolCreate(&pool, &props));
  uint64_t threshold = UINT64_MAX;
  BFLY_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold));
  cudaDeviceProp p;
  BFLY_CUDA(cudaGetDeviceProperties(&p, dev));
  sm_count = p.multiProcessorCount;
  // explicit up-front reservation (otherwise sized from the previous
  // factorization's peak, see reserve_pool)
  if (const char* e = std::getenv("BFLY_POOL_RESERVE_GB")) reserve_pool((size_t)(std::atof(e) * (double)(1ull << 30)));
}

Ctx::~Ctx() {
  if (stream) {
    cudaStreamSynchronize(stream);
    cudaStreamDestroy(stream);
  }
  for (auto& u : stage_uses) cudaEventDestroy(u.done);
  if (stage_p) cudaFreeHost(stage_p);
  if (oz_flag) cudaFree(oz_flag);
  if (pool) cudaMemPoolDestroy(pool);
}

void* Ctx::alloc(size_t bytes) {
  void* p = nullptr;
  cudaError_t e = cudaMallocFromPoolAsync(&p, bytes, pool, stream);
  if (e != cudaSuccess)
    fail(CUDA_ERR, "device allocation of " + std::to_string(bytes) + " bytes failed: " + cudaGetErrorString(e));
  return p;
}

void Ctx::release(void* p) { cudaFreeAsync(p, stream); }

void Ctx::sync() { BFLY_CUDA(cudaStreamSynchronize(stream)); }

void Ctx::upload(void* dst, const void* src, size_t bytes) {
  constexpr size_t kRing = 64ull << 20;
  if (bytes == 0) return;
  if (bytes > kRing / 2) {
    BFLY_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, stream));
    return;
  }
  if (!stage_p) {
    BFLY_CUDA(cudaMallocHost(reinterpret_cast<void**>(&stage_p), kRing));
    stage_n = kRing;
  }
  size_t b = (stage_off + 255) / 256 * 256;
  if (b + bytes > stage_n) b = 0;  // wrap
  const size_t e = b + bytes;
  // wait for earlier copies that read [b, e) and retire them
  for (size_t i = 0; i < stage_uses.size();) {
    StageUse& u = stage_uses[i];
    if (u.begin < e && b < u.end) {
      BFLY_CUDA(cudaEventSynchronize(u.done));
      cudaEventDestroy(u.done);
      stage_uses[i] = stage_uses.back();
      stage_uses.pop_back();
    } else {
      ++i;
    }
  }
  std::memcpy(stage_p + b, src, bytes);
  BFLY_CUDA(cudaMemcpyAsync(dst, stage_p + b, bytes, cudaMemcpyHostToDevice, stream));
  cudaEvent_t ev;
  BFLY_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  BFLY_CUDA(cudaEventRecord(ev, stream));
  stage_uses.push_back(StageUse{b, e, ev});
  stage_off = e;
  // retire finished uses now and then (bounded bookkeeping)
  if (stage_uses.size() > 256)
    for (size_t i = 0; i < stage_uses.size();) {
      if (cudaEventQuery(stage_uses[i].done) == cudaSuccess) {
        cudaEventDestroy(stage_uses[i].done);
        stage_uses[i] = stage_uses.back();
        stage_uses.pop_back();
      } else {
        ++i;
      }
    }
}

void Ctx::resolve_records() {
  if (records.empty()) return;
  BFLY_CUDA(cudaStreamSynchronize(stream));
  for (auto& r : records) {
    float ms = 0;
    cudaEventElapsedTime(&ms, r.start, r.stop);
    cudaEventDestroy(r.start);
    cudaEventDestroy(r.stop);
    KStat* s = nullptr;
    for (auto& kv : stats)
      if (kv.first == r.name) s = &kv.second;
    if (!s) {
      stats.emplace_back(r.name, KStat{});
      s = &stats.back().second;
    }
    s->launches += 1;
    s->ms += ms;
    s->flops += r.flops;
    s->bytes += r.bytes;
  }
  records.clear();
}

void Ctx::clear_oz_flag() {
  if (oz_flag) BFLY_CUDA(cudaMemsetAsync(oz_flag, 0, sizeof(int), stream));
}

int* Ctx::oz_flag_dev() {
  if (!oz_flag) {
    BFLY_CUDA(cudaMalloc(&oz_flag, sizeof(int)));
    BFLY_CUDA(cudaMemsetAsync(oz_flag, 0, sizeof(int), stream));
  }
  return oz_flag;
}

bool Ctx::take_oz_overflow() {
  // every rank must join the all-reduce, including a rank that launched no
  // K2 product (its flag is created here, zero)
  if (comm_active(this)) oz_flag_dev();
  if (!oz_flag) return false;
  if (comm_active(this)) comm_allreduce_max_i32(this, oz_flag, 1);
  int h = 0;
  BFLY_CUDA(cudaMemcpyAsync(&h, oz_flag, sizeof(int), cudaMemcpyDeviceToHost, stream));
  BFLY_CUDA(cudaStreamSynchronize(stream));
  if (h) BFLY_CUDA(cudaMemsetAsync(oz_flag, 0, sizeof(int), stream));
  return h != 0;
}

// One contiguous pool chunk of at least `bytes`: many separately grown
// chunks fragment, and a multi-GB level buffer that fits none of them maps
// new physical memory mid-factorization (hundreds of ms to seconds).
void Ctx::reserve_pool(size_t bytes) {
  // enough free reserved memory already (results the caller still holds
  // count as used, so a kept butterfly does not eat the next one's room)
  uint64_t used = 0, reserved = 0;
  cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
  cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved);
  if (bytes == 0 || reserved >= used + bytes) return;
  BFLY_CUDA(cudaStreamSynchronize(stream));
  budget = -1;  // re-sampled by the next memory guard
  BFLY_CUDA(cudaMemPoolTrimTo(pool, 0));  // drop free chunks; live allocations stay
  void* q = nullptr;
  if (cudaMallocFromPoolAsync(&q, bytes, pool, stream) == cudaSuccess) {
    BFLY_CUDA(cudaFreeAsync(q, stream));
    BFLY_CUDA(cudaStreamSynchronize(stream));
    pool_reserved = bytes;
    // the reservation itself must not count as a factorization's peak
    uint64_t zero = 0;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrUsedMemHigh, &zero);
  } else {
    cudaGetLastError();  // not enough memory for one chunk: keep growing on demand
  }
}

double Ctx::device_budget() {
  if (budget < 0) {
    size_t free_b = 0, total_b = 0;
    BFLY_CUDA(cudaMemGetInfo(&free_b, &total_b));
    uint64_t reserved = 0;
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved);
    budget = (double)free_b + (double)reserved;
  }
  return budget;
}

// start of a factorization: its working set is measured from here
void Ctx::mark_pool_start() {
  uint64_t used = 0, zero = 0;
  cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
  pool_used_start = (size_t)used;
  cudaMemPoolSetAttribute(pool, cudaMemPoolAttrUsedMemHigh, &zero);
}

// after a factorization: remember its working set (peak minus what was
// already in use -- earlier results the caller keeps are not part of it)
void Ctx::note_pool_peak() {
  uint64_t high = 0;
  if (cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemHigh, &high) != cudaSuccess) return;
  const size_t ws = (size_t)high > pool_used_start ? (size_t)high - pool_used_start : 0;
  pool_hint = std::max<size_t>(pool_hint, ws + ws / 16);
}

}  // namespace bfly
