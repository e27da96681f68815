// context.cu -- per-GPU context implementation.
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
  BFLY_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
  // keep freed blocks cached in the pool: level buffers are re-allocated
  // every phase and must not go back to the driver each time.
  uint64_t threshold = UINT64_MAX;
  BFLY_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold));
  cudaDeviceProp p;
  BFLY_CUDA(cudaGetDeviceProperties(&p, dev));
  sm_count = p.multiProcessorCount;
}

Ctx::~Ctx() {
  if (stream) {
    cudaStreamSynchronize(stream);
    cudaStreamDestroy(stream);
  }
  if (pinned_p) cudaFreeHost(pinned_p);
  if (oz_flag) cudaFree(oz_flag);
}

void* Ctx::alloc(size_t bytes) {
  void* p = nullptr;
  cudaError_t e = cudaMallocFromPoolAsync(&p, bytes, pool, stream);
  if (e != cudaSuccess)
    fail(CUDA_ERR, "device allocation of " + std::to_string(bytes) + " bytes failed: " + cudaGetErrorString(e));
  return p;
}

void Ctx::release(void* p) { cudaFreeAsync(p, stream); }

void* Ctx::pinned(size_t bytes) {
  if (bytes > pinned_n) {
    if (pinned_p) cudaFreeHost(pinned_p);
  if (oz_flag) cudaFree(oz_flag);
    pinned_p = nullptr;
    pinned_n = 0;
    BFLY_CUDA(cudaMallocHost(&pinned_p, bytes));
    pinned_n = bytes;
  }
  return pinned_p;
}

void Ctx::sync() { BFLY_CUDA(cudaStreamSynchronize(stream)); }

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

int* Ctx::oz_flag_dev() {
  if (!oz_flag) {
    BFLY_CUDA(cudaMalloc(&oz_flag, sizeof(int)));
    BFLY_CUDA(cudaMemsetAsync(oz_flag, 0, sizeof(int), stream));
  }
  return oz_flag;
}

bool Ctx::take_oz_overflow() {
  if (!oz_flag) return false;
  if (world > 1 && comm) comm_allreduce_max_i32(this, oz_flag, 1);
  int h = 0;
  BFLY_CUDA(cudaMemcpyAsync(&h, oz_flag, sizeof(int), cudaMemcpyDeviceToHost, stream));
  BFLY_CUDA(cudaStreamSynchronize(stream));
  if (h) BFLY_CUDA(cudaMemsetAsync(oz_flag, 0, sizeof(int), stream));
  return h != 0;
}

}  // namespace bfly
