// Does DMMA (mma.sync m8n8k4 f64) share issue/pipe capacity with DFMA and
// with double-precision sincos on B200?  Warps in one CTA are split between
// a DMMA loop and a DFMA (or sincos) loop; compare against each alone.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = threadIdx.x * 2e-3;
  double c[8][2] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int t = 0; t < 8; ++t)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__device__ __forceinline__ void dfma_loop(double* out, int iters) {
  double x[8];
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = fma(x[k], 0.999, 1e-3);
  }
  double s = 0;
  for (int k = 0; k < 8; ++k) s += x[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__device__ __forceinline__ void sincos_loop(double* out, int iters) {
  double acc = 0, x = (blockIdx.x * blockDim.x + threadIdx.x) * 1e-3;
  for (int i = 0; i < iters; ++i) {
    double s, c;
    sincos(x * 26214.0 + i, &s, &c);
    acc += s * c;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// mode: 0 dmma only, 1 dfma only, 2 split dmma/dfma, 3 sincos only, 4 split dmma/sincos
__global__ void mixed(double* out, int mode, int it_mma, int it_fma, int it_sc) {
  int warp = threadIdx.x / 32;
  bool first = (warp & 1) == 0;
  if (mode == 0) dmma_loop(out, it_mma);
  else if (mode == 1) dfma_loop(out, it_fma);
  else if (mode == 2) { if (first) dmma_loop(out, it_mma); else dfma_loop(out, it_fma); }
  else if (mode == 3) sincos_loop(out, it_sc);
  else { if (first) dmma_loop(out, it_mma); else sincos_loop(out, it_sc); }
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, sizeof(double) * sms * 8 * 512);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 4, threads = 256;
  const int it_mma = 1024, it_fma = 1024, it_sc = 2048;
  const char* names[] = {"dmma only", "dfma only", "dmma || dfma (split warps)", "sincos only", "dmma || sincos"};
  for (int mode = 0; mode < 5; ++mode) {
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      mixed<<<blocks, threads>>>(out, mode, it_mma, it_fma, it_sc);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    // work per warp
    double warps = blocks * threads / 32.0;
    double w_mma = (mode == 0) ? warps : (mode == 2 || mode == 4) ? warps / 2 : 0;
    double w_fma = (mode == 1) ? warps : (mode == 2) ? warps / 2 : 0;
    double w_sc = (mode == 3) ? warps : (mode == 4) ? warps / 2 : 0;
    double mma_flops = w_mma * it_mma * 64.0 * 512.0;       // 64 mma x 256 fma x 2
    double fma_flops = w_fma * 32.0 * it_fma * 128.0 * 2.0;  // 32 lanes x 128 fma x 2
    double sc = w_sc * 32.0 * it_sc;
    printf("%-28s %8.3f ms  dmma %6.2f TF  dfma %6.2f TF  sincos %7.1f Gelem/s\n", names[mode], best,
           mma_flops / best / 1e9, fma_flops / best / 1e9, sc / best / 1e6);
  }
  return cudaGetLastError() != cudaSuccess;
}
