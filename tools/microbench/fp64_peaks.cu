// FP64 pipe microbenchmarks on B200 (sm_100a): DFMA vs DMMA (mma.sync m8n8k4 f64),
// plus per-element cost of the transcendentals used by the kernel-evaluated matvecs.
// Used to set the roofline denominator (MEASURED_PEAKS.json has no FP64 entry).
#include <cstdio>
#include <cuda_runtime.h>
#include <cmath>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

// FP32 FFMA peak (the complex64 recompression's pipe)
__global__ void ffma_kernel(float* out, int iters, float a, float b) {
  float x[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) x[j] = threadIdx.x + j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int j = 0; j < 16; ++j) x[j] = fmaf(x[j], a, b);
  }
  float s = 0;
#pragma unroll
  for (int j = 0; j < 16; ++j) s += x[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = threadIdx.x * 2e-3;
  double c[8][2];
  for (int t = 0; t < 8; ++t) { c[t][0] = 0; c[t][1] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
#pragma unroll
      for (int t = 0; t < 8; ++t)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
  for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void sincos_kernel(double* out, int iters, double scale) {
  double acc = 0, x = (blockIdx.x * blockDim.x + threadIdx.x) * 1e-3;
  for (int i = 0; i < iters; ++i) {
    double s, c;
    sincos(x * scale + i, &s, &c);
    acc += s * c;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void sincospi_kernel(double* out, int iters) {
  double acc = 0, x = (blockIdx.x * blockDim.x + threadIdx.x) * 1e-7;
  for (int i = 0; i < iters; ++i) {
    double s, c;
    sincospi(x + i * 1e-9, &s, &c);
    acc += s * c;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void rsqrt_kernel(double* out, int iters) {
  double acc = 0, x = 1.0 + (blockIdx.x * blockDim.x + threadIdx.x) * 1e-3;
  for (int i = 0; i < iters; ++i) { acc += rsqrt(x + i); }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int sms = p.multiProcessorCount;
  printf("device %s sms %d clock %d kHz\n", p.name, sms, p.clockRate);
  double* out; CK(cudaMalloc(&out, sizeof(double) * 148 * 64 * 1024));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  // DFMA
  for (int rep = 0; rep < 2; ++rep) {
    int blocks = sms * 4, threads = 512, iters = 4096;
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, threads>>>(out, iters, 0.999, 1e-3);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * blocks * threads * (double)iters * 16 * 8;
    printf("DFMA: %.2f TFLOP/s (%.3f ms)\n", flops / ms / 1e9, ms);
  }
  for (int rep = 0; rep < 2; ++rep) {
    int blocks = sms * 4, threads = 512, iters = 4096;
    cudaEventRecord(e0);
    ffma_kernel<<<blocks, threads>>>(reinterpret_cast<float*>(out), iters, 0.999f, 1e-3f);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * blocks * threads * (double)iters * 16 * 16;
    printf("FFMA (fp32): %.2f TFLOP/s (%.3f ms)\n", flops / ms / 1e9, ms);
  }
  for (int rep = 0; rep < 2; ++rep) {
    int blocks = sms * 4, threads = 256, iters = 2048;
    cudaEventRecord(e0);
    dmma_kernel<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 256 /*fma per mma*/ * (blocks * threads / 32) * (double)iters * 64;
    printf("DMMA m8n8k4: %.2f TFLOP/s (%.3f ms)\n", flops / ms / 1e9, ms);
  }
  {
    int blocks = sms * 8, threads = 256, iters = 4096;
    for (double sc : {1.0, 26214.0}) {
      cudaEventRecord(e0);
      sincos_kernel<<<blocks, threads>>>(out, iters, sc);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      printf("sincos(scale %.0f): %.2f Gelem/s\n", sc, blocks * threads * (double)iters / ms / 1e6);
    }
    cudaEventRecord(e0);
    sincospi_kernel<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("sincospi: %.2f Gelem/s\n", blocks * threads * (double)iters / ms / 1e6);
    cudaEventRecord(e0);
    rsqrt_kernel<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("rsqrt: %.2f Gelem/s\n", blocks * threads * (double)iters / ms / 1e6);
  }
  CK(cudaGetLastError());
  return 0;
}
