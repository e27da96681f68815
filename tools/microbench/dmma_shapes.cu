// dmma_shapes.cu -- FP64 mma.sync throughput by shape on sm_100a (m8n8k4 vs m16n8k16): both reach
// the same ~37 TF/s, so the DMMA GEMMs gain nothing from the larger shape.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 dmma_shapes.cu -o dmma_shapes
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k884(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = threadIdx.x * 2e-3, c[8][2] = {};
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int t = 0; t < 8; ++t)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
  double s = 0; for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k16816(double* out, int iters) {
  double a[8], b[4], c[4][4] = {};
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 1e-3 + j;
  for (int j = 0; j < 4; ++j) b[j] = threadIdx.x * 2e-3 + j;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int t = 0; t < 4; ++t)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[t][0]), "+d"(c[t][1]), "+d"(c[t][2]), "+d"(c[t][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  double s = 0; for (int t = 0; t < 4; ++t) s += c[t][0] + c[t][1] + c[t][2] + c[t][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  double* out; cudaMalloc(&out, 148 * 8 * 1024 * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 20000, blocks = 148 * 4, threads = 256;
  for (int rep = 0; rep < 2; ++rep) {
    float ms;
    cudaEventRecord(e0); k884<<<blocks, threads>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 8 * 8 * 4 * 8.0 * iters * blocks * (threads / 32);
    printf("m8n8k4:   %.2f TFLOP/s (%.3f ms)\n", fl / ms / 1e9, ms);
    cudaEventRecord(e0); k16816<<<blocks, threads>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    fl = 2.0 * 16 * 8 * 16 * 4.0 * iters * blocks * (threads / 32);
    printf("m16n8k16: %.2f TFLOP/s (%.3f ms)  err=%s\n", fl / ms / 1e9, ms, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
