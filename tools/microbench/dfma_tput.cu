// Scalar FP64 FMA throughput per SM (no memory traffic): 8 independent chains
// per thread, 16 warps per SM.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
__global__ void tput(double* out, long long* cyc, int n) {
  double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = 0.999, c = 1e-3;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
    a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  double* o;
  long long* c;
  cudaMalloc(&o, 148 * 1024 * 8);
  cudaMallocManaged(&c, 148 * 8);
  const int n = 4096;
  for (int threads : {128, 512, 1024}) {
    tput<<<148, threads>>>(o, c, n);
    cudaDeviceSynchronize();
    tput<<<148, threads>>>(o, c, n);
    cudaDeviceSynchronize();
    double mx = 0;
    for (int i = 0; i < 148; ++i) mx = c[i] > mx ? c[i] : mx;
    printf("%4d threads/SM: %.2f DFMA lanes/clk/SM\n", threads, (double)threads * 8 * n / mx);
  }
  return 0;
}
