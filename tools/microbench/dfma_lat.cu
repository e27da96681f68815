// Dependent-chain latency of DFMA / FFMA and of an LDS->DFMA pair on one warp
// (clock64 around 1024 chained ops).  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
__global__ void lat(double* out, long long* cyc, double a, double b, int n) {
  __shared__ double sm[64];
  sm[threadIdx.x] = threadIdx.x;
  __syncthreads();
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, a, b);
  long long t1 = clock64();
  float y = threadIdx.x;
  for (int i = 0; i < n; ++i) y = fmaf(y, (float)a, (float)b);
  long long t2 = clock64();
  int idx = threadIdx.x;
  double z = 0;
  for (int i = 0; i < n; ++i) {
    double v = sm[idx & 63];
    z = fma(v, a, z);
    idx = (int)z & 1;
  }
  long long t3 = clock64();
  out[threadIdx.x] = x + y + z;
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0;
    cyc[1] = t2 - t1;
    cyc[2] = t3 - t2;
  }
}
int main() {
  double* o;
  long long* c;
  cudaMalloc(&o, 64 * 8);
  cudaMallocManaged(&c, 3 * 8);
  const int n = 1024;
  lat<<<1, 32>>>(o, c, 0.999, 1e-3, n);
  cudaDeviceSynchronize();
  lat<<<1, 32>>>(o, c, 0.999, 1e-3, n);
  cudaDeviceSynchronize();
  printf("DFMA dep latency %.1f cyc, FFMA %.1f cyc, LDS->DFMA->idx loop %.1f cyc\n", (double)c[0] / n,
         (double)c[1] / n, (double)c[2] / n);
  return 0;
}
