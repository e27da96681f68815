// Latency of the apply-stage warp GEMV (16 x 32 complex128 block from shared
// memory, k = 1, two lanes per output) on one warp vs 14 warps per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2002_03400_b200/csrc
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void cfma(double2& acc, double2 a, double2 b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
}

template <int M, int K>
__global__ void gemv(double2* out, long long* cyc, int reps, int rt_k) {
  __shared__ double2 As[4][K * (M + 1)];
  __shared__ double2 Bs[4][K];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = lane; i < K * (M + 1); i += 32) As[warp][i] = make_double2(i * 1e-3, 1.0 / (i + 1));
  for (int i = lane; i < K; i += 32) Bs[warp][i] = make_double2(1.0, 0.5);
  __syncwarp();
  const int Q = 2, part = lane % Q, m = lane / Q;
  const int Kr = rt_k;  // runtime K as in the product
  long long t0 = clock64();
  double2 acc = make_double2(0, 0);
  for (int r = 0; r < reps; ++r) {
    double2 a0 = make_double2(0, 0), a1 = a0, a2 = a0, a3 = a0;
    const double2* as = As[warp] + m;
    const double2* bs = Bs[warp];
    int kk = part;
    for (; kk + 3 * Q < Kr; kk += 4 * Q) {
      cfma(a0, as[kk * (M + 1)], bs[kk]);
      cfma(a1, as[(kk + Q) * (M + 1)], bs[kk + Q]);
      cfma(a2, as[(kk + 2 * Q) * (M + 1)], bs[kk + 2 * Q]);
      cfma(a3, as[(kk + 3 * Q) * (M + 1)], bs[kk + 3 * Q]);
    }
    a0.x += a1.x + a2.x + a3.x;
    a0.y += a1.y + a2.y + a3.y;
    a0.x += __shfl_xor_sync(0xffffffffu, a0.x, 1);
    a0.y += __shfl_xor_sync(0xffffffffu, a0.y, 1);
    acc.x += a0.x;
    acc.y += a0.y;
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (lane == 0) cyc[blockIdx.x * 4 + warp] = t1 - t0;
}

int main() {
  double2* o;
  long long* c;
  cudaMalloc(&o, 2048 * 128 * sizeof(double2));
  cudaMallocManaged(&c, 2048 * 4 * sizeof(long long));
  for (int grid : {1, 148 * 4}) {
    for (int reps : {1, 100}) {
      gemv<16, 32><<<grid, 128>>>(o, c, reps, 32);
      cudaDeviceSynchronize();
      gemv<16, 32><<<grid, 128>>>(o, c, reps, 32);
      cudaDeviceSynchronize();
      double s = 0, mx = 0;
      for (int i = 0; i < grid * 4; ++i) {
        s += c[i];
        mx = c[i] > mx ? c[i] : mx;
      }
      printf("grid %4d x 4 warps, reps %3d: mean %.0f cyc/rep, max %.0f cyc/rep\n", grid, reps, s / (grid * 4) / reps,
             mx / reps);
    }
  }
  return 0;
}
