// Latency of the apply-stage warp GEMV (16 x 32 complex128 block from shared
// memory, k = 1, two lanes per output) on 16 warps per SM, for three inner-loop
// schedules: 4-way unrolled (V=0), all loads of a chunk of CH first (V=CH).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void cfma(double2& acc, double2 a, double2 b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
}

template <int CH, bool SPLIT_HI>
__global__ void __launch_bounds__(128) gemv(double2* out, long long* cyc, int reps, int K, int M) {
  __shared__ double2 As[4][32 * 17];
  __shared__ double2 Bs[4][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = lane; i < K * (M + 1); i += 32) As[warp][i] = make_double2(i * 1e-3, 1.0 / (i + 1));
  for (int i = lane; i < K; i += 32) Bs[warp][i] = make_double2(1.0, 0.5);
  __syncwarp();
  const int Q = 2, part = SPLIT_HI ? lane / 16 : lane % Q, m = SPLIT_HI ? lane % 16 : lane / Q, ks = M + 1;
  long long t0 = clock64();
  double2 acc = make_double2(0, 0);
  for (int r = 0; r < reps; ++r) {
    double2 a[4] = {};
    const double2* as = As[warp] + m;
    const double2* bs = Bs[warp];
    if constexpr (CH == 0) {
      int kk = part;
      for (; kk + 3 * Q < K; kk += 4 * Q) {
        cfma(a[0], as[kk * ks], bs[kk]);
        cfma(a[1], as[(kk + Q) * ks], bs[kk + Q]);
        cfma(a[2], as[(kk + 2 * Q) * ks], bs[kk + 2 * Q]);
        cfma(a[3], as[(kk + 3 * Q) * ks], bs[kk + 3 * Q]);
      }
    } else {
      for (int kb = part; kb < K; kb += CH * Q) {
        double2 av[CH > 0 ? CH : 1], bv[CH > 0 ? CH : 1];
#pragma unroll
        for (int j = 0; j < CH; ++j) {
          const int kk = kb + j * Q;
          av[j] = kk < K ? as[kk * ks] : make_double2(0, 0);
          bv[j] = kk < K ? bs[kk] : make_double2(0, 0);
        }
#pragma unroll
        for (int j = 0; j < CH; ++j) cfma(a[j & 3], av[j], bv[j]);
      }
    }
    a[0].x += a[1].x + a[2].x + a[3].x;
    a[0].y += a[1].y + a[2].y + a[3].y;
    a[0].x += __shfl_xor_sync(0xffffffffu, a[0].x, SPLIT_HI ? 16 : 1);
    a[0].y += __shfl_xor_sync(0xffffffffu, a[0].y, SPLIT_HI ? 16 : 1);
    acc.x += a[0].x;
    acc.y += a[0].y;
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (lane == 0) cyc[blockIdx.x * 4 + warp] = t1 - t0;
}

template <int CH, bool SH>
void run(double2* o, long long* c, int grid) {
  for (int reps : {1, 20}) {
    gemv<CH, SH><<<grid, 128>>>(o, c, reps, 32, 16);
    cudaDeviceSynchronize();
    gemv<CH, SH><<<grid, 128>>>(o, c, reps, 32, 16);
    cudaDeviceSynchronize();
    double s = 0, mx = 0;
    for (int i = 0; i < grid * 4; ++i) {
      s += c[i];
      mx = c[i] > mx ? c[i] : mx;
    }
    printf("SH %d CH %2d grid %4d x 4 warps, reps %2d: mean %.0f cyc/rep, max %.0f\n", (int)SH, CH, grid, reps, s / (grid * 4) / reps,
           mx / reps);
  }
}
int main() {
  double2* o;
  long long* c;
  cudaMalloc(&o, 2048 * 128 * sizeof(double2));
  cudaMallocManaged(&c, 2048 * 4 * sizeof(long long));
  for (int grid : {1, 148 * 4}) {
    run<0, false>(o, c, grid);
    run<0, true>(o, c, grid);
    run<16, true>(o, c, grid);
  }
  return 0;
}
