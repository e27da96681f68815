// %globaltimer resolution: smallest nonzero increment seen by a spinning thread
#include <cstdio>
__global__ void k(unsigned long long* out) {
  unsigned long long prev, t, mn = ~0ull;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(prev));
  int changes = 0;
  for (int i = 0; i < 200000 && changes < 1000; ++i) {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t != prev) {
      if (t - prev < mn) mn = t - prev;
      prev = t;
      ++changes;
    }
  }
  out[0] = mn;
  out[1] = changes;
}
int main() {
  unsigned long long* o;
  cudaMallocManaged(&o, 16);
  k<<<1, 1>>>(o);
  cudaDeviceSynchronize();
  printf("globaltimer min increment %llu ns over %llu changes\n", o[0], o[1]);
}
