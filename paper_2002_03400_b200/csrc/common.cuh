// common.cuh -- shared device/host utilities of the B200 butterfly library.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

namespace bfly {

// ---------------------------------------------------------------- errors
// Mirrors the reference hierarchy (core.hpp:43-60); converted to status codes
// at the C ABI.
enum Status { OK = 0, PRECONDITION = 1, DIMENSION = 2, SEQUENCING = 3, FORMAT = 4, CONDITIONING = 5, CUDA_ERR = 6, NCCL_ERR = 7 };

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }

#define BFLY_CUDA(call)                                                                        \
  do {                                                                                         \
    cudaError_t e_ = (call);                                                                   \
    if (e_ != cudaSuccess)                                                                     \
      ::bfly::fail(::bfly::CUDA_ERR, std::string(#call) + ": " + cudaGetErrorString(e_) +      \
                                         " (" + __FILE__ + ":" + std::to_string(__LINE__) + ")"); \
  } while (0)

// Every kernel launch goes through here: counts launches on the context and
// surfaces launch errors immediately.
void note_launch(const char* name);

#define BFLY_LAUNCH_CHECK(name)                                                 \
  do {                                                                          \
    cudaError_t e_ = cudaGetLastError();                                        \
    if (e_ != cudaSuccess)                                                      \
      ::bfly::fail(::bfly::CUDA_ERR, std::string("launch ") + (name) + ": " +  \
                                         cudaGetErrorString(e_));               \
    ::bfly::note_launch(name);                                                  \
  } while (0)

// ---------------------------------------------------------- complex types
template <typename R> struct cx_of;
template <> struct cx_of<double> { using type = double2; };
template <> struct cx_of<float> { using type = float2; };
template <typename R> using cx = typename cx_of<R>::type;

template <typename R> __host__ __device__ __forceinline__ cx<R> mkc(R re, R im) {
  cx<R> z;
  z.x = re;
  z.y = im;
  return z;
}
template <typename V> __host__ __device__ __forceinline__ V cconj(V a) {
  a.y = -a.y;
  return a;
}
template <typename V> __host__ __device__ __forceinline__ V cadd(V a, V b) {
  a.x += b.x;
  a.y += b.y;
  return a;
}
template <typename V> __host__ __device__ __forceinline__ V csub(V a, V b) {
  a.x -= b.x;
  a.y -= b.y;
  return a;
}
template <typename V> __host__ __device__ __forceinline__ V cmul(V a, V b) {
  V r;
  r.x = a.x * b.x - a.y * b.y;
  r.y = a.x * b.y + a.y * b.x;
  return r;
}
// acc += a * b
template <typename V> __host__ __device__ __forceinline__ void cfma(V& acc, V a, V b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
}
// acc += conj(a) * b
template <typename V> __host__ __device__ __forceinline__ void cfma_conj(V& acc, V a, V b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(-a.y, b.x, acc.y);
}
template <typename V> __host__ __device__ __forceinline__ auto cabs2(V a) { return a.x * a.x + a.y * a.y; }

// ----------------------------------------------------------------- RNG
// splitmix64 / seed_mix (core.hpp:70-88).  The stream is counter based: after
// c draws the state is s0 + c*gamma, so any entry can be produced directly.
constexpr uint64_t kGamma = 0x9e3779b97f4a7c15ULL;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

inline uint64_t seed_mix_host(uint64_t seed, std::initializer_list<uint64_t> words) {
  uint64_t h = seed;
  for (uint64_t w : words) h = mix64(h + kGamma) ^ (w + kGamma);
  return mix64(h + kGamma);
}
inline uint64_t seed_mix_host_n(uint64_t seed, int n, const uint64_t* words) {
  uint64_t h = seed;
  for (int i = 0; i < n; ++i) h = mix64(h + kGamma) ^ (words[i] + kGamma);
  return mix64(h + kGamma);
}

// Box-Muller pair t of the gaussian_matrix stream whose state starts at s0
// (= seed_mix(seed, "matr"), linalg.hpp:20): (rho cos, rho sin), core.hpp:106-118.
__device__ __forceinline__ void gauss_pair(uint64_t s0, uint64_t t, double& c, double& s) {
  uint64_t b1 = mix64(s0 + (2 * t + 1) * kGamma);
  uint64_t b2 = mix64(s0 + (2 * t + 2) * kGamma);
  double u1 = ((double)(b1 >> 11) + 1.0) * 0x1p-53;
  double u2 = ((double)(b2 >> 11) + 1.0) * 0x1p-53;
  double radius = sqrt(-2.0 * log(u1));
  double angle = 6.283185307179586476925286766559 * u2;
  double sn, cs;
  sincos(angle, &sn, &cs);
  c = radius * cs;
  s = radius * sn;
}

__host__ __device__ __forceinline__ int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace bfly
