// k_util.cu -- K1 seeded Gaussian probes and small elementwise kernels.
#include <algorithm>

#include "kernels.cuh"

namespace bfly {

namespace {

// gaussian_matrix (linalg.hpp:16-25): column-major entry t of a block takes
// Box-Muller pair t (complex) or half of pair t/2 (real: cos, then spare sin).
template <typename R>
__global__ void gauss_kernel(cx<R>* base, const GaussEnt* __restrict__ ents, int is_real) {
  const GaussEnt e = ents[blockIdx.y];
  const int64_t total = e.rows * e.cols;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = t % e.rows, c = t / e.rows;
    double re, im;
    if (!is_real) {
      gauss_pair(e.s0, (uint64_t)t, re, im);
    } else {
      double cs, sn;
      gauss_pair(e.s0, (uint64_t)(t >> 1), cs, sn);
      re = (t & 1) ? sn : cs;
      im = 0.0;
    }
    base[e.dst + i + c * e.ld] = mkc<R>((R)re, (R)im);
  }
}

template <typename R>
__global__ void conj_kernel(cx<R>* p, int64_t rows, int64_t cols, int64_t ld) {
  int64_t total = rows * cols;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = t % rows, c = t / rows;
    p[i + c * ld].y = -p[i + c * ld].y;
  }
}

template <typename R>
__global__ void permute_kernel(cx<R>* dst, int64_t ldd, const cx<R>* src, int64_t lds, int64_t rows, int64_t cols,
                               const int64_t* idx, int scatter) {
  int64_t total = rows * cols;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = t % rows, c = t / rows;
    if (scatter) dst[idx[i] + c * ldd] = src[i + c * lds];
    else dst[i + c * ldd] = src[idx[i] + c * lds];
  }
}

template <typename R>
__global__ void copy2d_kernel(cx<R>* dst, int64_t ldd, const cx<R>* src, int64_t lds, int64_t rows, int64_t cols) {
  int64_t total = rows * cols;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = t % rows, c = t / rows;
    dst[i + c * ldd] = src[i + c * lds];
  }
}

template <typename R>
__global__ void diff_norms_kernel(const cx<R>* a, const cx<R>* b, int64_t n, double* out) {
  double s0 = 0, s1 = 0;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    double dx = (double)a[t].x - (double)b[t].x, dy = (double)a[t].y - (double)b[t].y;
    s0 += dx * dx + dy * dy;
    s1 += (double)a[t].x * a[t].x + (double)a[t].y * a[t].y;
  }
  __shared__ double r0[256], r1[256];
  r0[threadIdx.x] = s0;
  r1[threadIdx.x] = s1;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      r0[threadIdx.x] += r0[threadIdx.x + o];
      r1[threadIdx.x] += r1[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    atomicAdd(out, r0[0]);
    atomicAdd(out + 1, r1[0]);
  }
}

template <typename R>
__global__ void copy_blocks_kernel(cx<R>* dst, const int64_t* idx_dst, const cx<R>* src, const int64_t* idx_src,
                                   int64_t nblocks, int64_t stride) {
  const int64_t total = nblocks * stride;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = t / stride, e = t % stride;
    const int64_t bd = idx_dst ? idx_dst[b] : b, bs = idx_src ? idx_src[b] : b;
    dst[bd * stride + e] = src[bs * stride + e];
  }
}

__global__ void copy_idx_i32_kernel(int32_t* dst, const int64_t* idx_dst, const int32_t* src, const int64_t* idx_src,
                                    int64_t n) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    dst[idx_dst ? idx_dst[t] : t] = src[idx_src ? idx_src[t] : t];
}

__global__ void d2f_kernel(const double2* s, float2* d, int64_t n) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    d[t] = make_float2((float)s[t].x, (float)s[t].y);
}
__global__ void f2d_kernel(const float2* s, double2* d, int64_t n) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    d[t] = make_double2(s[t].x, s[t].y);
}

inline unsigned grid_for(Ctx* c, int64_t total) {
  int64_t g = ceil_div(total, 256);
  int64_t cap = (int64_t)c->sm_count * 16;
  if (g > cap) g = cap;
  return (unsigned)(g < 1 ? 1 : g);
}

}  // namespace

template <typename R>
void launch_gauss(Ctx* c, cx<R>* base, const GaussEnt* ents, int nent, int64_t max_elems, bool is_real) {
  if (nent <= 0 || max_elems <= 0) return;
  int64_t gx = ceil_div(max_elems, 256);
  int64_t cap = std::max<int64_t>(1, (int64_t)c->sm_count * 16 / nent);
  if (gx > cap) gx = cap;
  KTimer timer(c, "gauss", 0.0, (double)sizeof(cx<R>) * (double)max_elems * nent);
  for (int off = 0; off < nent; off += 65535) {
    int n = std::min(65535, nent - off);
    gauss_kernel<R><<<dim3((unsigned)gx, n), 256, 0, c->stream>>>(base, ents + off, is_real ? 1 : 0);
    BFLY_LAUNCH_CHECK("gauss");
  }
}

template <typename R>
void launch_conj(Ctx* c, cx<R>* p, int64_t rows, int64_t cols, int64_t ld) {
  if (rows * cols <= 0) return;
  conj_kernel<R><<<grid_for(c, rows * cols), 256, 0, c->stream>>>(p, rows, cols, ld);
  BFLY_LAUNCH_CHECK("conj");
}

template <typename R>
void launch_permute_rows(Ctx* c, cx<R>* dst, int64_t ldd, const cx<R>* src, int64_t lds, int64_t rows, int64_t cols,
                         const int64_t* idx, bool scatter) {
  if (rows * cols <= 0) return;
  permute_kernel<R><<<grid_for(c, rows * cols), 256, 0, c->stream>>>(dst, ldd, src, lds, rows, cols, idx, scatter ? 1 : 0);
  BFLY_LAUNCH_CHECK("permute_rows");
}

template <typename R>
void launch_copy2d(Ctx* c, cx<R>* dst, int64_t ldd, const cx<R>* src, int64_t lds, int64_t rows, int64_t cols) {
  if (rows * cols <= 0) return;
  copy2d_kernel<R><<<grid_for(c, rows * cols), 256, 0, c->stream>>>(dst, ldd, src, lds, rows, cols);
  BFLY_LAUNCH_CHECK("copy2d");
}

template <typename R>
void launch_diff_norms(Ctx* c, const cx<R>* a, const cx<R>* b, int64_t n, double* out) {
  if (n <= 0) return;
  diff_norms_kernel<R><<<grid_for(c, n), 256, 0, c->stream>>>(a, b, n, out);
  BFLY_LAUNCH_CHECK("diff_norms");
}

template <typename R>
void launch_copy_blocks(Ctx* c, cx<R>* dst, const int64_t* idx_dst, const cx<R>* src, const int64_t* idx_src,
                        int64_t nblocks, int64_t stride) {
  if (nblocks * stride <= 0) return;
  copy_blocks_kernel<R><<<grid_for(c, nblocks * stride), 256, 0, c->stream>>>(dst, idx_dst, src, idx_src, nblocks,
                                                                               stride);
  BFLY_LAUNCH_CHECK("copy_blocks");
}

void launch_copy_idx_i32(Ctx* c, int32_t* dst, const int64_t* idx_dst, const int32_t* src, const int64_t* idx_src,
                         int64_t n) {
  if (n <= 0) return;
  copy_idx_i32_kernel<<<grid_for(c, n), 256, 0, c->stream>>>(dst, idx_dst, src, idx_src, n);
  BFLY_LAUNCH_CHECK("copy_idx_i32");
}

void launch_d2f(Ctx* c, const double2* s, float2* d, int64_t n) {
  if (n <= 0) return;
  d2f_kernel<<<grid_for(c, n), 256, 0, c->stream>>>(s, d, n);
  BFLY_LAUNCH_CHECK("d2f");
}
void launch_f2d(Ctx* c, const float2* s, double2* d, int64_t n) {
  if (n <= 0) return;
  f2d_kernel<<<grid_for(c, n), 256, 0, c->stream>>>(s, d, n);
  BFLY_LAUNCH_CHECK("f2d");
}

#define INST(R)                                                                                           \
  template void launch_gauss<R>(Ctx*, cx<R>*, const GaussEnt*, int, int64_t, bool);                       \
  template void launch_conj<R>(Ctx*, cx<R>*, int64_t, int64_t, int64_t);                                  \
  template void launch_permute_rows<R>(Ctx*, cx<R>*, int64_t, const cx<R>*, int64_t, int64_t, int64_t,    \
                                       const int64_t*, bool);                                              \
  template void launch_copy2d<R>(Ctx*, cx<R>*, int64_t, const cx<R>*, int64_t, int64_t, int64_t);         \
  template void launch_diff_norms<R>(Ctx*, const cx<R>*, const cx<R>*, int64_t, double*);                 \
  template void launch_copy_blocks<R>(Ctx*, cx<R>*, const int64_t*, const cx<R>*, const int64_t*, int64_t, int64_t);
INST(double)
INST(float)
#undef INST

}  // namespace bfly
