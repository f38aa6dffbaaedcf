// Elementwise / column-reduction HBM-bound kernels: bias-dropout-residual,
// column sums (bias gradients), exact-erf GeLU, the checker's loss head, and
// the in-process AllReduce used to emulate TMP ranks on one device.
#include "common.cuh"
#include "kernels.h"

namespace oases {
namespace {

constexpr int kThreads = 256;

unsigned grid_for(long long work_items, int per_block) {
  long long g = (work_items + per_block - 1) / per_block;
  const long long cap = 148LL * 16;
  if (g > cap) g = cap;
  return static_cast<unsigned>(g < 1 ? 1 : g);
}

// out = residual + dropout(x + bias[col])   (8 elements per thread-iteration)
template <typename T>
__global__ void __launch_bounds__(kThreads) bdr_fwd_kernel(const T* __restrict__ x, const T* __restrict__ bias,
                                                           const T* __restrict__ res, T* __restrict__ out, long long n,
                                                           int cols, uint32_t thr, float ks, int drop, uint64_t seed,
                                                           uint64_t offset) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x * 4;
  for (long long i = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) * 4; i < n; i += stride) {
    uint32_t u[4] = {0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu};
    if (drop) Philox::gen(seed, offset, static_cast<unsigned long long>(i) >> 2, u);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const long long e = i + q;
      if (e >= n) break;
      float v = to_f(x[e]);
      if (bias) v += to_f(bias[e % cols]);
      if (drop) v = (u[q] >= thr) ? v * ks : 0.f;
      if (res) v += to_f(res[e]);
      out[e] = from_f<T>(v);
    }
  }
}

// Column pass: dx = dropout'(dout) (optional, written if dx != null), and
// partial column sums of dx over a chunk of rows (deterministic).
template <typename T>
__global__ void __launch_bounds__(kThreads) col_pass_kernel(const T* __restrict__ in, T* __restrict__ dx,
                                                            float* __restrict__ part, long long rows, int cols,
                                                            int rows_per_chunk, uint32_t thr, float ks, int drop,
                                                            uint64_t seed, uint64_t offset) {
  const int c = blockIdx.x * kThreads + threadIdx.x;
  if (c >= cols) return;
  const long long r0 = static_cast<long long>(blockIdx.y) * rows_per_chunk;
  long long r1 = r0 + rows_per_chunk;
  if (r1 > rows) r1 = rows;
  float s = 0.f;
  for (long long r = r0; r < r1; ++r) {
    const long long e = r * cols + c;
    float v = to_f(in[e]);
    if (drop) {
      uint32_t u[4];
      Philox::gen(seed, offset, static_cast<unsigned long long>(e) >> 2, u);
      v = (u[e & 3] >= thr) ? v * ks : 0.f;
    }
    if (dx) dx[e] = from_f<T>(v);
    s += v;
  }
  if (part) part[static_cast<long long>(blockIdx.y) * cols + c] = s;
}

__global__ void col_finalize_kernel(const float* __restrict__ part, int chunks, int cols, float* __restrict__ out,
                                    int acc) {
  const int c = blockIdx.x * kThreads + threadIdx.x;
  if (c >= cols) return;
  float s = 0.f;
  for (int k = 0; k < chunks; ++k) s += part[static_cast<long long>(k) * cols + c];
  out[c] = acc ? out[c] + s : s;
}

template <typename T>
__global__ void __launch_bounds__(kThreads) gelu_fwd_kernel(const T* __restrict__ x, T* __restrict__ y, long long n) {
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    y[i] = from_f<T>(gelu_f(to_f(x[i])));
}
template <typename T>
__global__ void __launch_bounds__(kThreads) gelu_bwd_kernel(const T* __restrict__ x, const T* __restrict__ dy,
                                                            T* __restrict__ dx, long long n) {
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    dx[i] = from_f<T>(to_f(dy[i]) * gelu_grad_f(to_f(x[i])));
}

// loss partial per block (f64), dz = gelu(z) * gelu'(z)   (numerics.cpp:175-188)
template <typename T>
__global__ void __launch_bounds__(kThreads) gelu_sq_loss_kernel(const T* __restrict__ z, T* __restrict__ dz,
                                                                double* __restrict__ part, long long n) {
  double acc = 0.0;
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const float v = to_f(z[i]);
    const float g = gelu_f(v);
    acc += 0.5 * static_cast<double>(g) * static_cast<double>(g);
    if (dz) dz[i] = from_f<T>(g * gelu_grad_f(v));
  }
  acc = warp_sum(acc);
  __shared__ double sm[kThreads / 32];
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) s += sm[w];
    part[blockIdx.x] = s;
  }
}
__global__ void loss_finalize_kernel(const double* __restrict__ part, int nparts, double* __restrict__ out, int acc) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double s = 0.0;
  for (int i = 0; i < nparts; ++i) s += part[i];
  *out = acc ? *out + s : s;
}

struct BufList {
  void* p[8];
};
template <typename T>
__global__ void __launch_bounds__(kThreads) local_allreduce_kernel(BufList b, int w, long long n) {
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    float s = to_f(static_cast<const T*>(b.p[0])[i]);
    for (int k = 1; k < w; ++k) s += to_f(static_cast<const T*>(b.p[k])[i]);
    const T r = from_f<T>(s);
    for (int k = 0; k < w; ++k) static_cast<T*>(b.p[k])[i] = r;
  }
}

int chunks_for(long long rows) {
  long long c = (rows + 31) / 32;
  if (c > 512) c = 512;
  return static_cast<int>(c < 1 ? 1 : c);
}

}  // namespace

size_t colsum_workspace(long long rows, int cols) {
  return static_cast<size_t>(chunks_for(rows)) * cols * sizeof(float) + 256;
}

cudaError_t bias_dropout_residual_fwd(int dtype, const void* x, const void* bias, const void* res, void* out,
                                      long long rows, int cols, float p, uint64_t seed, uint64_t offset,
                                      cudaStream_t st) {
  const long long n = rows * cols;
  const unsigned g = grid_for(n, kThreads * 4);
  const int drop = p > 0.f;
  const uint32_t thr = dropout_threshold(p);
  const float ks = drop ? 1.f / (1.f - p) : 1.f;
  if (dtype == OASES_BF16)
    bdr_fwd_kernel<__nv_bfloat16><<<g, kThreads, 0, st>>>(
        static_cast<const __nv_bfloat16*>(x), static_cast<const __nv_bfloat16*>(bias),
        static_cast<const __nv_bfloat16*>(res), static_cast<__nv_bfloat16*>(out), n, cols, thr, ks, drop, seed, offset);
  else
    bdr_fwd_kernel<float><<<g, kThreads, 0, st>>>(static_cast<const float*>(x), static_cast<const float*>(bias),
                                                  static_cast<const float*>(res), static_cast<float*>(out), n, cols, thr,
                                                  ks, drop, seed, offset);
  return cudaGetLastError();
}

cudaError_t col_pass(int dtype, const void* in, void* dx, float* out, int acc, void* ws, long long rows, int cols,
                     float p, uint64_t seed, uint64_t offset, cudaStream_t st) {
  const int chunks = chunks_for(rows);
  const int rpc = static_cast<int>((rows + chunks - 1) / chunks);
  float* part = out ? static_cast<float*>(ws) : nullptr;
  dim3 grid((cols + kThreads - 1) / kThreads, chunks);
  const int drop = p > 0.f;
  const uint32_t thr = dropout_threshold(p);
  const float ks = drop ? 1.f / (1.f - p) : 1.f;
  if (dtype == OASES_BF16)
    col_pass_kernel<__nv_bfloat16><<<grid, kThreads, 0, st>>>(static_cast<const __nv_bfloat16*>(in),
                                                              static_cast<__nv_bfloat16*>(dx), part, rows, cols, rpc,
                                                              thr, ks, drop, seed, offset);
  else
    col_pass_kernel<float><<<grid, kThreads, 0, st>>>(static_cast<const float*>(in), static_cast<float*>(dx), part,
                                                      rows, cols, rpc, thr, ks, drop, seed, offset);
  if (out) col_finalize_kernel<<<(cols + kThreads - 1) / kThreads, kThreads, 0, st>>>(part, chunks, cols, out, acc);
  return cudaGetLastError();
}

cudaError_t gelu_fwd(int dtype, const void* x, void* y, long long n, cudaStream_t st) {
  const unsigned g = grid_for(n, kThreads);
  if (dtype == OASES_BF16)
    gelu_fwd_kernel<<<g, kThreads, 0, st>>>(static_cast<const __nv_bfloat16*>(x), static_cast<__nv_bfloat16*>(y), n);
  else
    gelu_fwd_kernel<<<g, kThreads, 0, st>>>(static_cast<const float*>(x), static_cast<float*>(y), n);
  return cudaGetLastError();
}

cudaError_t gelu_bwd(int dtype, const void* x, const void* dy, void* dx, long long n, cudaStream_t st) {
  const unsigned g = grid_for(n, kThreads);
  if (dtype == OASES_BF16)
    gelu_bwd_kernel<<<g, kThreads, 0, st>>>(static_cast<const __nv_bfloat16*>(x), static_cast<const __nv_bfloat16*>(dy),
                                            static_cast<__nv_bfloat16*>(dx), n);
  else
    gelu_bwd_kernel<<<g, kThreads, 0, st>>>(static_cast<const float*>(x), static_cast<const float*>(dy),
                                            static_cast<float*>(dx), n);
  return cudaGetLastError();
}

size_t loss_workspace() { return 1024 * sizeof(double); }

cudaError_t gelu_sq_loss(int dtype, const void* z, void* dz, double* loss, int acc, double* ws, long long n,
                         cudaStream_t st) {
  unsigned g = grid_for(n, kThreads * 4);
  if (g > 1024) g = 1024;
  if (dtype == OASES_BF16)
    gelu_sq_loss_kernel<<<g, kThreads, 0, st>>>(static_cast<const __nv_bfloat16*>(z), static_cast<__nv_bfloat16*>(dz),
                                                ws, n);
  else
    gelu_sq_loss_kernel<<<g, kThreads, 0, st>>>(static_cast<const float*>(z), static_cast<float*>(dz), ws, n);
  loss_finalize_kernel<<<1, 32, 0, st>>>(ws, static_cast<int>(g), loss, acc);
  return cudaGetLastError();
}

cudaError_t local_allreduce(int dtype, void* const* bufs, int w, long long n, cudaStream_t st) {
  if (w < 1 || w > 8) return cudaErrorInvalidValue;
  BufList b{};
  for (int i = 0; i < w; ++i) b.p[i] = bufs[i];
  const unsigned g = grid_for(n, kThreads);
  if (dtype == OASES_BF16) local_allreduce_kernel<__nv_bfloat16><<<g, kThreads, 0, st>>>(b, w, n);
  else local_allreduce_kernel<float><<<g, kThreads, 0, st>>>(b, w, n);
  return cudaGetLastError();
}

}  // namespace oases

namespace oases {
namespace {

template <typename T>
__global__ void __launch_bounds__(kThreads) fill_uniform_kernel(T* p, long long n, float scale, uint64_t seed,
                                                                uint64_t offset) {
  for (long long i = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) * 4; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x * 4) {
    uint32_t u[4];
    Philox::gen(seed, offset, static_cast<unsigned long long>(i) >> 2, u);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (i + q >= n) break;
      const float r = (static_cast<float>(u[q] >> 8) + 0.5f) * (1.0f / 16777216.0f);  // (0,1)
      p[i + q] = from_f<T>((2.f * r - 1.f) * scale);
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(kThreads) fill_const_kernel(T* p, long long n, float v) {
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    p[i] = from_f<T>(v);
}

template <typename S, typename D>
__global__ void __launch_bounds__(kThreads) convert_kernel(const S* src, D* dst, long long n) {
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    dst[i] = from_f<D>(to_f(src[i]));
}

}  // namespace

cudaError_t fill_uniform(int dtype, void* p, long long n, float scale, uint64_t seed, uint64_t offset,
                         cudaStream_t st) {
  const unsigned g = grid_for(n, kThreads * 4);
  if (dtype == OASES_BF16)
    fill_uniform_kernel<<<g, kThreads, 0, st>>>(static_cast<__nv_bfloat16*>(p), n, scale, seed, offset);
  else
    fill_uniform_kernel<<<g, kThreads, 0, st>>>(static_cast<float*>(p), n, scale, seed, offset);
  return cudaGetLastError();
}

cudaError_t fill_const(int dtype, void* p, long long n, float v, cudaStream_t st) {
  const unsigned g = grid_for(n, kThreads);
  if (dtype == OASES_BF16) fill_const_kernel<<<g, kThreads, 0, st>>>(static_cast<__nv_bfloat16*>(p), n, v);
  else fill_const_kernel<<<g, kThreads, 0, st>>>(static_cast<float*>(p), n, v);
  return cudaGetLastError();
}

cudaError_t convert(int sd, const void* src, int dd, void* dst, long long n, cudaStream_t st) {
  const unsigned g = grid_for(n, kThreads);
  if (sd == OASES_F32 && dd == OASES_BF16)
    convert_kernel<<<g, kThreads, 0, st>>>(static_cast<const float*>(src), static_cast<__nv_bfloat16*>(dst), n);
  else if (sd == OASES_BF16 && dd == OASES_F32)
    convert_kernel<<<g, kThreads, 0, st>>>(static_cast<const __nv_bfloat16*>(src), static_cast<float*>(dst), n);
  else if (sd == OASES_F32 && dd == OASES_F32)
    return cudaMemcpyAsync(dst, src, n * sizeof(float), cudaMemcpyDeviceToDevice, st);
  else
    return cudaMemcpyAsync(dst, src, n * 2, cudaMemcpyDeviceToDevice, st);
  return cudaGetLastError();
}

}  // namespace oases
