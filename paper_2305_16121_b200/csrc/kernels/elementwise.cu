// Elementwise / column-reduction HBM-bound kernels: bias-dropout-residual,
// column sums (bias gradients), exact-erf GeLU, the checker's loss head, the
// in-process AllReduce used to emulate TMP ranks on one device, and fills.
//
// All bulk paths move 16-byte vectors (8 bf16 / 4 f32) per thread; dropout
// masks come from Philox (one byte per element, 16 elements per call), so forward,
// recompute and backward regenerate them bit-exactly. Column reductions are
// two-stage with a fixed summation order (deterministic, no float atomics).
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

// ---------------------------------------------------------------- bias-dropout-residual
// out = residual + dropout(x + bias[col]); vector path (n % V == 0, cols % V == 0).
template <typename T>
__global__ void __launch_bounds__(kThreads) bdr_fwd_vec_kernel(const T* __restrict__ x, const T* __restrict__ bias,
                                                               const T* __restrict__ res, T* __restrict__ out,
                                                               long long n, int cols, uint32_t thr, float ks, int drop,
                                                               uint64_t seed, uint64_t offset) {
  constexpr int V = Vec<T>::N;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x * V;
  for (long long i = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) * V; i < n; i += stride) {
    float v[V];
    vload(x + i, v);
    if (bias) {
      float b[V];
      vload(bias + (i % cols), b);
#pragma unroll
      for (int q = 0; q < V; ++q) v[q] += b[q];
    }
    if (drop) apply_dropout<V>(v, static_cast<unsigned long long>(i), seed, offset, thr, ks);
    if (res) {
      float r[V];
      vload(res + i, r);
#pragma unroll
      for (int q = 0; q < V; ++q) v[q] += r[q];
    }
    vstore(out + i, v);
  }
}

// 16 elements per thread (one Philox counter, 2-4 vectors); cols % 16 == 0 so
// the 16 share one row. IDX = 32-bit indexing when n < 2^32.
template <typename T, typename IDX>
__global__ void __launch_bounds__(kThreads) bdr_fwd16_kernel(const T* __restrict__ x, const T* __restrict__ bias,
                                                             const T* __restrict__ res, T* __restrict__ out, IDX n,
                                                             IDX cols, uint32_t thr, float ks, int drop, uint64_t seed,
                                                             uint64_t offset) {
  pdl_trigger();
  pdl_wait();
  const IDX stride = static_cast<IDX>(gridDim.x) * blockDim.x * 16;
  for (IDX i = (static_cast<IDX>(blockIdx.x) * blockDim.x + threadIdx.x) * 16; i < n; i += stride) {
    float v[16];
    load16(x + i, v);
    if (res) {
      float r[16];
      load16(res + i, r);
      if (bias) {
        float b[16];
        load16(bias + (i % cols), b);
#pragma unroll
        for (int q = 0; q < 16; ++q) v[q] += b[q];
      }
      if (drop) apply_dropout16(v, static_cast<unsigned long long>(i), seed, offset, thr, ks);
#pragma unroll
      for (int q = 0; q < 16; ++q) v[q] += r[q];
    } else {
      if (bias) {
        float b[16];
        load16(bias + (i % cols), b);
#pragma unroll
        for (int q = 0; q < 16; ++q) v[q] += b[q];
      }
      if (drop) apply_dropout16(v, static_cast<unsigned long long>(i), seed, offset, thr, ks);
    }
    store16(out + i, v);
  }
}

// scalar fallback for shapes that are not 16-byte multiples (toy checker sizes)
template <typename T>
__global__ void __launch_bounds__(kThreads) bdr_fwd_kernel(const T* __restrict__ x, const T* __restrict__ bias,
                                                           const T* __restrict__ res, T* __restrict__ out, long long n,
                                                           int cols, uint32_t thr, float ks, int drop, uint64_t seed,
                                                           uint64_t offset) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x * 4;
  for (long long i = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) * 4; i < n; i += stride) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const long long e = i + q;
      if (e >= n) break;
      float v = to_f(x[e]);
      if (bias) v += to_f(bias[e % cols]);
      if (drop) v = dropout_one(v, static_cast<unsigned long long>(e), seed, offset, thr, ks);
      if (res) v += to_f(res[e]);
      out[e] = from_f<T>(v);
    }
  }
}

// ---------------------------------------------------------------- column pass
// dx = dropout'(in) (written if dx), partial column sums of dx over a chunk of
// rows (written if part). Each thread owns V consecutive columns.
template <typename T>
__global__ void __launch_bounds__(kThreads) col_pass_vec_kernel(const T* __restrict__ in, T* __restrict__ dx,
                                                                float* __restrict__ part, long long rows, int cols,
                                                                int rows_per_chunk, uint32_t thr, float ks, int drop,
                                                                uint64_t seed, uint64_t offset) {
  constexpr int V = Vec<T>::N;
  const int c = (blockIdx.x * kThreads + threadIdx.x) * V;
  if (c >= cols) return;
  const long long r0 = static_cast<long long>(blockIdx.y) * rows_per_chunk;
  const long long r1 = r0 + rows_per_chunk < rows ? r0 + rows_per_chunk : rows;
  float s[V] = {};
  for (long long r = r0; r < r1; ++r) {
    const long long e = r * cols + c;
    float v[V];
    vload(in + e, v);
    if (drop) apply_dropout<V>(v, static_cast<unsigned long long>(e), seed, offset, thr, ks);
    if (dx) vstore(dx + e, v);
#pragma unroll
    for (int q = 0; q < V; ++q) s[q] += v[q];
  }
  if (part) {
    float* p = part + static_cast<long long>(blockIdx.y) * cols + c;
#pragma unroll
    for (int q = 0; q < V; ++q) p[q] = s[q];
  }
}

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
    if (drop) v = dropout_one(v, static_cast<unsigned long long>(e), seed, offset, thr, ks);
    if (dx) dx[e] = from_f<T>(v);
    s += v;
  }
  if (part) part[static_cast<long long>(blockIdx.y) * cols + c] = s;
}

// Column-pass tiling for 16-column lanes: one warp per block covers 512
// columns (lane = 16 consecutive columns = one Philox counter) over a chunk of
// rows (4 rows in flight) and writes its column partials to part[chunk][col].
// No shared memory, few registers: the kernel co-resides with a persistent
// GEMM (which leaves < 3 KB of smem per SM), so on the side stream it runs
// under the GEMMs instead of after them.
template <typename T>
__global__ void __launch_bounds__(32) col_pass16_kernel(const T* __restrict__ in, T* __restrict__ dx,
                                                        float* __restrict__ part, long long rows, int cols,
                                                        int rows_per_chunk, uint32_t thr, float ks, int drop,
                                                        uint64_t seed, uint64_t offset) {
  pdl_trigger();
  pdl_wait();
  const int lane = threadIdx.x;
  const int c = blockIdx.x * 512 + lane * 16;
  if (c >= cols) return;
  const long long r0 = static_cast<long long>(blockIdx.y) * rows_per_chunk;
  const long long r1 = r0 + rows_per_chunk < rows ? r0 + rows_per_chunk : rows;
  float s[16] = {};
  long long r = r0;
  for (; r + 3 < r1; r += 4) {  // 4 rows in flight
    float v[4][16];
#pragma unroll
    for (int u = 0; u < 4; ++u) load16(in + (r + u) * cols + c, v[u]);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const long long e = (r + u) * cols + c;
      if (drop) apply_dropout16(v[u], static_cast<unsigned long long>(e), seed, offset, thr, ks);
      if (dx) store16(dx + e, v[u]);
#pragma unroll
      for (int q = 0; q < 16; ++q) s[q] += v[u][q];
    }
  }
  for (; r < r1; ++r) {
    const long long e = r * cols + c;
    float v[16];
    load16(in + e, v);
    if (drop) apply_dropout16(v, static_cast<unsigned long long>(e), seed, offset, thr, ks);
    if (dx) store16(dx + e, v);
#pragma unroll
    for (int q = 0; q < 16; ++q) s[q] += v[q];
  }
  if (!part) return;
  float* pp = part + static_cast<long long>(blockIdx.y) * cols + c;
#pragma unroll
  for (int q = 0; q < 16; q += 4) *reinterpret_cast<float4*>(pp + q) = make_float4(s[q], s[q + 1], s[q + 2], s[q + 3]);
}

// out[c] (+)= sum_k part[k][c]: a block covers 32 columns x 8 chunk lanes; lane
// group g sums chunks g, g+8, ... (4 loads in flight), then the 8 group sums
// are combined in g order -- a fixed summation order, so results are
// bit-reproducible.
__global__ void __launch_bounds__(kThreads) col_finalize_fast_kernel(const float* __restrict__ part, int chunks,
                                                                     int cols, float* __restrict__ out, int acc) {
  pdl_trigger();
  pdl_wait();
  __shared__ float sm[8][33];
  const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + lane;
  float t = 0.f;
  if (c < cols) {
    int k = g;
    for (; k + 24 < chunks; k += 32) {
      float v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = __ldg(part + static_cast<long long>(k + 8 * u) * cols + c);
#pragma unroll
      for (int u = 0; u < 4; ++u) t += v[u];
    }
    for (; k < chunks; k += 8) t += __ldg(part + static_cast<long long>(k) * cols + c);
  }
  sm[g][lane] = t;
  __syncthreads();
  if (g == 0 && c < cols) {
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += sm[j][lane];
    out[c] = acc ? out[c] + s : s;
  }
}

// out[c] (+)= sum_k part[k][c], fixed order: 8 interleaved partial sums per
// column, combined in index order.
__global__ void __launch_bounds__(kThreads) col_finalize_kernel(const float* __restrict__ part, int chunks, int cols,
                                                                float* __restrict__ out, int acc) {
  __shared__ float sm[8][33];
  const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + lane;
  float s = 0.f;
  if (c < cols)
    for (int k = g; k < chunks; k += 8) s += part[static_cast<long long>(k) * cols + c];
  sm[g][lane] = s;
  __syncthreads();
  if (g == 0 && c < cols) {
    float t = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) t += sm[j][lane];
    out[c] = acc ? out[c] + t : t;
  }
}

// ---------------------------------------------------------------- GeLU / loss
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
  pdl_trigger();
  pdl_wait();
  // 8 elements per step (16-byte bf16 vectors): f32 sum of the 8 terms, f64 across steps
  constexpr int V = 8;
  double acc = 0.0;
  const long long nv = n / V;
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < nv;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    float v[V], o[V];
    if constexpr (sizeof(T) == 2) {
      vload(z + i * V, v);
    } else {
      float a[4], b[4];
      vload(z + i * V, a);
      vload(z + i * V + 4, b);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        v[e] = a[e];
        v[4 + e] = b[e];
      }
    }
    float s = 0.f;
#pragma unroll
    for (int e = 0; e < V; ++e) {
      const float g = gelu_f(v[e]);
      s += 0.5f * g * g;
      o[e] = g * gelu_grad_f(v[e]);
    }
    acc += static_cast<double>(s);
    if (dz) {
      if constexpr (sizeof(T) == 2) {
        vstore(dz + i * V, o);
      } else {
        float a[4], b[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          a[e] = o[e];
          b[e] = o[4 + e];
        }
        vstore(dz + i * V, a);
        vstore(dz + i * V + 4, b);
      }
    }
  }
  // scalar tail
  for (long long i = nv * V + static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
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

// Deterministic tree over the block partials (fixed order).
__global__ void __launch_bounds__(kThreads) loss_finalize_kernel(const double* __restrict__ part, int nparts,
                                                                 double* __restrict__ out, int acc) {
  pdl_trigger();
  pdl_wait();
  __shared__ double sm[kThreads];
  double s = 0.0;
  for (int i = threadIdx.x; i < nparts; i += kThreads) s += part[i];
  sm[threadIdx.x] = s;
  __syncthreads();
  for (int w = kThreads / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) sm[threadIdx.x] += sm[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = acc ? *out + sm[0] : sm[0];
}

// ---------------------------------------------------------------- in-process AllReduce
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

// literal sum in worker order, 0 + x_0 + x_1 + ... (numerics.cpp:160-163)
__global__ void __launch_bounds__(kThreads) local_allreduce_f64_kernel(BufList b, int w, long long n) {
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    double s = static_cast<const double*>(b.p[0])[i];
    for (int k = 1; k < w; ++k) s = __dadd_rn(s, static_cast<const double*>(b.p[k])[i]);
    for (int k = 0; k < w; ++k) static_cast<double*>(b.p[k])[i] = s;
  }
}

__global__ void __launch_bounds__(kThreads) fill_f64_kernel(double* p, long long n, double v) {
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    p[i] = v;
}

__global__ void __launch_bounds__(kThreads) fill_uniform_f64_kernel(double* p, long long n, double scale,
                                                                    uint64_t seed, uint64_t offset) {
  for (long long i = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) * 4; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x * 4) {
    uint32_t u[4];
    Philox::gen(seed, offset, static_cast<unsigned long long>(i) >> 2, u);
    for (int q = 0; q < 4 && i + q < n; ++q) {
      const double r = (static_cast<double>(u[q]) + 0.5) * (1.0 / 4294967296.0);  // (0,1)
      p[i + q] = (2.0 * r - 1.0) * scale;
    }
  }
}

// ---------------------------------------------------------------- fills
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

// ---------------------------------------------------------------- f64 (value-level toy checks)
// The f64 mode runs the reference's toy checker (numerics.hpp:35-60) through the
// runtime: no dropout, no LayerNorm; plain scalar kernels in the reference's
// operation order (numerics.cpp:34-39 add, 175-188 loss head).
__global__ void __launch_bounds__(kThreads) bdr_f64_kernel(const double* __restrict__ x, const double* __restrict__ bias,
                                                           const double* __restrict__ res, double* __restrict__ out,
                                                           long long n, int cols) {
  for (long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    double v = x[e];
    if (bias) v = __dadd_rn(v, bias[e % cols]);
    out[e] = res ? __dadd_rn(res[e], v) : v;
  }
}

__global__ void __launch_bounds__(kThreads) gelu_sq_loss_f64_kernel(const double* __restrict__ z, double* __restrict__ dz,
                                                                    double* __restrict__ part, long long n) {
  double acc = 0.0;
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const double v = z[i];
    const double g = gelu_d(v);
    acc += 0.5 * g * g;
    if (dz) dz[i] = __dmul_rn(g, gelu_grad_d(v));
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

struct ColSplit {
  int chunks, rows_per_chunk;
};
// ~4 CTAs per SM over (column blocks x row chunks)
ColSplit col_split(long long rows, int col_blocks) {
  long long chunks = (4LL * 148 + col_blocks - 1) / col_blocks;
  if (chunks > rows) chunks = rows;
  if (chunks < 1) chunks = 1;
  const int rpc = static_cast<int>((rows + chunks - 1) / chunks);
  return {static_cast<int>((rows + rpc - 1) / rpc), rpc};
}

// (512-column groups) x (row chunks): ~8 single-warp CTAs per SM, >= 8 rows per chunk
ColSplit col_split16(long long rows, int cols) {
  const int groups = (cols + 511) / 512;
  long long chunks = (8LL * 148 + groups - 1) / groups;
  const long long maxc = (rows + 7) / 8;
  if (chunks > maxc) chunks = maxc;
  if (chunks < 1) chunks = 1;
  const int rpc = static_cast<int>((rows + chunks - 1) / chunks);
  return {static_cast<int>((rows + rpc - 1) / rpc), rpc};
}

template <typename T>
bool vec_ok(const void* a, const void* b, long long n, int cols) {
  constexpr int V = 16 / sizeof(T);
  auto al = [](const void* p) { return p == nullptr || (reinterpret_cast<uintptr_t>(p) % 16) == 0; };
  return n % V == 0 && cols % V == 0 && al(a) && al(b);
}

template <typename T>
void bdr16(const T* X, const T* B, const T* R, T* O, long long n, int cols, uint32_t thr, float ks, int drop,
           uint64_t seed, uint64_t offset, cudaStream_t st) {
  long long g = (n / 16 + kThreads - 1) / kThreads;
  if (g > 148LL * 8) g = 148LL * 8;
  if (g < 1) g = 1;
  if (n < (1LL << 31))  // 32-bit index arithmetic cannot wrap
    launch_pdl(bdr_fwd16_kernel<T, uint32_t>, dim3(static_cast<unsigned>(g)), dim3(kThreads), 0, st, X, B, R, O,
               static_cast<uint32_t>(n), static_cast<uint32_t>(cols), thr, ks, drop, seed, offset);
  else
    launch_pdl(bdr_fwd16_kernel<T, unsigned long long>, dim3(static_cast<unsigned>(g)), dim3(kThreads), 0, st, X, B,
               R, O, static_cast<unsigned long long>(n), static_cast<unsigned long long>(cols), thr, ks, drop, seed,
               offset);
}

}  // namespace

size_t colsum_workspace(long long rows, int cols) {
  // upper bound over both the vector (V columns per thread) and scalar layouts
  int chunks = 1;
  for (int v : {1, 4, 8}) {  // scalar, f32 and bf16 vector layouts
    const ColSplit s = col_split(rows, (cols + kThreads * v - 1) / (kThreads * v));
    if (s.chunks > chunks) chunks = s.chunks;
  }
  if (col_split16(rows, cols).chunks > chunks) chunks = col_split16(rows, cols).chunks;
  return static_cast<size_t>(chunks) * cols * sizeof(float) + 256;
}

cudaError_t bias_dropout_residual_fwd(int dtype, const void* x, const void* bias, const void* res, void* out,
                                      long long rows, int cols, float p, uint64_t seed, uint64_t offset,
                                      cudaStream_t st) {
  const long long n = rows * cols;
  const int drop = p > 0.f;
  const uint32_t thr = dropout_threshold(p);
  const float ks = dropout_keep_scale(p);
  if (dtype == OASES_F64) {
    if (drop) return cudaErrorNotSupported;  // the f64 toy mode has no dropout
    bdr_f64_kernel<<<grid_for(n, kThreads), kThreads, 0, st>>>(static_cast<const double*>(x),
                                                              static_cast<const double*>(bias),
                                                              static_cast<const double*>(res),
                                                              static_cast<double*>(out), n, cols);
    return cudaGetLastError();
  }
  if (dtype == OASES_BF16) {
    using T = __nv_bfloat16;
    auto X = static_cast<const T*>(x);
    auto B = static_cast<const T*>(bias);
    auto R = static_cast<const T*>(res);
    auto O = static_cast<T*>(out);
    if (cols % 16 == 0 && vec_ok<T>(x, out, n, cols) && vec_ok<T>(bias, res, n, cols))
      bdr16<T>(X, B, R, O, n, cols, thr, ks, drop, seed, offset, st);
    else if (vec_ok<T>(x, out, n, cols) && vec_ok<T>(bias, res, n, cols))
      bdr_fwd_vec_kernel<T><<<grid_for(n, kThreads * 8), kThreads, 0, st>>>(X, B, R, O, n, cols, thr, ks, drop, seed,
                                                                          offset);
    else
      bdr_fwd_kernel<T><<<grid_for(n, kThreads * 4), kThreads, 0, st>>>(X, B, R, O, n, cols, thr, ks, drop, seed,
                                                                      offset);
  } else {
    using T = float;
    auto X = static_cast<const T*>(x);
    auto B = static_cast<const T*>(bias);
    auto R = static_cast<const T*>(res);
    auto O = static_cast<T*>(out);
    if (cols % 16 == 0 && vec_ok<T>(x, out, n, cols) && vec_ok<T>(bias, res, n, cols))
      bdr16<T>(X, B, R, O, n, cols, thr, ks, drop, seed, offset, st);
    else if (vec_ok<T>(x, out, n, cols) && vec_ok<T>(bias, res, n, cols))
      bdr_fwd_vec_kernel<T><<<grid_for(n, kThreads * 4), kThreads, 0, st>>>(X, B, R, O, n, cols, thr, ks, drop, seed,
                                                                          offset);
    else
      bdr_fwd_kernel<T><<<grid_for(n, kThreads * 4), kThreads, 0, st>>>(X, B, R, O, n, cols, thr, ks, drop, seed,
                                                                      offset);
  }
  return cudaGetLastError();
}

template <typename T>
static bool col_pass_t(const void* in, void* dx, float* part, long long rows, int cols, uint32_t thr, float ks,
                       int drop, uint64_t seed, uint64_t offset, int* chunks_out, cudaStream_t st) {
  constexpr int V = 16 / sizeof(T);
  if (cols % 16 == 0 && vec_ok<T>(in, dx, rows * cols, cols) && vec_ok<T>(part, nullptr, cols, cols)) {
    const ColSplit sp = col_split16(rows, cols);
    launch_pdl(col_pass16_kernel<T>, dim3((cols + 511) / 512, sp.chunks), dim3(32), 0, st, static_cast<const T*>(in),
               static_cast<T*>(dx), part, rows, cols, sp.rows_per_chunk, thr, ks, drop, seed, offset);
    *chunks_out = sp.chunks;
    return true;
  }
  if (vec_ok<T>(in, dx, rows * cols, cols)) {
    const int cb = (cols + kThreads * V - 1) / (kThreads * V);
    const ColSplit sp = col_split(rows, cb);
    col_pass_vec_kernel<T><<<dim3(cb, sp.chunks), kThreads, 0, st>>>(static_cast<const T*>(in), static_cast<T*>(dx),
                                                                      part, rows, cols, sp.rows_per_chunk, thr, ks,
                                                                      drop, seed, offset);
    *chunks_out = sp.chunks;
  } else {
    const int cb = (cols + kThreads - 1) / kThreads;
    const ColSplit sp = col_split(rows, cb);
    col_pass_kernel<T><<<dim3(cb, sp.chunks), kThreads, 0, st>>>(static_cast<const T*>(in), static_cast<T*>(dx), part,
                                                                  rows, cols, sp.rows_per_chunk, thr, ks, drop, seed,
                                                                  offset);
    *chunks_out = sp.chunks;
  }
  return false;
}

cudaError_t col_pass(int dtype, const void* in, void* dx, float* out, int acc, void* ws, long long rows, int cols,
                     float p, uint64_t seed, uint64_t offset, cudaStream_t st) {
  float* part = out ? static_cast<float*>(ws) : nullptr;
  const int drop = p > 0.f;
  const uint32_t thr = dropout_threshold(p);
  const float ks = dropout_keep_scale(p);
  int chunks = 0;
  bool fast;
  if (dtype == OASES_BF16)
    fast = col_pass_t<__nv_bfloat16>(in, dx, part, rows, cols, thr, ks, drop, seed, offset, &chunks, st);
  else
    fast = col_pass_t<float>(in, dx, part, rows, cols, thr, ks, drop, seed, offset, &chunks, st);
  if (out) {
    if (fast)
      launch_pdl(col_finalize_fast_kernel, dim3((cols + 31) / 32), dim3(kThreads), 0, st,
                 static_cast<const float*>(part), chunks, cols, out, acc);
    else
      col_finalize_kernel<<<(cols + 31) / 32, kThreads, 0, st>>>(part, chunks, cols, out, acc);
  }
  return cudaGetLastError();
}

cudaError_t col_finalize(const float* part, long long chunks, int cols, float* out, int acc, cudaStream_t st) {
  launch_pdl(col_finalize_fast_kernel, dim3((cols + 31) / 32), dim3(kThreads), 0, st, part, static_cast<int>(chunks),
             cols, out, acc);
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
  unsigned g = grid_for(n, kThreads * 32);
  if (g > 1024) g = 1024;
  // 16-byte vector path needs aligned buffers
  const size_t es = dtype == OASES_BF16 ? 2 : (dtype == OASES_F64 ? 8 : 4);
  if (dtype != OASES_F64 && ((reinterpret_cast<uintptr_t>(z) | reinterpret_cast<uintptr_t>(dz)) & 15u))
    return cudaErrorMisalignedAddress;
  (void)es;
  if (dtype == OASES_F64)
    gelu_sq_loss_f64_kernel<<<g, kThreads, 0, st>>>(static_cast<const double*>(z), static_cast<double*>(dz), ws, n);
  else if (dtype == OASES_BF16)
    launch_pdl(gelu_sq_loss_kernel<__nv_bfloat16>, dim3(g), dim3(kThreads), 0, st, static_cast<const __nv_bfloat16*>(z),
               static_cast<__nv_bfloat16*>(dz), ws, n);
  else
    launch_pdl(gelu_sq_loss_kernel<float>, dim3(g), dim3(kThreads), 0, st, static_cast<const float*>(z),
               static_cast<float*>(dz), ws, n);
  return launch_pdl(loss_finalize_kernel, dim3(1), dim3(kThreads), 0, st, static_cast<const double*>(ws),
                    static_cast<int>(g), loss, acc);
}

cudaError_t local_allreduce(int dtype, void* const* bufs, int w, long long n, cudaStream_t st) {
  if (w < 1 || w > 8) return cudaErrorInvalidValue;
  BufList b{};
  for (int i = 0; i < w; ++i) b.p[i] = bufs[i];
  const unsigned g = grid_for(n, kThreads);
  if (dtype == OASES_F64) local_allreduce_f64_kernel<<<g, kThreads, 0, st>>>(b, w, n);
  else if (dtype == OASES_BF16) local_allreduce_kernel<__nv_bfloat16><<<g, kThreads, 0, st>>>(b, w, n);
  else local_allreduce_kernel<float><<<g, kThreads, 0, st>>>(b, w, n);
  return cudaGetLastError();
}

// In-process AllGather (1-GPU emulation of a TMP group's resharding
// AllGather): w buffers, each holding chunk i (n elements at offset i*n) of
// its own; afterwards every buffer holds all w chunks. blockIdx.y = (dst, src)
// pair, 16-byte copies.
__global__ void __launch_bounds__(kThreads) local_allgather_kernel(BufList b, int w, long long n16) {
  const int pair = blockIdx.y, dst = pair / w, src = pair % w;
  if (dst == src) return;
  const uint4* s = reinterpret_cast<const uint4*>(b.p[src]) + src * n16;
  uint4* d = reinterpret_cast<uint4*>(b.p[dst]) + src * n16;
  for (long long i = blockIdx.x * static_cast<long long>(kThreads) + threadIdx.x; i < n16;
       i += static_cast<long long>(gridDim.x) * kThreads)
    d[i] = s[i];
}

cudaError_t local_allgather(int dtype, void* const* bufs, int w, long long n, cudaStream_t st) {
  if (w < 1 || w > 8) return cudaErrorInvalidValue;
  const long long bytes = n * (dtype == OASES_BF16 ? 2 : dtype == OASES_F64 ? 8 : 4);
  BufList b{};
  for (int i = 0; i < w; ++i) {
    b.p[i] = bufs[i];
    if ((reinterpret_cast<uintptr_t>(bufs[i]) & 15u) != 0) return cudaErrorMisalignedAddress;
  }
  if (bytes % 16) return cudaErrorInvalidValue;
  if (w == 1) return cudaSuccess;
  const long long n16 = bytes / 16;
  long long gx = (n16 + kThreads * 4 - 1) / (kThreads * 4);
  if (gx > 1184) gx = 1184;
  local_allgather_kernel<<<dim3(static_cast<unsigned>(gx < 1 ? 1 : gx), static_cast<unsigned>(w * w)), kThreads, 0,
                           st>>>(b, w, n16);
  return cudaGetLastError();
}

cudaError_t fill_uniform(int dtype, void* p, long long n, float scale, uint64_t seed, uint64_t offset,
                         cudaStream_t st) {
  const unsigned g = grid_for(n, kThreads * 4);
  if (dtype == OASES_F64)
    fill_uniform_f64_kernel<<<g, kThreads, 0, st>>>(static_cast<double*>(p), n, scale, seed, offset);
  else if (dtype == OASES_BF16)
    fill_uniform_kernel<<<g, kThreads, 0, st>>>(static_cast<__nv_bfloat16*>(p), n, scale, seed, offset);
  else
    fill_uniform_kernel<<<g, kThreads, 0, st>>>(static_cast<float*>(p), n, scale, seed, offset);
  return cudaGetLastError();
}

cudaError_t fill_const(int dtype, void* p, long long n, float v, cudaStream_t st) {
  const unsigned g = grid_for(n, kThreads);
  if (dtype == OASES_F64) fill_f64_kernel<<<g, kThreads, 0, st>>>(static_cast<double*>(p), n, v);
  else if (dtype == OASES_BF16) fill_const_kernel<<<g, kThreads, 0, st>>>(static_cast<__nv_bfloat16*>(p), n, v);
  else fill_const_kernel<<<g, kThreads, 0, st>>>(static_cast<float*>(p), n, v);
  return cudaGetLastError();
}

cudaError_t convert(int sd, const void* src, int dd, void* dst, long long n, cudaStream_t st) {
  const unsigned g = grid_for(n, kThreads);
  if (sd == OASES_F64 || dd == OASES_F64) {
    if (sd != dd) return cudaErrorNotSupported;
    return cudaMemcpyAsync(dst, src, n * sizeof(double), cudaMemcpyDeviceToDevice, st);
  }
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
