// Row-wise HBM-bound kernels: LayerNorm fwd/bwd and causal softmax fwd/bwd.
//
// One warp per row, 16-byte vector loads, warp-shuffle reductions, f32
// statistics. The reference restates none of these (its toy FFN has no LN and
// no attention, numerics.hpp:37-44); the fp64 oracle (oracle/gpt_oracle.cpp)
// defines their parity semantics.
#include "common.cuh"
#include "kernels.h"

namespace oases {
namespace {

template <typename T>
struct Vec;
template <>
struct Vec<float> {
  static constexpr int N = 4;
  using raw = float4;
  __device__ static void unpack(const raw& r, float (&v)[4]) { v[0] = r.x; v[1] = r.y; v[2] = r.z; v[3] = r.w; }
  __device__ static raw pack(const float (&v)[4]) { return make_float4(v[0], v[1], v[2], v[3]); }
};
template <>
struct Vec<__nv_bfloat16> {
  static constexpr int N = 8;
  using raw = uint4;
  __device__ static void unpack(const raw& r, float (&v)[8]) {
    const uint32_t w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[j]));
      v[2 * j] = f.x;
      v[2 * j + 1] = f.y;
    }
  }
  __device__ static raw pack(const float (&v)[8]) {
    uint32_t w[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * j], v[2 * j + 1]);
      w[j] = *reinterpret_cast<uint32_t*>(&h);
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
  }
};

template <typename T>
__device__ __forceinline__ void vload(const T* p, float (&v)[Vec<T>::N]) {
  Vec<T>::unpack(*reinterpret_cast<const typename Vec<T>::raw*>(p), v);
}
template <typename T>
__device__ __forceinline__ void vstore(T* p, const float (&v)[Vec<T>::N]) {
  *reinterpret_cast<typename Vec<T>::raw*>(p) = Vec<T>::pack(v);
}

// Chan/Welford merge of (n, mean, M2) across a warp.
__device__ __forceinline__ void welford_warp(float& n, float& mean, float& m2) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float n2 = __shfl_xor_sync(0xffffffffu, n, o);
    const float mean2 = __shfl_xor_sync(0xffffffffu, mean, o);
    const float m22 = __shfl_xor_sync(0xffffffffu, m2, o);
    const float nt = n + n2;
    if (nt > 0.f) {
      const float d = mean2 - mean;
      mean += d * (n2 / nt);
      m2 += m22 + d * d * (n * n2 / nt);
      n = nt;
    }
  }
}

template <typename T>
__device__ __forceinline__ void row_stats(const T* x, int cols, float eps, float& mean, float& rstd) {
  constexpr int V = Vec<T>::N;
  const int lane = threadIdx.x & 31;
  float n = 0.f, mu = 0.f, m2 = 0.f;
  for (int c = lane * V; c < cols; c += 32 * V) {
    float v[V];
    vload(x + c, v);
#pragma unroll
    for (int i = 0; i < V; ++i) {
      n += 1.f;
      const float d = v[i] - mu;
      mu += d / n;
      m2 += d * (v[i] - mu);
    }
  }
  welford_warp(n, mu, m2);
  mean = mu;
  rstd = rsqrtf(m2 / static_cast<float>(cols) + eps);
}

template <typename T>
__global__ void __launch_bounds__(256) ln_fwd_kernel(const T* __restrict__ x, const T* __restrict__ gamma,
                                                     const T* __restrict__ beta, T* __restrict__ y, long long rows,
                                                     int cols, float eps) {
  constexpr int V = Vec<T>::N;
  const long long row = static_cast<long long>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  if (row >= rows) return;
  const int lane = threadIdx.x & 31;
  const T* xr = x + row * cols;
  float mean, rstd;
  row_stats(xr, cols, eps, mean, rstd);
  T* yr = y + row * cols;
  for (int c = lane * V; c < cols; c += 32 * V) {
    float v[V], g[V], b[V];
    vload(xr + c, v);
    vload(gamma + c, g);
    vload(beta + c, b);
#pragma unroll
    for (int i = 0; i < V; ++i) v[i] = (v[i] - mean) * rstd * g[i] + b[i];
    vstore(yr + c, v);
  }
}

// dx (+)= rstd * (g - mean(g) - xhat * mean(g * xhat)),  g = dy * gamma.
// Writes the row statistics for the parameter-gradient column pass.
template <typename T>
__global__ void __launch_bounds__(256) ln_bwd_kernel(const T* __restrict__ x, const T* __restrict__ gamma,
                                                     const T* __restrict__ dy, T* __restrict__ dx, int acc,
                                                     float2* __restrict__ stats, long long rows, int cols, float eps) {
  constexpr int V = Vec<T>::N;
  const long long row = static_cast<long long>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  if (row >= rows) return;
  const int lane = threadIdx.x & 31;
  const T* xr = x + row * cols;
  const T* dyr = dy + row * cols;
  float mean, rstd;
  row_stats(xr, cols, eps, mean, rstd);
  float s1 = 0.f, s2 = 0.f;
  for (int c = lane * V; c < cols; c += 32 * V) {
    float v[V], g[V], d[V];
    vload(xr + c, v);
    vload(gamma + c, g);
    vload(dyr + c, d);
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const float gg = d[i] * g[i];
      s1 += gg;
      s2 += gg * (v[i] - mean) * rstd;
    }
  }
  s1 = warp_sum(s1) / static_cast<float>(cols);
  s2 = warp_sum(s2) / static_cast<float>(cols);
  if (lane == 0) stats[row] = make_float2(mean, rstd);
  T* dxr = dx + row * cols;
  for (int c = lane * V; c < cols; c += 32 * V) {
    float v[V], g[V], d[V], o[V];
    vload(xr + c, v);
    vload(gamma + c, g);
    vload(dyr + c, d);
    if (acc) vload(dxr + c, o);
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const float xh = (v[i] - mean) * rstd;
      const float r = rstd * (d[i] * g[i] - s1 - xh * s2);
      o[i] = acc ? o[i] + r : r;
    }
    vstore(dxr + c, o);
  }
}

// Column partial sums over a chunk of rows: part[chunk][0][c] = sum dy*xhat,
// part[chunk][1][c] = sum dy. Threads own columns -> coalesced, deterministic.
template <typename T>
__global__ void __launch_bounds__(256) ln_param_partial_kernel(const T* __restrict__ x, const T* __restrict__ dy,
                                                               const float2* __restrict__ stats, float* __restrict__ part,
                                                               long long rows, int cols, int rows_per_chunk) {
  const int c = blockIdx.x * 256 + threadIdx.x;
  if (c >= cols) return;
  const long long r0 = static_cast<long long>(blockIdx.y) * rows_per_chunk;
  long long r1 = r0 + rows_per_chunk;
  if (r1 > rows) r1 = rows;
  float sg = 0.f, sb = 0.f;
  for (long long r = r0; r < r1; ++r) {
    const float2 st = stats[r];
    const float d = to_f(dy[r * cols + c]);
    sg += d * (to_f(x[r * cols + c]) - st.x) * st.y;
    sb += d;
  }
  part[(static_cast<long long>(blockIdx.y) * 2 + 0) * cols + c] = sg;
  part[(static_cast<long long>(blockIdx.y) * 2 + 1) * cols + c] = sb;
}

__global__ void colpair_finalize_kernel(const float* __restrict__ part, int chunks, int cols, float* __restrict__ out0,
                                        float* __restrict__ out1, int acc) {
  const int c = blockIdx.x * 256 + threadIdx.x;
  if (c >= cols) return;
  float a = 0.f, b = 0.f;
  for (int k = 0; k < chunks; ++k) {
    a += part[(static_cast<long long>(k) * 2 + 0) * cols + c];
    b += part[(static_cast<long long>(k) * 2 + 1) * cols + c];
  }
  if (out0) out0[c] = acc ? out0[c] + a : a;
  if (out1) out1[c] = acc ? out1[c] + b : b;
}

// ------------------------------------------------------------------ softmax
// Row r of S (viewed [batch*seq, seq]) is query position i = r % seq; keys
// j <= i are valid. P = softmax(scale * S) over valid keys, zeros elsewhere.
// The row is cached in registers: NV vectors per lane.
// Dropout element index uses the GLOBAL head (head_offset + local head) so the
// mask does not depend on the TMP degree: row r = (n*Hl + jl)*seq + i maps to
// global row (n*Hg + head_offset + jl)*seq + i.
__device__ __forceinline__ unsigned long long global_row(long long row, int seq, int hl, int hg, int hoff) {
  const long long per = static_cast<long long>(hl) * seq;
  const long long n = row / per, rem = row - n * per;
  const long long jl = rem / seq, i = rem - jl * seq;
  return static_cast<unsigned long long>((n * hg + hoff + jl) * seq + i);
}

template <typename T, int NV>
__global__ void __launch_bounds__(256) softmax_fwd_kernel(const T* __restrict__ s, T* __restrict__ p,
                                                          T* __restrict__ pd, long long rows, int seq, float scale,
                                                          uint32_t thr, float keep_scale, uint64_t seed,
                                                          uint64_t offset, int hl, int hg, int hoff) {
  constexpr int V = Vec<T>::N;
  const long long row = static_cast<long long>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  if (row >= rows) return;
  const int lane = threadIdx.x & 31;
  const int i = static_cast<int>(row % seq);
  const T* sr = s + row * seq;
  float v[NV][V];
  float mx = -INFINITY;
#pragma unroll
  for (int t = 0; t < NV; ++t) {
    const int c = (t * 32 + lane) * V;
    if (c < seq && c <= i) {
      vload(sr + c, v[t]);
#pragma unroll
      for (int e = 0; e < V; ++e) {
        v[t][e] = (c + e <= i) ? v[t][e] * scale : -INFINITY;
        mx = fmaxf(mx, v[t][e]);
      }
    } else {
#pragma unroll
      for (int e = 0; e < V; ++e) v[t][e] = -INFINITY;
    }
  }
  mx = warp_max(mx);
  float sum = 0.f;
#pragma unroll
  for (int t = 0; t < NV; ++t)
#pragma unroll
    for (int e = 0; e < V; ++e) {
      const float ex = v[t][e] == -INFINITY ? 0.f : __expf(v[t][e] - mx);
      v[t][e] = ex;
      sum += ex;
    }
  sum = warp_sum(sum);
  const float inv = 1.f / sum;
  T* pr = p + row * seq;
  T* pdr = pd ? pd + row * seq : nullptr;
#pragma unroll
  for (int t = 0; t < NV; ++t) {
    const int c = (t * 32 + lane) * V;
    if (c >= seq) continue;
#pragma unroll
    for (int e = 0; e < V; ++e) v[t][e] *= inv;
    vstore(pr + c, v[t]);
    if (pdr) {
      const unsigned long long base = global_row(row, seq, hl, hg, hoff) * seq + c;
#pragma unroll
      for (int e = 0; e < V; e += 4) {
        uint32_t u[4];
        Philox::gen(seed, offset, (base + e) >> 2, u);
#pragma unroll
        for (int q = 0; q < 4; ++q) v[t][e + q] = (u[q] >= thr) ? v[t][e + q] * keep_scale : 0.f;
      }
      vstore(pdr + c, v[t]);
    }
  }
}

// dS = scale * P o (dP - sum_j P_j dP_j), dP = dropout'(dP_drop).
template <typename T, int NV>
__global__ void __launch_bounds__(256) softmax_bwd_kernel(const T* __restrict__ p, const T* __restrict__ dpd,
                                                          T* __restrict__ ds, long long rows, int seq, float scale,
                                                          uint32_t thr, float keep_scale, int use_dropout,
                                                          uint64_t seed, uint64_t offset, int hl, int hg, int hoff) {
  constexpr int V = Vec<T>::N;
  const long long row = static_cast<long long>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  if (row >= rows) return;
  const int lane = threadIdx.x & 31;
  const int i = static_cast<int>(row % seq);
  float pv[NV][V], dv[NV][V];
  float dot = 0.f;
#pragma unroll
  for (int t = 0; t < NV; ++t) {
    const int c = (t * 32 + lane) * V;
    if (c < seq && c <= i) {
      vload(p + row * seq + c, pv[t]);
      vload(dpd + row * seq + c, dv[t]);
      if (use_dropout) {
        const unsigned long long base = global_row(row, seq, hl, hg, hoff) * seq + c;
#pragma unroll
        for (int e = 0; e < V; e += 4) {
          uint32_t u[4];
          Philox::gen(seed, offset, (base + e) >> 2, u);
#pragma unroll
          for (int q = 0; q < 4; ++q) dv[t][e + q] = (u[q] >= thr) ? dv[t][e + q] * keep_scale : 0.f;
        }
      }
#pragma unroll
      for (int e = 0; e < V; ++e) {
        if (c + e > i) { pv[t][e] = 0.f; dv[t][e] = 0.f; }
        dot += pv[t][e] * dv[t][e];
      }
    } else {
#pragma unroll
      for (int e = 0; e < V; ++e) { pv[t][e] = 0.f; dv[t][e] = 0.f; }
    }
  }
  dot = warp_sum(dot);
#pragma unroll
  for (int t = 0; t < NV; ++t) {
    const int c = (t * 32 + lane) * V;
    if (c >= seq) continue;
#pragma unroll
    for (int e = 0; e < V; ++e) pv[t][e] = scale * pv[t][e] * (dv[t][e] - dot);
    vstore(ds + row * seq + c, pv[t]);
  }
}

template <typename T, template <typename, int> class K, typename... Args>
cudaError_t launch_rows_nv(int seq, long long rows, cudaStream_t st, Args... args) {
  constexpr int V = Vec<T>::N;
  const int nv = (seq + 32 * V - 1) / (32 * V);
  const unsigned grid = static_cast<unsigned>((rows + 7) / 8);
  if (nv <= 1) K<T, 1>::launch(grid, st, args...);
  else if (nv <= 2) K<T, 2>::launch(grid, st, args...);
  else if (nv <= 4) K<T, 4>::launch(grid, st, args...);
  else if (nv <= 8) K<T, 8>::launch(grid, st, args...);
  else if (nv <= 16) K<T, 16>::launch(grid, st, args...);
  else return cudaErrorInvalidValue;
  return cudaGetLastError();
}

template <typename T, int NV>
struct SoftmaxFwdL {
  template <typename... A>
  static void launch(unsigned grid, cudaStream_t st, A... a) {
    softmax_fwd_kernel<T, NV><<<grid, 256, 0, st>>>(a...);
  }
};
template <typename T, int NV>
struct SoftmaxBwdL {
  template <typename... A>
  static void launch(unsigned grid, cudaStream_t st, A... a) {
    softmax_bwd_kernel<T, NV><<<grid, 256, 0, st>>>(a...);
  }
};

int param_chunks(long long rows) {
  long long c = (rows + 63) / 64;
  if (c > 256) c = 256;
  return static_cast<int>(c < 1 ? 1 : c);
}

}  // namespace

size_t layernorm_bwd_workspace(long long rows, int cols) {
  const int chunks = param_chunks(rows);
  return static_cast<size_t>(rows) * sizeof(float2) + static_cast<size_t>(chunks) * 2 * cols * sizeof(float) + 256;
}

cudaError_t layernorm_fwd(int dtype, const void* x, const void* gamma, const void* beta, void* y, long long rows,
                          int cols, float eps, cudaStream_t st) {
  const unsigned grid = static_cast<unsigned>((rows + 7) / 8);
  if (dtype == OASES_BF16)
    ln_fwd_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>(
        static_cast<const __nv_bfloat16*>(x), static_cast<const __nv_bfloat16*>(gamma),
        static_cast<const __nv_bfloat16*>(beta), static_cast<__nv_bfloat16*>(y), rows, cols, eps);
  else
    ln_fwd_kernel<float><<<grid, 256, 0, st>>>(static_cast<const float*>(x), static_cast<const float*>(gamma),
                                               static_cast<const float*>(beta), static_cast<float*>(y), rows, cols,
                                               eps);
  return cudaGetLastError();
}

cudaError_t layernorm_bwd(int dtype, const void* x, const void* gamma, const void* dy, void* dx, int acc_dx,
                          float* dgamma, float* dbeta, int acc_params, void* workspace, long long rows, int cols,
                          float eps, cudaStream_t st) {
  float2* stats = static_cast<float2*>(workspace);
  float* part = reinterpret_cast<float*>(static_cast<char*>(workspace) +
                                         ((static_cast<size_t>(rows) * sizeof(float2) + 255) & ~size_t(255)));
  const unsigned grid = static_cast<unsigned>((rows + 7) / 8);
  const int chunks = param_chunks(rows);
  const int rpc = static_cast<int>((rows + chunks - 1) / chunks);
  dim3 pgrid((cols + 255) / 256, chunks);
  if (dtype == OASES_BF16) {
    auto X = static_cast<const __nv_bfloat16*>(x);
    auto DY = static_cast<const __nv_bfloat16*>(dy);
    ln_bwd_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>(X, static_cast<const __nv_bfloat16*>(gamma), DY,
                                                       static_cast<__nv_bfloat16*>(dx), acc_dx, stats, rows, cols, eps);
    if (dgamma || dbeta) ln_param_partial_kernel<__nv_bfloat16><<<pgrid, 256, 0, st>>>(X, DY, stats, part, rows, cols, rpc);
  } else {
    auto X = static_cast<const float*>(x);
    auto DY = static_cast<const float*>(dy);
    ln_bwd_kernel<float><<<grid, 256, 0, st>>>(X, static_cast<const float*>(gamma), DY, static_cast<float*>(dx),
                                               acc_dx, stats, rows, cols, eps);
    if (dgamma || dbeta) ln_param_partial_kernel<float><<<pgrid, 256, 0, st>>>(X, DY, stats, part, rows, cols, rpc);
  }
  if (dgamma || dbeta)
    colpair_finalize_kernel<<<(cols + 255) / 256, 256, 0, st>>>(part, chunks, cols, dgamma, dbeta, acc_params);
  return cudaGetLastError();
}

cudaError_t softmax_fwd(int dtype, const void* s, void* p, void* pd, long long batch, int seq, float scale,
                        float dropout_p, uint64_t seed, uint64_t offset, int hl, int hg, int hoff, cudaStream_t st) {
  const long long rows = batch * seq;
  const uint32_t thr = dropout_threshold(dropout_p);
  const float ks = dropout_p > 0.f ? 1.f / (1.f - dropout_p) : 1.f;
  if (dropout_p <= 0.f) pd = nullptr;
  if (dtype == OASES_BF16)
    return launch_rows_nv<__nv_bfloat16, SoftmaxFwdL>(seq, rows, st, static_cast<const __nv_bfloat16*>(s),
                                                      static_cast<__nv_bfloat16*>(p), static_cast<__nv_bfloat16*>(pd),
                                                      rows, seq, scale, thr, ks, seed, offset, hl, hg, hoff);
  return launch_rows_nv<float, SoftmaxFwdL>(seq, rows, st, static_cast<const float*>(s), static_cast<float*>(p),
                                            static_cast<float*>(pd), rows, seq, scale, thr, ks, seed, offset, hl, hg, hoff);
}

cudaError_t softmax_bwd(int dtype, const void* p, const void* dpd, void* ds, long long batch, int seq, float scale,
                        float dropout_p, uint64_t seed, uint64_t offset, int hl, int hg, int hoff, cudaStream_t st) {
  const long long rows = batch * seq;
  const uint32_t thr = dropout_threshold(dropout_p);
  const float ks = dropout_p > 0.f ? 1.f / (1.f - dropout_p) : 1.f;
  const int use = dropout_p > 0.f ? 1 : 0;
  if (dtype == OASES_BF16)
    return launch_rows_nv<__nv_bfloat16, SoftmaxBwdL>(seq, rows, st, static_cast<const __nv_bfloat16*>(p),
                                                      static_cast<const __nv_bfloat16*>(dpd),
                                                      static_cast<__nv_bfloat16*>(ds), rows, seq, scale, thr, ks, use,
                                                      seed, offset, hl, hg, hoff);
  return launch_rows_nv<float, SoftmaxBwdL>(seq, rows, st, static_cast<const float*>(p), static_cast<const float*>(dpd),
                                            static_cast<float*>(ds), rows, seq, scale, thr, ks, use, seed, offset, hl, hg, hoff);
}

}  // namespace oases
