// Row-wise HBM-bound kernels: LayerNorm fwd/bwd and causal softmax fwd/bwd.
//
// One warp per row, 16-byte vector loads, warp-shuffle reductions, f32
// statistics. The reference restates none of these (its toy FFN has no LN and
// no attention, numerics.hpp:37-44); the fp64 oracle (oracle/gpt_oracle.cpp)
// defines their parity semantics.
#include <cstdlib>
#include "common.cuh"
#include "kernels.h"

namespace oases {
namespace {

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

// Register-cached variants: the row lives in NV 16-byte vectors per lane, so
// x (and dy) are read from HBM exactly once and the statistics are exact
// two-pass (mean, then centred variance) in f32.
template <typename T, int NV>
__global__ void __launch_bounds__(256) ln_fwd_cached_kernel(const T* __restrict__ x, const T* __restrict__ gamma,
                                                            const T* __restrict__ beta, T* __restrict__ y,
                                                            long long rows, int cols, float eps) {
  constexpr int V = Vec<T>::N;
  const long long row = static_cast<long long>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  if (row >= rows) return;
  const int lane = threadIdx.x & 31;
  const T* xr = x + row * cols;
  float v[NV][V];
  float sum = 0.f;
#pragma unroll
  for (int t = 0; t < NV; ++t) {
    const int c = (t * 32 + lane) * V;
    if (c < cols) {
      vload(xr + c, v[t]);
#pragma unroll
      for (int e = 0; e < V; ++e) sum += v[t][e];
    }
  }
  const float mean = warp_sum(sum) / static_cast<float>(cols);
  float var = 0.f;
#pragma unroll
  for (int t = 0; t < NV; ++t)
    if ((t * 32 + lane) * V < cols)
#pragma unroll
      for (int e = 0; e < V; ++e) var += (v[t][e] - mean) * (v[t][e] - mean);
  const float rstd = rsqrtf(warp_sum(var) / static_cast<float>(cols) + eps);
  T* yr = y + row * cols;
#pragma unroll
  for (int t = 0; t < NV; ++t) {
    const int c = (t * 32 + lane) * V;
    if (c >= cols) continue;
    float g[V], b[V];
    vload(gamma + c, g);
    vload(beta + c, b);
#pragma unroll
    for (int e = 0; e < V; ++e) v[t][e] = (v[t][e] - mean) * rstd * g[e] + b[e];
    vstore(yr + c, v[t]);
  }
}

template <typename T, int NV>
__global__ void __launch_bounds__(256) ln_bwd_cached_kernel(const T* __restrict__ x, const T* __restrict__ gamma,
                                                            const T* __restrict__ dy, T* __restrict__ dx, int acc,
                                                            float2* __restrict__ stats, long long rows, int cols,
                                                            float eps) {
  constexpr int V = Vec<T>::N;
  const long long row = static_cast<long long>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  if (row >= rows) return;
  const int lane = threadIdx.x & 31;
  const T* xr = x + row * cols;
  const T* dyr = dy + row * cols;
  float xv[NV][V], gv[NV][V];
  float sum = 0.f;
#pragma unroll
  for (int t = 0; t < NV; ++t) {
    const int c = (t * 32 + lane) * V;
    if (c < cols) {
      vload(xr + c, xv[t]);
      float d[V], g[V];
      vload(dyr + c, d);
      vload(gamma + c, g);
#pragma unroll
      for (int e = 0; e < V; ++e) {
        sum += xv[t][e];
        gv[t][e] = d[e] * g[e];
      }
    }
  }
  const float mean = warp_sum(sum) / static_cast<float>(cols);
  float var = 0.f;
#pragma unroll
  for (int t = 0; t < NV; ++t)
    if ((t * 32 + lane) * V < cols)
#pragma unroll
      for (int e = 0; e < V; ++e) var += (xv[t][e] - mean) * (xv[t][e] - mean);
  const float rstd = rsqrtf(warp_sum(var) / static_cast<float>(cols) + eps);
  float s1 = 0.f, s2 = 0.f;
#pragma unroll
  for (int t = 0; t < NV; ++t)
    if ((t * 32 + lane) * V < cols)
#pragma unroll
      for (int e = 0; e < V; ++e) {
        xv[t][e] = (xv[t][e] - mean) * rstd;  // xhat
        s1 += gv[t][e];
        s2 += gv[t][e] * xv[t][e];
      }
  s1 = warp_sum(s1) / static_cast<float>(cols);
  s2 = warp_sum(s2) / static_cast<float>(cols);
  if (lane == 0) stats[row] = make_float2(mean, rstd);
  T* dxr = dx + row * cols;
#pragma unroll
  for (int t = 0; t < NV; ++t) {
    const int c = (t * 32 + lane) * V;
    if (c >= cols) continue;
    float o[V];
    if (acc) vload(dxr + c, o);
#pragma unroll
    for (int e = 0; e < V; ++e) {
      const float r = rstd * (gv[t][e] - s1 - xv[t][e] * s2);
      o[e] = acc ? o[e] + r : r;
    }
    vstore(dxr + c, o);
  }
}

// Block-per-row variants (256 threads, NVEC 16-byte vectors per thread, cols ==
// 256 * V * NVEC): every thread holds a few vectors, so residency is high and
// the loads of many rows are in flight at once. Statistics are exact two-pass
// in f32 with fixed-order block reductions.
template <int N>
__device__ __forceinline__ void block_sum(float (&v)[N], float* sm) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int i = 0; i < N; ++i) v[i] = warp_sum(v[i]);
  if (lane == 0)
#pragma unroll
    for (int i = 0; i < N; ++i) sm[warp * N + i] = v[i];
  __syncthreads();
#pragma unroll
  for (int i = 0; i < N; ++i) {
    float t = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += sm[w * N + i];
    v[i] = t;
  }
  __syncthreads();
}

template <typename T, int NVEC, int R>
__global__ void __launch_bounds__(256) ln_fwd_block_kernel(const T* __restrict__ x, const T* __restrict__ gamma,
                                                           const T* __restrict__ beta, T* __restrict__ y, long long rows,
                                                           int cols, float eps) {
  constexpr int V = Vec<T>::N;
  __shared__ float sm[8 * R];
  const long long row0 = static_cast<long long>(blockIdx.x) * R;
  float v[R][NVEC][V], g[NVEC][V], b[NVEC][V];
#pragma unroll
  for (int t = 0; t < NVEC; ++t) {
    const int c = (t * 256 + threadIdx.x) * V;
    vload(gamma + c, g[t]);
    vload(beta + c, b[t]);
#pragma unroll
    for (int k = 0; k < R; ++k) {
      if (row0 + k < rows) vload(x + (row0 + k) * cols + c, v[k][t]);
      else
#pragma unroll
        for (int e = 0; e < V; ++e) v[k][t][e] = 0.f;
    }
  }
  float s[R];
#pragma unroll
  for (int k = 0; k < R; ++k) {
    s[k] = 0.f;
#pragma unroll
    for (int t = 0; t < NVEC; ++t)
#pragma unroll
      for (int e = 0; e < V; ++e) s[k] += v[k][t][e];
  }
  block_sum<R>(s, sm);
  float mean[R], q[R];
#pragma unroll
  for (int k = 0; k < R; ++k) {
    mean[k] = s[k] / static_cast<float>(cols);
    q[k] = 0.f;
#pragma unroll
    for (int t = 0; t < NVEC; ++t)
#pragma unroll
      for (int e = 0; e < V; ++e) q[k] += (v[k][t][e] - mean[k]) * (v[k][t][e] - mean[k]);
  }
  block_sum<R>(q, sm);
#pragma unroll
  for (int k = 0; k < R; ++k) {
    if (row0 + k >= rows) continue;
    const float rstd = rsqrtf(q[k] / static_cast<float>(cols) + eps);
#pragma unroll
    for (int t = 0; t < NVEC; ++t) {
#pragma unroll
      for (int e = 0; e < V; ++e) v[k][t][e] = (v[k][t][e] - mean[k]) * rstd * g[t][e] + b[t][e];
      vstore(y + (row0 + k) * cols + (t * 256 + threadIdx.x) * V, v[k][t]);
    }
  }
}

// DROP: also writes gout = dropout'(dx) (the hidden-dropout gradient of the
// bias-dropout-residual backward, computed from the stored bf16 dx exactly as
// the separate column pass would), saving that pass's re-read of dx.
template <typename T, int NVEC, int R, bool DROP = false>
__global__ void __launch_bounds__(256) ln_bwd_block_kernel(const T* __restrict__ x, const T* __restrict__ gamma,
                                                           const T* __restrict__ dy, T* __restrict__ dx, int acc,
                                                           float2* __restrict__ stats, long long rows, int cols,
                                                           float eps, T* __restrict__ gout = nullptr,
                                                           uint32_t thr = 0, float ks = 1.f, uint64_t seed = 0,
                                                           uint64_t offset = 0,
                                                           const uint16_t* __restrict__ keep_bits = nullptr) {
  if constexpr (DROP) {
    pdl_trigger();
    pdl_wait();
  }
  constexpr int V = Vec<T>::N;
  __shared__ float sm[16 * R];
  const long long row0 = static_cast<long long>(blockIdx.x) * R;
  float xv[R][NVEC][V], gv[R][NVEC][V], o[R][NVEC][V];
#pragma unroll
  for (int t = 0; t < NVEC; ++t) {
    const int c = (t * 256 + threadIdx.x) * V;
    float g[V];
    vload(gamma + c, g);
#pragma unroll
    for (int k = 0; k < R; ++k) {
      float d[V];
      if (row0 + k < rows) {
        vload(x + (row0 + k) * cols + c, xv[k][t]);
        vload(dy + (row0 + k) * cols + c, d);
        if (acc) vload(dx + (row0 + k) * cols + c, o[k][t]);
      } else {
#pragma unroll
        for (int e = 0; e < V; ++e) xv[k][t][e] = d[e] = 0.f;
      }
#pragma unroll
      for (int e = 0; e < V; ++e) gv[k][t][e] = d[e] * g[e];
    }
  }
  float s[R];
#pragma unroll
  for (int k = 0; k < R; ++k) {
    s[k] = 0.f;
#pragma unroll
    for (int t = 0; t < NVEC; ++t)
#pragma unroll
      for (int e = 0; e < V; ++e) s[k] += xv[k][t][e];
  }
  block_sum<R>(s, sm);
  float mean[R], q[R];
#pragma unroll
  for (int k = 0; k < R; ++k) {
    mean[k] = s[k] / static_cast<float>(cols);
    q[k] = 0.f;
#pragma unroll
    for (int t = 0; t < NVEC; ++t)
#pragma unroll
      for (int e = 0; e < V; ++e) q[k] += (xv[k][t][e] - mean[k]) * (xv[k][t][e] - mean[k]);
  }
  block_sum<R>(q, sm);
  float rstd[R], s12[2 * R];
#pragma unroll
  for (int k = 0; k < R; ++k) {
    rstd[k] = rsqrtf(q[k] / static_cast<float>(cols) + eps);
    s12[2 * k] = 0.f;
    s12[2 * k + 1] = 0.f;
#pragma unroll
    for (int t = 0; t < NVEC; ++t)
#pragma unroll
      for (int e = 0; e < V; ++e) {
        xv[k][t][e] = (xv[k][t][e] - mean[k]) * rstd[k];  // xhat
        s12[2 * k] += gv[k][t][e];
        s12[2 * k + 1] += gv[k][t][e] * xv[k][t][e];
      }
  }
  block_sum<2 * R>(s12, sm);
#pragma unroll
  for (int k = 0; k < R; ++k) {
    if (row0 + k >= rows) continue;
    const float m1 = s12[2 * k] / static_cast<float>(cols), m2 = s12[2 * k + 1] / static_cast<float>(cols);
    if (threadIdx.x == 0) stats[row0 + k] = make_float2(mean[k], rstd[k]);
#pragma unroll
    for (int t = 0; t < NVEC; ++t) {
#pragma unroll
      for (int e = 0; e < V; ++e) {
        const float r = rstd[k] * (gv[k][t][e] - m1 - xv[k][t][e] * m2);
        o[k][t][e] = acc ? o[k][t][e] + r : r;
      }
      const long long off = (row0 + k) * cols + (t * 256 + threadIdx.x) * V;
      vstore(dx + off, o[k][t]);
      if constexpr (DROP) {
        if constexpr (sizeof(T) == 2) {  // what a re-read of the stored dx sees
#pragma unroll
          for (int e = 0; e < V; ++e) o[k][t][e] = __bfloat162float(__float2bfloat16_rn(o[k][t][e]));
        }
        if (keep_bits) {  // decisions cached by the forward pass
          const uint32_t bits = keep_bits[off >> 4] >> (off & 15);
#pragma unroll
          for (int e = 0; e < V; ++e) o[k][t][e] = (bits >> e) & 1u ? o[k][t][e] * ks : 0.f;
        } else {
          apply_dropout<V>(o[k][t], static_cast<unsigned long long>(off), seed, offset, thr, ks);
        }
        vstore(gout + off, o[k][t]);
      }
    }
  }
}

// LN parameter-gradient partials with 16-column lanes: one warp per block
// covers 512 columns over a chunk of rows (2 rows in flight); no shared
// memory, so it co-resides with the persistent GEMMs on the side stream.
// part[chunk][0][c] = sum dy * xhat, part[chunk][1][c] = sum dy.
template <typename T>
__global__ void __launch_bounds__(32) ln_param16_kernel(const T* __restrict__ x, const T* __restrict__ dy,
                                                        const float2* __restrict__ stats, float* __restrict__ part,
                                                        long long rows, int cols, int rows_per_chunk) {
  pdl_trigger();
  pdl_wait();
  const int lane = threadIdx.x;
  const int c = blockIdx.x * 512 + lane * 16;
  if (c >= cols) return;
  const long long r0 = static_cast<long long>(blockIdx.y) * rows_per_chunk;
  const long long r1 = r0 + rows_per_chunk < rows ? r0 + rows_per_chunk : rows;
  float sg[16] = {}, sb[16] = {};
  long long r = r0;
  for (; r + 1 < r1; r += 2) {  // 2 rows in flight
    float d[2][16], xv[2][16];
    float2 st[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      load16(dy + (r + u) * cols + c, d[u]);
      load16(x + (r + u) * cols + c, xv[u]);
      st[u] = stats[r + u];
    }
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        sg[e] += d[u][e] * (xv[u][e] - st[u].x) * st[u].y;
        sb[e] += d[u][e];
      }
  }
  for (; r < r1; ++r) {
    float d[16], xv[16];
    load16(dy + r * cols + c, d);
    load16(x + r * cols + c, xv);
    const float2 st = stats[r];
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      sg[e] += d[e] * (xv[e] - st.x) * st.y;
      sb[e] += d[e];
    }
  }
  float* p0 = part + (static_cast<long long>(blockIdx.y) * 2 + 0) * cols + c;
  float* p1 = part + (static_cast<long long>(blockIdx.y) * 2 + 1) * cols + c;
#pragma unroll
  for (int q = 0; q < 16; q += 4) {
    *reinterpret_cast<float4*>(p0 + q) = make_float4(sg[q], sg[q + 1], sg[q + 2], sg[q + 3]);
    *reinterpret_cast<float4*>(p1 + q) = make_float4(sb[q], sb[q + 1], sb[q + 2], sb[q + 3]);
  }
}

// out0/out1[c] (+)= sum_k part[k][0/1][c]: 32 columns x 8 chunk lanes per
// block, group g sums chunks g, g+8, ... (2x2 loads in flight), group sums
// combined in g order (fixed order, bit-reproducible).
__global__ void __launch_bounds__(256) colpair_finalize_fast_kernel(const float* __restrict__ part, int chunks,
                                                                    int cols, float* __restrict__ out0,
                                                                    float* __restrict__ out1, int acc) {
  pdl_trigger();
  pdl_wait();
  __shared__ float sm[2][8][33];
  const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + lane;
  float ta = 0.f, tb = 0.f;
  if (c < cols) {
    int k = g;
    for (; k + 8 < chunks; k += 16) {
      float a[2], b[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        a[u] = __ldg(part + (static_cast<long long>(k + 8 * u) * 2 + 0) * cols + c);
        b[u] = __ldg(part + (static_cast<long long>(k + 8 * u) * 2 + 1) * cols + c);
      }
      ta += a[0];
      ta += a[1];
      tb += b[0];
      tb += b[1];
    }
    for (; k < chunks; k += 8) {
      ta += __ldg(part + (static_cast<long long>(k) * 2 + 0) * cols + c);
      tb += __ldg(part + (static_cast<long long>(k) * 2 + 1) * cols + c);
    }
  }
  sm[0][g][lane] = ta;
  sm[1][g][lane] = tb;
  __syncthreads();
  if (g == 0 && c < cols) {
    float sa = 0.f, sb = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      sa += sm[0][j][lane];
      sb += sm[1][j][lane];
    }
    if (out0) out0[c] = acc ? out0[c] + sa : sa;
    if (out1) out1[c] = acc ? out1[c] + sb : sb;
  }
}

// Column partial sums over a chunk of rows: part[chunk][0][c] = sum dy*xhat,
// part[chunk][1][c] = sum dy. Each thread owns V consecutive columns.
template <typename T>
__global__ void __launch_bounds__(256) ln_param_partial_kernel(const T* __restrict__ x, const T* __restrict__ dy,
                                                               const float2* __restrict__ stats, float* __restrict__ part,
                                                               long long rows, int cols, int rows_per_chunk) {
  constexpr int V = Vec<T>::N;
  const int c = (blockIdx.x * 256 + threadIdx.x) * V;
  if (c >= cols) return;
  const long long r0 = static_cast<long long>(blockIdx.y) * rows_per_chunk;
  const long long r1 = r0 + rows_per_chunk < rows ? r0 + rows_per_chunk : rows;
  float sg[V] = {}, sb[V] = {};
  for (long long r = r0; r < r1; ++r) {
    const float2 st = stats[r];
    float d[V], xv[V];
    vload(dy + r * cols + c, d);
    vload(x + r * cols + c, xv);
#pragma unroll
    for (int e = 0; e < V; ++e) {
      sg[e] += d[e] * (xv[e] - st.x) * st.y;
      sb[e] += d[e];
    }
  }
  float* p0 = part + (static_cast<long long>(blockIdx.y) * 2 + 0) * cols + c;
  float* p1 = part + (static_cast<long long>(blockIdx.y) * 2 + 1) * cols + c;
#pragma unroll
  for (int e = 0; e < V; ++e) {
    p0[e] = sg[e];
    p1[e] = sb[e];
  }
}

// out0/out1[c] (+)= sum_k part[k][0/1][c] in a fixed order (8 interleaved
// partial sums per column combined in index order).
__global__ void __launch_bounds__(256) colpair_finalize_kernel(const float* __restrict__ part, int chunks, int cols,
                                                               float* __restrict__ out0, float* __restrict__ out1,
                                                               int acc) {
  __shared__ float sm[2][8][33];
  const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + lane;
  float a = 0.f, b = 0.f;
  if (c < cols)
    for (int k = g; k < chunks; k += 8) {
      a += part[(static_cast<long long>(k) * 2 + 0) * cols + c];
      b += part[(static_cast<long long>(k) * 2 + 1) * cols + c];
    }
  sm[0][g][lane] = a;
  sm[1][g][lane] = b;
  __syncthreads();
  if (g == 0 && c < cols) {
    float ta = 0.f, tb = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      ta += sm[0][j][lane];
      tb += sm[1][j][lane];
    }
    if (out0) out0[c] = acc ? out0[c] + ta : ta;
    if (out1) out1[c] = acc ? out1[c] + tb : tb;
  }
}

// ------------------------------------------------------------------ softmax
// Row r of S (viewed [batch*seq, seq]) is query position i = r % seq; keys
// j <= i are valid. P = softmax(scale * S) over valid keys, zeros elsewhere.
// The row is cached in registers: NV vectors per lane.
// Dropout element index uses the GLOBAL head (head_offset + local head) so the
// mask does not depend on the TMP degree: row r = (n*Hl + jl)*seq + i maps to
// global row (n*Hg + head_offset + jl)*seq + i.
struct RowIdx {
  int i;                    // query position within the sequence
  unsigned long long ebase; // global element index of (row, 0) for the dropout key
};
__device__ __forceinline__ RowIdx row_index(unsigned row, int seq, int hl, int hg, int hoff) {
  const unsigned per = static_cast<unsigned>(hl) * static_cast<unsigned>(seq);
  const unsigned n = row / per, rem = row - n * per;
  const unsigned jl = rem / static_cast<unsigned>(seq), i = rem - jl * static_cast<unsigned>(seq);
  const unsigned long long grow =
      (static_cast<unsigned long long>(n) * hg + hoff + jl) * static_cast<unsigned long long>(seq) + i;
  return {static_cast<int>(i), grow * static_cast<unsigned long long>(seq)};
}

template <typename T, int NV>
__global__ void __launch_bounds__(256) softmax_fwd_kernel(const T* __restrict__ s, T* __restrict__ p,
                                                          T* __restrict__ pd, long long rows, int seq, float scale,
                                                          uint32_t thr, float keep_scale, uint64_t seed,
                                                          uint64_t offset, int hl, int hg, int hoff) {
  constexpr int V = Vec<T>::N;
  const unsigned row = blockIdx.x * 8u + (threadIdx.x >> 5);
  if (row >= rows) return;
  const int lane = threadIdx.x & 31;
  const RowIdx ri = row_index(row, seq, hl, hg, hoff);
  const int i = ri.i;
  const size_t roff = static_cast<size_t>(row) * seq;
  const T* sr = s + roff;
  const float sl2 = scale * 1.44269504088896341f;  // exp(x*scale) = exp2(x*scale*log2 e)
  float v[NV][V];
  float mx = -INFINITY;
#pragma unroll
  for (int t = 0; t < NV; ++t) {
    const int c = (t * 32 + lane) * V;
    if (c <= i) {  // c <= i < seq
      vload(sr + c, v[t]);
#pragma unroll
      for (int e = 0; e < V; ++e) {
        v[t][e] = (c + e <= i) ? v[t][e] * sl2 : -INFINITY;
        mx = fmaxf(mx, v[t][e]);
      }
    }
  }
  mx = warp_max(mx);
  float sum = 0.f;
#pragma unroll
  for (int t = 0; t < NV; ++t) {
    const int c = (t * 32 + lane) * V;
    if (c <= i) {
#pragma unroll
      for (int e = 0; e < V; ++e) {
        v[t][e] = exp2f(v[t][e] - mx);  // exp2(-inf) = 0
        sum += v[t][e];
      }
    } else {
#pragma unroll
      for (int e = 0; e < V; ++e) v[t][e] = 0.f;
    }
  }
  sum = warp_sum(sum);
  const float inv = 1.f / sum;
  T* pr = p + roff;
  T* pdr = pd ? pd + roff : nullptr;
  // Only the band [0, round_up(i+1, 128)) is ever read by the causal P.V /
  // P^T.dO GEMMs (their K ranges stop at the 128-row tile edge), so the zero
  // tail beyond it is never written.
  const int band = min(seq, ((i + 128) / 128) * 128);
#pragma unroll
  for (int t = 0; t < NV; ++t) {
    const int c = (t * 32 + lane) * V;
    if (c >= band) continue;
#pragma unroll
    for (int e = 0; e < V; ++e) v[t][e] *= inv;
    vstore(pr + c, v[t]);
    if (pdr) {
      if (c <= i) apply_dropout<V>(v[t], ri.ebase + c, seed, offset, thr, keep_scale);
      vstore(pdr + c, v[t]);  // beyond i: zeros, no mask needed
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
  const unsigned row = blockIdx.x * 8u + (threadIdx.x >> 5);
  if (row >= rows) return;
  const int lane = threadIdx.x & 31;
  const RowIdx ri = row_index(row, seq, hl, hg, hoff);
  const int i = ri.i;
  const size_t roff = static_cast<size_t>(row) * seq;
  float pv[NV][V], dv[NV][V];
  float dot = 0.f;
#pragma unroll
  for (int t = 0; t < NV; ++t) {
    const int c = (t * 32 + lane) * V;
    if (c <= i) {
      vload(p + roff + c, pv[t]);
      vload(dpd + roff + c, dv[t]);
      if (use_dropout) apply_dropout<V>(dv[t], ri.ebase + c, seed, offset, thr, keep_scale);
#pragma unroll
      for (int e = 0; e < V; ++e) {
        if (c + e > i) dv[t][e] = 0.f;  // P is 0 there; dP_drop may be unwritten
        dot += pv[t][e] * dv[t][e];
      }
    } else {
#pragma unroll
      for (int e = 0; e < V; ++e) { pv[t][e] = 0.f; dv[t][e] = 0.f; }
    }
  }
  dot = warp_sum(dot);
  const int band = min(seq, ((i + 128) / 128) * 128);  // see softmax_fwd_kernel
#pragma unroll
  for (int t = 0; t < NV; ++t) {
    const int c = (t * 32 + lane) * V;
    if (c >= band) continue;
#pragma unroll
    for (int e = 0; e < V; ++e) pv[t][e] = scale * pv[t][e] * (dv[t][e] - dot);
    vstore(ds + roff + c, pv[t]);
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

template <typename T, int NV>
struct LnFwdL {
  template <typename... A>
  static void launch(unsigned grid, cudaStream_t st, A... a) {
    ln_fwd_cached_kernel<T, NV><<<grid, 256, 0, st>>>(a...);
  }
};
template <typename T, int NV>
struct LnBwdL {
  template <typename... A>
  static void launch(unsigned grid, cudaStream_t st, A... a) {
    ln_bwd_cached_kernel<T, NV><<<grid, 256, 0, st>>>(a...);
  }
};

// (column blocks) x (row chunks) ~ 4 CTAs per SM
struct ParamSplit {
  int col_blocks, chunks, rows_per_chunk;
};
template <typename T>
ParamSplit param_split(long long rows, int cols) {
  constexpr int V = Vec<T>::N;
  const int cb = (cols + 256 * V - 1) / (256 * V);
  long long chunks = (4LL * 148 + cb - 1) / cb;
  if (chunks > rows) chunks = rows;
  if (chunks < 1) chunks = 1;
  const int rpc = static_cast<int>((rows + chunks - 1) / chunks);
  return {cb, static_cast<int>((rows + rpc - 1) / rpc), rpc};
}

// (512-column groups) x (row chunks): ~8 single-warp CTAs per SM, >= 8 rows per chunk
ParamSplit param_split16(long long rows, int cols) {
  const int groups = (cols + 511) / 512;
  long long chunks = (8LL * 148 + groups - 1) / groups;
  const long long maxc = (rows + 7) / 8;
  if (chunks > maxc) chunks = maxc;
  if (chunks < 1) chunks = 1;
  const int rpc = static_cast<int>((rows + chunks - 1) / chunks);
  return {groups, static_cast<int>((rows + rpc - 1) / rpc), rpc};
}

// NVEC for the block-per-row kernels (0 = not applicable)
template <typename T>
int block_nvec(int cols) {
  constexpr int V = Vec<T>::N;
  if (cols % (256 * V)) return 0;
  const int n = cols / (256 * V);
  return (n == 1 || n == 2 || n == 4) ? n : 0;
}

// which: 1 = dx (+ row statistics into the workspace), 2 = dgamma/dbeta from
// those statistics, 3 = both. Splitting lets the parameter reduction run on a
// side stream under the next GEMMs (its outputs are only needed at step end).
// NV for the row-group kernel (0: shape not covered -> older kernels).
inline int ln_rows_nv(int cols) {
  if (cols % 16) return 0;
  for (int nv = 1; nv <= 4; nv *= 2) {
    const int v = cols / 16;
    if (v % nv) return 0;
    const int tpr = v / nv;
    if (tpr <= 256 && tpr >= 32 && tpr % 32 == 0) return nv;
  }
  return 0;
}

template <typename T>
cudaError_t ln_bwd_t(const void* x, const void* gamma, const void* dy, void* dx, int acc_dx, float* dgamma,
                     float* dbeta, int acc_params, void* workspace, long long rows, int cols, float eps,
                     cudaStream_t st, int which = 3, void* gout = nullptr, float drop_p = 0.f, uint64_t seed = 0,
                     uint64_t offset = 0, const uint16_t* keep_bits = nullptr) {
  float2* stats = static_cast<float2*>(workspace);
  float* part = reinterpret_cast<float*>(static_cast<char*>(workspace) +
                                         ((static_cast<size_t>(rows) * sizeof(float2) + 255) & ~size_t(255)));
  auto X = static_cast<const T*>(x);
  auto DY = static_cast<const T*>(dy);
  auto G = static_cast<const T*>(gamma);
  auto DX = static_cast<T*>(dx);
  const unsigned grid = static_cast<unsigned>((rows + 7) / 8);
  const int nvec = block_nvec<T>(cols);
  if (!(which & 1)) {
    // parameter pass only
  } else if (gout) {
    // fused dropout output: the block-per-row kernel (one row of 256 threads, 8
    // elements each; measured faster than the row-group geometry backward)
    if (!nvec || rows >= (1LL << 31)) return cudaErrorNotSupported;
    const uint32_t thr = dropout_threshold(drop_p);
    const float ks = dropout_keep_scale(drop_p);
    T* GO = static_cast<T*>(gout);
    const dim3 gr(static_cast<unsigned>(rows));
    if (nvec == 1)
      launch_pdl(ln_bwd_block_kernel<T, 1, 1, true>, gr, dim3(256), 0, st, X, G, DY, DX, acc_dx, stats, rows, cols,
                 eps, GO, thr, ks, seed, offset, keep_bits);
    else if (nvec == 2)
      launch_pdl(ln_bwd_block_kernel<T, 2, 1, true>, gr, dim3(256), 0, st, X, G, DY, DX, acc_dx, stats, rows, cols,
                 eps, GO, thr, ks, seed, offset, keep_bits);
    else
      launch_pdl(ln_bwd_block_kernel<T, 4, 1, true>, gr, dim3(256), 0, st, X, G, DY, DX, acc_dx, stats, rows, cols,
                 eps, GO, thr, ks, seed, offset, keep_bits);
  } else if (nvec && rows < (1LL << 31)) {
    // one row per block (measured faster than 2 for the backward)
    if (nvec == 1)
      ln_bwd_block_kernel<T, 1, 1><<<static_cast<unsigned>(rows), 256, 0, st>>>(X, G, DY, DX, acc_dx, stats, rows,
                                                                                cols, eps);
    else if (nvec == 2)
      ln_bwd_block_kernel<T, 2, 1><<<static_cast<unsigned>(rows), 256, 0, st>>>(X, G, DY, DX, acc_dx, stats, rows,
                                                                                cols, eps);
    else
      ln_bwd_block_kernel<T, 4, 1><<<static_cast<unsigned>(rows), 256, 0, st>>>(X, G, DY, DX, acc_dx, stats, rows,
                                                                                cols, eps);
  } else if (cols <= 16 * 32 * Vec<T>::N) {
    const cudaError_t e = launch_rows_nv<T, LnBwdL>(cols, rows, st, X, G, DY, DX, acc_dx, stats, rows, cols, eps);
    if (e != cudaSuccess) return e;
  } else {
    ln_bwd_kernel<T><<<grid, 256, 0, st>>>(X, G, DY, DX, acc_dx, stats, rows, cols, eps);
  }
  if ((which & 2) && (dgamma || dbeta)) {
    if (cols % 16 == 0) {
      const ParamSplit sp = param_split16(rows, cols);
      launch_pdl(ln_param16_kernel<T>, dim3(sp.col_blocks, sp.chunks), dim3(32), 0, st, X, DY,
                 static_cast<const float2*>(stats), part, rows, cols, sp.rows_per_chunk);
      launch_pdl(colpair_finalize_fast_kernel, dim3((cols + 31) / 32), dim3(256), 0, st,
                 static_cast<const float*>(part), sp.chunks, cols, dgamma, dbeta, acc_params);
    } else {
      const ParamSplit sp = param_split<T>(rows, cols);
      ln_param_partial_kernel<T><<<dim3(sp.col_blocks, sp.chunks), 256, 0, st>>>(X, DY, stats, part, rows, cols,
                                                                                 sp.rows_per_chunk);
      colpair_finalize_kernel<<<(cols + 31) / 32, 256, 0, st>>>(part, sp.chunks, cols, dgamma, dbeta, acc_params);
    }
  }
  return cudaGetLastError();
}

// Row-group LayerNorm forward: TPR = cols / (16 NV) threads per row, 16 NV
// consecutive-by-16 elements per thread (one Philox dropout counter per 16),
// RB = 256 / TPR rows per 256-thread block; exact two-pass f32 statistics with
// fixed-order reductions. BDR fuses the producing bias-dropout-residual
// (x = res + dropout(in + bias), the bdr_fwd16 arithmetic in the same order)
// and stores x: HBM traffic read in+res / write x+y instead of a separate
// bias-dropout-residual pass plus a re-read of x. The plain and fused variants
// share every f32 operation of the normalisation, so LN(x) is bit-identical
// whichever kernel produced x (Oases recompute == CrossPass replay).
template <typename T, int NV, bool BDR>
__global__ void __launch_bounds__(256) ln_rows_kernel(const T* __restrict__ in, const T* __restrict__ bias,
                                                      const T* __restrict__ res, T* __restrict__ xout,
                                                      const T* __restrict__ gamma, const T* __restrict__ beta,
                                                      T* __restrict__ y, long long rows, int cols, float eps,
                                                      uint32_t thr, float ks, int drop, uint64_t seed,
                                                      uint64_t offset, uint16_t* __restrict__ keep_bits) {
  pdl_trigger();
  pdl_wait();
  __shared__ float sm[2][8][8];  // [statistic][row of the block][warp of the row]
  const int tpr = cols / (16 * NV), rb = 256 / tpr, wpr = tpr / 32;
  const int sub = threadIdx.x / tpr, t = threadIdx.x - sub * tpr, wi = t >> 5;
  const long long row = static_cast<long long>(blockIdx.x) * rb + sub;
  const bool ok = row < rows;
  const long long base = row * cols;
  float v[NV][16];
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const int c = (k * tpr + t) * 16;
    if (!ok) {
#pragma unroll
      for (int e = 0; e < 16; ++e) v[k][e] = 0.f;
      continue;
    }
    load16(in + base + c, v[k]);
    if constexpr (BDR) {
      if (bias) {
        float b[16];
        load16(bias + c, b);
#pragma unroll
        for (int e = 0; e < 16; ++e) v[k][e] += b[e];
      }
      if (drop) {
        // one Philox call for the 16 elements; the keep decisions optionally
        // cached (1 bit each) for the backward's dropout gradient
        uint32_t u[4];
        Philox::gen(seed, offset, static_cast<unsigned long long>(base + c) >> 4, u);
        uint32_t bits = 0;
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const bool kp = keep_byte(u, q, thr);
          v[k][q] = kp ? v[k][q] * ks : 0.f;
          bits |= static_cast<uint32_t>(kp) << q;
        }
        if (keep_bits) keep_bits[(base + c) >> 4] = static_cast<uint16_t>(bits);
      }
      if (res) {
        float r[16];
        load16(res + base + c, r);
#pragma unroll
        for (int e = 0; e < 16; ++e) v[k][e] += r[e];
      }
      store16(xout + base + c, v[k]);
      if constexpr (sizeof(T) == 2) {  // normalise the stored (rounded) x, exactly what a re-read would see
#pragma unroll
        for (int e = 0; e < 16; ++e) v[k][e] = __bfloat162float(__float2bfloat16_rn(v[k][e]));
      }
    }
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < NV; ++k)
#pragma unroll
    for (int e = 0; e < 16; ++e) s += v[k][e];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) sm[0][sub][wi] = s;
  __syncthreads();
  s = 0.f;
  for (int w = 0; w < wpr; ++w) s += sm[0][sub][w];
  const float mean = s / static_cast<float>(cols);
  float q = 0.f;
#pragma unroll
  for (int k = 0; k < NV; ++k)
#pragma unroll
    for (int e = 0; e < 16; ++e) q += (v[k][e] - mean) * (v[k][e] - mean);
  q = warp_sum(q);
  if ((threadIdx.x & 31) == 0) sm[1][sub][wi] = q;
  __syncthreads();
  q = 0.f;
  for (int w = 0; w < wpr; ++w) q += sm[1][sub][w];
  if (!ok) return;
  const float rstd = rsqrtf(q / static_cast<float>(cols) + eps);
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const int c = (k * tpr + t) * 16;
    float g[16], b[16];
    load16(gamma + c, g);
    load16(beta + c, b);
#pragma unroll
    for (int e = 0; e < 16; ++e) v[k][e] = (v[k][e] - mean) * rstd * g[e] + b[e];
    store16(y + base + c, v[k]);
  }
}

template <typename T, bool BDR>
cudaError_t ln_rows_launch(const void* in, const void* bias, const void* res, void* xout, const void* gamma,
                           const void* beta, void* y, long long rows, int cols, float eps, float p, uint64_t seed,
                           uint64_t offset, cudaStream_t st, uint16_t* keep_bits = nullptr) {
  const int nv = ln_rows_nv(cols);
  if (!nv || rows >= (1LL << 31) * 4) return cudaErrorNotSupported;
  const int rb = 256 / (cols / (16 * nv));
  const unsigned grid = static_cast<unsigned>((rows + rb - 1) / rb);
  const uint32_t thr = dropout_threshold(p);
  const float ks = dropout_keep_scale(p);
  const int drop = p > 0.f;
  auto I = static_cast<const T*>(in);
  auto Bi = static_cast<const T*>(bias);
  auto R = static_cast<const T*>(res);
  auto X = static_cast<T*>(xout);
  auto G = static_cast<const T*>(gamma);
  auto Be = static_cast<const T*>(beta);
  auto Y = static_cast<T*>(y);
  switch (nv) {
    case 1: launch_pdl(ln_rows_kernel<T, 1, BDR>, dim3(grid), dim3(256), 0, st, I, Bi, R, X, G, Be, Y, rows, cols, eps, thr, ks, drop, seed, offset, keep_bits); break;
    case 2: launch_pdl(ln_rows_kernel<T, 2, BDR>, dim3(grid), dim3(256), 0, st, I, Bi, R, X, G, Be, Y, rows, cols, eps, thr, ks, drop, seed, offset, keep_bits); break;
    default: launch_pdl(ln_rows_kernel<T, 4, BDR>, dim3(grid), dim3(256), 0, st, I, Bi, R, X, G, Be, Y, rows, cols, eps, thr, ks, drop, seed, offset, keep_bits); break;
  }
  return cudaGetLastError();
}

template <typename T>
cudaError_t ln_fwd_t(const void* x, const void* gamma, const void* beta, void* y, long long rows, int cols, float eps,
                     cudaStream_t st) {
  auto X = static_cast<const T*>(x);
  auto G = static_cast<const T*>(gamma);
  auto B = static_cast<const T*>(beta);
  auto Y = static_cast<T*>(y);
  if (ln_rows_nv(cols) && rows < (1LL << 31))
    return ln_rows_launch<T, false>(x, nullptr, nullptr, nullptr, gamma, beta, y, rows, cols, eps, 0.f, 0, 0, st);
  const int nvec = block_nvec<T>(cols);
  if (nvec && rows < (1LL << 31)) {
    if (nvec == 1)
      ln_fwd_block_kernel<T, 1, 4><<<static_cast<unsigned>((rows + 3) / 4), 256, 0, st>>>(X, G, B, Y, rows, cols, eps);
    else if (nvec == 2)
      ln_fwd_block_kernel<T, 2, 2><<<static_cast<unsigned>((rows + 1) / 2), 256, 0, st>>>(X, G, B, Y, rows, cols, eps);
    else
      ln_fwd_block_kernel<T, 4, 1><<<static_cast<unsigned>(rows), 256, 0, st>>>(X, G, B, Y, rows, cols, eps);
    return cudaGetLastError();
  }
  if (cols <= 16 * 32 * Vec<T>::N) return launch_rows_nv<T, LnFwdL>(cols, rows, st, X, G, B, Y, rows, cols, eps);
  ln_fwd_kernel<T><<<static_cast<unsigned>((rows + 7) / 8), 256, 0, st>>>(X, G, B, Y, rows, cols, eps);
  return cudaGetLastError();
}

}  // namespace

size_t layernorm_bwd_workspace(long long rows, int cols) {
  const ParamSplit a = param_split<float>(rows, cols), b = param_split<__nv_bfloat16>(rows, cols);
  long long chunks = a.chunks > b.chunks ? a.chunks : b.chunks;
  if (param_split16(rows, cols).chunks > chunks) chunks = param_split16(rows, cols).chunks;
  // the persistent kernel's [prows][3][cols] partials (rowpipe.cu)
  const long long lnp3 = 3 * lnp_partial_rows_max(rows, cols);
  if ((lnp3 + 1) / 2 > chunks) chunks = (lnp3 + 1) / 2;
  return ((static_cast<size_t>(rows) * sizeof(float2) + 255) & ~size_t(255)) +
         static_cast<size_t>(chunks) * 2 * cols * sizeof(float) + 256;
}

cudaError_t layernorm_fwd(int dtype, const void* x, const void* gamma, const void* beta, void* y, long long rows,
                          int cols, float eps, cudaStream_t st, int max_sms) {
  if (lnp_enabled() && lnp_supported(rows, cols))
    return lnp_layernorm_fwd(dtype, x, nullptr, nullptr, nullptr, gamma, beta, y, rows, cols, eps, 0.f, 0, 0, nullptr,
                             max_sms, st);
  if (dtype == OASES_BF16) return ln_fwd_t<__nv_bfloat16>(x, gamma, beta, y, rows, cols, eps, st);
  return ln_fwd_t<float>(x, gamma, beta, y, rows, cols, eps, st);
}

bool bdr_layernorm_supported(long long rows, int cols) {
  return (lnp_enabled() && lnp_supported(rows, cols)) || (ln_rows_nv(cols) && rows < (1LL << 31));
}

bool ln_bwd_dropout_supported(int dtype, long long rows, int cols) {
  const int nv = dtype == OASES_BF16 ? block_nvec<__nv_bfloat16>(cols) : block_nvec<float>(cols);
  return nv && rows < (1LL << 31);
}

cudaError_t bias_dropout_residual_layernorm_fwd(int dtype, const void* in, const void* bias, const void* res,
                                                void* xout, const void* gamma, const void* beta, void* y,
                                                long long rows, int cols, float eps, float p, uint64_t seed,
                                                uint64_t offset, cudaStream_t st, uint16_t* keep_bits, int max_sms) {
  if (lnp_enabled() && lnp_supported(rows, cols))
    return lnp_layernorm_fwd(dtype, in, bias, res, xout, gamma, beta, y, rows, cols, eps, p, seed, offset, keep_bits,
                             max_sms, st);
  if (!bdr_layernorm_supported(rows, cols)) return cudaErrorNotSupported;
  if (dtype == OASES_BF16)
    return ln_rows_launch<__nv_bfloat16, true>(in, bias, res, xout, gamma, beta, y, rows, cols, eps, p, seed, offset,
                                               st, keep_bits);
  return ln_rows_launch<float, true>(in, bias, res, xout, gamma, beta, y, rows, cols, eps, p, seed, offset, st,
                                     keep_bits);
}

cudaError_t layernorm_bwd_part(int which, int dtype, const void* x, const void* gamma, const void* dy, void* dx,
                               int acc_dx, float* dgamma, float* dbeta, int acc_params, void* workspace,
                               long long rows, int cols, float eps, cudaStream_t st, void* gout, float drop_p,
                               uint64_t seed, uint64_t offset, const uint16_t* keep_bits) {
  if (dtype == OASES_BF16)
    return ln_bwd_t<__nv_bfloat16>(x, gamma, dy, dx, acc_dx, dgamma, dbeta, acc_params, workspace, rows, cols, eps, st,
                                   which, gout, drop_p, seed, offset, keep_bits);
  return ln_bwd_t<float>(x, gamma, dy, dx, acc_dx, dgamma, dbeta, acc_params, workspace, rows, cols, eps, st, which,
                         gout, drop_p, seed, offset, keep_bits);
}

cudaError_t layernorm_bwd(int dtype, const void* x, const void* gamma, const void* dy, void* dx, int acc_dx,
                          float* dgamma, float* dbeta, int acc_params, void* workspace, long long rows, int cols,
                          float eps, cudaStream_t st, int max_sms) {
  if (lnp_enabled() && lnp_supported(rows, cols)) {
    // the persistent kernel: column partials of the parameter gradients in the workspace, then
    // one fixed-order finalize
    float* part = reinterpret_cast<float*>(static_cast<char*>(workspace) +
                                           ((static_cast<size_t>(rows) * sizeof(float2) + 255) & ~size_t(255)));
    const bool params = dgamma || dbeta;
    cudaError_t e = lnp_layernorm_bwd(dtype, x, gamma, dy, dx, acc_dx, nullptr, 0.f, 0, 0, nullptr,
                                      params ? part : nullptr, nullptr, rows, cols, eps, max_sms, st);
    if (e != cudaSuccess || !params) return e;
    return lnp_finalize(part, lnp_partial_rows(dtype, rows, cols, acc_dx, max_sms), cols, dgamma, dbeta, nullptr,
                        acc_params, acc_params, 0, st);
  }
  if (dtype == OASES_BF16)
    return ln_bwd_t<__nv_bfloat16>(x, gamma, dy, dx, acc_dx, dgamma, dbeta, acc_params, workspace, rows, cols, eps, st);
  return ln_bwd_t<float>(x, gamma, dy, dx, acc_dx, dgamma, dbeta, acc_params, workspace, rows, cols, eps, st);
}

cudaError_t softmax_fwd(int dtype, const void* s, void* p, void* pd, long long batch, int seq, float scale,
                        float dropout_p, uint64_t seed, uint64_t offset, int hl, int hg, int hoff, cudaStream_t st) {
  const long long rows = batch * seq;
  const uint32_t thr = dropout_threshold(dropout_p);
  const float ks = dropout_keep_scale(dropout_p);
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
  const float ks = dropout_keep_scale(dropout_p);
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
