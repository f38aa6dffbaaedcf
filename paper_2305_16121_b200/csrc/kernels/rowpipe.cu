// Persistent, bulk-copy-pipelined LayerNorm kernels (the HBM-bound row work of
// every block boundary).
//
// Each CTA owns a fixed set of row groups (item i of the tensor goes to CTA
// i % gridDim.x) and keeps S of them in flight: one thread issues 1-D
// cp.async.bulk copies of the next items' input rows into an S-stage shared
// ring (completion counted on an mbarrier per stage) while every thread
// normalises the current item from shared memory and stores its outputs with
// 16-byte global stores. The in-flight depth (S stages x inputs x row bytes,
// ~100-200 KB per SM) is what a one-shot row kernel cannot sustain.
//
// Thread mapping: TPR = cols / 16 threads per row, each owning 16 consecutive
// columns (one Philox dropout counter); RB = max(1,
// 256 / TPR) rows per item. Since a CTA always owns the same columns, the
// per-column operands (gamma, beta, the row bias) are loaded once per CTA, and
// the LayerNorm backward accumulates its parameter-gradient column sums
// (sum dy * xhat, sum dy) and the preceding row-parallel GEMM's bias gradient
// (sum of the dropout gradient it writes) in registers across the CTA's rows:
// the separate column passes over x and dy (ln_param16 / col_pass16 in
// rowwise.cu / elementwise.cu) are gone. Partials go to part[cta * RB + r][3]
// [cols] and a fixed-order finalize reduces them, so results are
// bit-reproducible run to run.
//
// Row statistics are exact two-pass f32 (mean, then centred variance) with
// fixed-order reductions; the plain and bias-dropout-residual forward variants
// share every f32 operation of the normalisation, so LN(x) is bit-identical
// whichever kernel produced x (Oases recompute == CrossPass replay, bitwise).
// Semantics follow oracle/gpt_oracle.cpp (the fp64 restatement the parity
// tests compare against).
#include <cstdlib>

#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.h"

namespace oases {
namespace {

constexpr int kStagesMax = 8;
// CTAs per cluster of the LayerNorm backward (column partials reduced through
// DSMEM): 2 unless OASES_LNP_CLUSTER (1, 2, 4 or 8) says otherwise (measured at
// C2/C3 sub-batch shapes: 1 and 2 equal, 4 and 8 slower -- fewer co-resident clusters).
int lnp_cluster() {
  static int c = 0;
  if (!c) {
    const char* e = std::getenv("OASES_LNP_CLUSTER");
    c = e ? std::atoi(e) : 2;
    if (c != 1 && c != 2 && c != 4 && c != 8) c = 2;
  }
  return c;
}

template <typename T>
struct Lnp {
  // forward
  const T* in;      // plain: x ; BDR: the row-GEMM output / AllReduce result
  const T* bias;    // BDR: row bias (optional)
  const T* res;     // BDR: residual x_{b-1} (optional)
  T* xout;          // BDR: x_b
  const T* gamma;
  const T* beta;
  T* y;
  uint16_t* keep_bits_out;  // BDR with dropout: keep decisions (optional)
  // backward
  const T* x;        // LN input
  const T* dy;       // gradient of the LN output
  T* dx;             // (+)= LN input gradient (acc reads the old dx)
  T* gout;           // dropout'(dx) (optional)
  const uint16_t* keep_bits;  // cached keep decisions for gout (optional; else Philox)
  float* part;       // [gridDim.x * RB][3][cols] column partials (optional)
  float2* stats;     // per-row (mean, rstd) (optional)
  long long rows;
  int cols;
  float eps;
  uint32_t thr;
  float ks;
  int drop;
  uint64_t seed;
  uint64_t offset;
  int stages;
};

// Row statistics: shifted sums. K = the row's first element as stored (every
// thread of the row reads it: from the staged input, or -- for the fused
// bias-dropout-residual forward, which computes x -- from shared memory after
// the barrier that also releases the stage), each thread sums xc = x - K and
// xc^2 over its 16 elements (and, in the backward, gd = dy * gamma and gd *
// xc), and the row's threads add the sums (xor butterfly inside a warp, then
// the row's warps in index order: fixed order, identical in every thread).
// mean = K + s1/n, var = s2/n - (s1/n)^2: with K an element of the row the
// shift keeps the cancellation at the level of two-pass statistics.
template <int TPR, int NP>
__device__ __forceinline__ void row_sum2(float2 (&v)[NP], float2* sm, int r, int wi) {
  constexpr int LIM = TPR < 32 ? TPR : 32;
#pragma unroll
  for (int o = 1; o < LIM; o <<= 1)
#pragma unroll
    for (int i = 0; i < NP; ++i) {
      float2 t;
      t.x = __shfl_xor_sync(0xffffffffu, v[i].x, o);
      t.y = __shfl_xor_sync(0xffffffffu, v[i].y, o);
      v[i] = __fadd2_rn(v[i], t);
    }
  if constexpr (TPR > 32) {
    constexpr int W = TPR / 32;
    if ((threadIdx.x & 31) == 0)
#pragma unroll
      for (int i = 0; i < NP; ++i) sm[(r * W + wi) * NP + i] = v[i];
    __syncthreads();
    const float2* q = sm + r * W * NP;
#pragma unroll
    for (int i = 0; i < NP; ++i) {
      float2 t = q[i];
#pragma unroll
      for (int w = 1; w < W; ++w) t = __fadd2_rn(t, q[w * NP + i]);
      v[i] = t;
    }
  }
}

// 16 consecutive elements as 8 float2 (pairs (2i, 2i+1)); bf16 unpacks with a
// shift / mask per element, f32 is a plain reinterpretation.
template <typename T>
__device__ __forceinline__ void ld16(const T* p, float2 (&v)[8]) {
  if constexpr (sizeof(T) == 2) {
    const uint4 a = reinterpret_cast<const uint4*>(p)[0], b = reinterpret_cast<const uint4*>(p)[1];
    const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = make_float2(__uint_as_float(w[i] << 16), __uint_as_float(w[i] & 0xFFFF0000u));
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float4 f = reinterpret_cast<const float4*>(p)[i];
      v[2 * i] = make_float2(f.x, f.y);
      v[2 * i + 1] = make_float2(f.z, f.w);
    }
  }
}
// Packed words of 16 elements (8 for bf16, 16 for f32).
template <typename T>
struct Words16 {
  static constexpr int N = 16 * static_cast<int>(sizeof(T)) / 4;
  uint32_t w[N];
};
template <typename T>
__device__ __forceinline__ void pack16(const float2 (&v)[8], Words16<T>& o) {
  if constexpr (sizeof(T) == 2) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const __nv_bfloat162 b = __float22bfloat162_rn(v[i]);
      o.w[i] = *reinterpret_cast<const uint32_t*>(&b);
    }
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      o.w[2 * i] = __float_as_uint(v[i].x);
      o.w[2 * i + 1] = __float_as_uint(v[i].y);
    }
  }
}
template <typename T>
__device__ __forceinline__ void unpack16(const Words16<T>& o, float2 (&v)[8]) {
  if constexpr (sizeof(T) == 2) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      v[i] = make_float2(__uint_as_float(o.w[i] << 16), __uint_as_float(o.w[i] & 0xFFFF0000u));
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = make_float2(__uint_as_float(o.w[2 * i]), __uint_as_float(o.w[2 * i + 1]));
  }
}
template <typename T>
__device__ __forceinline__ void st16(T* p, const Words16<T>& o) {
#pragma unroll
  for (int i = 0; i < Words16<T>::N / 4; ++i)
    reinterpret_cast<uint4*>(p)[i] = make_uint4(o.w[4 * i], o.w[4 * i + 1], o.w[4 * i + 2], o.w[4 * i + 3]);
}
template <typename T>
__device__ __forceinline__ void ldw16(const T* p, Words16<T>& o) {
#pragma unroll
  for (int i = 0; i < Words16<T>::N / 4; ++i) {
    const uint4 u = reinterpret_cast<const uint4*>(p)[i];
    o.w[4 * i] = u.x;
    o.w[4 * i + 1] = u.y;
    o.w[4 * i + 2] = u.z;
    o.w[4 * i + 3] = u.w;
  }
}
template <typename T>
__device__ __forceinline__ float ld1(const T* p) {
  if constexpr (sizeof(T) == 2) return __bfloat162float(*p);
  else return *p;
}

// Keep decisions of 16 elements (one Philox call, byte e >= thr keeps element e)
// as a 16-bit mask: a SIMD byte compare per 4 elements, bit 7 of each byte
// gathered with one multiply.
__device__ __forceinline__ uint32_t keep_mask16(const uint32_t (&u)[4], uint32_t thr) {
  const uint32_t t4 = thr * 0x01010101u;
  uint32_t bits = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t m = __vcmpgeu4(u[i], t4) & 0x80808080u;  // bit 7 of byte b = keep(4i + b)
    bits |= ((m * 0x00204081u) >> 28) << (4 * i);            // bits 7,15,23,31 -> 28..31
  }
  return bits;
}
// v *= (bit e of mask ? ks : 0) for the 16 elements
__device__ __forceinline__ void apply_mask16(float2 (&v)[8], uint32_t mask, float ks) {
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    v[i].x = (mask >> (2 * i)) & 1u ? v[i].x * ks : 0.f;
    v[i].y = (mask >> (2 * i + 1)) & 1u ? v[i].y * ks : 0.f;
  }
}

template <int TPR>
struct Geo {
  static constexpr int RB = TPR >= 256 ? 1 : 256 / TPR;  // rows per item
  static constexpr int THREADS = RB * TPR;
  static constexpr int W = TPR > 32 ? TPR / 32 : 1;       // warps per row
};

// Issue the bulk copies of item `item` (NIN inputs) into stage s.
template <typename T, int NIN>
__device__ __forceinline__ void issue_item(unsigned char* stage, uint64_t* bar, const T* const (&src)[NIN],
                                           long long item, int RB, long long rows, int cols) {
  const long long r0 = item * RB;
  const long long nr = rows - r0 < RB ? rows - r0 : RB;
  const uint32_t bytes = static_cast<uint32_t>(nr * cols * static_cast<long long>(sizeof(T)));
  const size_t slot = static_cast<size_t>(RB) * cols * sizeof(T);
  mbar_arrive_expect_tx(bar, bytes * NIN);
#pragma unroll
  for (int i = 0; i < NIN; ++i) bulk_load(stage + i * slot, src[i] + r0 * cols, bytes, bar);
}

// ------------------------------------------------------------------ forward
template <typename T, int TPR, bool BDR>
__global__ void __launch_bounds__(Geo<TPR>::THREADS, Geo<TPR>::THREADS <= 256 ? 3 : 1) lnp_fwd_kernel(const Lnp<T> a) {
  using G = Geo<TPR>;
  constexpr int RB = G::RB, W = G::W;
  constexpr int NIN = BDR ? 2 : 1;
  extern __shared__ __align__(128) unsigned char dsm[];
  __shared__ uint64_t full[kStagesMax];
  __shared__ float2 red[2][RB * W];  // double-buffered by item parity
  __shared__ float kbuf[2][RB];
  pdl_trigger();
  const int tid = threadIdx.x, r = tid / TPR, j = tid - r * TPR, wi = j >> 5;
  const int cols = a.cols, S = a.stages;
  const long long nitems = (a.rows + RB - 1) / RB;
  const size_t slot = static_cast<size_t>(RB) * cols * sizeof(T);
  const size_t stage_bytes = slot * NIN;
  const bool has_res = BDR && a.res != nullptr;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
    fence_barrier_init();
  }
  // the per-column parameters are not produced inside the step: read them before
  // the programmatic-dependency wait, under the previous kernel's tail
  const int c = j * 16;
  float2 g2[8], b2[8], bi2[8];
  ld16(a.gamma + c, g2);
  ld16(a.beta + c, b2);
  if constexpr (BDR) {
    if (a.bias) ld16(a.bias + c, bi2);
    else
#pragma unroll
      for (int i = 0; i < 8; ++i) bi2[i] = make_float2(0.f, 0.f);
  }
  __syncthreads();
  pdl_wait();
  const T* src[NIN];
  src[0] = a.in;
  if constexpr (BDR) src[NIN - 1] = has_res ? a.res : a.in;  // no residual: a harmless re-read of in
  if (tid == 0)
    for (int s = 0; s < S; ++s) {
      const long long it = blockIdx.x + static_cast<long long>(s) * gridDim.x;
      if (it < nitems) issue_item<T, NIN>(dsm + s * stage_bytes, &full[s], src, it, RB, a.rows, cols);
    }
  const float inv_cols = 1.f / static_cast<float>(cols);
  // ring slot s = k % S and its phase (k / S) & 1 as running counters (no 64-bit division per item)
  int s = 0;
  uint32_t ph = 0u;
  for (long long k = 0;; ++k, (++s == S) ? (s = 0, ph ^= 1u) : 0u) {
    const long long item = blockIdx.x + k * gridDim.x;
    if (item >= nitems) break;
    mbar_wait(&full[s], ph);
    const long long row = item * RB + r;
    const bool ok = row < a.rows;
    const long long base = row * cols + c;
    const T* srow = reinterpret_cast<const T*>(dsm + s * stage_bytes) + r * cols;
    float2 v[8];
    float K = 0.f;
    if (ok) ld16(srow + c, v);
    else
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = make_float2(0.f, 0.f);
    if constexpr (BDR) {
      if (ok) {
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = __fadd2_rn(v[i], bi2[i]);
        if (a.drop) {
          uint32_t u[4];
          Philox::gen(a.seed, a.offset, static_cast<unsigned long long>(base) >> 4, u);
          const uint32_t m = keep_mask16(u, a.thr);
          apply_mask16(v, m, a.ks);
          if (a.keep_bits_out) a.keep_bits_out[base >> 4] = static_cast<uint16_t>(m);
        }
        if (has_res) {
          float2 rr[8];
          ld16(reinterpret_cast<const T*>(reinterpret_cast<const unsigned char*>(srow) + slot) + c, rr);
#pragma unroll
          for (int i = 0; i < 8; ++i) v[i] = __fadd2_rn(v[i], rr[i]);
        }
        Words16<T> xw;
        pack16<T>(v, xw);
        st16(a.xout + base, xw);
        unpack16<T>(xw, v);  // normalise the stored (rounded) x, exactly what a re-read sees
        if (j == 0) kbuf[k & 1][r] = v[0].x;
      }
      __syncthreads();  // the stage is consumed and K is visible
      if (tid == 0) {
        const long long nxt = item + static_cast<long long>(S) * gridDim.x;
        if (nxt < nitems) issue_item<T, NIN>(dsm + s * stage_bytes, &full[s], src, nxt, RB, a.rows, cols);
      }
      K = kbuf[k & 1][r];
    } else {
      if (ok) K = ld1(srow);
      if constexpr (TPR <= 32) __syncthreads();  // (the row sum's barrier otherwise)
    }
    float2 a1 = make_float2(0.f, 0.f), a2 = make_float2(0.f, 0.f);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      v[i] = __fadd2_rn(v[i], make_float2(-K, -K));  // xc
      a1 = __fadd2_rn(a1, v[i]);
      a2 = __ffma2_rn(v[i], v[i], a2);
    }
    float2 st2[1] = {make_float2(a1.x + a1.y, a2.x + a2.y)};
    row_sum2<TPR, 1>(st2, red[k & 1], r, wi);
    if constexpr (!BDR) {  // every thread has read stage s: hand it to the next item
      if (tid == 0) {
        const long long nxt = item + static_cast<long long>(S) * gridDim.x;
        if (nxt < nitems) issue_item<T, NIN>(dsm + s * stage_bytes, &full[s], src, nxt, RB, a.rows, cols);
      }
    }
    if (!ok) continue;
    const float dm = st2[0].x * inv_cols;
    const float var = fmaxf(st2[0].y * inv_cols - dm * dm, 0.f);
    const float rstd = rsqrtf(var + a.eps);
    const float2 r2 = make_float2(rstd, rstd), ndm = make_float2(-dm, -dm);
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __ffma2_rn(__fadd2_rn(v[i], ndm), __fmul2_rn(g2[i], r2), b2[i]);
    Words16<T> yw;
    pack16<T>(v, yw);
    st16(a.y + base, yw);
  }
}

// ------------------------------------------------------------------ backward
// dx (+)= rstd * (gd - mean(gd) - xhat * mean(gd * xhat)),  gd = dy * gamma;
// gout = dropout'(dx as stored); column partials of dy * xhat, dy, gout.
template <typename T, int TPR, bool ACC, bool DROP>
__global__ void __launch_bounds__(Geo<TPR>::THREADS, Geo<TPR>::THREADS <= 256 ? 2 : 1) lnp_bwd_kernel(const Lnp<T> a) {
  using G = Geo<TPR>;
  constexpr int RB = G::RB, W = G::W;
  constexpr int NIN = ACC ? 3 : 2;
  extern __shared__ __align__(128) unsigned char dsm[];
  __shared__ uint64_t full[kStagesMax];
  __shared__ float2 red[2][RB * W * 2];  // double-buffered by item parity
  pdl_trigger();
  const int tid = threadIdx.x, r = tid / TPR, j = tid - r * TPR, wi = j >> 5;
  const int cols = a.cols, S = a.stages;
  const long long nitems = (a.rows + RB - 1) / RB;
  const size_t slot = static_cast<size_t>(RB) * cols * sizeof(T);
  const size_t stage_bytes = slot * NIN;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
    fence_barrier_init();
  }
  const int c = j * 16;
  // gamma: 16 elements per thread, parked in a private shared-memory slot (read
  // back per row) so the register budget goes to the column partials; a
  // parameter, so read before the programmatic-dependency wait
  uint4* gsm = reinterpret_cast<uint4*>(dsm + static_cast<size_t>(S) * stage_bytes) + tid * (Words16<T>::N / 4);
  {
    Words16<T> gw;
    ldw16(a.gamma + c, gw);
#pragma unroll
    for (int i = 0; i < Words16<T>::N / 4; ++i) gsm[i] = make_uint4(gw.w[4 * i], gw.w[4 * i + 1], gw.w[4 * i + 2], gw.w[4 * i + 3]);
  }
  __syncthreads();
  pdl_wait();
  const T* src[NIN];
  src[0] = a.x;
  src[1] = a.dy;
  if constexpr (ACC) src[NIN - 1] = a.dx;
  float2 pg[8], pb[8], po[8];  // column partials: dy * xhat, dy, out
#pragma unroll
  for (int i = 0; i < 8; ++i) pg[i] = pb[i] = po[i] = make_float2(0.f, 0.f);
  if (tid == 0)
    for (int s = 0; s < S; ++s) {
      const long long it = blockIdx.x + static_cast<long long>(s) * gridDim.x;
      if (it < nitems) issue_item<T, NIN>(dsm + s * stage_bytes, &full[s], src, it, RB, a.rows, cols);
    }
  const float inv_cols = 1.f / static_cast<float>(cols);
  int s = 0;  // ring slot k % S and its phase (k / S) & 1, as running counters
  uint32_t ph = 0u;
  for (long long k = 0;; ++k, (++s == S) ? (s = 0, ph ^= 1u) : 0u) {
    const long long item = blockIdx.x + k * gridDim.x;
    if (item >= nitems) break;
    const long long row = item * RB + r;
    const bool ok = row < a.rows;
    const long long base = row * cols + c;
    // the forward's keep bits of this thread's 16 elements: a dependent global
    // load, issued before the stage wait so its latency hides under the wait and
    // the row statistics (it was 22 % of the stall samples where dropout' used it)
    uint32_t keep = 0;
    if constexpr (DROP)
      if (a.keep_bits && ok) keep = a.keep_bits[base >> 4];
    mbar_wait(&full[s], ph);
    const T* srow = reinterpret_cast<const T*>(dsm + s * stage_bytes) + r * cols;
    float2 xc[8];
    Words16<T> dw, ow;
    float K = 0.f;
    if (ok) {
      K = ld1(srow);
      ld16(srow + c, xc);
      ldw16(reinterpret_cast<const T*>(reinterpret_cast<const unsigned char*>(srow) + slot) + c, dw);
      if constexpr (ACC) ldw16(reinterpret_cast<const T*>(reinterpret_cast<const unsigned char*>(srow) + 2 * slot) + c, ow);
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) xc[i] = make_float2(0.f, 0.f);
#pragma unroll
      for (int i = 0; i < Words16<T>::N; ++i) dw.w[i] = ow.w[i] = 0u;
    }
    float2 g2[8], d[8];
    {
      Words16<T> gw;
      ldw16(reinterpret_cast<const T*>(gsm), gw);
      unpack16<T>(gw, g2);
    }
    unpack16<T>(dw, d);
    float2 a1 = make_float2(0.f, 0.f), a2 = a1, a3 = a1, a4 = a1;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      xc[i] = __fadd2_rn(xc[i], make_float2(-K, -K));
      const float2 gd = __fmul2_rn(d[i], g2[i]);
      a1 = __fadd2_rn(a1, xc[i]);
      a2 = __ffma2_rn(xc[i], xc[i], a2);
      a3 = __fadd2_rn(a3, gd);
      a4 = __ffma2_rn(gd, xc[i], a4);
    }
    float2 st2[2] = {make_float2(a1.x + a1.y, a2.x + a2.y), make_float2(a3.x + a3.y, a4.x + a4.y)};
    if constexpr (TPR <= 32) __syncthreads();  // (the row sum's barrier otherwise)
    row_sum2<TPR, 2>(st2, red[k & 1], r, wi);
    // every thread has read stage s: hand it to the next item
    if (tid == 0) {
      const long long nxt = item + static_cast<long long>(S) * gridDim.x;
      if (nxt < nitems) issue_item<T, NIN>(dsm + s * stage_bytes, &full[s], src, nxt, RB, a.rows, cols);
    }
    if (!ok) continue;
    const float dm = st2[0].x * inv_cols;
    const float var = fmaxf(st2[0].y * inv_cols - dm * dm, 0.f);
    const float rstd = rsqrtf(var + a.eps);
    const float m1 = st2[1].x * inv_cols, m2 = rstd * (st2[1].y - dm * st2[1].x) * inv_cols;
    if (a.stats && j == 0) a.stats[row] = make_float2(K + dm, rstd);
    const float2 r2 = make_float2(rstd, rstd), ndm = make_float2(-dm, -dm), nm1 = make_float2(-m1, -m1),
                 nm2 = make_float2(-m2, -m2);
    {
      Words16<T> gw;
      ldw16(reinterpret_cast<const T*>(gsm), gw);
      unpack16<T>(gw, g2);
    }
    float2 o[8];
    if constexpr (ACC) unpack16<T>(ow, o);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float2 xh = __fmul2_rn(__fadd2_rn(xc[i], ndm), r2);
      pg[i] = __ffma2_rn(d[i], xh, pg[i]);
      pb[i] = __fadd2_rn(pb[i], d[i]);
      const float2 t = __ffma2_rn(xh, nm2, __fadd2_rn(__fmul2_rn(d[i], g2[i]), nm1));
      o[i] = ACC ? __ffma2_rn(t, r2, o[i]) : __fmul2_rn(t, r2);
    }
    Words16<T> w;
    pack16<T>(o, w);
    st16(a.dx + base, w);
    unpack16<T>(w, o);  // what a re-read of the stored dx sees
    if constexpr (DROP) {
      uint32_t m;
      if (a.keep_bits) {
        m = keep;
      } else {
        uint32_t u[4];
        Philox::gen(a.seed, a.offset, static_cast<unsigned long long>(base) >> 4, u);
        m = keep_mask16(u, a.thr);
      }
      apply_mask16(o, m, a.ks);
      pack16<T>(o, w);
      st16(a.gout + base, w);
      unpack16<T>(w, o);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) po[i] = __fadd2_rn(po[i], o[i]);
  }
  if (!a.part) return;
  // Column partials: every row slot stores its partials into its own
  // [3][cols] plane of shared memory (the ring is idle now; one barrier, no
  // read-modify-write rounds), then the CTAs of the cluster reduce them through
  // distributed shared memory -- CTA rank q sums column chunk q of every rank's
  // planes, slots in order within a rank, ranks in order -- and write one
  // [3][cols] partial row per cluster (lnp_cluster() times fewer rows for the
  // finalize to read).
  float* psm = reinterpret_cast<float*>(dsm);  // [RB][3][cols]
  {
    float* q0 = psm + static_cast<size_t>(r) * 3 * cols + c;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      reinterpret_cast<float4*>(q0)[i] = make_float4(pg[2 * i].x, pg[2 * i].y, pg[2 * i + 1].x, pg[2 * i + 1].y);
      reinterpret_cast<float4*>(q0 + cols)[i] = make_float4(pb[2 * i].x, pb[2 * i].y, pb[2 * i + 1].x, pb[2 * i + 1].y);
      reinterpret_cast<float4*>(q0 + 2 * cols)[i] =
          make_float4(po[2 * i].x, po[2 * i].y, po[2 * i + 1].x, po[2 * i + 1].y);
    }
  }
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  cl.sync();  // (also the CTA barrier for the planes)
  const int ncl = static_cast<int>(cl.num_blocks()), rank = static_cast<int>(cl.block_rank());
  const int nf4 = 3 * cols / 4, chunk = (nf4 + ncl - 1) / ncl;
  const int f0 = rank * chunk, f1 = f0 + chunk < nf4 ? f0 + chunk : nf4;
  float4* out = reinterpret_cast<float4*>(a.part + static_cast<long long>(blockIdx.x / ncl) * 3 * cols);
  for (int f = f0 + tid; f < f1; f += G::THREADS) {
    float4 t;
    for (int q = 0; q < ncl; ++q) {
      const float4* pq = reinterpret_cast<const float4*>(cl.map_shared_rank(psm, q)) + f;
      float4 u = pq[0];
#pragma unroll 4
      for (int rr = 1; rr < RB; ++rr) {
        const float4 v = pq[static_cast<size_t>(rr) * nf4];
        u.x += v.x; u.y += v.y; u.z += v.z; u.w += v.w;
      }
      if (q == 0) {
        t = u;
      } else {
        t.x += u.x; t.y += u.y; t.z += u.z; t.w += u.w;
      }
    }
    out[f] = t;
  }
  cl.sync();  // the peers' shared memory stays valid until every rank has read it
}

// out_q[c] (+)= sum_p part[p][q][c] (null outputs skipped): block (x, q)
// covers 128 columns of quantity q with 32 lanes x 4 columns (16-byte loads) x
// 32 partial-row groups; group g sums rows g, g+32, ... (4 loads in flight) and
// the 32 group sums are combined in g order (fixed order, bit-reproducible).
__global__ void __launch_bounds__(1024) lnp_finalize_kernel(const float* __restrict__ part, int prows, int cols,
                                                            float* o0, float* o1, float* o2, int acc0, int acc1,
                                                            int acc2) {
  pdl_trigger();
  const int q = blockIdx.y;
  float* out = q == 0 ? o0 : q == 1 ? o1 : o2;
  if (!out) return;
  const int acc = q == 0 ? acc0 : q == 1 ? acc1 : acc2;
  pdl_wait();
  __shared__ float4 sm[32][32];
  const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int c = blockIdx.x * 128 + lane * 4;
  float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
  if (c < cols) {
    const float* base = part + static_cast<long long>(q) * cols + c;
    const long long stride = 3LL * cols;
    int k = g;
    for (; k + 96 < prows; k += 128) {
      float4 u[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) u[i] = __ldg(reinterpret_cast<const float4*>(base + (k + 32 * i) * stride));
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        t.x += u[i].x; t.y += u[i].y; t.z += u[i].z; t.w += u[i].w;
      }
    }
    for (; k < prows; k += 32) {
      const float4 u = __ldg(reinterpret_cast<const float4*>(base + k * stride));
      t.x += u.x; t.y += u.y; t.z += u.z; t.w += u.w;
    }
  }
  sm[g][lane] = t;
  __syncthreads();
  if (g == 0 && c < cols) {
    float4 sacc = sm[0][lane];
#pragma unroll
    for (int w = 1; w < 32; ++w) {
      const float4 u = sm[w][lane];
      sacc.x += u.x; sacc.y += u.y; sacc.z += u.z; sacc.w += u.w;
    }
    float4* o = reinterpret_cast<float4*>(out + c);
    if (acc) {
      const float4 u = *o;
      sacc.x += u.x; sacc.y += u.y; sacc.z += u.z; sacc.w += u.w;
    }
    *o = sacc;
  }
}

// ------------------------------------------------------------------ launch
int tpr_of(int cols) {
  if (cols % 16) return 0;
  const int t = cols / 16;
  return (t >= 8 && t <= 512 && (t & (t - 1)) == 0) ? t : 0;
}

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// Stage count and CTAs per SM: up to 200 KB of ring per SM split over the
// resident CTAs (2..8 stages each).
struct Plan {
  int stages, per_sm;
  size_t smem;
};
Plan plan_with(size_t bytes_per_stage, int per_sm) {
  int s = static_cast<int>((200 * 1024 / per_sm) / bytes_per_stage);
  s = s < 2 ? 2 : (s > kStagesMax ? kStagesMax : s);
  return {s, per_sm, static_cast<size_t>(s) * bytes_per_stage};
}
// Forward: as many CTAs per SM (<= 4) as registers, threads and a >= 2-stage
// ring allow, from the occupancy calculator (cached per kernel and stage size).
template <typename K>
Plan plan_occupancy(K kernel, size_t bytes_per_stage, int threads) {
  struct Key {
    const void* k;
    size_t b;
  };
  static Key keys[64];
  static Plan plans[64];
  static int n = 0;
  for (int i = 0; i < n; ++i)
    if (keys[i].k == reinterpret_cast<const void*>(kernel) && keys[i].b == bytes_per_stage) return plans[i];
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, threads, 0);
  int per = occ < 4 ? occ : 4;
  Plan pl = plan_with(bytes_per_stage, 1);
  for (; per >= 1; --per) {
    const Plan cand = plan_with(bytes_per_stage, per);
    if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(cand.smem)) !=
        cudaSuccess)
      continue;
    int got = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&got, kernel, threads, cand.smem);
    if (got >= per) {
      pl = cand;
      break;
    }
  }
  if (n < 64) {
    keys[n] = {reinterpret_cast<const void*>(kernel), bytes_per_stage};
    plans[n++] = pl;
  }
  return pl;
}

int grid_for_items(long long nitems, int per_sm, int max_sms) {
  int sms = num_sms();
  if (max_sms > 0 && max_sms < sms) sms = max_sms;
  long long g = static_cast<long long>(sms) * per_sm;
  if (g > nitems) g = nitems;
  return static_cast<int>(g < 1 ? 1 : g);
}

template <typename T, int TPR, bool BDR>
cudaError_t fwd_tpr(Lnp<T> a, int max_sms, cudaStream_t st) {
  using G = Geo<TPR>;
  const size_t stage = static_cast<size_t>(BDR ? 2 : 1) * G::RB * a.cols * sizeof(T);
  auto k = lnp_fwd_kernel<T, TPR, BDR>;
  const Plan pl = plan_occupancy(k, stage, G::THREADS);
  a.stages = pl.stages;
  const long long nitems = (a.rows + G::RB - 1) / G::RB;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(pl.smem));
  if (e != cudaSuccess) return e;
  e = launch_pdl(k, dim3(grid_for_items(nitems, pl.per_sm, max_sms)), dim3(G::THREADS), pl.smem, st, a);
  return e != cudaSuccess ? e : cudaGetLastError();
}

// Geometry of a backward launch: the grid (and so the number of partial rows,
// grid / lnp_cluster()) is a pure function of (element size, cols, acc, rows,
// max_sms): as many whole clusters as the occupancy calculator says can be
// co-resident (a persistent grid must not spill into a second wave), capped
// by the work.
struct BwdGeo {
  Plan pl;
  int rb, threads, grid;
};
template <typename T, bool ACC>
const void* bwd_kernel_ptr(int tpr) {
  switch (tpr) {
    case 8: return reinterpret_cast<const void*>(lnp_bwd_kernel<T, 8, ACC, false>);
    case 16: return reinterpret_cast<const void*>(lnp_bwd_kernel<T, 16, ACC, false>);
    case 32: return reinterpret_cast<const void*>(lnp_bwd_kernel<T, 32, ACC, false>);
    case 64: return reinterpret_cast<const void*>(lnp_bwd_kernel<T, 64, ACC, false>);
    case 128: return reinterpret_cast<const void*>(lnp_bwd_kernel<T, 128, ACC, false>);
    case 256: return reinterpret_cast<const void*>(lnp_bwd_kernel<T, 256, ACC, false>);
    default: return reinterpret_cast<const void*>(lnp_bwd_kernel<T, 512, ACC, false>);
  }
}
// Co-resident clusters of the backward kernel (cached; all DROP variants share
// the launch bounds and the shared-memory size, so the DROP=false instance stands in).
int bwd_max_clusters(size_t esize, int tpr, bool acc, int threads, size_t smem) {
  struct Key {
    size_t e;
    int t;
    bool a;
    size_t m;
    int v;
  };
  static Key cache[32];
  static int n = 0;
  for (int i = 0; i < n; ++i)
    if (cache[i].e == esize && cache[i].t == tpr && cache[i].a == acc && cache[i].m == smem) return cache[i].v;
  const void* k = esize == 2 ? (acc ? bwd_kernel_ptr<__nv_bfloat16, true>(tpr) : bwd_kernel_ptr<__nv_bfloat16, false>(tpr))
                             : (acc ? bwd_kernel_ptr<float, true>(tpr) : bwd_kernel_ptr<float, false>(tpr));
  int v = 0;
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) == cudaSuccess) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(lnp_cluster() * 64);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = lnp_cluster();
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaOccupancyMaxActiveClusters(&v, k, &cfg) != cudaSuccess) v = 0;
  }
  cudaGetLastError();
  if (v < 1) v = 1;
  if (n < 32) cache[n++] = {esize, tpr, acc, smem, v};
  return v;
}
BwdGeo bwd_geo(size_t esize, int cols, bool acc, long long rows, int max_sms) {
  const int tpr = tpr_of(cols);
  const int rb = tpr >= 256 ? 1 : 256 / tpr;
  const int threads = rb * tpr;
  const size_t stage = static_cast<size_t>(acc ? 3 : 2) * rb * cols * esize;
  // 2 CTAs per SM (the kernel's launch bounds guarantee the registers) up to 256 threads
  Plan pl = plan_with(stage, threads <= 256 ? 2 : 1);
  pl.smem += static_cast<size_t>(threads) * 16 * esize;  // private gamma slots
  // the column-partial planes overlay the ring at kernel end: [rb][3][cols] f32
  const size_t planes = static_cast<size_t>(rb) * 3 * cols * sizeof(float);
  if (pl.smem < planes) pl.smem = planes;
  int sms = num_sms();
  long long clusters = bwd_max_clusters(esize, tpr, acc, threads, pl.smem);
  if (max_sms > 0 && max_sms < sms) clusters = clusters * max_sms / sms;  // leave the capped SMs' share
  const long long need = ((rows + rb - 1) / rb + lnp_cluster() - 1) / lnp_cluster();  // whole clusters of work
  if (clusters > need) clusters = need;
  if (clusters < 1) clusters = 1;
  return {pl, rb, threads, static_cast<int>(clusters) * lnp_cluster()};
}

template <typename T, int TPR, bool ACC, bool DROP>
cudaError_t bwd_tpr(Lnp<T> a, int max_sms, cudaStream_t st) {
  const BwdGeo g = bwd_geo(sizeof(T), a.cols, ACC, a.rows, max_sms);
  a.stages = g.pl.stages;
  auto k = lnp_bwd_kernel<T, TPR, ACC, DROP>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(g.pl.smem));
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(g.grid);
  cfg.blockDim = dim3(g.threads);
  cfg.dynamicSmemBytes = g.pl.smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = lnp_cluster();
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  e = cudaLaunchKernelEx(&cfg, k, a);
  return e != cudaSuccess ? e : cudaGetLastError();
}

template <typename T, bool BDR>
cudaError_t fwd_dispatch(const Lnp<T>& a, int max_sms, cudaStream_t st) {
  switch (tpr_of(a.cols)) {
    case 8: return fwd_tpr<T, 8, BDR>(a, max_sms, st);
    case 16: return fwd_tpr<T, 16, BDR>(a, max_sms, st);
    case 32: return fwd_tpr<T, 32, BDR>(a, max_sms, st);
    case 64: return fwd_tpr<T, 64, BDR>(a, max_sms, st);
    case 128: return fwd_tpr<T, 128, BDR>(a, max_sms, st);
    case 256: return fwd_tpr<T, 256, BDR>(a, max_sms, st);
    case 512: return fwd_tpr<T, 512, BDR>(a, max_sms, st);
    default: return cudaErrorNotSupported;
  }
}

template <typename T, bool ACC, bool DROP>
cudaError_t bwd_dispatch2(const Lnp<T>& a, int max_sms, cudaStream_t st) {
  switch (tpr_of(a.cols)) {
    case 8: return bwd_tpr<T, 8, ACC, DROP>(a, max_sms, st);
    case 16: return bwd_tpr<T, 16, ACC, DROP>(a, max_sms, st);
    case 32: return bwd_tpr<T, 32, ACC, DROP>(a, max_sms, st);
    case 64: return bwd_tpr<T, 64, ACC, DROP>(a, max_sms, st);
    case 128: return bwd_tpr<T, 128, ACC, DROP>(a, max_sms, st);
    case 256: return bwd_tpr<T, 256, ACC, DROP>(a, max_sms, st);
    case 512: return bwd_tpr<T, 512, ACC, DROP>(a, max_sms, st);
    default: return cudaErrorNotSupported;
  }
}

template <typename T>
cudaError_t bwd_dispatch(const Lnp<T>& a, bool acc, bool drop, int max_sms, cudaStream_t st) {
  if (acc) return drop ? bwd_dispatch2<T, true, true>(a, max_sms, st) : bwd_dispatch2<T, true, false>(a, max_sms, st);
  return drop ? bwd_dispatch2<T, false, true>(a, max_sms, st) : bwd_dispatch2<T, false, false>(a, max_sms, st);
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

}  // namespace

bool lnp_supported(long long rows, int cols) { return tpr_of(cols) != 0 && rows > 0 && rows < (1LL << 40); }

long long lnp_partial_rows_max(long long rows, int cols) {
  const int tpr = tpr_of(cols);
  if (!tpr) return 0;
  const int rb = tpr >= 256 ? 1 : 256 / tpr;
  const long long nitems = (rows + rb - 1) / rb;
  const long long g = 2LL * num_sms() < nitems ? 2LL * num_sms() : nitems;
  return g * rb;
}

bool lnp_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = std::getenv("OASES_LNP");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}

long long lnp_partial_rows(int dtype, long long rows, int cols, int acc_dx, int max_sms) {
  if (!lnp_supported(rows, cols)) return 0;
  const BwdGeo g = bwd_geo(dtype == OASES_BF16 ? 2 : 4, cols, acc_dx != 0, rows, max_sms);
  return g.grid / lnp_cluster();
}

cudaError_t lnp_layernorm_fwd(int dtype, const void* in, const void* bias, const void* res, void* xout,
                              const void* gamma, const void* beta, void* y, long long rows, int cols, float eps,
                              float p, uint64_t seed, uint64_t offset, uint16_t* keep_bits, int max_sms,
                              cudaStream_t st) {
  if (!lnp_supported(rows, cols) || !aligned16(in) || (res && !aligned16(res))) return cudaErrorNotSupported;
  const bool bdr = xout != nullptr;
  auto fill = [&](auto a) {
    using T = std::remove_pointer_t<decltype(a.xout)>;
    a.in = static_cast<const T*>(in);
    a.bias = static_cast<const T*>(bias);
    a.res = static_cast<const T*>(res);
    a.xout = static_cast<T*>(xout);
    a.gamma = static_cast<const T*>(gamma);
    a.beta = static_cast<const T*>(beta);
    a.y = static_cast<T*>(y);
    a.keep_bits_out = keep_bits;
    a.rows = rows;
    a.cols = cols;
    a.eps = eps;
    a.thr = dropout_threshold(p);
    a.ks = dropout_keep_scale(p);
    a.drop = bdr && p > 0.f;
    a.seed = seed;
    a.offset = offset;
    return a;
  };
  if (dtype == OASES_BF16) {
    const Lnp<__nv_bfloat16> a = fill(Lnp<__nv_bfloat16>{});
    return bdr ? fwd_dispatch<__nv_bfloat16, true>(a, max_sms, st) : fwd_dispatch<__nv_bfloat16, false>(a, max_sms, st);
  }
  const Lnp<float> a = fill(Lnp<float>{});
  return bdr ? fwd_dispatch<float, true>(a, max_sms, st) : fwd_dispatch<float, false>(a, max_sms, st);
}

cudaError_t lnp_layernorm_bwd(int dtype, const void* x, const void* gamma, const void* dy, void* dx, int acc_dx,
                              void* gout, float p, uint64_t seed, uint64_t offset, const uint16_t* keep_bits,
                              float* part, float2* stats, long long rows, int cols, float eps, int max_sms,
                              cudaStream_t st) {
  if (!lnp_supported(rows, cols) || !aligned16(x) || !aligned16(dy) || !aligned16(dx)) return cudaErrorNotSupported;
  const bool drop = gout != nullptr;
  auto fill = [&](auto a) {
    using T = std::remove_pointer_t<decltype(a.dx)>;
    a.x = static_cast<const T*>(x);
    a.gamma = static_cast<const T*>(gamma);
    a.dy = static_cast<const T*>(dy);
    a.dx = static_cast<T*>(dx);
    a.gout = static_cast<T*>(gout);
    a.keep_bits = keep_bits;
    a.part = part;
    a.stats = stats;
    a.rows = rows;
    a.cols = cols;
    a.eps = eps;
    a.thr = dropout_threshold(p);
    a.ks = dropout_keep_scale(p);
    a.drop = drop;
    a.seed = seed;
    a.offset = offset;
    return a;
  };
  if (dtype == OASES_BF16) return bwd_dispatch(fill(Lnp<__nv_bfloat16>{}), acc_dx != 0, drop, max_sms, st);
  return bwd_dispatch(fill(Lnp<float>{}), acc_dx != 0, drop, max_sms, st);
}

cudaError_t lnp_finalize(const float* part, long long prows, int cols, float* dgamma, float* dbeta, float* dbias,
                         int acc_gamma, int acc_beta, int acc_bias, cudaStream_t st) {
  if (!dgamma && !dbeta && !dbias) return cudaSuccess;
  if (cols % 4) return cudaErrorNotSupported;
  launch_pdl(lnp_finalize_kernel, dim3((cols + 127) / 128, 3), dim3(1024), 0, st, part, static_cast<int>(prows), cols,
             dgamma, dbeta, dbias, acc_gamma, acc_beta, acc_bias);
  return cudaGetLastError();
}

}  // namespace oases
