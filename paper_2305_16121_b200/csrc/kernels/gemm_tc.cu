// Persistent, warp-specialised tcgen05 GEMM for sm_100a (bf16 in, f32 accumulate in TMEM).
//
// C[z](m,n) = epilogue(alpha * sum_k A[z](m,k) * B[z](n,k))
//
// This is the B200 replacement of the reference's fp64 `matmul`
// (proj/src/numerics.cpp:13-24) for every GEMM of the TMP layer: the
// column-parallel QKV/FC1, row-parallel proj/FC2, their dgrad/wgrad
// (numerics.cpp:202-206) and the batched attention contractions. Transposes
// (numerics.cpp:26-32) are expressed as operand major-ness in the TMA box and
// the UMMA smem descriptor, never as a kernel.
//
// Two kernels share the pipeline structure (320 threads, 1 CTA per SM,
// persistent over a static tile schedule):
//   warp 0      TMA producer (one lane): gmem -> SWIZZLE_128B smem ring, mbarrier tx
//   warp 1      MMA issuer (one lane): tcgen05.mma into a double-buffered TMEM
//               accumulator; also owns TMEM alloc/dealloc
//   warps 2..9  epilogue: two warps per TMEM lane quarter, each owning half of
//               the tile's columns: tcgen05.ld -> registers -> swizzled smem ->
//               row-contiguous 16-byte segments -> fused bias / erf-GeLU /
//               dGeLU / f32-accumulate -> global. The epilogue is specialised at
//               compile time (output type x epilogue x accumulate) so its inner
//               loop is branch-free pointer arithmetic.
// * gemm_tc_kernel<BN,...>: one CTA computes 128 x BN (BN = 128 | 256); used for
//   the causal attention GEMMs and small problems.
// * gemm_tc2_kernel: a 2-CTA cluster (cta_group::2) computes 256 x 256; each CTA
//   stages half of A and half of B, the leader issues M=256 MMAs reading both
//   CTAs' smem (half the operand traffic per MAC of the single-CTA tile).
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <type_traits>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "gemm.h"

namespace oases {

namespace {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int EPI_WARPS = 8;
constexpr int THREADS = 64 + 32 * EPI_WARPS;
constexpr int STG_FLOAT4 = EPI_WARPS * 256;  // 4 KB staging per epilogue warp (static smem)

template <int BN>
struct TcCfg {
  static constexpr int STAGES = (BN == 256) ? 4 : 6;
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int BAR_BYTES = 256;
  static constexpr int SMEM = STAGES * STAGE_BYTES + BAR_BYTES + 1024;  // + 32 KB static staging
  static constexpr uint32_t TMEM_COLS = 2 * BN;                       // two accumulator buffers
};

struct TcParams {
  int M, N, K;
  int batch, batch_inner;
  int tiles_m, tiles_n;
  int kblocks;
  int a_x_off[2], a_y_off[2], b_x_off[2], b_y_off[2];
  void* c;
  void* c2;
  const void* aux;
  const void* bias;
  long long ldc;
  long long c_row_off[2], c_col_off[2];
  int c_f32;
  int epilogue;
  int causal;
  int accumulate;
  float alpha;
  float* rowdot;  // EPI_ROWDOT output
  int rd_group, rd_seq, rd_heads;
  float* colsum;  // EPI_MUL column-sum partials [ceil(M/32)][N] (or null)
  int zigzag;     // causal K ranges: serpentine tile order (sched_tile)
};

struct TileInfo {
  int z, m0, n0, kb0, kb1;
};

template <int BN>
__device__ __forceinline__ bool decode_tile(const TcParams& p, int t, TileInfo& ti) {
  int mt, nt;
  if (p.causal == OASES_CAUSAL_K_UPTO_M || p.causal == OASES_CAUSAL_K_FROM_M) {
    // Causal K ranges make tile cost grow (UPTO) or shrink (FROM) with the
    // m-tile: order tiles heaviest-first across the whole batch (m-tile is the
    // slowest index) so the static persistent stride balances like LPT.
    const int per_m = p.batch * p.tiles_n;
    const int mi = t / per_m;
    const int r = t - mi * per_m;
    mt = p.causal == OASES_CAUSAL_K_UPTO_M ? p.tiles_m - 1 - mi : mi;
    ti.z = r / p.tiles_n;
    nt = r - ti.z * p.tiles_n;
  } else {
    const int per_z = p.tiles_m * p.tiles_n;
    ti.z = t / per_z;
    const int r = t - ti.z * per_z;
    mt = r / p.tiles_n;
    nt = r - mt * p.tiles_n;
  }
  ti.m0 = mt * BM;
  ti.n0 = nt * BN;
  if (p.causal == OASES_CAUSAL_SKIP_UPPER && ti.n0 > ti.m0 + BM - 1) return false;
  ti.kb0 = 0;
  ti.kb1 = p.kblocks;
  if (p.causal == OASES_CAUSAL_K_UPTO_M) {
    const int lim = (ti.m0 + BM + BK - 1) / BK;
    ti.kb1 = lim < ti.kb1 ? lim : ti.kb1;
  } else if (p.causal == OASES_CAUSAL_K_FROM_M) {
    ti.kb0 = ti.m0 / BK;
  }
  return ti.kb0 < ti.kb1;
}

// Tile of this CTA's r-th round. Causal K-range tiles come heaviest first
// (decode_tile); a plain stride hands CTA b the b-th tile of every round, so
// the low CTAs collect the heaviest tile of each round (C2 dQ: 20 vs an average
// of 15.6 k-blocks of 128). Serpentine order (the stride reversed on odd rounds)
// pairs each round's heavy tiles with the next round's light ones.
__device__ __forceinline__ int sched_tile(const TcParams& p, int r) {
  const int G = static_cast<int>(gridDim.x), b = static_cast<int>(blockIdx.x);
  return r * G + ((p.zigzag && (r & 1)) ? G - 1 - b : b);
}

// ----------------------------------------------------------------- epilogue
// erf-GeLU and its derivative for the bf16 tensor-core epilogues. The normal
// CDF uses Abramowitz & Stegun 7.1.26 (|erf error| <= 1.5e-7, four orders of
// magnitude below the bf16 output's resolution): one rcp and one ex2 on the
// SFU, shared between Phi(x) and phi(x), ~16 instructions instead of erff +
// expf (~45). The f32 parity path (gemm_simt) and the standalone GeLU kernels
// keep the exact erff of numerics.cpp:50-55.
__device__ __forceinline__ void norm_cdf_pdf(float x, float& cdf, float& pdf) {
  const float u = fabsf(x) * 0.70710678118654752f;
  float t, e;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(t) : "f"(fmaf(0.3275911f, u, 1.0f)));
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(-0.72134752044448170f * x * x));  // exp(-x^2/2)
  const float poly =
      t * fmaf(t, fmaf(t, fmaf(t, fmaf(t, 1.061405429f, -1.453152027f), 1.421413741f), -0.284496736f), 0.254829592f);
  const float half_erf = fmaf(-0.5f * poly, e, 0.5f);  // erf(|x|/sqrt2) / 2
  cdf = 0.5f + copysignf(half_erf, x);
  pdf = 0.39894228040143268f * e;
}
__device__ __forceinline__ float gelu_fast(float x) {
  float c, d;
  norm_cdf_pdf(x, c, d);
  return x * c;
}
__device__ __forceinline__ float gelu_grad_fast(float x) {
  float c, d;
  norm_cdf_pdf(x, c, d);
  return fmaf(x, d, c);
}

// E elements (E = 8 bf16 / 4 f32, one 16-byte vector) of one output row.
template <typename OutT, int E>
__device__ __forceinline__ void st_vec(OutT* p, const float (&v)[E]) {
  if constexpr (sizeof(OutT) == 2) {
    uint32_t w[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * j], v[2 * j + 1]);
      w[j] = *reinterpret_cast<uint32_t*>(&h);
    }
    *reinterpret_cast<uint4*>(p) = make_uint4(w[0], w[1], w[2], w[3]);
  } else {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  }
}
// E bias values starting at column n (bias is bf16 in the tensor-core path).
template <int E>
__device__ __forceinline__ void ld_bias(const __nv_bfloat16* b, int n, int valid, float (&v)[E]) {
  if (valid >= E && (E % 8 == 0)) {
    const uint4 u = *reinterpret_cast<const uint4*>(b + n);
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int j = 0; j < E / 2; ++j) {
      const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[j]));
      v[2 * j] = f.x;
      v[2 * j + 1] = f.y;
    }
  } else {
#pragma unroll
    for (int i = 0; i < E; ++i) v[i] = i < valid ? __bfloat162float(b[n + i]) : 0.f;
  }
}

// 16-byte vector (E elements) -> floats.
template <typename OutT, int E>
__device__ __forceinline__ void unpack_vec(const uint4 u, float (&v)[E]) {
  if constexpr (sizeof(OutT) == 2) {
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[j]));
      v[2 * j] = f.x;
      v[2 * j + 1] = f.y;
    }
  } else {
    v[0] = __uint_as_float(u.x); v[1] = __uint_as_float(u.y); v[2] = __uint_as_float(u.z); v[3] = __uint_as_float(u.w);
  }
}

// Geometry of one warp's epilogue stripe: lane (lr, lc) owns 16-byte column
// group lc of rows lr, lr + RPI, ... of each 32-column chunk.
template <typename OutT>
struct StripeGeo {
  static constexpr int E = 16 / sizeof(OutT);  // elements per lane per row
  static constexpr int LPR = 32 / E;           // lanes per row (4 | 8)
  static constexpr int RPI = 32 / LPR;         // rows per iteration (8 | 4)
  static constexpr int IT = 32 / RPI;          // row iterations per chunk
};

// Loads of the global operands an epilogue reads (dGeLU pre-activation,
// f32 accumulate of C) for chunk c into registers.
template <typename OutT, int EPI, bool ACC>
__device__ __forceinline__ void epi_prefetch(const TcParams& p, int c, int nbeg, int lc, int lr, int rows_left,
                                             long long lane_base, long long step,
                                             uint4 (&pa)[StripeGeo<OutT>::IT], uint4 (&pc)[StripeGeo<OutT>::IT]) {
  using G = StripeGeo<OutT>;
  const int n = nbeg + c * 32 + lc * G::E;
  const bool full = n + G::E <= p.N;  // partial groups use the scalar tail path
  // every element gets a value (zero where not loaded): no merge with stale
  // register contents, so the buffers never need to live in local memory
#pragma unroll
  for (int it = 0; it < G::IT; ++it) {
    const bool ok = full && it * G::RPI + lr < rows_left;
    const long long off = lane_base + nbeg + c * 32 + it * step;
    if constexpr (EPI == OASES_EPI_DGELU || EPI == OASES_EPI_MUL || EPI == OASES_EPI_ROWDOT) {
      pa[it] = make_uint4(0u, 0u, 0u, 0u);
      if (ok) pa[it] = __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const OutT*>(p.aux) + off));
    }
    if constexpr (ACC) {
      pc[it] = make_uint4(0u, 0u, 0u, 0u);
      if (ok) pc[it] = *reinterpret_cast<const uint4*>(reinterpret_cast<const OutT*>(p.c) + off);
    }
  }
}

// One 32-column chunk of a stripe: TMEM -> swizzled smem -> fused epilogue -> global.
template <typename OutT, int EPI, bool ACC>
__device__ __forceinline__ void epi_chunk(const TcParams& p, int c, int nbeg, long long row0, long long col0, int lr,
                                          int lc, int rows_left, long long step, uint32_t taddr, float4* stg, int lane,
                                          float (&racc)[StripeGeo<OutT>::IT], const uint4 (&pa)[StripeGeo<OutT>::IT],
                                          const uint4 (&pc)[StripeGeo<OutT>::IT]) {
  using G = StripeGeo<OutT>;
  constexpr int E = G::E, RPI = G::RPI, IT = G::IT;
  constexpr bool BIAS = EPI == OASES_EPI_BIAS || EPI == OASES_EPI_BIAS_GELU || EPI == OASES_EPI_BIAS_GELU_GRAD;
  constexpr bool RD = EPI == OASES_EPI_ROWDOT;
  constexpr bool DG = EPI == OASES_EPI_DGELU || EPI == OASES_EPI_MUL || RD;  // epilogues reading AUX
  constexpr bool CS = EPI == OASES_EPI_MUL;  // optional column-sum partials of the stored C
  const int nc = nbeg + c * 32;
  // pa / pc: the chunk's global operands, loaded by epilogue_stripe ahead of time
  {
    uint32_t r[32];
    tmem_ld32(taddr + static_cast<uint32_t>(c * 32), r);
    tmem_wait_ld();
    if (nc >= p.N) return;  // warp-uniform
#pragma unroll
    for (int j = 0; j < 8; ++j)
      stg[lane * 8 + (j ^ (lane & 7))] = make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                                                     __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3]));
  }
  __syncwarp();
  const int n = nc + lc * E;
  const int valid = p.N - n;  // elements of this lane's group inside the problem
  float cs[E];
#pragma unroll
  for (int i = 0; i < E; ++i) cs[i] = 0.f;
  if (valid > 0) {
    float b[E];
    if constexpr (BIAS) {
      if (p.bias) ld_bias<E>(reinterpret_cast<const __nv_bfloat16*>(p.bias), n, valid, b);
      else
#pragma unroll
        for (int i = 0; i < E; ++i) b[i] = 0.f;
    }
    OutT* cp = reinterpret_cast<OutT*>(p.c) + (row0 + lr) * p.ldc + col0 + n;
    const bool scale = p.alpha != 1.f;
#pragma unroll
    for (int it = 0; it < IT; ++it, cp += step) {
      const int row = it * RPI + lr;
      if (row >= rows_left) break;
      float v[E];
#pragma unroll
      for (int q = 0; q < E / 4; ++q) {
        const int ch = lc * (E / 4) + q;
        const float4 a = stg[row * 8 + (ch ^ (row & 7))];
        v[4 * q] = a.x; v[4 * q + 1] = a.y; v[4 * q + 2] = a.z; v[4 * q + 3] = a.w;
      }
      if (scale)
#pragma unroll
        for (int i = 0; i < E; ++i) v[i] *= p.alpha;
      if constexpr (BIAS)
#pragma unroll
        for (int i = 0; i < E; ++i) v[i] += b[i];
      const long long rel = cp - reinterpret_cast<OutT*>(p.c);
      if (valid >= E) {
        if constexpr (RD) {
          // C stored as is; its bf16 values dotted with AUX over this lane's columns
          float x[E];
          unpack_vec<OutT, E>(pa[it], x);
          float dsum = 0.f;
#pragma unroll
          for (int i = 0; i < E; ++i) dsum = fmaf(to_f(from_f<OutT>(v[i])), x[i], dsum);
          racc[it] += dsum;
        } else if constexpr (DG) {
          float x[E];
          unpack_vec<OutT, E>(pa[it], x);
#pragma unroll
          for (int i = 0; i < E; ++i) v[i] *= EPI == OASES_EPI_MUL ? x[i] : gelu_grad_fast(x[i]);
        }
        if constexpr (ACC) {
          float o[E];
          unpack_vec<OutT, E>(pc[it], o);
#pragma unroll
          for (int i = 0; i < E; ++i) v[i] += o[i];
        }
        if constexpr (CS)
#pragma unroll
          for (int i = 0; i < E; ++i) cs[i] += to_f(from_f<OutT>(v[i]));  // the value stored
        if constexpr (EPI == OASES_EPI_BIAS_GELU) {
          // C2 == null: only the activation is wanted (pre-activation dead), into C
          if (p.c2) st_vec<OutT, E>(cp, v);
#pragma unroll
          for (int i = 0; i < E; ++i) v[i] = gelu_fast(v[i]);
          st_vec<OutT, E>(p.c2 ? reinterpret_cast<OutT*>(p.c2) + rel : cp, v);
        } else if constexpr (EPI == OASES_EPI_BIAS_GELU_GRAD) {
          // C = gelu'(v) (what the dgrad epilogue multiplies by), C2 = gelu(v)
          float d[E];
#pragma unroll
          for (int i = 0; i < E; ++i) {
            float cdf, pdf;
            norm_cdf_pdf(v[i], cdf, pdf);
            d[i] = fmaf(v[i], pdf, cdf);
            v[i] *= cdf;
          }
          st_vec<OutT, E>(cp, d);
          st_vec<OutT, E>(reinterpret_cast<OutT*>(p.c2) + rel, v);
        } else {
          st_vec<OutT, E>(cp, v);
        }
      } else {
#pragma unroll
        for (int i = 0; i < E; ++i) {  // compile-time indices keep v[] in registers
          if (i >= valid) break;
          float x = v[i];
          if constexpr (EPI == OASES_EPI_DGELU) x *= gelu_grad_fast(to_f(reinterpret_cast<const OutT*>(p.aux)[rel + i]));
          if constexpr (EPI == OASES_EPI_MUL) x *= to_f(reinterpret_cast<const OutT*>(p.aux)[rel + i]);
          if constexpr (ACC) x += to_f(cp[i]);
          if constexpr (EPI == OASES_EPI_BIAS_GELU_GRAD) {
            cp[i] = from_f<OutT>(gelu_grad_fast(x));
            reinterpret_cast<OutT*>(p.c2)[rel + i] = from_f<OutT>(gelu_fast(x));
          } else if constexpr (EPI == OASES_EPI_BIAS_GELU) {
            if (p.c2) {
              cp[i] = from_f<OutT>(x);
              reinterpret_cast<OutT*>(p.c2)[rel + i] = from_f<OutT>(gelu_fast(x));
            } else {
              cp[i] = from_f<OutT>(gelu_fast(x));
            }
          } else {
            cp[i] = from_f<OutT>(x);
          }
        }
      }
    }
  }
  if constexpr (CS) {
    if (p.colsum) {  // N % 32 == 0 (host-checked): every lane's group is whole
      // reduce over the rows of the stripe (lanes of equal lc), fixed order
#pragma unroll
      for (int o = G::LPR; o < 32; o <<= 1)
#pragma unroll
        for (int i = 0; i < E; ++i) cs[i] += __shfl_xor_sync(0xffffffffu, cs[i], o);
      if (lr == 0) {
        float* dst = p.colsum + (row0 >> 5) * static_cast<long long>(p.N) + n;
#pragma unroll
        for (int i = 0; i < E; i += 4)
          *reinterpret_cast<float4*>(dst + i) = make_float4(cs[i], cs[i + 1], cs[i + 2], cs[i + 3]);
      }
    }
  }
  __syncwarp();
}

// One warp's 32-row x (32*NCH)-column stripe of an accumulator tile.
// TMEM -> registers (thread = row) -> 128B-swizzled smem staging -> each lane
// takes one 16-byte column group of a row, so a warp's global access covers
// 32/LPR full row segments -> fused epilogue -> global.
// Epilogues that READ global memory (the gelu' / pre-activation operand, the
// f32 accumulate of C) keep those loads a chunk ahead: chunk 0's are issued
// before waiting for the accumulator (tfull), chunk c+1's before chunk c is
// drained, so one DRAM latency per stripe is exposed instead of one per chunk
// (NCH chunks per tile: the per-tile epilogue latency is what the double-
// buffered accumulator must hide under the next tile's main loop).
template <typename OutT, int EPI, bool ACC, int NCH>
__device__ __forceinline__ void epilogue_stripe(const TcParams& p, int z, int m_base, int nbeg, uint32_t taddr,
                                                float4* stg, int lane, uint64_t* tfull, uint32_t tphase) {
  using G = StripeGeo<OutT>;
  const int zo = z / p.batch_inner, zi = z - zo * p.batch_inner;
  const long long row0 = p.c_row_off[0] * zo + p.c_row_off[1] * zi + m_base;
  const long long col0 = p.c_col_off[0] * zo + p.c_col_off[1] * zi;
  const int lr = lane / G::LPR, lc = lane % G::LPR;
  const int rows_left = p.M - m_base;  // rows of this stripe inside the problem
  const long long step = static_cast<long long>(G::RPI) * p.ldc;
  const long long lane_base = (row0 + lr) * p.ldc + col0 + lc * G::E;  // element offset of (row lr, column 0)
  float racc[G::IT];
#pragma unroll
  for (int it = 0; it < G::IT; ++it) racc[it] = 0.f;
  constexpr bool LD = EPI == OASES_EPI_DGELU || EPI == OASES_EPI_MUL || EPI == OASES_EPI_ROWDOT || ACC;
  uint4 pa[G::IT], pc[G::IT];
  if constexpr (LD) epi_prefetch<OutT, EPI, ACC>(p, 0, nbeg, lc, lr, rows_left, lane_base, step, pa, pc);
  mbar_wait(tfull, tphase);
  tc_fence_after();
  auto rowdot_flush = [&](int c) {
    if constexpr (EPI == OASES_EPI_ROWDOT) {
      const int cend = static_cast<int>(col0) + nbeg + (c + 1) * 32;  // column after this chunk
      if (cend % p.rd_group == 0 && cend <= p.N) {
        // the group (head) ends here: reduce over the LPR lanes of each row, one lane writes
        const int g = (cend - 1) / p.rd_group;
#pragma unroll
        for (int it = 0; it < G::IT; ++it) {
          float t = racc[it];
#pragma unroll
          for (int o = 1; o < G::LPR; o <<= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
          const int row = it * G::RPI + lr;
          if (lc == 0 && row < rows_left) {
            const long long m = row0 + row;
            const long long smp = m / p.rd_seq, i = m - smp * p.rd_seq;
            p.rowdot[(smp * p.rd_heads + g) * p.rd_seq + i] = t;
          }
          racc[it] = 0.f;
        }
      }
    }
  };
  // bf16 operands (4 vectors) run a chunk ahead in two named buffers (chunks in
  // pairs); the f32 accumulate of C (8 vectors) would not fit twice in the
  // register budget and is loaded at the start of its chunk
  constexpr bool PIPE = LD && !ACC && NCH % 2 == 0;
  if constexpr (PIPE) {
    uint4 qa[G::IT], qc[G::IT];
#pragma unroll 1
    for (int c = 0; c < NCH; c += 2) {
      epi_prefetch<OutT, EPI, ACC>(p, c + 1, nbeg, lc, lr, rows_left, lane_base, step, qa, qc);
      epi_chunk<OutT, EPI, ACC>(p, c, nbeg, row0, col0, lr, lc, rows_left, step, taddr, stg, lane, racc, pa, pc);
      rowdot_flush(c);
      if (c + 2 < NCH) epi_prefetch<OutT, EPI, ACC>(p, c + 2, nbeg, lc, lr, rows_left, lane_base, step, pa, pc);
      epi_chunk<OutT, EPI, ACC>(p, c + 1, nbeg, row0, col0, lr, lc, rows_left, step, taddr, stg, lane, racc, qa, qc);
      rowdot_flush(c + 1);
    }
  } else {
#pragma unroll 1
    for (int c = 0; c < NCH; ++c) {
      if constexpr (LD)
        if (c > 0) epi_prefetch<OutT, EPI, ACC>(p, c, nbeg, lc, lr, rows_left, lane_base, step, pa, pc);
      epi_chunk<OutT, EPI, ACC>(p, c, nbeg, row0, col0, lr, lc, rows_left, step, taddr, stg, lane, racc, pa, pc);
      rowdot_flush(c);
    }
  }
}

// Calls BODY(OutT, EPI, ACC) for the runtime mode of p (compile-time specialised).
#define OASES_EPI_DISPATCH(p, BODY)                                                       \
  do {                                                                                    \
    const int mode_ = ((p).c_f32 ? 16 : 0) + (p).epilogue * 2 + ((p).accumulate ? 1 : 0); \
    switch (mode_) {                                                                      \
      case 0: BODY(__nv_bfloat16, 0, false); break;                                       \
      case 2: BODY(__nv_bfloat16, 1, false); break;                                       \
      case 4: BODY(__nv_bfloat16, 2, false); break;                                       \
      case 6: BODY(__nv_bfloat16, 3, false); break;                                       \
      case 8: BODY(__nv_bfloat16, 4, false); break;                                       \
      case 10: BODY(__nv_bfloat16, 5, false); break;                                      \
      case 12: BODY(__nv_bfloat16, 6, false); break;                                      \
      case 16: BODY(float, 0, false); break;                                              \
      case 17: BODY(float, 0, true); break;                                               \
      case 18: BODY(float, 1, false); break;                                              \
      default: BODY(float, 1, true); break;                                               \
    }                                                                                     \
  } while (0)

// ----------------------------------------------------------------- single-CTA kernel
template <typename OutT, int EPI, bool ACC, int BN>
__device__ __forceinline__ void epilogue_role_single(const TcParams& p, uint64_t* tfull, uint64_t* tempty,
                                                     uint32_t tmem_base, float4* stg, int warp, int lane) {
  const int q = warp & 3;            // TMEM lane quarter this warp may access
  const int half = (warp - 2) >> 2;  // which half of the tile's columns
  const int total = p.batch * p.tiles_m * p.tiles_n;
  int acc = 0;
  uint32_t acc_phase = 0;
  for (int r = 0, t = sched_tile(p, 0); t < total; t = sched_tile(p, ++r)) {
    TileInfo ti;
    if (!decode_tile<BN>(p, t, ti)) continue;
    const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) +
                           static_cast<uint32_t>(acc * BN + half * (BN / 2));
    epilogue_stripe<OutT, EPI, ACC, BN / 64>(p, ti.z, ti.m0 + q * 32, ti.n0 + half * (BN / 2), taddr, stg, lane,
                                             &tfull[acc], acc_phase);
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(&tempty[acc]);
    if (++acc == 2) { acc = 0; acc_phase ^= 1; }
  }
}

template <int BN, int A_MN, int B_MN>
__global__ void __launch_bounds__(THREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
                   const TcParams p) {
  pdl_trigger();
  using Cfg = TcCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  // Statically shared staging so the compiler emits STS/LDS (a generic-pointer
  // LD after STG stalls on store ordering).
  __shared__ __align__(16) float4 stg_all[STG_FLOAT4];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::STAGES * Cfg::STAGE_BYTES);
  uint64_t* empty = full + Cfg::STAGES;
  uint64_t* tfull = empty + Cfg::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int total_tiles = p.batch * p.tiles_m * p.tiles_n;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tma_a);
    tma_prefetch(&tma_b);
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], EPI_WARPS);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();

  if (warp == 0) {
    // ------------------------------------------------ TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int r = 0, t = sched_tile(p, 0); t < total_tiles; t = sched_tile(p, ++r)) {
        TileInfo ti;
        if (!decode_tile<BN>(p, t, ti)) continue;
        const int zo = ti.z / p.batch_inner, zi = ti.z - zo * p.batch_inner;
        const int ax = p.a_x_off[0] * zo + p.a_x_off[1] * zi;
        const int ay = p.a_y_off[0] * zo + p.a_y_off[1] * zi;
        const int bx = p.b_x_off[0] * zo + p.b_x_off[1] * zi;
        const int by = p.b_y_off[0] * zo + p.b_y_off[1] * zi;
        for (int kb = ti.kb0; kb < ti.kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], Cfg::STAGE_BYTES);
          uint8_t* sa = smem + stage * Cfg::STAGE_BYTES;
          uint8_t* sb = sa + Cfg::A_BYTES;
          const int k0 = kb * BK;
          if (A_MN) {
#pragma unroll
            for (int j = 0; j < BM / 64; ++j)
              tma_load_2d(sa + j * 8192, &tma_a, &full[stage], ax + ti.m0 + 64 * j, ay + k0);
          } else {
            tma_load_2d(sa, &tma_a, &full[stage], ax + k0, ay + ti.m0);
          }
          if (B_MN) {
#pragma unroll
            for (int j = 0; j < BN / 64; ++j)
              tma_load_2d(sb + j * 8192, &tma_b, &full[stage], bx + ti.n0 + 64 * j, by + k0);
          } else {
            tma_load_2d(sb, &tma_b, &full[stage], bx + k0, by + ti.n0);
          }
          if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(BM, BN, A_MN, B_MN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      const uint32_t smem_base = smem_u32(smem);
      for (int r = 0, t = sched_tile(p, 0); t < total_tiles; t = sched_tile(p, ++r)) {
        TileInfo ti;
        if (!decode_tile<BN>(p, t, ti)) continue;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * BN);
        for (int kb = ti.kb0; kb < ti.kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_base + stage * Cfg::STAGE_BYTES;
          const uint32_t sb = sa + Cfg::A_BYTES;
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            const uint64_t adesc = A_MN ? umma_desc_sw128(sa + kk * 2048, 8192, 1024)
                                        : umma_desc_sw128(sa + kk * 32, 16, 1024);
            const uint64_t bdesc = B_MN ? umma_desc_sw128(sb + kk * 2048, 8192, 1024)
                                        : umma_desc_sw128(sb + kk * 32, 16, 1024);
            umma_bf16(d_tmem, adesc, bdesc, idesc, (kb > ti.kb0 || kk > 0) ? 1u : 0u);
          }
          umma_commit(&empty[stage]);
          if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1; }
        }
        umma_commit(&tfull[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else {
    // ------------------------------------------------ epilogue (warps 2..9)
    float4* stg = stg_all + (warp - 2) * 256;
#define OASES_SINGLE_BODY(T, E, A) epilogue_role_single<T, E, A, BN>(p, tfull, tempty, tmem_base, stg, warp, lane)
    OASES_EPI_DISPATCH(p, OASES_SINGLE_BODY);
#undef OASES_SINGLE_BODY
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
  }
}

// ----------------------------------------------------------------- CTA-pair kernel
// cta_group::2 variant for large non-causal GEMMs: a cluster of 2 CTAs on one
// TPC computes a 256 x 256 tile. Each CTA stages its own 128-row half of A and
// 128-row half of B (TMA completion counted on the leader's barrier); the
// leader's single thread issues tcgen05.mma.cta_group::2 (M = 256) reading
// both CTAs' smem. Accumulators: 2 x 256 TMEM columns per CTA. Causal K ranges
// are defined at 128-row granularity, so attention stays on the single-CTA kernel.
constexpr int PAIR_BM = 256, PAIR_BN = 256, PAIR_STAGES = 6;
constexpr int PAIR_HALF_BYTES = 128 * BK * 2;          // 16 KB
constexpr int PAIR_STAGE_BYTES = 2 * PAIR_HALF_BYTES;  // A half + B half
constexpr int PAIR_SMEM = PAIR_STAGES * PAIR_STAGE_BYTES + 256 + 1024;  // + 32 KB static staging
constexpr uint32_t PAIR_TMEM_COLS = 512;

// Tile order: groups of PAIR_GROUP_M m-tiles walked n-major inside the group,
// so the ~74 tiles in flight at once share a few A and B panels (a wave
// touches ~8 A + ~9 B panels instead of 2-3 A + every B panel). Keeps the
// operand panels L2-resident across waves: DRAM traffic stays near A + B + C
// once even when B is larger than the L2 share it gets (wgrad: B = 64 MB).
constexpr int PAIR_GROUP_M = 8;
__device__ __forceinline__ void pair_decode(const TcParams& p, int t, int& z, int& m0, int& n0) {
  const int per_z = p.tiles_m * p.tiles_n;
  z = t / per_z;
  const int r = t - z * per_z;
  const int group = PAIR_GROUP_M * p.tiles_n;
  const int grp = r / group;
  const int first_m = grp * PAIR_GROUP_M;
  const int gm = min(PAIR_GROUP_M, p.tiles_m - first_m);
  const int idx = r - grp * group;
  m0 = (first_m + idx % gm) * PAIR_BM;
  n0 = (idx / gm) * PAIR_BN;
}

// Up to two independent GEMM problems in one persistent launch (a "group"):
// their tiles form one list (problem 0 first, the host puts the problem with
// the longer K first), walked with the usual static pair striding. Used for
// the backward's dgrad + wgrad pairs, which read the same gradient and are
// independent: together they fill the 74 CTA pairs' waves far better than
// either alone. Operand majorness is a runtime property of each problem.
struct TcGroup {
  TcParams p[2];
  int a_mn[2], b_mn[2];
  int tiles0, total;
};

__device__ __forceinline__ int group_tile(const TcGroup& g, int t, int& lt) {
  if (t < g.tiles0) {
    lt = t;
    return 0;
  }
  lt = t - g.tiles0;
  return 1;
}

template <typename OutT, int EPI, bool ACC>
__device__ __forceinline__ void pair_tile_epilogue(const TcParams& p, int lt, uint32_t taddr, float4* stg, int q,
                                                   int half, int lane, uint32_t rank, uint64_t* tfull,
                                                   uint32_t tphase) {
  int z, m0, n0;
  pair_decode(p, lt, z, m0, n0);
  const int mb = m0 + static_cast<int>(rank) * 128 + q * 32;
  epilogue_stripe<OutT, EPI, ACC, PAIR_BN / 64>(p, z, mb, n0 + half * (PAIR_BN / 2), taddr, stg, lane, tfull, tphase);
}

// Producer: TMA of one k-block of a tile (compile-time operand layout).
template <int A_MN, int B_MN>
__device__ __forceinline__ void pair_load(uint8_t* sa, uint8_t* sb, const CUtensorMap* tma_a, const CUtensorMap* tma_b,
                                          uint64_t* bar, int ax, int ay, int bx, int by, int am, int bn, int k0) {
  if (A_MN) {
    tma_load_2d_pair(sa, tma_a, bar, ax + am, ay + k0);
    tma_load_2d_pair(sa + 8192, tma_a, bar, ax + am + 64, ay + k0);
  } else {
    tma_load_2d_pair(sa, tma_a, bar, ax + k0, ay + am);
  }
  if (B_MN) {
    tma_load_2d_pair(sb, tma_b, bar, bx + bn, by + k0);
    tma_load_2d_pair(sb + 8192, tma_b, bar, bx + bn + 64, by + k0);
  } else {
    tma_load_2d_pair(sb, tma_b, bar, bx + k0, by + bn);
  }
}

// MMA issuer: all k-blocks of one tile into the TMEM accumulator d_tmem.
template <int A_MN, int B_MN>
__device__ __forceinline__ void pair_mma_tile(uint32_t smem_base, uint64_t* full, uint64_t* empty, int& stage,
                                              uint32_t& phase, uint32_t d_tmem, int kblocks) {
  constexpr uint32_t idesc = umma_idesc_bf16(PAIR_BM, PAIR_BN, A_MN, B_MN);
  for (int kb = 0; kb < kblocks; ++kb) {
    mbar_wait(&full[stage], phase);
    tc_fence_after();
    const uint32_t sa = smem_base + stage * PAIR_STAGE_BYTES;
    const uint32_t sb = sa + PAIR_HALF_BYTES;
#pragma unroll
    for (int kk = 0; kk < BK / 16; ++kk) {
      const uint64_t adesc = A_MN ? umma_desc_sw128(sa + kk * 2048, 8192, 1024) : umma_desc_sw128(sa + kk * 32, 16, 1024);
      const uint64_t bdesc = B_MN ? umma_desc_sw128(sb + kk * 2048, 8192, 1024) : umma_desc_sw128(sb + kk * 32, 16, 1024);
      umma_bf16_pair(d_tmem, adesc, bdesc, idesc, (kb > 0 || kk > 0) ? 1u : 0u);
    }
    umma_commit_pair(&empty[stage], 0x3);
    if (++stage == PAIR_STAGES) { stage = 0; phase ^= 1; }
  }
}

// Operand layouts are template parameters per problem slot (A0,B0 | A1,B1): a
// single problem instantiates A1 = A0, B1 = B0; the backward's wgrad + dgrad
// group is <1,1,0,1>.
template <int A0, int B0, int A1, int B1>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
    gemm_tc2_kernel(const __grid_constant__ CUtensorMap ta0, const __grid_constant__ CUtensorMap tb0,
                    const __grid_constant__ CUtensorMap ta1, const __grid_constant__ CUtensorMap tb1,
                    const TcGroup g) {
  pdl_trigger();
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(16) float4 stg_all[STG_FLOAT4];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + PAIR_STAGES * PAIR_STAGE_BYTES);
  uint64_t* empty = full + PAIR_STAGES;
  uint64_t* tfull = empty + PAIR_STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int total_tiles = g.total;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&ta0);
    tma_prefetch(&tb0);
    if (g.total > g.tiles0) {
      tma_prefetch(&ta1);
      tma_prefetch(&tb1);
    }
    for (int s = 0; s < PAIR_STAGES; ++s) {
      mbar_init(&full[s], 1);   // leader's arrive.expect_tx; both CTAs' TMA bytes
      mbar_init(&empty[s], 1);  // multicast commit from the leader's MMA
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 2 * EPI_WARPS);  // epilogue warps of both CTAs (leader's copy is used)
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_pair(tmem_slot, PAIR_TMEM_COLS);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();  // the previous kernel's outputs (our operands) are complete from here on

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = pair; t < total_tiles; t += npairs) {
        int lt;
        const int pi = group_tile(g, t, lt);
        const TcParams& p = g.p[pi];
        int z, m0, n0;
        pair_decode(p, lt, z, m0, n0);
        const int zo = z / p.batch_inner, zi = z - zo * p.batch_inner;
        const int ax = p.a_x_off[0] * zo + p.a_x_off[1] * zi, ay = p.a_y_off[0] * zo + p.a_y_off[1] * zi;
        const int bx = p.b_x_off[0] * zo + p.b_x_off[1] * zi, by = p.b_y_off[0] * zo + p.b_y_off[1] * zi;
        const int am = m0 + static_cast<int>(rank) * 128, bn = n0 + static_cast<int>(rank) * 128;
        for (int kb = 0; kb < p.kblocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (leader) mbar_arrive_expect_tx(&full[stage], 2 * PAIR_STAGE_BYTES);
          uint8_t* sa = smem + stage * PAIR_STAGE_BYTES;
          uint8_t* sb = sa + PAIR_HALF_BYTES;
          if (pi == 0)
            pair_load<A0, B0>(sa, sb, &ta0, &tb0, &full[stage], ax, ay, bx, by, am, bn, kb * BK);
          else
            pair_load<A1, B1>(sa, sb, &ta1, &tb1, &full[stage], ax, ay, bx, by, am, bn, kb * BK);
          if (++stage == PAIR_STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      const uint32_t smem_base = smem_u32(smem);
      for (int t = pair; t < total_tiles; t += npairs) {
        int lt;
        const int pi = group_tile(g, t, lt);
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * PAIR_BN);
        if (pi == 0)
          pair_mma_tile<A0, B0>(smem_base, full, empty, stage, phase, d_tmem, g.p[0].kblocks);
        else
          pair_mma_tile<A1, B1>(smem_base, full, empty, stage, phase, d_tmem, g.p[1].kblocks);
        umma_commit_pair(&tfull[acc], 0x3);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else {
    // ------------------------------------------------ epilogue (warps 2..9), per-tile mode dispatch
    float4* stg = stg_all + (warp - 2) * 256;
    const int q = warp & 3, half = (warp - 2) >> 2;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = pair; t < total_tiles; t += npairs) {
      int lt;
      const int pi = group_tile(g, t, lt);
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) +
                             static_cast<uint32_t>(acc * PAIR_BN + half * (PAIR_BN / 2));
      // static problem index: the parameters stay constant-bank operands
      if (pi == 0) {
#define OASES_PAIR_BODY(T, E, A) \
  pair_tile_epilogue<T, E, A>(g.p[0], lt, taddr, stg, q, half, lane, rank, &tfull[acc], acc_phase)
        OASES_EPI_DISPATCH(g.p[0], OASES_PAIR_BODY);
#undef OASES_PAIR_BODY
      } else {
#define OASES_PAIR_BODY(T, E, A) \
  pair_tile_epilogue<T, E, A>(g.p[1], lt, taddr, stg, q, half, lane, rank, &tfull[acc], acc_phase)
        OASES_EPI_DISPATCH(g.p[1], OASES_PAIR_BODY);
#undef OASES_PAIR_BODY
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_leader(&tempty[acc]);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  }

  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, PAIR_TMEM_COLS);
  }
}

// ----------------------------------------------------------------- host side
PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess) {
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    }
  });
  return fn;
}

bool make_map(CUtensorMap* map, const oases_gemm_operand& o, uint32_t box_inner, uint32_t box_outer,
              std::string* err) {
  return make_tma_bf16_2d(map, o.ptr, o.rows, o.cols, o.ld, box_inner, box_outer, err);
}

template <int BN, int A_MN, int B_MN>
cudaError_t launch_tc(const CUtensorMap& ma, const CUtensorMap& mb, const TcParams& p, int grid,
                      cudaStream_t stream) {
  using Cfg = TcCfg<BN>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(gemm_tc_kernel<BN, A_MN, B_MN>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  return launch_pdl(gemm_tc_kernel<BN, A_MN, B_MN>, dim3(grid), dim3(THREADS), Cfg::SMEM, stream, ma, mb, p);
}

template <int A0, int B0, int A1, int B1>
cudaError_t launch_group_t(const CUtensorMap (&maps)[4], const TcGroup& g, int grid, cudaStream_t stream) {
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(gemm_tc2_kernel<A0, B0, A1, B1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         PAIR_SMEM);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  return launch_pdl(gemm_tc2_kernel<A0, B0, A1, B1>, dim3(grid), dim3(THREADS), PAIR_SMEM, stream, maps[0], maps[1],
                    maps[2], maps[3], g);
}

// false: no instantiation for this combination of operand layouts
bool launch_group(const CUtensorMap (&maps)[4], const TcGroup& g, int grid, cudaStream_t stream, cudaError_t* e) {
  const int key = g.a_mn[0] * 8 + g.b_mn[0] * 4 + g.a_mn[1] * 2 + g.b_mn[1];
  switch (key) {
    case 0: *e = launch_group_t<0, 0, 0, 0>(maps, g, grid, stream); return true;
    case 5: *e = launch_group_t<0, 1, 0, 1>(maps, g, grid, stream); return true;
    case 10: *e = launch_group_t<1, 0, 1, 0>(maps, g, grid, stream); return true;
    case 15: *e = launch_group_t<1, 1, 1, 1>(maps, g, grid, stream); return true;
    case 13: *e = launch_group_t<1, 1, 0, 1>(maps, g, grid, stream); return true;  // wgrad + dgrad
    case 7: *e = launch_group_t<0, 1, 1, 1>(maps, g, grid, stream); return true;   // dgrad + wgrad
    default: return false;
  }
}

template <int BN>
cudaError_t dispatch_major(int a_mn, int b_mn, const CUtensorMap& ma, const CUtensorMap& mb, const TcParams& p,
                           int grid, cudaStream_t s) {
  if (!a_mn && !b_mn) return launch_tc<BN, 0, 0>(ma, mb, p, grid, s);
  if (!a_mn && b_mn) return launch_tc<BN, 0, 1>(ma, mb, p, grid, s);
  if (a_mn && !b_mn) return launch_tc<BN, 1, 0>(ma, mb, p, grid, s);
  return launch_tc<BN, 1, 1>(ma, mb, p, grid, s);
}

// OASES_GEMM_PAIR=0 forces the single-CTA kernel (A/B comparisons).
bool use_pairs() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("OASES_GEMM_PAIR");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

int sm_count() {
  static int n = -1;
  if (n < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) n = 148;
  }
  return n;
}

}  // namespace

bool make_tma_bf16_2d(CUtensorMap* map, const void* ptr, int64_t rows, int64_t cols, int64_t ld, uint32_t box_inner,
                      uint32_t box_outer, std::string* err) {
  auto enc = get_encode();
  if (!enc) {
    *err = "cuTensorMapEncodeTiled unavailable";
    return false;
  }
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 2};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    *err = "cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(r)) + ")";
    return false;
  }
  return true;
}

namespace {

struct Prepared {
  TcParams p;
  CUtensorMap ma, mb;
  bool pair;
  int BN;
  long long tiles;
};

// Validation + TMA maps + kernel parameters for one problem.
bool prepare(const oases_gemm_desc& d, Prepared& out, std::string* err) {
  // Shape / alignment checks: TMA needs 16 B aligned strides and bases; the
  // vectorised epilogue needs 16 B aligned output rows.
  auto aligned = [](const void* p, int a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; };
  if (d.a.ld % 8 || d.b.ld % 8 || !aligned(d.a.ptr, 16) || !aligned(d.b.ptr, 16)) {
    *err = "gemm_tc: operand base/ld must be 16-byte aligned (ld % 8 == 0)";
    return false;
  }
  if (d.ldc % 8 || !aligned(d.c, 16) || (d.c_col_off[0] % 8) || (d.c_col_off[1] % 8) ||
      (d.c2 && !aligned(d.c2, 16)) || (d.aux && !aligned(d.aux, 16)) || (d.bias && !aligned(d.bias, 16))) {
    *err = "gemm_tc: output/aux/bias bases, ld and column offsets must be 16-byte aligned";
    return false;
  }
  if (d.M <= 0 || d.N <= 0 || d.K <= 0 || d.batch <= 0 || d.batch_inner <= 0) {
    *err = "gemm_tc: empty problem";
    return false;
  }
  if (d.epilogue == OASES_EPI_ROWDOT &&
      (!d.rowdot || !d.aux || d.c_dtype == OASES_F32 || d.rowdot_group <= 0 || d.rowdot_group % 32 ||
       d.N % d.rowdot_group || d.rowdot_seq <= 0 || d.M % d.rowdot_seq || d.batch != 1 ||
       d.N != static_cast<int64_t>(d.rowdot_group) * d.rowdot_heads)) {
    *err = "gemm_tc: ROWDOT needs bf16 C, AUX, rowdot, unbatched, N = heads*group (group % 32 == 0), M % seq == 0";
    return false;
  }
  if (d.colsum && (d.epilogue != OASES_EPI_MUL || d.batch != 1 || d.N % 32 || d.c_row_off[0] || d.c_row_off[1] ||
                   (reinterpret_cast<uintptr_t>(d.colsum) % 16))) {
    *err = "gemm_tc: COLSUM partials need the MUL epilogue, unbatched, N % 32 == 0, no row offsets, 16 B aligned";
    return false;
  }
  if (d.epilogue < OASES_EPI_NONE || d.epilogue > OASES_EPI_ROWDOT) {
    *err = "gemm_tc: unknown epilogue";
    return false;
  }
  // Instantiated epilogue modes (OASES_EPI_DISPATCH): bf16 output without
  // accumulation (any epilogue); f32 output with NONE or BIAS, +-accumulate.
  if (d.c_dtype != OASES_F32 && d.accumulate) {
    *err = "gemm_tc: accumulate needs an f32 output";
    return false;
  }
  if (d.c_dtype == OASES_F32 && d.epilogue != OASES_EPI_NONE && d.epilogue != OASES_EPI_BIAS) {
    *err = "gemm_tc: f32 output supports the NONE and BIAS epilogues only";
    return false;
  }
  const int BN = (d.N <= 128) ? 128 : 256;
  // Reads past the logical K would pull in neighbouring data (TMA zero-fills
  // only at the storage edge): K must be a multiple of 64 unless it spans the
  // whole storage extent of both operands. M/N tails are masked in the epilogue.
  if (d.K % BK) {
    const int64_t ka = d.a.mn_major ? d.a.rows : d.a.cols;
    const int64_t kb = d.b.mn_major ? d.b.rows : d.b.cols;
    if (d.batch > 1 || ka != d.K || kb != d.K) {
      *err = "gemm_tc: K % 64 != 0 requires K to span both operands' full extent (unbatched)";
      return false;
    }
  }
  if (d.causal != OASES_CAUSAL_NONE && d.M != d.K && d.causal != OASES_CAUSAL_SKIP_UPPER) {
    *err = "gemm_tc: causal K-range modes need M == K";
    return false;
  }
  const bool pair = use_pairs() && d.causal == OASES_CAUSAL_NONE && d.M > BM && d.N > 128;
  if (d.epilogue == OASES_EPI_ROWDOT && ((pair ? PAIR_BN / 2 : BN / 2) % d.rowdot_group)) {
    // each epilogue warp reduces its own column stripe: a group must not straddle two
    *err = "gemm_tc: ROWDOT groups must tile the epilogue stripe (" + std::to_string(pair ? PAIR_BN / 2 : BN / 2) +
           " columns)";
    return false;
  }
  if (!make_map(&out.ma, d.a, 64, d.a.mn_major ? 64 : BM, err)) return false;
  if (!make_map(&out.mb, d.b, 64, d.b.mn_major ? 64 : (pair ? 128 : BN), err)) return false;
  TcParams& p = out.p;
  p = TcParams{};
  p.M = static_cast<int>(d.M);
  p.N = static_cast<int>(d.N);
  p.K = static_cast<int>(d.K);
  p.batch = static_cast<int>(d.batch);
  p.batch_inner = static_cast<int>(d.batch_inner);
  const int tm = pair ? PAIR_BM : BM, tn = pair ? PAIR_BN : BN;
  p.tiles_m = static_cast<int>((d.M + tm - 1) / tm);
  p.tiles_n = static_cast<int>((d.N + tn - 1) / tn);
  p.kblocks = static_cast<int>((d.K + BK - 1) / BK);
  for (int i = 0; i < 2; ++i) {
    p.a_x_off[i] = static_cast<int>(d.a.col_off[i]);
    p.a_y_off[i] = static_cast<int>(d.a.row_off[i]);
    p.b_x_off[i] = static_cast<int>(d.b.col_off[i]);
    p.b_y_off[i] = static_cast<int>(d.b.row_off[i]);
    p.c_row_off[i] = d.c_row_off[i];
    p.c_col_off[i] = d.c_col_off[i];
  }
  p.c = d.c;
  p.c2 = d.c2;
  p.aux = d.aux;
  p.rowdot = d.rowdot;
  p.rd_group = d.rowdot_group;
  p.rd_seq = d.rowdot_seq;
  p.rd_heads = d.rowdot_heads;
  p.colsum = d.colsum;
  p.bias = d.bias;
  p.ldc = d.ldc;
  p.c_f32 = d.c_dtype == OASES_F32;
  p.epilogue = d.epilogue;
  p.causal = d.causal;
  {
    static const bool zz = [] {
      const char* e = std::getenv("OASES_GEMM_ZIGZAG");
      return !(e && e[0] == '0');
    }();
    p.zigzag = zz && (d.causal == OASES_CAUSAL_K_UPTO_M || d.causal == OASES_CAUSAL_K_FROM_M);
  }
  p.accumulate = d.accumulate;
  p.alpha = d.alpha;
  out.pair = pair;
  out.BN = BN;
  out.tiles = static_cast<long long>(p.batch) * p.tiles_m * p.tiles_n;
  return true;
}

GemmStatus launch_status(cudaError_t e) {
  GemmStatus st;
  if (e != cudaSuccess) {
    st.err = std::string("gemm_tc launch: ") + cudaGetErrorString(e);
    st.cuda = true;
    return st;
  }
  st.ok = true;
  return st;
}

int grid_cap(int max_ctas) {
  int grid = sm_count();
  if (max_ctas > 0 && max_ctas < grid) grid = max_ctas;
  return grid;
}

GemmStatus launch_pairs(const oases_gemm_desc* const* ds, const Prepared* const* pr, int n, int max_ctas,
                        cudaStream_t stream) {
  TcGroup g{};
  CUtensorMap maps[4];
  long long total = 0;
  for (int i = 0; i < 2; ++i) {
    const int k = i < n ? i : 0;  // a group of one repeats its maps in the unused slots
    g.p[i] = pr[k]->p;
    g.a_mn[i] = ds[k]->a.mn_major ? 1 : 0;
    g.b_mn[i] = ds[k]->b.mn_major ? 1 : 0;
    maps[2 * i] = pr[k]->ma;
    maps[2 * i + 1] = pr[k]->mb;
  }
  for (int i = 0; i < n; ++i) total += pr[i]->tiles;
  g.tiles0 = static_cast<int>(pr[0]->tiles);
  g.total = static_cast<int>(total);
  int pairs = grid_cap(max_ctas) / 2;
  if (pairs < 1) pairs = 1;
  if (total < pairs) pairs = static_cast<int>(total);
  cudaError_t e = cudaSuccess;
  if (!launch_group(maps, g, 2 * pairs, stream, &e)) {
    GemmStatus st;
    st.err = "gemm_tc: no grouped kernel for this operand-layout combination";
    return st;
  }
  return launch_status(e);
}

}  // namespace

GemmStatus gemm_tc(const oases_gemm_desc& d, cudaStream_t stream) {
  GemmStatus st;
  Prepared pr;
  if (!prepare(d, pr, &st.err)) return st;
  if (pr.pair) {
    const oases_gemm_desc* ds[1] = {&d};
    const Prepared* ps[1] = {&pr};
    return launch_pairs(ds, ps, 1, d.max_ctas, stream);
  }
  int grid = grid_cap(d.max_ctas);
  if (pr.tiles < grid) grid = static_cast<int>(pr.tiles);
  const cudaError_t e = pr.BN == 128 ? dispatch_major<128>(d.a.mn_major, d.b.mn_major, pr.ma, pr.mb, pr.p, grid, stream)
                                     : dispatch_major<256>(d.a.mn_major, d.b.mn_major, pr.ma, pr.mb, pr.p, grid, stream);
  return launch_status(e);
}

GemmStatus gemm_tc_group(const oases_gemm_desc* d, int n, cudaStream_t stream) {
  GemmStatus st;
  if (n == 2) {
    Prepared a, b;
    if (!prepare(d[0], a, &st.err) || !prepare(d[1], b, &st.err)) return st;
    // instantiated mixed groups: (wgrad: MN/MN) with (dgrad: K/MN), either order
    const int ka = (d[0].a.mn_major ? 2 : 0) + (d[0].b.mn_major ? 1 : 0);
    const int kb = (d[1].a.mn_major ? 2 : 0) + (d[1].b.mn_major ? 1 : 0);
    const bool supported = ka == kb || (ka == 3 && kb == 1) || (ka == 1 && kb == 3);
    if (a.pair && b.pair && supported) {
      // longer-K problem first: its tiles are the heavier ones in the shared list
      const bool swap = b.p.kblocks > a.p.kblocks;
      const oases_gemm_desc* ds[2] = {swap ? &d[1] : &d[0], swap ? &d[0] : &d[1]};
      const Prepared* ps[2] = {swap ? &b : &a, swap ? &a : &b};
      return launch_pairs(ds, ps, 2, d[0].max_ctas, stream);
    }
  }
  for (int i = 0; i < n; ++i) {
    st = gemm_tc(d[i], stream);
    if (!st.ok) return st;
  }
  st.ok = true;
  return st;
}

}  // namespace oases
