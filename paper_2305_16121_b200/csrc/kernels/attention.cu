// Fused causal self-attention on tcgen05 (bf16, head_dim 64 | 128, seq % 128 == 0).
//
// The reference's attention (proj/src/numerics.cpp, the per-head
// softmax(Q K^T / sqrt(d)) V of the TMP layer, with attention dropout on the
// probabilities) is computed here without materialising the [seq, seq]
// probability matrix in HBM:
//
//   attn_fwd_kernel   persistent (one CTA per SM, zigzag order over (sample x
//                     local head, 128-query tile) items). S_j = Q K_j^T into
//                     three TMEM buffers, issued two KV tiles ahead; online
//                     softmax in registers (one query row per thread, 16 warps:
//                     4 per TMEM lane quarter x 32 key columns, row max / sum
//                     exchanged through smem), the dropout keep-mask of
//                     DESIGN.md "Dropout keys" applied to the unnormalised
//                     probabilities; P_j (bf16) written back over S_j in TMEM
//                     and consumed from there by the TS-form MMA O += P_j V_j
//                     (O rescaled in place only when the running max grows by
//                     more than 8). Writes ctx (bf16), the row log-sum-exp
//                     (log2 domain, f32) and optionally the keep bits.
//                     Warps: 0 Q/K TMA, 1 MMA issuer + TMEM owner, 2 V TMA,
//                     3..18 softmax.
//   attn_dsum_kernel  D_i = sum_d dO_i,d * O_i,d  (= sum_j P_ij dP_ij), when the
//                     dO-producing GEMM did not emit it (EPI_ROWDOT).
//   attn_dkdv_kernel  one CTA per (sample x head, 128-key tile), streaming the
//                     query tiles at or below the diagonal: S = Q K^T and
//                     dP_drop = dO V^T into TMEM, P = exp2(S - lse), the
//                     dropped P -> smem -> dV += P_drop^T dO; dS = P o (dP - D)
//                     -> smem -> dK += dS^T Q. dS is also TMA-stored to HBM so
//                     dQ = dS K runs as one batched causal tcgen05 GEMM
//                     (deterministic: no atomics anywhere). Warps: 0 TMA,
//                     1 MMA issuer + TMEM owner, 2..9 row math (warp w owns
//                     TMEM lanes 32*(w%4) .. +31 and half (w-2)/4 of the 128
//                     key columns).
//
// Dropout keep bits: Philox4x32-10 with the seed's round keys in the kernel
// parameters; the forward pass can store one bit per causal-band element
// (mask_mode 1) which the recompute forward and the backward read (mode 2).
#include <cmath>
#include <cstdlib>
#include <string>

#include "common.cuh"
#include "gemm.h"
#include "kernels.h"

namespace oases {

namespace {

constexpr int kTile = 128;
constexpr int kRowWarps = 8;                    // backward: two warps per TMEM lane quarter, 64 columns each
constexpr int kThreads = 64 + 32 * kRowWarps;  // + TMA warp + MMA warp
constexpr int kFwdRowWarps = 16;                      // forward: four warps per lane quarter, 32 columns each
constexpr int kFwdThreads = 96 + 32 * kFwdRowWarps;  // + Q/K producer, MMA, V producer: 19 warps
constexpr float kLog2e = 1.44269504088896341f;

#ifdef OASES_EXP_TRACE
__device__ unsigned long long g_attn_trace[8][64];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define ATRACE(ev, g) \
  do {                 \
    if (blockIdx.x == 0 && (g) < 64) g_attn_trace[ev][g] = gtime(); \
  } while (0)
// per-CTA start / end / SM id of the dK/dV kernel (first 1024 CTAs; tools/attn_cta_timeline.py)
__device__ unsigned long long g_cta_trace[3][1024];
#define CTRACE(ev)                                                                   \
  do {                                                                               \
    if (threadIdx.x == 64 && blockIdx.x < 1024) {                                    \
      unsigned smid;                                                                 \
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));                             \
      g_cta_trace[ev][blockIdx.x] = gtime();                                         \
      g_cta_trace[2][blockIdx.x] = smid;                                             \
    }                                                                                \
  } while (0)
#else
#define CTRACE(ev) \
  do {             \
  } while (0)
#define ATRACE(ev, g) \
  do {                 \
  } while (0)
#endif
struct AttnParams {
  int seq, hl, hg, hoff, Z, nq;
  int n0;  // dropout keys: first sample of this tensor in the keyed sub-batch
  int q_col, k_col, v_col;  // columns of head 0 of Q / K / V in the qkv (and dqkv) rows
  int do_col;               // column of head 0 in dout / out rows
  long long ld_out;         // fwd: ctx row stride; bwd: dqkv row stride
  void* out;                // fwd: ctx; bwd: dqkv
  float* lse;               // [Z * seq], log2 domain
  const float* dsum;        // [Z * seq]
  float sl2;                // scale * log2(e)
  float scale;
  uint32_t thr;             // dropout byte threshold (0 = no dropout)
  float ks;                 // keep scale
  uint64_t seed, offset;
  uint32_t rk0[10], rk1[10];  // Philox round keys of `seed` (constant-bank operands of the round LOP3s)
  uint32_t* mask_bits;        // keep-bit cache [Z][causal tile][128 rows][4 words] (null: always Philox)
  int mask_mode;              // 0 generate, 1 generate + store, 2 load
  int pv_wait;                // attn_fwd2_kernel: S(j+1) waits for PV(j) (1) or relies on in-order MMAs (0)
};

// Word index of (row, 32-column group w) of causal tile (qt, kt) of head z in
// the keep-bit cache: tiles of a head in row-major causal order.
__device__ __forceinline__ long long mask_word(const AttnParams& p, int z, int qt, int kt, int row, int w) {
  const long long tile = static_cast<long long>(z) * (p.nq * (p.nq + 1) / 2) + qt * (qt + 1) / 2 + kt;
  return (tile * kTile + row) * 4 + w;
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ float2 unpack_bf16(uint32_t w) {
  return __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w));
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// Packed f32x2 arithmetic (FFMA2 / FADD2: two lanes of work per instruction).
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
  unsigned long long r, x, y, z;
  asm("mov.b64 %0, {%1, %2};" : "=l"(x) : "f"(a.x), "f"(a.y));
  asm("mov.b64 %0, {%1, %2};" : "=l"(y) : "f"(b.x), "f"(b.y));
  asm("mov.b64 %0, {%1, %2};" : "=l"(z) : "f"(c.x), "f"(c.y));
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(x), "l"(y), "l"(z));
  float2 o;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(o.x), "=f"(o.y) : "l"(r));
  return o;
}
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
  unsigned long long r, x, y;
  asm("mov.b64 %0, {%1, %2};" : "=l"(x) : "f"(a.x), "f"(a.y));
  asm("mov.b64 %0, {%1, %2};" : "=l"(y) : "f"(b.x), "f"(b.y));
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(x), "l"(y));
  float2 o;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(o.x), "=f"(o.y) : "l"(r));
  return o;
}
// 16-byte chunk `ch` (8 bf16 columns, ch in 0..15 over 128 columns) of row r of a
// [128 x 128] bf16 tile stored as two SW128 K-major [128 x 64] halves 16 KB apart.
__device__ __forceinline__ uint4* tile_chunk(uint8_t* tile, int r, int ch) {
  return reinterpret_cast<uint4*>(tile + (ch >> 3) * 16384 + r * 128 + (((ch & 7) ^ (r & 7)) << 4));
}
// Philox4x32-10 (common.cuh) with the round keys and
// the offset words hoisted out of the per-call path: they are the same for
// every call of a launch.
// Philox4x32-10 (common.cuh): the offset words live
// in registers, the round keys of the seed in the kernel parameters
// (AttnParams::rk0/rk1, constant-bank operands of the round LOP3s).
struct PhiloxLite {
  uint32_t s0, s1, o0, o1, thr4;
};
__device__ __forceinline__ void philox_init(const AttnParams& p, PhiloxLite& ps) {
  ps.s0 = static_cast<uint32_t>(p.seed);
  ps.s1 = static_cast<uint32_t>(p.seed >> 32);
  ps.o0 = static_cast<uint32_t>(p.offset);
  ps.o1 = static_cast<uint32_t>(p.offset >> 32);
  ps.thr4 = p.thr * 0x01010101u;
}
// Keep masks of 16 consecutive elements (Philox counter ctr) as 8 bf16x2 lane
// masks: m[k] covers elements 2k (low half) and 2k+1.
__device__ __forceinline__ void keep_masks16(const PhiloxLite& ps, const AttnParams& prm, unsigned long long ctr,
                                             uint32_t (&m)[8]) {
  uint32_t c0 = static_cast<uint32_t>(ctr), c1 = static_cast<uint32_t>(ctr >> 32), c2 = ps.o0, c3 = ps.o1;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const unsigned long long p0 = static_cast<unsigned long long>(0xD2511F53u) * c0;
    const unsigned long long p1 = static_cast<unsigned long long>(0xCD9E8D57u) * c2;
    const uint32_t n0 = static_cast<uint32_t>(p1 >> 32) ^ c1 ^ prm.rk0[r];
    const uint32_t n2 = static_cast<uint32_t>(p0 >> 32) ^ c3 ^ prm.rk1[r];
    c1 = static_cast<uint32_t>(p1);
    c3 = static_cast<uint32_t>(p0);
    c0 = n0;
    c2 = n2;
  }
  const uint32_t u[4] = {c0, c1, c2, c3};
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    const uint32_t k = __vcmpgeu4(u[w], ps.thr4);
    m[2 * w] = __byte_perm(k, 0, 0x1100);
    m[2 * w + 1] = __byte_perm(k, 0, 0x3322);
  }
}
// keep_masks16 plus the 16 keep bits (bit e = element e of the group).
__device__ __forceinline__ uint32_t keep_masks16_bits(const PhiloxLite& ps, const AttnParams& prm,
                                                      unsigned long long ctr, uint32_t (&m)[8]) {
  uint32_t c0 = static_cast<uint32_t>(ctr), c1 = static_cast<uint32_t>(ctr >> 32), c2 = ps.o0, c3 = ps.o1;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const unsigned long long p0 = static_cast<unsigned long long>(0xD2511F53u) * c0;
    const unsigned long long p1 = static_cast<unsigned long long>(0xCD9E8D57u) * c2;
    const uint32_t n0 = static_cast<uint32_t>(p1 >> 32) ^ c1 ^ prm.rk0[r];
    const uint32_t n2 = static_cast<uint32_t>(p0 >> 32) ^ c3 ^ prm.rk1[r];
    c1 = static_cast<uint32_t>(p1);
    c3 = static_cast<uint32_t>(p0);
    c0 = n0;
    c2 = n2;
  }
  const uint32_t u[4] = {c0, c1, c2, c3};
  uint32_t bits = 0;
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    const uint32_t k = __vcmpgeu4(u[w], ps.thr4);
    m[2 * w] = __byte_perm(k, 0, 0x1100);
    m[2 * w + 1] = __byte_perm(k, 0, 0x3322);
    bits |= (((k & 0x01010101u) * 0x01020408u) >> 24) << (4 * w);  // 4 byte flags -> 4 bits
  }
  return bits;
}
// The 8 bf16x2 lane masks of 16 cached keep bits.
__device__ __forceinline__ void masks16_from_bits(uint32_t bits, uint32_t (&m)[8]) {
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    const uint32_t nib = (bits >> (4 * w)) & 0xFu;
    const uint32_t k = ((nib * 0x00204081u) & 0x01010101u) * 0xFFu;  // 4 bits -> 4 byte flags
    m[2 * w] = __byte_perm(k, 0, 0x1100);
    m[2 * w + 1] = __byte_perm(k, 0, 0x3322);
  }
}

// Static zigzag schedule of work items over a persistent grid. Items are
// numbered heaviest first; round r hands CTA c item r*G + c (r even) or
// r*G + G-1-c (r odd), which balances the decreasing item sizes.
__device__ __forceinline__ int zigzag_item(int round, int G) {
  const int c = static_cast<int>(blockIdx.x);
  return round * G + ((round & 1) ? G - 1 - c : c);
}

template <int DH>
struct FwdCfg {
  static constexpr int TILE_BYTES = kTile * DH * 2;
  static constexpr int Q_OFF = 0;                        // [2] double-buffered across items
  static constexpr int K_OFF = 2 * TILE_BYTES;           // [2]
  static constexpr int V_OFF = K_OFF + 2 * TILE_BYTES;   // [2]
  // row-max exchange [2 parities][4 parts][128 rows] (one barrier per KV tile),
  // then the row-sum exchange of the item epilogue [4 parts][128 rows]
  static constexpr int RED_OFF = V_OFF + 2 * TILE_BYTES;
  static constexpr int REDL_OFF = RED_OFF + 2 * 4 * kTile * 4;
  static constexpr int BAR_OFF = REDL_OFF + 4 * kTile * 4;
  static constexpr int SMEM = BAR_OFF + 256;
  // TMEM: NS S/P buffers of 128 columns + NO O accumulators of DH columns.
  // Three S buffers give the S MMA of iteration g+3 the slack of a whole
  // iteration after PV_g (which reads P_g from the buffer) completes.
  static constexpr int NS = 3;
  static constexpr int NO = DH == 64 ? 2 : 1;
  static constexpr uint32_t O_COL = NS * kTile;
  static constexpr uint32_t TMEM_COLS = 512;
  static_assert(NS * kTile + NO * DH <= 512, "TMEM budget");
};

// Persistent flash forward: each CTA walks its zigzag item list as one flat
// sequence of (item, kv-tile) iterations; Q, K/V stages, the S buffers and the
// O accumulator are all double-buffered across item boundaries, so the next
// item's loads and first QK^T run under the current item's last softmax and
// epilogue.
template <int DH>
__global__ void __launch_bounds__(kFwdThreads, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tqkv, const AttnParams p) {
  pdl_trigger();
  using C = FwdCfg<DH>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
  uint64_t* q_full = bars;        // [2]
  uint64_t* q_empty = bars + 2;   // [2] freed by the item's last S MMA
  uint64_t* k_full = bars + 4;    // [2]
  uint64_t* k_empty = bars + 6;   // [2] freed by the S MMA
  uint64_t* v_full = bars + 8;    // [2]
  uint64_t* v_empty = bars + 10;  // [2] freed by the PV MMA
  uint64_t* s_full = bars + 12;   // [NS] S_g in TMEM buffer g % NS
  uint64_t* p_full = bars + 15;   // [NS] P_g (bf16) written over S_g by the row warps
  uint64_t* pv_done = bars + 18;  // [NS] PV_g done: buffer g % NS reusable
  uint64_t* o_free = bars + 21;   // [NO] row warps drained the O buffer
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 23);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = static_cast<int>(gridDim.x);
  const int total = p.Z * p.nq;
  auto item_of = [&](int t, int& qt, int& z) {
    qt = p.nq - 1 - t / p.Z;  // heaviest (longest causal rows) first
    z = t % p.Z;
  };

  if (threadIdx.x == 0) {
    if (smem_u32(smem) & 1023) __trap();
    for (int s = 0; s < 2; ++s) {
      mbar_init(&q_full[s], 1);
      mbar_init(&q_empty[s], 1);
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    for (int s = 0; s < C::NS; ++s) {
      mbar_init(&s_full[s], 1);
      mbar_init(&p_full[s], kFwdRowWarps);
      mbar_init(&pv_done[s], 1);
    }
    for (int s = 0; s < C::NO; ++s) mbar_init(&o_free[s], kFwdRowWarps);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();

  if (warp == 0 || warp == 2) {
    // TMA producers: warp 0 streams Q and K, warp 2 streams V. Separate
    // threads so a K load never queues behind the wait for a V stage (freed
    // only by the PV MMA at the end of a softmax): K gets a full extra
    // iteration of latency slack.
    if (lane == 0) {
      const bool kq = warp == 0;
      if (kq) tma_prefetch(&tqkv);
      int g = 0;  // global kv iteration
      for (int r = 0, k = 0;; ++r, ++k) {
        const int t = zigzag_item(r, G);
        if (t >= total) break;
        int qt, z;
        item_of(t, qt, z);
        const int n = z / p.hl, jl = z - n * p.hl, row0 = n * p.seq;
        const int qb = k & 1;
        if (kq) {
          mbar_wait(&q_empty[qb], ((k >> 1) & 1) ^ 1);
          mbar_arrive_expect_tx(&q_full[qb], C::TILE_BYTES);
#pragma unroll
          for (int gg = 0; gg < DH / 64; ++gg)
            tma_load_2d(smem + C::Q_OFF + qb * C::TILE_BYTES + gg * 16384, &tqkv, &q_full[qb],
                        p.q_col + jl * DH + gg * 64, row0 + qt * kTile);
        }
        for (int j = 0; j <= qt; ++j, ++g) {
          const int st = g & 1, ph = ((g >> 1) & 1) ^ 1;
          uint64_t* empty = kq ? &k_empty[st] : &v_empty[st];
          uint64_t* full = kq ? &k_full[st] : &v_full[st];
          const int off = kq ? C::K_OFF : C::V_OFF, col = kq ? p.k_col : p.v_col;
          mbar_wait(empty, ph);
          ATRACE(kq ? 6 : 7, g);
          mbar_arrive_expect_tx(full, C::TILE_BYTES);
#pragma unroll
          for (int gg = 0; gg < DH / 64; ++gg)
            tma_load_2d(smem + off + st * C::TILE_BYTES + gg * 16384, &tqkv, full, col + jl * DH + gg * 64,
                        row0 + j * kTile);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t id_s = umma_idesc_bf16(kTile, kTile, 0, 0);
      constexpr uint32_t id_o = umma_idesc_bf16(kTile, DH, 0, 1);  // A = P in TMEM (K-major), B = V (MN-major)
      const uint32_t sb = smem_u32(smem);
      // S for flat iteration (item k, kv tile j, global g) into TMEM buffer g&1,
      // once PV_{g-2} (which read P_{g-2} from that buffer) is done; commits
      // q_empty after the item's last tile.
      auto issue_s = [&](int k, int j, int g, bool last) {
        ATRACE(0, g);
        const int st = g % C::NS, kv = g & 1, qb = k & 1;
        if (j == 0) mbar_wait(&q_full[qb], (k >> 1) & 1);
        mbar_wait(&k_full[kv], (g >> 1) & 1);
        if (g >= C::NS) mbar_wait(&pv_done[st], ((g - C::NS) / C::NS) & 1);
        ATRACE(1, g);
        tc_fence_after();
        const uint32_t qa = sb + C::Q_OFF + qb * C::TILE_BYTES, kb = sb + C::K_OFF + kv * C::TILE_BYTES;
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk) {
          const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
          umma_bf16(tmem + st * kTile, umma_desc_sw128(qa + off, 16, 1024), umma_desc_sw128(kb + off, 16, 1024),
                    id_s, kk > 0 ? 1u : 0u);
        }
        umma_commit(&s_full[st]);
        umma_commit(&k_empty[kv]);
        if (last) umma_commit(&q_empty[qb]);
      };
      // O += P_g V_g with P_g read from TMEM (bf16, 64 columns over S_g).
      auto issue_pv = [&](int k, int j, int g) {
        ATRACE(2, g);
        const int st = g % C::NS, kv = g & 1, ob = k % C::NO;
        if (j == 0) mbar_wait(&o_free[ob], ((k / C::NO) & 1) ^ 1);
        mbar_wait(&p_full[st], (g / C::NS) & 1);
        mbar_wait(&v_full[kv], (g >> 1) & 1);
        ATRACE(3, g);
        tc_fence_after();
        const uint32_t vb = sb + C::V_OFF + kv * C::TILE_BYTES;
#pragma unroll
        for (int kk = 0; kk < kTile / 16; ++kk) {
          const uint64_t bd = umma_desc_sw128(vb + kk * 2048, 16384, 1024);
          umma_bf16_ts(tmem + C::O_COL + ob * DH, tmem + st * kTile + kk * 8, bd, id_o, (j > 0 || kk > 0) ? 1u : 0u);
        }
        umma_commit(&v_empty[kv]);
        umma_commit(&pv_done[st]);
      };
      // Flat iteration cursors (round r -> item k, kv tile j, global g). The S
      // MMAs run two iterations ahead of the PV MMAs (three S/P buffers), so
      // the commit -> mbarrier -> softmax latency of S_{g+1}, S_{g+2} hides
      // under the softmax of g.
      struct Cur {
        int r, k, j, qt, g;
        bool valid;
      };
      auto cur_load = [&](Cur& c) {
        const int t = zigzag_item(c.r, G);
        c.valid = t < total;
        if (c.valid) {
          int z;
          item_of(t, c.qt, z);
        }
      };
      auto cur_next = [&](Cur& c) {
        ++c.g;
        if (++c.j > c.qt) {
          ++c.r;
          ++c.k;
          c.j = 0;
          cur_load(c);
        }
      };
      Cur sc{0, 0, 0, 0, 0, false}, pc{0, 0, 0, 0, 0, false};
      cur_load(sc);
      cur_load(pc);
      for (int a = 0; a < C::NS - 1 && sc.valid; ++a) {
        issue_s(sc.k, sc.j, sc.g, sc.j == sc.qt);
        cur_next(sc);
      }
      while (pc.valid) {
        if (sc.valid) {
          issue_s(sc.k, sc.j, sc.g, sc.j == sc.qt);
          cur_next(sc);
        }
        issue_pv(pc.k, pc.j, pc.g);
        cur_next(pc);
      }
    }
  } else {
    // ------------------------------------------------ row warps
    // Warp w owns TMEM lane quarter q = w % 4 (query rows 32q .. 32q+31 of the
    // tile; one row per thread), key columns [32 part, 32 part + 32) of every
    // S tile and O columns [part DH/4, (part+1) DH/4). The four warps of a
    // quarter combine their partial row maxima / sums through smem.
    const int q = warp & 3, part = (warp - 3) >> 2;  // row warps 3 .. 18
    const int rr = q * 32 + lane;
    const int c0 = part * 32;
    constexpr int OC = DH / 4;  // O columns per warp
    const uint32_t tl = tmem + (static_cast<uint32_t>(q * 32) << 16);
    float* redm = reinterpret_cast<float*>(smem + C::RED_OFF);   // [parity][part][row]
    float* redl = reinterpret_cast<float*>(smem + C::REDL_OFF);  // [part][row]
    PhiloxLite ph;
    philox_init(p, ph);
    int g = 0;
    for (int r = 0, k = 0;; ++r, ++k) {
      const int t = zigzag_item(r, G);
      if (t >= total) break;
      int qt, z;
      item_of(t, qt, z);
      const int n = z / p.hl, jl = z - n * p.hl, row0 = n * p.seq;
      const int i = qt * kTile + rr;
      const int ob = k % C::NO;
      const uint32_t to = tl + C::O_COL + ob * DH + part * OC;  // this warp's columns of O
      const unsigned long long ebase =
          (static_cast<unsigned long long>((n + p.n0) * p.hg + p.hoff + jl) * p.seq + i) *
              static_cast<unsigned long long>(p.seq) +
          c0;
      float m = -INFINITY, l = 0.f;
      // cached keep bits: the word of tile j + 1 is loaded while tile j is processed
      const bool cached = p.thr && p.mask_mode == 2;
      uint32_t mword = cached ? p.mask_bits[mask_word(p, z, qt, 0, rr, part)] : 0u;
      for (int j = 0; j <= qt; ++j, ++g) {
        const int st = g % C::NS;
        const uint32_t bits_j = mword;
        if (cached && j < qt) mword = p.mask_bits[mask_word(p, z, qt, j + 1, rr, part)];
        mbar_wait(&s_full[st], (g / C::NS) & 1);
        if (warp == 3 && lane == 0) ATRACE(4, g);
        tc_fence_after();
        uint32_t u[32];
        tmem_ld32(tl + st * kTile + c0, u);
        tmem_wait_ld();
        if (j == qt) {
          int lim = rr - c0;                   // keys > row are masked
          asm volatile("" : "+r"(lim));        // keep the comparisons inside the (rare) diagonal branch
#pragma unroll
          for (int kk = 0; kk < 32; ++kk)
            if (kk > lim) u[kk] = __float_as_uint(-INFINITY);
        }
        float mpart;
        {  // 4 independent partial maxima (short dependency chains)
          float mp[4];
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) mp[kk] = __uint_as_float(u[kk]);
#pragma unroll
          for (int kk = 4; kk < 32; ++kk) mp[kk & 3] = fmaxf(mp[kk & 3], __uint_as_float(u[kk]));
          mpart = fmaxf(fmaxf(mp[0], mp[1]), fmaxf(mp[2], mp[3]));
        }
        // Partials alternate between two buffers: a warp can only write a buffer
        // again after the next tile's barrier, which every warp of the quarter
        // reaches after reading it. The barrier also orders every warp's S loads
        // before any P store over S below.
        float* rm = redm + (g & 1) * 4 * kTile;
        rm[part * kTile + rr] = mpart;
        tc_fence_before();
        named_bar_sync(1 + q, 128);
        tc_fence_after();
        const float mloc = fmaxf(fmaxf(rm[rr], rm[kTile + rr]), fmaxf(rm[2 * kTile + rr], rm[3 * kTile + rr]));
        // Conditional rescaling: keep the running max unless the row max grew by
        // more than 8 (log2 units). P = exp2(s - m) then stays <= 256 (exact in
        // bf16's range) and O, l are rescaled only when it pays; the result is
        // the same softmax since O and l always share one reference max.
        const float cand = fmaxf(m, mloc * p.sl2);
        const float mx = cand > m + 8.f ? cand : m;
        const float alpha = ex2(m - mx);
        const float nmx = -mx;
        float2 sp[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
        uint32_t pk[16];
        const float2 sl2x2 = make_float2(p.sl2, p.sl2), nmx2 = make_float2(nmx, nmx);
#pragma unroll
        for (int kk = 0; kk < 32; kk += 2) {
          // pairs on the packed pipe: one FFMA2 for the exponents, one FADD2 for the sums
          const float2 e = fma2(make_float2(__uint_as_float(u[kk]), __uint_as_float(u[kk + 1])), sl2x2, nmx2);
          const float2 ab = make_float2(ex2(e.x), ex2(e.y));
          sp[(kk >> 1) & 1] = add2(sp[(kk >> 1) & 1], ab);
          pk[kk >> 1] = pack_bf16(ab.x, ab.y);
        }
        const float sum = (sp[0].x + sp[1].x) + (sp[0].y + sp[1].y);
        l = l * alpha + sum;
        m = mx;
        if (p.thr) {
          if (cached) {  // keep bits stored by the forward pass
#pragma unroll
            for (int gq = 0; gq < 2; ++gq) {
              uint32_t km[8];
              masks16_from_bits(bits_j >> (16 * gq), km);
#pragma unroll
              for (int kk = 0; kk < 8; ++kk) pk[gq * 8 + kk] &= km[kk];
            }
          } else {
            uint32_t bits = 0;
#pragma unroll
            for (int gq = 0; gq < 2; ++gq) {
              uint32_t km[8];
              bits |= keep_masks16_bits(ph, p, (ebase + static_cast<unsigned long long>(j) * kTile + gq * 16) >> 4,
                                        km)
                      << (16 * gq);
#pragma unroll
              for (int kk = 0; kk < 8; ++kk) pk[gq * 8 + kk] &= km[kk];
            }
            if (p.mask_mode == 1) p.mask_bits[mask_word(p, z, qt, j, rr, part)] = bits;
          }
        }
        if (j > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {
          // O holds P_{j-1} V_{j-1} once PV_{g-1} is done: rescale it to the new
          // reference max (rare: only when the row max grew by more than 8)
          mbar_wait(&pv_done[(g - 1) % C::NS], ((g - 1) / C::NS) & 1);
          tc_fence_after();
          if constexpr (OC == 32) {
            uint32_t o[32];
            tmem_ld32(to, o);
            tmem_wait_ld();
#pragma unroll
            for (int kk = 0; kk < 32; ++kk) o[kk] = __float_as_uint(__uint_as_float(o[kk]) * alpha);
            tmem_st32(to, o);
          } else {
            uint32_t o[16];
            tmem_ld16(to, o);
            tmem_wait_ld();
#pragma unroll
            for (int kk = 0; kk < 16; ++kk) o[kk] = __float_as_uint(__uint_as_float(o[kk]) * alpha);
            tmem_st16(to, o);
          }
          tmem_wait_st();
        }
        // P_g (bf16 pairs) over this warp's S_g columns: the quarter's S loads all
        // precede the max exchange above, so no warp still needs them
        tmem_st16(tl + st * kTile + c0 / 2, pk);
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (warp == 3 && lane == 0) ATRACE(5, g);
        if (lane == 0) mbar_arrive(&p_full[st]);
      }
      // ---- item epilogue: O / l -> ctx, lse
      redl[part * kTile + rr] = l;  // previous item's sums were read before this item's tile barriers
      named_bar_sync(1 + q, 128);
      const float lt = (redl[rr] + redl[kTile + rr]) + (redl[2 * kTile + rr] + redl[3 * kTile + rr]);
      mbar_wait(&pv_done[(g - 1) % C::NS], ((g - 1) / C::NS) & 1);
      tc_fence_after();
      const float inv = p.ks / lt;
      __nv_bfloat16* orow = static_cast<__nv_bfloat16*>(p.out) + static_cast<long long>(row0 + i) * p.ld_out +
                            p.do_col + jl * DH + part * OC;
      uint32_t o[OC];
      if constexpr (OC == 32) tmem_ld32(to, o);
      else tmem_ld16(to, o);
      tmem_wait_ld();
#pragma unroll
      for (int kk = 0; kk < OC / 8; ++kk) {
        const float* f = reinterpret_cast<const float*>(o + 8 * kk);
        *reinterpret_cast<uint4*>(orow + kk * 8) =
            make_uint4(pack_bf16(f[0] * inv, f[1] * inv), pack_bf16(f[2] * inv, f[3] * inv),
                       pack_bf16(f[4] * inv, f[5] * inv), pack_bf16(f[6] * inv, f[7] * inv));
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&o_free[ob]);
      if (part == 0) p.lse[static_cast<long long>(z) * p.seq + i] = m + log2f(lt);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, C::TMEM_COLS);
  }
}

// ------------------------------------------------------------------ forward, ping-pong
// attn_fwd2_kernel: FA4-style forward. A work item is a PAIR of adjacent
// 128-query tiles (2m, 2m+1) of one (sample, head), streaming the same K/V
// tiles (both active on all but the last one, so the two softmax groups
// overlap each other's MMAs; pairing (m, nq-1-m) balances the items but leaves
// one tile running alone most of the time -- measured slower). Each
// tile has its own softmax warpgroup (4 warps, one query row per thread, all
// 128 key columns of the row in registers: the row max needs no cross-warp
// exchange) and its own TMEM S/P (128 columns) and O (DH columns) regions, so
// the tensor core alternates between the tiles: PV_A(j), S_A(j+1) run under
// softmax B(j); PV_B(j), S_B(j+1) under softmax A(j+1).
// Warps: 0-3 softmax of tile A (TMEM lane quarter w % 4), 4-7 softmax of tile
// B, 8 TMA (Q pair, K/V stages), 9 MMA issuer + TMEM owner (10 warps; the
// register file is split per SM sub-partition, so 3 warps on one of them cap
// a thread at 168 registers).
// Dropout keys, keep-bit cache layout (mask_word) and the conditional
// rescaling are those of attn_fwd_kernel, so both kernels compute the same
// softmax and either one's keep bits serve the other and attn_dkdv_kernel.
template <int DH>
struct Fwd2Cfg {
  static constexpr int TILE_BYTES = kTile * DH * 2;
  static constexpr int QA_OFF = 0, QB_OFF = TILE_BYTES;
  static constexpr int K_OFF = 2 * TILE_BYTES;          // [2] stages
  static constexpr int V_OFF = K_OFF + 2 * TILE_BYTES;  // [2] stages
  static constexpr int BAR_OFF = V_OFF + 2 * TILE_BYTES;
  static constexpr int SMEM = BAR_OFF + 256;
  __host__ __device__ static constexpr uint32_t s_col(int x) { return x ? kTile : 0u; }
  static constexpr uint32_t O_COL0 = 2 * kTile;  // O_A at O_COL0, O_B at O_COL0 + DH
  static constexpr uint32_t TMEM_COLS = 512;
  static_assert(2 * kTile + 2 * DH <= 512, "TMEM budget");
};
constexpr int kFwd2Threads = 320;

template <int DH>
__global__ void __launch_bounds__(kFwd2Threads, 1)
    attn_fwd2_kernel(const __grid_constant__ CUtensorMap tqkv, const AttnParams p) {
  pdl_trigger();
  using C = Fwd2Cfg<DH>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
  uint64_t* q_full = bars;        // Q pair loaded
  uint64_t* q_empty = bars + 1;   // the item's last S MMAs done
  uint64_t* k_full = bars + 2;    // [2]
  uint64_t* k_empty = bars + 4;   // [2]
  uint64_t* v_full = bars + 6;    // [2]
  uint64_t* v_empty = bars + 8;   // [2]
  uint64_t* s_full = bars + 10;   // [tile] S in TMEM
  uint64_t* p_full = bars + 12;   // [tile] P (bf16) written over S by the tile's 4 softmax warps
  uint64_t* pv_done = bars + 14;  // [tile] PV done (S/P region reusable, O current)
  uint64_t* o_free = bars + 16;   // [tile] epilogue drained O
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 18);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = static_cast<int>(gridDim.x);
  const int npair = (p.nq + 1) / 2;
  const int total = p.Z * npair;
  // item t -> (m, z): tiles A = 2m, B = 2m+1 (absent for the last of an odd
  // count), heaviest first
  auto item_of = [&](int t, int& m, int& z) {
    m = npair - 1 - t / p.Z;
    z = t % p.Z;
  };

  if (threadIdx.x == 0) {
    if (smem_u32(smem) & 1023) __trap();
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
      mbar_init(&s_full[s], 1);
      mbar_init(&p_full[s], 4);
      mbar_init(&pv_done[s], 1);
      mbar_init(&o_free[s], 4);
    }
    fence_barrier_init();
  }
  if (warp == 9) tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  if (warp == 8) {
    if (lane == 0) {
      tma_prefetch(&tqkv);
      int g = 0;
      for (int r = 0, k = 0;; ++r, ++k) {
        const int t = zigzag_item(r, G);
        if (t >= total) break;
        int m, z;
        item_of(t, m, z);
        const int n = z / p.hl, jl = z - n * p.hl, row0 = n * p.seq;
        const int qtb = 2 * m + 1;
        const bool hasb = qtb < p.nq;
        const int nkv = hasb ? qtb + 1 : 2 * m + 1;
        mbar_wait(q_empty, (k & 1) ^ 1);
        mbar_arrive_expect_tx(q_full, (hasb ? 2 : 1) * C::TILE_BYTES);
#pragma unroll
        for (int gg = 0; gg < DH / 64; ++gg) {
          tma_load_2d(smem + C::QA_OFF + gg * 16384, &tqkv, q_full, p.q_col + jl * DH + gg * 64,
                      row0 + 2 * m * kTile);
          if (hasb)
            tma_load_2d(smem + C::QB_OFF + gg * 16384, &tqkv, q_full, p.q_col + jl * DH + gg * 64,
                        row0 + qtb * kTile);
        }
        for (int j = 0; j < nkv; ++j, ++g) {
          const int st = g & 1, ph = ((g >> 1) & 1) ^ 1;
          mbar_wait(&k_empty[st], ph);
          mbar_arrive_expect_tx(&k_full[st], C::TILE_BYTES);
#pragma unroll
          for (int gg = 0; gg < DH / 64; ++gg)
            tma_load_2d(smem + C::K_OFF + st * C::TILE_BYTES + gg * 16384, &tqkv, &k_full[st],
                        p.k_col + jl * DH + gg * 64, row0 + j * kTile);
          mbar_wait(&v_empty[st], ph);
          mbar_arrive_expect_tx(&v_full[st], C::TILE_BYTES);
#pragma unroll
          for (int gg = 0; gg < DH / 64; ++gg)
            tma_load_2d(smem + C::V_OFF + st * C::TILE_BYTES + gg * 16384, &tqkv, &v_full[st],
                        p.v_col + jl * DH + gg * 64, row0 + j * kTile);
        }
      }
    }
  } else if (warp == 9) {
    if (lane == 0) {
      constexpr uint32_t id_s = umma_idesc_bf16(kTile, kTile, 0, 0);
      constexpr uint32_t id_o = umma_idesc_bf16(kTile, DH, 0, 1);  // A = P in TMEM (K-major), B = V (MN-major)
      const uint32_t sb = smem_u32(smem);
      int cnt[2] = {0, 0};  // S/PV iterations issued per tile (barrier phases)
      int itc[2] = {0, 0};  // items processed per tile (o_free phases; odd pairs have no tile B)
      int g = 0;
      auto issue_s = [&](int x, int st, uint32_t qa) {
        // PV read the previous P from this region: tcgen05.mma executes in issue
        // order, so S(j+1) issued after PV(j) cannot overwrite P(j) before PV(j)
        // consumed it; pv_wait = 1 keeps the explicit drain (A/B check)
        if (p.pv_wait && cnt[x] > 0) mbar_wait(&pv_done[x], (cnt[x] - 1) & 1);
        tc_fence_after();
        const uint32_t kb = sb + C::K_OFF + st * C::TILE_BYTES;
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk) {
          const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
          umma_bf16(tmem + C::s_col(x), umma_desc_sw128(qa + off, 16, 1024), umma_desc_sw128(kb + off, 16, 1024),
                    id_s, kk > 0 ? 1u : 0u);
        }
        umma_commit(&s_full[x]);
      };
      auto issue_pv = [&](int x, int st, int j) {
        if (j == 0) mbar_wait(&o_free[x], (itc[x]++ & 1) ^ 1);
        mbar_wait(&p_full[x], cnt[x] & 1);
        tc_fence_after();
        const uint32_t vb = sb + C::V_OFF + st * C::TILE_BYTES;
#pragma unroll
        for (int kk = 0; kk < kTile / 16; ++kk) {
          const uint64_t bd = umma_desc_sw128(vb + kk * 2048, 16384, 1024);
          umma_bf16_ts(tmem + C::O_COL0 + x * DH, tmem + C::s_col(x) + kk * 8, bd, id_o, (j > 0 || kk > 0) ? 1u : 0u);
        }
        umma_commit(&pv_done[x]);
        ++cnt[x];
      };
      for (int r = 0, k = 0;; ++r, ++k) {
        const int t = zigzag_item(r, G);
        if (t >= total) break;
        int m, z;
        item_of(t, m, z);
        const bool hasb = 2 * m + 1 < p.nq;
        const int na = 2 * m + 1, nb = hasb ? 2 * m + 2 : 0, nkv = hasb ? nb : na;
        const uint32_t qa = sb + C::QA_OFF, qb = sb + C::QB_OFF;
        mbar_wait(q_full, k & 1);
        // prologue: S_A(0), S_B(0)
        mbar_wait(&k_full[g & 1], (g >> 1) & 1);
        issue_s(0, g & 1, qa);
        if (nb > 0) issue_s(1, g & 1, qb);
        umma_commit(&k_empty[g & 1]);
        if (nkv == 1) umma_commit(q_empty);
        for (int j = 0; j < nkv; ++j) {
          const int st = g & 1, gn = g + 1;
          mbar_wait(&v_full[st], (g >> 1) & 1);
          // PV_A(j), then S_A(j+1) under softmax B(j)
          if (j < na) issue_pv(0, st, j);
          const bool more = j + 1 < nkv;
          if (more) mbar_wait(&k_full[gn & 1], (gn >> 1) & 1);
          if (j + 1 < na) issue_s(0, gn & 1, qa);
          // PV_B(j), then S_B(j+1) under softmax A(j+1)
          if (j < nb) issue_pv(1, st, j);
          umma_commit(&v_empty[st]);
          if (j + 1 < nb) issue_s(1, gn & 1, qb);
          if (more) {
            umma_commit(&k_empty[gn & 1]);
            if (j + 2 == nkv) umma_commit(q_empty);  // the item's last S MMAs were just issued
          }
          g = gn;
        }
      }
    }
  } else if (warp < 8) {
    // ------------------------------------------------ softmax warpgroups
    const int x = warp >> 2;  // 0: tile A (2m), 1: tile B (2m+1)
    const int q = warp & 3;
    const int rr = q * 32 + lane;
    const uint32_t tl = tmem + (static_cast<uint32_t>(q * 32) << 16);
    const uint32_t ts = tl + C::s_col(x), to = tl + C::O_COL0 + x * DH;
    int cnt = 0;
    for (int r = 0, k = 0;; ++r, ++k) {
      const int t = zigzag_item(r, G);
      if (t >= total) break;
      int m2, z;
      item_of(t, m2, z);
      const int qt = 2 * m2 + x;
      if (qt >= p.nq) continue;  // no tile B in the last pair of an odd count
      const int n = z / p.hl, jl = z - n * p.hl, row0 = n * p.seq;
      const int i = qt * kTile + rr;
      const bool cached = p.thr != 0;  // always cached in this kernel (mask_mode 2)
      float mrun = -INFINITY, l4[4] = {0.f, 0.f, 0.f, 0.f};
      for (int j = 0; j <= qt; ++j, ++cnt) {
        // this tile's keep-bit words (the load flies while the S MMA completes)
        uint4 bits4 = make_uint4(0u, 0u, 0u, 0u);
        if (cached) bits4 = __ldg(reinterpret_cast<const uint4*>(p.mask_bits + mask_word(p, z, qt, j, rr, 0)));
        mbar_wait(&s_full[x], cnt & 1);
        tc_fence_after();
        uint32_t u[128];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t (&uc)[32] = *reinterpret_cast<uint32_t(*)[32]>(u + 32 * c);
          tmem_ld32(ts + 32 * c, uc);
        }
        tmem_wait_ld();
        if (j == qt) {
          int lim = rr;  // keys > row are masked on the diagonal tile
          asm volatile("" : "+r"(lim));
#pragma unroll
          for (int kk = 0; kk < 128; ++kk)
            if (kk > lim) u[kk] = __float_as_uint(-INFINITY);
        }
        float mp[8];
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) mp[kk] = __uint_as_float(u[kk]);
#pragma unroll
        for (int kk = 8; kk < 128; ++kk) mp[kk & 7] = fmaxf(mp[kk & 7], __uint_as_float(u[kk]));
        const float mloc =
            fmaxf(fmaxf(fmaxf(mp[0], mp[1]), fmaxf(mp[2], mp[3])), fmaxf(fmaxf(mp[4], mp[5]), fmaxf(mp[6], mp[7])));
        // conditional rescaling (attn_fwd_kernel): keep the running max unless the
        // row max grew by more than 8 (log2 units)
        const float cand = fmaxf(mrun, mloc * p.sl2);
        const float mx = cand > mrun + 8.f ? cand : mrun;
        const float alpha = ex2(mrun - mx);
        const float2 sl2x2 = make_float2(p.sl2, p.sl2), nmx2 = make_float2(-mx, -mx);
        // row sums kept per 32-column group, each accumulated exactly like one
        // attn_fwd_kernel softmax warp's (same operation order), so both kernels
        // produce the same bits
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          float2 sp[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
          for (int kk = 32 * c; kk < 32 * c + 32; kk += 2) {
            const float2 e = fma2(make_float2(__uint_as_float(u[kk]), __uint_as_float(u[kk + 1])), sl2x2, nmx2);
            const float2 ab = make_float2(ex2(e.x), ex2(e.y));
            sp[(kk >> 1) & 1] = add2(sp[(kk >> 1) & 1], ab);
            u[kk >> 1] = pack_bf16(ab.x, ab.y);  // P pairs packed into u[0..63]
          }
          l4[c] = l4[c] * alpha + ((sp[0].x + sp[1].x) + (sp[0].y + sp[1].y));
        }
        mrun = mx;
        if (p.thr) {  // cached keep bits (the launcher routes Philox-generating modes to attn_fwd_kernel)
          const uint32_t w4[4] = {bits4.x, bits4.y, bits4.z, bits4.w};
#pragma unroll
          for (int gq = 0; gq < 8; ++gq) {
            uint32_t km[8];
            masks16_from_bits(w4[gq >> 1] >> (16 * (gq & 1)), km);
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) u[gq * 8 + kk] &= km[kk];
          }
        }
        if (j > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {
          // O holds P_{<j} V: PV(j-1) was issued before S(j), and s_full(j)'s commit
          // tracks every MMA issued before it
#pragma unroll
          for (int c = 0; c < DH / 32; ++c) {
            uint32_t o[32];
            tmem_ld32(to + 32 * c, o);
            tmem_wait_ld();
#pragma unroll
            for (int kk = 0; kk < 32; ++kk) o[kk] = __float_as_uint(__uint_as_float(o[kk]) * alpha);
            tmem_st32(to + 32 * c, o);
          }
          tmem_wait_st();
        }
        // P (bf16 pairs) over the first 64 columns of this tile's S region
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const uint32_t (&pc)[32] = *reinterpret_cast<const uint32_t(*)[32]>(u + 32 * c);
          tmem_st32(ts + 32 * c, pc);
        }
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[x]);
      }
      // ---- epilogue: O / l -> ctx, lse
      mbar_wait(&pv_done[x], (cnt - 1) & 1);
      tc_fence_after();
      const float l = (l4[0] + l4[1]) + (l4[2] + l4[3]);  // attn_fwd_kernel's combine order
      const float inv = p.ks / l;
      __nv_bfloat16* orow =
          static_cast<__nv_bfloat16*>(p.out) + static_cast<long long>(row0 + i) * p.ld_out + p.do_col + jl * DH;
#pragma unroll
      for (int c = 0; c < DH / 32; ++c) {
        uint32_t o[32];
        tmem_ld32(to + 32 * c, o);
        tmem_wait_ld();
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const float* f = reinterpret_cast<const float*>(o + 8 * kk);
          *reinterpret_cast<uint4*>(orow + 32 * c + kk * 8) =
              make_uint4(pack_bf16(f[0] * inv, f[1] * inv), pack_bf16(f[2] * inv, f[3] * inv),
                         pack_bf16(f[4] * inv, f[5] * inv), pack_bf16(f[6] * inv, f[7] * inv));
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&o_free[x]);
      p.lse[static_cast<long long>(z) * p.seq + i] = mrun + log2f(l);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 9) {
    tc_fence_after();
    tmem_dealloc(tmem, C::TMEM_COLS);
  }
}

// Keep bits of every causal-band element (the attention-dropout masks of
// DESIGN.md section 5), one 32-key word per thread: a separate, fully parallel
// pass so that the forward's softmax warps -- the critical path of the fused
// kernels -- only expand cached bits (mask_mode 2) instead of running Philox.
__global__ void __launch_bounds__(512) attn_mask_kernel(const AttnParams p) {
  // block = one causal tile (z, qt, kt) in mask_word's order; thread = (row, 32-key word)
  pdl_trigger();
  pdl_wait();
  const int ntile = p.nq * (p.nq + 1) / 2;
  const int tile = static_cast<int>(blockIdx.x);
  const int z = tile / ntile, rem = tile - z * ntile;
  int qt = static_cast<int>((sqrtf(8.f * rem + 1.f) - 1.f) * 0.5f);  // largest qt with qt(qt+1)/2 <= rem
  if ((qt + 1) * (qt + 2) / 2 <= rem) ++qt;
  if (qt * (qt + 1) / 2 > rem) --qt;
  const int kt = rem - qt * (qt + 1) / 2;
  const int n = z / p.hl, jl = z - n * p.hl;
  const int row = threadIdx.x >> 2, w = threadIdx.x & 3;
  const unsigned long long e =
      (static_cast<unsigned long long>((n + p.n0) * p.hg + p.hoff + jl) * p.seq + qt * kTile + row) *
          static_cast<unsigned long long>(p.seq) +
      static_cast<unsigned long long>(kt) * kTile + 32 * w;
  PhiloxLite ph;
  philox_init(p, ph);
  uint32_t km[8];
  const uint32_t b0 = keep_masks16_bits(ph, p, e >> 4, km);
  const uint32_t b1 = keep_masks16_bits(ph, p, (e + 16) >> 4, km);
  p.mask_bits[static_cast<long long>(tile) * 512 + threadIdx.x] = b0 | (b1 << 16);
}

// D[z, i] = sum_d dO[i, d] * O[i, d] (head z's columns); DH/8 threads per row,
// one 16-byte vector of each operand per thread.
template <int DH>
__global__ void __launch_bounds__(256) attn_dsum_kernel(const __nv_bfloat16* __restrict__ dout,
                                                        const __nv_bfloat16* __restrict__ out, long long ld,
                                                        float* __restrict__ dsum, int seq, int hl, int col0,
                                                        long long rows) {
  pdl_trigger();
  pdl_wait();
  constexpr int TPR = DH / 8;  // threads per row (power of two <= 32)
  const long long row = (static_cast<long long>(blockIdx.x) * 256 + threadIdx.x) / TPR;
  const int sub = threadIdx.x % TPR;
  float acc = 0.f;
  if (row < rows) {
    const long long per = static_cast<long long>(hl) * seq;
    const int n = static_cast<int>(row / per);
    const int rem = static_cast<int>(row - n * per);
    const int jl = rem / seq, i = rem - jl * seq;
    const long long off = static_cast<long long>(n * seq + i) * ld + col0 + jl * DH + sub * 8;
    float a[8], b[8];
    vload(dout + off, a);
    vload(out + off, b);
#pragma unroll
    for (int e = 0; e < 8; ++e) acc += a[e] * b[e];
  }
#pragma unroll
  for (int o = TPR / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (row < rows && sub == 0) dsum[row] = acc;
}

template <int DH>
struct BwdCfg {
  static constexpr int TILE_BYTES = kTile * DH * 2;
  static constexpr int K_OFF = 0;
  static constexpr int V_OFF = TILE_BYTES;
  static constexpr int STAGE_OFF = 2 * TILE_BYTES;
  static constexpr int STAGE_BYTES = 2 * TILE_BYTES + 1024;  // Q_i, dO_i, lse_i[128], D_i[128]
  static constexpr int BUF_OFF = STAGE_OFF + 2 * STAGE_BYTES;
  static constexpr int BAR_OFF = BUF_OFF + kTile * kTile * 2;
  static constexpr int SMEM = BAR_OFF + 256;
  static constexpr uint32_t TMEM_COLS = 512;  // S, dP (128 each), dV, dK (DH each)
};

template <int DH>
__global__ void __launch_bounds__(kThreads, 1)
    attn_dkdv_kernel(const __grid_constant__ CUtensorMap tqkv, const __grid_constant__ CUtensorMap tdo,
                     const __grid_constant__ CUtensorMap tds, const AttnParams p) {
  pdl_trigger();
  using C = BwdCfg<DH>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
  uint64_t* kv_full = bars;
  uint64_t* st_full = bars + 1;   // [2] Q_i, dO_i, lse_i, D_i
  uint64_t* st_empty = bars + 3;  // [2]
  uint64_t* s_full = bars + 5;    // S_i in TMEM
  uint64_t* s_free = bars + 6;    // row warps read S_i
  uint64_t* dp_full = bars + 7;   // dP_i in TMEM
  uint64_t* dp_free = bars + 8;   // row warps read dP_i
  uint64_t* pd_full = bars + 9;   // keep o P_i in the buffer
  uint64_t* buf_free1 = bars + 10;  // dV MMA done with it
  uint64_t* ds_full = bars + 11;    // dS_i in the buffer
  uint64_t* buf_free2 = bars + 12;  // dK MMA done with it
  uint64_t* acc_full = bars + 13;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 14);

  CTRACE(0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kt = static_cast<int>(blockIdx.x) / p.Z;  // longest column (kt = 0) first
  const int z = static_cast<int>(blockIdx.x) % p.Z;
  const int n = z / p.hl, jl = z - n * p.hl;
  const int ni = p.nq - kt;
  const int row0 = n * p.seq;
  const uint32_t t_s = 0, t_dp = kTile, t_dv = 2 * kTile, t_dk = 2 * kTile + DH;

  if (threadIdx.x == 0) {
    if (smem_u32(smem) & 1023) __trap();
    mbar_init(kv_full, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&st_full[s], 1);
      mbar_init(&st_empty[s], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(s_free, kRowWarps);
    mbar_init(dp_full, 1);
    mbar_init(dp_free, kRowWarps);
    mbar_init(pd_full, kRowWarps);
    mbar_init(buf_free1, 1);
    mbar_init(ds_full, 1);
    mbar_init(buf_free2, 1);
    mbar_init(acc_full, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();

  if (warp == 0) {
    if (lane == 0) {
      tma_prefetch(&tqkv);
      tma_prefetch(&tdo);
      mbar_arrive_expect_tx(kv_full, 2 * C::TILE_BYTES);
#pragma unroll
      for (int g = 0; g < DH / 64; ++g) {
        tma_load_2d(smem + C::K_OFF + g * 16384, &tqkv, kv_full, p.k_col + jl * DH + g * 64, row0 + kt * kTile);
        tma_load_2d(smem + C::V_OFF + g * 16384, &tqkv, kv_full, p.v_col + jl * DH + g * 64, row0 + kt * kTile);
      }
      for (int it = 0; it < ni; ++it) {
        const int st = it & 1, i = kt + it;
        mbar_wait(&st_empty[st], ((it >> 1) & 1) ^ 1);
        ATRACE(0, it);
        uint8_t* sp = smem + C::STAGE_OFF + st * C::STAGE_BYTES;
        mbar_arrive_expect_tx(&st_full[st], C::STAGE_BYTES);
#pragma unroll
        for (int g = 0; g < DH / 64; ++g) {
          tma_load_2d(sp + g * 16384, &tqkv, &st_full[st], p.q_col + jl * DH + g * 64, row0 + i * kTile);
          tma_load_2d(sp + C::TILE_BYTES + g * 16384, &tdo, &st_full[st], p.do_col + jl * DH + g * 64,
                      row0 + i * kTile);
        }
        const long long ro = static_cast<long long>(z) * p.seq + i * kTile;
        bulk_load(sp + 2 * C::TILE_BYTES, p.lse + ro, 512, &st_full[st]);
        bulk_load(sp + 2 * C::TILE_BYTES + 512, p.dsum + ro, 512, &st_full[st]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // Issue order per query tile i: dV_i, S_{i+1}, dK_i, dP_{i+1} -- S_{i+1} runs under
      // the row warps' dS pass of tile i, dP_{i+1} under their P pass of tile i+1.
      constexpr uint32_t id_s = umma_idesc_bf16(kTile, kTile, 0, 0);
      constexpr uint32_t id_g = umma_idesc_bf16(kTile, DH, 1, 1);
      const uint32_t sb = smem_u32(smem);
      const uint32_t ka = sb + C::K_OFF, va = sb + C::V_OFF, buf = sb + C::BUF_OFF;
      auto stage_addr = [&](int it) { return sb + C::STAGE_OFF + (it & 1) * C::STAGE_BYTES; };
      auto issue_s = [&](int it) {  // S = Q_i K^T
        mbar_wait(&st_full[it & 1], (it >> 1) & 1);
        mbar_wait(s_free, (it & 1) ^ 1);
        tc_fence_after();
        const uint32_t qa = stage_addr(it);
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk) {
          const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
          umma_bf16(tmem + t_s, umma_desc_sw128(qa + off, 16, 1024), umma_desc_sw128(ka + off, 16, 1024), id_s,
                    kk > 0 ? 1u : 0u);
        }
        umma_commit(s_full);
      };
      auto issue_dp = [&](int it) {  // dP_drop = dO_i V^T
        mbar_wait(dp_free, (it & 1) ^ 1);
        tc_fence_after();
        const uint32_t da = stage_addr(it) + C::TILE_BYTES;
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk) {
          const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
          umma_bf16(tmem + t_dp, umma_desc_sw128(da + off, 16, 1024), umma_desc_sw128(va + off, 16, 1024), id_s,
                    kk > 0 ? 1u : 0u);
        }
        umma_commit(dp_full);
      };
      mbar_wait(kv_full, 0);
      issue_s(0);
      issue_dp(0);
      for (int it = 0; it < ni; ++it) {
        const uint32_t qa = stage_addr(it), da = qa + C::TILE_BYTES;
        // dV += (keep o P)^T dO   (A: keys x queries, MN-major view of the [query][key] buffer)
        mbar_wait(pd_full, it & 1);
        ATRACE(1, it);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < kTile / 16; ++kk)
          umma_bf16(tmem + t_dv, umma_desc_sw128(buf + kk * 2048, 16384, 1024),
                    umma_desc_sw128(da + kk * 2048, 16384, 1024), id_g, (it > 0 || kk > 0) ? 1u : 0u);
        umma_commit(buf_free1);
        if (it + 1 < ni) issue_s(it + 1);
        // dK += dS^T Q
        mbar_wait(ds_full, it & 1);
        ATRACE(2, it);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < kTile / 16; ++kk)
          umma_bf16(tmem + t_dk, umma_desc_sw128(buf + kk * 2048, 16384, 1024),
                    umma_desc_sw128(qa + kk * 2048, 16384, 1024), id_g, (it > 0 || kk > 0) ? 1u : 0u);
        umma_commit(&st_empty[it & 1]);
        umma_commit(buf_free2);
        if (it + 1 < ni) issue_dp(it + 1);
      }
      umma_commit(acc_full);
    }
  } else {
    // ------------------------------------------------ row warps: query row r of tile i, keys [c0, c0 + 64)
    const int q = warp & 3, hf = (warp - 2) >> 2;
    const int r = q * 32 + lane;
    const int c0 = hf * 64;
    const uint32_t tl = tmem + (static_cast<uint32_t>(q * 32) << 16);
    uint8_t* buf = smem + C::BUF_OFF;
    const bool leader = threadIdx.x == 64;
    PhiloxLite ph;
    philox_init(p, ph);
    // cached keep bits: the two words of query tile it + 1 load while tile it is processed
    const bool cached = p.thr && p.mask_mode == 2;
    uint32_t mw0 = 0u, mw1 = 0u;
    if (cached) {
      mw0 = p.mask_bits[mask_word(p, z, kt, kt, r, hf * 2)];
      mw1 = p.mask_bits[mask_word(p, z, kt, kt, r, hf * 2 + 1)];
    }
    for (int it = 0; it < ni; ++it) {
      const int st = it & 1, i = kt + it;
      const uint32_t bw0 = mw0, bw1 = mw1;
      if (cached && it + 1 < ni) {
        mw0 = p.mask_bits[mask_word(p, z, i + 1, kt, r, hf * 2)];
        mw1 = p.mask_bits[mask_word(p, z, i + 1, kt, r, hf * 2 + 1)];
      }
      const uint8_t* sp = smem + C::STAGE_OFF + st * C::STAGE_BYTES;
      mbar_wait(&st_full[st], (it >> 1) & 1);
      const float nlse = -reinterpret_cast<const float*>(sp + 2 * C::TILE_BYTES)[r];
      const float dsum = reinterpret_cast<const float*>(sp + 2 * C::TILE_BYTES + 512)[r];
      int lim = it == 0 ? r - c0 : 1 << 20;  // keys c0 + k > r are masked on the diagonal tile
      asm volatile("" : "+r"(lim));
      const unsigned long long ebase =
          (static_cast<unsigned long long>((n + p.n0) * p.hg + p.hoff + jl) * p.seq + i * kTile + r) *
              static_cast<unsigned long long>(p.seq) +
          static_cast<unsigned long long>(kt) * kTile + c0;
      // pass 1: P = exp2(S*sl2 - lse) (kept in registers as bf16), keep o P -> buffer
      mbar_wait(s_full, it & 1);
      if (warp == 2 && lane == 0) ATRACE(3, it);
      tc_fence_after();
      uint32_t u[2][32];
      tmem_ld32(tl + t_s + c0, u[0]);
      tmem_ld32(tl + t_s + c0 + 32, u[1]);
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(s_free);
      uint32_t pp[32];  // P, bf16x2
      const float2 sl2x2 = make_float2(p.sl2, p.sl2), nlse2 = make_float2(nlse, nlse);
#pragma unroll
      for (int k = 0; k < 64; k += 2) {
        const float2 e = fma2(make_float2(__uint_as_float(u[k >> 5][k & 31]), __uint_as_float(u[k >> 5][(k & 31) + 1])),
                              sl2x2, nlse2);
        float a = ex2(e.x), b = ex2(e.y);
        if (k > lim) a = 0.f;
        if (k + 1 > lim) b = 0.f;
        pp[k >> 1] = pack_bf16(a, b);
      }
      uint32_t pk[32];
#pragma unroll
      for (int k = 0; k < 32; ++k) pk[k] = pp[k];
      if (p.thr) {
        if (cached) {  // keep bits stored by the forward pass
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            uint32_t km[8];
            masks16_from_bits(((g >> 1) ? bw1 : bw0) >> (16 * (g & 1)), km);
#pragma unroll
            for (int k = 0; k < 8; ++k) pk[g * 8 + k] &= km[k];
          }
        } else {
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            uint32_t km[8];
            keep_masks16(ph, p, (ebase + g * 16) >> 4, km);
#pragma unroll
            for (int k = 0; k < 8; ++k) pk[g * 8 + k] &= km[k];
          }
        }
      }
      // the previous dK MMA and dS store must be done with the buffer
      if (it > 0) {
        mbar_wait(buf_free2, (it - 1) & 1);
        if (leader) bulk_wait_read0();
        named_bar_sync(1, 32 * kRowWarps);
      }
#pragma unroll
      for (int ch = 0; ch < 8; ++ch)
        *tile_chunk(buf, r, hf * 8 + ch) = make_uint4(pk[4 * ch], pk[4 * ch + 1], pk[4 * ch + 2], pk[4 * ch + 3]);
      fence_proxy_async();
      __syncwarp();
      if (warp == 2 && lane == 0) ATRACE(4, it);
      if (lane == 0) mbar_arrive(pd_full);
      // pass 2: dS = scale * (ks * (keep o P) o dP_drop - P D) -> buffer (after the dV MMA read it)
      mbar_wait(dp_full, it & 1);
      if (warp == 2 && lane == 0) ATRACE(5, it);
      tc_fence_after();
      uint32_t v[2][32];
      tmem_ld32(tl + t_dp + c0, v[0]);
      tmem_ld32(tl + t_dp + c0 + 32, v[1]);
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(dp_free);
      const float c1 = p.scale * p.ks, c2 = -p.scale * dsum;
      const float2 c1x2 = make_float2(c1, c1), c2x2 = make_float2(c2, c2), z2 = make_float2(0.f, 0.f);
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        const float2 pr = unpack_bf16(pp[k]);
        const float2 kp = unpack_bf16(pk[k]);
        // dS = (kp c1) dP + pr c2, two columns per packed instruction
        const float2 dp = make_float2(__uint_as_float(v[k >> 4][(2 * k) & 31]), __uint_as_float(v[k >> 4][(2 * k + 1) & 31]));
        const float2 d = fma2(fma2(kp, c1x2, z2), dp, fma2(pr, c2x2, z2));
        pk[k] = pack_bf16(d.x, d.y);
      }
      mbar_wait(buf_free1, it & 1);
      if (warp == 2 && lane == 0) ATRACE(6, it);
#pragma unroll
      for (int ch = 0; ch < 8; ++ch)
        *tile_chunk(buf, r, hf * 8 + ch) = make_uint4(pk[4 * ch], pk[4 * ch + 1], pk[4 * ch + 2], pk[4 * ch + 3]);
      fence_proxy_async();
      named_bar_sync(1, 32 * kRowWarps);
      if (leader) {
        ATRACE(7, it);
        mbar_arrive(ds_full);
        const int y = z * p.seq + i * kTile;
        tma_store_2d(&tds, buf, kt * kTile, y);
        tma_store_2d(&tds, buf + 16384, kt * kTile + 64, y);
        bulk_commit();
      }
    }
    // epilogue: rows r of this CTA's key tile, columns [hf*DH/2, +DH/2) of dV (x keep scale) and dK
    mbar_wait(acc_full, 0);
    tc_fence_after();
    __nv_bfloat16* base = static_cast<__nv_bfloat16*>(p.out) + static_cast<long long>(row0 + kt * kTile + r) * p.ld_out;
#pragma unroll
    for (int which = 0; which < 2; ++which) {
      __nv_bfloat16* dst = base + (which ? p.k_col : p.v_col) + jl * DH + hf * (DH / 2);
      const uint32_t tc = (which ? t_dk : t_dv) + hf * (DH / 2);
      const float sc = which ? 1.f : p.ks;
#pragma unroll
      for (int c = 0; c < DH / 64; ++c) {
        uint32_t o[32];
        tmem_ld32(tl + tc + c * 32, o);
        tmem_wait_ld();
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float* f = reinterpret_cast<const float*>(o + 8 * k);
          *reinterpret_cast<uint4*>(dst + c * 32 + k * 8) =
              make_uint4(pack_bf16(f[0] * sc, f[1] * sc), pack_bf16(f[2] * sc, f[3] * sc),
                         pack_bf16(f[4] * sc, f[5] * sc), pack_bf16(f[6] * sc, f[7] * sc));
        }
      }
    }
    if (leader) bulk_wait0();
    CTRACE(1);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, C::TMEM_COLS);
  }
}

template <typename K>
cudaError_t set_smem(K kernel, int bytes) {
  return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

bool fill_common(AttnParams& p, const oases_attn_desc& d, std::string* err) {
  if (d.head_dim != 64 && d.head_dim != 128) {
    *err = "attention: head_dim must be 64 or 128";
    return false;
  }
  if (d.seq <= 0 || d.seq % kTile) {
    *err = "attention: seq must be a positive multiple of 128";
    return false;
  }
  if (d.samples <= 0 || d.heads_local <= 0 || d.heads_total < d.heads_local || d.head_offset < 0 ||
      d.head_offset + d.heads_local > d.heads_total) {
    *err = "attention: bad head / sample counts";
    return false;
  }
  const long long hd = static_cast<long long>(d.heads_local) * d.head_dim;
  if (d.ld_qkv < 3 * hd || d.ld_qkv % 8 || d.ld_out < hd || d.ld_out % 8) {
    *err = "attention: qkv rows need >= 3*heads*head_dim columns, ctx rows >= heads*head_dim (ld % 8 == 0)";
    return false;
  }
  p.seq = d.seq;
  p.hl = d.heads_local;
  p.hg = d.heads_total;
  p.hoff = d.head_offset;
  p.n0 = d.sample_offset;
  p.Z = d.samples * d.heads_local;
  p.nq = d.seq / kTile;
  p.q_col = 0;
  p.k_col = static_cast<int>(hd);
  p.v_col = static_cast<int>(2 * hd);
  p.do_col = 0;
  p.sl2 = d.scale * kLog2e;
  p.scale = d.scale;
  p.thr = dropout_threshold(d.dropout_p);
  p.ks = dropout_keep_scale(d.dropout_p);
  p.seed = d.seed;
  p.offset = d.offset;
  p.mask_bits = d.mask_bits;
  p.mask_mode = (d.mask_bits && p.thr) ? d.mask_mode : 0;
  if (p.mask_mode < 0 || p.mask_mode > 2) {
    *err = "attention: mask_mode must be 0, 1 or 2";
    return false;
  }
  uint32_t a = static_cast<uint32_t>(d.seed), b = static_cast<uint32_t>(d.seed >> 32);
  for (int r = 0; r < 10; ++r) {
    p.rk0[r] = a;
    p.rk1[r] = b;
    a += 0x9E3779B9u;
    b += 0xBB67AE85u;
  }
  return true;
}

}  // namespace

#ifdef OASES_EXP_TRACE
extern "C" int oases_attn_trace_dump(unsigned long long* host) {
  return static_cast<int>(cudaMemcpyFromSymbol(host, g_attn_trace, sizeof(unsigned long long) * 8 * 64));
}
extern "C" int oases_attn_cta_dump(unsigned long long* host) {
  return static_cast<int>(cudaMemcpyFromSymbol(host, g_cta_trace, sizeof(unsigned long long) * 3 * 1024));
}
#endif

bool attention_supported(int dtype, int head_dim, int seq) {
  return dtype == OASES_BF16 && (head_dim == 64 || head_dim == 128) && seq > 0 && seq % kTile == 0;
}

size_t attention_mask_bytes(const oases_attn_desc& d) {
  if (d.seq <= 0 || d.seq % kTile) return 0;
  const long long nq = d.seq / kTile;
  return static_cast<size_t>(d.samples) * d.heads_local * (nq * (nq + 1) / 2) * kTile * 4 * sizeof(uint32_t);
}

size_t attention_bwd_workspace(const oases_attn_desc& d) {
  return static_cast<size_t>(d.samples) * d.heads_local * d.seq * sizeof(float);
}

GemmStatus attention_fwd(const oases_attn_desc& d, cudaStream_t stream) {
  GemmStatus st;
  AttnParams p{};
  if (d.dtype != OASES_BF16) {
    st.err = "attention: fused kernels are bf16-only";
    return st;
  }
  if (!fill_common(p, d, &st.err)) return st;
  if (!d.qkv || !d.out || !d.lse) {
    st.err = "attention_fwd: null qkv / out / lse";
    return st;
  }
  const long long rows = static_cast<long long>(d.samples) * d.seq;
  CUtensorMap tqkv;
  if (!make_tma_bf16_2d(&tqkv, d.qkv, rows, 3LL * d.heads_local * d.head_dim, d.ld_qkv, 64, kTile, &st.err))
    return st;
  p.out = d.out;
  p.ld_out = d.ld_out;
  p.lse = d.lse;
  static const bool fwd2_on = [] {
    const char* e = std::getenv("OASES_ATTN_FWD2");
    return !(e && e[0] == '0');
  }();
  // The ping-pong kernel reads cached keep bits only (the stack's mask pass,
  // mask_mode 2), and needs enough tile pairs to balance its persistent grid:
  // measured at the C2 sub-batch (256 pairs) 36.3 vs 38.8 us, at a C3 TMP=8
  // rank (128 pairs of very unequal length) 46 vs 31 us.
  int nsm = 148;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  static const int pv_wait = [] {
    const char* e = std::getenv("OASES_ATTN_PV_WAIT");
    return e && e[0] == '1' ? 1 : 0;
  }();
  p.pv_wait = pv_wait;
  const bool fwd2 = fwd2_on && (!p.thr || p.mask_mode == 2) && 2LL * p.Z * ((p.nq + 1) / 2) >= 3LL * nsm;
  unsigned grid = static_cast<unsigned>(fwd2 ? p.Z * ((p.nq + 1) / 2) : p.Z * p.nq);
  {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (grid > static_cast<unsigned>(sms)) grid = static_cast<unsigned>(sms);  // persistent: one CTA per SM
    // leave SMs to the overlapped collectives when the caller caps the persistent grids
    if (d.max_ctas > 0 && grid > static_cast<unsigned>(d.max_ctas)) grid = static_cast<unsigned>(d.max_ctas);
  }
  cudaError_t e;
  if (fwd2 && d.head_dim == 128) {
    static cudaError_t once = set_smem(attn_fwd2_kernel<128>, Fwd2Cfg<128>::SMEM);
    if ((e = once) == cudaSuccess)
      e = launch_pdl(attn_fwd2_kernel<128>, dim3(grid), dim3(kFwd2Threads), Fwd2Cfg<128>::SMEM, stream, tqkv, p);
  } else if (fwd2) {
    static cudaError_t once = set_smem(attn_fwd2_kernel<64>, Fwd2Cfg<64>::SMEM);
    if ((e = once) == cudaSuccess)
      e = launch_pdl(attn_fwd2_kernel<64>, dim3(grid), dim3(kFwd2Threads), Fwd2Cfg<64>::SMEM, stream, tqkv, p);
  } else if (d.head_dim == 128) {
    static cudaError_t once = set_smem(attn_fwd_kernel<128>, FwdCfg<128>::SMEM);
    if ((e = once) == cudaSuccess) {
      e = launch_pdl(attn_fwd_kernel<128>, dim3(grid), dim3(kFwdThreads), FwdCfg<128>::SMEM, stream, tqkv, p);
    }
  } else {
    static cudaError_t once = set_smem(attn_fwd_kernel<64>, FwdCfg<64>::SMEM);
    if ((e = once) == cudaSuccess) {
      e = launch_pdl(attn_fwd_kernel<64>, dim3(grid), dim3(kFwdThreads), FwdCfg<64>::SMEM, stream, tqkv, p);
    }
  }
  if (e != cudaSuccess) {
    st.err = std::string("attention_fwd launch: ") + cudaGetErrorString(e);
    st.cuda = true;
    return st;
  }
  st.ok = true;
  return st;
}

GemmStatus attention_masks(const oases_attn_desc& d, cudaStream_t stream) {
  GemmStatus st;
  AttnParams p{};
  if (!fill_common(p, d, &st.err)) return st;
  if (!d.mask_bits || !p.thr) {
    st.err = "attention_masks: needs mask_bits and dropout_p > 0";
    return st;
  }
  const long long tiles = static_cast<long long>(p.Z) * (p.nq * (p.nq + 1) / 2);
  const cudaError_t e = launch_pdl(attn_mask_kernel, dim3(static_cast<unsigned>(tiles)), dim3(512), 0, stream, p);
  if (e != cudaSuccess) {
    st.err = std::string("attention_masks launch: ") + cudaGetErrorString(e);
    st.cuda = true;
    return st;
  }
  st.ok = true;
  return st;
}

GemmStatus attention_bwd(const oases_attn_desc& d, cudaStream_t stream) {
  GemmStatus st;
  AttnParams p{};
  if (d.dtype != OASES_BF16) {
    st.err = "attention: fused kernels are bf16-only";
    return st;
  }
  if (!fill_common(p, d, &st.err)) return st;
  if (!d.qkv || !d.out || !d.lse || !d.dout || !d.dqkv || !d.ds || !d.workspace) {
    st.err = "attention_bwd: null qkv / out / lse / dout / dqkv / ds / workspace";
    return st;
  }
  if (d.ld_dout < static_cast<long long>(d.heads_local) * d.head_dim || d.ld_dout % 8 || d.ld_dqkv % 8 ||
      d.ld_dqkv < 3LL * d.heads_local * d.head_dim) {
    st.err = "attention_bwd: bad dout / dqkv leading dimensions";
    return st;
  }
  const long long rows = static_cast<long long>(d.samples) * d.seq;
  const long long hd = static_cast<long long>(d.heads_local) * d.head_dim;
  CUtensorMap tqkv, tdo, tds;
  if (!make_tma_bf16_2d(&tqkv, d.qkv, rows, 3 * hd, d.ld_qkv, 64, kTile, &st.err)) return st;
  if (!make_tma_bf16_2d(&tdo, d.dout, rows, hd, d.ld_dout, 64, kTile, &st.err)) return st;
  if (!make_tma_bf16_2d(&tds, d.ds, static_cast<long long>(p.Z) * d.seq, d.seq, d.seq, 64, kTile, &st.err))
    return st;
  float* dsum = static_cast<float*>(d.workspace);
  // D = rowsum(dO o O) (ld of out must equal ld of dout for the shared row walk)
  if (d.ld_out != d.ld_dout) {
    st.err = "attention_bwd: out and dout must share a leading dimension";
    return st;
  }
  const long long drows = static_cast<long long>(p.Z) * d.seq;
  const unsigned dgrid = static_cast<unsigned>((drows * (d.head_dim / 8) + 255) / 256);
  const auto* dO = static_cast<const __nv_bfloat16*>(d.dout);
  const auto* O = static_cast<const __nv_bfloat16*>(d.out);
  cudaError_t e = cudaSuccess;
  if (!d.dsum_ready)  // else the GEMM that produced dO wrote D (EPI_ROWDOT)
    e = d.head_dim == 128 ? launch_pdl(attn_dsum_kernel<128>, dim3(dgrid), dim3(256), 0, stream, dO, O, d.ld_dout,
                                       dsum, d.seq, d.heads_local, 0, drows)
                          : launch_pdl(attn_dsum_kernel<64>, dim3(dgrid), dim3(256), 0, stream, dO, O, d.ld_dout,
                                       dsum, d.seq, d.heads_local, 0, drows);
  if (e == cudaSuccess) {
    p.out = d.dqkv;
    p.ld_out = d.ld_dqkv;
    p.lse = const_cast<float*>(d.lse);
    p.dsum = dsum;
    const unsigned grid = static_cast<unsigned>(p.Z * p.nq);
    if (d.head_dim == 128) {
      static cudaError_t once = set_smem(attn_dkdv_kernel<128>, BwdCfg<128>::SMEM);
      if ((e = once) == cudaSuccess) {
        e = launch_pdl(attn_dkdv_kernel<128>, dim3(grid), dim3(kThreads), BwdCfg<128>::SMEM, stream, tqkv, tdo,
                       tds, p);
      }
    } else {
      static cudaError_t once = set_smem(attn_dkdv_kernel<64>, BwdCfg<64>::SMEM);
      if ((e = once) == cudaSuccess) {
        e = launch_pdl(attn_dkdv_kernel<64>, dim3(grid), dim3(kThreads), BwdCfg<64>::SMEM, stream, tqkv, tdo,
                       tds, p);
      }
    }
  }
  if (e != cudaSuccess) {
    st.err = std::string("attention_bwd launch: ") + cudaGetErrorString(e);
    st.cuda = true;
    return st;
  }
  // dQ = dS K per (sample, head): causal K range, deterministic tcgen05 GEMM.
  oases_gemm_desc g{};
  g.dtype = OASES_BF16;
  g.c_dtype = OASES_BF16;
  g.M = d.seq;
  g.N = d.head_dim;
  g.K = d.seq;
  g.batch = p.Z;
  g.batch_inner = d.heads_local;
  g.a = oases_gemm_operand{d.ds, static_cast<long long>(p.Z) * d.seq, d.seq, d.seq, 0, 0,
                           {static_cast<long long>(d.heads_local) * d.seq, d.seq}, {0, 0}};
  g.b = oases_gemm_operand{static_cast<const char*>(d.qkv) + hd * 2, rows, 2 * hd, d.ld_qkv, 1, 0,
                           {d.seq, 0}, {0, d.head_dim}};
  g.c = d.dqkv;
  g.ldc = d.ld_dqkv;
  g.c_row_off[0] = d.seq;
  g.c_col_off[1] = d.head_dim;
  g.alpha = 1.f;
  g.causal = OASES_CAUSAL_K_UPTO_M;
  g.max_ctas = d.max_ctas;
  return gemm_tc(g, stream);
}

}  // namespace oases
