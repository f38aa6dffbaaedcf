// TMP transformer layer stack on one device: parameters, the saved post-
// AllReduce boundary tensors, workspaces, and the kernel list of every plan op
// (F_b forward, R_b recompute, B_b backward, the LN_0 tail) for one worker.
//
// Block partition (SURVEY.md §8(a) note; the value semantics are the fp64
// oracle's, oracle/gpt_oracle.cpp, whose FFN-only reduction is the reference
// toy numerics.cpp:158-210):
//   F_b : x_b = (res ? x_{b-1} : 0) + dropout(AR_{b-1} + bias_row_{b-1})   [bdr, b > 0]
//         ln = LN(x_b); col = ln W_col^T + b_col; attention(qkv) | gelu(pre);
//         partial_b = act W_row^T  -> AR_b (forward g)
//   R_b : same from the STORED x_b, without the row GEMM and without any
//         collective (Oases elision, Eq. 1 / numerics.cpp:198-199); CrossPass
//         replays the unit, rebuilding x_b from the replayed AR_{b-1}.
//   B_b : LN_{b+1} backward on the all-reduced d_ln_{b+1} (+ residual add),
//         or the loss head for the last block; dropout'/bias grad; row GEMM
//         wgrad/dgrad; attention or dGeLU backward; column GEMM wgrad;
//         d_ln partial -> AR_b (backward f).
//   tail: LN_0 backward after the last backward AR -> dX.
// Weight gradients accumulate in f32 across the two sub-batches in issue
// order; column reductions (bias, LN gamma/beta) are deterministic.
#include "stack.h"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../kernels/gemm.h"
#include "../kernels/kernels.h"
#include "status.h"

namespace oases {

using tmpsim::ConfigError;

// ================================================================== context
Context::~Context() {
  if (nccl) ncclCommDestroy(nccl);
  if (compute) cudaStreamDestroy(compute);
  if (comm) cudaStreamDestroy(comm);
  if (side) cudaStreamDestroy(side);
  if (fork_ev) cudaEventDestroy(fork_ev);
  if (join_ev) cudaEventDestroy(join_ev);
}

static void check_nccl(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw NcclError(std::string(what) + ": " + ncclGetErrorString(r));
}

std::unique_ptr<Context> make_context(const oases_ctx_desc& d) {
  if (d.tp < 1) throw ConfigError("ctx: tp must be >= 1");
  if (d.local_workers != 1 && d.local_workers != d.tp)
    throw ConfigError("ctx: local_workers must be 1 (one rank per process) or equal tp (in-process emulation)");
  if (d.local_workers > 8) throw ConfigError("ctx: at most 8 in-process workers");
  if (d.tp > 1 && d.local_workers == 1 && !d.unique_id && !d.comm_disabled)
    throw ConfigError("ctx: tp > 1 with one rank per process needs the NCCL unique id");
  if (d.rank < 0 || (d.local_workers == 1 && d.rank >= d.tp)) throw ConfigError("ctx: rank out of range");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    throw CudaError("no CUDA device: the Oases runtime has no CPU fallback");
  }
  check_cuda(cudaSetDevice(d.device), "cudaSetDevice");
  auto ctx = std::make_unique<Context>();
  ctx->tp = d.tp;
  ctx->rank = d.local_workers == 1 ? d.rank : 0;
  ctx->device = d.device;
  ctx->local_workers = d.local_workers;
  ctx->gemm_max_ctas = d.gemm_max_ctas;
  ctx->nccl_max_ctas = d.nccl_max_ctas;
  int lo = 0, hi = 0;
  check_cuda(cudaDeviceGetStreamPriorityRange(&lo, &hi), "stream priorities");
  check_cuda(cudaStreamCreateWithPriority(&ctx->compute, cudaStreamNonBlocking, lo), "compute stream");
  // The comm stream gets the highest priority so NCCL's CTAs are scheduled as
  // soon as the overlapped GEMM frees SMs.
  check_cuda(cudaStreamCreateWithPriority(&ctx->comm, cudaStreamNonBlocking, hi), "comm stream");
  check_cuda(cudaStreamCreateWithPriority(&ctx->side, cudaStreamNonBlocking, lo), "side stream");
  check_cuda(cudaEventCreateWithFlags(&ctx->fork_ev, cudaEventDisableTiming), "fork event");
  check_cuda(cudaEventCreateWithFlags(&ctx->join_ev, cudaEventDisableTiming), "join event");
  ctx->comm_disabled = d.comm_disabled != 0;
  // tp == 1 with an id: a single-rank NCCL communicator (AllReduce is the
  // identity) -- exercises the NCCL path, including graph capture, on one GPU.
  if (d.local_workers == 1 && !ctx->comm_disabled && (d.tp > 1 || d.unique_id)) {
    ncclUniqueId id;
    static_assert(sizeof(ncclUniqueId) == OASES_UNIQUE_ID_BYTES, "unique id size");
    std::memcpy(&id, d.unique_id, sizeof(id));
    ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
    if (d.nccl_max_ctas > 0) cfg.maxCTAs = d.nccl_max_ctas;
    check_nccl(ncclCommInitRankConfig(&ctx->nccl, d.tp, id, d.rank, &cfg), "ncclCommInitRankConfig");
  }
  return ctx;
}

// ================================================================== arena
DeviceArena::~DeviceArena() {
  for (auto& b : blocks_) cudaFree(b.first);
}

void DeviceArena::release(void* p) {
  if (!p) return;
  for (size_t i = 0; i < blocks_.size(); ++i)
    if (blocks_[i].first == p) {
      check_cuda(cudaFree(p), "cudaFree");
      total_ -= blocks_[i].second;
      blocks_.erase(blocks_.begin() + static_cast<std::ptrdiff_t>(i));
      return;
    }
  throw ConfigError("arena: release of a pointer it does not own");
}

void* DeviceArena::alloc(size_t bytes) {
  bytes = (bytes + 255) & ~size_t(255);
  if (bytes == 0) bytes = 256;
  void* p = nullptr;
  check_cuda(cudaMalloc(&p, bytes), "cudaMalloc");
  check_cuda(cudaMemset(p, 0, bytes), "cudaMemset");
  blocks_.emplace_back(p, bytes);
  total_ += bytes;
  return p;
}

// ================================================================== stack
namespace {
uint64_t drop_offset(int block, int sb, int kind) { return (static_cast<uint64_t>(block) * 2 + sb) * 4 + kind; }

oases_gemm_operand operand(const void* ptr, int64_t rows, int64_t cols, int64_t ld, bool mn, int64_t r0 = 0,
                           int64_t r1 = 0, int64_t c0 = 0, int64_t c1 = 0) {
  oases_gemm_operand o{};
  o.ptr = ptr;
  o.rows = rows;
  o.cols = cols;
  o.ld = ld;
  o.mn_major = mn ? 1 : 0;
  o.row_off[0] = r0;
  o.row_off[1] = r1;
  o.col_off[0] = c0;
  o.col_off[1] = c1;
  return o;
}
}  // namespace

Stack::Stack(Context& ctx, const ModelCfg& cfg, const std::vector<int>& degrees) : ctx_(ctx), cfg_(cfg) {
  const int t = ctx.tp;
  if (cfg.h <= 0 || cfg.s <= 0 || cfg.b <= 0 || cfg.layers < 0) throw ConfigError("stack: sizes must be positive");
  if (cfg.b % 2) throw ConfigError("stack: global_batch must be even (two sub-batches)");
  if (cfg.bytes != 2 && cfg.bytes != 4 && cfg.bytes != 8)
    throw ConfigError("stack: bytes_per_element must be 2 (bf16), 4 (f32) or 8 (f64 value-level toy mode)");
  if (cfg.bytes == 8 && (cfg.attention || cfg.ln || cfg.p_hidden > 0.f || cfg.p_attn > 0.f))
    throw ConfigError("stack: f64 mode runs the reference's toy FFN blocks (numerics.hpp:35-60): no attention, "
                      "LayerNorm or dropout");
  // 16-byte vector loads in LayerNorm / softmax rows
  if ((cfg.ln && cfg.h % 8) || (cfg.attention && (cfg.s % 8 || cfg.h % 8)))
    throw ConfigError("stack: hidden (with LayerNorm/attention) and seq must be multiples of 8");
  nblocks_ = oases::num_blocks(cfg);
  // per-block degrees (F2): each divides the world; a degree-d block runs on N/d
  // data-parallel groups, each with an even number of samples (two sub-batches)
  deg_ = resolve_degrees(cfg, t, degrees, &mixed_);
  if (mixed_ && cfg.p_hidden > 0.f)
    throw ConfigError("stack: mixed per-block degrees need hidden_dropout 0 (hidden-dropout masks are keyed per "
                      "sub-batch tensor, which the degree changes re-slice)");
  if (mixed_ && ctx.comm_disabled) throw ConfigError("stack: mixed per-block degrees need the collectives");
  if (mixed_ && cfg.bytes == 8) throw ConfigError("stack: mixed per-block degrees run in bf16 or f32");
  // heads per rank at the world degree: (samples per sub-batch) x (local heads) is
  // the same at every degree, so the attention buffers are sized with it
  hl_ = cfg.attention ? cfg.heads / t : 0;
  dh_ = cfg.attention ? cfg.h / cfg.heads : 0;
  for (int b = 0; b < nblocks_; ++b) {
    const int d = degree(b);
    if (dtype() == OASES_BF16) {
      // tcgen05 tiles: K extents must be multiples of 64 (TMA zero-fill only at
      // buffer edges), attention sequences whole 128-row tiles.
      const int64_t k_dims[] = {cfg.h, cfg.f / d, ts(b)};
      for (int64_t k : k_dims)
        if (k % 64) throw ConfigError("stack: bf16 mode needs hidden, ffn/degree and tokens per sub-batch % 64 == 0");
      if (cfg.attention && (cfg.s % 128 || dh_ % 64 || nrow(b) % 64))
        throw ConfigError("stack: bf16 attention needs seq % 128 == 0 and head dim % 64 == 0");
    }
  }
  // Fused bias-dropout-residual + LayerNorm unless OASES_FUSED_BDR_LN=0 (A/B runs).
  {
    const char* e = std::getenv("OASES_FUSED_BDR_LN");
    fuse_bdr_ln_ = !(e && e[0] == '0');
  }
  // the fused forward kernel caches the hidden-dropout decisions for the backward
  // persistent LayerNorm backward with the parameter / row-bias column sums folded in (rowpipe.cu)
  lnp_bwd_ = cfg.ln && lnp_enabled() && lnp_supported(static_cast<int64_t>(cfg.b / 2) * cfg.s, static_cast<int>(cfg.h));
  hbits_ = cfg.ln && fuse_bdr_ln_ && cfg.p_hidden > 0.f && cfg.h % 16 == 0 &&
           bdr_layernorm_supported(static_cast<int64_t>(cfg.b / 2) * cfg.s, static_cast<int>(cfg.h)) &&
           (lnp_bwd_ || ln_bwd_dropout_supported(cfg.bytes == 2 ? OASES_BF16 : OASES_F32,
                                                 static_cast<int64_t>(cfg.b / 2) * cfg.s, static_cast<int>(cfg.h)));
  // FFN column-bias gradient from the FC2 dgrad epilogue's partials unless OASES_FUSED_COLSUM=0
  {
    const char* e = std::getenv("OASES_FUSED_COLSUM");
    colsum_ = cfg.bias && cfg.bytes == 2 && !(e && e[0] == '0');
    for (int b = 0; b < nblocks_; ++b)
      if (!is_attention(b) && (ts(b) % 32 || ncol(b) % 32)) colsum_ = false;
  }
  // Fused tcgen05 attention unless OASES_FUSED_ATTN=0 (A/B runs of the unfused chain).
  {
    const char* e = std::getenv("OASES_FUSED_ATTN");
    fused_attn_ = cfg.attention && attention_supported(dtype(), dh_, static_cast<int>(cfg.s)) && !(e && e[0] == '0');
  }
  const int W = ctx.local_workers;
  workers_.resize(static_cast<size_t>(W));
  for (int w = 0; w < W; ++w) workers_[static_cast<size_t>(w)].rank = W > 1 ? w : ctx.rank;
  alloc_all();
  touched_.assign(static_cast<size_t>(W), std::vector<std::array<bool, OASES_P_COUNT>>(static_cast<size_t>(nblocks_)));
  bwd_seen_.assign(static_cast<size_t>(W), std::vector<bool>(static_cast<size_t>(nblocks_), false));
  loss_touched_.assign(static_cast<size_t>(W), false);
  computed_at_.assign(static_cast<size_t>(nblocks_), {});
  // NCCL sub-communicators of the mixed degrees, split in the same order on every rank
  if (mixed_ && ctx.local_workers == 1 && ctx.nccl) {
    std::vector<int> ds(deg_.begin(), deg_.end());
    std::sort(ds.begin(), ds.end());
    ds.erase(std::unique(ds.begin(), ds.end()), ds.end());
    for (int d : ds) {
      if (d == t) continue;
      ncclComm_t c = nullptr;
      check_nccl(ncclCommSplit(ctx.nccl, group_of(ctx.rank, d), rank_in_group(ctx.rank, d), &c, nullptr),
                 "ncclCommSplit (tp group)");
      tp_comms_.emplace_back(d, c);
      check_nccl(ncclCommSplit(ctx.nccl, rank_in_group(ctx.rank, d), group_of(ctx.rank, d), &c, nullptr),
                 "ncclCommSplit (dp group)");
      dp_comms_.emplace_back(d, c);
    }
  }
}

Stack::~Stack() {
  for (cudaEvent_t e : tev_) cudaEventDestroy(e);
  for (auto& c : tp_comms_) ncclCommDestroy(c.second);
  for (auto& c : dp_comms_) ncclCommDestroy(c.second);
}

void Stack::kernel_stats(double* gemm_ms, double* gemm_flops, int* launches) {
  double ms = 0.0, fl = 0.0;
  if (timed_) check_cuda(cudaEventSynchronize(tev_[2 * timed_ - 1]), "kernel stats sync");
  for (size_t i = 0; i < timed_; ++i) {
    float t = 0.f;
    check_cuda(cudaEventElapsedTime(&t, tev_[2 * i], tev_[2 * i + 1]), "elapsed");
    ms += t;
    fl += tflops_[i];
  }
  *gemm_ms = ms;
  *gemm_flops = fl;
  *launches = static_cast<int>(timed_);
}

int64_t Stack::param_numel(int block, int p) const {
  if (block < 0 || block >= nblocks_ || p < 0 || p >= OASES_P_COUNT) return 0;
  return workers_.front().params[static_cast<size_t>(block)].numel[p];
}

void* Stack::gp(void* base, const Worker& w, int b, int sb, int64_t cols) const {
  return static_cast<char*>(base) + static_cast<size_t>(row0(w, b) + sb * ts(b)) * cols * esize();
}

void* Stack::lp(void* base, int b, int sb, int64_t cols) const {
  return static_cast<char*>(base) + static_cast<size_t>(sb) * ts(b) * cols * esize();
}

void Stack::alloc_all() {
  const int64_t T = static_cast<int64_t>(cfg_.b) * cfg_.s, h = cfg_.h;
  const size_t es = esize();
  // Per-rank extents: a block's tokens per sub-batch grow with its degree while
  // its column widths shrink, so the workspaces are sized by the largest
  // products over the blocks (all equal when the degrees are uniform).
  int64_t Ts = 0, tcol = 0, trow = 0, tffn = 0;
  for (int b = 0; b < nblocks_; ++b) {
    Ts = std::max(Ts, ts(b));
    tcol = std::max(tcol, ts(b) * ncol(b));
    trow = std::max(trow, ts(b) * std::max<int64_t>(nrow(b), 1));
    if (!is_attention(b)) tffn = std::max(tffn, ts(b) * ncol(b));
  }
  if (nblocks_ == 0) Ts = tokens_sub();
  // the attention extents (samples x local heads) do not depend on the degree
  const int64_t bh = cfg_.b / 2;
  const int64_t prob = cfg_.attention ? bh * hl_ * cfg_.s * static_cast<int64_t>(cfg_.s) : 0;
  const int nslots = cfg_.recompute ? std::min(2, nblocks_) : nblocks_;
  size_t colws = colsum_workspace(2 * Ts, static_cast<int>(h));
  for (int b = 0; b < nblocks_; ++b)
    colws = std::max(colws, colsum_workspace(2 * ts(b), static_cast<int>(std::max<int64_t>(ncol(b), 1))));
  for (Worker& w : workers_) {
    w.params.resize(static_cast<size_t>(nblocks_));
    for (int b = 0; b < nblocks_; ++b) {
      BlockParams& bp = w.params[static_cast<size_t>(b)];
      const int64_t nc = ncol(b), nr = nrow(b);
      bp.numel[OASES_P_LN_GAMMA] = cfg_.ln ? h : 0;
      bp.numel[OASES_P_LN_BETA] = cfg_.ln ? h : 0;
      bp.numel[OASES_P_W_COL] = nc * h;
      bp.rows[OASES_P_W_COL] = static_cast<int>(nc);
      bp.numel[OASES_P_B_COL] = cfg_.bias ? nc : 0;
      bp.numel[OASES_P_W_ROW] = h * nr;
      bp.rows[OASES_P_W_ROW] = static_cast<int>(h);
      bp.numel[OASES_P_B_ROW] = cfg_.bias ? h : 0;
      for (int p = 0; p < OASES_P_COUNT; ++p) {
        if (!bp.numel[p]) continue;
        bp.p[p] = arena_.alloc(static_cast<size_t>(bp.numel[p]) * es);
        bp.g[p] = static_cast<float*>(arena_.alloc(static_cast<size_t>(bp.numel[p]) * gsize()));
      }
      if (cfg_.ln) {
        check_cuda(fill_const(dtype(), bp.p[OASES_P_LN_GAMMA], h, 1.f, nullptr), "fill gamma");
      }
    }
    w.input = arena_.alloc(static_cast<size_t>(T * h) * es);
    w.grad = arena_.alloc(static_cast<size_t>(T * h) * es);
    // x_0 is the input; the other residual-stream buffers are placed by
    // bind_storage (all dedicated until a plan is bound)
    w.xbase.assign(static_cast<size_t>(nblocks_), nullptr);
    w.x_own.assign(static_cast<size_t>(nblocks_), nullptr);
    if (nblocks_ > 0) w.xbase[0] = w.x_own[0] = w.input;
    for (int par = 0; par < 2; ++par) {
      w.fwd_ar[par] = arena_.alloc(static_cast<size_t>(T * h) * es);
      w.bwd_ar[par] = arena_.alloc(static_cast<size_t>(T * h) * es);
      if (cfg_.recompute) w.rec_ar[par] = arena_.alloc(static_cast<size_t>(T * h) * es);
    }
    w.ws.resize(static_cast<size_t>(nslots));
    w.ln_full.assign(static_cast<size_t>(nslots), nullptr);
    w.act_full.assign(static_cast<size_t>(nslots), nullptr);
    for (int slot = 0; slot < nslots; ++slot) {
      // the weight-gradient GEMMs read the two sub-batches' LN output and
      // activation as one [2 T_sub, .] operand: both halves of a slot are one
      // allocation (ws_for points ws.ln / ws.act at the block's halves)
      w.ln_full[static_cast<size_t>(slot)] = cfg_.ln ? arena_.alloc(static_cast<size_t>(2 * Ts * h) * es) : nullptr;
      w.act_full[static_cast<size_t>(slot)] = arena_.alloc(static_cast<size_t>(2 * trow) * es);
      for (int sb = 0; sb < 2; ++sb) {
        Workspace& ws = w.ws[static_cast<size_t>(slot)][static_cast<size_t>(sb)];
        ws.col = arena_.alloc(static_cast<size_t>(tcol) * es);
        if (prob && fused_attn_) {
          ws.lse = static_cast<float*>(arena_.alloc(static_cast<size_t>(bh * hl_ * cfg_.s) * sizeof(float)));
        } else if (prob) {
          ws.p = arena_.alloc(static_cast<size_t>(prob) * es);
          ws.pd = cfg_.p_attn > 0.f ? arena_.alloc(static_cast<size_t>(prob) * es) : ws.p;
        }
      }
    }
    w.gar = arena_.alloc(static_cast<size_t>(2 * Ts * h) * es);  // [sb][T_sub, h]
    w.du = arena_.alloc(static_cast<size_t>(trow) * es);
    w.dcol = arena_.alloc(static_cast<size_t>(2 * tcol) * es);  // [sb][T_sub, ncol] of the block
    if (prob) w.dp = arena_.alloc(static_cast<size_t>(prob) * es);
    if (prob && fused_attn_) w.attn_ws = arena_.alloc(static_cast<size_t>(bh * hl_ * cfg_.s) * sizeof(float));
    if (hbits_) {
      w.hbits.assign(static_cast<size_t>(nblocks_), {nullptr, nullptr});
      for (int b = 0; b + 1 < nblocks_; ++b)
        for (int sb = 0; sb < 2; ++sb)
          w.hbits[static_cast<size_t>(b)][static_cast<size_t>(sb)] =
              static_cast<uint16_t*>(arena_.alloc(static_cast<size_t>(Ts * h / 16) * sizeof(uint16_t)));
    }
    if (prob && fused_attn_ && cfg_.p_attn > 0.f) {
      oases_attn_desc md{};
      md.samples = static_cast<int>(bh);
      md.heads_local = hl_;
      md.seq = static_cast<int>(cfg_.s);
      const size_t mbytes = attention_mask_bytes(md);
      w.mask_bits.assign(static_cast<size_t>(nblocks_ / 2 + 1), {nullptr, nullptr});
      for (int b = 0; b < nblocks_; b += 2)
        for (int sb = 0; sb < 2; ++sb)
          w.mask_bits[static_cast<size_t>(b / 2)][static_cast<size_t>(sb)] = static_cast<uint32_t*>(arena_.alloc(mbytes));
    }
    w.y = arena_.alloc(static_cast<size_t>(T * h) * es);
    // row statistics of both sub-batches (the parameter pass runs once over 2 T_sub rows)
    w.ln_ws = arena_.alloc(layernorm_bwd_workspace(2 * Ts, static_cast<int>(h)));
    // [2 sub-batches][partial rows][3][h] column partials of the persistent LayerNorm backward
    if (lnp_bwd_)
      w.lnp_part = static_cast<float*>(arena_.alloc(
          static_cast<size_t>(2 * lnp_partial_rows_max(Ts, static_cast<int>(h)) * 3 * h) * sizeof(float)));
    w.col_ws = arena_.alloc(colws);
    w.col_ws2 = arena_.alloc(colws);
    // [2 T_sub / 32, ncol_ffn] partials of the fused FFN column-bias gradient (own buffer: the
    // attention blocks' side-stream column sums may run between the two sub-batches' FC2 dgrads)
    w.col_part = colsum_ ? static_cast<float*>(arena_.alloc(static_cast<size_t>(2 * tffn / 32) * sizeof(float)))
                         : nullptr;
    w.loss = static_cast<double*>(arena_.alloc(sizeof(double)));
    w.loss_ws = static_cast<double*>(arena_.alloc(loss_workspace()));
  }
  check_cuda(cudaDeviceSynchronize(), "stack allocation");
  // residual-stream buffers of blocks > 0 are placed when a plan is bound
  x_stored_.assign(static_cast<size_t>(nblocks_), false);
  if (nblocks_ > 0) x_stored_[0] = true;
}

void Stack::bind_storage(const std::vector<bool>& stored) {
  if (static_cast<int>(stored.size()) != nblocks_) throw ConfigError("bind_storage: one flag per block");
  const int64_t T = static_cast<int64_t>(cfg_.b) * cfg_.s, h = cfg_.h;
  const size_t bytes = static_cast<size_t>(T * h) * esize();
  // buffers the previous plan needed and this one does not are freed, so the
  // reported device bytes are those of the bound plan (a rebound stack measures
  // the same peak_memory as a fresh one)
  check_cuda(cudaDeviceSynchronize(), "bind_storage sync");
  bool any_scratch = false;
  for (int b = 1; b < nblocks_; ++b) any_scratch = any_scratch || !stored[static_cast<size_t>(b)];
  for (Worker& w : workers_) {
    for (int b = 1; b < nblocks_; ++b) {
      void*& own = w.x_own[static_cast<size_t>(b)];
      if (stored[static_cast<size_t>(b)]) {
        if (!own) own = arena_.alloc(bytes);
        w.xbase[static_cast<size_t>(b)] = own;
      } else {
        if (own) {
          arena_.release(own);
          own = nullptr;
        }
        if (!w.x_scratch) w.x_scratch = arena_.alloc(bytes);
        w.xbase[static_cast<size_t>(b)] = w.x_scratch;
      }
    }
    if (!any_scratch && w.x_scratch) {
      arena_.release(w.x_scratch);
      w.x_scratch = nullptr;
    }
  }
  x_stored_ = stored;
  if (nblocks_ > 0) x_stored_[0] = true;
}

Workspace Stack::ws_for(Worker& w, int block, int sb) {
  size_t slot = cfg_.recompute ? static_cast<size_t>(block % 2) : static_cast<size_t>(block);
  slot = std::min(slot, w.ws.size() - 1);
  Workspace ws = w.ws[slot][static_cast<size_t>(sb)];
  ws.ln = w.ln_full[slot] ? lp(w.ln_full[slot], block, sb, cfg_.h) : nullptr;
  ws.act = lp(w.act_full[slot], block, sb, std::max<int64_t>(nrow(block), 1));
  return ws;
}

bool Stack::touch(const Worker& w, int block, int p, int computed_at) {
  const size_t wi = static_cast<size_t>(&w - workers_.data());
  bool& t = touched_[wi][static_cast<size_t>(block)][static_cast<size_t>(p)];
  const bool was = t;
  t = true;
  computed_at_[static_cast<size_t>(block)][static_cast<size_t>(p)] = computed_at ? computed_at : degree(block);
  return was;
}

void Stack::begin_step() {
  for (auto& per_worker : touched_)
    for (auto& a : per_worker) a.fill(false);
  for (auto& per_worker : bwd_seen_) std::fill(per_worker.begin(), per_worker.end(), false);
  std::fill(loss_touched_.begin(), loss_touched_.end(), false);
  for (auto& a : computed_at_) a.fill(0);
}

// GEMM timing events: plain records when issued eagerly; external event-record
// nodes when the step is being captured (graph_kernel_stats), so a replay of the
// captured step re-records them.
cudaError_t Stack::record_timing(cudaEvent_t e) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  const cudaError_t q = cudaStreamIsCapturing(ctx_.compute, &cs);
  if (q != cudaSuccess) return q;
  return cs == cudaStreamCaptureStatusActive ? cudaEventRecordWithFlags(e, ctx_.compute, cudaEventRecordExternal)
                                             : cudaEventRecord(e, ctx_.compute);
}

void Stack::gemm(const oases_gemm_desc& d0) {
  oases_gemm_desc d = d0;
  d.dtype = dtype();
  d.max_ctas = ctx_.gemm_max_ctas;
  const bool timed = timing_ && d.causal == OASES_CAUSAL_NONE && d.batch == 1;
  if (timed) {
    while (tev_.size() < 2 * (timed_ + 1)) {
      cudaEvent_t e;
      check_cuda(cudaEventCreate(&e), "event");
      tev_.push_back(e);
    }
    if (tflops_.size() < timed_ + 1) tflops_.resize(timed_ + 1);
    tflops_[timed_] = 2.0 * static_cast<double>(d.M) * static_cast<double>(d.N) * static_cast<double>(d.K);
    check_cuda(record_timing(tev_[2 * timed_]), "record");
  }
  GemmStatus st = d.dtype == OASES_BF16 ? gemm_tc(d, ctx_.compute) : gemm_simt(d, ctx_.compute);
  if (!st.ok) {
    if (st.cuda) throw CudaError(st.err);
    throw ConfigError(st.err);
  }
  if (timed) {
    check_cuda(record_timing(tev_[2 * timed_ + 1]), "record");
    ++timed_;
  }
  ++launches_;
}

// Two independent GEMMs (a backward dgrad + wgrad pair) in one launch when the
// tcgen05 CTA-pair kernel takes both (kernels/gemm_tc.cu, TcGroup).
void Stack::gemm2(const oases_gemm_desc& d0, const oases_gemm_desc& d1) {
  if (dtype() != OASES_BF16) {
    gemm(d0);
    gemm(d1);
    return;
  }
  oases_gemm_desc d[2] = {d0, d1};
  for (auto& x : d) {
    x.dtype = dtype();
    x.max_ctas = ctx_.gemm_max_ctas;
  }
  const bool timed = timing_;
  if (timed) {
    while (tev_.size() < 2 * (timed_ + 1)) {
      cudaEvent_t e;
      check_cuda(cudaEventCreate(&e), "event");
      tev_.push_back(e);
    }
    if (tflops_.size() < timed_ + 1) tflops_.resize(timed_ + 1);
    tflops_[timed_] = 0.0;
    for (const auto& x : d)
      tflops_[timed_] += 2.0 * static_cast<double>(x.M) * static_cast<double>(x.N) * static_cast<double>(x.K);
    check_cuda(record_timing(tev_[2 * timed_]), "record");
  }
  GemmStatus st = gemm_tc_group(d, 2, ctx_.compute);
  if (!st.ok) {
    if (st.cuda) throw CudaError(st.err);
    throw ConfigError(st.err);
  }
  if (timed) {
    check_cuda(record_timing(tev_[2 * timed_ + 1]), "record");
    ++timed_;
  }
  launches_ += 1;
}

void Stack::fork_side() {
  check_cuda(cudaEventRecord(ctx_.fork_ev, ctx_.compute), "fork record");
  check_cuda(cudaStreamWaitEvent(ctx_.side, ctx_.fork_ev, 0), "fork wait");
  side_forked_ = true;
}

void Stack::join_side() {
  if (!side_forked_) return;
  check_cuda(cudaEventRecord(ctx_.join_ev, ctx_.side), "join record");
  check_cuda(cudaStreamWaitEvent(ctx_.compute, ctx_.join_ev, 0), "join wait");
  side_forked_ = false;
}

// x_b = x_{b-1} + dropout(ar + bias_row_{b-1}), then LN_b(x_b) -> ln: one
// fused HBM pass where the row-group kernel covers the shape (its LN is
// bit-identical to ln_fwd of the stored x_b), else the two kernels.
void Stack::bdr_then_ln(Worker& w, int block, int sb, const void* ar, void* x, void* ln, bool store_bits) {
  const int64_t Ts = ts(block), h = cfg_.h;
  const BlockParams& prev = w.params[static_cast<size_t>(block - 1)];
  const BlockParams& bp = w.params[static_cast<size_t>(block)];
  const void* bias = cfg_.bias ? prev.p[OASES_P_B_ROW] : nullptr;
  const void* res = cfg_.residual ? gp(w.xbase[static_cast<size_t>(block - 1)], w, block, sb, h) : nullptr;
  if (cfg_.ln && fuse_bdr_ln_ && bdr_layernorm_supported(Ts, static_cast<int>(h))) {
    uint16_t* bits = store_bits && hbits_ ? w.hbits[static_cast<size_t>(block - 1)][static_cast<size_t>(sb)] : nullptr;
    check_cuda(bias_dropout_residual_layernorm_fwd(dtype(), ar, bias, res, x, bp.p[OASES_P_LN_GAMMA],
                                                   bp.p[OASES_P_LN_BETA], ln, Ts, static_cast<int>(h), cfg_.eps,
                                                   cfg_.p_hidden, cfg_.seed, drop_offset(block - 1, sb, 0),
                                                   ctx_.compute, bits, ctx_.gemm_max_ctas),
               "bdr + layernorm");
    ++launches_;
    return;
  }
  check_cuda(bias_dropout_residual_fwd(dtype(), ar, bias, res, x, Ts, static_cast<int>(h), cfg_.p_hidden, cfg_.seed,
                                       drop_offset(block - 1, sb, 0), ctx_.compute),
             "bdr_fwd");
  ++launches_;
  if (cfg_.ln) ln_fwd(x, bp.p[OASES_P_LN_GAMMA], bp.p[OASES_P_LN_BETA], ln, Ts);
}

void Stack::ln_fwd(const void* x, const void* g, const void* b, void* y, int64_t rows) {
  check_cuda(layernorm_fwd(dtype(), x, g, b, y, rows, cfg_.h, cfg_.eps, ctx_.compute, ctx_.gemm_max_ctas),
             "layernorm_fwd");
  ++launches_;
}

// ------------------------------------------------------------------ params / io
// Host views use the oracle layout [in, out] (f64); the device keeps [out, in].

void Stack::set_param(int worker, int block, int p, const double* host) {
  if (worker < 0 || worker >= num_workers() || block < 0 || block >= nblocks_ || p < 0 || p >= OASES_P_COUNT)
    throw ConfigError("set_param: index out of range");
  BlockParams& bp = workers_[static_cast<size_t>(worker)].params[static_cast<size_t>(block)];
  const int64_t n = bp.numel[p];
  if (!n) throw ConfigError("set_param: block has no such parameter");
  if (dtype() == OASES_F64) {  // value-level toy mode: the host values as they are
    std::vector<double> d(static_cast<size_t>(n));
    if (p == OASES_P_W_COL || p == OASES_P_W_ROW) {
      const int64_t out = bp.rows[p], in = n / out;
      for (int64_t o = 0; o < out; ++o)
        for (int64_t i = 0; i < in; ++i) d[static_cast<size_t>(o * in + i)] = host[i * out + o];
    } else {
      for (int64_t i = 0; i < n; ++i) d[static_cast<size_t>(i)] = host[i];
    }
    check_cuda(cudaMemcpy(bp.p[p], d.data(), static_cast<size_t>(n) * 8, cudaMemcpyHostToDevice), "H2D");
    return;
  }
  std::vector<float> f(static_cast<size_t>(n));
  if (p == OASES_P_W_COL || p == OASES_P_W_ROW) {
    const int64_t out = bp.rows[p], in = n / out;  // device [out, in]; host [in, out]
    for (int64_t o = 0; o < out; ++o)
      for (int64_t i = 0; i < in; ++i) f[static_cast<size_t>(o * in + i)] = static_cast<float>(host[i * out + o]);
  } else {
    for (int64_t i = 0; i < n; ++i) f[static_cast<size_t>(i)] = static_cast<float>(host[i]);
  }
  void* staging = nullptr;
  check_cuda(cudaMalloc(&staging, static_cast<size_t>(n) * sizeof(float)), "staging");
  check_cuda(cudaMemcpy(staging, f.data(), static_cast<size_t>(n) * sizeof(float), cudaMemcpyHostToDevice), "H2D");
  check_cuda(convert(OASES_F32, staging, dtype(), bp.p[p], n, nullptr), "convert");
  check_cuda(cudaDeviceSynchronize(), "set_param");
  cudaFree(staging);
}

void Stack::get_grad(int worker, int block, int p, double* host) {
  if (worker < 0 || worker >= num_workers() || block < 0 || block >= nblocks_ || p < 0 || p >= OASES_P_COUNT)
    throw ConfigError("get_grad: index out of range");
  BlockParams& bp = workers_[static_cast<size_t>(worker)].params[static_cast<size_t>(block)];
  const int64_t n = bp.numel[p];
  if (!n) throw ConfigError("get_grad: block has no such parameter");
  std::vector<double> f(static_cast<size_t>(n));
  check_cuda(cudaDeviceSynchronize(), "get_grad sync");
  if (gdtype() == OASES_F64) {
    check_cuda(cudaMemcpy(f.data(), bp.g[p], static_cast<size_t>(n) * 8, cudaMemcpyDeviceToHost), "D2H");
  } else {
    std::vector<float> f32(static_cast<size_t>(n));
    check_cuda(cudaMemcpy(f32.data(), bp.g[p], static_cast<size_t>(n) * sizeof(float), cudaMemcpyDeviceToHost), "D2H");
    for (int64_t i = 0; i < n; ++i) f[static_cast<size_t>(i)] = f32[static_cast<size_t>(i)];
  }
  if (p == OASES_P_W_COL || p == OASES_P_W_ROW) {
    const int64_t out = bp.rows[p], in = n / out;
    for (int64_t o = 0; o < out; ++o)
      for (int64_t i = 0; i < in; ++i) host[i * out + o] = f[static_cast<size_t>(o * in + i)];
  } else {
    for (int64_t i = 0; i < n; ++i) host[i] = f[static_cast<size_t>(i)];
  }
}

void Stack::init_random(uint64_t seed) {
  // numerics.cpp:146-152 conventions: input U(-1,1), W_col U(+-1/sqrt(h)),
  // W_row U(+-1/sqrt(fan_in)); LN gamma 1, beta 0, biases 0.
  const int64_t T = 2 * tokens_sub();
  for (Worker& w : workers_) {
    check_cuda(fill_uniform(dtype(), w.input, T * cfg_.h, 1.f, seed, 0x1000000, ctx_.compute), "init input");
    for (int b = 0; b < nblocks_; ++b) {
      BlockParams& bp = w.params[static_cast<size_t>(b)];
      // the shard is keyed by the rank in the block's group: data-parallel groups of
      // a lower-degree block hold identical replicas
      const uint64_t off = 0x2000000 + (static_cast<uint64_t>(b) * 64 + static_cast<uint64_t>(rig(w, b))) * 8;
      check_cuda(fill_uniform(dtype(), bp.p[OASES_P_W_COL], bp.numel[OASES_P_W_COL],
                              1.f / std::sqrt(static_cast<float>(cfg_.h)), seed, off, ctx_.compute),
                 "init w_col");
      const float fan = static_cast<float>(is_attention(b) ? cfg_.h : cfg_.f);
      check_cuda(fill_uniform(dtype(), bp.p[OASES_P_W_ROW], bp.numel[OASES_P_W_ROW], 1.f / std::sqrt(fan), seed,
                              off + 1, ctx_.compute),
                 "init w_row");
    }
  }
  // every worker sees the same input (replicated across the TMP group)
  for (size_t w = 1; w < workers_.size(); ++w)
    check_cuda(cudaMemcpyAsync(workers_[w].input, workers_[0].input, static_cast<size_t>(T * cfg_.h) * esize(),
                               cudaMemcpyDeviceToDevice, ctx_.compute),
               "replicate input");
  check_cuda(cudaStreamSynchronize(ctx_.compute), "init_random");
}

void Stack::set_input(const void* host, int host_dtype, cudaStream_t st) {
  const int64_t n = 2 * tokens_sub() * cfg_.h;
  const int my = dtype();
  const void* src = host;
  std::vector<float> f32;
  std::vector<uint16_t> b16;
  int src_dtype = host_dtype;
  if (host_dtype == 2 && my != OASES_F64) {  // f64 -> activation dtype on the host
    const double* d = static_cast<const double*>(host);
    if (my == OASES_F32) {
      f32.resize(static_cast<size_t>(n));
      for (int64_t i = 0; i < n; ++i) f32[static_cast<size_t>(i)] = static_cast<float>(d[i]);
      src = f32.data();
    } else {
      b16.resize(static_cast<size_t>(n));
      for (int64_t i = 0; i < n; ++i) {
        const float v = static_cast<float>(d[i]);
        uint32_t u;
        std::memcpy(&u, &v, 4);
        u += 0x7FFFu + ((u >> 16) & 1u);  // round to nearest even
        b16[static_cast<size_t>(i)] = static_cast<uint16_t>(u >> 16);
      }
      src = b16.data();
    }
    src_dtype = my;
  }
  if (src_dtype != my) throw ConfigError("set_input: host dtype must match the activation dtype (or be f64)");
  for (Worker& w : workers_)
    check_cuda(cudaMemcpyAsync(w.input, src, static_cast<size_t>(n) * esize(), cudaMemcpyHostToDevice, st), "H2D input");
  if (host_dtype == 2) check_cuda(cudaStreamSynchronize(st), "set_input");
}

namespace {
void download(const void* dev, int dtype, int64_t n, double* host) {
  check_cuda(cudaDeviceSynchronize(), "download sync");
  if (dtype == OASES_F64) {
    check_cuda(cudaMemcpy(host, dev, static_cast<size_t>(n) * 8, cudaMemcpyDeviceToHost), "D2H");
  } else if (dtype == OASES_F32) {
    std::vector<float> f(static_cast<size_t>(n));
    check_cuda(cudaMemcpy(f.data(), dev, static_cast<size_t>(n) * 4, cudaMemcpyDeviceToHost), "D2H");
    for (int64_t i = 0; i < n; ++i) host[i] = f[static_cast<size_t>(i)];
  } else {
    std::vector<uint16_t> b(static_cast<size_t>(n));
    check_cuda(cudaMemcpy(b.data(), dev, static_cast<size_t>(n) * 2, cudaMemcpyDeviceToHost), "D2H");
    for (int64_t i = 0; i < n; ++i) {
      const uint32_t u = static_cast<uint32_t>(b[static_cast<size_t>(i)]) << 16;
      float v;
      std::memcpy(&v, &u, 4);
      host[i] = v;
    }
  }
}
}  // namespace

void Stack::get_input_grad(double* host) {
  // dX rows of each data-parallel group of block 0 (its rank 0 holds them)
  const int64_t h = cfg_.h;
  if (nblocks_ == 0 || degree(0) == world() || workers_.size() == 1) {
    download(workers_[0].grad, dtype(), 2 * tokens_sub() * h, host);
    return;
  }
  const int64_t rows = 2 * ts(0);
  for (const Worker& w : workers_) {
    if (rig(w, 0) != 0) continue;
    const int64_t r0 = row0(w, 0);
    download(static_cast<const char*>(w.grad) + static_cast<size_t>(r0 * h) * esize(), dtype(), rows * h,
             host + r0 * h);
  }
}

void Stack::get_activation(int worker, int block, int sb, double* host) {
  if (block >= 0 && block < nblocks_ && !x_stored_[static_cast<size_t>(block)])
    throw ConfigError("activation: x_" + std::to_string(block) +
                      " is not kept by the bound plan (rebuilt in recompute; bind an Oases plan to read it)");
  if (worker < 0 || worker >= num_workers() || block < 0 || block > nblocks_ || sb < 0 || sb > 1)
    throw ConfigError("get_activation: index out of range");
  Worker& w = workers_[static_cast<size_t>(worker)];
  // rows of sub-batch sb of the block's group of this worker (T_sub of a uniform stack)
  if (block == nblocks_) {
    const int last = nblocks_ - 1;  // x_B, the stack's output
    download(gp(w.y, w, last, sb, cfg_.h), dtype(), ts(last) * cfg_.h, host);
    return;
  }
  download(gp(w.xbase[static_cast<size_t>(block)], w, block, sb, cfg_.h), dtype(), ts(block) * cfg_.h, host);
}

double Stack::read_loss() {
  // in-process: one value per data-parallel group of the last block (its rank 0),
  // summed; one rank per process: this rank's group's value
  double l = 0.0;
  for (const Worker& w : workers_) {
    if (workers_.size() > 1 && nblocks_ > 0 && rig(w, nblocks_ - 1) != 0) continue;
    double v = 0.0;
    check_cuda(cudaMemcpy(&v, w.loss, sizeof(double), cudaMemcpyDeviceToHost), "loss D2H");
    l += v;
    if (nblocks_ == 0) break;
  }
  return l;
}

// ------------------------------------------------------------------ attention
// Attention-dropout keys of a sub-batch tensor: the key
// sub-batch is the half of the micro-batch holding its samples and sample
// n of the tensor is sample n0 + n there, so the masks do not depend on the
// block's degree (data-parallel groups of a mixed-degree stack hold slices).
namespace {
struct AttnKey {
  int sb_key;
  int n0;
};
}  // namespace
static AttnKey attn_key(int64_t first_sample, int64_t half_batch) {
  return {static_cast<int>(first_sample / half_batch), static_cast<int>(first_sample % half_batch)};
}

oases_attn_desc Stack::attn_desc(Worker& w, int block, int sb, const Workspace& ws) {
  oases_attn_desc a{};
  const int64_t nc = ncol(block), nr = nrow(block);
  a.dtype = dtype();
  a.samples = static_cast<int>(bsub(block));
  a.heads_local = hl(block);
  a.heads_total = static_cast<int>(cfg_.heads);
  a.head_offset = rig(w, block) * hl(block);
  a.head_dim = dh_;
  a.seq = static_cast<int>(cfg_.s);
  a.max_ctas = ctx_.gemm_max_ctas;
  a.qkv = ws.col;
  a.ld_qkv = nc;
  a.out = ws.act;
  a.ld_out = nr;
  a.lse = ws.lse;
  a.dout = w.du;
  a.ld_dout = nr;
  a.dqkv = lp(w.dcol, block, sb, nc);
  a.ld_dqkv = nc;
  a.ds = w.dp;
  a.workspace = w.attn_ws;
  // keep-bit cache unless OASES_ATTN_MASK_CACHE=0 (A/B runs: Philox in every pass)
  static const bool cache = [] {
    const char* e = std::getenv("OASES_ATTN_MASK_CACHE");
    return !(e && e[0] == '0');
  }();
  if (cache && !w.mask_bits.empty())
    a.mask_bits = w.mask_bits[static_cast<size_t>(block / 2)][static_cast<size_t>(sb)];
  a.scale = 1.f / std::sqrt(static_cast<float>(dh_));
  a.dropout_p = cfg_.p_attn;
  a.seed = cfg_.seed;
  const AttnKey k = attn_key(row0(w, block) / cfg_.s + sb * bsub(block), cfg_.b / 2);
  a.offset = drop_offset(block, k.sb_key, 1);
  a.sample_offset = k.n0;
  return a;
}

void Stack::attention_fwd(Worker& w, int block, int sb, const Workspace& ws, int mask_mode) {
  const int hlb = hl(block);
  const int64_t s = cfg_.s, Ts = ts(block), bh = bsub(block), Z = bh * hlb, nc = ncol(block), nr = nrow(block);
  const int64_t hd = static_cast<int64_t>(hlb) * dh_;
  const AttnKey key = attn_key(row0(w, block) / cfg_.s + sb * bh, cfg_.b / 2);
  // unfused softmax: the sample offset of the dropout keys folds into the head offset
  const int hoff = key.n0 * cfg_.heads + rig(w, block) * hlb;
  const char* qkv = static_cast<const char*>(ws.col);
  const size_t es = esize();
  if (fused_attn_) {
    oases_attn_desc a = attn_desc(w, block, sb, ws);
    a.mask_mode = mask_mode;
    // OASES_ATTN_MASK_PASS=1: the forward's keep bits from the separate mask pass and
    // every fused-attention pass reads cached bits. Off by default: the pass costs
    // ~18 us per C2 sub-batch (Philox is issue-bound wherever it runs), as much as
    // generating the bits inside the split-warp forward saves (A/B on one B200:
    // 76.11 / 76.12 ms with the pass vs 75.81 / 76.14 without). The recompute and
    // backward read the bits the forward stored either way.
    static const bool mask_pass = [] {
      const char* e = std::getenv("OASES_ATTN_MASK_PASS");
      return e && e[0] == '1';
    }();
    if (mask_mode == 1 && mask_pass && a.mask_bits && cfg_.p_attn > 0.f) {
      const GemmStatus ms = oases::attention_masks(a, ctx_.compute);
      if (!ms.ok) {
        if (ms.cuda) throw CudaError(ms.err);
        throw ConfigError(ms.err);
      }
      ++launches_;
      a.mask_mode = 2;
    }
    const GemmStatus st = oases::attention_fwd(a, ctx_.compute);
    if (!st.ok) {
      if (st.cuda) throw CudaError(st.err);
      throw ConfigError(st.err);
    }
    ++launches_;
    return;
  }
  oases_gemm_desc d{};
  // S = Q K^T per (sample, head); tiles above the diagonal are skipped.
  d = oases_gemm_desc{};
  d.c_dtype = dtype();
  d.M = s; d.N = s; d.K = dh_;
  d.batch = Z; d.batch_inner = hlb;
  d.a = operand(qkv, Ts, nc, nc, false, s, 0, 0, dh_);
  d.b = operand(qkv + hd * es, Ts, nc - hd, nc, false, s, 0, 0, dh_);
  d.c = ws.p; d.ldc = s; d.c_row_off[0] = hlb * s; d.c_row_off[1] = s;
  d.alpha = 1.f; d.causal = OASES_CAUSAL_SKIP_UPPER;
  gemm(d);
  check_cuda(softmax_fwd(dtype(), ws.p, ws.p, cfg_.p_attn > 0.f ? ws.pd : nullptr, Z, static_cast<int>(s),
                         1.f / std::sqrt(static_cast<float>(dh_)), cfg_.p_attn, cfg_.seed, drop_offset(block, key.sb_key, 1),
                         hlb, cfg_.heads, hoff, ctx_.compute),
             "softmax_fwd");
  ++launches_;
  // ctx = P_drop V  (K limited to the causal prefix of each 128-row tile)
  d = oases_gemm_desc{};
  d.c_dtype = dtype();
  d.M = s; d.N = dh_; d.K = s;
  d.batch = Z; d.batch_inner = hlb;
  d.a = operand(ws.pd, Z * s, s, s, false, hlb * s, s);
  d.b = operand(qkv + 2 * hd * es, Ts, nc - 2 * hd, nc, true, s, 0, 0, dh_);
  d.c = ws.act; d.ldc = nr; d.c_row_off[0] = s; d.c_col_off[1] = dh_;
  d.alpha = 1.f; d.causal = OASES_CAUSAL_K_UPTO_M;
  gemm(d);
}

void Stack::attention_bwd(Worker& w, int block, int sb, const Workspace& ws) {
  const int hlb = hl(block);
  const int64_t s = cfg_.s, Ts = ts(block), bh = bsub(block), Z = bh * hlb, nc = ncol(block), nr = nrow(block);
  const int64_t hd = static_cast<int64_t>(hlb) * dh_;
  const AttnKey key = attn_key(row0(w, block) / cfg_.s + sb * bh, cfg_.b / 2);
  const int hoff = key.n0 * cfg_.heads + rig(w, block) * hlb;
  const size_t es = esize();
  const char* qkv = static_cast<const char*>(ws.col);
  char* dqkv = static_cast<char*>(lp(w.dcol, block, sb, nc));
  if (fused_attn_) {
    oases_attn_desc a = attn_desc(w, block, sb, ws);
    a.mask_mode = 2;                // the forward pass stored the keep bits
    a.dsum_ready = rowdot_ ? 1 : 0;  // the proj dgrad's ROWDOT epilogue wrote D
    const GemmStatus st = oases::attention_bwd(a, ctx_.compute);
    if (!st.ok) {
      if (st.cuda) throw CudaError(st.err);
      throw ConfigError(st.err);
    }
    launches_ += 3;  // rowsum(dO o O), dK/dV kernel, dQ GEMM
    return;
  }
  oases_gemm_desc d{};
  // dP_drop = dctx V^T
  d.c_dtype = dtype();
  d.M = s; d.N = s; d.K = dh_;
  d.batch = Z; d.batch_inner = hlb;
  d.a = operand(w.du, Ts, nr, nr, false, s, 0, 0, dh_);
  d.b = operand(qkv + 2 * hd * es, Ts, nc - 2 * hd, nc, false, s, 0, 0, dh_);
  d.c = w.dp; d.ldc = s; d.c_row_off[0] = hlb * s; d.c_row_off[1] = s;
  d.alpha = 1.f; d.causal = OASES_CAUSAL_SKIP_UPPER;
  gemm(d);
  // dV = P_drop^T dctx
  d = oases_gemm_desc{};
  d.c_dtype = dtype();
  d.M = s; d.N = dh_; d.K = s;
  d.batch = Z; d.batch_inner = hlb;
  d.a = operand(ws.pd, Z * s, s, s, true, hlb * s, s);
  d.b = operand(w.du, Ts, nr, nr, true, s, 0, 0, dh_);
  d.c = dqkv + 2 * hd * es; d.ldc = nc; d.c_row_off[0] = s; d.c_col_off[1] = dh_;
  d.alpha = 1.f; d.causal = OASES_CAUSAL_K_FROM_M;
  gemm(d);
  // dS (in place over dP)
  check_cuda(softmax_bwd(dtype(), ws.p, w.dp, w.dp, Z, static_cast<int>(s), 1.f / std::sqrt(static_cast<float>(dh_)),
                         cfg_.p_attn, cfg_.seed, drop_offset(block, key.sb_key, 1), hlb, cfg_.heads, hoff,
                         ctx_.compute),
             "softmax_bwd");
  ++launches_;
  // dQ = dS K
  d = oases_gemm_desc{};
  d.c_dtype = dtype();
  d.M = s; d.N = dh_; d.K = s;
  d.batch = Z; d.batch_inner = hlb;
  d.a = operand(w.dp, Z * s, s, s, false, hlb * s, s);
  d.b = operand(qkv + hd * es, Ts, nc - hd, nc, true, s, 0, 0, dh_);
  d.c = dqkv; d.ldc = nc; d.c_row_off[0] = s; d.c_col_off[1] = dh_;
  d.alpha = 1.f; d.causal = OASES_CAUSAL_K_UPTO_M;
  gemm(d);
  // dK = dS^T Q
  d = oases_gemm_desc{};
  d.c_dtype = dtype();
  d.M = s; d.N = dh_; d.K = s;
  d.batch = Z; d.batch_inner = hlb;
  d.a = operand(w.dp, Z * s, s, s, true, hlb * s, s);
  d.b = operand(qkv, Ts, nc, nc, true, s, 0, 0, dh_);
  d.c = dqkv + hd * es; d.ldc = nc; d.c_row_off[0] = s; d.c_col_off[1] = dh_;
  d.alpha = 1.f; d.causal = OASES_CAUSAL_K_FROM_M;
  gemm(d);
}

// ------------------------------------------------------------------ plan ops
void Stack::forward(int wi, int block, int sb, bool with_bdr, bool with_row) {
  Worker& w = workers_[static_cast<size_t>(wi)];
  const int64_t Ts = ts(block), h = cfg_.h;
  void* x = gp(w.xbase[static_cast<size_t>(block)], w, block, sb, h);
  Workspace ws = ws_for(w, block, sb);
  const BlockParams& bp = w.params[static_cast<size_t>(block)];
  const bool att = is_attention(block);
  const int64_t ncol = this->ncol(block), nrow = this->nrow(block);
  const void* ln = x;
  if (block > 0 && with_bdr) {
    bdr_then_ln(w, block, sb, gp(w.fwd_ar[(block - 1) % 2], w, block, sb, h), x, ws.ln, true);
  } else if (cfg_.ln) {
    ln_fwd(x, bp.p[OASES_P_LN_GAMMA], bp.p[OASES_P_LN_BETA], ws.ln, Ts);
  }
  if (cfg_.ln) ln = ws.ln;
  oases_gemm_desc d{};
  d.c_dtype = dtype();
  d.M = Ts; d.N = ncol; d.K = h;
  d.batch = 1; d.batch_inner = 1;
  d.a = operand(ln, Ts, h, h, false);
  d.b = operand(bp.p[OASES_P_W_COL], ncol, h, h, false);
  d.c = ws.col; d.ldc = ncol;
  d.alpha = 1.f;
  d.bias = cfg_.bias ? bp.p[OASES_P_B_COL] : nullptr;
  if (att) {
    d.epilogue = OASES_EPI_BIAS;
    gemm(d);
    attention_fwd(w, block, sb, ws, 1);  // generate + store the keep bits
  } else {
    if (cfg_.recompute) {
      // the recompute pass regenerates gelu'(pre) for the backward; here only
      // the activation feeding FC2 is live
      d.epilogue = OASES_EPI_BIAS_GELU;
      d.c = ws.act;
      d.c2 = nullptr;
    } else {
      d.epilogue = OASES_EPI_BIAS_GELU_GRAD;  // ws.col = gelu'(pre) for the dgrad, ws.act = gelu(pre)
      d.c2 = ws.act;
    }
    gemm(d);
  }
  if (with_row) {
    d = oases_gemm_desc{};
    d.c_dtype = dtype();
    d.M = Ts; d.N = h; d.K = nrow;
    d.batch = 1; d.batch_inner = 1;
    d.a = operand(ws.act, Ts, nrow, nrow, false);
    d.b = operand(bp.p[OASES_P_W_ROW], h, nrow, nrow, false);
    d.c = gp(w.fwd_ar[block % 2], w, block, sb, h);
    d.ldc = h;
    d.alpha = 1.f;
    gemm(d);
  }
}

void Stack::recompute(int wi, int block, int sb, bool rebuild_x, bool with_row) {
  Worker& w = workers_[static_cast<size_t>(wi)];
  const int64_t Ts = ts(block), h = cfg_.h;
  void* x = gp(w.xbase[static_cast<size_t>(block)], w, block, sb, h);
  // Same kernels as the forward from the stored x_b (or x_b rebuilt from the
  // replayed AllReduce); the row GEMM only when this variant replays the
  // block's AllReduce.
  Workspace ws = ws_for(w, block, sb);
  const BlockParams& bp = w.params[static_cast<size_t>(block)];
  const bool att = is_attention(block);
  const int64_t ncol = this->ncol(block), nrow = this->nrow(block);
  const void* ln = x;
  if (rebuild_x && block > 0) {
    bdr_then_ln(w, block, sb, gp(w.rec_ar[(block - 1) % 2], w, block, sb, h), x, ws.ln, false);
  } else if (cfg_.ln) {
    ln_fwd(x, bp.p[OASES_P_LN_GAMMA], bp.p[OASES_P_LN_BETA], ws.ln, Ts);
  }
  if (cfg_.ln) ln = ws.ln;
  oases_gemm_desc d{};
  d.c_dtype = dtype();
  d.M = Ts; d.N = ncol; d.K = h;
  d.batch = 1; d.batch_inner = 1;
  d.a = operand(ln, Ts, h, h, false);
  d.b = operand(bp.p[OASES_P_W_COL], ncol, h, h, false);
  d.c = ws.col; d.ldc = ncol;
  d.alpha = 1.f;
  d.bias = cfg_.bias ? bp.p[OASES_P_B_COL] : nullptr;
  if (att) {
    d.epilogue = OASES_EPI_BIAS;
    gemm(d);
    attention_fwd(w, block, sb, ws, 2);  // the forward pass stored the keep bits
  } else {
    // ws.col = gelu'(pre) (the factor the FC2 dgrad epilogue multiplies by), ws.act = gelu(pre)
    d.epilogue = OASES_EPI_BIAS_GELU_GRAD;
    d.c2 = ws.act;
    gemm(d);
  }
  if (with_row) {
    d = oases_gemm_desc{};
    d.c_dtype = dtype();
    d.M = Ts; d.N = h; d.K = nrow;
    d.batch = 1; d.batch_inner = 1;
    d.a = operand(ws.act, Ts, nrow, nrow, false);
    d.b = operand(bp.p[OASES_P_W_ROW], h, nrow, nrow, false);
    d.c = gp(w.rec_ar[block % 2], w, block, sb, h);
    d.ldc = h;
    d.alpha = 1.f;
    gemm(d);
  }
}

void Stack::backward(int wi, int block, int sb, bool g_ready) {
  Worker& w = workers_[static_cast<size_t>(wi)];
  const int64_t Ts = ts(block), h = cfg_.h;
  const int hi = static_cast<int>(h);
  void* g = gp(w.grad, w, block, sb, h);
  void* gar_sb = lp(w.gar, block, sb, h);
  // The weight gradients of a block are computed once per step, by its second
  // backward call (the other sub-batch's), over both sub-batches at once:
  // K = 2 T_sub, no f32 read-modify-write of dW between the sub-batches.
  const bool wgrad_now = bwd_seen_[static_cast<size_t>(wi)][static_cast<size_t>(block)];
  bwd_seen_[static_cast<size_t>(wi)][static_cast<size_t>(block)] = true;
  // 1. gradient arriving at x_{b+1}; with LayerNorm the same pass also writes
  //    g_ar = dropout'(g) (step 2) when the row-group kernel covers the width
  bool gar_done = false, row_bias_done = false;
  if (g_ready) {
    // reshard_bwd already gathered g + LN_{b+1}'(dln_{b+1}) over this block's slice
  } else if (block == nblocks_ - 1) {
    const BlockParams& bp = w.params[static_cast<size_t>(block)];
    void* y = gp(w.y, w, block, sb, h);
    check_cuda(bias_dropout_residual_fwd(dtype(), gp(w.fwd_ar[block % 2], w, block, sb, h),
                                         cfg_.bias ? bp.p[OASES_P_B_ROW] : nullptr,
                                         cfg_.residual ? gp(w.xbase[static_cast<size_t>(block)], w, block, sb, h) : nullptr,
                                         y, Ts, hi,
                                         cfg_.p_hidden, cfg_.seed, drop_offset(block, sb, 0), ctx_.compute),
               "bdr_fwd (loss head)");
    const bool acc = loss_touched_[static_cast<size_t>(wi)];
    loss_touched_[static_cast<size_t>(wi)] = true;
    check_cuda(gelu_sq_loss(dtype(), y, g, w.loss, acc ? 1 : 0, w.loss_ws, Ts * h, ctx_.compute), "loss head");
    launches_ += 3;
  } else {
    const BlockParams& nxt = w.params[static_cast<size_t>(block + 1)];
    const void* dln = gp(w.bwd_ar[(block + 1) % 2], w, block, sb, h);
    if (cfg_.ln && lnp_bwd_) {
      // one persistent pass: dx (+ residual), g_ar = dropout'(dx) and this sub-batch's column
      // partials of dgamma/dbeta (block b+1) and of the row-bias gradient (block b)
      const void* xn = gp(w.xbase[static_cast<size_t>(block + 1)], w, block, sb, h);
      const bool drop = cfg_.p_hidden > 0.f;
      const int acc_dx = cfg_.residual ? 1 : 0;
      const long long prows = lnp_partial_rows(dtype(), Ts, hi, acc_dx, ctx_.gemm_max_ctas);
      check_cuda(lnp_layernorm_bwd(dtype(), xn, nxt.p[OASES_P_LN_GAMMA], dln, g, acc_dx, drop ? gar_sb : nullptr,
                                   cfg_.p_hidden, cfg_.seed, drop_offset(block, sb, 0),
                                   drop && hbits_ ? w.hbits[static_cast<size_t>(block)][static_cast<size_t>(sb)] : nullptr,
                                   w.lnp_part + static_cast<int64_t>(sb) * prows * 3 * h, nullptr, Ts, hi, cfg_.eps,
                                   ctx_.gemm_max_ctas, ctx_.compute),
                 "layernorm_bwd (persistent)");
      gar_done = drop;
      row_bias_done = true;
      ++launches_;
      if (wgrad_now) {
        // dgamma/dbeta and the row-bias gradient over both sub-batches' partials: side stream
        const bool acc_ln = touch(w, block + 1, OASES_P_LN_GAMMA, degree(block));
        const bool acc_b = cfg_.bias ? touch(w, block, OASES_P_B_ROW) : false;
        BlockParams& cur = w.params[static_cast<size_t>(block)];
        fork_side();
        check_cuda(lnp_finalize(w.lnp_part, 2 * prows, hi, nxt.g[OASES_P_LN_GAMMA], nxt.g[OASES_P_LN_BETA],
                                cfg_.bias ? cur.g[OASES_P_B_ROW] : nullptr, acc_ln ? 1 : 0, acc_ln ? 1 : 0,
                                acc_b ? 1 : 0, ctx_.side),
                   "layernorm params + row bias finalize");
        ++launches_;
      }
    } else if (cfg_.ln) {
      const void* xn = gp(w.xbase[static_cast<size_t>(block + 1)], w, block, sb, h);
      const bool fuse = cfg_.p_hidden > 0.f && fuse_bdr_ln_ && ln_bwd_dropout_supported(dtype(), Ts, hi);
      // this sub-batch's row statistics land in rows [sb T_sub, (sb+1) T_sub) of the workspace
      void* stats_sb = static_cast<char*>(w.ln_ws) + static_cast<size_t>(sb) * Ts * 2 * sizeof(float);
      check_cuda(layernorm_bwd_part(1, dtype(), xn, nxt.p[OASES_P_LN_GAMMA], dln, g, cfg_.residual ? 1 : 0, nullptr,
                                    nullptr, 0, stats_sb, Ts, hi, cfg_.eps, ctx_.compute, fuse ? gar_sb : nullptr,
                                    cfg_.p_hidden, cfg_.seed, drop_offset(block, sb, 0),
                                    fuse && hbits_ ? w.hbits[static_cast<size_t>(block)][static_cast<size_t>(sb)] : nullptr),
                 "layernorm_bwd");
      gar_done = fuse;
      ++launches_;
      if (wgrad_now) {
        // dgamma/dbeta over both sub-batches: side stream, under this op's GEMMs (joined at the op's end)
        const bool acc = touch(w, block + 1, OASES_P_LN_GAMMA, degree(block));
        fork_side();
        check_cuda(layernorm_bwd_part(2, dtype(), gp(w.xbase[static_cast<size_t>(block + 1)], w, block, 0, h),
                                      nxt.p[OASES_P_LN_GAMMA], gp(w.bwd_ar[(block + 1) % 2], w, block, 0, h), nullptr, 0, nxt.g[OASES_P_LN_GAMMA],
                                      nxt.g[OASES_P_LN_BETA], acc ? 1 : 0, w.ln_ws, 2 * Ts, hi, cfg_.eps, ctx_.side),
                   "layernorm_bwd params");
        launches_ += 2;
      }
    } else {
      check_cuda(bias_dropout_residual_fwd(dtype(), dln, nullptr, cfg_.residual ? g : nullptr, g, Ts, hi, 0.f, 0, 0,
                                           ctx_.compute),
                 "residual grad add");
      ++launches_;
    }
  }
  // 2. through bias-dropout: g_ar = dropout'(g), dbias_row += colsum(g_ar)
  BlockParams& bp = w.params[static_cast<size_t>(block)];
  const void* gar = g;
  if (cfg_.p_hidden > 0.f) {
    if (!gar_done) {
      check_cuda(col_pass(dtype(), g, gar_sb, nullptr, 0, w.col_ws, Ts, hi, cfg_.p_hidden, cfg_.seed,
                          drop_offset(block, sb, 0), ctx_.compute),
                 "dropout bwd");
      ++launches_;
    }
    gar = gar_sb;
  }
  if (cfg_.bias && wgrad_now && !row_bias_done) {
    // row-bias gradient = column sums of g_ar over both sub-batches: side stream, under the row GEMMs
    const bool acc = touch(w, block, OASES_P_B_ROW);
    fork_side();
    check_cuda(col_pass(dtype(), gar == gar_sb ? w.gar : gp(w.grad, w, block, 0, h), nullptr, bp.g[OASES_P_B_ROW],
                        acc ? 1 : 0, w.col_ws,
                        2 * Ts, hi, 0.f, 0, 0, ctx_.side),
               "row bias grad");
    launches_ += 2;
  }
  Workspace ws = ws_for(w, block, sb);
  const bool att = is_attention(block);
  const int64_t ncol = this->ncol(block), nrow = this->nrow(block);
  // 3. row-parallel GEMM: dW_row (+)= g_ar^T act over both sub-batches ; d(act) = g_ar W_row
  // (g_ar is the sub-batch half of w.gar unless the dropout is off and g_ar == g,
  // a half of w.grad: both hold the two sub-batches contiguously)
  const void* gar_base = gar == gar_sb ? w.gar : gp(w.grad, w, block, 0, h);
  oases_gemm_desc dw{};
  if (wgrad_now) {
    dw.c_dtype = gdtype();
    dw.M = h; dw.N = nrow; dw.K = 2 * Ts;
    dw.batch = 1; dw.batch_inner = 1;
    dw.a = operand(gar_base, 2 * Ts, h, h, true);
    dw.b = operand(ws_for(w, block, 0).act, 2 * Ts, nrow, nrow, true);
    dw.c = bp.g[OASES_P_W_ROW]; dw.ldc = nrow;
    dw.alpha = 1.f; dw.accumulate = touch(w, block, OASES_P_W_ROW) ? 1 : 0;
  }
  oases_gemm_desc d{};
  d.c_dtype = dtype();
  d.M = Ts; d.N = nrow; d.K = h;
  d.batch = 1; d.batch_inner = 1;
  d.a = operand(gar, Ts, h, h, false);
  d.b = operand(bp.p[OASES_P_W_ROW], h, nrow, nrow, true);
  d.alpha = 1.f;
  if (att) {
    d.c = w.du; d.ldc = nrow;
    // ROWDOT: each 128-column epilogue stripe of the CTA-pair kernel holds whole heads
    rowdot_ = fused_attn_ && nrow > 128 && Ts > 128 && 128 % dh_ == 0;
    if (rowdot_) {
      // D = rowsum(dO o O) per head for the attention backward, from the dgrad epilogue
      d.epilogue = OASES_EPI_ROWDOT;
      d.aux = ws.act;
      d.rowdot = static_cast<float*>(w.attn_ws);
      d.rowdot_group = dh_;
      d.rowdot_seq = static_cast<int>(cfg_.s);
      d.rowdot_heads = hl(block);
    }
    if (wgrad_now) gemm2(dw, d);
    else gemm(d);
    attention_bwd(w, block, sb, ws);
  } else {
    // dpre = (g_ar W_row) o gelu'(pre)   (hadamard + gelu_grad, numerics.cpp:203-204; gelu'(pre)
    // was stored by the FC1 epilogue that produced the activation)
    d.c = lp(w.dcol, block, sb, ncol); d.ldc = ncol;
    d.epilogue = OASES_EPI_MUL;
    d.aux = ws.col;
    // column-bias gradient partials (32-row sums of dpre) from the same epilogue: this
    // sub-batch's rows [sb T_sub / 32, (sb + 1) T_sub / 32) of the partials
    if (colsum_) d.colsum = w.col_part + static_cast<int64_t>(sb) * (Ts / 32) * ncol;
    if (wgrad_now) gemm2(dw, d);
    else gemm(d);
  }
  // 4. column bias
  if (cfg_.bias && wgrad_now) {
    // the column-bias gradient (both sub-batches) only feeds the step's result: side stream, under
    // the column GEMMs
    const bool acc = touch(w, block, OASES_P_B_COL);
    fork_side();
    if (colsum_ && !att) {  // partials of both sub-batches' FC2 dgrad epilogues
      check_cuda(col_finalize(w.col_part, 2 * Ts / 32, static_cast<int>(ncol),
                              bp.g[OASES_P_B_COL], acc ? 1 : 0, ctx_.side),
                 "colsum finalize");
      launches_ += 1;
    } else {
      check_cuda(col_pass(dtype(), w.dcol, nullptr, bp.g[OASES_P_B_COL], acc ? 1 : 0, w.col_ws2, 2 * Ts,
                          static_cast<int>(ncol), 0.f, 0, 0, ctx_.side),
                 "colsum");
      launches_ += 2;
    }
  }
  // 5. column-parallel GEMM: dW_col (+)= dcol^T ln over both sub-batches ; d_ln partial = dcol W_col
  //    -> AR_b (backward f)
  const void* ln_base = cfg_.ln ? ws_for(w, block, 0).ln : gp(w.xbase[static_cast<size_t>(block)], w, block, 0, h);
  dw = oases_gemm_desc{};
  if (wgrad_now) {
    dw.c_dtype = gdtype();
    dw.M = ncol; dw.N = h; dw.K = 2 * Ts;
    dw.batch = 1; dw.batch_inner = 1;
    dw.a = operand(w.dcol, 2 * Ts, ncol, ncol, true);
    dw.b = operand(ln_base, 2 * Ts, h, h, true);
    dw.c = bp.g[OASES_P_W_COL]; dw.ldc = h;
    dw.alpha = 1.f; dw.accumulate = touch(w, block, OASES_P_W_COL) ? 1 : 0;
  }
  d = oases_gemm_desc{};
  d.c_dtype = dtype();
  d.M = Ts; d.N = h; d.K = ncol;
  d.batch = 1; d.batch_inner = 1;
  d.a = operand(lp(w.dcol, block, sb, ncol), Ts, ncol, ncol, false);
  d.b = operand(bp.p[OASES_P_W_COL], ncol, h, h, true);
  d.c = gp(w.bwd_ar[block % 2], w, block, sb, h); d.ldc = h;
  d.alpha = 1.f;
  if (wgrad_now) gemm2(dw, d);
  else gemm(d);
  join_side();
}

void Stack::tail(int wi, int sb) {
  Worker& w = workers_[static_cast<size_t>(wi)];
  const int64_t Ts = ts(0), h = cfg_.h;
  void* g = gp(w.grad, w, 0, sb, h);
  const void* dln = gp(w.bwd_ar[0], w, 0, sb, h);
  if (cfg_.ln) {
    const BlockParams& bp = w.params[0];
    const bool acc = touch(w, 0, OASES_P_LN_GAMMA, degree(0));
    check_cuda(layernorm_bwd(dtype(), gp(w.xbase[0], w, 0, sb, h), bp.p[OASES_P_LN_GAMMA], dln, g, cfg_.residual ? 1 : 0,
                             bp.g[OASES_P_LN_GAMMA], bp.g[OASES_P_LN_BETA], acc ? 1 : 0, w.ln_ws, Ts,
                             static_cast<int>(h), cfg_.eps, ctx_.compute, ctx_.gemm_max_ctas),
               "layernorm_bwd (tail)");
    launches_ += 3;
  } else {
    check_cuda(bias_dropout_residual_fwd(dtype(), dln, nullptr, cfg_.residual ? g : nullptr, g, Ts,
                                         static_cast<int>(h), 0.f, 0, 0, ctx_.compute),
               "residual grad add (tail)");
    ++launches_;
  }
}

void Stack::allreduce(tmpsim::Pass pass, int block, int sb, bool both) {
  if (ctx_.comm_disabled || (ctx_.tp == 1 && !ctx_.nccl)) return;
  const int par = block % 2, d = degree(block);
  auto pick = [&](Worker& w) -> void* {
    void* base = pass == tmpsim::Pass::Forward ? w.fwd_ar[par] : pass == tmpsim::Pass::Recompute ? w.rec_ar[par] : w.bwd_ar[par];
    return gp(base, w, block, both ? 0 : sb, cfg_.h);
  };
  const int64_t count = ts(block) * cfg_.h * (both ? 2 : 1);
  if (ctx_.local_workers > 1) {
    // one literal sum per group of the block's degree (worker order inside the group)
    if (d == 1) return;
    for (int g0 = 0; g0 < num_workers(); g0 += d) {
      std::vector<void*> bufs;
      for (int k = 0; k < d; ++k) bufs.push_back(pick(workers_[static_cast<size_t>(g0 + k)]));
      check_cuda(local_allreduce(dtype(), bufs.data(), d, count, ctx_.comm), "local allreduce");
      ++launches_;
    }
    return;
  }
  if (d == 1 && ctx_.tp > 1) return;
  void* p = pick(workers_[0]);
  check_nccl(ncclAllReduce(p, p, static_cast<size_t>(count), dtype() == OASES_BF16 ? ncclBfloat16 : ncclFloat32,
                           ncclSum, group_comm(d), ctx_.comm),
             "ncclAllReduce");
  ++launches_;
}

// ------------------------------------------------------------------ mixed degrees (F2)
// NCCL sub-communicators, split once per degree from the world communicator in
// a fixed order on every rank (Stack construction): the TMP group of degree d
// (color rank / d) and its data-parallel complement (color rank % d).
ncclComm_t Stack::group_comm(int d) {
  if (d == ctx_.tp) return ctx_.nccl;
  for (auto& c : tp_comms_)
    if (c.first == d) return c.second;
  throw ConfigError("stack: no communicator for degree " + std::to_string(d));
}

ncclComm_t Stack::dp_comm(int d) {
  for (auto& c : dp_comms_)
    if (c.first == d) return c.second;
  throw ConfigError("stack: no data-parallel communicator for degree " + std::to_string(d));
}

void Stack::gather_tokens(const std::vector<void*>& bases, int from_b, int to_b) {
  // to_b's group (degree du) covers du / dv slices of from_b (degree dv); split
  // its slice into du chunks: rank r of the group holds chunk r inside its own
  // slice of from_b, so this is an in-place AllGather of one chunk per rank
  const int du = degree(to_b);
  if (degree(from_b) >= du) throw ConfigError("gather_tokens: the target block's groups must be the larger ones");
  const int64_t h = cfg_.h, chunk = 2 * ts(to_b) / du;  // rows
  const int dt = dtype();
  if (ctx_.local_workers > 1) {
    for (int g0 = 0; g0 < num_workers(); g0 += du) {
      std::vector<void*> bufs;
      for (int k = 0; k < du; ++k) {
        const Worker& w = workers_[static_cast<size_t>(g0 + k)];
        bufs.push_back(static_cast<char*>(bases[static_cast<size_t>(g0 + k)]) +
                       static_cast<size_t>(row0(w, to_b) * h) * esize());
      }
      check_cuda(local_allgather(dt, bufs.data(), du, chunk * h, ctx_.comm), "local allgather");
      ++launches_;
    }
    return;
  }
  const Worker& w = workers_[0];
  char* base = static_cast<char*>(bases[0]) + static_cast<size_t>(row0(w, to_b) * h) * esize();
  const size_t cnt = static_cast<size_t>(chunk * h);
  check_nccl(ncclAllGather(base + static_cast<size_t>(rig(w, to_b)) * cnt * esize(), base, cnt,
                           dt == OASES_BF16 ? ncclBfloat16 : ncclFloat32, group_comm(du), ctx_.comm),
             "ncclAllGather");
  ++launches_;
}

void Stack::reshard_fwd(int v) {
  const int u = v + 1;
  const int64_t h = cfg_.h;
  std::vector<void*> bases;
  for (Worker& w : workers_) {
    const BlockParams& pv = w.params[static_cast<size_t>(v)];
    for (int sb = 0; sb < 2; ++sb) {
      // x_u = x_v + AR_v + bias_v on block v's slice (mixed degrees run without hidden dropout)
      check_cuda(bias_dropout_residual_fwd(dtype(), gp(w.fwd_ar[v % 2], w, v, sb, h),
                                           cfg_.bias ? pv.p[OASES_P_B_ROW] : nullptr,
                                           cfg_.residual ? gp(w.xbase[static_cast<size_t>(v)], w, v, sb, h) : nullptr,
                                           gp(w.xbase[static_cast<size_t>(u)], w, v, sb, h), ts(v),
                                           static_cast<int>(h), 0.f, 0, 0, ctx_.comm),
                 "reshard bdr");
      ++launches_;
    }
    bases.push_back(w.xbase[static_cast<size_t>(u)]);
  }
  gather_tokens(bases, v, u);
}

void Stack::reshard_bwd(int u) {
  const int v = u - 1;
  const int64_t h = cfg_.h, rows = 2 * ts(u);
  std::vector<void*> bases;
  for (Worker& w : workers_) {
    // g_u = g + LN_u'(dln_u) (+ the residual) over both sub-batches of block u's slice
    void* g = gp(w.grad, w, u, 0, h);
    const void* dln = gp(w.bwd_ar[u % 2], w, u, 0, h);
    if (cfg_.ln) {
      const BlockParams& bp = w.params[static_cast<size_t>(u)];
      const bool acc = touch(w, u, OASES_P_LN_GAMMA, degree(u));
      check_cuda(layernorm_bwd(dtype(), gp(w.xbase[static_cast<size_t>(u)], w, u, 0, h), bp.p[OASES_P_LN_GAMMA], dln,
                               g, cfg_.residual ? 1 : 0, bp.g[OASES_P_LN_GAMMA], bp.g[OASES_P_LN_BETA], acc ? 1 : 0,
                               w.ln_ws, rows, static_cast<int>(h), cfg_.eps, ctx_.comm, 0),
                 "reshard layernorm_bwd");
      launches_ += 3;
    } else {
      check_cuda(bias_dropout_residual_fwd(dtype(), dln, nullptr, cfg_.residual ? g : nullptr, g, rows,
                                           static_cast<int>(h), 0.f, 0, 0, ctx_.comm),
                 "reshard residual grad");
      ++launches_;
    }
    bases.push_back(w.grad);
  }
  gather_tokens(bases, u, v);
}

void Stack::dp_reduce_grads() {
  if (!mixed_) return;
  const int N = world();
  for (int b = 0; b < nblocks_; ++b) {
    for (int p = 0; p < OASES_P_COUNT; ++p) {
      const int64_t n = workers_[0].params[static_cast<size_t>(b)].numel[p];
      // LayerNorm beta follows gamma (one touch covers both)
      const int d = computed_at_[static_cast<size_t>(b)][static_cast<size_t>(p == OASES_P_LN_BETA ? OASES_P_LN_GAMMA : p)];
      if (!n || d == 0 || d == N) continue;
      if (ctx_.local_workers > 1) {
        for (int r = 0; r < d; ++r) {
          std::vector<void*> bufs;
          for (int k = r; k < N; k += d) bufs.push_back(workers_[static_cast<size_t>(k)].params[static_cast<size_t>(b)].g[p]);
          check_cuda(local_allreduce(gdtype(), bufs.data(), N / d, n, ctx_.comm), "dp grad allreduce");
          ++launches_;
        }
      } else {
        float* gptr = workers_[0].params[static_cast<size_t>(b)].g[p];
        check_nccl(ncclAllReduce(gptr, gptr, static_cast<size_t>(n), ncclFloat32, ncclSum, dp_comm(d), ctx_.comm),
                   "dp grad allreduce");
        ++launches_;
      }
    }
  }
}

}  // namespace oases
