// Runtime objects behind the C-ABI: the device/stream/NCCL context, the TMP
// layer stack (weights, saved boundary tensors, workspaces) and the plan
// executor that turns a tmpsim::SchedulePlan into kernels on a compute stream
// and AllReduces on a dedicated comm stream.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <array>
#include <memory>
#include <string>
#include <vector>

#include "../../../include/oases.h"
#include "../../../include/oases/tmpsim.hpp"
#include "layout.h"

namespace oases {

// ------------------------------------------------------------------ context
struct Context {
  int tp = 1;
  int rank = 0;
  int device = 0;
  int local_workers = 1;  // >1: all TMP ranks emulated in-process on `device`
  int gemm_max_ctas = 0;
  int nccl_max_ctas = 0;
  bool comm_disabled = false;  // calibration: one rank's shard, no collectives
  cudaStream_t compute = nullptr;
  cudaStream_t comm = nullptr;
  // side compute stream: parameter-gradient reductions forked off the compute
  // stream inside an op and joined before the op ends (off the critical path)
  cudaStream_t side = nullptr;
  cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
  ncclComm_t nccl = nullptr;
  ~Context();
};

std::unique_ptr<Context> make_context(const oases_ctx_desc& d);

// ------------------------------------------------------------------ memory
class DeviceArena {
 public:
  ~DeviceArena();
  void* alloc(size_t bytes);  // 256-byte aligned, zero-initialised
  void release(void* p);      // frees a block returned by alloc (no-op for nullptr)
  size_t bytes() const { return total_; }

 private:
  std::vector<std::pair<void*, size_t>> blocks_;
  size_t total_ = 0;
};

// ------------------------------------------------------------------ stack
// ModelCfg and the rank geometry (tokens / heads / columns per rank and block): layout.h

// Per-block parameters of one TMP worker (device layout [out, in]).
struct BlockParams {
  void* p[OASES_P_COUNT] = {};   // activation dtype
  float* g[OASES_P_COUNT] = {};  // f32 gradients
  int64_t numel[OASES_P_COUNT] = {};
  int rows[OASES_P_COUNT] = {};  // device layout rows (out features) for 2-D weights
};

// Activations of one (block, sub-batch) forward/recompute instance.
// (ws_for() returns a copy whose ln / act point at the sub-batch half of the
// slot's [2 T_sub, .] allocations for the block's own T_sub and row width.)
struct Workspace {
  void* ln = nullptr;   // [T_sub, h]  (aliases x when LN is off)
  void* col = nullptr;  // [T_sub, ncol]  qkv | pre
  void* act = nullptr;  // [T_sub, nrow]  ctx | gelu(pre)
  void* p = nullptr;    // [bh*Hl*s, s]   S then P (in place)
  void* pd = nullptr;   // dropped P (== p when attention dropout is 0)
  float* lse = nullptr; // [bh*Hl*s] row log-sum-exp of the fused attention (log2 domain)
};

// Token-indexed ("global") buffers hold [T, h] rows of the whole micro-batch
// (T = b * s); a block of degree d runs on N/d groups of d ranks (N = the
// world), group g owning the contiguous sample slice g of the micro-batch, and
// sub-batch sb of the block is half sb of that slice (Stack::gp). With every
// block at degree N this is the plain TMP layout (one group, the halves of T).
struct Worker {
  int rank = 0;  // rank in the world (the in-process worker index, or the NCCL rank)
  std::vector<BlockParams> params;
  // residual stream x_b (b = 0..nblocks-1), token-indexed [T, h]; x_0 is the
  // input. Blocks whose x_b the bound plan keeps until backward own a buffer;
  // the others (interior tensors of CrossPass-replayed layer units) share
  // x_scratch, rebuilt by their recompute (Stack::bind_storage).
  std::vector<void*> xbase;
  std::vector<void*> x_own;  // dedicated buffers, allocated on first need
  void* x_scratch = nullptr;
  void* fwd_ar[2] = {}, *rec_ar[2] = {}, *bwd_ar[2] = {};  // [block parity], token-indexed [T, h]
  std::vector<std::array<Workspace, 2>> ws;  // [slot][sb]
  std::vector<void*> ln_full, act_full;      // [slot] [2 T_sub, .] bases of ws.ln / ws.act
  void* input = nullptr;                     // [T, h]
  void* grad = nullptr;                      // [T, h] residual gradient g (token-indexed) == dX at the end
  // backward scratch (the compute stream serialises all B_b)
  void* gar = nullptr;   // [T_sub, h]  dropout'(g)
  void* du = nullptr;    // [T_sub, nmax] d(row GEMM input)
  void* dcol = nullptr;  // [T_sub, ncol_max]
  void* dp = nullptr;    // [bh*Hl*s, s]  dP_drop then dS (fused attention: dS only)
  void* attn_ws = nullptr;  // fused attention backward workspace (rowsum(dO o O))
  // attention-dropout keep bits per [attention block][sb], written by the
  // forward pass, read by the recompute forward and the backward
  std::vector<std::array<uint32_t*, 2>> mask_bits;
  // hidden-dropout keep bits per [block b][sb] of the dropout on AR_b's output,
  // written by the forward's fused bias-dropout-residual + LN of block b+1,
  // read by the backward's fused LN-backward + dropout'
  std::vector<std::array<uint16_t*, 2>> hbits;
  void* y = nullptr;     // [T, h] final output x_B (token-indexed) for the loss head
  void* ln_ws = nullptr;
  float* lnp_part = nullptr;  // persistent LayerNorm backward column partials [2][prows][3][h]
  void* col_ws = nullptr;
  void* col_ws2 = nullptr;  // side-stream column sums (bias gradients)
  float* col_part = nullptr;  // FC2 dgrad epilogue's 32-row column-sum partials (FFN column bias)
  double* loss = nullptr;     // device scalar (f64)
  double* loss_ws = nullptr;  // partials
};

class Stack {
 public:
  // degrees: per-block TMP degree (each divides the world size ctx.tp); empty =
  // every block at ctx.tp. Mixed degrees: a block of
  // degree d < N runs data-parallel over N/d groups of d ranks.
  Stack(Context& ctx, const ModelCfg& cfg, const std::vector<int>& degrees = {});
  ~Stack();
  int degree(int b) const { return deg_[static_cast<size_t>(b)]; }
  int world() const { return ctx_.tp; }
  bool mixed() const { return mixed_; }

  const ModelCfg& cfg() const { return cfg_; }
  Context& ctx() { return ctx_; }
  int num_blocks() const { return nblocks_; }
  int num_workers() const { return static_cast<int>(workers_.size()); }
  bool is_attention(int b) const { return attention_block(cfg_, b); }
  int dtype() const { return cfg_.bytes == 2 ? OASES_BF16 : (cfg_.bytes == 8 ? OASES_F64 : OASES_F32); }
  // gradient dtype: f32 (f64 in the value-level toy mode)
  int gdtype() const { return cfg_.bytes == 8 ? OASES_F64 : OASES_F32; }
  size_t gsize() const { return cfg_.bytes == 8 ? 8 : 4; }
  size_t esize() const { return static_cast<size_t>(cfg_.bytes); }
  int64_t tokens_sub() const { return static_cast<int64_t>(cfg_.b / 2) * cfg_.s; }
  int64_t param_numel(int block, int p) const;
  size_t device_bytes() const { return arena_.bytes(); }

  void set_param(int worker, int block, int p, const double* host);
  void get_grad(int worker, int block, int p, double* host);
  void init_random(uint64_t seed);
  void set_input(const void* host, int host_dtype, cudaStream_t st);
  void get_input_grad(double* host);
  void get_activation(int worker, int block, int sb, double* host);
  // Residual-stream storage for a plan: stored[b] (b > 0) keeps x_b in its own
  // HBM buffer from forward to backward; false maps it onto a scratch buffer
  // (the plan rebuilds it in recompute). Called by plan_bind.
  void bind_storage(const std::vector<bool>& stored);

  // ---- per-op kernel lists (issued on ctx.compute for every worker) ----
  void forward(int worker, int block, int sb, bool with_bdr, bool with_row);
  // recompute: replay_input: -1 = saved x_b; else rebuild x_b from rec_ar of block-1
  void recompute(int worker, int block, int sb, bool rebuild_x, bool with_row);
  // g_ready: the gradient at x_{b+1} (LN_{b+1} backward included) is already in
  // the residual-gradient rows (gathered by reshard_bwd)
  void backward(int worker, int block, int sb, bool g_ready = false);
  void tail(int worker, int sb);  // LN_0 backward after the last backward AR
  // ---- resharding between blocks of different degree (the AllGathers of
  //      sim.cpp:101-175), issued on ctx.comm for every worker ----
  // degree grows at v -> v+1: x_{v+1} = x_v + AR_v + bias on each rank's slice of
  // block v, then gathered over block v+1's groups (F_{v+1} skips its BDR)
  void reshard_fwd(int v);
  // degree shrinks at u-1 -> u: g + LN_u'(dln_u) on block u's slice, then
  // gathered over block u-1's groups (B_{u-1} runs with g_ready)
  void reshard_bwd(int u);
  // sums every gradient computed data-parallel (on groups smaller than the
  // world) over the groups, on ctx.comm: after it each rank holds the
  // micro-batch gradient of its shard
  void dp_reduce_grads();
  // ---- communication (issued on ctx.comm) ----
  void allreduce(tmpsim::Pass pass, int block, int sb, bool both_halves);

  void begin_step();  // resets first-touch flags of gradient accumulation
  double read_loss();

  int64_t kernel_launches() const { return launches_; }
  // Live per-launch timing of the linear-layer GEMMs (QKV/proj/FC1/FC2 and their
  // dgrad/wgrad) with cudaEvents on the compute stream, for the roofline.
  void set_kernel_timing(bool on) { timing_ = on; }
  void reset_kernel_stats() { timed_ = 0; }
  void kernel_stats(double* gemm_ms, double* gemm_flops, int* launches);

 private:
  void alloc_all();
  void gemm(const oases_gemm_desc& d);
  cudaError_t record_timing(cudaEvent_t e);
  void gemm2(const oases_gemm_desc& d0, const oases_gemm_desc& d1);
  void fork_side();  // side stream waits for the compute stream's current tail
  void join_side();  // compute stream waits for the side stream's current tail
  bool side_forked_ = false;
  void ln_fwd(const void* x, const void* g, const void* b, void* y, int64_t rows);
  void bdr_then_ln(Worker& w, int block, int sb, const void* ar, void* x, void* ln, bool store_bits);
  // bases[w]: a token-indexed [T, h] buffer per worker whose rows of block
  // from_b's slice are valid; gathers the rows of block to_b's (larger) slice
  // from the peers of to_b's group (ncclAllGather on the group communicator,
  // or a copy kernel between the in-process workers)
  void gather_tokens(const std::vector<void*>& bases, int from_b, int to_b);
  ncclComm_t group_comm(int d);  // the TMP group communicator of degree d (NCCL mode)
  ncclComm_t dp_comm(int d);     // ranks with the same rank-in-group of degree d
  oases_attn_desc attn_desc(Worker& w, int block, int sb, const Workspace& ws);
  void attention_fwd(Worker& w, int block, int sb, const Workspace& ws, int mask_mode);
  void attention_bwd(Worker& w, int block, int sb, const Workspace& ws);
  Workspace ws_for(Worker& w, int block, int sb);
  bool touch(const Worker& w, int block, int p, int computed_at = 0);  // true if the gradient must accumulate
  // per-block geometry (degree-dependent)
  // rank geometry: layout.h (shared with the host-only oases_rank_layout)
  int hl(int b) const { return heads_local(cfg_, degree(b)); }
  int64_t ncol(int b) const { return col_width(cfg_, degree(b), is_attention(b)); }
  int64_t nrow(int b) const { return row_width(cfg_, degree(b), is_attention(b)); }
  int64_t bsub(int b) const { return samples_per_sub(cfg_, world(), degree(b)); }  // samples per sub-batch
  int64_t ts(int b) const { return tokens_per_sub(cfg_, world(), degree(b)); }     // tokens per sub-batch
  int rig(const Worker& w, int b) const { return rank_in_group(w.rank, degree(b)); }  // rank in the block's group
  int64_t row0(const Worker& w, int b) const { return token_row0(cfg_, world(), degree(b), w.rank); }
  // rows of sub-batch sb of block b (this worker's group) in a token-indexed buffer
  void* gp(void* base, const Worker& w, int b, int sb, int64_t cols) const;
  // half sb of a local [2 ts(b), cols] buffer
  void* lp(void* base, int b, int sb, int64_t cols) const;

  Context& ctx_;
  ModelCfg cfg_;
  DeviceArena arena_;
  std::vector<Worker> workers_;
  int nblocks_ = 0;
  bool fused_attn_ = false;  // tcgen05 flash attention (attention.cu) instead of QK^T / softmax / PV
  bool fuse_bdr_ln_ = true;
  bool rowdot_ = false;  // attention D = rowsum(dO o O) comes from the proj dgrad epilogue
  bool lnp_bwd_ = false;  // persistent LayerNorm backward with folded column sums (rowpipe.cu)
  bool hbits_ = false;   // hidden-dropout keep bits cached (fused forward kernel covers the shape)
  bool colsum_ = false;  // FFN column-bias gradient partials come from the FC2 dgrad (MUL) epilogue
  int hl_ = 0, dh_ = 0;  // local heads at the world degree, head dim
  std::vector<std::vector<std::array<bool, OASES_P_COUNT>>> touched_;  // [worker][block]
  // degree of the groups a gradient was computed on this step (0: untouched); < world -> dp_reduce_grads
  std::vector<std::array<int, OASES_P_COUNT>> computed_at_;  // [block] (same on every worker)
  std::vector<int> deg_;  // [block]
  bool mixed_ = false;
  std::vector<std::pair<int, ncclComm_t>> tp_comms_, dp_comms_;  // NCCL sub-communicators by degree
  std::vector<bool> loss_touched_;
  std::vector<std::vector<bool>> bwd_seen_;  // [worker][block] first backward call of the step done
  std::vector<bool> x_stored_;  // [block] x_b readable after a step (bind_storage)
  int64_t launches_ = 0;
  bool timing_ = false;
  size_t timed_ = 0;
  std::vector<cudaEvent_t> tev_;
  std::vector<double> tflops_;
};

// ------------------------------------------------------------------ executor
struct ExecOp {
  int id = 0;
  tmpsim::OpKind kind = tmpsim::OpKind::ForwardCompute;
  tmpsim::Pass pass = tmpsim::Pass::Forward;
  int stream = 0;  // 0 compute, 1 comm
  int block = 0;
  int sb = 0;
  bool both_halves = false;  // unsplit (Default) plans: one op covers both sub-batches
  bool rebuild_x = false;    // recompute restarts from a replayed comm (CrossPass inside a unit)
  bool with_row = false;     // recompute also runs the row-parallel GEMM (its AR is replayed)
  bool with_bdr = true;      // forward: builds x_b itself (false after a degree-growing reshard)
  bool g_ready = false;      // backward: a degree-shrinking reshard gathered its input gradient
  int seq = 0;               // position in plan order (reshards right after their anchors)
  std::vector<int> waits;    // cross-stream deps (op ids)
};

class Executor {
 public:
  Executor(Stack& stack, const tmpsim::SchedulePlan& plan);
  ~Executor();
  // One step; returns measured SimResult (trace when `trace`).
  tmpsim::SimResult step(bool trace);
  bool capture_graph();
  // Captures a separate graph of the step with the per-GEMM timing events as
  // graph nodes, replays it twice and leaves the second replay's GEMM timings
  // in the stack's kernel stats (the roofline of the graph-replayed step).
  void timed_graph_replay();
  const tmpsim::SchedulePlan& plan() const { return plan_; }
  const std::vector<oases_trace_event>& events() const { return events_; }

 private:
  void issue(bool trace);
  // resharding AllGathers between blocks of different degree, at the anchors
  // of sim.cpp:101-175 (after the upstream block's last forward comm when the
  // degree grows; after the downstream block's backward tail when it shrinks)
  void inject_reshards(int n);
  Stack& stack_;
  tmpsim::SchedulePlan plan_;
  std::vector<ExecOp> ops_;
  std::vector<cudaEvent_t> done_;   // per op (+ tails) completion, sync-only
  std::vector<cudaEvent_t> t0_, t1_;  // per op timing
  cudaEvent_t begin_ = nullptr, end_ = nullptr, fork_ = nullptr;
  std::array<int, 2> tail_wait_ = {-1, -1};  // last backward AR (per sb) the LN_0 tail waits for
  std::vector<int> stream_of_;  // [op id] 0 compute / 1 comm (plan ops, then the injected reshards)
  int nreshard_ = 0;            // injected AllGathers: op ids n .. n + nreshard_ - 1
  cudaGraph_t graph_ = nullptr;
  cudaGraphExec_t graph_exec_ = nullptr;
  std::vector<oases_trace_event> events_;
};

}  // namespace oases
