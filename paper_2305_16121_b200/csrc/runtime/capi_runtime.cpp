// extern "C" runtime entry points of include/oases.h: context, stack, plan
// binding and the measured step. Handles are opaque; every call maps C++
// exceptions to status codes (status.h).
#include <nccl.h>

#include <cstring>
#include <memory>

#include "../../../include/oases.h"
#include "stack.h"
#include "status.h"

// Contexts are reference counted: every stack holds one reference, so the
// destruction order chosen by a garbage collector cannot free the streams or
// the NCCL communicator under a live stack.
struct oases_ctx {
  std::unique_ptr<oases::Context> ctx;
  int refs = 1;
};

namespace {
void ctx_release(oases_ctx* c) {
  if (c && --c->refs == 0) delete c;
}
}  // namespace

struct oases_stack {
  oases_ctx* owner = nullptr;
  std::unique_ptr<oases::Stack> stack;
  std::unique_ptr<oases::Executor> exec;
  std::vector<oases_trace_event> events;
};

using oases::guarded;
using tmpsim::ConfigError;

namespace {

oases::ModelCfg to_cfg(const oases_model_desc& m) {
  oases::ModelCfg c;
  c.h = m.hidden_size;
  c.f = m.ffn_hidden > 0 ? m.ffn_hidden : 4 * m.hidden_size;
  c.heads = m.attention_heads;
  c.s = m.seq_len;
  c.b = m.global_batch;
  c.layers = m.num_layers;
  c.bytes = m.bytes_per_element;
  c.recompute = m.recompute_enabled != 0;
  c.attention = m.use_attention != 0;
  c.ln = m.use_layernorm != 0;
  c.bias = m.use_bias != 0;
  c.residual = m.use_residual != 0;
  c.p_hidden = m.hidden_dropout;
  c.p_attn = m.attention_dropout;
  c.eps = m.ln_eps > 0.f ? m.ln_eps : 1e-5f;
  c.seed = m.seed;
  return c;
}

tmpsim::SchedulePlan unflatten(const oases_flat_plan& f) {
  if (f.n_ops < 0 || f.n_forward < 0 || f.n_forward > f.n_ops || (f.n_ops && !f.ops) || f.n_deps < 0 ||
      (f.n_deps > 0 && !f.deps))
    throw ConfigError("plan_bind: malformed flat plan");
  if (f.variant < 0 || f.variant > static_cast<int>(tmpsim::ScheduleVariant::Oases))
    throw ConfigError("plan_bind: unknown schedule variant " + std::to_string(f.variant));
  tmpsim::SchedulePlan p;
  p.variant = static_cast<tmpsim::ScheduleVariant>(f.variant);
  p.split_batch = f.split_batch != 0;
  p.has_recompute = f.has_recompute != 0;
  for (int i = 0; i < f.n_ops; ++i) {
    const oases_plan_op& o = f.ops[i];
    // enum and index ranges (the executor indexes per-sub-batch and per-block arrays with them)
    if (o.kind < 0 || o.kind > static_cast<int>(tmpsim::OpKind::AllGather) || o.pass < 0 ||
        o.pass > static_cast<int>(tmpsim::Pass::Backward) || o.stream < 0 ||
        o.stream > static_cast<int>(tmpsim::Stream::Comm))
      throw ConfigError("plan_bind: op " + std::to_string(i) + " has an out-of-range kind/pass/stream");
    if (o.sub_batch < 0 || o.sub_batch > 1 || o.block < 0)
      throw ConfigError("plan_bind: op " + std::to_string(i) + " has sub_batch outside {0,1} or a negative block");
    tmpsim::ScheduledOp op;
    op.id = o.id;
    op.base_id = o.base_id;
    op.kind = static_cast<tmpsim::OpKind>(o.kind);
    op.pass = static_cast<tmpsim::Pass>(o.pass);
    op.stream = static_cast<tmpsim::Stream>(o.stream);
    op.block = o.block;
    op.sub_batch = o.sub_batch;
    op.blocking = o.blocking != 0;
    if (o.dep_begin < 0 || o.dep_count < 0 || o.dep_begin + o.dep_count > f.n_deps)
      throw ConfigError("plan_bind: dependency range out of bounds");
    op.deps.assign(f.deps + o.dep_begin, f.deps + o.dep_begin + o.dep_count);
    (i < f.n_forward ? p.forward_ops : p.backward_ops).push_back(std::move(op));
  }
  return p;
}

oases::Stack& S(oases_stack* s) {
  if (!s || !s->stack) throw ConfigError("null stack");
  return *s->stack;
}

}  // namespace

extern "C" {

oases_status oases_get_unique_id(void* out) {
  return guarded([&] {
    if (!out) throw ConfigError("null output");
    ncclUniqueId id;
    const ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) throw oases::NcclError(std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
    std::memcpy(out, &id, sizeof(id));
  });
}

oases_status oases_ctx_create(const oases_ctx_desc* desc, oases_ctx** out) {
  return guarded([&] {
    if (!desc || !out) throw ConfigError("null argument");
    auto h = std::make_unique<oases_ctx>();
    h->ctx = oases::make_context(*desc);
    *out = h.release();
  });
}

oases_status oases_ctx_destroy(oases_ctx* ctx) {
  return guarded([&] { ctx_release(ctx); });
}

oases_status oases_stack_create(oases_ctx* ctx, const oases_model_desc* model, oases_stack** out) {
  return guarded([&] {
    if (!ctx || !ctx->ctx || !model || !out) throw ConfigError("null argument");
    auto h = std::make_unique<oases_stack>();
    h->stack = std::make_unique<oases::Stack>(*ctx->ctx, to_cfg(*model));
    h->owner = ctx;
    ++ctx->refs;
    *out = h.release();
  });
}

oases_status oases_stack_create_mixed(oases_ctx* ctx, const oases_model_desc* model, const int32_t* block_degrees,
                                      int32_t num_blocks, oases_stack** out) {
  return guarded([&] {
    if (!ctx || !ctx->ctx || !model || !out || (num_blocks > 0 && !block_degrees)) throw ConfigError("null argument");
    if (num_blocks < 0) throw ConfigError("num_blocks must be >= 0");
    std::vector<int> deg(block_degrees, block_degrees + num_blocks);
    auto h = std::make_unique<oases_stack>();
    h->stack = std::make_unique<oases::Stack>(*ctx->ctx, to_cfg(*model), deg);
    h->owner = ctx;
    ++ctx->refs;
    *out = h.release();
  });
}

oases_status oases_rank_layout(const oases_model_desc* model, int32_t world, const int32_t* block_degrees,
                               int32_t num_blocks, int32_t rank, oases_block_layout* out) {
  return guarded([&] {
    if (!model || !out) throw ConfigError("oases_rank_layout: null argument");
    const oases::ModelCfg cfg = to_cfg(*model);
    if (cfg.b <= 0 || cfg.s <= 0 || cfg.h <= 0 || cfg.layers < 0)
      throw ConfigError("oases_rank_layout: sizes must be positive");
    if (cfg.b % 2) throw ConfigError("stack: global_batch must be even (two sub-batches)");
    if (num_blocks != oases::num_blocks(cfg))
      throw ConfigError((block_degrees ? "stack: one degree per block (" : "oases_rank_layout: num_blocks must be (") +
                        std::to_string(oases::num_blocks(cfg)) + ")");
    if (rank < 0 || rank >= world) throw ConfigError("oases_rank_layout: rank outside [0, world)");
    std::vector<int> deg;
    if (block_degrees) deg.assign(block_degrees, block_degrees + num_blocks);
    deg = oases::resolve_degrees(cfg, world, deg, nullptr);
    for (int b = 0; b < num_blocks; ++b) {
      const int d = deg[static_cast<size_t>(b)];
      const bool att = oases::attention_block(cfg, b);
      oases_block_layout& o = out[b];
      o = oases_block_layout{};
      o.degree = d;
      o.group = oases::group_of(rank, d);
      o.rank_in_group = oases::rank_in_group(rank, d);
      o.groups = world / d;
      o.heads_local = att ? oases::heads_local(cfg, d) : 0;
      o.attention = att ? 1 : 0;
      o.samples_per_sub_batch = oases::samples_per_sub(cfg, world, d);
      o.tokens_per_sub_batch = oases::tokens_per_sub(cfg, world, d);
      o.token_row0 = oases::token_row0(cfg, world, d, rank);
      o.col_width = oases::col_width(cfg, d, att);
      o.row_width = oases::row_width(cfg, d, att);
    }
  });
}

int oases_stack_block_degree(const oases_stack* s, int block) {
  return (s && s->stack && block >= 0 && block < s->stack->num_blocks()) ? s->stack->degree(block) : 0;
}

oases_status oases_stack_destroy(oases_stack* s) {
  return guarded([&] {
    if (s) {
      if (s->stack) cudaStreamSynchronize(s->stack->ctx().compute);
      s->exec.reset();
      s->stack.reset();
      ctx_release(s->owner);
      delete s;
    }
  });
}

int64_t oases_stack_param_numel(const oases_stack* s, int block, int param) {
  return (s && s->stack) ? s->stack->param_numel(block, param) : 0;
}
int oases_stack_num_blocks(const oases_stack* s) { return (s && s->stack) ? s->stack->num_blocks() : 0; }
int oases_stack_num_workers(const oases_stack* s) { return (s && s->stack) ? s->stack->num_workers() : 0; }

oases_status oases_stack_set_param(oases_stack* s, int worker, int block, int param, const double* host) {
  return guarded([&] { S(s).set_param(worker, block, param, host); });
}

oases_status oases_stack_get_grad(oases_stack* s, int worker, int block, int param, double* host) {
  return guarded([&] { S(s).get_grad(worker, block, param, host); });
}

oases_status oases_stack_init_random(oases_stack* s, uint64_t seed) {
  return guarded([&] { S(s).init_random(seed); });
}

oases_status oases_plan_bind(oases_stack* s, const oases_flat_plan* plan) {
  return guarded([&] {
    if (!plan) throw ConfigError("null plan");
    oases::Stack& st = S(s);
    s->exec.reset();
    s->exec = std::make_unique<oases::Executor>(st, unflatten(*plan));
  });
}

oases_status oases_stack_set_input(oases_stack* s, const void* host, int input_dtype) {
  return guarded([&] {
    oases::Stack& st = S(s);
    st.set_input(host, input_dtype, st.ctx().compute);
    oases::check_cuda(cudaStreamSynchronize(st.ctx().compute), "set_input");
  });
}

oases_status oases_step(oases_stack* s, const void* input_host, int input_dtype, int trace, oases_step_result* out) {
  return guarded([&] {
    oases::Stack& st = S(s);
    if (!s->exec) throw ConfigError("oases_step: no plan bound");
    if (input_host) st.set_input(input_host, input_dtype, st.ctx().compute);
    tmpsim::SimResult r = s->exec->step(trace != 0);
    if (out) {
      std::memset(out, 0, sizeof(*out));
      out->makespan = r.makespan;
      out->compute_busy_fraction = r.compute_busy_fraction;
      out->comm_exposed = r.comm_exposed;
      out->peak_memory = r.peak_memory;
      out->loss = st.read_loss();
      s->events = s->exec->events();
      out->n_events = static_cast<int32_t>(s->events.size());
      out->events = s->events.empty() ? nullptr : s->events.data();
    }
  });
}

oases_status oases_stack_get_input_grad(oases_stack* s, double* host) {
  return guarded([&] { S(s).get_input_grad(host); });
}

oases_status oases_stack_get_activation(oases_stack* s, int worker, int block, int sb, double* host) {
  return guarded([&] { S(s).get_activation(worker, block, sb, host); });
}

oases_status oases_stack_capture_graph(oases_stack* s) {
  return guarded([&] {
    S(s);
    if (!s->exec) throw ConfigError("capture_graph: no plan bound");
    s->exec->capture_graph();
  });
}

oases_status oases_stack_sync(oases_stack* s) {
  return guarded([&] { oases::check_cuda(cudaDeviceSynchronize(), "sync"); (void)S(s); });
}

oases_status oases_stack_set_kernel_timing(oases_stack* s, int on) {
  return guarded([&] {
    S(s).set_kernel_timing(on != 0);
    S(s).reset_kernel_stats();
  });
}

oases_status oases_stack_kernel_stats(oases_stack* s, oases_kernel_stats* out) {
  return guarded([&] {
    if (!out) throw ConfigError("null output");
    std::memset(out, 0, sizeof(*out));
    int n = 0;
    S(s).kernel_stats(&out->gemm_ms, &out->gemm_flops, &n);
    out->gemm_launches = n;
    S(s).reset_kernel_stats();
  });
}

oases_status oases_stack_graph_kernel_stats(oases_stack* s, oases_kernel_stats* out) {
  return guarded([&] {
    if (!out) throw ConfigError("null output");
    S(s);
    if (!s->exec) throw ConfigError("graph_kernel_stats: no plan bound");
    s->exec->timed_graph_replay();
    std::memset(out, 0, sizeof(*out));
    int n = 0;
    S(s).kernel_stats(&out->gemm_ms, &out->gemm_flops, &n);
    out->gemm_launches = n;
    S(s).reset_kernel_stats();
  });
}

int oases_stack_kernel_launches(const oases_stack* s) {
  return (s && s->stack) ? static_cast<int>(s->stack->kernel_launches()) : 0;
}

}  // extern "C"
