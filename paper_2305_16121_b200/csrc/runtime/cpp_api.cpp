// C++ entry points of the measured runtime (include/oases/runtime.hpp):
// tmpsim::Context / execute / calibrate / allreduce_seconds, the §8(b)
// "execute() -> SimResult" and "calibrate() -> MeasuredRow" of SURVEY.md,
// on the same oases::Stack + Executor as the C-ABI.
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <memory>
#include <tuple>

#include "../kernels/kernels.h"
#include "oases/runtime.hpp"
#include "stack.h"
#include "status.h"

namespace tmpsim {

using oases::check_cuda;

struct Context::Impl {
  ContextOptions opts;
  std::unique_ptr<oases::Context> ctx;
  // cached stack of the last execute() (rebuilt when the model changes)
  std::unique_ptr<oases::Stack> stack;
  std::tuple<int, int, int, int, int, int, int, int, int, int, int, int, double, double, std::uint64_t> key{};
  bool seeded = false;
  std::vector<int> degrees;
};

namespace {

oases_ctx_desc to_desc(const ContextOptions& o) {
  oases_ctx_desc d{};
  d.tp = o.tp;
  d.rank = o.rank;
  d.device = o.device;
  d.local_workers = o.local_workers;
  d.unique_id = o.nccl_unique_id.empty() ? nullptr : o.nccl_unique_id.data();
  d.nccl_max_ctas = o.nccl_max_ctas;
  d.gemm_max_ctas = o.gemm_max_ctas;
  d.comm_disabled = o.comm_disabled ? 1 : 0;
  return d;
}

oases::ModelCfg to_cfg(const ModelSpec& s, const ExecOptions& o) {
  s.validate();
  oases::ModelCfg c;
  c.h = s.hidden_size;
  c.f = o.ffn_hidden > 0 ? o.ffn_hidden : 4 * s.hidden_size;
  c.heads = s.attention_heads;
  c.s = s.seq_len;
  c.b = s.global_batch;
  c.layers = s.num_layers;
  c.bytes = s.bytes_per_element;
  c.recompute = s.recompute_enabled;
  c.attention = o.attention;
  c.ln = o.layernorm;
  c.bias = o.bias;
  c.residual = o.residual;
  c.p_hidden = static_cast<float>(o.hidden_dropout);
  c.p_attn = static_cast<float>(o.attention_dropout);
  c.seed = o.seed;
  return c;
}

// The strategy's per-block degrees (each dividing the context's world size
// ctx tp); mixed degrees run data-parallel groups with resharding AllGathers.
std::vector<int> strategy_degrees(const SchedulePlan& plan, const Strategy& st, int tp) {
  int max_block = -1;
  for (int i = 0; i < plan.total_ops(); ++i) max_block = std::max(max_block, plan.op(i).block);
  if (static_cast<int>(st.degrees.size()) != max_block + 1)
    throw ConfigError("execute: strategy needs one degree per block (" + std::to_string(max_block + 1) + ")");
  for (int d : st.degrees)
    if (d < 1 || tp % d) throw ConfigError("execute: every block degree must divide the context's world size " + std::to_string(tp));
  return st.degrees;
}

}  // namespace

std::string nccl_unique_id() {
  ncclUniqueId id;
  const ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) throw oases::NcclError(std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
  return std::string(reinterpret_cast<const char*>(&id), sizeof(id));
}

Context::Context(const ContextOptions& options) : impl_(std::make_unique<Impl>()) {
  impl_->opts = options;
  if (!options.nccl_unique_id.empty() && options.nccl_unique_id.size() != OASES_UNIQUE_ID_BYTES)
    throw ConfigError("Context: nccl_unique_id must hold " + std::to_string(OASES_UNIQUE_ID_BYTES) + " bytes");
  impl_->ctx = oases::make_context(to_desc(options));
}

Context::~Context() = default;
const ContextOptions& Context::options() const { return impl_->opts; }
Context::Impl& Context::impl() { return *impl_; }

SimResult execute(const SchedulePlan& plan, const Strategy& strategy, Context& ctx, const ExecOptions& opts) {
  Context::Impl& I = ctx.impl();
  const std::vector<int> degrees = strategy_degrees(plan, strategy, I.opts.tp);
  if (opts.steps < 1 || opts.warmup < 0) throw ConfigError("execute: steps >= 1 and warmup >= 0");
  const oases::ModelCfg c = to_cfg(opts.spec, opts);
  const auto key = std::make_tuple(c.h, c.f, c.heads, c.s, c.b, c.layers, c.bytes, int(c.recompute), int(c.attention),
                                   int(c.ln), int(c.bias), int(c.residual), double(c.p_hidden), double(c.p_attn),
                                   c.seed);
  if (!I.stack || key != I.key || degrees != I.degrees) {
    I.stack.reset();
    I.stack = std::make_unique<oases::Stack>(*I.ctx, c, degrees);
    I.degrees = degrees;
    I.stack->init_random(c.seed);
    I.key = key;
  }
  oases::Executor ex(*I.stack, plan);
  if (opts.cuda_graph) ex.capture_graph();
  for (int i = 0; i < opts.warmup; ++i) ex.step(false);
  SimResult r;
  for (int i = 0; i < opts.steps; ++i) r = ex.step(!opts.cuda_graph);
  return r;
}

double allreduce_seconds(Context& ctx, double message_bytes, int bytes_per_element, int iters) {
  Context::Impl& I = ctx.impl();
  oases::Context& c = *I.ctx;
  if (bytes_per_element != 2 && bytes_per_element != 4) throw ConfigError("allreduce_seconds: bf16 or f32");
  if (iters < 1) throw ConfigError("allreduce_seconds: iters >= 1");
  const long long n = static_cast<long long>(message_bytes) / bytes_per_element;
  if (n < 1) throw ConfigError("allreduce_seconds: empty message");
  const int W = c.local_workers;
  if (W == 1 && !c.nccl) throw ConfigError("allreduce_seconds: the context has no communicator (tp == 1)");
  std::vector<void*> bufs(static_cast<size_t>(W), nullptr);
  for (auto& b : bufs) {
    check_cuda(cudaMalloc(&b, static_cast<size_t>(n) * bytes_per_element), "cudaMalloc");
    check_cuda(cudaMemset(b, 0, static_cast<size_t>(n) * bytes_per_element), "cudaMemset");
  }
  cudaEvent_t e0, e1;
  check_cuda(cudaEventCreate(&e0), "event");
  check_cuda(cudaEventCreate(&e1), "event");
  const int dt = bytes_per_element == 2 ? OASES_BF16 : OASES_F32;
  auto issue = [&] {
    if (W > 1) {
      check_cuda(oases::local_allreduce(dt, bufs.data(), W, n, c.comm), "local allreduce");
    } else {
      const ncclResult_t r = ncclAllReduce(bufs[0], bufs[0], static_cast<size_t>(n),
                                           dt == OASES_BF16 ? ncclBfloat16 : ncclFloat32, ncclSum, c.nccl, c.comm);
      if (r != ncclSuccess) throw oases::NcclError(std::string("ncclAllReduce: ") + ncclGetErrorString(r));
    }
  };
  for (int i = 0; i < 3; ++i) issue();
  std::vector<double> t;
  for (int i = 0; i < iters; ++i) {
    check_cuda(cudaEventRecord(e0, c.comm), "record");
    issue();
    check_cuda(cudaEventRecord(e1, c.comm), "record");
    check_cuda(cudaEventSynchronize(e1), "sync");
    float ms = 0.f;
    check_cuda(cudaEventElapsedTime(&ms, e0, e1), "elapsed");
    t.push_back(ms * 1e-3);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  for (void* b : bufs) cudaFree(b);
  std::sort(t.begin(), t.end());
  return t[t.size() / 2];
}

std::vector<MeasuredRow> calibrate(const ModelGraph& graph, const ModelSpec& spec, Context& ctx,
                                   const std::vector<int>& degrees, const ExecOptions& opts, int steps) {
  if (degrees.empty()) throw ConfigError("calibrate: no degrees");
  if (steps < 1) throw ConfigError("calibrate: steps >= 1");
  Context::Impl& I = ctx.impl();
  const SchedulePlan plan = schedule_oases(graph);
  const double half_bytes =
      static_cast<double>(spec.global_batch / 2) * spec.seq_len * spec.hidden_size * spec.bytes_per_element;
  std::vector<MeasuredRow> rows;
  for (int d : degrees) {
    if (d < 1) throw ConfigError("calibrate: degrees must be positive");
    // one rank's shard of a d-way group on this context's device, collectives skipped
    ContextOptions o;
    o.tp = d;
    o.device = I.opts.device;
    o.comm_disabled = d > 1;
    const std::unique_ptr<oases::Context> rc = oases::make_context(to_desc(o));
    oases::Stack stack(*rc, to_cfg(spec, opts));
    stack.init_random(opts.seed);
    if (graph.block_count() != stack.num_blocks())
      throw ConfigError("calibrate: graph and spec disagree on the number of blocks");
    oases::Executor ex(stack, plan);
    ex.step(false);  // warm-up
    std::map<int, std::vector<double>> fwd, bwd;
    for (int it = 0; it < steps; ++it) {
      const SimResult r = ex.step(true);
      std::map<std::tuple<int, int, int>, double> per;  // (block, sb, pass) -> seconds
      for (const TraceEvent& ev : r.trace) {
        if (ev.op_id >= plan.total_ops()) continue;
        const ScheduledOp& op = plan.op(ev.op_id);
        if (is_comm(op.kind)) continue;
        per[std::make_tuple(op.block, op.sub_batch, static_cast<int>(op.pass))] += ev.end - ev.start;
      }
      for (int b = 0; b < stack.num_blocks(); ++b)
        for (int sb = 0; sb < 2; ++sb) {
          auto f = per.find(std::make_tuple(b, sb, static_cast<int>(Pass::Forward)));
          if (f != per.end()) fwd[b].push_back(f->second);
          auto bw = per.find(std::make_tuple(b, sb, static_cast<int>(Pass::Backward)));
          auto rc2 = per.find(std::make_tuple(b, sb, static_cast<int>(Pass::Recompute)));
          if (bw != per.end()) bwd[b].push_back(bw->second + (rc2 != per.end() ? rc2->second : 0.0));
        }
    }
    double c = 0.0;
    if (d > 1) {
      const bool own = (I.opts.tp == d) && (I.ctx->nccl || I.ctx->local_workers == d) && !I.opts.comm_disabled;
      c = own ? allreduce_seconds(ctx, half_bytes, spec.bytes_per_element)
              : comm_time(allreduce_volume(half_bytes, d), d, b200_profile(std::max(d, 2)));
    }
    auto median = [](std::vector<double> v) {
      std::sort(v.begin(), v.end());
      return v.empty() ? 0.0 : v[v.size() / 2];
    };
    for (int b = 0; b < stack.num_blocks(); ++b) {
      const std::pair<const char*, double> vals[] = {{"d_fwd", median(fwd[b])}, {"d_bwd", median(bwd[b])},
                                                     {"c_fwd", c},          {"c_bwd", c},
                                                     {"m_saved", 2 * half_bytes}};
      for (const auto& [field, v] : vals) rows.push_back(MeasuredRow{b, d, field, v});
    }
  }
  return rows;
}

}  // namespace tmpsim
