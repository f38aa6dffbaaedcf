// Plan executor: a tmpsim::SchedulePlan becomes kernels on the compute stream
// and AllReduces on the comm stream. Every cross-stream plan dependency --
// data edges AND the weave gates of Alg. 1 (the host `Sync(handler)`,
// PAPER.md:239-240) -- becomes a cudaStreamWaitEvent, never a host sync, so
// one sub-batch's AllReduce runs under the other sub-batch's GEMMs.
//
// The measured step is reported in the reference's SimResult shape
// (sim.hpp:13-26): per-op cudaEvent intervals, makespan, compute-busy
// fraction, exposed communication by the same interval algebra as
// simulate() (sim.cpp:178-199), and the device bytes of the stack.
#include <algorithm>
#include <cstdlib>
#include <deque>
#include <map>
#include <set>

#include "stack.h"
#include "status.h"

namespace oases {

using tmpsim::ConfigError;
using tmpsim::OpKind;
using tmpsim::Pass;

namespace {

// validate_plan (schedule.cpp:470-521) accepts graphs with several compute ops
// per block (custom operator sequences); this executor maps ONE plan op to a
// block's whole kernel list and shares activation workspaces between blocks, so
// it also needs:
//  * exactly one forward, (recompute,) backward compute op per (block, sub-batch)
//    and at most one comm op per (pass, block, sub-batch);
//  * the second backward op of a block (which computes the weight gradients over
//    both sub-batches) directly follows the first among backward computes (the
//    per-sub-batch gradient scratch is shared by all blocks), and
//  * every backward op finds its block's forward/recompute activations still in
//    the workspace slot they were written to (slot = block % 2 with recompute).
// A plan that breaks these would run and produce wrong gradients, so it is
// rejected with ConfigError instead.
void check_buffer_discipline(const tmpsim::SchedulePlan& plan, int nblocks, bool recompute) {
  const int n = plan.total_ops();
  const int halves = plan.split_batch ? 2 : 1;
  std::map<std::tuple<int, int, int>, int> ncomp, ncomm;
  for (int id = 0; id < n; ++id) {
    const auto& op = plan.op(id);
    if (op.block < 0 || op.block >= nblocks) throw ConfigError("plan_bind: op " + std::to_string(id) + " block out of range");
    if (!plan.split_batch && op.sub_batch != 0)
      throw ConfigError("plan_bind: unsplit plan with sub_batch != 0 at op " + std::to_string(id));
    auto key = std::make_tuple(static_cast<int>(op.pass), op.block, op.sub_batch);
    if (tmpsim::is_comm(op.kind)) {
      if (++ncomm[key] > 1)
        throw ConfigError("plan_bind: more than one comm op for (pass, block " + std::to_string(op.block) +
                          ", sub-batch " + std::to_string(op.sub_batch) + ")");
    } else if (++ncomp[key] > 1) {
      throw ConfigError("plan_bind: more than one compute op for (pass, block " + std::to_string(op.block) +
                        ", sub-batch " + std::to_string(op.sub_batch) + "); the executor runs one kernel list per block");
    }
  }
  std::vector<Pass> passes = {Pass::Forward, Pass::Backward};
  if (plan.has_recompute) passes.push_back(Pass::Recompute);
  for (int b = 0; b < nblocks; ++b)
    for (Pass p : passes)
      for (int sb = 0; sb < halves; ++sb)
        if (!ncomp.count(std::make_tuple(static_cast<int>(p), b, sb)))
          throw ConfigError("plan_bind: block " + std::to_string(b) + " lacks a " + tmpsim::to_string(p) +
                            " compute op for sub-batch " + std::to_string(sb));
  // workspace ownership walk in compute-stream issue order
  std::map<std::pair<int, int>, int> owner;  // (slot, sb) -> block whose activations it holds
  auto slot = [&](int b) { return recompute ? b % 2 : b; };
  int prev_b = -1, prev_block = -1;
  std::vector<int> seen(static_cast<size_t>(nblocks), 0);
  for (int id = 0; id < n; ++id) {
    const auto& op = plan.op(id);
    if (tmpsim::is_comm(op.kind)) continue;
    if (op.kind == OpKind::ForwardCompute || op.kind == OpKind::RecomputeCompute) {
      // forward ops of a recompute plan only feed their own row GEMM (the saved x_b is
      // separate); the recompute op (or, without recompute, the forward) fills the slot
      if (op.kind == OpKind::RecomputeCompute || !plan.has_recompute)
        for (int sb = 0; sb < 2; ++sb)
          if (halves == 2 ? sb == op.sub_batch : true) owner[{slot(op.block), sb}] = op.block;
      if (op.kind == OpKind::ForwardCompute && plan.has_recompute)
        for (int sb = 0; sb < 2; ++sb)
          if (halves == 2 ? sb == op.sub_batch : true) owner[{slot(op.block), sb}] = -1 - op.block;
      continue;
    }
    // backward compute
    const int b = op.block;
    const int k = ++seen[static_cast<size_t>(b)];
    auto holds = [&](int sb) {
      auto it = owner.find({slot(b), sb});
      return it != owner.end() && it->second == b;
    };
    const bool ok = halves == 1 ? holds(0) && holds(1)
                                : (k == 1 ? holds(op.sub_batch) : holds(0) && holds(1) && prev_b == id && prev_block == b);
    if (!ok)
      throw ConfigError("plan_bind: backward op " + std::to_string(id) + " of block " + std::to_string(b) +
                        " would read activations or gradient scratch overwritten by another block (the two "
                        "backward ops of a block must follow each other and their recompute)");
    // the next backward op must be this block's second one when the plan is split
    prev_b = -1;
    prev_block = -1;
    if (halves == 2 && k == 1) {
      for (int j = id + 1; j < n; ++j)
        if (plan.op(j).kind == OpKind::BackwardCompute) {
          prev_b = j;
          prev_block = b;
          break;
        }
    }
  }
}

}  // namespace

Executor::Executor(Stack& stack, const tmpsim::SchedulePlan& plan) : stack_(stack), plan_(plan) {
  const auto bad = tmpsim::validate_plan(plan);
  if (!bad.empty()) throw ConfigError("plan_bind: invalid plan: " + bad.front().code + ": " + bad.front().detail);
  if (plan.has_recompute != stack.cfg().recompute)
    throw ConfigError("plan_bind: plan.has_recompute must match the stack's recompute_enabled");
  const int n = plan.total_ops();
  int max_block = -1;
  std::set<std::pair<int, int>> rec_comm;
  for (int id = 0; id < n; ++id) {
    const auto& op = plan.op(id);
    max_block = std::max(max_block, op.block);
    if (op.kind == OpKind::AllGather)
      throw ConfigError("plan_bind: AllGather ops are injected from the stack's per-block degrees, not planned");
    if (tmpsim::is_comm(op.kind) && op.pass == Pass::Recompute) rec_comm.emplace(op.block, op.sub_batch);
  }
  if (max_block + 1 != stack.num_blocks())
    throw ConfigError("plan_bind: plan has " + std::to_string(max_block + 1) + " blocks, stack has " +
                      std::to_string(stack.num_blocks()));
  check_buffer_discipline(plan, stack.num_blocks(), stack.cfg().recompute);
  // WAR protection: a compute op that writes an AllReduce buffer waits for the
  // last comm op that used the same buffer (the plan's data edges cover RAW).
  std::map<std::tuple<int, int, int>, int> last_comm_on;
  auto buf_key = [](Pass p, int block, int sb) { return std::make_tuple(static_cast<int>(p), block % 2, sb); };
  ops_.reserve(static_cast<size_t>(n));
  for (int id = 0; id < n; ++id) {
    const auto& op = plan.op(id);
    ExecOp e;
    e.id = id;
    e.kind = op.kind;
    e.pass = op.pass;
    e.stream = op.stream == tmpsim::Stream::Comm ? 1 : 0;
    e.block = op.block;
    e.sb = op.sub_batch;
    e.both_halves = !plan.split_batch;
    if (op.kind == OpKind::RecomputeCompute) {
      e.with_row = rec_comm.count({op.block, op.sub_batch}) > 0;
      for (int d : op.deps) {
        const auto& dop = plan.op(d);
        if (tmpsim::is_comm(dop.kind) && dop.pass == Pass::Recompute) e.rebuild_x = true;
      }
    }
    std::set<int> waits;
    for (int d : op.deps) {
      const int ds = plan.op(d).stream == tmpsim::Stream::Comm ? 1 : 0;
      if (ds != e.stream) waits.insert(d);
    }
    if (e.stream == 0) {
      const bool writes = op.kind == OpKind::ForwardCompute || op.kind == OpKind::BackwardCompute ||
                          (op.kind == OpKind::RecomputeCompute && e.with_row);
      if (writes) {
        auto it = last_comm_on.find(buf_key(op.pass, op.block, op.sub_batch));
        if (it != last_comm_on.end()) waits.insert(it->second);
      }
    } else {
      last_comm_on[buf_key(op.pass, op.block, op.sub_batch)] = id;
    }
    e.waits.assign(waits.begin(), waits.end());
    ops_.push_back(std::move(e));
  }
  if (stack.mixed()) inject_reshards(n);
  // Residual-stream storage: x_b stays in its own HBM buffer unless the plan
  // rebuilds it from a replayed AllReduce (interior of a CrossPass unit).
  {
    std::vector<bool> stored(static_cast<size_t>(stack.num_blocks()), true);
    for (const ExecOp& e : ops_)
      if (e.kind == OpKind::RecomputeCompute && e.rebuild_x) stored[static_cast<size_t>(e.block)] = false;
    stack.bind_storage(stored);
  }
  // LN_0 backward tail: after the last backward comm (or compute) of block 0.
  for (int id = 0; id < n; ++id) {
    const auto& op = plan.op(id);
    if (op.pass == Pass::Backward && op.block == 0) tail_wait_[static_cast<size_t>(op.sub_batch)] = id;
  }
  stream_of_.assign(static_cast<size_t>(n + nreshard_), 0);
  for (const ExecOp& e : ops_) stream_of_[static_cast<size_t>(e.id)] = e.stream;
  const int nev = n + nreshard_ + 2;
  t0_.resize(static_cast<size_t>(nev));
  t1_.resize(static_cast<size_t>(nev));
  for (int i = 0; i < nev; ++i) {
    check_cuda(cudaEventCreate(&t0_[static_cast<size_t>(i)]), "event");
    check_cuda(cudaEventCreate(&t1_[static_cast<size_t>(i)]), "event");
  }
  check_cuda(cudaEventCreate(&begin_), "event");
  check_cuda(cudaEventCreate(&end_), "event");
  check_cuda(cudaEventCreateWithFlags(&fork_, cudaEventDisableTiming), "event");
}

void Executor::inject_reshards(int n) {
  const int B = stack_.num_blocks();
  std::vector<int> last_fwd_comm(static_cast<size_t>(B), -1), last_bwd_comm(static_cast<size_t>(B), -1),
      last_bwd_compute(static_cast<size_t>(B), -1);
  std::vector<std::array<int, 2>> first_fwd(static_cast<size_t>(B), {-1, -1}), first_bwd(static_cast<size_t>(B), {-1, -1});
  for (int id = 0; id < n; ++id) {
    const auto& op = plan_.op(id);
    const size_t b = static_cast<size_t>(op.block), sb = static_cast<size_t>(op.sub_batch);
    if (op.pass == Pass::Forward) {
      if (tmpsim::is_comm(op.kind)) last_fwd_comm[b] = id;
      if (op.kind == OpKind::ForwardCompute && first_fwd[b][sb] < 0) first_fwd[b][sb] = id;
    } else if (op.pass == Pass::Backward) {
      if (tmpsim::is_comm(op.kind)) last_bwd_comm[b] = id;
      if (op.kind == OpKind::BackwardCompute) {
        last_bwd_compute[b] = id;
        if (first_bwd[b][sb] < 0) first_bwd[b][sb] = id;
      }
    }
  }
  for (const ExecOp& e : ops_)
    if (e.kind == OpKind::RecomputeCompute && e.rebuild_x && e.block > 0 &&
        stack_.degree(e.block) != stack_.degree(e.block - 1))
      throw ConfigError("plan_bind: the recompute of block " + std::to_string(e.block) +
                        " rebuilds x_b from a replayed AllReduce across a degree change (keep x_b: an Oases or "
                        "policy plan storing it)");
  struct Reshard {
    int after;
    std::array<int, 2> gates;
    bool fwd;
    int block;  // v (forward) or u (backward)
  };
  std::vector<Reshard> rs;
  for (int v = 0; v + 1 < B; ++v) {
    const int u = v + 1, dv = stack_.degree(v), du = stack_.degree(u);
    if (dv == du) continue;
    if (dv < du) {
      if (last_fwd_comm[static_cast<size_t>(v)] >= 0)
        rs.push_back({last_fwd_comm[static_cast<size_t>(v)], first_fwd[static_cast<size_t>(u)], true, v});
    } else {
      const int anchor = last_bwd_comm[static_cast<size_t>(u)] >= 0 ? last_bwd_comm[static_cast<size_t>(u)]
                                                                     : last_bwd_compute[static_cast<size_t>(u)];
      if (anchor >= 0) rs.push_back({anchor, first_bwd[static_cast<size_t>(v)], false, u});
    }
  }
  nreshard_ = static_cast<int>(rs.size());
  if (rs.empty()) return;
  std::map<int, size_t> pos;  // plan id -> index in ops_
  for (size_t i = 0; i < ops_.size(); ++i) pos[ops_[i].id] = i;
  std::vector<std::vector<ExecOp>> after(ops_.size());
  for (int r = 0; r < nreshard_; ++r) {
    const Reshard& x = rs[static_cast<size_t>(r)];
    ExecOp e;
    e.id = n + r;
    e.kind = OpKind::AllGather;
    e.pass = x.fwd ? Pass::Forward : Pass::Backward;
    e.stream = 1;
    e.block = x.block;
    if (ops_[pos[x.after]].stream == 0) e.waits.push_back(x.after);  // comm anchors: same stream, in order
    after[pos[x.after]].push_back(e);
    for (int g : x.gates) {
      if (g < 0) continue;
      ExecOp& go = ops_[pos[g]];
      go.waits.push_back(n + r);
    }
    // F_u builds no x_u of its own; B_v starts from the gathered gradient
    for (ExecOp& o : ops_) {
      if (x.fwd && o.kind == OpKind::ForwardCompute && o.block == x.block + 1) o.with_bdr = false;
      if (!x.fwd && o.kind == OpKind::BackwardCompute && o.block == x.block - 1) o.g_ready = true;
    }
  }
  std::vector<ExecOp> merged;
  for (size_t i = 0; i < ops_.size(); ++i) {
    merged.push_back(ops_[i]);
    for (ExecOp& e : after[i]) merged.push_back(e);
  }
  // Host issue order: a gated compute op can precede its AllGather's anchor in
  // plan order (F_u^0 before AR_v^1 in the weave), and a stream wait needs the
  // event recorded first. Re-interleave the two streams' in-order queues,
  // taking at each step the earliest head whose waits are already issued; the
  // order WITHIN each stream is the plan's.
  std::deque<ExecOp> q[2];
  for (size_t i = 0; i < merged.size(); ++i) {
    merged[i].seq = static_cast<int>(i);
    q[merged[i].stream].push_back(std::move(merged[i]));
  }
  std::set<int> issued;
  ops_.clear();
  auto ready = [&](const ExecOp& e) {
    for (int d : e.waits)
      if (!issued.count(d)) return false;
    return true;
  };
  while (!q[0].empty() || !q[1].empty()) {
    int pick = -1;
    for (int st = 0; st < 2; ++st)
      if (!q[st].empty() && ready(q[st].front()) &&
          (pick < 0 || q[st].front().seq < q[pick].front().seq))
        pick = st;
    if (pick < 0) throw ConfigError("plan_bind: the resharding AllGathers make the stream dependencies cyclic");
    issued.insert(q[pick].front().id);
    ops_.push_back(std::move(q[pick].front()));
    q[pick].pop_front();
  }
}

Executor::~Executor() {
  if (graph_exec_) cudaGraphExecDestroy(graph_exec_);
  if (graph_) cudaGraphDestroy(graph_);
  for (auto e : t0_) cudaEventDestroy(e);
  for (auto e : t1_) cudaEventDestroy(e);
  if (begin_) cudaEventDestroy(begin_);
  if (end_) cudaEventDestroy(end_);
  if (fork_) cudaEventDestroy(fork_);
}

void Executor::issue(bool trace) {
  Context& c = stack_.ctx();
  check_cuda(cudaEventRecord(begin_, c.compute), "record");
  check_cuda(cudaStreamWaitEvent(c.comm, begin_, 0), "fork");
  stack_.begin_step();
  const int W = stack_.num_workers();
  for (const ExecOp& op : ops_) {
    cudaStream_t s = op.stream ? c.comm : c.compute;
    for (int d : op.waits) check_cuda(cudaStreamWaitEvent(s, t1_[static_cast<size_t>(d)], 0), "wait");
    if (trace) check_cuda(cudaEventRecord(t0_[static_cast<size_t>(op.id)], s), "record");
    if (op.kind == OpKind::AllGather) {
      if (op.pass == Pass::Forward) stack_.reshard_fwd(op.block);
      else stack_.reshard_bwd(op.block);
    } else if (op.stream == 1) {
      stack_.allreduce(op.pass, op.block, op.sb, op.both_halves);
    } else {
      const int sb0 = op.both_halves ? 0 : op.sb, sb1 = op.both_halves ? 1 : op.sb;
      for (int w = 0; w < W; ++w) {
        for (int sb = sb0; sb <= sb1; ++sb) {
          switch (op.kind) {
            case OpKind::ForwardCompute: stack_.forward(w, op.block, sb, op.with_bdr, true); break;
            case OpKind::RecomputeCompute: stack_.recompute(w, op.block, sb, op.rebuild_x, op.with_row); break;
            case OpKind::BackwardCompute: stack_.backward(w, op.block, sb, op.g_ready); break;
            default: break;
          }
        }
      }
    }
    check_cuda(cudaEventRecord(t1_[static_cast<size_t>(op.id)], s), "record");
  }
  const int n = static_cast<int>(ops_.size());  // plan ops + injected reshards
  for (int k = 0; k < 2; ++k) {
    const int wait = plan_.split_batch ? tail_wait_[static_cast<size_t>(k)] : tail_wait_[0];
    if (wait >= 0 && stream_of_[static_cast<size_t>(wait)] == 1)
      check_cuda(cudaStreamWaitEvent(c.compute, t1_[static_cast<size_t>(wait)], 0), "wait tail");
    if (trace) check_cuda(cudaEventRecord(t0_[static_cast<size_t>(n + k)], c.compute), "record");
    if (stack_.num_blocks() > 0)  // an empty stack has no LN_0 to run backward through
      for (int w = 0; w < W; ++w) stack_.tail(w, k);
    check_cuda(cudaEventRecord(t1_[static_cast<size_t>(n + k)], c.compute), "record");
  }
  if (stack_.mixed()) {
    // data-parallel gradient sums of the blocks below the world degree
    check_cuda(cudaEventRecord(fork_, c.compute), "record");
    check_cuda(cudaStreamWaitEvent(c.comm, fork_, 0), "fork");
    stack_.dp_reduce_grads();
  }
  check_cuda(cudaEventRecord(fork_, c.comm), "record");
  check_cuda(cudaStreamWaitEvent(c.compute, fork_, 0), "join");
  check_cuda(cudaEventRecord(end_, c.compute), "record");
}

bool Executor::capture_graph() {
  Context& c = stack_.ctx();
  if (graph_exec_) return true;
  check_cuda(cudaStreamSynchronize(c.compute), "sync");
  check_cuda(cudaStreamBeginCapture(c.compute, cudaStreamCaptureModeRelaxed), "begin capture");
  try {
    issue(false);
  } catch (...) {
    cudaGraph_t g = nullptr;
    cudaStreamEndCapture(c.compute, &g);
    if (g) cudaGraphDestroy(g);
    throw;
  }
  check_cuda(cudaStreamEndCapture(c.compute, &graph_), "end capture");
  // Keep the per-node stream priorities of the capture (comm stream highest)
  // instead of running every node at the launching stream's priority.
  const char* np = std::getenv("OASES_GRAPH_NODE_PRIO");
  const unsigned long long flags = (np && np[0] == '0') ? 0ull : static_cast<unsigned long long>(cudaGraphInstantiateFlagUseNodePriority);
  check_cuda(cudaGraphInstantiateWithFlags(&graph_exec_, graph_, flags), "instantiate");
  return true;
}

void Executor::timed_graph_replay() {
  Context& c = stack_.ctx();
  check_cuda(cudaStreamSynchronize(c.compute), "sync");
  stack_.set_kernel_timing(true);
  stack_.reset_kernel_stats();
  cudaGraph_t g = nullptr;
  cudaGraphExec_t ge = nullptr;
  check_cuda(cudaStreamBeginCapture(c.compute, cudaStreamCaptureModeRelaxed), "begin capture");
  try {
    issue(false);
  } catch (...) {
    cudaStreamEndCapture(c.compute, &g);
    if (g) cudaGraphDestroy(g);
    stack_.set_kernel_timing(false);
    throw;
  }
  stack_.set_kernel_timing(false);
  check_cuda(cudaStreamEndCapture(c.compute, &g), "end capture");
  check_cuda(cudaGraphInstantiateWithFlags(&ge, g, static_cast<unsigned long long>(cudaGraphInstantiateFlagUseNodePriority)),
             "instantiate");
  for (int rep = 0; rep < 2; ++rep) check_cuda(cudaGraphLaunch(ge, c.compute), "graph launch");
  check_cuda(cudaStreamSynchronize(c.compute), "sync");
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
}

tmpsim::SimResult Executor::step(bool trace) {
  Context& c = stack_.ctx();
  tmpsim::SimResult r;
  if (graph_exec_ && !trace) {
    check_cuda(cudaEventRecord(begin_, c.compute), "record");
    check_cuda(cudaGraphLaunch(graph_exec_, c.compute), "graph launch");
    check_cuda(cudaEventRecord(end_, c.compute), "record");
  } else {
    issue(trace);
  }
  check_cuda(cudaEventSynchronize(end_), "step sync");
  float ms = 0.f;
  check_cuda(cudaEventElapsedTime(&ms, begin_, end_), "elapsed");
  r.makespan = ms * 1e-3;
  r.peak_memory = static_cast<double>(stack_.device_bytes());
  events_.clear();
  if (trace) {
    std::vector<std::pair<double, double>> comp, comm;
    double busy = 0.0;
    const int n = static_cast<int>(ops_.size());
    for (int i = 0; i < n + 2; ++i) {
      float a = 0.f, b = 0.f;
      check_cuda(cudaEventElapsedTime(&a, begin_, t0_[static_cast<size_t>(i)]), "elapsed");
      check_cuda(cudaEventElapsedTime(&b, begin_, t1_[static_cast<size_t>(i)]), "elapsed");
      const int stream = i < n ? stream_of_[static_cast<size_t>(i)] : 0;
      const double s0 = a * 1e-3, s1 = std::max(a, b) * 1e-3;
      events_.push_back({i, stream, s0, s1});
      r.trace.push_back({i, stream ? tmpsim::Stream::Comm : tmpsim::Stream::Compute, s0, s1});
      if (stream) {
        // tp == 1 AllReduces are empty: they contribute no interval
        const Context& cx = stack_.ctx();
        if (!cx.comm_disabled && (cx.tp > 1 || cx.nccl)) comm.emplace_back(s0, s1);
      } else {
        comp.emplace_back(s0, s1);
        busy += s1 - s0;
      }
    }
    r.comm_exposed = tmpsim::exposed_comm_time(comp, comm);
    r.compute_busy_fraction = r.makespan > 0.0 ? busy / r.makespan : 0.0;
  }
  return r;
}

}  // namespace oases
