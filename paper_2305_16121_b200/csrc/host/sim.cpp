// Two-stream timing model of a plan, and the exposed-communication metric.
//
// `simulate` predicts what the GPU executor (runtime/executor.cpp) measures:
// same plan, same two streams, same metric definitions. It follows the
// reference's list scheduler (proj/src/sim.cpp:44-380): per-op durations from
// CostVectors (forward/recompute d_fwd split over the block's computes,
// backward d_bwd minus d_fwd when it includes recompute, AR c_fwd/c_bwd, x2
// when the batch is not split), blocking resharding AllGathers injected
// between blocks of different degree, each free stream dispatching the first
// ready op in plan order, exposed comm by interval subtraction, and a peak
// memory sweep. Pinned against the reference by tests/golden/sim_cases.json.
#include <algorithm>
#include <array>
#include <cmath>
#include <limits>
#include <map>

#include "oases/tmpsim.hpp"

namespace tmpsim {

double exposed_comm_time(std::vector<std::pair<double, double>> compute,
                         std::vector<std::pair<double, double>> comm) {
  std::sort(compute.begin(), compute.end());
  std::sort(comm.begin(), comm.end());
  double exposed = 0.0;
  std::size_t c = 0;  // first compute interval that may still cover something
  for (const auto& [lo, hi] : comm) {
    double t = lo;
    while (t < hi) {
      while (c < compute.size() && compute[c].second <= t) ++c;
      if (c == compute.size() || compute[c].first >= hi) {
        exposed += hi - t;
        break;
      }
      if (compute[c].first > t) exposed += std::min(hi, compute[c].first) - t;
      t = std::max(t, compute[c].second);
    }
  }
  return exposed;
}

namespace {

struct Node {
  int trace_id = 0;
  int stream = 0;  // 0 compute, 1 comm
  bool blocking = false;
  double duration = 0.0;
  std::vector<int> deps;
};

struct Timeline {
  std::vector<Node> nodes;
  std::vector<int> node_of;  // plan id -> node index
};

double op_duration(const SchedulePlan& plan, const CostVectors& costs, const Strategy& st, const ScheduledOp& op,
                   const std::vector<int>& computes_per_block) {
  const double scale = plan.split_batch ? 1.0 : 2.0;
  const int slot = costs.degree_index(st.degrees[static_cast<std::size_t>(op.block)]);
  const BlockCosts& bc = costs.blocks[static_cast<std::size_t>(op.block)];
  const auto s = static_cast<std::size_t>(slot);
  const double per = static_cast<double>(computes_per_block[static_cast<std::size_t>(op.block)]);
  switch (op.kind) {
    case OpKind::ForwardCompute:
    case OpKind::RecomputeCompute:
      return scale * bc.d_fwd[s] / per;
    case OpKind::BackwardCompute: {
      double d = bc.d_bwd[s];
      if (plan.has_recompute && costs.backward_includes_recompute) d = std::max(0.0, d - bc.d_fwd[s]);
      return scale * d / per;
    }
    case OpKind::AllReduce:
      return scale * (op.pass == Pass::Backward ? bc.c_bwd[s] : bc.c_fwd[s]);
    case OpKind::AllGather:
      return scale * bc.c_fwd[s];
  }
  return 0.0;
}

Timeline lower(const SchedulePlan& plan, const CostVectors& costs, const Strategy& st) {
  const int n = plan.total_ops();
  const int nb = costs.block_count();
  std::vector<int> per_block(static_cast<std::size_t>(nb), 0);
  for (const ScheduledOp& op : plan.forward_ops)
    if (op.kind == OpKind::ForwardCompute && op.sub_batch == 0 && op.block < nb) ++per_block[static_cast<std::size_t>(op.block)];
  for (int& c : per_block) c = std::max(c, 1);

  // anchors for resharding insertion
  std::vector<int> fwd_comm_last(nb, -1), bwd_comm_last(nb, -1), bwd_compute_last(nb, -1);
  std::vector<std::array<int, 2>> fwd_first(nb, {-1, -1}), bwd_first(nb, {-1, -1});
  for (int id = 0; id < n; ++id) {
    const ScheduledOp& op = plan.op(id);
    const auto b = static_cast<std::size_t>(op.block);
    const auto sb = static_cast<std::size_t>(op.sub_batch);
    if (op.pass == Pass::Forward) {
      if (is_comm(op.kind)) fwd_comm_last[b] = id;
      if (op.kind == OpKind::ForwardCompute && fwd_first[b][sb] < 0) fwd_first[b][sb] = id;
    } else if (op.pass == Pass::Backward) {
      if (is_comm(op.kind)) bwd_comm_last[b] = id;
      if (op.kind == OpKind::BackwardCompute) {
        bwd_compute_last[b] = id;
        if (bwd_first[b][sb] < 0) bwd_first[b][sb] = id;
      }
    }
  }
  // A degree change between blocks v and v+1 costs an exclusive AllGather at
  // group max(dv, du): after the forward tail of v when growing, after the
  // backward tail of v+1 when shrinking; it gates both sub-batches' consumers.
  struct Reshard {
    int after;
    std::array<int, 2> gates;
    double duration;
  };
  std::vector<Reshard> rs;
  for (int v = 0; v + 1 < nb; ++v) {
    const int dv = st.degrees[static_cast<std::size_t>(v)], du = st.degrees[static_cast<std::size_t>(v + 1)];
    if (dv == du) continue;
    const double ag = costs.blocks[static_cast<std::size_t>(v)].allgather_time[static_cast<std::size_t>(
        costs.degree_index(std::max(dv, du)))];
    if (dv < du) {
      if (fwd_comm_last[static_cast<std::size_t>(v)] >= 0)
        rs.push_back({fwd_comm_last[static_cast<std::size_t>(v)], fwd_first[static_cast<std::size_t>(v + 1)], ag});
    } else {
      const int anchor = bwd_comm_last[static_cast<std::size_t>(v + 1)] >= 0
                             ? bwd_comm_last[static_cast<std::size_t>(v + 1)]
                             : bwd_compute_last[static_cast<std::size_t>(v + 1)];
      if (anchor >= 0) rs.push_back({anchor, bwd_first[static_cast<std::size_t>(v)], ag});
    }
  }
  std::map<int, std::vector<int>> after, gated;
  for (int r = 0; r < static_cast<int>(rs.size()); ++r) {
    after[rs[static_cast<std::size_t>(r)].after].push_back(r);
    for (int gte : rs[static_cast<std::size_t>(r)].gates)
      if (gte >= 0) gated[gte].push_back(r);
  }

  Timeline tl;
  tl.node_of.assign(static_cast<std::size_t>(n), -1);
  std::vector<int> rs_node(rs.size(), -1);
  for (int id = 0; id < n; ++id) {
    const ScheduledOp& op = plan.op(id);
    Node nd;
    nd.trace_id = id;
    nd.stream = op.stream == Stream::Comm ? 1 : 0;
    nd.blocking = op.blocking;
    nd.duration = op_duration(plan, costs, st, op, per_block);
    for (int d : op.deps) nd.deps.push_back(tl.node_of[static_cast<std::size_t>(d)]);
    if (auto it = gated.find(id); it != gated.end())
      for (int r : it->second)
        if (rs_node[static_cast<std::size_t>(r)] >= 0) nd.deps.push_back(rs_node[static_cast<std::size_t>(r)]);
    tl.node_of[static_cast<std::size_t>(id)] = static_cast<int>(tl.nodes.size());
    tl.nodes.push_back(std::move(nd));
    if (auto it = after.find(id); it != after.end()) {
      for (int r : it->second) {
        Node ag;
        ag.trace_id = n + r;
        ag.stream = 1;
        ag.blocking = true;
        ag.duration = rs[static_cast<std::size_t>(r)].duration;
        ag.deps.push_back(tl.node_of[static_cast<std::size_t>(id)]);
        rs_node[static_cast<std::size_t>(r)] = static_cast<int>(tl.nodes.size());
        tl.nodes.push_back(std::move(ag));
      }
    }
  }
  return tl;
}

}  // namespace

SimResult simulate(const SchedulePlan& plan, const CostVectors& costs, const Strategy& strategy, SimOptions options) {
  const auto bad = validate_plan(plan);
  if (!bad.empty()) throw ConfigError("simulate: invalid plan: " + bad.front().code + ": " + bad.front().detail);
  validate_strategy(strategy, costs);
  for (int id = 0; id < plan.total_ops(); ++id) {
    if (plan.op(id).block >= costs.block_count())
      throw ConfigError("simulate: plan references block " + std::to_string(plan.op(id).block) +
                        " with no cost entry");
  }
  SimResult result;
  if (plan.total_ops() == 0) return result;

  const Timeline tl = lower(plan, costs, strategy);
  const int n = static_cast<int>(tl.nodes.size());
  std::vector<double> start(static_cast<std::size_t>(n), -1.0), finish(static_cast<std::size_t>(n), -1.0);
  std::vector<char> issued(static_cast<std::size_t>(n), 0);
  std::vector<int> queue[2];
  for (int i = 0; i < n; ++i) queue[tl.nodes[static_cast<std::size_t>(i)].stream].push_back(i);
  std::size_t head[2] = {0, 0};
  double busy_until[2] = {0.0, 0.0};
  double now = 0.0;
  int left = n;

  auto ready = [&](int i) {
    for (int d : tl.nodes[static_cast<std::size_t>(i)].deps) {
      const double f = finish[static_cast<std::size_t>(d)];
      if (f < 0.0 || f > now) return false;
    }
    return true;
  };

  while (left > 0) {
    for (bool progress = true; progress;) {
      progress = false;
      for (int s = 0; s < 2; ++s) {
        if (busy_until[s] > now) continue;
        auto& q = queue[s];
        while (head[s] < q.size() && issued[static_cast<std::size_t>(q[head[s]])]) ++head[s];
        for (std::size_t k = head[s]; k < q.size(); ++k) {
          const int i = q[k];
          if (issued[static_cast<std::size_t>(i)] || !ready(i)) continue;
          const Node& nd = tl.nodes[static_cast<std::size_t>(i)];
          if (nd.blocking && busy_until[1 - s] > now) break;  // exclusive op waits at the head
          double dur = nd.duration;
          if (s == 1 && !nd.blocking && options.overlap_slowdown != 1.0 && busy_until[0] > now)
            dur *= options.overlap_slowdown;
          issued[static_cast<std::size_t>(i)] = 1;
          start[static_cast<std::size_t>(i)] = now;
          finish[static_cast<std::size_t>(i)] = now + dur;
          busy_until[s] = now + dur;
          if (nd.blocking) busy_until[1 - s] = now + dur;
          --left;
          progress = true;
          break;
        }
      }
    }
    if (left == 0) break;
    double next = std::numeric_limits<double>::infinity();
    for (int s = 0; s < 2; ++s)
      if (busy_until[s] > now) next = std::min(next, busy_until[s]);
    for (int i = 0; i < n; ++i)
      if (issued[static_cast<std::size_t>(i)] && finish[static_cast<std::size_t>(i)] > now)
        next = std::min(next, finish[static_cast<std::size_t>(i)]);
    if (!std::isfinite(next)) throw ConfigError("simulate: schedule deadlocked; plan dependencies are unsatisfiable");
    now = next;
  }

  std::vector<std::pair<double, double>> comp_iv, comm_iv;
  double makespan = 0.0, busy = 0.0;
  result.trace.reserve(static_cast<std::size_t>(n));
  for (int i = 0; i < n; ++i) {
    const Node& nd = tl.nodes[static_cast<std::size_t>(i)];
    const double s0 = start[static_cast<std::size_t>(i)], s1 = finish[static_cast<std::size_t>(i)];
    result.trace.push_back({nd.trace_id, nd.stream == 1 ? Stream::Comm : Stream::Compute, s0, s1});
    makespan = std::max(makespan, s1);
    if (nd.stream == 0) {
      busy += s1 - s0;
      comp_iv.emplace_back(s0, s1);
    } else {
      comm_iv.emplace_back(s0, s1);
    }
  }
  result.makespan = makespan;
  result.compute_busy_fraction = makespan > 0.0 ? busy / makespan : 0.0;
  result.comm_exposed = exposed_comm_time(comp_iv, comm_iv);

  // Memory: parameter state resident throughout; saved boundary tensors live
  // from their forward unit's start to the last backward of their blocks;
  // recompute/backward working sets are transient.
  double resident = 0.0;
  for (int b = 0; b < costs.block_count(); ++b)
    resident += costs.blocks[static_cast<std::size_t>(b)]
                    .m_param[static_cast<std::size_t>(costs.degree_index(strategy.degrees[static_cast<std::size_t>(b)]))];
  const double share = plan.split_batch ? 0.5 : 1.0;
  std::vector<std::pair<double, double>> events;
  std::map<std::pair<int, int>, double> bwd_done;
  auto slot_of = [&](int block) {
    return static_cast<std::size_t>(costs.degree_index(strategy.degrees[static_cast<std::size_t>(block)]));
  };
  for (int id = 0; id < plan.total_ops(); ++id) {
    const ScheduledOp& op = plan.op(id);
    const auto m = static_cast<std::size_t>(tl.node_of[static_cast<std::size_t>(id)]);
    if (op.kind == OpKind::BackwardCompute) {
      double& f = bwd_done[{op.block, op.sub_batch}];
      f = std::max(f, finish[m]);
    }
    if (op.kind == OpKind::BackwardCompute || op.kind == OpKind::RecomputeCompute) {
      const double r = share * costs.blocks[static_cast<std::size_t>(op.block)].m_runtime[slot_of(op.block)];
      events.emplace_back(start[m], r);
      events.emplace_back(finish[m], -r);
    }
  }
  auto keep_saved = [&](int block, int sb, double from, const std::vector<int>& blocks) {
    const double bytes = share * costs.blocks[static_cast<std::size_t>(block)].m_saved[slot_of(block)];
    double latest = -1.0;
    for (int blk : blocks)
      if (auto it = bwd_done.find({blk, sb}); it != bwd_done.end()) latest = std::max(latest, it->second);
    events.emplace_back(from, bytes);
    events.emplace_back(latest >= 0.0 ? latest : makespan, -bytes);
  };
  if (!plan.saved_sequences.empty()) {
    for (const auto& seq : plan.saved_sequences) {
      if (seq.empty()) continue;
      const ScheduledOp& first = plan.op(seq.front());
      std::vector<int> blocks;
      for (int id : seq) blocks.push_back(plan.op(id).block);
      keep_saved(first.block, first.sub_batch,
                 start[static_cast<std::size_t>(tl.node_of[static_cast<std::size_t>(seq.front())])], blocks);
    }
  } else {
    std::map<std::pair<int, int>, double> first_fwd;
    for (int id = 0; id < plan.total_ops(); ++id) {
      const ScheduledOp& op = plan.op(id);
      if (op.kind != OpKind::ForwardCompute) continue;
      const double t = start[static_cast<std::size_t>(tl.node_of[static_cast<std::size_t>(id)])];
      auto [it, fresh] = first_fwd.emplace(std::make_pair(op.block, op.sub_batch), t);
      if (!fresh) it->second = std::min(it->second, t);
    }
    for (const auto& [key, t] : first_fwd) keep_saved(key.first, key.second, t, {key.first});
  }
  std::sort(events.begin(), events.end());
  double mem = resident, peak = resident;
  for (const auto& [t, delta] : events) {
    (void)t;
    mem += delta;
    peak = std::max(peak, mem);
  }
  result.peak_memory = peak;
  return result;
}

Breakdown breakdown(const SimResult& r) {
  if (r.makespan <= 0.0) throw ConfigError("breakdown: zero makespan");
  Breakdown b;
  b.comm_fraction = r.comm_exposed / r.makespan;
  b.compute_fraction = r.compute_busy_fraction;
  b.idle_fraction = std::max(0.0, 1.0 - b.comm_fraction - b.compute_fraction);
  return b;
}

}  // namespace tmpsim
