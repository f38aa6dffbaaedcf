// Schedule construction: the issue order and cross-stream dependencies the
// GPU executor honours (Algorithms 1 and 2 of the paper).
//
// Semantics are those of the reference's schedule module
// (proj/src/schedule.cpp:62-530) and are pinned op-for-op by
// tests/golden/plans.json (all four variants, L = 0..3, recompute on/off,
// generated from the reference itself) and by the reference's shipped golden
// plan proj/tests/golden/oases_l1_plan.json:
//   * two sub-batches alternate at every communication (Alg. 1 weave);
//   * every compute waits for the second-most-recently started
//     communication -- the host `Sync(handler)` of Alg. 1;
//   * Oases recomputation starts from the stored post-AllReduce tensor and
//     issues no collective (Eq. 1);
//   * CrossPass/IntraPass replay per-layer units including their AllReduces.
#include <algorithm>
#include <array>
#include <functional>
#include <set>

#include "json.hpp"
#include "oases/tmpsim.hpp"

namespace tmpsim {

const char* to_string(ScheduleVariant v) {
  static const char* names[] = {"Default", "IntraPass", "CrossPass", "Oases"};
  const int i = static_cast<int>(v);
  return (i >= 0 && i < 4) ? names[i] : "?";
}
const char* to_string(Stream s) { return s == Stream::Compute ? "Compute" : "Comm"; }
const char* to_string(Pass p) {
  static const char* names[] = {"Forward", "Recompute", "Backward"};
  const int i = static_cast<int>(p);
  return (i >= 0 && i < 3) ? names[i] : "?";
}
const char* to_string(OpKind k) {
  static const char* names[] = {"ForwardCompute", "RecomputeCompute", "BackwardCompute", "AllReduce", "AllGather"};
  const int i = static_cast<int>(k);
  return (i >= 0 && i < 5) ? names[i] : "?";
}

ScheduleVariant variant_from_string(const std::string& name) {
  for (ScheduleVariant v : {ScheduleVariant::Default, ScheduleVariant::IntraPass, ScheduleVariant::CrossPass,
                            ScheduleVariant::Oases}) {
    if (name == to_string(v)) return v;
  }
  throw ConfigError("unknown schedule variant '" + name + "'");
}

const ScheduledOp& SchedulePlan::op(int id) const {
  if (id < 0 || id >= total_ops()) throw ConfigError("plan op id out of range");
  const int nf = static_cast<int>(forward_ops.size());
  return id < nf ? forward_ops[static_cast<std::size_t>(id)] : backward_ops[static_cast<std::size_t>(id - nf)];
}

namespace {

// One program step: a compute of a block (in some pass) or its trailing comm.
struct Step {
  bool comm;
  OpKind kind;
  Pass pass;
  int block;
  int base_id;
};
using Program = std::vector<Step>;

constexpr int kNone = -1;
using PerSb = std::array<int, 2>;

// Per-layer replay units [first, last] (attention/FFN pair of one layer).
std::vector<std::pair<int, int>> layer_units(const ModelGraph& g) {
  std::vector<std::pair<int, int>> units;
  int prev_layer = -1;
  for (int b = 0; b < g.block_count(); ++b) {
    const int layer = g.blocks[static_cast<std::size_t>(b)].compute_ops.front().layer;
    if (!units.empty() && layer == prev_layer) units.back().second = b;
    else units.emplace_back(b, b);
    prev_layer = layer;
  }
  return units;
}

Program forward_steps(const ModelGraph& g) {
  Program p;
  for (const Block& blk : g.blocks) {
    for (const Operator& c : blk.compute_ops) p.push_back({false, OpKind::ForwardCompute, Pass::Forward, blk.index, c.id});
    if (blk.comm_op) p.push_back({true, blk.comm_op->kind, Pass::Forward, blk.index, blk.comm_op->id});
  }
  return p;
}

void add_recompute(const ModelGraph& g, int b, bool replay_comm, Program& p) {
  const Block& blk = g.blocks[static_cast<std::size_t>(b)];
  for (const Operator& c : blk.compute_ops) p.push_back({false, OpKind::RecomputeCompute, Pass::Recompute, b, c.id});
  if (replay_comm && blk.comm_op) p.push_back({true, blk.comm_op->kind, Pass::Recompute, b, blk.comm_op->id});
}

void add_backward(const ModelGraph& g, int b, Program& p) {
  const Block& blk = g.blocks[static_cast<std::size_t>(b)];
  for (auto it = blk.compute_ops.rbegin(); it != blk.compute_ops.rend(); ++it)
    p.push_back({false, OpKind::BackwardCompute, Pass::Backward, b, it->id});
  if (blk.comm_op) p.push_back({true, blk.comm_op->kind, Pass::Backward, b, blk.comm_op->id});
}

// Emits ScheduledOps and keeps the per-(pass, block, sub-batch) bookkeeping
// the dependency rules read.
class Emitter {
 public:
  Emitter(const ModelGraph& g, ScheduleVariant v, bool split) : graph_(g) {
    plan_.variant = v;
    plan_.split_batch = split;
    plan_.has_recompute = g.recompute_enabled;
    const auto n = static_cast<std::size_t>(g.block_count());
    for (int p = 0; p < 3; ++p) {
      comm_[p].assign(n, PerSb{kNone, kNone});
      last_[p].assign(n, PerSb{kNone, kNone});
    }
    fwd_ids_.assign(n, {});
  }

  SchedulePlan& plan() { return plan_; }
  int next_id() const { return next_; }
  int comm(Pass p, int b, int sb) const { return comm_[idx(p)][static_cast<std::size_t>(b)][static_cast<std::size_t>(sb)]; }
  int last(Pass p, int b, int sb) const { return last_[idx(p)][static_cast<std::size_t>(b)][static_cast<std::size_t>(sb)]; }
  const std::vector<int>& forward_ids(int b, int sb) const {
    return fwd_ids_[static_cast<std::size_t>(b)][static_cast<std::size_t>(sb)];
  }

  // The loss reduces over the whole batch: nothing in backward starts before
  // the forward phase (including its trailing comm) has drained.
  void enter_backward() {
    backward_ = true;
    started_.clear();
    for (const ScheduledOp& op : plan_.forward_ops) (op.stream == Stream::Comm ? join_comm_ : join_compute_) = op.id;
  }
  void reset_gate() { started_.clear(); }

  int emit(const Step& s, int sb, std::vector<int> deps) {
    ScheduledOp op;
    op.id = next_++;
    op.base_id = s.base_id;
    op.kind = s.kind;
    op.pass = s.pass;
    op.stream = s.comm ? Stream::Comm : Stream::Compute;
    op.blocking = s.kind == OpKind::AllGather;
    op.block = s.block;
    op.sub_batch = sb;
    if (backward_) {
      deps.push_back(join_compute_);
      deps.push_back(join_comm_);
    }
    std::set<int> uniq(deps.begin(), deps.end());
    uniq.erase(kNone);
    op.deps.assign(uniq.begin(), uniq.end());
    const auto b = static_cast<std::size_t>(s.block);
    const auto u = static_cast<std::size_t>(sb);
    if (s.comm) {
      started_.push_back(op.id);
      comm_[idx(s.pass)][b][u] = op.id;
    } else {
      last_[idx(s.pass)][b][u] = op.id;
      if (s.pass == Pass::Forward) fwd_ids_[b][u].push_back(op.id);
    }
    (backward_ ? plan_.backward_ops : plan_.forward_ops).push_back(std::move(op));
    return next_ - 1;
  }

  // Alg. 1: run one sub-batch until its next comm, start it, switch. Computes
  // are gated on the second-most-recently started comm.
  template <typename Deps>
  void weave(const Program& prog, int first_sb, const Deps& data_deps) {
    std::size_t pos[2] = {0, 0};
    int x = first_sb;
    while (pos[0] < prog.size() || pos[1] < prog.size()) {
      if (pos[x] >= prog.size()) {
        x ^= 1;
        continue;
      }
      const Step& s = prog[pos[x]++];
      std::vector<int> deps;
      data_deps(s, x, deps);
      if (!s.comm && started_.size() >= 2) deps.push_back(started_[started_.size() - 2]);
      emit(s, x, std::move(deps));
      if (s.comm) x ^= 1;
    }
  }

  // Default: one sub-batch, strictly serial.
  template <typename Deps>
  void serial(const Program& prog, const Deps& data_deps) {
    for (const Step& s : prog) {
      std::vector<int> deps;
      data_deps(s, 0, deps);
      if (next_ > 0) deps.push_back(next_ - 1);
      emit(s, 0, std::move(deps));
    }
  }

 private:
  static std::size_t idx(Pass p) { return static_cast<std::size_t>(p); }
  const ModelGraph& graph_;
  SchedulePlan plan_;
  int next_ = 0;
  bool backward_ = false;
  int join_compute_ = kNone, join_comm_ = kNone;
  std::vector<int> started_;
  std::vector<PerSb> comm_[3], last_[3];
  std::vector<std::array<std::vector<int>, 2>> fwd_ids_;
};

// Data dependencies common to every variant; `replay_source(b, sb)` names the
// op whose output a recompute of block b starts from.
struct DataDeps {
  const ModelGraph& g;
  const Emitter& e;
  std::function<int(int, int)> replay_source;

  void operator()(const Step& s, int sb, std::vector<int>& deps) const {
    const int b = s.block;
    switch (s.pass) {
      case Pass::Forward:
        if (s.comm) deps.push_back(e.last(Pass::Forward, b, sb));
        else if (b > 0) deps.push_back(e.comm(Pass::Forward, b - 1, sb));
        return;
      case Pass::Recompute:
        deps.push_back(s.comm ? e.last(Pass::Recompute, b, sb) : replay_source(b, sb));
        return;
      case Pass::Backward:
        if (s.comm) {
          deps.push_back(e.last(Pass::Backward, b, sb));
          return;
        }
        // incoming gradient: downstream block's backward comm, or this
        // sub-batch's own forward tail for the last block
        if (b + 1 < g.block_count()) {
          deps.push_back(e.comm(Pass::Backward, b + 1, sb));
        } else {
          const int tail = e.comm(Pass::Forward, b, sb);
          deps.push_back(tail != kNone ? tail : e.last(Pass::Forward, b, sb));
        }
        // activations: the replay if there was one, else the forward
        const int rec = e.last(Pass::Recompute, b, sb);
        deps.push_back(rec != kNone ? rec : e.last(Pass::Forward, b, sb));
        return;
    }
  }
};

void save_per_unit(Emitter& e, const std::vector<std::pair<int, int>>& units, int sub_batches) {
  for (const auto& [first, last] : units) {
    for (int sb = 0; sb < sub_batches; ++sb) {
      std::vector<int> seq;
      for (int b = first; b <= last; ++b) {
        const auto& ids = e.forward_ids(b, sb);
        seq.insert(seq.end(), ids.begin(), ids.end());
      }
      e.plan().saved_sequences.push_back(std::move(seq));
    }
  }
}

// `keep[u]` (per layer unit, Oases/CrossPass only): the unit's interior
// post-AllReduce tensors stay in HBM, so its recompute starts from them and
// replays no collective (Oases, Eq. 1); otherwise the unit is replayed from
// its input with the recompute AllReduces (CrossPass). All-true is Oases,
// all-false CrossPass; a mixed vector is the fine-grained memory policy
// (SURVEY.md 8(f) F4), built with the same weave and dependency rules.
SchedulePlan build_pipelined(const ModelGraph& g, ScheduleVariant v, const std::vector<bool>* keep_in = nullptr) {
  Emitter e(g, v, /*split=*/true);
  if (g.block_count() == 0) return e.plan();
  const bool rec = g.recompute_enabled;
  const auto units = layer_units(g);
  std::vector<bool> keep(units.size(), v == ScheduleVariant::Oases);
  if (keep_in) keep = *keep_in;
  std::vector<int> unit_of(static_cast<std::size_t>(g.block_count()));
  for (std::size_t u = 0; u < units.size(); ++u)
    for (int b = units[u].first; b <= units[u].second; ++b) unit_of[static_cast<std::size_t>(b)] = static_cast<int>(u);
  auto kept = [&](int b) { return static_cast<bool>(keep[static_cast<std::size_t>(unit_of[static_cast<std::size_t>(b)])]); };

  DataDeps deps{g, e, [&](int b, int sb) -> int {
                  const auto& unit = units[static_cast<std::size_t>(unit_of[static_cast<std::size_t>(b)])];
                  // stored post-AR tensor (kept unit, or the unit's own input)
                  if (kept(b) || b == unit.first) return b > 0 ? e.comm(Pass::Forward, b - 1, sb) : kNone;
                  return e.comm(Pass::Recompute, b - 1, sb);  // replayed comm inside the unit
                }};

  e.weave(forward_steps(g), 0, deps);
  if (rec) {
    for (std::size_t u = 0; u < units.size(); ++u) {
      if (keep[u]) {
        for (int b = units[u].first; b <= units[u].second; ++b)
          for (int sb = 0; sb < 2; ++sb) e.plan().saved_sequences.push_back(e.forward_ids(b, sb));
      } else {
        save_per_unit(e, {units[u]}, 2);
      }
    }
  }

  e.enter_backward();
  if (keep_in || v == ScheduleVariant::Oases || v == ScheduleVariant::CrossPass || !rec) {
    Program bwd;
    for (auto it = units.rbegin(); it != units.rend(); ++it) {
      if (!rec) {
        for (int b = it->second; b >= it->first; --b) add_backward(g, b, bwd);
      } else if (kept(it->first)) {
        for (int b = it->second; b >= it->first; --b) {
          add_recompute(g, b, /*replay_comm=*/false, bwd);
          add_backward(g, b, bwd);
        }
      } else {
        for (int b = it->first; b <= it->second; ++b) add_recompute(g, b, true, bwd);
        for (int b = it->second; b >= it->first; --b) add_backward(g, b, bwd);
      }
    }
    e.weave(bwd, 1, deps);
    return e.plan();
  }

  // IntraPass: each recompute pass and each backward pass is pipelined on its
  // own; a barrier (deps on every op of the previous pass) joins them.
  std::vector<int> prev;
  auto run = [&](const Program& prog) {
    const int begin = e.next_id();
    e.reset_gate();
    auto gated = [&](const Step& s, int sb, std::vector<int>& d) {
      deps(s, sb, d);
      d.insert(d.end(), prev.begin(), prev.end());
    };
    e.weave(prog, 1, gated);
    prev.clear();
    for (int id = begin; id < e.next_id(); ++id) prev.push_back(id);
  };
  for (auto it = units.rbegin(); it != units.rend(); ++it) {
    Program rp, bp;
    for (int b = it->first; b <= it->second; ++b) add_recompute(g, b, true, rp);
    run(rp);
    for (int b = it->second; b >= it->first; --b) add_backward(g, b, bp);
    run(bp);
  }
  return e.plan();
}

}  // namespace

SchedulePlan schedule_default(const ModelGraph& g) {
  Emitter e(g, ScheduleVariant::Default, /*split=*/false);
  if (g.block_count() == 0) return e.plan();
  DataDeps deps{g, e, [&](int b, int) -> int { return b > 0 ? e.comm(Pass::Forward, b - 1, 0) : kNone; }};
  e.serial(forward_steps(g), deps);
  const auto units = layer_units(g);
  if (g.recompute_enabled) save_per_unit(e, units, 1);
  e.enter_backward();
  Program bwd;
  for (auto it = units.rbegin(); it != units.rend(); ++it) {
    if (g.recompute_enabled)
      for (int b = it->first; b <= it->second; ++b) add_recompute(g, b, true, bwd);
    for (int b = it->second; b >= it->first; --b) add_backward(g, b, bwd);
  }
  e.serial(bwd, deps);
  return e.plan();
}

SchedulePlan schedule_intra_pass(const ModelGraph& g) { return build_pipelined(g, ScheduleVariant::IntraPass); }
SchedulePlan schedule_cross_pass(const ModelGraph& g) { return build_pipelined(g, ScheduleVariant::CrossPass); }
SchedulePlan schedule_oases(const ModelGraph& g) { return build_pipelined(g, ScheduleVariant::Oases); }

SchedulePlan schedule_oases_policy(const ModelGraph& g, const std::vector<bool>& keep) {
  const auto units = layer_units(g);
  if (keep.size() != units.size())
    throw ConfigError("schedule_oases_policy: keep has " + std::to_string(keep.size()) + " entries, the model has " +
                      std::to_string(units.size()) + " layer units");
  const bool all = std::all_of(keep.begin(), keep.end(), [](bool k) { return k; });
  // a plan that replays any collective is labelled CrossPass (validate_plan
  // forbids recompute comms only in Oases plans)
  return build_pipelined(g, all ? ScheduleVariant::Oases : ScheduleVariant::CrossPass, &keep);
}

int layer_unit_count(const ModelGraph& g) { return static_cast<int>(layer_units(g).size()); }

SchedulePlan make_schedule(const ModelGraph& g, ScheduleVariant v) {
  switch (v) {
    case ScheduleVariant::Default: return schedule_default(g);
    case ScheduleVariant::IntraPass: return schedule_intra_pass(g);
    case ScheduleVariant::CrossPass: return schedule_cross_pass(g);
    case ScheduleVariant::Oases: return schedule_oases(g);
  }
  throw ConfigError("unknown schedule variant");
}

std::vector<Violation> validate_plan(const SchedulePlan& plan) {
  std::vector<Violation> out;
  const int n = plan.total_ops();
  std::set<std::pair<int, int>> produced_fwd, produced_rec;
  auto tag = [](int id) { return std::to_string(id); };
  for (int id = 0; id < n; ++id) {
    const ScheduledOp& op = plan.op(id);
    if (op.id != id) out.push_back({"id-order", "op at position " + tag(id) + " has id " + tag(op.id)});
    for (int d : op.deps) {
      if (d < 0 || d >= n) out.push_back({"dangling-dep", "op " + tag(id) + " depends on unknown id " + tag(d)});
      else if (d >= id)
        out.push_back({"cycle", "op " + tag(id) + " depends on op " + tag(d) + " that is not before it"});
    }
    const bool comm = is_comm(op.kind);
    if (comm != (op.stream == Stream::Comm)) out.push_back({"stream", "op " + tag(id) + " kind/stream mismatch"});
    if (op.kind == OpKind::AllGather && !op.blocking)
      out.push_back({"non-blocking-gather", "op " + tag(id) + " must stall both streams"});
    if (plan.variant == ScheduleVariant::Oases && comm && op.pass == Pass::Recompute)
      out.push_back({"recompute-comm", "op " + tag(id) + " replays a communication"});
    const auto key = std::make_pair(op.block, op.sub_batch);
    if (op.kind == OpKind::ForwardCompute) produced_fwd.insert(key);
    if (op.kind == OpKind::RecomputeCompute) produced_rec.insert(key);
    if (op.kind == OpKind::BackwardCompute) {
      const auto& pool = plan.has_recompute ? produced_rec : produced_fwd;
      if (!pool.count(key))
        out.push_back({"missing-producer", "backward op " + tag(id) + " on block " + tag(op.block) + " has no " +
                                               (plan.has_recompute ? "recompute" : "forward") + " producer"});
    }
  }
  return out;
}

int comm_op_count(const SchedulePlan& plan) {
  std::set<std::pair<int, int>> logical;
  for (int id = 0; id < plan.total_ops(); ++id) {
    const ScheduledOp& op = plan.op(id);
    if (is_comm(op.kind)) logical.emplace(op.base_id, static_cast<int>(op.pass));
  }
  return static_cast<int>(logical.size());
}

std::string plan_to_json_text(const SchedulePlan& plan, int indent) {
  using nlohmann::json;
  auto ops = [](const std::vector<ScheduledOp>& v) {
    json arr = json::array();
    for (const ScheduledOp& op : v) {
      arr.push_back({{"id", op.id},
                     {"base_id", op.base_id},
                     {"kind", to_string(op.kind)},
                     {"pass", to_string(op.pass)},
                     {"stream", to_string(op.stream)},
                     {"block", op.block},
                     {"sub_batch", op.sub_batch},
                     {"deps", op.deps}});
    }
    return arr;
  };
  json j = {{"variant", to_string(plan.variant)},
            {"split_batch", plan.split_batch},
            {"has_recompute", plan.has_recompute},
            {"forward_ops", ops(plan.forward_ops)},
            {"backward_ops", ops(plan.backward_ops)},
            {"saved_sequences", plan.saved_sequences}};
  return j.dump(indent);
}

}  // namespace tmpsim
