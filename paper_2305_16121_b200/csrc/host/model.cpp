// Layer -> operator sequence -> block chain (the unit the schedule, the
// planner and the GPU executor all index by).
//
// Behaviour follows the reference's model module (proj/src/model.cpp:19-120,
// SPEC.md "MODULE model"): per layer an attention compute (4H^2 params) and an
// FFN compute (8H^2), each followed by its AllReduce; blocks are maximal
// compute runs plus their trailing communication.
#include <string>

#include "oases/tmpsim.hpp"

namespace tmpsim {

bool is_compute(OpKind k) {
  switch (k) {
    case OpKind::ForwardCompute:
    case OpKind::RecomputeCompute:
    case OpKind::BackwardCompute:
      return true;
    default:
      return false;
  }
}

bool is_comm(OpKind k) { return k == OpKind::AllReduce || k == OpKind::AllGather; }

void ModelSpec::validate() const {
  struct Field {
    const char* name;
    long long value;
  };
  const Field positive[] = {{"hidden_size", hidden_size}, {"seq_len", seq_len}, {"attention_heads", attention_heads},
                            {"global_batch", global_batch}, {"bytes_per_element", bytes_per_element}};
  if (hidden_size <= 0) throw ConfigError("model spec: field 'hidden_size' must be positive");
  if (num_layers < 0) throw ConfigError("model spec: field 'num_layers' must be nonnegative");
  for (const Field& f : positive) {
    if (f.value <= 0) throw ConfigError(std::string("model spec: field '") + f.name + "' must be positive");
  }
  if (hidden_size % attention_heads != 0)
    throw ConfigError("model spec: 'hidden_size' must be divisible by 'attention_heads'");
  if (global_batch % 2 != 0)
    throw ConfigError("model spec: 'global_batch' must be even (the schedule splits it into two sub-batches)");
}

std::vector<Operator> build_operator_sequence(const ModelSpec& spec) {
  spec.validate();
  const std::int64_t h = spec.hidden_size;
  const std::int64_t boundary = static_cast<std::int64_t>(spec.seq_len) * h;
  std::vector<Operator> seq;
  seq.reserve(static_cast<std::size_t>(spec.num_layers) * 4);
  auto push = [&](OpKind kind, int layer, Sublayer sub, std::int64_t params) {
    Operator op;
    op.id = static_cast<int>(seq.size());
    op.kind = kind;
    op.layer = layer;
    op.sublayer = sub;
    op.param_count = params;
    op.tensor_elements = boundary;
    seq.push_back(op);
  };
  for (int layer = 0; layer < spec.num_layers; ++layer) {
    push(OpKind::ForwardCompute, layer, Sublayer::Attention, 4 * h * h);
    push(OpKind::AllReduce, layer, Sublayer::Attention, 0);
    push(OpKind::ForwardCompute, layer, Sublayer::Ffn, 8 * h * h);
    push(OpKind::AllReduce, layer, Sublayer::Ffn, 0);
  }
  return seq;
}

std::vector<Operator> build_ffn_sequence(const ModelSpec& spec) {
  spec.validate();
  std::vector<Operator> seq;
  const std::int64_t h = spec.hidden_size;
  for (int layer = 0; layer < spec.num_layers; ++layer) {
    for (OpKind kind : {OpKind::ForwardCompute, OpKind::AllReduce}) {
      Operator op;
      op.id = static_cast<int>(seq.size());
      op.kind = kind;
      op.layer = layer;
      op.sublayer = Sublayer::Ffn;
      op.param_count = kind == OpKind::ForwardCompute ? 8 * h * h : 0;
      op.tensor_elements = static_cast<std::int64_t>(spec.seq_len) * h;
      seq.push_back(op);
    }
  }
  return seq;
}

ModelGraph build_block_graph(const std::vector<Operator>& ops) {
  ModelGraph g;
  std::vector<Operator> pending;
  auto close = [&](const Operator* comm) {
    Block blk;
    blk.index = g.block_count();
    blk.compute_ops = std::move(pending);
    pending.clear();
    for (const Operator& c : blk.compute_ops) blk.param_count += c.param_count;
    if (comm) {
      blk.comm_op = *comm;
      blk.comm_op->blocking = comm->kind == OpKind::AllGather;
      blk.activation_elements = comm->tensor_elements;
    } else {
      blk.activation_elements = blk.compute_ops.back().tensor_elements;
    }
    g.blocks.push_back(std::move(blk));
  };
  for (const Operator& op : ops) {
    if (!is_comm(op.kind)) {
      pending.push_back(op);
      continue;
    }
    // A communication must close a non-empty compute run (no leading comm, no
    // two comms in a row).
    if (pending.empty())
      throw ConfigError("block graph: adjacent communication operators at op id " + std::to_string(op.id));
    close(&op);
  }
  if (!pending.empty()) close(nullptr);
  for (int i = 0; i + 1 < g.block_count(); ++i) g.edges.emplace_back(i, i + 1);
  return g;
}

ModelGraph build_block_graph(const std::vector<Operator>& ops, const ModelSpec& spec) {
  ModelGraph g = build_block_graph(ops);
  g.recompute_enabled = spec.recompute_enabled;
  return g;
}

std::vector<Operator> flatten(const ModelGraph& graph) {
  std::vector<Operator> out;
  for (const Block& b : graph.blocks) {
    out.insert(out.end(), b.compute_ops.begin(), b.compute_ops.end());
    if (b.comm_op) out.push_back(*b.comm_op);
  }
  return out;
}

}  // namespace tmpsim
