// tmpsim-compatible C++ API of the B200 Oases build.
//
// Drop-in for the reference's host API on the TMP hot path (SURVEY.md §8(b),
// row B1): the same namespace, type names and fields as
// proj/include/tmpsim/{errors,model,costs,schedule,sim,planner}.hpp, so a
// caller of the reference recompiles against this header unchanged. The
// implementations are this repo's own (paper_2305_16121_b200/csrc/host/*).
// On top of the reference surface it adds the real-hardware entry points
// `execute` (measured SimResult) and `calibrate` (measured-cost rows), see
// include/oases/runtime.hpp.
#pragma once

#include <cstdint>
#include <filesystem>
#include <map>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace tmpsim {

// ------------------------------------------------------------- errors.hpp:11-26
class ConfigError : public std::runtime_error {
 public:
  explicit ConfigError(const std::string& w) : std::runtime_error(w) {}
};
class InfeasibleError : public std::runtime_error {
 public:
  explicit InfeasibleError(const std::string& w) : std::runtime_error(w) {}
};
class IoError : public std::runtime_error {
 public:
  explicit IoError(const std::string& w) : std::runtime_error(w) {}
};
// B200 extension: a CUDA or NCCL failure (no device, launch error, collective
// error). The runtime has no CPU fallback, so value-level and execution entry
// points raise this instead of silently computing on the host.
class DeviceError : public std::runtime_error {
 public:
  explicit DeviceError(const std::string& w) : std::runtime_error(w) {}
};

// ------------------------------------------------------------- model.hpp:13-84
enum class OpKind { ForwardCompute, RecomputeCompute, BackwardCompute, AllReduce, AllGather };
enum class Sublayer { Attention, Ffn };

bool is_compute(OpKind k);
bool is_comm(OpKind k);

struct ModelSpec {
  int hidden_size = 0;
  int num_layers = 0;
  int seq_len = 0;
  int attention_heads = 0;
  int global_batch = 0;
  int bytes_per_element = 2;
  bool recompute_enabled = true;
  void validate() const;
};

struct Operator {
  int id = 0;
  OpKind kind = OpKind::ForwardCompute;
  int layer = 0;
  Sublayer sublayer = Sublayer::Attention;
  int sub_batch = 0;
  bool blocking = false;
  std::int64_t param_count = 0;
  std::int64_t tensor_elements = 0;
};

struct Block {
  int index = 0;
  std::vector<Operator> compute_ops;
  std::optional<Operator> comm_op;
  std::int64_t param_count = 0;
  std::int64_t activation_elements = 0;
};

struct ModelGraph {
  std::vector<Block> blocks;
  std::vector<std::pair<int, int>> edges;
  bool recompute_enabled = true;
  int block_count() const { return static_cast<int>(blocks.size()); }
};

std::vector<Operator> build_operator_sequence(const ModelSpec& spec);
// Extension: FFN-only layers (compute + AllReduce per layer) -- the shape of the
// reference's toy checker (numerics.hpp:37-44) as a block chain.
std::vector<Operator> build_ffn_sequence(const ModelSpec& spec);
ModelGraph build_block_graph(const std::vector<Operator>& ops);
ModelGraph build_block_graph(const std::vector<Operator>& ops, const ModelSpec& spec);
std::vector<Operator> flatten(const ModelGraph& graph);

// ------------------------------------------------------------- costs.hpp:15-73
struct HardwareProfile {
  int num_devices = 0;
  std::int64_t memory_capacity = 0;
  double compute_throughput = 0.0;
  std::map<int, double> bandwidth_by_group;
  std::map<int, double> latency_by_group;
  std::vector<int> candidate_degrees;
  double optimizer_bytes_per_element = 16.0;
  void validate() const;
};

struct Strategy {
  std::vector<int> degrees;
};

struct BlockCosts {
  std::vector<double> d_fwd, d_bwd, c_fwd, c_bwd, m_param, m_saved, m_runtime, allgather_time;
};

struct CostVectors {
  std::vector<int> degrees;
  std::vector<BlockCosts> blocks;
  std::vector<double> boundary_bytes_half;
  bool backward_includes_recompute = true;
  int degree_index(int degree) const;
  int block_count() const { return static_cast<int>(blocks.size()); }
};

double allreduce_volume(double message_bytes, int degree);
double allgather_volume(double message_bytes, int degree);
double comm_time(double volume_bytes, int degree, const HardwareProfile& profile);
CostVectors build_cost_vectors(const ModelGraph& graph, const ModelSpec& spec, const HardwareProfile& profile);
CostVectors load_measured_costs(const std::filesystem::path& path, CostVectors base);
void validate_strategy(const Strategy& strategy, const CostVectors& costs);

// ------------------------------------------------------------- schedule.hpp:14-78
enum class ScheduleVariant { Default, IntraPass, CrossPass, Oases };
enum class Stream { Compute, Comm };
enum class Pass { Forward, Recompute, Backward };

const char* to_string(ScheduleVariant v);
const char* to_string(Stream s);
const char* to_string(Pass p);
const char* to_string(OpKind k);
ScheduleVariant variant_from_string(const std::string& name);

struct ScheduledOp {
  int id = 0;
  int base_id = 0;
  OpKind kind = OpKind::ForwardCompute;
  Pass pass = Pass::Forward;
  Stream stream = Stream::Compute;
  int block = 0;
  int sub_batch = 0;
  bool blocking = false;
  std::vector<int> deps;
};

struct SchedulePlan {
  ScheduleVariant variant = ScheduleVariant::Default;
  bool split_batch = false;
  bool has_recompute = true;
  std::vector<ScheduledOp> forward_ops;
  std::vector<ScheduledOp> backward_ops;
  std::vector<std::vector<int>> saved_sequences;
  int total_ops() const { return static_cast<int>(forward_ops.size() + backward_ops.size()); }
  const ScheduledOp& op(int id) const;
};

SchedulePlan schedule_default(const ModelGraph& graph);
SchedulePlan schedule_intra_pass(const ModelGraph& graph);
SchedulePlan schedule_cross_pass(const ModelGraph& graph);
SchedulePlan schedule_oases(const ModelGraph& graph);
SchedulePlan make_schedule(const ModelGraph& graph, ScheduleVariant variant);
// Extension (fine-grained recomputation): per layer unit,
// keep[u] keeps the unit's interior post-AllReduce tensors (Oases: recompute
// from them, no collective) or replays the unit from its input with its
// recompute AllReduces (CrossPass). All-true == schedule_oases, all-false ==
// schedule_cross_pass; a mixed plan carries variant CrossPass.
SchedulePlan schedule_oases_policy(const ModelGraph& graph, const std::vector<bool>& keep);
int layer_unit_count(const ModelGraph& graph);

struct Violation {
  std::string code;
  std::string detail;
};
std::vector<Violation> validate_plan(const SchedulePlan& plan);
int comm_op_count(const SchedulePlan& plan);
// JSON text of the plan (same schema as the reference's plan_to_json).
std::string plan_to_json_text(const SchedulePlan& plan, int indent = -1);

// ------------------------------------------------------------- sim.hpp:13-47
struct TraceEvent {
  int op_id = 0;
  Stream stream = Stream::Compute;
  double start = 0.0;
  double end = 0.0;
};

struct SimResult {
  double makespan = 0.0;
  double compute_busy_fraction = 0.0;
  double comm_exposed = 0.0;
  double peak_memory = 0.0;
  std::vector<TraceEvent> trace;
};

struct SimOptions {
  double overlap_slowdown = 1.0;
};

SimResult simulate(const SchedulePlan& plan, const CostVectors& costs, const Strategy& strategy,
                   SimOptions options = {});

struct Breakdown {
  double comm_fraction = 0.0;
  double compute_fraction = 0.0;
  double idle_fraction = 0.0;
};
Breakdown breakdown(const SimResult& result);

// Exposed communication: comm-interval time not covered by any compute interval
// (the interval algebra of sim.cpp:178-199), shared by simulate() and the
// measured-trace path of execute().
double exposed_comm_time(std::vector<std::pair<double, double>> compute,
                         std::vector<std::pair<double, double>> comm);

// Extension: the policy choosing keep[] under an HBM budget (host/policy.cpp).
struct RecomputePolicy {
  std::vector<bool> keep;
  double predicted_time = 0.0;
  double predicted_memory = 0.0;
};
RecomputePolicy choose_recompute_policy(const ModelGraph& graph, const CostVectors& costs, const Strategy& strategy,
                                        double budget_bytes, SimOptions options = {});

// ------------------------------------------------------------- planner.hpp:18-82
struct EdgeCostMatrix {
  int p = 0;
  std::vector<double> entries;
  double at(int i, int j) const { return entries[static_cast<std::size_t>(i) * p + j]; }
  double& at(int i, int j) { return entries[static_cast<std::size_t>(i) * p + j]; }
};

struct PlanResult {
  Strategy strategy;
  double predicted_time = 0.0;
  double predicted_memory = 0.0;
  double solve_time_ms = 0.0;
  std::uint64_t evaluated = 0;
};

struct SolveOptions {
  double mem_granularity = 1 << 20;
  std::size_t frontier_cap = 20000;
  std::uint64_t brute_force_cap = 1000000;
};

double node_cost(const CostVectors& costs, const Strategy& strategy, Pass pass);
EdgeCostMatrix edge_cost_matrix(const CostVectors& costs, int v, int u, const HardwareProfile& profile);
std::vector<EdgeCostMatrix> build_edge_costs(const CostVectors& costs, const HardwareProfile& profile);
double objective(const CostVectors& costs, const std::vector<EdgeCostMatrix>& edges, const Strategy& strategy);
double memory_usage(const CostVectors& costs, const Strategy& strategy);
PlanResult solve(const ModelGraph& graph, const CostVectors& costs, const std::vector<EdgeCostMatrix>& edges,
                 const HardwareProfile& profile, double budget_bytes, SolveOptions options = {});
PlanResult brute_force(const ModelGraph& graph, const CostVectors& costs, const std::vector<EdgeCostMatrix>& edges,
                       const HardwareProfile& profile, double budget_bytes, SolveOptions options = {});
double rank_correlation(const CostVectors& costs, const std::vector<EdgeCostMatrix>& edges,
                        const std::vector<Strategy>& strategies, const std::vector<double>& measured_times);
double spearman(const std::vector<double>& a, const std::vector<double>& b);
std::string run_length_notation(const std::vector<int>& degrees);

// ------------------------------------------------------------- numerics.hpp:10-60
// The reference's value-level checker API. Same types, fields and semantics;
// every function computes ON THE GPU (f64): the Matrix primitives in device
// kernels with the reference's scalar arithmetic (no FMA contraction, same
// summation order), and the ToyShardedModel checks by running the toy as an
// f64 FFN block stack through this build's runtime -- the literal in-process
// AllReduce is the runtime's worker-order sum kernel, and
// recompute_elision_equivalence executes the CrossPass (replayed AllReduce)
// and Oases (elided) plans with the plan executor. Throws DeviceError without
// a CUDA device.
struct Matrix {
  int rows = 0;
  int cols = 0;
  std::vector<double> data;

  Matrix() = default;
  Matrix(int r, int c) : rows(r), cols(c), data(static_cast<std::size_t>(r) * c, 0.0) {}
  double& at(int r, int c) { return data[static_cast<std::size_t>(r) * cols + c]; }
  double at(int r, int c) const { return data[static_cast<std::size_t>(r) * cols + c]; }
};

Matrix matmul(const Matrix& a, const Matrix& b);
Matrix transpose(const Matrix& a);
Matrix add(const Matrix& a, const Matrix& b);
Matrix hadamard(const Matrix& a, const Matrix& b);
Matrix gelu(const Matrix& a);
Matrix gelu_grad(const Matrix& a);  // elementwise derivative at a
double max_abs_diff(const Matrix& a, const Matrix& b);

struct GradIdentityCheck {
  double autodiff_deviation = 0.0;
  double finite_difference_deviation = 0.0;
};
GradIdentityCheck allreduce_grad_identity(int workers, int rows, int cols, unsigned seed);

struct ToyShardedModel {
  int workers = 1;
  Matrix input;              // batch x model_dim
  std::vector<Matrix> w_in;  // model_dim x (hidden/workers) column shards
  std::vector<Matrix> w_out; // (hidden/workers) x model_dim row shards
};

ToyShardedModel make_toy_sharded_model(int workers, int batch, int model_dim, int hidden_dim, unsigned seed);
double sharded_output_deviation(const ToyShardedModel& model);

struct ElisionCheck {
  double grad_deviation = 0.0;
  bool loss_bit_identical = false;
};
ElisionCheck recompute_elision_equivalence(const ToyShardedModel& model);

// ------------------------------------------------------------- trace_export.hpp:15-22
void write_chrome_trace(const SimResult& result, const SchedulePlan& plan, const std::filesystem::path& path);
void write_svg_timeline(const SimResult& result, const SchedulePlan& plan, const std::filesystem::path& path);

// ------------------------------------------------------------- json_io.hpp:40-43
// The reference's named hardware presets ("3090", "nvlink-3090", same values)
// plus "b200" (b200_profile(8), runtime.hpp). Unknown names: ConfigError.
HardwareProfile preset_profile(const std::string& name);
std::vector<std::string> preset_profile_names();
std::string sim_result_to_json_text(const SimResult& result);

}  // namespace tmpsim
