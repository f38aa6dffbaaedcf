// Real-hardware extensions of the tmpsim API (SURVEY.md §8(b) "What the B200
// replacement must export"): the calibration output rows that the reference's
// load_measured_costs ingests (proj/src/costs.cpp:162-214), and a B200
// HardwareProfile preset in the reference's schema (costs.hpp:17-28).
//
// Measured execution: `execute` runs a SchedulePlan on the GPU and returns the
// reference's SimResult shape filled from cudaEvent intervals (the measured
// counterpart of simulate, sim.hpp:38-39); `calibrate` measures the per-block
// per-degree rows load_measured_costs ingests. Both drive the same runtime as
// the C-ABI (include/oases.h: oases_plan_bind / oases_step), which
// paper_2305_16121_b200/runtime.py wraps for one process per GPU.
#pragma once

#include <cstdint>
#include <filesystem>
#include <memory>
#include <string>
#include <vector>

#include "oases/tmpsim.hpp"

namespace tmpsim {

// One override row of a measured-cost table (costs.cpp:174-211 schema).
struct MeasuredRow {
  int block_index = 0;
  int degree = 1;
  std::string field;  // d_fwd | d_bwd | c_fwd | c_bwd | m_param | m_saved | m_runtime
  double seconds_or_bytes = 0.0;
};

// Writes rows as the JSON array load_measured_costs reads.
void write_measured_costs(const std::vector<MeasuredRow>& rows, const std::filesystem::path& path);

// B200 NVSwitch node: 180 GB HBM3e per GPU, one bandwidth tier for every group
// size (NVSwitch gives each GPU full bandwidth to every peer), candidate
// degrees 1..num_devices. compute_throughput is MAC/s (the reference's
// "elements per second"); callers replace it and the comm terms with measured
// rows from calibration.
HardwareProfile b200_profile(int num_devices, double nvlink_bytes_per_s = 770e9, double latency_s = 10e-6);

// ------------------------------------------------------------- measured execution
// The devices, streams and NCCL communicator of one TMP rank (or of all `tp`
// ranks emulated in-process on one device with local_workers == tp).
struct ContextOptions {
  int tp = 1;
  int rank = 0;
  int device = 0;
  int local_workers = 1;
  std::string nccl_unique_id;  // nccl_unique_id() bytes from rank 0 (tp > 1, one rank per process)
  int nccl_max_ctas = 0;       // 0: NCCL default
  int gemm_max_ctas = 0;       // persistent-kernel grid cap leaving SMs to NCCL (0: all SMs)
  bool comm_disabled = false;  // one rank's shard of a tp-way group with the collectives skipped
};

std::string nccl_unique_id();  // OASES_UNIQUE_ID_BYTES bytes, broadcast out of band

class Context {
 public:
  explicit Context(const ContextOptions& options = {});
  ~Context();
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  const ContextOptions& options() const;
  struct Impl;
  Impl& impl();

 private:
  std::unique_ptr<Impl> impl_;
};

// What `execute` runs: the ModelSpec dimensions (global_batch = the micro-batch
// split into two sub-batches; bytes_per_element 2 = bf16 tensor-core path,
// 4 = f32 parity path) plus the numerics knobs of the real layer.
struct ExecOptions {
  ModelSpec spec;
  int ffn_hidden = 0;  // 0: 4 * hidden
  bool attention = true, layernorm = true, bias = true, residual = true;
  double hidden_dropout = 0.0, attention_dropout = 0.0;
  std::uint64_t seed = 1234;  // dropout keys and the synthetic weights / input
  int warmup = 1;
  int steps = 1;
  bool cuda_graph = false;  // replay the captured step (no per-op trace: trace = {})
};

// Runs `plan` on the GPU (warmup + steps; the last step is returned): per-op
// cudaEvent intervals as the trace (op_id = plan id; the two LN_0 tails get
// ids total_ops() and total_ops() + 1), makespan, compute-busy fraction,
// exposed communication by exposed_comm_time, device bytes as peak_memory.
// strategy: per-block degrees, each dividing ctx.options().tp (the world); a block
// below the world degree runs data-parallel groups, with the resharding AllGathers
// of simulate() between blocks of different degree.
SimResult execute(const SchedulePlan& plan, const Strategy& strategy, Context& ctx, const ExecOptions& opts);

// Per-block rows for every degree in `degrees`: d_fwd (forward op of a
// sub-batch), d_bwd (recompute + backward op, the reference's convention,
// costs.cpp:117,136), c_fwd / c_bwd (the half-batch AllReduce: timed on ctx's
// NCCL communicator when ctx.options().tp == degree, else the alpha-beta
// comm_time of b200_profile), m_saved. Compute is measured on ONE rank's shard
// of a degree-way group on ctx's device (collectives skipped): the kernels,
// shapes and HBM traffic of a real rank.
std::vector<MeasuredRow> calibrate(const ModelGraph& graph, const ModelSpec& spec, Context& ctx,
                                   const std::vector<int>& degrees, const ExecOptions& opts = {}, int steps = 3);

// Seconds of one AllReduce of `message_bytes` on ctx's communicator (NCCL,
// comm stream), median of `iters` cudaEvent-timed calls after warm-up; with
// local_workers > 1 the in-process worker-order sum kernel is timed instead.
double allreduce_seconds(Context& ctx, double message_bytes, int bytes_per_element, int iters = 20);

}  // namespace tmpsim
