// Real-hardware extensions of the tmpsim API (SURVEY.md §8(b) "What the B200
// replacement must export"): the calibration output rows that the reference's
// load_measured_costs ingests (proj/src/costs.cpp:162-214), and a B200
// HardwareProfile preset in the reference's schema (costs.hpp:17-28).
//
// Measured execution itself (`execute` -> SimResult) is driven through the
// C-ABI runtime (include/oases.h: oases_plan_bind / oases_step) so that one
// process per GPU can issue it; paper_2305_16121_b200/runtime.py wraps it.
#pragma once

#include <filesystem>
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

}  // namespace tmpsim
