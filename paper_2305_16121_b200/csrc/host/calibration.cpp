// Calibration boundary: measured rows out (-> load_measured_costs), and the
// B200 hardware preset in the reference's HardwareProfile schema.
#include <fstream>

#include "json.hpp"
#include "oases/runtime.hpp"

namespace tmpsim {

void write_measured_costs(const std::vector<MeasuredRow>& rows, const std::filesystem::path& path) {
  nlohmann::json arr = nlohmann::json::array();
  for (const MeasuredRow& r : rows) {
    static const char* fields[] = {"d_fwd", "d_bwd", "c_fwd", "c_bwd", "m_param", "m_saved", "m_runtime"};
    bool ok = false;
    for (const char* f : fields) ok = ok || r.field == f;
    if (!ok) throw ConfigError("measured-cost row: unknown field '" + r.field + "'");
    if (r.seconds_or_bytes < 0.0) throw ConfigError("measured-cost row: negative value");
    arr.push_back({{"block_index", r.block_index},
                   {"degree", r.degree},
                   {"field", r.field},
                   {"seconds_or_bytes", r.seconds_or_bytes}});
  }
  std::ofstream out(path);
  if (!out) throw IoError("cannot write " + path.string());
  out << arr.dump(1) << "\n";
}

HardwareProfile b200_profile(int num_devices, double nvlink_bytes_per_s, double latency_s) {
  if (num_devices < 1) throw ConfigError("b200_profile: num_devices must be positive");
  HardwareProfile hp;
  hp.num_devices = num_devices;
  hp.memory_capacity = 180LL * 1000 * 1000 * 1000;
  hp.compute_throughput = 0.5 * 1696.6e12;  // MAC/s at the measured bf16 dense burst (MEASURED_PEAKS.json, round 2)
  for (int d = 1; d <= num_devices; d *= 2) {
    hp.candidate_degrees.push_back(d);
    if (d > 1) {
      hp.bandwidth_by_group[d] = nvlink_bytes_per_s;
      hp.latency_by_group[d] = latency_s;
    }
  }
  hp.validate();
  return hp;
}

// Named presets of the reference (json_io.cpp:160-178: two synthetic 3090
// clusters, kept value-for-value so configs naming them still load) and this
// build's B200 node.
HardwareProfile preset_profile(const std::string& name) {
  if (name == "b200") return b200_profile(8);
  HardwareProfile hw;
  hw.num_devices = 8;
  hw.memory_capacity = 24LL * 1024 * 1024 * 1024;
  hw.compute_throughput = 1.4e13;
  hw.candidate_degrees = {2, 4, 8};
  hw.latency_by_group = {{2, 5e-6}, {4, 1e-5}, {8, 2e-5}};
  if (name == "nvlink-3090")
    hw.bandwidth_by_group = {{2, 2.0e10}, {4, 1.7e9}, {8, 1.2e9}};
  else if (name == "3090")
    hw.bandwidth_by_group = {{2, 5.0e9}, {4, 4.2e9}, {8, 3.0e9}};
  else
    throw ConfigError("unknown hardware preset '" + name + "' (have: 3090, nvlink-3090, b200)");
  return hw;
}

std::vector<std::string> preset_profile_names() { return {"3090", "nvlink-3090", "b200"}; }

}  // namespace tmpsim
