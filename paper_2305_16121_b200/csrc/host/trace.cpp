// Trace export: the reference's Chrome-trace schema (proj/src/trace_export.cpp:31-46:
// complete "X" events, microseconds, tid 0 compute / 1 comm, args.op_id),
// used here for MEASURED two-stream timelines from the GPU executor as well
// as for simulated ones.
#include <fstream>

#include "json.hpp"
#include "oases/tmpsim.hpp"

namespace tmpsim {

namespace {
std::string label(const SchedulePlan& plan, const TraceEvent& ev) {
  if (ev.op_id >= plan.total_ops()) return ev.stream == Stream::Comm ? "Reshard" : "Tail";
  const ScheduledOp& op = plan.op(ev.op_id);
  std::string s = std::string(to_string(op.kind)) + " b" + std::to_string(op.block);
  if (plan.split_batch) s += " s" + std::to_string(op.sub_batch);
  return s;
}
}  // namespace

void write_chrome_trace(const SimResult& result, const SchedulePlan& plan, const std::filesystem::path& path) {
  nlohmann::json events = nlohmann::json::array();
  for (const TraceEvent& ev : result.trace) {
    const bool comm = ev.stream == Stream::Comm;
    events.push_back({{"name", label(plan, ev)},
                      {"cat", comm ? "comm" : "compute"},
                      {"ph", "X"},
                      {"ts", ev.start * 1e6},
                      {"dur", (ev.end - ev.start) * 1e6},
                      {"pid", 0},
                      {"tid", comm ? 1 : 0},
                      {"args", {{"op_id", ev.op_id}}}});
  }
  std::ofstream out(path);
  if (!out) throw IoError("cannot write " + path.string());
  out << events.dump(1) << "\n";
}

std::string sim_result_to_json_text(const SimResult& r) {
  nlohmann::json trace = nlohmann::json::array();
  for (const TraceEvent& ev : r.trace)
    trace.push_back({{"op_id", ev.op_id}, {"stream", to_string(ev.stream)}, {"start", ev.start}, {"end", ev.end}});
  return nlohmann::json{{"makespan", r.makespan},
                        {"compute_busy_fraction", r.compute_busy_fraction},
                        {"comm_exposed", r.comm_exposed},
                        {"peak_memory", r.peak_memory},
                        {"trace", trace}}
      .dump();
}

}  // namespace tmpsim
