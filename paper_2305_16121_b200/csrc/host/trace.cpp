// Trace export: the reference's Chrome-trace schema (proj/src/trace_export.cpp:31-46:
// complete "X" events, microseconds, tid 0 compute / 1 comm, args.op_id),
// used here for MEASURED two-stream timelines from the GPU executor as well
// as for simulated ones.
#include <algorithm>
#include <cmath>
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

// SVG timeline (the reference's write_svg_timeline entry point, trace_export.hpp:19):
// one lane per stream, time axis in ms with ticks, bars coloured by pass
// (forward / recompute / backward, AllReduce, resharding or tail), the exposed
// part of every comm interval (not covered by any compute interval, the
// exposed_comm_time algebra) hatched in the comm lane. Works for measured
// (executor) and simulated results alike.
void write_svg_timeline(const SimResult& result, const SchedulePlan& plan, const std::filesystem::path& path) {
  const double W = 1400.0, lane = 40.0, top = 56.0, left = 90.0, right = 20.0;
  double span = result.makespan;
  for (const TraceEvent& ev : result.trace) span = std::max(span, ev.end);
  if (!(span > 0.0)) span = 1.0;
  const double sx = (W - left - right) / span;
  std::ofstream out(path);
  if (!out) throw IoError("cannot write " + path.string());
  const double H = top + 2 * (lane + 16) + 40;
  out << "<svg xmlns=\"http://www.w3.org/2000/svg\" width=\"" << W << "\" height=\"" << H
      << "\" font-family=\"sans-serif\">\n";
  out << "<defs><pattern id=\"hatch\" width=\"6\" height=\"6\" patternUnits=\"userSpaceOnUse\">"
      << "<path d=\"M0,6 L6,0\" stroke=\"black\" stroke-width=\"1\"/></pattern></defs>\n";
  out << "<text x=\"" << left << "\" y=\"20\" font-size=\"14\">" << to_string(plan.variant) << ": makespan "
      << result.makespan * 1e3 << " ms, exposed comm " << result.comm_exposed * 1e3 << " ms ("
      << (result.makespan > 0 ? 100.0 * result.comm_exposed / result.makespan : 0.0) << " %), compute busy "
      << 100.0 * result.compute_busy_fraction << " %</text>\n";
  const double lane_y[2] = {top, top + lane + 16};
  const char* names[2] = {"compute", "comm"};
  for (int l = 0; l < 2; ++l)
    out << "<text x=\"8\" y=\"" << lane_y[l] + lane * 0.6 << "\" font-size=\"12\">" << names[l] << "</text>\n";
  // time ticks
  const double raw = span / 10.0, mag = std::pow(10.0, std::floor(std::log10(raw)));
  const double step = raw / mag < 2 ? 2 * mag : raw / mag < 5 ? 5 * mag : 10 * mag;
  for (double t = 0.0; t <= span * 1.0001; t += step) {
    const double x = left + t * sx;
    out << "<line x1=\"" << x << "\" y1=\"" << top - 6 << "\" x2=\"" << x << "\" y2=\"" << H - 30
        << "\" stroke=\"#ddd\"/><text x=\"" << x << "\" y=\"" << H - 14 << "\" font-size=\"10\" "
        << "text-anchor=\"middle\">" << t * 1e3 << "</text>\n";
  }
  out << "<text x=\"" << W - right << "\" y=\"" << H - 2 << "\" font-size=\"10\" text-anchor=\"end\">ms</text>\n";
  std::vector<std::pair<double, double>> comp;
  for (const TraceEvent& ev : result.trace)
    if (ev.stream == Stream::Compute) comp.emplace_back(ev.start, ev.end);
  std::sort(comp.begin(), comp.end());
  for (const TraceEvent& ev : result.trace) {
    const int l = ev.stream == Stream::Comm ? 1 : 0;
    std::string fill = l ? "#c0504d" : "#4f81bd";
    if (ev.op_id >= plan.total_ops()) {
      fill = "#8064a2";
    } else {
      const Pass p = plan.op(ev.op_id).pass;
      if (!l && p == Pass::Recompute) fill = "#9bbb59";
      if (!l && p == Pass::Backward) fill = "#1f497d";
      if (l && p == Pass::Recompute) fill = "#f79646";
    }
    const double x = left + ev.start * sx, w = std::max(0.6, (ev.end - ev.start) * sx);
    out << "<rect x=\"" << x << "\" y=\"" << lane_y[l] << "\" width=\"" << w << "\" height=\"" << lane
        << "\" fill=\"" << fill << "\" stroke=\"white\" stroke-width=\"0.3\"><title>" << label(plan, ev) << ": "
        << ev.start * 1e3 << " - " << ev.end * 1e3 << " ms</title></rect>\n";
    if (l) {  // exposed sub-intervals of this comm op
      double cur = ev.start;
      auto emit = [&](double a, double b) {
        if (b > a)
          out << "<rect x=\"" << left + a * sx << "\" y=\"" << lane_y[1] << "\" width=\"" << std::max(0.6, (b - a) * sx)
              << "\" height=\"" << lane << "\" fill=\"url(#hatch)\"/>\n";
      };
      for (const auto& c : comp) {
        if (c.second <= cur) continue;
        if (c.first >= ev.end) break;
        emit(cur, std::min(c.first, ev.end));
        cur = std::max(cur, c.second);
        if (cur >= ev.end) break;
      }
      emit(cur, ev.end);
    }
  }
  out << "</svg>\n";
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
