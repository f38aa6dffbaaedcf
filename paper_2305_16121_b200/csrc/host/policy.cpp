// Fine-grained recomputation policy (north star: "the
// fine-grained recomputation policy picks which post-all-reduce tensors are
// kept in HBM so the recompute pass issues no collective").
//
// The reference only has the all-or-nothing variants: Oases keeps every
// block's post-AllReduce boundary tensor (two per layer, schedule.cpp:384-392
// of the reference) and never replays a collective (Eq. 1); CrossPass keeps
// the layer input only and replays the layer's AllReduces in recompute
// (schedule.cpp:404-412). Per layer unit this chooses between the two under
// an HBM budget, evaluating every candidate plan with the reference's own
// timing and memory semantics (simulate, sim.cpp:203-380) on the given --
// analytic or calibrated (load_measured_costs) -- cost vectors.
#include <limits>

#include "oases/tmpsim.hpp"

namespace tmpsim {

RecomputePolicy choose_recompute_policy(const ModelGraph& graph, const CostVectors& costs, const Strategy& strategy,
                                        double budget_bytes, SimOptions options) {
  if (!graph.recompute_enabled) throw ConfigError("choose_recompute_policy: the model has recomputation disabled");
  const int units = layer_unit_count(graph);
  RecomputePolicy best;
  best.keep.assign(static_cast<std::size_t>(units), true);
  {
    const SimResult all = simulate(schedule_oases_policy(graph, best.keep), costs, strategy, options);
    if (all.peak_memory <= budget_bytes) {
      best.predicted_time = all.makespan;
      best.predicted_memory = all.peak_memory;
      return best;
    }
  }
  best.keep.assign(static_cast<std::size_t>(units), false);
  const SimResult none = simulate(schedule_oases_policy(graph, best.keep), costs, strategy, options);
  if (none.peak_memory > budget_bytes)
    throw InfeasibleError("choose_recompute_policy: even full recomputation (CrossPass) needs " +
                          std::to_string(none.peak_memory) + " bytes > budget " + std::to_string(budget_bytes));
  best.predicted_time = none.makespan;
  best.predicted_memory = none.peak_memory;
  // Greedy: keep the unit whose plan is fastest while it fits; a unit whose
  // keep does not slow the step is taken too (one replayed collective pair
  // fewer on NVLink), so the budget is spent before it is left unused.
  constexpr double kTie = 1e-12;
  for (;;) {
    int pick = -1;
    SimResult pick_r;
    for (int u = 0; u < units; ++u) {
      if (best.keep[static_cast<std::size_t>(u)]) continue;
      std::vector<bool> trial = best.keep;
      trial[static_cast<std::size_t>(u)] = true;
      const SimResult r = simulate(schedule_oases_policy(graph, trial), costs, strategy, options);
      if (r.peak_memory > budget_bytes || r.makespan > best.predicted_time + kTie) continue;
      if (pick < 0 || r.makespan < pick_r.makespan - kTie ||
          (r.makespan <= pick_r.makespan + kTie && r.peak_memory < pick_r.peak_memory)) {
        pick = u;
        pick_r = r;
      }
    }
    if (pick < 0) break;
    best.keep[static_cast<std::size_t>(pick)] = true;
    best.predicted_time = pick_r.makespan;
    best.predicted_memory = pick_r.peak_memory;
  }
  return best;
}

}  // namespace tmpsim
