"""BASELINE config C5: planner-chosen per-block TMP degrees for a 24-layer
h=4096 GPT under an HBM budget at 2/4/8 GPUs, with the cost model CALIBRATED
from measured B200 block timings (paper_2305_16121_b200.calibrate).

    python tools/plan_c5.py [--out profiles/c5_plan.json] [--budget-gb 60]
"""
import argparse
import json
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2305_16121_b200.tmpsim as t  # noqa: E402
from paper_2305_16121_b200.calibrate import calibrate, replicate_layers  # noqa: E402
from paper_2305_16121_b200.runtime import ModelConfig  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="profiles/c5_plan.json")
    ap.add_argument("--layers", type=int, default=24)
    ap.add_argument("--budget-gb", type=float, default=0.0, help="0: 180 GB")
    ap.add_argument("--steps", type=int, default=3)
    args = ap.parse_args()
    one = ModelConfig(hidden=4096, heads=32, seq=2048, batch=8, layers=1, dtype="bf16", hidden_dropout=0.1,
                      attention_dropout=0.1)
    degrees = [1, 2, 4, 8]
    rows1 = calibrate(one, degrees, steps=args.steps)
    rows = replicate_layers(rows1, 2, args.layers)
    full = ModelConfig(hidden=4096, heads=32, seq=2048, batch=8, layers=args.layers)
    spec = full.spec()
    graph = t.build_block_graph(t.build_operator_sequence(spec), spec)
    report = {"config": "C5: 24-layer h4096 s2048 b8 GPT, planner over measured B200 block costs",
              "calibration_rows_layer0": [[r.block_index, r.degree, r.field, r.seconds_or_bytes] for r in rows1],
              "gpus": {}}
    for n in (2, 4, 8):
        hw = t.b200_profile(n)
        base = t.build_cost_vectors(graph, spec, hw)
        with tempfile.NamedTemporaryFile("w", suffix=".json", delete=False) as f:
            path = f.name
        try:
            t.write_measured_costs([r for r in rows if r.degree <= n], path)
            costs = t.load_measured_costs(path, base)
        finally:
            os.unlink(path)
        edges = t.build_edge_costs(costs, hw)
        budget = args.budget_gb * 1e9 if args.budget_gb else float(hw.memory_capacity)
        entry = {"budget_bytes": budget, "uniform": {}}
        for d in hw.candidate_degrees:
            s = t.Strategy([d] * graph.block_count())
            entry["uniform"][d] = {"predicted_s": t.objective(costs, edges, s), "memory": t.memory_usage(costs, s),
                                   "simulated_oases_s": t.simulate(t.schedule_oases(graph), costs, s).makespan}
        try:
            pr = t.solve(graph, costs, edges, hw, budget)
            entry["plan"] = {"strategy": t.run_length_notation(list(pr.strategy.degrees)),
                             "predicted_s": pr.predicted_time, "memory": pr.predicted_memory,
                             "solve_ms": pr.solve_time_ms,
                             "simulated_oases_s": t.simulate(t.schedule_oases(graph), costs, pr.strategy).makespan}
        except t.InfeasibleError as e:
            entry["plan"] = {"infeasible": str(e)}
        # fine-grained recomputation policy at the uniform degree n:
        # which layers keep their mid-layer post-AllReduce tensor under budgets
        # between full recomputation (CrossPass) and Oases
        s_n = t.Strategy([n] * graph.block_count())
        lo = t.simulate(t.schedule_cross_pass(graph), costs, s_n)
        hi = t.simulate(t.schedule_oases(graph), costs, s_n)
        pol = {"crosspass": {"s": lo.makespan, "memory": lo.peak_memory, "exposed_comm_s": lo.comm_exposed},
               "oases": {"s": hi.makespan, "memory": hi.peak_memory, "exposed_comm_s": hi.comm_exposed},
               "budgets": []}
        for frac in (0.0, 0.25, 0.5, 0.75, 1.0):
            budget_p = lo.peak_memory + frac * (hi.peak_memory - lo.peak_memory)
            rp = t.choose_recompute_policy(graph, costs, s_n, budget_p)
            pol["budgets"].append({"budget_bytes": budget_p, "kept_layers": sum(rp.keep),
                                   "keep": "".join("K" if k else "r" for k in rp.keep),
                                   "predicted_s": rp.predicted_time, "memory": rp.predicted_memory})
        entry["recompute_policy"] = pol
        report["gpus"][n] = entry
        print(n, json.dumps(entry["plan"]), flush=True)
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(report, f, indent=1)


if __name__ == "__main__":
    main()
