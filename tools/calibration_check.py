"""Predicted vs measured: the reference's cost model and simulator, fed rows
measured on this B200, against the executor's measured step makespans
(the paper's Appendix C method, and the
reference's rank_correlation, planner.cpp:432-445).

For every case (a model shape, depth and TMP arrangement on this GPU):
  1. one traced step of the Oases plan -> per-block rows: d_fwd = forward op of
     a sub-batch, d_bwd = recompute + backward op (costs.cpp:117,136), c_fwd /
     c_bwd = the measured AllReduce op (emulated TMP=2: the worker-order sum
     kernel on the comm stream; TMP=1 and comm-disabled rank slices: 0);
  2. load_measured_costs(rows) -> CostVectors; simulate() of the Default,
     IntraPass, CrossPass and Oases plans -> predicted makespans;
  3. the executor runs each plan (CUDA graph, mean of `steps` replays) ->
     measured makespans.
Writes predicted/measured pairs, their Spearman rank correlation and the
relative errors to profiles/r02_calibration.json. All numbers are measured or
simulated from measured rows; no alpha-beta constants are involved.

    python tools/calibration_check.py [--out profiles/r02_calibration.json] [--quick]
"""
import argparse
import json
import os
import statistics
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2305_16121_b200.tmpsim as t  # noqa: E402
from paper_2305_16121_b200.runtime import Context, LayerStack, ModelConfig, graph_for, plan_for  # noqa: E402

VARIANTS = ("Default", "IntraPass", "CrossPass", "Oases")


def rows_from_trace(plan, res, tp, degree_comm):
    ops = list(plan.forward_ops) + list(plan.backward_ops)
    per = {}
    comm = {}
    for op_id, stream, s0, s1 in res.events:
        if op_id >= len(ops):
            continue
        op = ops[op_id]
        if stream == 1:
            comm.setdefault((op.block, op.pass_), []).append(s1 - s0)
        else:
            key = (op.block, op.sub_batch, op.pass_)
            per[key] = per.get(key, 0.0) + (s1 - s0)
    nblocks = 1 + max(op.block for op in ops)
    # an unsplit plan's op covers both halves; the simulator doubles per-sub-batch costs for it (sim.cpp:44-74)
    halves = (0, 1) if plan.split_batch else (0,)
    div = 1.0 if plan.split_batch else 2.0
    rows = []
    for b in range(nblocks):
        fwd = [per[(b, sb, t.Pass.Forward)] / div for sb in halves]
        bwd = [(per[(b, sb, t.Pass.Backward)] + per.get((b, sb, t.Pass.Recompute), 0.0)) / div for sb in halves]
        cf = statistics.mean(comm.get((b, t.Pass.Forward), [0.0])) / div if degree_comm else 0.0
        cb = statistics.mean(comm.get((b, t.Pass.Backward), [0.0])) / div if degree_comm else 0.0
        for field, v in (("d_fwd", statistics.mean(fwd)), ("d_bwd", statistics.mean(bwd)), ("c_fwd", cf),
                         ("c_bwd", cb)):
            r = t.MeasuredRow()
            r.block_index, r.degree, r.field, r.seconds_or_bytes = b, tp, field, float(v)
            rows.append(r)
    return rows


def costs_from(st, plan, mc, tp, emulated):
    """Rows from 3 traced steps of `plan` (median per field) -> CostVectors."""
    st.bind(plan)
    st.step(trace=True)
    rows = [rows_from_trace(plan, st.step(trace=True), tp, emulated) for _ in range(3)]
    merged = []
    for i, r in enumerate(rows[0]):
        m = t.MeasuredRow()
        m.block_index, m.degree, m.field = r.block_index, r.degree, r.field
        m.seconds_or_bytes = statistics.median(rr[i].seconds_or_bytes for rr in rows)
        merged.append(m)
    graph = graph_for(mc)
    base = t.build_cost_vectors(graph, mc.spec(), t.b200_profile(max(2, tp)))
    with tempfile.NamedTemporaryFile("w", suffix=".json", delete=False) as f:
        path = f.name
    try:
        t.write_measured_costs(merged, path)
        return t.load_measured_costs(path, base)
    finally:
        os.unlink(path)


def run_case(name, mc, tp, local_workers, comm_disabled, steps):
    ctx = Context(tp=tp, local_workers=local_workers, comm_disabled=comm_disabled)
    st = LayerStack(ctx, mc)
    st.init_random(1234)
    emulated = local_workers > 1
    # the planner's view: one row table (from the Oases plan) predicts every variant
    costs = costs_from(st, plan_for(mc, "Oases"), mc, tp, emulated)
    strategy = t.Strategy([tp] * graph_for(mc).block_count())
    out = {}
    for v in VARIANTS:
        plan = plan_for(mc, v)
        sim = t.simulate(plan, costs, strategy)
        # the simulator's timing semantics alone: rows measured from this variant's own trace
        own = t.simulate(plan, costs_from(st, plan, mc, tp, emulated), strategy)
        st.bind(plan)
        st.capture_graph()
        for _ in range(2):
            st.step(trace=False)
        ms = [st.step(trace=False).makespan for _ in range(steps)]
        traced_v = st.step(trace=True)
        measured = statistics.mean(ms)
        out[v] = {"predicted_s": sim.makespan, "measured_s": measured, "rel_err": (sim.makespan - measured) / measured,
                  "predicted_own_rows_s": own.makespan, "rel_err_own_rows": (own.makespan - measured) / measured,
                  "measured_exposed_comm_s": traced_v.comm_exposed,
                  "predicted_exposed_comm_s": sim.comm_exposed,
                  "predicted_own_rows_exposed_comm_s": own.comm_exposed}
    st.close()
    ctx.close()
    return {"case": name, "tp": tp, "local_workers": local_workers, "comm_disabled": comm_disabled,
            "layers": mc.layers, "variants": out}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="profiles/r02_calibration.json")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--quick", action="store_true", help="two small cases (CI smoke)")
    args = ap.parse_args()
    c2 = dict(hidden=2048, heads=16, seq=1024, batch=8)
    c3 = dict(hidden=4096, heads=32, seq=2048, batch=8)
    c4 = dict(hidden=8192, heads=64, seq=2048, batch=8)
    kw = dict(dtype="bf16", hidden_dropout=0.1, attention_dropout=0.1)
    cases = []
    if args.quick:
        cases = [("small L2 TMP=1", ModelConfig(hidden=256, heads=2, seq=256, batch=4, layers=2, **kw), 1, 1, False),
                 ("small L2 TMP=2 emulated", ModelConfig(hidden=256, heads=2, seq=256, batch=4, layers=2, **kw), 2, 2,
                  False)]
    else:
        for L in (2, 4, 8, 24):
            cases.append((f"C2 L{L} TMP=1", ModelConfig(layers=L, **c2, **kw), 1, 1, False))
        for L in (2, 4):
            cases.append((f"C2 L{L} TMP=2 emulated in-process", ModelConfig(layers=L, **c2, **kw), 2, 2, False))
        for L in (2, 8):
            cases.append((f"C3 L{L} rank slice of TMP=8", ModelConfig(layers=L, **c3, **kw), 8, 1, True))
        cases.append(("C4 L2 rank slice of TMP=8", ModelConfig(layers=2, **c4, **kw), 8, 1, True))
        cases.append(("C4 L2 rank slice of TMP=4", ModelConfig(layers=2, **c4, **kw), 4, 1, True))
    results = [run_case(n, mc, tp, lw, cd, args.steps) for n, mc, tp, lw, cd in cases]
    pred = [v["predicted_s"] for r in results for v in r["variants"].values()]
    meas = [v["measured_s"] for r in results for v in r["variants"].values()]
    errs = [abs(v["rel_err"]) for r in results for v in r["variants"].values()]
    within = []  # rank agreement of the four variants inside each case (what the planner decides on)
    for r in results:
        p = [r["variants"][v]["predicted_s"] for v in VARIANTS]
        m = [r["variants"][v]["measured_s"] for v in VARIANTS]
        within.append(t.spearman(p, m))
    own = [v["predicted_own_rows_s"] for r in results for v in r["variants"].values()]
    own_err = [abs(v["rel_err_own_rows"]) for r in results for v in r["variants"].values()]
    report = {"method": ("predicted: rows measured from traced Oases steps of each case -> load_measured_costs -> "
                         "simulate() of each variant's plan; own_rows: the same from that variant's own trace "
                         "(isolates the simulator's list-scheduling semantics); measured: the executor's "
                         "CUDA-graph makespan (mean of replays)"),
              "spearman_all": t.spearman(pred, meas), "spearman_within_case_mean": statistics.mean(within),
              "max_abs_rel_err": max(errs), "mean_abs_rel_err": statistics.mean(errs),
              "own_rows": {"spearman_all": t.spearman(own, meas), "max_abs_rel_err": max(own_err),
                           "mean_abs_rel_err": statistics.mean(own_err)},
              "cases": results}
    os.makedirs(os.path.dirname(os.path.abspath(args.out)), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(report, f, indent=1)
    print(json.dumps({k: report[k] for k in ("spearman_all", "spearman_within_case_mean", "max_abs_rel_err",
                                             "mean_abs_rel_err", "own_rows")}))


if __name__ == "__main__":
    main()
