"""Regenerate tests/golden/* from the REFERENCE itself (run in the build container).

Needs `make -C oracle ref` (builds /root/reference/proj into oracle/_ref: the
tmpsim library, its own pybind11 module and oracle/ref_dump.cpp). Nothing here
runs on the GPU box; the JSON fixtures it writes are committed.

Fixtures:
  toy_*.json          every tensor of the reference toy checker (ref_dump)
  plans.json          plan_to_json of all 4 variants, L=0..3, recompute on/off
  sim_cases.json      simulate() on random measured-cost tables (load_measured_costs)
  planner_cases.json  node_cost / edge costs / objective / memory / solve / brute_force
  misc.json           volumes, comm_time, spearman, run_length_notation, cost vectors
  reference_smoke_test.py.txt  the reference's own Python smoke test, byte for byte
                      (proj/tests/python/smoke_test.py; its sha256 in
                      reference_smoke_test.sha256) -- run against this build's
                      module under the name `tmpsim` by tests/test_numerics_gpu.py,
                      because /root/reference does not exist on the GPU box
"""
import json
import os
import random
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF = os.path.join(ROOT, "oracle", "_ref")
sys.path.insert(0, REF)
import tmpsim as t  # noqa: E402  (the reference's own pybind11 module)

TOYS = [(1, 4, 6, 8, 78), (2, 4, 6, 16, 79), (4, 4, 6, 32, 81),  # main.cpp:237 verify-numerics
        (1, 4, 4, 4, 3), (2, 4, 4, 8, 4),                         # test_numerics.cpp:65,71
        (4, 3, 5, 8, 0), (4, 3, 5, 8, 7), (4, 3, 5, 8, 19),       # test_numerics.cpp:78
        (2, 3, 4, 6, 9), (2, 8, 16, 64, 2024)]


def spec(L, recompute=True, h=64, seq=8, heads=4, batch=4, bpe=2):
    s = t.ModelSpec()
    s.hidden_size, s.num_layers, s.seq_len, s.attention_heads = h, L, seq, heads
    s.global_batch, s.bytes_per_element, s.recompute_enabled = batch, bpe, recompute
    return s


def flat_profile(degrees=(1, 2, 4, 8)):
    hw = t.HardwareProfile()
    hw.num_devices = 8
    hw.memory_capacity = 1 << 34
    hw.compute_throughput = 1e9
    hw.bandwidth_by_group = {2: 1e9, 4: 8e8, 8: 6e8}
    hw.latency_by_group = {2: 1e-6, 4: 2e-6, 8: 4e-6}
    hw.candidate_degrees = list(degrees)
    return hw


def profile_json(hw):
    return {"num_devices": hw.num_devices, "memory_capacity": hw.memory_capacity,
            "compute_throughput": hw.compute_throughput,
            "bandwidth_by_group": {str(k): v for k, v in hw.bandwidth_by_group.items()},
            "latency_by_group": {str(k): v for k, v in hw.latency_by_group.items()},
            "candidate_degrees": list(hw.candidate_degrees),
            "optimizer_bytes_per_element": hw.optimizer_bytes_per_element}


def spec_json(s):
    return {"hidden_size": s.hidden_size, "num_layers": s.num_layers, "seq_len": s.seq_len,
            "attention_heads": s.attention_heads, "global_batch": s.global_batch,
            "bytes_per_element": s.bytes_per_element, "recompute_enabled": s.recompute_enabled}


def random_rows(rng, nblocks, degrees, comm_scale, comp_scale):
    rows = []
    for b in range(nblocks):
        for d in degrees:
            df = rng.uniform(0.1, 1.0) * comp_scale
            rows.append({"block_index": b, "degree": d, "field": "d_fwd", "seconds_or_bytes": df})
            rows.append({"block_index": b, "degree": d, "field": "d_bwd",
                         "seconds_or_bytes": df * rng.uniform(2.0, 3.5)})
            c = 0.0 if d == 1 else rng.uniform(0.05, 1.0) * comm_scale
            rows.append({"block_index": b, "degree": d, "field": "c_fwd", "seconds_or_bytes": c})
            rows.append({"block_index": b, "degree": d, "field": "c_bwd",
                         "seconds_or_bytes": c * rng.uniform(0.8, 1.2)})
            rows.append({"block_index": b, "degree": d, "field": "m_runtime",
                         "seconds_or_bytes": rng.uniform(1e6, 5e7) / d})
    return rows


def load_costs(graph, s, hw, rows):
    base = t.build_cost_vectors(graph, s, hw)
    if not rows:
        return base
    with tempfile.NamedTemporaryFile("w", suffix=".json", delete=False) as f:
        json.dump(rows, f)
        path = f.name
    try:
        return t.load_measured_costs(path, base)
    finally:
        os.unlink(path)


def sim_json(r):
    return {"makespan": r.makespan, "compute_busy_fraction": r.compute_busy_fraction,
            "comm_exposed": r.comm_exposed, "peak_memory": r.peak_memory,
            "trace": [[e.op_id, 0 if e.stream == t.Stream.Compute else 1, e.start, e.end] for e in r.trace]}


VARIANTS = [("Default", t.ScheduleVariant.Default), ("IntraPass", t.ScheduleVariant.IntraPass),
            ("CrossPass", t.ScheduleVariant.CrossPass), ("Oases", t.ScheduleVariant.Oases)]


def make_toys():
    exe = os.path.join(REF, "ref_dump")
    for cfg in TOYS:
        out = subprocess.check_output([exe] + [str(v) for v in cfg]).decode()
        json.loads(out)
        name = "toy_" + "_".join(str(v) for v in cfg) + ".json"
        with open(os.path.join(HERE, name), "w") as f:
            f.write(out)


def make_plans():
    plans = {}
    for L in range(0, 4):
        for rec in (True, False):
            s = spec(L, rec)
            g = t.build_block_graph(t.build_operator_sequence(s), s)
            for name, v in VARIANTS:
                p = t.make_schedule(g, v)
                plans[f"{name}_L{L}_{'rec' if rec else 'norec'}"] = {
                    "plan": json.loads(p.to_json()), "comm_op_count": t.comm_op_count(p),
                    "violations": [repr(x) for x in t.validate_plan(p)]}
    # the reference's shipped golden file must equal what its code emits
    with open("/root/reference/proj/tests/golden/oases_l1_plan.json") as f:
        shipped = json.load(f)
    assert shipped == plans["Oases_L1_rec"]["plan"], "reference golden plan drifted"
    with open(os.path.join(HERE, "plans.json"), "w") as f:
        json.dump(plans, f, separators=(",", ":"))


def make_sim_cases():
    rng = random.Random(20260101)
    cases = []
    for i in range(24):
        L = rng.choice([1, 2, 3])
        rec = rng.random() < 0.8
        degrees = [1, 2, 4, 8]
        s = spec(L, rec, h=rng.choice([64, 128]), seq=rng.choice([8, 16]), batch=rng.choice([2, 4, 8]))
        hw = flat_profile(degrees)
        g = t.build_block_graph(t.build_operator_sequence(s), s)
        regime = rng.choice(["comm", "compute", "mixed", "analytic"])
        rows = [] if regime == "analytic" else random_rows(
            rng, g.block_count(), degrees, comm_scale=2.0 if regime == "comm" else 0.5,
            comp_scale=0.3 if regime == "comm" else 1.0)
        costs = load_costs(g, s, hw, rows)
        strategies = [[rng.choice(degrees[1:]) for _ in range(g.block_count())], [2] * g.block_count(),
                      [rng.choice(degrees) for _ in range(g.block_count())]]
        slow = rng.choice([1.0, 1.0, 1.25])
        res = {}
        for name, v in VARIANTS:
            plan = t.make_schedule(g, v)
            res[name] = [sim_json(t.simulate(plan, costs, t.Strategy(st), slow)) for st in strategies]
        cases.append({"spec": spec_json(s), "profile": profile_json(hw), "rows": rows, "strategies": strategies,
                      "overlap_slowdown": slow, "results": res})
    with open(os.path.join(HERE, "sim_cases.json"), "w") as f:
        json.dump(cases, f, separators=(",", ":"))


def make_planner_cases():
    rng = random.Random(777)
    cases = []
    for i in range(16):
        L = rng.choice([1, 2, 3, 4])
        degrees = rng.choice([[1, 2, 4], [2, 4, 8], [1, 2, 4, 8]])
        s = spec(L, True, h=rng.choice([64, 256]), seq=rng.choice([8, 64]), batch=rng.choice([4, 8]))
        hw = flat_profile(degrees)
        g = t.build_block_graph(t.build_operator_sequence(s), s)
        rows = random_rows(rng, g.block_count(), degrees, comm_scale=rng.choice([0.2, 1.0, 3.0]), comp_scale=1.0)
        costs = load_costs(g, s, hw, rows)
        edges = t.build_edge_costs(costs, hw)
        n = g.block_count()
        strategies = [[rng.choice(degrees) for _ in range(n)] for _ in range(5)]
        rec = {"spec": spec_json(s), "profile": profile_json(hw), "rows": rows, "strategies": strategies,
               "node_fwd": [], "node_bwd": [], "objective": [], "memory": [],
               "edges": [[[e.at(a, b) for b in range(e.p)] for a in range(e.p)] for e in edges]}
        for st in strategies:
            S = t.Strategy(st)
            rec["node_fwd"].append(t.node_cost(costs, S, t.Pass.Forward))
            rec["node_bwd"].append(t.node_cost(costs, S, t.Pass.Backward))
            rec["objective"].append(t.objective(costs, edges, S))
            rec["memory"].append(t.memory_usage(costs, S))
        mems = sorted(rec["memory"])
        budgets = [mems[len(mems) // 2] * 1.01, mems[-1] * 2.0]
        rec["solve"] = []
        for budget in budgets:
            try:
                pr = t.solve(g, costs, edges, hw, budget)
                entry = {"budget": budget, "degrees": list(pr.strategy.degrees), "time": pr.predicted_time,
                         "memory": pr.predicted_memory}
            except t.InfeasibleError:
                entry = {"budget": budget, "infeasible": True}
            if len(degrees) ** n <= 200000:
                try:
                    bf = t.brute_force(g, costs, edges, hw, budget)
                    entry["brute"] = {"degrees": list(bf.strategy.degrees), "time": bf.predicted_time,
                                      "evaluated": bf.evaluated}
                except t.InfeasibleError:
                    entry["brute"] = {"infeasible": True}
            rec["solve"].append(entry)
        cases.append(rec)
    with open(os.path.join(HERE, "planner_cases.json"), "w") as f:
        json.dump(cases, f, separators=(",", ":"))


def make_misc():
    rng = random.Random(5)
    misc = {"allreduce_volume": [], "allgather_volume": [], "spearman": [], "rle": [], "cost_vectors": []}
    for _ in range(10):
        k, d = rng.uniform(0, 1e9), rng.choice([1, 2, 4, 8])
        misc["allreduce_volume"].append([k, d, t.allreduce_volume(k, d)])
        misc["allgather_volume"].append([k, d, t.allgather_volume(k, d)])
    for _ in range(6):
        n = rng.randint(3, 12)
        a = [rng.choice([1.0, 2.0, 3.0, rng.random()]) for _ in range(n)]
        b = [rng.random() for _ in range(n)]
        misc["spearman"].append([a, b, t.spearman(a, b)])
    for v in ([2] * 8 + [4] * 16, [1], [], [8, 8, 4, 8]):
        misc["rle"].append([v, t.run_length_notation(v)])
    for rec in (True, False):
        for bpe in (2, 4):
            s = spec(2, rec, h=128, seq=16, batch=4, bpe=bpe)
            hw = flat_profile([1, 2, 4, 8])
            g = t.build_block_graph(t.build_operator_sequence(s), s)
            c = t.build_cost_vectors(g, s, hw)
            # observable through the public bindings: node costs per uniform degree + memory
            entry = {"spec": spec_json(s), "profile": profile_json(hw), "per_degree": []}
            for d in hw.candidate_degrees:
                S = t.Strategy([d] * g.block_count())
                entry["per_degree"].append([d, t.node_cost(c, S, t.Pass.Forward), t.node_cost(c, S, t.Pass.Backward),
                                            t.memory_usage(c, S)])
            misc["cost_vectors"].append(entry)
    with open(os.path.join(HERE, "misc.json"), "w") as f:
        json.dump(misc, f, separators=(",", ":"))


def make_smoke_fixture():
    import hashlib
    import shutil

    src = "/root/reference/proj/tests/python/smoke_test.py"
    dst = os.path.join(HERE, "reference_smoke_test.py.txt")  # .txt: never collected by pytest
    shutil.copyfile(src, dst)
    with open(src, "rb") as f:
        digest = hashlib.sha256(f.read()).hexdigest()
    with open(os.path.join(HERE, "reference_smoke_test.sha256"), "w") as f:
        f.write(digest + "  proj/tests/python/smoke_test.py\n")


if __name__ == "__main__":
    make_smoke_fixture()
    make_toys()
    make_plans()
    make_sim_cases()
    make_planner_cases()
    make_misc()
    print("golden fixtures written to", HERE)
