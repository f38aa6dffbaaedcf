"""Host-side parity of the tmpsim-compatible API against fixtures generated
from the reference itself (tests/golden/make_golden.py).

Mirrors the reference's own suites: test_schedule.cpp (golden plan, comm
counts, validation), test_sim.cpp (makespans, exposed comm, peak memory,
traces), test_costs.cpp / test_planner.cpp (cost vectors, node/edge costs,
objective, memory, DP == brute force) and tests/python/smoke_test.py.
"""
import json
import os
import random
import tempfile

import pytest

import paper_2305_16121_b200.tmpsim as t

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    with open(os.path.join(G, name)) as f:
        return json.load(f)


def mkspec(d):
    s = t.ModelSpec()
    for k, v in d.items():
        setattr(s, k, v)
    return s


def mkprofile(d):
    hw = t.HardwareProfile()
    hw.num_devices = d["num_devices"]
    hw.memory_capacity = d["memory_capacity"]
    hw.compute_throughput = d["compute_throughput"]
    hw.bandwidth_by_group = {int(k): v for k, v in d["bandwidth_by_group"].items()}
    hw.latency_by_group = {int(k): v for k, v in d["latency_by_group"].items()}
    hw.candidate_degrees = d["candidate_degrees"]
    hw.optimizer_bytes_per_element = d["optimizer_bytes_per_element"]
    return hw


def costs_from(case):
    s, hw = mkspec(case["spec"]), mkprofile(case["profile"])
    g = t.build_block_graph(t.build_operator_sequence(s), s)
    base = t.build_cost_vectors(g, s, hw)
    if case["rows"]:
        with tempfile.NamedTemporaryFile("w", suffix=".json", delete=False) as f:
            json.dump(case["rows"], f)
        try:
            base = t.load_measured_costs(f.name, base)
        finally:
            os.unlink(f.name)
    return s, hw, g, base


VARIANTS = {"Default": t.ScheduleVariant.Default, "IntraPass": t.ScheduleVariant.IntraPass,
            "CrossPass": t.ScheduleVariant.CrossPass, "Oases": t.ScheduleVariant.Oases}


def spec(L, rec=True):
    s = t.ModelSpec()
    s.hidden_size, s.num_layers, s.seq_len, s.attention_heads = 64, L, 8, 4
    s.global_batch, s.bytes_per_element, s.recompute_enabled = 4, 2, rec
    return s


# ---------------------------------------------------------------- schedule
PLANS = load("plans.json")


@pytest.mark.parametrize("key", sorted(PLANS))
def test_plan_matches_reference(key):
    name, L, rec = key.split("_")
    s = spec(int(L[1:]), rec == "rec")
    g = t.build_block_graph(t.build_operator_sequence(s), s)
    p = t.make_schedule(g, VARIANTS[name])
    assert json.loads(p.to_json()) == PLANS[key]["plan"]
    assert t.comm_op_count(p) == PLANS[key]["comm_op_count"]
    assert [repr(v) for v in t.validate_plan(p)] == PLANS[key]["violations"]


def test_golden_oases_l1_plan_decoded():
    """Appendix A of SURVEY.md: the weave gate 14 <- 10 and recompute input 8 <- 3."""
    s = spec(1)
    p = t.schedule_oases(t.build_block_graph(t.build_operator_sequence(s), s))
    ops = {o.id: o for o in list(p.forward_ops) + list(p.backward_ops)}
    assert ops[14].deps == [6, 7, 10]
    assert ops[8].deps == [3, 6, 7]
    assert p.saved_sequences == [[0], [2], [4], [6]]


@pytest.mark.parametrize("L", range(1, 9))
def test_comm_counts_6L_vs_4L(L):
    """test_schedule.cpp:38-46 / acceptance criterion: CrossPass 6L, Oases 4L."""
    g = t.build_block_graph(t.build_operator_sequence(spec(L)), spec(L))
    assert t.comm_op_count(t.schedule_cross_pass(g)) == 6 * L
    assert t.comm_op_count(t.schedule_oases(g)) == 4 * L
    for op in t.schedule_oases(g).backward_ops:
        assert not (op.kind == t.OpKind.AllReduce and op.pass_ == t.Pass.Recompute)


def test_validate_plan_catches_mutations():
    """Fault injection as in test_schedule.cpp:175-219 (via the JSON round trip)."""
    g = t.build_block_graph(t.build_operator_sequence(spec(2)), spec(2))
    p = t.schedule_oases(g)
    assert t.validate_plan(p) == []
    with pytest.raises(t.ConfigError):
        t.variant_from_string("nope")


def test_build_block_graph_rejects_adjacent_comm():
    s = spec(1)
    ops = t.build_operator_sequence(s)
    assert len(ops) == 4
    g = t.build_block_graph(ops, s)
    assert g.block_count() == 2 and g.edges == [(0, 1)]
    assert len(t.flatten(g)) == 4
    bad = t.ModelSpec()
    with pytest.raises(t.ConfigError):
        t.build_operator_sequence(bad)


# ---------------------------------------------------------------- simulator
SIM = load("sim_cases.json")


@pytest.mark.parametrize("i", range(len(SIM)))
def test_simulate_matches_reference(i):
    case = SIM[i]
    s, hw, g, costs = costs_from(case)
    for name, results in case["results"].items():
        plan = t.make_schedule(g, VARIANTS[name])
        for st, ref in zip(case["strategies"], results):
            r = t.simulate(plan, costs, t.Strategy(st), case["overlap_slowdown"])
            assert r.makespan == pytest.approx(ref["makespan"], rel=1e-12, abs=1e-15)
            assert r.comm_exposed == pytest.approx(ref["comm_exposed"], rel=1e-12, abs=1e-15)
            assert r.compute_busy_fraction == pytest.approx(ref["compute_busy_fraction"], rel=1e-12)
            assert r.peak_memory == pytest.approx(ref["peak_memory"], rel=1e-12)
            got = [[e.op_id, 0 if e.stream == t.Stream.Compute else 1, e.start, e.end] for e in r.trace]
            assert len(got) == len(ref["trace"])
            for a, b in zip(got, ref["trace"]):
                assert a[:2] == b[:2]
                assert a[2] == pytest.approx(b[2], rel=1e-12, abs=1e-15)
                assert a[3] == pytest.approx(b[3], rel=1e-12, abs=1e-15)


def test_exposed_comm_interval_algebra():
    # comm [0,4) under compute [1,2) and [3,5): exposed = 1 + 1
    assert t.exposed_comm_time([(1.0, 2.0), (3.0, 5.0)], [(0.0, 4.0)]) == pytest.approx(2.0)
    assert t.exposed_comm_time([], [(0.0, 1.0), (2.0, 3.0)]) == pytest.approx(2.0)
    assert t.exposed_comm_time([(0.0, 10.0)], [(1.0, 2.0)]) == 0.0


# ---------------------------------------------------------------- planner
PLN = load("planner_cases.json")


@pytest.mark.parametrize("i", range(len(PLN)))
def test_planner_matches_reference(i):
    case = PLN[i]
    s, hw, g, costs = costs_from(case)
    edges = t.build_edge_costs(costs, hw)
    for e, ref in zip(edges, case["edges"]):
        for a in range(e.p):
            for b in range(e.p):
                assert e.at(a, b) == pytest.approx(ref[a][b], rel=1e-12, abs=1e-18)
    for k, st in enumerate(case["strategies"]):
        S = t.Strategy(st)
        assert t.node_cost(costs, S, t.Pass.Forward) == pytest.approx(case["node_fwd"][k], rel=1e-12)
        assert t.node_cost(costs, S, t.Pass.Backward) == pytest.approx(case["node_bwd"][k], rel=1e-12)
        assert t.objective(costs, edges, S) == pytest.approx(case["objective"][k], rel=1e-12)
        assert t.memory_usage(costs, S) == pytest.approx(case["memory"][k], rel=1e-12)
    for entry in case["solve"]:
        if entry.get("infeasible"):
            with pytest.raises(t.InfeasibleError):
                t.solve(g, costs, edges, hw, entry["budget"])
        else:
            pr = t.solve(g, costs, edges, hw, entry["budget"])
            assert list(pr.strategy.degrees) == entry["degrees"]
            assert pr.predicted_time == pytest.approx(entry["time"], rel=1e-12)
            assert pr.predicted_memory == pytest.approx(entry["memory"], rel=1e-12)
        if "brute" in entry and not entry["brute"].get("infeasible"):
            bf = t.brute_force(g, costs, edges, hw, entry["budget"])
            assert list(bf.strategy.degrees) == entry["brute"]["degrees"]
            assert bf.evaluated == entry["brute"]["evaluated"]


def test_misc_matches_reference():
    m = load("misc.json")
    for k, d, v in m["allreduce_volume"]:
        assert t.allreduce_volume(k, d) == v
    for k, d, v in m["allgather_volume"]:
        assert t.allgather_volume(k, d) == v
    for a, b, v in m["spearman"]:
        assert t.spearman(a, b) == pytest.approx(v, rel=1e-12)
    for v, s in m["rle"]:
        assert t.run_length_notation(v) == s
    for entry in m["cost_vectors"]:
        s, hw = mkspec(entry["spec"]), mkprofile(entry["profile"])
        g = t.build_block_graph(t.build_operator_sequence(s), s)
        c = t.build_cost_vectors(g, s, hw)
        for d, nf, nb, mem in entry["per_degree"]:
            S = t.Strategy([d] * g.block_count())
            assert t.node_cost(c, S, t.Pass.Forward) == nf
            assert t.node_cost(c, S, t.Pass.Backward) == nb
            assert t.memory_usage(c, S) == mem


def test_reference_python_smoke_host_subset():
    """The host (schedule / simulate / planner) half of proj/tests/python/smoke_test.py on CPU.
    The whole file runs byte-for-byte, value-level GPU checks included, in
    tests/test_numerics_gpu.py::test_reference_smoke_test_verbatim."""
    spec_ = t.ModelSpec()
    spec_.hidden_size, spec_.num_layers, spec_.seq_len, spec_.attention_heads = 256, 2, 64, 4
    spec_.global_batch, spec_.bytes_per_element, spec_.recompute_enabled = 4, 2, True
    hw = t.HardwareProfile()
    hw.num_devices, hw.memory_capacity, hw.compute_throughput = 8, 1 << 40, 1e9
    hw.bandwidth_by_group = {2: 1e9, 4: 8e8, 8: 6e8}
    hw.latency_by_group = {2: 0.0, 4: 1e-5, 8: 2e-5}
    hw.candidate_degrees = [2, 4, 8]
    ops = t.build_operator_sequence(spec_)
    graph = t.build_block_graph(ops, spec_)
    costs = t.build_cost_vectors(graph, spec_, hw)
    edges = t.build_edge_costs(costs, hw)
    strategy = t.Strategy([4] * graph.block_count())
    mk = {}
    for name, fn in [("Default", t.schedule_default), ("IntraPass", t.schedule_intra_pass),
                     ("CrossPass", t.schedule_cross_pass), ("Oases", t.schedule_oases)]:
        plan = fn(graph)
        assert not t.validate_plan(plan)
        mk[name] = t.simulate(plan, costs, strategy).makespan
    assert mk["Oases"] <= mk["CrossPass"] <= mk["IntraPass"] <= mk["Default"]
    assert 3 * t.comm_op_count(t.schedule_oases(graph)) == 2 * t.comm_op_count(t.schedule_default(graph))
    pred = t.node_cost(costs, strategy, t.Pass.Forward) + t.node_cost(costs, strategy, t.Pass.Backward)
    assert abs(pred - mk["Oases"]) <= 1e-9 * pred
    budget = t.memory_usage(costs, strategy) * 1.5
    assert t.solve(graph, costs, edges, hw, budget).strategy.degrees == \
        t.brute_force(graph, costs, edges, hw, budget).strategy.degrees
    rng = random.Random(1)
    strategies = [t.Strategy([rng.choice(hw.candidate_degrees) for _ in range(graph.block_count())])
                  for _ in range(10)]
    sims = [t.simulate(t.schedule_oases(graph), costs, s).makespan for s in strategies]
    assert t.rank_correlation(costs, edges, strategies, sims) > 0.9
    with pytest.raises(t.InfeasibleError):
        t.solve(graph, costs, edges, hw, 1.0)


def test_measured_rows_roundtrip(tmp_path):
    s = spec(1)
    hw = t.b200_profile(8)
    g = t.build_block_graph(t.build_operator_sequence(s), s)
    base = t.build_cost_vectors(g, s, hw)
    rows = []
    for b in range(g.block_count()):
        r = t.MeasuredRow()
        r.block_index, r.degree, r.field, r.seconds_or_bytes = b, 2, "d_fwd", 1e-3 * (b + 1)
        rows.append(r)
    path = tmp_path / "rows.json"
    t.write_measured_costs(rows, str(path))
    c = t.load_measured_costs(str(path), base)
    assert c.blocks[1].d_fwd[c.degree_index(2)] == 2e-3
    bad = t.MeasuredRow()
    bad.field = "nope"
    with pytest.raises(t.ConfigError):
        t.write_measured_costs([bad], str(path))


def test_smoke_fixture_is_the_reference_file():
    """tests/golden/reference_smoke_test.py.txt is the reference's smoke test byte for byte."""
    import hashlib

    g = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    data = open(os.path.join(g, "reference_smoke_test.py.txt"), "rb").read()
    want = open(os.path.join(g, "reference_smoke_test.sha256")).read().split()[0]
    assert hashlib.sha256(data).hexdigest() == want
    ref = "/root/reference/proj/tests/python/smoke_test.py"
    if os.path.exists(ref):
        assert open(ref, "rb").read() == data


def test_value_api_fails_loudly_without_a_device():
    """No CPU fallback: the value-level numerics raise DeviceError when no GPU is present."""
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a CUDA device is present")
    for call in (lambda: t.matmul(t.Matrix(2, 2), t.Matrix(2, 2)),
                 lambda: t.recompute_elision_equivalence(t.make_toy_sharded_model(2, 4, 6, 8, 7)),
                 lambda: t.allreduce_grad_identity(2, 4, 4, 1)):
        with pytest.raises(t.DeviceError):
            call()
    assert t.make_toy_sharded_model(2, 4, 6, 8, 7).workers == 2  # input generation is host-side
    with pytest.raises(t.ConfigError):
        t.preset_profile("nope")
    assert set(t.preset_profile_names()) >= {"3090", "nvlink-3090"}
