"""Fine-grained recomputation policy: per layer unit, keep the
interior post-AllReduce tensor (Oases: recompute issues no collective, Eq. 1) or
replay the unit from its input with its AllReduces (CrossPass).

The endpoints are pinned to the reference's own variants: all-keep must be the
exact Oases plan and all-replay the exact CrossPass plan (schedule.cpp:360-444 of
the reference; fixtures in tests/golden via test_tmpsim_api). Mixed plans are
checked with the reference's invariants (validate_plan, comm counts,
saved-sequence coverage) and its timing/memory semantics (simulate).
"""
import itertools

import pytest

import paper_2305_16121_b200.tmpsim as t
from paper_2305_16121_b200.runtime import ModelConfig, graph_for, plan_for, recompute_policy


def gpt(layers, h=4096, heads=32, seq=2048, batch=8):
    spec = t.ModelSpec()
    spec.hidden_size, spec.num_layers, spec.seq_len = h, layers, seq
    spec.attention_heads, spec.global_batch, spec.bytes_per_element = heads, batch, 2
    spec.recompute_enabled = True
    return spec, t.build_block_graph(t.build_operator_sequence(spec), spec)


def ops_key(plan):
    return [(o.id, o.base_id, o.kind, o.pass_, o.stream, o.block, o.sub_batch, list(o.deps))
            for o in list(plan.forward_ops) + list(plan.backward_ops)]


@pytest.mark.parametrize("layers", [1, 2, 3, 5])
def test_endpoints_are_the_reference_variants(layers):
    _, g = gpt(layers)
    assert t.layer_unit_count(g) == layers
    a = t.schedule_oases_policy(g, [True] * layers)
    b = t.schedule_oases(g)
    assert ops_key(a) == ops_key(b) and a.saved_sequences == b.saved_sequences and a.variant == b.variant
    a = t.schedule_oases_policy(g, [False] * layers)
    b = t.schedule_cross_pass(g)
    assert ops_key(a) == ops_key(b) and a.saved_sequences == b.saved_sequences and a.variant == b.variant


@pytest.mark.parametrize("layers", [2, 3, 4])
def test_mixed_plans_valid_and_counted(layers):
    spec, g = gpt(layers)
    hw = t.b200_profile(8)
    costs = t.build_cost_vectors(g, spec, hw)
    s = t.Strategy([8] * g.block_count())
    fwd_ids = set()
    for keep in itertools.product([False, True], repeat=layers):
        plan = t.schedule_oases_policy(g, list(keep))
        assert t.validate_plan(plan) == []
        dropped = layers - sum(keep)
        # 2 fwd + 2 bwd collectives per layer, + 2 replayed per CrossPass unit (test_schedule.cpp:38-46)
        assert t.comm_op_count(plan) == 4 * layers + 2 * dropped
        rec_comm_blocks = {o.block for o in plan.backward_ops
                           if o.pass_ == t.Pass.Recompute and o.kind == t.OpKind.AllReduce}
        assert rec_comm_blocks == {b for l in range(layers) if not keep[l] for b in (2 * l, 2 * l + 1)}
        # every forward compute in exactly one saved sequence (test_schedule.cpp:133-149)
        flat = [i for seq in plan.saved_sequences for i in seq]
        fwd_ids = {o.id for o in plan.forward_ops if o.kind == t.OpKind.ForwardCompute}
        assert sorted(flat) == sorted(fwd_ids)
        # kept units save two boundary tensors per sub-batch, replayed units one
        assert len(plan.saved_sequences) == 2 * (2 * sum(keep) + dropped)
        r = t.simulate(plan, costs, s)
        assert r.makespan > 0


def test_memory_monotone_in_kept_units():
    spec, g = gpt(4)
    hw = t.b200_profile(8)
    costs = t.build_cost_vectors(g, spec, hw)
    s = t.Strategy([8] * g.block_count())
    mem = []
    for k in range(5):
        keep = [i < k for i in range(4)]
        mem.append(t.simulate(t.schedule_oases_policy(g, keep), costs, s).peak_memory)
    assert all(b > a for a, b in zip(mem, mem[1:]))
    # each kept unit costs one more [T_sub, h] boundary tensor per sub-batch, live across the step
    step = mem[1] - mem[0]
    assert all(abs((b - a) - step) <= 1e-6 * step for a, b in zip(mem, mem[1:]))


def test_policy_respects_budget():
    spec, g = gpt(6)
    hw = t.b200_profile(8)
    costs = t.build_cost_vectors(g, spec, hw)
    s = t.Strategy([8] * g.block_count())
    lo = t.simulate(t.schedule_cross_pass(g), costs, s).peak_memory
    hi = t.simulate(t.schedule_oases(g), costs, s).peak_memory
    full = t.choose_recompute_policy(g, costs, s, hi)
    assert full.keep == [True] * 6 and full.predicted_memory == hi
    none = t.choose_recompute_policy(g, costs, s, lo)
    assert none.keep == [False] * 6 and none.predicted_memory == lo
    with pytest.raises(t.InfeasibleError):
        t.choose_recompute_policy(g, costs, s, lo * 0.5)
    for frac in (0.25, 0.5, 0.75):
        budget = lo + frac * (hi - lo)
        pol = t.choose_recompute_policy(g, costs, s, budget)
        r = t.simulate(t.schedule_oases_policy(g, pol.keep), costs, s)
        assert r.peak_memory <= budget and r.peak_memory == pol.predicted_memory
        assert r.makespan == pol.predicted_time
        # the budget is spent: keeping one more unit would not fit
        per_unit = (hi - lo) / 6
        assert budget - r.peak_memory < per_unit * 1.000001
        # never slower than replaying everything
        assert pol.predicted_time <= none.predicted_time + 1e-12


def test_python_runtime_policy_helpers():
    mc = ModelConfig(hidden=1024, heads=8, seq=512, batch=4, layers=3)
    g = graph_for(mc)
    p = plan_for(mc, keep=[True, False, True])
    assert t.validate_plan(p) == [] and t.comm_op_count(p) == 4 * 3 + 2
    pol = recompute_policy(mc, 1e15, tp=2)
    assert pol.keep == [True] * 3
    assert t.layer_unit_count(g) == 3
    with pytest.raises(t.ConfigError):
        t.schedule_oases_policy(g, [True])
