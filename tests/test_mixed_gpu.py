"""Mixed per-block TMP degrees on one GPU, ranks emulated
in-process, against the fp64 oracle of the unsharded model.

A block of degree d < N (N = the world) runs data-parallel on N/d groups of d
ranks, each group on its slice of the micro-batch; between blocks of different
degree the executor injects the resharding AllGathers at the anchors of the
reference simulator (/root/reference/proj/src/sim.cpp:101-175):
  * degree grows v -> v+1: after v's last forward AllReduce, x_{v+1} is built
    on v's slices and gathered over v+1's groups;
  * degree shrinks v -> v+1: after v+1's backward tail, the gradient at x_{v+1}
    is gathered over v's groups;
and sums the data-parallel gradients at step end. The result must be the
micro-batch step of the unsharded model: loss, dX and every rank's shard of
every gradient within the stated tolerance. Attention dropout is on (its keys
follow the samples, not the slicing); hidden dropout is off (mixed degrees
require it).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle.oracle import PARAMS, LayerCfg, Oracle  # noqa: E402

from .test_stack_gpu import rel  # noqa: E402


def run_mixed(world, degrees, dtype, *, layers, variant="Oases", hidden=256, heads=4, seq=128, batch=4,
              attention_dropout=0.1, seed=11, graph=False):
    from paper_2305_16121_b200.runtime import Context, LayerStack, ModelConfig, plan_for, shard_parameter

    ocfg = LayerCfg(hidden=hidden, heads=heads, seq=seq, batch=batch, layers=layers, tp=1, hidden_dropout=0.0,
                    attention_dropout=attention_dropout)
    orc = Oracle(ocfg)
    orc.init_params(seed, extras=True)
    loss = orc.run()
    mc = ModelConfig(hidden=hidden, heads=heads, seq=seq, batch=batch, layers=layers, ffn=ocfg.ffn, dtype=dtype,
                     hidden_dropout=0.0, attention_dropout=attention_dropout, seed=ocfg.seed)
    ctx = Context(tp=world, local_workers=world)
    st = LayerStack(ctx, mc, degrees=degrees)
    assert st.degrees == list(degrees)
    att = lambda b: b % 2 == 0  # noqa: E731
    for b in range(orc.num_blocks):
        d = degrees[b]
        for w in range(world):
            for p in PARAMS:
                if st.param_numel(b, p):
                    full = np.array(orc.param(0, b, p))
                    st.set_param(w, b, p, shard_parameter(p, full, tp=d, rank=w % d, attention=att(b), heads=heads,
                                                          hidden=hidden))
    st.set_input(np.array(orc.input))
    st.bind(plan_for(mc, variant))
    if graph:
        st.capture_graph()
        st.step(trace=False)
    res = st.step(trace=True)
    return orc, loss, st, res


def check(orc, loss, st, res, degrees, world, tol):
    from paper_2305_16121_b200.runtime import shard_parameter

    errs = {"loss": abs(res.loss - loss) / abs(loss), "input_grad": rel(st.input_grad(), orc.input_grad)}
    for b in range(orc.num_blocks):
        d = degrees[b]
        for w in range(world):
            for p in PARAMS:
                if st.param_numel(b, p):
                    full = np.array(orc.grad(0, b, p))
                    want = shard_parameter(p, full, tp=d, rank=w % d, attention=b % 2 == 0,
                                           heads=st.cfg.heads, hidden=st.cfg.hidden)
                    errs[f"g[b{b},w{w},p{p}]"] = rel(st.grad(w, b, p), np.asarray(want).ravel())
    from tests.test_parity_baseline_gpu import log

    log(f"mixed_world{world}_{st.cfg.dtype}{degrees}", dict(hidden=st.cfg.hidden, heads=st.cfg.heads, seq=st.cfg.seq,
                                                          batch=st.cfg.batch, layers=st.cfg.layers,
                                                          degrees=list(degrees)), st.cfg.dtype, tol, errs,
        {"oracle_loss": loss, "gpu_loss": res.loss})
    bad = {k: v for k, v in errs.items() if not v <= tol}
    assert not bad, f"tolerance {tol} exceeded: {bad}"
    return errs


def gathers(res, nplan):
    """Injected AllGathers in the measured trace (op ids past the plan's)."""
    return [e for e in res.events if e[0] >= nplan and e[1] == 1]


@pytest.mark.parametrize("degrees", [[1, 1, 2, 2], [2, 2, 1, 1], [1, 2, 1, 2], [2, 1, 2, 1]])
def test_mixed_world2_bf16(cuda, degrees):
    orc, loss, st, res = run_mixed(2, degrees, "bf16", layers=2)
    check(orc, loss, st, res, degrees, 2, 3e-2)
    # one injected AllGather per degree change, on the comm stream, in the measured trace
    changes = sum(1 for a, b in zip(degrees, degrees[1:]) if a != b)
    nplan = st._plan.total_ops()
    ag = gathers(res, nplan)
    assert len(ag) == changes and all(e[3] >= e[2] for e in ag)


@pytest.mark.parametrize("degrees", [[1, 2, 1, 2], [2, 2, 1, 1]])
def test_mixed_world2_f32(cuda, degrees):
    """f32 mode: the north star's 1e-4 relative bound holds through the reshards."""
    orc, loss, st, res = run_mixed(2, degrees, "f32", layers=2)
    check(orc, loss, st, res, degrees, 2, 1e-4)


def test_mixed_world4_planner_style(cuda):
    """The planner's non-uniform shape ([[2]*8 + [4]*16] of acceptance_tests.cpp:262-307,
    scaled to 6 layers on a 4-rank world): degree 2 then 4, one growing reshard."""
    degrees = [2] * 4 + [4] * 8
    orc, loss, st, res = run_mixed(4, degrees, "bf16", layers=6, batch=8)
    check(orc, loss, st, res, degrees, 4, 3e-2)


def test_mixed_world4_all_degrees(cuda):
    degrees = [1, 2, 4, 2, 1, 4]
    orc, loss, st, res = run_mixed(4, degrees, "bf16", layers=3, batch=8)
    check(orc, loss, st, res, degrees, 4, 3e-2)


def test_mixed_graph_replay_matches_eager(cuda):
    """The injected AllGathers and gradient sums capture into the step's CUDA graph."""
    degrees = [1, 2, 1, 2]
    _, _, st_e, res_e = run_mixed(2, degrees, "bf16", layers=2)
    _, _, st_g, res_g = run_mixed(2, degrees, "bf16", layers=2, graph=True)
    assert res_e.loss == res_g.loss
    assert np.array_equal(st_e.input_grad(), st_g.input_grad())


def test_mixed_crosspass_allowed_inside_units(cuda):
    """CrossPass rebuilds x_b only inside a layer unit: legal when the degree changes at
    layer boundaries, rejected when a rebuilt tensor sits on a degree change."""
    degrees = [1, 1, 2, 2]
    orc, loss, st, res = run_mixed(2, degrees, "bf16", layers=2, variant="CrossPass")
    check(orc, loss, st, res, degrees, 2, 3e-2)
    from paper_2305_16121_b200._capi import OasesError

    with pytest.raises(OasesError, match="degree change"):
        run_mixed(2, [1, 2, 1, 2], "bf16", layers=2, variant="CrossPass")


def test_mixed_requires_no_hidden_dropout(cuda):
    from paper_2305_16121_b200._capi import OasesError
    from paper_2305_16121_b200.runtime import Context, LayerStack, ModelConfig

    mc = ModelConfig(hidden=256, heads=4, seq=128, batch=4, layers=1, dtype="bf16", hidden_dropout=0.1)
    with pytest.raises(OasesError, match="hidden_dropout"):
        LayerStack(Context(tp=2, local_workers=2), mc, degrees=[1, 2])
