"""TMP over NCCL with one process per GPU (the product's multi-rank path).

Needs >= 2 visible GPUs (skips otherwise; the round-end box has one). Two ranks
(torch.multiprocessing, spawn) each own a Megatron shard of the same oracle-
generated weights, bind the Oases plan and step with real ncclAllReduce calls on
the comm stream; the result must equal the in-process TMP=2 emulation (the same
shards on one GPU, worker-order sum kernel) and the fp64 oracle, and the measured
trace must carry the comm intervals (comm_exposed populated by the interval
algebra of sim.cpp:178-199).
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASE = dict(hidden=256, heads=4, seq=128, batch=4, layers=2, hidden_dropout=0.1, attention_dropout=0.1)


def _rank_main(rank, uid, dtype, q):
    import torch

    from oracle.oracle import PARAMS, LayerCfg, Oracle
    from paper_2305_16121_b200.runtime import Context, LayerStack, ModelConfig, plan_for

    torch.cuda.set_device(rank)
    orc = Oracle(LayerCfg(tp=2, **CASE))
    orc.init_params(7, extras=True)
    c = orc.cfg
    mc = ModelConfig(hidden=c.hidden, heads=c.heads, seq=c.seq, batch=c.batch, layers=c.layers, dtype=dtype,
                     hidden_dropout=c.hidden_dropout, attention_dropout=c.attention_dropout, seed=c.seed)
    ctx = Context(tp=2, rank=rank, device=rank, unique_id=uid)
    st = LayerStack(ctx, mc)
    for b in range(orc.num_blocks):
        for p in PARAMS:
            if st.param_numel(b, p):
                st.set_param(0, b, p, np.array(orc.param(rank, b, p)))
    st.set_input(np.array(orc.input))
    st.bind(plan_for(mc, "Oases"))
    res = st.step(trace=True)
    st.capture_graph()
    graph_loss = st.step(trace=False).loss
    grads = {(b, p): st.grad(0, b, p) for b in range(orc.num_blocks) for p in PARAMS if st.param_numel(b, p)}
    comm = [e for e in res.events if e[1] == 1]
    q.put((rank, res.loss, graph_loss, st.input_grad(), grads, len(comm), res.comm_exposed, res.makespan))
    st.close()
    ctx.close()


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_tmp2_over_nccl_matches_emulation_and_oracle(cuda, dtype):
    import torch
    import torch.multiprocessing as mp

    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs (one process per GPU over NCCL)")
    from oracle.oracle import PARAMS
    from paper_2305_16121_b200.runtime import unique_id
    from tests.test_stack_gpu import make_pair, rel, run_variant

    uid = unique_id()
    ctx_mp = mp.get_context("spawn")
    q = ctx_mp.Queue()
    procs = [ctx_mp.Process(target=_rank_main, args=(r, uid, dtype, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(2):
        r = q.get(timeout=300)
        out[r[0]] = r
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # in-process emulation of the same two ranks on GPU 0
    orc, ctx, st, mc = make_pair(CASE, 2, dtype)
    emu = run_variant(st, mc, "Oases")
    loss_ref = orc.run()
    tol = 1e-4 if dtype == "f32" else 3e-2
    for rank in (0, 1):
        _, loss, gloss, dx, grads, ncomm, exposed, makespan = out[rank]
        assert loss == gloss  # graph replay of the NCCL step
        assert abs(loss - emu.loss) <= 1e-6 * abs(emu.loss)
        assert rel(dx, st.input_grad()) <= 1e-5
        assert abs(loss - loss_ref) <= tol * abs(loss_ref)
        for (b, p), g in grads.items():
            assert rel(g, st.grad(rank, b, p)) <= 1e-5, (rank, b, p)
            assert rel(g, np.array(orc.grad(rank, b, p)).ravel()) <= tol
        assert ncomm == 8 * mc.layers  # per layer: 2 blocks x 2 sub-batches x (forward g, backward f)
        assert 0.0 <= exposed <= makespan
    del PARAMS


MIXED = dict(hidden=256, heads=4, seq=128, batch=4, layers=2, attention_dropout=0.1)
MIXED_DEGREES = [1, 2, 1, 2]


def _mixed_rank_main(rank, uid, q):
    import torch

    from oracle.oracle import PARAMS, LayerCfg, Oracle
    from paper_2305_16121_b200.runtime import Context, LayerStack, ModelConfig, plan_for, shard_parameter

    torch.cuda.set_device(rank)
    orc = Oracle(LayerCfg(tp=1, hidden_dropout=0.0, **MIXED))
    orc.init_params(11, extras=True)
    c = orc.cfg
    mc = ModelConfig(hidden=c.hidden, heads=c.heads, seq=c.seq, batch=c.batch, layers=c.layers, dtype="bf16",
                     hidden_dropout=0.0, attention_dropout=c.attention_dropout, seed=c.seed)
    ctx = Context(tp=2, rank=rank, device=rank, unique_id=uid)
    st = LayerStack(ctx, mc, degrees=MIXED_DEGREES)  # splits the degree-1 communicators (ncclCommSplit)
    for b in range(orc.num_blocks):
        d = MIXED_DEGREES[b]
        for p in PARAMS:
            if st.param_numel(b, p):
                st.set_param(0, b, p, shard_parameter(p, np.array(orc.param(0, b, p)), tp=d, rank=rank % d,
                                                      attention=b % 2 == 0, heads=c.heads, hidden=c.hidden))
    st.set_input(np.array(orc.input))
    st.bind(plan_for(mc, "Oases"))
    res = st.step(trace=True)
    grads = {(b, p): st.grad(0, b, p) for b in range(orc.num_blocks) for p in PARAMS if st.param_numel(b, p)}
    q.put((rank, res.loss, st.input_grad(), grads))
    st.close()
    ctx.close()


def test_mixed_degrees_over_nccl_match_emulation(cuda):
    """F2 over NCCL: degree-1 blocks on split communicators, ncclAllGather reshards and
    data-parallel gradient sums equal the in-process emulation of the same strategy."""
    import torch
    import torch.multiprocessing as mp

    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs (one process per GPU over NCCL)")
    from paper_2305_16121_b200.runtime import unique_id
    from tests.test_mixed_gpu import run_mixed
    from tests.test_stack_gpu import rel

    uid = unique_id()
    ctx_mp = mp.get_context("spawn")
    q = ctx_mp.Queue()
    procs = [ctx_mp.Process(target=_mixed_rank_main, args=(r, uid, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(2):
        r = q.get(timeout=300)
        out[r[0]] = r
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    orc, loss_ref, st, res = run_mixed(2, MIXED_DEGREES, "bf16", **MIXED)
    half = MIXED["batch"] // 2 * MIXED["seq"]
    dx_emu = st.input_grad()
    for rank in (0, 1):
        _, loss, dx, grads = out[rank]
        assert abs(loss - res.loss) <= 1e-6 * abs(res.loss)
        rows = slice(rank * half, (rank + 1) * half)  # block 0 (degree 1): this rank's group slice
        assert rel(dx[rows], dx_emu[rows]) <= 1e-5
        for (b, p), g in grads.items():
            assert rel(g, st.grad(rank, b, p)) <= 1e-5, (rank, b, p)
