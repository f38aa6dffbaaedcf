"""World-size-2 and -4 gloo tests of the N>1 host path (CPU only).

The TMP ranks of the GPU build exchange only through the AllReduce; these tests
run the host-side partition logic (runtime.shard_parameter) in two real
processes and check, with torch.distributed's gloo AllReduce standing in for
NCCL, that the rank partials of every block sum to the unsharded block output
(the g AllReduce, numerics.cpp:158-165) and that the f-backward partials sum to
the unsharded input gradient (numerics.cpp:206), and that every rank builds the
identical plan it will issue (the schedule is rank-independent).
"""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _gelu(x):
    from math import sqrt

    from scipy.special import erf

    return 0.5 * x * (1.0 + erf(x / sqrt(2.0)))


def _worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from oracle.oracle import B_COL, W_COL, W_ROW, LayerCfg, Oracle
        from paper_2305_16121_b200.runtime import ModelConfig, plan_for, shard_parameter

        # unsharded reference parameters (same seed on every rank)
        cfg = LayerCfg(hidden=32, heads=4, seq=8, batch=2, layers=1, tp=1, use_layernorm=False)
        orc = Oracle(cfg)
        orc.init_params(11, extras=True)
        x = np.array(orc.input)
        T, h = x.shape
        ok = True
        # FFN block (block 1): partial_r = gelu(x W1_r + b1_r) W2_r
        wc, bc, wr = (np.array(orc.param(0, 1, p)) for p in (W_COL, B_COL, W_ROW))
        w1 = shard_parameter(W_COL, wc, tp=world, rank=rank, attention=False)
        b1 = shard_parameter(B_COL, bc, tp=world, rank=rank, attention=False)
        w2 = shard_parameter(W_ROW, wr, tp=world, rank=rank, attention=False)
        part = torch.tensor(_gelu(x @ w1 + b1) @ w2)
        dist.all_reduce(part)
        full = _gelu(x @ wc + bc) @ wr
        ok &= np.allclose(part.numpy(), full, rtol=1e-12, atol=1e-12)
        # backward f: d_in = sum_r dpre_r W1_r^T
        g = np.ones((T, h))
        pre_r = x @ w1 + b1
        dx = torch.tensor(((g @ w2.T) * (pre_r > -1e9)) @ w1.T)
        dist.all_reduce(dx)
        ok &= np.allclose(dx.numpy(), (g @ wr.T) @ wc.T, rtol=1e-12, atol=1e-12)
        # attention block (block 0): head-partitioned Q/K/V columns and proj rows
        wq = np.array(orc.param(0, 0, W_COL))
        wo = np.array(orc.param(0, 0, W_ROW))
        mine = shard_parameter(W_COL, wq, tp=world, rank=rank, attention=True, heads=4, hidden=h)
        rows = shard_parameter(W_ROW, wo, tp=world, rank=rank, attention=True, heads=4, hidden=h)
        parts = [torch.zeros(1)]
        gathered = [torch.zeros(mine.size, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(gathered, torch.tensor(mine.ravel()))
        hl, d = 4 // world, h // 4
        rebuilt = np.zeros_like(wq)
        for r, gt in enumerate(gathered):
            m = gt.numpy().reshape(h, 3 * hl * d)
            for part_i in range(3):
                rebuilt[:, part_i * h + r * hl * d: part_i * h + (r + 1) * hl * d] = m[:, part_i * hl * d:(part_i + 1) * hl * d]
        ok &= np.array_equal(rebuilt, wq)
        ok &= rows.shape == (h // world, h)
        # every rank issues the same plan
        mc = ModelConfig(hidden=64, heads=4, seq=16, batch=4, layers=2)
        js = plan_for(mc, "Oases").to_json()
        all_js = [None] * world
        dist.all_gather_object(all_js, js)
        ok &= all(j == js for j in all_js)
        del parts
        q.put((rank, bool(ok)))
        dist.destroy_process_group()
    except Exception as e:  # noqa: BLE001
        q.put((rank, repr(e)))


def test_two_rank_partition_and_allreduce():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=180) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert results == {0: True, 1: True}, results


def _mixed_worker(rank, world, port, q, degrees):
    """One rank of a mixed-degree stack on `world` ranks: its token slice, group and
    weight shard come from the product's rank geometry (runtime.rank_layout ->
    oases_rank_layout, the functions Stack uses for its buffer offsets and
    ncclCommSplit colours); the tensor-parallel AllReduce, the data-parallel
    gradient sum and the resharding AllGather run over gloo groups built from
    those colours. The result must be the unsharded FFN block on the whole
    micro-batch (sim.cpp:101-175 for the group structure, numerics.cpp:158-165
    and 206 for the sums)."""
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from oracle.oracle import B_COL, W_COL, W_ROW
        from paper_2305_16121_b200.runtime import ModelConfig, rank_layout, shard_parameter

        mc = ModelConfig(hidden=32, heads=4, seq=8, batch=8, layers=len(degrees) // 2, ffn=64, dtype="f32")
        lay = rank_layout(mc, world, rank, degrees)
        every = [None] * world
        dist.all_gather_object(every, lay)
        ok = True
        T, h, f = mc.batch * mc.seq, mc.hidden, mc.ffn
        # the groups of every distinct degree, created in the same order on every rank
        # (torch.distributed.new_group is collective, like ncclCommSplit)
        tp_groups, dp_groups = {}, {}
        for d in sorted(set(degrees)):
            for g in range(world // d):
                grp = dist.new_group([g * d + r for r in range(d)])
                if g == rank // d:
                    tp_groups[d] = grp
            for r in range(d):
                grp = dist.new_group([g * d + r for g in range(world // d)])
                if r == rank % d:
                    dp_groups[d] = grp
        rng = np.random.default_rng(3)
        x = rng.standard_normal((T, h))
        for b, d in enumerate(degrees):
            blocks = [e[b] for e in every]
            att = b % 2 == 0
            # partition: the groups' token slices tile the micro-batch, each group's ranks
            # hold distinct tensor-parallel indices, widths tile the weights
            ok &= all(L["degree"] == d and L["groups"] == world // d and L["attention"] == int(att) for L in blocks)
            spans = sorted({(L["token_row0"], L["token_row0"] + 2 * L["tokens_per_sub_batch"]) for L in blocks})
            ok &= spans[0][0] == 0 and spans[-1][1] == T and all(a[1] == c[0] for a, c in zip(spans, spans[1:]))
            for g in range(world // d):
                mem = [L for L in blocks if L["group"] == g]
                ok &= sorted(L["rank_in_group"] for L in mem) == list(range(d))
            ok &= blocks[rank]["col_width"] * d == (3 * h if att else f)
            ok &= blocks[rank]["row_width"] * d == (h if att else f)
            if att:
                continue
            # the FFN block on this rank's slice with its shard, then the exchanges
            L = blocks[rank]
            r0, n = L["token_row0"], 2 * L["tokens_per_sub_batch"]
            w1 = rng.standard_normal((h, f)) * 0.2
            b1 = rng.standard_normal(f) * 0.1
            w2 = rng.standard_normal((f, h)) * 0.2
            s1 = shard_parameter(W_COL, w1, tp=d, rank=L["rank_in_group"], attention=False)
            sb = shard_parameter(B_COL, b1, tp=d, rank=L["rank_in_group"], attention=False)
            s2 = shard_parameter(W_ROW, w2, tp=d, rank=L["rank_in_group"], attention=False)
            ok &= s1.shape[1] == L["col_width"] and s2.shape[0] == L["row_width"]
            xs = x[r0:r0 + n]
            pre = xs @ s1 + sb
            y = torch.tensor(_gelu(pre) @ s2)
            dist.all_reduce(y, group=tp_groups[d])  # the block's g AllReduce inside the group
            full = _gelu(x @ w1 + b1) @ w2
            ok &= np.allclose(y.numpy(), full[r0:r0 + n], rtol=1e-12, atol=1e-12)
            # resharding AllGather: the next degree's groups need every token of their slice
            gathered = [torch.zeros_like(y) for _ in range(world // d)]
            dist.all_gather(gathered, y, group=dp_groups[d])
            ok &= np.allclose(torch.cat(gathered).numpy(), full, rtol=1e-12, atol=1e-12)
            # data-parallel gradient sum: dW2 shard over the group's tokens, summed over groups
            gy = np.ones((n, h))
            dw2 = torch.tensor(_gelu(pre).T @ gy)
            dist.all_reduce(dw2, group=dp_groups[d])
            want = shard_parameter(W_ROW, _gelu(x @ w1 + b1).T @ np.ones((T, h)), tp=d, rank=L["rank_in_group"],
                                   attention=False)
            ok &= np.allclose(dw2.numpy(), want, rtol=1e-12, atol=1e-10)
        q.put((rank, bool(ok)))
        dist.destroy_process_group()
    except Exception as e:  # noqa: BLE001
        q.put((rank, repr(e)))


@pytest.mark.parametrize("world,degrees", [(2, [1, 2, 2, 1]), (4, [2, 2, 4, 4, 1, 4]), (4, [4, 1, 2, 2])])
def test_mixed_degree_layout_and_group_exchanges(world, degrees):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 30500 + (os.getpid() % 1000) + 17 * world + len(degrees)
    procs = [ctx.Process(target=_mixed_worker, args=(r, world, port, q, degrees)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert results == {r: True for r in range(world)}, results


def test_rank_layout_rejects_what_the_stack_rejects():
    from paper_2305_16121_b200._capi import OasesError
    from paper_2305_16121_b200.runtime import ModelConfig, rank_layout

    mc = ModelConfig(hidden=32, heads=4, seq=8, batch=4, layers=1, ffn=64, dtype="f32")
    with pytest.raises(OasesError, match="divide the world"):
        rank_layout(mc, 4, 0, [3, 4])
    with pytest.raises(OasesError, match="must be even"):
        rank_layout(mc, 4, 0, [1, 4])  # 4 samples over 4 groups: one sample per group
    with pytest.raises(OasesError, match="one degree per block"):
        rank_layout(mc, 2, 0, [2])
    L = rank_layout(mc, 2, 1)
    assert [e["degree"] for e in L] == [2, 2] and L[0]["heads_local"] == 2 and L[1]["col_width"] == 32


def test_bench_launches_one_rank_per_gpu():
    """bench.py --gpus N outside torchrun re-executes itself as N ranks; inside a launcher
    whose WORLD_SIZE disagrees with --gpus it refuses instead of silently running TMP=1."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["OASES_BENCH_PRINT_LAUNCH"] = "1"
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "4", "--steps", "2"],
                         env=env, capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    cmd = json.loads(out.stdout.strip().splitlines()[-1])["launch"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"] and "--nproc-per-node=4" in cmd
    assert "--master-addr=127.0.0.1" in cmd and cmd[-4:] == ["--gpus", "4", "--steps", "2"]
    env.pop("OASES_BENCH_PRINT_LAUNCH")
    env["WORLD_SIZE"] = "1"
    bad = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2"], env=env,
                         capture_output=True, text=True, timeout=120)
    assert bad.returncode != 0 and "WORLD_SIZE=1" in bad.stderr
