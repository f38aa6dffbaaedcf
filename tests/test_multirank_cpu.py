"""World-size-2 gloo tests of the N>1 host path (CPU only).

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
