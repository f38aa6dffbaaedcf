#!/usr/bin/env python
"""Benchmark: TMP train step (forward + Oases recompute + backward) of a GPT
layer stack on B200, samples/s and exposed AllReduce % of step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N = 1 runs BASELINE config C2 (h=2048, 16 heads, seq 1024, micro-batch 8,
24 layers, bf16, TMP=1). Under torchrun (N > 1) the same stack runs as one TMP
group of N ranks (NCCL over NVLink, one process per GPU): total work per step
is fixed, so scaling is "strong". One JSON line is printed by rank 0.

Timing: W untimed warm-up steps, then K steps of the CUDA-graph-captured plan,
each device-timed with cudaEvents on the compute stream inside the library
(barrier + synchronize on both sides, max over ranks). The working set
(2.4 GB of weights, 1.6 GB of saved activations) exceeds the 126 MB L2, so no
explicit flush is needed. `e2e` re-times the same step through the public
API with the input batch copied from pinned host memory every step and the
loss read back. `roofline` uses live cudaEvent timings of every linear-layer
GEMM launch of one extra step. `cpu_baseline` times the reference's own CPU
implementation of the path (oracle/_ref/ref_bench, built from /root/reference)
on a bounded sample.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS = {"hbm_gbs": 6532.9, "bf16_tflops": 1611.4, "bf16_tflops_sustained": 1356.2, "source": "fallback"}
try:
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
        _p = json.load(f)
    PEAKS.update({k: _p[k] for k in ("hbm_gbs", "bf16_tflops", "bf16_tflops_sustained") if k in _p})
    PEAKS["source"] = "measured"
except (OSError, ValueError):
    pass

METRIC = "TMP train step samples/s at 1/2/4/8 B200; exposed comm % of step"
CONFIGS = {
    # BASELINE.json configs[1] (C2) -- the N=1 headline
    "c2": dict(hidden=2048, heads=16, seq=1024, batch=8, layers=24),
    # configs[2] (C3) -- TMP=8 target, too large for one GPU at full depth
    "c3": dict(hidden=4096, heads=32, seq=2048, batch=8, layers=24),
    # configs[3] (C4)
    "c4": dict(hidden=8192, heads=64, seq=2048, batch=8, layers=8),
}


def step_flops(c, variant="Oases"):
    """Algorithmic FLOPs of one step for the whole TMP group."""
    T, h, s = c["batch"] * c["seq"], c["hidden"], c["seq"]
    f_fwd = 24 * T * h * h + 4 * T * s * h
    f_rec = f_fwd - 10 * T * h * h if variant == "Oases" else f_fwd
    return c["layers"] * (f_fwd + f_rec + 2 * f_fwd)


class ClockSampler:
    """nvidia-smi clock/throttle sampling during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device, self.rows, self.proc = device, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def cpu_baseline(cfg, seconds=12.0):
    """The reference's own CPU path (tmpsim::recompute_elision_equivalence) on the host cores."""
    exe = os.path.join(ROOT, "oracle", "_ref", "ref_bench")
    threads = os.cpu_count() or 1
    rows = 16  # one reference call ~ 3.8 GMAC at C2 widths: a few seconds per sample
    h, f = cfg["hidden"], 4 * cfg["hidden"]
    macs_per_sample = step_flops(cfg) / 2.0 / cfg["batch"]
    if os.path.exists(exe):
        out = subprocess.check_output([exe, "1", str(rows), str(h), str(f), str(seconds), str(threads)], text=True)
        r = json.loads(out)
        return {"value": r["macs_per_s"] / macs_per_sample, "unit": "samples/s", "cores": threads,
                "kind": "reference",
                "sample": (f"reference toy FFN checker (recompute_elision_equivalence, numerics.cpp:234) "
                           f"{rows} tokens x h{h} x ffn{f}, {threads} independent threads for {r['seconds']:.1f} s; "
                           f"{r['macs_per_s'] / 1e9:.2f} GMAC/s scaled by the step's MAC count"),
                "macs_per_s": r["macs_per_s"]}
    # fallback: the fp64 oracle port (full layer) on a small sample
    from oracle.oracle import LayerCfg, Oracle

    c = LayerCfg(hidden=256, heads=2, seq=128, batch=2, layers=1)
    o = Oracle(c)
    o.init_params(1)
    t0 = time.time()
    n = 0
    while time.time() - t0 < seconds:
        o.run()
        n += 1
    dt = time.time() - t0
    sample_macs = step_flops(dict(hidden=256, heads=2, seq=128, batch=2, layers=1), "CrossPass") / 2.0 * 0.75
    return {"value": n * sample_macs / dt / macs_per_sample, "unit": "samples/s", "cores": threads, "kind": "port",
            "sample": "fp64 oracle full layer h256 s128 b2, scaled by MAC count"}


def load_traffic():
    """dram bytes/launch of the dominant GEMM from the committed ncu summary, if any."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get("dominant_dram_bytes_per_launch"), d
    except (OSError, ValueError):
        return None, None


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    vals = []
    for _ in range(args.warmup + args.steps):
        vals.append(cpu_baseline(cfg, seconds=args.ref_seconds))
    timed = vals[args.warmup:]
    v = statistics.mean(x["value"] for x in timed)
    cb = dict(timed[-1])
    cb["value"] = v
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "samples/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": cfg["batch"] / v * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (mt19937 U(-1,1) inputs, numerics.cpp:136-154 init)",
            "config": dict(workload=f"{args.config} GPT layer stack, reference CPU numerics", **cfg,
                           parallelism=f"tp{args.gpus}"),
            "cpu_baseline": cb,
            "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=int(os.environ.get("WORLD_SIZE", "1")))
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--layers", type=int, default=0)
    ap.add_argument("--variant", default="Oases")
    ap.add_argument("--dropout", type=float, default=0.1)
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-seconds", type=float, default=3.0)
    ap.add_argument("--trace-out", default="")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config])
    if args.layers:
        cfg["layers"] = args.layers
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args, cfg)

    import numpy as np
    import torch

    from paper_2305_16121_b200.runtime import Context, LayerStack, ModelConfig, plan_for, unique_id

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    uid = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        obj = [unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    tp = world
    mc = ModelConfig(dtype="bf16", hidden_dropout=args.dropout, attention_dropout=args.dropout, **cfg)
    # TMP > 1: the persistent GEMM / attention grids leave SMs to NCCL so the
    # AllReduce of one sub-batch can run under the other sub-batch's compute
    # (a full-width persistent grid would block the collective until it ends)
    reserve = int(os.environ.get("OASES_NCCL_SMS", "16")) if tp > 1 else 0
    sms = torch.cuda.get_device_properties(local).multi_processor_count
    ctx = Context(tp=tp, rank=rank, device=local, unique_id=uid, nccl_max_ctas=reserve,
                  gemm_max_ctas=(sms - reserve) // 2 * 2 if reserve else 0)
    stack = LayerStack(ctx, mc)
    stack.init_random(1234)
    plan = plan_for(mc, args.variant)
    stack.bind(plan)
    if not args.no_graph:
        stack.capture_graph()

    def barrier():
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    launches0 = stack.kernel_launches()
    for _ in range(args.warmup):
        stack.step(trace=False)
    barrier()
    with ClockSampler(local) as clk:
        t0 = time.perf_counter()
        dev = [stack.step(trace=False).makespan for _ in range(args.steps)]
        wall = time.perf_counter() - t0
    barrier()
    total = sum(dev)
    if dist:
        t = torch.tensor([total], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total = t.item()
    ms_per_step = total / args.steps * 1e3
    value = mc.batch / (total / args.steps)
    # kernels launched by our library inside the timed region (graph replays issue the same kernels)
    per_step_launches = (stack.kernel_launches() - launches0) / max(1, args.warmup) if args.no_graph else None

    # one traced step: measured SimResult (exposed comm, compute busy)
    traced = stack.step(trace=True)
    launches_per_step = per_step_launches or 0
    if not launches_per_step:
        before = stack.kernel_launches()
        stack.step(trace=True)
        launches_per_step = stack.kernel_launches() - before
    if args.trace_out and rank == 0:
        import paper_2305_16121_b200.tmpsim as tm

        tm.write_chrome_trace(traced.sim_result(), plan, args.trace_out)
    # live GEMM timings for the roofline (one eager step with per-launch events)
    stack.set_kernel_timing(True)
    stack.step(trace=True)  # eager issue (graph replays bypass the per-launch events)
    ks = stack.kernel_stats()
    stack.set_kernel_timing(False)

    # e2e: public API with the input copied from pinned host memory + loss read back every step
    T = mc.batch * mc.seq
    host_in = torch.empty((T, mc.hidden), dtype=torch.bfloat16).uniform_(-1, 1).pin_memory()
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        stack.step(input=host_in, trace=False)
    barrier()
    e2e_wall = time.perf_counter() - t0
    if dist:
        t = torch.tensor([e2e_wall], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_wall = t.item()
    e2e = {"value": mc.batch * args.steps / e2e_wall, "unit": "samples/s",
           "h2d_bytes_per_step": T * mc.hidden * 2, "d2h_bytes_per_step": 8}

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    achieved = ks["gemm_flops"] / (ks["gemm_ms"] * 1e-3) / 1e12 if ks["gemm_ms"] > 0 else 0.0
    peak = PEAKS["bf16_tflops_sustained"]
    traffic, _ = load_traffic()
    step_tf = step_flops(cfg, args.variant) / tp / (total / args.steps) / 1e12
    line = {
        "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (device Philox U(-1,1) input, U(+-1/sqrt(fan_in)) weights, numerics.cpp conventions)",
        "config": {"workload": f"{args.config}: GPT layer stack h{cfg['hidden']} a{cfg['heads']} s{cfg['seq']} "
                               f"b{cfg['batch']} L{cfg['layers']}, TMP={tp}, {args.variant} schedule",
                   "global_batch": cfg["batch"], "seq_len": cfg["seq"], "hidden": cfg["hidden"],
                   "heads": cfg["heads"], "layers": cfg["layers"], "parallelism": f"tp{tp}",
                   "schedule": args.variant, "dropout": args.dropout, "cuda_graph": not args.no_graph,
                   "sms_reserved_for_nccl": reserve,
                   "l2": "working set (>4 GB) exceeds the 126 MB L2; no flush"},
        "exposed_comm_pct": 100.0 * traced.comm_exposed / traced.makespan if traced.makespan else 0.0,
        "measured_sim": {"makespan_s": traced.makespan, "comm_exposed_s": traced.comm_exposed,
                         "compute_busy_fraction": traced.compute_busy_fraction,
                         "peak_memory_bytes": traced.peak_memory},
        "step_tflops_per_gpu": step_tf,
        "step_roofline_frac": step_tf / peak,
        "roofline": {"bound": "tensor", "kernel": "gemm_tc (tcgen05 linear-layer GEMMs, all launches of a step)",
                     "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak if peak else 0,
                     "peak_source": f"{PEAKS['source']} bf16_tflops_sustained",
                     "gemm_launches": ks["gemm_launches"], "traffic": traffic},
        "gpu_launches": int(launches_per_step * args.steps),
        "clocks": clk.summary(),
        "wall_s_timed": wall,
        "e2e": e2e,
    }
    if not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline(cfg)
        except Exception as e:  # noqa: BLE001
            line["cpu_baseline"] = {"value": None, "error": str(e)}
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    del np


if __name__ == "__main__":
    main()
