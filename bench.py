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
loss read back. `roofline` uses cudaEvent timings of every linear-layer GEMM
launch inside a replay of the captured step. `cpu_baseline` (and the
`--impl reference` arm, one sample per step) runs the fp64 full-layer CPU
restatement on a bounded sample of the configured workload with every host
core, plus the reference's own toy checker (oracle/_ref, built from
/root/reference) per call at its shipped sizes.

`--gpus N` outside torchrun re-executes itself under torch.distributed.run with
N ranks. Extras (skip with --no-extras): at N=1 one rank of the north-star
config C3 at TMP=8 (`c3_tp8`, collectives disabled) and TMP=2 emulated
in-process (`emulated_tp2_exposure`, real comm-stream AllReduce kernels); at
N=8 the C3 config itself at TMP=8 over NCCL.
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


def oracle_sample(cfg, sample_batch=2, threads=None):
    """One bounded sample of the configured workload on the host cores: the fp64
    full-layer restatement (oracle/gpt_oracle.cpp, OpenMP on every host core)
    running `sample_batch` sequences of the config's shape through ONE of its
    identical layers, forward + backward. The stack's step is `layers` such
    layers, so the sample is 1/layers of the per-layer work of `sample_batch`
    samples: samples/s = sample_batch / layers / seconds."""
    from oracle.oracle import LayerCfg, Oracle

    threads = threads or os.cpu_count() or 1
    os.environ.setdefault("OMP_NUM_THREADS", str(threads))
    c = LayerCfg(hidden=cfg["hidden"], heads=cfg["heads"], seq=cfg["seq"], batch=sample_batch, layers=1,
                 hidden_dropout=0.1, attention_dropout=0.1)
    o = Oracle(c)
    o.init_params(1, extras=True)
    t0 = time.perf_counter()
    o.run()
    dt = time.perf_counter() - t0
    return {"seconds": dt, "value": sample_batch / cfg["layers"] / dt, "unit": "samples/s", "cores": threads,
            "kind": "port",
            "sample": (f"fp64 full-layer restatement (oracle/gpt_oracle.cpp; LN, causal attention, GeLU FFN, "
                       f"bias-dropout-residual, dropout 0.1): {sample_batch} sequences x s{cfg['seq']} x "
                       f"h{cfg['hidden']} through 1 of the {cfg['layers']} identical layers, fwd+bwd, "
                       f"{threads} OpenMP threads, {dt:.2f} s measured; value = {sample_batch}/{cfg['layers']} "
                       f"samples / time")}


def reference_toy_calls(threads=1, seconds=1.0):
    """The reference's own CPU implementation of the path (tmpsim::recompute_elision_equivalence,
    proj/src/numerics.cpp:234-256, built from /root/reference into oracle/_ref) timed per call
    at its shipped sizes (main.cpp:236-240 verify-numerics (w,4,6,8w)) and at the FFN-only
    scaled shape of BASELINE.md 5.2 (256x256x1024), single-threaded."""
    exe = os.path.join(ROOT, "oracle", "_ref", "ref_bench")
    if not os.path.exists(exe):
        return {"error": "oracle/_ref/ref_bench not built"}
    out = {}
    for name, (w, rows, d, h) in {"toy_w2_4x6x16": (2, 4, 6, 16), "toy_w4_4x6x32": (4, 4, 6, 32),
                                  "ffn_256x256x1024": (2, 256, 256, 1024)}.items():
        r = json.loads(subprocess.check_output([exe, str(w), str(rows), str(d), str(h), str(seconds), str(threads)],
                                               text=True))
        out[name] = {"us_per_call": r["seconds"] / r["calls"] * 1e6, "gmac_per_s": r["macs_per_s"] / 1e9,
                     "threads": threads}
    return out


def cpu_baseline(cfg):
    cb = oracle_sample(cfg)
    try:
        cb["reference_toy"] = reference_toy_calls()
    except Exception as e:  # noqa: BLE001
        cb["reference_toy"] = {"error": str(e)}
    return cb


def load_traffic():
    """dram bytes/launch of the dominant GEMM (the FC1 forward) from the committed ncu
    --set full summary of this round (profiles/r02_gemm_ncu.json), else round 1's."""
    p2 = os.path.join(ROOT, "profiles", "r02_gemm_ncu.json")
    try:
        with open(p2) as f:
            d = json.load(f)
        k = d["kernels"][0]
        return (k["dram_read_mb"] + k["dram_write_mb"]) * 1e6, d
    except (OSError, ValueError, KeyError, IndexError):
        pass
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get("dominant_dram_bytes_per_launch"), d
    except (OSError, ValueError):
        return None, None


def run_reference(args, cfg):
    """Reference arm: the CPU implementation of the path on the host cores, one bounded
    sample of the configured workload per step (rank 0 only under torchrun)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    samples = [oracle_sample(cfg, args.ref_batch) for _ in range(args.warmup + args.steps)]
    timed = samples[args.warmup:]
    secs = [x["seconds"] for x in timed]
    v = args.ref_batch / cfg["layers"] / statistics.mean(secs)
    cb = dict(timed[-1])
    cb["value"] = v
    try:
        cb["reference_toy"] = reference_toy_calls()
    except Exception as e:  # noqa: BLE001
        cb["reference_toy"] = {"error": str(e)}
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "samples/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": statistics.mean(secs) * 1e3,
            "ms_per_step_sd": statistics.pstdev(secs) * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (mt19937 U(-1,1) input, U(+-1/sqrt(fan_in)) weights, numerics.cpp:136-154 conventions)",
            "config": dict(workload=(f"{args.config} GPT layer stack on the host CPU: each step = {args.ref_batch} "
                                     f"sequences through 1 of {cfg['layers']} identical layers (fwd+bwd, fp64)"),
                           **cfg, parallelism="host OpenMP"),
            "cpu_baseline": cb,
            "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def self_launch(args):
    """`bench.py --gpus N` outside torchrun re-executes itself as N ranks (one per GPU)."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    if os.environ.get("OASES_BENCH_PRINT_LAUNCH"):
        print(json.dumps({"launch": cmd}), flush=True)
        return
    os.execv(sys.executable, cmd)


def c3_rank_slice(steps=10, warmup=3):
    """One TMP rank of the north-star config C3 at TMP=8 (h4096, 32 heads, s2048, b8,
    24 layers; per rank QKV N=1536, proj K=512, 4 heads), collectives disabled: the
    compute side of that rank's step on this GPU."""
    from paper_2305_16121_b200.runtime import Context, LayerStack, ModelConfig, plan_for

    cfg = dict(CONFIGS["c3"])
    mc = ModelConfig(dtype="bf16", hidden_dropout=0.1, attention_dropout=0.1, **cfg)
    ctx = Context(tp=8, comm_disabled=True)
    st = LayerStack(ctx, mc)
    st.init_random(1234)
    st.bind(plan_for(mc, "Oases"))
    st.capture_graph()
    for _ in range(warmup):
        st.step(trace=False)
    ms = [st.step(trace=False).makespan * 1e3 for _ in range(steps)]
    mem = st.step(trace=True).peak_memory
    st.close()
    ctx.close()
    t = statistics.mean(ms)
    tf = step_flops(cfg) / 8 / (t * 1e-3) / 1e12
    return {"config": "c3 (h4096 a32 s2048 b8 L24), one rank of TMP=8, collectives disabled", "ms_per_step": t,
            "ms_per_step_sd": statistics.pstdev(ms), "tflops": tf,
            "frac_of_sustained_peak": tf / PEAKS["bf16_tflops_sustained"], "peak_memory_bytes": mem}


def emulated_tp2(cfg, layers=4, steps=5):
    """TMP=2 emulated in-process on this GPU (local_workers=2): both ranks' kernels on the
    compute stream, the worker-order AllReduce kernel on the comm stream, so the exposed-
    communication accounting (exposed_comm_time on cudaEvent intervals) runs on real comm-
    stream work. Not a multi-GPU number: the two ranks share one GPU."""
    from paper_2305_16121_b200.runtime import Context, LayerStack, ModelConfig, plan_for

    c = dict(cfg, layers=layers)
    mc = ModelConfig(dtype="bf16", hidden_dropout=0.1, attention_dropout=0.1, **c)
    out = {}
    for variant in ("Oases", "CrossPass", "Default"):
        ctx = Context(tp=2, local_workers=2)
        st = LayerStack(ctx, mc)
        st.init_random(1234)
        st.bind(plan_for(mc, variant))
        st.step(trace=True)
        rs = [st.step(trace=True) for _ in range(steps)]
        out[variant] = {"makespan_ms": statistics.mean(r.makespan for r in rs) * 1e3,
                        "comm_exposed_ms": statistics.mean(r.comm_exposed for r in rs) * 1e3,
                        "exposed_comm_pct": 100.0 * statistics.mean(r.comm_exposed / r.makespan for r in rs),
                        "comm_ops": sum(1 for e in rs[-1].events if e[1] == 1)}
        st.close()
        ctx.close()
    return {"config": f"{c['hidden']}h s{c['seq']} b{c['batch']} L{layers}, TMP=2 as 2 in-process workers",
            "variants": out}


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
    ap.add_argument("--no-extras", action="store_true", help="skip the C3 line and the emulated-TP2 exposure")
    ap.add_argument("--ref-batch", type=int, default=2, help="sequences per reference-arm sample")
    ap.add_argument("--trace-out", default="")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config])
    if args.layers:
        cfg["layers"] = args.layers
    if args.warmup < 3:
        args.warmup = 3
    world_env = os.environ.get("WORLD_SIZE")
    if args.impl == "reference":
        return run_reference(args, cfg)
    if args.gpus > 1 and world_env is None:
        return self_launch(args)  # one process per GPU
    world = int(world_env or "1")
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch one rank per GPU "
                         f"(torchrun --nproc-per-node {args.gpus}) or omit WORLD_SIZE to self-launch")

    import torch

    from paper_2305_16121_b200.runtime import Context, LayerStack, ModelConfig, plan_for, unique_id

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

    def max_over_ranks(v):
        if not dist:
            return v
        t = torch.tensor([v], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    for _ in range(args.warmup):
        stack.step(trace=False)
    barrier()
    launches0 = stack.kernel_launches()
    with ClockSampler(local) as clk:
        t0 = time.perf_counter()
        dev = [stack.step(trace=False).makespan for _ in range(args.steps)]
        wall = time.perf_counter() - t0
    barrier()
    # our kernels launched inside the timed region: counted by the library per issued
    # launch (a graph replay issues the kernels its capture counted once)
    launched = stack.kernel_launches() - launches0
    total = max_over_ranks(sum(dev))
    ms_per_step = total / args.steps * 1e3
    value = mc.batch / (total / args.steps)

    # one traced step: measured SimResult (exposed comm, compute busy)
    traced = stack.step(trace=True)
    if args.no_graph:
        launches_per_step = launched / args.steps
    else:
        before = stack.kernel_launches()
        stack.step(trace=True)
        launches_per_step = stack.kernel_launches() - before
    if args.trace_out and rank == 0:
        import paper_2305_16121_b200.tmpsim as tm

        tm.write_chrome_trace(traced.sim_result(), plan, args.trace_out)
        tm.write_svg_timeline(traced.sim_result(), plan, os.path.splitext(args.trace_out)[0] + ".svg")
    # live GEMM timings for the roofline, measured inside a replay of the captured step
    ks = stack.graph_kernel_stats() if not args.no_graph else None
    if ks is None:
        stack.set_kernel_timing(True)
        stack.step(trace=True)
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
    e2e_wall = max_over_ranks(time.perf_counter() - t0)
    e2e = {"value": mc.batch * args.steps / e2e_wall, "unit": "samples/s",
           "h2d_bytes_per_step": T * mc.hidden * 2, "d2h_bytes_per_step": 8}
    stack.close()
    ctx.close()

    # the north-star config at the target degree: real TMP=8 on 8 GPUs, else one rank's slice
    c3 = None
    if not args.no_extras and args.config == "c2":
        if tp == 8:
            c3 = c3_full_tp8(dist, rank, local, uid_fn=unique_id, reserve=reserve, sms=sms, steps=args.steps)
        elif tp == 1 and rank == 0:
            c3 = c3_rank_slice()
    emu = emulated_tp2(cfg) if (not args.no_extras and tp == 1 and rank == 0) else None

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
        "warmup": args.warmup, "ms_per_step": ms_per_step, "ms_per_step_sd": statistics.pstdev(dev) * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
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
        "roofline": {"bound": "tensor",
                     "kernel": "gemm_tc (tcgen05 linear-layer GEMMs, all launches of one graph-replayed step)",
                     "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak if peak else 0,
                     "peak_source": f"{PEAKS['source']} bf16_tflops_sustained",
                     "gemm_launches": ks["gemm_launches"], "traffic": traffic,
                     "traffic_source": "ncu --set full capture of the FC1 forward GEMM (profiles/r02_gemm_ncu.json)"},
        "gpu_launches": int(round(launches_per_step * args.steps)),
        "clocks": clk.summary(),
        "wall_s_timed": wall,
        "e2e": e2e,
    }
    if c3:
        line["c3_tp8"] = c3
    if emu:
        line["emulated_tp2_exposure"] = emu
    if not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline(cfg)
        except Exception as e:  # noqa: BLE001
            line["cpu_baseline"] = {"value": None, "error": str(e)}
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def c3_full_tp8(dist, rank, local, uid_fn, reserve, sms, steps=10, warmup=3):
    """C3 (h4096, 32 heads, s2048, b8, 24 layers) at TMP=8 over NCCL, Oases plan: the
    north-star target, measured when the bench runs on 8 GPUs."""
    from paper_2305_16121_b200.runtime import Context, LayerStack, ModelConfig, plan_for
    import torch

    cfg = dict(CONFIGS["c3"])
    obj = [uid_fn() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    mc = ModelConfig(dtype="bf16", hidden_dropout=0.1, attention_dropout=0.1, **cfg)
    ctx = Context(tp=8, rank=rank, device=local, unique_id=obj[0], nccl_max_ctas=reserve,
                  gemm_max_ctas=(sms - reserve) // 2 * 2)
    st = LayerStack(ctx, mc)
    st.init_random(1234)
    st.bind(plan_for(mc, "Oases"))
    st.capture_graph()
    for _ in range(warmup):
        st.step(trace=False)
    dist.barrier()
    torch.cuda.synchronize()
    ms = [st.step(trace=False).makespan * 1e3 for _ in range(steps)]
    t = torch.tensor([sum(ms)], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    tr = st.step(trace=True)
    st.close()
    ctx.close()
    mean = t.item() / steps
    tf = step_flops(cfg) / 8 / (mean * 1e-3) / 1e12
    return {"config": "c3 (h4096 a32 s2048 b8 L24), TMP=8 over NCCL", "value": cfg["batch"] / (mean * 1e-3),
            "unit": "samples/s", "ms_per_step": mean, "tflops_per_gpu": tf,
            "frac_of_sustained_peak": tf / PEAKS["bf16_tflops_sustained"],
            "exposed_comm_pct": 100.0 * tr.comm_exposed / tr.makespan if tr.makespan else 0.0}


if __name__ == "__main__":
    main()
