"""One TMP rank's share of a north-star config on this GPU (collectives disabled):
the compute side of a TMP=t step at the target shapes, e.g. C3 (h4096, 32 heads,
s2048, b8, 24 layers) at t=8. Prints one JSON line with the measured per-rank
step time, its algorithmic TFLOP/s (SURVEY.md 8(d) step FLOPs / t) and the
fraction of the measured sustained bf16 peak; the AllReduce side is the
calibrated simulation of tools/plan_c5.py.

    python tools/rank_slice.py [--config c3] [--tp 8] [--layers 24] [--steps 5]
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402
from paper_2305_16121_b200.runtime import Context, LayerStack, ModelConfig, plan_for  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3", choices=sorted(bench.CONFIGS))
    ap.add_argument("--tp", type=int, default=8)
    ap.add_argument("--layers", type=int, default=24)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--variant", default="Oases")
    args = ap.parse_args()
    cfg = dict(bench.CONFIGS[args.config])
    cfg["layers"] = args.layers
    mc = ModelConfig(dtype="bf16", hidden_dropout=0.1, attention_dropout=0.1, **cfg)
    ctx = Context(tp=args.tp, comm_disabled=True)
    st = LayerStack(ctx, mc)
    st.init_random(1234)
    st.bind(plan_for(mc, args.variant))
    st.capture_graph()
    for _ in range(3):
        st.step(trace=False)
    ms = [st.step(trace=False).makespan * 1e3 for _ in range(args.steps)]
    t = statistics.median(ms)
    tf = bench.step_flops(cfg, args.variant) / args.tp / (t * 1e-3) / 1e12
    print(json.dumps({"config": args.config, "tp": args.tp, "layers": args.layers, "variant": args.variant,
                      "rank_step_ms": t, "rank_tflops": tf,
                      "frac_of_sustained_peak": tf / bench.PEAKS["bf16_tflops_sustained"],
                      "samples_per_s_if_comm_hidden": cfg["batch"] / (t * 1e-3),
                      "peak_memory_bytes": st.step(trace=True).peak_memory}), flush=True)


if __name__ == "__main__":
    main()
