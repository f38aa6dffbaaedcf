"""Assemble the committed profiles/r02_* summaries from one tools/profile_round2.sh
run (gpurun_out/final) plus a bench line (default gpurun_out/b3/bench2.json).

    python tools/assemble_r02_profiles.py [final_dir] [bench_json]
"""
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
F = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "final")
BENCH = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out", "b3", "bench2.json")
P = os.path.join(ROOT, "profiles")
peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
HBM, BURST = peaks["hbm_gbs"], peaks["bf16_tflops"]


def load(name):
    return json.load(open(os.path.join(F, name)))


def short(k):
    return k.replace("void unnamed>::", "").replace("unnamed>::", "")


# LayerNorm kernels: algorithmic bytes = tensors read and written once (bf16)
ln = {"source": "ncu --set full --clock-control none, one cold launch each (tools/lnp_one.py: plain LN forward, "
                "bias-dropout-residual + LN forward p=0.1, LN backward with residual accumulate + dgamma/dbeta "
                "partials, finalize); tools/profile_round2.sh",
      "hbm_peak_gbs": HBM, "hbm_peak_source": "MEASURED_PEAKS.json hbm_gbs (burst copy; kernels timed alone)",
      "note": "algorithmic bytes = the tensors the kernel must read and write once (bf16); ncu dram__bytes_write "
              "under-counts writes still in L2 at kernel end, so the fraction uses algorithmic bytes / duration",
      "shapes": {}}
for tag, (T, h) in (("c2_sub_batch", (4096, 2048)), ("c3_tp8_rank", (8192, 4096))):
    t = T * h * 2 / 1e6
    alg = [2 * t, 4 * t + T * h / 8 / 1e6, 4 * t, None]  # fwd, bdr (+keep bits), bwd (x, dy, dx r/w), finalize
    ks = []
    for k, a in zip(load(f"ncu_lnp_{T}x{h}.json"), alg):
        e = {"kernel": short(k["kernel"]), "time_us": k["time_us"], "dram_read_mb": k["dram_read_mb"],
             "dram_write_mb": k["dram_write_mb"], "issue_active_pct": k["issue_active_pct"],
             "registers": k["registers"], "grid": k["grid"]}
        if a:
            e.update(algorithmic_mb=round(a, 2), achieved_gbs=round(a * 1e3 / k["time_us"], 1),
                     frac_of_hbm=round(a * 1e3 / k["time_us"] / HBM, 3))
        ks.append(e)
    ln["shapes"][tag] = {"T_sub": T, "hidden": h, "kernels": ks}
json.dump(ln, open(os.path.join(P, "r02_hbm_ncu.json"), "w"), indent=1)

# attention: algorithmic FLOPs, causal (fwd 4 s^2 d / 2, dK/dV 8 s^2 d / 2 per (sample, head))
att = {"source": "ncu --set full --clock-control none, one cold launch each (tools/attn_one.py); "
                 "tools/profile_round2.sh", "burst_peak_tflops": BURST, "cases": {}}
for tag, fn, (n, hl, s) in (("c2_sub_batch_cached_bits", "ncu_attn_c2_cached.json", (4, 16, 1024)),
                            ("c2_sub_batch_philox_in_kernel", "ncu_attn_c2_philox.json", (4, 16, 1024)),
                            ("c3_tp8_rank_sub_batch_cached_bits", "ncu_attn_c3rank_cached.json", (4, 4, 2048))):
    ks = []
    for k in load(fn):
        mult = 8 if "dkdv" in k["kernel"] else 4
        gf = mult * n * hl * s * s * 128 / 2 / 1e9
        ks.append({**{x: k[x] for x in ("time_us", "tensor_pipe_pct", "issue_active_pct", "xu_pct", "dram_read_mb",
                                        "dram_write_mb", "sm_ghz", "grid")},
                   "kernel": short(k["kernel"]).split("(")[0], "algorithmic_gflop": round(gf, 2),
                   "achieved_tflops": round(gf / k["time_us"] * 1e3, 1),
                   "frac_of_burst_peak": round(gf / k["time_us"] * 1e3 / BURST, 3)})
    att["cases"][tag] = {"samples": n, "heads_local": hl, "seq": s, "head_dim": 128, "dropout": 0.1, "kernels": ks}
json.dump(att, open(os.path.join(P, "r02_attention_ncu.json"), "w"), indent=1)

# GEMMs (bench.py reads the FC1 capture's DRAM bytes for the roofline `traffic`)
gm = {"source": "ncu --set full --clock-control none (tools/gemm_one.py FC1 forward 4096x8192x2048; "
                "tools/epi_one.py FC2 dgrad with the dGeLU epilogue + FC2 wgrad)",
      "kernels": load("ncu_gemm_fc1.json") + load("ncu_gemm_epi.json")}
json.dump(gm, open(os.path.join(P, "r02_gemm_ncu.json"), "w"), indent=1)

# launch lists
shutil.copy(os.path.join(F, "launches_bench.csv"), os.path.join(P, "r02_launches_bench.csv"))
hdr = ("ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none "
       "launch list of 'bench.py --steps 1 --warmup 3' (C2 L24, cold-cache serialised per launch: shares, not "
       "absolutes); second half of the launches (= the timed region's graph replay)\n")
tab = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "launch_table.py"),
                      os.path.join(F, "launches_bench.csv")], capture_output=True, text=True).stdout
open(os.path.join(P, "r02_launch_summary.txt"), "w").write(hdr + tab)
tab = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "launch_table.py"),
                      os.path.join(F, "c3_tp8_launches.csv")], capture_output=True, text=True).stdout
open(os.path.join(P, "r02_c3_tp8_launch_summary.txt"), "w").write(
    "C3 TMP=8 rank slice, 2 layers, eager step, ncu launch list (tools/profile_slice.py), last step\n" + tab)
for c in ("c3", "c4"):
    line = [x for x in open(os.path.join(F, f"{c}_tp8.log")) if x.startswith("{")][-1]
    open(os.path.join(P, f"r02_{c}_tp8_rank_slice.json"), "w").write(line)
shutil.copy(BENCH, os.path.join(P, "r02_bench.json"))
print("ok")
