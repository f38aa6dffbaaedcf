"""Summarise `ncu --set full` captures of single GEMM / attention launches into
profiles/ncu_summary.json (the `traffic` field of bench.py's roofline object).

usage: python tools/ncu_gemm_summary.py OUT.json NAME=REP[#i]:M,N,K,OUT_BYTES [...]
  REP        an .ncu-rep holding one launch of the kernel (tools/gemm_one.py);
             REP#i selects launch i of a multi-launch capture
  M,N,K      GEMM shape; algorithmic bytes = 2*(M*K + N*K) + OUT_BYTES*M*N
The first entry is the dominant kernel bench.py reports.
"""
import csv
import io
import json
import subprocess
import sys

WANT = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_active_pct",
    "lts__t_bytes.sum": "l2_bytes",
    "sm__cycles_elapsed.avg.per_second": "sm_clock",
    "launch__grid_size": "grid",
    "launch__registers_per_thread": "registers",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
         "second": 1, "us": 1e-6, "ns": 1e-9, "ms": 1e-3, "%": 1, "": 1, "cycle/second": 1, "cycle/nsecond": 1e9, "cycle/usecond": 1e6,
         "Ghz": 1e9, "Mhz": 1e6, "hz": 1, "register/thread": 1, "block": 1}


def raw(rep):
    out = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], text=True)
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    res = []
    for v in rows[2:]:
        d = {}
        for i, k in enumerate(h):
            if k in WANT and v[i] not in ("", "n/a"):
                d[WANT[k]] = float(v[i].replace(",", "")) * SCALE.get(u[i], 1)
        d["kernel"] = v[h.index("Kernel Name")][:120]
        res.append(d)
    return res


def main():
    out_path = sys.argv[1]
    entries = []
    for arg in sys.argv[2:]:
        name, rest = arg.split("=", 1)
        rep, shape = rest.split(":")
        M, N, K, ob = (int(x) for x in shape.split(","))
        idx = None
        if "#" in rep:  # REP#i: the i-th launch of a multi-launch capture
            rep, i = rep.split("#")
            idx = int(i)
        launches = raw(rep)
        for d in (launches if idx is None else [launches[idx]]):
            alg = 2 * (M * K + N * K) + ob * M * N
            traffic = d.get("dram_read", 0) + d.get("dram_write", 0)
            e = {"name": name, "shape": [M, N, K], "out_bytes_per_elem": ob, "algorithmic_bytes": alg,
                 "dram_bytes": traffic, "traffic_over_algorithmic": traffic / alg,
                 "tflops": 2 * M * N * K / d["duration"] / 1e12 if d.get("duration") else None, **d}
            entries.append(e)
    top = entries[0]
    summary = {
        "source": "ncu --set full --clock-control none (cold cache, one launch each); tools/ncu_gemm_summary.py",
        "dominant_kernel": top["kernel"],
        "dominant_dram_bytes_per_launch": top["dram_bytes"],
        "dominant_algorithmic_bytes_per_launch": top["algorithmic_bytes"],
        "note": ("traffic = dram__bytes_read.sum + dram__bytes_write.sum of the dominant tcgen05 GEMM launch "
                 "(FC1 forward shape of C2); algorithmic bytes = A + B + C once"),
        "launches": entries,
    }
    with open(out_path, "w") as f:
        json.dump(summary, f, indent=1)
    for e in entries:
        print(f"{e['name']:8s} {e['duration']*1e6:8.1f} us  {e['tflops'] or 0:7.1f} TF/s  dram {e['dram_bytes']/1e6:7.1f} MB "
              f"(alg {e['algorithmic_bytes']/1e6:7.1f} MB)  tensor {e.get('tensor_active_pct', 0):5.1f}%")


if __name__ == "__main__":
    main()
