"""Key metrics of every kernel in an ncu --set full report (.ncu-rep), as JSON:
time, DRAM bytes, achieved DRAM GB/s, tensor-pipe / issue / XU utilisation.

    python tools/ncu_kernel_summary.py report.ncu-rep [algorithmic_bytes_by_kernel_substring=...]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "time_us": ("gpu__time_duration.sum", 1e-3),
    "dram_read_mb": ("dram__bytes_read.sum", None),
    "dram_write_mb": ("dram__bytes_write.sum", None),
    "sm_ghz": ("sm__cycles_elapsed.avg.per_second", None),
    "tensor_pipe_pct": ("sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active", 1),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
    "xu_pct": ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", 1),
    "dram_throughput_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "achieved_occupancy_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    "registers": ("launch__registers_per_thread", 1),
}
UNIT = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3,
        "Ghz": 1.0, "Mhz": 1e-3, "hz": 1e-9}


def main():
    rep = sys.argv[1]
    alg = {}
    for a in sys.argv[2:]:
        k, v = a.split("=")
        alg[k] = float(v)
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(h, r))
        u = dict(zip(h, units))
        e = {"kernel": d.get("Kernel Name", "")[:120], "grid": d.get("Grid Size"), "block": d.get("Block Size")}
        for key, (m, _) in KEYS.items():
            if m in d and d[m] not in ("", "n/a"):
                v = float(d[m].replace(",", ""))
                unit = u.get(m, "")
                if key == "time_us":
                    v *= {"nsecond": 1e-3, "usecond": 1, "msecond": 1e3, "second": 1e6}.get(unit, 1e-3)
                elif key.endswith("_mb"):
                    v *= {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1, "Gbyte": 1e3}.get(unit, 1e-6)
                elif key == "sm_ghz":
                    v *= {"hz": 1e-9, "Khz": 1e-6, "Mhz": 1e-3, "Ghz": 1}.get(unit, 1e-9)
                e[key] = round(v, 3)
        if "time_us" in e and "dram_read_mb" in e:
            e["dram_gbs"] = round((e["dram_read_mb"] + e.get("dram_write_mb", 0)) / e["time_us"] * 1e3, 1)
        for k, v in alg.items():
            if k in e["kernel"] and "time_us" in e:
                e["algorithmic_mb"] = v
                e["algorithmic_gbs"] = round(v / e["time_us"] * 1e3, 1)
        res.append(e)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
