"""Registers and spills per kernel from an nvcc -Xptxas -v log: python tools/ptxas_summary.py log [filter]"""
import re
import subprocess
import sys

txt = open(sys.argv[1]).read()
flt = sys.argv[2] if len(sys.argv) > 2 else ""
cur = None
out = {}
for line in txt.splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", line) or re.search(r"Function properties for (\S+)", line)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        out.setdefault(cur, {})["spill"] = int(m.group(1)) + int(m.group(2))
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        out.setdefault(cur, {})["regs"] = int(m.group(1))
names = list(out)
dem = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.splitlines()
for n, d in zip(names, dem):
    if flt in d:
        d = re.sub(r"oases::\(anonymous namespace\)::", "", d)
        print(f"regs {out[n].get('regs', '?'):>4} spill {out[n].get('spill', 0):>4}  {d[:110]}")
