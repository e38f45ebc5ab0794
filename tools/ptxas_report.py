"""Summarise `nvcc -Xptxas -v` output: kernel, registers, spills, smem (reads stdin)."""
import re
import subprocess
import sys

cur = None
rows = []
for line in sys.stdin:
    m = re.search(r"Compiling entry function '([^']+)'", line)
    if m:
        cur = {"name": m.group(1), "regs": None, "spill": "", "smem": ""}
        rows.append(cur)
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        cur["spill"] = f"{m.group(1)}/{m.group(2)}"
    m = re.search(r"Used (\d+) registers", line)
    if m:
        cur["regs"] = int(m.group(1))
    m = re.search(r"(\d+) bytes smem", line)
    if m:
        cur["smem"] = m.group(1)
names = [r["name"] for r in rows]
try:
    dem = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.split("\n")
except Exception:
    dem = names
pat = sys.argv[1] if len(sys.argv) > 1 else ""
for r, d in zip(rows, dem):
    d = d.replace("pdg::", "").split("(")[0]
    if pat in d:
        print(f"{d[:70]:70s} regs={r['regs']} spill(st/ld)={r['spill']} smem={r['smem']}")
