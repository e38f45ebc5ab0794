"""Per-launch table (time, DRAM bytes) of the library's kernels from an ncu --csv launch list.

usage: python tools/ncu_launches.py launches.csv
(the list comes from `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
 -k regex:... --csv --log-file launches.csv <command>`; torch's own kernels are dropped)."""
import csv
import sys
from collections import defaultdict

OURS = ("sweep", "relax", "zslab", "lattice", "equilibrium", "check_state", "partial_moments", "source")

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, mi, vi, idi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
d = defaultdict(dict)
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].split("(")[0].replace("void ", "").replace("pdg::", "")
    if not any(o in name for o in OURS) or "at::" in name:
        continue
    d[(int(r[idi]), name)][r[mi]] = float(r[vi].replace(",", ""))
for (i, name), v in sorted(d.items()):
    t = v.get("gpu__time_duration.sum", 0)
    rd = v.get("dram__bytes_read.sum", 0)
    wr = v.get("dram__bytes_write.sum", 0)
    print(f"{i:5d} {name[:48]:48s} {t / 1e6:9.3f} ms  R {rd / 1e9:8.2f} GB  W {wr / 1e9:8.2f} GB  "
          f"{(rd + wr) / t if t else 0:8.1f} GB/s")
