"""One-line summaries of `ncu --set full` captures (key throughput metrics + stall-sample shares).

usage: python tools/ncu_full_summary.py cap1.ncu-rep [cap2.ncu-rep ...]
Reads each report with `ncu -i <rep> --page raw --csv` (the ncu of this image) and prints, per
kernel launch, the metrics the roofline and the DESIGN.md kernel notes quote."""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "lts__t_sector_hit_rate.pct",
        "lts__t_bytes.sum"]
STALL = "smsp__pcsamp_warps_issue_stalled_"


def summarise(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head = rows[0]
    units = rows[1]
    for r in rows[2:]:
        if len(r) != len(head):
            continue
        rec = dict(zip(head, r))
        unit = dict(zip(head, units))
        parts = [f"Kernel Name={rec.get('Kernel Name', '?').split('(')[0]}"]
        for k in KEYS:
            if k in rec and rec[k] != "":
                parts.append(f"{k}={rec[k]} {unit.get(k, '')}".rstrip())
        print(" ; ".join(parts))
        st = {}
        for k, v in rec.items():
            if k.startswith(STALL) and not k.endswith("_not_issued"):
                try:
                    st[k[len(STALL):]] = float(v.replace(",", ""))
                except ValueError:
                    pass
        tot = sum(st.values())
        if tot > 0:
            top = sorted(st.items(), key=lambda kv: -kv[1])[:6]
            print("   stall samples (share): " + ", ".join(f"{k} {v / tot:.2f}" for k, v in top))


if __name__ == "__main__":
    for rep in sys.argv[1:]:
        summarise(rep)
