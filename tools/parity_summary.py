"""Markdown summary of the full-size parity records (profiles/r02_parity/parity_long_*.json,
written by tests/test_gpu_long.py on the GPU box)."""
import glob
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def ranges(xs):
    """[86, 87, 88, 90] -> '86-88, 90'"""
    out, i = [], 0
    while i < len(xs):
        j = i
        while j + 1 < len(xs) and xs[j + 1] == xs[j] + 1:
            j += 1
        out.append(str(xs[i]) if i == j else f"{xs[i]}–{xs[j]}")
        i = j + 1
    return ", ".join(out) or "—"


def fmt(x):
    return "—" if x is None else (f"{x:.1e}" if isinstance(x, float) else str(x))


def main(d=os.path.join(ROOT, "profiles", "r02_parity")):
    rows = []
    order = ["cfg2", "cfg3", "cfg4", "cfg5", "cfg2s", "cfg3s", "cfg4s", "cfg5s"]
    for name in order:
        path = os.path.join(d, f"parity_long_{name}.json")
        if not os.path.exists(path):
            continue
        r = json.load(open(path))
        ps = r["per_step"]
        rs = [e["resync_f"] for e in ps if "resync_f" in e and e.get("oracle_nonphysical_in", 0) == 0]
        rs_bad = [e["step"] for e in ps if "resync_f" in e and e.get("oracle_nonphysical_in", 0) > 0]
        free = [e["free_f"] for e in ps if "free_f" in e]
        # amplification of a 1e-13 twin perturbation up to the last step whose state is physical
        phys = [e for e in ps if e.get("nonphysical_gpu", 0) == 0 and e.get("nonfinite_oracle", 0) == 0]
        twin = [e.get("gpu_twin_amplification") for e in phys if "gpu_twin_amplification" in e]
        otw = [e.get("oracle_twin_amplification") for e in phys if "oracle_twin_amplification" in e]
        last_phys = phys[-1]["step"] if phys else None
        first_bad = next((e["step"] for e in ps if e.get("nonphysical_gpu", 0) > 0), None)
        last = ps[-1]
        rows.append([name, r["N"], r["p"], r["lambda"], r["steps"], len(rs), fmt(max(rs) if rs else None),
                     ranges(rs_bad),
                     fmt(free[-1] if free else None), fmt(r.get("fused_free_f")),
                     (r.get("last_step_finite_and_agree_1e-12") if free else
                      (r["steps"] if (r.get("fused_free_f") or 1.0) <= 1e-12 else None)),
                     fmt(twin[-1] if twin else r.get("gpu_twin_amplification_final")),
                     fmt(otw[-1] if otw else None), fmt(last_phys if twin else r["steps"]), fmt(first_bad), r.get("stopped_at_step") or "—",
                     f"{r['oracle_seconds'] / 60:.1f}"])
    hdr = ["case", "N", "p", "λ", "steps", "re-synced steps (physical input)", "max re-synced rel err f",
           "re-synced steps with non-physical input", "free-running rel err f (last step, lockstep)",
           "one pdg_step(steps) call rel err f", "last step free-running <= 1e-12",
           "GPU twin amplification", "oracle twin amplification", "at step (last physical)", "first non-physical step",
           "oracle stopped (non-finite)", "oracle min"]
    out = ["| " + " | ".join(hdr) + " |", "|" + "---|" * len(hdr)]
    out += ["| " + " | ".join(str(c) for c in r) + " |" for r in rows]
    print("\n".join(out))


if __name__ == "__main__":
    main(*sys.argv[1:])
