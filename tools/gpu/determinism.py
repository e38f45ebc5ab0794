"""Repeated lattice steps at bench sizes must be bit-identical (a race in a cross-CTA hand-over
-- tagged words, per-warp row progress, segment halo flags -- would show as a difference)."""
import sys
import os
sys.path.insert(0, os.getcwd())
import torch
from paper_1702_00169_b200 import pdg
from pdg_inputs import lbm_config, w0_grid

REPS = int(sys.argv[1]) if len(sys.argv) > 1 else 20
for lat, N in (("D3Q15", 128), ("D3Q27", 96), ("D2Q9", 1024), ("D2Q9", 2048)):
    cfg = lbm_config(lat, N, nu=2.0)
    S = pdg.Solver(pdg.problem_from_config(cfg))
    w0 = w0_grid(cfg, device="cuda").reshape(-1)
    ref = None
    bad = 0
    for _ in range(REPS):
        S.set_equilibrium(w0)
        S.step(3)
        torch.cuda.synchronize()
        h = S.get_state().clone()
        if ref is None:
            ref = h
        elif not torch.equal(h, ref):
            bad += 1
    S.destroy()
    print(f"{lat} N={N}: {REPS} repeats of 3 M2 steps, {bad} differing", flush=True)
