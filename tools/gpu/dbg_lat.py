"""Debug helper: one T2 of a lattice set at a given size (exit code != 0 on a CUDA fault)."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_1702_00169_b200 import pdg
from pdg_inputs import lbm_config, w0_grid
lat, N, nsteps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
cfg = lbm_config(lat, N, nu=2.0)
S = pdg.Solver(pdg.problem_from_config(cfg, flags=pdg.PDG_SYNC_ERRORS))
S.set_equilibrium(w0_grid(cfg, device="cuda").reshape(-1))
if nsteps == 0:
    S.transport(cfg.dt)
else:
    S.step(nsteps)
torch.cuda.synchronize()
print(lat, N, nsteps, "ok", flush=True)
