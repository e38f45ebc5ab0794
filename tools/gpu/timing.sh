cp paper_1702_00169_b200/libpdg_timing.so paper_1702_00169_b200/libpdg.so
python - <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_1702_00169_b200 import pdg
from pdg_inputs import lbm_config, w0_grid
for lat in ("D3Q15", "D3Q19"):
    cfg = lbm_config(lat, 128, nu=2.0)
    S = pdg.Solver(pdg.problem_from_config(cfg))
    S.set_equilibrium(w0_grid(cfg, device="cuda").reshape(-1))
    S.transport(cfg.dt)
    torch.cuda.synchronize()
    S.destroy()
PY
