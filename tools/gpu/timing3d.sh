# per-phase cycle counters of the D3Q15 sweeps (timing build, -DPDG_LAT_TIMING)
cp paper_1702_00169_b200/libpdg_timing.so paper_1702_00169_b200/libpdg.so
touch paper_1702_00169_b200/libpdg.so
python - <<'PY' > gpurun_out/timing3d.txt 2>&1
import sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_1702_00169_b200 import pdg
from pdg_inputs import lbm_config, w0_grid
cfg = lbm_config("D3Q15", 128, nu=2.0)
S = pdg.Solver(pdg.problem_from_config(cfg))
S.set_equilibrium(w0_grid(cfg, device="cuda").reshape(-1))
torch.cuda.synchronize()
S.transport(cfg.dt / 2)
torch.cuda.synchronize()
S.destroy()
PY
