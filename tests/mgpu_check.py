"""Multi-GPU parity check, launched by tests/test_gpu_multi.py under torchrun (one rank per GPU).

Every rank runs the same small problem decomposed over the ranks (velocity shards with one
NCCL sum of the moments per collision, or the exact z-slab decomposition with the NCCL
all-gather of carry planes) and compares its share with a single-GPU run of the whole
problem on its own device.  Rank 0 prints one JSON line with the worst relative error.
"""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1702_00169_b200 import dist as pdist  # noqa: E402
from paper_1702_00169_b200 import pdg  # noqa: E402
from pdg_inputs import CONFIGS, lbm_config, w0_grid, wb_grid  # noqa: E402


def main():
    decomp = sys.argv[1]
    case = sys.argv[2]
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    rank, world = dist.get_rank(), dist.get_world_size()
    cfg = {"iso": CONFIGS[3].resized(8).stabilised(), "lbm": lbm_config("D3Q27", 6)}[case]
    steps = 3
    w0 = w0_grid(cfg)
    wb = wb_grid(cfg, w0)
    # reference: the whole problem on this device
    R = pdg.Solver(pdg.problem_from_config(cfg), device=dev)
    R.set_equilibrium(w0.reshape(-1).to(dev), wb.reshape(-1).to(dev))
    R.step(steps)
    ref_f = R.get_state().view((cfg.nv,) + cfg.grid_shape)
    ref_w = R.moments().view((cfg.m,) + cfg.grid_shape)
    # decomposed
    d = pdg.PDG_DECOMP_ZSLAB if decomp == "zslab" else pdg.PDG_DECOMP_VELOCITY
    S = pdist.sharded_solver(cfg, dev, decomposition=d)
    sz = S.sizes
    if d == pdg.PDG_DECOMP_ZSLAB:
        z0 = int(sz.cell_begin) * cfg.n
        z1 = z0 + int(sz.cell_count) * cfg.n
        S.set_equilibrium(w0[:, z0:z1].reshape(-1).to(dev).contiguous(), wb[:, z0:z1].reshape(-1).to(dev).contiguous())
        S.step(steps)
        got = S.get_state().view((cfg.nv, z1 - z0) + cfg.grid_shape[1:])
        ref = ref_f[:, z0:z1]
        w = S.moments().view((cfg.m, z1 - z0) + cfg.grid_shape[1:])
        wref = ref_w[:, z0:z1]
    else:
        v0, nvl = int(sz.v_begin), int(sz.nv_local)
        S.set_equilibrium(w0.reshape(-1).to(dev), wb.reshape(-1).to(dev))
        S.step(steps)
        got = S.get_state().view((nvl,) + cfg.grid_shape)
        ref = ref_f[v0:v0 + nvl]
        w = S.moments().view((cfg.m,) + cfg.grid_shape)
        wref = ref_w
    err = float(((got - ref).abs().max() / ref.abs().max()).item())
    errw = float(((w - wref).abs().max() / wref.abs().max()).item())
    t = torch.tensor([err, errw], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({"decomp": decomp, "case": case, "world": world, "err_f": t[0].item(),
                          "err_w": t[1].item()}), flush=True)
    S.destroy()
    R.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
