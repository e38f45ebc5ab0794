"""Multi-GPU parity of both decompositions (row e), gated on the device count (NCCL rejects
two ranks of one communicator on one GPU).  Each case launches
tests/mgpu_check.py under torchrun on 2 and (if present) 4 / 8 GPUs and requires the
decomposed run to equal the single-GPU run of the whole problem to 1e-12 (velocity shards
change only the order of the moment sum; the z-slab superposition is exact)."""
import json
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NDEV = torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.skipif(NDEV < 2, reason="needs >= 2 GPUs (NCCL: one rank per device)")
@pytest.mark.parametrize("decomp,case", [("velocity", "iso"), ("zslab", "iso"), ("velocity", "lbm")])
@pytest.mark.parametrize("G", [2, 4, 8])
def test_multi_gpu_decomposition_parity(decomp, case, G):
    if G > NDEV:
        pytest.skip("not enough GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={G}",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + G), os.path.join(ROOT, "tests", "mgpu_check.py"),
           decomp, case]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    line = [ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1]
    res = json.loads(line)
    assert res["err_f"] <= 1e-12 and res["err_w"] <= 1e-12, res
