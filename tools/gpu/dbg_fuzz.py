import sys, os, math
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
from oracle import oracle as O
from paper_1702_00169_b200 import pdg
from pdg_inputs import lattice
from gpu_helpers import lattice_planes, rel_maxnorm, to_dev, to_np

def run(name, ncell, p, nu, steps, hi, transport_only=False, perturb=0.0):
    dim = 3
    lam = 1.0
    vel, wts = lattice(name, lam)
    fparams = [lam / math.sqrt(3.0)] + list(wts)
    h = min(hi[d] / ncell[d] for d in range(dim))
    dt = nu * h / lam
    pb = pdg.make_problem(dim, ncell, p, dim + 1, vel, [0] * len(vel), lam, pdg.PDG_FLUX_LBM, fparams, dt, hi=tuple(hi))
    ob = O.Problem(dim, ncell, p, vel, [0] * len(vel), dim + 1, lam, 3, fparams, dt, hi=list(hi))
    rng = np.random.default_rng(1)
    shape = ob.grid_shape(); nv = ob.nv
    f = (1.0 + 0.2 * (rng.random((nv,) + shape) - 0.5)) / nv
    fb = (1.0 + 0.2 * rng.random((nv,) + shape)) / nv
    S = pdg.Solver(pb)
    class C: pass
    cv = C(); cv.dim, cv.grid_shape = dim, shape; cv.velocities = lambda: (ob.vel.tolist(), None)
    S.set_state(to_dev(f), to_dev(lattice_planes(cv, fb, S.sizes.plane_stride)))
    if transport_only:
        S.transport(dt); got = to_np(S.get_state(), f.shape)
        fc = ob.grid_to_cells(f); O.t2_all(ob, dt, fc, ob.grid_to_cells(fb)); ref = ob.cells_to_grid(fc)
    else:
        S.step(steps); got = to_np(S.get_state(), f.shape); ref = O.scheme_run(ob, f, fb, steps, "m2")
    S.destroy()
    # oracle self-sensitivity: perturb f by 1e-15 relative and rerun
    f2 = f * (1.0 + 1e-15 * (rng.random(f.shape) - 0.5))
    if transport_only:
        fc2 = ob.grid_to_cells(f2); O.t2_all(ob, dt, fc2, ob.grid_to_cells(fb)); ref2 = ob.cells_to_grid(fc2)
    else:
        ref2 = O.scheme_run(ob, f2, fb, steps, "m2")
    print(name, ncell, p, nu, steps, "T" if transport_only else "M2", "gpu-vs-oracle %.2e" % rel_maxnorm(got, ref), "oracle twin %.2e" % rel_maxnorm(ref2, ref), flush=True)

hi = (1.0 + 0.0, 1.0, 1.0)
import itertools
for nu in (-0.123, 0.123):
    for p in (2, 3):
        run("D3Q15", [7, 4, 2], p, nu, 2, (1.6, 0.9, 1.3))
run("D3Q15", [7, 4, 2], 3, -0.123, 1, (1.6, 0.9, 1.3), transport_only=True)
run("D3Q19", [7, 4, 2], 3, -0.123, 1, (1.6, 0.9, 1.3), transport_only=True)
