# one-cell axes through the config pipeline vs the fuzz pipeline
import sys; sys.path.insert(0, 'tests'); sys.path.insert(0, '.')
import numpy as np
from oracle import oracle as O
from paper_1702_00169_b200 import pdg
from pdg_inputs import CONFIGS, velocity_set, w0_grid, wb_grid
from gpu_helpers import rel_maxnorm, to_np, to_dev, full_grid_to_planes
import test_gpu_parity as T

def run(ncell, p, init):
    dim = len(ncell); m = dim + 1; lam = 3.5
    vel, comp = velocity_set(dim, m, lam)
    hi = [1.0 * c / ncell[0] for c in ncell] + [1.0] * (3 - dim)
    h = 1.0 / ncell[0]; dt = 1.0 * h / lam
    pb = pdg.make_problem(dim, list(ncell), p, m, vel, comp, lam, pdg.PDG_FLUX_ISOTHERMAL, [1.0], dt, hi=tuple(hi))
    ob = O.Problem(dim, list(ncell), p, vel, comp, m, lam, pdg.PDG_FLUX_ISOTHERMAL, [1.0], dt, hi=list(hi))
    shape = ob.grid_shape(); nv = ob.nv
    rng = np.random.default_rng(5)
    if init == "random":
        f = (1.0 + 0.05 * (rng.random((nv,) + shape) - 0.5)) / (2 * dim)
        fb = (1.0 + 0.05 * rng.random((nv,) + shape)) / (2 * dim)
    else:  # equilibrium of a smooth state
        w = np.zeros((m,) + shape); w[0] = 1.0 + 0.1 * rng.random(shape); w[1] = 0.05
        f, fb = O.initial_data(ob, w, w.copy())
    out = []
    for flags in (0, pdg.PDG_NO_SMALL):
        pbb = pdg.make_problem(dim, list(ncell), p, m, vel, comp, lam, pdg.PDG_FLUX_ISOTHERMAL, [1.0], dt, hi=tuple(hi), flags=flags)
        S = pdg.Solver(pbb)
        class _C: pass
        cv = _C(); cv.dim, cv.grid_shape = dim, shape
        S.set_state(to_dev(f), to_dev(full_grid_to_planes(cv, fb, S.sizes.plane_stride)))
        S.step(1)
        out.append(rel_maxnorm(to_np(S.get_state(), f.shape), O.m2_run(ob, f, fb, 1)))
        S.destroy()
    print(ncell, p, init, ['%.2e' % e for e in out], flush=True)

for nc in ([1, 1, 1], [2, 1, 1], [1, 2, 1], [1, 1, 2], [2, 2, 2], [1, 1], [3, 1], [1, 3]):
    for p in (2, 3):
        for init in ("random", "eq"):
            run(nc, p, init)
# config pipeline, N = 1 and 2
for key, N in [(4, 1), (4, 2), (3, 1), (1, 1), (2, 1)]:
    cfg = CONFIGS[key].resized(N)
    if key != 1: cfg = cfg.stabilised()
    pbo, f0, fbg = T.seeded_equilibrium(cfg)
    S = T.gpu_with_state(cfg, f0, fbg); S.step(1)
    print('cfg', key, N, '%.2e' % rel_maxnorm(to_np(S.get_state(), f0.shape), O.m2_run(pbo, f0, fbg, 1)), 'L', cfg.grid_shape, flush=True)
    S.destroy()
