"""GPU parity of the source step S2 and the Strang scheme M2s (SURVEY §8(f) NEXT-3:
P:456-463, Euler with gravity P:1101-1194) against the CPU oracle.

The oracle solves the CN source equation by Picard iteration; the CUDA
path applies the closed form f + h g(f) fused with the collision (S2 C2 S2 in one pass
over f).  Bar: <= 1e-13 for one operator, <= 1e-12 for M2s steps (reading C17).
"""
from dataclasses import replace

import numpy as np
import pytest

from oracle import oracle as O
from pdg_inputs import gravity_config, lbm_config, random_state, w0_grid
from gpu_helpers import lattice_planes, make_solver, oracle_problem, rel_maxnorm, to_dev, to_np

pytestmark = pytest.mark.gpu


def _cfgs():
    return [gravity_config(10, dt=0.006, t_max=0.03), replace(lbm_config("D3Q19", 5), gravity=(0.3, 0.0, -1.0)),
            replace(lbm_config("D3Q27", 4), gravity=(0.0, 0.5, 0.2)),
            replace(lbm_config("D3Q15", 4), gravity=(0.0, 0.0, -2.0))]


@pytest.mark.parametrize("k", range(4))
def test_source_operator_parity(k):
    from paper_1702_00169_b200 import pdg
    cfg = _cfgs()[k]
    f = random_state(cfg, 21, 0.5).numpy()
    S = make_solver(cfg, scheme=pdg.PDG_SCHEME_M2S)
    S.set_state(to_dev(f), to_dev(np.zeros(S.sizes.fb_elems)))
    S.source(0.3)
    got = to_np(S.get_state(), f.shape)
    pb = oracle_problem(cfg)
    ref = np.ascontiguousarray(f.copy())
    O.source(pb, ref, 0.3)
    S.destroy()
    assert rel_maxnorm(got, ref) <= 1e-13


@pytest.mark.parametrize("k", range(4))
@pytest.mark.parametrize("tau_dt", [0.0, 0.4])
def test_m2s_scheme_parity(k, tau_dt):
    """Free-running M2s steps from the equilibrium of the initial state (readings C12/C13)."""
    from paper_1702_00169_b200 import pdg
    cfg = _cfgs()[k]
    steps = 4
    tau = tau_dt * cfg.dt
    w0 = w0_grid(cfg)
    S = make_solver(cfg, scheme=pdg.PDG_SCHEME_M2S, tau=tau)
    S.set_equilibrium(w0.reshape(-1).cuda())
    S.step(steps)
    got = to_np(S.get_state(), (cfg.nv,) + cfg.grid_shape)
    pb = oracle_problem(cfg, tau=tau)
    f0, fb = O.initial_data(pb, w0.numpy(), w0.numpy())
    ref = O.scheme_run(pb, f0, fb, steps, "m2s")
    S.destroy()
    assert rel_maxnorm(got, ref) <= 1e-12


def test_gravity_order_on_gpu():
    """The Euler-with-gravity time-order study (Fig. euler_gravity_order) run through the C-ABI:
    relative L2 error of w vs the analytic fluid at rest, t_max = 0.12, slopes in [1.75, 2.25]."""
    from paper_1702_00169_b200 import pdg
    errs = []
    for dt in [0.012, 0.006, 0.003, 0.0015]:
        cfg = gravity_config(16, dt=dt)
        w0 = w0_grid(cfg)
        S = make_solver(cfg, scheme=pdg.PDG_SCHEME_M2S)
        S.set_equilibrium(w0.reshape(-1).cuda())
        S.step(cfg.steps)
        w = to_np(S.moments(), (cfg.m,) + cfg.grid_shape)
        S.destroy()
        w0n = w0.numpy()
        errs.append(float(np.sqrt(np.sum((w - w0n) ** 2) / np.sum(w0n ** 2))))
    slopes = [np.log2(errs[i] / errs[i + 1]) for i in range(3)]
    assert all(1.75 <= s <= 2.25 for s in slopes), (errs, slopes)
