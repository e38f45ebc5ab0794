"""GPU parity of the lattice velocity sets: D2Q9 and
D3Q15/19/27 with the isothermal LBM equilibrium, against the CPU oracle.

The oracle assembles the full eq DG_reduit blocks of each velocity, orders cells with
Kahn's algorithm on the dependency graph and solves every cell with a
dense LU; the CUDA path applies the pre-inverted dense (p+1)^d block along diagonal
wavefronts (pdg_lattice.cuh).  Bar: <= 1e-13 for one operator, <= 1e-12 for M2 steps
(relative max-norm, reading C17).  PDG_LATTICE_WARPS forces one warp per CTA so that
the cross-CTA hand-over (global traces + progress flags) runs on small grids.
"""
import os

import numpy as np
import pytest
import torch

from oracle import oracle as O
from pdg_inputs import lbm_config, random_state, w0_grid, wb_grid
from gpu_helpers import lattice_planes, make_solver, oracle_problem, rel_maxnorm, to_dev, to_np

pytestmark = pytest.mark.gpu

TOL_OP = 1e-13
TOL_STEP = 1e-12


@pytest.fixture
def warps(request):
    old = os.environ.get("PDG_LATTICE_WARPS")
    if request.param:
        os.environ["PDG_LATTICE_WARPS"] = request.param
    else:
        os.environ.pop("PDG_LATTICE_WARPS", None)
    yield request.param
    if old is None:
        os.environ.pop("PDG_LATTICE_WARPS", None)
    else:
        os.environ["PDG_LATTICE_WARPS"] = old


def cases():
    return [
        ("D2Q9", 37, 2), ("D2Q9", 8, 1), ("D2Q9", 9, 3),
        ("D3Q15", 5, 2), ("D3Q19", 5, 2), ("D3Q27", 5, 2),
        ("D3Q19", 4, 3), ("D3Q27", 3, 1), ("D3Q15", 33, 2),
    ]


def random_lattice_inputs(cfg, seed):
    f = random_state(cfg, seed, 0.5).numpy()
    rng = np.random.default_rng(seed + 7)
    fb_full = rng.random((cfg.nv,) + cfg.grid_shape) / cfg.nv
    return f, fb_full


@pytest.mark.parametrize("warps", [None, "1,1", "2,2"], indirect=True)
@pytest.mark.parametrize("lat,N,p", cases())
@pytest.mark.parametrize("dtp_nu", [0.5, -0.05, 2.0])
def test_lattice_transport_parity(lat, N, p, dtp_nu, warps):
    """One T2(dt') of every velocity (rows a1/a3 for lattice sets) == the oracle's Kahn sweep."""
    if warps and N < 30 and lat != "D2Q9":
        pytest.skip("hand-over variants are exercised on the larger grids")
    cfg = lbm_config(lat, N, p=p)
    f, fb_full = random_lattice_inputs(cfg, 11 + N + p)
    S = make_solver(cfg)
    S.set_state(to_dev(f), to_dev(lattice_planes(cfg, fb_full, S.sizes.plane_stride)))
    dtp = dtp_nu * cfg.h / cfg.lam
    S.transport(dtp)
    got = to_np(S.get_state(), f.shape)
    pb = oracle_problem(cfg)
    fc = pb.grid_to_cells(f)
    fbc = pb.grid_to_cells(fb_full)
    O.t2_all(pb, dtp, fc, fbc)
    ref = pb.cells_to_grid(fc)
    S.destroy()
    assert rel_maxnorm(got, ref) <= TOL_OP


@pytest.mark.parametrize("lat", ["D2Q9", "D3Q15", "D3Q19", "D3Q27"])
@pytest.mark.parametrize("tau_dt", [0.0, 0.7])
def test_lbm_collision_parity(lat, tau_dt):
    """C2(dt) with P = [1; v^T] and the lattice equilibrium (eq collision_cn)."""
    cfg = lbm_config(lat, 6 if lat == "D2Q9" else 3)
    tau = tau_dt * cfg.dt
    f, fb_full = random_lattice_inputs(cfg, 3)
    S = make_solver(cfg, tau=tau)
    S.set_state(to_dev(f), to_dev(lattice_planes(cfg, fb_full, S.sizes.plane_stride)))
    S.collide(cfg.dt)
    got = to_np(S.get_state(), f.shape)
    w = to_np(S.moments(), (cfg.m,) + cfg.grid_shape)
    pb = oracle_problem(cfg, tau=tau)
    ref = np.ascontiguousarray(f.copy())
    O.collide(pb, ref, cfg.dt)
    S.destroy()
    assert rel_maxnorm(got, ref) <= TOL_OP
    assert rel_maxnorm(w, O.moments(pb, ref)) <= TOL_OP


@pytest.mark.parametrize("lat,N,p,scheme", [("D2Q9", 12, 2, "m2"), ("D2Q9", 34, 2, "m2kin"), ("D3Q15", 6, 2, "m2"),
                                            ("D3Q19", 6, 2, "m2"), ("D3Q27", 5, 2, "m2"), ("D3Q19", 4, 3, "m2"),
                                            ("D3Q27", 5, 1, "m4")])
def test_lbm_scheme_parity(lat, N, p, scheme):
    """Free-running palindromic steps from f^eq(w0) with inflow f^eq(w0(x_b)) (readings C12/C13)."""
    from paper_1702_00169_b200 import pdg
    cfg = lbm_config(lat, N, p=p, steps=3)
    w0 = w0_grid(cfg)
    wb = wb_grid(cfg, w0)
    sch = {"m2": pdg.PDG_SCHEME_M2, "m2kin": pdg.PDG_SCHEME_M2KIN, "m4": pdg.PDG_SCHEME_M4}[scheme]
    tau = 0.0 if scheme == "m2" else 0.3 * cfg.dt
    S = make_solver(cfg, scheme=sch, tau=tau)
    S.set_equilibrium(w0.reshape(-1).cuda(), wb.reshape(-1).cuda())
    S.step(cfg.steps)
    got = to_np(S.get_state(), (cfg.nv,) + cfg.grid_shape)
    w = to_np(S.moments(), (cfg.m,) + cfg.grid_shape)
    pb = oracle_problem(cfg, tau=tau)
    f0, fb = O.initial_data(pb, w0.numpy(), wb.numpy())
    ref = O.scheme_run(pb, f0, fb, cfg.steps, scheme)
    S.destroy()
    assert rel_maxnorm(got, ref) <= TOL_STEP
    assert rel_maxnorm(w, O.moments(pb, ref)) <= TOL_STEP


def test_lattice_equilibrium_init_matches_oracle():
    cfg = lbm_config("D3Q27", 4)
    w0 = w0_grid(cfg)
    S = make_solver(cfg)
    S.set_equilibrium(w0.reshape(-1).cuda())
    got = to_np(S.get_state(), (cfg.nv,) + cfg.grid_shape)
    fb = S.fb.cpu().numpy().reshape(cfg.nv, cfg.dim, -1)
    pb = oracle_problem(cfg)
    f0, fbf = O.initial_data(pb, w0.numpy(), w0.numpy())
    ref_planes = lattice_planes(cfg, fbf, S.sizes.plane_stride)
    S.destroy()
    assert rel_maxnorm(got, f0) <= TOL_OP
    assert rel_maxnorm(fb, ref_planes) <= TOL_OP


def test_lattice_p3_body_diagonal_unsupported():
    from paper_1702_00169_b200 import pdg
    cfg = lbm_config("D3Q15", 3, p=3)
    with pytest.raises(pdg.PdgError) as e:
        pdg.query_sizes(pdg.problem_from_config(cfg))
    assert e.value.status == pdg.PDG_E_UNSUPPORTED
