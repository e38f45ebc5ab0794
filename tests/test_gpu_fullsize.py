"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

* One M2 step from the seeded equilibrium of configs 2-5 at full size: the CUDA
  result is compared with the oracle on sampled cells, the oracle evaluating each
  sample exactly on its dependency cone (oracle.m2_cone_step: closures of the
  upwind graph), from the same seeded w0.
* The fused multi-step pass structure bench.py times (consecutive T2(dt/2) swept in
  one pass, collision fused with the x-sweeps) equals separate single-step calls:
  a property that holds at any size.
"""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from pdg_inputs import CONFIGS
from gpu_helpers import make_solver, rel_maxnorm

pytestmark = pytest.mark.gpu

TOL = 1e-12


def fill_w0(cfg, w_flat):
    from pdg_inputs import w0_grid
    w = w_flat.view((cfg.m,) + cfg.grid_shape)
    if cfg.dim == 2:
        w.copy_(w0_grid(cfg, device=w_flat.device))
        return
    L = cfg.N * cfg.n
    slab = max(1, min(L, (1 << 24) // (L * L)))
    for z0 in range(0, L, slab):
        w[:, z0:z0 + slab].copy_(w0_grid(cfg, device=w_flat.device, zslab=(z0, min(L, z0 + slab))))


def cell_node_index(cfg, cells: np.ndarray) -> torch.Tensor:
    """Grid node indices [len(cells), Nd] of the nodes of `cells` (cell-blocked order)."""
    n, N, D = cfg.n, cfg.N, cfg.dim
    L = N * n
    cells = torch.as_tensor(cells, dtype=torch.int64)
    cc = []
    r = cells.clone()
    for _ in range(D):
        cc.append(r % N)
        r = r // N
    a = torch.arange(n ** D, dtype=torch.int64)
    aa = []
    r = a.clone()
    for _ in range(D):
        aa.append(r % n)
        r = r // n
    idx = torch.zeros((cells.numel(), n ** D), dtype=torch.int64)
    stride = 1
    for d in range(D):
        coord = cc[d].view(-1, 1) * n + aa[d].view(1, -1)
        idx += coord * stride
        stride *= L
    return idx


def sample_cells(cfg):
    N, D = cfg.N, cfg.dim
    rng = np.random.default_rng(17)
    pts = [[0] * D, [N // 2] * D, list(rng.integers(0, N, D))]
    out = []
    for p in pts:
        c = 0
        for d in reversed(range(D)):
            c = c * N + int(p[d])
        out.append(c)
    return np.array(sorted(set(out)), dtype=np.int64)


@pytest.mark.parametrize("key", [2, 3, 4, 5])
def test_fullsize_one_step_sampled(key):
    cfg = CONFIGS[key]
    torch.cuda.empty_cache()
    S = make_solver(cfg)
    fill_w0(cfg, S.w)
    S.set_equilibrium(S.w)
    pb = O.Problem.from_config(cfg)
    samples = sample_cells(cfg)
    plan = O.m2_cone_plan(pb, samples)
    # inputs of the oracle: the same seeded w0, gathered at the cells each pass needs
    need = np.unique(np.concatenate(plan["first"]))
    idx = cell_node_index(cfg, need).to(S.w.device)
    w_need = S.w.view(cfg.m, -1)[:, idx.view(-1)].view(cfg.m, need.size, -1).cpu().numpy()
    f_need = O.equilibrium_field(pb, np.ascontiguousarray(w_need))  # [nv, ncell_need, Nd]
    def f0_of(i, cells):
        return np.ascontiguousarray(f_need[i][np.searchsorted(need, cells)])

    S.step(1)
    sidx = cell_node_index(cfg, samples).to(S.f.device)
    got = S.f.view(cfg.nv, -1)[:, sidx.view(-1)].view(cfg.nv, samples.size, -1).cpu().numpy()
    ref = O.m2_cone_step(pb, plan, f0_of, f0_of)  # w_b = w0 (reading C12): f^b = f0 on the faces
    assert rel_maxnorm(got, ref) < TOL
    S.destroy()
    del S
    torch.cuda.empty_cache()


@pytest.mark.parametrize("key", [3, 5])
def test_fullsize_fused_passes_equal_separate_steps(key):
    """step(3) (fused TT passes, NPASS=2 kernels) == 3 x step(1) (NPASS=1 kernels)."""
    cfg = CONFIGS[key]
    torch.cuda.empty_cache()
    S = make_solver(cfg)
    fill_w0(cfg, S.w)
    g = torch.Generator(device="cpu").manual_seed(3)
    pick = torch.randint(0, S.sizes.f_elems, (1 << 20,), generator=g).to(S.f.device)
    S.set_equilibrium(S.w)
    S.step(3)
    a = S.f[pick].cpu().numpy()
    fill_w0(cfg, S.w)
    S.set_equilibrium(S.w)
    for _ in range(3):
        S.step(1)
    b = S.f[pick].cpu().numpy()
    assert rel_maxnorm(a, b) < 1e-13
    S.destroy()
    del S
    torch.cuda.empty_cache()


# --------------------------------------------------------------------------
# Lattice sets at the bench size: one T2 of every velocity on 128^3 cells (D3Q27: every
# wavefront class, the warp scans, the skewed warps and the cross-CTA hand-over in
# bench.py's launch configuration), compared with the oracle on sampled cells.  For each
# velocity the samples lie on the three domain edges through its upstream corner (plus a
# few cells near it): their dependency cones are single lines or small boxes, and the
# full-length lines cross every CTA boundary along x and along the pipe axis.
# --------------------------------------------------------------------------
def _smooth_field(X, Y, Z, i, nv, amp):
    sin = torch.sin if isinstance(X, torch.Tensor) else np.sin
    return (1.0 + amp * sin(0.37 * X + 0.71 * Y + 1.13 * Z + 0.5 * i + 0.3 * X * Y / 97.0)) / nv


@pytest.mark.parametrize("lat,N", [("D3Q27", 128), ("D2Q9", 1024), ("D2Q9", 2048), ("D3Q15", 128)])
def test_lattice_fullsize_sampled_transport(lat, N):
    from pdg_inputs import lbm_config
    cfg = lbm_config(lat, N, nu=2.0)
    torch.cuda.empty_cache()
    S = make_solver(cfg)
    dev = S.f.device
    D, n = cfg.dim, cfg.n
    xs = [torch.arange(cfg.N * n, device=dev, dtype=torch.float64) for _ in range(D)]  # node indices
    if D == 3:
        X, Y, Z = xs[0].view(1, 1, -1), xs[1].view(1, -1, 1), xs[2].view(-1, 1, 1)
    else:
        X, Y, Z = xs[0].view(1, -1), xs[1].view(-1, 1), torch.zeros((), device=dev, dtype=torch.float64)
    f = S.f.view((cfg.nv,) + cfg.grid_shape)
    fbv = S.fb.view(cfg.nv, D, -1)
    vel, _ = cfg.velocities()
    for i in range(cfg.nv):
        f[i].copy_(_smooth_field(X, Y, Z, i, cfg.nv, 0.3).expand(cfg.grid_shape))
        full = _smooth_field(X, Y, Z, 100 + i, cfg.nv, 0.2).expand(cfg.grid_shape)  # one f^b field (C22)
        for k in range(D):
            if vel[i][k] == 0:
                continue
            ax = D - 1 - k
            sl = [slice(None)] * D
            sl[ax] = 0 if vel[i][k] > 0 else cfg.grid_shape[ax] - 1
            pl = full[tuple(sl)].reshape(-1)
            fbv[i, k, :pl.numel()].copy_(pl)
    f0_full = S.f.clone()
    S.set_state(f0_full)
    S.transport(cfg.dt)
    pb = O.Problem.from_config(cfg)
    Nd = n ** D
    errs = []
    for i in range(cfg.nv):
        v = vel[i]
        if not any(v[:D]):
            continue
        # samples in flow coordinates -> physical cell indices
        flow = []
        for d in range(D):
            for a in (1, N // 3, N - 1):
                p = [0] * D
                p[d] = a
                flow.append(p)
        flow.append([1] * D)
        flow.append([min(2, N - 1)] * D)
        cells = set()
        for p in flow:
            c = 0
            for d in reversed(range(D)):
                pd_ = p[d] if v[d] >= 0 else N - 1 - p[d]
                c = c * N + pd_
            cells.add(c)
        samples = np.array(sorted(cells), dtype=np.int64)
        clos = np.flatnonzero(O.upstream_closure(pb, v, samples)).astype(np.int64)
        idx = cell_node_index(cfg, clos).to(dev)                           # [ncl, Nd] node indices
        coords = []
        r = idx.clone()
        for d in range(D):
            coords.append((r % (N * n)).double())
            r = r // (N * n)
        Xc, Yc = coords[0], coords[1]
        Zc = coords[2] if D == 3 else torch.zeros_like(Xc)
        # the same values the GPU run used: f0 gathered from its input, f^b re-evaluated by the same
        # torch expression on the same device (elementwise, so bitwise the plane values)
        f0c = np.ascontiguousarray(f0_full.view(cfg.nv, -1)[i][idx.view(-1)].view(idx.shape).cpu().numpy())
        fbc = np.ascontiguousarray(_smooth_field(Xc, Yc, Zc, 100 + i, cfg.nv, 0.2).cpu().numpy())
        O.t2_velocity(pb, v, cfg.dt, f0c, fbc, clos)
        pos = np.searchsorted(clos, samples)
        ref = f0c[pos]
        sidx = cell_node_index(cfg, samples).to(dev)
        got = S.f.view(cfg.nv, -1)[i][sidx.view(-1)].view(samples.size, Nd).cpu().numpy()
        errs.append(rel_maxnorm(got, ref))
    S.destroy()
    del S
    torch.cuda.empty_cache()
    assert max(errs) <= 1e-13, errs


# --------------------------------------------------------------------------
# The parity protocol on whole arrays at full size (tests/parity_harness.py; the long runs of every
# config are in test_gpu_long.py, gated): the fast cases that run in every `pytest -m gpu`.
# --------------------------------------------------------------------------
def test_fullsize_cfg2_stabilised_free_running_whole_arrays():
    """Config 2's stabilised twin (lambda = 3.5, same nu) at full 256^2 over its 100 steps: the GPU
    (pdg_step(1) per step, and one pdg_step(100) call) against the oracle on the whole f and w at
    every step, plus re-synced steps 1, 50, 100: all <= 1e-12."""
    from parity_harness import run_protocol
    rec = run_protocol(CONFIGS[2].stabilised(), {1, 50, 100}, lockstep=True, gpu_twin=False)
    for e in rec["per_step"]:
        assert e["free_f"] <= TOL and e["free_w"] <= TOL and e["free_nonfinite_gpu"] == 0, e
        if "resync_f" in e:
            assert e["resync_f"] <= TOL and e["resync_w"] <= TOL, e
    assert rec["fused_free_f"] <= TOL and rec["fused_free_w"] <= TOL, rec


def test_fullsize_cfg3_as_written_resynced_whole_arrays():
    """Config 3 as written at full 64^3: steps 1-3 re-synced and free-running on the whole arrays."""
    from parity_harness import run_protocol
    rec = run_protocol(CONFIGS[3], {1, 2, 3}, lockstep=True, gpu_twin=False, steps=3)
    for e in rec["per_step"]:
        assert e["resync_f"] <= TOL and e["resync_w"] <= TOL, e
        assert e["free_f"] <= TOL and e["free_w"] <= TOL, e
    assert rec["fused_free_f"] <= TOL, rec
