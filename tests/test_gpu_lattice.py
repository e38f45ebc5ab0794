"""GPU parity of the lattice velocity sets: D2Q9 and
D3Q15/19/27 with the isothermal LBM equilibrium, against the CPU oracle.

The oracle assembles the full eq DG_reduit blocks of each velocity, orders cells with
Kahn's algorithm on the dependency graph and solves every cell with a
dense LU; the CUDA path applies the pre-inverted dense (p+1)^d block along diagonal
wavefronts (pdg_lattice.cuh).  Bar: <= 1e-13 for one operator, <= 1e-12 for M2 steps
(relative max-norm, reading C17).  pdg_problem.lattice_cta forces small CTAs (one warp per
CTA) so that the cross-CTA hand-over (global traces + progress flags) runs on small grids.
"""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from pdg_inputs import lbm_config, random_state, w0_grid, wb_grid
import gpu_helpers
from gpu_helpers import lattice_planes, make_solver, oracle_problem, rel_maxnorm, to_dev, to_np

pytestmark = pytest.mark.gpu

TOL_OP = 1e-13
TOL_STEP = 1e-12


def _cta(warps):
    return tuple(int(x) for x in warps.split(",")) if warps else (0, 0)


@pytest.fixture
def warps(request):
    """Forced CTA shape "wx,wy" (pdg_problem.lattice_cta) for the solvers the test creates."""
    gpu_helpers.LATTICE_PLAN["lattice_cta"] = _cta(request.param)
    yield request.param
    gpu_helpers.LATTICE_PLAN["lattice_cta"] = (0, 0)


def cases():
    return [
        ("D2Q9", 37, 2), ("D2Q9", 8, 1), ("D2Q9", 9, 3),
        ("D3Q15", 5, 2), ("D3Q19", 5, 2), ("D3Q27", 5, 2),
        ("D3Q19", 4, 3), ("D3Q27", 3, 1), ("D3Q15", 33, 2),
        ("D3Q27", 1, 2), ("D2Q9", 1, 2), ("D3Q19", 2, 3),   # degenerate: one / two cells per axis
        ("D3Q15", 3, 3), ("D3Q27", 2, 3),                   # p = 3 body diagonals (64 x 64 block)
    ]


def random_lattice_inputs(cfg, seed):
    f = random_state(cfg, seed, 0.5).numpy()
    rng = np.random.default_rng(seed + 7)
    fb_full = rng.random((cfg.nv,) + cfg.grid_shape) / cfg.nv
    return f, fb_full


def _transport_params():
    """Every case with the default CTA shape; the grids large enough for several CTAs along x or
    the pipe axis also with 1x1 and 2x2 warps per CTA (cross-CTA hand-over)."""
    out = []
    for lat, N, p in cases():
        for warps in ([None, "1,1", "2,2"] if (N >= 30 or lat == "D2Q9") else [None]):
            for nu in (0.5, -0.05, 2.0):
                out.append(pytest.param(lat, N, p, nu, warps, id=f"{lat}-N{N}-p{p}-nu{nu}-w{warps}"))
    return out


@pytest.mark.parametrize("lat,N,p,dtp_nu,warps", _transport_params(), indirect=["warps"])
def test_lattice_transport_parity(lat, N, p, dtp_nu, warps):
    """One T2(dt') of every velocity (rows a1/a3 for lattice sets) == the oracle's Kahn sweep."""
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
                                            ("D3Q27", 5, 1, "m4"), ("D3Q15", 3, 3, "m2")])
def test_lbm_scheme_parity(lat, N, p, scheme):
    """Free-running palindromic steps from f^eq(w0) with inflow f^eq(w0(x_b)) (readings C12/C13)."""
    from paper_1702_00169_b200 import pdg
    cfg = lbm_config(lat, N, p=p, steps=3)
    w0 = w0_grid(cfg)
    wb = wb_grid(cfg, w0)
    sch = {"m2": pdg.PDG_SCHEME_M2, "m2kin": pdg.PDG_SCHEME_M2KIN, "m4": pdg.PDG_SCHEME_M4}[scheme]
    # M4's middle substep is negative (g2 = 1 - 2 g1 < 0): tau > 0 needs 2 tau + g2 dt/2 > 0
    tau = {"m2": 0.0, "m2kin": 0.3 * cfg.dt, "m4": 0.6 * cfg.dt}[scheme]
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


# --------------------------------------------------------------------------
# Sharded collision, NCCL communicator path, CUDA-graph capture (lattice sets)
# --------------------------------------------------------------------------
def test_lattice_sharded_collision_standin():
    """Row a4 for the LBM model: 4 uneven velocity shards of D3Q27, partial moments (P = [1; v^T]),
    reduction by torch, relax from the reduced w, with a source step fused."""
    from dataclasses import replace
    from paper_1702_00169_b200 import pdg
    cfg = replace(lbm_config("D3Q27", 3), gravity=(0.0, 0.3, -1.0))
    f = random_state(cfg, 4, 0.5).numpy()
    G = 4  # uneven shards: 7, 7, 7, 6 velocities
    shards = []
    for r in range(G):
        S = make_solver(cfg, rank=r, nranks=G, scheme=pdg.PDG_SCHEME_M2S)
        v0, nvl = S.sizes.v_begin, S.sizes.nv_local
        assert nvl == (7 if r < 3 else 6) and v0 == 7 * r
        S.set_state(to_dev(f[v0:v0 + nvl]), to_dev(np.zeros(S.sizes.fb_elems)))
        S.partial_moments()
        shards.append(S)
    wsum = sum(S.w for S in shards)
    for S in shards:
        S.w.copy_(wsum)
        S.relax_from_w(cfg.dt)
    got = np.concatenate([to_np(S.get_state(), (S.sizes.nv_local,) + cfg.grid_shape) for S in shards])
    pb = oracle_problem(cfg)
    ref = np.ascontiguousarray(f.copy())
    O.collide(pb, ref, cfg.dt)
    assert rel_maxnorm(got, ref) <= TOL_OP
    with pytest.raises(Exception):
        shards[0].collide(cfg.dt)  # no communicator: fails loudly
    for S in shards:
        S.destroy()


def test_lattice_nccl_single_rank_m2s():
    """M2s steps through libpdg's NCCL communicator with one rank (partial moments, ncclAllReduce,
    relax_from_w with the fused source steps)."""
    from paper_1702_00169_b200 import pdg
    from pdg_inputs import gravity_config
    cfg = gravity_config(8, dt=0.006, t_max=0.024)
    w0 = w0_grid(cfg)
    S = make_solver(cfg, scheme=pdg.PDG_SCHEME_M2S, nccl_id=pdg.nccl_unique_id(), flags=pdg.PDG_PROFILE)
    S.set_equilibrium(w0.reshape(-1).cuda())
    S.step(cfg.steps)
    got = to_np(S.get_state(), (cfg.nv,) + cfg.grid_shape)
    prof = S.profile_read()
    S.destroy()
    assert prof["allreduce"][1] == cfg.steps and prof["relax_from_w"][1] == cfg.steps
    pb = oracle_problem(cfg)
    f0, fb = O.initial_data(pb, w0.numpy(), w0.numpy())
    assert rel_maxnorm(got, O.scheme_run(pb, f0, fb, cfg.steps, "m2s")) <= TOL_STEP


def test_lattice_cuda_graph_capture():
    """pdg_step of a lattice set (ticket/progress memsets + persistent sweep kernels) is capturable."""
    cfg = lbm_config("D3Q15", 6, steps=4)
    w0 = w0_grid(cfg)
    torch.cuda.synchronize()
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        S = make_solver(cfg, stream=stream.cuda_stream)
        S.set_equilibrium(w0.reshape(-1).cuda())
        f0 = S.get_state().clone()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            S.step(2)
        S.set_state(f0)
        g.replay()
        g.replay()
        stream.synchronize()
    got = to_np(S.get_state(), (cfg.nv,) + cfg.grid_shape)
    S.destroy()
    pb = oracle_problem(cfg)
    f0n, fb = O.initial_data(pb, w0.numpy(), w0.numpy())
    assert rel_maxnorm(got, O.scheme_run(pb, f0n, fb, 4, "m2")) <= TOL_STEP


# --------------------------------------------------------------------------
# Bench sizes (the launch configuration bench.py times): properties that hold at any size
# --------------------------------------------------------------------------
def _perp_basis(v):
    v = np.asarray(v[:3], dtype=np.float64)
    n = v / np.linalg.norm(v)
    a = np.array([1.0, 0.0, 0.0]) if abs(n[0]) < 0.9 else np.array([0.0, 1.0, 0.0])
    u1 = np.cross(n, a)
    u1 /= np.linalg.norm(u1)
    u2 = np.cross(n, u1)
    return u1, u2


@pytest.mark.parametrize("lat,N", [("D3Q27", 128), ("D2Q9", 1024)])
def test_lattice_fullsize_transport_of_invariant_data(lat, N):
    """At the bench size: data of degree <= p that is constant along each velocity, with matching
    inflow data, is a steady state of the exact transport and lies in the DG space, where L_h is
    exact: T2 must leave it unchanged.  Exercises every wavefront class,
    the warp scans and the cross-CTA hand-over in bench.py's launch configuration."""
    from pdg_inputs import node_axis
    cfg = lbm_config(lat, N, nu=2.0)
    vel, _ = cfg.velocities()
    S = make_solver(cfg)
    dev = torch.device("cuda")
    xs = [node_axis(cfg, a, device=dev) for a in range(cfg.dim)]
    if cfg.dim == 3:
        X, Y, Z = xs[0].view(1, 1, -1), xs[1].view(1, -1, 1), xs[2].view(-1, 1, 1)
    else:
        X, Y, Z = xs[0].view(1, -1), xs[1].view(-1, 1), torch.zeros((), dtype=torch.float64, device=dev)
    f = S.f.view((cfg.nv,) + cfg.grid_shape)
    fbv = S.fb.view(cfg.nv, cfg.dim, -1)
    rng = np.random.default_rng(5)
    for i, v in enumerate(vel):
        if not any(v[:cfg.dim]):
            u1, u2 = np.array([1.0, 0, 0]), np.array([0, 1.0, 0])
        else:
            vv = list(v[:cfg.dim]) + [0.0] * (3 - cfg.dim)
            if cfg.dim == 2:
                u1 = np.array([-vv[1], vv[0], 0.0]) / np.hypot(vv[0], vv[1])
                u2 = u1
            else:
                u1, u2 = _perp_basis(vv)
        c = rng.random(3)
        s1 = u1[0] * X + u1[1] * Y + u1[2] * Z
        s2 = u2[0] * X + u2[1] * Y + u2[2] * Z
        val = (1.0 + c[0] * s1 + c[1] * s2 * s2 + c[2] * s1 * s2).expand(cfg.grid_shape)
        f[i].copy_(val)
        for k in range(cfg.dim):
            if v[k] == 0:
                continue
            ax = cfg.dim - 1 - k
            idx = [slice(None)] * cfg.dim
            idx[ax] = 0 if v[k] > 0 else cfg.grid_shape[ax] - 1
            pl = val[tuple(idx)].reshape(-1)
            fbv[i, k, :pl.numel()].copy_(pl)
    f0 = S.f.clone()
    S.set_state(f0)
    S.transport(cfg.dt)
    err = float((S.f - f0).abs().max() / f0.abs().max())
    S.destroy()
    assert err <= 1e-12, err


@pytest.mark.parametrize("lat", ["D3Q19", "D3Q15"])
def test_lattice_fullsize_equilibrium_fixed_point(lat):
    """At the bench size (128^3, p = 2): a constant equilibrium state with f^b = f^eq(w) is a fixed
    point of the whole M2 step (constants are transported exactly, the collision of an equilibrium
    is the identity)."""
    cfg = lbm_config(lat, 128, nu=2.0)
    S = make_solver(cfg)
    w = torch.empty((cfg.m, cfg.nnodes), dtype=torch.float64, device="cuda")
    w[0].fill_(1.1)
    for d in range(cfg.dim):
        w[1 + d].fill_(1.1 * 0.03 * (d + 1))
    S.set_equilibrium(w.reshape(-1))
    f0 = S.f.clone()
    S.step(1)
    err = float((S.f - f0).abs().max() / f0.abs().max())
    S.destroy()
    assert err <= 1e-13, err


# --------------------------------------------------------------------------
# Anisotropic boxes: different cell counts (and cell sizes) per axis, so that the lane, chain,
# pipe and batch extents of every wavefront class differ
# --------------------------------------------------------------------------
def _aniso(lat, ncell, p, lam=1.0, hi=(1.0, 1.0, 1.0)):
    from paper_1702_00169_b200 import pdg
    from pdg_inputs import lattice
    import math
    dim = 2 if lat.startswith("D2") else 3
    vel, wts = lattice(lat, lam)
    c = lam / math.sqrt(3.0)
    fparams = [c] + list(wts)
    h = min(hi[d] / ncell[d] for d in range(dim))
    dt = 0.7 * h / lam
    pb = pdg.make_problem(dim, list(ncell), p, dim + 1, vel, [0] * len(vel), lam, pdg.PDG_FLUX_LBM, fparams, dt,
                          hi=tuple(hi), **gpu_helpers.LATTICE_PLAN)
    ob = O.Problem(dim, list(ncell), p, vel, [0] * len(vel), dim + 1, lam, 3, fparams, dt, hi=list(hi))
    return pb, ob, dt


@pytest.mark.parametrize("lat,ncell,p,hi", [
    ("D3Q27", (37, 5, 3), 2, (1.0, 0.5, 0.25)),
    ("D3Q19", (3, 33, 6), 2, (1.0, 1.0, 1.0)),
    ("D3Q15", (6, 4, 35), 1, (0.3, 1.0, 2.0)),
    ("D2Q9", (40, 7), 3, (1.0, 0.2, 1.0)),
    ("D2Q9", (3, 45), 2, (1.0, 1.0, 1.0)),
])
@pytest.mark.parametrize("warps", [None, "1,1"], indirect=True)
def test_lattice_anisotropic_transport_and_steps(lat, ncell, p, hi, warps):
    from paper_1702_00169_b200 import pdg
    pb, ob, dt = _aniso(lat, ncell, p, hi=hi)
    S = pdg.Solver(pb)
    dim = ob.dim
    shape = ob.grid_shape()
    rng = np.random.default_rng(sum(ncell) + p)
    f = (1.0 + 0.5 * (rng.random((ob.nv,) + shape) - 0.5)) / ob.nv
    fb_full = rng.random((ob.nv,) + shape) / ob.nv

    class _C:  # minimal config view for lattice_planes
        pass
    cv = _C()
    cv.dim, cv.grid_shape = dim, shape
    cv.velocities = lambda: (ob.vel.tolist(), None)
    S.set_state(to_dev(f), to_dev(lattice_planes(cv, fb_full, S.sizes.plane_stride)))
    S.transport(dt)
    got = to_np(S.get_state(), f.shape)
    fc = ob.grid_to_cells(f)
    fbc = ob.grid_to_cells(fb_full)
    O.t2_all(ob, dt, fc, fbc)
    assert rel_maxnorm(got, ob.cells_to_grid(fc)) <= TOL_OP
    # two M2 steps (fused half-steps) from the transported state
    S.step(2)
    got2 = to_np(S.get_state(), f.shape)
    ref2 = O.m2_run(ob, ob.cells_to_grid(fc), fb_full, 2)
    S.destroy()
    assert rel_maxnorm(got2, ref2) <= TOL_STEP


def test_lattice_check_state_counts_nonpositive_density():
    """pdg_check_state for a lattice set: rho = sum of all n_v populations (P = [1; v^T])."""
    from paper_1702_00169_b200 import pdg
    cfg = lbm_config("D2Q9", 4)
    w0 = w0_grid(cfg)
    S = make_solver(cfg)
    S.set_equilibrium(w0.reshape(-1).cuda())
    assert S.check_state() == 0
    state = S.get_state()
    f = state.view((cfg.nv,) + cfg.grid_shape)
    f[:, 2, 3] = -0.1          # one node with rho < 0
    f[4, 5, 6] = float("nan")  # one node with a non-finite population
    S.set_state(state)
    assert S.check_state() == 2
    S.destroy()
    cfgc = lbm_config("D2Q9", 4)
    pb = pdg.problem_from_config(cfgc, flags=pdg.PDG_CHECK_STATE)
    S2 = pdg.Solver(pb)
    S2.set_equilibrium(w0.reshape(-1).cuda())
    S2.step(1)  # healthy: no error
    S2.destroy()


def test_lattice_host_pointer_paths():
    """pdg_set_equilibrium with HOST w and w_b (staged through w_dev), pdg_get_state and
    pdg_moments into host memory, for a lattice set."""
    cfg = lbm_config("D3Q19", 4)
    w0 = w0_grid(cfg)
    wb = 1.01 * w0
    S = make_solver(cfg)
    S.set_equilibrium(w0.reshape(-1).clone(), wb.reshape(-1).clone())   # host tensors
    f = S.get_state(torch.empty(S.sizes.f_elems, dtype=torch.float64))  # host out
    fb = S.fb.cpu().numpy().reshape(cfg.nv, cfg.dim, -1)
    w = S.moments(torch.empty(S.sizes.w_elems, dtype=torch.float64))
    S.destroy()
    pb = oracle_problem(cfg)
    f0, fbf = O.initial_data(pb, w0.numpy(), wb.numpy())
    assert rel_maxnorm(f.numpy().reshape(f0.shape), f0) <= TOL_OP
    assert rel_maxnorm(fb, lattice_planes(cfg, fbf, S.sizes.plane_stride)) <= TOL_OP
    assert rel_maxnorm(w.numpy().reshape((cfg.m,) + cfg.grid_shape), O.moments(pb, f0)) <= TOL_OP


# --------------------------------------------------------------------------
# Chain segments: a class without a pipe axis is cut along its chain into
# segments swept concurrently, each starting `halo` rows early from a zero chain trace, the
# halo taken from the norm bound of the chain operator (pdg_tables.hpp lattice_chain_halo).
# pdg_problem.lattice_segment forces the segment length so that small grids run several segments.
# --------------------------------------------------------------------------
@pytest.fixture
def seglen(request):
    gpu_helpers.LATTICE_PLAN["lattice_segment"] = int(request.param)
    yield request.param
    gpu_helpers.LATTICE_PLAN["lattice_segment"] = 0


def _d2q9_box(ncell, p, dt, lam=1.0, hi=(1.0, 1.0, 1.0)):
    from paper_1702_00169_b200 import pdg
    from pdg_inputs import lattice
    import math
    vel, wts = lattice("D2Q9", lam)
    fparams = [lam / math.sqrt(3.0)] + list(wts)
    pb = pdg.make_problem(2, list(ncell), p, 3, vel, [0] * len(vel), lam, pdg.PDG_FLUX_LBM, fparams, dt, hi=tuple(hi),
                          **gpu_helpers.LATTICE_PLAN)
    ob = O.Problem(2, list(ncell), p, vel, [0] * len(vel), 3, lam, 3, fparams, dt, hi=list(hi))
    return pb, ob


def _planes_view(ob):
    class _C:
        pass
    cv = _C()
    cv.dim, cv.grid_shape = ob.dim, ob.grid_shape()
    cv.velocities = lambda: (ob.vel.tolist(), None)
    return cv


# (cells x, y), p, kappa = lambda dt'/h, forced segment length, CTA shape.  kappa 0.25 / 0.5 / 1
# give halos of 12-16 / 16 / 28 rows (<= the segment: segmented); kappa 4 needs > 100 rows and
# dt' < 0 has no bound (both run unsegmented: the fallback path).
SEG_CASES = [
    ((40, 150), 2, 0.25, 24, None),
    ((70, 200), 2, 1.0, 40, "1,1"),
    ((33, 130), 1, 0.5, 32, None),
    ((37, 97), 3, 1.0, 30, "2,2"),
    ((65, 90), 2, 0.5, 17, "1,1"),
    ((40, 150), 2, 4.0, 24, None),
    ((40, 120), 2, -0.05, 24, "1,1"),
]


@pytest.mark.parametrize("ncell,p,kappa,seglen,warps", SEG_CASES, indirect=["seglen", "warps"],
                         ids=[f"{c[0][0]}x{c[0][1]}-p{c[1]}-k{c[2]}-L{c[3]}-w{c[4]}" for c in SEG_CASES])
def test_lattice_chain_segments_parity(ncell, p, kappa, seglen, warps):
    """One T2(dt') and two M2 steps of D2Q9 with the chain cut into segments == the oracle."""
    h = 1.0 / ncell[0]
    dtp = kappa * h
    hi = (1.0, ncell[1] / ncell[0], 1.0)  # square cells: kappa on both axes
    pb, ob = _d2q9_box(ncell, p, dt=2.0 * dtp if dtp > 0 else 0.5 * h, hi=hi)
    from paper_1702_00169_b200 import pdg
    S = pdg.Solver(pb)
    shape = ob.grid_shape()
    rng = np.random.default_rng(sum(ncell) + p)
    f = (1.0 + 0.5 * (rng.random((ob.nv,) + shape) - 0.5)) / ob.nv
    fb_full = rng.random((ob.nv,) + shape) / ob.nv
    S.set_state(to_dev(f), to_dev(lattice_planes(_planes_view(ob), fb_full, S.sizes.plane_stride)))
    S.transport(dtp)
    got = to_np(S.get_state(), f.shape)
    fc = ob.grid_to_cells(f)
    fbc = ob.grid_to_cells(fb_full)
    O.t2_all(ob, dtp, fc, fbc)
    assert rel_maxnorm(got, ob.cells_to_grid(fc)) <= TOL_OP
    S.step(2)
    got2 = to_np(S.get_state(), f.shape)
    ref2 = O.m2_run(ob, ob.cells_to_grid(fc), fb_full, 2)
    S.destroy()
    assert rel_maxnorm(got2, ref2) <= TOL_STEP


@pytest.mark.parametrize("N", [512, 1024])
def test_lattice_chain_segments_match_unsegmented(N):
    """At bench-like sizes the default segmentation (halo from the bound) and the whole-chain sweep
    agree to the last bits: the truncated trace differs by <= 2^-64 of the true one."""
    cfg = lbm_config("D2Q9", N, nu=2.0)
    outs = []
    for seg in (-1, 0):  # never segmented, the default plan
        S = make_solver(cfg, lattice_segment=seg)
        S.set_equilibrium(w0_grid(cfg, device="cuda").reshape(-1))
        S.step(2)
        outs.append(S.get_state().clone())
        S.destroy()
    err = float((outs[0] - outs[1]).abs().max() / outs[0].abs().max())
    assert err <= 1e-15, err


@pytest.mark.parametrize("lat,N,warps", [("D2Q9", 1024, None), ("D2Q9", 300, "1,1"), ("D3Q27", 48, None),
                                         ("D3Q15", 40, "2,2")], indirect=["warps"])
def test_lattice_sweeps_bitwise_deterministic(lat, N, warps):
    """The cross-CTA hand-overs (tagged x/y words, fenced y traces, segment halo flags) are races if
    wrong: a stale or torn trace changes the result.  Tasks are claimed dynamically, so repeated
    launches exercise different CTA interleavings; every repeat must be bit-identical, including
    replays of a captured CUDA graph (the consumers empty the tagged slots for the next launch)."""
    cfg = lbm_config(lat, N, nu=2.0)
    S = make_solver(cfg)
    w0 = w0_grid(cfg, device="cuda").reshape(-1)
    outs = []
    for _ in range(3):
        S.set_equilibrium(w0)
        S.step(2)
        outs.append(S.get_state().clone())
    torch.cuda.synchronize()
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        S2 = make_solver(cfg, stream=st.cuda_stream)
        S2.set_equilibrium(w0)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            S2.step(2)
        for _ in range(2):
            S2.set_equilibrium(w0)
            g.replay()
            st.synchronize()
            outs.append(S2.get_state().clone())
        st.synchronize()
    S.destroy()
    S2.destroy()
    for o in outs[1:]:
        assert torch.equal(o, outs[0])


@pytest.mark.parametrize("seglen", [16, 40])
def test_lattice_chain_segments_3d_two_axis_classes(seglen):
    """Chain segments on the 3-D classes without a pipe axis (x,y and x,z active: D3Q19's face
    diagonals) against the oracle: one T2 and two M2 steps on a box whose chains span several
    segments."""
    from paper_1702_00169_b200 import pdg
    from pdg_inputs import lattice
    import math
    ncell = (10, 48, 48)
    h = 1.0 / ncell[0]
    hi = (1.0, ncell[1] * h, ncell[2] * h)
    kappa = 0.5
    dtp = kappa * h
    vel, wts = lattice("D3Q19", 1.0)
    fparams = [1.0 / math.sqrt(3.0)] + list(wts)
    if True:  # (indentation kept from the env-knob version)
        pb = pdg.make_problem(3, list(ncell), 2, 4, vel, [0] * len(vel), 1.0, pdg.PDG_FLUX_LBM, fparams, 2.0 * dtp, hi=hi,
                              lattice_segment=seglen)
        S = pdg.Solver(pb)
        ob = O.Problem(3, list(ncell), 2, vel, [0] * len(vel), 4, 1.0, 3, fparams, 2.0 * dtp, hi=list(hi))
        shape = ob.grid_shape()
        rng = np.random.default_rng(123 + seglen)
        f = (1.0 + 0.5 * (rng.random((ob.nv,) + shape) - 0.5)) / ob.nv
        fb_full = rng.random((ob.nv,) + shape) / ob.nv
        S.set_state(to_dev(f), to_dev(lattice_planes(_planes_view(ob), fb_full, S.sizes.plane_stride)))
        S.transport(dtp)
        got = to_np(S.get_state(), f.shape)
        fc = ob.grid_to_cells(f)
        fbc = ob.grid_to_cells(fb_full)
        O.t2_all(ob, dtp, fc, fbc)
        assert rel_maxnorm(got, ob.cells_to_grid(fc)) <= TOL_OP
        S.step(2)
        got2 = to_np(S.get_state(), f.shape)
        S.destroy()
    ref2 = O.m2_run(ob, ob.cells_to_grid(fc), fb_full, 2)
    assert rel_maxnorm(got2, ref2) <= TOL_STEP
