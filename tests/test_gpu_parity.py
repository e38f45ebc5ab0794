"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle.

Bar: relative max-norm (reading C17) <= 1e-12 for the palindromic step (north
star), <= 1e-13 for a single transport / collision operator.  Sizes span
several x-chunks (32 cells), ragged tails and every axis/sign; full config
sizes are checked on sampled cells through dependency cones
(test_gpu_fullsize.py).
"""
from dataclasses import replace

import numpy as np
import pytest
import torch

from oracle import oracle as O
from pdg_inputs import CONFIGS, random_state, w0_grid, wb_grid
from gpu_helpers import (full_grid_to_planes, make_solver, oracle_problem, planes_to_full_grid, rel_maxnorm,
                               to_dev, to_np)

pytestmark = pytest.mark.gpu

TOL_OP = 1e-13
TOL_STEP = 1e-12


def random_inputs(cfg, seed, scale=0.5):
    f = random_state(cfg, seed, scale).numpy()
    rng = np.random.default_rng(seed + 1)
    fb_full = planes_to_full_grid(cfg, rng.random((cfg.nv, (cfg.N * cfg.n) ** (cfg.dim - 1))) / cfg.nv)
    return f, fb_full


def gpu_with_state(cfg, f, fb_full, **kw):
    S = make_solver(cfg, **kw)
    planes = full_grid_to_planes(cfg, fb_full, S.sizes.plane_stride)
    S.set_state(to_dev(f), to_dev(planes))
    return S


def small_cases():
    return [
        CONFIGS[1],                                   # 8x8, p=2, advection
        CONFIGS[1].resized(37, name="adv37"),         # 2 x-chunks + ragged tail
        CONFIGS[2].resized(40, name="euler40"),       # Euler, ragged 40 = 32 + 8
        CONFIGS[3].resized(5, name="iso5"),           # 3-D, p=2
        CONFIGS[4].resized(4, name="iso4p3"),         # 3-D, p=3, kappa=2
        replace(CONFIGS[3].resized(3), p=1, name="iso3p1"),  # p=1
    ]


# --------------------------------------------------------------------------
# Cell block (setup of row a5) against the oracle's single-cell solve
# --------------------------------------------------------------------------
@pytest.mark.parametrize("p,kappa", [(1, 0.25), (2, 0.125), (2, 1.0), (3, 2.0), (3, -0.5), (2, 7.0)])
def test_cell_block_matches_oracle(p, kappa):
    cfg = replace(CONFIGS[3].resized(2), p=p)
    S = make_solver(cfg)
    dtp = kappa * cfg.h / cfg.lam
    M, g, beta = S.cell_block(0, dtp)
    pb = O.Problem(1, 1, p, [[1.0, 0, 0]], [0], 1, 1.0, 0, [1.0], dt=1.0)
    n = p + 1
    Mo = np.zeros((n, n))
    for j in range(n):
        f = np.zeros((1, n))
        f[0, j] = 1.0
        O.t2_velocity(pb, pb.vel[0], kappa, f, np.zeros((1, n)))
        Mo[:, j] = f[0]
    f = np.zeros((1, n))
    O.t2_velocity(pb, pb.vel[0], kappa, f, np.full((1, n), 0.5))
    assert rel_maxnorm(np.array(M), Mo) < 1e-14
    assert rel_maxnorm(np.array(g), f[0]) < 1e-14
    assert abs(beta - f[0][-1]) <= 1e-15 * max(1.0, abs(f[0][-1]))


# --------------------------------------------------------------------------
# Row a1/a3: one transport operator T2(dt') on every velocity
# --------------------------------------------------------------------------
@pytest.mark.parametrize("case", range(6))
@pytest.mark.parametrize("npass_dt", [0.5, -0.05, 1.3])
def test_transport_parity(case, npass_dt):
    cfg = small_cases()[case]
    f, fb_full = random_inputs(cfg, 100 + case)
    dtp = npass_dt * cfg.dt
    S = gpu_with_state(cfg, f, fb_full)
    S.transport(dtp)
    got = to_np(S.get_state(), f.shape)
    pb = oracle_problem(cfg)
    fc = pb.grid_to_cells(f)
    O.t2_all(pb, dtp, fc, pb.grid_to_cells(fb_full))
    assert rel_maxnorm(got, pb.cells_to_grid(fc)) < TOL_OP


# --------------------------------------------------------------------------
# Row a2: collision fused with moments, every model, tau = 0 and tau > 0
# --------------------------------------------------------------------------
MODEL_CASES = [
    ("adv2", CONFIGS[1]), ("euler2", CONFIGS[2].resized(6)), ("iso3", CONFIGS[3].resized(3)),
    ("adv3", replace(CONFIGS[3].resized(3), m=1, flux=0, fparams=(1.0, -0.5, 0.25))),
    ("euler3", replace(CONFIGS[3].resized(3), m=5, flux=1, fparams=(1.4,))),
    ("iso2", replace(CONFIGS[2].resized(6), m=3, flux=2, fparams=(0.7,))),
]


@pytest.mark.parametrize("name,cfg", MODEL_CASES)
@pytest.mark.parametrize("tau", [0.0, 0.01])
def test_collision_parity(name, cfg, tau):
    f, fb_full = random_inputs(cfg, 7)
    S = gpu_with_state(cfg, f, fb_full, tau=tau)
    S.collide(cfg.dt)
    got = to_np(S.get_state(), f.shape)
    pb = oracle_problem(cfg, tau=tau)
    ref = np.ascontiguousarray(f.copy())
    O.collide(pb, ref, cfg.dt, tau=tau)
    assert rel_maxnorm(got, ref) < TOL_OP
    w = to_np(S.moments(), (cfg.m,) + cfg.grid_shape)
    assert rel_maxnorm(w, O.moments(pb, ref)) < TOL_OP


# --------------------------------------------------------------------------
# Equilibrium initialisation (readings C12, C13)
# --------------------------------------------------------------------------
@pytest.mark.parametrize("key", [1, 2, 3])
@pytest.mark.parametrize("host", [True, False])
def test_set_equilibrium_parity(key, host):
    cfg = CONFIGS[key] if key == 1 else CONFIGS[key].resized(6)
    w0 = w0_grid(cfg)
    wb = wb_grid(cfg, w0)
    S = make_solver(cfg)
    if host:
        S.set_equilibrium(w0.reshape(-1), wb.reshape(-1) if cfg.wb_zero else None)
    else:
        S.set_equilibrium(w0.reshape(-1).cuda(), wb.reshape(-1).cuda())
    pb = oracle_problem(cfg)
    f0, fbg = O.initial_data(pb, w0.numpy(), wb.numpy())
    assert rel_maxnorm(to_np(S.get_state(), f0.shape), f0) < TOL_OP
    planes = to_np(S.fb, (cfg.nv, S.sizes.plane_stride))
    assert rel_maxnorm(planes, full_grid_to_planes(cfg, fbg, S.sizes.plane_stride)) < TOL_OP


# --------------------------------------------------------------------------
# The palindromic step M2 (rows a1-a3 + a5)
# --------------------------------------------------------------------------
def seeded_equilibrium(cfg):
    w0 = w0_grid(cfg)
    wb = wb_grid(cfg, w0)
    pb = oracle_problem(cfg)
    f0, fbg = O.initial_data(pb, w0.numpy(), wb.numpy())
    return pb, f0, fbg


def test_config1_free_running_full():
    """Config 1 exactly as written: 10 free-running steps, f and w <= 1e-12."""
    cfg = CONFIGS[1]
    pb, f0, fbg = seeded_equilibrium(cfg)
    S = gpu_with_state(cfg, f0, fbg)
    S.step(cfg.steps)
    got = to_np(S.get_state(), f0.shape)
    ref = O.m2_run(pb, f0, fbg, cfg.steps)
    assert rel_maxnorm(got, ref) < TOL_STEP
    w = to_np(S.moments(), (cfg.m,) + cfg.grid_shape)
    assert rel_maxnorm(w, O.moments(pb, ref)) < TOL_STEP


@pytest.mark.parametrize("key,N,steps", [(2, 24, 6), (3, 6, 5), (4, 4, 4), (5, 8, 4)])
def test_m2_resynced_each_step(key, N, steps):
    """One-step parity re-synced from the oracle's f^n (parity protocol step 1)."""
    cfg = CONFIGS[key].resized(N)
    pb, f, fbg = seeded_equilibrium(cfg)
    S = gpu_with_state(cfg, f, fbg)
    for s in range(steps):
        ref = O.m2_run(pb, f, fbg, 1)
        S.set_state(to_dev(f))
        S.step(1)
        got = to_np(S.get_state(), f.shape)
        assert rel_maxnorm(got, ref) < TOL_STEP, s
        f = ref


@pytest.mark.parametrize("key,N,steps", [(2, 20, 10), (3, 6, 8), (4, 4, 6), (5, 8, 6)])
def test_m2_stabilised_twin_free_running(key, N, steps):
    """Stabilised twins (lambda = 3.5, same nu) free-running: <= 1e-12 (protocol step 3)."""
    cfg = CONFIGS[key].resized(N, steps=steps).stabilised()
    pb, f0, fbg = seeded_equilibrium(cfg)
    S = gpu_with_state(cfg, f0, fbg)
    S.step(steps)
    got = to_np(S.get_state(), f0.shape)
    ref = O.m2_run(pb, f0, fbg, steps)
    assert rel_maxnorm(got, ref) < TOL_STEP


def test_fused_equals_unfused():
    from paper_1702_00169_b200 import pdg
    cfg = CONFIGS[3].resized(6).stabilised()
    pb, f0, fbg = seeded_equilibrium(cfg)
    A = gpu_with_state(cfg, f0, fbg)
    B = gpu_with_state(cfg, f0, fbg, flags=pdg.PDG_NO_FUSION)
    A.step(5)
    B.step(5)
    a = to_np(A.get_state(), f0.shape)
    b = to_np(B.get_state(), f0.shape)
    assert rel_maxnorm(a, b) < 1e-14


def test_m2kin_scheme():
    """M2kin = T2(dt/4) C2(dt/2) T2(dt/2) C2(dt/2) T2(dt/4) vs oracle composition."""
    from paper_1702_00169_b200 import pdg
    cfg = CONFIGS[2].resized(12).stabilised()
    pb, f0, fbg = seeded_equilibrium(cfg)
    S = gpu_with_state(cfg, f0, fbg, scheme=pdg.PDG_SCHEME_M2KIN)
    S.step(3)
    fc = pb.grid_to_cells(f0)
    fbc = pb.grid_to_cells(fbg)
    for _ in range(3):
        O.t2_all(pb, cfg.dt / 4, fc, fbc)
        O.collide(pb, fc, cfg.dt / 2)
        O.t2_all(pb, cfg.dt / 2, fc, fbc)
        O.collide(pb, fc, cfg.dt / 2)
        O.t2_all(pb, cfg.dt / 4, fc, fbc)
    assert rel_maxnorm(to_np(S.get_state(), f0.shape), pb.cells_to_grid(fc)) < TOL_STEP


# --------------------------------------------------------------------------
# Row a4 on one GPU: sharded collision halves with the reduction done by torch
# --------------------------------------------------------------------------
@pytest.mark.parametrize("G", [2, 4, 8])
def test_sharded_collision_standin(G):
    cfg = CONFIGS[3].resized(4)
    f, fb_full = random_inputs(cfg, 3)
    nvl = cfg.nv // G
    shards = []
    for r in range(G):
        S = make_solver(cfg, rank=r, nranks=G)
        assert S.sizes.nv_local == nvl and S.sizes.v_begin == r * nvl
        planes = full_grid_to_planes(cfg, fb_full[r * nvl:(r + 1) * nvl], S.sizes.plane_stride, v_begin=r * nvl)
        S.set_state(to_dev(f[r * nvl:(r + 1) * nvl]), to_dev(planes))
        S.partial_moments()
        shards.append(S)
    wsum = sum(S.w for S in shards)
    for S in shards:
        S.w.copy_(wsum)
        S.relax_from_w(cfg.dt)
    got = np.concatenate([to_np(S.get_state(), (nvl,) + cfg.grid_shape) for S in shards])
    pb = oracle_problem(cfg)
    ref = np.ascontiguousarray(f.copy())
    O.collide(pb, ref, cfg.dt)
    assert rel_maxnorm(got, ref) < TOL_OP
    with pytest.raises(Exception):
        shards[0].collide(cfg.dt)  # no communicator: must fail loudly, not fall back


# --------------------------------------------------------------------------
# Edge cases and error behaviour
# --------------------------------------------------------------------------
def test_single_cell_and_zero_steps():
    cfg = CONFIGS[3].resized(1).stabilised()
    pb, f0, fbg = seeded_equilibrium(cfg)
    S = gpu_with_state(cfg, f0, fbg)
    S.step(0)
    assert rel_maxnorm(to_np(S.get_state(), f0.shape), f0) == 0.0
    S.step(2)
    assert rel_maxnorm(to_np(S.get_state(), f0.shape), O.m2_run(pb, f0, fbg, 2)) < TOL_STEP


def test_gpu_time_symmetry():
    """T2(-dt') T2(dt') = I on the GPU path too (eq prop_sym), small nu."""
    cfg = CONFIGS[2].resized(4)
    f, fb_full = random_inputs(cfg, 5)
    S = gpu_with_state(cfg, f, fb_full)
    S.transport(0.05 * cfg.dt)
    S.transport(-0.05 * cfg.dt)
    assert rel_maxnorm(to_np(S.get_state(), f.shape), f) < 1e-12


def test_errors_are_reported():
    from paper_1702_00169_b200 import pdg
    cfg = CONFIGS[1]
    S = make_solver(cfg)
    with pytest.raises(pdg.PdgError) as e:
        S.step(1)
    assert e.value.status == pdg.PDG_E_STATE_NOT_SET
    with pytest.raises(pdg.PdgError) as e:
        S.step(-1)
    assert e.value.status == pdg.PDG_E_INVALID_ARGUMENT


def test_check_state_flags_nonphysical():
    from paper_1702_00169_b200 import pdg
    cfg = CONFIGS[3].resized(3)
    pb, f0, fbg = seeded_equilibrium(cfg)
    S = gpu_with_state(cfg, f0, fbg)
    assert S.check_state() == 0
    bad = f0.copy()
    bad[0, 0, 0, 0] = np.nan
    bad[:6, 1, 1, 1] = -1.0
    S.set_state(to_dev(bad))
    assert S.check_state() == 2
    S2 = gpu_with_state(cfg, bad, fbg, flags=pdg.PDG_CHECK_STATE)
    with pytest.raises(pdg.PdgError) as e:
        S2.step(1)
    assert e.value.status == pdg.PDG_E_NONPHYSICAL


def test_cuda_graph_capture_of_step():
    """pdg_step is capturable: replaying the graph equals eager steps."""
    cfg = CONFIGS[3].resized(6).stabilised()
    pb, f0, fbg = seeded_equilibrium(cfg)
    torch.cuda.synchronize()
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        S = gpu_with_state(cfg, f0, fbg)
        S.set_state(to_dev(f0))
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            S.step(2)
        S.set_state(to_dev(f0))
        g.replay()
        g.replay()
        stream.synchronize()
    ref = O.m2_run(pb, f0, fbg, 4)
    assert rel_maxnorm(to_np(S.get_state(), f0.shape), ref) < TOL_STEP


@pytest.mark.parametrize("N", [3, 37, 100, 300])
def test_m2_fused_relax_xsweep_line_lengths(N):
    """The fused collision + x-sweep kernel over segment sizes K = 2, 4, 8 and a
    line longer than one 32K-cell super-chunk (N = 300), ragged tails included."""
    cfg = CONFIGS[1].resized(N, steps=3)
    pb, f0, fbg = seeded_equilibrium(cfg)
    S = gpu_with_state(cfg, f0, fbg)
    S.step(3)
    ref = O.m2_run(pb, f0, fbg, 3)
    assert rel_maxnorm(to_np(S.get_state(), f0.shape), ref) < TOL_STEP


def test_odd_line_count():
    """p=2 with an odd cell count gives odd node rows and odd line counts."""
    cfg = CONFIGS[3].resized(5).stabilised()
    pb, f0, fbg = seeded_equilibrium(cfg)
    S = gpu_with_state(cfg, f0, fbg)
    S.step(3)
    assert rel_maxnorm(to_np(S.get_state(), f0.shape), O.m2_run(pb, f0, fbg, 3)) < TOL_STEP


def test_nccl_communicator_path_single_rank():
    """The sharded collision through libpdg's own NCCL communicator (1 rank): dlopen of
    libnccl, ncclCommInitRank, partial moments, ncclAllReduce, relax_from_w."""
    from paper_1702_00169_b200 import pdg
    cfg = CONFIGS[3].resized(6).stabilised()
    pb, f0, fbg = seeded_equilibrium(cfg)
    S = gpu_with_state(cfg, f0, fbg, nccl_id=pdg.nccl_unique_id(), flags=pdg.PDG_PROFILE)
    S.step(3)
    got = to_np(S.get_state(), f0.shape)
    prof = S.profile_read()
    assert prof["allreduce"][1] == 3 and prof["relax_from_w"][1] == 3 and prof["relax_xsweep"][1] == 0
    assert rel_maxnorm(got, O.m2_run(pb, f0, fbg, 3)) < TOL_STEP
    w = to_np(S.moments(), (cfg.m,) + cfg.grid_shape)
    assert rel_maxnorm(w, O.moments(pb, O.m2_run(pb, f0, fbg, 3))) < TOL_STEP


@pytest.mark.parametrize("scheme_name,tau", [("m2kin", 0.0), ("m4", 0.05), ("m4", 0.0)])
def test_composed_schemes(scheme_name, tau):
    """M2kin (NEXT-1) and the fourth-order composition M4 (NEXT-4) vs the oracle."""
    from paper_1702_00169_b200 import pdg
    code = {"m2kin": pdg.PDG_SCHEME_M2KIN, "m4": pdg.PDG_SCHEME_M4}[scheme_name]
    # the negative substep of M4 sweeps with kappa < 0, where the carry factor |beta| grows
    # quickly: only small CFL numbers are stable (config-1 model, nu = 0.5)
    cfg = CONFIGS[1].resized(16) if scheme_name == "m4" else CONFIGS[3].resized(5).stabilised()
    pb, f0, fbg = seeded_equilibrium(cfg)
    pb.tau = tau
    S = gpu_with_state(cfg, f0, fbg, scheme=code, tau=tau)
    S.step(3)
    ref = O.scheme_run(pb, f0, fbg, 3, scheme_name)
    assert rel_maxnorm(to_np(S.get_state(), f0.shape), ref) < TOL_STEP


# --------------------------------------------------------------------------
# Row e: z-slab decomposition, emulated on one GPU with sub-slabs (same arithmetic as
# one slab per rank: zero-inflow slab sweeps, affine carry scan, correction)
# --------------------------------------------------------------------------
@pytest.mark.parametrize("key,N,S,steps", [(3, 8, 2, 3), (3, 8, 4, 3), (3, 10, 4, 2), (4, 6, 3, 2),
                                           (5, 16, 8, 2), (2, 24, 5, 3), (1, 37, 6, 3)])
def test_zslab_emulated_parity(key, N, S, steps):
    from paper_1702_00169_b200 import pdg
    cfg = CONFIGS[key].resized(N)
    if key != 1:
        cfg = cfg.stabilised()
    pb, f0, fbg = seeded_equilibrium(cfg)
    Z = gpu_with_state(cfg, f0, fbg, decomposition=pdg.PDG_DECOMP_ZSLAB, slabs_per_rank=S, flags=pdg.PDG_PROFILE)
    Z.step(steps)
    assert Z.profile_read()["zslab"][1] > 0
    got = to_np(Z.get_state(), f0.shape)
    assert rel_maxnorm(got, O.m2_run(pb, f0, fbg, steps)) < TOL_STEP


@pytest.mark.parametrize("dtp_frac", [0.5, 1.7, -0.05])
def test_zslab_single_transport(dtp_frac):
    from paper_1702_00169_b200 import pdg
    cfg = CONFIGS[4].resized(6)
    f, fb_full = random_inputs(cfg, 21)
    Z = gpu_with_state(cfg, f, fb_full, decomposition=pdg.PDG_DECOMP_ZSLAB, slabs_per_rank=3)
    dtp = dtp_frac * cfg.dt
    Z.transport(dtp)
    pb = oracle_problem(cfg)
    fc = pb.grid_to_cells(f)
    O.t2_all(pb, dtp, fc, pb.grid_to_cells(fb_full))
    assert rel_maxnorm(to_np(Z.get_state(), f.shape), pb.cells_to_grid(fc)) < TOL_OP


def test_zslab_m2kin_and_unfused():
    from paper_1702_00169_b200 import pdg
    cfg = CONFIGS[3].resized(8).stabilised()
    pb, f0, fbg = seeded_equilibrium(cfg)
    for kw in (dict(scheme=pdg.PDG_SCHEME_M2KIN), dict(flags=pdg.PDG_NO_FUSION)):
        Z = gpu_with_state(cfg, f0, fbg, decomposition=pdg.PDG_DECOMP_ZSLAB, slabs_per_rank=4, **kw)
        Z.step(2)
        ref = O.scheme_run(pb, f0, fbg, 2, "m2kin" if "scheme" in kw else "m2")
        assert rel_maxnorm(to_np(Z.get_state(), f0.shape), ref) < TOL_STEP


# --------------------------------------------------------------------------
# Anisotropic boxes (vectorial sets): different cell counts and sizes per axis
# --------------------------------------------------------------------------
@pytest.mark.parametrize("dim,ncell,p,flux,fparams,m,hi", [
    (3, (37, 5, 9), 2, 2, (1.0,), 4, (1.0, 0.4, 0.7)),
    (3, (4, 33, 3), 3, 2, (1.0,), 4, (0.5, 1.0, 0.3)),
    (2, (40, 7), 2, 1, (1.4,), 4, (1.0, 0.25, 1.0)),
    (2, (3, 70), 1, 0, (1.0, -0.5), 1, (1.0, 1.0, 1.0)),
])
def test_anisotropic_transport_and_steps(dim, ncell, p, flux, fparams, m, hi):
    from paper_1702_00169_b200 import pdg
    from pdg_inputs import velocity_set
    lam = 3.5
    vel, comp = velocity_set(dim, m, lam)
    h = min(hi[d] / ncell[d] for d in range(dim))
    dt = 0.6 * h / lam
    pb = pdg.make_problem(dim, list(ncell), p, m, vel, comp, lam, flux, list(fparams), dt, hi=tuple(hi))
    ob = O.Problem(dim, list(ncell), p, vel, comp, m, lam, flux, list(fparams), dt, hi=list(hi))
    S = pdg.Solver(pb)
    shape = ob.grid_shape()
    rng = np.random.default_rng(sum(ncell))
    # positive density state near equilibrium-like magnitudes (Euler needs positive pressure)
    base = {0: 0.5, 1: 1.0, 2: 1.0}[flux]
    f = base * (1.0 + 0.05 * (rng.random((ob.nv,) + shape) - 0.5)) / (2 * dim)
    if flux == 1:  # energy component: keep E large enough for p > 0
        f[3 * 2 * dim:] *= 3.0
    fb_full = base * (1.0 + 0.05 * rng.random((ob.nv,) + shape)) / (2 * dim)

    class _C:
        pass
    cv = _C()
    cv.dim, cv.grid_shape = dim, shape
    S.set_state(to_dev(f), to_dev(full_grid_to_planes(cv, fb_full, S.sizes.plane_stride)))
    S.transport(dt)
    got = to_np(S.get_state(), f.shape)
    fc = ob.grid_to_cells(f)
    fbc = ob.grid_to_cells(fb_full)
    O.t2_all(ob, dt, fc, fbc)
    assert rel_maxnorm(got, ob.cells_to_grid(fc)) < TOL_OP
    S.step(3)
    got3 = to_np(S.get_state(), f.shape)
    ref3 = O.m2_run(ob, ob.cells_to_grid(fc), fb_full, 3)
    S.destroy()
    assert rel_maxnorm(got3, ref3) < TOL_STEP


def test_async_host_mode_equals_sync():
    """PDG_ASYNC_HOST: host-pointer uploads staged in the extra work region, downloads on the
    copy stream, no synchronisation until pdg_synchronize -- same results as the synchronous
    calls, step by step (each step re-initialised from host w0, as in bench.py's e2e loop)."""
    import torch
    from paper_1702_00169_b200 import pdg
    from pdg_inputs import lbm_config
    for cfg in (CONFIGS[3].resized(6).stabilised(), lbm_config("D3Q19", 5)):
        w0 = w0_grid(cfg).reshape(-1)
        outs = {}
        for mode in ("sync", "async"):
            flags = pdg.PDG_ASYNC_HOST if mode == "async" else 0
            S = make_solver(cfg, flags=flags)
            if mode == "async":
                assert S.sizes.work_bytes >= 8 * cfg.m * cfg.nnodes
            w_host = w0.clone().pin_memory()
            res = [torch.empty(S.sizes.w_elems, dtype=torch.float64).pin_memory() for _ in range(3)]
            for k in range(3):
                S.set_equilibrium(w_host)
                S.step(k + 1)
                S.moments(res[k])
            S.synchronize()
            outs[mode] = [r.numpy().copy() for r in res]
            S.destroy()
        for a, b in zip(outs["sync"], outs["async"]):
            assert np.array_equal(a, b)


def test_nccl_pipelined_sharded_collision_chunks():
    """The sharded collision pipelined over node chunks (partial moments of chunk k, its NCCL sum on
    the communicator stream, relaxation of chunk k once summed; SURVEY §8(e) mitigation 2), through
    libpdg's own single-rank communicator on a grid large enough for several chunks (>= 2^20 nodes
    each): equal to the oracle's M2 steps."""
    from paper_1702_00169_b200 import pdg
    cfg = CONFIGS[3].resized(48).stabilised()        # 144^3 = 2.99 M nodes -> 2 chunks
    pb, f0, fbg = seeded_equilibrium(cfg)
    S = gpu_with_state(cfg, f0, fbg, nccl_id=pdg.nccl_unique_id(), flags=pdg.PDG_PROFILE)
    S.step(2)
    got = to_np(S.get_state(), f0.shape)
    prof = S.profile_read()
    assert prof["allreduce"][1] == 2 * 2 and prof["partial_moments"][1] == 2 * 2, prof
    assert rel_maxnorm(got, O.m2_run(pb, f0, fbg, 2)) < TOL_STEP
    S.destroy()


@pytest.mark.parametrize("dim,ncell,p,flux,fparams,m,nu", [
    (2, (16, 16), 2, 1, (1.4,), 4, 2.0),       # 2-D Euler: 48-node lines tile by 16
    (2, (32, 32), 2, 1, (1.4,), 4, 2.0),
    (2, (20, 20), 3, 1, (1.4,), 4, 2.0),       # p = 3: 80-node lines
    (2, (40, 24), 1, 2, (1.0,), 3, 2.0),       # p = 1, anisotropic
    # 3-D with few strided lines: y and z tiles.  nu = 0.6: at nu = 2 this random state amplifies a
    # one-ulp perturbation to 2.7e-11 in three steps in the oracle itself (3.0e-14 at nu = 0.6)
    (3, (4, 30, 30), 3, 2, (1.0,), 4, 0.6),
])
def test_strided_tile_kernel_parity(dim, ncell, p, flux, fparams, m, nu):
    """sweep_cols_kernel (grids with few strided lines: tiles of 8 adjacent lines staged in shared
    memory, warp-scan sweeps; the config-2 y-velocity path) inside free-running M2 steps (fused
    two-sweep passes and single passes) against the oracle."""
    from paper_1702_00169_b200 import pdg
    from pdg_inputs import velocity_set
    lam = 3.5
    vel, comp = velocity_set(dim, m, lam)
    h = 1.0 / ncell[0]
    hi = tuple(ncell[d] * h for d in range(dim)) + (1.0,) * (3 - dim)
    dt = nu * h / lam
    pb = pdg.make_problem(dim, list(ncell), p, m, vel, comp, lam, flux, list(fparams), dt, hi=hi)
    ob = O.Problem(dim, list(ncell), p, vel, comp, m, lam, flux, list(fparams), dt, hi=list(hi))
    S = pdg.Solver(pb)
    shape = ob.grid_shape()
    rng = np.random.default_rng(sum(ncell) + p)
    base = {1: 1.0, 2: 1.0}[flux]
    f = base * (1.0 + 0.05 * (rng.random((ob.nv,) + shape) - 0.5)) / (2 * dim)
    if flux == 1:
        f[3 * 2 * dim:] *= 3.0  # energy large enough for a positive pressure
    fb_full = base * (1.0 + 0.05 * rng.random((ob.nv,) + shape)) / (2 * dim)
    if flux == 1:
        fb_full[3 * 2 * dim:] *= 3.0

    class _C:
        pass
    cv = _C()
    cv.dim, cv.grid_shape = dim, shape
    S.set_state(to_dev(f), to_dev(full_grid_to_planes(cv, fb_full, S.sizes.plane_stride)))
    S.step(3)
    got = to_np(S.get_state(), f.shape)
    S.destroy()
    assert rel_maxnorm(got, O.m2_run(ob, f, fb_full, 3)) < TOL_STEP


@pytest.mark.parametrize("G", [2, 3, 4, 8])
def test_velocity_sharded_steps_standin(G):
    """The velocity decomposition over whole M2 steps, G shards on one GPU (row a4/e): each shard
    context transports only its velocity block (T2 is block-diagonal over velocities),
    the collision is split into the shards' partial moments, a sum over shards (torch here, NCCL
    in libpdg) and the relaxation of each block from the summed moments.  Two steps against the
    oracle's M2 on the undecomposed problem; G = 3 gives uneven blocks (24 = 8 + 8 + 8 is even, so
    use the 16-velocity 2-D Euler model: 6 + 5 + 5)."""
    cfg = (CONFIGS[2].resized(20) if G == 3 else CONFIGS[3].resized(5)).stabilised()
    pb, f0, fbg = seeded_equilibrium(cfg)
    shards = []
    for r in range(G):
        S = make_solver(cfg, rank=r, nranks=G)
        v0, nvl = S.sizes.v_begin, S.sizes.nv_local
        planes = full_grid_to_planes(cfg, fbg[v0:v0 + nvl], S.sizes.plane_stride, v_begin=v0)
        S.set_state(to_dev(f0[v0:v0 + nvl]), to_dev(planes))
        shards.append(S)
    for _ in range(2):
        for S in shards:
            S.transport(0.5 * cfg.dt)
            S.partial_moments()
        wsum = sum(S.w for S in shards)
        for S in shards:
            S.w.copy_(wsum)
            S.relax_from_w(cfg.dt)
            S.transport(0.5 * cfg.dt)
    got = np.concatenate([to_np(S.get_state(), (S.sizes.nv_local,) + cfg.grid_shape) for S in shards])
    for S in shards:
        S.destroy()
    assert rel_maxnorm(got, O.m2_run(pb, f0, fbg, 2)) < TOL_STEP


@pytest.mark.parametrize("kind,steps", [("iso", 7), ("iso", 300), ("lbm", 5), ("zslab", 4)])
def test_step_graph_replay_equals_direct_launches(kind, steps):
    """pdg_step(n) replays a CUDA graph of its launch sequence (captured once per n on a library
    stream, launched on the caller's): bit-identical to the direct launches (PDG_NO_GRAPH), on the
    default stream, twice in a row (the second call replays the cached graph), for a long call
    (n = 300), a lattice set and the emulated z-slab decomposition."""
    from paper_1702_00169_b200 import pdg
    from pdg_inputs import lbm_config
    if kind == "lbm":
        cfg = lbm_config("D3Q19", 6)
    else:
        cfg = CONFIGS[3].resized(4 if steps > 100 else 6).stabilised()
    kw = dict(decomposition=pdg.PDG_DECOMP_ZSLAB, slabs_per_rank=3) if kind == "zslab" else {}
    w0 = w0_grid(cfg).reshape(-1).cuda()
    outs = []
    for flags in (0, pdg.PDG_NO_GRAPH):
        S = make_solver(cfg, flags=flags, **kw)
        S.set_equilibrium(w0)
        S.step(steps)
        S.step(steps)
        outs.append(S.get_state().clone())
        S.destroy()
    assert torch.equal(outs[0], outs[1])


def test_profile_pause_and_resume():
    """pdg_profile_enable: paused events record nothing (and let pdg_step replay its graph), resumed
    events count every launch again; same results either way."""
    from paper_1702_00169_b200 import pdg
    cfg = CONFIGS[3].resized(6).stabilised()
    pb, f0, fbg = seeded_equilibrium(cfg)
    S = gpu_with_state(cfg, f0, fbg, flags=pdg.PDG_PROFILE)
    S.profile_enable(False)
    S.step(3)
    assert sum(v[1] for v in S.profile_read().values()) == 0
    S.profile_enable(True)
    S.step(3)
    prof = S.profile_read()
    assert prof["relax_xsweep"][1] == 3 and prof["sweep_strided"][1] == 4, prof
    assert rel_maxnorm(to_np(S.get_state(), f0.shape), O.m2_run(pb, f0, fbg, 6)) < TOL_STEP
    S.destroy()
    T = make_solver(cfg)
    with pytest.raises(pdg.PdgError):
        T.profile_enable(True)  # created without PDG_PROFILE
    T.destroy()


@pytest.mark.parametrize("key,N,scheme_name,tau,steps", [
    (1, 8, "m2", 0.0, 10),       # config 1 as written: 30 operators, one launch
    (1, 8, "m2", 0.0, 40),       # 120 operators: three launches (48 per launch)
    (1, 5, "m2kin", 0.02, 7),
    (1, 8, "m4", 0.05, 3),       # four distinct T2 step sizes in one launch, a negative one
    (2, 3, "m2", 0.0, 6),        # 2-D Euler, 16 velocities (f = 41 KB)
    (3, 2, "m2", 0.0, 5),        # 3-D isothermal, 24 velocities (f = 41 KB)
    (4, 1, "m2kin", 0.01, 4),    # p = 3, one cell per axis
])
def test_small_problem_run(key, N, scheme_name, tau, steps):
    """Small problems (f <= 64 KB): pdg_step runs its operators in one CTA with f in shared memory
    (small_run_kernel) -- against the oracle, against the general per-operator kernels
    (PDG_NO_SMALL) to rounding, and the launch count (ceil(operators / 48) per call)."""
    from paper_1702_00169_b200 import pdg
    code = {"m2": pdg.PDG_SCHEME_M2, "m2kin": pdg.PDG_SCHEME_M2KIN, "m4": pdg.PDG_SCHEME_M4}[scheme_name]
    cfg = CONFIGS[key].resized(N)
    if key != 1:
        cfg = cfg.stabilised()
    pb, f0, fbg = seeded_equilibrium(cfg)
    pb.tau = tau
    ref = O.scheme_run(pb, f0, fbg, steps, scheme_name)
    outs = []
    for flags in (pdg.PDG_PROFILE, pdg.PDG_PROFILE | pdg.PDG_NO_SMALL):
        S = gpu_with_state(cfg, f0, fbg, scheme=code, tau=tau, flags=flags)
        S.step(steps)
        prof = S.profile_read()
        got = to_np(S.get_state(), f0.shape)
        S.destroy()
        assert rel_maxnorm(got, ref) < TOL_STEP, flags
        outs.append(got)
        small = prof["small_run"][1]
        if flags & pdg.PDG_NO_SMALL:
            assert small == 0, prof
        else:
            nops = {"m2": 3, "m2kin": 5, "m4": 15}[scheme_name] * steps
            assert small == -(-nops // 48), prof
            assert sum(v[1] for k, v in prof.items() if k != "small_run") == 0, prof
    assert rel_maxnorm(outs[0], outs[1]) < 1e-13
