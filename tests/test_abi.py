"""CPU checks of the boundary: the library loads, exports every symbol declared in
include/pdg.h, and validates problem statements host-side (no GPU needed)."""
import ctypes
import os
import re

import pytest

from paper_1702_00169_b200 import pdg
from pdg_inputs import CONFIGS

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    txt = open(os.path.join(ROOT, "include", "pdg.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(pdg_[a-z_0-9]+)\s*\(", txt)))


def test_header_symbols_exported():
    lib = pdg.load()
    names = declared_symbols()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(pdg.EXPORTED)


def test_checked_build_exports_the_same_symbols():
    """The bounds-checked build (build.py --checked) is the same C-ABI."""
    path = os.path.join(ROOT, "paper_1702_00169_b200", "libpdg_checked.so")
    if not os.path.exists(path):
        from paper_1702_00169_b200 import build
        build.build(checked=True)
    lib = ctypes.CDLL(path)
    for n in declared_symbols():
        assert hasattr(lib, n), n


def test_version_and_status_strings():
    assert "sm_100a" in pdg.version()
    assert pdg.status_string(pdg.PDG_E_VELOCITY_SET) == "PDG_E_VELOCITY_SET"


@pytest.mark.parametrize("key", [1, 2, 3, 4, 5])
def test_query_sizes_configs(key):
    cfg = CONFIGS[key]
    s = pdg.query_sizes(pdg.problem_from_config(cfg))
    assert s.nnodes == cfg.nnodes
    assert s.f_elems == cfg.nv * cfg.nnodes
    assert s.w_elems == cfg.m * cfg.nnodes
    assert s.plane_stride == (cfg.N * cfg.n) ** (cfg.dim - 1)
    assert s.nv_local == cfg.nv and s.v_begin == 0


def test_query_sizes_sharded():
    cfg = CONFIGS[5]
    for G in (2, 4, 8):
        for r in range(G):
            s = pdg.query_sizes(pdg.problem_from_config(cfg, rank=r, nranks=G))
            assert s.nv_local == 24 // G and s.v_begin == r * (24 // G)
            assert s.f_elems == (24 // G) * cfg.nnodes


def _bad(cfg, **over):
    vel, comp = cfg.velocities()
    kw = dict(dim=cfg.dim, ncell=cfg.N, degree=cfg.p, m=cfg.m, vel=vel, comp=comp, lam=cfg.lam, flux=cfg.flux,
              flux_params=list(cfg.fparams), dt=cfg.dt)
    kw.update(over)
    with pytest.raises(pdg.PdgError) as e:
        pdg.query_sizes(pdg.make_problem(**kw))
    return e.value.status


def _good(cfg, **over) -> bool:
    vel, comp = cfg.velocities()
    kw = dict(dim=cfg.dim, ncell=cfg.N, degree=cfg.p, m=cfg.m, vel=vel, comp=comp, lam=cfg.lam, flux=cfg.flux,
              flux_params=list(cfg.fparams), dt=cfg.dt)
    kw.update(over)
    return pdg.query_sizes(pdg.make_problem(**kw)).f_elems > 0


def test_validation_errors():
    cfg = CONFIGS[3]
    assert _bad(cfg, dim=4) == pdg.PDG_E_DIMENSION
    assert _bad(cfg, degree=5) == pdg.PDG_E_DEGREE
    assert _bad(cfg, lam=-1.0) == pdg.PDG_E_INVALID_ARGUMENT
    assert _bad(cfg, dt=0.0) == pdg.PDG_E_INVALID_ARGUMENT
    assert _bad(cfg, m=3) == pdg.PDG_E_FLUX_MODEL
    assert _bad(cfg, flux=7) == pdg.PDG_E_FLUX_MODEL
    vel, comp = cfg.velocities()
    vel2 = [list(v) for v in vel]
    vel2[3][1] = 1.0  # not axis-aligned
    assert _bad(cfg, vel=vel2) == pdg.PDG_E_VELOCITY_SET
    comp2 = list(comp)
    comp2[0] = 1
    assert _bad(cfg, comp=comp2) == pdg.PDG_E_VELOCITY_SET
    assert _bad(cfg, ncell=0) == pdg.PDG_E_INVALID_ARGUMENT
    # tau > 0: every collision substep h of the scheme needs 2 tau + h > 0 (eq collision_cn)
    dt = cfg.dt
    assert _bad(cfg, tau=0.2 * dt, dt=-dt) == pdg.PDG_E_INVALID_ARGUMENT            # M2, C2(-dt)
    assert _bad(cfg, tau=0.1 * dt, scheme=pdg.PDG_SCHEME_M4) == pdg.PDG_E_INVALID_ARGUMENT  # g2 dt/2 < 0
    ok = dict(tau=0.6 * dt, scheme=pdg.PDG_SCHEME_M4)  # 2 tau + g2 dt/2 = (1.2 - 0.85) dt > 0
    assert _good(cfg, **ok) and _good(cfg, tau=0.0, dt=-dt) and _good(cfg, tau=0.3 * dt, dt=-dt,
                                                                       scheme=pdg.PDG_SCHEME_M2KIN)


def test_solver_refuses_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        pdg.Solver(pdg.problem_from_config(CONFIGS[1]))


def test_query_sizes_zslab():
    cfg = CONFIGS[5]
    G = 8
    begins = []
    for r in range(G):
        s = pdg.query_sizes(pdg.problem_from_config(cfg, rank=r, nranks=G, decomposition=pdg.PDG_DECOMP_ZSLAB))
        assert s.nv_local == cfg.nv and s.v_begin == 0
        assert s.cell_count == cfg.N // G and s.cell_begin == r * (cfg.N // G)
        assert s.nnodes_local == cfg.nnodes // G and s.nnodes == cfg.nnodes
        assert s.f_elems == cfg.nv * cfg.nnodes // G
        begins.append(s.cell_begin)
        # carry planes: 8 slabs x 8 z-velocities x 2 passes x 768^2 doubles
        assert s.work_bytes >= 8 * (2 * 8 * 8 * 2 * 768 * 768)
    assert begins == sorted(begins)
    s = pdg.query_sizes(pdg.problem_from_config(CONFIGS[3].resized(10), decomposition=pdg.PDG_DECOMP_ZSLAB,
                                                slabs_per_rank=4))
    assert s.cell_count == 10 and s.nnodes_local == s.nnodes
    with pytest.raises(pdg.PdgError):
        pdg.query_sizes(pdg.problem_from_config(CONFIGS[3].resized(4), decomposition=pdg.PDG_DECOMP_ZSLAB,
                                                slabs_per_rank=8))


# ---- lattice sets (NEXT-2) and the source step (NEXT-3): host-side validation ----------
@pytest.mark.parametrize("lat", ["D2Q9", "D3Q15", "D3Q19", "D3Q27"])
def test_query_sizes_lattice(lat):
    from pdg_inputs import lbm_config
    cfg = lbm_config(lat, 9)
    s = pdg.query_sizes(pdg.problem_from_config(cfg))
    assert s.f_elems == cfg.nv * cfg.nnodes and s.w_elems == cfg.m * cfg.nnodes
    assert s.fb_elems == cfg.nv * cfg.dim * s.plane_stride  # one inflow plane per axis
    for G in (2, 3, 4, 8):  # contiguous blocks, sizes nv//G or nv//G + 1 (first nv % G ranks)
        begin = 0
        for r in range(G):
            t = pdg.query_sizes(pdg.problem_from_config(cfg, rank=r, nranks=G))
            assert t.v_begin == begin and t.nv_local == cfg.nv // G + (1 if r < cfg.nv % G else 0)
            begin += t.nv_local
        assert begin == cfg.nv


def test_lattice_validation_errors():
    from pdg_inputs import lbm_config
    cfg = lbm_config("D2Q9", 4)
    vel, comp = cfg.velocities()
    base = dict(dim=2, ncell=4, degree=2, m=3, vel=vel, comp=comp, lam=cfg.lam, flux=pdg.PDG_FLUX_LBM,
                flux_params=list(cfg.flux_params()), dt=cfg.dt)

    def bad(**over):
        kw = dict(base)
        kw.update(over)
        with pytest.raises(pdg.PdgError) as e:
            pdg.query_sizes(pdg.make_problem(**kw))
        return e.value.status

    assert pdg.query_sizes(pdg.make_problem(**base)).f_elems == 9 * cfg.nnodes
    v2 = [list(v) for v in vel]
    v2[5][0] = 0.5 * cfg.lam  # component not in {0, +-lambda}
    assert bad(vel=v2) == pdg.PDG_E_VELOCITY_SET
    assert bad(flux_params=[cfg.flux_params()[0]]) == pdg.PDG_E_FLUX_MODEL  # weights missing
    assert bad(m=4) == pdg.PDG_E_FLUX_MODEL
    assert bad(vel=vel[:8], comp=comp[:8], flux_params=list(cfg.flux_params())[:9]) == pdg.PDG_E_UNSUPPORTED
    assert bad(scheme=pdg.PDG_SCHEME_M2S) == pdg.PDG_E_INVALID_ARGUMENT  # M2s without a source
    ok = pdg.make_problem(**base, scheme=pdg.PDG_SCHEME_M2S, gravity=(0.0, -1.0))
    assert pdg.query_sizes(ok).nv_local == 9
    assert bad(decomposition=pdg.PDG_DECOMP_ZSLAB, nranks=2) == pdg.PDG_E_UNSUPPORTED
    c3 = CONFIGS[3]
    v3, c3comp = c3.velocities()
    with pytest.raises(pdg.PdgError) as e:  # gravity needs the LBM model
        pdg.query_sizes(pdg.make_problem(3, 4, 2, 4, v3, c3comp, c3.lam, c3.flux, list(c3.fparams), c3.dt,
                                         gravity=(0.0, 0.0, -1.0)))
    assert e.value.status == pdg.PDG_E_UNSUPPORTED


def test_product_never_uses_the_oracle():
    """The product path (package + CUDA sources) neither imports nor links anything under oracle/;
    only tests, __graft_entry__.smoke() and bench.py's baseline legs may."""
    pkg = os.path.join(ROOT, "paper_1702_00169_b200")
    offenders = []
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".hpp", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, fn), errors="ignore").read()
                if re.search(r"(import\s+oracle|from\s+oracle|liboracle|#\s*include[^\n]*oracle|pdg_oracle)", txt):
                    offenders.append(fn)
    assert offenders == []
