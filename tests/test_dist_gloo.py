"""World-size-2 gloo tests (CPU) of the host logic of the velocity-sharded path:
NCCL-id bootstrap, shard partition, max-over-ranks timing, and the decomposition
of the collision into per-rank partial moments + a sum over ranks (checked with the
oracle's arithmetic standing in for the kernels)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, fn, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def run_world(fn, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, fn, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    return [out[r] for r in range(world)]


def _bootstrap(rank, world):
    from paper_1702_00169_b200 import dist as pd
    return pd.bootstrap_nccl_id()


def test_nccl_id_bootstrap_is_identical_on_all_ranks():
    ids = run_world(_bootstrap)
    assert all(isinstance(i, bytes) and len(i) == 128 for i in ids), ids
    assert ids[0] == ids[1]


def _maxrank(rank, world):
    from paper_1702_00169_b200 import dist as pd
    return pd.max_over_ranks(10.0 + rank)


def test_max_over_ranks():
    assert run_world(_maxrank) == [11.0, 11.0]


def _shards(rank, world):
    from paper_1702_00169_b200 import dist as pd
    from pdg_inputs import CONFIGS, lbm_config
    return [pd.shard(c, rank, world) for c in (CONFIGS[2], CONFIGS[5], lbm_config("D3Q27", 4))]


def test_shards_partition_the_velocities():
    res = run_world(_shards)
    for k, nv in enumerate((16, 24)):
        got = sorted(r[k] for r in res)
        assert got == [(0, nv // 2), (nv // 2, nv // 2)]
    # odd lattice set: uneven contiguous blocks (14 + 13)
    assert sorted(r[2] for r in res) == [(0, 14), (14, 13)]


def _sharded_collision(rank, world):
    """Partial moments of this rank's velocity block, summed with all_reduce, then the
    collision of the local block only: must equal the full single-process collision."""
    from oracle import oracle as O
    from paper_1702_00169_b200 import dist as pd
    from pdg_inputs import CONFIGS, random_state
    cfg = CONFIGS[3].resized(3)
    pb = O.Problem.from_config(cfg)
    f = random_state(cfg, 11).numpy().reshape(cfg.nv, -1)
    v0, nvl = pd.shard(cfg, rank, world)
    local = np.zeros_like(f)
    local[v0:v0 + nvl] = f[v0:v0 + nvl]
    w = torch.from_numpy(O.moments(pb, local))       # partial moments of this rank
    dist.all_reduce(w)                                # the exchange step
    full = np.ascontiguousarray(f.copy())
    O.collide(pb, full, cfg.dt)
    # collision of the local block from the reduced w: f^eq(w) is the same on every rank
    feq = O.equilibrium_field(pb, w.numpy())
    mine = 2.0 * feq[v0:v0 + nvl] - f[v0:v0 + nvl]
    return float(np.max(np.abs(mine - full[v0:v0 + nvl])) / np.max(np.abs(full)))


def test_sharded_collision_decomposition():
    errs = run_world(_sharded_collision)
    assert all(isinstance(e, float) and e < 1e-14 for e in errs), errs


# --------------------------------------------------------------------------
# The exact z-slab decomposition (row e): each rank sweeps its slab of cell planes with
# zero inflow, the outgoing carries of every slab are all-gathered (gloo here, NCCL in libpdg),
# the true slab inflows follow from the affine carry scan with the product's tables
# (pdg_zslab_table: B = beta^len, C), and the first leff cells are corrected with its P, Q
# responses.  The slab sweeps themselves are the oracle's (standing in for the CUDA kernels); the
# result must equal the oracle's sweep of the whole domain.
# --------------------------------------------------------------------------
def _zslab_world(rank, world, p=2, nu_half=1.0, nz=64):
    from oracle import oracle as O
    from paper_1702_00169_b200 import pdg
    n, nx, ny, lam = p + 1, 2, 3, 2.0
    h = 1.0 / nz
    dtp = nu_half * h / lam           # kappa = lambda dt' / h
    lo, hi = (0.0, 0.0, 0.0), (nx * h, ny * h, 1.0)
    lines = (nx * n) * (ny * n)
    rng = np.random.default_rng(5)
    fz = rng.random((nz * n, ny * n, nx * n))          # one z-velocity's node grid [Z][Y][X]
    fbz = rng.random((ny * n, nx * n))                 # its inflow plane
    out = {}
    for sgn in (+1.0, -1.0):
        v = [0.0, 0.0, sgn * lam]
        # the whole domain, two consecutive T2(dt') sweeps (the fused y/z pass of pdg_step)
        full = O.Problem(3, [nx, ny, nz], p, [v], [0], 1, lam, 0, [1.0, 0.0, 0.0], 2 * dtp, lo=lo, hi=hi)
        fb_full = np.zeros_like(fz)
        fb_full[0 if sgn > 0 else -1] = fbz
        fc = full.grid_to_cells(fz[None])[0]
        O.t2_velocity(full, v, dtp, fc, full.grid_to_cells(fb_full[None])[0])
        O.t2_velocity(full, v, dtp, fc, full.grid_to_cells(fb_full[None])[0])
        ref = full.cells_to_grid(fc[None])[0]
        # this rank's slab, swept with zero inflow unless the velocity enters the domain here
        z0, z1 = rank * nz // world, (rank + 1) * nz // world
        ln = z1 - z0
        entry = (rank == 0) if sgn > 0 else (rank == world - 1)
        sub = O.Problem(3, [nx, ny, ln], p, [v], [0], 1, lam, 0, [1.0, 0.0, 0.0], 2 * dtp,
                        lo=(0.0, 0.0, z0 * h), hi=(nx * h, ny * h, z1 * h))
        f0 = fz[z0 * n:z1 * n].copy()
        fb_sub = np.zeros_like(f0)
        if entry:
            fb_sub[0 if sgn > 0 else -1] = fbz
        c = sub.grid_to_cells(f0[None])[0]
        fbc = sub.grid_to_cells(fb_sub[None])[0]
        O.t2_velocity(sub, v, dtp, c, fbc)
        f1 = sub.cells_to_grid(c[None])[0]
        O.t2_velocity(sub, v, dtp, c, fbc)
        f2 = sub.cells_to_grid(c[None])[0]
        # outgoing carries of the two zero-inflow passes: old + new trace at the outflow face
        o = -1 if sgn > 0 else 0
        A = torch.from_numpy(np.stack([f0[o] + f1[o], f1[o] + f2[o]]).reshape(2, lines).copy())
        gathered = [torch.zeros_like(A) for _ in range(world)]
        dist.all_gather(gathered, A)                    # the carry-plane exchange
        # product tables for every slab length (the tables depend on p and kappa of the outer axis)
        from pdg_inputs import velocity_set
        vs, cs = velocity_set(3, 1, lam)
        pb = pdg.make_problem(3, [nx, ny, nz], p, 1, vs, cs, lam, 0, [1.0, 0.0, 0.0], 2 * dtp, lo=lo, hi=hi)
        P_, Q_, B_, C_, leff = pdg.zslab_table(pb, dtp, 2, ln)
        tabs = {}
        for r in range(world):
            lr = (r + 1) * nz // world - r * nz // world
            tabs[r] = pdg.zslab_table(pb, dtp, 2, lr)
        # affine scan over the slabs upstream of this one (flow order)
        order = list(range(world)) if sgn > 0 else list(reversed(range(world)))
        s1 = s2 = None
        for r in order:
            if r == rank:
                break
            a1, a2 = gathered[r][0].numpy(), gathered[r][1].numpy()
            if s1 is None:
                s1, s2 = a1, a2                           # the entry slab: true carries
            else:
                Br, Cr = tabs[r][2], tabs[r][3]
                s1, s2 = a1 + Br * s1, a2 + Br * s2 + Cr * s1
        got = f2.copy()
        if s1 is not None:
            S1, S2 = s1.reshape(ny * n, nx * n), s2.reshape(ny * n, nx * n)
            for l in range(min(ln, leff)):
                for a in range(n):
                    zz = (l * n + a) if sgn > 0 else (ln * n - 1 - (l * n + a))
                    got[zz] += Q_[l][a] * S2 + P_[l][a] * S1
        mine = ref[z0 * n:z1 * n]
        out[sgn] = float(np.max(np.abs(got - mine)) / np.max(np.abs(ref)))
        out[("leff", sgn)] = leff
    return out


def _zslab_p2(rank, world):
    return _zslab_world(rank, world, p=2, nu_half=1.0, nz=64)


def _zslab_p3(rank, world):
    return _zslab_world(rank, world, p=3, nu_half=2.0, nz=32)


@pytest.mark.parametrize("world,fn", [(2, _zslab_p2), (4, _zslab_p2), (2, _zslab_p3), (4, _zslab_p3)])
def test_zslab_carry_scan_with_product_tables(world, fn):
    res = run_world(fn, world=world)
    for r in res:
        assert isinstance(r, dict), r
        assert r[1.0] < 1e-13 and r[-1.0] < 1e-13, r
    if fn is _zslab_p2 and world == 2:
        assert res[0][("leff", 1.0)] < 64 // world  # the correction stops inside the slab (reading C26)
