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
