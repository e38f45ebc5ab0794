"""Host-side plumbing of the velocity-sharded multi-GPU path.

Velocities are independent during transport (L_h is block-diagonal over
velocities), so rank r owns the contiguous velocity block [r nv/G, (r+1) nv/G) and the
only exchange is one fp64 sum of the moment fields per collision, done by
libpdg's own NCCL communicator inside pdg_step / pdg_collide.  torch.distributed only
bootstraps that communicator (the 128-byte ncclUniqueId broadcast) and provides
barriers and the max-over-ranks timing reduction.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import pdg


def shard(cfg, rank: int, world: int):
    """(v_begin, nv_local) of `rank` as libpdg computes it (pdg_query_sizes)."""
    s = pdg.query_sizes(pdg.problem_from_config(cfg, rank=rank, nranks=world))
    return s.v_begin, s.nv_local


def bootstrap_nccl_id(group=None, device=None) -> bytes:
    """Rank 0 creates an ncclUniqueId, every rank returns the same 128 bytes."""
    rank = dist.get_rank(group)
    backend = dist.get_backend(group)
    dev = device if (backend == "nccl") else torch.device("cpu")
    buf = torch.zeros(128, dtype=torch.uint8, device=dev)
    if rank == 0:
        buf.copy_(torch.frombuffer(bytearray(pdg.nccl_unique_id()), dtype=torch.uint8))
    dist.broadcast(buf, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    return bytes(buf.cpu().numpy().tobytes())


def max_over_ranks(value: float, device=None, group=None) -> float:
    """Max of a per-rank scalar (device times: the slowest rank defines the step)."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return float(value)
    backend = dist.get_backend(group)
    dev = device if backend == "nccl" else torch.device("cpu")
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def sum_over_ranks(value: float, device=None, group=None) -> float:
    """Sum of a per-rank scalar (e.g. counts of non-physical nodes)."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return float(value)
    backend = dist.get_backend(group)
    dev = device if backend == "nccl" else torch.device("cpu")
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return float(t.item())


def sharded_solver(cfg, device, flags=0, stream=None, tau=0.0, scheme=pdg.PDG_SCHEME_M2,
                   decomposition=pdg.PDG_DECOMP_VELOCITY, slabs_per_rank=1, **plan):
    """A libpdg context for this rank's share (velocity block or z-slab), with its NCCL communicator."""
    world = dist.get_world_size() if dist.is_initialized() else 1
    rank = dist.get_rank() if dist.is_initialized() else 0
    # a communicator only with several ranks: one rank keeps the fused single-GPU path
    # (collision fused with the x sweeps, no partial-moment round trip through HBM)
    nccl_id = bootstrap_nccl_id(device=device) if dist.is_initialized() and world > 1 else None
    pb = pdg.problem_from_config(cfg, tau=tau, scheme=scheme, rank=rank, nranks=world, nccl_id=nccl_id,
                                 flags=flags, stream=stream, decomposition=decomposition,
                                 slabs_per_rank=slabs_per_rank, **plan)
    return pdg.Solver(pb, device=device)
