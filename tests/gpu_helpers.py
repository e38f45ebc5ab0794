"""Helpers shared by the GPU parity tests (test infrastructure; layout plumbing only).

The CUDA side keeps the inflow data of velocity i as a plane (the node grid with
the velocity axis removed); the oracle keeps f^b at the boundary cell's own face
nodes in a full cell-blocked array.  These helpers move data between the two
layouts -- index permutations, no arithmetic of the method.
"""
from __future__ import annotations

import numpy as np
import torch

from oracle import oracle as O


def rel_maxnorm(x, y) -> float:
    """||x - y||_inf / ||y||_inf over the whole array (reading C17)."""
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    den = np.max(np.abs(y))
    return float(np.max(np.abs(x - y)) / (den if den > 0 else 1.0))


def vel_axis_sign(i: int, dim: int):
    return (i % (2 * dim)) // 2, (-1 if i % 2 else 1)


def planes_to_full_grid(cfg, planes: np.ndarray, v_begin: int = 0) -> np.ndarray:
    """[nvl, plane_stride] GPU planes -> [nvl, grid...] with values on inflow faces, 0 elsewhere."""
    dim = cfg.dim
    shape = cfg.grid_shape  # slow..fast: (Z, Y, X)
    nvl = planes.shape[0]
    out = np.zeros((nvl,) + shape)
    for j in range(nvl):
        k, s = vel_axis_sign(v_begin + j, dim)
        ax = dim - 1 - k  # numpy axis of physical axis k
        pshape = tuple(shape[a] for a in range(dim) if a != ax)
        npl = int(np.prod(pshape))
        plane = planes[j, :npl].reshape(pshape)
        idx = [slice(None)] * dim
        idx[ax] = 0 if s > 0 else shape[ax] - 1
        out[j][tuple(idx)] = plane
    return out


def full_grid_to_planes(cfg, full: np.ndarray, plane_stride: int, v_begin: int = 0) -> np.ndarray:
    """[nvl, grid...] -> [nvl, plane_stride] inflow planes (the face slice of each velocity)."""
    dim = cfg.dim
    shape = cfg.grid_shape
    nvl = full.shape[0]
    out = np.zeros((nvl, plane_stride))
    for j in range(nvl):
        k, s = vel_axis_sign(v_begin + j, dim)
        ax = dim - 1 - k
        idx = [slice(None)] * dim
        idx[ax] = 0 if s > 0 else shape[ax] - 1
        pl = full[j][tuple(idx)].reshape(-1)
        out[j, :pl.size] = pl
    return out


# Launch plan of the lattice sweeps forced by a test (pdg_problem.lattice_cta / lattice_segment;
# zeros: the library's default plan).  Set through the `warps` / `seglen` fixtures.
LATTICE_PLAN = {"lattice_cta": (0, 0), "lattice_segment": 0}


def make_solver(cfg, **kw):
    from paper_1702_00169_b200 import pdg
    pb = pdg.problem_from_config(cfg, **{**LATTICE_PLAN, **kw})
    return pdg.Solver(pb)


def to_dev(a: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64).reshape(-1)).cuda()


def to_np(t: torch.Tensor, shape) -> np.ndarray:
    return t.detach().cpu().numpy().reshape(shape)


def oracle_problem(cfg, tau=0.0):
    return O.Problem.from_config(cfg, tau=tau)


def lattice_planes(cfg, full: np.ndarray, plane_stride: int, v_begin: int = 0) -> np.ndarray:
    """Lattice sets (PDG_FLUX_LBM): [nvl, grid...] -> [nvl, dim, plane_stride]; plane k of velocity i
    is the face slice of its inflow face across axis k (include/pdg.h), unused when v_i^k = 0."""
    vel, _ = cfg.velocities()
    dim, shape = cfg.dim, cfg.grid_shape
    nvl = full.shape[0]
    out = np.zeros((nvl, dim, plane_stride))
    for j in range(nvl):
        for k in range(dim):
            vk = vel[v_begin + j][k]
            if vk == 0:
                continue
            ax = dim - 1 - k
            idx = [slice(None)] * dim
            idx[ax] = 0 if vk > 0 else shape[ax] - 1
            pl = full[j][tuple(idx)].reshape(-1)
            out[j, k, :pl.size] = pl
    return out
