"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the PDG method: it only describes the five
BASELINE.json configurations (and their stabilised twins, DESIGN.md "parity
protocol"), draws their random phases with a counter-based SplitMix64, and
evaluates the macroscopic initial state w0(x) on the node grid.  Turning w0
into kinetic data f0 = f^eq(w0) and inflow data f^b = f^eq(w_b) is done by
each side on its own (oracle: oracle/oracle.py, product: pdg_set_equilibrium).

The paper uses no public dataset (its torus mesh, is not
available); these recipes stand in for its workloads with the shapes, sizes
and smooth value distributions of the configs (SURVEY.md §8(d) "Synthetic
inputs").  Node positions: x = lo + (c + (xhat_a + 1)/2) h per axis, with xhat
the 1-D Gauss-Lobatto points (textbook closed forms; used here only as the
sample positions of the input fields).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field, replace

import torch

# flux model ids (same numbering on both sides is part of the problem statement)
FLUX_ADVECTION = 0
FLUX_EULER = 1
FLUX_ISOTHERMAL = 2
FLUX_LBM = 3

# Lattice-Boltzmann velocity sets (unit vectors; scaled by lambda) and weights.
# D2Q9 in the paper's order and with its weights; the 3-D lattices are the
# standard D3Q15/D3Q19/D3Q27 sets the paper benchmarks.
def _lattice(name):
    axis2 = [(1, 0), (0, 1), (-1, 0), (0, -1)]
    if name == "D2Q9":
        v = [(0, 0)] + axis2 + [(1, 1), (-1, 1), (-1, -1), (1, -1)]
        w = [4 / 9] + [1 / 9] * 4 + [1 / 36] * 4
        return [list(x) + [0] for x in v], w
    axis3 = [(1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1)]
    edges = [(a, b, 0) for a in (1, -1) for b in (1, -1)] + [(a, 0, b) for a in (1, -1) for b in (1, -1)] + \
            [(0, a, b) for a in (1, -1) for b in (1, -1)]
    corners = [(a, b, c) for a in (1, -1) for b in (1, -1) for c in (1, -1)]
    if name == "D3Q15":
        return [(0, 0, 0)] + axis3 + corners, [2 / 9] + [1 / 9] * 6 + [1 / 72] * 8
    if name == "D3Q19":
        return [(0, 0, 0)] + axis3 + edges, [1 / 3] + [1 / 18] * 6 + [1 / 36] * 12
    if name == "D3Q27":
        return [(0, 0, 0)] + axis3 + edges + corners, [8 / 27] + [2 / 27] * 6 + [1 / 54] * 12 + [1 / 216] * 8
    raise ValueError(name)


def lattice(name: str, lam: float):
    """(velocities [nv][3], weights [nv]) of a lattice scaled by lambda."""
    v, w = _lattice(name)
    return [[lam * float(c) for c in x] for x in v], [float(x) for x in w]

MASK64 = (1 << 64) - 1


def splitmix64(seed: int):
    """Counter-based SplitMix64 stream of 64-bit integers."""
    state = seed & MASK64
    while True:
        state = (state + 0x9E3779B97F4A7C15) & MASK64
        z = state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        yield z ^ (z >> 31)


def phases(seed: int, count: int) -> list[float]:
    """phi = 2 pi u, u = (SplitMix64 >> 11) * 2^-53, drawn in order."""
    g = splitmix64(seed)
    return [2.0 * math.pi * ((next(g) >> 11) * 2.0 ** -53) for _ in range(count)]


def gl_sample_points(p: int) -> list[float]:
    """1-D Gauss-Lobatto points on [-1, 1] (sample positions only)."""
    s5 = 1.0 / math.sqrt(5.0)
    s37 = math.sqrt(3.0 / 7.0)
    table = {1: [-1.0, 1.0], 2: [-1.0, 0.0, 1.0], 3: [-1.0, -s5, s5, 1.0],
             4: [-1.0, -s37, 0.0, s37, 1.0]}
    if p not in table:
        raise ValueError(f"degree {p} not supported by the input generator")
    return table[p]


def velocity_set(dim: int, m: int, lam: float):
    """Vectorial D2Q4/D3Q6 per component (reading C6): velocity index
    i = c*2D + 2k + (0 for +lambda e_k, 1 for -lambda e_k); comp[i] = c."""
    vel, comp = [], []
    for c in range(m):
        for k in range(dim):
            for s in (1.0, -1.0):
                v = [0.0, 0.0, 0.0]
                v[k] = s * lam
                vel.append(v)
                comp.append(c)
    return vel, comp


@dataclass(frozen=True)
class Config:
    name: str
    dim: int
    N: int              # cells per axis
    p: int              # degree
    m: int              # conservative variables
    lam: float          # lattice speed lambda
    flux: int
    fparams: tuple      # advection: a[dim]; Euler: (gamma,); isothermal: (c,)
    dt: float
    steps: int
    seed: int
    recipe: str
    wb_zero: bool = False   # config 1: inflow f^b = f^eq(0) = 0
    lo: tuple = (0.0, 0.0, 0.0)
    hi: tuple = (1.0, 1.0, 1.0)
    lattice: str = ""       # LBM lattice name (flux == FLUX_LBM); fparams = (c,) then
    gravity: tuple = ()     # gravity vector G of the Euler-with-gravity source, () if none
    rho0_g: tuple = ()      # (rho0, g) of the hydrostatic initial state

    @property
    def n(self) -> int:
        return self.p + 1

    @property
    def nv(self) -> int:
        if self.lattice:
            return len(_lattice(self.lattice)[1])
        return self.m * 2 * self.dim

    @property
    def h(self) -> float:
        return (self.hi[0] - self.lo[0]) / self.N

    @property
    def grid_shape(self) -> tuple:
        """Node-grid shape, slowest axis first: (Z, Y, X) or (Y, X)."""
        return tuple([self.N * self.n] * self.dim)

    @property
    def nnodes(self) -> int:
        return (self.N * self.n) ** self.dim

    @property
    def updates_per_step(self) -> int:
        return self.nnodes * self.nv

    def velocities(self):
        if self.lattice:
            v, _ = lattice(self.lattice, self.lam)
            return v, [0] * len(v)
        return velocity_set(self.dim, self.m, self.lam)

    def flux_params(self):
        """Model parameters as both sides take them: LBM -> (c, w_0..w_{nv-1})."""
        if self.lattice:
            return tuple(self.fparams) + tuple(lattice(self.lattice, self.lam)[1])
        return tuple(self.fparams)

    def resized(self, N: int, steps: int | None = None, name: str | None = None) -> "Config":
        """Same recipe and CFL number nu = lambda dt / h on an N-cell grid."""
        nu = self.lam * self.dt / self.h
        h = (self.hi[0] - self.lo[0]) / N
        return replace(self, N=N, dt=nu * h / self.lam, steps=self.steps if steps is None else steps,
                       name=name or f"{self.name}@N{N}")

    def stabilised(self, lam: float = 3.5) -> "Config":
        """Twin with lambda = 3.5 and the same nu (DESIGN.md parity protocol)."""
        nu = self.lam * self.dt / self.h
        return replace(self, lam=lam, dt=nu * self.h / lam, name=self.name + "s")


CONFIGS = {
    1: Config("cfg1_adv2d", 2, 8, 2, 1, 2.0, FLUX_ADVECTION, (1.0, 0.5), 1.0 / 32.0, 10,
              0x5EED0001, "gauss_bump", wb_zero=True),
    2: Config("cfg2_euler2d", 2, 256, 2, 4, 3.0, FLUX_EULER, (1.4,), 1.0 / 384.0, 100,
              0x5EED0002, "euler2d_modes"),
    3: Config("cfg3_iso3d", 3, 64, 2, 4, 2.0, FLUX_ISOTHERMAL, (1.0,), 1.0 / 64.0, 50,
              0x5EED0003, "iso3d_pulse_vortical"),
    4: Config("cfg4_iso3d_p3", 3, 128, 3, 4, 2.0, FLUX_ISOTHERMAL, (1.0,), 1.0 / 64.0, 20,
              0x5EED0004, "iso3d_pulse_vortical"),
    5: Config("cfg5_iso3d_scale", 3, 256, 2, 4, 2.0, FLUX_ISOTHERMAL, (1.0,), 1.0 / 256.0, 10,
              0x5EED0005, "iso3d_multimode"),
}


def lbm_config(lattice_name: str, N: int, p: int = 2, lam: float = 1.0, nu: float = 0.5, steps: int = 4,
               seed: int = 0x5EED0009) -> Config:
    """An isothermal LBM workload (NEXT-2): c = lambda/sqrt(3), density pulse plus a
    small seeded vortical velocity; inflow data f^eq(w0(x_b))."""
    dim = 2 if lattice_name.startswith("D2") else 3
    h = 1.0 / N
    return Config(f"lbm_{lattice_name}_N{N}", dim, N, p, dim + 1, lam, FLUX_LBM, (lam / math.sqrt(3.0),),
                  nu * h / lam, steps, seed, "lbm_pulse", lattice=lattice_name)


def gravity_config(N: int, p: int = 2, lam: float = 2.0, g: float = 1.0, rho0: float = 1.0, dt: float = 0.024,
                   t_max: float = 0.12, seed: int = 0x5EED000A) -> Config:
    """The paper's Euler-with-gravity test: isothermal Euler in 2-D with the D2Q9
    model (c = lambda/sqrt(3)), gravity G = -g e_y, starting from the fluid at rest
    rho = rho0 exp(-g y / c^2), u = 0; steps = t_max / dt."""
    steps = max(1, int(round(t_max / dt)))
    return Config(f"gravity_D2Q9_N{N}", 2, N, p, 3, lam, FLUX_LBM, (lam / math.sqrt(3.0),), dt, steps, seed,
                  "hydrostatic", lattice="D2Q9", gravity=(0.0, -g), rho0_g=(rho0, g))


def node_axis(cfg: Config, axis: int, dtype=torch.float64, device="cpu") -> torch.Tensor:
    """1-D coordinates of the node grid along `axis`: X = c*n + a."""
    xh = torch.tensor(gl_sample_points(cfg.p), dtype=dtype)
    hh = (cfg.hi[axis] - cfg.lo[axis]) / cfg.N
    c = torch.arange(cfg.N, dtype=dtype).unsqueeze(1)
    x = cfg.lo[axis] + (c + (xh.unsqueeze(0) + 1.0) * 0.5) * hh
    return x.reshape(-1).to(device)


def _fields(cfg: Config, X, Y, Z):
    """w0 at broadcastable coordinate tensors; returns a list of m tensors."""
    two_pi = 2.0 * math.pi
    if cfg.recipe == "gauss_bump":
        r2 = (X - 0.5) ** 2 + (Y - 0.5) ** 2
        return [torch.exp(-100.0 * r2)]
    if cfg.recipe == "euler2d_modes":
        ph = phases(cfg.seed, 4)
        gamma = cfg.fparams[0]
        rho = 1.0 + 0.2 * torch.sin(two_pi * X + ph[0]) * torch.sin(two_pi * Y + ph[1])
        u = 0.3 * torch.sin(two_pi * Y + ph[2])
        v = 0.3 * torch.sin(two_pi * X + ph[3])
        pr = 1.0
        E = pr / (gamma - 1.0) + rho * (u * u + v * v) * 0.5
        return [rho, rho * u, rho * v, E]
    if cfg.recipe == "iso3d_pulse_vortical":
        ph = phases(cfg.seed, 3)
        r2 = (X - 0.5) ** 2 + (Y - 0.5) ** 2 + (Z - 0.5) ** 2
        rho = 1.0 + 0.1 * torch.exp(-100.0 * r2)
        u = 0.05 * torch.sin(two_pi * Y + ph[0])
        v = 0.05 * torch.sin(two_pi * Z + ph[1])
        w = 0.05 * torch.sin(two_pi * X + ph[2])
        return [rho, rho * u, rho * v, rho * w]
    if cfg.recipe == "iso3d_multimode":
        ph = phases(cfg.seed, 4 + 12)
        phi = ph[:4]
        psi = [[ph[4 + 3 * k + d] for d in range(3)] for k in range(4)]
        rho = 1.0
        for k in range(4):
            rho = rho + 0.02 * torch.sin(two_pi * (k + 1) * (X + Y + Z) + phi[k])
        coords = (X, Y, Z)
        vel = []
        for d in range(3):
            ud = 0.0
            for k in range(4):
                ud = ud + 0.02 * torch.sin(two_pi * (k + 1) * coords[(d + 1) % 3] + psi[k][d])
            vel.append(ud)
        return [rho, rho * vel[0], rho * vel[1], rho * vel[2]]
    if cfg.recipe == "hydrostatic":
        # fluid at rest in the gravity field: rho = rho0 exp(-g y / c^2), u = 0
        rho0, g = cfg.rho0_g
        c = cfg.fparams[0]
        rho = rho0 * torch.exp(-g * Y / (c * c)) + 0.0 * X
        return [rho, 0.0 * rho, 0.0 * rho]
    if cfg.recipe == "lbm_pulse":
        ph = phases(cfg.seed, 3)
        r2 = (X - 0.5) ** 2 + (Y - 0.5) ** 2 + ((Z - 0.5) ** 2 if cfg.dim == 3 else 0.0)
        rho = 1.0 + 0.05 * torch.exp(-50.0 * r2)
        u = 0.02 * cfg.lam * torch.sin(two_pi * Y + ph[0])
        v = 0.02 * cfg.lam * torch.sin(two_pi * X + ph[1])
        out = [rho, rho * u, rho * v]
        if cfg.dim == 3:
            out.append(rho * 0.02 * cfg.lam * torch.sin(two_pi * X + ph[2]) * torch.cos(two_pi * Y))
        return out
    raise ValueError(cfg.recipe)


def w0_grid(cfg: Config, device="cpu", zslab: tuple | None = None) -> torch.Tensor:
    """w0 on the node grid, shape [m, Z, Y, X] (3-D) or [m, Y, X] (2-D), fp64.
    zslab=(z0, z1) restricts a 3-D grid to node planes z0 <= Z < z1."""
    xs = node_axis(cfg, 0, device=device)
    ys = node_axis(cfg, 1, device=device)
    if cfg.dim == 2:
        X = xs.view(1, -1)
        Y = ys.view(-1, 1)
        zero = torch.zeros((), dtype=torch.float64, device=device)
        F = _fields(cfg, X, Y, zero)
        shape = (ys.numel(), xs.numel())
    else:
        zs = node_axis(cfg, 2, device=device)
        if zslab is not None:
            zs = zs[zslab[0]:zslab[1]]
        X = xs.view(1, 1, -1)
        Y = ys.view(1, -1, 1)
        Z = zs.view(-1, 1, 1)
        F = _fields(cfg, X, Y, Z)
        shape = (zs.numel(), ys.numel(), xs.numel())
    out = torch.empty((cfg.m,) + shape, dtype=torch.float64, device=device)
    for c in range(cfg.m):
        out[c].copy_(torch.as_tensor(F[c], dtype=torch.float64, device=device).expand(shape))
    return out


def wb_grid(cfg: Config, w0: torch.Tensor) -> torch.Tensor:
    """Macroscopic state whose equilibrium gives the inflow data (reading C12):
    w_b = w0(x_b) (configs 2-5) or 0 (config 1)."""
    return torch.zeros_like(w0) if cfg.wb_zero else w0


def random_state(cfg: Config, seed: int, scale: float = 1.0) -> torch.Tensor:
    """Non-equilibrium kinetic test data f[nv, grid] ~ 1 + scale*U(-1/2, 1/2)/nv
    (positive density), drawn from torch's seeded CPU generator."""
    g = torch.Generator().manual_seed(seed)
    f = torch.rand((cfg.nv,) + cfg.grid_shape, generator=g, dtype=torch.float64)
    return (1.0 + scale * (f - 0.5)) / cfg.nv
