"""Python driver of the CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import this module.  It wraps oracle/pdg_oracle.c (plain C,
fp64, no FMA contraction) with ctypes and composes the palindromic step

    M2(dt) = T2(dt/2) C2(dt) T2(dt/2)

It shares no code with the CUDA product (paper_1702_00169_b200/).  Storage is
the paper's cell-blocked numbering F_{k N_d + i} = f_{L_k, i},
per velocity; conversions to/from the canonical node grid f[i][Z][Y][X]
(X = c_x (p+1) + a_x fastest) are plain index permutations.

Parity status of each function is listed in DESIGN.md ("Oracle pins").
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

FLUX_LBM = 3  # lattice-Boltzmann isothermal model

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "pdg_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with plain IEEE binary64 semantics (no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
                               "-shared", "-fPIC", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class Mesh(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int32), ("p", ctypes.c_int32), ("ncell", ctypes.c_int64 * 3),
                ("lo", ctypes.c_double * 3), ("hi", ctypes.c_double * 3)]


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.POINTER
        d, i32, i64 = ctypes.c_double, ctypes.c_int32, ctypes.c_int64
        pd, pi64, pi32 = P(d), P(i64), P(i32)
        pm = P(Mesh)
        sig = {
            "or_gl_1d": [ctypes.c_int, pd, pd],
            "or_lagrange_deriv_matrix": [ctypes.c_int, pd],
            "or_cell_operator": [pm, pd, pd, pd],
            "or_topo_order": [pm, pd, i64, pi64, pi64, pi32],
            "or_upstream_closure": [pm, pd, i64, pi64, P(ctypes.c_uint8)],
            "or_t2": [pm, pd, d, i64, pi64, pd, pd],
            "or_t2_all": [pm, ctypes.c_int, pd, d, pd, pd],
            "or_apply_L": [pm, pd, pd, pd, pd],
            "or_flux": [ctypes.c_int, ctypes.c_int, pd, pd, pd],
            "or_equilibrium": [ctypes.c_int, ctypes.c_int, pd, pi32, ctypes.c_int, d, ctypes.c_int, pd, pd, pd],
            "or_moments": [ctypes.c_int, pi32, ctypes.c_int, i64, pd, pd],
            "or_moments_lbm": [ctypes.c_int, ctypes.c_int, pd, i64, pd, pd],
            "or_collide": [ctypes.c_int, ctypes.c_int, pd, pi32, ctypes.c_int, d, ctypes.c_int, pd, d, d, i64, pd],
            "or_equilibrium_field": [ctypes.c_int, ctypes.c_int, pd, pi32, ctypes.c_int, d, ctypes.c_int, pd,
                                     i64, pd, pd],
            "or_source": [ctypes.c_int, ctypes.c_int, pd, pd, pd, d, i64, pd],
        }
        for name, args in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = ctypes.c_int
        _lib = L
    return _lib


def _pd(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _pi64(a: np.ndarray):
    assert a.dtype == np.int64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))


def _pi32(a: np.ndarray):
    assert a.dtype == np.int32 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))


def _check(rc: int, what: str):
    if rc != 0:
        raise RuntimeError(f"oracle {what} failed with code {rc}")


# ----------------------------------------------------------------------------
# Problem statement
# ----------------------------------------------------------------------------
class Problem:
    """Everything the paper's problem statement fixes."""

    def __init__(self, dim, N, p, vel, comp, m, lam, flux, fparams, dt, tau=0.0, lo=None, hi=None, gravity=None):
        self.dim, self.p, self.m = int(dim), int(p), int(m)
        self.N = [int(N)] * dim if np.isscalar(N) else [int(x) for x in N]
        self.vel = np.ascontiguousarray(np.asarray(vel, dtype=np.float64).reshape(-1, 3))
        self.comp = np.ascontiguousarray(np.asarray(comp, dtype=np.int32))
        self.nv = self.vel.shape[0]
        self.lam, self.flux = float(lam), int(flux)
        self.fparams = np.ascontiguousarray(np.asarray(fparams, dtype=np.float64).reshape(-1))
        if self.fparams.size < 3:
            self.fparams = np.concatenate([self.fparams, np.zeros(3 - self.fparams.size)])
        self.dt, self.tau = float(dt), float(tau)
        self.lo = list(lo) if lo is not None else [0.0] * 3
        self.hi = list(hi) if hi is not None else [1.0] * 3
        self.n = self.p + 1
        self.Nd = self.n ** self.dim
        # gravity vector G of the Euler-with-gravity source, or None
        self.gravity = None if gravity is None else np.ascontiguousarray(
            (list(gravity) + [0.0, 0.0, 0.0])[:3], dtype=np.float64)
        self.ncell = int(np.prod(self.N))
        self.nnodes = self.ncell * self.Nd

    @classmethod
    def from_config(cls, cfg, tau=0.0):
        vel, comp = cfg.velocities()
        return cls(cfg.dim, cfg.N, cfg.p, vel, comp, cfg.m, cfg.lam, cfg.flux, cfg.flux_params(), cfg.dt, tau,
                   lo=cfg.lo, hi=cfg.hi, gravity=cfg.gravity or None)

    def mesh(self) -> Mesh:
        m = Mesh()
        m.dim, m.p = self.dim, self.p
        for d in range(3):
            m.ncell[d] = self.N[d] if d < self.dim else 1
            m.lo[d], m.hi[d] = self.lo[d], self.hi[d]
        return m

    # --- layouts ------------------------------------------------------------
    def grid_shape(self):
        return tuple(self.N[d] * self.n for d in reversed(range(self.dim)))

    def grid_to_cells(self, g: np.ndarray) -> np.ndarray:
        """[..., (Z), Y, X] node grid -> [..., ncell, Nd] cell-blocked."""
        lead = g.shape[: g.ndim - self.dim]
        n, D = self.n, self.dim
        shp = []
        for d in reversed(range(D)):
            shp += [self.N[d], n]
        a = g.reshape(lead + tuple(shp))
        L = len(lead)
        cell_axes = [L + 2 * k for k in range(D)]      # slow..fast cell coords
        node_axes = [L + 2 * k + 1 for k in range(D)]  # slow..fast local coords
        a = a.transpose(tuple(range(L)) + tuple(cell_axes) + tuple(node_axes))
        out = np.ascontiguousarray(a.reshape(lead + (self.ncell, self.Nd)))
        # with one cell per axis the reordering is the identity and numpy returns a view: the
        # drivers update their cell arrays in place, so the caller's grid must never be aliased
        return out.copy() if np.may_share_memory(out, g) else out

    def cells_to_grid(self, c: np.ndarray) -> np.ndarray:
        lead = c.shape[:-2]
        n, D = self.n, self.dim
        shp = tuple(self.N[d] for d in reversed(range(D))) + (n,) * D
        a = c.reshape(lead + shp)
        L = len(lead)
        perm = []
        for k in range(D):
            perm += [L + k, L + D + k]
        a = a.transpose(tuple(range(L)) + tuple(perm))
        return np.ascontiguousarray(a.reshape(lead + self.grid_shape()))


# ----------------------------------------------------------------------------
# Reference-element and operator access (pins)
# ----------------------------------------------------------------------------
def gl_1d(p: int):
    x = np.zeros(p + 1)
    w = np.zeros(p + 1)
    _check(lib().or_gl_1d(p, _pd(x), _pd(w)), "gl_1d")
    return x, w


def deriv_matrix(p: int) -> np.ndarray:
    D = np.zeros((p + 1) * (p + 1))
    _check(lib().or_lagrange_deriv_matrix(p, _pd(D)), "deriv")
    return D.reshape(p + 1, p + 1)


def cell_operator(pb: Problem, v):
    v = np.ascontiguousarray(np.asarray(v, dtype=np.float64).reshape(3))
    GLL = np.zeros(pb.Nd * pb.Nd)
    GLR = np.zeros(6 * pb.Nd)
    m = pb.mesh()
    _check(lib().or_cell_operator(ctypes.byref(m), _pd(v), _pd(GLL), _pd(GLR)), "cell_operator")
    return GLL.reshape(pb.Nd, pb.Nd), GLR.reshape(6, pb.Nd)


def topo_order(pb: Problem, v, cells=None):
    v = np.ascontiguousarray(np.asarray(v, dtype=np.float64).reshape(3))
    m = pb.mesh()
    if cells is None:
        nsub, cp = 0, None
        count = pb.ncell
    else:
        cells = np.ascontiguousarray(np.asarray(cells, dtype=np.int64))
        nsub, cp, count = cells.size, _pi64(cells), cells.size
    order = np.zeros(count, dtype=np.int64)
    level = np.zeros(count, dtype=np.int32)
    _check(lib().or_topo_order(ctypes.byref(m), _pd(v), nsub, cp, _pi64(order), _pi32(level)), "topo_order")
    return order, level


def upstream_closure(pb: Problem, v, seed_cells, mask=None) -> np.ndarray:
    v = np.ascontiguousarray(np.asarray(v, dtype=np.float64).reshape(3))
    seed = np.ascontiguousarray(np.asarray(seed_cells, dtype=np.int64))
    if mask is None:
        mask = np.zeros(pb.ncell, dtype=np.uint8)
    m = pb.mesh()
    _check(lib().or_upstream_closure(ctypes.byref(m), _pd(v), seed.size, _pi64(seed),
                                     mask.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))), "closure")
    return mask


def apply_L(pb: Problem, v, f_cells: np.ndarray, fb_cells: np.ndarray) -> np.ndarray:
    """(L_h F) for one velocity, cell-blocked [ncell, Nd]."""
    v = np.ascontiguousarray(np.asarray(v, dtype=np.float64).reshape(3))
    f = np.ascontiguousarray(f_cells, dtype=np.float64)
    fb = np.ascontiguousarray(fb_cells, dtype=np.float64)
    out = np.zeros_like(f)
    m = pb.mesh()
    _check(lib().or_apply_L(ctypes.byref(m), _pd(v), _pd(f), _pd(fb), _pd(out)), "apply_L")
    return out


def dense_L(pb: Problem, v):
    """Dense transport matrix L (ncell*Nd square) and ghost vector b with
    (L_h F) = L F + b(fb) linear in fb: returns (L, Bmat) so L_h F = L F + Bmat fb."""
    n = pb.ncell * pb.Nd
    zeros = np.zeros((pb.ncell, pb.Nd))
    L = np.zeros((n, n))
    B = np.zeros((n, n))
    for j in range(n):
        e = np.zeros(n)
        e[j] = 1.0
        L[:, j] = apply_L(pb, v, e.reshape(pb.ncell, pb.Nd), zeros).reshape(-1)
        B[:, j] = apply_L(pb, v, zeros, e.reshape(pb.ncell, pb.Nd)).reshape(-1)
    return L, B


# ----------------------------------------------------------------------------
# Transport, collision, moments
# ----------------------------------------------------------------------------
def t2_velocity(pb: Problem, v, dtp: float, f_cells: np.ndarray, fb_cells: np.ndarray, cells=None):
    """T2(dt') for one velocity, in place on cell-blocked f ([ncell or nsub, Nd])."""
    v = np.ascontiguousarray(np.asarray(v, dtype=np.float64).reshape(3))
    assert f_cells.flags["C_CONTIGUOUS"] and fb_cells.flags["C_CONTIGUOUS"]
    m = pb.mesh()
    if cells is None:
        rc = lib().or_t2(ctypes.byref(m), _pd(v), dtp, 0, None, _pd(f_cells), _pd(fb_cells))
    else:
        cells = np.ascontiguousarray(np.asarray(cells, dtype=np.int64))
        rc = lib().or_t2(ctypes.byref(m), _pd(v), dtp, cells.size, _pi64(cells), _pd(f_cells), _pd(fb_cells))
    _check(rc, "t2")


def t2_all(pb: Problem, dtp: float, f_cells: np.ndarray, fb_cells: np.ndarray):
    """T2(dt') for every velocity, in place on [nv, ncell, Nd]."""
    m = pb.mesh()
    _check(lib().or_t2_all(ctypes.byref(m), pb.nv, _pd(pb.vel), dtp, _pd(f_cells), _pd(fb_cells)), "t2_all")


def flux(pb: Problem, w):
    w = np.ascontiguousarray(np.asarray(w, dtype=np.float64))
    q = np.zeros(3 * 8)
    _check(lib().or_flux(pb.dim, pb.flux, _pd(pb.fparams), _pd(w), _pd(q)), "flux")
    return q[: pb.dim * pb.m].reshape(pb.dim, pb.m)


def equilibrium(pb: Problem, w):
    w = np.ascontiguousarray(np.asarray(w, dtype=np.float64))
    feq = np.zeros(pb.nv)
    _check(lib().or_equilibrium(pb.dim, pb.nv, _pd(pb.vel), _pi32(pb.comp), pb.m, pb.lam, pb.flux,
                                _pd(pb.fparams), _pd(w), _pd(feq)), "equilibrium")
    return feq


def equilibrium_field(pb: Problem, w_nodes: np.ndarray) -> np.ndarray:
    """w [m, nodes...] -> f^eq [nv, nodes...] (any node ordering)."""
    w = np.ascontiguousarray(w_nodes, dtype=np.float64)
    nn = w[0].size
    out = np.zeros((pb.nv,) + w.shape[1:])
    _check(lib().or_equilibrium_field(pb.dim, pb.nv, _pd(pb.vel), _pi32(pb.comp), pb.m, pb.lam, pb.flux,
                                      _pd(pb.fparams), nn, _pd(w), _pd(out)), "equilibrium_field")
    return out


def moments(pb: Problem, f_nodes: np.ndarray) -> np.ndarray:
    """w = P f: block sums for the vectorial models, P = [1; v^T] for LBM."""
    f = np.ascontiguousarray(f_nodes, dtype=np.float64)
    nn = f[0].size
    w = np.zeros((pb.m,) + f.shape[1:])
    if pb.flux == FLUX_LBM:
        _check(lib().or_moments_lbm(pb.dim, pb.nv, _pd(pb.vel), nn, _pd(f), _pd(w)), "moments")
    else:
        _check(lib().or_moments(pb.nv, _pi32(pb.comp), pb.m, nn, _pd(f), _pd(w)), "moments")
    return w


def collide(pb: Problem, f_nodes: np.ndarray, dt: float, tau: float | None = None):
    """C2(dt) in place on f [nv, nodes...] (eq collision_cn; tau=0: P:474-477)."""
    assert f_nodes.flags["C_CONTIGUOUS"]
    tau = pb.tau if tau is None else tau
    nn = f_nodes[0].size
    _check(lib().or_collide(pb.dim, pb.nv, _pd(pb.vel), _pi32(pb.comp), pb.m, pb.lam, pb.flux,
                            _pd(pb.fparams), tau, dt, nn, _pd(f_nodes)), "collide")


def source(pb: Problem, f_nodes: np.ndarray, h: float) -> int:
    """S2(h) in place on f [nv, nodes...] (gravity source of P:1101-1160, reading C24).
    Returns the number of Picard iterations the worst node needed."""
    assert f_nodes.flags["C_CONTIGUOUS"] and pb.flux == FLUX_LBM and pb.gravity is not None
    nn = f_nodes[0].size
    it = lib().or_source(pb.dim, pb.nv, _pd(pb.vel), _pd(pb.fparams), _pd(pb.gravity), h, nn, _pd(f_nodes))
    if it < 1:
        raise RuntimeError("oracle source failed")
    return it


# ----------------------------------------------------------------------------
# Palindromic step M2 on the whole mesh
# ----------------------------------------------------------------------------
def m2_run(pb: Problem, f_grid: np.ndarray, fb_grid: np.ndarray, nsteps: int, callback=None) -> np.ndarray:
    """nsteps of M2(dt) = T2(dt/2) C2(dt) T2(dt/2), never collapsing the
    trailing and leading half-steps (P:1173-1177 is a different map).
    f_grid, fb_grid: canonical [nv, (Z), Y, X]; returns the new f_grid."""
    fc = pb.grid_to_cells(np.asarray(f_grid, dtype=np.float64))
    fbc = pb.grid_to_cells(np.asarray(fb_grid, dtype=np.float64))
    for s in range(nsteps):
        t2_all(pb, 0.5 * pb.dt, fc, fbc)
        collide(pb, fc, pb.dt)
        t2_all(pb, 0.5 * pb.dt, fc, fbc)
        if callback is not None:
            callback(s + 1, fc)
    return pb.cells_to_grid(fc)


def m2kin_substep(pb: Problem, fc, fbc, h: float):
    """M2kin(h) = T2(h/4) C2(h/2) T2(h/2) C2(h/2) T2(h/4), in place, cell-blocked."""
    t2_all(pb, h / 4, fc, fbc)
    collide(pb, fc, h / 2)
    t2_all(pb, h / 2, fc, fbc)
    collide(pb, fc, h / 2)
    t2_all(pb, h / 4, fc, fbc)


def scheme_run(pb: Problem, f_grid: np.ndarray, fb_grid: np.ndarray, nsteps: int, scheme: str) -> np.ndarray:
    """nsteps of 'm2', 'm2kin', 'm4': the symmetric triple-jump
    composition M2kin(g1 dt) M2kin(g2 dt) M2kin(g1 dt), g1 = 1/(2 - 2^(1/3)), g2 = 1 - 2 g1
    (palindromic composition to higher even order), or 'm2s': the Strang scheme
    with source M2s(dt) = T2(dt/2) S2(dt/2) C2(dt) S2(dt/2) T2(dt/2)."""
    fc = pb.grid_to_cells(np.asarray(f_grid, dtype=np.float64))
    fbc = pb.grid_to_cells(np.asarray(fb_grid, dtype=np.float64))
    g1 = 1.0 / (2.0 - 2.0 ** (1.0 / 3.0))
    g2 = 1.0 - 2.0 * g1
    for _ in range(nsteps):
        if scheme == "m2":
            t2_all(pb, 0.5 * pb.dt, fc, fbc)
            collide(pb, fc, pb.dt)
            t2_all(pb, 0.5 * pb.dt, fc, fbc)
        elif scheme == "m2kin":
            m2kin_substep(pb, fc, fbc, pb.dt)
        elif scheme == "m2s":
            t2_all(pb, 0.5 * pb.dt, fc, fbc)
            source(pb, fc, 0.5 * pb.dt)
            collide(pb, fc, pb.dt)
            source(pb, fc, 0.5 * pb.dt)
            t2_all(pb, 0.5 * pb.dt, fc, fbc)
        elif scheme == "m4":
            m2kin_substep(pb, fc, fbc, g1 * pb.dt)
            m2kin_substep(pb, fc, fbc, g2 * pb.dt)
            m2kin_substep(pb, fc, fbc, g1 * pb.dt)
        else:
            raise ValueError(scheme)
    return pb.cells_to_grid(fc)


def initial_data(pb: Problem, w0_grid: np.ndarray, wb_grid: np.ndarray):
    """f0 = f^eq(w0) at every node, f^b = f^eq(w_b) (readings C12, C13)."""
    return equilibrium_field(pb, w0_grid), equilibrium_field(pb, wb_grid)


# ----------------------------------------------------------------------------
# M2 on sampled cells of a large mesh (dependency-cone evaluation)
# ----------------------------------------------------------------------------
def m2_cone_plan(pb: Problem, sample_cells):
    """Cells each pass needs so that one M2 step can be evaluated exactly at
    `sample_cells`: second T2 of velocity i on closure_i(S); collision on
    R = U_i closure_i(S); first T2 of velocity i on closure_i(R).  Closures
    follow the dependency graph, not the velocity directions."""
    S = np.asarray(sample_cells, dtype=np.int64)
    second = []
    Rmask = np.zeros(pb.ncell, dtype=np.uint8)
    for i in range(pb.nv):
        mk = upstream_closure(pb, pb.vel[i], S)
        second.append(np.flatnonzero(mk).astype(np.int64))
        Rmask |= mk
    R = np.flatnonzero(Rmask).astype(np.int64)
    first = [np.flatnonzero(upstream_closure(pb, pb.vel[i], R)).astype(np.int64) for i in range(pb.nv)]
    return {"S": S, "R": R, "second": second, "first": first}


def m2_cone_step(pb: Problem, plan, f0_of_cells, fb_of_cells, threads: int | None = None):
    """Evaluate one M2 step at plan['S'].
    f0_of_cells(i, cells) -> [len(cells), Nd] initial f_i on those cells;
    fb_of_cells(i, cells) -> [len(cells), Nd] boundary data of velocity i.
    Velocities are independent in transport, so they run on a thread pool
    (the C solver releases the GIL).  Returns f at S: [nv, len(S), Nd]."""
    from concurrent.futures import ThreadPoolExecutor
    R = plan["R"]
    fR = np.zeros((pb.nv, R.size, pb.Nd))
    threads = threads or min(pb.nv, os.cpu_count() or 1)

    def first(i):
        cells = plan["first"][i]
        f = np.ascontiguousarray(f0_of_cells(i, cells), dtype=np.float64)
        fb = np.ascontiguousarray(fb_of_cells(i, cells), dtype=np.float64)
        t2_velocity(pb, pb.vel[i], 0.5 * pb.dt, f, fb, cells)
        fR[i] = f[np.searchsorted(cells, R)]

    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(first, range(pb.nv)))
    collide(pb, fR, pb.dt)
    out = np.zeros((pb.nv, plan["S"].size, pb.Nd))

    def second(i):
        cells = plan["second"][i]
        f = np.ascontiguousarray(fR[i][np.searchsorted(R, cells)])
        fb = np.ascontiguousarray(fb_of_cells(i, cells), dtype=np.float64)
        t2_velocity(pb, pb.vel[i], 0.5 * pb.dt, f, fb, cells)
        out[i] = f[np.searchsorted(cells, plan["S"])]

    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(second, range(pb.nv)))
    return out
