"""Pins of the CPU oracle against what the paper and the mathematics fix.

Each test names the passage it checks.  None of them compares the oracle with
itself by re-typing its formulas: they use closed forms (golden/), invariants
(constant preservation, polynomial exactness, dissipation, conservation,
time symmetry), brute-force dense solves and convergence orders.
"""
import math
from fractions import Fraction

import numpy as np
import pytest

from oracle import oracle as O
from pdg_inputs import CONFIGS, FLUX_ADVECTION, FLUX_EULER, FLUX_ISOTHERMAL, velocity_set, w0_grid, wb_grid


def _val(s):
    if isinstance(s, (int, float)):
        return float(s)
    s = s.replace("sqrt5", str(math.sqrt(5.0)))
    if "/" in s:
        a, b = s.split("/")
        return float(eval(a)) / float(eval(b))
    return float(eval(s))


def scalar_problem(dim, N, p, v, lo=None, hi=None):
    return O.Problem(dim, N, p, [v], [0], 1, 1.0, FLUX_ADVECTION, [1.0, 0.0, 0.0], dt=0.1, lo=lo, hi=hi)


def node_positions(pb):
    """Physical node coordinates, cell-blocked [ncell, Nd, dim], from the closed-form GL points."""
    x1 = {1: [-1.0, 1.0], 2: [-1.0, 0.0, 1.0], 3: [-1.0, -1 / math.sqrt(5), 1 / math.sqrt(5), 1.0]}[pb.p]
    n = pb.n
    pos = np.zeros((pb.ncell, pb.Nd, pb.dim))
    for c in range(pb.ncell):
        cc, r = [], c
        for d in range(pb.dim):
            cc.append(r % pb.N[d])
            r //= pb.N[d]
        for i in range(pb.Nd):
            a, r = [], i
            for d in range(pb.dim):
                a.append(r % n)
                r //= n
            for d in range(pb.dim):
                h = (pb.hi[d] - pb.lo[d]) / pb.N[d]
                pos[c, i, d] = pb.lo[d] + (cc[d] + (x1[a[d]] + 1) / 2) * h
    return pos


# --------------------------------------------------------------------------
# Reference element
# --------------------------------------------------------------------------
@pytest.mark.parametrize("p", [1, 2, 3])
def test_gl_closed_forms(p, golden):
    g = golden("gl_tables.json")
    x, w = O.gl_1d(p)
    np.testing.assert_allclose(x, [_val(s) for s in g["points"][str(p)]], rtol=0, atol=1e-15)
    np.testing.assert_allclose(w, [_val(s) for s in g["weights"][str(p)]], rtol=0, atol=1e-15)
    assert abs(w.sum() - 2.0) < 1e-15
    for k in range(0, 2 * p):  # Lobatto exactness: degree <= 2p-1
        exact = 0.0 if k % 2 else 2.0 / (k + 1)
        assert abs(np.dot(w, x ** k) - exact) < 1e-14


def test_deriv_matrix_golden(golden):
    g = golden("gl_tables.json")
    np.testing.assert_allclose(O.deriv_matrix(1), g["D_p1"], atol=1e-15)
    np.testing.assert_allclose(O.deriv_matrix(2), g["D_p2"], atol=1e-15)


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_deriv_matrix_exact_on_polynomials(p):
    x, _ = O.gl_1d(p)
    D = O.deriv_matrix(p)
    for k in range(0, p + 1):
        expect = k * x ** (k - 1) if k > 0 else np.zeros_like(x)
        np.testing.assert_allclose(D @ x ** k, expect, atol=1e-13)


# --------------------------------------------------------------------------
# The 1-D cell block against exact rationals
# --------------------------------------------------------------------------
def one_cell_block(p, kappa):
    """M and g of one T2 solve on a single 1-D cell of width 1 with velocity 2:
    f_new = M f_old + g s, s = sum of ghost old/new values (= 2 f^b)."""
    pb = O.Problem(1, 1, p, [[2.0, 0, 0]], [0], 1, 2.0, FLUX_ADVECTION, [1.0], dt=1.0)
    dtp = kappa / 2.0  # kappa = v dt'/h
    n = p + 1
    M = np.zeros((n, n))
    for j in range(n):
        f = np.zeros((1, n))
        f[0, j] = 1.0
        O.t2_velocity(pb, pb.vel[0], dtp, f, np.zeros((1, n)))
        M[:, j] = f[0]
    f = np.zeros((1, n))
    O.t2_velocity(pb, pb.vel[0], dtp, f, np.full((1, n), 0.5))
    return M, f[0]


@pytest.mark.parametrize("kappa", ["0.125", "0.25", "1.0", "2.0"])
def test_cell_block_p2_appendix_A(kappa, golden):
    g = golden("cell_block_p2.json")["p2"][kappa]
    M, gv = one_cell_block(2, float(kappa))
    Ainv = (M + np.eye(3)) / 2.0   # M = Ainv (2I - A) = 2 Ainv - I
    np.testing.assert_allclose(Ainv, np.array(g["Ainv_num"]) / g["Ainv_den"], atol=2e-15)
    assert abs(gv[2] - g["beta"][0] / g["beta"][1]) < 1e-15
    if "M_num" in g:
        np.testing.assert_allclose(M, np.array(g["M_num"]) / g["M_den"], atol=2e-15)
    k = float(kappa)
    det_closed = (6 * k ** 3 + 9 * k ** 2 + 6 * k + 2) / 2
    assert abs(np.linalg.det(2 * np.linalg.inv(M + np.eye(3))) - det_closed) < 1e-12 * det_closed


def test_cell_block_p3_beta(golden):
    g = golden("cell_block_p2.json")["p3"]["2.0"]
    _, gv = one_cell_block(3, 2.0)
    assert abs(gv[3] - g["beta"][0] / g["beta"][1]) < 1e-15
    M, _ = one_cell_block(3, 2.0)
    k = 2.0
    det_closed = (45 * k ** 4 + 60 * k ** 3 + 36 * k ** 2 + 12 * k + 2) / 2
    assert abs(np.linalg.det(2 * np.linalg.inv(M + np.eye(4))) - det_closed) < 1e-11 * det_closed


def test_cell_block_exact_rational_derivation():
    """Independent exact derivation for p=2 from the GL weak form with Fractions:
    G = W^{-1}(D^T W - e_out e_out^T), then (I - kG)^{-1} and beta at k = 1."""
    xs = [Fraction(-1), Fraction(0), Fraction(1)]
    ws = [Fraction(1, 3), Fraction(4, 3), Fraction(1, 3)]

    def dl(b, t):
        s = Fraction(0)
        for k in range(3):
            if k == b:
                continue
            term = 1 / (xs[b] - xs[k])
            for j in range(3):
                if j not in (b, k):
                    term *= (t - xs[j]) / (xs[b] - xs[j])
            s += term
        return s
    D = [[dl(b, xs[a]) for b in range(3)] for a in range(3)]
    G = [[(D[j][i] * ws[j] - (1 if (i == 2 and j == 2) else 0)) / ws[i] for j in range(3)] for i in range(3)]
    k = Fraction(1)
    A = [[(1 if i == j else 0) - k * G[i][j] for j in range(3)] for i in range(3)]
    # exact inverse by Gauss-Jordan
    aug = [A[i] + [Fraction(1 if i == j else 0) for j in range(3)] for i in range(3)]
    for c in range(3):
        piv = next(r for r in range(c, 3) if aug[r][c] != 0)
        aug[c], aug[piv] = aug[piv], aug[c]
        pv = aug[c][c]
        aug[c] = [v / pv for v in aug[c]]
        for r in range(3):
            if r != c and aug[r][c] != 0:
                fac = aug[r][c]
                aug[r] = [a - fac * b for a, b in zip(aug[r], aug[c])]
    Ainv = [row[3:] for row in aug]
    M, gv = one_cell_block(2, 1.0)
    np.testing.assert_allclose((M + np.eye(3)) / 2, np.array([[float(v) for v in r] for r in Ainv]), atol=2e-15)
    beta = sum(Ainv[2][j] * (k / ws[0] if j == 0 else 0) for j in range(3))
    assert abs(gv[2] - float(beta)) < 1e-15


# --------------------------------------------------------------------------
# Local block structure: axis-aligned velocities give I (x) B_1D
# --------------------------------------------------------------------------
@pytest.mark.parametrize("dim,axis,sign", [(2, 0, 1), (2, 1, -1), (3, 2, 1), (3, 0, -1)])
def test_local_block_is_kronecker(dim, axis, sign):
    p = 2
    v = [0.0, 0.0, 0.0]
    v[axis] = 2.0 * sign
    pb = scalar_problem(dim, 3, p, v)
    GLL, _ = O.cell_operator(pb, v)
    pb1 = scalar_problem(1, 3, p, [2.0 * sign, 0, 0])
    G1, _ = O.cell_operator(pb1, [2.0 * sign, 0, 0])
    # 1-D operator scaled by the cell measure ratio: same h -> identical entries
    mats = [np.eye(3)] * dim
    mats = list(mats)
    mats[axis] = G1
    K = mats[dim - 1]
    for d in reversed(range(dim - 1)):
        K = np.kron(K, mats[d])
    assert np.max(np.abs(GLL - K)) == 0.0


# --------------------------------------------------------------------------
# Properties of L_h
# --------------------------------------------------------------------------
VELS2 = [(2.0, 0.0, 0.0), (0.0, -2.0, 0.0), (2.0, 2.0, 0.0), (-1.0, 0.5, 0.0)]
VELS3 = [(0.0, 0.0, 2.0), (1.0, -0.5, 0.25), (-2.0, 0.0, 0.0)]


@pytest.mark.parametrize("dim,v", [(2, v) for v in VELS2] + [(3, v) for v in VELS3])
def test_constants_preserved(dim, v):
    """L_h F = 0 if all components of F (ghosts included) are the same."""
    pb = scalar_problem(dim, 3, 2, v)
    one = np.ones((pb.ncell, pb.Nd))
    out = O.apply_L(pb, v, one, one)
    assert np.max(np.abs(out)) < 1e-13


@pytest.mark.parametrize("p", [1, 2, 3])
@pytest.mark.parametrize("dim,v", [(2, v) for v in VELS2] + [(3, v) for v in VELS3])
def test_polynomial_exactness(dim, v, p):
    """For f in Q_p (degree <= p per variable) with exact ghost traces, the DG
    operator is exact: (L_h F)_j = -v . grad f(x_j) (GL exactness P:341-347)."""
    pb = scalar_problem(dim, 3, p, v, lo=[0.1, -0.3, 0.2], hi=[1.3, 0.6, 0.8])
    rng = np.random.default_rng(7 + p)
    coef = rng.standard_normal((p + 1,) * dim)
    X = node_positions(pb)

    def f_and_grad(X):
        f = np.zeros(X.shape[:-1])
        g = np.zeros(X.shape)
        for idx in np.ndindex(*coef.shape):
            mono = np.ones(X.shape[:-1])
            for d in range(dim):
                mono = mono * X[..., d] ** idx[d]
            f += coef[idx] * mono
            for d in range(dim):
                if idx[d] == 0:
                    continue
                dm = np.ones(X.shape[:-1]) * idx[d]
                for e in range(dim):
                    dm = dm * X[..., e] ** (idx[e] - (1 if e == d else 0))
                g[..., d] += coef[idx] * dm
        return f, g
    f, g = f_and_grad(X)
    out = O.apply_L(pb, v, f, f)  # ghost = exact trace of f at the boundary nodes
    expect = -np.einsum("cid,d->ci", g, np.asarray(v[:dim]))
    scale = max(1.0, np.max(np.abs(expect)))
    assert np.max(np.abs(out - expect)) < 1e-12 * scale


@pytest.mark.parametrize("dim,v", [(2, v) for v in VELS2] + [(3, v) for v in VELS3[:2]])
def test_dissipation_mass_weighted(dim, v):
    """F^T L_h F <= 0 with zero ghost, in the mass-weighted inner
    product M = diag(omega_{L,i}) (reading C9)."""
    pb = scalar_problem(dim, 3 if dim == 2 else 2, 2, v)
    L, _ = O.dense_L(pb, v)
    _, w = O.gl_1d(pb.p)
    wl = np.ones(1)
    for _d in range(dim):
        wl = np.kron(w, wl)
    h = 1.0 / pb.N[0]
    Mw = np.tile(wl * (h / 2) ** dim, pb.ncell)
    S = Mw[:, None] * L
    ev = np.linalg.eigvalsh(0.5 * (S + S.T))
    assert ev.max() < 1e-12 * np.abs(ev).max()


# --------------------------------------------------------------------------
# Dependency graph and triangular structure
# --------------------------------------------------------------------------
def test_levels_fig_dependency_graph(golden):
    g = golden("dependency_levels.json")
    pb = scalar_problem(2, g["mesh"][0], 2, g["velocity"])
    order, level = O.topo_order(pb, g["velocity"])
    groups = {}
    for c, l in zip(order, level):
        groups.setdefault(int(l), []).append(int(c))
    assert [sorted(groups[k]) for k in sorted(groups)] == g["levels"]


def test_graph_special_cases():
    pb = scalar_problem(2, 4, 1, (0.0, 0.0, 0.0))
    order, level = O.topo_order(pb, (0.0, 0.0, 0.0))
    assert list(order) == list(range(16)) and level.max() == 0  # v = 0: no edges
    pb = O.Problem(2, [5, 1], 1, [[1.0, 0, 0]], [0], 1, 1.0, 0, [1.0], 0.1)
    order, level = O.topo_order(pb, (1.0, 0.0, 0.0))
    assert list(order) == [0, 1, 2, 3, 4] and list(level) == [0, 1, 2, 3, 4]  # 1xN strip: chain
    pbn = O.Problem(2, [5, 1], 1, [[-1.0, 0, 0]], [0], 1, 1.0, 0, [1.0], 0.1)
    order, level = O.topo_order(pbn, (-1.0, 0.0, 0.0))
    assert list(order) == [4, 3, 2, 1, 0]  # -v reverses the edges


@pytest.mark.parametrize("v", [(2.0, 2.0, 0.0), (-1.0, 0.5, 0.0), (0.0, -2.0, 0.0)])
def test_block_triangular_in_topological_order(v):
    pb = scalar_problem(2, 3, 2, v)
    L, _ = O.dense_L(pb, v)
    order, _ = O.topo_order(pb, v)
    perm = np.concatenate([np.arange(c * pb.Nd, (c + 1) * pb.Nd) for c in order])
    Lp = L[np.ix_(perm, perm)]
    Nd = pb.Nd
    for bi in range(pb.ncell):
        for bj in range(bi + 1, pb.ncell):
            assert np.all(Lp[bi * Nd:(bi + 1) * Nd, bj * Nd:(bj + 1) * Nd] == 0.0)


# --------------------------------------------------------------------------
# T2 sweep
# --------------------------------------------------------------------------
@pytest.mark.parametrize("dim,v,dtp", [(2, (2.0, 0.0, 0.0), 0.3), (2, (2.0, 2.0, 0.0), 0.05),
                                       (2, (-1.0, 0.5, 0.0), 0.4), (3, (0.0, 0.0, -2.0), 0.2),
                                       (3, (1.0, -0.5, 0.25), 0.1)])
def test_sweep_equals_dense_cn_solve(dim, v, dtp):
    """Cell-by-cell sweep = dense (I - theta L)^{-1}((I + theta L) F + 2 theta B fb)."""
    pb = scalar_problem(dim, 3 if dim == 2 else 2, 2, v)
    rng = np.random.default_rng(3)
    F = rng.standard_normal((pb.ncell, pb.Nd))
    fb = rng.standard_normal((pb.ncell, pb.Nd))
    L, B = O.dense_L(pb, v)
    th = dtp / 2
    I = np.eye(L.shape[0])
    expect = np.linalg.solve(I - th * L, (I + th * L) @ F.reshape(-1) + 2 * th * B @ fb.reshape(-1))
    f = F.copy()
    O.t2_velocity(pb, v, dtp, f, fb)
    assert np.max(np.abs(f.reshape(-1) - expect)) < 1e-13 * max(1.0, np.max(np.abs(expect)))


def test_sweep_invariance_along_v():
    """Data constant along v, with matching ghost, is left unchanged by T2."""
    pb = scalar_problem(2, 4, 2, (2.0, 0.0, 0.0))
    rng = np.random.default_rng(5)
    rows = rng.standard_normal(pb.N[1] * pb.n)            # depends on Y only
    g = np.broadcast_to(rows[:, None], pb.grid_shape()).copy()
    f = pb.grid_to_cells(g)
    O.t2_velocity(pb, (2.0, 0.0, 0.0), 0.7, f, f.copy())
    assert np.max(np.abs(pb.cells_to_grid(f) - g)) < 1e-14


def test_sweep_time_symmetry():
    """T2(-dt') T2(dt') = I (eq prop_sym), on a small mesh at nu <= 0.1."""
    for v in [(1.0, 0.0, 0.0), (0.5, -1.0, 0.0)]:
        pb = scalar_problem(2, 3, 2, v)
        rng = np.random.default_rng(11)
        F = rng.standard_normal((pb.ncell, pb.Nd))
        fb = rng.standard_normal((pb.ncell, pb.Nd))
        f = F.copy()
        O.t2_velocity(pb, v, 0.02, f, fb)
        O.t2_velocity(pb, v, -0.02, f, fb)
        assert np.max(np.abs(f - F)) < 1e-12


# --------------------------------------------------------------------------
# Kinetic model and collision
# --------------------------------------------------------------------------
def model_problem(model, dim, lam=2.0, params=None):
    if model == "advection":
        m, flux, fp = 1, FLUX_ADVECTION, params or [1.0, 0.5, 0.0]
    elif model == "euler":
        m, flux, fp = dim + 2, FLUX_EULER, params or [1.4]
    else:
        m, flux, fp = dim + 1, FLUX_ISOTHERMAL, params or [1.0]
    vel, comp = velocity_set(dim, m, lam)
    return O.Problem(dim, 2, 1, vel, comp, m, lam, flux, fp, dt=0.1)


def test_flux_special_states(golden):
    for case in golden("flux_special_states.json")["cases"]:
        params = {"euler": [case.get("gamma", 1.4)], "isothermal": [case.get("c", 1.0)],
                  "advection": case.get("a", [1.0, 0.5]) + [0.0]}[case["model"]]
        pb = model_problem(case["model"], case["dim"], params=params)
        q = O.flux(pb, case["w"])
        for k, key in enumerate(["qx", "qy", "qz"][: case["dim"]]):
            np.testing.assert_allclose(q[k], case[key], atol=1e-14)


def random_physical_w(model, dim, rng):
    rho = 0.5 + rng.random()
    u = 0.4 * (rng.random(dim) - 0.5)
    if model == "advection":
        return np.array([rng.standard_normal()])
    if model == "isothermal":
        return np.concatenate([[rho], rho * u])
    E = 1.0 / 0.4 + 0.5 * rho * np.dot(u, u)
    return np.concatenate([[rho], rho * u, [E]])


@pytest.mark.parametrize("model,dim", [("advection", 2), ("euler", 2), ("euler", 3), ("isothermal", 2),
                                       ("isothermal", 3)])
def test_equilibrium_moments(model, dim):
    """P f^eq = w and sum_i v_i^k f^eq_i = q^k(w)."""
    pb = model_problem(model, dim)
    rng = np.random.default_rng(1)
    for _ in range(10):
        w = random_physical_w(model, dim, rng)
        feq = O.equilibrium(pb, w)
        P = np.zeros((pb.m, pb.nv))
        P[pb.comp, np.arange(pb.nv)] = 1.0
        np.testing.assert_allclose(P @ feq, w, atol=1e-14 * max(1, np.abs(w).max()))
        q = O.flux(pb, w)
        for k in range(dim):
            np.testing.assert_allclose(P @ (pb.vel[:, k] * feq), q[k], atol=1e-14 * max(1, np.abs(q).max()))


@pytest.mark.parametrize("model,dim", [("advection", 2), ("euler", 2), ("isothermal", 3)])
def test_collision_conservation_and_involution(model, dim):
    """C2 keeps w = P f; at tau = 0 C2(C2(f)) = f (w preserved => same f^eq)."""
    pb = model_problem(model, dim)
    rng = np.random.default_rng(2)
    nn = 50
    w = np.stack([random_physical_w(model, dim, rng) for _ in range(nn)], axis=1)
    f = O.equilibrium_field(pb, w) + 0.01 * rng.standard_normal((pb.nv, nn))
    f0 = f.copy()
    w0 = O.moments(pb, f)
    O.collide(pb, f, 0.1, tau=0.0)
    ulp = np.finfo(np.float64).eps
    assert np.max(np.abs(O.moments(pb, f) - w0)) <= 8 * ulp * max(1.0, np.abs(w0).max()) * pb.nv
    O.collide(pb, f, 0.1, tau=0.0)
    assert np.max(np.abs(f - f0)) < 1e-13


def test_collision_tau_positive_time_symmetric():
    """For tau > 0, C2(-dt) = C2(dt)^{-1} (eq prop_sym) and C2 keeps w."""
    pb = model_problem("isothermal", 3)
    rng = np.random.default_rng(4)
    w = np.stack([random_physical_w("isothermal", 3, rng) for _ in range(20)], axis=1)
    f = O.equilibrium_field(pb, w) + 0.01 * rng.standard_normal((pb.nv, 20))
    f0 = f.copy()
    O.collide(pb, f, 0.3, tau=0.05)
    assert np.max(np.abs(O.moments(pb, f) - O.moments(pb, f0))) < 1e-14
    O.collide(pb, f, -0.3, tau=0.05)
    assert np.max(np.abs(f - f0)) < 1e-13
    # tau -> 0 limit of eq collision_cn is 2 f^eq - f
    g = f0.copy()
    O.collide(pb, g, 0.3, tau=1e-13)
    h = f0.copy()
    O.collide(pb, h, 0.3, tau=0.0)
    assert np.max(np.abs(g - h)) < 1e-11


def test_config1_left_equilibrium_vanishes():
    """Config 1: f^eq_{x-} = w/4 - a_x w/(2 lambda) = 0 for a_x = 1, lambda = 2."""
    cfg = CONFIGS[1]
    pb = O.Problem.from_config(cfg)
    feq = O.equilibrium(pb, [0.7])
    assert feq[1] == 0.0 and abs(feq[0] - 0.35) < 1e-16


# --------------------------------------------------------------------------
# The palindromic step M2
# --------------------------------------------------------------------------
def test_m2_constant_equilibrium_fixed_point():
    """A constant equilibrium state with f^b = f^eq(w_const) is invariant."""
    cfg = CONFIGS[3].resized(3, steps=2)
    pb = O.Problem.from_config(cfg)
    w = np.array([1.1, 0.05, -0.02, 0.03])
    wg = np.broadcast_to(w.reshape(4, 1, 1, 1), (4,) + pb.grid_shape()).copy()
    f0 = O.equilibrium_field(pb, wg)
    f = O.m2_run(pb, f0, f0, 2)
    assert np.max(np.abs(f - f0)) < 1e-14


def test_m2_second_order_in_time():
    """Self-convergence of w at fixed mesh (config-1 model, N=16, p=2, T=0.25):
    slopes over the last two halvings in [1.9, 2.1]."""
    base = CONFIGS[1].resized(16)
    from pdg_inputs import w0_grid, wb_grid
    w0 = w0_grid(base).numpy()
    T = 0.25

    def run(nsteps):
        pb = O.Problem.from_config(base)
        pb.dt = T / nsteps
        f0, fb = O.initial_data(pb, w0, wb_grid(base, w0_grid(base)).numpy())
        f = O.m2_run(pb, f0, fb, nsteps)
        return O.moments(pb, f)
    ref = run(1024)
    errs = [np.max(np.abs(run(s) - ref)) for s in (16, 32, 64, 128)]
    slopes = [math.log2(errs[k] / errs[k + 1]) for k in range(3)]
    assert all(1.9 <= s <= 2.1 for s in slopes[-2:]), (errs, slopes)


def _advection_exact_errors(dim, Ns, p=2, nu=0.5, T=0.25, lam=2.0, a=(1.0, 0.5), c=(0.35, 0.4), k=200.0,
                            half_step=True):
    """max |w - w_exact| at t = T for the config-1 model (vectorial D1Q2 / D2Q4, q = a w,
    lambda = 2), Gaussian bump w0 = exp(-k |x - c|^2), mesh and dt refined together at fixed
    nu = lambda dt / h.  The exact solution of the limit system (eq macro_limit_system) is
    w0(x - a t) (P M2 converges to the macroscopic identity); with the bump at
    <= 2e-11 on the inflow faces for t <= T, the inflow data f^b = f^eq(0) is exact to that
    level.  half_step=False composes T2(dt) C2(dt) T2(dt) -- the plausible mistake of a full
    transport step on each side -- as a negative control."""
    errs = []
    for N in Ns:
        vel, comp = [], []
        for kk in range(dim):
            for s in (1.0, -1.0):
                v = [0.0, 0.0, 0.0]
                v[kk] = s * lam
                vel.append(v)
                comp.append(0)
        h = 1.0 / N
        nsteps = int(round(T / (nu * h / lam)))
        dt = T / nsteps
        pb = O.Problem(dim, N, p, vel, comp, 1, lam, 0, list(a[:dim]), dt)
        xg = {1: [-1.0, 1.0], 2: [-1.0, 0.0, 1.0], 3: [-1.0, -1 / math.sqrt(5), 1 / math.sqrt(5), 1.0]}[p]
        xs = [((np.arange(N)[:, None] + (np.asarray(xg)[None, :] + 1) / 2) * h).reshape(-1) for _ in range(dim)]

        def wfield(t):
            r2 = (xs[0] - c[0] - a[0] * t) ** 2
            if dim == 2:
                r2 = r2[None, :] + ((xs[1] - c[1] - a[1] * t) ** 2)[:, None]
            return np.exp(-k * r2)[None]
        w0 = wfield(0.0)
        f0, fb = O.initial_data(pb, w0, np.zeros_like(w0))
        if half_step:
            f = O.m2_run(pb, f0, fb, nsteps)
        else:
            fc, fbc = pb.grid_to_cells(f0), pb.grid_to_cells(fb)
            for _ in range(nsteps):
                O.t2_all(pb, dt, fc, fbc)
                O.collide(pb, fc, dt)
                O.t2_all(pb, dt, fc, fbc)
            f = pb.cells_to_grid(fc)
        errs.append(float(np.max(np.abs(O.moments(pb, f) - wfield(T)))))
    return errs


@pytest.mark.parametrize("dim,Ns", [(1, (32, 64, 128, 256)), (2, (16, 32, 64, 128))])
def test_m2_converges_to_exact_advection(dim, Ns):
    """M2 at tau = 0 against an exact solution, not itself: w -> w0(x - a t) at second order
    when h and dt are refined together; measured slopes 2.08/2.04/2.01
    (1-D) and 2.03/2.09/2.07 (2-D).  A wrong transport step (T2(dt) instead of T2(dt/2))
    moves the bump twice as far and does not converge at all."""
    errs = _advection_exact_errors(dim, Ns)
    slopes = [math.log2(errs[j] / errs[j + 1]) for j in range(len(errs) - 1)]
    assert all(1.85 <= s <= 2.25 for s in slopes[-2:]), (errs, slopes)
    assert errs[-1] < 3.5e-3, errs
    bad = _advection_exact_errors(dim, Ns[-2:], half_step=False)
    assert min(bad) > 0.3, bad


def test_cone_evaluation_matches_full_mesh():
    """Evaluating one M2 step on dependency cones of sampled cells equals the
    full-mesh step there (used for sampled parity at full config sizes)."""
    cfg = CONFIGS[3].resized(5)
    pb = O.Problem.from_config(cfg)
    from pdg_inputs import w0_grid
    w0 = w0_grid(cfg).numpy()
    f0, fb = O.initial_data(pb, w0, w0)
    rng = np.random.default_rng(9)
    f0 = f0 * (1 + 0.01 * rng.standard_normal(f0.shape))
    full = pb.grid_to_cells(O.m2_run(pb, f0, fb, 1))
    f0c, fbc = pb.grid_to_cells(f0), pb.grid_to_cells(fb)
    S = np.array([0, 31, 62, 124], dtype=np.int64)
    plan = O.m2_cone_plan(pb, S)
    got = O.m2_cone_step(pb, plan, lambda i, cells: f0c[i][cells], lambda i, cells: fbc[i][cells])
    assert np.max(np.abs(got - full[:, S])) == 0.0


def test_layout_roundtrip():
    cfg = CONFIGS[4].resized(3)
    pb = O.Problem.from_config(cfg)
    g = np.arange(np.prod(pb.grid_shape()), dtype=np.float64).reshape(pb.grid_shape())
    c = pb.grid_to_cells(g)
    assert np.array_equal(pb.cells_to_grid(c), g)
    # cell (cx,cy,cz)=(1,0,2), local (ax,ay,az)=(3,1,0) -> grid [Z=2*4+0, Y=0*4+1, X=1*4+3]
    cell = 1 + 3 * (0 + 3 * 2)
    loc = 3 + 4 * (1 + 4 * 0)
    assert c[cell, loc] == g[8, 1, 7]


@pytest.mark.parametrize("scheme,tau,order", [("m2kin", 0.05, 2.0), ("m2kin", 0.0, 2.0), ("m4", 0.05, 4.0)])
def test_palindromic_composition_orders(scheme, tau, order):
    """M2kin is second order also at tau = 0; its symmetric triple-jump
    composition is fourth order.  Config-1 model, N = 8, T = 0.25."""
    base = CONFIGS[1].resized(8)
    from pdg_inputs import w0_grid, wb_grid
    w0 = w0_grid(base).numpy()
    wb = wb_grid(base, w0_grid(base)).numpy()

    def run(nsteps):
        pb = O.Problem.from_config(base, tau=tau)
        pb.dt = 0.25 / nsteps
        f0, fb = O.initial_data(pb, w0, wb)
        return O.scheme_run(pb, f0, fb, nsteps, scheme)
    ref = run(512)
    errs = [np.max(np.abs(run(s) - ref)) for s in (16, 32, 64)]
    slopes = [math.log2(errs[k] / errs[k + 1]) for k in range(2)]
    assert all(abs(s - order) < 0.15 for s in slopes), (errs, slopes)


# --------------------------------------------------------------------------
# Lattice-Boltzmann models (NEXT-2)
# --------------------------------------------------------------------------
def test_d2q9_matches_paper(golden):
    from pdg_inputs import lattice
    g = golden("d2q9.json")
    lam = 1.7
    v, w = lattice("D2Q9", lam)
    assert [[x / lam for x in vi[:2]] for vi in v] == g["velocities_unit"]
    np.testing.assert_allclose(w, [_val(x) for x in g["weights"]], atol=1e-16)
    P = np.vstack([np.ones(9), np.array(v)[:, :2].T])
    np.testing.assert_allclose(P, np.array(g["P_rows_unit"]) * np.array([[1.0], [lam], [lam]]), atol=0)


@pytest.mark.parametrize("lat", ["D2Q9", "D3Q15", "D3Q19", "D3Q27"])
def test_lbm_equilibrium_moments(lat):
    """P f^eq = w (rho, rho u conserved) and the second moment is the isothermal
    Euler flux Pi = rho c^2 I + rho u u; at rest f^eq_i = w_i rho."""
    from pdg_inputs import lbm_config
    cfg = lbm_config(lat, 2, lam=1.3)
    pb = O.Problem.from_config(cfg)
    D = cfg.dim
    rng = np.random.default_rng(8)
    c2 = (cfg.lam / math.sqrt(3.0)) ** 2
    P = np.vstack([np.ones(pb.nv), pb.vel[:, :D].T])
    for _ in range(5):
        rho = 0.5 + rng.random()
        u = 0.1 * (rng.random(D) - 0.5)
        w = np.concatenate([[rho], rho * u])
        feq = O.equilibrium(pb, w)
        np.testing.assert_allclose(P @ feq, w, atol=1e-15)
        Pi = np.einsum("i,ia,ib->ab", feq, pb.vel[:, :D], pb.vel[:, :D])
        np.testing.assert_allclose(Pi, rho * c2 * np.eye(D) + rho * np.outer(u, u), atol=2e-15)
    feq = O.equilibrium(pb, np.concatenate([[1.3], np.zeros(D)]))
    np.testing.assert_allclose(feq, 1.3 * np.array(cfg.flux_params()[1:]), atol=1e-15)


def test_lbm_collision_conserves_and_m2_order():
    from pdg_inputs import lbm_config, w0_grid, wb_grid
    cfg = lbm_config("D2Q9", 6)
    pb = O.Problem.from_config(cfg)
    rng = np.random.default_rng(3)
    f = O.equilibrium_field(pb, w0_grid(cfg).numpy()) * (1 + 0.01 * rng.standard_normal((9,) + cfg.grid_shape))
    f = np.ascontiguousarray(f)
    w0 = O.moments(pb, f)
    O.collide(pb, f, cfg.dt)
    assert np.max(np.abs(O.moments(pb, f) - w0)) < 1e-14
    # second order in time of M2 on the D2Q9 model (diagonal transports included)
    base = lbm_config("D2Q9", 8)
    w0 = w0_grid(base).numpy()

    def run(nsteps):
        p2 = O.Problem.from_config(base)
        p2.dt = 0.1 / nsteps
        f0, fb = O.initial_data(p2, w0, wb_grid(base, w0_grid(base)).numpy())
        return O.moments(p2, O.m2_run(p2, f0, fb, nsteps))
    ref = run(256)
    errs = [np.max(np.abs(run(s) - ref)) for s in (8, 16, 32)]
    slopes = [math.log2(errs[k] / errs[k + 1]) for k in range(2)]
    assert all(1.85 <= s <= 2.15 for s in slopes), (errs, slopes)


# --------------------------------------------------------------------------
# NEXT-3: source step S2 and the Euler-with-gravity case
# --------------------------------------------------------------------------
def _gravity_problem(N=6, lat=None, G=(0.0, -1.0)):
    from dataclasses import replace
    from pdg_inputs import gravity_config, lbm_config
    cfg = gravity_config(N) if lat is None else replace(lbm_config(lat, N), gravity=tuple(G))
    return cfg, O.Problem.from_config(cfg)


@pytest.mark.parametrize("lat,G", [(None, (0.0, -1.0)), ("D3Q19", (0.3, 0.0, -1.0)), ("D3Q27", (0.0, 0.5, 0.2))])
def test_source_step_moments_closed_form(lat, G):
    """S2(h) leaves rho unchanged and adds exactly h rho G to the momentum (P g = s with
    s = (0, rho G); the source is linear in w and nilpotent, so CN is exact)."""
    from pdg_inputs import random_state
    cfg, pb = _gravity_problem(3 if lat else 6, lat, G)
    f = np.ascontiguousarray(random_state(cfg, 5, 0.5).numpy())
    w0 = O.moments(pb, f)
    h = 0.37
    O.source(pb, f, h)
    w1 = O.moments(pb, f)
    assert np.max(np.abs(w1[0] - w0[0])) <= 1e-15
    for d in range(cfg.dim):
        assert np.max(np.abs(w1[1 + d] - (w0[1 + d] + h * w0[0] * G[d]))) <= 1e-15


def test_source_step_time_symmetric_and_one_picard_iteration():
    """S2(-h) S2(h) = I (eq prop_sym) and the Picard solve of the CN source equation
    converges after one iteration (the check iteration is the second)."""
    from pdg_inputs import random_state
    cfg, pb = _gravity_problem(6)
    f = np.ascontiguousarray(random_state(cfg, 9, 0.5).numpy())
    g = f.copy()
    assert O.source(pb, g, 0.2) <= 2
    O.source(pb, g, -0.2)
    assert np.max(np.abs(g - f)) <= 4e-16


def _gravity_error(N, dt, scheme):
    from pdg_inputs import gravity_config, w0_grid
    cfg = gravity_config(N, dt=dt)
    pb = O.Problem.from_config(cfg)
    w0 = w0_grid(cfg).numpy()
    f0, fb = O.initial_data(pb, w0, w0)
    f = O.scheme_run(pb, f0, fb, cfg.steps, scheme)
    w = O.moments(pb, f)
    return float(np.sqrt(np.sum((w - w0) ** 2) / np.sum(w0 ** 2)))  # relative L2 (Fig. euler_gravity_order)


def test_gravity_m2s_second_order_in_time():
    """Fig. euler_gravity_order: the Strang scheme M2s = T2 S2 C2 S2 T2 on
    the fluid at rest in the gravity field, relative L2 error of w against the analytic stationary
    solution rho0 exp(-g y/c^2), u = 0 at t_max = 0.12, dt halved from 0.012: slopes in
    [1.75, 2.25].  Without the source step (M2) the error does not go to zero (negative control)."""
    dts = [0.012, 0.006, 0.003, 0.0015]
    e = [_gravity_error(16, dt, "m2s") for dt in dts]
    slopes = [np.log2(e[i] / e[i + 1]) for i in range(len(e) - 1)]
    assert all(1.75 <= s <= 2.25 for s in slopes), (e, slopes)
    e_nosrc = _gravity_error(16, dts[-1], "m2")
    assert e_nosrc > 30 * e[-1], (e_nosrc, e[-1])


# --------------------------------------------------------------------------
# The full-size parity harness (tests/parity_harness.py) builds the oracle's state in z-chunks
# with inflow data only on the inflow cell layers; on small boxes it must equal oracle.m2_run
# exactly (same oracle calls, different plumbing).
# --------------------------------------------------------------------------
@pytest.mark.parametrize("key,N,chunk", [(1, 8, 1 << 25), (2, 12, 1 << 25), (3, 5, 300), (4, 3, 1 << 25),
                                         (5, 6, 2000)])
def test_parity_harness_oracle_state_equals_m2_run(key, N, chunk):
    import torch
    from parity_harness import OracleRun, cells_to_grid_t, fill_w0
    from pdg_inputs import w0_grid, wb_grid
    cfg = CONFIGS[key].resized(N)
    w0 = torch.empty(cfg.m * cfg.nnodes, dtype=torch.float64)
    fill_w0(cfg, w0)
    orun = OracleRun(cfg, w0, chunk_elems=chunk)
    for _ in range(2):
        orun.step()
    pb = O.Problem.from_config(cfg)
    wg = w0_grid(cfg)
    f0, fb = O.initial_data(pb, wg.numpy(), wb_grid(cfg, wg).numpy())
    ref = O.m2_run(pb, f0, fb, 2)
    got = np.stack([cells_to_grid_t(torch.from_numpy(orun.fc[i]), orun.N, cfg.n, cfg.dim).numpy()
                    for i in range(cfg.nv)])
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("key,N,scheme", [(1, 1, "m2"), (3, 1, "m2kin"), (4, 1, "m4"), (2, 1, "m2"), (1, 3, "m2")])
def test_oracle_drivers_leave_their_inputs_unchanged(key, N, scheme):
    """The drivers update cell-blocked copies in place; with one cell per axis the grid -> cell
    reordering is the identity, and an aliased view would advance the caller's f (found when a
    parity test computed the reference before the GPU run).  Inputs stay bit-identical, and the
    result equals the one from a private copy."""
    cfg = CONFIGS[key].resized(N)
    w0 = w0_grid(cfg)
    pb = O.Problem.from_config(cfg)
    f0, fb = O.initial_data(pb, w0.numpy(), wb_grid(cfg, w0).numpy())
    fa, fba = f0.copy(), fb.copy()
    out = O.scheme_run(pb, f0, fb, 2, scheme)
    out2 = O.m2_run(pb, f0, fb, 1)
    assert np.array_equal(f0, fa) and np.array_equal(fb, fba)
    assert np.array_equal(out, O.scheme_run(pb, fa.copy(), fba.copy(), 2, scheme))
    assert not np.shares_memory(out, f0) and not np.shares_memory(out2, f0)
