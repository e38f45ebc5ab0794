"""Seeded randomized parity sweep: small boxes with random cell counts per axis, degrees,
velocity-set kinds, time steps (both signs), schemes and relaxation times, through the
C-ABI against the oracle.  Complements the hand-picked cases with combinations nobody
chose (ragged tails on every axis, one-cell axes, every wavefront class)."""
import math

import numpy as np
import pytest

from oracle import oracle as O
from gpu_helpers import full_grid_to_planes, lattice_planes, rel_maxnorm, to_dev, to_np

pytestmark = pytest.mark.gpu

LATTICES = {2: ["D2Q9"], 3: ["D3Q15", "D3Q19", "D3Q27"]}


def _case(seed, backward=False):
    from paper_1702_00169_b200 import pdg
    from pdg_inputs import lattice, velocity_set
    rng = np.random.default_rng((3000 if backward else 1000) + seed)
    dim = int(rng.integers(2, 4))
    p = int(rng.integers(1, 4))
    lat = bool(rng.integers(0, 2))
    ncell = [int(rng.integers(1, 41 if dim == 2 else 11)) for _ in range(dim)]
    hi = [float(rng.uniform(0.5, 2.0)) for _ in range(dim)] + [1.0] * (3 - dim)
    scheme = ["m2", "m2kin"][int(rng.integers(0, 2))]
    steps = int(rng.integers(1, 3))
    if lat:
        name = LATTICES[dim][int(rng.integers(0, len(LATTICES[dim])))]
        lam = 1.0
        vel, wts = lattice(name, lam)
        comp = [0] * len(vel)
        m, flux = dim + 1, pdg.PDG_FLUX_LBM
        fparams = [lam / math.sqrt(3.0)] + list(wts)
    else:
        name = "vectorial"
        lam = 3.5
        m, flux = dim + 1, pdg.PDG_FLUX_ISOTHERMAL
        vel, comp = velocity_set(dim, m, lam)
        fparams = [1.0]
    h = min(hi[d] / ncell[d] for d in range(dim))
    nu = float(rng.uniform(0.05, 2.0)) if not backward else -float(rng.uniform(0.005, 0.2))
    dt = nu * h / lam
    if scheme == "m2":
        tau = 0.0
    elif not backward:
        tau = float(rng.uniform(0.0, 1.0)) * abs(dt)
    else:  # collision substeps h = dt/2 < 0 need 2 tau + h > 0 (eq collision_cn; checked by pdg_create)
        tau = 0.0 if rng.random() < 0.3 else float(rng.uniform(0.3, 1.0)) * abs(dt)
    sch = {"m2": pdg.PDG_SCHEME_M2, "m2kin": pdg.PDG_SCHEME_M2KIN}[scheme]
    pb = pdg.make_problem(dim, ncell, p, m, vel, comp, lam, flux, fparams, dt, tau=tau, scheme=sch, hi=tuple(hi))
    ob = O.Problem(dim, ncell, p, vel, comp, m, lam, flux, fparams, dt, tau=tau, hi=hi)
    desc = f"seed {seed}: {name} dim {dim} cells {ncell} p {p} nu {nu:.3f} {scheme} tau {tau:.2e} steps {steps}"
    return pb, ob, rng, desc, steps, scheme, lat


def _run_case(seed, backward):
    from paper_1702_00169_b200 import pdg
    pb, ob, rng, desc, steps, scheme, lat = _case(seed, backward)
    S = pdg.Solver(pb)
    shape = ob.grid_shape()
    nv = ob.nv
    # a positive state near equilibrium magnitudes, and positive inflow data
    base = 1.0 / nv
    f = base * (1.0 + 0.2 * (rng.random((nv,) + shape) - 0.5))
    fb = base * (1.0 + 0.2 * rng.random((nv,) + shape))

    class _C:
        pass
    cv = _C()
    cv.dim, cv.grid_shape = ob.dim, shape
    cv.velocities = lambda: (ob.vel.tolist(), None)
    planes = lattice_planes(cv, fb, S.sizes.plane_stride) if lat else full_grid_to_planes(cv, fb, S.sizes.plane_stride)
    S.set_state(to_dev(f), to_dev(planes))
    S.step(steps)
    got = to_np(S.get_state(), f.shape)
    w = to_np(S.moments(), (ob.m,) + shape)
    S.destroy()
    ref = O.scheme_run(ob, f, fb, steps, scheme)
    return f, fb, ob, steps, scheme, desc, rel_maxnorm(got, ref), rel_maxnorm(w, O.moments(ob, ref)), ref


def _ulp_spread(ob, f, fb, steps, scheme, ref, seed, samples=3):
    """The map's own amplification of rounding, measured on the oracle: the largest relative change
    of its result when f is perturbed by one ulp (relative 2^-52, random signs), over `samples`
    perturbations (one sample can underestimate it by two orders of magnitude: seed 803 of the
    backward sweep gave 4.9e-14 with one sign pattern and 5.2e-12 with another)."""
    eps = 2.0 ** -52
    out = 0.0
    for k in range(samples):
        sg = np.where(np.random.default_rng(seed + 7919 * k).random(f.shape) < 0.5, -1.0, 1.0)
        out = max(out, rel_maxnorm(O.scheme_run(ob, f * (1.0 + eps * sg), fb, steps, scheme), ref))
    return out


# A case whose map amplifies a one-ulp change of its input above 1e-13 is ill-conditioned: two
# correct fp64 implementations differ there by about that spread (DESIGN.md parity protocol,
# readings C7/C28).  Such a case is held to 64 ulp-equivalents of its measured spread (the rounding
# a path accumulates over the ~10 operator applications of two steps); every other case to 1e-12.
ILL_CONDITIONED = 1e-13


@pytest.mark.parametrize("seed", range(int(__import__("os").environ.get("PDG_FUZZ_SEEDS_MAIN", "40"))))
def test_fuzz_parity(seed):
    """Forward steps (dt > 0): <= 1e-12, the north star's bar, for every well-conditioned case.
    A case above it must be ill-conditioned (its oracle 1-ulp spread > 1e-13: random states that
    blow up -- e.g. seed 2769 of the 4000-seed campaign, max|f| 0.04 -> 6.4e5 in two steps, spread
    3.8e-11) and within 64 times its spread; both numbers are printed."""
    f, fb, ob, steps, scheme, desc, err_f, err_w, ref = _run_case(seed, backward=False)
    if err_f <= 1e-12 and err_w <= 1e-12:
        return
    spread = _ulp_spread(ob, f, fb, steps, scheme, ref, seed)
    print(f"forward {desc}: err_f {err_f:.2e} err_w {err_w:.2e} 1-ulp spread {spread:.2e} "
          f"ratio {err_f / max(spread, 1e-300):.1f}")
    assert spread > ILL_CONDITIONED, (desc, err_f, err_w, spread)
    assert err_f <= 64.0 * spread and err_w <= 64.0 * spread, (desc, err_f, err_w, spread)


@pytest.mark.parametrize("seed", range(int(__import__("os").environ.get("PDG_FUZZ_SEEDS_BACKWARD", "12"))))
def test_fuzz_backward_steps(seed):
    """Backward steps (dt < 0, T2(-dt') = T2(dt')^{-1}, eq prop_sym) are outside the
    configs and reported separately: the backward map amplifies rounding (the carry factor |beta|
    grows, and with tau > 0 the collision factor (2 tau - dt)/(2 tau + dt) exceeds 1), so the bar
    scales with the map's own amplification measured on the oracle (_ulp_spread) -- 64
    ulp-equivalents for the rounding a path accumulates over the ~10 operator applications of two
    steps (DESIGN.md parity protocol); never below 1e-12."""
    f, fb, ob, steps, scheme, desc, err_f, err_w, ref = _run_case(seed, backward=True)
    if err_f <= 1e-12 and err_w <= 1e-12:
        return
    spread = _ulp_spread(ob, f, fb, steps, scheme, ref, seed)
    tol = max(1e-12, 64.0 * spread)
    print(f"backward {desc}: err_f {err_f:.2e} err_w {err_w:.2e} 1-ulp spread {spread:.2e} "
          f"ratio {err_f / max(spread, 1e-300):.1f}")
    assert err_f <= tol and err_w <= tol, (desc, err_f, err_w, spread, tol)


# --------------------------------------------------------------------------
# Protocol fuzz: lattice sets with the cross-CTA hand-overs and chain segments, with random
# CTA shapes forced through the launch plan (pdg_problem.lattice_cta / lattice_segment, DESIGN.md
# §12), on boxes large enough for several CTAs and segments.  PDG_FUZZ_SEEDS widens the sweep (default 24 seeds).
# --------------------------------------------------------------------------
N_PROTO = int(__import__("os").environ.get("PDG_FUZZ_SEEDS", "24"))


@pytest.mark.parametrize("seed", range(N_PROTO))
def test_fuzz_lattice_protocols(seed):
    from paper_1702_00169_b200 import pdg
    from pdg_inputs import lattice
    rng = np.random.default_rng(5000 + seed)
    dim = int(rng.integers(2, 4))
    p = int(rng.integers(1, 4)) if dim == 2 else int(rng.integers(1, 3))
    name = LATTICES[dim][int(rng.integers(0, len(LATTICES[dim])))]
    ncell = ([int(rng.integers(20, 81)) for _ in range(2)] if dim == 2
             else [int(rng.integers(4, 13)), int(rng.integers(4, 13)), int(rng.integers(12, 33))])
    kappa = float(rng.choice([0.1, 0.25, 0.5, 1.0]))
    h = 1.0 / ncell[0]
    hi = [ncell[d] * h for d in range(dim)] + [1.0] * (3 - dim)  # square cells: equal kappas
    dt = 2.0 * kappa * h
    cta = [(1, 1), (2, 2), (1, 2), (2, 1), (4, 2)][int(rng.integers(0, 5))]
    seg = int(rng.choice([-1, 12, 16, 20, 30]))
    plan = {"lattice_cta": cta, "lattice_segment": seg}
    vel, wts = lattice(name, 1.0)
    fparams = [1.0 / math.sqrt(3.0)] + list(wts)
    if True:  # (indentation kept from the env-knob version)
        pb = pdg.make_problem(dim, ncell, p, dim + 1, vel, [0] * len(vel), 1.0, pdg.PDG_FLUX_LBM, fparams, dt,
                              hi=tuple(hi), **plan)
        S = pdg.Solver(pb)
        ob = O.Problem(dim, ncell, p, vel, [0] * len(vel), dim + 1, 1.0, 3, fparams, dt, hi=hi)
        shape = ob.grid_shape()
        base = 1.0 / ob.nv
        f = base * (1.0 + 0.2 * (rng.random((ob.nv,) + shape) - 0.5))
        fb = base * (1.0 + 0.2 * rng.random((ob.nv,) + shape))

        class _C:
            pass
        cv = _C()
        cv.dim, cv.grid_shape = ob.dim, shape
        cv.velocities = lambda: (ob.vel.tolist(), None)
        S.set_state(to_dev(f), to_dev(lattice_planes(cv, fb, S.sizes.plane_stride)))
        S.step(2)
        got = to_np(S.get_state(), f.shape)
        S.destroy()
    ref = O.scheme_run(ob, f, fb, 2, "m2")
    err = rel_maxnorm(got, ref)
    assert err <= 1e-12, (seed, name, dim, ncell, p, kappa, plan, err)
