"""Full-size parity harness (SURVEY §8(c) parity protocol) -- test infrastructure.

The oracle (oracle/, plain C, fp64, dense LU per cell, Kahn order) advances the WHOLE state of
a BASELINE config on the host; the CUDA path advances the same seeded state on the GPU through
the C-ABI.  Compared, over whole arrays (relative max-norm, reading C17):

  * re-synced one-step parity: the oracle's f^{n-1} is loaded into the GPU context, one pdg_step,
    compared with the oracle's f^n (isolates implementation error from the scheme's own
    amplification of rounding, reading C7);
  * free-running parity: the GPU run from the seeded equilibrium (pdg_step(1) per step in lockstep,
    and one pdg_step(steps) call -- the fused passes bench.py times) against the oracle run;
  * twin amplification of the map itself, measured in the same harness: the GPU path (and, where
    affordable, the oracle) rerun from f0 perturbed by a relative 1e-13;
  * non-physical states (rho <= 0 or non-finite values), reported per step.

Memory: the oracle keeps f cell-blocked ([nv][cell][node]) on the host, built in z-chunks
from the seeded w0; its inflow array f^b is allocated with np.zeros (untouched pages stay unmapped)
and filled only on the inflow cell layers, so config 5 (87 GB of f) fits a 196 GB host.  Layout
conversions (cell-blocked <-> node grid) are index permutations done with torch on the GPU: no
arithmetic of the method.
"""
from __future__ import annotations

import json
import math
import os
import time

import numpy as np
import torch

from oracle import oracle as O
from pdg_inputs import w0_grid

TWIN_EPS = 1e-13


def _log(msg):
    print(f"[{time.strftime('%H:%M:%S')}] {msg}", flush=True)


# ----------------------------------------------------------------------------
# layout plumbing (torch, on the GPU)
# ----------------------------------------------------------------------------
def cells_to_grid_t(t: torch.Tensor, N: list, n: int, dim: int) -> torch.Tensor:
    """[ncell, Nd] cell-blocked (cell = (cz*Ny + cy)*Nx + cx, node = (az*n + ay)*n + ax) -> node grid."""
    if dim == 3:
        v = t.view(N[2], N[1], N[0], n, n, n).permute(0, 3, 1, 4, 2, 5)
        return v.reshape(N[2] * n, N[1] * n, N[0] * n)
    v = t.view(N[1], N[0], n, n).permute(0, 2, 1, 3)
    return v.reshape(N[1] * n, N[0] * n)


def grid_to_cells_t(g: torch.Tensor, N: list, n: int, dim: int) -> torch.Tensor:
    """Inverse of cells_to_grid_t; the leading axis count of g may be a z-chunk (N[2] from g)."""
    if dim == 3:
        nz = g.shape[0] // n
        v = g.view(nz, n, N[1], n, N[0], n).permute(0, 2, 4, 1, 3, 5)
        return v.reshape(nz * N[1] * N[0], n ** 3)
    v = g.view(N[1], n, N[0], n).permute(0, 2, 1, 3)
    return v.reshape(N[1] * N[0], n * n)


# ----------------------------------------------------------------------------
# the oracle's state of a whole config
# ----------------------------------------------------------------------------
class OracleRun:
    """The oracle's M2 run of a config, cell-blocked on the host."""

    def __init__(self, cfg, w0_dev: torch.Tensor, perturb: float = 0.0, seed: int = 7, chunk_elems: int = 1 << 25):
        self.cfg = cfg
        self.pb = O.Problem.from_config(cfg)
        pb, n, D = self.pb, cfg.n, cfg.dim
        self.N = list(pb.N)
        nn = pb.nnodes
        t0 = time.time()
        self.fc = np.empty((pb.nv, pb.ncell, pb.Nd))
        # f0 = f^eq(w0) by the oracle, in z-chunks of cell layers (reading C13)
        w0 = w0_dev.view((cfg.m,) + cfg.grid_shape)
        if D == 3:
            per_layer = pb.N[0] * pb.N[1]
            chunk = max(1, chunk_elems // (per_layer * pb.Nd))
            for z0 in range(0, pb.N[2], chunk):
                z1 = min(pb.N[2], z0 + chunk)
                wl = np.ascontiguousarray(w0[:, z0 * n:z1 * n].cpu().numpy())
                fe = torch.from_numpy(O.equilibrium_field(pb, wl)).to(w0_dev.device)
                for i in range(pb.nv):
                    self.fc[i, z0 * per_layer:z1 * per_layer] = grid_to_cells_t(fe[i], self.N, n, D).cpu().numpy()
                del fe
        else:
            fe = torch.from_numpy(O.equilibrium_field(pb, np.ascontiguousarray(w0.cpu().numpy()))).to(w0_dev.device)
            for i in range(pb.nv):
                self.fc[i] = grid_to_cells_t(fe[i], self.N, n, D).cpu().numpy()
            del fe
        if perturb:
            rng = np.random.default_rng(seed)
            for i in range(pb.nv):
                self.fc[i] *= 1.0 + perturb * (rng.random(self.fc[i].shape) - 0.5)
        # f^b = f^eq(w_b), w_b = w0(x_b) (configs 2-5) or 0 (config 1) (reading C12), only on the
        # inflow cell layers
        self.fbc = np.zeros((pb.nv, pb.ncell, pb.Nd))  # calloc: untouched pages are never mapped
        wb = torch.zeros_like(w0) if cfg.wb_zero else w0
        for k in range(D):
            for s in (+1, -1):
                self._fill_inflow_layer(wb, k, s)
        self.steps_done = 0
        _log(f"oracle {cfg.name}: initial data ready ({time.time() - t0:.1f} s, f {self.fc.nbytes / 1e9:.1f} GB)")

    def _fill_inflow_layer(self, w0, k, s):
        cfg, pb, n, D = self.cfg, self.pb, self.cfg.n, self.cfg.dim
        ax = D - 1 - k  # numpy axis of physical axis k in the node grid
        L = cfg.N * n
        sl = [slice(None)] * (D + 1)
        sl[1 + ax] = slice(0, n) if s > 0 else slice(L - n, L)
        wl = np.ascontiguousarray(w0[tuple(sl)].cpu().numpy())          # [m, layer grid]
        Nl = list(pb.N)
        Nl[k] = 1
        lay = O.Problem(D, Nl, cfg.p, pb.vel, pb.comp, pb.m, pb.lam, pb.flux, pb.fparams, pb.dt)
        fe = O.equilibrium_field(pb, wl)                                 # oracle's f^eq at those nodes
        fe_c = lay.grid_to_cells(fe)                                     # [nv, layer cells, Nd]
        # global cell index of each layer cell: insert c_k = 0 (s = +) or N-1 (s = -)
        idx = np.arange(lay.ncell)
        cc, r = [], idx.copy()
        for d in range(D):
            cc.append(r % Nl[d])
            r //= Nl[d]
        cc[k] = np.full_like(idx, 0 if s > 0 else pb.N[k] - 1)
        g = np.zeros_like(idx)
        for d in reversed(range(D)):
            g = g * pb.N[d] + cc[d]
        for i in range(pb.nv):
            kk = (i % (2 * D)) // 2
            ss = -1 if i % 2 else 1
            if kk == k and ss == s:
                self.fbc[i, g] = fe_c[i]

    def step(self):
        pb = self.pb
        O.t2_all(pb, 0.5 * pb.dt, self.fc, self.fbc)
        O.collide(pb, self.fc, pb.dt)
        O.t2_all(pb, 0.5 * pb.dt, self.fc, self.fbc)
        self.steps_done += 1

    def moments(self):
        return O.moments(self.pb, self.fc)                                # [m, ncell, Nd]

    def nonphysical(self) -> int:
        """Nodes of the oracle's current state with rho <= 0 or a non-finite value (component 0 of w
        is the density of the Euler / isothermal models; the advection model has none)."""
        if self.pb.flux == 0:
            return int(sum(int((~np.isfinite(self.fc[i])).sum()) for i in range(self.pb.nv)))
        w = self.moments()
        bad = ~(w[0] > 0.0)
        for c in range(1, w.shape[0]):
            bad |= ~np.isfinite(w[c])
        return int(bad.sum())


# ----------------------------------------------------------------------------
# GPU side
# ----------------------------------------------------------------------------
def load_into(S, orun: OracleRun):
    """Copy the oracle's f (cell-blocked, host) into the context's f buffer (node grid)."""
    cfg = orun.cfg
    nn = cfg.nnodes
    for i in range(orun.pb.nv):
        t = torch.from_numpy(orun.fc[i]).to(S.f.device)
        S.f[i * nn:(i + 1) * nn].view(cfg.grid_shape).copy_(cells_to_grid_t(t, orun.N, cfg.n, cfg.dim))
        del t
    torch.cuda.synchronize(S.f.device)


def compare_f(f_dev: torch.Tensor, orun: OracleRun):
    """(max |f_gpu - f_oracle|, max |f_oracle|, non-finite count on each side) over the whole f."""
    cfg = orun.cfg
    nn = cfg.nnodes
    dmax, rmax, bad_g, bad_o = 0.0, 0.0, 0, 0
    for i in range(orun.pb.nv):
        ref = cells_to_grid_t(torch.from_numpy(orun.fc[i]).to(f_dev.device), orun.N, cfg.n, cfg.dim)
        got = f_dev[i * nn:(i + 1) * nn].view(cfg.grid_shape)
        bad_g += int((~torch.isfinite(got)).sum())
        bad_o += int((~torch.isfinite(ref)).sum())
        dmax = max(dmax, float((got - ref).abs().max()))
        rmax = max(rmax, float(ref.abs().max()))
        del ref
    return dmax, rmax, bad_g, bad_o


def compare_w(S, orun: OracleRun):
    cfg = orun.cfg
    wg = S.moments().view((cfg.m,) + cfg.grid_shape)
    wo = orun.moments()
    dmax, rmax = 0.0, 0.0
    for c in range(cfg.m):
        ref = cells_to_grid_t(torch.from_numpy(np.ascontiguousarray(wo[c])).to(wg.device), orun.N, cfg.n, cfg.dim)
        dmax = max(dmax, float((wg[c] - ref).abs().max()))
        rmax = max(rmax, float(ref.abs().max()))
    return dmax / rmax if rmax > 0 else dmax


def rel(d, r):
    return d / r if r > 0 else d


def spread(a: torch.Tensor, b: torch.Tensor, nv: int) -> float:
    """||a - b||_inf / ||b||_inf over the whole f (velocity by velocity to bound memory; b may be on
    the host)."""
    nn = a.numel() // nv
    dmax, rmax = 0.0, 0.0
    for i in range(nv):
        x, y = a[i * nn:(i + 1) * nn], b[i * nn:(i + 1) * nn].to(a.device)
        dmax = max(dmax, float((x - y).abs().max()))
        rmax = max(rmax, float(y.abs().max()))
    return rel(dmax, rmax)


def perturb_(f_dev: torch.Tensor, nv: int, eps: float = TWIN_EPS, seed: int = 11):
    g = torch.Generator(device=f_dev.device).manual_seed(seed)
    nn = f_dev.numel() // nv
    for i in range(nv):
        x = f_dev[i * nn:(i + 1) * nn]
        x.mul_(1.0 + eps * (torch.rand(x.shape, generator=g, device=x.device, dtype=x.dtype) - 0.5))


def fill_w0(cfg, w_flat):
    w = w_flat.view((cfg.m,) + cfg.grid_shape)
    if cfg.dim == 2:
        w.copy_(w0_grid(cfg, device=w_flat.device))
        return
    L = cfg.N * cfg.n
    slab = max(1, min(L, (1 << 24) // (L * L)))
    for z0 in range(0, L, slab):
        w[:, z0:z0 + slab].copy_(w0_grid(cfg, device=w_flat.device, zslab=(z0, min(L, z0 + slab))))


def nonphysical(S) -> int:
    return int(S.check_state())


# ----------------------------------------------------------------------------
# the protocol
# ----------------------------------------------------------------------------
def run_protocol(cfg, resync_steps, lockstep=True, oracle_twin=False, gpu_twin=True, steps=None,
                 out_path=None, stop_on_nonfinite=True):
    """Run the parity protocol on `cfg` (full size); returns the record dict (also written to out_path)."""
    from paper_1702_00169_b200 import pdg
    steps = cfg.steps if steps is None else steps
    dev = torch.device("cuda", torch.cuda.current_device())
    rec = {"config": cfg.name, "N": cfg.N, "p": cfg.p, "lambda": cfg.lam, "dt": cfg.dt, "nu": cfg.lam * cfg.dt / cfg.h,
           "steps": steps, "nv": cfg.nv, "nodes": cfg.nnodes, "twin_eps": TWIN_EPS, "per_step": [],
           "host_threads": os.environ.get("OMP_NUM_THREADS") or os.cpu_count()}

    def solver():
        return pdg.Solver(pdg.problem_from_config(cfg))

    R = solver()                                     # re-synced steps, then the fused free run
    w0 = torch.empty_like(R.w)
    fill_w0(cfg, w0)
    wb = torch.zeros_like(w0) if cfg.wb_zero else w0   # reading C12
    R.set_equilibrium(w0, wb)
    F = T = None
    if lockstep:
        F = solver()
        F.set_equilibrium(w0, wb)
        if gpu_twin:
            T = solver()
            T.set_equilibrium(w0, wb)
            perturb_(T.f, cfg.nv)
    torch.cuda.synchronize()
    orun = OracleRun(cfg, w0)
    otwin = OracleRun(cfg, w0, perturb=TWIN_EPS) if oracle_twin else None
    t_start = time.time()
    last_agree = 0
    for n in range(1, steps + 1):
        e = {"step": n}
        if n in resync_steps:
            # the input state of the re-synced step: a state with rho <= 0 somewhere makes the
            # collision (1/rho in the flux) arbitrarily ill-conditioned, so the 1e-12 bar applies to
            # physical inputs only (reading C7)
            e["oracle_nonphysical_in"] = orun.nonphysical()
            load_into(R, orun)                       # oracle f^{n-1}
            R.step(1)                                # runs on the GPU while the oracle computes f^n
        if F is not None:
            F.step(1)
            if T is not None:
                T.step(1)
        t0 = time.time()
        orun.step()
        if otwin is not None:
            otwin.step()
        e["oracle_s"] = round(time.time() - t0, 2)
        if n in resync_steps:
            d, r, bg, bo = compare_f(R.f, orun)
            e["resync_f"] = rel(d, r)
            e["resync_w"] = compare_w(R, orun)
            e["resync_nonfinite_gpu"], e["nonfinite_oracle"] = bg, bo
        if F is not None:
            d, r, bg, bo = compare_f(F.f, orun)
            e["free_f"], e["free_nonfinite_gpu"], e["nonfinite_oracle"] = rel(d, r), bg, bo
            e["free_w"] = compare_w(F, orun)
            e["nonphysical_gpu"] = nonphysical(F)
            if T is not None:
                e["gpu_twin_spread"] = spread(T.f, F.f, cfg.nv)
                e["gpu_twin_amplification"] = e["gpu_twin_spread"] / TWIN_EPS
            if bg == 0 and bo == 0 and e["free_f"] <= 1e-12:
                last_agree = n
        if otwin is not None:
            dmax, rmax = 0.0, 0.0
            dmax = float(np.max(np.abs(otwin.fc - orun.fc)))
            rmax = float(np.max(np.abs(orun.fc)))
            e["oracle_twin_spread"] = rel(dmax, rmax)
            e["oracle_twin_amplification"] = e["oracle_twin_spread"] / TWIN_EPS
        rec["per_step"].append(e)
        _log(json.dumps(e))
        if stop_on_nonfinite and e.get("nonfinite_oracle", 0) > 0:
            rec["stopped_at_step"] = n
            break
    rec["last_step_finite_and_agree_1e-12"] = last_agree if F is not None else None
    rec["oracle_seconds"] = round(time.time() - t_start, 1)
    # one pdg_step(steps) call from the seeded equilibrium: the fused passes bench.py times
    if rec.get("stopped_at_step") is None:
        R.set_equilibrium(w0, wb)
        R.step(steps)
        d, r, bg, bo = compare_f(R.f, orun)
        rec["fused_free_f"] = rel(d, r)
        rec["fused_free_w"] = compare_w(R, orun)
        rec["fused_nonfinite_gpu"] = bg
        rec["fused_nonphysical_gpu"] = nonphysical(R)
        if not lockstep and gpu_twin:
            # twin amplification of the whole run with one context: keep the unperturbed result on the
            # host, rerun from the perturbed equilibrium (the oracle's state is freed first)
            del orun
            orun = None
            keep = R.f.cpu()
            R.set_equilibrium(w0, wb)
            perturb_(R.f, cfg.nv)
            R.step(steps)
            rec["gpu_twin_spread_final"] = spread(R.f, keep, cfg.nv)
            rec["gpu_twin_amplification_final"] = rec["gpu_twin_spread_final"] / TWIN_EPS
            del keep
    for X in (R, F, T):
        if X is not None:
            X.destroy()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    if out_path:
        with open(out_path, "w") as fh:
            json.dump(rec, fh, indent=1)
    _log(f"{cfg.name}: " + json.dumps({k: v for k, v in rec.items() if k != "per_step"}))
    return rec
