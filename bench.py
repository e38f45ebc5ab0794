"""bench.py -- node.velocity updates/s of the palindromic PDG step on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--impl product|reference]

One "step" is one palindromic step M2(dt) = T2(dt/2) C2(dt) T2(dt/2)
over the whole workload (all rows of SURVEY §8(a)).  The default workload is
BASELINE config 5 (3-D isothermal, 256^3 cells, p=2, D3Q6 x 4 components: 10.9 G
node.velocity updates per step; f = 87 GB in place, far larger than L2, so no L2
flush is needed between steps).  Multi-GPU (torchrun): the exact z-slab decomposition by
default (--decomp zslab: slabs of cell planes, NCCL all-gather of carry planes), or
velocity shards with one NCCL sum of the moments per collision, pipelined over node chunks
(--decomp velocity: the north star's partition; the default for --lattice workloads); the
line's `alt_decomposition` times the other one in the same run (--one-decomp skips it);
strong scaling: total work fixed.

The JSON line adds:
  roofline     : the dominant kernel's algorithmic bytes / its CUDA-event time (on the
                 library stream), against MEASURED_PEAKS.json hbm_gbs.
  cpu_baseline : the CPU oracle (oracle/, as it stands) timed on this host on a bounded
                 sample of the same workload (N=128 sub-box of config 5, same p, nu, model:
                 ~10 s of CPU work), with the CPU model, RAM and a single-thread timing
                 (N=32 sub-box).
  e2e          : the same metric through the public C-ABI with HOST buffers: per step,
                 pdg_set_equilibrium(host w0, pinned) + pdg_step(1) + pdg_moments(host w), with
                 PDG_ASYNC_HOST so that uploads and downloads of consecutive steps overlap.
  clocks       : nvidia-smi samples taken during the timed region.
--impl reference times the oracle (the base contract's reference arm for this tier).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "node·velocity updates/s per palindromic PDG step (fp64), % of HBM roofline"
UNIT = "node·velocity updates/s"
FALLBACK_HBM_GBS = 6650.0


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            pk = json.load(fh)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def ncu_traffic(cfg, kernel):
    """DRAM bytes per launch of `kernel` from the committed ncu --set full summary of this workload."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as fh:
            t = json.load(fh)
        if t.get("workload") == cfg.name and kernel in t["kernels"]:
            return float(t["kernels"][kernel]["dram_bytes_per_launch"]), t.get("source")
    except Exception:
        pass
    return None, None


# ----------------------------------------------------------------------------
# clocks sampled during the timed region
# ----------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, val in zip(names, parts[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        sm.sort()
        med = sm[len(sm) // 2] if sm else None
        return {"sm_mhz": med, "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------
# CPU oracle baseline (rank 0, N=1) and the --impl reference arm
# ----------------------------------------------------------------------------
def oracle_sample_cfg(cfg, N_sub):
    return cfg.resized(N_sub, name=f"{cfg.name}@N{N_sub}")


def oracle_prepare(cfg, N_sub):
    import numpy as np
    from oracle import oracle as O
    from pdg_inputs import w0_grid, wb_grid
    sub = oracle_sample_cfg(cfg, min(N_sub, cfg.N))
    pb = O.Problem.from_config(sub)
    w0 = w0_grid(sub)
    f0, fb = O.initial_data(pb, w0.numpy(), wb_grid(sub, w0).numpy())
    fc = pb.grid_to_cells(f0)
    fbc = pb.grid_to_cells(fb)
    return sub, pb, fc, fbc, np


def oracle_step(pb, fc, fbc):
    from oracle import oracle as O
    O.t2_all(pb, 0.5 * pb.dt, fc, fbc)
    O.collide(pb, fc, pb.dt)
    O.t2_all(pb, 0.5 * pb.dt, fc, fbc)


def omp_threads():
    try:
        return int(os.environ.get("OMP_NUM_THREADS", "")) or os.cpu_count()
    except ValueError:
        return os.cpu_count()


def host_info():
    """CPU model and RAM of the host the oracle runs on (state them)."""
    model, ram = None, None
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
        with open("/proc/meminfo") as fh:
            for ln in fh:
                if ln.startswith("MemTotal"):
                    ram = round(int(ln.split()[1]) / 1024 ** 2, 1)
                    break
    except OSError:
        pass
    return model, ram


def single_thread_baseline(cfg, N_sub):
    """The same oracle step on one thread (OMP_NUM_THREADS=1 in a child process)."""
    code = ("import sys, time, json; sys.path.insert(0, %r); import bench; from pdg_inputs import CONFIGS, lbm_config; "
            "cfg = %s; sub, pb, fc, fbc, _ = bench.oracle_prepare(cfg, %d); t0 = time.perf_counter(); "
            "bench.oracle_step(pb, fc, fbc); dt = time.perf_counter() - t0; "
            "print(json.dumps({'value': sub.updates_per_step / dt, 'seconds': dt, 'N': sub.N, "
            "'updates': sub.updates_per_step}))")
    expr = (f"lbm_config({cfg.lattice!r}, {cfg.N}, p={cfg.p}, nu=2.0)" if cfg.lattice else
            f"[c for c in CONFIGS.values() if c.name == {cfg.name!r}][0]")
    env = dict(os.environ, OMP_NUM_THREADS="1")
    try:
        out = subprocess.run([sys.executable, "-c", code % (ROOT, expr, N_sub)], env=env, capture_output=True,
                             text=True, timeout=120)
        r = json.loads(out.stdout.strip().splitlines()[-1])
        return {"value": r["value"], "unit": UNIT, "cores": 1,
                "sample": f"1 M2 step of the {r['N']}^{cfg.dim}-cell sub-box ({r['updates']} node.velocity "
                          f"updates, {r['seconds']:.2f} s)"}
    except Exception as e:  # reported, never fatal
        return {"error": repr(e)[:200]}


def cpu_baseline(cfg, N_sub=64):
    sub, pb, fc, fbc, _ = oracle_prepare(cfg, N_sub)
    N_sub = sub.N
    t0 = time.perf_counter()
    oracle_step(pb, fc, fbc)
    dt = time.perf_counter() - t0
    ups = sub.updates_per_step / dt
    model, ram = host_info()
    return {"value": ups, "unit": UNIT, "cores": omp_threads(), "kind": "oracle",
            "sample": f"1 M2 step of the {N_sub}^{cfg.dim}-cell sub-box of {cfg.name} (same p, lambda, nu, model; "
                      f"{sub.updates_per_step} node.velocity updates, {dt:.2f} s), oracle/pdg_oracle.c -O2 "
                      f"-ffp-contract=off, OpenMP over velocities/nodes",
            "cpu_model": model, "ram_gb": ram,
            "single_thread": single_thread_baseline(cfg, max(4, N_sub // 4))}


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    N_sub = args.ref_cells
    sub, pb, fc, fbc, _ = oracle_prepare(cfg, N_sub)
    for _ in range(args.warmup):
        oracle_step(pb, fc, fbc)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle_step(pb, fc, fbc)
    dt = time.perf_counter() - t0
    ups = sub.updates_per_step * args.steps / dt
    sample = (f"each step = 1 M2 step of the {N_sub}^{cfg.dim}-cell sub-box of {cfg.name} (same p, lambda, nu, "
              f"model; {sub.updates_per_step} node.velocity updates)")
    line = {"impl": "reference", "metric": METRIC, "value": ups, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded, pdg_inputs)",
            "config": dict(config_block(cfg, args.gpus),
                           oracle_timed_on=f"{N_sub}^{cfg.dim}-cell sub-box of this workload per step "
                                           f"({sub.updates_per_step} node.velocity updates); value is per-update "
                                           f"throughput, comparable with the product arm's"),
            "cpu_baseline": {"value": ups, "unit": UNIT, "cores": omp_threads(), "kind": "oracle", "sample": sample},
            "e2e": {"value": ups, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)


def oracle_config_timing(key, steps):
    """One child process: `steps` oracle M2 steps of BASELINE config `key` at full size."""
    from pdg_inputs import CONFIGS
    cfg = CONFIGS[key]
    sub, pb, fc, fbc, _ = oracle_prepare(cfg, cfg.N)
    t0 = time.perf_counter()
    for _ in range(steps):
        oracle_step(pb, fc, fbc)
    dt = time.perf_counter() - t0
    return {"config": cfg.name, "steps": steps, "seconds": dt, "updates_per_s": cfg.updates_per_step * steps / dt}


def run_oracle_table(args):
    """the oracle on configs 1-3 at full size, single-thread and on all host cores
    (each in a child process with OMP_NUM_THREADS set), one JSON line."""
    model, ram = host_info()
    rows = []
    for key, steps in ((1, 100), (2, 2), (3, 1)):
        for threads in (1, os.cpu_count()):
            code = ("import sys, json; sys.path.insert(0, %r); import bench; "
                    "print(json.dumps(bench.oracle_config_timing(%d, %d)))") % (ROOT, key, steps)
            env = dict(os.environ, OMP_NUM_THREADS=str(threads))
            out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=1800)
            r = json.loads(out.stdout.strip().splitlines()[-1])
            r["threads"] = threads
            rows.append(r)
    print(json.dumps({"oracle_table": rows, "cpu_model": model, "ram_gb": ram, "cores": os.cpu_count()}), flush=True)


def config_block(cfg, G, decomp="velocity", spr=1):
    return {"workload": cfg.name, "dim": cfg.dim, "cells_per_axis": cfg.N, "degree": cfg.p, "m": cfg.m,
            "nv": cfg.nv, "lambda": cfg.lam, "dt": cfg.dt, "nodes": cfg.nnodes,
            "updates_per_step": cfg.updates_per_step, "f_bytes": 8 * cfg.nv * cfg.nnodes,
            "l2": "inputs larger than L2 (f = %.1f GB >> 126 MB); no flush" % (8e-9 * cfg.nv * cfg.nnodes)
            if 8 * cfg.nv * cfg.nnodes > 4 * 126e6 else "f fits in L2: HBM fraction not meaningful",
            "parallelism": (f"velocity-sharded x{G}" + (" + NCCL allreduce of w" if G > 1 else "")) if decomp == "velocity"
            else f"z-slab x{G} ({spr} slab(s)/rank) + NCCL all-gather of carry planes",
            "scheme": "M2 = T2(dt/2) C2(dt) T2(dt/2), consecutive half-steps swept in one pass"}


# ----------------------------------------------------------------------------
# product arm
# ----------------------------------------------------------------------------
def fill_w0(cfg, w_flat, device, sizes=None):
    """Seeded w0 of this rank's node planes (all of them unless z-slab decomposed), generated
    in slabs straight into w_flat ([m][local nodes])."""
    import torch
    from pdg_inputs import w0_grid
    L = cfg.N * cfg.n
    p0 = 0 if sizes is None else int(sizes.cell_begin) * cfg.n
    p1 = L if sizes is None else (int(sizes.cell_begin) + int(sizes.cell_count)) * cfg.n
    shape = (cfg.m, p1 - p0) + cfg.grid_shape[1:]
    w = w_flat.view(shape)
    if cfg.dim == 2:
        w.copy_(w0_grid(cfg, device=device)[:, p0:p1])
        return
    slab = max(1, min(L, (1 << 25) // (L * L)))
    for z0 in range(p0, p1, slab):
        z1 = min(p1, z0 + slab)
        w[:, z0 - p0:z1 - p0].copy_(w0_grid(cfg, device=device, zslab=(z0, z1)))
    torch.cuda.synchronize(device)


def run_product(args, cfg):
    import torch
    import torch.distributed as dist

    from paper_1702_00169_b200 import dist as pdist
    from paper_1702_00169_b200 import pdg

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    launched = "RANK" in os.environ and "MASTER_ADDR" in os.environ  # torchrun (any world size)
    if launched:
        dist.init_process_group("nccl", device_id=device)
    stream = torch.cuda.Stream(device)
    with torch.cuda.stream(stream):
        decomp = {"velocity": pdg.PDG_DECOMP_VELOCITY, "zslab": pdg.PDG_DECOMP_ZSLAB}[args.decomp]
        flags = pdg.PDG_PROFILE | (0 if args.no_e2e else pdg.PDG_ASYNC_HOST) | (pdg.PDG_NO_TMA if args.no_tma else 0) | (pdg.PDG_NO_SMALL if args.no_small else 0)
        plan = {}
        if args.lattice_cta:
            plan["lattice_cta"] = tuple(int(x) for x in args.lattice_cta.split(","))
        if args.lattice_segment:
            plan["lattice_segment"] = args.lattice_segment
        S = pdist.sharded_solver(cfg, device, flags=flags, stream=stream.cuda_stream,
                                 decomposition=decomp, slabs_per_rank=args.slabs_per_rank, **plan)
        fill_w0(cfg, S.w, device, S.sizes)
        S.set_equilibrium(S.w)
        # the timed region runs as a user's call does: no per-launch events (they are recorded in a
        # separate profiled pass below), pdg_step(K) replaying the CUDA graph of its launch sequence
        # that an earlier call with the same K captured (include/pdg.h pdg_step)
        S.profile_enable(False)
        S.step(args.warmup)
        if world == 1:
            S.step(args.steps)  # untimed: captures the K-step graph the timed call replays
        # the timed steps start again from the initial state: they stay inside the configuration's
        # physical horizon (configs 2-5 as written go non-physical after tens of steps)
        fill_w0(cfg, S.w, device, S.sizes)
        S.set_equilibrium(S.w)
        stream.synchronize()
        if launched:
            dist.barrier()
        clocks = ClockSampler(local)
        clocks.start()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(device)
        e0.record(stream)
        S.step(args.steps)
        e1.record(stream)
        torch.cuda.synchronize(device)
        ms = e0.elapsed_time(e1)
        clk = clocks.stop()
        if launched:
            dist.barrier()
        # profiled pass (untimed for the headline): per-launch CUDA events of the same K steps, for the
        # kernel table and the roofline fractions
        # non-physical states reached by the timed steps (parity protocol item 4): rho <= 0 or non-finite f
        bad = S.check_state()
        bad = int(pdist.sum_over_ranks(float(bad), device=device)) if launched else bad
        fill_w0(cfg, S.w, device, S.sizes)
        S.set_equilibrium(S.w)
        S.profile_enable(True)
        S.profile_read()
        S.step(args.steps)
        prof = S.profile_read()
        S.profile_enable(False)
        ms = pdist.max_over_ranks(ms, device=device)
        value = cfg.updates_per_step * args.steps / (ms * 1e-3)

        # dominant kernel roofline (per launch = its algorithmic bytes / its event time)
        peak, peak_src = peaks()
        dom = max((k for k in prof if prof[k][1] > 0 and k != "allreduce"), key=lambda k: prof[k][0])
        dms, dn, db = prof[dom]
        achieved = db / (dms * 1e-3) / 1e9
        launches = int(sum(v[1] for k, v in prof.items() if k != "allreduce"))
        kernels = {k: {"ms_total": v[0], "launches": v[1], "alg_GB": v[2] / 1e9,
                       "GB_per_s": (v[2] / (v[0] * 1e-3) / 1e9) if v[0] > 0 else None} for k, v in prof.items()
                   if v[1] > 0}
        traffic, traffic_src = ncu_traffic(cfg, dom)
        # whole-step roofline: the algorithmic bytes every launch of the timed region must move (the
        # fused schedule: one pass [C + 2 x-sweeps] over all velocities and one [2 y/z-sweeps] pass per
        # step, plus the run's leading T2 and the inflow planes), over the step time, against HBM
        sched = sum(v[2] for k, v in prof.items() if k != "allreduce")
        sched_ach = sched / (ms * 1e-3) / 1e9
        step_roof = {"bound": "hbm", "alg_bytes_per_step": sched / args.steps, "achieved": sched_ach, "peak": peak,
                     "unit": "GB/s", "frac": sched_ach / peak,
                     "bytes": "sum of the algorithmic bytes of every launch in the timed region (16 B per "
                              "node.velocity per pass over f + inflow planes + z-slab carries)"}
        if cfg.lattice:
            # whole-step HBM roofline of a lattice workload: per node and velocity, 16 B for the
            # relaxation plus 16 B per pass over f that the path needs at least (axis velocities and
            # 3-D two-axis classes: both half-steps can share one pass; body diagonals and 2-D
            # diagonals: one pass each).  Algorithmic bytes: the 3-D two-axis classes now run one
            # launch per half-step (measured faster), which moves more than this.
            vel, _ = cfg.velocities()
            b = 0.0
            for v in vel:
                na = sum(1 for x in v[:cfg.dim] if x != 0)
                b += 16.0 + (0.0 if na == 0 else (16.0 if (na == 1 or (na == 2 and cfg.dim == 3)) else 32.0))
            alg = b * cfg.nnodes
            ach = alg / (ms / args.steps * 1e-3) / 1e9
            step_roof["min_passes_model"] = {
                "alg_bytes_per_step": alg, "achieved": ach, "frac": ach / peak,
                "note": "minimum passes the lattice path needs; lattice classes run concurrently on forked "
                        "streams, so per-kernel event times overlap; this is the whole step against HBM"}
        roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                    "traffic": traffic, "traffic_source": traffic_src, "kernel": dom, "peak_source": peak_src,
                    "alg_bytes_per_launch": db / dn}

        # end to end through the C-ABI with host buffers
        e2e = None
        if not args.no_e2e:
            n_e2e = max(1, min(args.steps, args.e2e_steps))
            w_host = torch.empty(S.sizes.w_elems, dtype=torch.float64, pin_memory=True)
            w_out = torch.empty(S.sizes.w_elems, dtype=torch.float64, pin_memory=True)
            fill_w0(cfg, S.w, device, S.sizes)
            w_host.copy_(S.w)
            torch.cuda.synchronize(device)
            if launched:
                dist.barrier()
            t0 = time.perf_counter()
            a0 = torch.cuda.Event(enable_timing=True)
            a1 = torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            for _ in range(n_e2e):
                S.set_equilibrium(w_host)       # H2D of the step's input (pinned host)
                S.step(1)
                S.moments(w_out)                # D2H of the step's result (library copy stream)
            S.synchronize()                     # PDG_ASYNC_HOST: every copy of the loop has landed
            a1.record(stream)
            torch.cuda.synchronize(device)
            ems = a0.elapsed_time(a1)
            wall = time.perf_counter() - t0
            ems = pdist.max_over_ranks(ems, device=device)
            e2e = {"value": cfg.updates_per_step * n_e2e / (ems * 1e-3), "unit": UNIT,
                   "h2d_bytes_per_step": int(8 * S.sizes.w_elems), "d2h_bytes_per_step": int(8 * S.sizes.w_elems),
                   "steps": n_e2e, "ms_per_step": ems / n_e2e, "wall_s": wall,
                   "call": "pdg_set_equilibrium(host w0) + pdg_step(1) + pdg_moments(host w) per step, "
                           "PDG_ASYNC_HOST (upload of step k+1 overlaps the download of step k; timed to "
                           "pdg_synchronize)"}
            S.profile_read()
            del w_host, w_out


        cpu = None
        if world == 1 and rank == 0 and not args.no_cpu_baseline:
            cpu = cpu_baseline(cfg, args.cpu_cells)

        S.destroy()
        # several ranks: also time the other decomposition (velocity sharding is the north star's
        # partition, the exact z-slab decomposition the scalable one; both exact)
        alt = None
        if world > 1 and not args.lattice and not args.one_decomp:
            other = "velocity" if args.decomp == "zslab" else "zslab"
            T = pdist.sharded_solver(cfg, device, flags=pdg.PDG_PROFILE, stream=stream.cuda_stream,
                                     decomposition={"velocity": pdg.PDG_DECOMP_VELOCITY,
                                                    "zslab": pdg.PDG_DECOMP_ZSLAB}[other],
                                     slabs_per_rank=1)
            fill_w0(cfg, T.w, device, T.sizes)
            T.set_equilibrium(T.w)
            T.step(args.warmup)
            T.profile_read()
            torch.cuda.synchronize(device)
            dist.barrier()
            a0 = torch.cuda.Event(enable_timing=True)
            a1 = torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            T.step(args.steps)
            a1.record(stream)
            torch.cuda.synchronize(device)
            oms = pdist.max_over_ranks(a0.elapsed_time(a1), device=device)
            oprof = T.profile_read()
            T.destroy()
            alt = {"decomposition": other, "value": cfg.updates_per_step * args.steps / (oms * 1e-3),
                   "unit": UNIT, "ms_per_step": oms / args.steps,
                   "parallelism": config_block(cfg, world, other, 1)["parallelism"],
                   "kernels": {k: {"ms_total": v[0], "launches": v[1]} for k, v in oprof.items() if v[1] > 0}}

        if rank == 0:
            line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                    "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
                    "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                    "data": "synthetic (seeded pdg_inputs recipe of the config)",
                    "config": config_block(cfg, world, args.decomp, args.slabs_per_rank), "roofline": roofline,
                    "cpu_baseline": cpu, "e2e": e2e,
                    "gpu_launches": launches, "clocks": clk, "kernels": kernels, "step_roofline": step_roof,
                    "nonphysical_nodes": bad,
                    "updates_vs_48B_model": value * 48.0 / (peak * 1e9 * world),
                    "updates_vs_48B_model_note": "updates/s x 48 B (SURVEY 8(d) three-pass model) / (HBM peak x "
                                                 "GPUs); exceeds 1 because consecutive half-steps share a pass: "
                                                 "a throughput ratio, not a roofline fraction"}
            if alt is not None:
                line["alt_decomposition"] = alt
            print(json.dumps(line), flush=True)
    if launched:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--impl", default="product", choices=["product", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-cells", type=int, default=128, help="cells per axis of the oracle's timed sub-box")
    ap.add_argument("--ref-cells", type=int, default=32)
    ap.add_argument("--decomp", default=None, choices=["velocity", "zslab"],
                    help="multi-GPU decomposition (default: zslab when launched on several ranks)")
    ap.add_argument("--slabs-per-rank", type=int, default=1)
    ap.add_argument("--oracle-table", action="store_true",
                    help="time the CPU oracle on configs 1-3 at full size (1 thread and all cores) and exit")
    ap.add_argument("--no-small", action="store_true",
                    help="small problems: the general per-operator kernels instead of one CTA with f in shared memory (PDG_NO_SMALL)")
    ap.add_argument("--no-tma", action="store_true",
                    help="register-staged collision + x-sweep pass instead of bulk-copy staging (PDG_NO_TMA)")
    ap.add_argument("--one-decomp", action="store_true",
                    help="several ranks: time only --decomp (default: also the other decomposition)")
    ap.add_argument("--lattice", default=None, choices=["D2Q9", "D3Q15", "D3Q19", "D3Q27"],
                    help="NEXT-2 workload: isothermal LBM on this lattice (replaces --config)")
    ap.add_argument("--cells", type=int, default=128, help="cells per axis of the --lattice workload")
    ap.add_argument("--lattice-cta", default=None, help="forced lattice CTA shape 'wx,wy' (pdg_problem.lattice_cta)")
    ap.add_argument("--lattice-segment", type=int, default=0,
                    help="forced lattice chain-segment rows (pdg_problem.lattice_segment; < 0: none)")
    ap.add_argument("--degree", type=int, default=2, help="degree p of the --lattice workload")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "product":
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)
    from pdg_inputs import CONFIGS, lbm_config
    cfg = lbm_config(args.lattice, args.cells, p=args.degree, nu=2.0) if args.lattice else CONFIGS[args.config]
    if args.lattice:
        args.cpu_cells = min(args.cpu_cells, 64 if cfg.dim == 3 else 512)
        args.ref_cells = min(args.ref_cells, 16 if cfg.dim == 3 else 128)
    if args.decomp is None:  # the z-slab decomposition is implemented for axis-aligned sets only
        args.decomp = "zslab" if int(os.environ.get("WORLD_SIZE", "1")) > 1 and not args.lattice else "velocity"
    if args.oracle_table:
        run_oracle_table(args)
    elif args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_product(args, cfg)


if __name__ == "__main__":
    main()
