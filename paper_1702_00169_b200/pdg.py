"""Thin ctypes binding of libpdg (include/pdg.h): argument marshalling only.

Every arithmetic step of the hot path runs in the sm_100a kernels behind the
C-ABI.  PyTorch is used for device memory, the CUDA stream and (multi-GPU)
process groups.  There is no CPU fallback: without the built extension or a
CUDA device every entry point raises.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# PDG_CHECKED=1 selects the bounds-checked build of the same library (build.py --checked)
LIB_PATH = os.path.join(_HERE, "libpdg_checked.so" if os.environ.get("PDG_CHECKED") == "1" else "libpdg.so")

# status codes (include/pdg.h)
PDG_OK = 0
PDG_E_INVALID_ARGUMENT = 1
PDG_E_DIMENSION = 2
PDG_E_DEGREE = 3
PDG_E_VELOCITY_SET = 4
PDG_E_FLUX_MODEL = 5
PDG_E_STATE_NOT_SET = 6
PDG_E_NONPHYSICAL = 7
PDG_E_CUDA = 8
PDG_E_NCCL = 9
PDG_E_BUFFER = 10
PDG_E_UNSUPPORTED = 11

PDG_FLUX_LINEAR_ADVECTION = 0
PDG_FLUX_EULER = 1
PDG_FLUX_ISOTHERMAL = 2
PDG_FLUX_LBM = 3
PDG_SCHEME_M2 = 0
PDG_SCHEME_M2KIN = 1
PDG_SCHEME_M4 = 2
PDG_SCHEME_M2S = 3
PDG_SOURCE_NONE = 0
PDG_SOURCE_GRAVITY = 1
PDG_CHECK_STATE = 0x1
PDG_SYNC_ERRORS = 0x2
PDG_NO_FUSION = 0x4
PDG_PROFILE = 0x8
PDG_ASYNC_HOST = 0x10
PDG_NO_TMA = 0x20
PDG_NO_GRAPH = 0x40
PDG_NO_SMALL = 0x80
KERNEL_KINDS = ["sweep_strided", "sweep_x", "relax", "partial_moments", "relax_from_w", "allreduce", "other",
                "relax_xsweep", "zslab", "lattice", "small_run"]
PDG_DECOMP_VELOCITY = 0
PDG_DECOMP_ZSLAB = 1

EXPORTED = [
    "pdg_query_sizes", "pdg_create", "pdg_set_state", "pdg_set_equilibrium", "pdg_get_state", "pdg_step",
    "pdg_transport", "pdg_collide", "pdg_source", "pdg_partial_moments", "pdg_relax_from_w", "pdg_moments",
    "pdg_check_state", "pdg_cell_block", "pdg_synchronize", "pdg_destroy", "pdg_nccl_unique_id",
    "pdg_status_string", "pdg_last_error", "pdg_version", "pdg_profile_read", "pdg_zslab_table",
    "pdg_profile_enable",
]


class pdg_problem(ctypes.Structure):
    _fields_ = [
        ("dim", ctypes.c_int32), ("ncell", ctypes.c_int64 * 3), ("lo", ctypes.c_double * 3),
        ("hi", ctypes.c_double * 3), ("degree", ctypes.c_int32), ("m", ctypes.c_int32), ("nv", ctypes.c_int32),
        ("vel", ctypes.POINTER(ctypes.c_double)), ("comp", ctypes.POINTER(ctypes.c_int32)),
        ("lam", ctypes.c_double), ("flux", ctypes.c_int32), ("flux_params", ctypes.POINTER(ctypes.c_double)),
        ("n_flux_params", ctypes.c_int32), ("tau", ctypes.c_double), ("dt", ctypes.c_double),
        ("scheme", ctypes.c_int32), ("rank", ctypes.c_int32), ("nranks", ctypes.c_int32),
        ("nccl_id", ctypes.c_void_p), ("cuda_stream", ctypes.c_void_p), ("flags", ctypes.c_uint32),
        ("decomposition", ctypes.c_int32), ("slabs_per_rank", ctypes.c_int32),
        ("source", ctypes.c_int32), ("source_params", ctypes.POINTER(ctypes.c_double)),
        ("n_source_params", ctypes.c_int32),
        ("lattice_cta", ctypes.c_int32 * 2), ("lattice_segment", ctypes.c_int32),
    ]


class pdg_sizes(ctypes.Structure):
    _fields_ = [("f_elems", ctypes.c_size_t), ("fb_elems", ctypes.c_size_t), ("w_elems", ctypes.c_size_t),
                ("work_bytes", ctypes.c_size_t), ("nnodes", ctypes.c_int64), ("plane_stride", ctypes.c_int64),
                ("nv_local", ctypes.c_int32), ("v_begin", ctypes.c_int32), ("nnodes_local", ctypes.c_int64),
                ("cell_begin", ctypes.c_int64), ("cell_count", ctypes.c_int64)]


class PdgError(RuntimeError):
    def __init__(self, status, where, detail):
        super().__init__(f"{where}: {status_string(status)} ({detail})")
        self.status = status


_lib = None


def load() -> ctypes.CDLL:
    """Load the in-tree libpdg.so; raise if it is missing (no silent fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
    P = ctypes.POINTER
    d, i64, vp, st = ctypes.c_double, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int
    pd = P(d)
    ctx = vp
    sig = {
        "pdg_query_sizes": ([P(pdg_problem), P(pdg_sizes)], st),
        "pdg_create": ([P(pdg_problem), vp, vp, vp, vp, P(ctx)], st),
        "pdg_set_state": ([ctx, vp, vp, ctypes.c_int], st),
        "pdg_set_equilibrium": ([ctx, vp, vp, ctypes.c_int], st),
        "pdg_get_state": ([ctx, vp, ctypes.c_int], st),
        "pdg_step": ([ctx, i64], st),
        "pdg_transport": ([ctx, d], st),
        "pdg_collide": ([ctx, d], st),
        "pdg_source": ([ctx, d], st),
        "pdg_partial_moments": ([ctx], st),
        "pdg_relax_from_w": ([ctx, d], st),
        "pdg_moments": ([ctx, vp, ctypes.c_int], st),
        "pdg_check_state": ([ctx, P(i64)], st),
        "pdg_cell_block": ([ctx, ctypes.c_int, d, pd, pd, pd], st),
        "pdg_synchronize": ([ctx], st),
        "pdg_destroy": ([ctx], None),
        "pdg_nccl_unique_id": ([vp], st),
        "pdg_status_string": ([st], ctypes.c_char_p),
        "pdg_last_error": ([], ctypes.c_char_p),
        "pdg_version": ([], ctypes.c_char_p),
        "pdg_profile_read": ([ctx, pd, P(i64), pd], st),
        "pdg_profile_enable": ([ctx, ctypes.c_int], st),
        "pdg_zslab_table": ([P(pdg_problem), d, ctypes.c_int, i64, pd, pd, pd, pd, P(ctypes.c_int32)], st),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _lib = L
    return L


def status_string(s: int) -> str:
    return load().pdg_status_string(s).decode()


def last_error() -> str:
    return load().pdg_last_error().decode()


def _check(status: int, where: str):
    if status != PDG_OK:
        raise PdgError(status, where, last_error())


def version() -> str:
    return load().pdg_version().decode()


def make_problem(dim, ncell, degree, m, vel, comp, lam, flux, flux_params, dt, tau=0.0, scheme=PDG_SCHEME_M2,
                 rank=0, nranks=1, nccl_id=None, stream=None, flags=0, lo=(0.0, 0.0, 0.0), hi=(1.0, 1.0, 1.0),
                 decomposition=PDG_DECOMP_VELOCITY, slabs_per_rank=1, gravity=None, lattice_cta=(0, 0),
                 lattice_segment=0):
    """Build a pdg_problem; the returned object keeps its host arrays alive."""
    pb = pdg_problem()
    pb.dim = dim
    nc = [ncell] * dim if isinstance(ncell, int) else list(ncell)
    for d in range(3):
        pb.ncell[d] = nc[d] if d < dim else 1
        pb.lo[d] = lo[d]
        pb.hi[d] = hi[d]
    pb.degree, pb.m = degree, m
    flat = [float(x) for v in vel for x in (list(v) + [0.0] * (3 - len(v)))[:3]]
    pb.nv = len(vel)
    pb._vel = (ctypes.c_double * len(flat))(*flat)
    pb._comp = (ctypes.c_int32 * len(comp))(*comp)
    pb._fp = (ctypes.c_double * max(1, len(flux_params)))(*flux_params)
    pb.vel = ctypes.cast(pb._vel, ctypes.POINTER(ctypes.c_double))
    pb.comp = ctypes.cast(pb._comp, ctypes.POINTER(ctypes.c_int32))
    pb.lam, pb.flux = lam, flux
    pb.flux_params = ctypes.cast(pb._fp, ctypes.POINTER(ctypes.c_double))
    pb.n_flux_params = len(flux_params)
    pb.tau, pb.dt, pb.scheme = tau, dt, scheme
    pb.rank, pb.nranks = rank, nranks
    if nccl_id is not None:
        pb._id = ctypes.create_string_buffer(bytes(nccl_id), 128)
        pb.nccl_id = ctypes.cast(pb._id, ctypes.c_void_p)
    pb.cuda_stream = stream
    pb.flags = flags
    pb.decomposition = decomposition
    pb.slabs_per_rank = slabs_per_rank
    pb.lattice_cta[0], pb.lattice_cta[1] = int(lattice_cta[0]), int(lattice_cta[1])
    pb.lattice_segment = int(lattice_segment)
    if gravity:
        pb._src = (ctypes.c_double * len(gravity))(*gravity)
        pb.source = PDG_SOURCE_GRAVITY
        pb.source_params = ctypes.cast(pb._src, ctypes.POINTER(ctypes.c_double))
        pb.n_source_params = len(gravity)
    return pb


def query_sizes(pb: pdg_problem) -> pdg_sizes:
    out = pdg_sizes()
    _check(load().pdg_query_sizes(ctypes.byref(pb), ctypes.byref(out)), "pdg_query_sizes")
    return out


def zslab_table(pb: pdg_problem, dtp: float, npass: int, length: int):
    """(P [len][n], Q [len][n], B, C, leff): the z-slab carry tables (pdg_zslab_table, host-only)."""
    n = pb.degree + 1
    P_ = (ctypes.c_double * (length * n))()
    Q_ = (ctypes.c_double * (length * n))()
    B_, C_, le = ctypes.c_double(), ctypes.c_double(), ctypes.c_int32()
    _check(load().pdg_zslab_table(ctypes.byref(pb), float(dtp), int(npass), int(length), P_, Q_, ctypes.byref(B_),
                                  ctypes.byref(C_), ctypes.byref(le)), "pdg_zslab_table")
    rows = lambda a: [list(a[i * n:(i + 1) * n]) for i in range(length)]  # noqa: E731
    return rows(P_), rows(Q_), B_.value, C_.value, le.value


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(load().pdg_nccl_unique_id(buf), "pdg_nccl_unique_id")
    return buf.raw


def _ptr(t) -> int:
    return t.data_ptr()


class Solver:
    """One libpdg context on the current CUDA device with torch-owned buffers.

    Methods map 1:1 onto the C-ABI (same names without the pdg_ prefix)."""

    def __init__(self, pb: pdg_problem, device=None):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("libpdg needs a CUDA device (no CPU fallback)")
        self.torch = torch
        self.lib = load()
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        if pb.cuda_stream is None:
            pb.cuda_stream = torch.cuda.current_stream(self.device).cuda_stream
        self.pb = pb
        self.sizes = query_sizes(pb)
        s = self.sizes
        kw = dict(dtype=torch.float64, device=self.device)
        self.f = torch.empty(s.f_elems, **kw)
        self.fb = torch.zeros(max(1, s.fb_elems), **kw)
        self.w = torch.empty(s.w_elems, **kw)
        self.work = torch.zeros(max(64, s.work_bytes // 8), **kw)
        self.ctx = ctypes.c_void_p()
        self._keep = []
        with torch.cuda.device(self.device):  # the context records the current device
            _check(self.lib.pdg_create(ctypes.byref(pb), _ptr(self.f), _ptr(self.fb), _ptr(self.w),
                                       _ptr(self.work), ctypes.byref(self.ctx)), "pdg_create")

    # --- state ---------------------------------------------------------------
    def set_state(self, f=None, fb=None):
        """f, fb: torch tensors (both on the device or both on the host) in the canonical layout."""
        if f is None and fb is None:
            return
        if f is not None and fb is not None and f.is_cuda != fb.is_cuda:
            raise ValueError("f and fb must both be device or both be host tensors")
        on_dev = int((f if f is not None else fb).is_cuda)
        # contiguous copies bound to locals: they must outlive the (possibly asynchronous) copy
        if f is not None:
            assert f.numel() == self.sizes.f_elems and f.dtype == self.torch.float64
            f = f.contiguous()
        if fb is not None:
            assert fb.numel() == self.sizes.fb_elems and fb.dtype == self.torch.float64
            fb = fb.contiguous()
        fp = _ptr(f) if f is not None else None
        fbp = _ptr(fb) if fb is not None else None
        _check(self.lib.pdg_set_state(self.ctx, fp, fbp, on_dev), "pdg_set_state")
        self._keep_until_sync(on_dev, f, fb)

    def _keep_until_sync(self, on_dev, *tensors):
        # PDG_ASYNC_HOST: a host-input call returns before its copy ran; keep the (pinned) sources
        # alive until the next pdg_synchronize.  Device inputs are ordered on the context stream.
        if not on_dev and (self.pb.flags & PDG_ASYNC_HOST):
            self._keep.append(tensors)

    def set_equilibrium(self, w, wb=None):
        assert w.numel() == self.sizes.w_elems and w.dtype == self.torch.float64
        w = w.contiguous()
        wbp = None
        if wb is not None:
            wb = wb.contiguous()
            assert wb.numel() == self.sizes.w_elems and wb.is_cuda == w.is_cuda
            wbp = _ptr(wb)
        _check(self.lib.pdg_set_equilibrium(self.ctx, _ptr(w), wbp, int(w.is_cuda)), "pdg_set_equilibrium")
        self._keep_until_sync(int(w.is_cuda), w, wb)

    def get_state(self, out=None):
        if out is None:
            out = self.torch.empty(self.sizes.f_elems, dtype=self.torch.float64, device=self.device)
        _check(self.lib.pdg_get_state(self.ctx, _ptr(out), int(out.is_cuda)), "pdg_get_state")
        return out

    # --- hot path --------------------------------------------------------------
    def step(self, nsteps: int = 1):
        _check(self.lib.pdg_step(self.ctx, int(nsteps)), "pdg_step")

    def transport(self, dtp: float):
        _check(self.lib.pdg_transport(self.ctx, float(dtp)), "pdg_transport")

    def collide(self, dt: float):
        _check(self.lib.pdg_collide(self.ctx, float(dt)), "pdg_collide")

    def source(self, h: float):
        _check(self.lib.pdg_source(self.ctx, float(h)), "pdg_source")

    def partial_moments(self):
        _check(self.lib.pdg_partial_moments(self.ctx), "pdg_partial_moments")

    def relax_from_w(self, dt: float):
        _check(self.lib.pdg_relax_from_w(self.ctx, float(dt)), "pdg_relax_from_w")

    def moments(self, out=None):
        if out is None:
            out = self.torch.empty(self.sizes.w_elems, dtype=self.torch.float64, device=self.device)
        _check(self.lib.pdg_moments(self.ctx, _ptr(out), int(out.is_cuda)), "pdg_moments")
        return out

    def check_state(self) -> int:
        n = ctypes.c_int64(0)
        _check(self.lib.pdg_check_state(self.ctx, ctypes.byref(n)), "pdg_check_state")
        return n.value

    def cell_block(self, axis: int, dtp: float):
        n = self.pb.degree + 1
        M = (ctypes.c_double * (n * n))()
        g = (ctypes.c_double * n)()
        beta = ctypes.c_double()
        _check(self.lib.pdg_cell_block(self.ctx, axis, dtp, M, g, ctypes.byref(beta)), "pdg_cell_block")
        return [list(M[i * n:(i + 1) * n]) for i in range(n)], list(g), beta.value

    def profile_read(self):
        """{kind: (ms, launches, algorithmic_bytes)} since the last read (needs PDG_PROFILE)."""
        k = len(KERNEL_KINDS)
        ms = (ctypes.c_double * k)()
        n = (ctypes.c_int64 * k)()
        b = (ctypes.c_double * k)()
        _check(self.lib.pdg_profile_read(self.ctx, ms, n, b), "pdg_profile_read")
        return {KERNEL_KINDS[i]: (ms[i], n[i], b[i]) for i in range(k)}

    def profile_enable(self, on: bool):
        """Pause / resume the PDG_PROFILE per-launch events (paused: graph replay allowed)."""
        _check(self.lib.pdg_profile_enable(self.ctx, int(bool(on))), "pdg_profile_enable")

    def synchronize(self):
        _check(self.lib.pdg_synchronize(self.ctx), "pdg_synchronize")
        self._keep.clear()

    def destroy(self):
        if getattr(self, "ctx", None) is not None and self.ctx.value:
            self.lib.pdg_destroy(self.ctx)
            self.ctx = ctypes.c_void_p()

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


def problem_from_config(cfg, tau=0.0, scheme=PDG_SCHEME_M2, rank=0, nranks=1, nccl_id=None, flags=0, stream=None,
                        decomposition=PDG_DECOMP_VELOCITY, slabs_per_rank=1, lattice_cta=(0, 0), lattice_segment=0):
    """pdg_problem for a pdg_inputs.Config (the seeded workload descriptions)."""
    vel, comp = cfg.velocities()
    return make_problem(cfg.dim, cfg.N, cfg.p, cfg.m, vel, comp, cfg.lam, cfg.flux, list(cfg.flux_params()), cfg.dt,
                        tau=tau, scheme=scheme, rank=rank, nranks=nranks, nccl_id=nccl_id, flags=flags,
                        stream=stream, lo=cfg.lo, hi=cfg.hi, decomposition=decomposition,
                        slabs_per_rank=slabs_per_rank, gravity=getattr(cfg, "gravity", None) or None,
                        lattice_cta=lattice_cta, lattice_segment=lattice_segment)
