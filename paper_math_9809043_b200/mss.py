"""Thin ctypes binding of ``libmss.so`` (include/mss.h): argument marshalling only.

Every step of the solver runs in the library's CUDA kernels.  PyTorch supplies device
memory (float64 CUDA tensors) and the current CUDA stream; nothing here computes.
If the library is missing this module raises — there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import List, Optional, Sequence

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libmss.so")

MSS_OK = 0
MSS_NOT_CONVERGED = 1
MAX_LEVELS = 12

NEUMANN = 0
DIRICHLET = 1


class MSSError(RuntimeError):
    def __init__(self, code, where, detail=""):
        super().__init__(f"{where}: status {code} ({detail})")
        self.code = code


class BC(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("value", ctypes.c_double)]


class Params(ctypes.Structure):
    _fields_ = [
        ("scale", ctypes.c_int),
        ("m", ctypes.c_int),
        ("f", ctypes.c_double),
        ("interp", ctypes.c_int),
        ("max_iter", ctypes.c_int),
        ("coarse_min", ctypes.c_int),
        ("use_lift", ctypes.c_int),
        ("tail_cells", ctypes.c_int64),
        ("gather_below", ctypes.c_int64),
        ("method", ctypes.c_int),
        ("splitting", ctypes.c_int),
        ("dims_mode", ctypes.c_int),
        ("n_level_dims", ctypes.c_int),
        ("level_dims", (ctypes.c_int64 * 3) * MAX_LEVELS),
        ("log_events", ctypes.c_int),
    ]

METHODS = {"multiscale": 0, "tatebe": 1, "polynomial": 2, "multigrid": 3}


class Info(ctypes.Structure):
    _fields_ = [
        ("levels", ctypes.c_int),
        ("dims", (ctypes.c_int64 * 3) * MAX_LEVELS),
        ("iters", ctypes.c_int64 * MAX_LEVELS),
        ("calls", ctypes.c_int64 * MAX_LEVELS),
        ("not_converged", ctypes.c_int),
        ("breakdown_level", ctypes.c_int),
        ("true_rel_res", ctypes.c_double),
        ("bnorm2", ctypes.c_double),
        ("kernel_launches", ctypes.c_int64),
        ("tail_level", ctypes.c_int),
        ("tail_kind", ctypes.c_int),
        ("setup_ms", ctypes.c_double),
        ("setup_coarsest_ms", ctypes.c_double),
        ("graph", ctypes.c_int),
    ]


class FieldParams(ctypes.Structure):
    """mss_field_params (include/mss.h, NEXT-4)."""
    _fields_ = [("model", ctypes.c_int), ("ell", ctypes.c_double * 3), ("theta", ctypes.c_double),
                ("log_mean", ctypes.c_double), ("log_var", ctypes.c_double), ("seed", ctypes.c_uint64)]


P = ctypes.c_void_p
I64P = ctypes.POINTER(ctypes.c_int64)
DP = ctypes.POINTER(ctypes.c_double)

# (name, restype, argtypes) for every symbol include/mss.h declares.
SIGNATURES = [
    ("mss_field_generate", ctypes.c_int, [ctypes.c_int, I64P, ctypes.POINTER(FieldParams), P, P]),
    ("mss_manufacture_rhs", ctypes.c_int, [P, P, P]),
    ("mss_default_params", ctypes.c_int, [ctypes.POINTER(Params)]),
    ("mss_strerror", ctypes.c_char_p, [ctypes.c_int]),
    ("mss_last_error", ctypes.c_char_p, []),
    ("mss_setup", ctypes.c_int, [ctypes.POINTER(P), ctypes.c_int, I64P, DP, P, ctypes.c_int,
                                 ctypes.POINTER(BC), ctypes.c_int, ctypes.POINTER(Params), P]),
    ("mss_free", ctypes.c_int, [P]),
    ("mss_num_levels", ctypes.c_int, [P, ctypes.POINTER(ctypes.c_int)]),
    ("mss_level_dims", ctypes.c_int, [P, ctypes.c_int, I64P]),
    ("mss_solve", ctypes.c_int, [P, P, P, ctypes.c_double, I64P, DP]),
    ("mss_solve_host", ctypes.c_int, [P, P, P, ctypes.c_double, I64P, DP]),
    ("mss_solve_host_batch", ctypes.c_int, [P, ctypes.c_int, P, P, ctypes.c_double, I64P, DP]),
    ("mss_get_info", ctypes.c_int, [P, ctypes.POINTER(Info)]),
    ("mss_level_events", ctypes.c_int, [P, ctypes.POINTER(ctypes.c_int), ctypes.c_int, ctypes.POINTER(ctypes.c_int)]),
    ("mss_get_faces", ctypes.c_int, [P, ctypes.c_int, ctypes.c_int, P]),
    ("mss_apply_A", ctypes.c_int, [P, ctypes.c_int, P, P]),
    ("mss_dot", ctypes.c_int, [P, ctypes.c_int, P, P, DP]),
    ("mss_smooth", ctypes.c_int, [P, ctypes.c_int, P, P, ctypes.c_int, ctypes.c_int, ctypes.c_int]),
    ("mss_residual_restrict", ctypes.c_int, [P, ctypes.c_int, P, P, P]),
    ("mss_prolong_add", ctypes.c_int, [P, ctypes.c_int, P, P, ctypes.c_int]),
    ("mss_precond", ctypes.c_int, [P, ctypes.c_int, P, P, ctypes.c_double, I64P]),
    ("mss_coarse_solve", ctypes.c_int, [P, P, P]),
    ("mss_rhs_lift", ctypes.c_int, [P, P, P, P]),
    ("mss_cg_direction", ctypes.c_int, [P, ctypes.c_int, P, P, ctypes.c_double, ctypes.c_double, ctypes.c_int, P, P,
                                        DP]),
    ("mss_cg_update", ctypes.c_int, [P, ctypes.c_int, P, P, P, P, ctypes.c_double, ctypes.c_double, DP]),
    ("mss_residual", ctypes.c_int, [P, ctypes.c_int, P, P, P, DP]),
    ("mss_presmooth_restrict", ctypes.c_int, [P, ctypes.c_int, P, P, P]),
    ("mss_prolong_postsmooth", ctypes.c_int, [P, ctypes.c_int, P, P, P, DP]),
    ("mss_nccl_unique_id", ctypes.c_int, [ctypes.c_char_p]),
    ("mss_slab_range", ctypes.c_int, [I64P, ctypes.c_int, ctypes.POINTER(Params), ctypes.c_int, ctypes.c_int,
                                      ctypes.c_int, I64P, I64P]),
    ("mss_loopback_create", ctypes.c_int, [ctypes.c_int, ctypes.POINTER(P)]),
    ("mss_loopback_destroy", ctypes.c_int, [P]),
    ("mss_setup_loopback", ctypes.c_int, [ctypes.POINTER(P), P, ctypes.c_int, ctypes.c_int, I64P, DP, P,
                                          ctypes.c_int, ctypes.POINTER(BC), ctypes.c_int, ctypes.POINTER(Params),
                                          P]),
    ("mss_setup_dist", ctypes.c_int, [ctypes.POINTER(P), ctypes.c_int, ctypes.c_int, ctypes.c_char_p,
                                      ctypes.c_int, I64P, DP, P, ctypes.c_int, ctypes.POINTER(BC),
                                      ctypes.c_int, ctypes.POINTER(Params), P]),
    ("mss_kernel_launches", ctypes.c_int, [P, I64P]),
    ("mss_profile", ctypes.c_int, [P, ctypes.c_int, ctypes.c_int]),
    ("mss_profile_read", ctypes.c_int, [P, ctypes.c_int, ctypes.c_int, I64P, DP, DP]),
]

KCLASS = ["halfsweep", "halfsweep_first", "residual", "restrict", "prolong_add", "pdir_spmv_dot",
          "axpy_norm", "dot", "coarse_solve", "tail", "pair_sweep", "halo", "allreduce_gather"]

_lib = None


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libmss.so (raises if it was not built: no fallback path exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} not built; run `python -m paper_math_9809043_b200.build` "
                          "(or __graft_entry__.build()).  There is no CPU fallback.")
    lib = ctypes.CDLL(path)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def _check(rc, where, allow_nc=True):
    if rc == MSS_OK or (allow_nc and rc == MSS_NOT_CONVERGED):
        return rc
    lib = load_library()
    raise MSSError(rc, where, f"{lib.mss_strerror(rc).decode()}: {lib.mss_last_error().decode()}")


def _dev_ptr(t: torch.Tensor, n: Optional[int] = None) -> int:
    if not (t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
        raise ValueError("expected a contiguous float64 CUDA tensor")
    if n is not None and t.numel() != n:
        raise ValueError(f"expected {n} elements, got {t.numel()}")
    return t.data_ptr()


def default_params(**kw) -> Params:
    p = Params()
    load_library().mss_default_params(ctypes.byref(p))
    for k, v in kw.items():
        if not hasattr(p, k):
            raise KeyError(k)
        if k == "level_dims":
            for i, dd in enumerate(v):
                dd = list(dd) + [1] * (3 - len(dd))
                for a in range(3):
                    p.level_dims[i][a] = int(dd[a])
            p.n_level_dims = len(v)
            if "dims_mode" not in kw:
                p.dims_mode = 2
            continue
        setattr(p, k, v)
    return p


def slab_range(n_global, rank: int, nranks: int, params: Optional[dict] = None, depth: Optional[int] = None):
    """[z_begin, z_end) of level-0 planes owned by `rank` (mss_slab_range)."""
    lib = load_library()
    prm = default_params(**(params or {}))
    nn = (ctypes.c_int64 * 3)(*[int(v) for v in n_global])
    zb, ze = ctypes.c_int64(), ctypes.c_int64()
    _check(lib.mss_slab_range(nn, 3, ctypes.byref(prm), -1 if depth is None else int(depth), int(rank), int(nranks),
                              ctypes.byref(zb), ctypes.byref(ze)), "mss_slab_range", allow_nc=False)
    return zb.value, ze.value


def generate_field(ndim: int, n, model: int = 1, ell=(8.0, 1.0, 1.0), theta: float = 0.0, log_mean: float = 0.0,
                   log_var: float = 1.0, seed: int = 0, device=None, stream=None) -> torch.Tensor:
    """Log-normal permeability field on the device (mss_field_generate, NEXT-4):
    model 0 Gaussian, 1 power law (1 + r^T Lambda r)^(-1/4); lengths in cells; shape
    (nz, ny, nx) / (ny, nx)."""
    lib = load_library()
    nx, ny = int(n[0]), int(n[1])
    nz = int(n[2]) if ndim == 3 else 1
    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    shape = (nz, ny, nx) if ndim == 3 else (ny, nx)
    K = torch.empty(shape, dtype=torch.float64, device=dev)
    fp = FieldParams()
    fp.model = int(model)
    ell = list(ell) + [1.0] * (3 - len(ell))
    for d in range(3):
        fp.ell[d] = float(ell[d])
    fp.theta, fp.log_mean, fp.log_var, fp.seed = float(theta), float(log_mean), float(log_var), int(seed) & (2 ** 64 - 1)
    st = (stream if stream is not None else torch.cuda.current_stream(dev)).cuda_stream
    nn = (ctypes.c_int64 * 3)(nx, ny, nz)
    _check(lib.mss_field_generate(int(ndim), nn, ctypes.byref(fp), ctypes.c_void_p(K.data_ptr()), ctypes.c_void_p(st)),
           "mss_field_generate")
    return K


def nccl_unique_id() -> bytes:
    lib = load_library()
    buf = ctypes.create_string_buffer(128)
    _check(lib.mss_nccl_unique_id(buf), "mss_nccl_unique_id", allow_nc=False)
    return buf.raw


class LoopbackGroup:
    """P ranks as host threads of one process on one GPU (tests of the decomposition)."""

    def __init__(self, size: int):
        self.lib = load_library()
        self.size = size
        h = P()
        _check(self.lib.mss_loopback_create(int(size), ctypes.byref(h)), "mss_loopback_create", allow_nc=False)
        self.handle = h

    def close(self):
        if self.handle:
            self.lib.mss_loopback_destroy(self.handle)
            self.handle = None


@dataclass
class SolveReport:
    rc: int
    iters: List[int]
    calls: List[int]
    dims: List[tuple]
    not_converged: bool
    true_rel_res: float
    kernel_launches: int
    tail_level: int = -1
    tail_kind: int = 0
    setup_ms: float = 0.0
    setup_coarsest_ms: float = 0.0
    graph: bool = False


class Solver:
    """mss_setup / mss_solve / mss_free on CUDA tensors (see include/mss.h)."""

    def __init__(self, ndim: int, n: Sequence[int], K: torch.Tensor, bc, depth: Optional[int] = None,
                 params: Optional[dict] = None, extent: Optional[Sequence[float]] = None, stream=None,
                 comm=None):
        """n: global grid.  comm: None (one GPU), ("nccl", rank, nranks, id_bytes) or
        ("loop", LoopbackGroup, rank); with a comm, K is the rank's z-slab (mss_slab_range)
        and solve() takes / returns the rank's slab of f and x."""
        lib = load_library()
        self.lib = lib
        self.ndim = ndim
        nx, ny = int(n[0]), int(n[1])
        nz = int(n[2]) if ndim == 3 else 1
        self.n_global = (nx, ny, nz)
        depth_arg = -1 if depth is None else int(depth)
        prm = default_params(**(params or {}))
        self.ev_cap = int(prm.log_events)
        self.z_range = (0, nz)
        if comm is not None:
            rank = comm[2] if comm[0] == "loop" else comm[1]
            nranks = comm[1].size if comm[0] == "loop" else comm[2]
            self.z_range = slab_range((nx, ny, nz), rank, nranks, params=params, depth=depth)
        nzl = self.z_range[1] - self.z_range[0]
        self.n = (nx, ny, nzl)
        self.N = nx * ny * nzl
        if K.dim() == ndim:
            K = K.unsqueeze(0)
        K = K.contiguous()
        k_comp = K.shape[0]
        _dev_ptr(K, k_comp * self.N)
        self.stream = stream if stream is not None else torch.cuda.current_stream()
        bcs = (BC * 6)(*[BC(int(k), float(v)) for k, v in bc] + [BC(0, 0.0)] * (6 - len(bc)))
        nn = (ctypes.c_int64 * 3)(nx, ny, nz)
        ext = (ctypes.c_double * 3)(*(list(extent) + [1.0] * (3 - len(extent)))) if extent else None
        ctx = P()
        st = ctypes.c_void_p(self.stream.cuda_stream)
        if comm is None:
            rc = lib.mss_setup(ctypes.byref(ctx), ndim, nn, ext, K.data_ptr(), k_comp, bcs, depth_arg,
                               ctypes.byref(prm), st)
            where = "mss_setup"
        elif comm[0] == "loop":
            rc = lib.mss_setup_loopback(ctypes.byref(ctx), comm[1].handle, int(comm[2]), ndim, nn, ext, K.data_ptr(),
                                        k_comp, bcs, depth_arg, ctypes.byref(prm), st)
            where = "mss_setup_loopback"
        elif comm[0] == "nccl":
            idb = bytes(comm[3])
            assert len(idb) == 128
            rc = lib.mss_setup_dist(ctypes.byref(ctx), int(comm[1]), int(comm[2]), idb, ndim, nn, ext,
                                    K.data_ptr(), k_comp, bcs, depth_arg, ctypes.byref(prm), st)
            where = "mss_setup_dist"
        else:
            raise ValueError(comm)
        _check(rc, where, allow_nc=False)
        self.ctx = ctx
        L1 = ctypes.c_int()
        lib.mss_num_levels(ctx, ctypes.byref(L1))
        self.levels = L1.value

    # ---------------------------------------------------------------- lifecycle
    def close(self):
        if getattr(self, "ctx", None):
            self.lib.mss_free(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def level_dims(self, level: int):
        out = (ctypes.c_int64 * 3)()
        _check(self.lib.mss_level_dims(self.ctx, level, out), "mss_level_dims")
        return tuple(out)

    def level_N(self, level: int) -> int:
        d = self.level_dims(level)
        return d[0] * d[1] * d[2]

    def level_events(self):
        """mss_level_events: the last solve's level tree as the oracle logs it,
        [(k, "enter"), ..., (k, "leave", iterations), ...] (needs params log_events > 0)."""
        n = ctypes.c_int()
        _check(self.lib.mss_level_events(self.ctx, None, 0, ctypes.byref(n)), "mss_level_events", allow_nc=False)
        cap = min(n.value, self.ev_cap)   # the log keeps the first ev_cap events
        buf = (ctypes.c_int * (2 * max(cap, 1)))()
        _check(self.lib.mss_level_events(self.ctx, buf, cap, ctypes.byref(n)), "mss_level_events", allow_nc=False)
        out = []
        for i in range(min(cap, n.value)):
            code, it = buf[2 * i], buf[2 * i + 1]
            out.append((code >> 1, "enter") if (code & 1) == 0 else (code >> 1, "leave", it))
        return out, n.value

    def info(self) -> SolveReport:
        inf = Info()
        self.lib.mss_get_info(self.ctx, ctypes.byref(inf))
        L1 = inf.levels
        return SolveReport(0, list(inf.iters[:L1]), list(inf.calls[:L1]),
                           [tuple(inf.dims[k]) for k in range(L1)], bool(inf.not_converged),
                           inf.true_rel_res, inf.kernel_launches, inf.tail_level, inf.tail_kind,
                           inf.setup_ms, inf.setup_coarsest_ms, bool(inf.graph))

    def manufacture_rhs(self, x_exact: torch.Tensor) -> torch.Tensor:
        """f' with discrete solution x_exact (mss_manufacture_rhs)."""
        n = self.level_N(0)
        f = torch.empty(n, dtype=torch.float64, device=x_exact.device)
        _check(self.lib.mss_manufacture_rhs(self.ctx, _dev_ptr(x_exact, n), f.data_ptr()), "mss_manufacture_rhs")
        return f

    def profile(self, enable: bool, max_level: int = 0):
        _check(self.lib.mss_profile(self.ctx, 1 if enable else 0, int(max_level)), "mss_profile")

    def profile_read(self):
        """{(class name, level): (launches, ms, algorithmic bytes)} for nonzero entries."""
        out = {}
        c, ms, by = ctypes.c_int64(), ctypes.c_double(), ctypes.c_double()
        for ci, name in enumerate(KCLASS):
            for lvl in range(self.levels):
                self.lib.mss_profile_read(self.ctx, ci, lvl, ctypes.byref(c), ctypes.byref(ms), ctypes.byref(by))
                if c.value:
                    out[(name, lvl)] = (c.value, ms.value, by.value)
        return out

    def kernel_launches(self) -> int:
        c = ctypes.c_int64()
        self.lib.mss_kernel_launches(self.ctx, ctypes.byref(c))
        return c.value

    # ---------------------------------------------------------------- solve
    def solve(self, f: torch.Tensor, x: Optional[torch.Tensor] = None, rel_tol: float = 1e-10):
        if x is None:
            x = torch.zeros(self.N, dtype=torch.float64, device=f.device)
        its = (ctypes.c_int64 * self.levels)()
        tr = ctypes.c_double()
        rc = self.lib.mss_solve(self.ctx, _dev_ptr(f, self.N), _dev_ptr(x, self.N), float(rel_tol), its,
                                ctypes.byref(tr))
        _check(rc, "mss_solve")
        rep = self.info()
        rep.rc = rc
        return x, rep

    def solve_host(self, f_host: torch.Tensor, x_host: torch.Tensor, rel_tol: float = 1e-10):
        """End-to-end: host (ideally pinned) f in, host x out; copies inside the call."""
        for t in (f_host, x_host):
            if t.is_cuda or t.dtype != torch.float64 or not t.is_contiguous() or t.numel() != self.N:
                raise ValueError("expected contiguous float64 host tensors of N elements")
        its = (ctypes.c_int64 * self.levels)()
        tr = ctypes.c_double()
        rc = self.lib.mss_solve_host(self.ctx, f_host.data_ptr(), x_host.data_ptr(), float(rel_tol), its,
                                     ctypes.byref(tr))
        _check(rc, "mss_solve_host")
        rep = self.info()
        rep.rc = rc
        return x_host, rep

    def solve_host_batch(self, f_hosts, x_hosts, rel_tol: float = 1e-10):
        """mss_solve_host_batch: host f_hosts[i] -> x_hosts[i] with the copies pipelined
        against the solves (pinned buffers overlap).  Returns (iters [nrhs][L1],
        true_rel_res [nrhs], status)."""
        n = len(f_hosts)
        if len(x_hosts) != n:
            raise ValueError("f_hosts and x_hosts differ in length")
        for t in list(f_hosts) + list(x_hosts):
            if t.is_cuda or t.dtype != torch.float64 or not t.is_contiguous() or t.numel() != self.N:
                raise ValueError("expected contiguous float64 host tensors of N elements")
        fp = (ctypes.c_void_p * max(n, 1))(*[t.data_ptr() for t in f_hosts])
        xp = (ctypes.c_void_p * max(n, 1))(*[t.data_ptr() for t in x_hosts])
        its = (ctypes.c_int64 * max(n * self.levels, 1))()
        tr = (ctypes.c_double * max(n, 1))()
        rc = self.lib.mss_solve_host_batch(self.ctx, n, fp, xp, float(rel_tol), its, tr)
        _check(rc, "mss_solve_host_batch")
        iters = [[its[i * self.levels + k] for k in range(self.levels)] for i in range(n)]
        return iters, [tr[i] for i in range(n)], rc

    # ---------------------------------------------------------------- hooks
    def faces(self, level: int, d: int) -> torch.Tensor:
        nx, ny, nz = self.level_dims(level)
        dims = [nx, ny, nz]
        dims[d] += 1
        T = torch.empty(dims[0] * dims[1] * dims[2], dtype=torch.float64, device="cuda")
        _check(self.lib.mss_get_faces(self.ctx, level, d, T.data_ptr()), "mss_get_faces")
        return T

    def apply_A(self, level: int, x: torch.Tensor) -> torch.Tensor:
        y = torch.empty_like(x)
        _check(self.lib.mss_apply_A(self.ctx, level, _dev_ptr(x, self.level_N(level)), y.data_ptr()), "mss_apply_A")
        return y

    def dot(self, level: int, a: torch.Tensor, b: torch.Tensor) -> float:
        out = ctypes.c_double()
        n = self.level_N(level)
        _check(self.lib.mss_dot(self.ctx, level, _dev_ptr(a, n), _dev_ptr(b, n), ctypes.byref(out)), "mss_dot")
        return out.value

    def smooth(self, level: int, r: torch.Tensor, z: Optional[torch.Tensor], n_half: int, first_color: int = 0):
        n = self.level_N(level)
        zero = z is None
        zz = torch.zeros_like(r) if zero else z.clone()
        _check(self.lib.mss_smooth(self.ctx, level, _dev_ptr(r, n), _dev_ptr(zz, n), n_half, first_color,
                                   1 if zero else 0), "mss_smooth")
        return zz

    def residual_restrict(self, level: int, r: torch.Tensor, z: torch.Tensor) -> torch.Tensor:
        n = self.level_N(level)
        out = torch.empty(self.level_N(level + 1), dtype=torch.float64, device=r.device)
        _check(self.lib.mss_residual_restrict(self.ctx, level, _dev_ptr(r, n), _dev_ptr(z, n), out.data_ptr()),
               "mss_residual_restrict")
        return out

    def prolong_add(self, level: int, y: torch.Tensor, z: torch.Tensor, color: int = -1) -> torch.Tensor:
        zz = z.clone()
        _check(self.lib.mss_prolong_add(self.ctx, level, _dev_ptr(y, self.level_N(level + 1)),
                                        _dev_ptr(zz, self.level_N(level)), color), "mss_prolong_add")
        return zz

    def precond(self, level: int, r: torch.Tensor, rel_tol: float = 1e-10):
        n = self.level_N(level)
        z = torch.empty_like(r)
        its = (ctypes.c_int64 * self.levels)()
        _check(self.lib.mss_precond(self.ctx, level, _dev_ptr(r, n), z.data_ptr(), float(rel_tol), its),
               "mss_precond")
        return z, list(its)

    def coarse_solve(self, b: torch.Tensor) -> torch.Tensor:
        x = torch.empty_like(b)
        _check(self.lib.mss_coarse_solve(self.ctx, _dev_ptr(b, self.level_N(self.levels - 1)), x.data_ptr()),
               "mss_coarse_solve")
        return x

    def rhs_lift(self, f: torch.Tensor):
        b = torch.empty_like(f)
        x0 = torch.empty_like(f)
        _check(self.lib.mss_rhs_lift(self.ctx, _dev_ptr(f, self.N), b.data_ptr(), x0.data_ptr()), "mss_rhs_lift")
        return b, x0

    # ---------------------------------------------------------------- production-path hooks
    def cg_direction(self, level: int, z: torch.Tensor, p_in: Optional[torch.Tensor], rho: float, rho_prev: float,
                     first: bool):
        """(p_out, q, p_out.q) by the solver's own a10 kernel (mss_cg_direction)."""
        n = self.level_N(level)
        p_out = torch.empty_like(z)
        q = torch.empty_like(z)
        pq = ctypes.c_double()
        _check(self.lib.mss_cg_direction(self.ctx, level, _dev_ptr(z, n), None if p_in is None else _dev_ptr(p_in, n),
                                         float(rho), float(rho_prev), 1 if first else 0, p_out.data_ptr(),
                                         q.data_ptr(), ctypes.byref(pq)), "mss_cg_direction")
        return p_out, q, pq.value

    def cg_update(self, level: int, x: torch.Tensor, r: torch.Tensor, p: torch.Tensor, q: torch.Tensor, rho: float,
                  pq: float):
        """(x + alpha p, r - alpha q, ||r||^2) by the solver's own a11 kernel (mss_cg_update)."""
        n = self.level_N(level)
        xx, rr_ = x.clone(), r.clone()
        out = ctypes.c_double()
        _check(self.lib.mss_cg_update(self.ctx, level, _dev_ptr(xx, n), _dev_ptr(rr_, n), _dev_ptr(p, n),
                                      _dev_ptr(q, n), float(rho), float(pq), ctypes.byref(out)), "mss_cg_update")
        return xx, rr_, out.value

    def residual(self, level: int, b: torch.Tensor, x: torch.Tensor):
        """(b - A x, ||b - A x||^2) by the solver's residual kernel (mss_residual)."""
        n = self.level_N(level)
        r = torch.empty_like(b)
        out = ctypes.c_double()
        _check(self.lib.mss_residual(self.ctx, level, _dev_ptr(b, n), _dev_ptr(x, n), r.data_ptr(),
                                     ctypes.byref(out)), "mss_residual")
        return r, out.value

    def presmooth_restrict(self, level: int, r: torch.Tensor):
        """(z, R (r - A z)) with z = 2m+1 half-sweeps from zero (mss_presmooth_restrict)."""
        n = self.level_N(level)
        z = torch.empty_like(r)
        cb = torch.empty(self.level_N(level + 1), dtype=torch.float64, device=r.device)
        _check(self.lib.mss_presmooth_restrict(self.ctx, level, _dev_ptr(r, n), z.data_ptr(), cb.data_ptr()),
               "mss_presmooth_restrict")
        return z, cb

    def prolong_postsmooth(self, level: int, y: torch.Tensor, r: torch.Tensor, z: torch.Tensor):
        """(z', r.z') with z' = 2m+1 half-sweeps on z + E y (mss_prolong_postsmooth)."""
        n = self.level_N(level)
        zz = z.clone()
        rho = ctypes.c_double()
        _check(self.lib.mss_prolong_postsmooth(self.ctx, level, _dev_ptr(y, self.level_N(level + 1)), _dev_ptr(r, n),
                                               _dev_ptr(zz, n), ctypes.byref(rho)), "mss_prolong_postsmooth")
        return zz, rho.value
