"""paper_1706_06844_b200 -- B200-native CN-WSGD time-step solver.

Python mirror of the reference's C++ entry points for the hot path
(``/root/reference/proj/include/fde``), bound over the C ABI in
``include/fde_b200.h`` (``libfde_b200.so``, CUDA sm_100a).  Names follow the
reference: :class:`StructuredFdeOperator` (structured.hpp:57-97),
:class:`MgHierarchy` (multigrid.hpp:107-134), :func:`make_preconditioner`
(precond.hpp:94-98), :func:`gmres` (krylov.hpp:38-40), :func:`time_march`
(driver.hpp:39-40).  Errors map to the reference's exception classes:
``ValueError`` for ``std::invalid_argument``, ``RuntimeError`` for
``std::runtime_error`` / CUDA failures.

Device vectors are ``torch.Tensor`` objects on CUDA (float64, contiguous);
torch is only the allocator/stream plumbing.  There is no CPU fallback: the
CUDA library must load, and device calls fail loudly without a GPU.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

__all__ = [
    "load_library", "library_path", "wsgd_weights", "binom_coeffs", "Problem",
    "StructuredFdeOperator", "MgHierarchy", "Preconditioner", "make_preconditioner",
    "SolverConfig", "KrylovResult", "gmres", "bicgstab", "DriverConfig", "March",
    "SolveReport", "time_march", "SlabMarch", "vdist_run", "plan_level_dims", "transfer", "kernel_launches",
    "PRECOND_NONE", "PRECOND_P2", "PRECOND_MGM", "PRECOND_P2_EXACT", "PRECOND_MGM_GALERKIN",
    "COARSE_LU", "COARSE_SWEEPS", "COARSE_NONE",
]

PKG_DIR = Path(__file__).resolve().parent
LIB_PATH = PKG_DIR / "libfde_b200.so"

PRECOND_NONE, PRECOND_P2, PRECOND_MGM = 0, 1, 2
PRECOND_P2_EXACT, PRECOND_MGM_GALERKIN = 3, 4  # precond.cpp:90-133 (oracle-size variants)
COARSE_LU, COARSE_SWEEPS, COARSE_NONE = 0, 1, 2

_c_size = ctypes.c_size_t
_c_dbl = ctypes.c_double
_c_int = ctypes.c_int
_c_vp = ctypes.c_void_p
_P = ctypes.POINTER(ctypes.c_double)

FIELD_FN = ctypes.CFUNCTYPE(_c_dbl, _c_dbl, _c_dbl, _c_dbl, _c_vp)
INITIAL_FN = ctypes.CFUNCTYPE(_c_dbl, _c_dbl, _c_dbl, _c_vp)


class _FdeProblem(ctypes.Structure):
    _fields_ = [("alpha", _c_dbl), ("beta", _c_dbl), ("ax", _c_dbl), ("bx", _c_dbl),
                ("ay", _c_dbl), ("by", _c_dbl), ("t_final", _c_dbl),
                ("time_dependent_coeffs", _c_int), ("pq", _c_int),
                ("d_plus", FIELD_FN), ("d_minus", FIELD_FN), ("e_plus", FIELD_FN),
                ("e_minus", FIELD_FN), ("source", FIELD_FN), ("initial", INITIAL_FN),
                ("ctx", _c_vp), ("preset", _c_int), ("source_kind", _c_int),
                ("seed", ctypes.c_ulonglong)]


class _SolverConfig(ctypes.Structure):
    _fields_ = [("tol", _c_dbl), ("restart", _c_size), ("max_outer", _c_size)]


class _KrylovResult(ctypes.Structure):
    _fields_ = [("total_iterations", _c_size), ("converged", _c_int), ("n_history", _c_size),
                ("history_length", _c_size), ("history", _P), ("history_capacity", _c_size)]


class _DriverConfig(ctypes.Structure):
    _fields_ = [("precond", _c_int), ("tol", _c_dbl), ("restart", _c_size),
                ("max_outer", _c_size), ("omega", _c_dbl), ("cycles", _c_size),
                ("coarse", _c_int), ("coarse_sweeps", _c_size), ("solver", _c_int)]


# exported symbols and their ctypes signatures (kept in sync with include/fde_b200.h)
_SIGS = {
    "fde_last_error": (ctypes.c_char_p, []),
    "fde_abi_version": (_c_int, []),
    "fde_kernel_launches": (ctypes.c_ulonglong, []),
    "fde_fp64_peak": (_c_int, [ctypes.POINTER(_c_dbl), _c_vp]),
    "fde_wsgd_weights": (_c_int, [_c_dbl, _c_size, _c_int, _P, _P]),
    "fde_op_create": (_c_int, [_c_size, _c_size, _c_dbl, _c_dbl] + [_P] * 8 + [ctypes.POINTER(_c_vp)]),
    "fde_op_create_fractional": (_c_int, [_c_size, _c_size, _c_dbl, _c_dbl, _c_dbl, _c_dbl, _c_int]
                                 + [_P] * 4 + [ctypes.POINTER(_c_vp)]),
    "fde_op_size": (_c_int, [_c_vp, ctypes.POINTER(_c_size)]),
    "fde_op_apply": (_c_int, [_c_vp, _c_vp, _c_vp, _c_vp]),
    "fde_op_apply_rhs": (_c_int, [_c_vp, _c_vp, _c_vp, _c_vp]),
    "fde_op_diagonal": (_c_int, [_c_vp, _P]),
    "fde_op_scale": (_c_int, [_c_vp, _c_dbl]),
    "fde_op_destroy": (_c_int, [_c_vp]),
    "fde_problem_preset": (_c_int, [_c_int, ctypes.c_ulonglong, _c_int, _c_size, _c_dbl,
                                    ctypes.POINTER(_FdeProblem), ctypes.POINTER(_c_size),
                                    ctypes.POINTER(_c_size)]),
    "fde_problem_example": (_c_int, [_c_int, _c_dbl, _c_dbl, _c_dbl, _c_dbl, _c_dbl, _c_dbl,
                                     ctypes.POINTER(_FdeProblem)]),
    "fde_problem_example_default": (_c_int, [_c_int, _c_dbl, _c_dbl, ctypes.POINTER(_FdeProblem)]),
    "fde_error_inf": (_c_int, [ctypes.POINTER(_FdeProblem), _c_size, _c_size, _c_size, _c_dbl, _P,
                               ctypes.POINTER(_c_dbl)]),
    "fde_grid": (_c_int, [ctypes.POINTER(_FdeProblem), _c_size, _c_size, _c_size, _P]),
    "fde_assemble_step_operator": (_c_int, [ctypes.POINTER(_FdeProblem), _c_size, _c_size,
                                            _c_size, _c_size, ctypes.POINTER(_c_vp)]),
    "fde_sample_initial": (_c_int, [ctypes.POINTER(_FdeProblem), _c_size, _c_size, _c_size, _P]),
    "fde_sample_source": (_c_int, [ctypes.POINTER(_FdeProblem), _c_size, _c_size, _c_size,
                                   _c_size, _P]),
    "fde_plan_level_dims": (_c_int, [_c_size, _c_size, _c_dbl, _c_dbl, _c_dbl,
                                     ctypes.POINTER(_c_size), _c_size, ctypes.POINTER(_c_size)]),
    "fde_anisotropy_ratio": (_c_int, [_c_vp, _c_dbl, _c_dbl, _P]),
    "fde_transfer": (_c_int, [_c_size, _c_size, _c_int, _c_int, _c_int, _c_vp, _c_vp, _c_vp]),
    "fde_mg_build_geometric": (_c_int, [ctypes.POINTER(_FdeProblem), _c_size, _c_size, _c_size,
                                        _c_size, _c_dbl, _c_int, _c_size, ctypes.POINTER(_c_vp)]),
    "fde_mg_create": (_c_int, [ctypes.POINTER(_c_vp), _c_size, _c_dbl, _c_int, _c_size,
                               ctypes.POINTER(_c_vp)]),
    "fde_mg_build_p2": (_c_int, [_c_vp, _c_dbl, ctypes.POINTER(_c_vp)]),
    "fde_mg_depth": (_c_int, [_c_vp, ctypes.POINTER(_c_size)]),
    "fde_mg_level_dims": (_c_int, [_c_vp, _c_size, ctypes.POINTER(_c_size), ctypes.POINTER(_c_size)]),
    "fde_mg_vcycle": (_c_int, [_c_vp, _c_vp, _c_vp, _c_int, _c_vp]),
    "fde_mg_destroy": (_c_int, [_c_vp]),
    "fde_precond_create": (_c_int, [_c_int, ctypes.POINTER(_FdeProblem), _c_size, _c_size,
                                    _c_size, _c_size, _c_vp, _c_dbl, _c_size, _c_int, _c_size,
                                    ctypes.POINTER(_c_vp)]),
    "fde_precond_apply": (_c_int, [_c_vp, _c_vp, _c_vp, _c_vp]),
    "fde_precond_destroy": (_c_int, [_c_vp]),
    "fde_gmres": (_c_int, [_c_vp, _c_vp, ctypes.POINTER(_SolverConfig), _c_vp, _c_vp,
                           ctypes.POINTER(_KrylovResult), _c_vp]),
    "fde_bicgstab": (_c_int, [_c_vp, _c_vp, ctypes.POINTER(_SolverConfig), _c_vp, _c_vp,
                              ctypes.POINTER(_KrylovResult), _c_vp]),
    "fde_driver_config_default": (None, [ctypes.POINTER(_DriverConfig)]),
    "fde_march_create": (_c_int, [ctypes.POINTER(_FdeProblem), _c_size, _c_size, _c_size,
                                  ctypes.POINTER(_DriverConfig), ctypes.POINTER(_c_vp)]),
    "fde_march_step": (_c_int, [_c_vp, _c_vp, _c_int, _c_vp, ctypes.POINTER(_c_size), _P]),
    "fde_march_steps_taken": (_c_int, [_c_vp, ctypes.POINTER(_c_size)]),
    "fde_march_solution": (_c_int, [_c_vp, _c_vp, _c_int, _c_vp]),
    "fde_march_solution_ptr": (_c_int, [_c_vp, ctypes.POINTER(_c_vp)]),
    "fde_march_prefetch_source": (_c_int, [_c_vp, _c_vp]),
    "fde_march_solution_async": (_c_int, [_c_vp, _c_vp]),
    "fde_march_wait": (_c_int, [_c_vp]),
    "fde_march_destroy": (_c_int, [_c_vp]),
    "fde_time_march": (_c_int, [ctypes.POINTER(_FdeProblem), _c_size, _c_size, _c_size,
                                ctypes.POINTER(_DriverConfig), _P, ctypes.POINTER(_c_size), _P, _P]),
    "fde_slab_create": (_c_int, [ctypes.POINTER(_FdeProblem)] + [_c_size] * 10 + [ctypes.POINTER(_c_vp)]),
    "fde_slab_ypass": (_c_int, [_c_vp, _c_vp, _c_vp, _c_dbl, _c_vp]),
    "fde_slab_xpass": (_c_int, [_c_vp, _c_vp, _c_vp, _c_vp, _c_dbl, _c_int, _c_vp, _c_vp, _c_dbl,
                                _c_vp, _c_dbl, _c_vp]),
    "fde_slab_diagonal": (_c_int, [_c_vp, _P]),
    "fde_slab_destroy": (_c_int, [_c_vp]),
    "fde_transpose": (_c_int, [_c_vp, _c_vp, _c_size, _c_size, _c_vp]),
    "fde_transfer_rows": (_c_int, [_c_size, _c_size, _c_int, _c_int, _c_int, _c_int, _c_vp, _c_size,
                                   _c_vp, _c_size, _c_size, _c_vp]),
    "fde_vec": (_c_int, [_c_int, _c_size, _c_dbl, _c_vp, _c_vp, _c_vp, _c_vp]),
    "fde_block_permute": (_c_int, [_c_vp, _c_vp, _c_size, _c_size, ctypes.POINTER(ctypes.c_longlong),
                                   _c_int, _c_int, _c_vp]),
    "fde_axpy_dev": (_c_int, [_c_size, _c_vp, _c_dbl, _c_vp, _c_vp, _c_vp]),
    "fde_dot": (_c_int, [_c_size, _c_vp, _c_vp, _c_vp, _c_int, _c_vp]),
    "fde_dist_unique_id": (_c_int, [ctypes.c_char_p]),
    "fde_dist_comm_create": (_c_int, [ctypes.c_char_p, _c_int, _c_int, ctypes.POINTER(_c_vp)]),
    "fde_dist_comm_destroy": (_c_int, [_c_vp]),
    "fde_dist_march_create": (_c_int, [_c_vp, ctypes.POINTER(_FdeProblem), _c_size, _c_size, _c_size,
                                       ctypes.POINTER(_DriverConfig), _c_size, ctypes.POINTER(_c_vp)]),
    "fde_dist_march_rows": (_c_int, [_c_vp, ctypes.POINTER(_c_size), ctypes.POINTER(_c_size)]),
    "fde_dist_march_step": (_c_int, [_c_vp, _c_vp, _c_vp, ctypes.POINTER(_c_size), _P]),
    "fde_dist_march_solution": (_c_int, [_c_vp, _c_vp, _c_int, _c_vp]),
    "fde_dist_march_solution_ptr": (_c_int, [_c_vp, ctypes.POINTER(_c_vp)]),
    "fde_dist_march_apply": (_c_int, [_c_vp, _c_vp, _c_vp, _c_vp]),
    "fde_dist_march_vcycle": (_c_int, [_c_vp, _c_vp, _c_vp, _c_vp]),
    "fde_dist_march_collectives": (_c_int, [_c_vp, ctypes.POINTER(ctypes.c_ulonglong)]),
    "fde_dist_march_destroy": (_c_int, [_c_vp]),
    "fde_dist_split_rows": (_c_int, [_c_size, _c_int, ctypes.POINTER(_c_size)]),
    "fde_dist_induced_rows": (_c_int, [ctypes.POINTER(_c_size), _c_int, _c_size, _c_int,
                                       ctypes.POINTER(_c_size)]),
    "fde_vdist_run": (_c_int, [ctypes.POINTER(_FdeProblem), _c_size, _c_size, _c_size,
                               ctypes.POINTER(_DriverConfig), _c_int, _c_size, _c_int, _c_size,
                               _c_vp, _c_vp, ctypes.POINTER(_c_size), _c_vp,
                               ctypes.POINTER(ctypes.c_ulonglong)]),
}
EXPORTED_SYMBOLS = tuple(_SIGS)

_lib = None


def library_path() -> Path:
    return Path(os.environ.get("FDE_B200_LIB", LIB_PATH))


def build_library(force: bool = False) -> Path:
    """Compile libfde_b200.so for sm_100a in-tree (nvcc; no GPU needed)."""
    if force or not LIB_PATH.exists():
        subprocess.run(["make", "-s", "-C", str(PKG_DIR / "csrc"), "-j8"], check=True)
    return LIB_PATH


def load_library() -> ctypes.CDLL:
    """Load the CUDA library (building it if absent).  Never falls back to CPU."""
    global _lib
    if _lib is None:
        path = library_path()
        if not path.exists():
            build_library()
        lib = ctypes.CDLL(str(path))
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


class FdeError(RuntimeError):
    pass


def _check(rc: int) -> None:
    if rc == 0:
        return
    msg = load_library().fde_last_error().decode()
    if rc == 1:
        raise ValueError(msg)
    raise RuntimeError(msg)


def kernel_launches() -> int:
    return int(load_library().fde_kernel_launches())


def fp64_peak_tflops() -> float:
    """Measured DFMA throughput of the current device (TFLOP/s)."""
    v = _c_dbl(0.0)
    _check(load_library().fde_fp64_peak(ctypes.byref(v), None))
    return float(v.value)


# ------------------------------------------------------------------ tensors
def _torch():
    import torch
    return torch


def _dev_ptr(t) -> int:
    torch = _torch()
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float64:
        raise ValueError("expected a CUDA float64 tensor")
    if not t.is_contiguous():
        raise ValueError("expected a contiguous tensor")
    return t.data_ptr()


def _stream(stream=None) -> int:
    if stream is not None:
        return int(stream)
    return _torch().cuda.current_stream().cuda_stream


def _empty_like_n(n: int, like=None):
    torch = _torch()
    dev = like.device if like is not None else torch.device("cuda")
    return torch.empty(n, dtype=torch.float64, device=dev)


def _np(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_P)


# ------------------------------------------------------------------ weights
def wsgd_weights(gamma: float, K: int, pq: int = 0) -> np.ndarray:
    """weights.cpp:30-51 (pq=0) / the (1,-1) extension (pq=1)."""
    g, w = np.zeros(K + 1), np.zeros(K + 1)
    _check(load_library().fde_wsgd_weights(gamma, K, pq, _ptr(g), _ptr(w)))
    return w


def binom_coeffs(gamma: float, K: int) -> np.ndarray:
    g, w = np.zeros(K + 1), np.zeros(K + 1)
    _check(load_library().fde_wsgd_weights(gamma, max(K, 2), 0, _ptr(g), _ptr(w)))
    return g[:K + 1]


# ------------------------------------------------------------------ problem
@dataclass
class Problem:
    """FdeProblem (problem.hpp:22-33): a BASELINE preset or Python callbacks."""
    alpha: float = 1.5
    beta: float = 1.5
    ax: float = 0.0
    bx: float = 1.0
    ay: float = 0.0
    by: float = 1.0
    t_final: float = 1.0
    pq: int = 0
    time_dependent_coeffs: bool = False
    d_plus: object = None
    d_minus: object = None
    e_plus: object = None
    e_minus: object = None
    source: object = None
    initial: object = None
    preset: int = 0
    source_kind: int = 0
    seed: int = 0
    n: int = 0        # preset grid size
    steps: int = 0    # preset step count
    _keep: list = field(default_factory=list, repr=False)

    @classmethod
    def preset_config(cls, cfg: int, seed: int = 0, source_kind: int = -1, steps: int = 0,
                      tau: float = 0.0) -> "Problem":
        s = _FdeProblem()
        n, st = _c_size(), _c_size()
        _check(load_library().fde_problem_preset(cfg, seed, source_kind, steps, tau,
                                                 ctypes.byref(s), ctypes.byref(n), ctypes.byref(st)))
        return cls(alpha=s.alpha, beta=s.beta, ax=s.ax, bx=s.bx, ay=s.ay, by=s.by,
                   t_final=s.t_final, pq=s.pq, preset=cfg, source_kind=s.source_kind,
                   seed=seed, n=n.value, steps=st.value)

    @classmethod
    def example(cls, which: int, alpha: float, beta: float, domain=None) -> "Problem":
        """make_example_on / make_example (problem.cpp:172-260): the reference's
        manufactured problem 1..3 (example 2: time-dependent coefficients),
        evaluated natively (device-side per-step re-assembly)."""
        s = _FdeProblem()
        lib = load_library()
        if domain is None:
            _check(lib.fde_problem_example_default(which, alpha, beta, ctypes.byref(s)))
        else:
            ax, bx, ay, by = domain
            _check(lib.fde_problem_example(which, alpha, beta, ax, bx, ay, by, ctypes.byref(s)))
        return cls(alpha=s.alpha, beta=s.beta, ax=s.ax, bx=s.bx, ay=s.ay, by=s.by,
                   t_final=s.t_final, preset=s.preset,
                   time_dependent_coeffs=bool(s.time_dependent_coeffs))

    def error_inf(self, u, n1: int, n2: int, steps: int, t: float) -> float:
        """error_inf (problem.hpp:69-70) against the exact solution at time t."""
        u = np.ascontiguousarray(np.asarray(u, dtype=np.float64))
        e = _c_dbl()
        s = self.c_struct()
        _check(load_library().fde_error_inf(ctypes.byref(s), n1, n2, steps, t, _ptr(u),
                                            ctypes.byref(e)))
        return e.value

    def c_struct(self) -> _FdeProblem:
        s = _FdeProblem()
        for k in ("alpha", "beta", "ax", "bx", "ay", "by", "t_final", "pq", "preset",
                  "source_kind", "seed"):
            setattr(s, k, getattr(self, k))
        s.time_dependent_coeffs = int(bool(self.time_dependent_coeffs))
        if not self.preset:
            self._keep.clear()
            for name in ("d_plus", "d_minus", "e_plus", "e_minus", "source"):
                fn = getattr(self, name)
                if fn is not None:
                    cb = FIELD_FN(lambda x, y, t, _c, f=fn: float(f(x, y, t)))
                    self._keep.append(cb)
                    setattr(s, name, cb)
            if self.initial is not None:
                cb = INITIAL_FN(lambda x, y, _c, f=self.initial: float(f(x, y)))
                self._keep.append(cb)
                s.initial = cb
        return s

    def grid(self, n1: int, n2: int, steps: int) -> dict:
        out = np.zeros(5)
        s = self.c_struct()
        _check(load_library().fde_grid(ctypes.byref(s), n1, n2, steps, _ptr(out)))
        return dict(zip(("hx", "hy", "dt", "inv_r", "s_over_r"), out.tolist()))

    def sample_initial(self, n1: int, n2: int, steps: int) -> np.ndarray:
        u = np.zeros(n1 * n2)
        s = self.c_struct()
        _check(load_library().fde_sample_initial(ctypes.byref(s), n1, n2, steps, _ptr(u)))
        return u

    def sample_source(self, n1: int, n2: int, steps: int, m: int) -> np.ndarray:
        v = np.zeros(n1 * n2)
        s = self.c_struct()
        _check(load_library().fde_sample_source(ctypes.byref(s), n1, n2, steps, m, _ptr(v)))
        return v


# ------------------------------------------------------------------ operator
class StructuredFdeOperator:
    """Device-resident StructuredFdeOperator (structured.hpp:57-97)."""

    def __init__(self, handle):
        self._h = handle
        n = _c_size()
        _check(load_library().fde_op_size(self._h, ctypes.byref(n)))
        self.n = n.value

    @classmethod
    def from_blocks(cls, n1, n2, inv_r, s_over_r, col_x, row_x, col_y, row_y, dp, dm, ep, em):
        arrs = [_np(a) for a in (col_x, row_x, col_y, row_y, dp, dm, ep, em)]
        h = _c_vp()
        _check(load_library().fde_op_create(n1, n2, inv_r, s_over_r, *map(_ptr, arrs), ctypes.byref(h)))
        return cls(h)

    @classmethod
    def fractional(cls, n1, n2, inv_r, s_over_r, alpha, beta, dp, dm, ep, em, pq=0):
        arrs = [_np(a) for a in (dp, dm, ep, em)]
        h = _c_vp()
        _check(load_library().fde_op_create_fractional(n1, n2, inv_r, s_over_r, alpha, beta, pq,
                                                       *map(_ptr, arrs), ctypes.byref(h)))
        return cls(h)

    @classmethod
    def assemble(cls, problem: Problem, n1: int, n2: int, steps: int, m: int = 1):
        """assemble_step_operator (problem.hpp:54-55)."""
        h = _c_vp()
        s = problem.c_struct()
        _check(load_library().fde_assemble_step_operator(ctypes.byref(s), n1, n2, steps, m, ctypes.byref(h)))
        return cls(h)

    def size(self) -> int:
        return self.n

    def apply(self, x, y=None, stream=None):
        y = _empty_like_n(self.n, x) if y is None else y
        _check(load_library().fde_op_apply(self._h, _dev_ptr(x), _dev_ptr(y), _stream(stream)))
        return y

    def apply_rhs(self, x, y=None, stream=None):
        y = _empty_like_n(self.n, x) if y is None else y
        _check(load_library().fde_op_apply_rhs(self._h, _dev_ptr(x), _dev_ptr(y), _stream(stream)))
        return y

    def diagonal(self) -> np.ndarray:
        d = np.zeros(self.n)
        _check(load_library().fde_op_diagonal(self._h, _ptr(d)))
        return d

    def scale(self, s: float) -> None:
        _check(load_library().fde_op_scale(self._h, s))

    def anisotropy_ratio(self, alpha, beta) -> float:
        r = _c_dbl()
        _check(load_library().fde_anisotropy_ratio(self._h, alpha, beta, ctypes.byref(r)))
        return r.value

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.fde_op_destroy(self._h)
            self._h = None


def plan_level_dims(n1, n2, ratio0, alpha, beta):
    """mg::plan_level_dims (multigrid.hpp:39-40)."""
    dims = (_c_size * 256)()
    nl = _c_size()
    _check(load_library().fde_plan_level_dims(n1, n2, ratio0, alpha, beta, dims, 128, ctypes.byref(nl)))
    return [(dims[2 * l], dims[2 * l + 1]) for l in range(nl.value)]


def transfer(n1, n2, coarsen_x, coarsen_y, op, x, out, stream=None):
    """GridTransfer: op 0 prolong, 1 restrict_full, 2 restrict_transpose (device)."""
    _check(load_library().fde_transfer(n1, n2, int(coarsen_x), int(coarsen_y), op, _dev_ptr(x),
                                       _dev_ptr(out), _stream(stream)))
    return out


class MgHierarchy:
    """Device-resident MgHierarchy (multigrid.hpp:107-134)."""

    def __init__(self, handle, keep=()):
        self._h = handle
        self._keep = list(keep)

    @classmethod
    def build_geometric(cls, problem: Problem, n1, n2, steps, m=1, omega=0.9,
                        coarse=COARSE_LU, coarse_sweeps=3):
        h = _c_vp()
        s = problem.c_struct()
        _check(load_library().fde_mg_build_geometric(ctypes.byref(s), n1, n2, steps, m, omega,
                                                     coarse, coarse_sweeps, ctypes.byref(h)))
        return cls(h, [problem])

    @classmethod
    def from_levels(cls, levels, omega=0.9, coarse=COARSE_LU, coarse_sweeps=3):
        arr = (_c_vp * len(levels))(*[lv._h for lv in levels])
        h = _c_vp()
        _check(load_library().fde_mg_create(arr, len(levels), omega, coarse, coarse_sweeps, ctypes.byref(h)))
        return cls(h, levels)

    @classmethod
    def build_p2(cls, fine: StructuredFdeOperator, omega=0.9):
        h = _c_vp()
        _check(load_library().fde_mg_build_p2(fine._h, omega, ctypes.byref(h)))
        return cls(h, [fine])

    def depth(self) -> int:
        d = _c_size()
        _check(load_library().fde_mg_depth(self._h, ctypes.byref(d)))
        return d.value

    def dims(self):
        out = []
        for l in range(self.depth()):
            a, b = _c_size(), _c_size()
            _check(load_library().fde_mg_level_dims(self._h, l, ctypes.byref(a), ctypes.byref(b)))
            out.append((a.value, b.value))
        return out

    def vcycle(self, b, x=None, zero_guess=None, stream=None):
        torch = _torch()
        if x is None:
            x = torch.zeros_like(b)
            zero_guess = True
        if zero_guess is None:
            zero_guess = not bool(torch.any(x != 0).item())
        _check(load_library().fde_mg_vcycle(self._h, _dev_ptr(b), _dev_ptr(x), int(zero_guess), _stream(stream)))
        return x

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.fde_mg_destroy(self._h)
            self._h = None


class Preconditioner:
    """Precond (krylov.hpp:11-14) built by make_preconditioner."""

    def __init__(self, handle, keep=()):
        self._h = handle
        self._keep = list(keep)

    def apply(self, r, z=None, stream=None):
        z = _empty_like_n(r.numel(), r) if z is None else z
        _check(load_library().fde_precond_apply(self._h, _dev_ptr(r), _dev_ptr(z), _stream(stream)))
        return z

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.fde_precond_destroy(self._h)
            self._h = None


def make_preconditioner(kind, problem, n1, n2, steps, m, op, omega, cycles=1,
                        coarse=COARSE_SWEEPS, coarse_sweeps=3) -> Preconditioner:
    """make_preconditioner (precond.hpp:94-98); kind 0 none, 1 p2, 2 mgm, 3 p2-exact,
    4 mgm-galerkin (the problem is needed for 2 and 4)."""
    h = _c_vp()
    s = problem.c_struct() if problem is not None else None
    _check(load_library().fde_precond_create(kind, ctypes.byref(s) if s is not None else None, n1, n2,
                                             steps, m, op._h, omega, cycles, coarse, coarse_sweeps,
                                             ctypes.byref(h)))
    return Preconditioner(h, [op, problem])


@dataclass
class SolverConfig:
    tol: float = 1e-7
    restart: int = 20
    max_outer: int = 100


@dataclass
class KrylovResult:
    solution: object
    total_iterations: int
    residual_history: list
    converged: bool


def _krylov(fn, op, cfg, b, precond, stream):
    torch = _torch()
    x = torch.empty_like(b)
    hist = np.zeros(65536)
    res = _KrylovResult(history=_ptr(hist), history_capacity=len(hist))
    c = _SolverConfig(cfg.tol, cfg.restart, cfg.max_outer)
    _check(fn(op._h, precond._h if precond is not None else None, ctypes.byref(c), _dev_ptr(b),
              _dev_ptr(x), ctypes.byref(res), _stream(stream)))
    return KrylovResult(x, int(res.total_iterations), hist[:res.n_history].tolist(), bool(res.converged))


def gmres(op: StructuredFdeOperator, cfg: SolverConfig, b, precond=None, stream=None) -> KrylovResult:
    """gmres (krylov.hpp:38-40) with zero initial guess."""
    return _krylov(load_library().fde_gmres, op, cfg, b, precond, stream)


def bicgstab(op: StructuredFdeOperator, cfg: SolverConfig, b, precond=None, stream=None) -> KrylovResult:
    """Left-preconditioned BiCGSTAB (extension; same stopping rule as gmres)."""
    return _krylov(load_library().fde_bicgstab, op, cfg, b, precond, stream)


@dataclass
class DriverConfig:
    """DriverConfig (driver.hpp:12-21) + solver (0 gmres, 1 bicgstab)."""
    precond: int = PRECOND_NONE
    tol: float = 1e-7
    restart: int = 20
    max_outer: int = 100
    omega: float = 0.9
    cycles: int = 1
    coarse: int = COARSE_SWEEPS
    coarse_sweeps: int = 3
    solver: int = 0

    def c_struct(self) -> _DriverConfig:
        return _DriverConfig(self.precond, self.tol, self.restart, self.max_outer, self.omega,
                             self.cycles, self.coarse, self.coarse_sweeps, self.solver)


@dataclass
class SolveReport:
    """SolveReport (driver.hpp:23-36)."""
    n1: int
    n2: int
    steps: int
    step_iterations: list
    step_residuals: list
    avg_iterations: float
    all_converged: bool
    wall_seconds: float
    solution: np.ndarray
    has_error: bool = False
    error_inf: float = float("nan")


class March:
    """Step-by-step time_march: device-resident u^m, one CN-WSGD step per call."""

    def __init__(self, problem: Problem, n1: int, n2: int, steps: int, cfg: DriverConfig):
        self.problem, self.n1, self.n2, self.steps = problem, n1, n2, steps
        self._s = problem.c_struct()
        self._cfg = cfg.c_struct()
        self._h = _c_vp()
        _check(load_library().fde_march_create(ctypes.byref(self._s), n1, n2, steps,
                                               ctypes.byref(self._cfg), ctypes.byref(self._h)))

    PREFETCHED = "prefetched"

    def step(self, source=None, stream=None):
        """Advance one step.  source: None (library evaluates it), a numpy host
        array (copied H2D inside the call), a CUDA tensor (used in place) or
        March.PREFETCHED (the array given to prefetch_source)."""
        it, res = _c_size(), _c_dbl()
        if source is None:
            ptr, mode = None, 0
        elif isinstance(source, str) and source == March.PREFETCHED:
            ptr, mode = None, 3
        elif isinstance(source, np.ndarray):
            ptr, mode = source.ctypes.data, 1
        else:
            ptr, mode = _dev_ptr(source), 2
        _check(load_library().fde_march_step(self._h, ptr, mode, _stream(stream),
                                             ctypes.byref(it), ctypes.byref(res)))
        return it.value, res.value

    def solution(self, out=None, stream=None) -> np.ndarray:
        if out is None:
            out = np.zeros(self.n1 * self.n2)
        _check(load_library().fde_march_solution(self._h, out.ctypes.data, 1, _stream(stream)))
        return out

    def prefetch_source(self, host_source: np.ndarray) -> None:
        """Start the H2D copy of a coming step's source, at most two ahead
        (keep the array alive until that step; pinned memory makes the copy
        asynchronous).  step(March.PREFETCHED) consumes the oldest."""
        _check(load_library().fde_march_prefetch_source(self._h, host_source.ctypes.data))

    def solution_async(self, out: np.ndarray) -> None:
        """Start the D2H copy of u^m into `out` (valid after wait())."""
        _check(load_library().fde_march_solution_async(self._h, out.ctypes.data))

    def wait(self) -> None:
        _check(load_library().fde_march_wait(self._h))

    def solution_device_ptr(self) -> int:
        p = _c_vp()
        _check(load_library().fde_march_solution_ptr(self._h, ctypes.byref(p)))
        return p.value

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.fde_march_destroy(self._h)
            self._h = None


def time_march(problem: Problem, n1: int, n2: int, steps: int, cfg: DriverConfig) -> SolveReport:
    """time_march (driver.hpp:39-40) on the GPU; host outputs."""
    u = np.zeros(n1 * n2)
    its = (_c_size * steps)()
    res = np.zeros(steps)
    wall = _c_dbl()
    s = problem.c_struct()
    c = cfg.c_struct()
    _check(load_library().fde_time_march(ctypes.byref(s), n1, n2, steps, ctypes.byref(c), _ptr(u),
                                         its, _ptr(res), ctypes.byref(wall)))
    its_l = [int(v) for v in its]
    rep = SolveReport(n1, n2, steps, its_l, res.tolist(), sum(its_l) / max(steps, 1),
                      bool(all(r <= cfg.tol for r in res)), wall.value, u)
    if problem.preset > 100:  # manufactured examples carry the exact solution (driver.cpp:63-66)
        rep.has_error = True
        rep.error_inf = problem.error_inf(u, n1, n2, steps, problem.t_final)
    return rep


# ------------------------------------------------------------------ multi-GPU
class SlabMarch:
    """time_march on y-slabs, one process per GPU (csrc/dist.cu over NCCL): this
    rank's rows [r0, r1) of u^m stay on its device.  The NCCL id is made on
    rank 0 and moved by torch.distributed (any backend) when world > 1."""

    def __init__(self, problem: Problem, n1: int, n2: int, steps: int, cfg: DriverConfig,
                 rank: int = 0, world: int = 1, agglomerate: int = 65536):
        lib = load_library()
        idbuf = ctypes.create_string_buffer(128)
        if rank == 0:
            _check(lib.fde_dist_unique_id(idbuf))
        if world > 1:
            import torch
            import torch.distributed as dist
            t = torch.frombuffer(bytearray(idbuf.raw), dtype=torch.uint8).clone()
            if dist.get_backend() == "nccl":
                t = t.cuda()
            dist.broadcast(t, src=0)
            idbuf = ctypes.create_string_buffer(bytes(t.cpu().numpy().tobytes()), 128)
        self._comm = _c_vp()
        _check(lib.fde_dist_comm_create(idbuf, rank, world, ctypes.byref(self._comm)))
        self._s, self._cfg = problem.c_struct(), cfg.c_struct()
        self._h = _c_vp()
        _check(lib.fde_dist_march_create(self._comm, ctypes.byref(self._s), n1, n2, steps,
                                         ctypes.byref(self._cfg), agglomerate, ctypes.byref(self._h)))
        r0, r1 = _c_size(), _c_size()
        _check(lib.fde_dist_march_rows(self._h, ctypes.byref(r0), ctypes.byref(r1)))
        self.n1, self.n2, self.r0, self.r1 = n1, n2, r0.value, r1.value
        self.local_size = (self.r1 - self.r0) * n1

    def step(self, source_local=None, stream=None):
        """source_local: CUDA tensor with this rank's rows of the source, or None."""
        it, res = _c_size(), _c_dbl()
        ptr = None if source_local is None else _dev_ptr(source_local)
        _check(load_library().fde_dist_march_step(self._h, ptr, _stream(stream), ctypes.byref(it),
                                                  ctypes.byref(res)))
        return it.value, res.value

    def solution_local(self) -> np.ndarray:
        out = np.zeros(self.local_size)
        _check(load_library().fde_dist_march_solution(self._h, out.ctypes.data, 1, _stream()))
        return out

    def solution_to(self, tensor, stream=None) -> None:
        """Copy this rank's rows of u^m into a CUDA tensor (stream ordered)."""
        _check(load_library().fde_dist_march_solution(self._h, _dev_ptr(tensor), 0, _stream(stream)))

    def apply(self, x_local, y_local, stream=None) -> None:
        _check(load_library().fde_dist_march_apply(self._h, _dev_ptr(x_local), _dev_ptr(y_local),
                                                   _stream(stream)))

    def vcycle(self, b_local, x_local, stream=None) -> None:
        _check(load_library().fde_dist_march_vcycle(self._h, _dev_ptr(b_local), _dev_ptr(x_local),
                                                    _stream(stream)))

    def collectives(self) -> int:
        n = ctypes.c_ulonglong()
        _check(load_library().fde_dist_march_collectives(self._h, ctypes.byref(n)))
        return int(n.value)

    def __del__(self):
        if _lib is not None:
            if getattr(self, "_h", None):
                _lib.fde_dist_march_destroy(self._h)
                self._h = None
            if getattr(self, "_comm", None):
                _lib.fde_dist_comm_destroy(self._comm)
                self._comm = None


def vdist_run(problem: Problem, n1: int, n2: int, steps: int, cfg: DriverConfig, nranks: int,
              what: str = "march", nrun: int = 1, inp: np.ndarray | None = None,
              agglomerate: int = 65536):
    """The multi-GPU code path on `nranks` virtual ranks of the current device.
    what: "march" -> (u^nrun, iterations, residuals, collectives);
    "apply" / "vcycle" -> the full-grid result vector (host arrays)."""
    code = {"march": 0, "apply": 1, "vcycle": 2}[what]
    out = np.zeros(n1 * n2)
    its = (_c_size * max(nrun, 1))()
    res = np.zeros(max(nrun, 1))
    ncoll = ctypes.c_ulonglong()
    s, c = problem.c_struct(), cfg.c_struct()
    src = None
    if code:
        src = np.ascontiguousarray(inp, dtype=np.float64)
        assert src.size == n1 * n2
    _check(load_library().fde_vdist_run(ctypes.byref(s), n1, n2, steps, ctypes.byref(c), nranks,
                                        agglomerate, code, nrun,
                                        src.ctypes.data if src is not None else None,
                                        out.ctypes.data, its, res.ctypes.data, ctypes.byref(ncoll)))
    if code:
        return out
    return out, [int(v) for v in its][:nrun], res[:nrun].tolist(), int(ncoll.value)
