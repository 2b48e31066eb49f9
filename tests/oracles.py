"""ctypes loaders for the CPU checkers (test infrastructure only).

* ``Oracle``  -- oracle/liboracle.so, our plain-C restatement (always built).
* ``RefLib``  -- oracle/_ref/libfde_ref.so, the UNMODIFIED reference sources
  compiled by oracle/Makefile; present wherever it was built (it travels to
  the GPU box in the gpurun snapshot), skipped otherwise.

* ``Adapter`` -- oracle/_ref/libfde_adapter.so: the reference's own gmres and
  step loop driving libfde_b200.so through fde::LinOp / fde::Precond adapters
  (the drop-in check of INTEGRATION.md); needs a GPU to call.

Oracle and RefLib expose the same flat entry points (``orc_*`` / ``ref_*``) over one spec
struct, so a test can run either checker with identical arguments.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
ORACLE_DIR = ROOT / "oracle"
ORACLE_SO = ORACLE_DIR / "liboracle.so"
REF_SO = ORACLE_DIR / "_ref" / "libfde_ref.so"
ADAPTER_SO = ORACLE_DIR / "_ref" / "libfde_adapter.so"

_P = ctypes.POINTER(ctypes.c_double)
_I = ctypes.POINTER(ctypes.c_int)

# defaults of each BASELINE config: (n, alpha, beta, tau, steps, pq, source_kind)
CONFIGS = {
    1: (63, 1.8, 1.6, 1 / 64, 64, 0, 0),
    2: (255, 1.5, 1.7, 1 / 256, 32, 0, 0),
    3: (1023, 1.1, 1.9, 1 / 128, 16, 1, 1),
    4: (2047, 1.6, 1.4, 1 / 64, 8, 0, 0),
    5: (2047, 1.7, 1.3, 1 / 64, 1, 0, 0),
}


class Spec(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int) for n in (
        "cfg n1 n2 steps precond restart max_outer cycles coarse coarse_sweeps pq "
        "source_kind").split()] + [
        (n, ctypes.c_double) for n in "tol omega alpha beta tau".split()] + [
        ("seed", ctypes.c_ulonglong)]


def spec(cfg: int, **kw) -> Spec:
    """Spec with the BASELINE defaults; 0/-1 fields mean 'config default'."""
    s = Spec(cfg=cfg, n1=0, n2=0, steps=0, precond=2, restart=20, max_outer=100, cycles=1,
             coarse=1, coarse_sweeps=3, pq=-1, source_kind=-1, tol=1e-8, omega=0.7,
             alpha=0.0, beta=0.0, tau=0.0, seed=0)
    if cfg == 3:
        s.restart, s.tol = 30, 1e-10
    for k, v in kw.items():
        setattr(s, k, v)
    return s


def dims_of(s: Spec):
    if s.cfg > 100:  # manufactured example k = cfg - 100 (harness default n = 32)
        n1 = s.n1 or 32
        return (n1, s.n2 or n1)
    n = CONFIGS[s.cfg if s.cfg else 1][0]
    return (s.n1 or n, s.n2 or n)


def _p(a):
    return a.ctypes.data_as(_P)


class _Checker:
    prefix = ""

    def __init__(self, path: Path):
        self.lib = ctypes.CDLL(str(path))
        getattr(self.lib, f"{self.prefix}last_error").restype = ctypes.c_char_p

    def _call(self, name, *args):
        rc = getattr(self.lib, self.prefix + name)(*args)
        if rc != 0:
            msg = getattr(self.lib, self.prefix + "last_error")()
            raise RuntimeError(f"{self.prefix}{name}: {msg.decode() if msg else rc}")
        return rc

    def weights(self, gamma, K, pq=0):
        g, w = np.zeros(K + 1), np.zeros(K + 1)
        self._call("wsgd_weights", ctypes.c_double(gamma), K, pq, _p(g), _p(w))
        return g, w

    def toeplitz_both(self, gamma, x, pq=0):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y, yt = np.zeros_like(x), np.zeros_like(x)
        self._call("toeplitz_apply_both", ctypes.c_double(gamma), len(x), pq, _p(x), _p(y), _p(yt))
        return y, yt

    def toeplitz_colrow(self, col, row, x):
        col, row, x = (np.ascontiguousarray(a, dtype=np.float64) for a in (col, row, x))
        y, yt = np.zeros_like(x), np.zeros_like(x)
        self._call("toeplitz_apply_colrow", len(x), _p(col), _p(row), _p(x), _p(y), _p(yt))
        return y, yt

    def grid(self, s):
        out = np.zeros(5)
        self._call("grid", ctypes.byref(s), _p(out))
        return dict(zip("hx hy dt inv_r s_over_r".split(), out))

    def coefficients(self, s):
        n1, n2 = dims_of(s)
        arrs = [np.zeros(n1 * n2) for _ in range(4)]
        self._call("coefficients", ctypes.byref(s), *map(_p, arrs))
        return arrs

    def apply(self, s, x, sign=1):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros_like(x)
        self._call("op_apply", ctypes.byref(s), sign, _p(x), _p(y))
        return y

    def diagonal(self, s):
        n1, n2 = dims_of(s)
        d = np.zeros(n1 * n2)
        self._call("op_diagonal", ctypes.byref(s), _p(d))
        return d

    def plan(self, s):
        dims = np.zeros(256, np.int32)
        r0 = ctypes.c_double()
        nl = self.lib[self.prefix + "plan"](ctypes.byref(s), dims.ctypes.data_as(_I), 128, ctypes.byref(r0))
        assert nl > 0
        return [tuple(d) for d in dims[:2 * nl].reshape(-1, 2).tolist()], r0.value

    def plan_raw(self, n1, n2, ratio0, alpha, beta):
        dims = np.zeros(256, np.int32)
        nl = self.lib[self.prefix + "plan_raw"](n1, n2, ctypes.c_double(ratio0), ctypes.c_double(alpha),
                                                ctypes.c_double(beta), dims.ctypes.data_as(_I), 128)
        assert nl > 0
        return [tuple(d) for d in dims[:2 * nl].reshape(-1, 2).tolist()]

    def transfer(self, n1, n2, cx, cy, op, v):
        k1 = (n1 - n1 % 2) // 2 if cx else n1
        k2 = (n2 - n2 % 2) // 2 if cy else n2
        v = np.ascontiguousarray(v, dtype=np.float64)
        out = np.zeros(n1 * n2 if op == 0 else k1 * k2)
        self._call("transfer", n1, n2, int(cx), int(cy), op, _p(v), _p(out))
        return out

    def vcycle(self, s, b, x0=None):
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.zeros_like(b) if x0 is None else np.array(x0, dtype=np.float64)
        self._call("vcycle", ctypes.byref(s), _p(b), _p(x))
        return x

    def precond(self, s, r):
        r = np.ascontiguousarray(r, dtype=np.float64)
        z = np.zeros_like(r)
        self._call("precond_apply", ctypes.byref(s), _p(r), _p(z))
        return z

    def initial(self, s):
        n1, n2 = dims_of(s)
        u = np.zeros(n1 * n2)
        self._call("initial", ctypes.byref(s), _p(u))
        return u

    def source(self, s, m):
        n1, n2 = dims_of(s)
        v = np.zeros(n1 * n2)
        self._call("source", ctypes.byref(s), m, _p(v))
        return v

    def rhs(self, s, m, u):
        u = np.ascontiguousarray(u, dtype=np.float64)
        b = np.zeros_like(u)
        self._call("rhs", ctypes.byref(s), m, _p(u), _p(b))
        return b

    def gmres(self, s, b):
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.zeros_like(b)
        it, conv, nh = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        hist = np.zeros(4096)
        self._call("gmres", ctypes.byref(s), _p(b), _p(x), ctypes.byref(it), ctypes.byref(conv),
                   _p(hist), 4096, ctypes.byref(nh))
        return x, it.value, bool(conv.value), hist[:nh.value].copy()

    def march(self, s, record=False):
        n1, n2 = dims_of(s)
        steps = s.steps or CONFIGS[s.cfg if s.cfg else 1][4]
        u = np.zeros(n1 * n2)
        its = np.zeros(steps, np.int32)
        res = np.zeros(steps)
        us = np.zeros((steps, n1 * n2)) if record else None
        wall = ctypes.c_double()
        self._march(s, u, its, res, us, wall)
        return dict(u=u, its=its, res=res, u_steps=us, wall=wall.value)

    def time_apply(self, s, reps):
        sec = np.zeros(reps)
        self._call("time_apply", ctypes.byref(s), reps, _p(sec))
        return sec

    def time_vcycle(self, s, reps):
        sec = np.zeros(reps)
        self._call("time_vcycle", ctypes.byref(s), reps, _p(sec))
        return sec


class Oracle(_Checker):
    prefix = "orc_"

    _solver = 0

    def _march(self, s, u, its, res, us, wall):
        self._call("march", ctypes.byref(s), self._solver, _p(u), its.ctypes.data_as(_I), _p(res),
                   _p(us) if us is not None else None, ctypes.byref(wall))

    def march(self, s, record=False, solver=0):
        """solver 0: GMRES(restart) (reference), 1: BiCGSTAB (extension)."""
        self._solver = solver
        try:
            return super().march(s, record)
        finally:
            self._solver = 0

    def bicgstab(self, s, b):
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.zeros_like(b)
        it, conv, nh = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        hist = np.zeros(8192)
        self._call("bicgstab", ctypes.byref(s), _p(b), _p(x), ctypes.byref(it), ctypes.byref(conv),
                   _p(hist), 8192, ctypes.byref(nh))
        return x, it.value, bool(conv.value), hist[:nh.value].copy()

    def fft(self, a, inverse=False):
        a = np.ascontiguousarray(a, dtype=np.complex128).copy()
        self._call("fft", len(a), a.ctypes.data_as(_P), int(inverse))
        return a

    def naive_dft(self, a, inverse=False):
        a = np.ascontiguousarray(a, dtype=np.complex128)
        out = np.zeros_like(a)
        self._call("naive_dft", len(a), a.ctypes.data_as(_P), out.ctypes.data_as(_P), int(inverse))
        return out


class RefLib(_Checker):
    prefix = "ref_"

    def _march(self, s, u, its, res, us, wall):
        self._call("march", ctypes.byref(s), _p(u), its.ctypes.data_as(_I), _p(res),
                   _p(us) if us is not None else None, ctypes.byref(wall))

    def march_timed(self, s):
        """Per-step loop of time_march with per-step wall times (setup excluded)."""
        n1, n2 = dims_of(s)
        steps = s.steps or CONFIGS[s.cfg][4]
        u, its, res = np.zeros(n1 * n2), np.zeros(steps, np.int32), np.zeros(steps)
        sec, wall = np.zeros(steps), ctypes.c_double()
        self._call("march_timed", ctypes.byref(s), _p(u), its.ctypes.data_as(_I), _p(res), None,
                   ctypes.byref(wall), _p(sec))
        return dict(u=u, its=its, res=res, step_seconds=sec, wall=wall.value)

    def time_march(self, s):
        n1, n2 = dims_of(s)
        steps = s.steps or CONFIGS[s.cfg][4]
        u, its, res, wall = np.zeros(n1 * n2), np.zeros(steps, np.int32), np.zeros(steps), ctypes.c_double()
        self._call("time_march", ctypes.byref(s), _p(u), its.ctypes.data_as(_I), _p(res), ctypes.byref(wall))
        return dict(u=u, its=its, res=res, wall=wall.value)

    def error_inf(self, s, u, t):
        u = np.ascontiguousarray(u, dtype=np.float64)
        e = ctypes.c_double()
        self._call("error_inf", ctypes.byref(s), _p(u), ctypes.c_double(t), ctypes.byref(e))
        return e.value

    def dense(self, s):
        n1, n2 = dims_of(s)
        n = n1 * n2
        a = np.zeros(n * n)
        self._call("dense", ctypes.byref(s), _p(a))
        return a.reshape(n, n, order="F")


class Adapter(_Checker):
    prefix = "adapter_"

    def gmres(self, s, b, gpu_op: bool, gpu_pc: bool):
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.zeros_like(b)
        it, conv, nh = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        hist = np.zeros(4096)
        self._call("gmres", ctypes.byref(s), int(gpu_op), int(gpu_pc), _p(b), _p(x),
                   ctypes.byref(it), ctypes.byref(conv), _p(hist), 4096, ctypes.byref(nh))
        return x, it.value, bool(conv.value), hist[:nh.value].copy()

    def march(self, s):
        n1, n2 = dims_of(s)
        steps = s.steps or CONFIGS[s.cfg if s.cfg else 1][4]
        u, its, res = np.zeros(n1 * n2), np.zeros(steps, np.int32), np.zeros(steps)
        self._call("march", ctypes.byref(s), _p(u), its.ctypes.data_as(_I), _p(res))
        return dict(u=u, its=its, res=res)


def build_oracle() -> None:
    """Build oracle/liboracle.so (and oracle/_ref when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", str(ORACLE_DIR), "oracle"], check=True)
    if Path(os.environ.get("FDE_REFERENCE", "/root/reference/proj")).exists():
        subprocess.run(["make", "-s", "-C", str(ORACLE_DIR), "ref"], check=True)
        subprocess.run(["make", "-s", "-C", str(ORACLE_DIR), "adapter"], check=True)


def oracle() -> Oracle:
    if not ORACLE_SO.exists():
        subprocess.run(["make", "-s", "-C", str(ORACLE_DIR), "oracle"], check=True)
    return Oracle(ORACLE_SO)


def reflib() -> RefLib | None:
    return RefLib(REF_SO) if REF_SO.exists() else None


def adapter() -> Adapter | None:
    return Adapter(ADAPTER_SO) if ADAPTER_SO.exists() else None
