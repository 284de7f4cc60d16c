"""TEST INFRASTRUCTURE ONLY — ctypes bindings to the CPU oracle.

`Oracle` wraps oracle/_build/libpsw_oracle.so (the C restatement,
psw_oracle.c) and `Reference` wraps oracle/_ref/libpsw_ref.so (the
unmodified reference headers compiled by oracle/Makefile). Both expose the
same numpy-level API so tests can run every check against either.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
`--impl reference`) may import this module. The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libpsw_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libpsw_ref.so")            # parity build (no FP contraction)
REF_PERF_SO = os.path.join(HERE, "_ref", "libpsw_ref_perf.so")  # CMake Release flags, CPU baseline

OK, INVALID_ARGUMENT, PIVOT_BREAKDOWN, TOO_MANY_PES, NOT_SUPPORTED = 0, 1, 2, 3, 4
NOT_SYMMETRIZABLE, ORACLE_FALLBACK = 8, 9
# GRowStrategy (dichotomy/preliminary.hpp:18-24)
AUTO, DIRECT_SYMMETRIC, SYMMETRIZE, EXPLICIT_INVERSE, TRANSPOSE_SOLVE = 0, 1, 2, 3, 4

_d = C.POINTER(C.c_double)
_i64 = C.POINTER(C.c_int64)
_u64 = C.POINTER(C.c_uint64)


class OracleError(RuntimeError):
    def __init__(self, code: int, index: int = -1):
        super().__init__(f"oracle status {code} (index {index})")
        self.code = code
        self.index = index


def build(ref: bool | None = None) -> None:
    """Compile the restatement (and the reference shim when headers exist)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    if ref is None:
        ref = os.path.isdir("/root/reference/proj/include")
    if ref:
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


def _dp(a: np.ndarray):
    return a.ctypes.data_as(_d)


def _ip(a: np.ndarray):
    return a.ctypes.data_as(_i64)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


class _Base:
    prefix = "orc_"

    def __init__(self, path: str):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle` (and `make -C oracle ref`)")
        self.lib = C.CDLL(path)
        L, p = self.lib, self.prefix
        self._thomas = getattr(L, p + "thomas")
        self._thomas.argtypes = [C.c_int64, _d, _d, _d, _d, _d, _i64]
        self._decompose = getattr(L, p + "decompose")
        self._decompose.argtypes = [C.c_int64, C.c_int64, _i64]
        self._levels = getattr(L, p + "level_sets")
        self._levels.argtypes = [C.c_int64, _i64, _i64]
        self._levels.restype = C.c_int64
        self._prelim = getattr(L, p + "preliminary")
        self._prelim.argtypes = [C.c_int64, _d, _d, _d, C.c_int64, _i64, _d, _d, _d, _d, _i64]
        self._batch = getattr(L, p + "solve_batch")
        self._batch.argtypes = [C.c_int64, _d, _d, _d, C.c_int64, _i64, C.c_int64, _d, C.c_int64,
                                _d, C.c_int64, _i64]
        self._prelim_ex = getattr(L, p + "preliminary_ex")
        self._prelim_ex.argtypes = [C.c_int64, _d, _d, _d, C.c_int64, _i64, C.c_int,
                                    C.POINTER(C.c_int), _d, _d, _d, _d, _i64]
        self._batch_ex = getattr(L, p + "solve_batch_ex")
        self._batch_ex.argtypes = [C.c_int64, _d, _d, _d, C.c_int64, _i64, C.c_int, C.c_int64, _d,
                                   C.c_int64, _d, C.c_int64, _i64]

    @staticmethod
    def _check(rc: int, bad: np.ndarray | None = None):
        if rc != OK:
            raise OracleError(rc, int(bad[0]) if bad is not None else -1)

    def thomas(self, sub, diag, sup, f):
        sub, diag, sup, f = map(_f64, (sub, diag, sup, f))
        n = diag.size
        x = np.empty(n)
        bad = np.zeros(1, np.int64)
        self._check(self._thomas(n, _dp(sub), _dp(diag), _dp(sup), _dp(f), _dp(x), _ip(bad)), bad)
        return x

    def decompose(self, n: int, P: int) -> np.ndarray:
        b = np.zeros(max(P - 1, 1), np.int64)
        rc = self._decompose(n, P, _ip(b))
        if rc != OK:
            raise OracleError(rc)
        return b[: P - 1].copy()

    def level_sets(self, p: int) -> list[list[int]]:
        order = np.zeros(max(p, 1), np.int64)
        off = np.zeros(72, np.int64)
        depth = self._levels(p, _ip(order), _ip(off))
        return [order[off[l]: off[l + 1]].tolist() for l in range(depth)]

    def preliminary(self, sub, diag, sup, bnd, strategy: int = AUTO):
        sub, diag, sup = map(_f64, (sub, diag, sup))
        bnd = np.ascontiguousarray(bnd, dtype=np.int64)
        n, p = diag.size, bnd.size
        g = np.zeros((max(p, 1), n))
        zr = np.zeros((max(p, 1), max(p, 1)))
        zl = np.zeros_like(zr)
        mz = np.zeros(1)
        bad = np.zeros(1, np.int64)
        used = C.c_int(-1)
        rc = self._prelim_ex(n, _dp(sub), _dp(diag), _dp(sup), p, _ip(bnd), strategy,
                             C.byref(used), _dp(g), _dp(zr), _dp(zl), _dp(mz), _ip(bad))
        self._check(rc, bad)
        return {"g": g[:p], "zr": zr[:p, :p], "zl": zl[:p, :p], "max_z": float(mz[0]),
                "strategy_used": int(used.value)}

    def solve_batch(self, sub, diag, sup, bnd, F, strategy: int = AUTO):
        """F: (N, n) system-contiguous series; returns X (N, n)."""
        sub, diag, sup = map(_f64, (sub, diag, sup))
        F = _f64(F)
        bnd = np.ascontiguousarray(bnd, dtype=np.int64)
        N, n = F.shape
        X = np.empty_like(F)
        bad = np.zeros(1, np.int64)
        rc = self._batch_ex(n, _dp(sub), _dp(diag), _dp(sup), bnd.size, _ip(bnd), strategy, N,
                            _dp(F), n, _dp(X), n, _ip(bad))
        self._check(rc, bad)
        return X


class Oracle(_Base):
    """The C restatement (psw_oracle.c)."""

    prefix = "orc_"

    def __init__(self, path: str = ORACLE_SO):
        super().__init__(path)
        L = self.lib
        L.orc_betas.argtypes = [C.c_int64, C.c_int64, _i64, _d, _d, _d, _d]
        L.orc_betas.restype = None
        L.orc_solve_boundaries.argtypes = [C.c_int64, _d, _d, _d, _d, _d, _u64]
        L.orc_solve_boundaries.restype = None
        L.orc_solve_boundaries_two_sided.argtypes = [C.c_int64, _d, _d, _d, _d, _d, _u64]
        L.orc_solve_boundaries_two_sided.restype = None
        L.orc_solve_local.argtypes = [C.c_int64, _d, _d, _d, C.c_int64, _i64, C.c_int64, _d,
                                      C.c_int, C.c_double, C.c_int, C.c_double, _d, _i64]
        L.orc_solve_batch_threads.argtypes = [C.c_int64, _d, _d, _d, C.c_int64, _i64, C.c_int64,
                                              _d, C.c_int64, _d, C.c_int64, C.c_int, _d, _d, _i64]
        L.orc_comm_rounds.argtypes = [C.c_int64]
        L.orc_comm_rounds.restype = C.c_uint64
        L.orc_partition_validate.argtypes = [C.c_int64, C.c_int64, _i64]
        L.orc_fill_uniform.argtypes = [_d, C.c_int64, C.c_uint64, C.c_uint64, C.c_double, C.c_double]
        L.orc_fill_uniform.restype = None

    def betas(self, bnd, g, f):
        bnd = np.ascontiguousarray(bnd, dtype=np.int64)
        f = _f64(f)
        g = _f64(g) if g.size else np.zeros(1)
        p, n = bnd.size, f.size
        left, right = np.zeros(p + 1), np.zeros(p + 1)
        self.lib.orc_betas(n, p, _ip(bnd), _dp(g), _dp(f), _dp(left), _dp(right))
        return left, right

    def solve_boundaries(self, zr, zl, left, right, two_sided: bool = False):
        p = zr.shape[0]
        zr, zl, left, right = map(_f64, (zr, zl, left, right))
        if p == 0:
            return np.zeros(0), 0
        v = np.zeros(p)
        terms = C.c_uint64(0)
        fn = self.lib.orc_solve_boundaries_two_sided if two_sided else self.lib.orc_solve_boundaries
        fn(p, _dp(zr), _dp(zl), _dp(left), _dp(right), _dp(v), C.byref(terms))
        return v, int(terms.value)

    def solve_local(self, sub, diag, sup, bnd, t, f, first=None, last=None):
        sub, diag, sup, f = map(_f64, (sub, diag, sup, f))
        bnd = np.ascontiguousarray(bnd, dtype=np.int64)
        n, p = diag.size, bnd.size
        lo = 1 if t == 0 else int(bnd[t - 1])
        hi = n if t == p else int(bnd[t])
        out = np.zeros(hi - lo + 1)
        bad = np.zeros(1, np.int64)
        rc = self.lib.orc_solve_local(n, _dp(sub), _dp(diag), _dp(sup), p, _ip(bnd), t, _dp(f),
                                      int(first is not None), float(first or 0.0),
                                      int(last is not None), float(last or 0.0), _dp(out), _ip(bad))
        self._check(rc, bad)
        return out

    def solve_batch_threads(self, sub, diag, sup, bnd, F, nthreads: int):
        sub, diag, sup = map(_f64, (sub, diag, sup))
        F = _f64(F)
        bnd = np.ascontiguousarray(bnd, dtype=np.int64)
        N, n = F.shape
        X = np.empty_like(F)
        su, so = C.c_double(0), C.c_double(0)
        bad = np.zeros(1, np.int64)
        rc = self.lib.orc_solve_batch_threads(n, _dp(sub), _dp(diag), _dp(sup), bnd.size, _ip(bnd),
                                              N, _dp(F), n, _dp(X), n, nthreads, C.byref(su),
                                              C.byref(so), _ip(bad))
        self._check(rc, bad)
        return X, su.value, so.value

    def comm_rounds(self, p: int) -> int:
        return int(self.lib.orc_comm_rounds(p))

    def validate(self, n, bnd) -> bool:
        bnd = np.ascontiguousarray(bnd, dtype=np.int64)
        return self.lib.orc_partition_validate(n, bnd.size, _ip(bnd)) == OK

    def fill_uniform(self, count: int, seed: int, lo: float, hi: float, offset: int = 0):
        out = np.empty(count)
        self.lib.orc_fill_uniform(_dp(out), count, seed, offset, lo, hi)
        return out


class Reference(_Base):
    """The reference itself, compiled from /root/reference headers (oracle/_ref)."""

    prefix = "ref_"

    def __init__(self, path: str = REF_SO):
        super().__init__(path)
        L = self.lib
        L.ref_betas_boundaries.argtypes = [C.c_int64, _d, _d, _d, C.c_int64, _i64, _d, _d, _d, _d,
                                           _u64, _i64]
        L.ref_run_batch.argtypes = [C.c_int, C.c_int64, C.c_int64, _d, _d, _d, C.c_int64, _i64,
                                    C.c_int64, _d, C.c_int64, _d, C.c_int64, C.c_char_p,
                                    C.c_int64, _i64]
        L.ref_solve_rhs_parallel.argtypes = [C.c_int64, _d, _d, _d, C.c_int64, _i64, C.c_int64,
                                             _d, C.c_int64, _d, C.c_int64, C.c_int, _d, _d, _i64]
        L.ref_hardware_concurrency.restype = C.c_int
        L.ref_adi_iteration_bound.argtypes = [C.c_int64, C.c_double]
        L.ref_adi_iteration_bound.restype = C.c_int64
        L.ref_adi_parameters.argtypes = [C.c_int64, C.c_int64, C.c_double, C.c_double, C.c_int64,
                                         C.c_int64, _d]
        L.ref_adi_steps.argtypes = [C.c_int64, C.c_int64, C.c_double, C.c_double, C.c_int64,
                                    C.c_int64, _d, _d, C.c_int64]
        L.ref_adi_solve.argtypes = [C.c_int64, C.c_int64, C.c_double, C.c_double, C.c_int64,
                                    C.c_int64, C.c_double, _d, _d, _d, _d, _i64]
        L.ref_model_problem.argtypes = [C.c_int64, C.c_int64, _d, _d]
        L.ref_fourier_solve.argtypes = [C.c_int64, C.c_int64, C.c_double, C.c_double, C.c_int64,
                                        _d, _d, _i64, _i64]

    # ---- poisson/adi.hpp (the ADI consumer) -------------
    def adi_iteration_bound(self, n: int, eps: float) -> int:
        return int(self.lib.ref_adi_iteration_bound(n, eps))

    def adi_parameters(self, n1, n2, h1, h2, cycle, pes=1):
        taus = np.zeros(max(cycle, 1))
        self._check(self.lib.ref_adi_parameters(n1, n2, h1, h2, cycle, pes, _dp(taus)))
        return taus

    def adi_steps(self, n1, n2, h1, h2, cycle, pes, f, u, steps):
        f, u = _f64(f), _f64(u).copy()
        self._check(self.lib.ref_adi_steps(n1, n2, h1, h2, cycle, pes, _dp(f), _dp(u), steps))
        return u

    def adi_solve(self, n1, n2, h1, h2, cycle, pes, eps, f, u0, exact=None):
        f, u0 = _f64(f), _f64(u0)
        u = np.empty_like(u0)
        its = np.zeros(1, np.int64)
        ex = _f64(exact) if exact is not None else None
        rc = self.lib.ref_adi_solve(n1, n2, h1, h2, cycle, pes, eps, _dp(f), _dp(u0),
                                    _dp(ex) if ex is not None else None, _dp(u), _ip(its))
        self._check(rc)
        return u, int(its[0])

    # ---- poisson/fourier.hpp (the Fourier consumer) -----
    def fourier_solve(self, n1, n2, h1, h2, pes, f):
        f = _f64(f)
        u = np.empty_like(f)
        bnd = np.zeros(max(n1, 1), np.int64)
        p = np.zeros(1, np.int64)
        self._check(self.lib.ref_fourier_solve(n1, n2, h1, h2, pes, _dp(f), _dp(u), _ip(bnd), _ip(p)))
        return u, bnd[: int(p[0])]

    def model_problem(self, n1, n2):
        f = np.zeros((n1 + 1, n2 + 1))
        ex = np.zeros_like(f)
        self.lib.ref_model_problem(n1, n2, _dp(f), _dp(ex))
        return f, ex

    def betas_boundaries(self, sub, diag, sup, bnd, f):
        sub, diag, sup, f = map(_f64, (sub, diag, sup, f))
        bnd = np.ascontiguousarray(bnd, dtype=np.int64)
        n, p = diag.size, bnd.size
        left, right, v = np.zeros(p + 1), np.zeros(p + 1), np.zeros(max(p, 1))
        terms = C.c_uint64(0)
        bad = np.zeros(1, np.int64)
        rc = self.lib.ref_betas_boundaries(n, _dp(sub), _dp(diag), _dp(sup), p, _ip(bnd), _dp(f),
                                           _dp(left), _dp(right), _dp(v), C.byref(terms), _ip(bad))
        self._check(rc, bad)
        return left, right, v[:p], int(terms.value)

    def run_batch(self, sub, diag, sup, bnd, F, threaded: bool = False, workers: int = 1):
        import json
        sub, diag, sup = map(_f64, (sub, diag, sup))
        F = _f64(F)
        bnd = np.ascontiguousarray(bnd, dtype=np.int64)
        N, n = F.shape
        X = np.empty_like(F)
        buf = C.create_string_buffer(256)
        bad = np.zeros(1, np.int64)
        rc = self.lib.ref_run_batch(int(threaded), workers, n, _dp(sub), _dp(diag), _dp(sup),
                                    bnd.size, _ip(bnd), N, _dp(F), n, _dp(X), n, buf, 256, _ip(bad))
        self._check(rc, bad)
        return X, json.loads(buf.value.decode())

    def solve_rhs_parallel(self, sub, diag, sup, bnd, F, nthreads: int):
        sub, diag, sup = map(_f64, (sub, diag, sup))
        F = _f64(F)
        bnd = np.ascontiguousarray(bnd, dtype=np.int64)
        N, n = F.shape
        X = np.empty_like(F)
        su, so = C.c_double(0), C.c_double(0)
        bad = np.zeros(1, np.int64)
        rc = self.lib.ref_solve_rhs_parallel(n, _dp(sub), _dp(diag), _dp(sup), bnd.size, _ip(bnd),
                                             N, _dp(F), n, _dp(X), n, nthreads, C.byref(su),
                                             C.byref(so), _ip(bad))
        self._check(rc, bad)
        return X, su.value, so.value

    def hardware_concurrency(self) -> int:
        return int(self.lib.ref_hardware_concurrency())

    def plan(self, sub, diag, sup, bnd, workers: int = 1) -> "RefPlan":
        """compute_preliminary once (on a WorkerPool of `workers`), then
        RefPlan.solve(F, nthreads) over disjoint RHS slices."""
        return RefPlan(self, sub, diag, sup, bnd, workers)


class RefPlan:
    def __init__(self, ref: "Reference", sub, diag, sup, bnd, workers: int):
        sub, diag, sup = map(_f64, (sub, diag, sup))
        bnd = np.ascontiguousarray(bnd, dtype=np.int64)
        L = ref.lib
        L.ref_plan_create.restype = C.c_void_p
        L.ref_plan_create.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
                                      C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]
        L.ref_plan_solve.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p,
                                     C.c_int64, C.c_int, C.c_void_p, C.c_void_p]
        L.ref_plan_destroy.argtypes = [C.c_void_p]
        self.lib, self.n = L, diag.size
        su = C.c_double(0)
        bad = np.zeros(1, np.int64)
        self.h = L.ref_plan_create(diag.size, _dp(sub), _dp(diag), _dp(sup), bnd.size, _ip(bnd),
                                   workers, C.byref(su), _ip(bad))
        if not self.h:
            raise OracleError(-1, int(bad[0]))
        self.setup_s = su.value

    def solve(self, F, nthreads: int = 1):
        """Returns (X, solve seconds)."""
        F = _f64(F)
        N, n = F.shape
        X = np.empty_like(F)
        so = C.c_double(0)
        bad = np.zeros(1, np.int64)
        rc = self.lib.ref_plan_solve(self.h, N, _dp(F), n, _dp(X), n, nthreads, C.byref(so),
                                     _ip(bad))
        if rc != 0:
            raise OracleError(rc, int(bad[0]))
        return X, so.value

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.ref_plan_destroy(self.h)
            self.h = None


def reference_available() -> bool:
    return os.path.exists(REF_SO)
