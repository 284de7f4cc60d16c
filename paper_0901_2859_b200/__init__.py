"""parsweep_b200 — B200-native batched dichotomy tridiagonal solver.

Python mirror of the reference `parsweep` hot-path API (C++20 header-only,
/root/reference/proj/include/parsweep) over the C ABI in
include/parsweep_b200.h. Names, argument meaning and error behaviour follow
the reference so parity tests read like its own tests:

    reference (C++)                              this package
    -------------------------------------------  ---------------------------------
    TridiagMatrix (core/tridiag.hpp:31-67)       TridiagMatrix
    Partition (dichotomy/partition.hpp:16-73)    Partition
    decompose(n,p).induced_partition()           decompose(n, P).induced_partition()
      (runtime/decompose.hpp:23-47)
    compute_preliminary(A, part)                 compute_preliminary(A, part, dtype=, device=)
      (dichotomy/preliminary.hpp:171-199)          -> Plan (resident in HBM)
    solve_with_preliminary_into / solve_batch    Plan.solve(F, X) on CUDA tensors,
      (dichotomy/batch.hpp:20-75)                  solve_batch(A, part, series) on host data
    SolverError, PivotBreakdown, TooManyPEs      same names (core/errors.hpp:9-62)

The product path is the CUDA library only: there is no CPU fallback, and
every call fails loudly when the extension or a GPU is missing.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

__all__ = [
    "TridiagMatrix", "Partition", "Decomposition", "decompose", "compute_preliminary", "Plan",
    "solve_batch", "solve_multi", "MultiPlan", "SolverError", "PivotBreakdown", "TooManyPEs", "NotSupported", "NotSymmetrizable", "OracleFallbackRequired", "CudaError",
    "F64", "F32", "LAYOUT_R", "LAYOUT_S", "PATH_AUTO", "PATH_STAGED", "PATH_FUSED", "PATH_CHUNKED",
    "PATH_RESWEEP", "PATH_CLUSTER", "PATH_HOLD", "last_path", "lib", "library_path", "Comm", "NcclError",
]

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_lib", "libparsweep_b200.so")
if os.environ.get("PSW_LIB_VARIANT"):  # experiments: _lib/<variant>/ built with other constants
    LIB_PATH = os.path.join(HERE, "_lib", os.environ["PSW_LIB_VARIANT"], "libparsweep_b200.so")

F64, F32 = 0, 1
LAYOUT_R, LAYOUT_S = 0, 1
PATH_AUTO, PATH_STAGED, PATH_FUSED, PATH_CHUNKED, PATH_RESWEEP, PATH_CLUSTER = 0, 1, 2, 5, 6, 7
PATH_HOLD = 8
OK, INVALID_ARGUMENT, PIVOT_BREAKDOWN, TOO_MANY_PES, NOT_SUPPORTED, CUDA_ERROR, NCCL_ERROR, OOM = range(8)
NOT_SYMMETRIZABLE, ORACLE_FALLBACK_REQUIRED = 8, 9
# GRowStrategy (dichotomy/preliminary.hpp:18-24)
GROW_AUTO, GROW_DIRECT_SYMMETRIC, GROW_SYMMETRIZE, GROW_EXPLICIT_INVERSE, GROW_TRANSPOSE_SOLVE = range(5)


# ---------------------------------------------------------------- errors
class SolverError(RuntimeError):
    """core/errors.hpp:9-12"""


class PivotBreakdown(SolverError):
    """core/errors.hpp:16-22 — carries the failing row."""

    def __init__(self, row: int, msg: str | None = None):
        super().__init__(msg or f"pivot breakdown during forward elimination at row {row}")
        self.row = row


class TooManyPEs(SolverError):
    """core/errors.hpp:42-47"""


class NotSymmetrizable(SolverError):
    """core/errors.hpp:29-38 (index = the failing off-diagonal k)"""

    def __init__(self, index: int, msg: str | None = None):
        super().__init__(msg or f"off-diagonal product sub[{index}]*super[{index}] is not positive")
        self.index = index


class OracleFallbackRequired(SolverError):
    """core/errors.hpp:40-43"""


class NotSupported(SolverError):
    pass


class CudaError(SolverError):
    pass


class NcclError(SolverError):
    """PSW_NCCL_ERROR: NCCL missing or a collective of the row-sharded solve failed."""


# ---------------------------------------------------------------- library
_lib = None


def library_path() -> str:
    return LIB_PATH


def lib() -> C.CDLL:
    """Load the in-tree CUDA library; raises if it was not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `make -C paper_0901_2859_b200/csrc` "
                "(or __graft_entry__.build()); there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        d, i64, vp = C.POINTER(C.c_double), C.POINTER(C.c_int64), C.c_void_p
        L.psw_last_error_message.restype = C.c_char_p
        L.psw_last_error_index.restype = C.c_int64
        L.psw_last_launch_count.restype = C.c_int64
        L.psw_last_path.restype = C.c_int
        L.psw_debug_trace.argtypes = [vp]
        L.psw_decompose.argtypes = [C.c_int64, C.c_int64, i64]
        L.psw_partition_validate.argtypes = [C.c_int64, C.c_int64, i64]
        L.psw_plan_create.argtypes = [C.POINTER(vp), C.c_int64, d, d, d, C.c_int64, i64, C.c_int, C.c_int]
        L.psw_plan_create_flags.argtypes = [C.POINTER(vp), C.c_int64, d, d, d, C.c_int64, i64,
                                            C.c_int, C.c_int, C.c_int, C.c_int]
        L.psw_plan_create_ex.argtypes = [C.POINTER(vp), C.c_int64, d, d, d, C.c_int64, i64, C.c_int,
                                         C.c_int, C.c_int]
        L.psw_shard_plan_create.argtypes = [C.POINTER(vp), C.c_int64, d, d, d, C.c_int64, i64,
                                            C.c_int, C.c_int, C.c_int, C.c_int]
        L.psw_plan_destroy.argtypes = [vp]
        L.psw_plan_info.argtypes = [vp, vp]
        L.psw_solve.argtypes = [vp, vp, C.c_int64, vp, C.c_int64, C.c_int64, C.c_int, vp]
        L.psw_solve_ex.argtypes = [vp, vp, C.c_int64, vp, C.c_int64, C.c_int64, C.c_int, vp, vp]
        L.psw_solve_host.argtypes = [vp, vp, C.c_int64, vp, C.c_int64, C.c_int64, C.c_int]
        L.psw_solve_multi.argtypes = [C.POINTER(vp), C.c_int64, vp, C.c_int64, vp, C.c_int64, vp]
        L.psw_dst_rows.argtypes = [vp, C.c_int64, vp, C.c_int64, C.c_int64, C.c_int64, C.c_double, vp]
        L.psw_multi_create.argtypes = [C.POINTER(vp), C.POINTER(vp), C.c_int64]
        L.psw_multi_destroy.argtypes = [vp]
        L.psw_multi_destroy.restype = None
        L.psw_multi_solve.argtypes = [vp, vp, C.c_int64, vp, C.c_int64, vp]
        L.psw_shard_partials_count.argtypes = [vp]
        L.psw_shard_partials_count.restype = C.c_int64
        L.psw_shard_row_offset.argtypes = [vp]
        L.psw_shard_row_offset.restype = C.c_int64
        L.psw_shard_rows.argtypes = [vp]
        L.psw_shard_rows.restype = C.c_int64
        L.psw_shard_workspace_bytes.argtypes = [vp, C.c_int64]
        L.psw_shard_workspace_bytes.restype = C.c_int64
        L.psw_shard_forward.argtypes = [vp, vp, C.c_int64, C.c_int64, vp, vp, vp]
        L.psw_shard_backward.argtypes = [vp, vp, C.c_int64, vp, C.c_int64, C.c_int64, vp, vp, vp]
        L.psw_shard_solve.argtypes = [vp, vp, C.c_int64, vp, C.c_int64, C.c_int64, vp, vp]
        L.psw_comm_unique_id.argtypes = [vp]
        L.psw_comm_create.argtypes = [C.POINTER(vp), C.c_int, C.c_int, vp, C.c_int]
        L.psw_comm_destroy.argtypes = [vp]
        L.psw_fill_uniform.argtypes = [vp, C.c_int, C.c_int64, C.c_uint64, C.c_uint64, C.c_double,
                                       C.c_double, vp]
        L.psw_fill_normal.argtypes = [vp, C.c_int, C.c_int64, C.c_uint64, C.c_uint64, vp]
        L.psw_l2_flush.argtypes = [vp, C.c_int64, vp]
        _lib = L
    return _lib


def _raise(rc: int):
    L = lib()
    msg = (L.psw_last_error_message() or b"").decode()
    idx = int(L.psw_last_error_index())
    if rc == INVALID_ARGUMENT:
        raise ValueError(msg)  # std::invalid_argument
    if rc == PIVOT_BREAKDOWN:
        raise PivotBreakdown(idx, msg)
    if rc == TOO_MANY_PES:
        raise TooManyPEs(msg)
    if rc == NOT_SUPPORTED:
        raise NotSupported(msg)
    if rc == NOT_SYMMETRIZABLE:
        raise NotSymmetrizable(idx, msg)
    if rc == ORACLE_FALLBACK_REQUIRED:
        raise OracleFallbackRequired(msg)
    if rc == OOM:
        raise MemoryError(msg)
    if rc == NCCL_ERROR:
        raise NcclError(msg)
    raise CudaError(f"status {rc}: {msg}")


def _check(rc: int):
    if rc != OK:
        _raise(rc)


def last_launch_count() -> int:
    return int(lib().psw_last_launch_count())


PATH_NAMES = {PATH_STAGED: "staged", PATH_FUSED: "fused", PATH_CHUNKED: "chunked",
              PATH_RESWEEP: "resweep", PATH_CLUSTER: "cluster", PATH_HOLD: "hold"}


def last_path() -> str:
    """Name of the solve path the last solve on this thread took."""
    return PATH_NAMES.get(int(lib().psw_last_path()), "none")


# ---------------------------------------------------------------- types
@dataclass
class TridiagMatrix:
    """core/tridiag.hpp:31-67: sub = a_2..a_n, diag = b_1..b_n, super = c_1..c_{n-1}."""

    sub: np.ndarray
    diag: np.ndarray
    super: np.ndarray

    def __post_init__(self):
        self.sub = np.ascontiguousarray(self.sub, dtype=np.float64)
        self.diag = np.ascontiguousarray(self.diag, dtype=np.float64)
        self.super = np.ascontiguousarray(self.super, dtype=np.float64)

    def n(self) -> int:
        return int(self.diag.size)

    def is_symmetric(self) -> bool:  # tridiag.hpp:43 (exact compare)
        return bool(np.array_equal(self.sub, self.super))

    @staticmethod
    def constant(n: int, a: float, b: float, c: float) -> "TridiagMatrix":
        return TridiagMatrix(np.full(n - 1, a), np.full(n, b), np.full(n - 1, c))

    @staticmethod
    def symmetric(a: np.ndarray, b: np.ndarray) -> "TridiagMatrix":
        a = np.ascontiguousarray(a, dtype=np.float64)
        return TridiagMatrix(a, b, a.copy())

    def validate(self):  # tridiag.hpp:57-66
        n = self.n()
        if n < 2:
            raise ValueError("TridiagMatrix: order must be >= 2")
        if self.sub.size != n - 1 or self.super.size != n - 1:
            raise ValueError("TridiagMatrix: off-diagonal lengths must be n-1")
        if not (np.isfinite(self.sub).all() and np.isfinite(self.diag).all() and np.isfinite(self.super).all()):
            raise ValueError("TridiagMatrix: entries must be finite")

    def mat_vec(self, x: np.ndarray) -> np.ndarray:  # tridiag.hpp:70-80
        y = self.diag * x
        y[1:] += self.sub * x[:-1]
        y[:-1] += self.super * x[1:]
        return y


@dataclass
class Partition:
    """dichotomy/partition.hpp:16-73 — 1-based interior boundaries."""

    n: int
    boundaries: list[int] = field(default_factory=list)

    def p(self) -> int:
        return len(self.boundaries)

    def blocks(self) -> int:
        return len(self.boundaries) + 1

    def block_begin(self, t: int) -> int:
        return 1 if t == 0 else self.boundaries[t - 1]

    def block_end(self, t: int) -> int:
        return self.n + 1 if t == self.p() else self.boundaries[t]

    def validate(self):
        b = np.ascontiguousarray(self.boundaries, dtype=np.int64)
        _check(lib().psw_partition_validate(self.n, b.size, b.ctypes.data_as(C.POINTER(C.c_int64))))

    def to_string(self) -> str:
        return ",".join(str(b) for b in self.boundaries)

    @staticmethod
    def parse(n: int, text: str) -> "Partition":
        items = []
        for item in text.split(","):
            if not item.strip():
                continue
            try:
                v = int(item)
            except ValueError:
                raise ValueError(f"Partition: bad boundary '{item}'") from None
            if v < 0:
                raise ValueError(f"Partition: bad boundary '{item}'")
            items.append(v)
        part = Partition(n, items)
        part.validate()
        return part


@dataclass
class Decomposition:
    """runtime/decompose.hpp:16-30"""

    n: int
    ranges: list[tuple[int, int]]

    def p(self) -> int:
        return len(self.ranges)

    def induced_partition(self) -> Partition:
        return Partition(self.n, [hi for (_, hi) in self.ranges[:-1]])


def decompose(n: int, P: int) -> Decomposition:
    """runtime/decompose.hpp:33-47 via psw_decompose (raises TooManyPEs)."""
    b = np.zeros(max(P - 1, 1), np.int64)
    _check(lib().psw_decompose(n, P, b.ctypes.data_as(C.POINTER(C.c_int64))))
    ends = list(b[: P - 1]) + [n]
    ranges, lo = [], 1
    for hi in ends:
        ranges.append((lo, int(hi)))
        lo = int(hi) + 1
    return Decomposition(n, ranges)


class _Info(C.Structure):
    _fields_ = [("n", C.c_int64), ("p", C.c_int64), ("dtype", C.c_int32), ("device", C.c_int32),
                ("uniform", C.c_int32), ("fused_ok", C.c_int32), ("device_bytes", C.c_int64),
                ("combine_terms", C.c_int64), ("comm_rounds", C.c_int64),
                ("setup_seconds", C.c_double), ("max_z_norm", C.c_double),
                ("strategy_used", C.c_int32), ("device_setup", C.c_int32)]


class _Opts(C.Structure):
    _fields_ = [("path", C.c_int32), ("nevents", C.c_int32), ("betas_left", C.c_void_p),
                ("betas_right", C.c_void_p), ("boundary_values", C.c_void_p),
                ("events", C.c_void_p)]


def _ptr(t) -> int:
    """Device (or host) address of a torch tensor / numpy array / int."""
    if t is None:
        return 0
    if isinstance(t, int):
        return t
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return int(t.data_ptr())


class Plan:
    """Device-resident preliminary data (the PreliminaryData of
    dichotomy/preliminary.hpp:53-101, restricted to what the kernels read)."""

    def __init__(self, A: TridiagMatrix, part: Partition, dtype: int = F64, device: int = 0,
                 rank: int | None = None, world: int | None = None,
                 strategy: int = GROW_AUTO, staged_only: bool = False):
        L = lib()
        A.validate() if A.n() >= 2 else None
        self.n = A.n()
        self.part = Partition(part.n, list(part.boundaries))
        self.dtype = dtype
        self.device = device
        shard = world is not None
        self._shard = shard
        self.rank, self.world = (rank or 0), (world or 1)
        b = np.ascontiguousarray(part.boundaries, dtype=np.int64)
        if b.size == 0:
            b = np.zeros(1, np.int64)
        dp = C.POINTER(C.c_double)
        h = C.c_void_p()
        args = (C.byref(h), self.n, A.sub.ctypes.data_as(dp), A.diag.ctypes.data_as(dp),
                A.super.ctypes.data_as(dp), len(part.boundaries),
                b.ctypes.data_as(C.POINTER(C.c_int64)), dtype, device)
        if not shard and staged_only:  # STAGED / multi-matrix solves only (cheap setup)
            _check(L.psw_plan_create_flags(*args, strategy, 1))
        elif not shard:
            _check(L.psw_plan_create_ex(*args, strategy))
        else:  # row shard of a multi-GPU solve (psw_shard_*)
            _check(L.psw_shard_plan_create(*args, self.rank, self.world))
        self._h = h
        info = _Info()
        _check(L.psw_plan_info(self._h, C.byref(info)))
        self.info = {k: getattr(info, k) for k, _ in _Info._fields_}

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                lib().psw_plan_destroy(h)
            except Exception:
                pass
            self._h = None

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def p(self) -> int:
        return self.part.p()

    # -- device-resident batched solve (psw_solve / psw_solve_ex) ----------
    def solve(self, F, X=None, *, nrhs: int | None = None, layout: int = LAYOUT_R,
              ldf: int | None = None, ldx: int | None = None, stream=None, path: int = PATH_AUTO,
              betas_left=None, betas_right=None, boundary_values=None, events=None):
        """Solve A X_k = F_k for every RHS in F (a CUDA tensor of the plan's
        dtype). layout R: F is (n, N) row-major [i*ld + k]; layout S: F is
        (N, n) [k*ld + i]. X defaults to F (in place)."""
        if X is None:
            X = F
        if layout not in (LAYOUT_R, LAYOUT_S):
            raise ValueError("layout must be LAYOUT_R or LAYOUT_S")
        self._check_device_tensor(F, "F")
        self._check_device_tensor(X, "X")
        if nrhs is None:
            nrhs = F.shape[1] if layout == LAYOUT_R else F.shape[0]
        if ldf is None:
            ldf = F.stride(0)
        if ldx is None:
            ldx = X.stride(0)
        for t, ld, name in ((F, ldf, "F"), (X, ldx, "X")):
            self._check_extent(t, ld, nrhs, layout, name)
        s = _stream_ptr(stream)
        opts = None
        if (path != PATH_AUTO or betas_left is not None or betas_right is not None
                or boundary_values is not None or events is not None):
            ev_arr = None
            if events is not None:
                ev_arr = (C.c_void_p * len(events))(*[e.cuda_event if hasattr(e, "cuda_event") else int(e)
                                                      for e in events])
            opts = _Opts(path, len(events) if events is not None else 0, _ptr(betas_left) or None,
                         _ptr(betas_right) or None, _ptr(boundary_values) or None,
                         C.cast(ev_arr, C.c_void_p) if ev_arr is not None else None)
            self._ev_keepalive = ev_arr
        rc = lib().psw_solve_ex(self._h, _ptr(F), ldf, _ptr(X), ldx, nrhs, layout, s,
                                C.byref(opts) if opts is not None else None)
        _check(rc)
        return X

    # -- argument checks (a wrong buffer must raise, never reach the kernels)
    def _check_device_tensor(self, t, name: str):
        import torch
        if not isinstance(t, torch.Tensor):
            raise ValueError(f"{name} must be a CUDA tensor")
        want = torch.float64 if self.dtype == F64 else torch.float32
        if t.dtype != want:
            raise ValueError(f"{name} has dtype {t.dtype}, the plan solves in {want}")
        if not t.is_cuda or t.device.index != self.device:
            raise ValueError(f"{name} must live on cuda:{self.device} (got {t.device})")
        if t.dim() != 2 or t.stride(-1) != 1:
            raise ValueError(f"{name} must be a 2-D tensor with unit inner stride")

    def _check_extent(self, t, ld: int, nrhs: int, layout: int, name: str):
        rows = self.rows() if self._shard else self.n
        if layout == LAYOUT_R:
            need_rows, need_cols = rows, nrhs
        else:
            need_rows, need_cols = nrhs, rows
        if nrhs < 0 or ld < need_cols:
            raise ValueError(f"{name}: leading dimension {ld} < {need_cols}")
        if nrhs == 0:
            return
        last = (need_rows - 1) * ld + need_cols  # elements the solve touches
        if t.shape[0] < need_rows or t.shape[1] < need_cols or \
                t.storage_offset() + last > t.untyped_storage().nbytes() // t.element_size():
            raise ValueError(f"{name} of shape {tuple(t.shape)} is too small for "
                             f"{need_rows} x {need_cols} (layout {'RS'[layout]})")

    def solve_host(self, F: np.ndarray, X: np.ndarray | None = None, layout: int = LAYOUT_S):
        """End-to-end solve on host arrays (psw_solve_host)."""
        dt = np.float64 if self.dtype == F64 else np.float32
        if layout not in (LAYOUT_R, LAYOUT_S):
            raise ValueError("layout must be LAYOUT_R or LAYOUT_S")
        if not isinstance(F, np.ndarray) or F.dtype != dt or not F.flags.c_contiguous or F.ndim != 2:
            raise ValueError("F must be a C-contiguous 2-D array of the plan dtype")
        if X is None:
            X = np.empty_like(F)
        if not isinstance(X, np.ndarray) or X.dtype != dt or not X.flags.c_contiguous or \
                X.shape != F.shape:
            raise ValueError("X must be a C-contiguous array of F's shape and the plan dtype")
        if (F.shape[0] if layout == LAYOUT_R else F.shape[1]) != self.n:
            raise ValueError(f"F must hold n = {self.n} rows per system "
                             f"({'rows' if layout == LAYOUT_R else 'columns'} of the array)")
        nrhs = F.shape[1] if layout == LAYOUT_R else F.shape[0]
        _check(lib().psw_solve_host(self._h, F.ctypes.data, F.shape[1], X.ctypes.data, X.shape[1],
                                    nrhs, layout))
        return X

    # -- row sharding (psw_shard_*) -----------------------------------------
    def partials_count(self) -> int:
        return int(lib().psw_shard_partials_count(self._h))

    def row_offset(self) -> int:
        return int(lib().psw_shard_row_offset(self._h))

    def rows(self) -> int:
        return int(lib().psw_shard_rows(self._h))

    def workspace_bytes(self, nrhs: int) -> int:
        return int(lib().psw_shard_workspace_bytes(self._h, nrhs))

    def shard_forward(self, F, nrhs: int, workspace, partials, stream=None):
        """K1 + fold + this rank's share of the p boundary values -> partials (p x nrhs fp64)."""
        self._check_device_tensor(F, "F")
        self._check_extent(F, F.stride(0), nrhs, LAYOUT_R, "F")
        _check(lib().psw_shard_forward(self._h, _ptr(F), F.stride(0), nrhs, _ptr(workspace),
                                       _ptr(partials), _stream_ptr(stream)))

    def shard_backward(self, F, X, nrhs: int, workspace, partials, stream=None):
        """Run carries from the reduced boundary values + the second sweep of F -> X."""
        self._check_device_tensor(F, "F")
        self._check_device_tensor(X, "X")
        self._check_extent(F, F.stride(0), nrhs, LAYOUT_R, "F")
        self._check_extent(X, X.stride(0), nrhs, LAYOUT_R, "X")
        _check(lib().psw_shard_backward(self._h, _ptr(F), F.stride(0), _ptr(X), X.stride(0), nrhs,
                                        _ptr(workspace), _ptr(partials), _stream_ptr(stream)))

    def shard_solve(self, F, X, comm: "Comm | None", nrhs: int | None = None, stream=None):
        """psw_shard_solve: forward, ncclAllReduce over `comm`, backward, on one stream."""
        self._check_device_tensor(F, "F")
        self._check_device_tensor(X, "X")
        if nrhs is None:
            nrhs = F.shape[1]
        self._check_extent(F, F.stride(0), nrhs, LAYOUT_R, "F")
        self._check_extent(X, X.stride(0), nrhs, LAYOUT_R, "X")
        _check(lib().psw_shard_solve(self._h, _ptr(F), F.stride(0), _ptr(X), X.stride(0), nrhs,
                                     comm.handle if comm is not None else None,
                                     _stream_ptr(stream)))
        return X


class Comm:
    """NCCL communicator of the row-sharded solve (psw_comm_*). `uid` is the
    128-byte id from Comm.unique_id() on rank 0, shared by the caller."""

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _check(lib().psw_comm_unique_id(buf))
        return buf.raw

    def __init__(self, nranks: int, rank: int, uid: bytes, device: int):
        if len(uid) != 128:
            raise ValueError("NCCL unique id must be 128 bytes")
        h = C.c_void_p()
        buf = C.create_string_buffer(uid, 128)
        _check(lib().psw_comm_create(C.byref(h), nranks, rank, buf, device))
        self._h = h
        self.nranks, self.rank, self.device = nranks, rank, device

    @property
    def handle(self):
        return self._h

    def close(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            lib().psw_comm_destroy(h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _stream_ptr(stream) -> int | None:
    if stream is None:
        try:
            import torch
            return torch.cuda.current_stream().cuda_stream
        except Exception:
            return None
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def compute_preliminary(A: TridiagMatrix, part: Partition, dtype: int = F64, device: int = 0) -> Plan:
    """dichotomy/preliminary.hpp:171-199 -> device-resident Plan."""
    return Plan(A, part, dtype=dtype, device=device)


def debug_preliminary(A: TridiagMatrix, part: Partition) -> dict:
    """Test hook (psw_debug_preliminary): the raw tables of the preliminary as
    plan creation produced them (host sweeps or the device kernels of
    psw_prelim.cu, by PSW_DEVICE_SETUP): gr / gl (g_j on blocks j / j+1),
    zr / zl (p x p samples), max_z, device_setup."""
    n, p = A.n(), part.p()
    dp = C.POINTER(C.c_double)
    L = lib()
    L.psw_debug_preliminary.restype = C.c_int
    L.psw_debug_preliminary.argtypes = [C.c_int64, dp, dp, dp, C.c_int64, C.POINTER(C.c_int64),
                                        dp, dp, dp, dp, dp, C.POINTER(C.c_int32)]
    sub = np.ascontiguousarray(A.sub, dtype=np.float64)
    diag = np.ascontiguousarray(A.diag, dtype=np.float64)
    sup = np.ascontiguousarray(A.super, dtype=np.float64)
    bnd = np.ascontiguousarray(part.boundaries, dtype=np.int64)
    gr, gl = np.zeros(n), np.zeros(n)
    zr, zl = np.zeros((max(p, 1), max(p, 1))), np.zeros((max(p, 1), max(p, 1)))
    mz, ds = C.c_double(0.0), C.c_int32(0)
    _check(L.psw_debug_preliminary(n, sub.ctypes.data_as(dp), diag.ctypes.data_as(dp),
                                   sup.ctypes.data_as(dp), p, bnd.ctypes.data_as(C.POINTER(C.c_int64)),
                                   gr.ctypes.data_as(dp), gl.ctypes.data_as(dp),
                                   zr.ctypes.data_as(dp), zl.ctypes.data_as(dp), C.byref(mz),
                                   C.byref(ds)))
    return {"gr": gr, "gl": gl, "zr": zr[:p, :p] if p else zr[:0, :0],
            "zl": zl[:p, :p] if p else zl[:0, :0], "max_z": mz.value, "device_setup": ds.value}


def solve_batch(A: TridiagMatrix, part: Partition, rhs_series: Sequence[Sequence[float]],
                dtype: int = F64, device: int = 0) -> list[np.ndarray]:
    """dichotomy/batch.hpp:57-75 on host data: validate, preliminary once,
    then the whole series on the GPU (psw_solve_host, layout S)."""
    part.validate()
    plan = Plan(A, part, dtype=dtype, device=device)
    dt = np.float64 if dtype == F64 else np.float32
    F = np.ascontiguousarray(np.asarray(rhs_series, dtype=dt).reshape(len(rhs_series), A.n()))
    X = plan.solve_host(F, layout=LAYOUT_S)
    return [X[k] for k in range(X.shape[0])]


def solve_multi(plans: Sequence["Plan"], F, X, stream=None):
    """psw_solve_multi: column k of the layout-R CUDA tensor F (n x ld) is
    solved with plans[k] into column k of X (the per-harmonic loop of
    poisson/fourier.hpp:157-164 as one pass)."""
    arr = (C.c_void_p * len(plans))(*[pl._h for pl in plans])
    _check(lib().psw_solve_multi(arr, len(plans), _ptr(F), F.stride(0), _ptr(X), X.stride(0),
                                 _stream_ptr(stream)))


class MultiPlan:
    """psw_multi: the plans' sweep tables gathered once (RHS-interleaved) for
    repeated multi-matrix solves; keeps the plans alive."""

    def __init__(self, plans: Sequence["Plan"]):
        self.plans = list(plans)
        self.nsys, self.n = len(self.plans), self.plans[0].n
        arr = (C.c_void_p * len(self.plans))(*[pl._h for pl in self.plans])
        h = C.c_void_p()
        _check(lib().psw_multi_create(C.byref(h), arr, len(self.plans)))
        self._h = h

    @classmethod
    def from_systems(cls, sub: np.ndarray, diag: np.ndarray, sup: np.ndarray, part: Partition,
                     dtype: int = F64, device: int = 0) -> "MultiPlan":
        """psw_multi_create_systems: the bundle of the symmetric systems
        (sub[k], diag[k], sup[k]), k = 0..nsys-1 (rows of 2-D arrays), sharing
        `part`, set up on the device in one pass (no per-system plans).
        Raises NotSupported for non-symmetric systems."""
        part.validate()
        sub = np.ascontiguousarray(sub, dtype=np.float64)
        diag = np.ascontiguousarray(diag, dtype=np.float64)
        sup = np.ascontiguousarray(sup, dtype=np.float64)
        if diag.ndim != 2 or sub.shape != (diag.shape[0], diag.shape[1] - 1) or sup.shape != sub.shape:
            raise ValueError("from_systems: diag (nsys, n), sub and super (nsys, n - 1)")
        nsys, n = diag.shape
        if part.n != n:
            raise ValueError("from_systems: partition order does not match the systems")
        dp = C.POINTER(C.c_double)
        L = lib()
        L.psw_multi_create_systems.restype = C.c_int
        L.psw_multi_create_systems.argtypes = [C.POINTER(C.c_void_p), C.c_int64, C.c_int64, dp, dp,
                                               dp, C.c_int64, C.POINTER(C.c_int64), C.c_int, C.c_int]
        bnd = np.ascontiguousarray(part.boundaries, dtype=np.int64)
        h = C.c_void_p()
        _check(L.psw_multi_create_systems(C.byref(h), n, nsys, sub.ctypes.data_as(dp),
                                          diag.ctypes.data_as(dp), sup.ctypes.data_as(dp), part.p(),
                                          bnd.ctypes.data_as(C.POINTER(C.c_int64)), dtype, device))
        self = cls.__new__(cls)
        self.plans = []
        self.nsys, self.n = nsys, n
        self._h = h
        return self

    def solve(self, F, X, stream=None):
        for t, nm in ((F, "F"), (X, "X")):
            if not getattr(t, "is_cuda", False) or t.dim() != 2 or t.stride(1) != 1:
                raise ValueError(f"{nm}: a CUDA matrix with contiguous rows")
            if t.shape[1] < self.nsys or t.shape[0] < self.n:
                raise ValueError(f"{nm}: too small for the bundle")
        _check(lib().psw_multi_solve(self._h, _ptr(F), F.stride(0), _ptr(X), X.stride(0),
                                     _stream_ptr(stream)))
        return X

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                lib().psw_multi_destroy(h)
            except Exception:  # noqa: BLE001
                pass
            self._h = None


def fill_uniform(t, seed: int, lo: float, hi: float, offset: int = 0, stream=None):
    """Seeded uniform fill of a CUDA tensor (SURVEY.md §8(d) generator)."""
    dt = F64 if str(t.dtype) == "torch.float64" else F32
    _check(lib().psw_fill_uniform(_ptr(t), dt, t.numel(), seed, offset, lo, hi, _stream_ptr(stream)))
    return t


def fill_normal(t, seed: int, offset: int = 0, stream=None):
    dt = F64 if str(t.dtype) == "torch.float64" else F32
    _check(lib().psw_fill_normal(_ptr(t), dt, t.numel(), seed, offset, _stream_ptr(stream)))
    return t


def l2_flush(t, stream=None):
    _check(lib().psw_l2_flush(_ptr(t), t.numel() * t.element_size(), _stream_ptr(stream)))
