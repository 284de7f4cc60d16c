"""ADI (Peaceman-Rachford) Poisson driver on the GPU: the first consumer of
the batched dichotomy solve (reference poisson/adi.hpp).

Mirrors the reference API: ``adi_iteration_bound``, ``adi_parameters``,
``AdiWorkspace`` (one pair of half-step plans per cyclic parameter),
``AdiIteration.step`` and ``adi_solve``. Fields are CUDA fp64 tensors in the
reference's Grid2D layout ((n1+1) x (n2+1) nodes, row-major, j contiguous,
zero Dirichlet boundary). Every half step is two device operations: the
stencil right-hand side (psw_adi_rhs, the reference's arithmetic) and one
batched solve of all lines through the plan of that parameter — direction 1
in layout R, solved straight into the interior of the half-step field,
direction 2 in layout S (SURVEY §8 C4 shapes).
"""
from __future__ import annotations

import ctypes as C
import math

from . import (F64, LAYOUT_R, LAYOUT_S, Partition, Plan, SolverError, TridiagMatrix, _check,
               _ptr, _stream_ptr, decompose, lib)


class NonConvergence(SolverError):
    """core/errors.hpp:51-54"""


def adi_iteration_bound(n: int, eps: float) -> int:
    """adi.hpp:20-25: n0(eps) = 0.2 ln(4N/pi) ln(4/eps), rounded up."""
    n0 = 0.2 * math.log(4.0 * float(n) / math.pi) * math.log(4.0 / eps)
    if n0 <= 0.0:
        return 0
    return int(math.ceil(n0 - 1e-12))


def geometric_parameters(lambda_min: float, lambda_max: float, n0: int) -> list[float]:
    """adi.hpp:32-43."""
    ratio = lambda_min / lambda_max
    taus = []
    for j in range(1, n0 + 1):
        exponent = (2.0 * float(j) - 1.0) / (2.0 * float(n0))
        taus.append(1.0 / (lambda_max * math.pow(ratio, exponent)))
    return taus


def _lambda_min(n: int, h: float) -> float:  # adi.hpp:102-105
    s = math.sin(math.pi / (2.0 * float(n)))
    return 4.0 / (h * h) * s * s


def _lambda_max(n: int, h: float) -> float:  # adi.hpp:106-109
    c = math.cos(math.pi / (2.0 * float(n)))
    return 4.0 / (h * h) * c * c


def adi_parameters(n: int, n0: int) -> list[float]:
    """adi.hpp:50-58: the cycle for the square N x N unit mesh."""
    h = 1.0 / float(n)
    return geometric_parameters(_lambda_min(n, h), _lambda_max(n, h), n0)


def _make_partition(order: int, dichotomy_pes: int) -> Partition:
    """adi.hpp:73-77."""
    pes = 1 if dichotomy_pes == 0 else dichotomy_pes
    while pes > 1 and order < 2 * pes:
        pes -= 1
    if pes == 1:
        return Partition(order, [])
    return decompose(order, pes).induced_partition()


class AdiWorkspace:
    """adi.hpp:63-117: the parameter cycle and, per parameter, the two
    half-step matrices with their device-resident plans."""

    class Step:
        def __init__(self, c1, c2, plan1, plan2):
            self.c1, self.c2, self.plan1, self.plan2 = c1, c2, plan1, plan2

    def __init__(self, n1: int, n2: int, h1: float, h2: float, cycle_length: int,
                 dichotomy_pes: int = 1, device: int = 0):
        self.n1, self.n2, self.h1, self.h2 = n1, n2, h1, h2
        lmin = min(_lambda_min(n1, h1), _lambda_min(n2, h2))
        lmax = max(_lambda_max(n1, h1), _lambda_max(n2, h2))
        self.taus = geometric_parameters(lmin, lmax, max(cycle_length, 1))
        self.part1 = _make_partition(n1 - 1, dichotomy_pes)
        self.part2 = _make_partition(n2 - 1, dichotomy_pes)
        self.steps = []
        for tau in self.taus:
            c1 = TridiagMatrix.constant(n1 - 1, 1.0, -2.0 - h1 * h1 / tau, 1.0)
            c2 = TridiagMatrix.constant(n2 - 1, 1.0, -2.0 - h2 * h2 / tau, 1.0)
            self.steps.append(AdiWorkspace.Step(c1, c2, Plan(c1, self.part1, F64, device),
                                                Plan(c2, self.part2, F64, device)))

    def parameters(self) -> list[float]:
        return self.taus

    def cycle_length(self) -> int:
        return len(self.taus)

    def step(self, k: int) -> "AdiWorkspace.Step":
        return self.steps[k % len(self.steps)]


def _adi_rhs(direction, u, f, rhs, ldr, n1, n2, h1, h2, tau, stream):
    L = lib()
    L.psw_adi_rhs.argtypes = [C.c_int, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p,
                              C.c_int64, C.c_int64, C.c_int64, C.c_double, C.c_double, C.c_double,
                              C.c_void_p]
    _check(L.psw_adi_rhs(direction, _ptr(u), u.stride(0), _ptr(f), f.stride(0), _ptr(rhs), ldr,
                         n1, n2, h1, h2, tau, stream))


def max_abs_diff_and_max(a, b, out=None, stream=None):
    """(max |a - b|, max |b|) of two fields on the device (grid2d.hpp:43-53)."""
    import torch
    L = lib()
    L.psw_grid_max_abs_diff.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_int64,
                                        C.c_int64, C.c_void_p, C.c_void_p]
    if a.shape != b.shape or a.dim() != 2 or a.stride(1) != 1 or b.stride(1) != 1:
        raise ValueError("max_abs_diff_and_max: two fields of one shape with contiguous rows")
    if out is None:
        out = torch.empty(2, dtype=torch.float64, device=a.device)
    _check(L.psw_grid_max_abs_diff(_ptr(a), a.stride(0), _ptr(b), b.stride(0), a.shape[0],
                                   a.shape[1], _ptr(out), _stream_ptr(stream)))
    v = out.tolist()
    return v[0], v[1]


def _is_padded(t) -> bool:
    return t.stride(0) % 16 == 0 and (t.data_ptr() + 8 * (t.stride(0) + 1)) % 128 == 0


def padded_field(n1: int, n2: int, device) -> "torch.Tensor":
    """A zero (n1+1) x (n2+1) Grid2D field whose rows have a pitch of a
    multiple of 16 doubles and whose interior node (1, 1) sits on 128 bytes:
    the layout-R solve of direction 1 then writes whole 128-byte lines of
    every grid row, and the layout-S solve of direction 2 whole 32-byte
    sectors of every line (the CLUSTER kernel's 256-bit store variant)."""
    import torch
    ld = (n2 + 1 + 15) // 16 * 16
    store = torch.zeros((n1 + 1) * ld + 16, dtype=torch.float64, device=device)
    return store.as_strided((n1 + 1, n2 + 1), (ld, 1), 15)


class AdiIteration:
    """adi.hpp:122-185: one Peaceman-Rachford iteration with reused buffers."""

    def __init__(self, ws: AdiWorkspace, f, stream=None):
        import torch
        self.ws, self.f = ws, f
        n1, n2 = ws.n1, ws.n2
        if tuple(f.shape) != (n1 + 1, n2 + 1) or f.dtype != torch.float64 or not f.is_cuda:
            raise ValueError("f must be a CUDA fp64 tensor of shape (n1+1, n2+1)")
        self.stream = _stream_ptr(stream)
        # right-hand sides of one half step (even pitch: 16-byte aligned rows)
        self.ldr = (n2 - 1 + 1) // 2 * 2
        self.rhs = torch.empty((n1 - 1, self.ldr), dtype=torch.float64, device=f.device)
        self.half = padded_field(n1, n2, f.device)  # half-step field (boundary stays zero)
        self.next = padded_field(n1, n2, f.device)

    def step(self, u, k: int) -> None:
        """Advances u (in place) by iteration k (parameter k mod n0)."""
        ws, f = self.ws, self.f
        n1, n2, h1, h2 = ws.n1, ws.n2, ws.h1, ws.h2
        st = ws.step(k)
        tau = ws.taus[k % ws.cycle_length()]
        # direction 1: lines j, unknowns along i -> layout R into the half field
        _adi_rhs(1, u, f, self.rhs, self.ldr, n1, n2, h1, h2, tau, self.stream)
        st.plan1.solve(self.rhs, self.half[1:, 1:], nrhs=n2 - 1, layout=LAYOUT_R,
                       ldf=self.ldr, ldx=self.half.stride(0), stream=self.stream)
        # direction 2: lines i, unknowns along j -> layout S into the next field
        _adi_rhs(2, self.half, f, self.rhs, self.ldr, n1, n2, h1, h2, tau, self.stream)
        st.plan2.solve(self.rhs, self.next[1:, 1:], nrhs=n1 - 1, layout=LAYOUT_S,
                       ldf=self.ldr, ldx=self.next.stride(0), stream=self.stream)
        u.data, self.next.data = self.next.data, u.data  # std::swap(u.values, next_.values)
        if not _is_padded(self.next):  # the caller's first field: keep the buffer padded
            self.next = padded_field(n1, n2, f.device)


def adi_solve(f, eps: float, u0, ws: AdiWorkspace, exact=None, stream=None):
    """adi.hpp:198-222: iterate until the relative successive difference is
    under eps (or, with `exact`, until the max-norm error shrank by eps).
    Returns (u, iterations); raises NonConvergence after 10 cycles."""
    import torch
    u = u0.clone()
    previous = torch.empty_like(u)
    it = AdiIteration(ws, f, stream)
    out = torch.empty(2, dtype=torch.float64, device=u.device)
    err0 = max_abs_diff_and_max(u, exact, out, stream)[0] if exact is not None else 0.0
    if exact is not None and err0 == 0.0:
        return u, 0
    max_iterations = 10 * ws.cycle_length()
    for k in range(max_iterations):
        previous.copy_(u)
        it.step(u, k)
        done = k + 1
        if exact is not None:
            if max_abs_diff_and_max(u, exact, out, stream)[0] <= eps * err0:
                return u, done
        else:
            diff, umax = max_abs_diff_and_max(previous, u, out, stream)
            if diff == 0.0 or diff <= eps * umax:
                return u, done
    raise NonConvergence(f"alternating-direction iteration exceeded {max_iterations} iterations")


def model_problem(n1: int, n2: int, device="cuda"):
    """model_problem.hpp:15-37 on the device (see model_problem_host)."""
    import torch
    f, exact = model_problem_host(n1, n2)
    return torch.from_numpy(f).to(device), torch.from_numpy(exact).to(device)


def model_problem_host(n1: int, n2: int):
    """model_problem.hpp:15-37: f = 8 pi^2 sin(2 pi x) sin(2 pi y) and the
    exact solution sin(2 pi x) sin(2 pi y), sampled at the mesh nodes."""
    import numpy as np
    h1, h2 = 1.0 / n1, 1.0 / n2
    two_pi = 2.0 * math.pi
    sx = np.array([math.sin(two_pi * (i * h1)) for i in range(n1 + 1)])
    sy = np.array([math.sin(two_pi * (j * h2)) for j in range(n2 + 1)])
    exact = np.outer(sx, sy)
    f = 8.0 * math.pi * math.pi * sx[:, None] * sy[None, :]
    exact[:, 0] = exact[:, n2] = 0.0
    exact[0, :] = exact[n1, :] = 0.0
    return f, exact
