"""Fourier (variable-separation) Poisson solver on the GPU: the second
consumer of the batched dichotomy solve (reference
poisson/fourier.hpp, poisson/dst.hpp).

Mirrors the reference API: ``harmonic_system``, ``FourierWorkspace`` (the
once-per-mesh phase: the direction-1 partition and, per direction-2 harmonic
l, the matrix B_l = tri(1, -(2 + d_l), 1) with its device-resident plan) and
``fourier_solve``. Fields are CUDA fp64 tensors in the reference's Grid2D
layout ((n1+1) x (n2+1) nodes, row-major, j contiguous, zero Dirichlet
boundary), as in the ADI driver (adi.py).

Per Poisson right-hand side:
  1. the DST-I of every interior row along direction 2 (dst.hpp:13-20:
     out_l = sum_j in_j sin(pi j l / N)), scaled by 2/N2 (fourier.hpp:130)
     and by -h1^2 (fourier.hpp:159) in the same pass — psw_dst_rows, a
     hand-written kernel restating the reference's paired radix-2 FFT of the
     odd extension (dst.hpp:85-149; direct sum for other N);
  2. ONE multi-matrix solve of all harmonics (psw_multi_solve on the
     workspace's MultiPlan bundle: column l of the coefficient grid with the
     plan of B_l; the reference's per-harmonic solve_harmonic loop,
     fourier.hpp:157-164);
  3. the inverse DST-I of every row (fourier.hpp:167-186).
The transforms follow the reference's FFT operation order (FMA contraction
aside); the solves are the dichotomy path of the reference.
"""
from __future__ import annotations

import math

import numpy as np
import torch

from . import F64, MultiPlan, NotSupported, Plan, TridiagMatrix
from .adi import _make_partition


class HarmonicSystem:
    """fourier.hpp:16-33 (the matrix is materialised on first use: the
    workspace sets all harmonics up from d_l alone)."""

    def __init__(self, l: int, d_l: float, order: int):
        self.l, self.d_l, self.order = l, d_l, order
        self._matrix = None

    @property
    def matrix(self) -> TridiagMatrix:
        if self._matrix is None:
            self._matrix = TridiagMatrix.constant(self.order, 1.0, -(2.0 + self.d_l), 1.0)
        return self._matrix


def harmonic_system(n1: int, n2: int, h1: float, h2: float, l: int) -> HarmonicSystem:
    """fourier.hpp:25-33: B_l = T - d_l I, d_l = 4 (h1/h2)^2 sin^2(pi l / (2 N2))."""
    s = math.sin(math.pi * float(l) / (2.0 * n2))
    d_l = 4.0 * (h1 * h1) / (h2 * h2) * s * s
    return HarmonicSystem(l, d_l, n1 - 1)


def dst_raw(x: torch.Tensor, out: torch.Tensor | None = None, scale: float = 1.0,
            stream=None) -> torch.Tensor:
    """out[..., l-1] = scale * sum_{j=1}^{N-1} x[..., j-1] sin(pi j l / N) for
    the rows of a CUDA fp64 matrix x of N-1 columns (psw_dst_rows: the
    reference's paired radix-2 FFT of the odd extension for power-of-two N,
    dst.hpp:93-149; the direct sum otherwise, :120-128)."""
    from . import _check, _ptr, _stream_ptr, lib
    if not (isinstance(x, torch.Tensor) and x.is_cuda and x.dtype == torch.float64 and x.dim() == 2
            and x.stride(1) == 1):
        raise ValueError("dst_raw: a CUDA fp64 matrix with contiguous rows")
    if out is None:
        out = torch.empty_like(x)
    if out.shape != x.shape or out.stride(1) != 1 or not out.is_cuda or out.dtype != torch.float64:
        raise ValueError("dst_raw: out must match x")
    rows, m = x.shape
    _check(lib().psw_dst_rows(_ptr(x), x.stride(0), _ptr(out), out.stride(0), rows, m + 1,
                              float(scale), _stream_ptr(stream)))
    return out


class FourierWorkspace:
    """fourier.hpp:35-105: the direction-1 partition (dichotomy_pes ranges,
    reduced while order < 2 pes) and one device plan per harmonic
    l = 1..n2-1 (the reference's cached HarmonicPlan list)."""

    def __init__(self, n1: int, n2: int, h1: float, h2: float, dichotomy_pes: int = 1,
                 device: int = 0):
        if n1 < 3 or n2 < 2:
            raise ValueError("FourierWorkspace: needs n1 >= 3 and n2 >= 2 cells")
        self.n1, self.n2, self.h1, self.h2 = n1, n2, h1, h2
        self.device = device
        order = n1 - 1
        self.part = _make_partition(order, dichotomy_pes)
        self.harmonics = [harmonic_system(n1, n2, h1, h2, l) for l in range(1, n2)]
        # every harmonic's tables in one device pass (psw_multi_create_systems):
        # B_l = tri(1, -(2 + d_l), 1) as rows of three arrays
        d = np.array([hs.d_l for hs in self.harmonics], dtype=np.float64)
        off = np.ones((len(self.harmonics), order - 1), dtype=np.float64)
        diag = np.repeat(-(2.0 + d)[:, None], order, axis=1)
        self._plans = None
        try:
            self._multi = MultiPlan.from_systems(off, diag, off, self.part, dtype=F64, device=device)
        except NotSupported:  # no room for the batched setup's scratch: one plan per harmonic
            self._multi = MultiPlan(self.plans)

    @property
    def plans(self):
        """One device plan per harmonic (the reference's cached HarmonicPlan
        list, fourier.hpp:53-60). The solver itself runs on the batched bundle;
        the per-harmonic plans are only built when asked for."""
        if self._plans is None:
            self._plans = [Plan(hs.matrix, self.part, dtype=F64, device=self.device, staged_only=True)
                           for hs in self.harmonics]
        return self._plans

    def partition(self):
        return self.part

    def solve_harmonics(self, coeff: torch.Tensor, out: torch.Tensor | None = None, stream=None):
        """All harmonic systems at once: column l-1 of `coeff` ((n1-1) x (n2-1),
        row i-1 = direction-1 node i) is the right-hand side of B_l."""
        if out is None:
            out = torch.empty_like(coeff)
        self._multi.solve(coeff, out, stream=stream)
        return out


def fourier_solve(f: torch.Tensor, ws: FourierWorkspace | None = None, h1: float | None = None,
                  h2: float | None = None) -> torch.Tensor:
    """fourier.hpp:111-186: Dirichlet Poisson laplace(u) = -f on the mesh of
    f ((n1+1) x (n2+1) CUDA fp64 tensor). Without a workspace, a single-PE one
    is built (fourier.hpp:189-193; h1, h2 default to the unit square)."""
    n1, n2 = f.shape[0] - 1, f.shape[1] - 1
    if ws is None:
        ws = FourierWorkspace(n1, n2, h1 if h1 is not None else 1.0 / n1,
                              h2 if h2 is not None else 1.0 / n2, 1, device=f.device.index or 0)
    if (ws.n1, ws.n2) != (n1, n2):
        raise ValueError("fourier_solve: workspace mesh does not match the field")
    interior = f[1:n1, 1:n2].to(torch.float64)
    # fourier.hpp:129-149 and :159 in one pass: rhs = -h1^2 (2 / N2) S f
    rhs = dst_raw(interior, scale=(-ws.h1 * ws.h1) * (2.0 / float(n2)))
    sol = ws.solve_harmonics(rhs)                           # fourier.hpp:157-164
    u = torch.zeros_like(f, dtype=torch.float64)
    dst_raw(sol, out=u[1:n1, 1:n2])                         # fourier.hpp:167-186
    return u
