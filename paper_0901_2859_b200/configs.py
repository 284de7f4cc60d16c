"""Seeded synthetic workloads of BASELINE.json `configs` (C0..C4).

No public dataset is involved: the reference's benchmark inputs are seeded
random matrices/RHS, so these generators restate the config text with a
documented counter-based generator:

    u(seed, i) = (splitmix64(seed ^ i) >> 11) * 2^-53          in [0, 1)
    U[lo, hi]  = lo + (hi - lo) * u                              (no FMA)
    N(0, 1)    = Box-Muller on (1 - u(2j), u(2j+1))

Streams: off-diagonal a uses seed+1, the diagonal slack seed+2, the RHS
seed+3 over the linear index of the buffer in its own layout. The device
fill kernels (psw_fill_uniform / psw_fill_normal) implement the same
streams, bitwise for the uniform one.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(x: np.ndarray) -> np.ndarray:
    x = x.astype(np.uint64, copy=True)
    with np.errstate(over="ignore"):
        x += np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        x = x ^ (x >> np.uint64(31))
    return x


def uniform01(seed: int, count: int, offset: int = 0) -> np.ndarray:
    idx = np.arange(offset, offset + count, dtype=np.uint64) ^ np.uint64(seed & 0xFFFFFFFFFFFFFFFF)
    return (splitmix64(idx) >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def uniform(seed: int, count: int, lo: float, hi: float, offset: int = 0) -> np.ndarray:
    return lo + (hi - lo) * uniform01(seed, count, offset)


def normal(seed: int, count: int, offset: int = 0) -> np.ndarray:
    pairs = (count + 1) // 2
    u = uniform01(seed, 2 * pairs, offset)
    r = np.sqrt(-2.0 * np.log(1.0 - u[0::2]))
    th = 2.0 * np.pi * u[1::2]
    out = np.empty(2 * pairs)
    out[0::2] = r * np.cos(th)
    out[1::2] = r * np.sin(th)
    return out[:count]


def dominant_matrix(n: int, seed: int, slack: tuple[float, float]):
    """a_i ~ U[-1,-0.5] (i = 1..n-1), b_i = |a_{i-1}| + |a_i| + U[slack]
    with a_0 = a_n = 0; symmetric (sub == super)."""
    a = uniform(seed + 1, n - 1, -1.0, -0.5)
    absa = np.abs(a)
    b = np.zeros(n)
    b[1:] += absa
    b[:-1] += absa
    b += uniform(seed + 2, n, slack[0], slack[1])
    return a, b


@dataclass(frozen=True)
class Config:
    name: str
    dtype: str       # "f64" | "f32"
    n: int
    nrhs: int
    P: int
    layout: str      # "R" | "S"
    rhs: str         # "uniform" | "normal" | "grid"
    matrix: str      # "dominant01" | "dominant05" | "laplace201" | "adi"

    def matrix_ab(self, seed: int = 0):
        if self.matrix == "dominant01":
            return dominant_matrix(self.n, seed, (0.1, 1.0))
        if self.matrix == "dominant05":
            return dominant_matrix(self.n, seed, (0.5, 2.0))
        if self.matrix == "laplace201":
            return -np.ones(self.n - 1), np.full(self.n, 2.01)
        if self.matrix == "adi":
            h = 1.0 / (self.n + 1)
            return -np.ones(self.n - 1), np.full(self.n, 2.0 + h * h * 10.0)
        raise ValueError(self.matrix)

    def bytes_min(self) -> int:
        """N n (s_F + s_X) + (2n - 1) s_A."""
        s = 8 if self.dtype == "f64" else 4
        return self.nrhs * self.n * 2 * s + (2 * self.n - 1) * s

    def with_(self, **kw) -> "Config":
        d = dict(self.__dict__)
        d.update(kw)
        return Config(**d)


CONFIGS = {
    "C0": Config("C0", "f64", 1024, 256, 4, "R", "uniform", "dominant01"),
    "C1": Config("C1", "f64", 4096, 4096, 16, "R", "normal", "laplace201"),
    "C2": Config("C2", "f32", 65536, 65536, 64, "R", "uniform", "dominant05"),
    "C3": Config("C3", "f64", 1 << 20, 1024, 64, "R", "uniform", "dominant01"),
    "C4": Config("C4", "f64", 4096, 4096, 16, "S", "grid", "adi"),
    # C4's second direction: the same grid field and matrix solved along the
    # columns (unknowns strided by the row pitch = layout R)
    "C4c": Config("C4c", "f64", 4096, 4096, 16, "R", "grid", "adi"),
}


def host_rhs(cfg: Config, seed: int = 0, nrhs: int | None = None) -> np.ndarray:
    """Host copy of the config's RHS buffer in its own layout (fp64 values;
    cast to fp32 for f32 configs). Layout R -> (n, N), layout S -> (N, n)."""
    N = cfg.nrhs if nrhs is None else nrhs
    count = cfg.n * N
    if cfg.rhs == "uniform":
        v = uniform(seed + 3, count, -1.0, 1.0)
    elif cfg.rhs == "normal":
        v = normal(seed + 3, count)
    elif cfg.rhs == "grid":
        return grid_rhs(cfg.n, N, seed)
    else:
        raise ValueError(cfg.rhs)
    shape = (cfg.n, N) if cfg.layout == "R" else (N, cfg.n)
    v = v.reshape(shape)
    return v.astype(np.float32) if cfg.dtype == "f32" else v


def grid_rhs(n: int, rows: int, seed: int = 0) -> np.ndarray:
    """C4 field on the interior grid, h = 1/(n+1): f_ij = sin(pi x_j) sin(pi y_i)
    + U[-0.01, 0.01]; row-major (grid row i contiguous) = layout S for the row
    sweep. `rows` grid rows are produced (rows == n for the full grid)."""
    h = 1.0 / (n + 1)
    x = np.arange(1, n + 1) * h
    y = np.arange(1, rows + 1) * h
    base = np.sin(math.pi * y)[:, None] * np.sin(math.pi * x)[None, :]
    return base + uniform(seed + 3, rows * n, -0.01, 0.01).reshape(rows, n)
