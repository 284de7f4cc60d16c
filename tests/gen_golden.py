"""Generate tests/golden/*.npz from the REFERENCE ITSELF.

Runs the unmodified reference headers compiled by oracle/Makefile
(oracle/_ref/libpsw_ref.so, i.e. parsweep::solve_batch, compute_preliminary,
compute_betas, solve_boundaries, run_batch) on small seeded inputs that
follow BASELINE.json's config shapes and value distributions, and stores
inputs + outputs. The fixtures travel with the repo; the GPU box (which has
no /root/reference) checks the product against them.

    python tests/gen_golden.py          # needs /root/reference (this container)
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.pyoracle import Reference, build  # noqa: E402
from paper_0901_2859_b200 import configs  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def case(name, a, b, bnd, F, ref: Reference, extras: bool = True, sup=None):
    sup = a if sup is None else sup
    X = ref.solve_batch(a, b, sup, bnd, F)
    d = {"sub": a, "diag": b, "super": sup, "bnd": np.asarray(bnd, np.int64), "F": F, "X": X}
    if extras and len(bnd) > 0:
        L, R, V = [], [], []
        terms = 0
        for k in range(F.shape[0]):
            l, r, v, terms = ref.betas_boundaries(a, b, sup, bnd, F[k])
            L.append(l); R.append(r); V.append(v)
        d.update(betas_left=np.array(L), betas_right=np.array(R), boundary=np.array(V),
                 combine_terms=np.int64(terms))
        pre = ref.preliminary(a, b, sup, bnd)
        d.update(zr=pre["zr"], zl=pre["zl"], max_z=np.float64(pre["max_z"]),
                 strategy_used=np.int64(pre["strategy_used"]))
    _, stats = ref.run_batch(a, b, sup, bnd, F[:1])
    d["comm_rounds"] = np.int64(stats["comm_rounds"])
    np.savez_compressed(os.path.join(OUT, name + ".npz"), **d)
    print(f"{name}: n={b.size} p={len(bnd)} N={F.shape[0]} -> {os.path.getsize(os.path.join(OUT, name + '.npz'))} B")


def nonsymmetric(ref: Reference, seed: int = 2026):
    """Non-symmetric matrices through the reference's Auto GRowStrategy:
    symmetrizable (-> Symmetrize), mixed off-diagonal signs (-> ExplicitInverse),
    a zero super entry (-> TransposeSolve) (preliminary.hpp:111-132)."""
    rng = np.random.default_rng(seed + 40)
    n = 300
    bnd = ref.decompose(n, 6)
    F = configs.uniform(seed + 41, 5 * n, -1, 1).reshape(5, n)
    sub = -rng.uniform(0.2, 1.0, n - 1)
    sup = -rng.uniform(0.2, 1.0, n - 1)
    diag = np.r_[0, np.abs(sub)] + np.r_[np.abs(sup), 0] + rng.uniform(0.5, 1.5, n)
    case("nonsym_symmetrizable_n300_P6", sub, diag, bnd, F, ref, sup=sup)
    sub = rng.uniform(-1, 1, n - 1)
    sup = rng.uniform(-1, 1, n - 1)
    sup[::3] = -np.sign(sub[::3]) * np.abs(sup[::3])
    diag = np.r_[0, np.abs(sub)] + np.r_[np.abs(sup), 0] + rng.uniform(0.5, 1.5, n)
    case("nonsym_mixed_n300_P6", sub, diag, bnd, F, ref, sup=sup)
    sup = sup.copy()
    sup[n // 3] = 0.0
    case("nonsym_reducible_n300_P6", sub, diag, bnd, F, ref, sup=sup)


def adi(ref: Reference, seed: int = 2026):
    """The ADI consumer (poisson/adi.hpp): three Peaceman-Rachford steps on a
    non-square mesh with a random start (1 and 3 dichotomy PEs), and a full
    adi_solve of the model problem."""
    for n1, n2, pes in ((24, 18, 1), (40, 33, 3)):
        h1, h2 = 1.0 / n1, 1.0 / n2
        f, exact = ref.model_problem(n1, n2)
        rng = np.random.default_rng(seed + n1)
        u0 = np.zeros((n1 + 1, n2 + 1))
        u0[1:-1, 1:-1] = rng.uniform(-1, 1, (n1 - 1, n2 - 1))
        cycle = 5
        u3 = ref.adi_steps(n1, n2, h1, h2, cycle, pes, f, u0, 3)
        taus = ref.adi_parameters(n1, n2, h1, h2, cycle, pes)
        np.savez_compressed(os.path.join(OUT, f"adi_steps_{n1}x{n2}_pes{pes}.npz"), n1=n1, n2=n2,
                            pes=pes, cycle=cycle, f=f, u0=u0, u3=u3, taus=taus)
        print(f"adi_steps_{n1}x{n2}_pes{pes}")
    n, eps, pes = 32, 1e-5, 2
    f, exact = ref.model_problem(n, n)
    cycle = ref.adi_iteration_bound(n, eps)
    u, its = ref.adi_solve(n, n, 1.0 / n, 1.0 / n, cycle, pes, eps, f, np.zeros_like(f))
    np.savez_compressed(os.path.join(OUT, "adi_solve_32x32.npz"), n=n, eps=eps, pes=pes,
                        cycle=cycle, f=f, exact=exact, u=u, iterations=its)
    print(f"adi_solve_32x32: {its} iterations (cycle {cycle})")


def fourier(ref: Reference, seed: int = 2026):
    """The Fourier consumer (poisson/fourier.hpp): fourier_solve of the model
    problem (1 and 4 dichotomy PEs) and of a seeded random field on a
    rectangular mesh."""
    for n1, n2, pes in ((32, 32, 1), (64, 64, 4), (24, 40, 3)):
        h1, h2 = 1.0 / n1, 1.0 / n2
        if n1 == n2:
            f, _ = ref.model_problem(n1, n2)
        else:
            rng = np.random.default_rng(seed + n1 + n2)
            f = np.zeros((n1 + 1, n2 + 1))
            f[1:-1, 1:-1] = rng.uniform(-1, 1, (n1 - 1, n2 - 1))
        u, bnd = ref.fourier_solve(n1, n2, h1, h2, pes, f)
        name = f"fourier_{n1}x{n2}_pes{pes}"
        np.savez_compressed(os.path.join(OUT, name + ".npz"), n1=n1, n2=n2, h1=h1, h2=h2, pes=pes,
                            f=f, u=u, bnd=bnd)
        print(name, "boundaries", list(bnd))


def main():
    build(ref=True)
    ref = Reference()
    os.makedirs(OUT, exist_ok=True)
    seed = 2026
    if len(sys.argv) > 1 and sys.argv[1] == "--nonsymmetric":
        nonsymmetric(ref, seed)
        return
    if len(sys.argv) > 1 and sys.argv[1] == "--adi":
        adi(ref, seed)
        return
    if len(sys.argv) > 1 and sys.argv[1] == "--fourier":
        fourier(ref, seed)
        return

    # C0 shape: n=1024, P=4, dominant (slack U[0.1,1]), F ~ U[-1,1]
    c0 = configs.CONFIGS["C0"]
    a, b = c0.matrix_ab(seed)
    bnd = ref.decompose(1024, 4)
    F = configs.uniform(seed + 3, 16 * 1024, -1, 1).reshape(16, 1024)
    case("c0_n1024_P4", a, b, bnd, F, ref)

    # C1 shape: n=4096, P=16, a=-1, b=2.01, F ~ N(0,1)
    a = -np.ones(4095); b = np.full(4096, 2.01)
    bnd = ref.decompose(4096, 16)
    F = configs.normal(seed + 3, 4 * 4096).reshape(4, 4096)
    case("c1_n4096_P16", a, b, bnd, F, ref)

    # C4 shape: the ill-conditioned ADI matrix (b = 2 + h^2 tau), grid rows
    h = 1.0 / 4097
    a = -np.ones(4095); b = np.full(4096, 2.0 + h * h * 10.0)
    bnd = ref.decompose(4096, 16)
    F = configs.grid_rhs(4096, 4, seed)
    case("c4_n4096_P16", a, b, bnd, F, ref)

    # C2 shape (fp32 config, fp64 oracle on fp32-rounded F), scaled-down n
    a, b = configs.dominant_matrix(8192, seed, (0.5, 2.0))
    for P in (8, 64, 512):
        bnd = ref.decompose(8192, P)
        F = configs.uniform(seed + 3, 4 * 8192, -1, 1).reshape(4, 8192).astype(np.float32).astype(np.float64)
        case(f"c2_n8192_P{P}", a, b, bnd, F, ref, extras=(P <= 64))

    # non-uniform / random partitions and edge shapes
    rng = np.random.default_rng(seed)
    a, b = configs.dominant_matrix(200, seed + 10, (0.1, 1.0))
    bnd = np.sort(rng.choice(np.arange(2, 200), size=7, replace=False))
    F = configs.uniform(seed + 11, 5 * 200, -1, 1).reshape(5, 200)
    case("rand_n200_p7", a, b, bnd, F, ref)
    # decompose with remainder (sizes differ by one)
    a, b = configs.dominant_matrix(333, seed + 12, (0.1, 1.0))
    bnd = ref.decompose(333, 9)
    F = configs.uniform(seed + 13, 6 * 333, -1, 1).reshape(6, 333)
    case("decomp_n333_P9", a, b, bnd, F, ref)
    # single block (p = 0): plain sweep
    a, b = configs.dominant_matrix(50, seed + 14, (0.1, 1.0))
    F = configs.uniform(seed + 15, 3 * 50, -1, 1).reshape(3, 50)
    case("p0_n50", a, b, np.zeros(0, np.int64), F, ref)
    # size-2 blocks at both ends and in the middle
    a, b = configs.dominant_matrix(12, seed + 16, (0.1, 1.0))
    bnd = np.array([2, 3, 5, 6, 10, 11], np.int64)
    F = configs.uniform(seed + 17, 4 * 12, -1, 1).reshape(4, 12)
    case("tiny_n12_p6", a, b, bnd, F, ref)
    # mixed-sign dominant symmetric matrix (reference helper style)
    n = 96
    mag = configs.uniform(seed + 18, n - 1, 0.2, 1.0)
    sgn = np.where(configs.uniform01(seed + 19, n - 1) < 0.5, -1.0, 1.0)
    a = mag * sgn
    off = np.zeros(n); off[1:] += np.abs(a); off[:-1] += np.abs(a)
    b = (off * (1.0 + configs.uniform(seed + 20, n, 0.05, 1.0)) + 0.1) * np.where(
        configs.uniform01(seed + 21, n) < 0.5, -1.0, 1.0)
    bnd = ref.decompose(n, 8)
    F = configs.uniform(seed + 22, 5 * n, -1, 1).reshape(5, n)
    case("mixed_n96_P8", a, b, bnd, F, ref)
    nonsymmetric(ref, seed)
    adi(ref, seed)
    fourier(ref, seed)


if __name__ == "__main__":
    main()
