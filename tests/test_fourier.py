"""Fourier consumer (paper_0901_2859_b200/fourier.py, reference
poisson/fourier.hpp + poisson/dst.hpp): the reference's fourier_solve
fixtures (tests/gen_golden.py --fourier), the reference's Fourier tests
restated (test_poisson.cpp:145-224), and the multi-matrix solve
(psw_solve_multi) against single-plan STAGED solves."""
import math

import numpy as np
import pytest

from conftest import load_golden


@pytest.mark.gpu
@pytest.mark.parametrize("n", [8, 13, 32, 1024, 4096, 6000])
def test_dst_raw_matches_the_sine_sum(psw, cuda, n):
    """psw_dst_rows against the dense sine sum (power-of-two N through the
    paired FFT, others through the direct sum; odd and even row counts)."""
    from paper_0901_2859_b200.fourier import dst_raw
    for rows in (1, 3, 8):
        x = np.random.default_rng(n + rows).standard_normal((rows, n - 1))
        j = np.arange(1, n)
        S = np.sin(np.pi * np.outer(j, j) / n)
        want = x @ S.T
        got = dst_raw(cuda.from_numpy(x).cuda()).cpu().numpy()
        assert np.max(np.abs(got - want)) <= 1e-12 * np.max(np.abs(want))
        # (2/N) S is the inverse of S (dst.hpp:13-17)
        back = dst_raw(cuda.from_numpy(got).cuda(), scale=2.0 / n).cpu().numpy()
        assert np.max(np.abs(back - x)) <= 1e-12 * np.max(np.abs(x))


def test_dst_raw_needs_a_cuda_matrix(psw):
    import torch
    from paper_0901_2859_b200.fourier import dst_raw
    with pytest.raises(ValueError):  # no CPU fallback
        dst_raw(torch.zeros(2, 7, dtype=torch.float64))


def test_harmonic_system_is_the_reference_matrix():
    from paper_0901_2859_b200.fourier import harmonic_system
    n1, n2, h1, h2 = 24, 40, 1 / 24, 1 / 40
    for l in (1, 7, 39):
        hs = harmonic_system(n1, n2, h1, h2, l)
        s = math.sin(math.pi * l / (2.0 * n2))
        d = 4.0 * (h1 * h1) / (h2 * h2) * s * s
        assert hs.d_l == d and hs.matrix.n() == n1 - 1
        assert np.all(hs.matrix.diag == -(2.0 + d)) and np.all(hs.matrix.sub == 1.0)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["fourier_32x32_pes1", "fourier_64x64_pes4", "fourier_24x40_pes3"])
def test_fourier_matches_reference(psw, cuda, name):
    from paper_0901_2859_b200.fourier import FourierWorkspace, fourier_solve
    g = load_golden(name)
    n1, n2, pes = int(g["n1"]), int(g["n2"]), int(g["pes"])
    ws = FourierWorkspace(n1, n2, float(g["h1"]), float(g["h2"]), pes)
    assert ws.partition().boundaries == [int(b) for b in g["bnd"]]
    u = fourier_solve(cuda.from_numpy(g["f"]).cuda(), ws).cpu().numpy()
    want = g["u"]
    assert np.linalg.norm(u - want) / np.linalg.norm(want) <= 1e-12
    assert np.max(np.abs(u - want)) <= 1e-12 * np.max(np.abs(want))
    assert np.all(u[0] == 0) and np.all(u[-1] == 0) and np.all(u[:, 0] == 0) and np.all(u[:, -1] == 0)


@pytest.mark.gpu
def test_fourier_zero_is_zero(psw, cuda):  # test_poisson.cpp:145-149
    from paper_0901_2859_b200.fourier import fourier_solve
    u = fourier_solve(cuda.zeros(17, 17, dtype=cuda.float64, device="cuda"))
    assert bool((u == 0).all())


@pytest.mark.gpu
def test_fourier_inverts_discrete_eigenfunction(psw, cuda):  # test_poisson.cpp:151-165
    from paper_0901_2859_b200.fourier import fourier_solve
    n, k, m = 32, 3, 5
    h = 1.0 / n
    x = np.arange(n + 1) * h
    f = np.outer(np.sin(np.pi * k * x), np.sin(np.pi * m * x))
    f[0, :] = f[-1, :] = f[:, 0] = f[:, -1] = 0.0
    lam = 4 / h**2 * math.sin(math.pi * k / (2 * n)) ** 2 + 4 / h**2 * math.sin(math.pi * m / (2 * n)) ** 2
    u = fourier_solve(cuda.from_numpy(f).cuda()).cpu().numpy()
    assert np.max(np.abs(u[1:-1, 1:-1] - f[1:-1, 1:-1] / lam)) <= 1e-12


def _laplacian(u, h1, h2):
    return ((u[2:, 1:-1] - 2 * u[1:-1, 1:-1] + u[:-2, 1:-1]) / h1**2 +
            (u[1:-1, 2:] - 2 * u[1:-1, 1:-1] + u[1:-1, :-2]) / h2**2)


@pytest.mark.gpu
def test_fourier_discrete_equations_and_convergence(psw, cuda, ref):  # test_poisson.cpp:167-190
    from paper_0901_2859_b200.fourier import fourier_solve
    prev = 0.0
    for n in (16, 32, 64, 128):
        f, exact = ref.model_problem(n, n)
        u = fourier_solve(cuda.from_numpy(f).cuda()).cpu().numpy()
        if n == 64:
            assert np.max(np.abs(_laplacian(u, 1 / n, 1 / n) + f[1:-1, 1:-1])) <= 1e-9 * np.max(np.abs(f))
        err = np.max(np.abs(u - exact))
        if prev:
            assert 3.5 < prev / err < 4.5
        prev = err


@pytest.mark.gpu
def test_fourier_rectangular_and_split(psw, cuda, ref):  # test_poisson.cpp:192-224
    from paper_0901_2859_b200.fourier import FourierWorkspace, fourier_solve
    n1, n2 = 24, 40
    x, y = np.arange(n1 + 1) / n1, np.arange(n2 + 1) / n2
    exact = np.outer(np.sin(2 * np.pi * x), np.sin(2 * np.pi * y))
    f = 8 * np.pi**2 * exact
    u = fourier_solve(cuda.from_numpy(f).cuda(), FourierWorkspace(n1, n2, 1 / n1, 1 / n2)).cpu().numpy()
    assert np.max(np.abs(u - exact)) < 0.05
    assert np.max(np.abs(_laplacian(u, 1 / n1, 1 / n2) + f[1:-1, 1:-1])) <= 1e-9 * np.max(np.abs(f))
    f64, _ = ref.model_problem(64, 64)
    fd = cuda.from_numpy(f64).cuda()
    plain = fourier_solve(fd, FourierWorkspace(64, 64, 1 / 64, 1 / 64, 1)).cpu().numpy()
    ws = FourierWorkspace(64, 64, 1 / 64, 1 / 64, 4)
    assert ws.partition().p() == 3
    split = fourier_solve(fd, ws).cpu().numpy()
    assert np.max(np.abs(plain - split)) <= 1e-11
    assert np.array_equal(split, fourier_solve(fd, ws).cpu().numpy())  # run to run


@pytest.mark.gpu
def test_solve_multi_equals_single_plan_staged(psw, cuda):
    """psw_solve_multi is, column by column, the single-plan STAGED solve."""
    rng = np.random.default_rng(5)
    n, K = 300, 37
    part = psw.decompose(n, 6).induced_partition()
    plans, As = [], []
    for k in range(K):
        a = rng.uniform(-1, -0.5, n - 1)
        b = np.abs(np.r_[0, a]) + np.abs(np.r_[a, 0]) + rng.uniform(0.1, 1, n)
        As.append((a, b))
        plans.append(psw.Plan(psw.TridiagMatrix.symmetric(a, b), part))
    F = cuda.from_numpy(rng.uniform(-1, 1, (n, K + 3))).cuda()
    X = cuda.zeros_like(F)
    psw.solve_multi(plans, F, X)
    for k in (0, 17, K - 1):
        xs = cuda.zeros(n, 1, dtype=cuda.float64, device="cuda")
        plans[k].solve(F[:, k:k + 1].contiguous(), xs, layout=psw.LAYOUT_R, path=psw.PATH_STAGED)
        assert cuda.equal(X[:, k], xs[:, 0])
    with pytest.raises(ValueError):  # plans must share the partition
        other = psw.Plan(psw.TridiagMatrix.symmetric(*As[0]), psw.decompose(n, 5).induced_partition())
        psw.solve_multi(plans[:2] + [other], F, X)


@pytest.mark.gpu
def test_multi_bundle_equals_solve_multi(psw, cuda):
    """psw_multi_solve (interleaved tables, one gather at creation) is bitwise
    psw_solve_multi (per-plan tables) on every column."""
    from paper_0901_2859_b200.fourier import FourierWorkspace
    n1, n2 = 300, 97
    ws = FourierWorkspace(n1, n2, 1.0 / n1, 1.0 / n2, 4)
    rhs = cuda.randn(n1 - 1, n2 - 1, dtype=cuda.float64, device="cuda")
    a = cuda.empty_like(rhs)
    psw.solve_multi(ws.plans, rhs, a)
    b = ws.solve_harmonics(rhs)
    b2 = psw.MultiPlan(ws.plans).solve(rhs, cuda.empty_like(rhs))
    cuda.cuda.synchronize()
    assert bool((a == b).all()) and bool((a == b2).all())


@pytest.mark.gpu
def test_staged_only_plan(psw, cuda):
    """PSW_PLAN_STAGED_ONLY: the same STAGED result as a full plan; the
    segment-table paths answer NotSupported and AUTO falls back to STAGED."""
    from test_parity_gpu import gpu_solve
    g = load_golden("c1_n4096_P16")
    A = psw.TridiagMatrix(g["sub"], g["diag"], g["super"])
    part = psw.Partition(A.n(), g["bnd"].tolist())
    full, lean = psw.Plan(A, part), psw.Plan(A, part, staged_only=True)
    assert lean.info["device_bytes"] < full.info["device_bytes"]
    a = gpu_solve(psw, cuda, full, g["F"], 0, path=psw.PATH_STAGED)
    b = gpu_solve(psw, cuda, lean, g["F"], 0, path=psw.PATH_AUTO)
    assert np.array_equal(a, b)
    for path in (psw.PATH_CLUSTER, psw.PATH_RESWEEP, psw.PATH_FUSED):
        with pytest.raises(psw.NotSupported):
            gpu_solve(psw, cuda, lean, g["F"], 0, path=path)


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["dominant", "mixed_sign", "harmonics", "fp32", "p0", "size2"])
def test_bundle_from_systems_is_bitwise_the_per_plan_bundle(psw, cuda, kind):
    """psw_multi_create_systems (every system's preliminary and block sweep
    coefficients in one device pass, [row][system] tables) against
    psw_multi_create over plans created one by one on the host: the same
    solution bit for bit on every column."""
    rng = np.random.default_rng({"dominant": 1, "mixed_sign": 2, "harmonics": 3, "fp32": 4,
                                 "p0": 5, "size2": 6}[kind])
    n, K = (700, 45) if kind != "harmonics" else (1500, 40)
    dt = psw.F32 if kind == "fp32" else psw.F64
    if kind == "p0":
        part = psw.Partition(n, [])
    elif kind == "size2":
        part = psw.Partition(n, [2, 4, 300, 302, 696, 698])
    else:
        part = psw.Partition(n, sorted(rng.choice(np.arange(2, n), 7, replace=False).tolist()))
    sub = np.empty((K, n - 1))
    diag = np.empty((K, n))
    for k in range(K):
        if kind == "harmonics":  # near-singular to strongly dominant Toeplitz systems
            sub[k] = 1.0
            diag[k] = -(2.0 + 10.0 ** rng.uniform(-7, 1))
        else:
            a = rng.uniform(0.5, 1.0, n - 1) * rng.choice([-1.0, 1.0], n - 1)
            b = np.abs(np.r_[0, a]) + np.abs(np.r_[a, 0]) + rng.uniform(0.1, 1, n)
            if kind == "mixed_sign":
                b *= rng.choice([-1.0, 1.0], n)
            sub[k], diag[k] = a, b
    plans = [psw.Plan(psw.TridiagMatrix.symmetric(sub[k], diag[k]), part, dtype=dt, staged_only=True)
             for k in range(K)]
    tdt = cuda.float32 if kind == "fp32" else cuda.float64
    F = cuda.from_numpy(rng.uniform(-1, 1, (n, K + 5))).cuda().to(tdt)
    want = psw.MultiPlan(plans).solve(F, cuda.zeros_like(F))
    got = psw.MultiPlan.from_systems(sub, diag, sub, part, dtype=dt).solve(F, cuda.zeros_like(F))
    cuda.cuda.synchronize()
    assert bool((want[:, :K] == got[:, :K]).all())
    assert bool(cuda.isfinite(got[:, :K]).all())


@pytest.mark.gpu
def test_bundle_from_systems_errors(psw, cuda):
    n, K = 40, 5
    part = psw.Partition(n, [10, 20, 30])
    sub = -np.ones((K, n - 1))
    diag = np.full((K, n), 2.5)
    sup = sub.copy()
    sup[3, 7] = -0.5
    with pytest.raises(psw.NotSupported):  # not symmetric: plans one by one
        psw.MultiPlan.from_systems(sub, diag, sup, part)
    diag[2] = 2.0  # the Neumann matrix of test_device_setup_pivot_breakdown: pivot 0 at row n-1
    diag[2, 0] = diag[2, -1] = 1.0
    with pytest.raises(psw.PivotBreakdown) as e:
        psw.MultiPlan.from_systems(sub, diag, sub, part)
    with pytest.raises(psw.PivotBreakdown) as e1:
        psw.Plan(psw.TridiagMatrix.symmetric(sub[2], diag[2]), part)
    assert e.value.row == e1.value.row == n - 1
    with pytest.raises(ValueError):
        psw.MultiPlan.from_systems(sub, diag[:, :-1], sub, part)
