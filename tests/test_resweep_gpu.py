"""RESWEEP path (psw_resweep.cu): F read twice, X written once, per-segment
checkpoints of the block sweeps. Betas and boundary values are the STAGED
path's (bitwise the reference's), so X agrees with STAGED to rounding; the fp64
gate against the reference on every golden case, both dtypes, ragged N,
padded leading dimensions, in place and out of place."""
import numpy as np
import pytest

from conftest import golden_cases, load_golden, rel_l2
from test_parity_gpu import FP32_TOL, FP64_TOL, gpu_solve, plan_for

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("layout", [0, 1])
@pytest.mark.parametrize("name", golden_cases())
def test_resweep_golden(psw, cuda, name, layout):
    g = load_golden(name)
    plan = plan_for(psw, g)
    ref = gpu_solve(psw, cuda, plan, g["F"], layout, path=psw.PATH_STAGED)
    X = gpu_solve(psw, cuda, plan, g["F"], layout, path=psw.PATH_RESWEEP)
    assert rel_l2(X, ref) <= 1e-12, (name, rel_l2(X, ref))
    assert rel_l2(X, g["X"]) <= FP64_TOL, (name, rel_l2(X, g["X"]))


@pytest.mark.parametrize("layout", [0, 1])
@pytest.mark.parametrize("N", [1, 5, 127, 129, 1000])
def test_resweep_ragged(psw, cuda, N, layout):
    g = load_golden("c1_n4096_P16")
    plan = plan_for(psw, g)
    F = np.random.default_rng(N).standard_normal((N, 4096))
    ref = gpu_solve(psw, cuda, plan, F, layout, path=psw.PATH_STAGED)
    X = gpu_solve(psw, cuda, plan, F, layout, path=psw.PATH_RESWEEP)
    X2 = gpu_solve(psw, cuda, plan, F, layout, path=psw.PATH_RESWEEP, inplace=False, pad=3)
    assert rel_l2(X, ref) <= 1e-13
    assert np.array_equal(X, X2)


@pytest.mark.parametrize("layout", [0, 1])
@pytest.mark.parametrize("name", ["c2_n8192_P8", "c2_n8192_P64", "c2_n8192_P512"])
def test_resweep_fp32(psw, cuda, name, layout):
    g = load_golden(name)
    plan = plan_for(psw, g, dtype=psw.F32)
    X = gpu_solve(psw, cuda, plan, g["F"], layout, path=psw.PATH_RESWEEP)
    assert rel_l2(X, g["X"]) <= FP32_TOL


def test_resweep_config_C1(psw, cuda):
    from paper_0901_2859_b200.configs import CONFIGS
    from oracle.pyoracle import Oracle
    cfg = CONFIGS["C1"]
    a, b = cfg.matrix_ab(0)
    A = psw.TridiagMatrix.symmetric(a, b)
    part = psw.decompose(cfg.n, cfg.P).induced_partition()
    plan = psw.Plan(A, part)
    F = cuda.empty((cfg.n, cfg.nrhs), dtype=cuda.float64, device="cuda")
    psw.fill_normal(F, 3)
    X = cuda.empty_like(F)
    plan.solve(F, X, path=psw.PATH_RESWEEP)
    ks = np.arange(0, 4096, 7)
    Fs = F[:, cuda.from_numpy(ks).cuda()].T.cpu().numpy()
    Xs = X[:, cuda.from_numpy(ks).cuda()].T.cpu().numpy()
    want = Oracle().solve_batch_threads(a, b, a, np.array(part.boundaries), Fs, 8)[0]
    assert rel_l2(Xs, want) <= FP64_TOL


def test_retired_paths(psw, cuda):
    """PIPE (3), TILE (4), CHUNKED (5) and HOLD (8) were explicit-only paths
    that lost to CLUSTER / RESWEEP; they are retired and answer NotSupported."""
    g = load_golden("c1_n4096_P16")
    plan = plan_for(psw, g)
    for path in (3, 4, psw.PATH_CHUNKED, psw.PATH_HOLD):
        with pytest.raises(psw.NotSupported):
            gpu_solve(psw, cuda, plan, g["F"], 0, path=path)


def test_resweep_c3_full(psw, cuda):
    """The headline config C3 at full size (n = 2^20, N = 1024) on the
    default path: a seeded RHS subset against the oracle, the rest through
    the size-independent backward error ||A x - f|| / ||f||."""
    from oracle.pyoracle import Oracle
    from paper_0901_2859_b200.configs import CONFIGS
    cfg = CONFIGS["C3"]
    a, b = cfg.matrix_ab(0)
    A = psw.TridiagMatrix.symmetric(a, b)
    part = psw.decompose(cfg.n, cfg.P).induced_partition()
    plan = psw.Plan(A, part)
    F = cuda.empty((cfg.n, cfg.nrhs), dtype=cuda.float64, device="cuda")
    psw.fill_uniform(F, 3, -1.0, 1.0)
    X = cuda.empty_like(F)
    plan.solve(F, X)
    assert psw.last_path() == "resweep"
    ks = np.arange(0, cfg.nrhs, 97)
    idx = cuda.from_numpy(ks).cuda()
    Fs = F[:, idx].T.cpu().numpy()
    Xs = X[:, idx].T.cpu().numpy()
    want = Oracle().solve_batch_threads(a, b, a, np.array(part.boundaries), Fs, 8)[0]
    assert rel_l2(Xs, want) <= FP64_TOL
    # every RHS: residual of the tridiagonal product on the device
    ad = cuda.from_numpy(a).cuda()
    bd = cuda.from_numpy(b).cuda()
    R = bd[:, None] * X
    R[1:] += ad[:, None] * X[:-1]
    R[:-1] += ad[:, None] * X[1:]
    res = ((R - F).norm(dim=0) / F.norm(dim=0)).max()
    assert float(res) <= 1e-13


@pytest.mark.parametrize("seed", range(16))
def test_resweep_tma_random_partitions(psw, cuda, seed):
    """The TMA-pipelined RESWEEP kernels (layout R, N >= one 256-byte chunk,
    16-byte row pitch) on random partitions: groups straddling several blocks
    (several runs per group, closed-form carries per run), short segments
    (the register fallback when a segment cannot lend its exchange rows),
    ragged last chunks and padded pitches; fp64 and fp32 against the oracle."""
    from oracle.pyoracle import Oracle
    rng = np.random.default_rng(7000 + seed)
    n = int(rng.integers(300, 6000))
    P = int(rng.integers(2, min(120, n // 3)))
    if seed % 3 == 0:
        bnd = psw.decompose(n, P).induced_partition().boundaries
    else:
        bnd = sorted(rng.choice(np.arange(2, n), size=P - 1, replace=False).tolist())
    sub = -rng.uniform(0.2, 1.0, n - 1)
    diag = np.r_[0, np.abs(sub)] + np.r_[np.abs(sub), 0] + rng.uniform(0.1, 1.0, n)
    f32 = seed % 4 == 3
    plan = psw.Plan(psw.TridiagMatrix(sub, diag, sub), psw.Partition(n, bnd),
                    dtype=psw.F32 if f32 else psw.F64)
    N = int(rng.integers(64, 400))
    F = rng.uniform(-1, 1, (N, n))
    if f32:
        F = F.astype(np.float32).astype(np.float64)
    want = Oracle().solve_batch_threads(sub, diag, sub, np.array(bnd, np.int64), F, 8)[0]
    pad = int(rng.integers(0, 3)) * (4 if f32 else 2)  # keeps 16-byte row pitches
    X = gpu_solve(psw, cuda, plan, F, 0, path=psw.PATH_RESWEEP, inplace=bool(seed % 2), pad=pad)
    tol = FP32_TOL if f32 else FP64_TOL
    assert rel_l2(X, want) <= tol, (seed, n, P, N, f32, rel_l2(X, want))
