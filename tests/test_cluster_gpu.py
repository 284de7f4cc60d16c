"""CLUSTER path (psw_cluster.cu): one persistent kernel, C-CTA clusters of
G-block strips, F read once and X written once. The fp64 gate against the
reference (golden fixtures, or the CPU oracle on the same inputs) on every
case, plus agreement with STAGED to rounding; ragged N, padded leading
dimensions, fp32, the full C1 config."""
import numpy as np
import pytest

from conftest import golden_cases, load_golden, rel_l2
from test_parity_gpu import FP32_TOL, FP64_TOL, gpu_solve, plan_for

pytestmark = pytest.mark.gpu


def _oracle(sub, diag, sup, bnd, F):
    from oracle.pyoracle import Oracle
    return Oracle().solve_batch_threads(sub, diag, sup, np.asarray(bnd, np.int64),
                                        np.ascontiguousarray(F), 8)[0]


def _supported(psw, cuda, plan, F):
    try:
        gpu_solve(psw, cuda, plan, F, 0, path=psw.PATH_CLUSTER)
        return True
    except psw.NotSupported:
        return False


@pytest.mark.parametrize("name", golden_cases())
def test_cluster_golden(psw, cuda, name):
    g = load_golden(name)
    plan = plan_for(psw, g)
    if not _supported(psw, cuda, plan, g["F"]):
        assert not name.startswith(("c0_", "c1_")), name  # the BASELINE C0/C1 shapes must run
        return
    ref = gpu_solve(psw, cuda, plan, g["F"], 0, path=psw.PATH_STAGED)
    X = gpu_solve(psw, cuda, plan, g["F"], 0, path=psw.PATH_CLUSTER)
    assert rel_l2(X, ref) <= 1e-12, (name, rel_l2(X, ref))
    assert rel_l2(X, g["X"]) <= FP64_TOL, (name, rel_l2(X, g["X"]))


@pytest.mark.parametrize("N", [2, 16, 18, 100, 1000, 5000])  # even: TMA row pitch
def test_cluster_ragged(psw, cuda, N):
    g = load_golden("c1_n4096_P16")
    plan = plan_for(psw, g)
    F = np.random.default_rng(N).standard_normal((N, 4096))
    ref = gpu_solve(psw, cuda, plan, F, 0, path=psw.PATH_STAGED)
    X = gpu_solve(psw, cuda, plan, F, 0, path=psw.PATH_CLUSTER)
    X2 = gpu_solve(psw, cuda, plan, F, 0, path=psw.PATH_CLUSTER, inplace=False, pad=2)
    assert rel_l2(X, ref) <= 1e-12
    assert np.array_equal(X, X2)
    assert rel_l2(X, _oracle(g["sub"], g["diag"], g["super"], g["bnd"], F)) <= FP64_TOL


def test_cluster_c0(psw, cuda):
    g = load_golden("c0_n1024_P4")
    plan = plan_for(psw, g)
    X = gpu_solve(psw, cuda, plan, g["F"], 0, path=psw.PATH_CLUSTER)
    assert rel_l2(X, g["X"]) <= FP64_TOL


def test_cluster_fp32(psw, cuda):
    g = load_golden("c1_n4096_P16")
    plan = plan_for(psw, g, dtype=psw.F32)
    F = g["F"]
    X = gpu_solve(psw, cuda, plan, F, 0, path=psw.PATH_CLUSTER)
    assert rel_l2(X, g["X"]) <= FP32_TOL


def test_cluster_config_C1(psw, cuda):
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
    plan.solve(F, X, path=psw.PATH_CLUSTER)
    X2 = cuda.empty_like(F)
    plan.solve(F, X2, path=psw.PATH_STAGED)
    cuda.cuda.synchronize()
    assert float(((X - X2).norm() / X2.norm()).item()) <= 1e-12
    ks = np.arange(0, 4096, 7)
    Fs = F[:, cuda.from_numpy(ks).cuda()].T.cpu().numpy()
    Xs = X[:, cuda.from_numpy(ks).cuda()].T.cpu().numpy()
    want = Oracle().solve_batch_threads(a, b, a, np.array(part.boundaries), Fs, 8)[0]
    assert rel_l2(Xs, want) <= FP64_TOL


@pytest.mark.parametrize("n,P,dtype", [(4096, 16, 0), (8192, 8, 0), (2048, 4, 0), (4096, 32, 0),
                                       (1024, 4, 0), (2048, 8, 1), (4096, 8, 1)])
def test_cluster_shapes(psw, cuda, n, P, dtype):
    """Cluster sizes 1..8, blocks of 128..1024 rows, both dtypes, against STAGED."""
    rng = np.random.default_rng(n + P)
    a = rng.uniform(-1, -0.5, n - 1)
    b = np.abs(np.r_[0, a]) + np.abs(np.r_[a, 0]) + rng.uniform(0.1, 1, n)
    plan = psw.Plan(psw.TridiagMatrix.symmetric(a, b), psw.decompose(n, P).induced_partition(),
                    dtype=psw.F64 if dtype == 0 else psw.F32)
    F = rng.uniform(-1, 1, (300, n))
    if dtype == 1:
        F = F.astype(np.float32).astype(np.float64)
    ref = gpu_solve(psw, cuda, plan, F, 0, path=psw.PATH_STAGED)
    X = gpu_solve(psw, cuda, plan, F, 0, path=psw.PATH_CLUSTER)
    tol = 1e-12 if dtype == 0 else 1e-5
    assert rel_l2(X, ref) <= tol, rel_l2(X, ref)
    bnd = psw.decompose(n, P).induced_partition().boundaries
    assert rel_l2(X, _oracle(a, b, a, bnd, F)) <= (FP64_TOL if dtype == 0 else FP32_TOL)


@pytest.mark.parametrize("n,P", [(4096, 16), (2048, 4), (4096, 32), (1024, 4), (2048, 8),
                                 (8192, 16), (8192, 8)])
def test_cluster_shapes_s(psw, cuda, n, P):
    """Layout S (fp64) over cluster sizes 2..16 and blocks of 128..1024 rows,
    against STAGED; shapes whose only configuration is one block per CTA
    (excluded for layout S) report NotSupported."""
    rng = np.random.default_rng(n + 3 * P)
    a = rng.uniform(-1, -0.5, n - 1)
    b = np.abs(np.r_[0, a]) + np.abs(np.r_[a, 0]) + rng.uniform(0.1, 1, n)
    plan = psw.Plan(psw.TridiagMatrix.symmetric(a, b), psw.decompose(n, P).induced_partition(),
                    dtype=psw.F64)
    F = rng.uniform(-1, 1, (300, n))
    try:
        X = gpu_solve(psw, cuda, plan, F, 1, path=psw.PATH_CLUSTER)
    except psw.NotSupported:
        assert (n, P) not in ((4096, 16), (2048, 4), (1024, 4)), (n, P)
        return
    ref = gpu_solve(psw, cuda, plan, F, 1, path=psw.PATH_STAGED)
    assert rel_l2(X, ref) <= 1e-12, rel_l2(X, ref)
    bnd = psw.decompose(n, P).induced_partition().boundaries
    assert rel_l2(X, _oracle(a, b, a, bnd, F)) <= FP64_TOL


@pytest.mark.parametrize("N", [2, 16, 18, 100, 1000])
def test_cluster_layout_s(psw, cuda, N):
    """Layout S (fp64): 16-row swizzled TMA boxes of 16 right-hand sides."""
    g = load_golden("c1_n4096_P16")
    plan = plan_for(psw, g)
    F = np.random.default_rng(N + 7).standard_normal((N, 4096))
    ref = gpu_solve(psw, cuda, plan, F, 1, path=psw.PATH_STAGED)
    X = gpu_solve(psw, cuda, plan, F, 1, path=psw.PATH_CLUSTER)
    X2 = gpu_solve(psw, cuda, plan, F, 1, path=psw.PATH_CLUSTER, inplace=False, pad=2)
    assert rel_l2(X, ref) <= 1e-12, rel_l2(X, ref)
    assert np.array_equal(X, X2)
    assert rel_l2(X, _oracle(g["sub"], g["diag"], g["super"], g["bnd"], F)) <= FP64_TOL


@pytest.mark.parametrize("name", ["c0_n1024_P4", "c1_n4096_P16", "c4_n4096_P16"])
def test_cluster_layout_s_golden(psw, cuda, name):
    g = load_golden(name)
    plan = plan_for(psw, g)
    X = gpu_solve(psw, cuda, plan, g["F"], 1, path=psw.PATH_CLUSTER)
    assert rel_l2(X, g["X"]) <= FP64_TOL, rel_l2(X, g["X"])
