"""CHUNKED path (psw_chunked.cu): segment-parallel sweeps over L2-sized RHS
chunks on two forked streams. Rounding-level agreement with STAGED, the
fp64 gate against the reference, every partition kind, ragged chunks."""
import numpy as np
import pytest

from conftest import golden_cases, load_golden, rel_l2
from test_parity_gpu import FP32_TOL, FP64_TOL, gpu_solve, plan_for
from test_pipe_gpu import _env

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", golden_cases())
def test_chunked_golden(psw, cuda, name):
    g = load_golden(name)
    plan = plan_for(psw, g)
    if len(g["bnd"]) + 1 > 96:  # block betas staged in shared memory
        with pytest.raises(psw.NotSupported):
            gpu_solve(psw, cuda, plan, g["F"], 0, path=psw.PATH_CHUNKED)
        return
    ref = gpu_solve(psw, cuda, plan, g["F"], 0, path=psw.PATH_STAGED)
    X = gpu_solve(psw, cuda, plan, g["F"], 0, path=psw.PATH_CHUNKED)
    assert rel_l2(X, ref) <= 1e-13, (name, rel_l2(X, ref))
    assert rel_l2(X, g["X"]) <= FP64_TOL


@pytest.mark.parametrize("mb", [1, 3, 24])
def test_chunked_many_chunks(psw, cuda, mb):
    """1 MiB chunks of n = 4096 fp64 -> 128-RHS chunks on alternating streams."""
    g = load_golden("c1_n4096_P16")
    plan = plan_for(psw, g)
    F = np.random.default_rng(9).standard_normal((1000, 4096))
    ref = gpu_solve(psw, cuda, plan, F, 0, path=psw.PATH_STAGED)
    with _env(PSW_CHUNK_MB=mb):
        X = gpu_solve(psw, cuda, plan, F, 0, path=psw.PATH_CHUNKED)
        X2 = gpu_solve(psw, cuda, plan, F, 0, path=psw.PATH_CHUNKED, inplace=False, pad=3)
    assert rel_l2(X, ref) <= 1e-13
    assert np.array_equal(X, X2)


@pytest.mark.parametrize("name", ["c2_n8192_P8", "c2_n8192_P64", "c2_n8192_P512"])
def test_chunked_fp32(psw, cuda, name):
    g = load_golden(name)
    plan = plan_for(psw, g, dtype=psw.F32)
    if "P512" in name:
        with pytest.raises(psw.NotSupported):
            gpu_solve(psw, cuda, plan, g["F"], 0, path=psw.PATH_CHUNKED)
        return
    X = gpu_solve(psw, cuda, plan, g["F"], 0, path=psw.PATH_CHUNKED)
    assert rel_l2(X, g["X"]) <= FP32_TOL


def test_chunked_config_C1(psw, cuda):
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
    plan.solve(F, X, path=psw.PATH_CHUNKED)
    ks = np.arange(0, 4096, 7)
    Fs = F[:, cuda.from_numpy(ks).cuda()].T.cpu().numpy()
    Xs = X[:, cuda.from_numpy(ks).cuda()].T.cpu().numpy()
    want = Oracle().solve_batch_threads(a, b, a, np.array(part.boundaries), Fs, 8)[0]
    assert rel_l2(Xs, want) <= FP64_TOL
