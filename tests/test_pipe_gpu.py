"""PIPE path (psw_pipe.cu): one persistent kernel, RHS chunks whose forward
intermediates stay in L2, ticket-ordered segment work items with exact
affine carries.

Against the reference the fp64 gate (rel L2 <= 1e-12) applies; against the
STAGED path (same algorithm, betas summed per segment instead of per block)
the difference is rounding only. Small chunk sizes force many chunks through
the scratch slots (slot reuse, counter ordering); lag 1 and few CTAs force
the ticket order to carry the dependencies.
"""
import os

import numpy as np
import pytest

from conftest import golden_cases, load_golden, rel_l2
from test_parity_gpu import FP32_TOL, FP64_TOL, gpu_solve, plan_for

pytestmark = pytest.mark.gpu


class _env:
    def __init__(self, **kw):
        self.kw = {k: str(v) for k, v in kw.items()}

    def __enter__(self):
        self.old = {k: os.environ.get(k) for k in self.kw}
        os.environ.update(self.kw)

    def __exit__(self, *a):
        for k, v in self.old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


@pytest.mark.parametrize("layout", [0, 1])
@pytest.mark.parametrize("name", golden_cases())
def test_pipe_golden_bitwise_staged(psw, cuda, name, layout):
    g = load_golden(name)
    plan = plan_for(psw, g)
    if len(g["bnd"]) + 1 > 64:
        pytest.skip("PIPE stages at most 64 block betas")
    ref = gpu_solve(psw, cuda, plan, g["F"], layout, path=psw.PATH_STAGED)
    X = gpu_solve(psw, cuda, plan, g["F"], layout, path=psw.PATH_PIPE)
    assert rel_l2(X, ref) <= 1e-13, (name, layout, rel_l2(X, ref))
    assert rel_l2(X, g["X"]) <= FP64_TOL


@pytest.mark.parametrize("cfg", [dict(PSW_PIPE_CHUNK_MB=1),
                                 dict(PSW_PIPE_CHUNK_MB=1, PSW_PIPE_LAG=1, PSW_PIPE_SLOTS=2,
                                      PSW_PIPE_CTAS_PER_SM=1),
                                 dict(PSW_PIPE_LAG=3, PSW_PIPE_SLOTS=5)])
@pytest.mark.parametrize("layout", [0, 1])
def test_pipe_many_chunks(psw, cuda, cfg, layout):
    """C1 golden matrix, 1000 RHS: 1 MiB chunks = 32 RHS -> 32 chunks."""
    g = load_golden("c1_n4096_P16")
    plan = plan_for(psw, g)
    rng = np.random.default_rng(5)
    F = rng.standard_normal((1000, 4096))
    ref = gpu_solve(psw, cuda, plan, F, layout, path=psw.PATH_STAGED)
    with _env(**cfg):
        X = gpu_solve(psw, cuda, plan, F, layout, path=psw.PATH_PIPE)
        X2 = gpu_solve(psw, cuda, plan, F, layout, path=psw.PATH_PIPE, inplace=False, pad=5)
    assert rel_l2(X, ref) <= 1e-13
    assert np.array_equal(X2, X)


@pytest.mark.parametrize("name", ["c2_n8192_P8", "c2_n8192_P64", "c2_n8192_P512"])
@pytest.mark.parametrize("layout", [0, 1])
def test_pipe_golden_fp32(psw, cuda, name, layout):
    g = load_golden(name)
    plan = plan_for(psw, g, dtype=psw.F32)
    if "P512" in name:
        with pytest.raises(psw.NotSupported):
            gpu_solve(psw, cuda, plan, g["F"], layout, path=psw.PATH_PIPE)
        return
    ref = gpu_solve(psw, cuda, plan, g["F"], layout, path=psw.PATH_STAGED)
    X = gpu_solve(psw, cuda, plan, g["F"], layout, path=psw.PATH_PIPE)
    assert rel_l2(X, ref) <= 1e-6
    assert rel_l2(X, g["X"]) <= FP32_TOL, rel_l2(X, g["X"])


def test_pipe_edge_shapes(psw, cuda):
    from oracle.pyoracle import Oracle
    g = load_golden("decomp_n333_P9")
    plan = plan_for(psw, g)
    rng = np.random.default_rng(3)
    F = rng.uniform(-1, 1, (161, 333))
    want = Oracle().solve_batch(g["sub"], g["diag"], g["super"], g["bnd"], F)
    for layout in (0, 1):
        for N in (1, 2, 5, 31, 33, 64, 161):
            for inplace, pad in ((True, 0), (False, 3)):
                X = gpu_solve(psw, cuda, plan, F[:N], layout, path=psw.PATH_PIPE, pad=pad,
                              inplace=inplace)
                assert rel_l2(X, want[:N]) <= FP64_TOL, (layout, N, inplace)


def test_pipe_rejects_too_many_blocks(psw, cuda):
    g = load_golden("c2_n8192_P512")
    plan = plan_for(psw, g)
    F = cuda.zeros((8192, 4), dtype=cuda.float64, device="cuda")
    with pytest.raises(psw.NotSupported):
        plan.solve(F, nrhs=4, layout=psw.LAYOUT_R, path=psw.PATH_PIPE)
    plan.solve(F, nrhs=4, layout=psw.LAYOUT_R)  # AUTO falls back to STAGED


def test_pipe_deterministic_and_repeatable(psw, cuda):
    g = load_golden("c4_n4096_P16")
    plan = plan_for(psw, g)
    a = gpu_solve(psw, cuda, plan, g["F"], 1, path=psw.PATH_PIPE)
    for _ in range(3):
        b = gpu_solve(psw, cuda, plan, g["F"], 1, path=psw.PATH_PIPE)
        assert np.array_equal(a, b)


def _cfg_pipe(psw, torch, cfg, check_rhs, layout=None, P=None):
    from oracle.pyoracle import Oracle
    from paper_0901_2859_b200 import configs
    cfg = cfg.with_(P=P or cfg.P, layout=layout or cfg.layout)
    a, b = cfg.matrix_ab(0)
    A = psw.TridiagMatrix.symmetric(a, b)
    part = psw.decompose(cfg.n, cfg.P).induced_partition()
    dt = psw.F64 if cfg.dtype == "f64" else psw.F32
    plan = psw.Plan(A, part, dtype=dt)
    tdt = torch.float64 if dt == psw.F64 else torch.float32
    lay = psw.LAYOUT_R if cfg.layout == "R" else psw.LAYOUT_S
    shape = (cfg.n, cfg.nrhs) if lay == psw.LAYOUT_R else (cfg.nrhs, cfg.n)
    F = torch.empty(shape, dtype=tdt, device="cuda")
    if cfg.rhs == "normal":
        psw.fill_normal(F, 3)
    else:
        psw.fill_uniform(F, 3, -1.0, 1.0)
    idx = torch.from_numpy(np.asarray(check_rhs)).cuda()
    Fs = (F[:, idx].T if lay == psw.LAYOUT_R else F[idx]).double().cpu().numpy()
    X = torch.empty_like(F)
    plan.solve(F, X, layout=lay, path=psw.PATH_PIPE)
    torch.cuda.synchronize()
    Xs = (X[:, idx].T if lay == psw.LAYOUT_R else X[idx]).double().cpu().numpy()
    want = Oracle().solve_batch_threads(a, b, a, np.array(part.boundaries), Fs, 8)[0]
    del F, X
    torch.cuda.empty_cache()
    return rel_l2(Xs, want)


@pytest.mark.parametrize("layout", ["R", "S"])
def test_pipe_config_C1(psw, cuda, layout):
    from paper_0901_2859_b200.configs import CONFIGS
    err = _cfg_pipe(psw, cuda, CONFIGS["C1"], np.arange(0, 4096, 5), layout=layout)
    assert err <= FP64_TOL, err


@pytest.mark.parametrize("P", [64])
def test_pipe_config_C2_subset(psw, cuda, P):
    from paper_0901_2859_b200.configs import CONFIGS
    ks = np.sort(np.random.default_rng(P).choice(65536, 24, replace=False))
    err = _cfg_pipe(psw, cuda, CONFIGS["C2"], ks, P=P)
    assert err <= FP32_TOL, err


def test_pipe_rejects_long_blocks(psw, cuda):
    """C3 blocks hold 512 segments: beyond the carry-fold scratch."""
    from paper_0901_2859_b200.configs import CONFIGS
    with pytest.raises(psw.NotSupported):
        _cfg_pipe(psw, cuda, CONFIGS["C3"].with_(nrhs=64), np.array([0, 1]))
