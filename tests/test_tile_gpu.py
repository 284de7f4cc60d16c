"""TILE path (psw_tile.cu): one CTA per RHS tile, two passes over the
tile's rows (segment partials, in-CTA scans + tabulated combination, exact
re-sweep), no cross-CTA exchange.

Gates: rel L2 <= 1e-12 (fp64) against the reference at the same partition;
against the STAGED path (exact dichotomy, block-order beta sums) the
difference is rounding only (combination matrix, segment-order sums).
"""
import os

import numpy as np
import pytest

from conftest import golden_cases, load_golden, rel_l2
from test_parity_gpu import FP32_TOL, FP64_TOL, gpu_solve, plan_for
from test_pipe_gpu import _env

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("layout", [0, 1])
@pytest.mark.parametrize("name", golden_cases())
def test_tile_golden(psw, cuda, name, layout):
    g = load_golden(name)
    plan = plan_for(psw, g)
    if len(g["bnd"]) + 1 > 256:
        pytest.skip("TILE stages at most 256 block betas")
    ref = gpu_solve(psw, cuda, plan, g["F"], layout, path=psw.PATH_STAGED)
    X = gpu_solve(psw, cuda, plan, g["F"], layout, path=psw.PATH_TILE)
    assert rel_l2(X, ref) <= 1e-13, (name, layout, rel_l2(X, ref))
    assert rel_l2(X, g["X"]) <= FP64_TOL


@pytest.mark.parametrize("cfg", [dict(), dict(PSW_TILE_THREADS=128, PSW_TILE_CTAS=3),
                                 dict(PSW_TILE_SMEM_KB=40), dict(PSW_TILE_THREADS=64)])
@pytest.mark.parametrize("layout", [0, 1])
def test_tile_variants(psw, cuda, cfg, layout):
    """Few CTAs walking many tiles, partials in global scratch, small CTAs,
    ragged last tile, padded leading dimension, out of place."""
    g = load_golden("c1_n4096_P16")
    plan = plan_for(psw, g)
    rng = np.random.default_rng(5)
    F = rng.standard_normal((333, 4096))
    ref = gpu_solve(psw, cuda, plan, F, layout, path=psw.PATH_STAGED)
    with _env(**cfg):
        X = gpu_solve(psw, cuda, plan, F, layout, path=psw.PATH_TILE)
        X2 = gpu_solve(psw, cuda, plan, F, layout, path=psw.PATH_TILE, inplace=False, pad=3)
    assert rel_l2(X, ref) <= 1e-13
    assert np.array_equal(X2, X)


@pytest.mark.parametrize("name", ["c2_n8192_P8", "c2_n8192_P64", "c2_n8192_P512"])
@pytest.mark.parametrize("layout", [0, 1])
def test_tile_golden_fp32(psw, cuda, name, layout):
    g = load_golden(name)
    plan = plan_for(psw, g, dtype=psw.F32)
    if "P512" in name:  # block betas staged in shared memory: P <= 256
        with pytest.raises(psw.NotSupported):
            gpu_solve(psw, cuda, plan, g["F"], layout, path=psw.PATH_TILE)
        return
    X = gpu_solve(psw, cuda, plan, g["F"], layout, path=psw.PATH_TILE)
    assert rel_l2(X, g["X"]) <= FP32_TOL, rel_l2(X, g["X"])


def test_tile_edge_shapes(psw, cuda):
    from oracle.pyoracle import Oracle
    g = load_golden("decomp_n333_P9")
    plan = plan_for(psw, g)
    rng = np.random.default_rng(3)
    F = rng.uniform(-1, 1, (161, 333))
    want = Oracle().solve_batch(g["sub"], g["diag"], g["super"], g["bnd"], F)
    for layout in (0, 1):
        for N in (1, 2, 5, 15, 17, 33, 161):
            X = gpu_solve(psw, cuda, plan, F[:N], layout, path=psw.PATH_TILE)
            assert rel_l2(X, want[:N]) <= FP64_TOL, (layout, N)


def test_tile_deterministic(psw, cuda):
    g = load_golden("c4_n4096_P16")
    plan = plan_for(psw, g)
    a = gpu_solve(psw, cuda, plan, g["F"], 1, path=psw.PATH_TILE)
    for _ in range(3):
        assert np.array_equal(a, gpu_solve(psw, cuda, plan, g["F"], 1, path=psw.PATH_TILE))


def _cfg_tile(psw, torch, cfg, check_rhs, layout=None, P=None):
    from oracle.pyoracle import Oracle
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
    plan.solve(F, X, layout=lay, path=psw.PATH_TILE)
    torch.cuda.synchronize()
    Xs = (X[:, idx].T if lay == psw.LAYOUT_R else X[idx]).double().cpu().numpy()
    want = Oracle().solve_batch_threads(a, b, a, np.array(part.boundaries), Fs, 8)[0]
    del F, X
    torch.cuda.empty_cache()
    return rel_l2(Xs, want)


@pytest.mark.parametrize("layout", ["R", "S"])
def test_tile_config_C1(psw, cuda, layout):
    from paper_0901_2859_b200.configs import CONFIGS
    err = _cfg_tile(psw, cuda, CONFIGS["C1"], np.arange(0, 4096, 5), layout=layout)
    assert err <= FP64_TOL, err


@pytest.mark.parametrize("P", [8, 64, 256])
def test_tile_config_C2_subset(psw, cuda, P):
    from paper_0901_2859_b200.configs import CONFIGS
    ks = np.sort(np.random.default_rng(P).choice(65536, 16, replace=False))
    err = _cfg_tile(psw, cuda, CONFIGS["C2"].with_(nrhs=4096), ks[ks < 4096] if (ks < 4096).any() else np.arange(8), P=P)
    assert err <= FP32_TOL, err


def test_tile_config_C3_subset(psw, cuda):
    from paper_0901_2859_b200.configs import CONFIGS
    err = _cfg_tile(psw, cuda, CONFIGS["C3"].with_(nrhs=64), np.array([0, 1, 31, 32, 63]))
    assert err <= FP64_TOL, err
