"""HOLD path (psw_hold.cu): fp32, layout R, one persistent cooperative launch
whose CTAs keep a whole 32-RHS tile of all n rows in shared memory (F read
once) and exchange run aggregates / block betas / boundary values through L2.
Gate: relative L2 <= 1e-5 against the fp64 oracle on the fp32-rounded F
(BASELINE.json north_star), on the reference-generated C2 goldens, random
partitions, ragged N, padded pitches, in and out of place; run-to-run bitwise
determinism; the full-size C2 shape through a seeded RHS subset and the
device residual."""
import numpy as np
import pytest

from conftest import load_golden, rel_l2
from test_parity_gpu import FP32_TOL, gpu_solve, plan_for

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["c2_n8192_P8", "c2_n8192_P64"])
def test_hold_golden(psw, cuda, name):
    g = load_golden(name)
    plan = plan_for(psw, g, dtype=psw.F32)
    # the goldens hold 4 RHS; HOLD needs N >= 32 (one tile): every RHS nine times
    F, want = np.tile(g["F"], (9, 1)), np.tile(g["X"], (9, 1))
    X = gpu_solve(psw, cuda, plan, F, 0, path=psw.PATH_HOLD)
    assert psw.last_path() == "hold"
    assert rel_l2(X, want) <= FP32_TOL, rel_l2(X, want)
    R = gpu_solve(psw, cuda, plan, F, 0, path=psw.PATH_RESWEEP)
    assert rel_l2(X, R) <= 2e-6, rel_l2(X, R)
    X2 = gpu_solve(psw, cuda, plan, F, 0, path=psw.PATH_HOLD, inplace=False, pad=4)
    assert np.array_equal(X, X2)  # deterministic, independent of pitch / in place


def test_hold_unsupported(psw, cuda):
    g = load_golden("c2_n8192_P512")  # P > 64: no HOLD tables
    plan = plan_for(psw, g, dtype=psw.F32)
    F = np.tile(g["F"], (9, 1))
    with pytest.raises(psw.NotSupported):
        gpu_solve(psw, cuda, plan, F, 0, path=psw.PATH_HOLD)
    g = load_golden("c1_n4096_P16")  # fp64 plan
    plan = plan_for(psw, g)
    with pytest.raises(psw.NotSupported):
        gpu_solve(psw, cuda, plan, np.tile(g["F"], (9, 1)), 0, path=psw.PATH_HOLD)
    g = load_golden("c2_n8192_P8")
    plan = plan_for(psw, g, dtype=psw.F32)
    with pytest.raises(psw.NotSupported):  # layout S
        gpu_solve(psw, cuda, plan, np.tile(g["F"], (9, 1)), 1, path=psw.PATH_HOLD)
    with pytest.raises(psw.NotSupported):  # less than one tile of RHS
        gpu_solve(psw, cuda, plan, g["F"], 0, path=psw.PATH_HOLD)


@pytest.mark.parametrize("N", [32, 33, 100, 1000])
def test_hold_ragged(psw, cuda, N):
    g = load_golden("c2_n8192_P64")
    plan = plan_for(psw, g, dtype=psw.F32)
    F = np.random.default_rng(N).uniform(-1, 1, (N, 8192)).astype(np.float32).astype(np.float64)
    pad = -N % 4  # TMA needs 16-byte row pitches
    ref = gpu_solve(psw, cuda, plan, F, 0, path=psw.PATH_RESWEEP)
    X = gpu_solve(psw, cuda, plan, F, 0, path=psw.PATH_HOLD, pad=pad)
    X2 = gpu_solve(psw, cuda, plan, F, 0, path=psw.PATH_HOLD, inplace=False, pad=pad + 8)
    assert rel_l2(X, ref) <= 2e-6, rel_l2(X, ref)
    assert np.array_equal(X, X2)


@pytest.mark.parametrize("seed", range(12))
def test_hold_random_partitions(psw, cuda, seed):
    """Random (mostly non-uniform) partitions with P <= 64: CTAs straddling
    several blocks (several runs per CTA), blocks spanning many CTAs, short
    segments, ragged last tiles."""
    from oracle.pyoracle import Oracle
    rng = np.random.default_rng(9100 + seed)
    n = int(rng.integers(600, 30000))
    P = int(rng.integers(2, 65))
    if seed % 3 == 0:
        bnd = psw.decompose(n, P).induced_partition().boundaries
    else:
        bnd = sorted(rng.choice(np.arange(2, n), size=P - 1, replace=False).tolist())
    sub = -rng.uniform(0.2, 1.0, n - 1)
    diag = np.r_[0, np.abs(sub)] + np.r_[np.abs(sub), 0] + rng.uniform(0.1, 1.0, n)
    plan = psw.Plan(psw.TridiagMatrix(sub, diag, sub), psw.Partition(n, bnd), dtype=psw.F32)
    N = int(rng.integers(32, 300))
    F = rng.uniform(-1, 1, (N, n)).astype(np.float32).astype(np.float64)
    want = Oracle().solve_batch_threads(sub, diag, sub, np.array(bnd, np.int64), F, 8)[0]
    X = gpu_solve(psw, cuda, plan, F, 0, path=psw.PATH_HOLD, inplace=bool(seed % 2),
                  pad=-N % 4 + 4 * int(rng.integers(0, 3)))
    assert rel_l2(X, want) <= FP32_TOL, (seed, n, P, N, rel_l2(X, want))


def test_hold_c2_shape(psw, cuda):
    """The fp32 config's system (n = 65536, P = 64, 14 segments per CTA, three
    tiles in flight) with 4096 RHS: HOLD is explicit only (AUTO keeps RESWEEP,
    which is faster there); a seeded RHS subset against the oracle, every RHS through the device residual, two runs
    bitwise equal."""
    from oracle.pyoracle import Oracle
    from paper_0901_2859_b200.configs import CONFIGS
    cfg = CONFIGS["C2"]
    a, b = cfg.matrix_ab(0)
    A = psw.TridiagMatrix.symmetric(a, b)
    part = psw.decompose(cfg.n, cfg.P).induced_partition()
    plan = psw.Plan(A, part, dtype=psw.F32)
    N = 4096
    F = cuda.empty((cfg.n, N), dtype=cuda.float32, device="cuda")
    psw.fill_uniform(F, 5, -1.0, 1.0)
    X = cuda.empty_like(F)
    plan.solve(F, X)
    assert psw.last_path() == "resweep"
    plan.solve(F, X, path=psw.PATH_HOLD)
    assert psw.last_path() == "hold"
    cuda.cuda.synchronize()
    X2 = cuda.empty_like(F)
    plan.solve(F, X2, path=psw.PATH_HOLD)
    assert cuda.equal(X, X2)
    ks = np.arange(0, N, 171)
    idx = cuda.from_numpy(ks).cuda()
    Fs = F[:, idx].T.double().cpu().numpy()
    Xs = X[:, idx].T.double().cpu().numpy()
    want = Oracle().solve_batch_threads(a, b, a, np.array(part.boundaries), Fs, 8)[0]
    assert rel_l2(Xs, want) <= FP32_TOL, rel_l2(Xs, want)
    ad = cuda.from_numpy(a).cuda().float()
    bd = cuda.from_numpy(b).cuda().float()
    R = bd[:, None] * X
    R[1:] += ad[:, None] * X[:-1]
    R[:-1] += ad[:, None] * X[1:]
    res = ((R - F).norm(dim=0) / F.norm(dim=0)).max()
    assert float(res) <= 2e-6, float(res)
