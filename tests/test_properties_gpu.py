"""Size-independent properties at the BASELINE configs' full sizes (where the
oracle cannot follow): the residual of the computed solution, linearity,
determinism, and randomized small cases against the oracle over paths,
layouts, dtypes and partitions."""
import numpy as np
import pytest

from conftest import rel_l2

pytestmark = pytest.mark.gpu


def _residual(torch, a, b, c, X, F, layout):
    """Normwise backward error max_k ||A x_k - f_k|| / (||A||_inf ||x_k|| + ||f_k||)
    for X, F in layout R (n, N) or S (N, n): a backward-stable solve keeps it
    at a modest multiple of the unit roundoff whatever the conditioning."""
    if layout == 1:
        X, F = X.T, F.T
    Xd, Fd = X.double(), F.double()
    a_t = torch.from_numpy(a).to(X.device)[:, None]
    b_t = torch.from_numpy(b).to(X.device)[:, None]
    c_t = torch.from_numpy(c).to(X.device)[:, None]
    r = b_t * Xd - Fd
    r[1:] += a_t * Xd[:-1]
    r[:-1] += c_t * Xd[1:]
    anorm = float(np.max(np.abs(b) + np.r_[0, np.abs(a)] + np.r_[np.abs(c), 0]))
    den = anorm * Xd.norm(dim=0) + Fd.norm(dim=0)
    return float((r.norm(dim=0) / den.clamp_min(1e-300)).max())


def _config(psw, torch, name, **over):
    from paper_0901_2859_b200.configs import CONFIGS
    cfg = CONFIGS[name].with_(**over) if over else CONFIGS[name]
    a, b = cfg.matrix_ab(0)
    A = psw.TridiagMatrix.symmetric(a, b)
    part = psw.decompose(cfg.n, cfg.P).induced_partition()
    dt = psw.F64 if cfg.dtype == "f64" else psw.F32
    plan = psw.Plan(A, part, dtype=dt)
    tdt = torch.float64 if dt == psw.F64 else torch.float32
    lay = psw.LAYOUT_R if cfg.layout == "R" else psw.LAYOUT_S
    shape = (cfg.n, cfg.nrhs) if lay == psw.LAYOUT_R else (cfg.nrhs, cfg.n)
    return cfg, a, b, plan, tdt, lay, shape


@pytest.mark.parametrize("name,tol", [("C1", 1e-14), ("C3", 1e-14), ("C4", 1e-14)])
def test_full_size_residual(psw, cuda, name, tol):
    cfg, a, b, plan, tdt, lay, shape = _config(psw, cuda, name)
    F = cuda.empty(shape, dtype=tdt, device="cuda")
    psw.fill_uniform(F, 5, -1.0, 1.0)
    X = plan.solve(F, cuda.empty_like(F), layout=lay)
    cuda.cuda.synchronize()
    assert _residual(cuda, a, b, a, X, F, lay) <= tol
    del F, X
    cuda.cuda.empty_cache()


def test_full_size_residual_C2_fp32(psw, cuda):
    """C2 at its full 65536 x 65536 fp32 size (16 GiB per operand)."""
    cfg, a, b, plan, tdt, lay, shape = _config(psw, cuda, "C2")
    F = cuda.empty(shape, dtype=tdt, device="cuda")
    psw.fill_uniform(F, 5, -1.0, 1.0)
    X = cuda.empty_like(F)
    plan.solve(F, X, layout=lay)
    cuda.cuda.synchronize()
    worst = 0.0
    for k0 in range(0, cfg.nrhs, 4096):  # residual in column slabs
        worst = max(worst, _residual(cuda, a, b, a, X[:, k0:k0 + 4096], F[:, k0:k0 + 4096], lay))
    assert worst <= 1e-6
    del F, X
    cuda.cuda.empty_cache()


@pytest.mark.parametrize("path", ["AUTO", "STAGED", "RESWEEP", "CLUSTER"])
def test_linearity_C1(psw, cuda, path):
    cfg, a, b, plan, tdt, lay, shape = _config(psw, cuda, "C1")
    p = getattr(psw, "PATH_" + path)
    F1 = cuda.empty(shape, dtype=tdt, device="cuda")
    F2 = cuda.empty_like(F1)
    psw.fill_normal(F1, 1)
    psw.fill_normal(F2, 2)
    X1 = plan.solve(F1, cuda.empty_like(F1), layout=lay, path=p)
    X2 = plan.solve(F2, cuda.empty_like(F1), layout=lay, path=p)
    X3 = plan.solve(F1 + 2.0 * F2, cuda.empty_like(F1), layout=lay, path=p)
    cuda.cuda.synchronize()
    err = float(((X3 - (X1 + 2.0 * X2)).norm() / X3.norm()))
    assert err <= 1e-13


def test_determinism_fused_C1(psw, cuda):
    cfg, a, b, plan, tdt, lay, shape = _config(psw, cuda, "C1")
    F = cuda.empty(shape, dtype=tdt, device="cuda")
    psw.fill_normal(F, 7)
    X1 = plan.solve(F, cuda.empty_like(F), layout=lay)
    X2 = plan.solve(F, cuda.empty_like(F), layout=lay)
    cuda.cuda.synchronize()
    assert bool((X1 == X2).all())


@pytest.mark.parametrize("seed", range(12))
def test_randomized_against_oracle(psw, cuda, seed):
    """Random n, partition (uniform or not), N, layout, dtype and path."""
    from oracle.pyoracle import Oracle
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(40, 1500))
    P = int(rng.integers(1, min(40, n // 2)))
    if rng.random() < 0.5:
        bnd = psw.decompose(n, P).induced_partition().boundaries
    else:
        bnd = sorted(rng.choice(np.arange(2, n), size=P - 1, replace=False).tolist()) if P > 1 else []
    sub = -rng.uniform(0.2, 1.0, n - 1)
    diag = np.r_[0, np.abs(sub)] + np.r_[np.abs(sub), 0] + rng.uniform(0.1, 1.0, n)
    A = psw.TridiagMatrix(sub, diag, sub)
    part = psw.Partition(n, bnd)
    N = int(rng.integers(1, 300))
    layout = int(rng.integers(0, 2))
    f32 = bool(rng.random() < 0.3)
    plan = psw.Plan(A, part, dtype=psw.F32 if f32 else psw.F64)
    F = rng.uniform(-1, 1, (N, n))
    if f32:
        F = F.astype(np.float32).astype(np.float64)
    want = Oracle().solve_batch(sub, diag, sub, np.array(bnd, np.int64), F)
    from test_parity_gpu import gpu_solve
    paths = [psw.PATH_AUTO, psw.PATH_STAGED, psw.PATH_RESWEEP, psw.PATH_CLUSTER, psw.PATH_FUSED]
    for path in paths:
        try:
            X = gpu_solve(psw, cuda, plan, F, layout, path=path)
        except psw.NotSupported:
            continue
        tol = 1e-5 if f32 else 1e-12
        assert rel_l2(X, want) <= tol, (seed, path, n, P, N, layout, f32, rel_l2(X, want))
