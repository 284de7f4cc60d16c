"""GPU parity: the CUDA path through the C ABI vs the reference / oracle.

Gates (BASELINE.json north_star): relative L2 <= 1e-12 for fp64 against the
reference CPU implementation at the same partition; <= 1e-5 for fp32
against the fp64 oracle run on the fp32-rounded F. Betas and boundary values
of the STAGED path are additionally bitwise the reference's.
"""
import numpy as np
import pytest

from conftest import golden_cases, load_golden, rel_l2

pytestmark = pytest.mark.gpu

FP64_TOL = 1e-12
FP32_TOL = 1e-5


def plan_for(psw, g, dtype=0):
    A = psw.TridiagMatrix(g["sub"], g["diag"], g["super"])
    return psw.Plan(A, psw.Partition(A.n(), [int(b) for b in g["bnd"]]), dtype=dtype)


def gpu_solve(psw, torch, plan, F_S, layout, path=0, pad=0, inplace=True):
    """F_S: host (N, n) system-contiguous series. Returns host (N, n)."""
    tdt = torch.float64 if plan.dtype == psw.F64 else torch.float32
    N, n = F_S.shape
    if layout == psw.LAYOUT_S:
        F = torch.zeros((N, n + pad), dtype=tdt, device="cuda")
        F[:, :n] = torch.from_numpy(F_S).to(tdt)
    else:
        F = torch.zeros((n, N + pad), dtype=tdt, device="cuda")
        F[:, :N] = torch.from_numpy(np.ascontiguousarray(F_S.T)).to(tdt)
    X = F if inplace else torch.full_like(F, float("nan"))
    plan.solve(F, X, nrhs=N, layout=layout, path=path)
    torch.cuda.synchronize()
    Xh = X.double().cpu().numpy()
    return Xh[:, :n] if layout == psw.LAYOUT_S else np.ascontiguousarray(Xh[:, :N].T)


@pytest.mark.parametrize("layout", [0, 1])
@pytest.mark.parametrize("name", golden_cases())
def test_golden_fp64(psw, cuda, name, layout):
    g = load_golden(name)
    plan = plan_for(psw, g)
    for path in (psw.PATH_STAGED, psw.PATH_AUTO):
        X = gpu_solve(psw, cuda, plan, g["F"], layout, path=path)
        assert rel_l2(X, g["X"]) <= FP64_TOL, (name, layout, path, rel_l2(X, g["X"]))
        for k in range(X.shape[0]):
            assert rel_l2(X[k], g["X"][k]) <= FP64_TOL


@pytest.mark.parametrize("name", [n for n in golden_cases() if "boundary" in load_golden(n)])
def test_golden_intermediates_bitwise(psw, cuda, name):
    g = load_golden(name)
    plan = plan_for(psw, g)
    N, n = g["F"].shape
    p = len(g["bnd"])
    F = cuda.from_numpy(np.ascontiguousarray(g["F"].T)).cuda()
    bl = cuda.zeros((p + 1, N), dtype=cuda.float64, device="cuda")
    br = cuda.zeros_like(bl)
    V = cuda.zeros((p, N), dtype=cuda.float64, device="cuda")
    plan.solve(F, layout=psw.LAYOUT_R, path=psw.PATH_STAGED, betas_left=bl, betas_right=br,
               boundary_values=V)
    cuda.cuda.synchronize()
    bl, br, V = bl.cpu().numpy().T, br.cpu().numpy().T, V.cpu().numpy().T
    # betas.hpp: left[0] and right[p] are never written (stay 0)
    assert np.array_equal(bl[:, 1:], g["betas_left"][:, 1:])
    assert np.array_equal(br[:, :p], g["betas_right"][:, :p])
    assert np.array_equal(V, g["boundary"])
    assert plan.info["combine_terms"] == int(g["combine_terms"])
    if "strategy_used" in g:  # GRowStrategy resolved like the reference (Auto)
        assert plan.info["strategy_used"] == int(g["strategy_used"])
    assert plan.info["comm_rounds"] == int(g["comm_rounds"])
    assert plan.info["max_z_norm"] == float(g["max_z"])


@pytest.mark.parametrize("name", golden_cases())
def test_fused_matches_staged_and_reference(psw, cuda, name):
    """The FUSED kernel (segmented sweeps, exact affine carries) agrees with
    the STAGED path to rounding and with the reference within the gate."""
    g = load_golden(name)
    for dtype, tol, gate in ((psw.F64, 1e-13, FP64_TOL), (psw.F32, 1e-6, FP32_TOL)):
        plan = plan_for(psw, g, dtype=dtype)
        if not plan.info["fused_ok"]:
            pytest.skip("partition not uniform: fused path not applicable")
        F = g["F"] if dtype == psw.F64 else g["F"].astype(np.float32).astype(np.float64)
        for N in (F.shape[0], 1):
            a = gpu_solve(psw, cuda, plan, F[:N], psw.LAYOUT_R, path=psw.PATH_FUSED, inplace=False,
                          pad=(-N) % 4)
            b = gpu_solve(psw, cuda, plan, F[:N], psw.LAYOUT_R, path=psw.PATH_STAGED)
            assert rel_l2(a, b) <= tol, (name, dtype, rel_l2(a, b))
            if dtype == psw.F64 or name.startswith("c2"):
                assert rel_l2(a, g["X"][:N]) <= gate, (name, dtype, rel_l2(a, g["X"][:N]))


def test_fused_wide_batches(psw, cuda):
    """Many tiles, ragged last tile, padded leading dimension."""
    from oracle.pyoracle import Oracle
    g = load_golden("c1_n4096_P16")
    plan = plan_for(psw, g)
    assert plan.info["fused_ok"]
    rng = np.random.default_rng(11)
    F = rng.standard_normal((301, 4096))
    want = Oracle().solve_batch_threads(g["sub"], g["diag"], g["super"], g["bnd"], F, 8)[0]
    X = gpu_solve(psw, cuda, plan, F, psw.LAYOUT_R, path=psw.PATH_FUSED, pad=3, inplace=False)
    assert rel_l2(X, want) <= FP64_TOL


@pytest.mark.parametrize("name", ["c2_n8192_P8", "c2_n8192_P64", "c2_n8192_P512"])
@pytest.mark.parametrize("layout", [0, 1])
def test_golden_fp32(psw, cuda, name, layout):
    g = load_golden(name)  # F already fp32-rounded; X is the fp64 reference
    plan = plan_for(psw, g, dtype=psw.F32)
    X = gpu_solve(psw, cuda, plan, g["F"], layout)
    assert rel_l2(X, g["X"]) <= FP32_TOL, rel_l2(X, g["X"])


def test_edge_shapes(psw, cuda):
    g = load_golden("decomp_n333_P9")
    plan = plan_for(psw, g)
    for layout in (0, 1):
        for N in (1, 2, 5):
            X = gpu_solve(psw, cuda, plan, g["F"][:N], layout)
            assert rel_l2(X, g["X"][:N]) <= FP64_TOL
        # padded leading dimension and out-of-place
        X = gpu_solve(psw, cuda, plan, g["F"], layout, pad=7, inplace=False)
        assert rel_l2(X, g["X"]) <= FP64_TOL
    # N not a multiple of the warp/CTA width: 33 and 161 RHS
    rng = np.random.default_rng(3)
    F = rng.uniform(-1, 1, (161, 333))
    from oracle.pyoracle import Oracle
    want = Oracle().solve_batch(g["sub"], g["diag"], g["super"], g["bnd"], F)
    for layout in (0, 1):
        for N in (33, 161):
            X = gpu_solve(psw, cuda, plan, F[:N], layout)
            assert rel_l2(X, want[:N]) <= FP64_TOL


def test_zero_and_unit_rhs(psw, cuda):
    g = load_golden("rand_n200_p7")
    plan = plan_for(psw, g)
    n = 200
    X = gpu_solve(psw, cuda, plan, np.zeros((3, n)), 0)
    assert np.all(X == 0)
    Xi = gpu_solve(psw, cuda, plan, np.eye(n), 0)  # columns of inv(A)
    A = np.diag(g["diag"]) + np.diag(g["sub"], -1) + np.diag(g["super"], 1)
    inv = np.linalg.inv(A)
    assert np.abs(Xi.T - inv).max() <= 1e-9 * max(np.abs(inv).max(), 1.0)


def test_bitwise_deterministic(psw, cuda):
    g = load_golden("c1_n4096_P16")
    plan = plan_for(psw, g)
    a = gpu_solve(psw, cuda, plan, g["F"], 0)
    b = gpu_solve(psw, cuda, plan, g["F"], 0)
    assert np.array_equal(a, b)


def test_solve_host_and_solve_batch(psw, cuda):
    g = load_golden("c0_n1024_P4")
    plan = plan_for(psw, g)
    X = plan.solve_host(np.ascontiguousarray(g["F"]), layout=psw.LAYOUT_S)
    assert rel_l2(X, g["X"]) <= FP64_TOL
    XR = plan.solve_host(np.ascontiguousarray(g["F"].T), layout=psw.LAYOUT_R)
    assert rel_l2(XR.T, X) <= 1e-13  # layout R runs the FUSED kernel
    A = psw.TridiagMatrix(g["sub"], g["diag"], g["super"])
    sols = psw.solve_batch(A, psw.Partition(1024, g["bnd"].tolist()), [row for row in g["F"]])
    assert rel_l2(np.array(sols), g["X"]) <= FP64_TOL


def test_device_generator_matches_host(psw, cuda):
    from paper_0901_2859_b200 import configs
    t = cuda.empty(100_003, dtype=cuda.float64, device="cuda")
    psw.fill_uniform(t, 77, -1.0, 1.0, offset=5)
    assert np.array_equal(t.cpu().numpy(), configs.uniform(77, 100_003, -1.0, 1.0, offset=5))
    psw.fill_normal(t, 77)
    assert np.allclose(t.cpu().numpy(), configs.normal(77, 100_003), rtol=1e-12, atol=1e-12)


# ------------------------------------------------------------------ full configs
def _config_run(psw, torch, cfg, seed=0, check_rhs=None, P=None, layout=None, path=0):
    """Device-generated config input, GPU solve, oracle check on a subset."""
    from oracle.pyoracle import Oracle
    from paper_0901_2859_b200 import configs
    cfg = cfg.with_(P=P or cfg.P, layout=layout or cfg.layout)
    a, b = cfg.matrix_ab(seed)
    A = psw.TridiagMatrix.symmetric(a, b)
    part = psw.decompose(cfg.n, cfg.P).induced_partition()
    dt = psw.F64 if cfg.dtype == "f64" else psw.F32
    plan = psw.Plan(A, part, dtype=dt)
    tdt = torch.float64 if dt == psw.F64 else torch.float32
    shape = (cfg.n, cfg.nrhs) if cfg.layout == "R" else (cfg.nrhs, cfg.n)
    F = torch.empty(shape, dtype=tdt, device="cuda")
    if cfg.rhs == "uniform":
        psw.fill_uniform(F, seed + 3, -1.0, 1.0)
    elif cfg.rhs == "normal":
        psw.fill_normal(F, seed + 3)
    else:
        F.copy_(torch.from_numpy(configs.grid_rhs(cfg.n, cfg.nrhs, seed)).to(tdt))
    ks = np.arange(cfg.nrhs) if check_rhs is None else np.asarray(check_rhs)
    lay = psw.LAYOUT_R if cfg.layout == "R" else psw.LAYOUT_S
    idx = torch.from_numpy(ks).cuda()
    Fs = (F[:, idx].T if lay == psw.LAYOUT_R else F[idx]).double().cpu().numpy()
    X = torch.empty_like(F)
    plan.solve(F, X, layout=lay, path=path)
    torch.cuda.synchronize()
    Xs = (X[:, idx].T if lay == psw.LAYOUT_R else X[idx]).double().cpu().numpy()
    want = Oracle().solve_batch_threads(a, b, a, np.array(part.boundaries), Fs, 8)[0]
    del F, X
    torch.cuda.empty_cache()
    return rel_l2(Xs, want), Xs, want


def test_config_C0_full(psw, cuda):
    from paper_0901_2859_b200.configs import CONFIGS
    err, _, _ = _config_run(psw, cuda, CONFIGS["C0"])
    assert err <= FP64_TOL, err


def test_config_C4c_full(psw, cuda):
    """C4's column direction on its own (layout R over the grid field)."""
    from paper_0901_2859_b200.configs import CONFIGS
    err, _, _ = _config_run(psw, cuda, CONFIGS["C4c"])
    assert err <= FP64_TOL, err


def test_config_C1_full(psw, cuda):
    from paper_0901_2859_b200.configs import CONFIGS
    err, _, _ = _config_run(psw, cuda, CONFIGS["C1"])
    assert err <= FP64_TOL, err


def test_config_C1_layout_S(psw, cuda):
    from paper_0901_2859_b200.configs import CONFIGS
    err, _, _ = _config_run(psw, cuda, CONFIGS["C1"], layout="S", check_rhs=np.arange(0, 4096, 7))
    assert err <= FP64_TOL, err


def test_config_C4_rows_then_columns(psw, cuda):
    """ADI-style: row sweep (systems along grid rows, layout S), then the
    column sweep (systems along columns, layout R) of the row result."""
    torch = cuda
    from oracle.pyoracle import Oracle
    from paper_0901_2859_b200.configs import CONFIGS, grid_rhs
    cfg = CONFIGS["C4"]
    a, b = cfg.matrix_ab()
    A = psw.TridiagMatrix.symmetric(a, b)
    part = psw.decompose(cfg.n, cfg.P).induced_partition()
    plan = psw.Plan(A, part)
    G = grid_rhs(cfg.n, cfg.n, 0)
    U = torch.from_numpy(G).cuda()
    plan.solve(U, layout=psw.LAYOUT_S)          # rows: U[i, :] solved in place
    plan.solve(U, layout=psw.LAYOUT_R)          # columns: U[:, j] solved in place
    torch.cuda.synchronize()
    bnd = np.array(part.boundaries)
    orc = Oracle()
    rows_ref = orc.solve_batch_threads(a, b, a, bnd, G, 8)[0]
    cols_ref = orc.solve_batch_threads(a, b, a, bnd, np.ascontiguousarray(rows_ref.T), 8)[0].T
    err = rel_l2(U.cpu().numpy(), cols_ref)
    assert err <= FP64_TOL, err


@pytest.mark.parametrize("P", [8, 64, 512])
def test_config_C2_subset(psw, cuda, P):
    from paper_0901_2859_b200.configs import CONFIGS
    rng = np.random.default_rng(P)
    ks = np.sort(rng.choice(65536, 24, replace=False))
    err, _, _ = _config_run(psw, cuda, CONFIGS["C2"], P=P, check_rhs=ks)
    assert err <= FP32_TOL, err


def test_config_C3_single_gpu_subset(psw, cuda):
    from paper_0901_2859_b200.configs import CONFIGS
    ks = np.array([0, 1, 511, 1023])
    err, _, _ = _config_run(psw, cuda, CONFIGS["C3"], check_rhs=ks)
    assert err <= FP64_TOL, err


@pytest.mark.parametrize("kind", ["symmetrizable", "mixed", "reducible"])
@pytest.mark.parametrize("strategy", [0, 1, 2, 3, 4])
def test_nonsymmetric_strategies(psw, cuda, kind, strategy):
    """GRowStrategy routes (preliminary.hpp:108-164) on the reference's
    non-symmetric goldens: the same strategy resolves (or fails) like the
    oracle, which is pinned bitwise to the reference (tests/test_strategies.py),
    and every path solves within the fp64 gate."""
    from oracle.pyoracle import Oracle, OracleError
    g = load_golden(f"nonsym_{kind}_n300_P6")
    A = psw.TridiagMatrix(g["sub"], g["diag"], g["super"])
    part = psw.Partition(A.n(), [int(b) for b in g["bnd"]])
    orc = Oracle()
    try:
        pre = orc.preliminary(g["sub"], g["diag"], g["super"], g["bnd"], strategy=strategy)
        want = orc.solve_batch(g["sub"], g["diag"], g["super"], g["bnd"], g["F"], strategy=strategy)
    except OracleError as e:
        with pytest.raises((psw.NotSymmetrizable, psw.OracleFallbackRequired)):
            psw.Plan(A, part, strategy=strategy)
        return
    plan = psw.Plan(A, part, strategy=strategy)
    assert plan.info["strategy_used"] == pre["strategy_used"]
    for path in (psw.PATH_STAGED, psw.PATH_AUTO, psw.PATH_RESWEEP):
        for layout in (0, 1):
            X = gpu_solve(psw, cuda, plan, g["F"], layout, path=path)
            assert rel_l2(X, want) <= FP64_TOL, (path, layout, rel_l2(X, want))
