"""ADI consumer on the GPU (paper_0901_2859_b200/adi.py + psw_adi_rhs):
Peaceman-Rachford steps and solves against fixtures produced by the
reference's own AdiIteration / adi_solve (tests/gen_golden.py), and the
reference's ADI tests restated (tests/test_poisson.cpp:250-312)."""
import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


@pytest.mark.parametrize("name", ["adi_steps_24x18_pes1", "adi_steps_40x33_pes3"])
def test_three_steps_match_reference(psw, cuda, name):
    from paper_0901_2859_b200 import adi
    g = load_golden(name)
    n1, n2, pes, cycle = int(g["n1"]), int(g["n2"]), int(g["pes"]), int(g["cycle"])
    ws = adi.AdiWorkspace(n1, n2, 1.0 / n1, 1.0 / n2, cycle, pes)
    assert np.array_equal(np.array(ws.parameters()), g["taus"])
    f = cuda.from_numpy(g["f"]).cuda()
    u = cuda.from_numpy(g["u0"]).cuda()
    it = adi.AdiIteration(ws, f)
    for k in range(3):
        it.step(u, k)
    cuda.cuda.synchronize()
    got = u.cpu().numpy()
    assert _rel(got, g["u3"]) <= 1e-12
    assert np.all(got[0] == 0) and np.all(got[-1] == 0) and np.all(got[:, 0] == 0)


def test_adi_solve_matches_reference(psw, cuda):
    from paper_0901_2859_b200 import adi
    g = load_golden("adi_solve_32x32")
    n, pes, cycle, eps = int(g["n"]), int(g["pes"]), int(g["cycle"]), float(g["eps"])
    ws = adi.AdiWorkspace(n, n, 1.0 / n, 1.0 / n, cycle, pes)
    f = cuda.from_numpy(g["f"]).cuda()
    u, its = adi.adi_solve(f, eps, cuda.zeros_like(f), ws)
    assert its == int(g["iterations"])
    assert _rel(u.cpu().numpy(), g["u"]) <= 1e-10


def test_zero_problem_one_iteration(psw, cuda):  # test_poisson.cpp:250-257
    from paper_0901_2859_b200 import adi
    ws = adi.AdiWorkspace(16, 16, 1 / 16, 1 / 16, adi.adi_iteration_bound(16, 1e-5))
    f = cuda.zeros((17, 17), dtype=cuda.float64, device="cuda")
    u, its = adi.adi_solve(f, 1e-5, cuda.zeros_like(f), ws)
    assert its == 1 and bool((u == 0).all())


def _discrete_solution(f, n):
    """The 5-point difference problem solved directly (sparse LU; test only)."""
    import scipy.sparse as sp
    import scipy.sparse.linalg as spla
    h = 1.0 / n
    m = n - 1
    T = sp.diags([np.ones(m - 1), -2 * np.ones(m), np.ones(m - 1)], [-1, 0, 1]) / (h * h)
    I = sp.identity(m)
    L = sp.kron(T, I) + sp.kron(I, T)
    u = np.zeros((n + 1, n + 1))
    u[1:-1, 1:-1] = spla.spsolve(L.tocsc(), -f[1:-1, 1:-1].ravel()).reshape(m, m)
    return u


@pytest.mark.parametrize("n", [64, 128])
def test_iteration_bound_with_exact_error(psw, cuda, n):  # test_poisson.cpp:259-274
    from paper_0901_2859_b200 import adi
    eps = 1e-5
    n0 = adi.adi_iteration_bound(n, eps)
    fh, _ = adi.model_problem_host(n, n)
    disc = _discrete_solution(fh, n)
    ws = adi.AdiWorkspace(n, n, 1.0 / n, 1.0 / n, n0)
    f = cuda.from_numpy(fh).cuda()
    exact = cuda.from_numpy(disc).cuda()
    u, its = adi.adi_solve(f, eps, cuda.zeros_like(f), ws, exact=exact)
    assert its <= n0 + 2
    assert np.abs(u.cpu().numpy() - disc).max() <= eps * np.abs(disc).max()


def test_error_decreases_across_cycles(psw, cuda):  # test_poisson.cpp:276-293
    from paper_0901_2859_b200 import adi
    n, n0 = 64, 4
    fh, _ = adi.model_problem_host(n, n)
    disc = _discrete_solution(fh, n)
    ws = adi.AdiWorkspace(n, n, 1.0 / n, 1.0 / n, n0)
    f = cuda.from_numpy(fh).cuda()
    it = adi.AdiIteration(ws, f)
    u = cuda.zeros_like(f)
    prev = np.abs(disc).max()
    k = 0
    for _ in range(4):
        for _ in range(n0):
            it.step(u, k)
            k += 1
        err = np.abs(u.cpu().numpy() - disc).max()
        assert err < prev
        prev = err


def test_nonconvergence(psw, cuda):  # test_poisson.cpp:305-312
    from paper_0901_2859_b200 import adi
    n = 32
    ws = adi.AdiWorkspace(n, n, 1.0 / n, 1.0 / n, 1)
    f, _ = adi.model_problem(n, n)
    with pytest.raises(adi.NonConvergence):
        adi.adi_solve(f, 1e-300, cuda.zeros_like(f), ws)


def test_large_grid_layouts_and_paths(psw, cuda):
    """C4-sized sweep (4096^2 grid lines would be 128 MB per field): one step
    on a 1024 x 768 mesh with 8 dichotomy PEs equals the step with 1 PE
    (different partitions, same linear systems) to rounding."""
    from paper_0901_2859_b200 import adi
    n1, n2 = 1024, 768
    fh, _ = adi.model_problem_host(n1, n2)
    f = cuda.from_numpy(fh).cuda()
    rng = np.random.default_rng(1)
    u0 = np.zeros((n1 + 1, n2 + 1))
    u0[1:-1, 1:-1] = rng.uniform(-1, 1, (n1 - 1, n2 - 1))
    outs = []
    for pes in (1, 8):
        ws = adi.AdiWorkspace(n1, n2, 1.0 / n1, 1.0 / n2, 3, pes)
        u = cuda.from_numpy(u0).cuda()
        it = adi.AdiIteration(ws, f)
        for k in range(2):
            it.step(u, k)
        outs.append(u.cpu().numpy())
    assert _rel(outs[1], outs[0]) <= 1e-10


def test_stencil_division_is_ieee(psw, cuda):
    """psw_adi_rhs divides by tau and h^2 with a reciprocal and one FMA
    residual step instead of an IEEE division per node: on a random field the
    right-hand sides equal the reference's operation order (numpy, IEEE
    division) bitwise."""
    import numpy as np
    from paper_0901_2859_b200.adi import _adi_rhs
    rng = np.random.default_rng(5)
    n1, n2, h1, h2, tau = 130, 97, 1 / 130, 1 / 97, 0.0123
    u = rng.standard_normal((n1 + 1, n2 + 1))
    f = rng.standard_normal((n1 + 1, n2 + 1))
    for d in (1, 2):
        rhs = cuda.empty((n1 - 1, n2 - 1), dtype=cuda.float64, device="cuda")
        _adi_rhs(d, cuda.from_numpy(u).cuda(), cuda.from_numpy(f).cuda(), rhs, n2 - 1, n1, n2, h1, h2,
                 tau, 0)
        c = u[1:n1, 1:n2]
        if d == 1:
            lam = ((u[1:n1, 2:] - 2.0 * c) + u[1:n1, :n2 - 1]) / (h2 * h2)
            hs = -h1 * h1
        else:
            lam = ((u[2:, 1:n2] - 2.0 * c) + u[:n1 - 1, 1:n2]) / (h1 * h1)
            hs = -h2 * h2
        want = hs * ((c / tau + lam) + f[1:n1, 1:n2])
        assert np.array_equal(rhs.cpu().numpy(), want)
