"""GPU-side preliminary (psw_prelim.cu): the 3p boundary
sweeps of compute_preliminary (preliminary.hpp:171-199) on the device must be
bitwise the host restatement (itself bitwise the reference): same betas, same
boundary values and solutions, same max_z_norm, same pivot breakdown row."""
import os

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu


class _env:
    def __init__(self, **kv):
        self.kv = kv

    def __enter__(self):
        self.old = {k: os.environ.get(k) for k in self.kv}
        os.environ.update({k: str(v) for k, v in self.kv.items()})

    def __exit__(self, *a):
        for k, v in self.old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def _plans(psw, A, part):
    with _env(PSW_DEVICE_SETUP=0):
        host = psw.Plan(A, part)
    with _env(PSW_DEVICE_SETUP=1):
        dev = psw.Plan(A, part)
    assert host.info["device_setup"] == 0 and dev.info["device_setup"] == 1
    return host, dev


def _solve_all(psw, cuda, plan, F):
    Fd = cuda.from_numpy(np.ascontiguousarray(F.T)).cuda()
    X = cuda.empty_like(Fd)
    N = F.shape[0]
    p = int(plan.info["p"])
    bl = cuda.zeros(p + 1, N, dtype=cuda.float64, device="cuda")
    br = cuda.zeros(p + 1, N, dtype=cuda.float64, device="cuda")
    V = cuda.zeros(max(p, 1), N, dtype=cuda.float64, device="cuda")
    plan.solve(Fd, X, layout=psw.LAYOUT_R, path=psw.PATH_STAGED, betas_left=bl, betas_right=br,
               boundary_values=V)
    X2 = cuda.empty_like(Fd)
    plan.solve(Fd, X2, layout=psw.LAYOUT_R)
    cuda.cuda.synchronize()
    return [t.cpu().numpy() for t in (X, bl, br, V, X2)]


@pytest.mark.parametrize("case", ["c1", "c0", "rand_nonuniform", "c2_P512", "p1"])
def test_device_setup_is_bitwise_the_host_setup(psw, cuda, case):
    rng = np.random.default_rng(11)
    if case in ("c1", "c0", "c2_P512"):
        name = {"c1": "c1_n4096_P16", "c0": "c0_n1024_P4", "c2_P512": "c2_n8192_P512"}[case]
        g = load_golden(name)
        A = psw.TridiagMatrix(g["sub"], g["diag"], g["super"])
        part = psw.Partition(A.n(), [int(b) for b in g["bnd"]])
        F = g["F"]
    else:
        n = 3000 if case == "rand_nonuniform" else 500
        a = rng.uniform(-1, -0.5, n - 1)
        b = np.abs(np.r_[0, a]) + np.abs(np.r_[a, 0]) + rng.uniform(0.1, 1, n)
        A = psw.TridiagMatrix.symmetric(a, b)
        bnd = sorted(rng.choice(np.arange(2, n), 36, replace=False).tolist()) if n == 3000 else [250]
        part = psw.Partition(n, bnd)
        F = rng.uniform(-1, 1, (9, n))
    host, dev = _plans(psw, A, part)
    assert host.info["max_z_norm"] == dev.info["max_z_norm"]
    for a_, b_ in zip(_solve_all(psw, cuda, host, F), _solve_all(psw, cuda, dev, F)):
        assert np.array_equal(a_, b_)


def test_device_setup_pivot_breakdown(psw, cuda):
    n = 40
    # a singular principal block: breakdown inside the g-row sweep of boundary 0
    A = psw.TridiagMatrix.constant(n, -1.0, 2.0, -1.0)
    A.diag[0] = 1.0  # Neumann ends: singular, the forward pivots reach zero at row n-1
    A.diag[n - 1] = 1.0
    part = psw.Partition(n, [10, 20, 30])
    rows = []
    for dev in (0, 1):
        with _env(PSW_DEVICE_SETUP=dev):
            with pytest.raises(psw.PivotBreakdown) as e:
                psw.Plan(A, part)
            rows.append(e.value.row)
    assert rows[0] == rows[1]


def test_device_setup_large(psw, cuda):
    """C3 shape (n = 2^20, P = 64): the device setup is bitwise the host setup
    on a probe of right-hand sides (timings printed; the host is the default)."""
    import time
    from paper_0901_2859_b200.configs import CONFIGS
    cfg = CONFIGS["C3"]
    a, b = cfg.matrix_ab(0)
    A = psw.TridiagMatrix.symmetric(a, b)
    part = psw.decompose(cfg.n, cfg.P).induced_partition()
    t0 = time.perf_counter()
    with _env(PSW_DEVICE_SETUP=0):
        host = psw.Plan(A, part)
    t1 = time.perf_counter()
    with _env(PSW_DEVICE_SETUP=1):
        dev = psw.Plan(A, part)
    t2 = time.perf_counter()
    assert dev.info["device_setup"] == 1
    assert host.info["max_z_norm"] == dev.info["max_z_norm"]
    F = np.random.default_rng(3).uniform(-1, 1, (4, cfg.n))
    for a_, b_ in zip(_solve_all(psw, cuda, host, F), _solve_all(psw, cuda, dev, F)):
        assert np.array_equal(a_, b_)
    print(f"C3 setup: host {t1 - t0:.3f} s, device {t2 - t1:.3f} s")
