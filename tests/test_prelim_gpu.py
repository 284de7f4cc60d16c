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
    assert host.info["device_setup"] == 0 and dev.info["device_setup"] in (1, 2)
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
    on a probe of right-hand sides and on the raw tables (timings printed)."""
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
    assert dev.info["device_setup"] == 1  # chunked pivot chain accepted (dominant matrix)
    assert host.info["max_z_norm"] == dev.info["max_z_norm"]
    F = np.random.default_rng(3).uniform(-1, 1, (4, cfg.n))
    for a_, b_ in zip(_solve_all(psw, cuda, host, F), _solve_all(psw, cuda, dev, F)):
        assert np.array_equal(a_, b_)
    print(f"C3 setup: host {t1 - t0:.3f} s, device {t2 - t1:.3f} s")
    _tables_bitwise(psw, A, part, expect=1)


def _tables(psw, A, part, dev, **env):
    with _env(PSW_DEVICE_SETUP=dev, **env):
        return psw.debug_preliminary(A, part)


def _tables_bitwise(psw, A, part, expect=None, **env):
    """The preliminary's raw tables, bit for bit (signed zeros included)."""
    h = _tables(psw, A, part, 0)
    d = _tables(psw, A, part, 1, **env)
    assert h["device_setup"] == 0 and d["device_setup"] in (1, 2)
    if expect is not None:
        assert d["device_setup"] == expect, d["device_setup"]
    for k in ("gr", "gl", "zr", "zl"):
        a, b = h[k].view(np.int64), d[k].view(np.int64)
        bad = np.flatnonzero(a.ravel() != b.ravel())
        assert bad.size == 0, (k, bad[:8], h[k].ravel()[bad[:8]], d[k].ravel()[bad[:8]])
    assert h["max_z"] == d["max_z"]
    return d


def _dominant(rng, n, lo=0.1, hi=1.0, sign=None, offsign=None):
    a = rng.uniform(0.5, 1.0, n - 1) * (rng.choice([-1.0, 1.0], n - 1) if offsign is None else offsign)
    b = np.abs(np.r_[0, a]) + np.abs(np.r_[a, 0]) + rng.uniform(lo, hi, n)
    if sign is None:
        b *= rng.choice([-1.0, 1.0], n)
    else:
        b *= sign
    return a, b


@pytest.mark.parametrize("kind", ["pos", "neg", "mixed_diag", "weak", "long_blocks_neg",
                                  "long_blocks_mixed", "size2_blocks"])
def test_device_tables_bitwise(psw, cuda, kind):
    """Raw tables against the host sweeps on matrices that exercise every
    branch: positive / negative / mixed-sign pivots (the anchor search of the
    signed-zero regions), blocks far longer than the betas' decay length
    (exact zeros inside the stored g rows and at the far Z samples), weak
    dominance (slow merges), size-2 blocks."""
    rng = np.random.default_rng({"pos": 1, "neg": 2, "mixed_diag": 3, "weak": 4,
                                 "long_blocks_neg": 5, "long_blocks_mixed": 6,
                                 "size2_blocks": 7}[kind])
    if kind in ("pos", "neg", "mixed_diag"):
        n = 6000
        a, b = _dominant(rng, n, sign={"pos": 1.0, "neg": -1.0, "mixed_diag": None}[kind])
        bnd = sorted(rng.choice(np.arange(2, n), 23, replace=False).tolist())
    elif kind == "weak":
        n = 5000
        a, b = _dominant(rng, n, lo=1e-3, hi=1e-2, sign=1.0, offsign=-1.0)
        bnd = sorted(rng.choice(np.arange(2, n), 9, replace=False).tolist())
    elif kind.startswith("long_blocks"):
        n = 40000
        a, b = _dominant(rng, n, sign=-1.0 if kind.endswith("neg") else None)
        bnd = [9000, 21000, 33000]
    else:
        n = 400
        a, b = _dominant(rng, n, sign=1.0)
        bnd = [2, 4, 6, 100, 102, 396, 398]
    A = psw.TridiagMatrix.symmetric(a, b)
    part = psw.Partition(n, bnd)
    d = _tables_bitwise(psw, A, part)
    if kind.startswith("long_blocks"):  # exact zeros really are inside the tables
        assert np.count_nonzero(d["gl"] == 0.0) > 1000 and np.count_nonzero(d["zr"] == 0.0) > 0


def test_device_tables_serial_chain(psw, cuda):
    """Matrices whose pivot chain does not contract ((-1, 2, -1): pivots
    (i+2)/(i+1)) refuse the chunked chain; the one-thread chain takes over and
    the non-decaying betas run the full length. Also forced by a zero warm-up."""
    n = 3000
    A = psw.TridiagMatrix.constant(n, -1.0, 2.0, -1.0)
    part = psw.Partition(n, [700, 1500, 2900])
    _tables_bitwise(psw, A, part, expect=2)
    rng = np.random.default_rng(8)
    a, b = _dominant(rng, 5000, sign=1.0)
    A = psw.TridiagMatrix.symmetric(a, b)
    part = psw.Partition(5000, [1000, 2500, 4000])
    _tables_bitwise(psw, A, part, expect=1)
    _tables_bitwise(psw, A, part, expect=2, PSW_PRELIM_WARM=0)
    _tables_bitwise(psw, A, part, expect=1, PSW_PRELIM_CHUNK=64, PSW_PRELIM_WARM=200)


def test_device_window_overflow_falls_back_to_host(psw, cuda):
    """A chain longer than the scratch window hands the sweeps to the host
    (device_setup = 0), with the same tables."""
    n = 3000
    A = psw.TridiagMatrix.constant(n, -1.0, 2.0, -1.0)
    part = psw.Partition(n, [700, 1500, 2900])
    h = _tables(psw, A, part, 0)
    d = _tables(psw, A, part, 1, PSW_PRELIM_WINDOW=512)
    assert d["device_setup"] == 0
    for k in ("gr", "gl", "zr", "zl"):
        assert np.array_equal(h[k].view(np.int64), d[k].view(np.int64))


def test_device_setup_is_the_default(psw, cuda):
    """Without PSW_DEVICE_SETUP the device takes the sweeps of systems with at
    least 2^21 row steps (3 p n); small ones stay on the host's threads."""
    os.environ.pop("PSW_DEVICE_SETUP", None)
    g = load_golden("c1_n4096_P16")
    A = psw.TridiagMatrix(g["sub"], g["diag"], g["super"])
    part = psw.Partition(A.n(), [int(b) for b in g["bnd"]])
    assert psw.Plan(A, part).info["device_setup"] == 0
    from paper_0901_2859_b200.configs import CONFIGS
    cfg = CONFIGS["C2"]
    a, b = cfg.matrix_ab(0)
    A = psw.TridiagMatrix.symmetric(a, b)
    part = psw.decompose(cfg.n, cfg.P).induced_partition()
    assert psw.Plan(A, part, dtype=psw.F32).info["device_setup"] == 1


def test_device_z_right_breakdown(psw, cuda):
    """A breakdown only a z_right system sees (its unit first row changes the
    pivots that follow): same row as the host."""
    n = 60
    rng = np.random.default_rng(9)
    a, b = _dominant(rng, n, sign=1.0, offsign=-1.0)
    # row 21's pivot in the system that starts with a unit row at row 20 is
    # b[21] + a[20] * (-0.0) = b[21]: make it vanish there only
    b[21] = 0.0
    A = psw.TridiagMatrix.symmetric(a, b)
    part = psw.Partition(n, [10, 21, 40])
    rows = []
    for dev in (0, 1):
        with _env(PSW_DEVICE_SETUP=dev):
            with pytest.raises(psw.PivotBreakdown) as e:
                psw.Plan(A, part)
            rows.append(e.value.row)
    assert rows[0] == rows[1] == 1
