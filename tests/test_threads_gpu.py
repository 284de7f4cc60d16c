"""Thread safety of the drop-in (SURVEY §8(b) "Threading"): a plan is
immutable after creation and psw_solve may be called from several host
threads on different streams at once (reference: pure functions over a
shared const PreliminaryData, executor.hpp:37-41). Every path's results are
bitwise the sequential ones."""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cfgname,paths", [("C1", ["AUTO", "CLUSTER", "RESWEEP", "STAGED"]),
                                           ("C4", ["AUTO", "RESWEEP"])])
def test_concurrent_streams_one_plan(psw, cuda, cfgname, paths):
    from paper_0901_2859_b200.configs import CONFIGS
    cfg = CONFIGS[cfgname]
    a, b = cfg.matrix_ab(0)
    A = psw.TridiagMatrix.symmetric(a, b)
    plan = psw.Plan(A, psw.decompose(cfg.n, cfg.P).induced_partition())
    lay = psw.LAYOUT_R if cfg.layout == "R" else psw.LAYOUT_S
    shape = (cfg.n, 1024) if lay == psw.LAYOUT_R else (1024, cfg.n)
    jobs = []
    for i, name in enumerate(paths * 2):
        F = cuda.empty(shape, dtype=cuda.float64, device="cuda")
        psw.fill_normal(F, 100 + i)
        jobs.append((getattr(psw, "PATH_" + name), F))
    cuda.cuda.synchronize()
    want = [plan.solve(F, cuda.empty_like(F), layout=lay, path=p) for p, F in jobs]
    cuda.cuda.synchronize()
    got = [None] * len(jobs)
    errs = []

    def run(i):
        try:
            s = cuda.cuda.Stream()
            p, F = jobs[i]
            with cuda.cuda.stream(s):
                X = cuda.empty_like(F)
                for _ in range(3):
                    plan.solve(F, X, layout=lay, path=p, stream=s)
                s.synchronize()
            got[i] = X
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=run, args=(i,)) for i in range(len(jobs))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for w, g in zip(want, got):
        assert bool((w == g).all())


def test_concurrent_plan_creation_with_device_setup(psw, cuda):
    """Plans created from several host threads at once, their preliminary
    sweeps on the device (psw_prelim.cu: own scratch per call, default-stream
    kernels), while another thread keeps solving: every table is bitwise the
    host setup's, and the solves are unaffected."""
    import os
    rng = np.random.default_rng(21)
    n = 30000
    mats = []
    for _ in range(4):
        a = rng.uniform(-1, -0.5, n - 1)
        b = np.abs(np.r_[0, a]) + np.abs(np.r_[a, 0]) + rng.uniform(0.1, 1, n)
        mats.append(psw.TridiagMatrix.symmetric(a, b))
    part = psw.decompose(n, 32).induced_partition()
    old = os.environ.get("PSW_DEVICE_SETUP")
    try:
        os.environ["PSW_DEVICE_SETUP"] = "0"
        want = [psw.debug_preliminary(A, part) for A in mats]
        os.environ["PSW_DEVICE_SETUP"] = "1"
        plan = psw.Plan(mats[0], part)
        F = cuda.empty((n, 256), dtype=cuda.float64, device="cuda")
        psw.fill_normal(F, 5)
        Xw = plan.solve(F, cuda.empty_like(F))
        cuda.cuda.synchronize()
        got = [None] * len(mats)
        errs, Xs = [], []

        def create(i):
            try:
                for _ in range(3):
                    got[i] = psw.debug_preliminary(mats[i], part)
            except Exception as e:  # noqa: BLE001
                errs.append(e)

        def solve():
            try:
                s = cuda.cuda.Stream()
                with cuda.cuda.stream(s):
                    for _ in range(20):
                        X = plan.solve(F, cuda.empty_like(F), stream=s)
                    s.synchronize()
                Xs.append(X)
            except Exception as e:  # noqa: BLE001
                errs.append(e)

        th = [threading.Thread(target=create, args=(i,)) for i in range(len(mats))]
        th.append(threading.Thread(target=solve))
        for t in th:
            t.start()
        for t in th:
            t.join()
    finally:
        if old is None:
            os.environ.pop("PSW_DEVICE_SETUP", None)
        else:
            os.environ["PSW_DEVICE_SETUP"] = old
    assert not errs, errs
    for w, g in zip(want, got):
        assert g["device_setup"] == 1 and w["device_setup"] == 0
        for key in ("gr", "gl", "zr", "zl"):
            assert np.array_equal(w[key].view(np.int64), g[key].view(np.int64)), key
        assert w["max_z"] == g["max_z"]
    assert bool((Xs[0] == Xw).all())
