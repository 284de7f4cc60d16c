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
