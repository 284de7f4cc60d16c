"""C4 e2e with the bench's inputs (grid field) vs random inputs."""
import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
import paper_0901_2859_b200 as psw
from paper_0901_2859_b200.configs import CONFIGS, grid_rhs

cfg = CONFIGS["C4"]
a, b = cfg.matrix_ab(0)
plan = psw.Plan(psw.TridiagMatrix.symmetric(a, b), psw.decompose(cfg.n, cfg.P).induced_partition())
for kind in ("grid", "randn", "grid-dev", "grid-dev-empty"):
    if kind == "grid":
        F = torch.from_numpy(grid_rhs(cfg.n, cfg.nrhs, 0)).double().contiguous().pin_memory()
    elif kind == "randn":
        F = torch.randn(cfg.nrhs, cfg.n, dtype=torch.float64).pin_memory()
    elif kind == "grid-dev":
        Fd = torch.from_numpy(grid_rhs(cfg.n, cfg.nrhs, 0)).double().cuda()
        F = Fd.cpu().pin_memory()
    else:
        Fd = torch.from_numpy(grid_rhs(cfg.n, cfg.nrhs, 0)).double().cuda()
        F = torch.empty(Fd.shape, dtype=Fd.dtype, pin_memory=True)
        F.copy_(Fd)
    X = torch.empty(F.shape, dtype=F.dtype, pin_memory=True) if kind == "grid-dev-empty" else torch.empty_like(F).pin_memory()
    plan.solve_host(F.numpy(), X.numpy(), layout=psw.LAYOUT_S)
    ts = []
    for _ in range(3):
        t0 = time.perf_counter(); plan.solve_host(F.numpy(), X.numpy(), layout=psw.LAYOUT_S); ts.append(time.perf_counter() - t0)
    print(kind, [round(1e3 * t, 2) for t in ts], "max|X|", float(X.abs().max()), "min nonzero |X|", float(X.abs()[X != 0].min()))
