"""psw_solve_host timing per config/path (diagnostics for the e2e leg)."""
import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
import paper_0901_2859_b200 as psw
from paper_0901_2859_b200.configs import CONFIGS, host_rhs

name = sys.argv[1]
cfg = CONFIGS[name]
a, b = cfg.matrix_ab(0)
plan = psw.Plan(psw.TridiagMatrix.symmetric(a, b), psw.decompose(cfg.n, cfg.P).induced_partition(),
                dtype=psw.F64 if cfg.dtype == "f64" else psw.F32)
layout = psw.LAYOUT_R if cfg.layout == "R" else psw.LAYOUT_S
shape = (cfg.n, cfg.nrhs) if layout == psw.LAYOUT_R else (cfg.nrhs, cfg.n)
dt = torch.float64 if cfg.dtype == "f64" else torch.float32
F = torch.randn(*shape, dtype=dt).pin_memory()
X = torch.empty_like(F).pin_memory()
Fn, Xn = F.numpy(), X.numpy()
plan.solve_host(Fn, Xn, layout=layout)
torch.cuda.synchronize()
ts = []
for _ in range(3):
    t0 = time.perf_counter(); plan.solve_host(Fn, Xn, layout=layout); ts.append(time.perf_counter() - t0)
print(name, "solve_host ms", [round(1e3 * t, 2) for t in ts], "path", psw.last_path())
# device-only solve of one chunk-sized batch for comparison
Fd = F.cuda(); Xd = torch.empty_like(Fd)
plan.solve(Fd, Xd, layout=layout); torch.cuda.synchronize()
t0 = time.perf_counter(); plan.solve(Fd, Xd, layout=layout); torch.cuda.synchronize()
print(name, "device solve ms", round(1e3 * (time.perf_counter() - t0), 3), psw.last_path())
