"""psw_solve_host end-to-end time on C1 for several chunk sizes (one process each)."""
import os
import subprocess
import sys

CODE = r'''
import time, numpy as np, torch, sys
sys.path.insert(0, ".")
import paper_0901_2859_b200 as psw
from paper_0901_2859_b200.configs import CONFIGS
cfg = CONFIGS["C1"]
a, b = cfg.matrix_ab(0)
plan = psw.Plan(psw.TridiagMatrix.symmetric(a, b), psw.decompose(cfg.n, cfg.P).induced_partition())
F = torch.randn(cfg.n, cfg.nrhs, dtype=torch.float64).pin_memory()
X = torch.empty_like(F).pin_memory()
Fn, Xn = F.numpy(), X.numpy()
plan.solve_host(Fn, Xn, layout=psw.LAYOUT_R)
ts = []
for _ in range(10):
    t0 = time.perf_counter(); plan.solve_host(Fn, Xn, layout=psw.LAYOUT_R); ts.append(time.perf_counter() - t0)
print(f"chunk {sys.argv[1]} MB: median {1e3*sorted(ts)[5]:.3f} ms  min {1e3*min(ts):.3f} ms")
'''
for mb in (2, 4, 8, 16, 32):
    env = dict(os.environ, PSW_HOST_CHUNK_MB=str(mb))
    subprocess.run([sys.executable, "-c", CODE, str(mb)], env=env, check=False)
