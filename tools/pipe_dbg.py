"""Debug driver: one PIPE solve vs STAGED on a golden case (layout, dtype from argv)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_0901_2859_b200 as psw
from conftest import load_golden, rel_l2
from test_parity_gpu import gpu_solve, plan_for

name, layout, dt = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
g = load_golden(name)
plan = plan_for(psw, g, dtype=dt)
N = int(sys.argv[4]) if len(sys.argv) > 4 else g["F"].shape[0]
ref = gpu_solve(psw, torch, plan, g["F"][:N], layout, path=psw.PATH_STAGED)
X = gpu_solve(psw, torch, plan, g["F"][:N], layout, path=psw.PATH_PIPE)
print(name, layout, dt, N, "bitwise", np.array_equal(X, ref), "rel", rel_l2(X, ref))
