"""Debug: PIPE layout S on a partition with 32-aligned (0-based) block starts."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_0901_2859_b200 as psw
from conftest import rel_l2
from test_parity_gpu import gpu_solve

n = 1024
rng = np.random.default_rng(0)
a = rng.uniform(-1, -0.5, n - 1)
b = np.abs(np.r_[0, a]) + np.abs(np.r_[a, 0]) + rng.uniform(0.1, 1, n)
A = psw.TridiagMatrix(a, b, a)
bnd = [int(x) for x in sys.argv[1].split(",")]
plan = psw.Plan(A, psw.Partition(n, bnd))
F = rng.uniform(-1, 1, (64, n))
ref = gpu_solve(psw, torch, plan, F, 1, path=psw.PATH_STAGED)
X = gpu_solve(psw, torch, plan, F, 1, path=psw.PATH_PIPE)
print(bnd, "bitwise", np.array_equal(X, ref), rel_l2(X, ref))
