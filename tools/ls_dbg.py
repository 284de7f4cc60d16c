import sys
import sys; sys.path.insert(0, "tests")
sys.path.insert(0, ".")
import numpy as np, torch
import paper_0901_2859_b200 as psw
from conftest import load_golden
from test_parity_gpu import plan_for, gpu_solve
g = load_golden("c1_n4096_P16")
plan = plan_for(psw, g)
F = np.random.default_rng(1).standard_normal((int(sys.argv[1]), 4096))
X = gpu_solve(psw, torch, plan, F, 1, path=psw.PATH_CLUSTER)
print("ok", X.shape)
