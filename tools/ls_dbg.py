"""Debug helper: CLUSTER layout S vs STAGED on the C1 golden matrix; prints
the rows and right-hand sides that differ."""
import sys
sys.path.insert(0, "tests")
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_0901_2859_b200 as psw
from conftest import load_golden
from test_parity_gpu import plan_for, gpu_solve

g = load_golden("c1_n4096_P16")
plan = plan_for(psw, g)
N = int(sys.argv[1]) if len(sys.argv) > 1 else 32
F = np.random.default_rng(1).standard_normal((N, 4096))
LAY = int(sys.argv[2]) if len(sys.argv) > 2 else 1
ref = gpu_solve(psw, torch, plan, F, LAY, path=psw.PATH_STAGED)
X = gpu_solve(psw, torch, plan, F, LAY, path=psw.PATH_CLUSTER)
d = np.abs(X - ref) > 1e-9 * (1 + np.abs(ref))
print("N", N, "bad", int(d.sum()), "of", d.size)
if d.any():
    rows = np.unique(np.nonzero(d)[1])
    print("bad rows", rows[:40], "count", len(rows))
    print("bad rhs", np.unique(np.nonzero(d)[0])[:20])
if d.any():
    r = np.nonzero(d.any(axis=0))[0]
    iv = []
    s0 = r[0]
    for u, v in zip(r[:-1], r[1:]):
        if v != u + 1:
            iv.append((s0, u)); s0 = v
    iv.append((s0, r[-1]))
    print("row intervals", iv)
    for k in (1, 2, 8, 9):
        print("rhs", k, "bad rows", np.nonzero(d[k])[0][:12])
if d.any():
    e = np.abs(X - ref)
    for k in (1, 8):
        top = np.argsort(-e[k])[:6]
        print("rhs", k, "largest errors at rows", sorted(top.tolist()), "max", e[k].max())
        print("  err rows 30..70:", np.array2string(e[k, 30:70], precision=1, max_line_width=250))
