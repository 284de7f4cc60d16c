"""psw_solve_host on C3 (pinned host buffers): wall time per call for the
current PSW_HOST_* settings, plus raw pitched-copy bandwidth by row width."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0901_2859_b200 as psw  # noqa: E402
from paper_0901_2859_b200.configs import CONFIGS  # noqa: E402

cfg = CONFIGS["C3"]
a, b = cfg.matrix_ab(0)
plan = psw.Plan(psw.TridiagMatrix.symmetric(a, b), psw.decompose(cfg.n, cfg.P).induced_partition())
Fh = torch.empty((cfg.n, cfg.nrhs), dtype=torch.float64, pin_memory=True)
Fh.uniform_(-1, 1)
Xh = torch.empty((cfg.n, cfg.nrhs), dtype=torch.float64, pin_memory=True)
out = {"env": {k: v for k, v in os.environ.items() if k.startswith("PSW_HOST")}}
plan.solve_host(Fh.numpy(), Xh.numpy(), layout=psw.LAYOUT_R)
ts = []
for _ in range(3):
    t = time.perf_counter()
    plan.solve_host(Fh.numpy(), Xh.numpy(), layout=psw.LAYOUT_R)
    ts.append((time.perf_counter() - t) * 1e3)
out["solve_host_ms"] = ts
print(json.dumps(out))

# the link itself: 8 GB contiguous H2D alone, D2H alone, both at once (two streams)
dev_a = torch.empty((cfg.n, cfg.nrhs), dtype=torch.float64, device="cuda")
dev_b = torch.empty_like(dev_a)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
nb = Fh.numel() * 8


def wall(fn):
    torch.cuda.synchronize()
    t = time.perf_counter()
    fn()
    torch.cuda.synchronize()
    return time.perf_counter() - t


for _ in range(2):
    h2d = wall(lambda: dev_a.copy_(Fh, non_blocking=True))
    d2h = wall(lambda: Xh.copy_(dev_b, non_blocking=True))

    def both():
        with torch.cuda.stream(s1):
            dev_a.copy_(Fh, non_blocking=True)
        with torch.cuda.stream(s2):
            Xh.copy_(dev_b, non_blocking=True)
    bo = wall(both)
link = {"h2d_gbs": nb / h2d / 1e9, "d2h_gbs": nb / d2h / 1e9, "both_ms": bo * 1e3,
        "both_aggregate_gbs": 2 * nb / bo / 1e9}
print(json.dumps({"link": link}))
