"""Times one Peaceman-Rachford ADI iteration on the device (the C4 grid:
4096 x 4096 interior nodes, h = 1/4097): the two half steps, each a stencil
pass (psw_adi_rhs) and one batched solve of all grid lines (direction 1 in
layout R, direction 2 in layout S), against the bytes a fused iteration
would move."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0901_2859_b200.adi import AdiIteration, AdiWorkspace  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4097  # cells: n - 1 interior nodes per line
pes = int(sys.argv[2]) if len(sys.argv) > 2 else 16
h = 1.0 / n
ws = AdiWorkspace(n, n, h, h, 4, pes)
f = torch.randn(n + 1, n + 1, dtype=torch.float64, device="cuda")
u = torch.zeros_like(f)
it = AdiIteration(ws, f)
for k in range(3):
    it.step(u, k)
torch.cuda.synchronize()
reps = 20
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for k in range(reps):
    it.step(u, k)
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / reps
nodes = (n - 1) ** 2
print(json.dumps({"cells": n, "pes": pes, "ms_per_iteration": ms, "nodes": nodes,
                  "bytes_moved_per_iteration": 2 * (3 + 2) * 8 * nodes,
                  "bytes_if_fused": 2 * 3 * 8 * nodes,
                  "achieved_gbs": 2 * (3 + 2) * 8 * nodes / (ms / 1e3) / 1e9}))
