"""Per-rank cost of the row-sharded C3 solve, measured on ONE GPU.

The pool has one GPU per call, so no multi-GPU run exists. This times what
one rank of a G-rank row-sharded solve executes on its own device — its
forward half (K1 + fold + its share of the p boundary values) and its
backward half (carries + K3) on its n/G rows of all 1024 RHS — with rank 0's
shard plan of the G-rank partition, no collective and no other rank running
(nothing waits on anything). The all-reduce of p x N fp64 (516 KB at
G = 8) is NOT measured; the projection adds a stated latency for it. Output:
one JSON line with per-rank ms and the implied strong-scaling efficiency
E(G) = T(1) / (G T(G)) under that assumption.

    python tools/shard_projection.py [allreduce_us]
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0901_2859_b200 as psw  # noqa: E402
from paper_0901_2859_b200.configs import CONFIGS  # noqa: E402

allreduce_us = float(sys.argv[1]) if len(sys.argv) > 1 else 25.0
cfg = CONFIGS["C3"]
a, b = cfg.matrix_ab(0)
A = psw.TridiagMatrix.symmetric(a, b)
part = psw.decompose(cfg.n, cfg.P).induced_partition()
flush = torch.empty(2 * torch.cuda.get_device_properties(0).L2_cache_size // 4 + 1,
                    dtype=torch.float32, device="cuda")


def timed(fn, reps=10):
    for _ in range(3):
        psw.l2_flush(flush)
        fn()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(reps):
        psw.l2_flush(flush)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        tot += s.elapsed_time(e)
    return tot / reps


out = {"config": "C3", "n": cfg.n, "nrhs": cfg.nrhs, "P": cfg.P,
       "allreduce_us_assumed": allreduce_us, "ranks": {}}
t1 = None
for G in (1, 2, 4, 8):
    if G == 1:
        plan = psw.Plan(A, part)
        F = torch.empty((cfg.n, cfg.nrhs), dtype=torch.float64, device="cuda")
        psw.fill_uniform(F, 3, -1.0, 1.0)
        X = torch.empty_like(F)
        ms = timed(lambda: plan.solve(F, X))
        t1 = ms
        out["ranks"]["1"] = {"ms": ms, "path": psw.last_path()}
    else:
        plan = psw.Plan(A, part, rank=0, world=G)
        rows = plan.rows()
        F = torch.empty((rows, cfg.nrhs), dtype=torch.float64, device="cuda")
        psw.fill_uniform(F, 3, -1.0, 1.0)
        X = torch.empty_like(F)
        ws = torch.empty(max(plan.workspace_bytes(cfg.nrhs), 1), dtype=torch.uint8, device="cuda")
        partials = torch.zeros((cfg.P - 1, cfg.nrhs), dtype=torch.float64, device="cuda")
        fwd = timed(lambda: plan.shard_forward(F, cfg.nrhs, ws, partials))
        both = timed(lambda: (plan.shard_forward(F, cfg.nrhs, ws, partials),
                              plan.shard_backward(F, X, cfg.nrhs, ws, partials)))
        step = both + allreduce_us / 1e3
        out["ranks"][str(G)] = {"rows": rows, "forward_ms": fwd, "forward_backward_ms": both,
                                "projected_step_ms": step,
                                "projected_efficiency": t1 / (G * step)}
    del F, X
    torch.cuda.empty_cache()
print(json.dumps(out))
