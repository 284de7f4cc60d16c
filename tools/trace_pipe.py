"""PIPE kernel item trace (psw_debug_trace): per item type, time waiting for
dependencies and time working; timeline of the solve. Usage:
  python tools/trace_pipe.py [C1|C2|C3|C4] [R|S]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_0901_2859_b200 as psw
from paper_0901_2859_b200.configs import CONFIGS

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C1"]
lay = sys.argv[2] if len(sys.argv) > 2 else cfg.layout
cfg = cfg.with_(layout=lay)
a, b = cfg.matrix_ab(0)
A = psw.TridiagMatrix.symmetric(a, b)
plan = psw.Plan(A, psw.decompose(cfg.n, cfg.P).induced_partition(),
                dtype=psw.F64 if cfg.dtype == "f64" else psw.F32)
tdt = torch.float64 if cfg.dtype == "f64" else torch.float32
shape = (cfg.n, cfg.nrhs) if lay == "R" else (cfg.nrhs, cfg.n)
F = torch.empty(shape, dtype=tdt, device="cuda")
psw.fill_uniform(F, 1, -1.0, 1.0)
X = torch.empty_like(F)
layout = psw.LAYOUT_R if lay == "R" else psw.LAYOUT_S
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
for _ in range(3):
    plan.solve(F, X, layout=layout, path=psw.PATH_PIPE)
tr = torch.zeros(8 << 22, dtype=torch.int64, device="cuda")
psw.lib().psw_debug_trace(psw._ptr(tr))
psw.l2_flush(flush)
torch.cuda.synchronize()
plan.solve(F, X, layout=layout, path=psw.PATH_PIPE)
torch.cuda.synchronize()
psw.lib().psw_debug_trace(None)
t = tr.cpu().numpy().reshape(-1, 8)
t = t[(t[:, 2] > 0) & (t[:, 1] > 0)]  # executed items (skipped tickets have no ready stamp)
t0 = t[:, 0].min()
start, ready, end = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3, (t[:, 2] - t0) / 1e3
typ = (t[:, 3] >> 32) & 0xff
print(f"{cfg.name} {lay}: {len(t)} items, span {end.max():.1f} us")
for k, nm in enumerate("ABC"):  # B is unused (combination runs inside A items)
    m = typ == k
    if m.any():
        w, d = ready[m] - start[m], end[m] - ready[m]
        tw = t[m, 4] / 1e3
        print(f"  {nm}: n={m.sum():5d} wait mean {w.mean():7.2f} max {w.max():7.2f} us | "
              f"work mean {d.mean():7.2f} p50 {np.median(d):7.2f} max {d.max():7.2f} us "
              f"(tma wait mean {tw.mean():6.2f}) | "
              f"first start {start[m].min():7.1f} last end {end[m].max():7.1f}")
# activity histogram (busy warps per 5 us bin, by type)
bins = np.arange(0, end.max() + 5, 5.0)
print("  t(us)  A-work  B-work  C-work  waiting")
for lo in bins[:: max(1, len(bins) // 24)]:
    hi = lo + 5
    row = []
    for k in range(3):
        m = typ == k
        ov = np.clip(np.minimum(end[m], hi) - np.maximum(ready[m], lo), 0, None).sum() / 5
        row.append(ov)
    wv = np.clip(np.minimum(ready, hi) - np.maximum(start, lo), 0, None).sum() / 5
    print(f"  {lo:6.0f} {row[0]:7.1f} {row[1]:7.1f} {row[2]:7.1f} {wv:8.1f}")
