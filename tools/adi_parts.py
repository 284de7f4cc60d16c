"""Times the four device operations of one ADI iteration separately (C4 grid)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0901_2859_b200 as psw  # noqa: E402
from paper_0901_2859_b200.adi import AdiIteration, AdiWorkspace, _adi_rhs  # noqa: E402

n = 4097
h = 1.0 / n
ws = AdiWorkspace(n, n, h, h, 4, 16)
f = torch.randn(n + 1, n + 1, dtype=torch.float64, device="cuda")
u = torch.zeros_like(f)
it = AdiIteration(ws, f)
it.step(u, 0)
st = ws.step(0)
tau = ws.taus[0]


def timed(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


r = {}
r["stencil1_ms"] = timed(lambda: _adi_rhs(1, u, f, it.rhs, it.ldr, n, n, h, h, tau, 0))
r["solve1_ms"] = timed(lambda: st.plan1.solve(it.rhs, it.half[1:, 1:], nrhs=n - 1, layout=psw.LAYOUT_R,
                                              ldf=it.ldr, ldx=it.half.stride(0)))
r["solve1_path"] = psw.last_path()
r["stencil2_ms"] = timed(lambda: _adi_rhs(2, it.half, f, it.rhs, it.ldr, n, n, h, h, tau, 0))
r["solve2_ms"] = timed(lambda: st.plan2.solve(it.rhs, it.next[1:, 1:], nrhs=n - 1, layout=psw.LAYOUT_S,
                                              ldf=it.ldr, ldx=it.next.stride(0)))
r["solve2_path"] = psw.last_path()
r["iteration_ms"] = timed(lambda: it.step(u, 0))
print(json.dumps(r))
