"""Times the Fourier consumer on the device: the DST-I (psw_dst_rows) against
the cuFFT-based odd-extension transform it replaced, and one fourier_solve
(DST, multi-plan solve of all harmonics, inverse DST) on an n x n mesh."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0901_2859_b200.fourier import FourierWorkspace, dst_raw, fourier_solve  # noqa: E402


def cufft_dst(x):
    m = x.shape[-1]
    n = m + 1
    v = torch.zeros(*x.shape[:-1], 2 * n, dtype=torch.float64, device=x.device)
    v[..., 1:n] = x
    v[..., n + 1:] = -torch.flip(x, dims=[-1])
    return -0.5 * torch.fft.fft(v, dim=-1)[..., 1:n].imag


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
pes = int(sys.argv[2]) if len(sys.argv) > 2 else 16
x = torch.randn(n - 1, n - 1, dtype=torch.float64, device="cuda")
out = torch.empty_like(x)
res = {"n": n, "pes": pes}
res["dst_ms"] = timed(lambda: dst_raw(x, out=out))
res["cufft_dst_ms"] = timed(lambda: cufft_dst(x))
res["dst_max_diff"] = float((dst_raw(x) - cufft_dst(x)).abs().max() / cufft_dst(x).abs().max())
t0 = time.perf_counter()
ws = FourierWorkspace(n, n, 1.0 / n, 1.0 / n, pes)
res["workspace_s"] = time.perf_counter() - t0
f = torch.randn(n + 1, n + 1, dtype=torch.float64, device="cuda")
res["fourier_solve_ms"] = timed(lambda: fourier_solve(f, ws), reps=5)
rhs = torch.randn(n - 1, n - 1, dtype=torch.float64, device="cuda")
res["solve_harmonics_ms"] = timed(lambda: ws.solve_harmonics(rhs), reps=5)
print(json.dumps(res))
