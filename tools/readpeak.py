"""Read-only and copy bandwidth of this B200 on an 8 GiB buffer (torch
kernels): what K1 (read F) and K3 (read F, write X) can reach at best."""
import json
import torch

x = torch.empty(1 << 30, dtype=torch.float64, device="cuda").uniform_()
y = torch.empty_like(x)
out = {}
for name, fn, nbytes in [("sum_read", lambda: x.sum(), 8 << 30),
                         ("copy", lambda: y.copy_(x), 16 << 30),
                         ("max_read", lambda: x.amax(), 8 << 30)]:
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(5):
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    out[name] = {"ms": best, "gbs": nbytes / (best / 1e3) / 1e9}
print(json.dumps(out))
