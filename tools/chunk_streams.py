"""Feasibility probe for C2 (fp32, n = N = 65536): the RESWEEP solve run over
RHS chunks of Nc columns (F of a chunk = n Nc 4 bytes, sized for L2) on S
round-robin streams, so that a chunk's K3 can re-read its F from L2 and the
chunks' combination kernels overlap other chunks' sweeps. Times the whole
sweep with events (L2 flushed before), checks it equals the full-batch solve
bitwise. Output: one JSON line per (Nc, S, graph)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0901_2859_b200 as psw  # noqa: E402
from paper_0901_2859_b200.configs import CONFIGS  # noqa: E402

cfg = CONFIGS["C2"]
n, N = cfg.n, cfg.nrhs
a, b = cfg.matrix_ab(0)
A = psw.TridiagMatrix.symmetric(a, b)
part = psw.decompose(n, cfg.P).induced_partition()
plan = psw.Plan(A, part, psw.F32)
F = torch.empty((n, N), dtype=torch.float32, device="cuda")
psw.fill_uniform(F, 3, -1.0, 1.0)
X = torch.empty_like(F)
flush = torch.empty(2 * torch.cuda.get_device_properties(0).L2_cache_size // 4 + 1,
                    dtype=torch.float32, device="cuda")


def full():
    plan.solve(F, X)


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        psw.l2_flush(flush)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    return best


t_full = timed(full)
ref = X.clone()
print(json.dumps({"full_ms": t_full, "path": psw.last_path()}), flush=True)
GRAPH = True
for Nc in (64, 128, 256):
    for S in (1, 2, 4, 8):
        streams = [torch.cuda.Stream() for _ in range(S)]

        def chunked():
            cur = torch.cuda.current_stream()
            ev = torch.cuda.Event()
            ev.record(cur)
            for s in streams:
                s.wait_event(ev)
            for c in range(N // Nc):
                st = streams[c % S]
                plan.solve(F[:, c * Nc:(c + 1) * Nc], X[:, c * Nc:(c + 1) * Nc], nrhs=Nc,
                           ldf=N, ldx=N, stream=st)
            for s in streams:
                e2 = torch.cuda.Event()
                e2.record(s)
                cur.wait_event(e2)

        X.zero_()
        ms = timed(chunked)
        ok = bool(torch.equal(X, ref))
        out = {"Nc": Nc, "streams": S, "ms": ms, "path": psw.last_path(), "bitwise_equal_full": ok}
        if GRAPH:
            try:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    chunked()
                X.zero_()
                out["graph_ms"] = timed(g.replay)
                out["graph_bitwise_equal_full"] = bool(torch.equal(X, ref))
            except Exception as exc:  # noqa: BLE001
                out["graph_error"] = str(exc)[:200]
        print(json.dumps(out), flush=True)
