"""Phase trace of the FUSED kernel (profiling aid, psw_debug_trace).

    python tools/trace_fused.py [--config C1] [--rb 128]

Runs one traced solve and prints, per phase, the median / p90 duration in
SM cycles over all CTAs, plus how many CTAs were resident at once.
"""
import argparse
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

PHASES = ["forward (chunk wait + sweep)", "sync + issue + scan + push", "exchange wait + combine",
          "sync", "backward (carries + sweep)", "reload d~ + sync + issue (LAG)"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C1")
    ap.add_argument("--nrhs", type=int, default=None)
    args = ap.parse_args()
    import torch
    import paper_0901_2859_b200 as psw
    from paper_0901_2859_b200.configs import CONFIGS
    cfg = CONFIGS[args.config]
    if args.nrhs:
        cfg = cfg.with_(nrhs=args.nrhs)
    a, b = cfg.matrix_ab(0)
    plan = psw.Plan(psw.TridiagMatrix.symmetric(a, b), psw.decompose(cfg.n, cfg.P).induced_partition(),
                    dtype=psw.F64 if cfg.dtype == "f64" else psw.F32)
    tdt = torch.float64 if cfg.dtype == "f64" else torch.float32
    F = torch.empty((cfg.n, cfg.nrhs), dtype=tdt, device="cuda")
    psw.fill_uniform(F, 3, -1, 1)
    X = torch.empty_like(F)
    plan.solve(F, X, path=psw.PATH_FUSED)
    torch.cuda.synchronize()
    buf = torch.zeros(1 << 22, dtype=torch.int64, device="cuda")
    L = psw.lib()
    L.psw_debug_trace.argtypes = [C.c_void_p]
    L.psw_debug_trace(buf.data_ptr())
    plan.solve(F, X, path=psw.PATH_FUSED)
    torch.cuda.synchronize()
    L.psw_debug_trace(None)
    tr = buf.cpu().numpy().reshape(-1, 16)
    used = tr[:, 6] > 0
    tr = tr[used]
    print(f"CTAs traced: {len(tr)}")
    for k, name in enumerate(PHASES):
        d = (tr[:, k + 1] - tr[:, k]).astype(np.float64)
        print(f"  {name:28s} median {np.median(d):8.0f}  p90 {np.percentile(d, 90):8.0f} cycles")
    tot = (tr[:, len(PHASES)] - tr[:, 0]).astype(np.float64)
    print(f"  {'CTA lifetime':28s} median {np.median(tot):8.0f}  p90 {np.percentile(tot, 90):8.0f} cycles")
    ks, ke, nt = tr[:, 10], tr[:, 11], tr[:, 12]
    if (ke > 0).all():
        per = (ke - ks) / np.maximum(nt, 1)
        print(f"whole kernel: span {(ke.max() - ks.min()) / 1e3:.1f} us, tiles/CTA {nt.min()}..{nt.max()}, "
              f"median per-tile time {np.median(per):.0f} ns, CTA start spread "
              f"{(ks.max() - ks.min()) / 1e3:.2f} us, end spread {(ke.max() - ke.min()) / 1e3:.2f} us")


if __name__ == "__main__":
    main()
