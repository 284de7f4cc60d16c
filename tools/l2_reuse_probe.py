"""Does a chunk's K3 find the F its K1 just read in L2? C2 system (fp32,
n = 65536), chunks of Nc right-hand sides solved one after the other on one
stream; run under `ncu --cache-control none --metrics dram__bytes_read.sum,...`
and compare rs_solve's DRAM reads with the chunk's bytes (n Nc 4)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0901_2859_b200 as psw  # noqa: E402
from paper_0901_2859_b200.configs import CONFIGS  # noqa: E402

cfg = CONFIGS["C2"]
n = cfg.n
N = 2048
a, b = cfg.matrix_ab(0)
plan = psw.Plan(psw.TridiagMatrix.symmetric(a, b), psw.decompose(n, cfg.P).induced_partition(), psw.F32)
F = torch.empty((n, N), dtype=torch.float32, device="cuda")
psw.fill_uniform(F, 3, -1.0, 1.0)
X = torch.empty_like(F)
for Nc in [int(v) for v in (sys.argv[1:] or ["64", "128", "256"])]:
    for c in range(0, 4):
        plan.solve(F[:, c * Nc:(c + 1) * Nc], X[:, c * Nc:(c + 1) * Nc], nrhs=Nc, ldf=N, ldx=N)
    torch.cuda.synchronize()
    print("Nc", Nc, "chunk MB", n * Nc * 4 / 1e6, psw.last_path())
