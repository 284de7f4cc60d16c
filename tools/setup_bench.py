"""Plan-creation time per BASELINE config: host sweeps (PSW_DEVICE_SETUP=0)
against the device preliminary (psw_prelim.cu), with the library's own
breakdown (PSW_SETUP_VERBOSE). Prints one JSON line."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0901_2859_b200 as psw  # noqa: E402
from paper_0901_2859_b200.configs import CONFIGS  # noqa: E402

os.environ["PSW_SETUP_VERBOSE"] = "1"
out = {}
for name in (sys.argv[1:] or ["C0", "C1", "C4", "C2", "C3"]):
    cfg = CONFIGS[name]
    a, b = cfg.matrix_ab(0)
    A = psw.TridiagMatrix.symmetric(a, b)
    part = psw.decompose(cfg.n, cfg.P).induced_partition()
    dt = psw.F32 if cfg.dtype == "f32" else psw.F64
    res = {}
    for mode in ("0", "1", "1", "0"):
        os.environ["PSW_DEVICE_SETUP"] = mode
        t0 = time.perf_counter()
        plan = psw.Plan(A, part, dtype=dt)
        t1 = time.perf_counter()
        res.setdefault("device" if mode == "1" else "host", []).append(round((t1 - t0) * 1e3, 3))
        res.setdefault("device_setup", []).append(int(plan.info["device_setup"]))
        del plan
    out[name] = {"n": cfg.n, "P": cfg.P, "plan_create_ms": res}
print(json.dumps(out))
