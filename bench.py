#!/usr/bin/env python
"""bench.py — batched dichotomy tridiagonal solve on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C1] [--impl ours|reference]

One "step" = one batched solve of the whole workload (every RHS of the
config) with the plan and the inputs resident in HBM (`value`), and the same
solve end to end through the C ABI on pinned host buffers (`e2e`,
psw_solve_host: H2D of F + solve + D2H of X inside the timed region).
Metric (BASELINE.json): RHS-unknowns solved per second (N * n / t), plus the
achieved HBM GB/s of the dominant kernel against MEASURED_PEAKS.json.

Workload: BASELINE.json configs[1] (C1: fp64, n=4096, N=4096, P=16,
a=-1, b=2.01, F ~ N(0,1) seeded, RHS-contiguous layout). Multi-GPU
(torchrun): every rank solves its own full batch of RHS (RHS-sharded, no
data-path collective) -> "scaling": "weak"; rank 0 prints the max-over-ranks
timing. `--impl reference` times the reference's own CPU implementation
(oracle/_ref = the reference headers compiled) on the host cores.

L2 hygiene: a 2x-L2 buffer is overwritten before every timed solve; only the
solve itself is inside the CUDA events.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C1")
    ap.add_argument("--P", type=int, default=None, help="override the partition count")
    ap.add_argument("--layout", default=None, choices=[None, "R", "S"])
    ap.add_argument("--path", default="auto", choices=["auto", "staged", "fused", "pipe", "tile", "chunked", "resweep", "cluster"])
    ap.add_argument("--cpu-seconds", type=float, default=10.0, help="cpu_baseline sample budget")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--mode", default="rhs", choices=["rhs", "rows"],
                    help="multi-GPU: rhs = every rank its own RHS batch (weak scaling); rows = "
                         "one system sharded by rows over the ranks + one NCCL all-reduce "
                         "(strong scaling, BASELINE C3)")
    return ap.parse_args()


def _dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """Polls NVML during the timed region (SM clock, throttle reasons)."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, index: int, period_s: float = 0.002):
        self.samples, self.reasons = [], 0
        self.period = period_s
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # noqa: BLE001
            self.err = str(e)

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.reasons |= nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": self.err}
        names = [v for k, v in self.REASONS.items() if self.reasons & k and v != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": names, "samples": len(self.samples)}


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback"


def _traffic(workload: str, kernel: str):
    """ncu dram bytes per launch from the committed profile summary."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(f"{workload}:{kernel}")
    except Exception:  # noqa: BLE001
        return None


# ------------------------------------------------------------------ CPU side
def _host_inputs(cfg, seed=0):
    from paper_0901_2859_b200 import configs
    a, b = cfg.matrix_ab(seed)
    F = configs.host_rhs(cfg, seed)
    # the reference works on one std::vector per system (layout S)
    FS = np.ascontiguousarray(F.T if cfg.layout == "R" else F, dtype=np.float64)
    return a, b, FS


def cpu_reference_rate(cfg, budget_s: float, threads: int, max_reps: int = 1000):
    """Reference per-RHS solve (oracle/_ref, the reference compiled) on all
    host threads over disjoint RHS slices; repeats the whole batch until the
    budget is spent. Returns (unknowns/s, sample description, setup s)."""
    from oracle.pyoracle import Reference, REF_SO, REF_PERF_SO
    if not os.path.exists(REF_SO):
        raise RuntimeError("oracle/_ref/libpsw_ref.so missing (built by __graft_entry__.build())")
    ref = Reference(REF_PERF_SO if os.path.exists(REF_PERF_SO) else REF_SO)
    a, b, FS = _host_inputs(cfg)
    bnd = ref.decompose(cfg.n, cfg.P)
    N = FS.shape[0]
    reps, solve_t, setup_t = 0, 0.0, 0.0
    t_end = time.perf_counter() + budget_s
    while reps < max_reps and (reps == 0 or time.perf_counter() < t_end):
        _, su, so = ref.solve_rhs_parallel(a, b, a, bnd, FS, threads)
        solve_t += so
        setup_t = su
        reps += 1
    rate = reps * N * cfg.n / solve_t
    sample = (f"{reps} x full {cfg.name} batch ({N} RHS x n={cfg.n}, P={cfg.P}), reference "
              f"compute_preliminary once + solve_with_preliminary_into per RHS on {threads} "
              f"std::threads over disjoint RHS slices (oracle/_ref)")
    return rate, sample, setup_t


def run_reference(args, cfg):
    rank, world, _ = _dist_env()
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    from oracle.pyoracle import Reference, REF_SO, REF_PERF_SO
    ref = Reference(REF_PERF_SO if os.path.exists(REF_PERF_SO) else REF_SO)
    a, b, FS = _host_inputs(cfg)
    bnd = ref.decompose(cfg.n, cfg.P)
    N = FS.shape[0]
    for _ in range(args.warmup):
        ref.solve_rhs_parallel(a, b, a, bnd, FS, threads)
    times = []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        _, _, so = ref.solve_rhs_parallel(a, b, a, bnd, FS, threads)
        times.append(so)
    wall = time.perf_counter() - t0
    total = sum(times)
    value = args.steps * N * cfg.n / total
    line = {
        "impl": "reference", "metric": "rhs_unknowns_per_s", "value": value,
        "unit": "unknowns/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, BASELINE configs[1])",
        "config": _config_dict(cfg),
        "cpu_baseline": {"value": value, "unit": "unknowns/s", "cores": threads,
                         "kind": "reference",
                         "sample": f"full {cfg.name} batch per step ({N} RHS x n={cfg.n}); "
                                   f"reference solve_with_preliminary_into on {threads} "
                                   "std::threads over disjoint RHS slices, shared preliminary "
                                   "(timed separately, excluded like the GPU plan)"},
        "e2e": {"value": value, "unit": "unknowns/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "wall_s": wall,
    }
    print(json.dumps(line), flush=True)


def _config_dict(cfg):
    return {"workload": cfg.name, "n": cfg.n, "nrhs": cfg.nrhs, "P": cfg.P,
            "layout": cfg.layout, "matrix": cfg.matrix, "rhs": cfg.rhs,
            "l2": "2x-L2 buffer overwritten before every timed solve (flushed)"}


# ------------------------------------------------------------------ GPU side
class _Ev:
    """Raw cudaEvent_t (cuda-python): psw_solve_ex records it between its
    own kernels on the launching stream."""

    def __init__(self):
        try:
            from cuda.bindings import runtime as cudart
        except ImportError:  # older cuda-python
            from cuda import cudart
        self.rt = cudart
        err, self.ev = cudart.cudaEventCreate()
        assert int(err) == 0, err

    def __int__(self):
        return int(self.ev)

    def elapsed_time(self, other: "_Ev") -> float:
        err, ms = self.rt.cudaEventElapsedTime(self.ev, other.ev)
        assert int(err) == 0, err
        return ms

    def __del__(self):
        try:
            self.rt.cudaEventDestroy(self.ev)
        except Exception:  # noqa: BLE001
            pass


def main():
    args = _args()
    from paper_0901_2859_b200.configs import CONFIGS
    cfg = CONFIGS[args.config]
    if args.P:
        cfg = cfg.with_(P=args.P)
    if args.layout:
        cfg = cfg.with_(layout=args.layout)
    if args.impl == "reference":
        return run_reference(args, cfg)
    if args.mode == "rows":
        return run_rows(args, cfg)

    import torch
    import paper_0901_2859_b200 as psw

    rank, world, local = _dist_env()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()

    a, b = cfg.matrix_ab(0)
    A = psw.TridiagMatrix.symmetric(a, b)
    part = psw.decompose(cfg.n, cfg.P).induced_partition()
    dt = psw.F64 if cfg.dtype == "f64" else psw.F32
    tdt = torch.float64 if dt == psw.F64 else torch.float32
    es = 8 if dt == psw.F64 else 4
    plan = psw.Plan(A, part, dtype=dt, device=local)
    layout = psw.LAYOUT_R if cfg.layout == "R" else psw.LAYOUT_S
    shape = (cfg.n, cfg.nrhs) if layout == psw.LAYOUT_R else (cfg.nrhs, cfg.n)
    F = torch.empty(shape, dtype=tdt, device=dev)
    seed = 3 + 1000 * rank  # each rank its own RHS shard
    if cfg.rhs == "normal":
        psw.fill_normal(F, seed)
    elif cfg.rhs == "uniform":
        psw.fill_uniform(F, seed, -1.0, 1.0)
    else:
        from paper_0901_2859_b200.configs import grid_rhs
        F.copy_(torch.from_numpy(grid_rhs(cfg.n, cfg.nrhs, rank)).to(tdt))
    X = torch.empty_like(F)
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush = torch.empty(2 * l2 // 4 + 1, dtype=torch.float32, device=dev)
    path = {"auto": psw.PATH_AUTO, "staged": psw.PATH_STAGED, "fused": psw.PATH_FUSED,
            "pipe": psw.PATH_PIPE, "tile": psw.PATH_TILE, "chunked": psw.PATH_CHUNKED,
            "resweep": psw.PATH_RESWEEP, "cluster": psw.PATH_CLUSTER}[args.path]

    # discover the kernel count of the chosen path
    plan.solve(F, X, layout=layout, path=path)
    torch.cuda.synchronize()
    launches_per_solve = psw.last_launch_count()
    taken = psw.last_path()
    # event marks per path: STAGED brackets its three kernels, the others the whole solve
    names = {"staged": ["fwd", "combine", "bwd"],
             "resweep": ["part", "comb", "solve"]}.get(taken, [taken])
    nk = len(names)

    def step(events=None):
        psw.l2_flush(flush)
        plan.solve(F, X, layout=layout, path=path, events=events)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    evs = [[_Ev() for _ in range(nk + 1)] for _ in range(args.steps)]
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        t0 = time.perf_counter()
        launches = 0
        for i in range(args.steps):
            step(evs[i])
            launches += psw.last_launch_count()  # == launches_per_solve
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
    if dist:
        dist.barrier()
    step_ms = [e[0].elapsed_time(e[-1]) for e in evs]
    kern_ms = [sum(e[j].elapsed_time(e[j + 1]) for e in evs) / args.steps for j in range(nk)]
    total_ms = sum(step_ms)
    if dist:
        t = torch.tensor([total_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    units = cfg.nrhs * cfg.n
    value = world * units * args.steps / (total_ms / 1e3)

    # roofline of the dominant kernel: algorithmic bytes per launch / time
    peak, peak_kind = _peaks()
    j = int(np.argmax(kern_ms))
    kname = names[j] if j < len(names) else f"k{j}"
    coef = (2 * cfg.n - 1) * es
    alg = {"fused": units * 2 * es + coef,      # read F, write X
           "pipe": units * 2 * es + coef,       # read F, write X (d round trip in L2)
           "tile": units * 2 * es + coef,       # read F, write X (second read from L2)
           "chunked": units * 2 * es + coef,    # read F, write X (d~ round trip in L2)
           "cluster": units * 2 * es + coef,    # read F, write X
           "fwd": units * 2 * es + coef,        # read F, write d0
           "bwd": units * 2 * es + coef,        # read d0, write X
           "part": units * es + coef,           # read F (segment checkpoints: small)
           "solve": units * 2 * es + coef,      # read F again, write X
           "comb": 2 * cfg.P * cfg.nrhs * 8 + max(cfg.P - 1, 1) * cfg.nrhs * 8,
           "combine": 2 * cfg.P * cfg.nrhs * 8 + max(cfg.P - 1, 1) * cfg.nrhs * 8}[kname]
    achieved = alg / (kern_ms[j] / 1e3) / 1e9
    solve_gbs = cfg.bytes_min() / (total_ms / args.steps / 1e3) / 1e9

    line = {
        "metric": "rhs_unknowns_per_s", "value": value, "unit": "unknowns/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": cfg.dtype, "data": "synthetic (seeded counter-based generator, BASELINE configs)",
        "config": dict(_config_dict(cfg), parallelism=f"rhs-shard x{world}" if world > 1 else "1 gpu",
                       path=taken, kernels=names),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": _traffic(cfg.name, kname),
                     "kernel": kname, "kernel_ms": kern_ms[j], "peak_kind": peak_kind,
                     "alg_bytes_per_launch": alg},
        "hbm_gbs_solve": solve_gbs, "hbm_frac_solve": solve_gbs / peak,
        "kernel_ms": dict(zip(names, kern_ms)),
        "gpu_launches": launches, "clocks": clk.summary(), "wall_s_timed": wall,
    }

    if not args.no_e2e:
        line["e2e"] = _e2e(psw, plan, cfg, F, layout, dt, args, dist, dev, world)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            rate, sample, setup = cpu_reference_rate(cfg, args.cpu_seconds, os.cpu_count() or 1)
            line["cpu_baseline"] = {"value": rate, "unit": "unknowns/s", "cores": os.cpu_count(),
                                    "kind": "reference", "sample": sample,
                                    "setup_s": setup}
        except Exception as e:  # noqa: BLE001
            line["cpu_baseline"] = {"value": None, "error": str(e)}
    line["plan"] = {"setup_s": plan.info["setup_seconds"], "device_bytes": plan.info["device_bytes"],
                    "combine_terms": plan.info["combine_terms"]}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def run_rows(args, cfg):
    """Row-sharded strong scaling: rank r owns the rows of
    blocks [r P/G, (r+1) P/G) of every RHS; one NCCL all-reduce of p values per
    RHS per solve. Timed region = forward + all-reduce + backward, max over ranks."""
    import torch
    import paper_0901_2859_b200 as psw
    from paper_0901_2859_b200.configs import uniform
    from paper_0901_2859_b200.sharded import ShardedSolver
    rank, world, local = _dist_env()
    torch.cuda.set_device(local)
    import datetime
    import torch.distributed as dist
    if world > 1 or "MASTER_ADDR" in os.environ:  # launched by torchrun (its env:// store)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local),
                                timeout=datetime.timedelta(seconds=120))
    else:  # plain single process: a private one-rank group for the same code path
        dist.init_process_group("gloo", init_method="tcp://127.0.0.1:%d" % _port(), rank=0,
                                world_size=1, timeout=datetime.timedelta(seconds=120))
    dev = torch.device("cuda", local)
    a, b = cfg.matrix_ab(0)
    A = psw.TridiagMatrix.symmetric(a, b)
    part = psw.decompose(cfg.n, cfg.P).induced_partition()
    dt = psw.F64 if cfg.dtype == "f64" else psw.F32
    tdt = torch.float64 if dt == psw.F64 else torch.float32
    solver = ShardedSolver(A, part, dtype=dt, device=local)
    sh = solver.shard
    F = torch.empty((sh.rows, cfg.nrhs), dtype=tdt, device=dev)
    psw.fill_uniform(F, 3 + rank, -1.0, 1.0)
    X = torch.empty_like(F)
    flush = torch.empty(2 * torch.cuda.get_device_properties(dev).L2_cache_size // 4 + 1,
                        dtype=torch.float32, device=dev)
    for _ in range(args.warmup):
        solver.solve(F, X)
    torch.cuda.synchronize()
    dist.barrier()
    ms = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            psw.l2_flush(flush)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            solver.solve(F, X)
            e1.record()
            ms.append((e0, e1))
        torch.cuda.synchronize()
    total = sum(a_.elapsed_time(b_) for a_, b_ in ms)
    on_gpu = dist.get_backend() == "nccl"
    t = torch.tensor([total], dtype=torch.float64, device=dev if on_gpu else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total = float(t.item())
    units = cfg.nrhs * cfg.n
    value = units * args.steps / (total / 1e3)
    peak, peak_kind = _peaks()
    es = 8 if dt == psw.F64 else 4
    per_gpu = (sh.rows * cfg.nrhs * 2 * es) / (total / args.steps / 1e3) / 1e9
    line = {
        "metric": "rhs_unknowns_per_s", "value": value, "unit": "unknowns/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": cfg.dtype,
        "data": "synthetic (seeded counter-based generator, BASELINE configs)",
        "config": dict(_config_dict(cfg), parallelism=f"row-shard x{world} (NCCL all-reduce of "
                       f"{cfg.P - 1} values/RHS)", path="staged shard kernels"),
        "roofline": {"bound": "hbm", "achieved": per_gpu, "peak": peak, "unit": "GB/s",
                     "frac": per_gpu / peak, "traffic": None, "kernel": "shard solve (rank 0)",
                     "peak_kind": peak_kind},
        "comm_bytes_per_step": solver.comm_bytes_per_rhs * cfg.nrhs,
        "gpu_launches": 3 * args.steps, "clocks": clk.summary(),
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def _port():
    import socket
    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        return s_.getsockname()[1]


def _e2e(psw, plan, cfg, F, layout, dt, args, dist, dev, world):
    """Same metric through psw_solve_host on pinned host buffers."""
    import torch
    Fh = torch.empty(F.shape, dtype=F.dtype, pin_memory=True)
    Fh.copy_(F)
    Xh = torch.empty(F.shape, dtype=F.dtype, pin_memory=True)
    Fn, Xn = Fh.numpy(), Xh.numpy()
    for _ in range(2):  # warm (first-touch of the pinned pages, staging buffers)
        plan.solve_host(Fn, Xn, layout=layout)
    steps = max(1, min(args.steps, 10))
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        plan.solve_host(Fn, Xn, layout=layout)
    el = time.perf_counter() - t0
    if dist:
        t = torch.tensor([el], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        el = float(t.item())
    nbytes = Fh.numel() * Fh.element_size()
    return {"value": world * cfg.nrhs * cfg.n * steps / el, "unit": "unknowns/s",
            "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes, "steps": steps,
            "ms_per_step": 1e3 * el / steps, "api": "psw_solve_host (pinned host buffers)"}


if __name__ == "__main__":
    main()
