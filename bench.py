#!/usr/bin/env python
"""bench.py — batched dichotomy tridiagonal solve on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3]
                    [--mode rows|rhs] [--impl ours|reference]

Metric (BASELINE.json): RHS-unknowns solved per second (N * n / t) and the
achieved HBM GB/s against MEASURED_PEAKS.json, at 1/2/4/8 B200s.

Workload: BASELINE.json configs[3] (C3: fp64, n = 2^20 rows, N = 1024 RHS,
P = 64 partitions, dominant random A, F ~ U[-1, 1] seeded, RHS-contiguous
layout) — the config the metric's "at 1/2/4/8 B200" is quoted on. One step =
one batched solve of the whole workload with the plan and the inputs
resident in HBM (`value`). Inputs (8 GiB) are larger than L2 and a 2x-L2
buffer is overwritten before every step besides; only the solve is inside
the CUDA events.

Multi-GPU (`--gpus N`; launched under torchrun by the driver, or re-executed
under torchrun by this script): `--mode rows` (default) shards the rows of
ONE system over the ranks (the paper's decomposition, GPUs as PEs) with one
NCCL all-reduce of p x N fp64 per solve inside the C ABI (psw_shard_solve):
strong scaling; `--mode rhs` is the no-communication comparison that splits
the same batch's RHS over the ranks. At N = 1 the row mode is the plain
single-GPU solve (psw_solve, no collective). Timing: barrier + synchronize on
both sides, CUDA events on the launching stream, max over ranks.

`e2e`: the same metric through the public API on pinned host buffers
(psw_solve_host; per rank H2D of its rows + psw_shard_solve + D2H for
N > 1), copies inside the timed region. `cpu_baseline`: the reference
compiled from its headers (oracle/_ref) on the host cores, bounded samples
(serial, run_batch(threaded(all cores)) as shipped, and the
labelled RHS-parallel harness). `--impl reference` times that CPU path on a
bounded sample per step (the driver's reference arm).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PATHS = ["auto", "staged", "fused", "resweep", "cluster"]


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C3")
    ap.add_argument("--P", type=int, default=None, help="override the partition count")
    ap.add_argument("--layout", default=None, choices=[None, "R", "S"])
    ap.add_argument("--nrhs", type=int, default=None, help="override N (not a bench line)")
    ap.add_argument("--path", default="auto", choices=PATHS)
    ap.add_argument("--mode", default="rows", choices=["rows", "rhs"],
                    help="multi-GPU: rows = one system sharded by rows + one NCCL all-reduce "
                         "(strong scaling); rhs = the batch's RHS split over the ranks, no "
                         "communication (comparison)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="cpu_baseline sample budget")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-secondary", action="store_true",
                    help="skip the other configs' report-only lines in the default run")
    ap.add_argument("--e2e-steps", type=int, default=None)
    return ap.parse_args()


def _dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def _relaunch_under_torchrun(args):
    """`python bench.py --gpus N` without a torchrun env: run N ranks."""
    import socket
    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1", "--master-port",
           str(port), os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """Polls NVML during the timed region (SM clock, throttle reasons)."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, index: int, period_s: float = 0.001):
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
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback (B200_PROFILING.md)"


def _traffic(key: str):
    """ncu dram bytes (read + write) per solve from this round's committed
    capture of exactly this workload and path (profiles/ncu_traffic.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            ent = json.load(f).get(key)
        return ent
    except Exception:  # noqa: BLE001
        return None


def _config_dict(cfg, **extra):
    d = {"workload": cfg.name, "n": cfg.n, "nrhs": cfg.nrhs, "P": cfg.P, "layout": cfg.layout,
         "dtype": cfg.dtype, "matrix": cfg.matrix, "rhs": cfg.rhs,
         "l2": "inputs larger than L2 where the config is (C2, C3) and a 2x-L2 buffer "
               "overwritten before every timed solve (flushed)"}
    d.update(extra)
    return d


# ------------------------------------------------------------------ CPU side
def _cpu_sample_rhs(cfg, rate_guess: float, budget_s: float, cap: int) -> int:
    """RHS in a bounded CPU sample: ~budget_s of work, at most 2^26 unknowns
    (512 MB of fp64 host memory per buffer)."""
    cap = min(cap, max(1, (1 << 26) // cfg.n))
    return int(max(1, min(cap, budget_s * rate_guess / cfg.n)))


def _host_matrix(cfg):
    a, b = cfg.matrix_ab(0)
    return a, b


def _sample_rows(cfg, nr: int) -> np.ndarray:
    """`nr` systems drawn from the config's generator and distribution, in
    the reference's std::vector-per-system layout (nr x n, fp64; fp32
    configs rounded): a bounded sample of the same workload."""
    from paper_0901_2859_b200 import configs
    if cfg.rhs == "grid" and cfg.layout == "R":
        # C4's column sweep: system k is column k of the whole grid field
        F = configs.grid_rhs(cfg.n, cfg.n)[:, :nr].T
    else:
        full = configs.host_rhs(cfg.with_(nrhs=nr))
        F = full.T if cfg.layout == "R" else full
    F = np.ascontiguousarray(F, dtype=np.float64)
    assert F.shape == (nr, cfg.n), (F.shape, nr, cfg.n)
    return F


def cpu_reference(cfg, budget_s: float):
    """The reference on the host cores (oracle/_ref, its Release flags),
    BASELINE.md §3: compute_preliminary once, then (1) the serial per-RHS
    loop on 1 core, (2) run_batch(ExecMode::threaded(all cores)) as shipped
    (wall time includes its preliminary), (3) the labelled RHS-parallel
    harness on all cores (the headline cpu_baseline value). Bounded samples
    of the config's RHS; rates are per RHS-unknown."""
    from oracle.pyoracle import REF_PERF_SO, REF_SO, Reference
    so = REF_PERF_SO if os.path.exists(REF_PERF_SO) else REF_SO
    if not os.path.exists(so):
        raise RuntimeError("oracle/_ref not built (built by __graft_entry__.build())")
    ref = Reference(so)
    cores = os.cpu_count() or 1
    a, b = _host_matrix(cfg)
    bnd = ref.decompose(cfg.n, cfg.P)
    plan = ref.plan(a, b, a, bnd, workers=cores)
    Nmax = cfg.nrhs
    rows = lambda nr: _sample_rows(cfg, nr)  # noqa: E731
    # calibrate on a small slice, then size each variant to its share of the budget
    probe = rows(min(Nmax, max(1, cores)))
    _, t = plan.solve(probe, cores)
    rate_par = probe.shape[0] * cfg.n / max(t, 1e-9)
    n_par = _cpu_sample_rhs(cfg, rate_par, 0.5 * budget_s, Nmax)
    F_par = rows(n_par)
    reps, tot = 0, 0.0
    t_end = time.perf_counter() + 0.5 * budget_s
    while reps == 0 or (time.perf_counter() < t_end and reps < 1000):
        _, t = plan.solve(F_par, cores)
        tot += t
        reps += 1
    par = reps * n_par * cfg.n / tot
    n_ser = _cpu_sample_rhs(cfg, par / cores, 0.2 * budget_s, Nmax)
    _, t = plan.solve(rows(n_ser), 1)
    ser = n_ser * cfg.n / t
    n_rb = _cpu_sample_rhs(cfg, ser * 2, 0.2 * budget_s, Nmax)
    F_rb = rows(n_rb)
    t0 = time.perf_counter()
    _, stats = ref.run_batch(a, b, a, bnd, F_rb, threaded=True, workers=cores)
    rb_wall = time.perf_counter() - t0
    rb = n_rb * cfg.n / rb_wall
    return {
        "value": par, "unit": "unknowns/s", "cores": cores, "kind": "reference",
        "sample": (f"{reps} x {n_par} of {cfg.nrhs} RHS of {cfg.name} (n={cfg.n}, P={cfg.P}, the "
                   "config's generator and distribution): "
                   f"reference solve_with_preliminary_into on {cores} std::threads over disjoint "
                   f"RHS slices with one shared compute_preliminary (oracle/_ref, -O3); rate "
                   "extrapolated per RHS-unknown"),
        "nproc": cores, "hardware_concurrency": ref.hardware_concurrency(),
        "setup_s": plan.setup_s, "setup_workers": cores,
        "variants": {
            "serial_1core": {"value": ser, "rhs": n_ser,
                             "api": "compute_preliminary once + solve_with_preliminary_into loop"},
            "run_batch_threaded": {"value": rb, "rhs": n_rb, "workers": cores, "wall_s": rb_wall,
                                   "api": "run_batch(ExecMode::threaded(W)) as shipped; wall "
                                          "includes its preliminary (run.hpp:85-87)",
                                   "stats": stats},
            "harness_rhs_parallel": {"value": par, "rhs": n_par, "threads": cores},
        },
    }


def run_reference(args, cfg):
    """The driver's reference arm: the reference's own CPU implementation
    (oracle/_ref) on all host threads; each step solves a bounded sample of
    the workload's RHS (the preliminary is built once, timed separately, and
    excluded like the GPU plan)."""
    rank, world, _ = _dist_env()
    if rank != 0:
        return
    from oracle.pyoracle import REF_PERF_SO, REF_SO, Reference
    ref = Reference(REF_PERF_SO if os.path.exists(REF_PERF_SO) else REF_SO)
    cores = os.cpu_count() or 1
    a, b = _host_matrix(cfg)
    bnd = ref.decompose(cfg.n, cfg.P)
    plan = ref.plan(a, b, a, bnd, workers=cores)
    n0 = max(1, min(cfg.nrhs, cores))
    _, t = plan.solve(_sample_rows(cfg, n0), cores)
    rate = n0 * cfg.n / max(t, 1e-9)
    # ~0.25 s of CPU work per step so K + W steps finish within a few minutes
    ns = _cpu_sample_rhs(cfg, rate, 0.25, cfg.nrhs)
    Fs = _sample_rows(cfg, ns)
    for _ in range(args.warmup):
        plan.solve(Fs, cores)
    times = []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        times.append(plan.solve(Fs, cores)[1])
    wall = time.perf_counter() - t0
    total = sum(times)
    value = args.steps * ns * cfg.n / total
    sample = (f"{ns} of {cfg.nrhs} RHS of {cfg.name} per step (n={cfg.n}, P={cfg.P}, the config's "
              "generator and distribution); reference "
              f"solve_with_preliminary_into on {cores} std::threads over disjoint RHS slices, one "
              f"shared compute_preliminary ({plan.setup_s:.2f} s on a {cores}-thread WorkerPool, "
              "excluded like the GPU plan)")
    line = {
        "impl": "reference", "metric": "rhs_unknowns_per_s", "value": value,
        "unit": "unknowns/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": f"synthetic (seeded, BASELINE configs {cfg.name})",
        "config": _config_dict(cfg, parallelism=f"{cores} host threads"),
        "cpu_baseline": {"value": value, "unit": "unknowns/s", "cores": cores,
                         "kind": "reference", "sample": sample},
        "e2e": {"value": value, "unit": "unknowns/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "wall_s": wall, "setup_s": plan.setup_s,
    }
    print(json.dumps(line), flush=True)


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


KERNEL_NAMES = {"staged": ["fwd", "combine", "bwd"], "resweep": ["part", "comb", "solve"]}


def _alg_bytes(name, cfg, nrhs, rows, es):
    """Algorithmic HBM bytes per launch of each kernel."""
    coef = (2 * rows - 1) * es
    u = nrhs * rows
    return {"part": u * es + coef,          # read F
            "solve": u * 2 * es + coef,     # read F again, write X
            "comb": 0,                      # run aggregates only (a few per 256 rows)
            "fwd": u * 2 * es, "bwd": u * 2 * es, "combine": 0}.get(name, u * 2 * es + coef)


def main():
    args = _args()
    from paper_0901_2859_b200.configs import CONFIGS
    cfg = CONFIGS[args.config]
    default_cfg = cfg
    if args.P:
        cfg = cfg.with_(P=args.P)
    if args.layout:
        cfg = cfg.with_(layout=args.layout)
    if args.nrhs:
        cfg = cfg.with_(nrhs=args.nrhs)
    if args.impl == "reference":
        return run_reference(args, cfg)
    rank, world, local = _dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return _relaunch_under_torchrun(args)
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    overridden = cfg != default_cfg or args.path != "auto"
    run(args, cfg, overridden)


def run(args, cfg, overridden):
    import torch
    import paper_0901_2859_b200 as psw
    from paper_0901_2859_b200.sharded import ShardedSolver, rhs_slice

    rank, world, local = _dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import datetime
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev, timeout=datetime.timedelta(seconds=300))

    a, b = cfg.matrix_ab(0)
    A = psw.TridiagMatrix.symmetric(a, b)
    part = psw.decompose(cfg.n, cfg.P).induced_partition()
    dt = psw.F64 if cfg.dtype == "f64" else psw.F32
    tdt = torch.float64 if dt == psw.F64 else torch.float32
    es = 8 if dt == psw.F64 else 4
    layout = psw.LAYOUT_R if cfg.layout == "R" else psw.LAYOUT_S
    path = {"auto": psw.PATH_AUTO, "staged": psw.PATH_STAGED, "fused": psw.PATH_FUSED,
            "resweep": psw.PATH_RESWEEP,
            "cluster": psw.PATH_CLUSTER}[args.path]
    sharded = args.mode == "rows" and world > 1
    if sharded and layout != psw.LAYOUT_R:
        raise SystemExit("row sharding runs layout R")

    # ---- the rank's share of the workload, generated on the device
    if sharded:
        solver = ShardedSolver(A, part, dtype=dt, device=local)
        rows, k0, nr = solver.shard.rows, 0, cfg.nrhs
        row0 = solver.shard.row0
        plan = solver.plan
    else:
        solver = None
        plan = psw.Plan(A, part, dtype=dt, device=local)
        rows, row0 = cfg.n, 0
        k0, k1 = rhs_slice(cfg.nrhs, world, rank) if world > 1 else (0, cfg.nrhs)
        nr = k1 - k0
    shape = (rows, nr) if layout == psw.LAYOUT_R else (nr, rows)
    F = torch.empty(shape, dtype=tdt, device=dev)
    seed = 3  # configs.host_rhs stream over ONE global buffer; each rank takes its slice
    if cfg.rhs in ("uniform", "normal"):
        fill = (lambda t, off: psw.fill_uniform(t, seed, -1.0, 1.0, offset=off)) \
            if cfg.rhs == "uniform" else (lambda t, off: psw.fill_normal(t, seed, offset=off))
        if layout == psw.LAYOUT_S:
            fill(F, k0 * cfg.n)
        elif nr == cfg.nrhs:
            fill(F, row0 * cfg.nrhs)
        else:  # an RHS slice of a layout-R batch: the rank's columns of the global buffer
            tmp = torch.empty((rows, cfg.nrhs), dtype=tdt, device=dev)
            fill(tmp, row0 * cfg.nrhs)
            F.copy_(tmp[:, k0:k0 + nr])
            del tmp
    else:  # the C4 grid field (128 MB)
        from paper_0901_2859_b200.configs import host_rhs
        full = host_rhs(cfg)
        sl = full[row0:row0 + rows, k0:k0 + nr] if layout == psw.LAYOUT_R else full[k0:k0 + nr]
        F.copy_(torch.from_numpy(np.ascontiguousarray(sl)).to(tdt))
    X = torch.empty_like(F)
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush = torch.empty(2 * l2 // 4 + 1, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()

    def solve(events=None):
        if sharded:
            solver.solve(F, X, stream=stream)
        else:
            plan.solve(F, X, layout=layout, path=path, events=events)
        return psw.last_launch_count()

    solve()
    torch.cuda.synchronize()
    taken = "shard" if sharded else psw.last_path()
    names = KERNEL_NAMES.get(taken, [taken]) if not sharded else ["shard_solve"]
    nk = len(names)
    for _ in range(args.warmup):
        psw.l2_flush(flush)
        solve()
    torch.cuda.synchronize()

    # timed steps: one event pair around each whole solve (nothing between
    # the kernels, so their programmatic dependent launches overlap)
    evs = [[_Ev(), _Ev()] for _ in range(args.steps)]
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    launches = 0
    with ClockSampler(local) as clk:
        # keep the GPU busy while the host queues the first steps, so that no
        # step's events bracket host-side launch time
        torch.cuda._sleep(int(2e7))
        t0 = time.perf_counter()
        for i in range(args.steps):
            psw.l2_flush(flush)
            evs[i][0].rt.cudaEventRecord(evs[i][0].ev, stream.cuda_stream)
            launches += solve()
            evs[i][1].rt.cudaEventRecord(evs[i][1].ev, stream.cuda_stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    step_ms = [e[0].elapsed_time(e[1]) for e in evs]
    # the per-kernel split comes from extra untimed steps with events
    # recorded between the kernels by psw_solve_ex (which serialises them)
    kern_ms = [0.0] * nk
    if nk > 1 and not sharded:
        nsplit = min(args.steps, 5)
        sevs = [[_Ev() for _ in range(nk + 1)] for _ in range(nsplit)]
        for i in range(nsplit):
            psw.l2_flush(flush)
            solve(sevs[i])
        torch.cuda.synchronize()
        kern_ms = [sum(e[j].elapsed_time(e[j + 1]) for e in sevs) / nsplit for j in range(nk)]
    else:
        kern_ms = [sum(step_ms) / args.steps]
    total_ms = sum(step_ms)
    if dist:
        t = torch.tensor([total_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms = total_ms / args.steps
    value = cfg.nrhs * cfg.n / (ms / 1e3)  # whole job: every rank's units / max-over-ranks time

    peak, peak_kind = _peaks()
    bmin_rank = nr * rows * 2 * es + (2 * rows - 1) * es  # this rank's algorithmic bytes
    achieved = bmin_rank / (ms / 1e3) / 1e9
    tkey = f"{cfg.name}:{taken}"
    tr = _traffic(tkey) if (world == 1 and not overridden) else None
    kernels = {}
    for j, nm in enumerate(names):
        ab = _alg_bytes(nm, cfg, nr, rows, es) if nk > 1 else bmin_rank
        kernels[nm] = {"ms": kern_ms[j], "alg_bytes": ab,
                       "gbs": ab / (kern_ms[j] / 1e3) / 1e9 if kern_ms[j] > 0 else None}
    if sharded:
        par = (f"row-shard x{world}: rank r owns blocks [r P/{world}, (r+1) P/{world}); one NCCL "
               f"all-reduce of p x N = {cfg.P - 1} x {cfg.nrhs} fp64 per solve (psw_shard_solve)")
    elif world > 1:
        par = f"rhs-shard x{world}: the batch's RHS split over the ranks, no communication"
    else:
        par = "1 gpu"
    line = {
        "metric": "rhs_unknowns_per_s", "value": value, "unit": "unknowns/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": cfg.dtype,
        "data": "synthetic (seeded counter-based generator of the BASELINE config, on device)",
        "config": _config_dict(cfg, parallelism=par, path=taken),
        "roofline": {
            "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak,
            "traffic": tr["dram_bytes_per_solve"] if tr else None,
            "scope": "whole solve (every kernel of the step): algorithmic bytes B_min = "
                     "N n (s_F + s_X) + (2n - 1) s_A of this rank / its device time per step",
            "alg_bytes_per_launch": bmin_rank, "peak_kind": peak_kind,
            "traffic_source": tr.get("source") if tr else None,
        },
        "kernels": kernels,
        "gpu_launches": launches, "clocks": clk.summary(), "wall_s_timed": wall,
        "step_ms": {"min": min(step_ms), "median": statistics.median(step_ms),
                    "max": max(step_ms)},
    }
    if sharded:
        line["comm"] = {"backend": "nccl", "ranks": world, "collective": "ncclAllReduce(sum, fp64)",
                        "bytes_per_step": 8 * (cfg.P - 1) * cfg.nrhs}

    if not args.no_e2e:
        line["e2e"] = _e2e(psw, plan, solver, cfg, F, layout, dt, args, dist, dev)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_reference(cfg, args.cpu_seconds)
        except Exception as e:  # noqa: BLE001
            line["cpu_baseline"] = {"value": None, "error": str(e)}
    line["plan"] = {"setup_s": plan.info["setup_seconds"],
                    "device_bytes": plan.info["device_bytes"],
                    "combine_terms": plan.info["combine_terms"]}
    if rank == 0 and world == 1 and not overridden and not args.no_secondary and not args.no_e2e:
        # the other BASELINE configs, measured the same way (report-only keys)
        del F, X
        torch.cuda.empty_cache()
        line["secondary"] = _secondary(psw, torch, dev, flush, stream, cfg.name)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if solver is not None:
        solver.close()
    if dist:
        dist.destroy_process_group()


def _secondary(psw, torch, dev, flush, stream, skip):
    """Every other BASELINE config through AUTO: plan, seeded device input,
    3 warm-up solves, 10 timed solves each bracketed by CUDA events after an L2
    flush (as the main line). Report-only: the headline is the main line."""
    from paper_0901_2859_b200.configs import CONFIGS
    out = {}
    peak, _ = _peaks()
    for name in ("C0", "C1", "C2", "C4", "C4c"):
        if name == skip:
            continue
        cfg = CONFIGS[name]
        try:
            a, b = cfg.matrix_ab(0)
            plan = psw.Plan(psw.TridiagMatrix.symmetric(a, b),
                            psw.decompose(cfg.n, cfg.P).induced_partition(),
                            dtype=psw.F64 if cfg.dtype == "f64" else psw.F32, device=dev.index or 0)
            tdt = torch.float64 if cfg.dtype == "f64" else torch.float32
            lay = psw.LAYOUT_R if cfg.layout == "R" else psw.LAYOUT_S
            shape = (cfg.n, cfg.nrhs) if lay == psw.LAYOUT_R else (cfg.nrhs, cfg.n)
            F = torch.empty(shape, dtype=tdt, device=dev)
            if cfg.rhs == "uniform":
                psw.fill_uniform(F, 3, -1.0, 1.0)
            elif cfg.rhs == "normal":
                psw.fill_normal(F, 3)
            else:
                from paper_0901_2859_b200.configs import host_rhs
                F.copy_(torch.from_numpy(np.ascontiguousarray(host_rhs(cfg))).to(tdt))
            X = torch.empty_like(F)
            for _ in range(3):
                psw.l2_flush(flush)
                plan.solve(F, X, layout=lay)
            torch.cuda.synchronize()
            evs = [(_Ev(), _Ev()) for _ in range(10)]
            torch.cuda._sleep(int(2e6))
            for e0, e1 in evs:
                psw.l2_flush(flush)
                e0.rt.cudaEventRecord(e0.ev, stream.cuda_stream)
                plan.solve(F, X, layout=lay)
                e1.rt.cudaEventRecord(e1.ev, stream.cuda_stream)
            torch.cuda.synchronize()
            ms = sum(e0.elapsed_time(e1) for e0, e1 in evs) / len(evs)
            es = 8 if cfg.dtype == "f64" else 4
            bmin = cfg.nrhs * cfg.n * 2 * es + (2 * cfg.n - 1) * es
            out[name] = {"path": psw.last_path(),
                         "ms_per_step": ms, "value": cfg.nrhs * cfg.n / (ms / 1e3),
                         "unit": "unknowns/s", "frac": bmin / (ms / 1e3) / 1e9 / peak,
                         "steps": len(evs), "n": cfg.n, "nrhs": cfg.nrhs, "P": cfg.P,
                         "layout": cfg.layout, "dtype": cfg.dtype}
            del F, X, plan
            torch.cuda.empty_cache()
        except Exception as e:  # noqa: BLE001
            out[name] = {"error": str(e)}
    return out


def _e2e(psw, plan, solver, cfg, F, layout, dt, args, dist, dev):
    """The same metric through the public API on pinned host buffers: H2D of
    the step's F, the solve, D2H of X inside the timed region."""
    import torch
    Fh = torch.empty(F.shape, dtype=F.dtype, pin_memory=True)
    Fh.copy_(F)
    Xh = torch.empty(F.shape, dtype=F.dtype, pin_memory=True)
    nbytes = Fh.numel() * Fh.element_size()
    steps = args.e2e_steps or max(1, min(args.steps, 3 if nbytes > (1 << 30) else 10))
    if solver is not None:
        call = lambda: solver.solve_host(Fh, Xh)  # noqa: E731
        api = "ShardedSolver.solve_host (pinned rows -> psw_shard_solve -> pinned rows)"
    else:
        Fn, Xn = Fh.numpy(), Xh.numpy()
        call = lambda: plan.solve_host(Fn, Xn, layout=layout)  # noqa: E731
        api = "psw_solve_host (pinned host buffers)"
    for _ in range(2):  # warm (first touch of the pinned pages, staging buffers)
        call()
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        call()
    el = time.perf_counter() - t0
    if dist:
        t = torch.tensor([el], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        el = float(t.item())
    out = {"value": cfg.nrhs * cfg.n * steps / el, "unit": "unknowns/s",
           "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes, "steps": steps,
           "ms_per_step": 1e3 * el / steps, "api": api}
    if solver is None:
        out["link"] = _link_floor(Fh, Xh, 1e3 * el / steps)
    return out


def _link_floor(Fh, Xh, e2e_ms):
    """The host link's own bound for the step's traffic: the same bytes as
    one contiguous H2D and one contiguous D2H, on two streams at once (the
    most a pipelined solve can overlap); e2e is at `frac` of it."""
    import torch
    dev_a = torch.empty(Fh.shape, dtype=Fh.dtype, device="cuda")
    dev_b = torch.empty_like(dev_a)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def both():
        with torch.cuda.stream(s1):
            dev_a.copy_(Fh, non_blocking=True)
        with torch.cuda.stream(s2):
            Xh.copy_(dev_b, non_blocking=True)

    best = None
    for _ in range(2):
        torch.cuda.synchronize()
        t = time.perf_counter()
        both()
        torch.cuda.synchronize()
        el = (time.perf_counter() - t) * 1e3
        best = el if best is None else min(best, el)
    del dev_a, dev_b
    torch.cuda.empty_cache()
    nb = Fh.numel() * Fh.element_size()
    return {"both_directions_ms": best, "aggregate_gbs": 2 * nb / best / 1e6,
            "frac": best / e2e_ms,
            "note": "F's bytes H2D and X's bytes D2H as two concurrent contiguous copies "
                    "(pinned); the solve itself adds the first chunk's upload and the last "
                    "chunk's download, which cannot overlap anything"}


if __name__ == "__main__":
    main()
