"""Row-sharded CUDA path (psw_shard_*) on one GPU.

* Emulated ranks: every rank's shard plan and kernels run in this process
  and the all-reduce is the in-process sum of the ranks' partial boundary
  values (no rank waits on another, so no collective is needed).
* psw_shard_solve with a real NCCL communicator of one rank: the C-ABI path
  the multi-GPU bench runs (forward, ncclAllReduce, backward on one stream).
"""
import numpy as np
import pytest

from conftest import load_golden, rel_l2

pytestmark = pytest.mark.gpu


def _emulate(psw, torch, A, part, F, world, dtype=0):
    from paper_0901_2859_b200.sharded import shard_layout
    tdt = torch.float64 if dtype == psw.F64 else torch.float32
    N = F.shape[1]
    shards = shard_layout(A.n(), part, world)
    plans = [psw.Plan(A, part, dtype=dtype, rank=r, world=world) for r in range(world)]
    p = part.p()
    Fl, Xl, Wl = [], [], []
    total = torch.zeros((max(p, 1), N), dtype=torch.float64, device="cuda")
    for sh, pl in zip(shards, plans):
        assert pl.row_offset() == sh.row0 and pl.rows() == sh.rows
        assert pl.partials_count() == p
        f = torch.from_numpy(np.ascontiguousarray(F[sh.row0:sh.row1])).to(tdt).cuda()
        x = torch.empty_like(f)
        ws = torch.empty(pl.workspace_bytes(N), dtype=torch.uint8, device="cuda")
        part_v = torch.zeros_like(total)
        pl.shard_forward(f, N, ws, part_v)
        total += part_v
        Fl.append(f)
        Xl.append(x)
        Wl.append(ws)
    for pl, f, x, ws in zip(plans, Fl, Xl, Wl):
        pl.shard_backward(f, x, N, ws, total)
    torch.cuda.synchronize()
    return np.concatenate([x.double().cpu().numpy() for x in Xl], axis=0)


@pytest.mark.parametrize("name,world", [("c1_n4096_P16", 1), ("c1_n4096_P16", 2),
                                        ("c1_n4096_P16", 4), ("c1_n4096_P16", 8),
                                        ("c0_n1024_P4", 4), ("decomp_n333_P9", 3),
                                        ("c4_n4096_P16", 16), ("rand_n200_p7", 2),
                                        ("mixed_n96_P8", 8)])
def test_row_sharded_matches_reference(psw, cuda, name, world):
    g = load_golden(name)
    A = psw.TridiagMatrix(g["sub"], g["diag"], g["super"])
    part = psw.Partition(A.n(), g["bnd"].tolist())
    X = _emulate(psw, cuda, A, part, np.ascontiguousarray(g["F"].T), world)
    assert rel_l2(X.T, g["X"]) <= 1e-12


@pytest.mark.parametrize("name,world", [("c2_n8192_P64", 4), ("c2_n8192_P512", 8)])
def test_row_sharded_fp32(psw, cuda, name, world):
    g = load_golden(name)
    A = psw.TridiagMatrix(g["sub"], g["diag"], g["super"])
    part = psw.Partition(A.n(), g["bnd"].tolist())
    F32 = np.ascontiguousarray(g["F"].T)
    X = _emulate(psw, cuda, A, part, F32, world, dtype=psw.F32)
    assert rel_l2(X.T, g["X"]) <= 1e-5


@pytest.mark.parametrize("world", [1, 2, 8])
def test_row_sharded_c3_shape(psw, cuda, world):
    """C3 shape (n = 2^20, P = 64) over emulated ranks, 64 RHS against the oracle."""
    from oracle.pyoracle import Oracle
    from paper_0901_2859_b200.configs import CONFIGS, uniform
    cfg = CONFIGS["C3"]
    a, b = cfg.matrix_ab(0)
    A = psw.TridiagMatrix.symmetric(a, b)
    part = psw.decompose(cfg.n, cfg.P).induced_partition()
    N = 64
    F = uniform(3, cfg.n * N, -1, 1).reshape(cfg.n, N)
    X = _emulate(psw, cuda, A, part, F, world)
    want = Oracle().solve_batch_threads(a, b, a, np.array(part.boundaries),
                                        np.ascontiguousarray(F.T), 8)[0]
    assert rel_l2(X.T, want) <= 1e-12


@pytest.mark.parametrize("name", ["c1_n4096_P16", "c0_n1024_P4", "decomp_n333_P9"])
def test_shard_solve_nccl_one_rank(psw, cuda, name):
    """psw_shard_solve through a 1-rank NCCL communicator (the C-ABI exchange)."""
    g = load_golden(name)
    A = psw.TridiagMatrix(g["sub"], g["diag"], g["super"])
    part = psw.Partition(A.n(), g["bnd"].tolist())
    plan = psw.Plan(A, part, rank=0, world=1)
    comm = psw.Comm(1, 0, psw.Comm.unique_id(), 0)
    F = cuda.from_numpy(np.ascontiguousarray(g["F"].T)).cuda()
    X = cuda.empty_like(F)
    plan.shard_solve(F, X, comm)
    X2 = plan.shard_solve(F.clone(), cuda.empty_like(F), None)  # no communicator
    cuda.cuda.synchronize()
    assert rel_l2(X.cpu().numpy().T, g["X"]) <= 1e-12
    assert np.array_equal(X.cpu().numpy(), X2.cpu().numpy())
    comm.close()


def test_shard_solve_graph_capture(psw, cuda):
    """The whole sharded solve (kernels + NCCL) captures into one CUDA graph."""
    g = load_golden("c1_n4096_P16")
    A = psw.TridiagMatrix(g["sub"], g["diag"], g["super"])
    part = psw.Partition(A.n(), g["bnd"].tolist())
    plan = psw.Plan(A, part, rank=0, world=1)
    comm = psw.Comm(1, 0, psw.Comm.unique_id(), 0)
    F = cuda.from_numpy(np.ascontiguousarray(g["F"].T)).cuda()
    X = cuda.zeros_like(F)
    s = cuda.cuda.Stream()
    plan.shard_solve(F, X, comm, stream=s)  # warm (NCCL lazy init) outside the capture
    s.synchronize()
    X.zero_()
    graph = cuda.cuda.CUDAGraph()
    with cuda.cuda.graph(graph, stream=s):
        plan.shard_solve(F, X, comm, stream=s)
    graph.replay()
    cuda.cuda.synchronize()
    assert rel_l2(X.cpu().numpy().T, g["X"]) <= 1e-12
    comm.close()


def test_shard_one_rank_equals_resweep(psw, cuda):
    """A 1-rank shard solve and the single-GPU RESWEEP path agree to rounding."""
    from paper_0901_2859_b200.configs import CONFIGS
    cfg = CONFIGS["C3"].with_(nrhs=96)
    a, b = cfg.matrix_ab(0)
    A = psw.TridiagMatrix.symmetric(a, b)
    part = psw.decompose(cfg.n, cfg.P).induced_partition()
    F = cuda.empty((cfg.n, cfg.nrhs), dtype=cuda.float64, device="cuda")
    psw.fill_uniform(F, 3, -1.0, 1.0)
    X1 = cuda.empty_like(F)
    psw.Plan(A, part).solve(F, X1, path=psw.PATH_RESWEEP)
    X2 = cuda.empty_like(F)
    psw.Plan(A, part, rank=0, world=1).shard_solve(F, X2, None)
    cuda.cuda.synchronize()
    d = (X1 - X2).norm() / X1.norm()
    assert float(d) <= 1e-13


def test_shard_rejects_bad_world(psw, cuda):
    g = load_golden("c1_n4096_P16")
    A = psw.TridiagMatrix(g["sub"], g["diag"], g["super"])
    part = psw.Partition(A.n(), g["bnd"].tolist())
    with pytest.raises(ValueError):
        psw.Plan(A, part, rank=0, world=3)  # 16 blocks over 3 ranks
    plan = psw.Plan(A, part, rank=1, world=2)
    F = cuda.zeros((plan.rows(), 8), dtype=cuda.float64, device="cuda")
    with pytest.raises(ValueError):  # world 2 needs a communicator
        plan.shard_solve(F, F.clone(), None)
    comm = psw.Comm(1, 0, psw.Comm.unique_id(), 0)
    with pytest.raises(ValueError):  # 1-rank communicator for a 2-rank plan
        plan.shard_solve(F, F.clone(), comm)
    comm.close()
    with pytest.raises(ValueError):  # a shard plan refuses psw_solve
        plan.solve(F, F.clone())


@pytest.mark.parametrize("world", [2, 3, 4])
def test_rhs_slices_equal_full_batch(psw, cuda, world):
    """RHS-sharded comparison mode: each rank's slice of one batch (rhs_slice)
    solved on its own is bitwise the full-batch solve of those RHS (RESWEEP:
    the per-RHS arithmetic does not depend on the batch width)."""
    from paper_0901_2859_b200.configs import CONFIGS
    from paper_0901_2859_b200.sharded import rhs_slice
    cfg = CONFIGS["C3"].with_(n=65536, nrhs=256)
    a, b = cfg.matrix_ab(0)
    A = psw.TridiagMatrix.symmetric(a, b)
    part = psw.decompose(cfg.n, 64).induced_partition()
    plan = psw.Plan(A, part)
    F = cuda.empty((cfg.n, cfg.nrhs), dtype=cuda.float64, device="cuda")
    psw.fill_uniform(F, 3, -1.0, 1.0)
    full = plan.solve(F, cuda.empty_like(F), path=psw.PATH_RESWEEP)
    for r in range(world):
        k0, k1 = rhs_slice(cfg.nrhs, world, r)
        Fs = F[:, k0:k1].contiguous()
        Xs = plan.solve(Fs, cuda.empty_like(Fs), path=psw.PATH_RESWEEP)
        cuda.cuda.synchronize()
        assert bool((Xs == full[:, k0:k1]).all())


@pytest.mark.parametrize("name,world", [("c1_n4096_P16", 2), ("decomp_n333_P9", 3), ("c0_n1024_P4", 4)])
def test_shard_solve_multi_process_through_the_c_abi(psw, cuda, name, world, tmp_path):
    """psw_shard_solve with world_size > 1: one PROCESS per rank, all on cuda:0,
    each with its own shard plan and a communicator of `world` ranks; the
    all-reduce between the two halves of the solve is the host-staged
    stand-in of tests/cpp/fake_nccl.cpp (PSW_NCCL_LIB), which sums the ranks'
    partial boundary values in rank order. What runs is the C-ABI path of the
    multi-GPU bench — rank > 0 plans, communicator checks, forward, in-place
    sum, backward — and the assembled solution matches the reference."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    fake = os.path.join(root, "paper_0901_2859_b200", "_lib", "libfake_nccl.so")
    if not os.path.exists(fake):
        pytest.skip("libfake_nccl.so not built")
    env = dict(os.environ, PSW_NCCL_LIB=fake)
    uid = str(tmp_path / "uid")
    outs = [str(tmp_path / f"x{r}.npy") for r in range(world)]
    procs = [subprocess.Popen([sys.executable, os.path.join(root, "tests", "_shard_worker.py"), name,
                               str(world), str(r), uid, outs[r]], env=env, stdout=subprocess.PIPE,
                              stderr=subprocess.STDOUT) for r in range(world)]
    logs = []
    for p in procs:
        out, _ = p.communicate(timeout=300)
        logs.append(out.decode()[-2000:])
    assert all(p.returncode == 0 for p in procs), logs
    g = load_golden(name)
    X = np.concatenate([np.load(o) for o in outs], axis=0)
    assert rel_l2(X.T, g["X"]) <= 1e-12
    # and bitwise the in-process emulation, whose sum also runs in rank order
    A = psw.TridiagMatrix(g["sub"], g["diag"], g["super"])
    part = psw.Partition(A.n(), g["bnd"].tolist())
    assert np.array_equal(X, _emulate(psw, cuda, A, part, np.ascontiguousarray(g["F"].T), world))
