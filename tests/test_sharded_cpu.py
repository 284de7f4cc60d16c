"""Row-sharded multi-GPU path on the CPU: the combination matrix (host
C ABI), the shard ownership, and the ShardedSolver orchestration over a
world_size 2/4 `gloo` process group, with the per-rank device work emulated
by the CPU oracle (test infrastructure) — the exchange protocol, the
block/row bookkeeping and the linearity argument are the product code."""
import os
import socket

import numpy as np
import pytest

from conftest import load_golden, rel_l2


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("name", ["c0_n1024_P4", "c1_n4096_P16", "c4_n4096_P16", "rand_n200_p7",
                                  "decomp_n333_P9", "tiny_n12_p6", "mixed_n96_P8"])
def test_combine_matrix_matches_dichotomy(psw, orc, name):
    """v = MR right + ML left reproduces solve_boundaries (boundary_solve.hpp:96-121)."""
    from paper_0901_2859_b200.sharded import combine_matrix
    g = load_golden(name)
    A = psw.TridiagMatrix(g["sub"], g["diag"], g["super"])
    part = psw.Partition(A.n(), g["bnd"].tolist())
    M = combine_matrix(A, part)
    P = part.p() + 1
    pre = orc.preliminary(g["sub"], g["diag"], g["super"], g["bnd"])
    for k in range(g["F"].shape[0]):
        left, right = orc.betas(g["bnd"], pre["g"], g["F"][k])
        v, _ = orc.solve_boundaries(pre["zr"], pre["zl"], left, right)
        vm = M[:, :P] @ right + M[:, P:] @ left
        assert np.abs(vm - v).max() <= 1e-13 * np.abs(v).max()


def test_shard_layout_tiles_rows(psw):
    from paper_0901_2859_b200.sharded import shard_layout, rhs_slice
    for n, P, world in ((1024, 4, 2), (4096, 16, 4), (4096, 16, 8), (333, 9, 3), (1 << 20, 64, 8)):
        part = psw.decompose(n, P).induced_partition()
        sh = shard_layout(n, part, world)
        assert sh[0].row0 == 0 and sh[-1].row1 == n
        for a, b in zip(sh, sh[1:]):
            assert a.row1 == b.row0 and a.blk1 == b.blk0
        assert sum(s.blk1 - s.blk0 for s in sh) == P
    with pytest.raises(ValueError):
        shard_layout(1024, psw.decompose(1024, 6).induced_partition(), 4)
    assert [rhs_slice(10, 3, r) for r in range(3)] == [(0, 4), (4, 7), (7, 10)]


class CpuShardPlan:
    """CPU stand-in for a rank's CUDA shard plan (same method names)."""

    def __init__(self, orc, g, shard, M):
        self.orc, self.g, self.shard, self.M = orc, g, shard, M
        self.pre = orc.preliminary(g["sub"], g["diag"], g["super"], g["bnd"])
        self.n = g["diag"].size
        self.bnd = g["bnd"]
        self.p = self.bnd.size
        self.P = self.p + 1

    def _full(self, F_local, k):
        f = np.zeros(self.n)
        f[self.shard.row0:self.shard.row1] = F_local[:, k].numpy()
        return f

    def workspace_bytes(self, N):
        return 1

    def shard_forward(self, F, N, ws, partials, stream=None):
        import torch
        for k in range(N):
            f = self._full(F, k)
            left, right = self.orc.betas(self.bnd, self.pre["g"], f)  # own rows only are nonzero
            own = np.zeros(self.P, bool)
            own[self.shard.blk0:self.shard.blk1] = True
            v = self.M[:, :self.P] @ np.where(own, right, 0) + self.M[:, self.P:] @ np.where(own, left, 0)
            partials[:, k] = torch.from_numpy(v)
        self._F = F.clone()

    def shard_backward(self, F, X, N, ws, partials, stream=None):
        import torch
        V = partials.numpy()
        g = self.g
        for k in range(N):
            f = self._full(self._F, k)
            for t in range(self.shard.blk0, self.shard.blk1):
                blk = self.orc.solve_local(g["sub"], g["diag"], g["super"], self.bnd, t, f,
                                           first=V[t - 1, k] if t > 0 else None,
                                           last=V[t, k] if t < self.p else None)
                lo = 0 if t == 0 else int(self.bnd[t - 1]) - 1
                hi = self.n if t == self.p else int(self.bnd[t]) - 1
                X[lo - self.shard.row0:hi - self.shard.row0, k] = torch.from_numpy(blk[:hi - lo])


def _worker(rank, world, port, name, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_0901_2859_b200 as psw
        from oracle.pyoracle import Oracle
        from paper_0901_2859_b200.sharded import ShardedSolver, combine_matrix, shard_layout
        g = load_golden(name)
        A = psw.TridiagMatrix(g["sub"], g["diag"], g["super"])
        part = psw.Partition(A.n(), g["bnd"].tolist())
        shard = shard_layout(A.n(), part, world)[rank]
        plan = CpuShardPlan(Oracle(), g, shard, combine_matrix(A, part))
        solver = ShardedSolver(A, part, plan=plan)
        assert solver.shard == shard and solver.comm_bytes_per_rhs == 8 * part.p()
        assert solver.comm is None  # a stand-in plan: the exchange is torch.distributed (gloo)
        F_local = torch.from_numpy(np.ascontiguousarray(g["F"].T[shard.row0:shard.row1]))
        X_local = torch.zeros_like(F_local)
        solver.solve(F_local, X_local)
        parts = [None] * world
        dist.all_gather_object(parts, (shard.row0, X_local.numpy()))
        if rank == 0:
            X = np.zeros_like(g["F"].T)
            for r0, xl in parts:
                X[r0:r0 + xl.shape[0]] = xl
            q.put(rel_l2(X.T, g["X"]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,world", [("c1_n4096_P16", 2), ("c1_n4096_P16", 4),
                                        ("c0_n1024_P4", 2), ("decomp_n333_P9", 3)])
def test_row_sharded_gloo(name, world):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p_ in procs:
        p_.start()
    for p_ in procs:
        p_.join(timeout=300)
        assert p_.exitcode == 0
    err = q.get(timeout=10)
    assert err <= 1e-12, err


def _rhs_worker(rank, world, port, name, q):
    """RHS-sharded comparison mode: rank r solves the RHS slice
    rhs_slice(N, world, r) of ONE batch with a replicated plan and no
    exchange; the oracle stands in for the device solve."""
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.pyoracle import Oracle
        from paper_0901_2859_b200.sharded import rhs_slice
        g = load_golden(name)
        N = g["F"].shape[0]
        k0, k1 = rhs_slice(N, world, rank)
        X = Oracle().solve_batch(g["sub"], g["diag"], g["super"], g["bnd"], g["F"][k0:k1])
        parts = [None] * world
        dist.all_gather_object(parts, (k0, k1, X))
        if rank == 0:
            Xall = np.zeros_like(g["F"])
            seen = np.zeros(N, int)
            for a, b, x in parts:
                Xall[a:b] = x
                seen[a:b] += 1
            q.put((int(seen.min()), int(seen.max()), rel_l2(Xall, g["X"])))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,world", [("c0_n1024_P4", 2), ("rand_n200_p7", 3)])
def test_rhs_sharded_gloo(name, world):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rhs_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p_ in procs:
        p_.start()
    for p_ in procs:
        p_.join(timeout=300)
        assert p_.exitcode == 0
    lo, hi, err = q.get(timeout=10)
    assert lo == hi == 1  # every RHS solved exactly once
    assert err <= 1e-12, err
