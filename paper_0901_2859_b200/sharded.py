"""Multi-GPU batched solves: one process per GPU.

Row sharding (the paper's data decomposition, with the
GPUs as the processing elements): rank r of `world` owns the blocks
[r*P/world, (r+1)*P/world) of ONE global partition and the rows of those
blocks, for every right-hand side. The dichotomy combination
(dichotomy/boundary_solve.hpp:96-121) is linear in the betas, so each rank
forms its share of every boundary value from its own blocks and the solve's
only exchange is one all-reduce(sum) of p values per RHS (NCCL over NVLink);
the reference merely counts that round (runtime/run.hpp:93-94).

RHS sharding (comparison mode): every rank solves a disjoint slice of the
RHS against a replicated plan, with no communication.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import F64, LAYOUT_R, Partition, Plan, TridiagMatrix, _check, lib


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    blk0: int   # first owned block
    blk1: int   # one past the last owned block
    row0: int   # first owned row (0-based, global)
    row1: int   # one past the last owned row

    @property
    def rows(self) -> int:
        return self.row1 - self.row0


def shard_layout(n: int, part: Partition, world: int) -> list[Shard]:
    """Ownership of every rank (mirrors psw_shard.cpp build_shard_tables).
    Block t owns rows [n_t, n_{t+1}) (partition.hpp:26-29, 1-based)."""
    P = part.p() + 1
    if world < 1 or P % world:
        raise ValueError(f"P = {P} blocks must be divisible by world = {world}")
    loc = P // world
    out = []
    for r in range(world):
        b0, b1 = r * loc, (r + 1) * loc
        row0 = part.block_begin(b0) - 1
        row1 = part.block_end(b1 - 1) - 1
        out.append(Shard(r, world, b0, b1, row0, row1))
    return out


def combine_matrix(A: TridiagMatrix, part: Partition) -> np.ndarray:
    """p x 2P matrix [MR | ML] with v = MR @ right + ML @ left (host, no GPU)."""
    p, P = part.p(), part.p() + 1
    out = np.zeros((max(p, 1), 2 * P))
    b = np.ascontiguousarray(part.boundaries if p else [0], dtype=np.int64)
    dp = C.POINTER(C.c_double)
    L = lib()
    L.psw_combine_matrix.argtypes = [C.c_int64, dp, dp, dp, C.c_int64, C.POINTER(C.c_int64), dp]
    _check(L.psw_combine_matrix(A.n(), A.sub.ctypes.data_as(dp), A.diag.ctypes.data_as(dp),
                                A.super.ctypes.data_as(dp), p,
                                b.ctypes.data_as(C.POINTER(C.c_int64)), out.ctypes.data_as(dp)))
    return out[:p]


def rhs_slice(nrhs: int, world: int, rank: int) -> tuple[int, int]:
    """RHS-sharded comparison mode: near-equal contiguous RHS ranges."""
    base, rem = divmod(nrhs, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


class ShardedSolver:
    """Row-sharded solve of A X = F over a torch.distributed process group.

    On GPUs the exchange is inside the C ABI: psw_shard_solve runs the
    forward sweep, an ncclAllReduce over the solver's own NCCL communicator
    (created from a unique id that rank 0 broadcasts over `group`) and the
    backward sweep on one stream. With `use_nccl=False`, or a `plan` stand-in
    (the CPU gloo tests), the two halves run around
    torch.distributed.all_reduce of the p x N partial boundary values.
    A stand-in needs workspace_bytes / shard_forward / shard_backward /
    row_offset / rows with the Plan signatures."""

    def __init__(self, A: TridiagMatrix, part: Partition, dtype: int = F64, device: int = 0,
                 group=None, plan=None, use_nccl: bool | None = None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.shard = shard_layout(A.n(), part, self.world)[self.rank]
        own_plan = plan is None
        self.plan = plan if plan is not None else Plan(A, part, dtype=dtype, device=device,
                                                       rank=self.rank, world=self.world)
        self.p = part.p()
        self.comm_bytes_per_rhs = 8 * self.p
        self.device = device
        self.comm = None
        if use_nccl is None:
            use_nccl = own_plan
        if use_nccl:
            from . import Comm
            box = [Comm.unique_id() if self.rank == 0 else None]
            dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group else 0,
                                       group=group)
            self.comm = Comm(self.world, self.rank, box[0], device)

    def close(self):
        if self.comm is not None:
            self.comm.close()
            self.comm = None

    def solve(self, F_local, X_local=None, nrhs: int | None = None, stream=None):
        """F_local: (rows, N) owned rows of the series (layout R); X_local
        defaults to F_local (in place). Returns X_local."""
        if X_local is None:
            X_local = F_local
        N = F_local.shape[1] if nrhs is None else nrhs
        if self.comm is not None:
            return self.plan.shard_solve(F_local, X_local, self.comm, N, stream=stream)
        import contextlib

        import torch
        on_gpu = getattr(F_local, "is_cuda", False)
        # the zero fill, the all-reduce and both halves are ordered on one stream
        ctx = torch.cuda.stream(stream) if on_gpu and stream is not None else contextlib.nullcontext()
        with ctx:
            ws = torch.empty(max(self.plan.workspace_bytes(N), 1), dtype=torch.uint8,
                             device=F_local.device)
            partials = torch.zeros((max(self.p, 1), N), dtype=torch.float64, device=F_local.device)
            cur = torch.cuda.current_stream() if on_gpu else None
            self.plan.shard_forward(F_local, N, ws, partials, stream=cur)
            if self.p > 0 and self.world > 1:
                self.dist.all_reduce(partials, op=self.dist.ReduceOp.SUM, group=self.group)
            self.plan.shard_backward(F_local, X_local, N, ws, partials, stream=cur)
        return X_local

    def solve_host(self, F_host, X_host=None, stream=None):
        """End to end from pinned host rows: H2D of this rank's F rows, the
        sharded solve, D2H of its X rows (the bench's e2e leg)."""
        import torch
        if X_host is None:
            X_host = torch.empty_like(F_host)
        dev = torch.device("cuda", self.device)
        Fd = F_host.to(dev, non_blocking=True)
        self.solve(Fd, Fd, stream=stream)
        X_host.copy_(Fd, non_blocking=True)
        torch.cuda.current_stream(dev).synchronize()
        return X_host


__all__ = ["Shard", "shard_layout", "combine_matrix", "rhs_slice", "ShardedSolver", "LAYOUT_R"]
