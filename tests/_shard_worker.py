"""One rank of the two-process sharded-solve test (tests/test_sharded_gpu.py):
psw_shard_solve through the C ABI with PSW_NCCL_LIB pointing at the host-staged
stand-in (tests/cpp/fake_nccl.cpp), every rank on cuda:0.

    python _shard_worker.py <golden> <world> <rank> <uid file> <out file>
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    name, world, rank, uid_path, out_path = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], sys.argv[5]
    import torch

    import paper_0901_2859_b200 as psw
    from conftest import load_golden
    from paper_0901_2859_b200.sharded import shard_layout
    g = load_golden(name)
    A = psw.TridiagMatrix(g["sub"], g["diag"], g["super"])
    part = psw.Partition(A.n(), g["bnd"].tolist())
    if rank == 0:
        uid = psw.Comm.unique_id()
        with open(uid_path + ".tmp", "wb") as f:
            f.write(uid)
        os.replace(uid_path + ".tmp", uid_path)
    else:
        t0 = time.time()
        while not os.path.exists(uid_path):
            if time.time() - t0 > 60:
                raise RuntimeError("rank 0 never published the communicator id")
            time.sleep(0.01)
        uid = open(uid_path, "rb").read()
    plan = psw.Plan(A, part, rank=rank, world=world)
    comm = psw.Comm(world, rank, uid, 0)
    sh = shard_layout(A.n(), part, world)[rank]
    F = np.ascontiguousarray(g["F"].T)  # layout R: (n, N)
    f = torch.from_numpy(np.ascontiguousarray(F[sh.row0:sh.row1])).cuda()
    x = torch.empty_like(f)
    for _ in range(2):  # twice: the communicator and its slots are reused
        plan.shard_solve(f, x, comm)
    torch.cuda.synchronize()
    np.save(out_path, x.cpu().numpy())
    comm.close()


if __name__ == "__main__":
    main()
