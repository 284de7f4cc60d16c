"""Row-sharded CUDA path on one GPU: every rank's shard plan and kernels run
in this process (no rank waits on another, so no collective is needed); the
all-reduce is the sum of the ranks' partial boundary values."""
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
    Fl, Xl = [], []
    total = torch.zeros((max(p, 1), N), dtype=torch.float64, device="cuda")
    for sh, pl in zip(shards, plans):
        assert pl.row_offset() == sh.row0 and pl.rows() == sh.rows
        assert pl.partials_count() == p
        f = torch.from_numpy(np.ascontiguousarray(F[sh.row0:sh.row1])).to(tdt).cuda()
        x = torch.empty_like(f)
        part_v = torch.zeros_like(total)
        pl.shard_forward(f, x, part_v, N)
        total += part_v
        Fl.append(f)
        Xl.append(x)
    for pl, x in zip(plans, Xl):
        pl.shard_backward(x, total, N)
    torch.cuda.synchronize()
    return np.concatenate([x.double().cpu().numpy() for x in Xl], axis=0)


@pytest.mark.parametrize("name,world", [("c1_n4096_P16", 1), ("c1_n4096_P16", 2),
                                        ("c1_n4096_P16", 4), ("c1_n4096_P16", 8),
                                        ("c0_n1024_P4", 4), ("decomp_n333_P9", 3),
                                        ("c4_n4096_P16", 16)])
def test_row_sharded_matches_reference(psw, cuda, name, world):
    g = load_golden(name)
    A = psw.TridiagMatrix(g["sub"], g["diag"], g["super"])
    part = psw.Partition(A.n(), g["bnd"].tolist())
    X = _emulate(psw, cuda, A, part, np.ascontiguousarray(g["F"].T), world)
    assert rel_l2(X.T, g["X"]) <= 1e-12


def test_row_sharded_c3_shape(psw, cuda):
    """C3 shape (n = 2^20, P = 64) over 8 emulated ranks, subset of RHS
    checked against the oracle."""
    from oracle.pyoracle import Oracle
    from paper_0901_2859_b200.configs import CONFIGS, uniform
    cfg = CONFIGS["C3"]
    a, b = cfg.matrix_ab(0)
    A = psw.TridiagMatrix.symmetric(a, b)
    part = psw.decompose(cfg.n, cfg.P).induced_partition()
    N = 8
    F = uniform(3, cfg.n * N, -1, 1).reshape(cfg.n, N)
    X = _emulate(psw, cuda, A, part, F, 8)
    want = Oracle().solve_batch_threads(a, b, a, np.array(part.boundaries),
                                        np.ascontiguousarray(F.T), 8)[0]
    assert rel_l2(X.T, want) <= 1e-12


def test_shard_rejects_bad_world(psw, cuda):
    g = load_golden("c1_n4096_P16")
    A = psw.TridiagMatrix(g["sub"], g["diag"], g["super"])
    part = psw.Partition(A.n(), g["bnd"].tolist())
    with pytest.raises(ValueError):
        psw.Plan(A, part, rank=0, world=3)  # 16 blocks over 3 ranks
