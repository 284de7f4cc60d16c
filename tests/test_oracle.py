"""Pin the CPU oracle (oracle/psw_oracle.c) before trusting it.

1. The reference's own known-answer tests, restated (file:line in
   /root/reference/proj/tests).
2. Bitwise agreement with the committed fixtures produced by the reference
   itself (tests/gen_golden.py -> tests/golden/*.npz).
3. Live bitwise agreement with oracle/_ref (the reference compiled from its
   headers) on random cases, when it is available.
"""
import numpy as np
import pytest

from conftest import golden_cases, load_golden, rel_max
from oracle.pyoracle import OracleError, PIVOT_BREAKDOWN, TOO_MANY_PES


def const(n, a, b, c):
    return np.full(n - 1, a), np.full(n, b), np.full(n - 1, c)


# ---------------------------------------------------------------- core
def test_thomas_order3(orc):  # test_core.cpp:21-30
    x = orc.thomas(*const(3, -1, 2, -1), [1, 0, 0])
    np.testing.assert_allclose(x, [0.75, 0.5, 0.25], rtol=1e-13)


def test_thomas_identity(orc):  # test_core.cpp:32-36
    f = np.array([5.0, -1.0, 0.0, 2.0])
    assert np.array_equal(orc.thomas(*const(4, 0, 1, 0), f), f)


def test_thomas_order7_closed_form(orc):  # test_core.cpp:38-46
    x = orc.thomas(*const(7, -1, 2, -1), np.ones(7))
    i = np.arange(1, 8)
    np.testing.assert_allclose(x, i * (8 - i) / 2, rtol=1e-13)


def test_thomas_pivot_breakdown(orc):  # test_core.cpp:48-55
    with pytest.raises(OracleError) as e:
        orc.thomas([-1.0, -1.0], [1.0, 2.0, 1.0], [-1.0, -1.0], [1, 0, 0])
    assert e.value.code == PIVOT_BREAKDOWN and e.value.index == 2


def test_thomas_random_corpus_vs_dense(orc):  # test_core.cpp:77-96 (numpy dense LU)
    rng = np.random.default_rng(7)
    for _ in range(60):
        n = int(rng.integers(2, 200))
        a = rng.uniform(0.2, 1, n - 1) * rng.choice([-1, 1], n - 1)
        c = rng.uniform(0.2, 1, n - 1) * rng.choice([-1, 1], n - 1)
        off = np.zeros(n); off[1:] += np.abs(a); off[:-1] += np.abs(c)
        b = (off * (1 + rng.uniform(0.05, 1, n)) + 0.1) * rng.choice([-1, 1], n)
        f = rng.uniform(-1, 1, n)
        x = orc.thomas(a, b, c, f)
        A = np.diag(b) + np.diag(a, -1) + np.diag(c, 1)
        assert rel_max(x, np.linalg.solve(A, f)) <= 1e-11
        assert np.abs(A @ x - f).max() <= 1e-10 * np.abs(f).max()


# ---------------------------------------------------------------- runtime/decompose
def test_decompose_even(orc):  # test_runtime.cpp:20-25
    assert orc.decompose(16, 4).tolist() == [4, 8, 12]


def test_decompose_single(orc):  # test_runtime.cpp:27-32
    assert orc.decompose(10, 1).tolist() == []


def test_decompose_remainder(orc):  # test_runtime.cpp:34-39: sizes 3,2,2
    assert orc.decompose(7, 3).tolist() == [3, 5]


def test_decompose_too_many(orc):  # test_runtime.cpp:63-68
    for n, P in ((7, 4), (4, 3)):
        with pytest.raises(OracleError) as e:
            orc.decompose(n, P)
        assert e.value.code == TOO_MANY_PES
    assert orc.decompose(8, 4).tolist() == [2, 4, 6]


def test_decompose_tiles(orc):  # test_runtime.cpp:41-61
    rng = np.random.default_rng(5)
    for _ in range(100):
        n = 4 + int(rng.integers(0, 500))
        P = 1 + int(rng.integers(0, n // 2))
        b = [0] + orc.decompose(n, P).tolist() + [n]
        sizes = np.diff(b)
        assert sizes.min() >= 2 and sizes.max() - sizes.min() <= 1 and sizes.sum() == n


# ---------------------------------------------------------------- dichotomy
def test_partition_validation(orc):  # test_dichotomy.cpp:38-49
    assert orc.validate(16, [4, 8, 12])
    assert not orc.validate(16, [4, 4, 12])
    assert not orc.validate(16, [1, 8])
    assert not orc.validate(16, [8, 16])


def test_level_sets_p15(orc):  # test_dichotomy.cpp:51-58
    assert orc.level_sets(15) == [[8], [4, 12], [2, 6, 10, 14], [1, 3, 5, 7, 9, 11, 13, 15]]


def test_level_sets_p1_p3_p63(orc):  # test_dichotomy.cpp:60-64, SURVEY App. B
    assert orc.level_sets(1) == [[1]]
    assert orc.level_sets(3) == [[2], [1, 3]]
    l63 = orc.level_sets(63)
    assert l63[:3] == [[32], [16, 48], [8, 24, 40, 56]]


def test_level_sets_disjoint_cover(orc):  # test_dichotomy.cpp:66-95
    for p in range(1, 1025):
        sets = orc.level_sets(p)
        flat = [x for lv in sets for x in lv]
        assert sorted(flat) == list(range(1, p + 1))
        for m, lv in enumerate(sets):
            stride = 1 << (len(sets) - 1 - m)
            assert all(pos % stride == 0 for pos in lv)


def test_preliminary_order3(orc):  # test_dichotomy.cpp:97-105
    pre = orc.preliminary(*const(3, -1, 2, -1), [2])
    np.testing.assert_allclose(pre["g"][0], [0.5, 1.0, 0.5], rtol=1e-13)


def test_z_right_order3(orc):  # test_dichotomy.cpp:107-118 (b_right_matrix(A,1))
    z = orc.thomas([-1.0, -1.0], [1.0, 2.0, 2.0], [0.0, -1.0], [1, 0, 0])
    np.testing.assert_allclose(z, [1.0, 2 / 3, 1 / 3], rtol=1e-13)


def test_preliminary_identity(orc):  # test_dichotomy.cpp:120-132
    pre = orc.preliminary(*const(6, 0, 1, 0), [2, 4])
    for j, r in enumerate([2, 4]):
        e = np.zeros(6); e[r - 1] = 1
        assert np.array_equal(pre["g"][j], e)


def test_preliminary_residuals(orc):  # test_dichotomy.cpp:134-153
    rng = np.random.default_rng(41)
    n = 60
    a = rng.uniform(0.2, 1, n - 1) * rng.choice([-1, 1], n - 1)
    off = np.zeros(n); off[1:] += np.abs(a); off[:-1] += np.abs(a)
    b = off * 1.5 + 0.1
    bnd = np.sort(rng.choice(np.arange(2, n), 5, replace=False))
    pre = orc.preliminary(a, b, a, bnd)
    A = np.diag(b) + np.diag(a, -1) + np.diag(a, 1)
    for j, r in enumerate(bnd):
        e = np.zeros(n); e[r - 1] = 1
        assert np.abs(A @ pre["g"][j] - e).max() <= 1e-10


def test_preliminary_deterministic(orc):  # test_dichotomy.cpp:155-167 (bitwise)
    a, b, c = const(48, -1, 2.5, -1)
    p1 = orc.preliminary(a, b, c, [5, 17, 30])
    p2 = orc.preliminary(a, b, c, [5, 17, 30])
    assert all(np.array_equal(p1[k], p2[k]) for k in ("g", "zr", "zl"))


def test_z_stability_bound(orc):  # test_dichotomy.cpp:169-185
    rng = np.random.default_rng(47)
    for _ in range(20):
        n = 40
        a = rng.uniform(0.2, 1, n - 1) * rng.choice([-1, 1], n - 1)
        off = np.zeros(n); off[1:] += np.abs(a); off[:-1] += np.abs(a)
        b = (off * (1 + rng.uniform(0.05, 1, n)) + 0.1) * rng.choice([-1, 1], n)
        bnd = np.sort(rng.choice(np.arange(2, n), 6, replace=False))
        assert orc.preliminary(a, b, a, bnd)["max_z"] <= 1 + 1e-14
    assert orc.preliminary(*const(12, -1, 0.5, -1), [6])["max_z"] > 1 + 1e-14


def _order7(orc):
    a, b, c = const(7, -1, 2, -1)
    bnd = [2, 4, 6]
    pre = orc.preliminary(a, b, c, bnd)
    return a, b, c, bnd, pre


def test_order7_betas(orc):  # test_dichotomy.cpp:196-212
    a, b, c, bnd, pre = _order7(orc)
    left, right = orc.betas(bnd, pre["g"], np.ones(7))
    np.testing.assert_allclose([right[0], left[1], right[1], left[2], right[2], left[3]],
                               [0.75, 2.75, 2.5, 3.5, 2.25, 2.25], rtol=1e-12)
    v, _ = orc.solve_boundaries(pre["zr"], pre["zl"], left, right, two_sided=True)
    assert abs(v[1] - 8.0) <= 1e-12 * 8


def test_order7_boundaries(orc):  # test_dichotomy.cpp:234-243
    a, b, c, bnd, pre = _order7(orc)
    left, right = orc.betas(bnd, pre["g"], np.ones(7))
    v, _ = orc.solve_boundaries(pre["zr"], pre["zl"], left, right)
    np.testing.assert_allclose(v, [6.0, 8.0, 6.0], rtol=1e-12)
    left0, right0 = orc.betas(bnd, pre["g"], np.zeros(7))
    v0, _ = orc.solve_boundaries(pre["zr"], pre["zl"], left0, right0)
    assert np.all(v0 == 0.0)


def test_combine_terms_complexity(orc):  # test_dichotomy.cpp:290-307
    n = 4096
    a, b, c = const(n, -1, 2.5, -1)
    f = np.ones(n)
    for p in (15, 63, 255):
        bnd = orc.decompose(n, p + 1)
        pre = orc.preliminary(a, b, c, bnd)
        left, right = orc.betas(bnd, pre["g"], f)
        _, terms = orc.solve_boundaries(pre["zr"], pre["zl"], left, right)
        assert terms <= 8 * p * np.ceil(np.log2(p + 1))
        _, terms2 = orc.solve_boundaries(pre["zr"], pre["zl"], left, right, two_sided=True)
        assert terms2 >= p * p // 2


def test_solve_local_order7(orc):  # test_dichotomy.cpp:354-378
    a, b, c = const(7, -1, 2, -1)
    blk = orc.solve_local(a, b, c, [2, 4, 6], 2, np.ones(7), first=8.0, last=6.0)
    np.testing.assert_allclose(blk, [8.0, 7.5, 6.0], rtol=1e-13)
    assert np.all(orc.solve_local(a, b, c, [2, 4, 6], 1, np.zeros(7), 0.0, 0.0) == 0)
    a6, b6, c6 = const(6, -1, 3, -1)
    two = orc.solve_local(a6, b6, c6, [3, 4], 1, np.arange(1.0, 7.0), 2.5, -1.25)
    assert two.tolist() == [2.5, -1.25]


def test_solve_batch_vs_dense(orc):  # test_dichotomy.cpp:380-393
    rng = np.random.default_rng(71)
    a, b, c = const(128, -1, 2, -1)
    bnd = np.sort(rng.choice(np.arange(2, 128), 7, replace=False))
    F = rng.uniform(-1, 1, (100, 128))
    X = orc.solve_batch(a, b, c, bnd, F)
    A = np.diag(b) + np.diag(a, -1) + np.diag(c, 1)
    Xd = np.linalg.solve(A, F.T).T
    for k in range(100):
        assert rel_max(X[k], Xd[k]) <= 1e-9


def test_solve_batch_unit_vectors_inverse(orc):  # test_dichotomy.cpp:395-412
    rng = np.random.default_rng(73)
    n = 24
    a = rng.uniform(0.2, 1, n - 1) * rng.choice([-1, 1], n - 1)
    off = np.zeros(n); off[1:] += np.abs(a); off[:-1] += np.abs(a)
    b = off * 1.4 + 0.1
    bnd = np.sort(rng.choice(np.arange(2, n), 3, replace=False))
    X = orc.solve_batch(a, b, a, bnd, np.eye(n))
    inv = np.linalg.inv(np.diag(b) + np.diag(a, -1) + np.diag(a, 1))
    assert np.abs(X.T - inv).max() <= 1e-9 * max(np.abs(inv).max(), 1)


def test_single_boundary_equals_sweep(orc):  # test_dichotomy.cpp:414-421
    a, b, c = const(9, -1, 2, -1)
    f = np.array([1.0, -2.0, 0.5, 3.0, 0.0, -1.0, 2.0, 1.0, -0.5])
    X = orc.solve_batch(a, b, c, [5], f[None])
    assert rel_max(X[0], orc.thomas(a, b, c, f)) <= 1e-10


def test_comm_rounds(orc):  # test_runtime.cpp:117-135
    assert orc.comm_rounds(14) <= 6
    assert orc.comm_rounds(254) - orc.comm_rounds(14) <= 4
    assert orc.comm_rounds(0) == 0


def test_threads_bitwise_serial(orc):  # test_runtime.cpp:137-162
    rng = np.random.default_rng(17)
    n = 333
    a = -rng.uniform(0.5, 1, n - 1)
    b = np.abs(np.r_[0, a]) + np.abs(np.r_[a, 0]) + 0.5
    bnd = orc.decompose(n, 9)
    F = rng.uniform(-1, 1, (6, n))
    X1 = orc.solve_batch(a, b, a, bnd, F)
    X4, _, _ = orc.solve_batch_threads(a, b, a, bnd, F, 4)
    assert np.array_equal(X1, X4)


# ---------------------------------------------------------------- goldens (reference outputs)
@pytest.mark.parametrize("name", golden_cases())
def test_oracle_matches_reference_golden(orc, name):
    g = load_golden(name)
    X = orc.solve_batch(g["sub"], g["diag"], g["super"], g["bnd"], g["F"])
    assert np.array_equal(X, g["X"]), f"max diff {np.abs(X - g['X']).max()}"
    if "boundary" in g:
        pre = orc.preliminary(g["sub"], g["diag"], g["super"], g["bnd"])
        assert np.array_equal(pre["zr"], g["zr"]) and np.array_equal(pre["zl"], g["zl"])
        assert pre["max_z"] == float(g["max_z"])
        for k in range(g["F"].shape[0]):
            left, right = orc.betas(g["bnd"], pre["g"], g["F"][k])
            assert np.array_equal(left, g["betas_left"][k]) and np.array_equal(right, g["betas_right"][k])
            v, terms = orc.solve_boundaries(pre["zr"], pre["zl"], left, right)
            assert np.array_equal(v, g["boundary"][k])
            assert terms == int(g["combine_terms"])
    assert orc.comm_rounds(len(g["bnd"])) == int(g["comm_rounds"])


def test_oracle_matches_reference_live(orc, ref):
    rng = np.random.default_rng(99)
    for _ in range(15):
        n = int(rng.integers(8, 700))
        P = int(rng.integers(1, max(2, n // 4)))
        a = -rng.uniform(0.5, 1.0, n - 1)
        b = np.abs(np.r_[0, a]) + np.abs(np.r_[a, 0]) + rng.uniform(0.1, 1, n)
        bnd = orc.decompose(n, P)
        assert np.array_equal(bnd, ref.decompose(n, P))
        F = rng.uniform(-1, 1, (3, n))
        assert np.array_equal(orc.solve_batch(a, b, a, bnd, F), ref.solve_batch(a, b, a, bnd, F))


def test_generator_host_matches_oracle(orc):
    from paper_0901_2859_b200 import configs
    v = configs.uniform(12345, 1000, -1.0, 1.0, offset=77)
    assert np.array_equal(v, orc.fill_uniform(1000, 12345, -1.0, 1.0, offset=77))
