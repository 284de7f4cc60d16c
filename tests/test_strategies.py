"""Non-symmetric setup: the GRowStrategy routes of compute_preliminary
(dichotomy/preliminary.hpp:18-24, 108-164; core/symmetrize.hpp:21-37;
core/inverse_rows.hpp:46-104) in the C restatement, pinned bitwise to the
compiled reference, plus the reference's own known answers restated
(tests/test_core.cpp:132-253, tests/test_dichotomy.cpp:423-457)."""
import numpy as np
import pytest

from oracle.pyoracle import (AUTO, DIRECT_SYMMETRIC, EXPLICIT_INVERSE, NOT_SYMMETRIZABLE,
                             ORACLE_FALLBACK, SYMMETRIZE, TRANSPOSE_SOLVE, OracleError)

STRATEGIES = [AUTO, DIRECT_SYMMETRIC, SYMMETRIZE, EXPLICIT_INVERSE, TRANSPOSE_SOLVE]


def symmetrizable(rng, n):
    """sub * super > 0 everywhere, dominant diagonal (test_util random_symmetrizable shape)."""
    sub = -rng.uniform(0.2, 1.0, n - 1)
    sup = -rng.uniform(0.2, 1.0, n - 1)
    diag = np.r_[0, np.abs(sub)] + np.r_[np.abs(sup), 0] + rng.uniform(0.5, 1.5, n)
    return sub, diag, sup


def mixed_signs(rng, n):
    """dominant with mixed off-diagonal signs: not symmetrizable."""
    sub = rng.uniform(-1, 1, n - 1)
    sup = rng.uniform(-1, 1, n - 1)
    sup[::3] = -np.sign(sub[::3]) * np.abs(sup[::3])
    diag = np.r_[0, np.abs(sub)] + np.r_[np.abs(sup), 0] + rng.uniform(0.5, 1.5, n)
    return sub, diag, sup


def reducible(rng, n):
    """a zero super entry: explicit inverse undefined -> transpose solves."""
    sub, diag, sup = mixed_signs(rng, n)
    sup[n // 3] = 0.0
    return sub, diag, sup


MATRICES = {"symmetrizable": symmetrizable, "mixed": mixed_signs, "reducible": reducible}


def _partition(rng, n, p):
    return np.sort(rng.choice(np.arange(2, n), size=p, replace=False)).astype(np.int64)


def _outcome(fn):
    try:
        return ("ok", fn())
    except OracleError as e:
        return ("err", (e.code, e.index if e.code == NOT_SYMMETRIZABLE else -1))


@pytest.mark.parametrize("kind", sorted(MATRICES))
@pytest.mark.parametrize("strategy", STRATEGIES)
def test_preliminary_bitwise_reference(orc, ref, kind, strategy):
    rng = np.random.default_rng(7 + strategy)
    n = 97
    A = MATRICES[kind](rng, n)
    bnd = _partition(rng, n, 6)
    a = _outcome(lambda: orc.preliminary(*A, bnd, strategy=strategy))
    b = _outcome(lambda: ref.preliminary(*A, bnd, strategy=strategy))
    assert a[0] == b[0], (a, b)
    if a[0] == "err":
        assert a[1] == b[1]
        return
    for key in ("g", "zr", "zl"):
        assert np.array_equal(a[1][key], b[1][key]), key
    assert a[1]["max_z"] == b[1]["max_z"]
    assert a[1]["strategy_used"] == b[1]["strategy_used"]


@pytest.mark.parametrize("kind", sorted(MATRICES))
@pytest.mark.parametrize("strategy", STRATEGIES)
def test_solve_batch_bitwise_reference(orc, ref, kind, strategy):
    rng = np.random.default_rng(11 + strategy)
    n = 150
    A = MATRICES[kind](rng, n)
    bnd = _partition(rng, n, 5)
    F = rng.uniform(-1, 1, (4, n))
    a = _outcome(lambda: orc.solve_batch(*A, bnd, F, strategy=strategy))
    b = _outcome(lambda: ref.solve_batch(*A, bnd, F, strategy=strategy))
    assert a[0] == b[0]
    if a[0] == "ok":
        assert np.array_equal(a[1], b[1])
    else:
        assert a[1] == b[1]


def test_auto_routes(orc):
    """Auto: DirectSymmetric for sub == super, else Symmetrize, falling back to
    ExplicitInverse and then TransposeSolve (preliminary.hpp:111-132)."""
    rng = np.random.default_rng(3)
    n = 60
    bnd = _partition(rng, n, 4)
    sub, diag, _ = symmetrizable(rng, n)
    assert orc.preliminary(sub, diag, sub, bnd)["strategy_used"] == DIRECT_SYMMETRIC
    assert orc.preliminary(*symmetrizable(rng, n), bnd)["strategy_used"] == SYMMETRIZE
    assert orc.preliminary(*mixed_signs(rng, n), bnd)["strategy_used"] == EXPLICIT_INVERSE
    assert orc.preliminary(*reducible(rng, n), bnd)["strategy_used"] == TRANSPOSE_SOLVE


def test_explicit_strategies_report_their_failures(orc):
    """test_core.cpp:153-159 (NotSymmetrizable) and :236-253 (OracleFallbackRequired)."""
    rng = np.random.default_rng(5)
    n = 40
    bnd = _partition(rng, n, 3)
    sub, diag, sup = mixed_signs(rng, n)
    k = int(np.argmax(sub * sup <= 0))
    with pytest.raises(OracleError) as e:
        orc.preliminary(sub, diag, sup, bnd, strategy=SYMMETRIZE)
    assert e.value.code == NOT_SYMMETRIZABLE and e.value.index == k
    # reducible: the product representation is undefined
    sub = -np.ones(5)
    sup = -np.ones(5)
    sup[2] = 0.0
    diag = 2.0 * np.ones(6)
    with pytest.raises(OracleError) as e:
        orc.preliminary(sub, diag, sup, np.array([3]), strategy=EXPLICIT_INVERSE)
    assert e.value.code == ORACLE_FALLBACK
    # long strongly dominant: corner entries of the inverse underflow (test_core.cpp:249-253)
    n = 3000
    with pytest.raises(OracleError) as e:
        orc.preliminary(-np.ones(n - 1), 16.0 * np.ones(n), -np.ones(n - 1), np.array([1500]),
                        strategy=EXPLICIT_INVERSE)
    assert e.value.code == ORACLE_FALLBACK
    # non-symmetric version: the similarity scale sqrt(2)^k overflows (Symmetrize
    # rejected), the ratio products 2^-j underflow (ExplicitInverse rejected), so
    # Auto ends on transpose solves
    assert orc.preliminary(-np.ones(n - 1), 16.0 * np.ones(n), -np.ones(n - 1) * 0.5,
                           np.array([1500]))["strategy_used"] == TRANSPOSE_SOLVE


def test_routes_agree_with_dense_solve(orc):
    """test_dichotomy.cpp:423-442: every route solves a symmetrizable
    non-symmetric system to 1e-8 of the dense solution."""
    rng = np.random.default_rng(79)
    for _ in range(5):
        n = int(32 + rng.integers(0, 150))
        sub, diag, sup = symmetrizable(rng, n)
        bnd = _partition(rng, n, 5)
        f = rng.uniform(-1, 1, (1, n))
        dense = np.diag(diag) + np.diag(sub, -1) + np.diag(sup, 1)
        want = np.linalg.solve(dense, f[0])
        for s in (SYMMETRIZE, EXPLICIT_INVERSE, TRANSPOSE_SOLVE):
            x = orc.solve_batch(sub, diag, sup, bnd, f, strategy=s)[0]
            assert np.linalg.norm(x - want) <= 1e-8 * np.linalg.norm(want)


def test_symmetrize_example_inverse_row(orc):
    """test_core.cpp:132-143 uses the pair sub = 2, super = 8 (scale 1/2,
    symmetrized off-diagonals 4). Embedded in an order-3 matrix, the inverse
    row obtained through the Symmetrize route equals the dense inverse row."""
    sub, diag, sup = np.array([2.0, 1.0]), np.array([1.0, 1.0, 3.0]), np.array([8.0, 1.0])
    pr = orc.preliminary(sub, diag, sup, np.array([2]), strategy=SYMMETRIZE)
    dense = np.diag(diag) + np.diag(sub, -1) + np.diag(sup, 1)
    assert np.allclose(pr["g"][0], np.linalg.inv(dense)[1], rtol=1e-13, atol=1e-15)
