"""ADI consumer (poisson/adi.hpp), host side: parameters, iteration bound,
partitions and the model problem against the compiled reference and its
known answers (tests/test_poisson.cpp:226-248)."""
import math

import numpy as np
import pytest

from conftest import load_golden


def test_iteration_bound_documented_cases():  # test_poisson.cpp:226-230
    from paper_0901_2859_b200 import adi
    assert adi.adi_iteration_bound(512, 1e-5) == 17
    assert adi.adi_iteration_bound(128, 1e-5) == 14
    assert adi.adi_iteration_bound(64, 4.0) == 0


def test_parameters_geometric_in_range():  # test_poisson.cpp:232-248
    from paper_0901_2859_b200 import adi
    n = 128
    h = 1.0 / n
    lmin = 4.0 / (h * h) * math.sin(math.pi / (2.0 * n)) ** 2
    lmax = 4.0 / (h * h) * math.cos(math.pi / (2.0 * n)) ** 2
    single = adi.adi_parameters(n, 1)
    assert len(single) == 1
    assert single[0] == pytest.approx(1.0 / math.sqrt(lmin * lmax), rel=1e-12)
    taus = adi.adi_parameters(n, 9)
    for j, t in enumerate(taus):
        assert 1.0 / lmax <= t <= 1.0 / lmin
        assert j == 0 or t > taus[j - 1]


@pytest.mark.parametrize("n1,n2,cycle,pes", [(24, 18, 5, 1), (40, 33, 5, 3), (64, 64, 14, 4)])
def test_workspace_parameters_match_reference(ref, n1, n2, cycle, pes):
    from paper_0901_2859_b200 import adi
    h1, h2 = 1.0 / n1, 1.0 / n2
    lmin = min(adi._lambda_min(n1, h1), adi._lambda_min(n2, h2))
    lmax = max(adi._lambda_max(n1, h1), adi._lambda_max(n2, h2))
    ours = np.array(adi.geometric_parameters(lmin, lmax, cycle))
    assert np.array_equal(ours, ref.adi_parameters(n1, n2, h1, h2, cycle, pes))
    for n, eps in ((64, 1e-5), (100, 1e-7), (32, 0.5)):
        assert adi.adi_iteration_bound(n, eps) == ref.adi_iteration_bound(n, eps)


def test_golden_parameters():
    from paper_0901_2859_b200 import adi
    for name in ("adi_steps_24x18_pes1", "adi_steps_40x33_pes3"):
        g = load_golden(name)
        n1, n2 = int(g["n1"]), int(g["n2"])
        h1, h2 = 1.0 / n1, 1.0 / n2
        lmin = min(adi._lambda_min(n1, h1), adi._lambda_min(n2, h2))
        lmax = max(adi._lambda_max(n1, h1), adi._lambda_max(n2, h2))
        assert np.array_equal(np.array(adi.geometric_parameters(lmin, lmax, int(g["cycle"]))),
                              g["taus"])


def test_model_problem_matches_reference(ref):
    from paper_0901_2859_b200 import adi
    for n1, n2 in ((8, 8), (24, 18)):
        f, ex = adi.model_problem_host(n1, n2)
        rf, rex = ref.model_problem(n1, n2)
        assert np.array_equal(f, rf) and np.array_equal(ex, rex)


def test_partitions_follow_reference_rule(orc):
    """adi.hpp:73-77: decompose(order, pes) with pes lowered until order >= 2 pes."""
    from paper_0901_2859_b200 import adi
    assert adi._make_partition(23, 1).boundaries == []
    assert adi._make_partition(39, 3).boundaries == orc.decompose(39, 3).tolist()
    assert adi._make_partition(5, 4).boundaries == orc.decompose(5, 2).tolist()
