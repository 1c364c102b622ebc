"""Host side of the statistics consumer: the library's regularized_gamma_q
(stats.cpp:13-60 restated) against the reference's own function on a grid,
and the reference's own argument checks. No GPU."""
import math

import pytest

import paper_2309_16682_b200 as V


def test_regularized_gamma_q_matches_reference(golden):
    pts = golden["stats"]["gamma_q"]
    worst = 0.0
    exact = 0
    for a, x, ref in pts:
        got = V.regularized_gamma_q(a, x)
        if got == ref:
            exact += 1
        else:
            worst = max(worst, abs(got - ref) / max(abs(ref), 1e-300))
    # same formulas; the reference build may contract a*d+b into FMAs
    assert worst <= 1e-12, worst
    assert exact >= len(pts) // 2


def test_regularized_gamma_q_edges():
    assert V.regularized_gamma_q(127.5, 0.0) == 1.0
    with pytest.raises(V.InvalidArgument):
        V.regularized_gamma_q(0.0, 1.0)
    with pytest.raises(V.InvalidArgument):
        V.regularized_gamma_q(1.0, -1.0)
    # Q(1, x) = exp(-x)
    for x in (0.5, 1.0, 3.0, 10.0):
        assert math.isclose(V.regularized_gamma_q(1.0, x), math.exp(-x), rel_tol=1e-13)
