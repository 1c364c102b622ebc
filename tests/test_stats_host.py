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
    # same formulas with the reference build's fused multiply-adds: bit-exact
    assert exact == len(pts), worst


def test_regularized_gamma_q_edges():
    assert V.regularized_gamma_q(127.5, 0.0) == 1.0
    with pytest.raises(V.InvalidArgument):
        V.regularized_gamma_q(0.0, 1.0)
    with pytest.raises(V.InvalidArgument):
        V.regularized_gamma_q(1.0, -1.0)
    # Q(1, x) = exp(-x)
    for x in (0.5, 1.0, 3.0, 10.0):
        assert math.isclose(V.regularized_gamma_q(1.0, x), math.exp(-x), rel_tol=1e-13)


def test_reports_from_counts_match_reference_self_test(golden):
    """monobit / chi2_bytes from counts on the constant 0xDEADBEEF source
    (the CLI's --self-test) equal the reference's reports exactly."""
    ref = golden["stats"]["self_test_0xDEADBEEF"]
    w, n = 0xDEADBEEF, 1000000
    import numpy as np
    bins = np.zeros(256, np.uint64)
    for b in (w & 0xFF, (w >> 8) & 0xFF, (w >> 16) & 0xFF, w >> 24):
        bins[b] += n
    m = V.monobit_from_counts(n, bin(w).count("1") * n)
    c = V.chi2_bytes_from_counts(n, bins)
    assert (m.statistic, m.p_value, m.pass_) == (ref[0]["statistic"], ref[0]["p_value"], ref[0]["pass"])
    assert (c.statistic, c.p_value, c.pass_) == (ref[1]["statistic"], ref[1]["p_value"], ref[1]["pass"])
    with pytest.raises(V.InvalidArgument):
        V.monobit_from_counts(999999, 0)
    with pytest.raises(V.InvalidArgument):
        V.chi2_bytes_from_counts(3199, bins)
