"""Host metrics (metrics.cpp error part) against the reference's own metric
tests (test_metrics.cpp:11-63) and the oracle's analytic LCO propagator."""
import math

import numpy as np
import pytest

import _oracle as O
from paper_2605_23727_b200 import metrics as M


def test_normalized_final_error_kats():  # test_metrics.cpp:11-38
    a = np.array([1.0, 2.0, 3.0, 4.0])
    assert M.normalized_final_error(a, a, 2) == 0.0
    b = a.copy()
    b[0] -= 3.0
    b[1] -= 4.0
    assert M.normalized_final_error(a, b, 2) == pytest.approx(5.0 / math.sqrt(2.0), rel=1e-15)
    assert M.normalized_final_error(np.zeros(7), np.ones(7), 7) == pytest.approx(1.0, rel=1e-15)
    with pytest.raises(ValueError):
        M.normalized_final_error(a, np.zeros(3), 2)
    with pytest.raises(ValueError):
        M.normalized_final_error(a, b, 0)
    r = O.rng_uniform(40, 0, 18, -1.0, 1.0).reshape(6, 3).T  # u, v, w interleaved like the draws
    u, v, w = r[0], r[1], r[2]
    assert M.normalized_final_error(u, v, 3) == pytest.approx(M.normalized_final_error(v, u, 3), rel=1e-15)
    assert M.normalized_final_error(u, w, 3) <= M.normalized_final_error(u, v, 3) + M.normalized_final_error(v, w, 3) + 1e-15


def test_real_local_error_kats():  # test_metrics.cpp:40-63
    x = O.rng_uniform(41, 0, 8, 0.0, 2.0)
    for h in (1e-3, 0.05, 0.5, 1.0):
        ex = M.lco_analytic(x, h)
        assert M.real_local_error(x, ex, h, 1e-8, 1e-6) <= 1e-13
    ident = np.array([1.0, 0.0, 1.0, 0.0])
    h = 1.5707963267948966
    xn = M.lco_analytic(ident, h).copy()
    xn[0] += 1e-8
    assert M.real_local_error(ident, xn, h, 1e-2, 1.0) == pytest.approx(1e-6, rel=1e-8)


@pytest.mark.parametrize("n", [1, 4, 33, 1024])
def test_lco_analytic_matches_oracle_bitwise(n):
    x = O.rng_uniform(7 + n, 1, 2 * n, -1.0, 1.0)
    for t in (0.0, 1e-3, 0.37, 2.5, 10.0):
        assert np.array_equal(M.lco_analytic(x, t), O.lco_analytic(x, t))
    with pytest.raises(ValueError):
        M.lco_analytic(np.zeros(3), 1.0)
