"""The K-level AHP closed form (tests/ahp_closed_form.py) against the oracle's explicit
pairwise matrix and against the hand-derived two-level form (CPU only): it is what pins the
GPU's AHP at full C5 scale (tests/test_gpu_parity2.py), so it is pinned here first."""
from fractions import Fraction

import numpy as np
import pytest

from oracle import oracle as O
from tests.ahp_closed_form import ahp_levels_l2


@pytest.mark.parametrize("rule", [0, 1])
def test_levels_form_equals_explicit_matrix(rule):
    rng = np.random.default_rng(17 + rule)
    for trial in range(40):
        m = int(rng.integers(2, 400))
        K = int(rng.integers(1, 30))
        levels = rng.choice(10 ** 6, size=K, replace=False)
        x = levels[rng.integers(0, K, size=m)]
        a = ahp_levels_l2(x, rule)
        b = O.ahp_priority(x.astype(np.float64), rule)
        assert np.allclose(a, b, rtol=1e-11, atol=0), (trial, np.max(np.abs(a - b) / b))
        assert abs(a.sum() - 1) < 1e-12


@pytest.mark.parametrize("n,m", [(16, 1), (1024, 7), (65536, 1), (65536, 3000)])
def test_levels_form_two_level_closed_form(n, m):
    """m servers "high" among n, literal rule: L2 = 9/(9m+n-m) (high), 1/(9m+n-m) (low)
    (derived by hand; e.g. n = 65536, m = 1: 3/21848 and 1/65544)."""
    x = np.zeros(n, np.int64)
    x[:m] = 1
    l2 = ahp_levels_l2(x, 0)
    hi, lo = Fraction(9, 9 * m + n - m), Fraction(1, 9 * m + n - m)
    assert np.allclose(l2[:m], float(hi), rtol=1e-14) and np.allclose(l2[m:], float(lo), rtol=1e-14)
    if (n, m) == (65536, 1):
        assert hi == Fraction(3, 21848) and lo == Fraction(1, 65544)
