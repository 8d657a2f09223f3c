"""AHP local priorities of a criterion with repeated values, from its distinct levels only
(SURVEY.md §8(c) "AHP", the quantised K-level closed form) — an independent formula used
to pin the GPU at full C5 scale, where the oracle's explicit |F| x |F| matrix is too slow.

Derivation (readings R7-R9).  With values x_i over F (|F| = m), hi > lo and
c = 9 / (hi - lo), the cell is a_ij = f(c (x_i - x_j)).  A cell depends only on the two
values, so with distinct levels v_0 < ... < v_{K-1} of multiplicities m_l:

    colsum(level l) = sum_k m_k f(c (v_k - v_l))                       (column j at level l)
    L2(level k)     = (1/m) sum_l m_l f(c (v_k - v_l)) / colsum(l)      (row i at level k)

f is R8's literal rule (d, 1/(-d), 1) or the shifted rule (1+d, 1/(1-d), 1).  hi = lo
gives 1/m everywhere (every cell 1).  Evaluated in float64 as a K x K matrix.
"""
from __future__ import annotations

import numpy as np


def cell(d: np.ndarray, rule: int) -> np.ndarray:
    d = np.asarray(d, np.float64)
    out = np.ones_like(d)
    pos, neg = d > 0, d < 0
    if rule == 0:
        out[pos] = d[pos]
        out[neg] = 1.0 / (-d[neg])
    else:
        out[pos] = 1.0 + d[pos]
        out[neg] = 1.0 / (1.0 - d[neg])
    return out


def ahp_levels_l2(x: np.ndarray, rule: int = 0) -> np.ndarray:
    """L2 of every element of x (int64 values) via the level form."""
    x = np.asarray(x, np.int64)
    m = x.size
    v, inv, cnt = np.unique(x, return_inverse=True, return_counts=True)
    if v.size == 1:
        return np.full(m, 1.0 / m)
    c = 9.0 / float(v[-1] - v[0])
    A = cell(c * (v[:, None] - v[None, :]).astype(np.float64), rule)  # A[k, l] = f(c (v_k - v_l))
    colsum = (cnt[:, None] * A).sum(axis=0)
    l2 = (A * (cnt / colsum)[None, :]).sum(axis=1) / m
    return l2[inv]
