"""Pins of the oracle's commit phase (readings R17, R18, R19; SURVEY §8(c) steps 2.1, 2.6
and 3) against hand-worked k=4 cases (tests/commit_cases.py: every expected value is
derived by hand in the case's docstring, not computed by the oracle).

R17 "flows": P:384 routes "each ... source and destination pair", the paper is silent on
    pods sharing a server; R17 aggregates per hosting server.
R18 "commit failure": P:383 routes after selection; R18 excludes and redoes.
R19 "allocation amounts": "mixing between the maximum and minimum requirements" P:456;
    DESIGN.md R19 tops up in container, then vlink, index order, bounded by the path minimum.
"""
import numpy as np
import pytest

from oracle import oracle as O
from tests import commit_cases as CC


@pytest.mark.parametrize("case", sorted(CC.CASES))
@pytest.mark.parametrize("method", ["ahp", "topsis"])
def test_commit_pin_sequential(case, method):
    snap, req, expect = CC.CASES[case]()
    out, cnt, state = O.schedule(snap, req, method, "flat", sequential=True)
    CC.check(expect, out, state, cnt["retries"], f"{case} {method}")


@pytest.mark.parametrize("case", sorted(CC.CASES))
def test_commit_pin_batch_same_placement(case):
    """Batch mode (R21) runs the same pod steps on a private overlay: same placement, the
    snapshot unchanged."""
    snap, req, expect = CC.CASES[case]()
    out, cnt, state = O.schedule(snap, req, "topsis", "flat", sequential=False)
    CC.check(expect, out, None, cnt["retries"], case)
    for key in ("cpu_res", "ram_res", "link_res", "active"):
        assert np.array_equal(state[key], snap[key])


def test_r17_is_one_flow_per_server_in_the_filter():
    """R17 in the filter (step 2.2): with the 800 path cut to 650 no single path carries the
    aggregated 700, so pod 2 has no feasible server and the request is rejected — although
    each vlink alone (300, 400) would fit a 650 path."""
    snap, req, _ = CC.r17_case()
    for l in CC.cross_path_links(0, 7, 1, 1):
        snap["link_res"][l] = 650
    out, cnt, state = O.schedule(snap, req, "topsis", "flat", sequential=True)
    assert out["status"][0] == 0 and cnt["pod_steps"] == 3
    assert np.array_equal(state["link_res"], snap["link_res"])
    r = O.rank(snap, "topsis", "flat", 5000, 100, flows=[(0, 700)])
    assert r["best"] == -1 and r["n_feasible"] == 0
    r = O.rank(snap, "topsis", "flat", 5000, 100, flows=[(0, 400)])
    assert r["best"] == 15


def test_r18_exhausting_f_rejects():
    """R18 + R20: when the only other candidate is removed, the exclusion empties F and the
    request is rejected atomically after two pod-2 attempts."""
    snap, req, _ = CC.r18_case()
    snap["cpu_res"][4] = 0
    out, cnt, state = O.schedule(snap, req, "ahp", "flat", sequential=True)
    assert out["status"][0] == 0 and cnt["retries"] == 1 and cnt["pod_steps"] == 4
    for key in ("cpu_res", "ram_res", "link_res", "active"):
        assert np.array_equal(state[key], snap[key])
