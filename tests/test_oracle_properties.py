"""Property-based pins of the oracle (SURVEY.md §4 layers 2-3: hypothesis properties and
metamorphic relations), CPU only.  Each property is fixed by the mathematics, not by the
oracle: brute-force path enumeration, relabelling symmetry, the exact inverse of a commit."""
import numpy as np
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

from inputs import gen
from oracle import oracle as O
from tests.test_oracle_graph import brute_force

SETTINGS = settings(max_examples=40, deadline=None, suppress_health_check=[HealthCheck.too_slow])


@st.composite
def tiny_graphs(draw):
    V = draw(st.integers(2, 7))
    n_links = draw(st.integers(0, 12))
    links = [draw(st.tuples(st.integers(0, V - 1), st.integers(0, V - 1)).filter(lambda t: t[0] != t[1]))
             for _ in range(n_links)]
    res = [draw(st.sampled_from([0, 5, 10, 20])) for _ in range(n_links)]
    i32 = lambda x: np.asarray(x, dtype=np.int32)
    return dict(n_vertices=V, n_servers=V, link_u=i32([a for a, _ in links]), link_v=i32([b for _, b in links]),
                link_res=i32(res))


@SETTINGS
@given(tiny_graphs(), st.sampled_from([0, 7, 15]))
def test_paths_equal_brute_force(g, demand):
    """R26 on any small multigraph: fewest hops, widest, lexicographically smallest path."""
    V = g["n_vertices"]
    src = [s for s in range(V) for t in range(V) if s != t]
    dst = [t for s in range(V) for t in range(V) if s != t]
    bn, hops, path = O.graph_paths(g, src, dst, [demand] * len(src), max_hops=V, nthreads=1)
    for i, (s, t) in enumerate(zip(src, dst)):
        b, h, p = brute_force(g, s, t, demand)
        assert (bn[i], hops[i]) == (b, h)
        assert [x for x in path[i] if x >= 0] == p


@SETTINGS
@given(st.integers(0, 2 ** 31 - 1), st.sampled_from(["topsis", "ahp"]), st.sampled_from(["flat", "network"]))
def test_rank_is_equivariant_under_server_relabelling(seed, method, schema):
    """Without flows the filter and the criteria see each server alone, so permuting the
    servers' rows (CPU, RAM, f_u, access link) permutes feasibility and scores the same way."""
    rng = np.random.default_rng(seed)
    s = gen.snapshot(4, seed=seed % 1000 + 1, quantised=bool(seed & 1))
    perm = rng.permutation(16)
    p = dict(s, cpu_res=s["cpu_res"][perm].copy(), ram_res=s["ram_res"][perm].copy(),
             active=s["active"][perm].copy(), link_res=s["link_res"].copy())
    p["link_res"][:16] = s["link_res"][:16][perm]
    dc, dr = int(rng.integers(1, 12000)), int(rng.integers(1, 150000))
    a = O.rank(s, method, schema, dc, dr)
    b = O.rank(p, method, schema, dc, dr)
    assert np.array_equal(b["mask"], a["mask"][perm])
    assert np.allclose(b["score"], a["score"][perm], rtol=1e-12, atol=1e-15)


@SETTINGS
@given(st.integers(0, 2 ** 31 - 1), st.sampled_from(["topsis", "ahp", "bf", "wf"]))
def test_release_of_a_schedule_is_the_identity(seed, method):
    """Commit + top-up followed by the release of every accepted request restores the state
    word for word, for any batch on a warm DC whose activity flags follow R22."""
    snap = gen.snapshot(4, seed=seed % 997 + 1)
    reqs = gen.requests(12, seed % 991 + 3, nc_hi=8)
    out, _, state = O.schedule(snap, reqs, method, "clustering", sequential=True, nthreads=1)
    back = O.release(state, reqs, out)
    for key in ("cpu_res", "ram_res", "active", "link_res"):
        assert np.array_equal(back[key], snap[key])


@SETTINGS
@given(st.integers(0, 2 ** 31 - 1), st.sampled_from(["topsis", "bf", "wf"]), st.sampled_from([0, 1]))
def test_simulation_conservation(seed, method, hol):
    """Every request is accepted once at most, never before it arrives; attempts add up; the
    queue drains at the last tick; per-tick counts stay within the DC."""
    reqs, arrival, duration = gen.sim_workload(40, seed=seed % 1009 + 1, horizon=12, max_duration=9)
    r = O.simulate(gen.snapshot(2, warm=False), reqs, arrival, duration, method, "flat", max_ticks=300, hol=hol)
    st_ = r["start"]
    acc = st_ >= 0
    assert np.all(st_[acc] >= arrival[acc]) and r["totals"]["accepted"] == acc.sum()
    assert r["totals"]["attempts"] == r["attempts"].sum() and np.all(r["attempts"][acc] >= 1)
    if r["totals"]["events"] < 300:
        assert acc.all() and r["tick_queue"][-1] == 0
    assert np.all(r["tick_servers"] <= 2) and np.all(r["tick_links"] <= 6)
