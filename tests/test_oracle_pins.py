"""Pins of the CPU oracle against things other than itself (CPU only, no GPU).

Each pin names what fixes the expected value: a closed form derived by hand
from the paper's definitions, a value printed in the paper, a value computed
independently by the surveyor, an invariant, or brute force
on an explicit graph.
"""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

from inputs import gen
from oracle import oracle as O
from oracle import milp

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def state_with_rows(rows, k=4):
    """A k=4 DC whose servers 0..len(rows)-1 carry `rows` and whose other servers have no CPU
    (so a CPU demand of 1 makes exactly the listed servers feasible)."""
    s = gen.snapshot(k, warm=False)
    for u, (c, r, a, b) in enumerate(rows):
        s["cpu_res"][u], s["ram_res"][u], s["active"][u], s["link_res"][u] = c, r, a, b
    for u in range(len(rows), k ** 3 // 4):
        s["cpu_res"][u] = 0
        s["active"][u] = 1
    return s


# ---------------------------------------------------------------- fat-tree ----
@pytest.mark.parametrize("k,n,sw,L", [(2, 2, 5, 6), (4, 16, 20, 48), (8, 128, 80, 384)])
def test_fat_tree_counts(k, n, sw, L):
    # |N^s| = k^3/4 (§IV-B1); 5k^2/4 switches and 3k^3/4 links (SPEC.md:65-67 for k=4)
    links = milp.fat_tree_links(k)
    nodes = {x for l in links for x in l}
    assert sum(1 for x in nodes if x[0] == "srv") == n == gen.sizes(k)["n"]
    assert sum(1 for x in nodes if x[0] != "srv") == sw
    assert len(links) == L == gen.sizes(k)["L"]
    assert gen.sizes(20)["n"] == 2000  # PAPER.md:396 §VI-A


@pytest.mark.parametrize("k", [4, 8])
def test_widest_path_matches_exhaustive_enumeration(k):
    """R16: the closed-form widest ECMP path equals BFS enumeration of all shortest paths
    of the explicit graph (max fabric bottleneck, hop count)."""
    rng = np.random.default_rng(7 + k)
    n = k ** 3 // 4
    L = 3 * k ** 3 // 4
    link = rng.integers(0, 1000, size=L).astype(np.int32)
    for _ in range(150):
        u, v = rng.choice(n, 2, replace=False)
        pid, fab, links = O.widest_path(k, link, int(u), int(v))
        paths = milp.shortest_paths(k, int(u), int(v))
        # the fabric bottleneck ignores the two access links u, v
        best = max(min([link[l] for l in p if l not in (u, v)], default=1e300) for p in paths)
        assert fab == best
        assert len(links) + 2 == len(paths[0])
        chosen = [p for p in paths if set(l for l in p if l not in (u, v)) == set(links)]
        assert len(chosen) == 1
    # ECMP counts: k/2 inside a pod, (k/2)^2 across pods
    h = k // 2
    assert len(milp.shortest_paths(k, 0, h)) == h          # same pod, other edge switch
    assert len(milp.shortest_paths(k, 0, n - 1)) == h * h  # other pod


@pytest.mark.parametrize("k", [4, 6])
def test_filter_matches_brute_force_paths(k):
    """a3 / R6: u is feasible iff it fits CPU/RAM and, for every flow (v, D) with v != u, some
    shortest path in the explicit graph has every link >= D, and u's access link carries sum D."""
    rng = np.random.default_rng(11 + k)
    n = k ** 3 // 4
    for trial in range(6):
        s = gen.snapshot(k, seed=100 + trial)
        s["link_res"] = rng.integers(0, 60, size=len(s["link_res"])).astype(np.int32)
        nf = int(rng.integers(1, 4))
        vs = rng.choice(n, nf, replace=False)
        flows = [(int(v), int(rng.integers(1, 40))) for v in vs]
        r = O.rank(s, "topsis", "flat", 1000, 1000, flows)
        for u in range(n):
            ok = s["cpu_res"][u] >= 1000 and s["ram_res"][u] >= 1000
            ok = ok and s["link_res"][u] >= sum(D for v, D in flows if v != u)
            for v, D in flows:
                if v == u:
                    continue
                paths = milp.shortest_paths(k, u, v)
                ok = ok and any(all(s["link_res"][l] >= D for l in p) for p in paths)
            assert bool(r["mask"][u]) == ok, (trial, u)


# --------------------------------------------------------------------- AHP ----
def test_ahp_all_equal_is_uniform():
    # hi == lo: every scaled value is 1, every cell 1 => L2 = 1/m (R7)
    assert np.allclose(O.ahp_priority([5, 5, 5, 5, 5]), 0.2, rtol=0, atol=1e-15)


@pytest.mark.parametrize("n,m", [(16, 1), (16, 15), (100, 7), (1024, 1), (1024, 300)])
def test_ahp_two_level_closed_form(n, m):
    """Hand-derived from R7-R9: with m servers at the high value and n-m at the low one, the
    scaled difference is +-9 so L2(high) = 9/(9m+n-m) and L2(low) = 1/(9m+n-m)."""
    x = np.array([7.0] * m + [3.0] * (n - m))
    L2 = O.ahp_priority(x)
    assert np.allclose(L2[:m], 9 / (9 * m + n - m), rtol=1e-12, atol=0)
    assert np.allclose(L2[m:], 1 / (9 * m + n - m), rtol=1e-12, atol=0)


def test_ahp_invariants_random():
    rng = np.random.default_rng(3)
    for rule in (0, 1):
        for _ in range(200):
            m = int(rng.integers(2, 40))
            x = rng.integers(0, 50, size=m).astype(float)
            L = O.ahp_priority(x, rule)
            assert abs(L.sum() - 1) < 1e-12 and (L > 0).all()
            # affine invariance of the [1,10] scaling (R7): x -> a x + b, a > 0
            a, b = float(rng.uniform(0.1, 10)), float(rng.uniform(-100, 100))
            assert np.allclose(O.ahp_priority(a * x + b, rule), L, rtol=1e-9, atol=1e-15)
            # relabelling alternatives permutes priorities
            perm = rng.permutation(m)
            assert np.allclose(O.ahp_priority(x[perm], rule), L[perm], rtol=1e-12, atol=1e-15)


def test_ahp_literal_rule_nonmonotone_example():
    # CPU residuals [0, 1, 24] cores give L2 = 0.135, 0.071, 0.795 under the
    # literal rule and 0.076, 0.095, 0.829 under the shifted rule.
    assert np.allclose(O.ahp_priority([0, 1, 24], 0), [0.135, 0.071, 0.795], atol=5e-4)
    assert np.allclose(O.ahp_priority([0, 1, 24], 1), [0.076, 0.095, 0.829], atol=5e-4)


def test_ahp_l1_values():
    g = json.load(open(os.path.join(GOLDEN, "survey_4server.json")))
    assert np.allclose(O.ahp_l1("flat"), 0.25, rtol=0, atol=1e-15)
    lit = g["l1_clustering_literal"]
    exp = np.array(lit["numerators"], float) / lit["denominator"]
    assert np.allclose(O.ahp_l1("clustering"), exp, rtol=1e-12)
    # Network is Clustering with the last two criteria swapped (T4 P:322-326)
    assert np.allclose(O.ahp_l1("network"), exp[[0, 1, 3, 2]], rtol=1e-12)
    sh = g["l1_clustering_shifted"]
    assert np.allclose(O.ahp_l1("clustering", ahp_rule=1), sh["values"], atol=1e-6)
    assert np.allclose(O.ahp_l1("clustering", l1_mode=1), [0.17, 0.17, 0.5, 0.16], rtol=0, atol=0)


def _worked_state():
    """SURVEY.md §8(c) worked example: a fresh k=4 DC after one pod (1500 mc, 3072 MiB) on server 0."""
    s = gen.snapshot(4, warm=False)
    s["cpu_res"][0] -= 1500
    s["ram_res"][0] -= 3072
    s["active"][0] = 1
    return s


def test_ahp_worked_example_closed_form():
    """Two-level closed forms per criterion (n=16): CPU, RAM: m=15 high -> 9/136, 1/136;
    Fragmentation: m=1 high -> 3/8, 1/24; Bandwidth: all equal -> 1/16.  Flat L1 = 1/4 gives
    PG[0] = 123/1088 and PG[u!=0] = 193/3264."""
    r = O.rank(_worked_state(), "ahp", "flat", 100, 100)
    assert r["best"] == 0
    pg0 = Fraction(1, 4) * (Fraction(1, 136) * 2 + Fraction(3, 8) + Fraction(1, 16))
    pgu = Fraction(1, 4) * (Fraction(9, 136) * 2 + Fraction(1, 24) + Fraction(1, 16))
    assert pg0 == Fraction(123, 1088) and pgu == Fraction(193, 3264)
    assert math.isclose(r["score"][0], float(pg0), rel_tol=1e-13)
    assert np.allclose(r["score"][1:], float(pgu), rtol=1e-13)
    assert abs(r["score"].sum() - 1) < 1e-13


# ------------------------------------------------------------------ TOPSIS ----
def test_topsis_identical_servers_all_zero():
    # identical rows => A+ = A- => Ed+ = Ed- = 0 => closeness 0 (R13)
    r = O.rank(gen.snapshot(4, warm=False), "topsis", "flat", 100, 100)
    assert (r["score"] == 0).all() and r["best"] == 0 and r["tie"].all()


def test_topsis_dominance_one_zero():
    # a server better on every criterion is the ideal point (1) and the other the anti-ideal (0)
    s = state_with_rows([(20000, 200000, 1, 900), (10000, 100000, 0, 400)])
    r = O.rank(s, "topsis", "clustering", 1, 1)
    assert r["score"][0] == 1.0 and r["score"][1] == 0.0 and r["best"] == 0


@pytest.mark.parametrize("schema,expected", [("flat", 0.984294471), ("clustering", 0.994604189),
                                             ("network", 0.983329239)])
def test_topsis_worked_example(schema, expected):
    """Two-level TOPSIS closed form: server 0 is the anti-ideal on CPU and RAM and the ideal on
    Fragmentation (Bandwidth equal), so Rank_0 = dF / (dF + sqrt(dC^2 + dR^2)) and every other
    server has 1 - Rank_0; values printed in SURVEY.md §8(c)."""
    w = O.SCHEMAS[schema]
    n = 16
    NC = math.sqrt(22500 ** 2 + (n - 1) * 24000 ** 2)
    NR = math.sqrt(259072 ** 2 + (n - 1) * 262144 ** 2)
    dC = w[0] * (24000 - 22500) / NC
    dR = w[1] * (262144 - 259072) / NR
    dF = w[2] * 1.0 / 1.0  # ||f|| = 1: only server 0 is active
    r0 = dF / (dF + math.sqrt(dC * dC + dR * dR))
    assert abs(r0 - expected) < 1e-9
    r = O.rank(_worked_state(), "topsis", schema, 100, 100)
    assert math.isclose(r["score"][0], r0, rel_tol=1e-12)
    assert np.allclose(r["score"][1:], 1 - r0, rtol=1e-11)


def test_topsis_invariants_random():
    rng = np.random.default_rng(5)
    for _ in range(60):
        s = gen.snapshot(4, seed=int(rng.integers(1 << 30)))
        for schema in ("flat", "clustering", "network"):
            r = O.rank(s, "topsis", schema, 1000, 1000)
            F = r["mask"].astype(bool)
            sc = r["score"][F]
            assert ((sc >= 0) & (sc <= 1)).all()
            # scale invariance (vector normalisation): x_c -> a x_c leaves closeness unchanged
            s2 = dict(s, ram_res=(s["ram_res"] // 2 * 2).astype(np.int32))
            r2 = O.rank(s2, "topsis", schema, 1000, 1000)
            s3 = dict(s2, ram_res=(s2["ram_res"] // 2).astype(np.int32))
            r3 = O.rank(s3, "topsis", schema, 1000, 500)
            assert np.array_equal(r2["mask"], r3["mask"])
            assert np.allclose(r2["score"], r3["score"], rtol=1e-12, atol=1e-15)


def test_topsis_monotone_in_one_criterion():
    """Increasing one server's value on one (benefit) criterion never lowers its rank position."""
    rng = np.random.default_rng(9)
    viol = 0
    for _ in range(300):
        rows = [(int(rng.integers(1, 24000)), int(rng.integers(1, 262144)), int(rng.integers(0, 2)),
                 int(rng.integers(1, 1000))) for _ in range(int(rng.integers(2, 8)))]
        s = state_with_rows(rows)
        r = O.rank(s, "topsis", "flat", 1, 1)
        pos = lambda sc, i: int(np.sum(sc[: len(rows)] > sc[i]))
        i = int(rng.integers(len(rows)))
        s2 = state_with_rows(rows)
        s2["cpu_res"][i] = min(24000, s2["cpu_res"][i] + int(rng.integers(1, 5000)))
        r2 = O.rank(s2, "topsis", "flat", 1, 1)
        viol += pos(r2["score"], i) > pos(r["score"], i)
    assert viol == 0


# ---------------------------------------------------------- golden vectors ----
def test_survey_golden_vectors():
    g = json.load(open(os.path.join(GOLDEN, "survey_4server.json")))
    s = state_with_rows(g["rows"])
    for case in g["cases"]:
        r = O.rank(s, case["method"], case["schema"], 1, 1, ahp_rule=case["ahp_rule"])
        assert r["n_feasible"] == 4
        got = r["score"][:4]
        assert np.allclose(got, case["scores"], rtol=0, atol=1.5 * 10.0 ** -g["digits"]), case
        assert r["best"] == case["argmax"]
        if case["method"] == "ahp":
            assert abs(got.sum() - 1) < 1e-12


def test_ahp_exact_rationals_small():
    """Extra check in exact arithmetic (fractions) of R7-R11 on random small cases."""
    rng = np.random.default_rng(21)
    for _ in range(20):
        m = int(rng.integers(2, 9))
        x = [int(v) for v in rng.integers(0, 30, size=m)]
        lo, hi = min(x), max(x)
        if lo == hi:
            continue

        def cell(i, j):
            d = Fraction(9 * (x[i] - x[j]), hi - lo)
            return d if d > 0 else (1 / (-d) if d < 0 else Fraction(1))
        col = [sum(cell(i, j) for i in range(m)) for j in range(m)]
        L = [sum(cell(i, j) / col[j] for j in range(m)) / m for i in range(m)]
        assert np.allclose(O.ahp_priority(x), [float(v) for v in L], rtol=1e-13)


# ---------------------------------------------------------- placement ---------
def test_fresh_dc_first_pod_on_server_0():
    s = gen.snapshot(8, warm=False)
    req = gen.requests(1, 123)
    for m in ("ahp", "topsis"):
        out, cnt, _ = O.schedule(s, req, m, "flat", sequential=True)
        assert out["status"][0] == 1 and out["server_of_container"][0] == 0


def _request(cpu, ram, pods, vlinks=()):
    """One CSR request: per-container (cpu, ram) with c^min = c^max, pod ids, vlinks (src, dst, bw)."""
    nC, nV = len(cpu), len(vlinks)
    i32 = lambda x: np.asarray(x, np.int32)
    return {"n_requests": 1, "container_off": i32([0, nC]), "cpu_min": i32(cpu), "cpu_max": i32(cpu),
            "ram_min": i32(ram), "ram_max": i32(ram), "pod_of": i32(pods), "vlink_off": i32([0, nV]),
            "vl_src": i32([v[0] for v in vlinks]), "vl_dst": i32([v[1] for v in vlinks]),
            "bw_min": i32([v[2] for v in vlinks]), "bw_max": i32([v[2] for v in vlinks])}


def test_rank_once_fresh_dc_colocates_on_rank_1():
    """R25: a request that fits on the rank-1 server goes there
    whole: on a fresh DC every server scores the same, server 0 is first in the order and stays
    admissible for every pod."""
    s = gen.snapshot(4, warm=False)
    req = _request([1000, 1500, 800, 1200, 900], [1024, 2048, 512, 1024, 4096], [0, 0, 1, 2, 2],
                   [(0, 2, 10), (2, 3, 5), (1, 4, 20)])
    for m in ("ahp", "topsis"):
        out, _, state = O.schedule(s, req, m, "flat", sequential=True, rank_once=True)
        assert out["status"][0] == 1 and (out["server_of_container"] == 0).all()
        assert (out["path_of_vlink"] == -1).all() and (out["bw_alloc"] == [10, 5, 20]).all()
        assert state["cpu_res"][0] == 24000 - 5400


def test_rank_once_walks_the_order_across_a_dominating_class():
    """R25 on two server classes: A (servers 0-3) dominates B in every criterion, so the order is
    A by index, then B (TOPSIS closeness 1 / 0, AHP by dominance).  Six single-container pods of
    2000 mc walk it first-fit: each A server takes two pods (5000 mc), in index order."""
    s = gen.snapshot(4, warm=False)
    for u in range(16):
        a = u < 4
        s["cpu_res"][u], s["ram_res"][u] = (5000, 50000) if a else (3000, 30000)
        s["active"][u] = 1 if a else 0
        s["link_res"][u] = 1000 if a else 500
    req = _request([2000] * 6, [1000] * 6, list(range(6)))
    for m in ("ahp", "topsis"):
        out, _, _ = O.schedule(s, req, m, "flat", sequential=True, rank_once=True)
        assert out["server_of_container"].tolist() == [0, 0, 1, 1, 2, 2], m


@pytest.mark.parametrize("method", ["ahp", "topsis"])
def test_rank_once_equals_per_pod_for_single_pod_requests(method):
    """With one pod per request the first pod step's order is the only ranking: R25 = R15."""
    snap, reqs = gen.config("C2")
    one = dict(reqs, pod_of=np.zeros_like(reqs["pod_of"]))
    a, _, sa = O.schedule(snap, one, method, "network", sequential=True)
    b, _, sb = O.schedule(snap, one, method, "network", sequential=True, rank_once=True)
    for key in a:
        assert np.array_equal(a[key], b[key]), key
    for key in ("cpu_res", "ram_res", "link_res"):
        assert np.array_equal(sa[key], sb[key])


@pytest.mark.parametrize("method", ["ahp", "topsis"])
def test_rank_once_invariants(method):
    snap, reqs = gen.config("C2")
    out, _, state = O.schedule(snap, reqs, method, "flat", sequential=True, rank_once=True)
    _check_invariants(snap, reqs, out, state, sequential=True)
    outb, _, stb = O.schedule(snap, reqs, method, "flat", sequential=False, rank_once=True)
    _check_invariants(snap, reqs, outb, stb, sequential=False)


@pytest.mark.parametrize("alpha", [0.0, 0.5, 1.0])
def test_c1_heuristic_is_milp_optimal(alpha):
    """SURVEY.md §8(c) C1 expectation: both methods and all schemas put the 3 pods on server 0,
    which attains the MILP optimum (1-alpha)/16 (one active server, no active link)."""
    snap, req = gen.config("C1")
    opt, assign = milp.milp_optimum(snap, req, alpha)
    assert math.isclose(opt, (1 - alpha) / 16, abs_tol=1e-12)
    for m in ("ahp", "topsis"):
        for schema in ("flat", "clustering", "network"):
            out, _, _ = O.schedule(snap, req, m, schema, sequential=True)
            assert (out["server_of_container"] == 0).all()
            val = milp.placement_objective(snap, req, out, alpha)
            assert math.isclose(val, opt, abs_tol=1e-12)


def test_milp_bound_on_warm_k2():
    """On tiny warm fat-trees (k=2, 2 servers) the heuristic's Eq.3 value is never below the
    brute-force optimum (sanity of both)."""
    for seed in range(8):
        s = gen.snapshot(2, seed=seed)
        s["link_res"][:] = 1000
        req = gen.requests(1, 500 + seed, nc_lo=2, nc_hi=3)
        for m in ("ahp", "topsis"):
            out, _, _ = O.schedule(s, req, m, "flat", sequential=True)
            if out["status"][0] != 1:
                continue
            for alpha in (0.0, 0.5, 1.0):
                opt, _ = milp.milp_optimum(s, req, alpha)
                assert milp.placement_objective(s, req, out, alpha) >= opt - 1e-12


def _check_invariants(snap, reqs, out, state, sequential):
    k = snap["k"]
    h, n, E = k // 2, k ** 3 // 4, k * k // 2
    co, vo = reqs["container_off"], reqs["vlink_off"]
    used_cpu = np.zeros(n, np.int64)
    used_ram = np.zeros(n, np.int64)
    used_link = np.zeros(3 * k ** 3 // 4, np.int64)
    for r in range(reqs["n_requests"]):
        cs, vs = slice(co[r], co[r + 1]), slice(vo[r], vo[r + 1])
        srv = out["server_of_container"][cs]
        if out["status"][r] != 1:
            assert (srv == -1).all() and (out["path_of_vlink"][vs] == -1).all()
            continue
        assert (srv >= 0).all()
        pods = reqs["pod_of"][cs]
        for p in set(pods.tolist()):
            assert len(set(srv[pods == p].tolist())) == 1  # Eq. 8 pod integrity
        assert ((out["cpu_alloc"][cs] >= reqs["cpu_min"][cs]) & (out["cpu_alloc"][cs] <= reqs["cpu_max"][cs])).all()
        assert ((out["ram_alloc"][cs] >= reqs["ram_min"][cs]) & (out["ram_alloc"][cs] <= reqs["ram_max"][cs])).all()
        assert ((out["bw_alloc"][vs] >= reqs["bw_min"][vs]) & (out["bw_alloc"][vs] <= reqs["bw_max"][vs])).all()
        np.add.at(used_cpu, srv, out["cpu_alloc"][cs])
        np.add.at(used_ram, srv, out["ram_alloc"][cs])
        for e in range(vo[r], vo[r + 1]):
            u = srv[reqs["vl_src"][e] - 0]
            v = srv[reqs["vl_dst"][e]]
            pid = out["path_of_vlink"][e]
            bw = out["bw_alloc"][e]
            if u == v:
                assert pid == -1 and bw == reqs["bw_max"][e]
                continue
            eu, ev = u // h, v // h
            if eu == ev:
                assert pid == 0
                links = []
            elif eu // h == ev // h:
                assert 1 <= pid <= h
                a = pid - 1
                links = [n + eu * h + a, n + ev * h + a]
            else:
                assert pid > h
                a, b = divmod(pid - 1 - h, h)
                links = [n + eu * h + a, n + ev * h + a, n + E * h + ((eu // h) * h + a) * h + b,
                         n + E * h + ((ev // h) * h + a) * h + b]
            for l in [u, v] + links:
                used_link[l] += bw
        if not sequential:
            pass
    if sequential:
        # exact integer conservation: residual + allocated = initial residual
        assert np.array_equal(state["cpu_res"].astype(np.int64) + used_cpu, snap["cpu_res"].astype(np.int64))
        assert np.array_equal(state["ram_res"].astype(np.int64) + used_ram, snap["ram_res"].astype(np.int64))
        assert np.array_equal(state["link_res"].astype(np.int64) + used_link, snap["link_res"].astype(np.int64))
        assert (state["cpu_res"] >= 0).all() and (state["ram_res"] >= 0).all() and (state["link_res"] >= 0).all()
        hosting = used_cpu > 0
        assert (state["active"][hosting] == 1).all()
        assert np.array_equal(state["active"].astype(bool), hosting | snap["active"].astype(bool))
    else:
        for key in ("cpu_res", "ram_res", "link_res", "active"):
            assert np.array_equal(state[key], snap[key])


@pytest.mark.parametrize("method", ["ahp", "topsis"])
@pytest.mark.parametrize("schema", ["flat", "clustering", "network"])
def test_c2_sequential_invariants(method, schema):
    snap, reqs = gen.config("C2")
    out, cnt, state = O.schedule(snap, reqs, method, schema, sequential=True)
    assert cnt["pod_steps"] >= int(sum(reqs["pod_of"][reqs["container_off"][r]:reqs["container_off"][r + 1]].max() + 1
                                       for r in range(reqs["n_requests"])) * 0)
    _check_invariants(snap, reqs, out, state, sequential=True)


def test_tight_links_exercise_retries_and_rejections():
    """A congested fabric makes flows compete for links: commits must stay exact (R18) and
    rejections atomic (R20)."""
    snap = gen.snapshot(4, seed=77)
    snap["link_res"] = np.random.default_rng(1).integers(0, 80, size=48).astype(np.int32)
    reqs = gen.requests(60, 78, bw_max_hi=60)
    out, cnt, state = O.schedule(snap, reqs, "topsis", "network", sequential=True)
    _check_invariants(snap, reqs, out, state, sequential=True)
    assert (out["status"] == 0).any()


def test_batch_is_snapshot_isolated_and_equals_single_sequential():
    snap, reqs = gen.config("C2")
    outb, cntb, stb = O.schedule(snap, reqs, "topsis", "flat", sequential=False)
    _check_invariants(snap, reqs, outb, stb, sequential=False)
    for r in (0, 17, 63):
        one = gen.subset(reqs, [r])
        outs, _, _ = O.schedule(snap, one, "topsis", "flat", sequential=True)
        cs = slice(reqs["container_off"][r], reqs["container_off"][r + 1])
        assert np.array_equal(outs["server_of_container"], outb["server_of_container"][cs])
        assert outs["status"][0] == outb["status"][r]


def test_rejection_is_atomic():
    snap = gen.snapshot(4, seed=3)
    req = gen.requests(1, 4)
    req["cpu_min"][:] = 30000  # no server has 30 cores: first pod step has F empty
    req["cpu_max"][:] = 30000
    out, cnt, state = O.schedule(snap, req, "ahp", "flat", sequential=True)
    assert out["status"][0] == 0 and cnt["pod_steps"] == 1
    for key in ("cpu_res", "ram_res", "link_res", "active"):
        assert np.array_equal(state[key], snap[key])


def test_invalid_request_status():
    snap = gen.snapshot(4, seed=3)
    req = gen.requests(2, 4)
    req["cpu_min"][0] = req["cpu_max"][0] + 1  # c_min > c_max
    out, cnt, _ = O.schedule(snap, req, "topsis", "flat", sequential=True)
    assert out["status"][0] == -1 and out["status"][1] == 1
