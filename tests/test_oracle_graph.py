"""Pins of the oracle's general-topology modified Dijkstra (P:383-386
§V-D, reading R26) and of the logical-bandwidth criterion (R2 alternative), CPU only.

Each expected value comes from something other than the oracle's Dijkstra: exhaustive
enumeration of every simple path (tiny graphs), SPEC's worked examples,
scipy's unweighted BFS (hop counts), or the fat-tree closed form (R16), itself pinned by
BFS enumeration in test_oracle_pins.py.
"""
import numpy as np
import pytest
from scipy.sparse import csr_matrix
from scipy.sparse.csgraph import shortest_path

from inputs import gen
from oracle import oracle as O
from oracle import milp


def brute_force(graph, src, dst, demand):
    """Every simple path src -> dst over links with residual >= demand; the best by
    (hops, -bottleneck, vertex sequence).  Returns (bottleneck, hops, path) or (-1, -1, [])."""
    V = graph["n_vertices"]
    adj = [[] for _ in range(V)]
    for u, v, r in zip(graph["link_u"], graph["link_v"], graph["link_res"]):
        if r >= demand:
            adj[u].append((v, r))
            adj[v].append((u, r))
    best = None

    def dfs(path, width, seen):
        nonlocal best
        x = path[-1]
        if x == dst:
            key = (len(path) - 1, -width, tuple(path))
            if best is None or key < best:
                best = key
            return
        for y, r in adj[x]:
            if y not in seen:
                seen.add(y)
                path.append(y)
                dfs(path, min(width, r), seen)
                path.pop()
                seen.discard(y)

    dfs([src], float("inf"), {src})
    if best is None:
        return -1, -1, []
    return int(-best[1]), best[0], list(best[2])


def tiny_graph(rng, V, n_links, levels=(0, 10, 20, 30)):
    """Random multigraph (no self-loops, parallel links allowed), residuals from a small set
    so that hop and width ties are common."""
    lu, lv = [], []
    while len(lu) < n_links:
        a, b = rng.integers(0, V, 2)
        if a != b:
            lu.append(a)
            lv.append(b)
    res = rng.choice(levels, size=n_links)
    i32 = lambda x: np.asarray(x, dtype=np.int32)
    return dict(n_vertices=V, n_servers=V, link_u=i32(lu), link_v=i32(lv), link_res=i32(res))


@pytest.mark.parametrize("seed", range(6))
def test_paths_equal_exhaustive_enumeration(seed):
    """Fewest hops, then widest, then lexicographically smallest vertex sequence (R26)
    = the minimum over every simple path."""
    rng = np.random.default_rng(100 + seed)
    V = int(rng.integers(4, 9))
    g = tiny_graph(rng, V, int(rng.integers(V, 2 * V + 3)))
    src, dst, dem = [], [], []
    for s in range(V):
        for t in range(V):
            if s != t:
                for d in (0, 15, 25):
                    src.append(s), dst.append(t), dem.append(d)
    bn, hops, path = O.graph_paths(g, src, dst, dem)
    for q in range(len(src)):
        b, h, p = brute_force(g, src[q], dst[q], dem[q])
        assert (bn[q], hops[q]) == (b, h), (seed, src[q], dst[q], dem[q])
        assert [x for x in path[q] if x >= 0] == p


def test_spec_examples():
    """fresh k=4 fat-tree, servers under one edge switch, demand 50 -> 2 hops,
    bottleneck 1000; demand 2000 -> infeasible; a diamond picks the higher-residual side."""
    g = gen.fat_tree_graph(gen.snapshot(4, warm=False))
    bn, hops, path = O.graph_paths(g, [0, 0], [1, 1], [50, 2000])
    assert (bn[0], hops[0]) == (1000, 2)
    assert (bn[1], hops[1]) == (-1, -1) and np.all(path[1] == -1)
    # diamond 0-1-3, 0-2-3: the side through 2 has more residual
    d = dict(n_vertices=4, n_servers=4, link_u=np.int32([0, 1, 0, 2]), link_v=np.int32([1, 3, 2, 3]),
             link_res=np.int32([100, 100, 300, 250]))
    bn, hops, path = O.graph_paths(d, [0, 3], [3, 0], [0, 0])
    assert (bn[0], hops[0], list(path[0][:3])) == (250, 2, [0, 2, 3])
    assert (bn[1], hops[1], list(path[1][:3])) == (250, 2, [3, 2, 0])  # undirected


def test_fat_tree_graph_matches_explicit_links():
    """gen.fat_tree_graph numbers the same links as milp.fat_tree_links (canonical order)."""
    for k in (2, 4, 6):
        g = gen.fat_tree_graph(gen.snapshot(k, warm=False))
        s = gen.sizes(k)
        n, E, h = s["n"], s["E"], s["h"]

        def vid(x):
            if x[0] == "srv":
                return x[1]
            if x[0] == "edge":
                return n + x[1]
            if x[0] == "agg":
                return n + E + x[1] * h + x[2]
            return n + E + k * h + x[1] * h + x[2]

        links = milp.fat_tree_links(k)
        assert [(vid(a), vid(b)) for a, b in links] == list(zip(g["link_u"].tolist(), g["link_v"].tolist()))
        assert g["n_vertices"] == n + 5 * k * k // 4


@pytest.mark.parametrize("k", [4, 8])
def test_fat_tree_equals_closed_form(k):
    """On a fat-tree the general Dijkstra (every link usable) has the ECMP hop count 2 / 4 / 6
    and the bottleneck min(access u, access v, widest fabric) of the closed form R16."""
    snap = gen.snapshot(k, 11 + k)
    g = gen.fat_tree_graph(snap)
    h, n = k // 2, k ** 3 // 4
    rng = np.random.default_rng(k)
    src = rng.integers(0, n, 200)
    dst = (src + rng.integers(1, n, 200)) % n
    bn, hops, path = O.graph_paths(g, src, dst, np.zeros(200, np.int32))
    link = snap["link_res"]
    for q in range(200):
        u, v = int(src[q]), int(dst[q])
        _, fab, _ = O.widest_path(k, link, u, v)
        exp_h = 2 if u // h == v // h else (4 if u // (h * h) == v // (h * h) else 6)
        assert hops[q] == exp_h
        assert bn[q] == min(link[u], link[v], fab)


def test_hops_equal_scipy_bfs():
    """Hop counts at the paper's DC size (k=20) equal scipy's unweighted shortest paths
    on the subgraph of usable links (residual >= demand)."""
    snap = gen.snapshot(20, 7)
    g = gen.fat_tree_graph(snap)
    q = gen.path_queries(g, 60, 3, bw_hi=900)   # large demands: some shortest paths blocked
    bn, hops, path = O.graph_paths(g, q["src"], q["dst"], q["demand"], max_hops=16)
    V = g["n_vertices"]
    for d in np.unique(q["demand"]):
        keep = g["link_res"] >= d
        m = csr_matrix((np.ones(keep.sum()), (g["link_u"][keep], g["link_v"][keep])), shape=(V, V))
        sel = np.nonzero(q["demand"] == d)[0]
        dist = shortest_path(m, directed=False, unweighted=True, indices=q["src"][sel])
        for i, qi in enumerate(sel):
            t = dist[i, q["dst"][qi]]
            assert hops[qi] == (-1 if np.isinf(t) else int(t))
    assert (hops == -1).any() and (hops > 0).any()  # blocked and routed queries both occur


@pytest.mark.parametrize("seed", range(3))
def test_path_invariants_random_dc(seed):
    """Returned paths are simple, run over usable links, start at src, end at dst, and their
    bottleneck is the min residual along them on a Jellyfish-style DC."""
    g = gen.random_graph(40, 5, 3, seed)
    q = gen.path_queries(g, 300, seed, bw_hi=700)
    bn, hops, path = O.graph_paths(g, q["src"], q["dst"], q["demand"], max_hops=20)
    best = {}
    for u, v, r in zip(g["link_u"], g["link_v"], g["link_res"]):
        key = (min(u, v), max(u, v))
        best[key] = max(best.get(key, -1), r)
    for i in range(300):
        if hops[i] < 0:
            continue
        p = [x for x in path[i] if x >= 0]
        assert p[0] == q["src"][i] and p[-1] == q["dst"][i] and len(p) == hops[i] + 1
        assert len(set(p)) == len(p)
        w = min(best[(min(a, b), max(a, b))] for a, b in zip(p, p[1:]))
        assert w == bn[i] >= q["demand"][i]


def test_unreachable():
    g = dict(n_vertices=5, n_servers=5, link_u=np.int32([0, 2]), link_v=np.int32([1, 3]),
             link_res=np.int32([10, 10]))
    bn, hops, _ = O.graph_paths(g, [0, 0, 4], [1, 2, 0], [0, 0, 0])
    assert bn.tolist() == [10, -1, -1] and hops.tolist() == [1, -1, -1]
    assert O.logical_bandwidth(g).tolist() == [10, 10, 10, 10, 0]


@pytest.mark.parametrize("seed", range(4))
def test_logical_bandwidth_brute_force(seed):
    """R2 alternative: sum over servers v != u of the widest-shortest bottleneck u -> v
    (every link usable), by exhaustive path enumeration."""
    rng = np.random.default_rng(200 + seed)
    V = int(rng.integers(4, 8))
    g = tiny_graph(rng, V, int(rng.integers(V, 2 * V)))
    g["n_servers"] = V - 1           # the last vertex is a switch
    got = O.logical_bandwidth(g)
    for u in range(V - 1):
        exp = sum(max(brute_force(g, u, v, 0)[0], 0) for v in range(V - 1) if v != u)
        assert got[u] == exp


def test_logical_bandwidth_fat_tree_closed_form():
    """Fat-tree k=4, warm: the logical bandwidth of u = sum_v min(acc_u, acc_v, widest fabric)."""
    snap = gen.snapshot(4, 9)
    g = gen.fat_tree_graph(snap)
    got = O.logical_bandwidth(g)
    link = snap["link_res"]
    for u in range(16):
        exp = sum(min(link[u], link[v], O.widest_path(4, link, u, v)[1]) for v in range(16) if v != u)
        assert got[u] == exp


def test_hops_equal_scipy_bfs_random_dc():
    """Jellyfish-style DC with large demands: blocked links force detours longer than the
    unconstrained shortest path; hop counts still equal scipy's BFS on the usable links."""
    g = gen.random_graph(60, 4, 2, 5)
    q = gen.path_queries(g, 200, 8, bw_hi=800)
    bn, hops, _ = O.graph_paths(g, q["src"], q["dst"], q["demand"], max_hops=40)
    V = g["n_vertices"]
    free = shortest_path(csr_matrix((np.ones(g["link_u"].size), (g["link_u"], g["link_v"])), shape=(V, V)),
                         directed=False, unweighted=True, indices=q["src"])
    detours = 0
    for i in range(200):
        keep = g["link_res"] >= q["demand"][i]
        m = csr_matrix((np.ones(keep.sum()), (g["link_u"][keep], g["link_v"][keep])), shape=(V, V))
        t = shortest_path(m, directed=False, unweighted=True, indices=[q["src"][i]])[0, q["dst"][i]]
        assert hops[i] == (-1 if np.isinf(t) else int(t))
        detours += bool(hops[i] > free[i, q["dst"][i]])
    assert detours > 0


def test_path_rows_longer_than_max_hops_are_empty():
    """Output convention (include/nacs.h): a path with more links than max_hops is not
    truncated; its row is all -1 while bottleneck and hops are still reported."""
    g = gen.fat_tree_graph(gen.snapshot(4, warm=False))
    bn, hops, path = O.graph_paths(g, [0, 0], [1, 15], [0, 0], max_hops=4)
    assert hops.tolist() == [2, 6] and bn.tolist() == [1000, 1000]
    assert path[0].tolist() == [0, 16, 1, -1, -1] and path[1].tolist() == [-1] * 5


def test_rank_with_logical_bandwidth_criterion():
    """R2 alternative in the ranking: the oracle's Bandwidth criterion equals the logical
    bandwidth of the general-graph Dijkstra on the same state (two independent routes: the
    fat-tree closed form inside orc_rank, the explicit-graph Dijkstra here).  Checked through a
    one-criterion TOPSIS: with weights (0, 0, 0, 1) the closeness orders servers by the
    criterion, so the argmax is the server of largest logical bandwidth (lowest index on ties)."""
    snap = gen.snapshot(4, 31)
    lb = O.logical_bandwidth(gen.fat_tree_graph(snap))
    r = O.rank(snap, "topsis", (0.0, 0.0, 0.0, 1.0), 1, 1, bw_criterion=1)
    feas = r["mask"].astype(bool)
    cand = np.nonzero(feas)[0]
    assert r["best"] == int(cand[np.argmax(lb[cand])])
    # closeness with one criterion: (x - min) / (max - min) over F
    x = lb[cand].astype(np.float64)
    exp = (x - x.min()) / (x.max() - x.min())
    assert np.allclose(r["score"][cand], exp, rtol=1e-12, atol=1e-15)
    r0 = O.rank(snap, "topsis", (0.0, 0.0, 0.0, 1.0), 1, 1, bw_criterion=0)
    acc = snap["link_res"][:16].astype(np.float64)[cand]
    assert np.allclose(r0["score"][cand], (acc - acc.min()) / (acc.max() - acc.min()), rtol=1e-12, atol=1e-15)
