"""GPU parity of the general-topology path kernels (reading
R26) through the C ABI, against the oracle's modified Dijkstra: bottleneck, hop count and the
whole vertex sequence must be identical (integer work: bit-exact)."""
import numpy as np
import pytest

from inputs import gen
from oracle import oracle as O
from tests.test_oracle_graph import tiny_graph

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_1909_07673_b200 import nacs
    c = nacs.Context(0)
    yield c
    c.close()


def check(ctx, g, q, max_hops, exp=None):
    ctx.load_graph(g)
    bn, hops, path = ctx.widest_paths(q["src"], q["dst"], q["demand"], max_hops=max_hops)
    if exp is None:
        exp = O.graph_paths(g, q["src"], q["dst"], q["demand"], max_hops=max_hops)
    np.testing.assert_array_equal(bn, exp[0])
    np.testing.assert_array_equal(hops, exp[1])
    np.testing.assert_array_equal(path, exp[2])
    return bn, hops, path


@pytest.mark.parametrize("seed", range(8))
def test_tiny_graphs_all_pairs(ctx, seed):
    """Multigraphs with many hop and width ties: every ordered pair, demands 0 / 15 / 25."""
    rng = np.random.default_rng(500 + seed)
    V = int(rng.integers(3, 40))
    g = tiny_graph(rng, V, int(rng.integers(V - 1, 3 * V)))
    s, t = np.meshgrid(np.arange(V), np.arange(V), indexing="ij")
    keep = s != t
    s, t = s[keep], t[keep]
    q = dict(src=np.tile(s, 3), dst=np.tile(t, 3), demand=np.repeat([0, 15, 25], s.size))
    check(ctx, g, q, max_hops=V)


@pytest.mark.parametrize("k", [4, 8, 20])
def test_fat_tree_warm(ctx, k):
    """The explicit fat-tree graph (k=20 is the paper's DC) with demands up to 900 Mbps:
    routed, detoured and blocked queries."""
    g = gen.fat_tree_graph(gen.snapshot(k, 40 + k))
    q = gen.path_queries(g, 600 if k == 20 else 1500, 7 + k, bw_hi=900)
    bn, hops, _ = check(ctx, g, q, max_hops=12)
    assert (hops == -1).any() and (hops > 0).any()


@pytest.mark.parametrize("seed,nsw,deg,sps", [(1, 64, 6, 4), (2, 97, 4, 3), (3, 300, 8, 5)])
def test_random_dc(ctx, seed, nsw, deg, sps):
    """Jellyfish-style DCs (ragged vertex counts) with large demands forcing detours."""
    g = gen.random_graph(nsw, deg, sps, seed)
    q = gen.path_queries(g, 1200, seed, bw_hi=800)
    check(ctx, g, q, max_hops=24)


def test_long_chain_wraps_level_counter(ctx):
    """A 700-vertex chain plus a parallel detour: hop counts beyond 255 (the kernel stores
    levels mod 256) and a path that must take the longer, wider branch."""
    V = 700
    lu = list(range(V - 1))
    lv = list(range(1, V))
    res = [500] * (V - 1)
    lu += [0, 650]
    lv += [650, 699]
    res += [10, 10]
    g = dict(n_vertices=V, n_servers=V, link_u=np.int32(lu), link_v=np.int32(lv), link_res=np.int32(res))
    q = dict(src=np.int32([0, 0, 699, 5, 300]), dst=np.int32([699, 600, 1, 600, 299]),
             demand=np.int32([20, 20, 5, 0, 0]))
    bn, hops, _ = check(ctx, g, q, max_hops=V)
    assert hops[0] == 699 and hops[2] == 3


def test_global_scratch_path(ctx):
    """A graph too large for per-warp scratch in shared memory (V = 16000)."""
    g = gen.random_graph(4000, 6, 3, 11)
    q = gen.path_queries(g, 64, 5, bw_hi=600)
    check(ctx, g, q, max_hops=30)


def test_max_hops_truncation_and_edge_cases(ctx):
    g = gen.fat_tree_graph(gen.snapshot(8, 3))
    q = dict(src=np.int32([0, 0, 0]), dst=np.int32([1, 5, 127]), demand=np.int32([0, 0, 0]))
    ctx.load_graph(g)
    bn, hops, path = ctx.widest_paths(q["src"], q["dst"], q["demand"], max_hops=3)
    exp = O.graph_paths(g, q["src"], q["dst"], q["demand"], max_hops=3)
    np.testing.assert_array_equal(hops, exp[1])
    assert hops[2] == 6 and np.all(path[2] == -1)     # longer than max_hops: row all -1
    np.testing.assert_array_equal(path, exp[2])
    # empty query set; graph without links; disconnected vertices
    e = ctx.widest_paths(np.zeros(0, np.int32), np.zeros(0, np.int32), np.zeros(0, np.int32))
    assert e[0].size == 0
    g0 = dict(n_vertices=6, n_servers=4, link_u=np.int32([0, 2]), link_v=np.int32([4, 4]),
              link_res=np.int32([7, 9]))
    check(ctx, g0, dict(src=np.int32([0, 0, 1, 5]), dst=np.int32([2, 1, 3, 0]), demand=np.int32([0, 0, 0, 8])),
          max_hops=5)
    np.testing.assert_array_equal(ctx.logical_bandwidth(), O.logical_bandwidth(g0))


def test_invalid_queries(ctx):
    from paper_1909_07673_b200 import nacs
    g = gen.fat_tree_graph(gen.snapshot(4, warm=False))
    ctx.load_graph(g)
    with pytest.raises(nacs.NacsError) as e:
        ctx.widest_paths(np.int32([0, 3]), np.int32([0, 99]), np.int32([1, 1]))
    assert e.value.status == nacs.NACS_EINVAL
    with pytest.raises(nacs.NacsError):
        ctx.load_graph(dict(n_vertices=3, n_servers=3, link_u=np.int32([0]), link_v=np.int32([0]),
                            link_res=np.int32([1])))
    import torch
    dev = lambda a: torch.tensor(a, dtype=torch.int32, device="cuda:0")
    with pytest.raises(nacs.NacsError):
        ctx.widest_paths(dev([0, 1]), dev([1, 1]), dev([5, 5]))
    bn, hops, _ = ctx.widest_paths(dev([0, 1]), dev([1, 1]), dev([5, 5]), flags=nacs.NACS_ASYNC)
    torch.cuda.synchronize()
    assert hops.cpu().tolist() == [2, -2]


def test_device_pointers_match_host(ctx):
    import torch
    g = gen.fat_tree_graph(gen.snapshot(16, 8))
    q = gen.path_queries(g, 4000, 2, bw_hi=700)
    ctx.load_graph(g)
    h = ctx.widest_paths(q["src"], q["dst"], q["demand"], max_hops=10)
    t = {k: torch.from_numpy(v).cuda() for k, v in q.items()}
    d = ctx.widest_paths(t["src"], t["dst"], t["demand"], max_hops=10)
    for a, b in zip(h, d):
        np.testing.assert_array_equal(a, b.cpu().numpy())
    # identical on a second call (determinism)
    h2 = ctx.widest_paths(q["src"], q["dst"], q["demand"], max_hops=10)
    for a, b in zip(h, h2):
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("which", ["ft8", "ft12", "jelly", "tiny"])
def test_logical_bandwidth(ctx, which):
    if which == "ft8":
        g = gen.fat_tree_graph(gen.snapshot(8, 21))
    elif which == "ft12":
        g = gen.fat_tree_graph(gen.snapshot(12, 22))
    elif which == "jelly":
        g = gen.random_graph(150, 5, 4, 23)
    else:
        rng = np.random.default_rng(5)
        g = tiny_graph(rng, 30, 45)
        g["n_servers"] = 25
    ctx.load_graph(g)
    np.testing.assert_array_equal(ctx.logical_bandwidth(), O.logical_bandwidth(g))
    assert ctx.last_stats()["edges_scanned"] > 0


def test_grouped_by_destination_and_deferred(ctx):
    """Many queries per destination: one BFS per destination answers the queries whose label
    width covers their demand; the others are re-run on their own (both paths exact)."""
    g = gen.fat_tree_graph(gen.snapshot(8, 77))
    q = gen.path_queries(g, 6000, 78, bw_hi=700)
    check(ctx, g, q, max_hops=8)
    st = ctx.last_stats()
    groups = np.unique(q["dst"]).size
    assert groups < st["bfs_runs"] < 6000  # some deferred, most answered by their group's BFS
    # all demands below every residual: nothing deferred, exactly one BFS per destination
    q2 = gen.path_queries(g, 6000, 79, bw_hi=40)
    check(ctx, g, q2, max_hops=8)
    assert ctx.last_stats()["bfs_runs"] == np.unique(q2["dst"]).size
