"""nacs_rank_topsis_many (the whole-GPU cluster ranking kernel, nacs_rank.cu) against the
oracle, state by state (needs a B200).  Every state is an independent pod step (SURVEY
§8(a) a0-a5T, a7), so per-state parity with O.rank is exact."""
import numpy as np
import pytest

from inputs import gen
from oracle import oracle as O
from tests.parity import assert_rank_parity

pytestmark = pytest.mark.gpu


def state_words(snap):
    """The ABI's state row: cpu | ram | active | links, int32."""
    return np.concatenate([snap["cpu_res"], snap["ram_res"], snap["active"].astype(np.int32),
                           snap["link_res"]]).astype(np.int32)


def snaps(k, B, seed, tight=False):
    out = []
    rng = np.random.default_rng(seed)
    for b in range(B):
        s = gen.snapshot(k, seed=seed * 100 + b, quantised=b % 3 == 2)
        if tight and b % 2:
            s["link_res"] = rng.integers(0, 120, size=len(s["link_res"])).astype(np.int32)
        out.append(s)
    return out


@pytest.fixture(scope="module")
def ctx():
    from paper_1909_07673_b200 import nacs
    c = nacs.Context(0)
    yield c
    c.close()


@pytest.mark.parametrize("k", [2, 4, 6, 8, 10, 16, 32, 64])
def test_rank_many_vs_oracle(ctx, k):
    """k = 6 and 10 have n = 54, 250 (n % 4 != 0: the 2-wide vector path); k = 64: a cluster of
    16 CTAs per state.  Flows, exclusions and congested links on alternate states."""
    B = 3 if k == 64 else 6
    ss = snaps(k, B, 40 + k, tight=True)
    ctx.load_topology(ss[0])
    states = np.stack([state_words(s) for s in ss])
    n = k ** 3 // 4
    rng = np.random.default_rng(k)
    flows = [(int(v), int(rng.integers(1, 60))) for v in rng.choice(n, size=min(3, n), replace=False)]
    ex = [int(x) for x in rng.choice(n, size=min(2, n), replace=False)]
    for fl, exc, schema in (([], [], "flat"), (flows, [], "network"), (flows, ex, "clustering")):
        got = ctx.rank_many(states, 1500, 3000, flows=fl, excluded=exc, weights=schema)
        for b, s in enumerate(ss):
            o = O.rank(s, "topsis", schema, 1500, 3000, fl, exc)
            g = dict(mask=got["mask"][b], scores=got["scores"][b], best=int(got["best"][b]))
            assert_rank_parity(g, o, (k, b, schema, len(fl), len(exc)))
        st = ctx.last_stats()
        assert st["pod_steps"] == B


def test_rank_many_device_pointers_and_path_filter(ctx):
    import torch
    ss = snaps(32, 10, 7)
    ctx.load_topology(ss[0])
    states = np.stack([state_words(s) for s in ss])
    # a padded stride (rows of a wider tensor) on the device
    pad = np.zeros((states.shape[0], states.shape[1] + 12), np.int32)
    pad[:, : states.shape[1]] = states
    d = torch.from_numpy(pad).cuda()
    flows = [(17, 30), (4000, 25)]
    for pf in (1, 0):
        got = ctx.rank_many(d, 800, 1000, flows=flows, weights="network", path_filter=pf)
        host = ctx.rank_many(states, 800, 1000, flows=flows, weights="network", path_filter=pf)
        assert np.array_equal(got["best"].cpu().numpy(), host["best"])
        assert np.array_equal(got["scores"].cpu().numpy().view(np.uint32), host["scores"].view(np.uint32))
        for b in (0, 5, 9):
            o = O.rank(ss[b], "topsis", "network", 800, 1000, flows, path_filter=pf)
            assert_rank_parity(dict(mask=host["mask"][b], scores=host["scores"][b], best=int(host["best"][b])), o)


def test_rank_many_unaligned_device_outputs(ctx):
    """Device outputs the vector / TMA stores cannot take (scores not 16-byte aligned, mask not
    4-byte aligned) are rejected with NACS_EINVAL before any launch; the context stays usable."""
    import torch
    from paper_1909_07673_b200 import nacs
    ss = snaps(16, 3, 12)
    ctx.load_topology(ss[0])
    states = torch.from_numpy(np.stack([state_words(s) for s in ss])).cuda()
    n = 1024
    best = torch.zeros(3, dtype=torch.int32, device="cuda")
    sc = torch.zeros(3 * n + 1, dtype=torch.float32, device="cuda")[1:].view(3, n)
    mk = torch.zeros(3 * n + 3, dtype=torch.uint8, device="cuda")[3:].view(3, n)
    ok_sc = torch.zeros((3, n), dtype=torch.float32, device="cuda")
    ok_mk = torch.zeros((3, n), dtype=torch.uint8, device="cuda")
    for m, s_ in ((ok_mk, sc), (mk, ok_sc)):
        with pytest.raises(nacs.NacsError) as e:
            ctx.rank_many(states, 700, 900, out=dict(mask=m, scores=s_, best=best))
        assert e.value.status == nacs.NACS_EINVAL
    out = ctx.rank_many(states, 700, 900, out=dict(mask=ok_mk, scores=ok_sc, best=best))
    for b, s in enumerate(ss):
        o = O.rank(s, "topsis", "flat", 700, 900)
        assert_rank_parity(dict(mask=out["mask"][b].cpu().numpy(), scores=out["scores"][b].cpu().numpy(),
                                best=int(out["best"][b])), o, b)


def test_rank_many_equals_single_rank_and_exact64(ctx):
    """One state through rank_many equals nacs_rank_topsis on the loaded state (both run the
    cluster kernel) and the FP64 re-decision flag picks the same server."""
    s = gen.snapshot(16, seed=3, quantised=True)
    ctx.load_topology(s)
    a = ctx.rank("topsis", "flat", 500, 700)
    b = ctx.rank_many(state_words(s)[None, :], 500, 700)
    assert a["best"] == int(b["best"][0]) and np.array_equal(a["mask"], b["mask"][0])
    assert np.array_equal(a["scores"].view(np.uint32), b["scores"][0].view(np.uint32))
    c = ctx.rank_many(state_words(s)[None, :], 500, 700, exact64=True)
    o = O.rank(s, "topsis", "flat", 500, 700)
    assert c["best"][0] == o["best"] or o["tie"][c["best"][0]]
    assert ctx.last_stats()["fp64_decisions"] == 1


def test_rank_many_edge_cases(ctx):
    from paper_1909_07673_b200 import nacs
    ss = snaps(8, 4, 9)
    ctx.load_topology(ss[0])
    states = np.stack([state_words(s) for s in ss])
    # nothing feasible in one state, everything in another
    states[1, :128] = 0
    got = ctx.rank_many(states, 1, 1)
    assert got["best"][1] == -1 and not got["mask"][1].any() and (got["scores"][1] == 0).all()
    # an out-of-range residual: best = -2 and NACS_EINVAL (synchronous call)
    bad = states.copy()
    bad[2, 5] = 10 ** 6
    with pytest.raises(nacs.NacsError) as e:
        ctx.rank_many(bad, 1, 1)
    assert e.value.status == nacs.NACS_EINVAL
    out = ctx.rank_many(bad, 1, 1, flags=nacs.NACS_ASYNC)
    import torch
    torch.cuda.synchronize()
    assert out["best"][2] == -2 and out["best"][0] >= 0
    # zero states
    empty = ctx.rank_many(states[:0], 1, 1)
    assert empty["best"].size == 0
    # AHP is not offered by the many-state call
    o = nacs.Context.options("ahp", "flat")
    q = nacs.PodQuery(1, 1, 0, None, None, 0, None)
    st = ctx._lib.nacs_rank_topsis_many(ctx._h, o, q, 1, states.ctypes.data, states.shape[1], None, None,
                                        np.zeros(1, np.int32).ctypes.data)
    assert st == nacs.NACS_EINVAL


def test_rank_many_cold_stream_sampled(ctx):
    """The bench's cold-snapshot configuration (k = 32, distinct device-generated states; 512
    here, 100 MB of state rows): sampled states against the oracle."""
    import torch
    from paper_1909_07673_b200 import nacs
    snap = gen.snapshot(32, gen.CONFIG_SEEDS["C4"])
    ctx.load_topology(snap)
    B = 512
    states = torch.from_numpy(np.tile(state_words(snap), (B, 1))).cuda()
    n = 8192
    g = torch.Generator(device="cuda").manual_seed(11)
    states[:, :n] = torch.randint(0, 24001, (B, n), device="cuda", generator=g, dtype=torch.int32)
    states[:, n:2 * n] = torch.randint(0, 262145, (B, n), device="cuda", generator=g, dtype=torch.int32)
    states[:, 2 * n:3 * n] = torch.randint(0, 2, (B, n), device="cuda", generator=g, dtype=torch.int32)
    states[:, 3 * n:4 * n] = torch.randint(50, 1001, (B, n), device="cuda", generator=g, dtype=torch.int32)
    out = ctx.rank_many(states, 1500, 3000, flags=nacs.NACS_ASYNC)
    torch.cuda.synchronize()
    h = states.cpu().numpy()
    best = out["best"].cpu().numpy()
    for b in (0, 1, 77, 300, 511):
        s = dict(snap, cpu_res=h[b, :n], ram_res=h[b, n:2 * n], active=h[b, 2 * n:3 * n].astype(np.uint8),
                 link_res=h[b, 3 * n:])
        o = O.rank(s, "topsis", "flat", 1500, 3000)
        assert_rank_parity(dict(mask=out["mask"][b].cpu().numpy(), scores=out["scores"][b].cpu().numpy(),
                                best=int(best[b])), o, b)


def test_rank_many_random_sweep(ctx):
    """Random geometries (every even k from 2 to 30 and a few large ones), demands, flows and
    exclusions: every state against the oracle."""
    rng = np.random.default_rng(77)
    for k in list(range(2, 32, 2)) + [36, 48]:
        n = k ** 3 // 4
        B = 3
        ss = [gen.snapshot(k, seed=int(rng.integers(1 << 30)), quantised=bool(rng.integers(2))) for _ in range(B)]
        for s in ss:
            if rng.random() < 0.5:
                s["link_res"] = rng.integers(0, 200, size=len(s["link_res"])).astype(np.int32)
        ctx.load_topology(ss[0])
        states = np.stack([state_words(s) for s in ss])
        nfl = int(rng.integers(0, min(4, n) + 1))
        flows = [(int(v), int(rng.integers(1, 80))) for v in rng.choice(n, size=nfl, replace=False)]
        nex = int(rng.integers(0, min(3, n) + 1))
        ex = [int(x) for x in rng.choice(n, size=nex, replace=False)]
        dc, dr = int(rng.integers(1, 20000)), int(rng.integers(1, 200000))
        schema = ("flat", "clustering", "network")[int(rng.integers(3))]
        got = ctx.rank_many(states, dc, dr, flows=flows, excluded=ex, weights=schema)
        for b, s in enumerate(ss):
            o = O.rank(s, "topsis", schema, dc, dr, flows, ex)
            assert_rank_parity(dict(mask=got["mask"][b], scores=got["scores"][b], best=int(got["best"][b])), o,
                               (k, b, len(flows), len(ex)))
