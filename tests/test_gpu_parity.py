"""GPU parity: the CUDA path through the C ABI against the CPU oracle (needs a B200)."""
import json
import os

import numpy as np
import pytest

from inputs import gen
from oracle import oracle as O
from tests.parity import assert_rank_parity, assert_schedule_parity, to_np

pytestmark = pytest.mark.gpu
SCHEMAS = ("flat", "clustering", "network")
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def ctx():
    from paper_1909_07673_b200 import nacs
    c = nacs.Context(0)
    yield c
    c.close()


def random_flows(rng, snap, nflow, dmax=60):
    n = snap["k"] ** 3 // 4
    vs = rng.choice(n, size=min(nflow, n), replace=False)
    return [(int(v), int(rng.integers(1, dmax))) for v in vs]


# ------------------------------------------------------------------ rank -----
@pytest.mark.parametrize("k", [2, 4, 6, 8, 16])
@pytest.mark.parametrize("method", ["topsis", "ahp"])
def test_rank_parity_random(ctx, k, method):
    rng = np.random.default_rng(1000 + k)
    for trial in range(6):
        snap = gen.snapshot(k, seed=200 + trial, quantised=trial % 3 == 2)
        if trial % 2:
            snap["link_res"] = rng.integers(0, 120, size=len(snap["link_res"])).astype(np.int32)
        ctx.load_topology(snap)
        flows = random_flows(rng, snap, int(rng.integers(0, 4)))
        dc, dr = int(rng.integers(100, 8000)), int(rng.integers(128, 30000))
        for schema in SCHEMAS:
            for rule in ((0, 1) if method == "ahp" else (0,)):
                g = ctx.rank(method, schema, dc, dr, flows, ahp_rule=rule)
                o = O.rank(snap, method, schema, dc, dr, flows, ahp_rule=rule)
                assert_rank_parity(g, o, (k, trial, schema, rule))


def test_rank_golden_vectors(ctx):
    gold = json.load(open(os.path.join(GOLDEN, "survey_4server.json")))
    snap = gen.snapshot(4, warm=False)
    for u, (c, r, a, b) in enumerate(gold["rows"]):
        snap["cpu_res"][u], snap["ram_res"][u], snap["active"][u], snap["link_res"][u] = c, r, a, b
    snap["cpu_res"][4:] = 0
    snap["active"][4:] = 1
    ctx.load_topology(snap)
    for case in gold["cases"]:
        g = ctx.rank(case["method"], case["schema"], 1, 1, ahp_rule=case["ahp_rule"])
        assert g["mask"][:4].all() and not g["mask"][4:].any()
        assert g["best"] == case["argmax"]
        assert np.allclose(g["scores"][:4], case["scores"], rtol=1e-5, atol=0), case


@pytest.mark.parametrize("method", ["topsis", "ahp"])
def test_rank_excluded_and_exact64(ctx, method):
    snap = gen.snapshot(8, seed=31)
    ctx.load_topology(snap)
    rng = np.random.default_rng(5)
    flows = random_flows(rng, snap, 3)
    g = ctx.rank(method, "network", 500, 1000, flows)
    ex = [g["best"], flows[0][0]]
    g2 = ctx.rank(method, "network", 500, 1000, flows, excluded=ex)
    o2 = O.rank(snap, method, "network", 500, 1000, flows, excluded=ex)
    assert_rank_parity(g2, o2)
    g3 = ctx.rank(method, "network", 500, 1000, flows, excluded=ex, exact64=True)
    assert g3["best"] == g2["best"] and np.array_equal(g3["mask"], g2["mask"])


def test_rank_no_feasible(ctx):
    ctx.load_topology(gen.snapshot(4, seed=1))
    g = ctx.rank("topsis", "flat", 10 ** 6, 1)
    assert g["best"] == -1 and not g["mask"].any()


# -------------------------------------------------------------- schedule -----
@pytest.mark.parametrize("method", ["topsis", "ahp"])
@pytest.mark.parametrize("schema", SCHEMAS)
def test_c1_sequential(ctx, method, schema):
    snap, reqs = gen.config("C1")
    ctx.load_topology(snap)
    out = to_np(ctx.schedule_request(reqs, method, schema))
    assert (out["server_of_container"] == 0).all()  # SURVEY §8(c) C1 expectation
    assert_schedule_parity(snap, reqs, out, method, schema, True, gpu_state=ctx.read_topology())


@pytest.mark.parametrize("method", ["topsis", "ahp"])
@pytest.mark.parametrize("schema", SCHEMAS)
def test_c2_sequential(ctx, method, schema):
    snap, reqs = gen.config("C2")
    ctx.load_topology(snap)
    out = ctx.schedule_request(reqs, method, schema)
    cnt = assert_schedule_parity(snap, reqs, out, method, schema, True, gpu_state=ctx.read_topology())
    st = ctx.last_stats()
    assert st["pod_steps"] == cnt["pod_steps"] and st["retries"] == cnt["retries"]


@pytest.mark.parametrize("method", ["topsis", "ahp"])
@pytest.mark.parametrize("rule", [0, 1])
def test_c2_batch(ctx, method, rule):
    snap, reqs = gen.config("C2")
    ctx.load_topology(snap)
    for schema in SCHEMAS:
        out = ctx.schedule_batch(reqs, method, schema, ahp_rule=rule)
        assert_schedule_parity(snap, reqs, out, method, schema, False, ahp_rule=rule)
    st = ctx.read_topology()
    for key in ("cpu_res", "ram_res", "active", "link_res"):
        assert np.array_equal(st[key], snap[key])  # batch never mutates (R21)


def test_congested_links_retries_and_rejections(ctx):
    """Tight fabric: flows compete for links, exercising R18 retries and R20 rejections."""
    snap = gen.snapshot(8, seed=77)
    snap["link_res"] = np.random.default_rng(1).integers(0, 90, size=len(snap["link_res"])).astype(np.int32)
    reqs = gen.requests(300, 78, bw_max_hi=60)
    for method in ("topsis", "ahp"):
        ctx.load_topology(snap)
        out = ctx.schedule_batch(reqs, method, "network")
        cnt = assert_schedule_parity(snap, reqs, out, method, "network", False)
        assert (to_np(out)["status"] == 0).any()
        out = ctx.schedule_request(reqs, method, "network")
        cnt = assert_schedule_parity(snap, reqs, out, method, "network", True, gpu_state=ctx.read_topology())
        assert cnt["retries"] == ctx.last_stats()["retries"]


def test_quantised_ties(ctx):
    snap = gen.snapshot(8, seed=9, quantised=True)
    reqs = gen.requests(150, 10)
    ctx.load_topology(snap)
    for method in ("topsis", "ahp"):
        out = ctx.schedule_batch(reqs, method, "clustering")
        assert_schedule_parity(snap, reqs, out, method, "clustering", False)


def test_c3_batch_subsample(ctx):
    snap, reqs = gen.config("C3")
    ctx.load_topology(snap)
    sub = gen.subset(reqs, np.arange(0, 10_000, 25))  # 400 requests
    out = ctx.schedule_batch(sub, "topsis", "flat")
    assert_schedule_parity(snap, sub, out, "topsis", "flat", False)
    sub2 = gen.subset(reqs, np.arange(0, 10_000, 200))  # 50 requests
    out = ctx.schedule_batch(sub2, "ahp", "flat")
    assert_schedule_parity(snap, sub2, out, "ahp", "flat", False)


def test_c4_full_batch_sampled_parity(ctx):
    """The bench launch configuration (C4, 100k requests, device pointers): parity on a
    sample of requests (requests are independent under R21) plus invariants on all."""
    import torch
    snap, reqs = gen.config("C4")
    ctx.load_topology(snap)
    dreqs = {k: (torch.from_numpy(v).cuda() if isinstance(v, np.ndarray) else v) for k, v in reqs.items()}
    out = to_np(ctx.schedule_batch(dreqs, "topsis", "flat"))
    co, vo = reqs["container_off"], reqs["vlink_off"]
    assert set(np.unique(out["status"]).tolist()) <= {0, 1}
    ok = np.repeat(out["status"] == 1, np.diff(co))
    assert (out["server_of_container"][ok] >= 0).all() and (out["server_of_container"][~ok] == -1).all()
    assert (out["cpu_alloc"][ok] >= reqs["cpu_min"][ok]).all() and (out["cpu_alloc"][ok] <= reqs["cpu_max"][ok]).all()
    idx = np.sort(np.random.default_rng(0).choice(reqs["n_requests"], 200, replace=False))
    sub = gen.subset(reqs, idx)
    cs = np.concatenate([np.arange(co[i], co[i + 1]) for i in idx])
    vs = np.concatenate([np.arange(vo[i], vo[i + 1]) for i in idx])
    gsub = dict(status=out["status"][idx], server_of_container=out["server_of_container"][cs],
                cpu_alloc=out["cpu_alloc"][cs], ram_alloc=out["ram_alloc"][cs],
                bw_alloc=out["bw_alloc"][vs], path_of_vlink=out["path_of_vlink"][vs])
    assert_schedule_parity(snap, sub, gsub, "topsis", "flat", False)


def test_determinism(ctx):
    snap, reqs = gen.config("C2")
    ctx.load_topology(snap)
    a = to_np(ctx.schedule_batch(reqs, "ahp", "network"))
    b = to_np(ctx.schedule_batch(reqs, "ahp", "network"))
    for k in a:
        assert np.array_equal(a[k], b[k])
    g1 = ctx.rank("topsis", "flat", 300, 300)
    g2 = ctx.rank("topsis", "flat", 300, 300)
    assert np.array_equal(g1["scores"].view(np.uint32), g2["scores"].view(np.uint32))


# ------------------------------------------------------------ edge cases -----
def test_empty_batch_and_errors(ctx):
    from paper_1909_07673_b200 import nacs
    snap, reqs = gen.config("C2")
    ctx.load_topology(snap)
    empty = gen.subset(reqs, [])
    out = ctx.schedule_batch(empty, "topsis", "flat")
    assert len(out["status"]) == 0
    bad = gen.subset(reqs, [0, 1])
    bad["cpu_min"] = bad["cpu_min"].copy()
    bad["cpu_min"][0] = bad["cpu_max"][0] + 1
    with pytest.raises(nacs.NacsError) as ei:
        ctx.schedule_batch(bad, "topsis", "flat")
    assert ei.value.status == nacs.NACS_EINVAL and "request 0" in str(ei.value)
    before = ctx.read_topology()
    with pytest.raises(nacs.NacsError):
        ctx.schedule_request(bad, "topsis", "flat")
    after = ctx.read_topology()
    for k in before:
        assert np.array_equal(before[k], after[k])  # errors leave the state unchanged
    with pytest.raises(nacs.NacsError):
        ctx.schedule_batch(reqs, "topsis", (0.5, 0.5, 0.5, 0.5))  # weights do not sum to 1
    with pytest.raises(nacs.NacsError) as ei:
        ctx.load_topology(dict(snap, k=5))
    assert ei.value.status == nacs.NACS_EINVAL


def test_device_pointer_invalid_request_status(ctx):
    import torch
    from paper_1909_07673_b200 import nacs
    snap, reqs = gen.config("C2")
    ctx.load_topology(snap)
    bad = gen.subset(reqs, [0, 1, 2])
    bad["pod_of"] = bad["pod_of"].copy()
    bad["pod_of"][0] = 50  # pod ids not 0..P-1
    d = {k: (torch.from_numpy(v).cuda() if isinstance(v, np.ndarray) else v) for k, v in bad.items()}
    out = ctx.schedule_batch(d, "topsis", "flat", flags=nacs.NACS_ASYNC)
    torch.cuda.synchronize()
    st = out["status"].cpu().numpy()
    assert st[0] == -1 and (st[1:] == 1).all()
    with pytest.raises(nacs.NacsError):
        ctx.schedule_batch(d, "topsis", "flat")


def test_rejected_request_is_atomic(ctx):
    snap = gen.snapshot(8, seed=3)
    reqs = gen.requests(3, 4)
    reqs["cpu_min"][reqs["container_off"][1]:reqs["container_off"][2]] = 24000
    reqs["cpu_max"][reqs["container_off"][1]:reqs["container_off"][2]] = 24000
    ctx.load_topology(snap)
    out = ctx.schedule_request(reqs, "topsis", "flat")
    assert to_np(out)["status"][1] == 0
    assert_schedule_parity(snap, reqs, out, "topsis", "flat", True, gpu_state=ctx.read_topology())


def _cta_only_ctx():
    from paper_1909_07673_b200 import nacs
    os.environ["NACS_CTA_ONLY"] = "1"
    try:
        return nacs.Context(0)
    finally:
        del os.environ["NACS_CTA_ONLY"]


def test_warp_kernel_equals_cta_kernel(ctx):
    """The warp-per-request fast path (k_batch_warp) and the CTA-per-request kernel
    (k_batch) give identical placements (both also match the oracle elsewhere)."""
    cta = _cta_only_ctx()
    try:
        cases = [(gen.config("C3")[0], gen.subset(gen.config("C3")[1], np.arange(0, 10_000, 10)))]
        tight = gen.snapshot(8, seed=77)
        tight["link_res"] = np.random.default_rng(1).integers(0, 90, size=len(tight["link_res"])).astype(np.int32)
        cases.append((tight, gen.requests(400, 78, bw_max_hi=60)))
        cases.append((gen.snapshot(6, seed=5, quantised=True), gen.requests(300, 6)))  # n = 54: ragged chunk
        for snap, reqs in cases:
            ctx.load_topology(snap)
            cta.load_topology(snap)
            for schema in SCHEMAS:
                a = to_np(ctx.schedule_batch(reqs, "topsis", schema))
                b = to_np(cta.schedule_batch(reqs, "topsis", schema))
                for key in a:
                    assert np.array_equal(a[key], b[key]), (schema, key)
    finally:
        cta.close()


def test_warp_kernel_pruned_scans_at_scale(ctx):
    """The warp kernel's chunk layout, whole-chunk statistics and best-first pruned scoring
    at k=32 (64 chunks): identical to the CTA kernel (which reads every server in index
    order) on exact-tie (quantised), congested-fabric (slow chunks) and exact-FP64 runs,
    and to the oracle on a sample."""
    from paper_1909_07673_b200 import nacs
    cta = _cta_only_ctx()
    try:
        quant = gen.snapshot(32, seed=21, quantised=True)
        tight = gen.snapshot(32, seed=22)
        tight["link_res"] = np.random.default_rng(3).integers(0, 120, size=len(tight["link_res"])).astype(np.int32)
        cases = [(quant, gen.requests(1500, 23), 0), (tight, gen.requests(1500, 24, bw_max_hi=60), 0),
                 (gen.config("C4")[0], gen.requests(600, 25), nacs.NACS_EXACT_FP64)]
        for snap, reqs, flags in cases:
            ctx.load_topology(snap)
            cta.load_topology(snap)
            for schema in SCHEMAS:
                a = to_np(ctx.schedule_batch(reqs, "topsis", schema, flags=flags))
                sa = ctx.last_stats()
                b = to_np(cta.schedule_batch(reqs, "topsis", schema, flags=flags))
                for key in a:
                    assert np.array_equal(a[key], b[key]), (schema, key)
                assert sa["scanned_b"] < sa["servers_ranked"] or flags
        sub = gen.subset(cases[0][1], np.arange(0, 1500, 15))
        ctx.load_topology(quant)
        out = ctx.schedule_batch(sub, "topsis", "clustering")
        assert_schedule_parity(quant, sub, out, "topsis", "clustering", False)
    finally:
        cta.close()


def test_large_requests_deferred_to_cta_kernel(ctx):
    """Requests with more than 32 containers or 64 vlinks leave the warp fast path for the
    CTA kernel; mixed batches stay exact."""
    snap = gen.snapshot(8, seed=41)
    reqs = gen.requests(120, 42, nc_lo=4, nc_hi=70, extra_edges=3)
    assert (np.diff(reqs["container_off"]) > 32).any() and (np.diff(reqs["container_off"]) <= 32).any()
    ctx.load_topology(snap)
    out = ctx.schedule_batch(reqs, "topsis", "flat")
    assert_schedule_parity(snap, reqs, out, "topsis", "flat", False)


# ------------------------------------------------------- server sharding -----
@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_server_sharded_loopback_equals_unsharded(world):
    """§8(e): G logical server shards on one GPU (exchange = device copy) give the same
    placements and final state as the unsharded sequential path, and match the oracle."""
    from paper_1909_07673_b200 import nacs
    snap, reqs = gen.config("C2")
    sub = gen.subset(reqs, np.arange(60))
    ref = nacs.Context(0)
    sh = nacs.Context(0, shard=(0, world, None))
    try:
        for schema in SCHEMAS:
            ref.load_topology(snap)
            sh.load_topology(snap)
            a = to_np(ref.schedule_request(sub, "topsis", schema))
            b = to_np(sh.schedule_request(sub, "topsis", schema))
            for key in a:
                assert np.array_equal(a[key], b[key]), (world, schema, key)
            sa, sb = ref.read_topology(), sh.read_topology()
            for key in sa:
                assert np.array_equal(sa[key], sb[key])
            assert_schedule_parity(snap, sub, b, "topsis", schema, True, gpu_state=sb)
    finally:
        ref.close()
        sh.close()


def test_server_sharded_congested_and_exact64():
    from paper_1909_07673_b200 import nacs
    snap = gen.snapshot(8, seed=77)
    snap["link_res"] = np.random.default_rng(1).integers(0, 90, size=len(snap["link_res"])).astype(np.int32)
    reqs = gen.requests(120, 78, bw_max_hi=60)
    sh = nacs.Context(0, shard=(0, 4, None))
    try:
        sh.load_topology(snap)
        out = sh.schedule_request(reqs, "topsis", "network")
        assert_schedule_parity(snap, reqs, out, "topsis", "network", True, gpu_state=sh.read_topology())
        sh.load_topology(snap)
        out2 = sh.schedule_request(reqs, "topsis", "network", flags=nacs.NACS_EXACT_FP64)
        for key in out:
            assert np.array_equal(to_np(out)[key], to_np(out2)[key])
    finally:
        sh.close()


def test_server_sharded_nccl_world1():
    """The NCCL exchange path with a real communicator (world size 1 on this box)."""
    from paper_1909_07673_b200 import nacs
    snap, reqs = gen.config("C2")
    sub = gen.subset(reqs, np.arange(30))
    uid = nacs.nccl_unique_id()
    sh = nacs.Context(0, shard=(0, 1, uid))
    try:
        sh.load_topology(snap)
        out = sh.schedule_request(sub, "topsis", "flat")
        assert_schedule_parity(snap, sub, out, "topsis", "flat", True, gpu_state=sh.read_topology())
    finally:
        sh.close()


@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("rule", [0, 1])
def test_server_sharded_ahp_loopback(world, rule):
    """AHP with the level-pair passes split over G logical ranks (sum-allreduce between
    passes = shared buffers in loopback) equals the single-CTA sequential path."""
    from paper_1909_07673_b200 import nacs
    snap, reqs = gen.config("C2")
    sub = gen.subset(reqs, np.arange(40))
    ref = nacs.Context(0)
    sh = nacs.Context(0, shard=(0, world, None))
    try:
        for schema in ("flat", "network"):
            ref.load_topology(snap)
            sh.load_topology(snap)
            a = to_np(ref.schedule_request(sub, "ahp", schema, ahp_rule=rule))
            b = to_np(sh.schedule_request(sub, "ahp", schema, ahp_rule=rule))
            assert_schedule_parity(snap, sub, b, "ahp", schema, True, gpu_state=sh.read_topology(), ahp_rule=rule)
            for key in a:
                assert np.array_equal(a[key], b[key]), (world, schema, key)
    finally:
        ref.close()
        sh.close()


@pytest.mark.parametrize("rule", [0, 1])
def test_ahp_grid_engine_large_topology(ctx, rule):
    """k=26 (4394 servers): sequential AHP runs through the grid-wide level passes
    (k_ahp_pass_tiled: thousands of levels per criterion, ragged last tiles, both rules)."""
    snap = gen.snapshot(26, seed=26)
    reqs = gen.requests(3, 27)
    ctx.load_topology(snap)
    out = ctx.schedule_request(reqs, "ahp", "clustering", ahp_rule=rule)
    assert_schedule_parity(snap, reqs, out, "ahp", "clustering", True, gpu_state=ctx.read_topology(),
                           ahp_rule=rule)


def test_server_sharded_ahp_nccl_world1():
    from paper_1909_07673_b200 import nacs
    snap, reqs = gen.config("C2")
    sub = gen.subset(reqs, np.arange(20))
    sh = nacs.Context(0, shard=(0, 1, nacs.nccl_unique_id()))
    try:
        sh.load_topology(snap)
        out = sh.schedule_request(sub, "ahp", "flat")
        assert_schedule_parity(snap, sub, out, "ahp", "flat", True, gpu_state=sh.read_topology())
    finally:
        sh.close()


# ------------------------------------------------ R25: rank once per request -----
@pytest.mark.parametrize("method", ["topsis", "ahp"])
def test_rank_once_c2_sequential_and_batch(ctx, method):
    """the first pod step's order, pods walk it (nacs_options.rank_mode)."""
    snap, reqs = gen.config("C2")
    for schema in SCHEMAS:
        ctx.load_topology(snap)
        out = ctx.schedule_request(reqs, method, schema, rank_once=True)
        cnt = assert_schedule_parity(snap, reqs, out, method, schema, True, gpu_state=ctx.read_topology(),
                                     rank_once=True)
        assert ctx.last_stats()["pod_steps"] == cnt["pod_steps"]
        ctx.load_topology(snap)
        out = ctx.schedule_batch(reqs, method, schema, rank_once=True)
        assert_schedule_parity(snap, reqs, out, method, schema, False, rank_once=True)


def test_rank_once_congested_and_c3(ctx):
    tight = gen.snapshot(8, seed=77)
    tight["link_res"] = np.random.default_rng(1).integers(0, 90, size=len(tight["link_res"])).astype(np.int32)
    reqs = gen.requests(300, 78, bw_max_hi=60)
    for method in ("topsis", "ahp"):
        ctx.load_topology(tight)
        out = ctx.schedule_request(reqs, method, "network", rank_once=True)
        cnt = assert_schedule_parity(tight, reqs, out, method, "network", True, gpu_state=ctx.read_topology(),
                                     rank_once=True)
        assert cnt["retries"] == ctx.last_stats()["retries"]
    snap, c3 = gen.config("C3")
    ctx.load_topology(snap)
    sub = gen.subset(c3, np.arange(0, 10_000, 50))
    for method in ("topsis", "ahp"):
        out = ctx.schedule_batch(sub, method, "clustering", rank_once=True)
        assert_schedule_parity(snap, sub, out, method, "clustering", False, rank_once=True)


def test_rank_once_not_on_sharded_contexts():
    from paper_1909_07673_b200 import nacs
    snap, reqs = gen.config("C2")
    sh = nacs.Context(0, shard=(0, 2, None))
    try:
        sh.load_topology(snap)
        with pytest.raises(nacs.NacsError) as ei:
            sh.schedule_request(reqs, "topsis", "flat", rank_once=True)
        assert ei.value.status == nacs.NACS_EINVAL
    finally:
        sh.close()


def test_rank_once_warp_kernel_equals_cta_kernel(ctx):
    """R25 on the warp fast path (no statistics after the first pod step, pruned walk over the
    first step's order on snapshot values) equals the CTA kernel and the oracle, at k=32."""
    cta = _cta_only_ctx()
    try:
        quant = gen.snapshot(32, seed=31, quantised=True)
        tight = gen.snapshot(16, seed=32)
        tight["link_res"] = np.random.default_rng(4).integers(0, 100, size=len(tight["link_res"])).astype(np.int32)
        for snap, reqs in ((gen.config("C4")[0], gen.requests(1200, 33)), (quant, gen.requests(800, 34)),
                           (tight, gen.requests(800, 35, bw_max_hi=60))):
            ctx.load_topology(snap)
            cta.load_topology(snap)
            for schema in SCHEMAS:
                a = to_np(ctx.schedule_batch(reqs, "topsis", schema, rank_once=True))
                b = to_np(cta.schedule_batch(reqs, "topsis", schema, rank_once=True))
                for key in a:
                    assert np.array_equal(a[key], b[key]), (schema, key)
            sub = gen.subset(reqs, np.arange(0, reqs["n_requests"], 20))
            out = ctx.schedule_batch(sub, "topsis", "network", rank_once=True)
            assert_schedule_parity(snap, sub, out, "topsis", "network", False, rank_once=True)
    finally:
        cta.close()


@pytest.mark.parametrize("k", [10, 12, 14, 20])
def test_warp_kernel_ragged_chunk_layouts(ctx, k):
    """n = k^3/4 not a multiple of 128 (250, 432, 686) and a mid size (2000): the chunk layout's
    padded last tile, whole-tile statistics and pruning give the CTA kernel's placements, in
    both ranking modes, and the oracle's on a sample."""
    cta = _cta_only_ctx()
    try:
        snap = gen.snapshot(k, seed=40 + k)
        reqs = gen.requests(600, 50 + k)
        ctx.load_topology(snap)
        cta.load_topology(snap)
        for ro in (False, True):
            a = to_np(ctx.schedule_batch(reqs, "topsis", "clustering", rank_once=ro))
            b = to_np(cta.schedule_batch(reqs, "topsis", "clustering", rank_once=ro))
            for key in a:
                assert np.array_equal(a[key], b[key]), (ro, key)
        sub = gen.subset(reqs, np.arange(0, 600, 30))
        out = ctx.schedule_batch(sub, "topsis", "flat")
        assert_schedule_parity(snap, sub, out, "topsis", "flat", False)
    finally:
        cta.close()


# ------------------------------------------- logical bandwidth criterion -----
@pytest.mark.parametrize("k", [4, 6, 8, 16])
@pytest.mark.parametrize("method", ["topsis", "ahp"])
def test_rank_logical_bandwidth_criterion(ctx, k, method):
    """R2's alternative reading (bw_criterion = logical): the Bandwidth
    criterion is the sum of widest-shortest bottlenecks to every other server."""
    rng = np.random.default_rng(3000 + k)
    for trial in range(1 if k == 16 else 3):  # the oracle's logical table is O(n^2 paths): 5 s at k=16
        snap = gen.snapshot(k, seed=400 + trial, quantised=trial == 2)
        ctx.load_topology(snap)
        flows = random_flows(rng, snap, int(rng.integers(0, 3)))
        dc, dr = int(rng.integers(100, 8000)), int(rng.integers(128, 30000))
        for schema in (("network",) if k == 16 else SCHEMAS):
            g = ctx.rank(method, schema, dc, dr, flows, bw_criterion=1)
            o = O.rank(snap, method, schema, dc, dr, flows, bw_criterion=1)
            assert_rank_parity(g, o, (k, trial, schema))


def test_logical_bandwidth_limits(ctx):
    from paper_1909_07673_b200 import nacs
    snap = gen.snapshot(32, 4, link_cap=4000)  # n x link_cap = 32.8M >= 2^24: not exact in FP32
    ctx.load_topology(snap)
    with pytest.raises(nacs.NacsError) as e:
        ctx.rank("topsis", "flat", 100, 100, bw_criterion=1)
    assert e.value.status == nacs.NACS_ETOOBIG
    snap, reqs = gen.config("C2")
    ctx.load_topology(snap)
    with pytest.raises(nacs.NacsError) as e:
        ctx.schedule_batch(reqs, "topsis", "flat", bw_criterion=1)
    assert e.value.status == nacs.NACS_EINVAL
