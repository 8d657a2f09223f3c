"""GPU parity of the BF / WF baselines, departures and the discrete-event simulator (SURVEY.md
§8(f) row 3, T5 P:416-426; readings R27, R28) through the C ABI,
against the oracle.  Integer work: placements, timelines and counters must be identical.  The
single-shot schedule tests resynchronise R14 near-ties through the oracle's hint (as in
test_gpu_parity); a simulation re-offers refused requests, so a per-request hint cannot name
the choices of its failed attempts: the simulation tests compare without hints, on fresh DCs
whose exact ties (identical servers) both sides break to the lowest index."""
import numpy as np
import pytest

from inputs import gen
from oracle import oracle as O
from tests.parity import OUT_KEYS, assert_schedule_parity
from tests.test_oracle_sim import single_container_requests

pytestmark = pytest.mark.gpu
STATE_KEYS = ("cpu_res", "ram_res", "active", "link_res")


@pytest.fixture(scope="module")
def ctx():
    from paper_1909_07673_b200 import nacs
    c = nacs.Context(0)
    yield c
    c.close()


@pytest.mark.parametrize("method", ["bf", "wf"])
@pytest.mark.parametrize("k,nreq", [(4, 30), (8, 100), (16, 300)])
def test_fit_schedule_parity(ctx, method, k, nreq):
    snap = gen.snapshot(k, 60 + k, quantised=k == 8)
    reqs = gen.requests(nreq, 61 + k)
    ctx.load_topology(snap)
    out = ctx.schedule_request(reqs, method, "flat")
    assert_schedule_parity(snap, reqs, out, method, "flat", True, gpu_state=ctx.read_topology())
    ctx.load_topology(snap)
    out = ctx.schedule_batch(reqs, method, "flat")
    assert_schedule_parity(snap, reqs, out, method, "flat", False)


def test_fit_congested_fabric_retries(ctx):
    """BF on a congested fabric: the CPU/RAM-only choice fails to route (R18 retries, rejections)."""
    snap = gen.snapshot(8, 5)
    snap["link_res"] = np.random.default_rng(3).integers(0, 60, size=snap["link_res"].size).astype(np.int32)
    reqs = gen.requests(80, 9)
    for m in ("bf", "wf"):
        ctx.load_topology(snap)
        out = ctx.schedule_request(reqs, m, "flat")
        cnt = assert_schedule_parity(snap, reqs, out, m, "flat", True, gpu_state=ctx.read_topology())
        assert cnt["retries"] > 0 and ctx.last_stats()["retries"] == cnt["retries"]


@pytest.mark.parametrize("method", ["topsis", "ahp", "bf", "wf"])
def test_release_is_exact_inverse(ctx, method):
    snap = gen.snapshot(8, 12)
    reqs = gen.requests(60, 13)
    ctx.load_topology(snap)
    out = ctx.schedule_request(reqs, method, "network")
    assert (out["status"] == 1).sum() > 40
    ctx.release(reqs, out)
    back = ctx.read_topology()
    for key in STATE_KEYS:
        assert np.array_equal(back[key], snap[key]), key


def test_release_partial_device_pointers_and_errors(ctx):
    import torch
    from paper_1909_07673_b200 import nacs
    snap = gen.snapshot(8, 14)
    reqs = gen.requests(50, 15)
    ctx.load_topology(snap)
    out = ctx.schedule_request(reqs, "topsis", "flat")
    after = ctx.read_topology()
    part = dict(out, status=np.where(np.arange(50) % 3 == 0, out["status"], 0).astype(np.int32))
    d = {k: (torch.from_numpy(np.asarray(v)).cuda() if isinstance(v, np.ndarray) else v) for k, v in reqs.items()}
    dp = {k: torch.from_numpy(np.asarray(part[k])).cuda() for k in OUT_KEYS}
    ctx.release(d, dp)
    exp = O.release(dict(snap, **after), reqs, part)
    got = ctx.read_topology()
    for key in STATE_KEYS:
        assert np.array_equal(got[key], exp[key]), key
    # releasing the same requests again would exceed capacities: error, state unchanged
    with pytest.raises(nacs.NacsError):
        ctx.release(reqs, part)
    got2 = ctx.read_topology()
    for key in STATE_KEYS:
        assert np.array_equal(got2[key], got[key]), key
    # a malformed placement (server out of range) is rejected
    bad = dict(out, server_of_container=np.full_like(out["server_of_container"], 10 ** 6))
    with pytest.raises(nacs.NacsError):
        ctx.release(reqs, bad)


def compare_sim(g, o, label=""):
    for key in ("start", "attempts", "status"):
        assert np.array_equal(g[key], o[key]), (label, key)
    for key in OUT_KEYS:
        assert np.array_equal(g["placements"][key], o["placements"][key]), (label, key)
    for key in ("tick_servers", "tick_links", "tick_queue"):
        assert np.array_equal(g[key], o[key]), (label, key)
    for key in ("events", "attempts", "accepted"):
        assert g["totals"][key] == o["totals"][key], (label, key)


def test_sim_hand_worked_timeline(ctx):
    """The timeline of tests/test_oracle_sim.py, worked by hand, through the GPU."""
    snap = gen.snapshot(2, warm=False)
    reqs = single_container_requests([16000, 16000, 16000, 16000, 4000])
    arrival = np.int32([0, 0, 1, 1, 1])
    duration = np.int32([3, 1, 1, 2, 1])
    for hol, start, queue in ((1, [0, 0, 1, 2, 2], [0, 2, 0]), (0, [0, 0, 1, 2, 1], [0, 1, 0])):
        ctx.load_topology(snap)
        r = ctx.simulate(reqs, arrival, duration, "wf", "flat", max_ticks=50, hol=hol)
        assert r["start"].tolist() == start and r["tick_queue"].tolist() == queue
        assert r["placements"]["server_of_container"].tolist() == [0, 1, 1, 1, 0]
        assert r["totals"]["events"] == 3


@pytest.mark.parametrize("method,schema", [("topsis", "flat"), ("topsis", "clustering"), ("ahp", "network"),
                                           ("bf", "flat"), ("wf", "flat")])
@pytest.mark.parametrize("hol", [1, 0])
def test_sim_parity_congested(ctx, method, schema, hol):
    """A small fresh DC under heavy load (queueing, retries, departures every tick)."""
    snap = gen.snapshot(4, warm=False)
    reqs, arrival, duration = gen.sim_workload(400, seed=21, horizon=30, max_duration=25)
    ctx.load_topology(snap)
    g = ctx.simulate(reqs, arrival, duration, method, schema, max_ticks=600, hol=hol)
    o = O.simulate(snap, reqs, arrival, duration, method, schema, max_ticks=600, hol=hol)
    compare_sim(g, o, (method, schema, hol))
    assert g["tick_queue"].max() > 0  # the run did queue
    state = ctx.read_topology()
    for key in STATE_KEYS:
        assert np.array_equal(state[key], o["state"][key]), key


@pytest.mark.parametrize("method", ["topsis", "bf", "wf"])
def test_sim_parity_e2_shape(ctx, method):
    """The E2 shape (4-container requests, 50 Mbps pairs) on a k=8 fresh DC, 800 requests."""
    snap = gen.snapshot(8, warm=False)
    reqs, arrival, duration = gen.sim_workload(800, seed=22, horizon=100, max_duration=50)
    ctx.load_topology(snap)
    g = ctx.simulate(reqs, arrival, duration, method, "network", max_ticks=2000)
    o = O.simulate(snap, reqs, arrival, duration, method, "network", max_ticks=2000)
    compare_sim(g, o, method)


def test_sim_max_ticks_cuts_the_run(ctx):
    """Requests still queued (or not yet arrived) at max_ticks end rejected with empty mappings."""
    snap = gen.snapshot(2, warm=False)
    reqs = single_container_requests([20000, 20000, 20000, 20000])
    arrival = np.int32([0, 0, 0, 9])
    duration = np.int32([5, 5, 5, 1])
    ctx.load_topology(snap)
    g = ctx.simulate(reqs, arrival, duration, "bf", "flat", max_ticks=4)
    o = O.simulate(snap, reqs, arrival, duration, "bf", "flat", max_ticks=4)
    compare_sim(g, o)
    assert g["start"].tolist() == [0, 0, -1, -1] and g["totals"]["events"] == 4
    assert g["placements"]["server_of_container"].tolist() == [0, 1, -1, -1]
