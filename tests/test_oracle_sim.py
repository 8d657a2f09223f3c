"""Pins of the oracle's BF / WF baselines, departures and discrete-event simulator (SURVEY.md
§8(f) row 3, T5 P:416-426; readings R27, R28), CPU only.

Expected values come from hand-worked timelines on tiny DCs, integer brute force, and exact
algebraic identities (apply-then-release), not from the oracle's own code.
"""
import numpy as np
import pytest

from inputs import gen
from oracle import oracle as O

I32 = lambda a: np.asarray(a, dtype=np.int32)


def single_container_requests(cpus, ram=1024):
    """One container per request, no vlinks, c^min = c^max."""
    R = len(cpus)
    return dict(n_requests=R, container_off=I32(range(R + 1)), cpu_min=I32(cpus), cpu_max=I32(cpus),
                ram_min=I32([ram] * R), ram_max=I32([ram] * R), pod_of=I32([0] * R),
                vlink_off=I32([0] * (R + 1)), vl_src=I32([]), vl_dst=I32([]), bw_min=I32([]), bw_max=I32([]))


def test_bf_consolidates_wf_spreads():
    """Fresh k=4 DC, two small requests in sequence: BF puts both on server 0 (bin packing,
    S:280), WF puts the second on server 1 (spread: server 0 is now the most loaded)."""
    snap = gen.snapshot(4, warm=False)
    reqs = single_container_requests([1000, 1000])
    bf, _, _ = O.schedule(snap, reqs, "bf", "flat", sequential=True)
    wf, _, _ = O.schedule(snap, reqs, "wf", "flat", sequential=True)
    assert bf["server_of_container"].tolist() == [0, 0]
    assert wf["server_of_container"].tolist() == [0, 1]


@pytest.mark.parametrize("seed", range(5))
def test_fit_selection_brute_force(seed):
    """BF = feasible server of smallest cpu/cpu_cap + ram/ram_cap (exact integer comparison),
    WF = largest; ties to the lowest index (R27)."""
    snap = gen.snapshot(8, 300 + seed, quantised=seed % 2 == 1)
    rng = np.random.default_rng(seed)
    dc, dr = int(rng.integers(100, 6000)), int(rng.integers(128, 60000))
    cpu = snap["cpu_res"].astype(np.int64)
    ram = snap["ram_res"].astype(np.int64)
    key = cpu * snap["ram_cap"] + ram * snap["cpu_cap"]
    feas = (cpu >= dc) & (ram >= dr)
    idx = np.nonzero(feas)[0]
    exp_bf = int(idx[np.argmin(key[idx])])   # argmin returns the first (lowest index) minimum
    exp_wf = int(idx[np.argmax(key[idx])])
    # flows are ignored by the BF/WF filter ("natively ignore the network requirements")
    flows = [(5, 900), (77, 900)]
    for m, exp in (("bf", exp_bf), ("wf", exp_wf)):
        r = O.rank(snap, m, "flat", dc, dr, flows)
        assert r["best"] == exp
        assert np.array_equal(r["mask"].astype(bool), feas)


def test_release_inverts_schedule():
    """apply then release is the identity on the state, for every method."""
    snap = gen.snapshot(8, 12)  # activity flags follow R22
    reqs = gen.requests(40, 99)
    for m in ("topsis", "ahp", "bf", "wf"):
        out, _, state = O.schedule(snap, reqs, m, "network", sequential=True)
        assert (out["status"] == 1).sum() > 30
        back = O.release(state, reqs, out)
        for key in ("cpu_res", "ram_res", "active", "link_res"):
            assert np.array_equal(back[key], snap[key]), (m, key)


def test_release_keeps_shared_server_active():
    """Two placements on one server, release one: the server stays active."""
    snap = gen.snapshot(4, warm=False)
    reqs = single_container_requests([1000, 2000])
    out, _, state = O.schedule(snap, reqs, "bf", "flat", sequential=True)
    first = dict(out, status=I32([1, 0]))  # release R0 only
    after = O.release(state, reqs, first)
    assert after["active"][0] == 1 and after["cpu_res"][0] == 24000 - 2000
    both = O.release(state, reqs, out)
    assert both["active"][0] == 0 and both["cpu_res"][0] == 24000


def tiny_timeline(hol):
    """k=2 fat-tree: 2 servers of 24 cores.  R0 (16 cores, t=0, 3 ticks), R1 (16, t=0, 1),
    R2 (16, t=1, 1), R3 (16, t=1, 2), R4 (4, t=1, 1), WF."""
    snap = gen.snapshot(2, warm=False)
    reqs = single_container_requests([16000, 16000, 16000, 16000, 4000])
    arrival = I32([0, 0, 1, 1, 1])
    duration = I32([3, 1, 1, 2, 1])
    return O.simulate(snap, reqs, arrival, duration, "wf", "flat", max_ticks=50, hol=hol)


def test_simulator_hand_worked_timeline():
    """Worked by hand: t=0 R0->s0, R1->s1 (s0 keeps 8 cores).  t=1 R1 departs first, then R2->s1;
    R3 fits nowhere (8 + 8 cores) and blocks R4 (head of line).  t=2 R2 departs; R3->s1, then
    R4->s0 (8 cores left on s0 vs 8 on s1: equal load, lowest index).  Queue empty after t=2:
    3 events (ticks); R4 is not offered at t=1 (blocked), so 6 attempts."""
    r = tiny_timeline(hol=1)
    assert r["start"].tolist() == [0, 0, 1, 2, 2]
    assert r["attempts"].tolist() == [1, 1, 1, 2, 1]
    assert r["placements"]["server_of_container"].tolist() == [0, 1, 1, 1, 0]
    assert r["totals"]["events"] == 3 and r["totals"]["attempts"] == 6 and r["totals"]["accepted"] == 5
    assert r["tick_queue"].tolist() == [0, 2, 0]
    assert r["tick_servers"].tolist() == [2, 2, 2]


def test_simulator_without_head_of_line_blocking():
    """Same workload, whole-queue scan: R4 (4 cores) passes the blocked R3 at t=1 and lands on
    s0 (8 cores left vs 8 on s1 after R2: equal, lowest index)."""
    r = tiny_timeline(hol=0)
    assert r["start"].tolist() == [0, 0, 1, 2, 1]
    assert r["placements"]["server_of_container"].tolist() == [0, 1, 1, 1, 0]
    assert r["tick_queue"].tolist() == [0, 1, 0]


@pytest.mark.parametrize("method", ["topsis", "ahp", "bf", "wf"])
def test_simulator_invariants(method):
    """Conservation, delays >= 0, one attempt at least per accepted request, and the DC empty
    again once every request has departed (fresh DC: fragmentation back to 0)."""
    snap = gen.snapshot(4, warm=False)
    reqs, arrival, duration = gen.sim_workload(60, seed=7, horizon=20, max_duration=10)
    r = O.simulate(snap, reqs, arrival, duration, method, "clustering", max_ticks=400)
    st = r["start"]
    acc = st >= 0
    assert r["totals"]["accepted"] == acc.sum()
    assert np.all(st[acc] >= arrival[acc])
    assert np.all(r["attempts"][acc] >= 1)
    assert r["totals"]["attempts"] == r["attempts"].sum()
    T = r["totals"]["events"]
    assert T == len(r["tick_queue"]) and r["tick_queue"][-1] == 0
    assert np.all(r["tick_servers"] <= 16) and np.all(r["tick_links"] <= 48)
    # run the same simulation long enough for every request to depart: the DC is empty again
    end = int((st[acc] + duration[acc]).max()) + 1
    arrival2 = np.concatenate([arrival, I32([end])])
    reqs2 = gen.subset(reqs, np.arange(60))
    one = single_container_requests([100])
    for k in ("container_off", "vlink_off"):
        reqs2[k] = np.concatenate([reqs2[k], [reqs2[k][-1] + one[k][-1]]]).astype(np.int32)
    for k in ("cpu_min", "cpu_max", "ram_min", "ram_max", "pod_of"):
        reqs2[k] = np.concatenate([reqs2[k], one[k]]).astype(np.int32)
    reqs2["n_requests"] = 61
    r2 = O.simulate(snap, reqs2, arrival2, np.concatenate([duration, I32([1])]), method, "clustering",
                    max_ticks=end + 400)
    assert r2["start"][:60].tolist() == st.tolist()
    s = r2["state"]
    # at tick `end` every request of the first 60 has departed; only the probe (100 mc) remains
    assert s["cpu_res"].sum() == 16 * 24000 - 100 and s["link_res"].sum() == 48 * 1000
