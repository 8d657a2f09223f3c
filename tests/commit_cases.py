"""Hand-built k=4 cases for readings R17 (flow aggregation), R18 (exclude-and-redo) and
R19 (request-end top-up) — inputs only, plus the values worked out by hand in each
docstring.  Used by the oracle pins (tests/test_oracle_commit_pins.py, CPU) and by the
GPU parity tests (tests/test_gpu_parity2.py), so the same hand-derived expectations bind
both sides.

k = 4: h = 2, n = 16 servers, E = 8 edge switches; server u under edge u // 2, edge e in
fat-tree pod e // 2.  Canonical links: access u -> u; edge-agg (e, a) -> 16 + 2e + a;
agg-core (pod, a, b) -> 32 + 2(2 pod + a) + b.  Path ids: -1 intra-server, 0 same edge,
1 + a same pod, 1 + h + a h + b = 3 + 2a + b cross pod (include/nacs.h).
"""
from __future__ import annotations

import numpy as np

from inputs import gen

K = 4
N = 16


def access(u):
    return u


def edge_agg(e, a):
    return 16 + 2 * e + a


def agg_core(pod, a, b):
    return 32 + 2 * (2 * pod + a) + b


def cross_path_links(e1, e2, a, b):
    """Fabric links of the cross-pod path edge e1 -> agg a -> core (a, b) -> agg a -> edge e2."""
    return [edge_agg(e1, a), edge_agg(e2, a), agg_core(e1 // 2, a, b), agg_core(e2 // 2, a, b)]


def snapshot(servers: dict, fabric=None, default_fabric=1000):
    """A k=4 DC where only the servers in `servers` (u -> (cpu, ram)) have CPU; every other
    server has cpu 0 (never feasible for a positive demand).  fabric: {link: residual}."""
    s = gen.snapshot(K, warm=False)
    s["cpu_res"][:] = 0
    for u, (c, r) in servers.items():
        s["cpu_res"][u], s["ram_res"][u] = c, r
    s["active"] = ((s["cpu_res"] < s["cpu_cap"]) | (s["ram_res"] < s["ram_cap"])).astype(np.uint8)
    s["link_res"][N:] = default_fabric
    for l, v in (fabric or {}).items():
        s["link_res"][l] = v
    return s


def request(containers, vlinks):
    """One CSR request.  containers: (cpu_min, cpu_max, ram_min, ram_max, pod) per container;
    vlinks: (src, dst, bw_min, bw_max)."""
    i32 = lambda x: np.asarray(x, np.int32)
    nC, nV = len(containers), len(vlinks)
    return {"n_requests": 1, "container_off": i32([0, nC]),
            "cpu_min": i32([c[0] for c in containers]), "cpu_max": i32([c[1] for c in containers]),
            "ram_min": i32([c[2] for c in containers]), "ram_max": i32([c[3] for c in containers]),
            "pod_of": i32([c[4] for c in containers]), "vlink_off": i32([0, nV]),
            "vl_src": i32([v[0] for v in vlinks]), "vl_dst": i32([v[1] for v in vlinks]),
            "bw_min": i32([v[2] for v in vlinks]), "bw_max": i32([v[3] for v in vlinks])}


def r17_case():
    """R17: the vlinks from pod p to placed pods hosted on one server v form ONE flow D_v
    routed on ONE path.

    Pods 0 and 1 fit only server 0 (RAM 1000 each; server 15 has RAM 500) and share it; pod 2
    (5000 mc) fits only server 15 (edge 7, fat-tree pod 3).  Pod 2's vlinks to pods 0 and 1
    (300 + 400 Mbps) are one flow D_0 = 700.  Fabric: every link 600 except the four links of
    the cross path (a=1, b=1) from edge 7 to edge 0, at 800 — the only path >= 700.

    Expected: accepted, servers (0, 0, 15); both vlinks on path 3 + 2*1 + 1 = 6; the four
    links of that path end at 800 - 700 = 100 and both access links at 1000 - 700 = 300.
    Per-peer-pod flows (the plausible mistake) would route 300 on the 800 path (-> 500) and
    then 400 on a 600 path: two different path ids."""
    path = cross_path_links(0, 7, 1, 1)
    snap = snapshot({0: (2000, 2000), 15: (5000, 500)}, fabric={l: 800 for l in path}, default_fabric=600)
    req = request([(500, 500, 1000, 1000, 0), (500, 500, 1000, 1000, 1), (5000, 5000, 100, 100, 2)],
                  [(0, 2, 300, 300), (1, 2, 400, 400)])
    expect = {"status": [1], "server_of_container": [0, 0, 15], "path_of_vlink": [6, 6], "bw_alloc": [300, 400],
              "links": {**{l: 100 for l in path}, access(0): 300, access(15): 300}, "retries": 0}
    return snap, req, expect


def r18_case():
    """R18: a commit whose flows conflict on a fabric link excludes u* and redoes the pod step.

    Pod 0 fits only server 0 (RAM 3000), pod 1 only server 2 (RAM 2000; server 0 then has no
    CPU).  Pod 2 (5000 mc, RAM 100) has flows to server 0 (300) and server 2 (300) and two
    feasible servers: 14 (edge 7, pod 3) and 4 (edge 2, pod 1).  Server 14 dominates 4 in
    CPU, RAM and access bandwidth (both active), so both methods rank 14 first.  Edge 7's
    uplinks: (7, a=0) = 500, (7, a=1) = 0, everything else 1000.  Each flow alone fits
    (500 >= 300), so 14 passes the filter; the commit routes v=0 via a=0 (500 -> 200) and
    then finds at most 200 < 300 towards edge 1: failure, 14 is excluded, the redo picks 4.
    From edge 2 every path is 1000: v=0 takes (a=0, b=0) = path 3; then towards edge 1
    (a=0, b=0) is 700, (a=0, b=1) 700 (edge 2's uplink 0), (a=1, b=0) 1000: path 3+2 = 5.

    Expected: accepted, servers (0, 2, 4), paths (3, 5), one retry.  Rejecting the request on
    the first routing failure (the plausible mistake) gives status 0."""
    snap = snapshot({0: (1000, 3000), 2: (1000, 2000), 14: (20000, 1500), 4: (10000, 1400)},
                    fabric={edge_agg(7, 0): 500, edge_agg(7, 1): 0})
    snap["link_res"][access(4)] = 900
    snap["active"][4] = snap["active"][14] = 1
    req = request([(1000, 1000, 3000, 3000, 0), (1000, 1000, 2000, 2000, 1), (5000, 5000, 100, 100, 2)],
                  [(0, 2, 300, 300), (1, 2, 300, 300)])
    expect = {"status": [1], "server_of_container": [0, 2, 4], "path_of_vlink": [3, 5], "bw_alloc": [300, 300],
              "links": {edge_agg(7, 0): 500, edge_agg(7, 1): 0, access(14): 1000, access(4): 300,
                        edge_agg(2, 0): 700, edge_agg(2, 1): 700, edge_agg(0, 0): 700, edge_agg(1, 1): 700},
              "retries": 1}
    return snap, req, expect


def r19_case():
    """R19: at request end containers are topped up in index order, then vlinks in index
    order, each vlink by at most the minimum residual along its path.

    Pod 0 = containers 0, 1 (c^min 1000 + 1000, RAM 1000 + 1000) fits only server 0 (CPU 2300;
    server 15 has RAM 1500 < 2000); pod 1 = container 2 (3000 mc) fits only server 15.  Every
    fabric link is 230, so all four cross paths edge 7 -> edge 0 tie and (a=0, b=0) = path 3
    carries the flow D_0 = 10 + 20.  At request end server 0 has 2300 - 2000 = 300 mc left:
    container 0 (wants 200) gets 200, container 1 (wants 500) gets the last 100 ->
    c^a = (1200, 1100).  The path has 230 - 30 = 200 left on its fabric links (970 on the
    access links): vlink 0 (wants 490) gets 200 -> 210, vlink 1 (wants 280) gets 0 -> 20.

    Plausible mistakes: reverse container order -> (1000, 1300); reverse vlink order ->
    (10, 220); access links only -> (500, 300)."""
    snap = snapshot({0: (2300, 5000), 15: (3000, 1500)}, default_fabric=230)
    req = request([(1000, 1200, 1000, 1000, 0), (1000, 1500, 1000, 1000, 0), (3000, 3000, 100, 100, 1)],
                  [(0, 2, 10, 500), (1, 2, 20, 300)])
    path = cross_path_links(0, 7, 0, 0)
    expect = {"status": [1], "server_of_container": [0, 0, 15], "cpu_alloc": [1200, 1100, 3000],
              "path_of_vlink": [3, 3], "bw_alloc": [210, 20],
              "links": {**{l: 0 for l in path}, access(0): 1000 - 230, access(15): 1000 - 230},
              "cpu_res": {0: 0, 15: 0}, "retries": 0}
    return snap, req, expect


CASES = {"R17": r17_case, "R18": r18_case, "R19": r19_case}


def check(expect, out, state, retries, label=""):
    """Compare a placement (and the final state of a sequential run) with the hand values."""
    for key in ("status", "server_of_container", "path_of_vlink", "bw_alloc", "cpu_alloc"):
        if key in expect:
            got = np.asarray(out[key]).tolist()[: len(expect[key])]
            assert got == expect[key], (label, key, got, expect[key])
    for l, v in (expect.get("links", {}) if state is not None else {}).items():
        assert int(state["link_res"][l]) == v, (label, "link", l, int(state["link_res"][l]), v)
    for u, v in (expect.get("cpu_res", {}) if state is not None else {}).items():
        assert int(state["cpu_res"][u]) == v, (label, "cpu_res", u)
    if retries is not None:
        assert retries == expect["retries"], (label, "retries", retries)
