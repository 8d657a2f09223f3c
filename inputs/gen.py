"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds NO arithmetic of the method (no filtering, scoring, selection or
commit).  It only draws integers with numpy's PCG64 and lays them out in the
C-ABI's structure-of-arrays / CSR form (include/nacs.h).  The recipe follows
SURVEY.md §8(d) "Inputs", which takes its magnitudes from the paper:

* homogeneous servers of 24 cores and 256 GB, every link 1 Gbps
  (§IV-B1 and PAPER.md:396 §VI-A), stored in integer units:
  CPU in millicores, RAM in MiB, bandwidth in Mbps (reading R5);
* a k-ary fat-tree with k^3/4 servers (§IV-B1);
* containers with CPU "up to 2" cores and RAM "up to 4" GB
  (§IV-B2), up to 50% of containers grouped in pods and
  pair bandwidth up to 50 Mbps (§VI-A); 4-20 containers per
  request.

Canonical link order (include/nacs.h): access[n] | edge-agg[E][h] | agg-core[k][h][h]
with h = k/2, E = k^2/2 edge switches, server u under edge switch u // h,
edge switch e in fat-tree pod e // h.
"""
from __future__ import annotations

import numpy as np

CPU_CAP = 24000     # millicores: 24 cores
RAM_CAP = 262144    # MiB: 256 GB
LINK_CAP = 1000     # Mbps: 1 Gbps

CONFIG_SEEDS = {"C1": 1, "C2": 2, "C3": 3, "C4": 4, "C5": 5}
CONFIG_K = {"C1": 4, "C2": 8, "C3": 16, "C4": 32, "C5": 64}
CONFIG_REQUESTS = {"C1": 1, "C2": 100, "C3": 10_000, "C4": 100_000, "C5": 1000}


def sizes(k: int) -> dict:
    """Fat-tree sizes: n servers, h = k/2, E edge switches, L physical links."""
    if k < 2 or k % 2:
        raise ValueError("k must be even and >= 2")
    h = k // 2
    return {"k": k, "h": h, "n": k ** 3 // 4, "E": k * k // 2, "L": 3 * k ** 3 // 4}


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def snapshot(k: int, seed: int | None = None, warm: bool = True, quantised: bool = False,
             p_active: float = 0.6, cpu_cap: int = CPU_CAP, ram_cap: int = RAM_CAP,
             link_cap: int = LINK_CAP) -> dict:
    """A DC state G^s(N^s, E^s): residual c^s_u[r] per server and residual per link.

    fresh (warm=False): every residual equals its capacity, no server active.
    warm: each server is active with probability p_active and then has used CPU
    ~U{100..cpu_cap} and used RAM ~U{128..ram_cap}; every link has used
    bandwidth ~U{0..950} (SURVEY.md §8(d) "Snapshots").  quantised: CPU residual
    rounded down to a multiple of 1000 and RAM to a multiple of 8192, which
    creates exactly equal criteria rows (ties).
    active_u = 1 iff some residual is below capacity (reading R22).
    """
    s = sizes(k)
    n, L = s["n"], s["L"]
    cpu = np.full(n, cpu_cap, dtype=np.int32)
    ram = np.full(n, ram_cap, dtype=np.int32)
    link = np.full(L, link_cap, dtype=np.int32)
    if warm:
        rng = _rng(seed)
        act = rng.random(n) < p_active
        used_cpu = rng.integers(100, cpu_cap, size=n, endpoint=True)
        used_ram = rng.integers(128, ram_cap, size=n, endpoint=True)
        cpu = np.where(act, cpu_cap - used_cpu, cpu_cap).astype(np.int32)
        ram = np.where(act, ram_cap - used_ram, ram_cap).astype(np.int32)
        if quantised:
            cpu = (cpu // 1000 * 1000).astype(np.int32)
            ram = (ram // 8192 * 8192).astype(np.int32)
        link = (link_cap - rng.integers(0, min(950, link_cap), size=L, endpoint=True)).astype(np.int32)
    active = ((cpu < cpu_cap) | (ram < ram_cap)).astype(np.uint8)
    return dict(k=k, cpu_cap=cpu_cap, ram_cap=ram_cap, link_cap=link_cap,
                cpu_res=cpu, ram_res=ram, active=active, link_res=link)


def _segment_ids(counts: np.ndarray) -> np.ndarray:
    return np.repeat(np.arange(counts.size, dtype=np.int64), counts)


def requests(n_req: int, seed: int, nc_lo: int = 4, nc_hi: int = 20, cpu_max_hi: int = 2000,
             ram_max_hi: int = 4096, bw_max_hi: int = 50, extra_edges: int = 0,
             bw_one: bool = False) -> dict:
    """A batch of Req(N^c, E^c) in CSR form (§II-A, Table 1).

    Per request: |N^c| ~ U{nc_lo..nc_hi}; per container c^max_CPU ~ U{100..2000}
    millicores, c^min_CPU ~ U{100..c^max}; c^max_RAM ~ U{128..4096} MiB,
    c^min_RAM ~ U{128..c^max}.  g ~ U{0..floor(|N^c|/2)} containers (a random
    subset, paired in draw order) form 2-container pods, the rest are singleton
    pods; pod ids are numbered by each pod's lowest container index, which is
    also the placement order.  Virtual links form a random tree (container i's
    parent is uniform over 0..i-1) plus `extra_edges` random extra pairs;
    bw^max ~ U{1..50} Mbps, bw^min ~ U{1..bw^max}; bw_one sets both to 1
    (the paper's 1 Mbps scenario).
    """
    rng = _rng(seed)
    nc = rng.integers(nc_lo, nc_hi, size=n_req, endpoint=True).astype(np.int64)
    C = int(nc.sum())
    coff = np.zeros(n_req + 1, dtype=np.int64)
    np.cumsum(nc, out=coff[1:])
    req_of = _segment_ids(nc)
    local = np.arange(C, dtype=np.int64) - coff[req_of]

    cpu_max = rng.integers(100, cpu_max_hi, size=C, endpoint=True)
    cpu_min = rng.integers(100, cpu_max, endpoint=True)
    ram_max = rng.integers(128, ram_max_hi, size=C, endpoint=True)
    ram_min = rng.integers(128, ram_max, endpoint=True)

    # pods: g containers of each request, chosen by a random permutation, are paired
    g = rng.integers(0, nc // 2, endpoint=True)
    keys = rng.random(C)
    order = np.lexsort((keys, req_of))            # random permutation inside each request
    rank_in_req = np.empty(C, dtype=np.int64)
    rank_in_req[order] = np.arange(C) - coff[req_of[order]]
    paired = rank_in_req < 2 * (g[req_of] // 2)
    # partner: positions 2t and 2t+1 of the permutation form a pod
    leader = local.copy()
    pos = order  # order[coff[r] + j] = global container id at permutation position j
    perm_pos = coff[req_of] + rank_in_req
    partner_pos = np.where(rank_in_req % 2 == 0, perm_pos + 1, perm_pos - 1)
    partner_pos = np.clip(partner_pos, 0, C - 1)
    partner_local = local[pos[partner_pos]]
    leader = np.where(paired, np.minimum(local, partner_local), local)
    is_leader = leader == local
    # pod id = rank of the leader among the request's leaders (ascending container index)
    incl = np.cumsum(is_leader)                      # leaders up to and including each container
    base = np.concatenate([[0], incl])[coff[:-1]]    # leaders before each request
    leader_global = coff[req_of] + leader
    pod_of = incl[leader_global] - 1 - base[req_of]

    # virtual links: random tree plus extras
    nv_tree = nc - 1
    nv = nv_tree + extra_edges
    V = int(nv.sum())
    voff = np.zeros(n_req + 1, dtype=np.int64)
    np.cumsum(nv, out=voff[1:])
    vreq = _segment_ids(nv)
    vloc = np.arange(V, dtype=np.int64) - voff[vreq]
    is_tree = vloc < nv_tree[vreq]
    child = vloc + 1
    u01 = rng.random(V)
    parent = np.floor(u01 * child).astype(np.int64)
    ex_a = np.floor(rng.random(V) * nc[vreq]).astype(np.int64)
    ex_b = (ex_a + 1 + np.floor(rng.random(V) * (nc[vreq] - 1)).astype(np.int64)) % nc[vreq]
    vsrc = np.where(is_tree, parent, ex_a)
    vdst = np.where(is_tree, child, ex_b)
    if bw_one:
        bw_max = np.ones(V, dtype=np.int64)
        bw_min = np.ones(V, dtype=np.int64)
    else:
        bw_max = rng.integers(1, bw_max_hi, size=V, endpoint=True)
        bw_min = rng.integers(1, bw_max, endpoint=True)

    i32 = lambda a: np.ascontiguousarray(a, dtype=np.int32)
    return dict(n_requests=n_req, container_off=i32(coff), cpu_min=i32(cpu_min), cpu_max=i32(cpu_max),
                ram_min=i32(ram_min), ram_max=i32(ram_max), pod_of=i32(pod_of),
                vlink_off=i32(voff), vl_src=i32(vsrc), vl_dst=i32(vdst), bw_min=i32(bw_min),
                bw_max=i32(bw_max))


def c1_request(seed: int = CONFIG_SEEDS["C1"]) -> dict:
    """C1: one request of 6 containers in 3 pods of 2 ({0,1},{2,3},{4,5}), tree vlinks."""
    rng = _rng(seed)
    cpu_max = rng.integers(100, 2000, size=6, endpoint=True)
    cpu_min = rng.integers(100, cpu_max, endpoint=True)
    ram_max = rng.integers(128, 4096, size=6, endpoint=True)
    ram_min = rng.integers(128, ram_max, endpoint=True)
    child = np.arange(1, 6)
    parent = np.floor(rng.random(5) * child).astype(np.int64)
    bw_max = rng.integers(1, 50, size=5, endpoint=True)
    bw_min = rng.integers(1, bw_max, endpoint=True)
    i32 = lambda a: np.ascontiguousarray(a, dtype=np.int32)
    return dict(n_requests=1, container_off=i32([0, 6]), cpu_min=i32(cpu_min), cpu_max=i32(cpu_max),
                ram_min=i32(ram_min), ram_max=i32(ram_max), pod_of=i32([0, 0, 1, 1, 2, 2]),
                vlink_off=i32([0, 5]), vl_src=i32(parent), vl_dst=i32(child), bw_min=i32(bw_min),
                bw_max=i32(bw_max))


def subset(reqs: dict, idx) -> dict:
    """Requests `idx` (ascending indices) of a batch, re-packed as their own CSR batch."""
    idx = np.asarray(idx, dtype=np.int64)
    co, vo = reqs["container_off"].astype(np.int64), reqs["vlink_off"].astype(np.int64)
    cidx = np.concatenate([np.arange(co[i], co[i + 1]) for i in idx]) if idx.size else np.zeros(0, np.int64)
    vidx = np.concatenate([np.arange(vo[i], vo[i + 1]) for i in idx]) if idx.size else np.zeros(0, np.int64)
    ncs = co[idx + 1] - co[idx]
    nvs = vo[idx + 1] - vo[idx]
    out = dict(n_requests=int(idx.size))
    out["container_off"] = np.concatenate([[0], np.cumsum(ncs)]).astype(np.int32)
    out["vlink_off"] = np.concatenate([[0], np.cumsum(nvs)]).astype(np.int32)
    for key in ("cpu_min", "cpu_max", "ram_min", "ram_max", "pod_of"):
        out[key] = np.ascontiguousarray(reqs[key][cidx], dtype=np.int32)
    for key in ("vl_src", "vl_dst", "bw_min", "bw_max"):
        out[key] = np.ascontiguousarray(reqs[key][vidx], dtype=np.int32)
    return out


def config(name: str) -> tuple[dict, dict]:
    """(snapshot, requests) of a BASELINE.json config C1..C5 (SURVEY.md §8(d) "Configs")."""
    k = CONFIG_K[name]
    seed = CONFIG_SEEDS[name]
    if name == "C1":
        return snapshot(k, warm=False), c1_request(seed)
    snap = snapshot(k, seed)
    return snap, requests(CONFIG_REQUESTS[name], seed + 1000)


# ---------------------------------------------------------------------------
# General topologies: G^s(N^s, E^s) as an explicit undirected
# graph, vertices 0..n_servers-1 are the servers (§II-A: "N^s ... all servers
# and switches", E^s "all physical links").  Only layout and random draws here.
# ---------------------------------------------------------------------------

def fat_tree_graph(snap: dict) -> dict:
    """The fat-tree of `snap` as an explicit graph.  Vertex ids: servers 0..n-1, edge
    switch e at n + e, aggregation switch a of pod p at n + E + p*h + a, core switch (a, b)
    at n + E + k*h + a*h + b.  Link l is the canonical link l of include/nacs.h, so
    link_res is the snapshot's link_res unchanged."""
    s = sizes(int(snap["k"]))
    k, h, n, E = s["k"], s["h"], s["n"], s["E"]
    agg0, core0 = n + E, n + E + k * h
    u = np.arange(n)
    acc_u, acc_v = u, n + u // h
    e, a = np.divmod(np.arange(E * h), h)
    ea_u, ea_v = n + e, agg0 + (e // h) * h + a
    p, ab = np.divmod(np.arange(k * h * h), h * h)
    a2, b2 = np.divmod(ab, h)
    ac_u, ac_v = agg0 + p * h + a2, core0 + a2 * h + b2
    i32 = lambda x: np.ascontiguousarray(x, dtype=np.int32)
    return dict(n_vertices=n + E + k * h + h * h, n_servers=n,
                link_u=i32(np.concatenate([acc_u, ea_u, ac_u])), link_v=i32(np.concatenate([acc_v, ea_v, ac_v])),
                link_res=i32(snap["link_res"]), link_cap=int(snap["link_cap"]))


def random_graph(n_switches: int, degree: int, servers_per_switch: int, seed: int, warm: bool = True,
                 link_cap: int = LINK_CAP) -> dict:
    """A Jellyfish-style DC: a random `degree`-regular graph over the switches (configuration
    model; the stubs of self-loops and repeated pairs are re-paired with random other pairs
    until the graph is simple) with `servers_per_switch` servers on each switch.  Vertex ids:
    servers 0..ns-1 (server s on switch s // servers_per_switch), switches ns.. .  Residuals
    ~ link_cap - U{0..950} when warm (as the fat-tree snapshots), else link_cap."""
    if (n_switches * degree) % 2 or degree >= n_switches:
        raise ValueError("need n_switches * degree even and degree < n_switches")
    rng = _rng(seed)
    ns = n_switches * servers_per_switch
    stubs = rng.permutation(np.repeat(np.arange(n_switches), degree))
    while True:
        a, b = stubs[0::2], stubs[1::2]
        lo, hi = np.minimum(a, b), np.maximum(a, b)
        key = lo * n_switches + hi
        _, first = np.unique(key, return_index=True)
        bad = np.ones(key.size, bool)
        bad[first] = False
        bad |= lo == hi
        if not bad.any():
            break
        # re-pair the stubs of the bad pairs together with as many random good pairs
        redo = np.nonzero(bad)[0]
        good = np.nonzero(~bad)[0]
        redo = np.concatenate([redo, rng.choice(good, size=min(good.size, redo.size), replace=False)])
        pos = np.concatenate([2 * redo, 2 * redo + 1])
        stubs[pos] = rng.permutation(stubs[pos])
    srv = np.arange(ns)
    lu = np.concatenate([srv, ns + lo])
    lv = np.concatenate([ns + srv // servers_per_switch, ns + hi])
    res = np.full(lu.size, link_cap, dtype=np.int64)
    if warm:
        res = link_cap - rng.integers(0, min(950, link_cap), size=lu.size, endpoint=True)
    i32 = lambda x: np.ascontiguousarray(x, dtype=np.int32)
    return dict(n_vertices=ns + n_switches, n_servers=ns, link_u=i32(lu), link_v=i32(lv), link_res=i32(res),
                link_cap=link_cap)


def path_queries(graph: dict, n_queries: int, seed: int, bw_hi: int = 50) -> dict:
    """(src, dst, demand) server pairs, src != dst, demand ~ U{1..bw_hi} Mbps (the pair
    bandwidth "up to 50 Mbps")."""
    rng = _rng(seed)
    ns = int(graph["n_servers"])
    src = rng.integers(0, ns, size=n_queries)
    dst = (src + rng.integers(1, ns, size=n_queries)) % ns
    dem = rng.integers(1, bw_hi, size=n_queries, endpoint=True)
    i32 = lambda x: np.ascontiguousarray(x, dtype=np.int32)
    return dict(src=i32(src), dst=i32(dst), demand=i32(dem))



# ---------------------------------------------------------------------------
# Discrete-event workload: the E2 campaign of P:396-398 — a fresh
# k=20 fat-tree, 6000 requests of 4 containers "with a running time up to 250 events from a
# complete execution of 500 events", up to 50% of containers in pods, pair bandwidth up to
# 50 Mbps.  Arrival ticks ~U{0..horizon-1}, durations ~U{1..max_duration} (reading R28).
# ---------------------------------------------------------------------------

def sim_workload(n_req: int = 6000, seed: int = 6, horizon: int = 500, max_duration: int = 250,
                 n_containers: int = 4) -> tuple[dict, np.ndarray, np.ndarray]:
    reqs = requests(n_req, seed, nc_lo=n_containers, nc_hi=n_containers)
    rng = _rng(seed + 500)
    arrival = rng.integers(0, horizon, size=n_req).astype(np.int32)
    duration = rng.integers(1, max_duration, size=n_req, endpoint=True).astype(np.int32)
    return reqs, arrival, duration
