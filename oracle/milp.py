"""Brute-force optimum of the paper's MILP (Eq. 3-8) on tiny fat-trees — TEST INFRASTRUCTURE ONLY.

PAPER.md §III: minimise
    alpha * ( sum_i (1 - U(i)) + sum_ij (1 - U(ij)) )
  + (1 - alpha) * ( sum_u f_u / |N^s| + sum_uv fl_uv / |E^s| )        (Eq. 3)
subject to server capacity (Eq. 4), link capacity (Eq. 5), min-max intervals
(Eq. 6-7) and pod integrity (Eq. 8), with U(i) from Eq. 1 and U(ij) from Eq. 2
(P:122-125).  Readings (R23): E^s = the physical links (48 at k=4);
U(ij) = bw^a_ij / bw^max_ij, one rate per vlink; a vlink whose endpoints share a
server uses no link and has U = 1; paths are restricted to the ECMP shortest
paths; f_u counts every server active after placement (previously active or
hosting a container of this request), fl_uv likewise for links.

For a fixed pod->server assignment and path choice the allocation optimum is
computed exactly: CPU/RAM by the greedy fractional fill (Eq. 1 is linear and
separable per server and resource), bandwidth by scipy's LP solver.  The search
is exhaustive over assignments and path combinations, with a branch-and-bound
cut by an admissible lower bound: (1 - alpha) * |active servers| / |N^s|.
"""
from __future__ import annotations

import itertools

import numpy as np
from scipy.optimize import linprog


def fat_tree_links(k: int):
    """Explicit physical links of a k-ary fat-tree, canonical order (include/nacs.h)."""
    h, n, E = k // 2, k ** 3 // 4, k * k // 2
    links = []
    for u in range(n):
        links.append((("srv", u), ("edge", u // h)))
    for e in range(E):
        p = e // h
        for a in range(h):
            links.append((("edge", e), ("agg", p, a)))
    for p in range(k):
        for a in range(h):
            for b in range(h):
                links.append((("agg", p, a), ("core", a, b)))
    return links


def shortest_paths(k: int, u: int, v: int):
    """All shortest server-to-server paths, as lists of link ids, by BFS layering."""
    links = fat_tree_links(k)
    adj = {}
    for lid, (x, y) in enumerate(links):
        adj.setdefault(x, []).append((y, lid))
        adj.setdefault(y, []).append((x, lid))
    src, dst = ("srv", u), ("srv", v)
    dist = {src: 0}
    frontier = [src]
    while frontier and dst not in dist:
        nxt = []
        for x in frontier:
            for y, _ in adj[x]:
                if y not in dist:
                    dist[y] = dist[x] + 1
                    nxt.append(y)
        frontier = nxt
    out = []

    def walk(x, acc):
        if x == dst:
            out.append(list(acc))
            return
        for y, lid in adj[x]:
            if dist.get(y) == dist[x] + 1 and (y[0] != "srv" or y == dst):
                acc.append(lid)
                walk(y, acc)
                acc.pop()
    walk(src, [])
    return out


def _alloc_objective(snap, req, assign, vpaths, alpha):
    """Optimal Eq.3 value for a fixed pod assignment and vlink paths, or None if infeasible."""
    k = snap["k"]
    n = k ** 3 // 4
    L = 3 * k ** 3 // 4
    cmin = {"cpu": req["cpu_min"], "ram": req["ram_min"]}
    cmax = {"cpu": req["cpu_max"], "ram": req["ram_max"]}
    res = {"cpu": snap["cpu_res"], "ram": snap["ram_res"]}
    pod_of = req["pod_of"]
    nc = len(pod_of)
    util_loss = 0.0
    for r in ("cpu", "ram"):
        for u in set(assign):
            items = [i for i in range(nc) if assign[pod_of[i]] == u]
            need = sum(int(cmin[r][i]) for i in items)
            spare = int(res[r][u]) - need
            if spare < 0:
                return None  # Eq. 4 with Eq. 6 lower bounds
            # greedy fill: largest marginal utility 1/c_max first (Eq. 1 linear)
            alloc = {i: float(cmin[r][i]) for i in items}
            for i in sorted(items, key=lambda i: (cmax[r][i], i)):
                add = min(float(cmax[r][i] - cmin[r][i]), spare)
                alloc[i] += add
                spare -= add
            for i in items:
                util_loss += (1.0 - alloc[i] / float(cmax[r][i])) / 2.0  # |R| = 2
    # bandwidth LP over inter-server vlinks
    inter = [e for e in range(len(req["vl_src"]))
             if assign[pod_of[req["vl_src"][e]]] != assign[pod_of[req["vl_dst"][e]]]]
    used_links = set()
    for e in inter:
        used_links.update(vpaths[e])
    if inter:
        m = len(inter)
        bmin = np.array([req["bw_min"][e] for e in inter], float)
        bmax = np.array([req["bw_max"][e] for e in inter], float)
        rows, rhs = [], []
        for l in sorted(used_links):
            rows.append([1.0 if l in vpaths[e] else 0.0 for e in inter])
            rhs.append(float(snap["link_res"][l]))
        c = -1.0 / bmax  # maximise sum bw/bwmax
        lp = linprog(c, A_ub=np.array(rows), b_ub=np.array(rhs), bounds=list(zip(bmin, bmax)), method="highs")
        if lp.status != 0:
            return None  # Eq. 5 with Eq. 7 lower bounds
        util_loss += float(np.sum(1.0 - lp.x / bmax))
    act = np.array(snap["active"], dtype=bool).copy()
    for u in assign:
        act[u] = True
    link_active = np.array(snap["link_res"]) < snap["link_cap"]
    for l in used_links:
        link_active[l] = True
    frag = act.sum() / n + link_active.sum() / L
    return alpha * util_loss + (1.0 - alpha) * frag


def milp_optimum(snap: dict, req: dict, alpha: float, servers=None):
    """Exhaustive MILP optimum of one request (n_requests == 1).  Returns (value, assignment)."""
    k = snap["k"]
    n = k ** 3 // 4
    pod_of = [int(x) for x in req["pod_of"]]
    P = max(pod_of) + 1
    servers = list(range(n)) if servers is None else list(servers)
    pre_active = int(np.sum(snap["active"]))
    best = (float("inf"), None)
    path_cache = {}
    for assign in itertools.product(servers, repeat=P):
        act = set(assign) | set(np.nonzero(snap["active"])[0].tolist())
        bound = (1.0 - alpha) * len(act) / n
        if bound >= best[0] and best[1] is not None:
            continue
        inter = [e for e in range(len(req["vl_src"]))
                 if assign[pod_of[req["vl_src"][e]]] != assign[pod_of[req["vl_dst"][e]]]]
        choices = []
        for e in inter:
            a, b = assign[pod_of[req["vl_src"][e]]], assign[pod_of[req["vl_dst"][e]]]
            key = (min(a, b), max(a, b))
            if key not in path_cache:
                path_cache[key] = shortest_paths(k, key[0], key[1])
            choices.append(path_cache[key])
        for combo in itertools.product(*choices) if choices else [()]:
            vpaths = {e: set(p) for e, p in zip(inter, combo)}
            val = _alloc_objective(snap, req, assign, vpaths, alpha)
            if val is not None and val < best[0] - 1e-12:
                best = (val, assign)
    del pre_active
    return best


def placement_objective(snap: dict, req: dict, placement: dict, alpha: float, k: int | None = None):
    """Eq. 3 value of a heuristic placement (its own allocations and paths)."""
    k = snap["k"] if k is None else k
    n = k ** 3 // 4
    L = 3 * k ** 3 // 4
    h = k // 2
    E = k * k // 2
    srv = placement["server_of_container"]
    loss = 0.0
    for i in range(len(srv)):
        loss += (1 - placement["cpu_alloc"][i] / req["cpu_max"][i]) / 2.0
        loss += (1 - placement["ram_alloc"][i] / req["ram_max"][i]) / 2.0
    act = np.array(snap["active"], dtype=bool).copy()
    for u in srv:
        act[u] = True
    link_active = np.array(snap["link_res"]) < snap["link_cap"]
    for e in range(len(req["vl_src"])):
        loss += 1 - placement["bw_alloc"][e] / req["bw_max"][e]
        pid = placement["path_of_vlink"][e]
        if pid < 0:
            continue
        u, v = srv[req["vl_src"][e]], srv[req["vl_dst"][e]]
        link_active[u] = link_active[v] = True
        eu, ev = u // h, v // h
        if pid == 0:
            continue
        if pid <= h:
            a = pid - 1
            link_active[n + eu * h + a] = link_active[n + ev * h + a] = True
        else:
            a, b = divmod(pid - 1 - h, h)
            pu, pv = eu // h, ev // h
            link_active[n + eu * h + a] = link_active[n + ev * h + a] = True
            link_active[n + E * h + (pu * h + a) * h + b] = True
            link_active[n + E * h + (pv * h + a) * h + b] = True
    return alpha * loss + (1 - alpha) * (act.sum() / n + link_active.sum() / L)
