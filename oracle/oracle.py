"""ctypes wrapper of the C++ oracle (oracle/nacs_oracle.cpp) — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference arm
may import this module.  It never imports the product package and the product
never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "nacs_oracle.cpp")
LIB = os.path.join(HERE, "liboracle.so")

METHOD = {"ahp": 0, "topsis": 1, "bf": 2, "wf": 3}
# Table 4: (CPU, RAM, Fragmentation, Bandwidth)
SCHEMAS = {"flat": (0.25, 0.25, 0.25, 0.25),
           "clustering": (0.17, 0.17, 0.5, 0.16),
           "network": (0.17, 0.17, 0.16, 0.5)}


# NACS_ORACLE_SANITIZE=1: an AddressSanitizer + UndefinedBehaviorSanitizer build of the same
# source (SURVEY §4 layer 6), loaded instead; the process must preload libasan
# (tests/test_oracle_sanitized.py runs the pins that way).
SANITIZE = os.environ.get("NACS_ORACLE_SANITIZE") == "1"
SAN_LIB = os.path.join(HERE, "liboracle_san.so")


def build(force: bool = False) -> str:
    out, extra = (SAN_LIB, ["-g", "-fsanitize=address,undefined", "-fno-sanitize-recover=undefined",
                            "-fno-omit-frame-pointer"]) if SANITIZE else (LIB, [])
    if force or not os.path.exists(out) or os.path.getmtime(out) < os.path.getmtime(SRC):
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-fopenmp", "-shared", "-fPIC", *extra,
                               "-o", out, SRC])
    return out


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        P = C.c_void_p
        _lib.orc_rank.restype = C.c_int
        _lib.orc_rank.argtypes = [C.c_int] * 4 + [P] * 4 + [C.c_int, P, C.c_int, C.c_int, C.c_int,
                                                          C.c_int, C.c_int, C.c_int, P, P, C.c_int, P,
                                                          P, P, P, P, C.c_int]
        _lib.orc_ahp_priority.argtypes = [C.c_int, P, C.c_int, P]
        _lib.orc_ahp_l1.argtypes = [P, C.c_int, C.c_int, P]
        _lib.orc_widest_path.restype = C.c_int
        _lib.orc_widest_path.argtypes = [C.c_int, P, C.c_int, C.c_int, P, P, P]
        _lib.orc_schedule.restype = C.c_int
        _lib.orc_schedule.argtypes = [C.c_int] * 4 + [P] * 4 + [C.c_int, P, C.c_int, C.c_int, C.c_int,
                                                          C.c_int, C.c_int, C.c_int] + [P] * 19 + [C.c_int]
        _lib.orc_release.restype = None
        _lib.orc_release.argtypes = [C.c_int] * 4 + [P] * 4 + [C.c_int] + [P] * 17
        _lib.orc_simulate.restype = None
        _lib.orc_simulate.argtypes = ([C.c_int] * 4 + [P] * 4 + [C.c_int, P, C.c_int, C.c_int, C.c_int, C.c_int]
                                      + [P] * 13 + [C.c_int, C.c_int] + [P] * 13)
        _lib.orc_graph_paths.restype = None
        _lib.orc_graph_paths.argtypes = [C.c_int, C.c_int, P, P, P, C.c_int, P, P, P, P, P, P, C.c_int, C.c_int]
        _lib.orc_logical_bandwidth.restype = None
        _lib.orc_logical_bandwidth.argtypes = [C.c_int, C.c_int, C.c_int, P, P, P, P, C.c_int]
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _weights(w):
    if isinstance(w, str):
        w = SCHEMAS[w]
    return np.ascontiguousarray(w, dtype=np.float64)


def rank(snap: dict, method: str, weights, dem_cpu: int, dem_ram: int, flows=(), excluded=(),
         ahp_rule: int = 0, l1_mode: int = 0, path_filter: int = 1, bw_criterion: int = 0):
    """One pod step's ranking.  flows: iterable of (server v, demand D_v).  bw_criterion=1:
    the Bandwidth criterion is the logical bandwidth of R2's alternative reading."""
    k = snap["k"]
    n = k ** 3 // 4
    cpu, ram = _i32(snap["cpu_res"]), _i32(snap["ram_res"])
    act = np.ascontiguousarray(snap["active"], dtype=np.uint8)
    link = _i32(snap["link_res"])
    fv = _i32([f[0] for f in flows]) if len(flows) else np.zeros(1, np.int32)
    fd = _i32([f[1] for f in flows]) if len(flows) else np.zeros(1, np.int32)
    ex = _i32(list(excluded)) if len(excluded) else np.zeros(1, np.int32)
    w = _weights(weights)
    mask = np.zeros(n, np.uint8)
    score = np.zeros(n, np.float64)
    tie = np.zeros(n, np.uint8)
    best = np.zeros(1, np.int32)
    nf = lib().orc_rank(k, snap["cpu_cap"], snap["ram_cap"], snap["link_cap"], _p(cpu), _p(ram), _p(act),
                        _p(link), METHOD[method], _p(w), ahp_rule, l1_mode, path_filter, int(dem_cpu),
                        int(dem_ram), len(flows), _p(fv), _p(fd), len(excluded), _p(ex), _p(mask),
                        _p(score), _p(best), _p(tie), int(bw_criterion))
    return dict(mask=mask, score=score, best=int(best[0]), tie=tie, n_feasible=nf)


def ahp_priority(x, rule: int = 0) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.zeros(x.size, np.float64)
    lib().orc_ahp_priority(x.size, _p(x), rule, _p(out))
    return out


def ahp_l1(weights, ahp_rule: int = 0, l1_mode: int = 0) -> np.ndarray:
    w = _weights(weights)
    out = np.zeros(4, np.float64)
    lib().orc_ahp_l1(_p(w), ahp_rule, l1_mode, _p(out))
    return out


def widest_path(k: int, link_res, u: int, v: int):
    link = _i32(link_res)
    fab = np.zeros(1, np.float64)
    links = np.zeros(4, np.int32)
    nl = np.zeros(1, np.int32)
    pid = lib().orc_widest_path(k, _p(link), u, v, _p(fab), _p(links), _p(nl))
    return pid, float(fab[0]), links[: nl[0]].tolist()


def schedule(snap: dict, reqs: dict, method: str, weights, sequential: bool, hint=None,
             ahp_rule: int = 0, l1_mode: int = 0, path_filter: int = 1, nthreads: int | None = None,
             rank_once: bool = False):
    """Schedule a CSR batch.  Returns (placements, counters, final_state).
    rank_once: R25 (rank once per request, pods walk the order) instead of R15.

    final_state is the state after the batch (sequential) or the unchanged snapshot (batch).
    counters: pod_steps, retries, excused_ties, hint_mismatch, servers_ranked.
    """
    k = snap["k"]
    cpu, ram = _i32(snap["cpu_res"]).copy(), _i32(snap["ram_res"]).copy()
    act = np.ascontiguousarray(snap["active"], dtype=np.uint8).copy()
    link = _i32(snap["link_res"]).copy()
    R = int(reqs["n_requests"])
    Cn = int(reqs["container_off"][-1])
    Vn = int(reqs["vlink_off"][-1])
    arr = {key: _i32(reqs[key]) for key in ("container_off", "cpu_min", "cpu_max", "ram_min", "ram_max",
                                            "pod_of", "vlink_off", "vl_src", "vl_dst", "bw_min", "bw_max")}
    out = dict(status=np.zeros(R, np.int32), server_of_container=np.zeros(max(Cn, 1), np.int32),
               cpu_alloc=np.zeros(max(Cn, 1), np.int32), ram_alloc=np.zeros(max(Cn, 1), np.int32),
               bw_alloc=np.zeros(max(Vn, 1), np.int32), path_of_vlink=np.zeros(max(Vn, 1), np.int32))
    cnt = np.zeros(5, np.int64)
    hint_a = None if hint is None else _i32(hint)
    if nthreads is None:
        nthreads = len(os.sched_getaffinity(0))
    w = _weights(weights)
    lib().orc_schedule(k, snap["cpu_cap"], snap["ram_cap"], snap["link_cap"], _p(cpu), _p(ram), _p(act),
                       _p(link), METHOD[method], _p(w), ahp_rule, l1_mode, path_filter, int(rank_once),
                       int(sequential), R,
                       _p(arr["container_off"]), _p(arr["cpu_min"]), _p(arr["cpu_max"]), _p(arr["ram_min"]),
                       _p(arr["ram_max"]), _p(arr["pod_of"]), _p(arr["vlink_off"]), _p(arr["vl_src"]),
                       _p(arr["vl_dst"]), _p(arr["bw_min"]), _p(arr["bw_max"]), _p(hint_a), _p(out["status"]),
                       _p(out["server_of_container"]), _p(out["cpu_alloc"]), _p(out["ram_alloc"]),
                       _p(out["bw_alloc"]), _p(out["path_of_vlink"]), _p(cnt), int(nthreads))
    for key in ("server_of_container", "cpu_alloc", "ram_alloc"):
        out[key] = out[key][:Cn]
    for key in ("bw_alloc", "path_of_vlink"):
        out[key] = out[key][:Vn]
    counters = dict(zip(("pod_steps", "retries", "excused_ties", "hint_mismatch", "servers_ranked"),
                        cnt.tolist()))
    state = dict(snap, cpu_res=cpu, ram_res=ram, active=act, link_res=link)
    return out, counters, state


def graph_paths(graph: dict, src, dst, demand, max_hops: int | None = None, nthreads: int | None = None):
    """Widest-shortest paths on a general graph (modified Dijkstra, reading R26).
    graph: dict(n_vertices, n_servers, link_u, link_v, link_res).  Returns (bottleneck, hops,
    path[nq, max_hops + 1]) with -1 for infeasible queries and -1 padding."""
    V = int(graph["n_vertices"])
    lu, lv, lr = _i32(graph["link_u"]), _i32(graph["link_v"]), _i32(graph["link_res"])
    src, dst, dem = _i32(src), _i32(dst), _i32(demand)
    nq = src.size
    if max_hops is None:
        max_hops = V - 1
    bn = np.zeros(max(nq, 1), np.int32)
    hops = np.zeros(max(nq, 1), np.int32)
    path = np.zeros((max(nq, 1), max_hops + 1), np.int32)
    if nthreads is None:
        nthreads = len(os.sched_getaffinity(0))
    lib().orc_graph_paths(V, lu.size, _p(lu), _p(lv), _p(lr), nq, _p(src), _p(dst), _p(dem), _p(bn), _p(hops),
                          _p(path), max_hops, int(nthreads))
    return bn[:nq], hops[:nq], path[:nq]


def logical_bandwidth(graph: dict, nthreads: int | None = None) -> np.ndarray:
    """R2 alternative: per server u, sum over servers v != u of the widest-shortest
    bottleneck u -> v with every link usable; int64[n_servers]."""
    V, ns = int(graph["n_vertices"]), int(graph["n_servers"])
    lu, lv, lr = _i32(graph["link_u"]), _i32(graph["link_v"]), _i32(graph["link_res"])
    out = np.zeros(ns, np.int64)
    if nthreads is None:
        nthreads = len(os.sched_getaffinity(0))
    lib().orc_logical_bandwidth(V, ns, lu.size, _p(lu), _p(lv), _p(lr), _p(out), int(nthreads))
    return out


REQ_KEYS = ("container_off", "cpu_min", "cpu_max", "ram_min", "ram_max", "pod_of", "vlink_off", "vl_src", "vl_dst",
            "bw_min", "bw_max")
OUT_KEYS = ("status", "server_of_container", "cpu_alloc", "ram_alloc", "bw_alloc", "path_of_vlink")


def _state(snap):
    return (_i32(snap["cpu_res"]).copy(), _i32(snap["ram_res"]).copy(),
            np.ascontiguousarray(snap["active"], dtype=np.uint8).copy(), _i32(snap["link_res"]).copy())


def release(snap: dict, reqs: dict, placements: dict) -> dict:
    """Departure of every accepted request (status 1): the state after releasing them."""
    cpu, ram, act, link = _state(snap)
    arr = [_i32(reqs[k]) for k in REQ_KEYS]
    out = [_i32(placements[k]) for k in OUT_KEYS]
    lib().orc_release(snap["k"], snap["cpu_cap"], snap["ram_cap"], snap["link_cap"], _p(cpu), _p(ram), _p(act),
                      _p(link), int(reqs["n_requests"]), *[_p(a) for a in arr], *[_p(a) for a in out])
    return dict(snap, cpu_res=cpu, ram_res=ram, active=act, link_res=link)


def simulate(snap: dict, reqs: dict, arrival, duration, method: str, weights, max_ticks: int, hol: int = 1,
             hint=None, ahp_rule: int = 0, l1_mode: int = 0, path_filter: int = 1) -> dict:
    """Discrete-event simulation (reading R28).  Returns per-request start / attempts / status,
    the final placements, per-tick series and totals."""
    cpu, ram, act, link = _state(snap)
    R = int(reqs["n_requests"])
    Cn, Vn = int(reqs["container_off"][-1]), int(reqs["vlink_off"][-1])
    arr = [_i32(reqs[k]) for k in REQ_KEYS]
    start, attempts, status = (np.zeros(max(R, 1), np.int32) for _ in range(3))
    server, cpu_a, ram_a = (np.zeros(max(Cn, 1), np.int32) for _ in range(3))
    bw_a, path = np.zeros(max(Vn, 1), np.int32), np.zeros(max(Vn, 1), np.int32)
    ts, tl, tq = (np.zeros(max_ticks, np.int32) for _ in range(3))
    tot = np.zeros(7, np.int64)
    hint_a = None if hint is None else _i32(hint)
    lib().orc_simulate(snap["k"], snap["cpu_cap"], snap["ram_cap"], snap["link_cap"], _p(cpu), _p(ram), _p(act),
                       _p(link), METHOD[method], _p(_weights(weights)), ahp_rule, l1_mode, path_filter, R,
                       *[_p(a) for a in arr], _p(_i32(arrival)), _p(_i32(duration)), int(max_ticks), int(hol),
                       _p(hint_a), _p(start), _p(attempts), _p(status), _p(server), _p(cpu_a), _p(ram_a), _p(bw_a),
                       _p(path), _p(ts), _p(tl), _p(tq), _p(tot))
    T = int(tot[0])
    return dict(start=start[:R], attempts=attempts[:R], status=status[:R],
                placements=dict(status=status[:R], server_of_container=server[:Cn], cpu_alloc=cpu_a[:Cn],
                                ram_alloc=ram_a[:Cn], bw_alloc=bw_a[:Vn], path_of_vlink=path[:Vn]),
                tick_servers=ts[:T], tick_links=tl[:T], tick_queue=tq[:T],
                totals=dict(zip(("events", "attempts", "accepted", "pod_steps", "retries", "excused_ties",
                                 "hint_mismatch"), tot.tolist())),
                state=dict(snap, cpu_res=cpu, ram_res=ram, active=act, link_res=link))
