"""Request sharding across ranks (one process per GPU), host logic only.

Requests of a batch are independent under snapshot isolation (R21), so a batch
shards across ranks with no data-path collective: every rank schedules a contiguous
block of requests on its own GPU, and the placements are gathered once at the end.
Blocks are balanced by container count (the work of a request grows with its pods).
"""
from __future__ import annotations

import numpy as np

REQ_C = ("cpu_min", "cpu_max", "ram_min", "ram_max", "pod_of")
REQ_V = ("vl_src", "vl_dst", "bw_min", "bw_max")
OUT_R = ("status",)
OUT_C = ("server_of_container", "cpu_alloc", "ram_alloc")
OUT_V = ("bw_alloc", "path_of_vlink")


def shard_bounds(container_off: np.ndarray, world: int) -> np.ndarray:
    """Request boundaries [b_0=0, ..., b_world=R] splitting the batch into `world` contiguous
    blocks of (nearly) equal container count."""
    co = np.asarray(container_off, dtype=np.int64)
    R = co.size - 1
    targets = co[-1] * np.arange(world + 1) / world
    b = np.searchsorted(co, targets, side="left").astype(np.int64)
    b[0], b[-1] = 0, R
    return np.maximum.accumulate(np.clip(b, 0, R))


def csr_block(reqs: dict, r0: int, r1: int) -> dict:
    """Requests r0..r1-1 of a CSR batch as their own batch (offsets rebased to 0)."""
    co = np.asarray(reqs["container_off"], dtype=np.int64)
    vo = np.asarray(reqs["vlink_off"], dtype=np.int64)
    c0, c1, v0, v1 = co[r0], co[r1], vo[r0], vo[r1]
    out = {"n_requests": int(r1 - r0),
           "container_off": np.ascontiguousarray(co[r0:r1 + 1] - c0, dtype=np.int32),
           "vlink_off": np.ascontiguousarray(vo[r0:r1 + 1] - v0, dtype=np.int32)}
    for k in REQ_C:
        out[k] = np.ascontiguousarray(reqs[k][c0:c1], dtype=np.int32)
    for k in REQ_V:
        out[k] = np.ascontiguousarray(reqs[k][v0:v1], dtype=np.int32)
    return out


def _np(x):
    return x.cpu().numpy() if hasattr(x, "cpu") else np.asarray(x)


def schedule_batch_sharded(reqs: dict, schedule, rank: int, world: int, group=None) -> dict:
    """Schedule a batch across `world` ranks and return the full placements on every rank.

    schedule(block) -> placements dict for this rank's block (e.g. a bound
    `Context.schedule_batch`).  Uses torch.distributed all_gather_object when world > 1.
    """
    b = shard_bounds(reqs["container_off"], world)
    mine = schedule(csr_block(reqs, int(b[rank]), int(b[rank + 1])))
    mine = {k: _np(v) for k, v in mine.items()}
    if world == 1:
        parts = [mine]
    else:
        import torch.distributed as dist
        parts = [None] * world
        dist.all_gather_object(parts, mine, group=group)
    out = {k: np.concatenate([p[k] for p in parts]).astype(np.int32)
           for k in OUT_R + OUT_C + OUT_V}
    return out


# ---------------------------------------------------------------------------------------
# Path queries (general topology): queries are independent, and the GPU
# answers all queries to one destination from one BFS, so they shard by
# DESTINATION: each rank owns whole destination groups and no BFS is repeated across ranks.
# ---------------------------------------------------------------------------------------

def shard_queries_by_destination(dst: np.ndarray, world: int) -> list[np.ndarray]:
    """Per-rank query index arrays (ascending): destination groups assigned largest-first to
    the least-loaded rank (deterministic: ties by destination id, then rank id)."""
    dst = np.asarray(dst, dtype=np.int64)
    if world == 1:
        return [np.arange(dst.size)]
    ids, counts = np.unique(dst, return_counts=True)
    order = np.lexsort((ids, -counts))
    load = np.zeros(world, np.int64)
    owner = np.empty(ids.size, np.int64)
    for g in order:
        r = int(np.argmin(load))
        owner[g] = r
        load[r] += counts[g]
    rank_of_query = owner[np.searchsorted(ids, dst)]
    return [np.nonzero(rank_of_query == r)[0] for r in range(world)]


def widest_paths_sharded(q: dict, solve, rank: int, world: int, group=None):
    """Answer the queries q = dict(src, dst, demand) across `world` ranks; every rank returns
    the full (bottleneck, hops, path).  solve(src, dst, demand) -> (bn, hops, path) for this
    rank's queries (e.g. a bound Context.widest_paths)."""
    parts_idx = shard_queries_by_destination(q["dst"], world)
    idx = parts_idx[rank]
    mine = solve(*(np.ascontiguousarray(np.asarray(q[k])[idx], dtype=np.int32) for k in ("src", "dst", "demand")))
    mine = tuple(_np(x) for x in mine)
    if world == 1:
        parts = [mine]
    else:
        import torch.distributed as dist
        parts = [None] * world
        dist.all_gather_object(parts, mine, group=group)
    n = np.asarray(q["src"]).size
    bn = np.empty(n, np.int32)
    hops = np.empty(n, np.int32)
    path = np.empty((n, parts[0][2].shape[1]), np.int32)
    for r in range(world):
        ir = parts_idx[r]
        bn[ir], hops[ir], path[ir] = parts[r][0], parts[r][1], parts[r][2]
    return bn, hops, path
