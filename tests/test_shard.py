"""Multi-process request sharding on CPU: gloo, world size 2.  The scheduler plugged in
here is the CPU oracle (the sharding logic is host code and does not depend on it); the
GPU bench plugs in Context.schedule_batch the same way."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from inputs import gen
from paper_1909_07673_b200 import shard


def test_shard_bounds_balance_and_cover():
    reqs = gen.requests(1000, 11)
    for world in (1, 2, 3, 8):
        b = shard.shard_bounds(reqs["container_off"], world)
        assert b[0] == 0 and b[-1] == 1000 and (np.diff(b) >= 0).all()
        co = reqs["container_off"]
        loads = co[b[1:]] - co[b[:-1]]
        assert loads.max() - loads.min() <= 2 * 20  # within two requests of each other


def test_csr_block_roundtrip():
    reqs = gen.requests(50, 3)
    b = shard.shard_bounds(reqs["container_off"], 3)
    parts = [shard.csr_block(reqs, int(b[i]), int(b[i + 1])) for i in range(3)]
    for key in ("cpu_min", "pod_of", "vl_src", "bw_max"):
        assert np.array_equal(np.concatenate([p[key] for p in parts]), reqs[key])
    assert sum(p["n_requests"] for p in parts) == 50


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, snap, reqs, q):
    import torch.distributed as dist
    from oracle import oracle as O
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = shard.schedule_batch_sharded(
            reqs, lambda block: O.schedule(snap, block, "topsis", "flat", sequential=False, nthreads=1)[0],
            rank, world)
        q.put((rank, {k: v.tolist() for k, v in out.items()}))
    finally:
        dist.destroy_process_group()


def test_sharded_batch_equals_single_process():
    from oracle import oracle as O
    snap, reqs = gen.config("C2")
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, snap, reqs, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref, _, _ = O.schedule(snap, reqs, "topsis", "flat", sequential=False, nthreads=1)
    for rank in range(world):
        for key, val in ref.items():
            assert np.array_equal(np.asarray(results[rank][key]), val), (rank, key)


def test_query_shards_cover_and_keep_destinations_whole():
    g = gen.fat_tree_graph(gen.snapshot(8, 3))
    q = gen.path_queries(g, 5000, 9)
    for world in (1, 2, 3, 8):
        parts = shard.shard_queries_by_destination(q["dst"], world)
        allq = np.sort(np.concatenate(parts))
        assert np.array_equal(allq, np.arange(5000))
        owners = [set(q["dst"][p].tolist()) for p in parts]
        for a in range(world):
            for b in range(a + 1, world):
                assert not owners[a] & owners[b]  # a destination lives on one rank
        loads = [p.size for p in parts]
        assert max(loads) - min(loads) <= np.bincount(q["dst"]).max()


def _paths_worker(rank, world, port, g, q, out):
    import torch.distributed as dist
    from oracle import oracle as O
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = shard.widest_paths_sharded(
            q, lambda s, d, dm: O.graph_paths(g, s, d, dm, max_hops=8, nthreads=1), rank, world)
        out.put((rank, [x.tolist() for x in res]))
    finally:
        dist.destroy_process_group()


def test_sharded_paths_equal_single_process():
    from oracle import oracle as O
    g = gen.fat_tree_graph(gen.snapshot(4, 5))
    q = gen.path_queries(g, 400, 6, bw_hi=600)
    world = 2
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_paths_worker, args=(r, world, port, g, q, out)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(out.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = O.graph_paths(g, q["src"], q["dst"], q["demand"], max_hops=8, nthreads=1)
    for rank in range(world):
        for a, b in zip(results[rank], ref):
            assert np.array_equal(np.asarray(a), b)
