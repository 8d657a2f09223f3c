#!/usr/bin/env python
"""C5: fat-tree k=64 (65536 servers), sequential TOPSIS scheduling with the servers sharded
over the ranks (nacs_create_sharded + ncclAllGather of (score, index) keys per pod step).

  python scripts/bench_c5.py [--requests 100]                       # 1 GPU: unsharded, NCCL x1, loopback x8
  torchrun --nproc-per-node 8 --master-addr 127.0.0.1 scripts/bench_c5.py   # 8 GPUs, one rank each

Prints one JSON line (rank 0) with pods/s per mode; all ranks must produce identical
placements (checked with an allgather of a hash).
"""
import argparse
import hashlib
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from inputs import gen  # noqa: E402
from paper_1909_07673_b200 import nacs  # noqa: E402


def run(ctx, snap, reqs, method):
    ctx.load_topology(snap)
    torch.cuda.synchronize()
    t = time.perf_counter()
    out = ctx.schedule_request(reqs, method, "flat")
    torch.cuda.synchronize()
    el = time.perf_counter() - t
    st = ctx.last_stats()
    h = hashlib.sha256(b"".join(np.ascontiguousarray(out[k]).tobytes() for k in sorted(out))).hexdigest()
    return st["pod_steps"] / el, el, st["pod_steps"], h


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--requests", type=int, default=100)
    ap.add_argument("--method", default="topsis")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    snap = gen.snapshot(64, gen.CONFIG_SEEDS["C5"])
    reqs = gen.requests(args.requests, gen.CONFIG_SEEDS["C5"] + 1000)
    res = {}
    if world == 1:
        uid = nacs.nccl_unique_id()
        for name, shard in (("unsharded", None), ("nccl_x1", (0, 1, uid)), ("loopback_x8", (0, 8, None))):
            ctx = nacs.Context(local, shard=shard)
            run(ctx, snap, gen.subset(reqs, np.arange(min(5, args.requests))), args.method)  # warm-up
            v, el, steps, h = run(ctx, snap, reqs, args.method)
            res[name] = {"pods_per_s": v, "seconds": el, "pod_steps": steps, "hash": h[:16]}
            ctx.close()
        same = len({r["hash"] for r in res.values()}) == 1
    else:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        obj = [nacs.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ctx = nacs.Context(local, shard=(rank, world, obj[0]))
        run(ctx, snap, gen.subset(reqs, np.arange(min(5, args.requests))), args.method)
        dist.barrier()
        v, el, steps, h = run(ctx, snap, reqs, args.method)
        t = torch.tensor([el], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        hashes = [None] * world
        dist.all_gather_object(hashes, h)
        same = len(set(hashes)) == 1
        res[f"nccl_x{world}"] = {"pods_per_s": steps / float(t.item()), "seconds": float(t.item()),
                                 "pod_steps": steps, "hash": h[:16]}
        ctx.close()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps({"workload": f"C5: fat-tree k=64 (65536 servers), {args.requests} requests, sequential "
                                      f"{args.method} flat, servers sharded", "n_gpus": world, "modes": res,
                          "identical_placements": same}))


if __name__ == "__main__":
    main()
