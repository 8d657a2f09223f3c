"""Cold-snapshot streaming rank (nacs_rank_topsis_many) throughput: B distinct device-generated
states, B * 16 n >> L2; CUDA events on the context stream.  python scripts/bench_rank_many.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from inputs import gen  # noqa: E402
from paper_1909_07673_b200 import nacs  # noqa: E402


def make_states(snap, B, seed=1):
    k = snap["k"]
    n = k ** 3 // 4
    row = np.concatenate([snap["cpu_res"], snap["ram_res"], snap["active"].astype(np.int32), snap["link_res"]])
    st = torch.from_numpy(np.tile(row.astype(np.int32), (B, 1))).cuda()
    g = torch.Generator(device="cuda").manual_seed(seed)
    st[:, :n] = torch.randint(0, 24001, (B, n), device="cuda", generator=g, dtype=torch.int32)
    st[:, n:2 * n] = torch.randint(0, 262145, (B, n), device="cuda", generator=g, dtype=torch.int32)
    st[:, 2 * n:3 * n] = torch.randint(0, 2, (B, n), device="cuda", generator=g, dtype=torch.int32)
    st[:, 3 * n:4 * n] = torch.randint(50, 1001, (B, n), device="cuda", generator=g, dtype=torch.int32)
    return st


def main():
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = nacs.Context(0, stream)
    for variant, k, B in [(v, k, B) for v in ("occ", "occ256", "many") for k, B in ((32, 4096), (64, 512), (16, 16384))]:
        os.environ["NACS_RANK_KERNEL"] = variant
        snap = gen.snapshot(k, 4)
        ctx.load_topology(snap)
        n = k ** 3 // 4
        st = make_states(snap, B)
        out = dict(mask=None, scores=torch.empty((B, n), dtype=torch.float32, device="cuda"),
                   best=torch.empty(B, dtype=torch.int32, device="cuda"))
        for _ in range(3):
            ctx.rank_many(st, 1500, 3000, out=out, mask=False, flags=nacs.NACS_ASYNC)
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        reps = 10
        ev[0].record(stream)
        for _ in range(reps):
            ctx.rank_many(st, 1500, 3000, out=out, mask=False, flags=nacs.NACS_ASYNC)
        ev[1].record(stream)
        torch.cuda.synchronize()
        ms = ev[0].elapsed_time(ev[1]) / reps
        byts = B * n * (16 + 4)
        print(f"{variant} k={k} B={B} n={n}: {ms:.3f} ms/call, {B * n / ms * 1e3:.3e} servers/s, "
              f"{byts / ms / 1e6:.1f} GB/s algorithmic (16 B read + 4 B score per server)")
        torch.cuda.synchronize()
        ctx.rank_many(st[:8], 1500, 3000)
        print("  stats", ctx.last_stats()["pod_steps"], ctx.last_stats()["fp64_decisions"])


if __name__ == "__main__":
    main()
