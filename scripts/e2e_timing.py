"""Per-call wall time of the C4 TOPSIS batch with host arrays (NACS_HOST_TIMING=1 prints the host phases)."""
import os, sys, time
sys.path.insert(0, '/root/repo')
import torch
from inputs import gen
from paper_1909_07673_b200 import nacs
snap, reqs = gen.config("C4")
ctx = nacs.Context(0)
ctx.load_topology(snap)
hout = ctx._alloc_out(reqs, False)[0]
for i in range(6):
    t = time.perf_counter()
    ctx.schedule_batch(reqs, "topsis", "flat", out=hout)
    torch.cuda.synchronize()
    print("e2e ms", (time.perf_counter() - t) * 1e3, flush=True)
