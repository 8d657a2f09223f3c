"""Where does the end-to-end (host buffers) time of one C4 schedule_batch call go?"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from inputs import gen
from paper_1909_07673_b200 import nacs
snap, reqs = gen.config("C4")
ctx = nacs.Context(0)
ctx.load_topology(snap)
d = {k: (torch.from_numpy(v).cuda() if isinstance(v, np.ndarray) else v) for k, v in reqs.items()}
outd = ctx._alloc_out(reqs, True)[0]
outh = ctx._alloc_out(reqs, False)[0]
for _ in range(2):
    ctx.schedule_batch(reqs, "topsis", "flat")
    ctx.schedule_batch(d, "topsis", "flat", out=outd)
def t(f, n=5):
    ts = []
    for _ in range(n):
        torch.cuda.synchronize(); a = time.perf_counter(); f(); torch.cuda.synchronize(); ts.append((time.perf_counter() - a) * 1e3)
    return round(min(ts), 2), round(float(np.median(ts)), 2)
print("device ptrs          ", t(lambda: ctx.schedule_batch(d, "topsis", "flat", out=outd)))
print("host, out reused     ", t(lambda: ctx.schedule_batch(reqs, "topsis", "flat", out=outh)))
print("host, out allocated  ", t(lambda: ctx.schedule_batch(reqs, "topsis", "flat")))
big = np.empty(42440040 // 4, np.int32); src = np.ones_like(big)
print("numpy copy 42MB      ", t(lambda: np.copyto(big, src)))
