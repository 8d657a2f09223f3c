"""Where does the time between consecutive schedule_batch calls go?  Variants of the bench loop."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from inputs import gen
from paper_1909_07673_b200 import nacs
snap, reqs = gen.config("C4")
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
ctx = nacs.Context(0, s); ctx.load_topology(snap)
d = {k: (torch.from_numpy(v).cuda() if isinstance(v, np.ndarray) else v) for k, v in reqs.items()}
out = ctx._alloc_out(reqs, True)[0]
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
for _ in range(3):
    ctx.schedule_batch(d, "topsis", "flat", out=out, flags=nacs.NACS_ASYNC)
torch.cuda.synchronize()
def run(tag, use_flush, sync_each):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(5)]
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    th = []
    t = time.perf_counter()
    a0.record(s)
    for i in range(5):
        t1 = time.perf_counter()
        if use_flush: flush.zero_()
        ev[i][0].record(s)
        ctx.schedule_batch(d, "topsis", "flat", out=out, flags=nacs.NACS_ASYNC)
        ev[i][1].record(s)
        th.append(round((time.perf_counter() - t1) * 1e3, 2))
        if sync_each: torch.cuda.synchronize()
    a1.record(s)
    host = time.perf_counter() - t
    torch.cuda.synchronize()
    per = [round(a.elapsed_time(b), 2) for a, b in ev]
    print(f"{tag:22s} total/step {a0.elapsed_time(a1)/5:7.2f} per-call {per} host ms/iter {th} host total {host*1e3:.1f}")
run("flush", True, False)
run("no flush", False, False)
run("flush, sync each", True, True)
os.environ["NACS_WARP_GROUP"] = "8"
run("flush again", True, False)
