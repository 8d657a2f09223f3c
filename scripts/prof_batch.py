"""One nacs_schedule_batch call (after warm-up) for ncu captures.

usage: python scripts/prof_batch.py [topsis|ahp] [C3|C4] [n_requests]   (NACS_RANK_ONCE=1: R25 mode)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from inputs import gen  # noqa: E402
from paper_1909_07673_b200 import nacs  # noqa: E402

method = sys.argv[1] if len(sys.argv) > 1 else "topsis"
KW = {"rank_once": True} if os.environ.get("NACS_RANK_ONCE") == "1" else {}
cfg = sys.argv[2] if len(sys.argv) > 2 else "C4"
nreq = int(sys.argv[3]) if len(sys.argv) > 3 else gen.CONFIG_REQUESTS[cfg]
snap = gen.snapshot(gen.CONFIG_K[cfg], gen.CONFIG_SEEDS[cfg])
reqs = gen.requests(nreq, gen.CONFIG_SEEDS[cfg] + 1000)
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
ctx = nacs.Context(0, s)
ctx.load_topology(snap)
d = {k: (torch.from_numpy(v).cuda() if isinstance(v, np.ndarray) else v) for k, v in reqs.items()}
out = ctx._alloc_out(reqs, True)[0]
for _ in range(2):
    ctx.schedule_batch(d, method, "flat", out=out, flags=nacs.NACS_ASYNC, **KW)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
ctx.schedule_batch(d, method, "flat", out=out, flags=nacs.NACS_ASYNC, **KW)
e1.record(s)
torch.cuda.synchronize()
st = ctx.last_stats()
print(f"{method} {cfg} {nreq} requests: {e0.elapsed_time(e1):.3f} ms, stats {st}")

if len(sys.argv) > 4 and sys.argv[4] == "loop":
    import time
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(6)]
    torch.cuda.synchronize()
    t = time.perf_counter()
    a0 = torch.cuda.Event(enable_timing=True)
    a1 = torch.cuda.Event(enable_timing=True)
    a0.record(s)
    for i in range(6):
        flush.zero_()
        evs[i][0].record(s)
        ctx.schedule_batch(d, method, "flat", out=out, flags=nacs.NACS_ASYNC, **KW)
        evs[i][1].record(s)
    a1.record(s)
    host = time.perf_counter() - t
    torch.cuda.synchronize()
    print("per-call ms:", [round(a.elapsed_time(b), 3) for a, b in evs], "total", round(a0.elapsed_time(a1), 3),
          "host enqueue s", round(host, 4))

if len(sys.argv) > 4 and sys.argv[4] == "loop":
    import time
    torch.cuda.synchronize()
    ts = []
    for i in range(6):
        t = time.perf_counter()
        ctx.schedule_batch(d, method, "flat", out=out, flags=nacs.NACS_ASYNC, **KW)
        ts.append(round((time.perf_counter() - t) * 1e3, 3))
    torch.cuda.synchronize()
    print("host ms per call (async):", ts)
    import cProfile, pstats, io
    pr = cProfile.Profile()
    pr.enable()
    ctx.schedule_batch(d, method, "flat", out=out, flags=nacs.NACS_ASYNC, **KW)
    pr.disable()
    sio = io.StringIO()
    pstats.Stats(pr, stream=sio).sort_stats("cumulative").print_stats(8)
    print(sio.getvalue()[:2500])

if len(sys.argv) > 4 and sys.argv[4] == "loop":
    torch.cuda.synchronize()
    tz, te, tc = [], [], []
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(12)]
    for i in range(6):
        t = time.perf_counter(); flush.zero_(); tz.append(round((time.perf_counter() - t) * 1e3, 3))
        t = time.perf_counter(); ev[2 * i].record(s); te.append(round((time.perf_counter() - t) * 1e3, 3))
        t = time.perf_counter(); ctx.schedule_batch(d, method, "flat", out=out, flags=nacs.NACS_ASYNC, **KW)
        tc.append(round((time.perf_counter() - t) * 1e3, 3))
        ev[2 * i + 1].record(s)
    torch.cuda.synchronize()
    print("host ms zero_", tz, "record", te, "call", tc)
