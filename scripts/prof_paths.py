"""Path kernels (general topology) after warm-up, for timing and ncu captures.

usage: python scripts/prof_paths.py [ft20|ft32|jelly] [n_queries] [paths|logical]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from inputs import gen  # noqa: E402
from paper_1909_07673_b200 import nacs  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "ft20"
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 20
kind = sys.argv[3] if len(sys.argv) > 3 else "paths"
if which == "ft20":
    g = gen.fat_tree_graph(gen.snapshot(20, 20))
elif which == "ft32":
    g = gen.fat_tree_graph(gen.snapshot(32, 4))
else:
    g = gen.random_graph(500, 12, 4, 3)   # 2000 servers on 500 switches, 12 switch ports each
q = gen.path_queries(g, nq, 7000)
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
ctx = nacs.Context(0, s)
ctx.load_graph(g)
d = {k: torch.from_numpy(v).cuda() for k, v in q.items()}
out = (torch.empty(nq, dtype=torch.int32, device="cuda"), torch.empty(nq, dtype=torch.int32, device="cuda"),
       torch.empty((nq, 9), dtype=torch.int32, device="cuda"))
lb = torch.empty(g["n_servers"], dtype=torch.int64, device="cuda")


def call():
    if kind == "paths":
        ctx.widest_paths(d["src"], d["dst"], d["demand"], max_hops=8, out=out, flags=nacs.NACS_ASYNC)
    else:
        ctx.logical_bandwidth(out=lb, flags=nacs.NACS_ASYNC)


for _ in range(2):
    call()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
call()
e1.record(s)
torch.cuda.synchronize()
st = ctx.last_stats()
ms = e0.elapsed_time(e1)
units = nq if kind == "paths" else g["n_servers"]
print(f"{which} {kind} V={g['n_vertices']} units={units}: {ms:.3f} ms, {units / ms * 1e3:.3e}/s, "
      f"edges/unit {st['edges_scanned'] / units:.1f}, edges/s {st['edges_scanned'] / ms * 1e3:.3e}")
