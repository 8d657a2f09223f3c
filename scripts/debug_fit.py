"""Debug: first request where the GPU's BF/WF sequential placement differs from the oracle."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from inputs import gen
from oracle import oracle as O
from paper_1909_07673_b200 import nacs

method = sys.argv[1] if len(sys.argv) > 1 else "wf"
k = int(sys.argv[2]) if len(sys.argv) > 2 else 4
snap = gen.snapshot(k, 60 + k)
reqs = gen.requests(30, 61 + k)
ctx = nacs.Context(0)
state = dict(snap)
for r in range(30):
    one = gen.subset(reqs, [r])
    ctx.load_topology(state)
    g = ctx.schedule_request(one, method, "flat")
    gs = ctx.read_topology()
    o, cnt, ost = O.schedule(state, one, method, "flat", sequential=True)
    if not np.array_equal(g["server_of_container"], o["server_of_container"]) or g["status"][0] != o["status"][0]:
        print("request", r, "gpu", g["status"], g["server_of_container"], "oracle", o["status"], o["server_of_container"], cnt)
        print("pod_of", one["pod_of"], "cpu_min", one["cpu_min"], "ram_min", one["ram_min"])
        n = k ** 3 // 4
        key = state["cpu_res"].astype(np.int64) * snap["ram_cap"] + state["ram_res"].astype(np.int64) * snap["cpu_cap"]
        print("cpu", state["cpu_res"][:n].tolist())
        print("ram", state["ram_res"][:n].tolist())
        print("acc", state["link_res"][:n].tolist())
        print("key order desc", np.argsort(-key, kind="stable")[:10].tolist())
        print("gpu stats", ctx.last_stats())
        break
    state = dict(snap, **{kk: ost[kk] for kk in ("cpu_res", "ram_res", "active", "link_res")})
else:
    print("no divergence")
