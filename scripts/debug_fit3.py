"""Debug: per-request retry counts of BF/WF on a congested fabric, GPU vs oracle."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from inputs import gen
from oracle import oracle as O
from paper_1909_07673_b200 import nacs

snap = gen.snapshot(8, 5)
snap["link_res"] = np.random.default_rng(3).integers(0, 60, size=snap["link_res"].size).astype(np.int32)
reqs = gen.requests(80, 9)
ctx = nacs.Context(0)
for m in ("bf", "wf"):
    state = dict(snap)
    shown = 0
    for r in range(80):
        one = gen.subset(reqs, [r])
        ctx.load_topology(state)
        g = ctx.schedule_request(one, m, "flat")
        st = ctx.last_stats()
        o, cnt, ost = O.schedule(state, one, m, "flat", sequential=True)
        if st["retries"] != cnt["retries"] or st["pod_steps"] != cnt["pod_steps"]:
            print(m, "request", r, "status", g["status"][0], o["status"][0], "gpu", st["pod_steps"], st["retries"],
                  "oracle", cnt["pod_steps"], cnt["retries"], "pods", one["pod_of"].tolist(),
                  "vl", list(zip(one["vl_src"].tolist(), one["vl_dst"].tolist())))
            print("  servers gpu", g["server_of_container"].tolist(), "oracle", o["server_of_container"].tolist())
            shown += 1
            if shown > 4:
                break
        state = dict(snap, **{kk: ost[kk] for kk in ("cpu_res", "ram_res", "active", "link_res")})
