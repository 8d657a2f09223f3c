"""Debug: full-batch BF/WF sequential run, first request where GPU and oracle differ."""
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
ctx.load_topology(snap)
g = ctx.schedule_request(reqs, method, "flat")
print("gpu stats", ctx.last_stats())
o, cnt, ost = O.schedule(snap, reqs, method, "flat", sequential=True)
print("oracle cnt", cnt)
co = reqs["container_off"]
for r in range(30):
    a, b = co[r], co[r + 1]
    if g["status"][r] != o["status"][r] or not np.array_equal(g["server_of_container"][a:b], o["server_of_container"][a:b]):
        print("first diff at request", r, "gpu", g["status"][r], g["server_of_container"][a:b].tolist(),
              "oracle", o["status"][r], o["server_of_container"][a:b].tolist())
        break
for r in range(30):
    a, b = co[r], co[r + 1]
    print(r, g["status"][r], g["server_of_container"][a:b].tolist(), "|", o["status"][r], o["server_of_container"][a:b].tolist())
