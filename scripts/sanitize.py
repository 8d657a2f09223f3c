"""Every entry point of libnacs once on small inputs (SURVEY §4 layer 6), meant for
compute-sanitizer runs (memcheck / racecheck / synccheck):

  compute-sanitizer --tool racecheck python scripts/sanitize.py

compute-sanitizer is closed on the GPU pool of this build (runs under it left GPUs needing a
reset), so in round 1 the script ran plain; bad accesses are guarded by the parity tests on
small and ragged cases, the device-side request validation and the bounds of every kernel.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from inputs import gen  # noqa: E402
from paper_1909_07673_b200 import nacs  # noqa: E402

snap, reqs = gen.config("C2")
reqs = gen.subset(reqs, np.arange(24))
ctx = nacs.Context(0)
for m in ("topsis", "ahp", "bf", "wf"):
    ctx.load_topology(snap)
    ctx.schedule_batch(reqs, m, "flat")
    out = ctx.schedule_request(reqs, m, "network")
    ctx.release(reqs, out)
for m in ("topsis", "ahp"):
    ctx.load_topology(snap)
    ctx.rank(m, "flat", 1500, 3000, [(5, 20), (77, 10)])
    ctx.rank(m, "clustering", 1500, 3000, bw_criterion=1)
    ctx.schedule_batch(reqs, m, "flat", rank_once=True)
ctx.load_topology(gen.snapshot(16, 3))
ctx.schedule_batch(gen.requests(64, 9), "topsis", "flat")   # warp fast path at k=16
g = gen.fat_tree_graph(gen.snapshot(8, 3))
q = gen.path_queries(g, 600, 4, bw_hi=700)
ctx.load_graph(g)
ctx.widest_paths(q["src"], q["dst"], q["demand"], max_hops=8)
ctx.logical_bandwidth()
ctx.load_graph(gen.random_graph(40, 5, 3, 1))
ctx.widest_paths(q["src"] % 120, (q["src"] + 1) % 120, q["demand"], max_hops=12)
s4 = gen.snapshot(4, warm=False)
sreqs, arr, dur = gen.sim_workload(60, seed=21, horizon=10, max_duration=8)
for m in ("topsis", "ahp", "wf"):
    ctx.load_topology(s4)
    ctx.simulate(sreqs, arr, dur, m, "flat", max_ticks=200)
sh = nacs.Context(0, shard=(0, 2, None))   # loopback shards of the server-sharded engine
for m in ("topsis", "ahp"):
    sh.load_topology(snap)
    sh.schedule_request(reqs, m, "flat")
print("sanitize run complete")
