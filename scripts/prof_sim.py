"""The E2 campaign through nacs_simulate (one k_simulate launch) for timing / ncu.
usage: python scripts/prof_sim.py [topsis|ahp|bf|wf] [schema] [n_requests]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from inputs import gen  # noqa: E402
from paper_1909_07673_b200 import nacs  # noqa: E402
method = sys.argv[1] if len(sys.argv) > 1 else "topsis"
schema = sys.argv[2] if len(sys.argv) > 2 else "flat"
nreq = int(sys.argv[3]) if len(sys.argv) > 3 else 6000
snap = gen.snapshot(20, warm=False)
reqs, arrival, duration = gen.sim_workload(nreq)
ctx = nacs.Context(0)
ctx.load_topology(snap)
r = ctx.simulate(reqs, arrival, duration, method, schema, max_ticks=5000)
print(method, schema, r["totals"], f"device {r['sched_seconds']:.3f} s wall {r['wall_seconds']:.3f} s", ctx.last_stats())
