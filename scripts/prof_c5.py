"""A few sequential C5 requests (k=64) for per-kernel launch lists: python scripts/prof_c5.py [ahp|topsis] [n]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
from inputs import gen  # noqa: E402
from paper_1909_07673_b200 import nacs  # noqa: E402
method = sys.argv[1] if len(sys.argv) > 1 else "ahp"
nreq = int(sys.argv[2]) if len(sys.argv) > 2 else 2
snap = gen.snapshot(64, gen.CONFIG_SEEDS["C5"])
reqs = gen.requests(nreq, gen.CONFIG_SEEDS["C5"] + 1000)
ctx = nacs.Context(0)
ctx.load_topology(snap)
out = ctx.schedule_request(reqs, method, "flat")
print(ctx.last_stats())
