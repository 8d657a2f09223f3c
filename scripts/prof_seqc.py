"""C5 sequential TOPSIS (k_seq_cluster) for ncu: python scripts/prof_seqc.py [n_requests]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from inputs import gen  # noqa: E402
from paper_1909_07673_b200 import nacs  # noqa: E402
nreq = int(sys.argv[1]) if len(sys.argv) > 1 else 8
snap = gen.snapshot(64, gen.CONFIG_SEEDS["C5"])
reqs = gen.requests(nreq, gen.CONFIG_SEEDS["C5"] + 1000)
ctx = nacs.Context(0)
for _ in range(2):
    ctx.load_topology(snap)
    ctx.schedule_request(reqs, "topsis", "flat")
print(ctx.last_stats())
