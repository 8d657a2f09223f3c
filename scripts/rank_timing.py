import sys, time
sys.path.insert(0, '/root/repo')
from inputs import gen
from paper_1909_07673_b200 import nacs
ctx = nacs.Context(0)
snap = gen.snapshot(32, 4)
ctx.load_topology(snap)
for bwc in (0, 1):
    ts = []
    for i in range(12):
        t = time.perf_counter(); ctx.rank("topsis", "flat", 1500, 3000, bw_criterion=bwc); ts.append(time.perf_counter() - t)
    print(bwc, [round(x * 1e3, 3) for x in ts])
import os
os.environ["NACS_RANK_KERNEL"] = "many"
ts = []
for i in range(6):
    t = time.perf_counter(); ctx.rank("topsis", "flat", 1500, 3000); ts.append(time.perf_counter() - t)
print("many", [round(x * 1e3, 3) for x in ts])
ts = []
for i in range(6):
    t = time.perf_counter(); ctx.rank("ahp", "flat", 1500, 3000); ts.append(time.perf_counter() - t)
print("ahp", [round(x * 1e3, 3) for x in ts])
