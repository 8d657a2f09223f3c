import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from inputs import gen
from paper_1909_07673_b200 import nacs
snap, reqs = gen.config("C2")
sub = gen.subset(reqs, np.arange(60))
ref = nacs.Context(0)
ref.load_topology(snap)
a = ref.schedule_request(sub, "topsis", "flat")
print("ref stats", ref.last_stats())
sh = nacs.Context(0, shard=(0, 2, None))
sh.load_topology(snap)
try:
    out = sh.schedule_request(sub, "topsis", "flat")
except Exception as e:
    print("ERR", e)
