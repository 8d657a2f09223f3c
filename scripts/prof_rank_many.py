"""Short nacs_rank_topsis_many run for ncu (k=32 or 64, a few launches).
python scripts/prof_rank_many.py [k] [B] [launches]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from inputs import gen  # noqa: E402
from paper_1909_07673_b200 import nacs  # noqa: E402
from scripts.bench_rank_many import make_states  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 32
B = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 4
ctx = nacs.Context(0)
snap = gen.snapshot(k, 4)
ctx.load_topology(snap)
st = make_states(snap, B)
n = k ** 3 // 4
out = dict(mask=None, scores=torch.empty((B, n), dtype=torch.float32, device="cuda"),
           best=torch.empty(B, dtype=torch.int32, device="cuda"))
for _ in range(reps):
    ctx.rank_many(st, 1500, 3000, out=out, mask=False, flags=nacs.NACS_ASYNC)
torch.cuda.synchronize()
print("ok", int(out["best"][0]))
