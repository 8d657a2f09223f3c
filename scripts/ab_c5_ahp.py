"""A/B of C5 AHP sequential scheduling (12 requests, the bench's object): device time per
pod step under the current environment.  usage: NACS_LEVELS_CLUSTER=16 python scripts/ab_c5_ahp.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from inputs import gen  # noqa: E402
from paper_1909_07673_b200 import nacs  # noqa: E402

snap = gen.snapshot(64, gen.CONFIG_SEEDS["C5"])
reqs = gen.requests(12, gen.CONFIG_SEEDS["C5"] + 1000)
ctx = nacs.Context(0)
ts = []
for it in range(3):
    ctx.load_topology(snap)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = ctx.schedule_request(reqs, "ahp", "flat")
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
st = ctx.last_stats()
import hashlib  # noqa: E402
import numpy as np  # noqa: E402
hsh = hashlib.sha256(b"".join(np.ascontiguousarray(np.asarray(out[k].cpu() if hasattr(out[k], "cpu") else out[k])).tobytes()
                              for k in sorted(out))).hexdigest()[:16]
print(f"LEVELS_CLUSTER={os.environ.get('NACS_LEVELS_CLUSTER', 'default')} ms={min(ts):.2f} "
      f"us/pod_step={1e3 * min(ts) / st['pod_steps']:.1f} pods/s={st['pod_steps'] / min(ts) * 1e3:.0f} placements {hsh}")
