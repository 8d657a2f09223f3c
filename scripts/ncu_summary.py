"""Summarise an ncu report: key metrics, stall mix, and hot SASS groups.

usage: python scripts/ncu_summary.py report.ncu-rep [n_groups]
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
ngroups = int(sys.argv[2]) if len(sys.argv) > 2 else 10


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


want = ['Duration', 'Compute (SM) Throughput', 'Issue Slots Busy', 'Executed Ipc Active', 'Registers Per Thread',
        'Block Size', 'Grid Size', 'Achieved Active Warps Per SM', 'Executed Instructions',
        'Dynamic Shared Memory Per Block', 'Eligible Warps Per Scheduler', 'No Eligible',
        'Warp Cycles Per Issued Instruction', 'DRAM Throughput', 'L1/TEX Cache Throughput']
r = list(csv.reader(io.StringIO(ncu("--page", "details", "--csv"))))
h = r[0]
for row in r[1:]:
    d = dict(zip(h, row))
    if d.get('Metric Name') in want:
        print(f"  {d['Metric Name']}: {d['Metric Value']} {d['Metric Unit']}")
rows = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv"))))
h = rows[1]
ia, isrc = h.index('Address'), h.index('Source')
iw, ie = h.index('Warp Stall Sampling (All Samples)'), h.index('Instructions Executed')
stalls = [c for c in h if c.startswith('stall_') and 'Not Issued' not in c]
data = []
for row in rows[2:]:
    if row and row[0] == "Kernel Name":  # a report with several kernels: the first one
        break
    if len(row) < len(h):
        continue
    data.append((row[isrc].strip(), float(row[iw] or 0), float(row[ie] or 0),
                 {s: float(row[h.index(s)] or 0) for s in stalls}))
tw = sum(d[1] for d in data) or 1
te = sum(d[2] for d in data) or 1
tot = {s: sum(d[3][s] for d in data) for s in stalls}
print("  stalls:", ", ".join(f"{s[6:]} {100 * v / tw:.1f}%" for v, s in sorted(((v, s) for s, v in tot.items()), reverse=True)[:8]))
g = collections.defaultdict(lambda: [0, 0, 0, []])
for i, d in enumerate(data):
    k = int(d[2])
    g[k][0] += d[2]; g[k][1] += d[1]; g[k][2] += 1; g[k][3].append(i)
print(f"  SASS instructions: {len(data)}; executed warp-instructions: {te:.4g}")
for k, (e, w, n, ids) in sorted(g.items(), key=lambda kv: -kv[1][0])[:ngroups]:
    print(f"  group exec/inst {k:12d}: {n:5d} instrs, {100 * e / te:5.1f}% of exec, {100 * w / tw:5.1f}% of samples")
