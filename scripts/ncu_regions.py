"""Stall samples and instructions of an ncu report grouped by the enclosing function of
nacs_warp.cu (regions found from the source), inlined headers separately.

usage: python scripts/ncu_regions.py report.ncu-rep [source.cu]
"""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
src = sys.argv[2] if len(sys.argv) > 2 else "paper_1909_07673_b200/csrc/nacs_warp.cu"
starts = []
for i, line in enumerate(open(src), 1):
    m = re.match(r"^(?:__device__|__global__)[^(]*?\b(\w+)\s*\(", line)
    if m:
        starts.append((i, m.group(1)))
    elif re.match(r"^\s*// ---- phase", line):
        starts.append((i, "main:" + line.strip()[8:30]))


def region(ln):
    name = "?"
    for s, n in starts:
        if s <= ln:
            name = n
    return name


txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg, cur, hdr = {}, "?", None
base = src.split("/")[-1]
for r in csv.reader(io.StringIO(txt)):
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
    elif r[0] == "Line No":
        hdr = r
    elif hdr and r[0].isdigit() and len(r) > 8 and r[2] == "-":
        ex, sm = float(r[hdr.index("Instructions Executed")] or 0), float(r[4] or 0)
        key = region(int(r[0])) if cur == base else "inlined:" + cur
        e = agg.setdefault(key, [0, 0])
        e[0] += ex
        e[1] += sm
te = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    if v[1] / ts > 0.002:
        print(f"{k:36s} inst {v[0] / te * 100:5.1f}%  samples {v[1] / ts * 100:5.1f}%")
