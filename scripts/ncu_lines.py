"""Per-source-line instruction and stall-sample shares of an ncu report (hot lines first).

usage: python scripts/ncu_lines.py report.ncu-rep [n_lines] [inst]   (inst: sort by executed instructions)
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
nl = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur, hdr, out = "?", None, []
for r in csv.reader(io.StringIO(txt)):
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
    elif r[0] == "Line No":
        hdr = r
    elif hdr and r[0].isdigit() and len(r) > 8 and r[2] == "-":
        ex, sm = float(r[hdr.index("Instructions Executed")] or 0), float(r[4] or 0)
        if ex or sm:
            out.append((ex, sm, f"{cur}:{r[0]}", r[1][:100]))
tot = sum(o[0] for o in out) or 1
ts = sum(o[1] for o in out) or 1
key = 0 if len(sys.argv) > 3 and sys.argv[3] == "inst" else 1
for ex, sm, loc, src in sorted(out, key=lambda o: -o[key])[:nl]:
    print(f"{ex / tot * 100:5.1f}% inst {sm / ts * 100:5.1f}% samples  {loc:22s} {src}")
