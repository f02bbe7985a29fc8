"""Top source lines (and their hottest SASS) by warp-stall samples of one kernel of an ncu report.

    python tools/ncu_hot_lines.py REPORT.ncu-rep [N] [kernel-regex]
"""
import csv
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
if len(sys.argv) > 3:
    cmd += ["-k", f"regex:{sys.argv[3]}"]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
hdr = None
by_line = defaultdict(float)
src = {}
sass = defaultdict(list)
for x in csv.reader(out.splitlines()):
    if len(x) > 4 and x[0] == "Line No":
        hdr = x
        i_s = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if not hdr or len(x) < len(hdr):
        continue
    try:
        v = float(x[i_s] or 0)
    except ValueError:
        continue
    line = x[0]
    src.setdefault(line, x[1])
    by_line[line] += v
    sass[line].append((v, x[3]))
tot = sum(by_line.values()) or 1.0
for line, v in sorted(by_line.items(), key=lambda kv: -kv[1])[:n]:
    top = sorted(sass[line], reverse=True)[:2]
    print(f"{v:>8.0f} {v / tot * 100:5.1f}%  L{line:<5} {src[line].strip()[:90]}")
    for sv, ins in top:
        if sv > 0:
            print(f"{'':16}{sv:>7.0f}  {ins[:90]}")
