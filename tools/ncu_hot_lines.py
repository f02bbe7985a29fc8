"""Top source lines by warp-stall samples from `ncu -i X --page source --csv --print-source cuda,sass`."""
import csv
import subprocess
import sys

rep, n = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows, hdr = [], None
for x in csv.reader(out.splitlines()):
    if len(x) > 4 and x[0] == "Line No":
        hdr = x
        continue
    if hdr and len(x) == len(hdr) and x[0].isdigit():
        rows.append(x)
i = hdr.index("Warp Stall Sampling (All Samples)")
tot = sum(float(x[i] or 0) for x in rows) or 1.0
rows.sort(key=lambda x: -float(x[i] or 0))
for x in rows[:n]:
    print(f"{x[i]:>7} {float(x[i]) / tot * 100:5.1f}%  L{x[0]:<5} {x[1][:110]}")
