"""Add (or replace) the entry of one bench roofline kernel in profiles/roofline_traffic.json (a list, one
entry per config's roofline kernel) from an ncu --set full capture of that kernel.

    python tools/ncu_traffic.py gpurun_out/roofline.ncu-rep "<kernel string from bench roofline.kernel>"
"""
import csv
import io
import json
import os
import subprocess
import sys

rep, kernel = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
units = rows[1]
ri, wi, ti = h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum"), h.index("gpu__time_duration.sum")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
vals = []
for r in rows[2:]:
    rd = float(r[ri]) * scale[units[ri]]
    wr = float(r[wi]) * scale[units[wi]]
    vals.append((rd, wr, float(r[ti])))
# the capture may hold several launches of the same template (qkv and gate|up share it):
# the roofline kernel is the longest one
rd, wr, _ = max(vals, key=lambda v: v[2])
d = {"kernel": kernel, "bytes_per_launch": int(rd + wr), "dram_read_bytes": int(rd), "dram_write_bytes": int(wr),
     "launches_captured": len(vals), "picked": "longest launch", "source": os.path.basename(rep),
     "note": "ncu --set full --clock-control none, cold-cache replay of the kernel inside the bench's timed steps"}
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "roofline_traffic.json")
try:
    with open(path) as f:
        old = json.load(f)
except (OSError, ValueError):
    old = []
entries = [e for e in (old if isinstance(old, list) else [old]) if e.get("kernel") != kernel] + [d]
with open(path, "w") as f:
    json.dump(entries, f, indent=1)
print(json.dumps(d))
