"""Summarise ncu captures for profiles/.

    python tools/ncu_summary.py launches <launches.csv>          # per-kernel share of one step
    python tools/ncu_summary.py full <report.ncu-rep> [...]      # key --set full metrics per launch
"""
from __future__ import annotations

import collections
import csv
import io
import re
import subprocess
import sys

UNIT = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3, "s": 1e3}


def short(name: str) -> str:
    m = re.search(r"gemm_tcgen05_pair_kernel<(\d+), (true|false|0|1), (\d)>", name)
    if m:
        bn, bmn, epi = m.groups()
        return f"gemm_tcgen05_pair<256x{bn},{'dX K2' if bmn in ('true', '1') else 'fwd K1'},epi={epi}>"
    m = re.search(r"gemm_tcgen05_kernel<(\d+), (\d), (\d), (\d)(?:, (\d+))?>", name)
    if m:
        bn, amn, bmn, epi, maxp = m.groups()
        if maxp and maxp != "1":
            return f"gemm_tcgen05<BN={bn},dW K3 (masked units, all matrices of a microbatch)>"
        role = {("0", "0"): "fwd K1", ("0", "1"): "dX K2", ("1", "1"): "dW K3 (masked units)"}.get((amn, bmn), "gemm")
        return f"gemm_tcgen05<BN={bn},{role},epi={epi}>"
    name = re.sub(r"\(.*", "", name)
    name = re.sub(r"^void ", "", name)
    name = re.sub(r"<(\d+(?:, \d+)*)>$", r"<\1>", name)  # keep numeric template args (tile / row widths)
    if not re.search(r"<\d+(?:, \d+)*>$", name):
        name = re.sub(r"<.*>", "<>", name)
    return name.replace("void ", "").replace("pf::(anonymous namespace)::", "").replace("pf::<unnamed>::", "")


def launches(path: str) -> str:
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, mi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) <= mi or not r[mi]:
            continue
        ms = float(r[mi].replace(",", "")) * UNIT.get(r[ui], 1e-6)
        n = short(r[ki])
        tot[n] += ms
        cnt[n] += 1
    T = sum(tot.values())
    out = [f"total device time {T:.2f} ms over {sum(cnt.values())} launches (ncu, serialised, cold-cache)", "",
           "| kernel | launches | ms | share |", "|---|---:|---:|---:|"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        out.append(f"| {k} | {cnt[k]} | {v:.2f} | {100 * v / T:.1f}% |")
    return "\n".join(out)


METRICS = ["gpu__time_duration.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__grid_size", "launch__registers_per_thread",
           "sm__warps_active.avg.pct_of_peak_sustained_active"]


def full(path: str) -> str:
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, units = rows[0], rows[1]
    idx = {m: h.index(m) for m in METRICS if m in h}
    out = [f"### {path}", "", "| kernel | " + " | ".join(f"{m} [{units[idx[m]]}]" for m in idx) + " |",
           "|---|" + "---:|" * len(idx)]
    for r in rows[2:]:
        out.append(f"| {short(r[h.index('Kernel Name')])} | " + " | ".join(r[idx[m]] for m in idx) + " |")
    return "\n".join(out)


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "launches":
        print(launches(sys.argv[2]))
    else:
        print("\n\n".join(full(p) for p in sys.argv[2:]))
