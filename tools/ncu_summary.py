"""Summaries of ncu output for profiles/ (run here, on the CPU box).

  python tools/ncu_summary.py launches <launches.csv> [out.md]
      per-kernel-class device time, share and launch count from a
      `ncu --metrics gpu__time_duration.sum --csv` launch list
  python tools/ncu_summary.py full <report.ncu-rep> [out.md]
      key metrics of each captured launch of a `ncu --set full` report
"""
import collections
import csv
import io
import re
import subprocess
import sys

UNITS = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def short(name):
    m = re.search(r"(\w+)<([^>]*)>\(", name)
    base = name.split("(")[0].split("::")[-1]
    if m:
        return f"{m.group(1)}<{m.group(2)}>"
    return base


def launches(path):
    text = open(path).read()
    lines = [ln for ln in text.splitlines() if ln.startswith('"')]
    rows = list(csv.reader(io.StringIO("\n".join(lines))))
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot, cnt = collections.Counter(), collections.Counter()
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        us = float(r[vi].replace(",", "")) * UNITS.get(r[ui], 1.0)
        k = short(r[ki])
        tot[k] += us
        cnt[k] += 1
    T = sum(tot.values())
    out = [f"launches: {sum(cnt.values())}, total device time {T / 1e3:.2f} ms (serialised, cold-cache)\n",
           "| kernel | launches | time (ms) | share |", "|---|---|---|---|"]
    for k, v in tot.most_common():
        out.append(f"| `{k}` | {cnt[k]} | {v / 1e3:.3f} | {100 * v / T:.1f}% |")
    return "\n".join(out) + "\n"


FULL_METRICS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread", "launch__grid_size",
    "launch__cluster_dim_x",
]


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        out.append(f"### `{short(r[h.index('Kernel Name')])}` (launch {r[h.index('ID')]})\n")
        out.append("| metric | value | unit |\n|---|---|---|")
        for m in FULL_METRICS:
            if m in h:
                i = h.index(m)
                out.append(f"| {m} | {r[i]} | {units[i]} |")
        out.append("")
    return "\n".join(out) + "\n"


if __name__ == "__main__":
    mode, src = sys.argv[1], sys.argv[2]
    text = launches(src) if mode == "launches" else full(src)
    if len(sys.argv) > 3:
        open(sys.argv[3], "w").write(text)
    print(text)
