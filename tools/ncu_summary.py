"""Summarise ncu output into profiles/ (run here, on the CPU box).

    python tools/ncu_summary.py launches <launches.csv> [--half]  -> per-kernel share table
    python tools/ncu_summary.py full <report.ncu-rep>              -> key metrics per captured launch
"""

from __future__ import annotations

import collections
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic",
]


def launches(path, half=False):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    if half:
        data = data[len(data) // 2:]
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for d in data:
        name = d["Kernel Name"].split("(")[0][:70]
        tot[name] += float(d["Metric Value"].replace(",", ""))
        cnt[name] += 1
    s = sum(tot.values())
    unit = data[0]["Metric Unit"] if data else "?"
    print(f"| kernel | launches | total ({unit}) | share |")
    print("|---|---:|---:|---:|")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"| `{k}` | {cnt[k]} | {v:,.0f} | {100 * v / s:.1f}% |")
    print(f"| **all** | {sum(cnt.values())} | {s:,.0f} | 100% |")


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    name_i = idx.get("Kernel Name")
    for n, r in enumerate(rows[2:]):
        print(f"### launch {n}: `{r[name_i][:90] if name_i is not None else '?'}`")
        for k in KEYS:
            if k in idx:
                print(f"- {k}: {r[idx[k]]} {units[idx[k]]}")
        print()


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], half="--half" in sys.argv)
    else:
        full(sys.argv[2])
