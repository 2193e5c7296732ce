"""Summarise ncu output brought back from a gpurun call into profiles/.

    python tools/ncu_summary.py launches gpurun_out/launches.csv [steps]
    python tools/ncu_summary.py full gpurun_out/prof.ncu-rep

`launches`: per-kernel launch count, total/avg device time and share of the
listed launches (ncu's serialised, cold-cache times: compare shares).
`full`: the headline counters of every profiled launch of an `ncu --set full`
report (duration, DRAM bytes and throughput, SM/issue activity, occupancy).
"""
from __future__ import annotations

import collections
import csv
import io
import subprocess
import sys


def launches(path: str, steps: float = 0.0) -> str:
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "s": 1e6, "second": 1e6}
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in data:
        if len(r) <= vi:
            continue
        us = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        name = r[ki].split("(")[0].replace("hetgpu::<unnamed>::", "").replace("unnamed>::", "").replace("void ", "")
        agg[name][0] += 1
        agg[name][1] += us
    tot = sum(v[1] for v in agg.values())
    out = ["| kernel | launches | total us | us/launch | share |", "|---|---:|---:|---:|---:|"]
    for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| `{n}` | {c} | {t:.1f} | {t / c:.2f} | {100 * t / tot:.1f}% |")
    out.append(f"\n{len(data)} launches, {tot:.1f} us total" +
               (f" ({tot / steps:.1f} us per step over {steps:g} steps)" if steps else ""))
    return "\n".join(out)


METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % of peak"),
    ("sm__cycles_active.avg", "SM active cycles"),
    ("gpc__cycles_elapsed.max", "elapsed cycles"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("launch__registers_per_thread", "registers"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def full(path: str) -> str:
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[0]
    out = ["| launch | kernel | " + " | ".join(lbl for _, lbl in METRICS) + " |",
           "|---|---|" + "---:|" * len(METRICS)]
    for r in rows[2:]:
        d = dict(zip(h, r))
        name = d.get("Kernel Name", "?").split("(")[0].replace("hetgpu::<unnamed>::", "").replace("unnamed>::", "").replace("void ", "")
        vals = [d.get(m, "n/a") for m, _ in METRICS]
        out.append(f"| {d.get('ID', '?')} | `{name}` | " + " | ".join(vals) + " |")
    units = rows[1]
    out.append("\nunits: " + ", ".join(f"{lbl} [{units[h.index(m)] if m in h else '-'}]" for m, lbl in METRICS))
    return "\n".join(out)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        print(launches(sys.argv[2], float(sys.argv[3]) if len(sys.argv) > 3 else 0.0))
    else:
        print(full(sys.argv[2]))
