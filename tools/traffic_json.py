"""Per-kernel-class DRAM traffic and tensor-pipe utilisation from one `ncu --set full`
capture of a bench step, stamped with the library digest and git head it was taken
on (bench.py reads it as roofline.traffic and checks the stamp).

    python tools/traffic_json.py gpurun_out/prof_step.ncu-rep "<ncu command>" > profiles/r02_traffic.json

Classes follow bench.py's profile classes: k_gather_mean / k_csc_gather launches of
the layer-1 blocks ("aggregate" / "csc_gather") and of the top layer's hop-1 blocks
("aggregate_top" / "csc_gather_top", the lighter launch of each pair); the sampler
("sample"); every k_umma instantiation is its own class (tensor pipe % reported).
"""
from __future__ import annotations

import collections
import csv
import hashlib
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
         "ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def rows_of(path):
    """Rows of an ncu report (`.ncu-rep`) or of its `--page raw --csv` export
    (`.csv` / `.csv.gz`), with byte and time metrics normalised to bytes and us."""
    if path.endswith(".csv.gz"):
        import gzip
        raw = gzip.open(path, "rt").read()
    elif path.endswith(".csv"):
        raw = open(path).read()
    else:
        raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True,
                             check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(h, r))
        for k, u in zip(h, units):
            if u in UNITS and k in d:
                try:
                    d[k] = str(float(d[k].replace(",", "")) * UNITS[u])
                except ValueError:
                    pass
        out.append(d)
    return out


def num(d, k):
    try:
        return float(str(d.get(k, "nan")).replace(",", ""))
    except ValueError:
        return float("nan")


def short(name):
    """Kernel name without namespaces and parameter list, template arguments kept."""
    n = name.strip()
    if n.endswith(")"):  # drop the parameter list (the trailing balanced group)
        depth = 0
        for i in range(len(n) - 1, -1, -1):
            depth += {")": 1, "(": -1}.get(n[i], 0)
            if depth == 0:
                n = n[:i]
                break
    base, tmpl = (n.split("<", 1) + [""])[:2] if "<" in n and not n.startswith("<") else (n, "")
    if n.startswith("<") or "unnamed>" in n:
        base = n.split("::")[-1] if "<" not in n.split("::")[-1] else n
        m = re.search(r"(k_\w+)(<.*>)?$", n)
        return (m.group(1) + (m.group(2) or "")) if m else n
    base = re.sub(r"^void ", "", base).split("::")[-1]
    return base + ("<" + tmpl if tmpl else "")


def main():
    path, cmd = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
    acc = collections.defaultdict(list)
    split = collections.defaultdict(list)
    for d in rows_of(path):
        nm = short(d.get("Kernel Name", "?"))
        if nm.startswith("k_gather_mean"):
            split[("aggregate", "aggregate_top")].append(d)
        elif nm.startswith("k_csc_gather"):
            split[("csc_gather", "csc_gather_top")].append(d)
        elif nm.startswith("k_sample_fused"):
            acc["sample"].append(d)
        else:
            acc[nm].append(d)
    # each of these kernels runs once per layer: the top layer's launch (hop-1 blocks,
    # 1024 destination rows) moves far fewer bytes than the layer-1 launch
    for (big, small), ds in split.items():
        vol = sorted(num(d, "dram__bytes_read.sum") + num(d, "dram__bytes_write.sum") for d in ds)
        cut = (vol[0] + vol[-1]) / 2
        for d in ds:
            v = num(d, "dram__bytes_read.sum") + num(d, "dram__bytes_write.sum")
            acc[big if v > cut else small].append(d)
    out = {}
    for cls, ds in acc.items():
        rd = sum(num(d, "dram__bytes_read.sum") for d in ds) / len(ds)
        wr = sum(num(d, "dram__bytes_write.sum") for d in ds) / len(ds)
        us = sum(num(d, "gpu__time_duration.sum") for d in ds) / len(ds)
        e = {"launches": len(ds), "dram_bytes_per_launch": int(rd + wr), "read": int(rd), "write": int(wr),
             "us_per_launch": us,
             "dram_pct_of_peak": sum(num(d, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed") for d in ds) / len(ds),
             "occupancy_pct": sum(num(d, "sm__warps_active.avg.pct_of_peak_sustained_active") for d in ds) / len(ds)}
        tp = [num(d, "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active") for d in ds]
        tp = [x for x in tp if x == x]
        if tp and max(tp) > 0:
            e["tensor_pipe_pct"] = sum(tp) / len(tp)
        out[cls] = e
    lib = os.path.join(ROOT, "paper_2408_09697_b200", "libhetgpu.so")
    with open(lib, "rb") as f:
        sha = hashlib.sha256(f.read()).hexdigest()[:16]
    head = subprocess.run(["git", "-C", ROOT, "rev-parse", "--short=12", "HEAD"], capture_output=True,
                          text=True).stdout.strip()
    rec = {"source": cmd, "metrics": "dram__bytes_read.sum + dram__bytes_write.sum per launch; "
                                     "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
           "lib_sha256_16": sha, "git_head_at_capture": head,
           "tensor_pipe_pct": {k: round(v["tensor_pipe_pct"], 2) for k, v in out.items() if "tensor_pipe_pct" in v},
           "kernels": out}
    print(json.dumps(rec, indent=1))


if __name__ == "__main__":
    main()
