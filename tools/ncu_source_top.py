"""Top SASS / source lines of one kernel in an ncu report by warp-stall samples.

    python tools/ncu_source_top.py report.ncu-rep [N]
"""
import csv
import io
import subprocess
import sys


def main():
    path = sys.argv[1]
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    for view in ("source", "sass"):
        cmd = ["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass" if view == "source" else "sass"]
        out = subprocess.run(cmd, capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        if not rows:
            continue
        hi = next((i for i, r in enumerate(rows) if any("Source" == c or "Address" == c for c in r)), 0)
        h = rows[hi]
        data = rows[hi + 1:]
        col = next((i for i, c in enumerate(h) if c.startswith("Warp Stall Sampling (All")), None)
        src = next((i for i, c in enumerate(h) if c in ("Source", "Sass")), 1)
        if col is None:
            print(view, "no stall column:", h[:12])
            continue
        def val(r):
            try:
                return float(r[col].replace(",", ""))
            except (ValueError, IndexError):
                return 0.0
        tot = sum(val(r) for r in data) or 1.0
        print(f"== {view}: top {n} of {len(data)} lines by stall samples ({tot:.0f} total)")
        for r in sorted(data, key=val, reverse=True)[:n]:
            print(f"{100 * val(r) / tot:5.1f}%  {r[src][:150]}")


if __name__ == "__main__":
    main()
