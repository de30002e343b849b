"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list.

usage: python tools/ncu_summary.py launches.csv [--frame]

Prints per-kernel launch counts, total time and share.  With --frame, also
prints the launches of the last complete frame (the launches between the last
two `k_integrate` launches, i.e. one wfk_process_frame) in order, so the
per-frame setup kernels around the flip-flop solves can be read off.
"""
import csv
import sys
from collections import defaultdict


def load(path):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for rec in csv.DictReader(lines):
        if rec.get("Metric Name") != "gpu__time_duration.sum":
            continue
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}.get(rec["Metric Unit"], 1e-6)
        name = rec["Kernel Name"].split("(")[0]
        rows.append((name, float(rec["Metric Value"].replace(",", "")) * scale, rec["Grid Size"]))
    return rows


def main():
    path = sys.argv[1]
    rows = load(path)
    tot = sum(r[1] for r in rows)
    agg = defaultdict(lambda: [0, 0.0])
    for n, ms, _ in rows:
        agg[n][0] += 1
        agg[n][1] += ms
    print(f"# {len(rows)} launches, total {tot:.3f} ms")
    print(f"{'kernel':70s} {'launches':>9s} {'total_ms':>10s} {'share':>7s}")
    for n, (k, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{n[:70]:70s} {k:9d} {ms:10.3f} {100 * ms / tot:6.2f}%")
    if "--frame" in sys.argv:
        idx = [i for i, r in enumerate(rows) if r[0].endswith("k_integrate")]
        if len(idx) >= 2:
            seg = rows[idx[-2] + 1: idx[-1] + 1]
            fs = sum(r[1] for r in seg)
            print(f"\n# last frame: {len(seg)} launches, {fs:.3f} ms (serialised, cold cache)")
            for n, ms, grid in seg:
                print(f"{ms * 1e3:10.1f} us  {n[:60]:60s} {grid}")


if __name__ == "__main__":
    main()
