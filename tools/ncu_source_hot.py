"""Aggregate warp-stall samples per CUDA source line from
`ncu -i rep --page source --csv --print-source cuda,sass` output.
usage: python tools/ncu_source_hot.py src.csv [top]"""
import csv
import sys
from collections import defaultdict


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    agg = defaultdict(lambda: defaultdict(float))
    text = {}
    cur_file, cur_line = "?", None
    hdr = None
    with open(path) as f:
        for rec in csv.reader(f):
            if not rec:
                continue
            if rec[0] == "File Path":
                cur_file = rec[1].split("/")[-1]
                continue
            if rec[0] == "Line No":
                hdr = rec
                continue
            if hdr is None or len(rec) < len(hdr):
                continue
            if rec[0] not in ("",):
                cur_line = (cur_file, int(rec[0]))
                text[cur_line] = rec[1].strip()
                continue
            if rec[2] in ("-", "..."):
                continue
            for i, h in enumerate(hdr):
                if i < 4:
                    continue
                if h in ("Warp Stall Sampling (All Samples)", "Instructions Executed") or (
                        h.startswith("stall_") and "Not Issued" not in h):
                    try:
                        agg[cur_line][h] += float(rec[i])
                    except ValueError:
                        pass
    tot = sum(v["Warp Stall Sampling (All Samples)"] for v in agg.values())
    print(f"total samples {tot:.0f}")
    keys = sorted(agg, key=lambda k: -agg[k]["Warp Stall Sampling (All Samples)"])[:top]
    for k in keys:
        v = agg[k]
        s = v["Warp Stall Sampling (All Samples)"]
        main_stalls = sorted(((v[h], h[6:]) for h in v if h.startswith("stall_")), reverse=True)[:3]
        ms = " ".join(f"{n}:{100 * x / max(s, 1):.0f}%" for x, n in main_stalls)
        print(f"{100 * s / tot:5.1f}% {k[0]}:{k[1]:<5d} {ms:40s} | {text.get(k, '')[:90]}")


if __name__ == "__main__":
    main()
