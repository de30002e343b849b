"""Per-kernel DRAM traffic from an `ncu --metrics gpu__time_duration.sum,
dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --csv` capture of
bench.py, against the SURVEY.md 8(d) algorithmic byte models (configs[2]:
n^3 = 128^3 lattice, W x H = 640 x 480 depth).  ncu serialises launches and
runs them cold, so times are per launch in isolation.

usage: python tools/ncu_dram_summary.py capture.csv [C_d] [V_fused]
"""
import csv
import sys
from collections import defaultdict

N3 = 128 ** 3
WH = 640 * 480


def models(cd, vf):
    # SURVEY.md 8(d) "Algorithmic bytes" per launch of each stage's kernels
    return {
        "fusion (k_integrate)": ("k_integrate", 5 * N3 + 52 * vf + 16 * WH),
        "active set (k_surface_cells + k_dilate)": (("k_surface_cells", "k_dilate"), 9 * N3),
        "marching cubes (k_mc_*)": (("k_mc_case", "k_mc_count", "k_mc_vertices", "k_mc_triangles"), 8 * N3),
        "raster (k_tri_setup + k_raster_z + k_raster_resolve)": (("k_tri_setup", "k_raster_z", "k_raster_resolve"),
                                                                40 * WH),
        "association (k_assoc_flag + k_assoc_write)": (("k_assoc_flag", "k_assoc_write"), 66 * WH + 44 * cd),
        "back-projection (k_backproject)": ("k_backproject", 30 * WH),
    }


def main():
    path = sys.argv[1]
    cd = float(sys.argv[2]) if len(sys.argv) > 2 else 62312.0
    vf = float(sys.argv[3]) if len(sys.argv) > 3 else 60000.0
    per = defaultdict(lambda: defaultdict(float))
    launches = defaultdict(set)
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for rec in csv.DictReader(lines):
        name = rec["Kernel Name"].split("(")[0].replace("wfk::", "").split("<")[0]
        v = float(rec["Metric Value"].replace(",", ""))
        unit = rec["Metric Unit"]
        m = rec["Metric Name"]
        if m == "gpu__time_duration.sum":
            v *= {"ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}.get(unit, 1e-6)
        elif unit in ("Kbyte", "KB"):
            v *= 1e3
        elif unit in ("Mbyte", "MB"):
            v *= 1e6
        elif unit in ("Gbyte", "GB"):
            v *= 1e9
        per[name][m] += v
        launches[name].add(rec["ID"])
    print(f"{'kernel':34s} {'launches':>8s} {'ms/launch':>10s} {'DRAM MB/launch':>15s} {'L2 MB/launch':>13s} "
          f"{'DRAM GB/s':>10s}")
    for name, d in sorted(per.items(), key=lambda kv: -kv[1]["gpu__time_duration.sum"]):
        n = len(launches[name])
        t = d["gpu__time_duration.sum"] / n
        dram = (d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]) / n
        l2 = d["lts__t_bytes.sum"] / n
        print(f"{name:34s} {n:8d} {t:10.4f} {dram / 1e6:15.2f} {l2 / 1e6:13.2f} {dram / (t * 1e-3) / 1e9:10.1f}")
    print()
    print(f"{'stage (SURVEY 8(d) model)':56s} {'model MB':>9s} {'DRAM MB':>8s} {'ms':>8s} {'model GB/s':>11s}")
    for stage, (names, model) in models(cd, vf).items():
        names = (names,) if isinstance(names, str) else names
        t = sum(per[k]["gpu__time_duration.sum"] / max(len(launches[k]), 1) for k in names if k in per)
        dram = sum((per[k]["dram__bytes_read.sum"] + per[k]["dram__bytes_write.sum"]) / max(len(launches[k]), 1)
                   for k in names if k in per)
        if t > 0:
            print(f"{stage:56s} {model / 1e6:9.2f} {dram / 1e6:8.2f} {t:8.4f} {model / (t * 1e-3) / 1e9:11.1f}")


if __name__ == "__main__":
    main()
