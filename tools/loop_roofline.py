"""Per-kernel roofline table of the loop body from an ncu CSV made with
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv
(one row per kernel launch and metric). Usage:
  python tools/loop_roofline.py launches.csv [peak_GBps] [steps] > profiles/<name>.txt"""
import collections
import csv
import sys


def main():
    path = sys.argv[1]
    peak = float(sys.argv[2]) if len(sys.argv) > 2 else 6537.0
    steps = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, mi, ui, vi, ii = (hdr.index(c) for c in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value", "ID"))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
             "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}
    per = collections.defaultdict(dict)
    names = {}
    for r in rows[h + 1:]:
        if len(r) <= vi:
            continue
        try:
            v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
        except ValueError:
            continue
        per[r[ii]][r[mi]] = v
        names[r[ii]] = r[ki].split("(")[0].replace("void ", "")[:48]
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for lid, m in per.items():
        a = agg[names[lid]]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
        a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    tot = sum(a[1] for a in agg.values())
    print(f"{'kernel':48s} {'launches':>8s} {'ms/step':>8s} {'share':>6s} {'DRAM MB':>9s} {'GB/s':>7s} {'frac':>5s}")
    for k, (n, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:48s} {n / steps:8.1f} {1e3 * t / steps:8.3f} {100 * t / tot:5.1f}% {b / steps / 1e6:9.1f} "
              f"{b / t / 1e9 if t else 0:7.0f} {b / t / 1e9 / peak if t else 0:5.2f}")
    print(f"{'total':48s} {'':8s} {1e3 * tot / steps:8.3f}  (cold-cache, serialised ncu replays; peak {peak:.0f} GB/s)")


if __name__ == "__main__":
    main()
