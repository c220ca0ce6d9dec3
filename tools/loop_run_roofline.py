"""Per-kernel table of ONE iteration of the device-controlled loop
(lsr_cuda_loop_run, graph replay) from an ncu CSV of tools/loopbench.py --run K
(ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv):
the launches between the last two loop_record kernels. Usage:
  python tools/loop_run_roofline.py launches.csv [peak_GBps] > profiles/<name>.txt"""
import collections
import csv
import sys


def main():
    path = sys.argv[1]
    peak = float(sys.argv[2]) if len(sys.argv) > 2 else 6537.0
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, mi, ui, vi, ii = (hdr.index(c) for c in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value", "ID"))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
             "ns": 1e-9, "us": 1e-6, "ms": 1e-3}
    per = collections.OrderedDict()
    names = {}
    for r in rows[h + 1:]:
        if len(r) <= vi:
            continue
        try:
            v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
        except ValueError:
            continue
        per.setdefault(int(r[ii]), {})[r[mi]] = v
        names[int(r[ii])] = r[ki].split("(")[0].replace("void ", "")[:52]
    recs = [i for i in per if "loop_record" in names[i]]
    lo, hi = recs[-2], recs[-1]
    agg = collections.OrderedDict()
    for lid in per:
        if not (lo < lid <= hi):
            continue
        a = agg.setdefault(names[lid], [0, 0.0, 0.0])
        m = per[lid]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
        a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    tot = sum(a[1] for a in agg.values())
    print(f"{'kernel (in launch order of first use)':52s} {'launches':>8s} {'ms':>8s} {'share':>6s} {'DRAM MB':>9s} {'GB/s':>7s} {'frac':>5s}")
    for k, (n, t, b) in agg.items():
        print(f"{k:52s} {n:8d} {1e3 * t:8.3f} {100 * t / tot:5.1f}% {b / 1e6:9.1f} "
              f"{b / t / 1e9 if t else 0:7.0f} {b / t / 1e9 / peak if t else 0:5.2f}")
    print(f"{'total':52s} {sum(a[0] for a in agg.values()):8d} {1e3 * tot:8.3f}  (one graph-replayed iteration; cold-cache, serialised ncu replays; peak {peak:.0f} GB/s)")


if __name__ == "__main__":
    main()
