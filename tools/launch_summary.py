"""Summarise an ncu launch list (CSV with gpu__time_duration.sum [+ dram bytes]) per kernel/grid."""
import collections
import csv
import sys


def main(path, top=30):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, data = rows[hi], rows[hi + 1:]
    ki, mi, vi, gi, ii = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Grid Size", "ID"))
    launch = collections.OrderedDict()
    for r in data:
        d = launch.setdefault(r[ii], {"name": r[ki], "grid": r[gi]})
        d[r[mi]] = float(r[vi].replace(",", ""))
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    tot = 0.0
    for d in launch.values():
        n = d["name"].split("(")[0].replace("void ", "").replace("hkd::", "").replace("(anonymous namespace)::", "")
        n = n.replace("unnamed>::", "")[:44]
        key = f"{n} g={d['grid']}"
        t = d["gpu__time_duration.sum"]
        b = d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
        agg[key][0] += 1
        agg[key][1] += t
        agg[key][2] += b
        tot += t
    print(f"{len(launch)} launches, {tot / 1e6:.3f} ms (ncu: serialised, caches flushed per kernel)")
    print(" share  count   avg_us   MB/launch  DRAM_GB/s  kernel")
    for k, (n, t, b) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"{t / tot * 100:5.1f}% {n:6d} {t / n / 1e3:8.2f} {b / n / 1e6:11.2f} {b / t:10.1f}  {k}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
