"""Summarise an ncu --csv launch list: per-kernel count, total/avg device time, DRAM bytes."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr, data = rows[hi], rows[hi + 1:]
    ki, mi, vi, ui = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    ii = hdr.index("ID")
    gi = hdr.index("Grid Size") if (BY_GRID and "Grid Size" in hdr) else None
    per = collections.defaultdict(dict)
    names = {}
    for r in data:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        u = r[ui]
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3, "second": 1e6,
                 "byte": 1, "Kbyte": 1e3, "KB": 1e3, "MB": 1e6, "GB": 1e9,
                 "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        per[r[ii]][r[mi]] = v * scale
        names[r[ii]] = r[ki].split("(")[0][:70] + (" grid" + r[gi] if gi is not None else "")
    return per, names


def main(path):
    per, names = load(path)
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for i, m in per.items():
        n = names[i]
        a = agg[n]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
        a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    tot = sum(a[1] for a in agg.values())
    print(f"{'total us':>10} {'share':>6} {'n':>6} {'avg us':>9} {'avg MB':>9} {'GB/s':>8}  kernel")
    for n, (c, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{t:10.1f} {100 * t / tot:5.1f}% {c:6d} {t / c:9.2f} {b / c / 1e6:9.2f} {b / max(t, 1e-9) / 1e3:8.0f}  {n}")


BY_GRID = "--grid" in sys.argv  # key on (kernel, grid size): separates prefill from decode launches

if __name__ == "__main__":
    main([x for x in sys.argv[1:] if not x.startswith("--")][0])
