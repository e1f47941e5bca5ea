"""Summarise an ncu --csv launch list (time + DRAM bytes per kernel name)."""
import collections
import csv
import sys

UNIT = {"ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3,
        "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, mi, vi, ui, idi = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value",
                                                 "Metric Unit", "ID"))
    per, names = collections.defaultdict(dict), {}
    for r in rows[hi + 1:]:
        per[r[idi]][r[mi]] = float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1)
        names[r[idi]] = r[ki].split("(")[0][:70]
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for i, m in per.items():
        a = agg[names[i]]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0)
        a[2] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
    tot = sum(a[1] for a in agg.values())
    print("| kernel | launches | µs / launch | share | DRAM MB / launch | DRAM GB/s |")
    print("|---|---|---|---|---|---|")
    for n, (c, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| `{n}` | {c} | {t / c:.2f} | {t / tot:.1%} | {b / c / 1e6:.2f} | {b / t / 1e3 if t else 0:.0f} |")


if __name__ == "__main__":
    main(sys.argv[1])
