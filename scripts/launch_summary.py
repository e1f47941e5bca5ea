"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV):
count and mean per kernel, in first-launch order.  Usage:
    python scripts/launch_summary.py gpurun_out/launches.csv"""
import collections
import csv
import sys


def summary(path):
    rows = list(csv.reader(open(path)))
    hdr, agg = None, collections.OrderedDict()
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                agg.setdefault(d["Kernel Name"][:100], []).append(float(d["Metric Value"]))
    return agg


if __name__ == "__main__":
    for k, v in summary(sys.argv[1]).items():
        print(f"{len(v):4d} {sum(v) / len(v) / 1000:9.1f} us  {k}")
