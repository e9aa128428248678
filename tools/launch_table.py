"""Mean per-launch duration by kernel from an ncu --csv launch list (gpu__time_duration.sum)."""
import collections
import csv
import sys


def table(path, metric="gpu__time_duration.sum"):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi or r[mi] != metric:
            continue
        agg.setdefault(r[ki].split("(")[0], []).append(float(r[vi].replace(",", "")))
    return agg


if __name__ == "__main__":
    agg = table(sys.argv[1])
    tot = sum(sum(v) for v in agg.values())
    for k, v in agg.items():
        print(f"{k:40s} n={len(v):4d} mean={sum(v) / len(v) / 1e3:8.2f} us  share={sum(v) / tot:6.1%}")
