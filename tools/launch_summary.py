"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per-kernel count,
total and mean device time, and share of the listed time."""
import csv
import sys
from collections import OrderedDict


def main(path, top=40):
    lines = open(path).read().splitlines()
    start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
    rows = list(csv.reader(lines[start:]))
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = OrderedDict()
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        n = r[ki].split("(")[0].replace("void ", "")[:72]
        a = agg.setdefault(n, [0, 0.0])
        a[0] += 1
        a[1] += float(r[vi].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    print(f"{'kernel':72s} {'n':>5s} {'total_us':>10s} {'mean_us':>9s} {'share':>6s}")
    for n, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f"{n:72s} {c:5d} {t / 1e3:10.1f} {t / 1e3 / c:9.1f} {t / tot:6.1%}")
    print(f"total listed device time: {tot / 1e3:.1f} us")


if __name__ == "__main__":
    main(sys.argv[1])
