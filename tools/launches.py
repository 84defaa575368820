#!/usr/bin/env python3
"""Summarise an ncu launch list (gpu__time_duration.sum CSV) per kernel."""
import collections
import csv
import sys


def main(path, steps=None):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
    h = rows[hi]
    ki, vi = h.index('Kernel Name'), h.index('Metric Value')
    agg = collections.defaultdict(lambda: [0, 0.0])
    tot = 0.0
    for r in rows[hi + 1:]:
        n = r[ki].split('(')[0][:70]
        v = float(r[vi].replace(',', ''))
        agg[n][0] += 1
        agg[n][1] += v
        tot += v
    print(f"total {tot/1e3:.1f} us over {sum(a[0] for a in agg.values())} launches")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{t/1e3:10.1f} us {100*t/tot:5.1f}% {n:5d}  {k}")


if __name__ == "__main__":
    main(sys.argv[1])
