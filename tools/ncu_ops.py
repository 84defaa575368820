#!/usr/bin/env python3
"""Executed warp-instructions per SASS opcode from `ncu --page source --csv --print-source sass`."""
import collections
import csv
import sys


def main(path, top=30):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if 'Source' in r and 'Address' in r)
    h = rows[hi]
    ei = h.index('Instructions Executed')
    agg = collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) <= ei or not r[ei].strip().replace('.', '').isdigit():
            continue
        s = r[1].strip()
        if s.startswith('@'):
            s = s.split(None, 1)[1] if ' ' in s else s
        op = s.split()[0] if s else '?'
        agg[op] += int(float(r[ei]))
    tot = sum(agg.values())
    print(f"{path}: {tot} warp-instructions")
    for op, n in agg.most_common(top):
        print(f"{n:10d} {100*n/tot:5.1f}% {op}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
