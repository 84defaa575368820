#!/usr/bin/env python3
"""Top SASS lines by warp-stall samples from `ncu --page source --csv --print-source sass`."""
import csv
import sys


def main(path, top=25):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if 'Source' in r and 'Address' in r)
    h = rows[hi]
    si = h.index('Warp Stall Sampling (All Samples)')
    stall_cols = [(i, n) for i, n in enumerate(h) if n.startswith('stall_') and '(Not Issued)' not in n]
    body = [r for r in rows[hi + 1:] if len(r) > si and r[si].strip().isdigit()]
    tot = sum(int(r[si]) for r in body) or 1
    print(f"{path}: {tot} samples, {len(body)} instructions")
    idx = {id(r): k for k, r in enumerate(body)}
    for r in sorted(body, key=lambda r: -int(r[si]))[:top]:
        why = sorted(((int(float(r[i] or 0)), n[6:]) for i, n in stall_cols), reverse=True)[:2]
        print(f"{idx[id(r)]:5d} {100*int(r[si])/tot:5.1f}%  {r[1].strip()[:60]:60s} {why}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
