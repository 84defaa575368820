#!/usr/bin/env python3
"""One-line summaries of `ncu --page raw --csv` exports: duration, DRAM bytes
and throughput, SM/tensor activity, occupancy, top warp-stall reasons."""
import csv
import sys

KEYS = [("gpu__time_duration.sum", "us", 1e-3), ("dram__bytes_read.sum", "MB_rd", 1e-6),
        ("dram__bytes_write.sum", "MB_wr", 1e-6), ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%", 1),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%", 1),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%", 1),
        ("launch__grid_size", "grid", 1), ("launch__registers_per_thread", "regs", 1),
        ("launch__occupancy_limit_registers", "lim_reg", 1), ("launch__occupancy_limit_shared_mem", "lim_smem", 1)]


def conv(v, unit):
    v = float(v.replace(",", ""))
    return v


def main(paths):
    for p in paths:
        rows = list(csv.reader(open(p)))
        h, units, v = rows[0], rows[1], rows[2]
        idx = {n: i for i, n in enumerate(h)}
        out = {"kernel": v[idx["Kernel Name"]][:40]}
        for k, name, sc in KEYS:
            if k in idx:
                u = units[idx[k]]
                x = conv(v[idx[k]], u)
                if k.startswith("gpu__time") and u == "ns":
                    x *= 1e-3
                elif k.startswith("gpu__time") and u == "usecond":
                    pass
                elif "bytes" in k:
                    x *= {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1, "Gbyte": 1e3}.get(u, 1e-6)
                out[name] = round(x, 2)
        stalls = []
        for i, n in enumerate(h):
            if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(v[i]), n[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        out["stalls"] = " ".join(f"{n}:{x:.1f}" for x, n in stalls[:4])
        print(out)


if __name__ == "__main__":
    main(sys.argv[1:])
