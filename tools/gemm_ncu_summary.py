"""Join an ncu --csv metrics log of one step's k_gemm_tc launches with
gpurun_out/gemm_order.json (tools/gemm_ncu_step.py) and print per-class
tensor-pipe utilisation, duration and DRAM traffic."""
import collections
import csv
import json
import sys


def main(csv_path, order_path):
    order = json.load(open(order_path))
    rows = [r for r in csv.reader(open(csv_path)) if len(r) > 10]
    h = rows[0]
    idx = {n: i for i, n in enumerate(h)}
    per = collections.OrderedDict()
    for r in rows[1:]:
        if not r[idx["ID"]].isdigit():
            continue
        k = int(r[idx["ID"]])
        per.setdefault(k, {})[r[idx["Metric Name"]]] = float(r[idx["Metric Value"]].replace(",", ""))
    cls = collections.OrderedDict()
    for i, (k, m) in enumerate(per.items()):
        o = order[i % len(order)]
        t = o["type"]
        name = o["op"] + " " + t
        c = cls.setdefault(name, [])
        c.append(m)
    print(f"{'class':70s} {'n':>3s} {'us':>7s} {'tensor%':>8s} {'utchmma%':>9s} {'sm%':>6s} {'MB_rd':>7s} {'MB_wr':>7s}")
    for name, ms in cls.items():
        avg = lambda key: sum(m.get(key, 0.0) for m in ms) / len(ms)  # noqa: E731
        us = avg("gpu__time_duration.sum") / 1e3
        print(f"{name[:70]:70s} {len(ms):3d} {us:7.2f} "
              f"{avg('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed'):8.1f} "
              f"{avg('sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32.sum.pct_of_peak_sustained_elapsed'):9.1f} "
              f"{avg('sm__throughput.avg.pct_of_peak_sustained_elapsed'):6.1f} "
              f"{avg('dram__bytes_read.sum') / 1e6:7.2f} {avg('dram__bytes_write.sum') / 1e6:7.2f}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
