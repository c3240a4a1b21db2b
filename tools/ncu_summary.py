"""Summarise an ncu --csv metrics log (gpu__time_duration / dram bytes) per
kernel: launches, mean time, mean DRAM read / write and the DRAM GB/s.
Usage: python tools/ncu_summary.py file.csv [peak_gbs]"""
import csv
import sys
from collections import defaultdict


def load(path):
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    rows = list(csv.reader(lines))
    hdr = rows[0]
    agg = defaultdict(lambda: defaultdict(list))
    for r in rows[1:]:
        if len(r) < len(hdr):
            continue
        d = dict(zip(hdr, r))
        name = d["Kernel Name"].split("(")[0].replace("<unnamed>::", "")
        agg[name][d["Metric Name"]].append(float(d["Metric Value"].replace(",", "")))
    return agg


def main():
    agg = load(sys.argv[1])
    peak = float(sys.argv[2]) if len(sys.argv) > 2 else 6549.1
    print(f"{'kernel':52s} {'n':>4s} {'us':>8s} {'read MB':>8s} {'write MB':>8s} {'GB/s':>7s} {'HBM frac':>8s}")
    for k, m in sorted(agg.items(), key=lambda kv: -sum(kv[1]["gpu__time_duration.sum"])):
        t = m["gpu__time_duration.sum"]
        rd, wr = m.get("dram__bytes_read.sum", [0]), m.get("dram__bytes_write.sum", [0])
        n = len(t)
        gbs = (sum(rd) + sum(wr)) / sum(t) if sum(t) else 0
        print(f"{k[:52]:52s} {n:4d} {sum(t) / n / 1e3:8.2f} {sum(rd) / len(rd) / 1e6:8.2f} "
              f"{sum(wr) / len(wr) / 1e6:8.2f} {gbs:7.0f} {gbs / peak:8.2f}")


if __name__ == "__main__":
    main()
