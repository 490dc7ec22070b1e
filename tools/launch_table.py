"""Per-kernel table from an ncu --metrics launch list (CSV):
    python tools/launch_table.py launches.csv > profiles/rNN_bench_launches.txt"""
import csv
import sys
from collections import defaultdict


def main(path):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.DictReader(lines))
    per = defaultdict(lambda: defaultdict(float))
    launches = defaultdict(set)
    for r in rows:
        k = r["Kernel Name"]
        launches[k].add(r["ID"])
        v = float(r["Metric Value"].replace(",", ""))
        per[k][r["Metric Name"]] += v
    tot = sum(m["gpu__time_duration.sum"] for m in per.values()) or 1.0
    print(f"{'kernel':70s} {'launches':>8s} {'total_us':>12s} {'share':>7s} {'rd_GB/launch':>13s} {'wr_GB/launch':>13s}")
    for k, m in sorted(per.items(), key=lambda kv: -kv[1]["gpu__time_duration.sum"]):
        n = len(launches[k])
        t = m["gpu__time_duration.sum"] / 1000.0  # ns -> us
        print(f"{k[:70]:70s} {n:8d} {t:12.1f} {100 * m['gpu__time_duration.sum'] / tot:6.1f}% "
              f"{m['dram__bytes_read.sum'] / n / 1e9:13.4f} {m['dram__bytes_write.sum'] / n / 1e9:13.4f}")


if __name__ == "__main__":
    main(sys.argv[1])
