"""Per-kernel time and DRAM bytes from an ncu launch list (`--metrics gpu__time_duration.sum,
dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file X`).  ncu serialises launches and runs them
cold, so compare SHARES of a step with the live bench, not absolute times.

    python profiles/launch_shares.py profiles/r01/launches_bench.csv
"""
import collections
import csv
import sys

SCALE = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ik, im, iv, iu = (h.index(c) for c in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    t = collections.defaultdict(float)
    by = collections.defaultdict(float)
    n = collections.Counter()
    for r in rows[1:]:
        k = r[ik].split("(")[0][:60]
        v = float(r[iv].replace(",", "")) * SCALE.get(r[iu], 1.0)
        if r[im] == "gpu__time_duration.sum":
            t[k] += v
            n[k] += 1
        elif r[im].startswith("dram__bytes"):
            by[k] += v
    tot = sum(t.values())
    print(f"{'us/launch':>10} {'launches':>8} {'share':>6} {'DRAM MB/launch':>14} {'GB/s':>7}  kernel")
    for k, v in sorted(t.items(), key=lambda x: -x[1]):
        per = v / n[k]
        mb = by[k] / n[k] / 1e6
        print(f"{per:10.1f} {n[k]:8d} {100 * v / tot:5.1f}% {mb:14.2f} {mb * 1e6 / (per * 1e-6) / 1e9:7.0f}  {k}")


if __name__ == "__main__":
    main(sys.argv[1])
