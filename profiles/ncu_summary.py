"""Summarise an ncu report here (no GPU): per-kernel headline metrics and the hottest source lines.

    python profiles/ncu_summary.py gpurun_out/prof.ncu-rep [--lines 25]
"""
import argparse
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "Executed Ipc Active", "Achieved Occupancy",
        "Registers Per Thread", "L2 Hit Rate", "L1/TEX Hit Rate", "Warp Cycles Per Issued Instruction",
        "Executed Instructions", "Grid Size", "Block Size", "Dynamic Shared Memory Per Block",
        "Theoretical Occupancy", "Eligible Warps Per Scheduler"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum", "lts__t_sector_hit_rate.pct",
       "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
       "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active"]


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def details(rep):
    rows = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "details", "--csv"))))
    h = rows[0]
    out = {}
    for r in rows[1:]:
        d = dict(zip(h, r))
        key = (d["ID"], d["Kernel Name"][:70])
        if d["Metric Name"] in KEYS:
            out.setdefault(key, {})[d["Metric Name"]] = f'{d["Metric Value"]} {d["Metric Unit"]}'.strip()
    return out


def raw(rep):
    rows = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "raw", "--csv"))))
    h, units = rows[0], dict(zip(rows[0], rows[1]))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
             "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "msecond": 1e-3, "ms": 1e-3, "nsecond": 1e-9}
    out = {}
    for r in rows[2:]:
        d = dict(zip(h, r))
        vals = {}
        for k in RAW:
            if k not in d:
                continue
            u = units.get(k, "")
            try:
                v = float(d[k].replace(",", ""))
            except ValueError:
                vals[k] = d[k]
                continue
            vals[k] = v * scale[u] if u in scale else v   # bytes / seconds when a unit is given
        out[(d.get("ID"), d.get("Kernel Name", "")[:70])] = vals
    return out


def hot_lines(rep, n, kernel_filter=None):
    """Aggregates SASS-level stall samples / executed instructions onto the CUDA source line above them
    (`--print-source cuda,sass` interleaves both)."""
    txt = ncu("-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass")
    agg = {}
    cur_file, cur_line, cur_src, func = None, None, "", ""
    for r in csv.reader(io.StringIO(txt)):
        if len(r) == 2 and r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if len(r) == 2 and r[0] == "Function Name":
            func = r[1]
            continue
        if len(r) < 8 or r[0] == "Line No":
            continue
        if kernel_filter and kernel_filter not in func:
            continue
        if r[0]:
            cur_line, cur_src = r[0], r[1].strip()[:90]
            continue
        try:
            samples = int(r[4]) if r[4] not in ("", "-") else 0
            inst = int(r[7]) if r[7] not in ("", "-") else 0
        except (ValueError, IndexError):
            continue
        key = (cur_file, cur_line, cur_src)
        a = agg.setdefault(key, [0, 0])
        a[0] += samples
        a[1] += inst
    tot = sum(v[0] for v in agg.values()) or 1
    res = sorted(((v[0], v[1], k) for k, v in agg.items()), reverse=True)
    return [(f"{100 * s / tot:5.1f}%", i, f"{k[0]}:{k[1]}", k[2]) for s, i, k in res[:n]]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--lines", type=int, default=25)
    ap.add_argument("--traffic", nargs=2, metavar=("KEY", "KERNEL_REGEX"),
                    help="record dram read+write bytes per launch of the matching kernels (summed over one "
                         "step's launches) under KEY in profiles/traffic.json")
    ap.add_argument("--launches", type=int, default=1, help="launches of the matched kernels per report")
    a = ap.parse_args()
    if a.traffic:
        import json, os, re
        key, rx = a.traffic
        tot = sum(v["dram__bytes_read.sum"] + v["dram__bytes_write.sum"] for k, v in raw(a.rep).items()
                  if re.search(rx, k[1]))
        path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "traffic.json")
        tab = json.load(open(path)) if os.path.exists(path) else {}
        tab[key] = tot / a.launches
        json.dump(tab, open(path, "w"), indent=1, sort_keys=True)
        print(key, tab[key])
        return 0
    for k, v in details(a.rep).items():
        print(k)
        for m in KEYS:
            if m in v:
                print(f"   {m:40s} {v[m]}")
    for k, v in raw(a.rep).items():
        print(k, v)
    print("hottest source lines (warp-stall samples %, instructions executed):")
    for row in hot_lines(a.rep, a.lines):
        print("  ", *row)


if __name__ == "__main__":
    sys.exit(main())
