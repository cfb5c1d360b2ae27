"""Dev: bench.py's ESC lines alone (fresh process), to separate kernel time from the full bench's
allocation history."""
import sys
sys.path.insert(0, ".")
import torch
import bench
import paper_2604_17198_b200 as N, workloads as W

timer = bench.Timer(torch, 2 * 126 * 2**20)
for sampled in (False, True):
    r = bench.bench_esc(N, W, torch, 1.0, 5, 2, timer, sampled=sampled)
    print("sampled" if sampled else "spgemm", {k: round(sum(v) / len(v), 3) for k, v in r["sec"].items()})
