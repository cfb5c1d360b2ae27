"""Dev: the C2 partition kernel alone, eager and CUDA-graph replay, at two P (L2 flushed)."""
import sys
sys.path.insert(0, ".")
import torch
import paper_2604_17198_b200 as N, workloads as W

wl = W.build("c2", 1.0, device="cuda")
ops = wl.ops
flush = torch.empty(300 << 20, dtype=torch.uint8, device="cuda")


def t(fn, n=15):
    for _ in range(3):
        flush.zero_(); fn()
    ts = []
    for _ in range(n):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    ts.sort()
    return sum(ts[3:-3]) / len(ts[3:-3])


for P in (14815, 9840, N.auto_partitions(ops, "spadd")):
    parts = N.Parts(P, 3, "cuda")
    te = t(lambda: N.partition(ops, P, out=parts))
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        N.partition(ops, P, out=parts)
    torch.cuda.current_stream().wait_stream(s); torch.cuda.synchronize()
    with torch.cuda.graph(g):
        N.partition(ops, P, out=parts)
    tg = t(lambda: g.replay())
    print(f"P={P}: eager {te:.4f} ms  graph {tg:.4f} ms  max_work {parts.max_work}")
