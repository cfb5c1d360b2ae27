"""Times partition + SpMV on a configuration (CUDA events, L2 flushed between runs)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2604_17198_b200 as N  # noqa: E402
import workloads as W  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 0.25
wl = W.build(cfg, scale, device="cuda")
A = wl.ops[0]
P = N.auto_partitions([A], "spmv")
parts = N.partition([A], P)
y = N.spmv(A, wl.x, parts)
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
ts = []
for i in range(8):
    flush.zero_()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); N.spmv(A, wl.x, parts, y=y); e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = sorted(ts)[len(ts) // 2]
print(f"{os.environ.get('NACHO_LIB', 'default')} {cfg} x{scale}: spmv {ms:.3f} ms, {A.nnz / ms / 1e6:.1f} GNNZ/s")
