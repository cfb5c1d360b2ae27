"""Times SpMM (C4 shape, scaled) with CUDA events."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2604_17198_b200 as N  # noqa: E402
import workloads as W  # noqa: E402

scale = float(sys.argv[1]) if len(sys.argv) > 1 else 0.25
wl = W.build("c4", scale, device="cuda")
A = wl.ops[0]
P = N.auto_partitions([A], "spmm")
parts = N.partition([A], P)
C = N.spmm(A, wl.x, parts)
ts = []
for i in range(5):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); N.spmm(A, wl.x, parts, C=C); e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = sorted(ts)[len(ts) // 2]
print(f"c4 x{scale}: spmm {ms:.3f} ms, {A.nnz / ms / 1e6:.1f} GNNZ/s")
