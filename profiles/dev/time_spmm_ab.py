"""Dev A/B: C4 SpMM (partition + nacho_spmm) with the library named by NACHO_LIB; CUDA events."""
import os, sys
sys.path.insert(0, ".")
import torch
import paper_2604_17198_b200 as N, workloads as W

scale = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
wl = W.build("c4", scale, device="cuda")
A = wl.ops[0]
P = N.auto_partitions([A], "spmm")
parts = N.partition([A], P)
C = torch.empty(A.nrows, wl.nb, dtype=A.val.dtype, device="cuda")
for _ in range(2):
    N.spmm(A, wl.x, parts, C=C)
ts = []
for _ in range(5):
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); N.spmm(A, wl.x, parts, C=C); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ts.sort()
print(f"{os.path.basename(os.environ.get('NACHO_LIB', 'libnacho.so'))} c4 scale {scale} spmm {ts[2]:.3f} ms "
      f"({A.nnz / ts[2] / 1e6:.1f} GNNZ/s)")
