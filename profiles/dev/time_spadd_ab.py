"""Dev A/B: nacho_spadd_k (the single-read path) on C2 with the library named by NACHO_LIB; CUDA
events, L2 flushed, trimmed mean of 21 launches.  Run alternately for several builds on one box."""
import os, sys
sys.path.insert(0, ".")
import torch
import paper_2604_17198_b200 as N, workloads as W

wl = W.build("c2", 1.0, device="cuda")
ops = wl.ops
P = N.auto_partitions(ops, "spadd")
parts = N.partition(ops, P)
cap = sum(A.nnz for A in ops)
zp = torch.empty(ops[0].nrows + 1, dtype=torch.int64, device="cuda")
zc = torch.empty(cap, dtype=torch.int32, device="cuda")
zv = torch.empty(cap, dtype=torch.float32, device="cuda")
ws = torch.empty(N.lib.nacho_spadd_k_workspace_size(N._matrices(ops), 3, P) + 512, dtype=torch.uint8, device="cuda")
flush = torch.empty(300 << 20, dtype=torch.uint8, device="cuda")
for _ in range(5):
    flush.zero_(); N.spadd_k_fused(ops, parts, zp, zc, zv, ws=ws)
ts = []
for _ in range(21):
    flush.zero_()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); N.spadd_k_fused(ops, parts, zp, zc, zv, ws=ws); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ts.sort()
print(f"{os.path.basename(os.environ.get('NACHO_LIB', 'libnacho.so'))} spadd {sum(ts[3:-3]) / len(ts[3:-3]):.4f} ms "
      f"min {ts[0]:.4f}")
