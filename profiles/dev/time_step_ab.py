"""Dev A/B: the C2 step (partition at the library's auto P + nacho_spadd_k) with the library named by
NACHO_LIB (its tile decides P); CUDA events, L2 flushed, trimmed mean of 21; Z checked against the
library's own two-pass path."""
import os, sys
sys.path.insert(0, ".")
import torch
import paper_2604_17198_b200 as N, workloads as W

wl = W.build("c2", 1.0, device="cuda")
ops = wl.ops
P = N.auto_partitions(ops, "spadd")
parts = N.Parts(P, 3, "cuda")
cap = sum(A.nnz for A in ops)
zp = torch.empty(ops[0].nrows + 1, dtype=torch.int64, device="cuda")
zc = torch.empty(cap, dtype=torch.int32, device="cuda")
zv = torch.empty(cap, dtype=torch.float32, device="cuda")
ws = torch.empty(N.lib.nacho_spadd_k_workspace_size(N._matrices(ops), 3, P) + 512, dtype=torch.uint8, device="cuda")
flush = torch.empty(300 << 20, dtype=torch.uint8, device="cuda")


def step():
    N.partition(ops, P, out=parts)
    N.spadd_k_fused(ops, parts, zp, zc, zv, ws=ws)


for _ in range(5):
    flush.zero_(); step()
ts = []
for _ in range(21):
    flush.zero_()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); step(); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ts.sort()
r_pos, r_crd, r_val = N.spadd_k(ops, parts)
nz = int(zp[-1])
ok = torch.equal(zp, r_pos) and torch.equal(zc[:nz], r_crd) and torch.equal(zv[:nz], r_val)
print(f"{os.path.basename(os.environ.get('NACHO_LIB', 'libnacho.so'))} P={P} step {sum(ts[3:-3]) / len(ts[3:-3]):.4f} ms "
      f"({cap / (sum(ts[3:-3]) / len(ts[3:-3])) / 1e6:.1f} GNNZ/s)  same-as-two-pass {ok}")
