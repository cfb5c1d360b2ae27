import torch, sys, os
sys.path.insert(0, ".")
import paper_2604_17198_b200 as N, workloads as W
wl = W.build("c2", 1.0, device="cuda"); ops = wl.ops
P = N.auto_partitions(ops, "spadd"); parts = N.partition(ops, P)
off = torch.empty(P + 1, dtype=torch.int64, device="cuda")
cap = sum(A.nnz for A in ops)
zp = torch.empty(ops[0].nrows + 1, dtype=torch.int64, device="cuda"); zc = torch.empty(cap, dtype=torch.int32, device="cuda"); zv = torch.empty(cap, dtype=torch.float32, device="cuda")
def t(fn, n=10):
    for i in range(3): fn()
    torch.cuda.synchronize()
    e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(n): fn()
    e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1)/n
ws = torch.empty(N.lib.nacho_spadd_k_staged_workspace_size(N._matrices(ops), len(ops), P), dtype=torch.uint8, device="cuda")
print(os.environ.get("NACHO_LIB"), "staged %.3f ms" % t(lambda: N.spadd_k_staged(ops, parts, zp, zc, zv, part_off=off, ws=ws)),
      "fused %.3f ms" % t(lambda: N.spadd_k_fused(ops, parts, zp, zc, zv, part_off=off)),
      "count %.3f ms" % t(lambda: N.spadd_k_count(ops, parts, off)), "fill %.3f" % t(lambda: N.spadd_k_fill(ops, parts, off, cap, zp, zc, zv)),
      "partition %.3f" % t(lambda: N.partition(ops, P, out=parts)))
