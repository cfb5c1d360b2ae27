"""Dev: the bench's C2 step as two CUDA graphs (partition, spadd) with per-section events and an L2
flush before every step; also the same step eager."""
import sys
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
po = torch.empty(P + 1, dtype=torch.int64, device="cuda")
arr = N._matrices(ops)
ws = torch.empty(max(N.lib.nacho_spadd_k_workspace_size(arr, 3, P), N.lib.nacho_spadd_k_staged_workspace_size(arr, 3, P)),
                 dtype=torch.uint8, device="cuda")
flush = torch.empty((2 * 126) << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    N.partition(ops, P, out=parts); N.spadd_k_fused(ops, parts, zp, zc, zv, part_off=po, ws=ws)
torch.cuda.current_stream().wait_stream(s); torch.cuda.synchronize()
gp, gs = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
with torch.cuda.graph(gp):
    N.partition(ops, P, out=parts)
with torch.cuda.graph(gs):
    N.spadd_k_fused(ops, parts, zp, zc, zv, part_off=po, ws=ws)
torch.cuda.synchronize()
for mode in ("graph", "eager", "graph"):
    secs = [[], []]
    for it in range(20):
        flush.zero_()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record()
        if mode == "graph":
            gp.replay()
        else:
            N.partition(ops, P, out=parts)
        e[1].record()
        if mode == "graph":
            gs.replay()
        else:
            N.spadd_k_fused(ops, parts, zp, zc, zv, part_off=po, ws=ws)
        e[2].record()
        torch.cuda.synchronize()
        if it >= 4:
            secs[0].append(e[0].elapsed_time(e[1])); secs[1].append(e[1].elapsed_time(e[2]))
    print(mode, "P", P, "partition %.4f spadd %.4f ms" % (sum(secs[0]) / len(secs[0]), sum(secs[1]) / len(secs[1])))
