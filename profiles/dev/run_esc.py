"""Dev: one ESC SpGEMM / SSSMM step on C2's operands (for ncu launch lists; never a bench number)."""
import sys
sys.path.insert(0, ".")
import torch
import paper_2604_17198_b200 as N, workloads as W

scale = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
wl = W.build("c2", scale, device="cuda")
A, B, S = wl.ops
for _ in range(2):
    N.spgemm(A, B)
    N.sssmm(S, A, B)
torch.cuda.synchronize()
