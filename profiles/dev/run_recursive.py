"""Dev: one C3-shaped DCSR Hadamard (Alg. 2) for an ncu launch list (never a bench number)."""
import sys
sys.path.insert(0, ".")
import torch
import paper_2604_17198_b200 as N, workloads as W

wl = W.build("c3", 1.0, device="cuda")
A = wl.ops[0]
g = torch.Generator(device="cuda"); g.manual_seed(3)
keep = torch.rand(A.nouter, device="cuda", generator=g) < 0.5
lens = A.pos[1:] - A.pos[:-1]
sel = torch.repeat_interleave(keep, lens)
bpos = torch.zeros(int(keep.sum().item()) + 1, dtype=torch.int64, device="cuda")
torch.cumsum(lens[keep], 0, out=bpos[1:])
B = W.SparseMatrix("dcsr", A.nrows, A.ncols, bpos, A.crd[sel].contiguous(), (A.val[sel] * 2).contiguous(),
                   A.outer_crd[keep].contiguous())
P = max(1, -(-(A.nnz + B.nnz) // 512))
N.dcsr_hadamard([A, B], P)
torch.cuda.synchronize()
