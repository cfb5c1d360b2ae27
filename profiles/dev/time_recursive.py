"""Dev: C3-shaped DCSR Hadamard (Alg. 2) at several P (entries per partition), as bench_recursive builds it."""
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
ops = [A, B]
ref = None
for per in (512, 256, 128, 64, 32):
    P = max(1, -(-(A.nnz + B.nnz) // per))
    for _ in range(2):
        out = N.dcsr_hadamard(ops, P)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); out = N.dcsr_hadamard(ops, P); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    sig = [int(x.numel()) for x in out if hasattr(x, "numel")]
    print(f"per {per} P {P}: {ts[2]:.3f} ms  outputs {sig}")
