"""Times the single-read SpAdd (nacho_spadd_k) on C2 with L2 flushed between runs (CUDA events);
the library variant comes from NACHO_LIB.  A tuning aid, never a bench number."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2604_17198_b200 as N  # noqa: E402
import workloads as W  # noqa: E402

wl = W.build("c2", float(os.environ.get("SCALE", "1.0")), device="cuda")
ops = wl.ops
P = N.auto_partitions(ops, "spadd")
parts = N.partition(ops, P)
off = torch.empty(P + 1, dtype=torch.int64, device="cuda")
cap = sum(A.nnz for A in ops)
zp = torch.empty(ops[0].nrows + 1, dtype=torch.int64, device="cuda")
zc = torch.empty(cap, dtype=torch.int32, device="cuda")
zv = torch.empty(cap, dtype=torch.float32, device="cuda")
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")


def t(fn, n=10):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(n):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        ts.append((e0, e1))
    torch.cuda.synchronize()
    v = sorted(a.elapsed_time(b) for a, b in ts)
    return v[len(v) // 2]


tf = t(lambda: N.spadd_k_fused(ops, parts, zp, zc, zv, part_off=off))
tp = t(lambda: N.partition(ops, P, out=parts))
print(f"{os.path.basename(os.environ.get('NACHO_LIB', 'libnacho.so'))}: P={P} spadd_k {tf:.3f} ms  partition {tp:.3f} ms")
