"""Phase timers of the SpAdd kernel (debug build libnacho_prof.so, -DNACHO_PROF): where one CTA's
consumer thread 0 spends its cycles.  NACHO_LIB=paper_2604_17198_b200/libnacho_prof.so python profiles/phases.py"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2604_17198_b200 as N  # noqa: E402
import workloads as W  # noqa: E402

NAMES = ["ticket+bounds", "loads", "marks", "keys", "union", "bitmap path / offset", "writes", "#bitmap (count)"]


def main():
    mode = sys.argv[1] if len(sys.argv) > 1 else "fused"
    wl = W.build("c2", 1.0, device="cuda")
    ops = wl.ops
    P = N.auto_partitions(ops, "spadd")
    parts = N.partition(ops, P)
    cap = sum(A.nnz for A in ops)
    zp = torch.empty(ops[0].nrows + 1, dtype=torch.int64, device="cuda")
    zc = torch.empty(cap, dtype=torch.int32, device="cuda")
    zv = torch.empty(cap, dtype=torch.float32, device="cuda")
    off = torch.empty(P + 1, dtype=torch.int64, device="cuda")
    buf = (ctypes.c_ulonglong * 16)()
    f = N.lib.nacho_debug_phases
    for it in range(3):
        torch.cuda.synchronize()
        f(buf, 1)
        if mode == "fused":
            N.spadd_k_fused(ops, parts, zp, zc, zv, part_off=off)
        elif mode == "staged":
            N.spadd_k_staged(ops, parts, zp, zc, zv, part_off=off)
        else:
            N.spadd_k_count(ops, parts, off)
        torch.cuda.synchronize()
    f(buf, 0)
    tot = sum(buf[i] for i in range(8)) or 1
    ns = (P + 15) // 16   # sampled partitions (every 16th), one launch
    print(mode, "sampled cycles:", tot, "per sampled partition: %.0f" % (tot / ns))
    for i, n in enumerate(NAMES):
        print(f"  {n:14s} {buf[i]:>12d} {100 * buf[i] / tot:5.1f}%  {buf[i] / ns:9.0f} cyc/part")


if __name__ == "__main__":
    main()
