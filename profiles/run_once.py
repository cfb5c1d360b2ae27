"""Runs one configuration's hot-path step a few times (for ncu / compute-sanitizer; never a bench number).

    python profiles/run_once.py c2|c5|c3|c4|c1 [--scale S] [--steps N]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2604_17198_b200 as N  # noqa: E402
import workloads as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cfg")
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--two-pass", action="store_true")
    a = ap.parse_args()
    wl = W.build(a.cfg, a.scale, device="cuda")
    ops = wl.ops
    if wl.kind == "spadd":
        P = N.auto_partitions(ops, "spadd")
        parts = N.Parts(P, len(ops), "cuda")
        cap = sum(A.nnz for A in ops)
        off = torch.empty(P + 1, dtype=torch.int64, device="cuda")
        zp = torch.empty(ops[0].nrows + 1, dtype=torch.int64, device="cuda")
        zc = torch.empty(cap, dtype=torch.int32, device="cuda")
        zv = torch.empty(cap, dtype=ops[0].val.dtype, device="cuda")

        def step():
            N.partition(ops, P, out=parts)
            if a.two_pass:
                N.spadd_k_count(ops, parts, off)
                N.spadd_k_fill(ops, parts, off, cap, zp, zc, zv)
            else:
                N.spadd_k_fused(ops, parts, zp, zc, zv, part_off=off)
    elif wl.kind == "spmm":
        A = ops[0]
        P = N.auto_partitions([A], "spmm")
        parts = N.Parts(P, 1, "cuda")
        C = torch.empty(A.nrows, wl.nb, dtype=A.val.dtype, device="cuda")

        def step():
            N.partition([A], P, out=parts)
            N.spmm(A, wl.x, parts, C=C)
    else:
        A = ops[0]
        P = wl.P or N.auto_partitions([A], "spmv")
        parts = N.Parts(P, 1, "cuda")

        def step():
            N.partition([A], P, out=parts)
            N.spmv(A, wl.x, parts)
    for _ in range(a.steps):
        step()
    torch.cuda.synchronize()
    print("done", a.cfg, "P =", P)


if __name__ == "__main__":
    main()
