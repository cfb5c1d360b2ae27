"""Debug aid (not a test): first SpAdd mismatch of nacho_spadd_k against the oracle, located by partition."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import oracle as O, workloads as W, paper_2604_17198_b200 as N
from tests.test_gpu_parity import _random_ops
DEV = torch.device("cuda:0")
for k in (8, 5, 3):
    rng = np.random.default_rng(200 + k)
    for trial in range(8):
        M, Nc = int(rng.integers(1, 2000)), int(rng.integers(1, 5000))
        ops = _random_ops(rng, k, M, Nc, float(rng.uniform(0.0005, 0.01)),
                          dense_rows=[int(rng.integers(M))] if trial % 2 == 0 else ())
        dops = [A.to(DEV) for A in ops]
        P = N.auto_partitions(dops, "spadd")
        parts = N.partition(dops, P)
        rp, rc, rv = O.spadd_k(ops)
        po = torch.full((P + 1,), -1, dtype=torch.int64, device=DEV)
        zp, zc, zv = N.spadd_k_fused(dops, parts, part_off=po)
        n = int(zp[-1].item())
        zc = zc[:n].cpu().numpy(); zv = zv[:n].cpu().numpy()
        bad = np.nonzero((zc != rc) | (zv.view(np.uint32) != rv.view(np.uint32)))[0] if n == len(rc) else np.array([-1])
        if len(bad):
            off = po.cpu().numpy()
            p = int(np.searchsorted(off, bad[0], side="right") - 1)
            rows = parts.row.cpu().numpy()
            print(f"k={k} trial={trial} M={M} P={P} nbad={len(bad)} first={bad[0]} part={p} rows {rows[p]}..{rows[p+1]}"
                  f" span={rows[p+1]-rows[p]} off={off[p]}..{off[p+1]} got={zc[bad[0]:bad[0]+6]} want={rc[bad[0]:bad[0]+6]}")
            bp = sorted(set(int(np.searchsorted(off, b, side='right') - 1) for b in bad))
            print("   bad partitions", bp[:20], "spans", [int(rows[q+1]-rows[q]) for q in bp[:20]])
        else:
            print(f"k={k} trial={trial} ok P={P} max span {int(np.diff(parts.row.cpu().numpy()).max())}")
