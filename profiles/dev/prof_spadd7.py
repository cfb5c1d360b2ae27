"""Dev aid: per-role cycle counters of a NACHO_S7_PROF build of spadd7 on C2 (not a bench number)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2604_17198_b200 as N, workloads as W
wl = W.build("c2", 1.0, device="cuda"); ops = wl.ops
P = N.auto_partitions(ops, "spadd"); parts = N.partition(ops, P)
need = N.lib.nacho_spadd_k_workspace_size(N._matrices(ops), 3, P)
ws = torch.zeros(need + 512, dtype=torch.uint8, device="cuda")
for _ in range(3):
    N.spadd_k_fused(ops, parts, ws=ws)
torch.cuda.synchronize()
c = ws.view(torch.int64)[P + 2:P + 2 + 9].cpu().tolist()
names = ["prod wait empty", "emit wait done", "emit lookback", "comp wait full", "comp bitmap", "comp merge", "n bitmap", "n merge", "emit write"]
for n_, v in zip(names, c):
    print(f"{n_:16s} {v:16d}")
grid = 444
print("per-CTA us: " + ", ".join(f"{n_}={v / grid / 1.9e3:.1f}" for n_, v in zip(names[:6], c[:6])))
print(f"emit write per CTA us = {c[8] / grid / 1.9e3:.1f}")
print("per job cycles bitmap", c[4] / max(1, c[6]), "merge", c[5] / max(1, c[7]))
