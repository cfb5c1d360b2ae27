import torch, sys, os
sys.path.insert(0, ".")
import paper_2604_17198_b200 as N, workloads as W
wl = W.build("c2", 1.0, device="cuda"); ops = wl.ops
P = N.auto_partitions(ops, "spadd"); parts = N.partition(ops, P)
for i in range(3): N.spadd_k_staged(ops, parts)
torch.cuda.synchronize()
