import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import oracle as O, paper_2604_17198_b200 as N
from tests.test_gpu_parity import _random_ops
k = int(sys.argv[1]) if len(sys.argv) > 1 else 8
rng = np.random.default_rng(200 + k)
M, Nc = int(rng.integers(1, 2000)), int(rng.integers(1, 5000))
ops = _random_ops(rng, k, M, Nc, float(rng.uniform(0.0005, 0.01)), dense_rows=[int(rng.integers(M))])
dops = [A.to("cuda") for A in ops]
P = N.auto_partitions(dops, "spadd"); parts = N.partition(dops, P)
zp, zc, zv = N.spadd_k_fused(dops, parts)
torch.cuda.synchronize()
rp, rc, rv = O.spadd_k(ops)
n = int(zp[-1].item())
print("k", k, "P", P, "ok", n == len(rc) and np.array_equal(zc[:n].cpu().numpy(), rc))
