"""Small runs of every kernel path for compute-sanitizer (memcheck / racecheck / synccheck):
    compute-sanitizer --tool racecheck python profiles/sanitize.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2604_17198_b200 as N  # noqa: E402
import workloads as W  # noqa: E402
from util import random_csr  # noqa: E402

rng = np.random.default_rng(5)
dev = torch.device("cuda:0")
# SpAdd: light and heavy rows (merge path + bitmap path), all modes
base = random_csr(rng, 300, 3000, 0.01, dense_rows=[7, 150])
ops = [base] + [random_csr(rng, 300, 3000, 0.006, base=base, share=0.5, dense_rows=[7]) for _ in range(2)]
dops = [A.to(dev) for A in ops]
for P in (None, 5):
    parts = N.partition(dops, P or N.auto_partitions(dops, "spadd"))
    off = N.spadd_k_count(dops, parts)
    N.spadd_k_fill(dops, parts, off, int(off[-1].item()))
    if P is None:   # the single-read paths need tile-sized partitions
        N.spadd_k_fused(dops, parts)
        N.spadd_k_staged(dops, parts)
# SpMV (CSR fp32 / fp64, DCSR), SpMM
A = random_csr(rng, 2000, 1500, 0.01, dense_rows=[3])
for dt in (np.float32, np.float64):
    B = W.SparseMatrix(A.format, A.nrows, A.ncols, A.pos, A.crd, A.val.astype(dt)).to(dev)
    x = torch.from_numpy(rng.uniform(0.5, 1.5, 1500).astype(dt)).to(dev)
    for P in (None, 3):
        N.spmv(B, x, N.partition([B], P) if P else None)
Bm = torch.from_numpy(rng.uniform(0.5, 1.5, (1500, 64)).astype(np.float32)).to(dev)
N.spmm(A.to(dev), Bm)
# intersections (Hadamard, inner product) on the SpAdd operands
parts = N.partition(dops, N.auto_partitions(dops, "spadd"))
N.hadamard_k(dops, parts)
N.inner_k(dops, parts)
# ESC scatter kernels: SpGEMM (work, partition, expand, sort, contract) and sampled SpGEMM
Ae = random_csr(rng, 200, 150, 0.03, dense_rows=[9]).to(dev)
Be = random_csr(rng, 150, 170, 0.04, dense_rows=[2]).to(dev)
Se = random_csr(rng, 200, 170, 0.1).to(dev)
for P in (None, 7):
    N.spgemm(Ae, Be, P=P)
    N.sssmm(Se, Ae, Be, P=P)
torch.cuda.synchronize()
print("sanitize run done")
