"""GPU parity of the COO + CSR addition (nacho_partition with COO row levels + nacho_mixed_spadd_k)
against the oracle: the partition bit-exact (every field, equal to the CSR partition of the same
matrices), Z's structure and left-fold values bit-exact."""
import numpy as np
import pytest

import oracle as O
import workloads as W
from tests.conftest import gpu_available
from tests.util import random_csr

pytestmark = pytest.mark.gpu

if gpu_available():
    import torch
    import paper_2604_17198_b200 as N
    DEV = torch.device("cuda:0")


def _check(ops, P):
    dops = [A.to(DEV) for A in ops]
    parts = N.partition(dops, P)
    op = O.partition_rank(ops, P)
    for f in ("query", "row", "row_pos", "col", "pos"):
        assert np.array_equal(getattr(parts, f).cpu().numpy(), getattr(op, f)), f
    zp, zc, zv = N.mixed_spadd_k(dops, parts)
    rp, rc, rv = O.mixed_spadd_k(ops)
    assert np.array_equal(zp.cpu().numpy(), rp), "Z.pos"
    assert np.array_equal(zc.cpu().numpy(), rc), "Z.crd"
    assert np.array_equal(zv.cpu().numpy().view(np.uint8), rv.view(np.uint8)), "Z.val bits"


@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_coo_csr_random(k):
    rng = np.random.default_rng(800 + k)
    for trial in range(5):
        M, Nc = int(rng.integers(1, 3000)), int(rng.integers(1, 3000))
        base = random_csr(rng, M, Nc, float(rng.uniform(0.001, 0.02)),
                          dense_rows=[int(rng.integers(M))] if trial % 2 == 0 else ())
        csr = [base] + [random_csr(rng, M, Nc, 0.01, base=base, share=0.5) for _ in range(k - 1)]
        ops = [W.to_coo(A) if (o + trial) % 2 == 0 else A for o, A in enumerate(csr)]
        for P in (1, 5, 64, 900):
            _check(ops, P)


def test_coo_csr_c2_scaled():
    wl = W.build("c2", 0.02)
    ops = [W.to_coo(wl.ops[0]), wl.ops[1], W.to_coo(wl.ops[2])]
    _check(ops, 200)
    _check(ops[:2], 77)
