"""GPU parity of the DCSR k-way SpAdd (nacho_partition with k compressed outer levels +
nacho_dcsr_spadd_k, Listing 2) against the oracle: the partition bit-exact (every field), Z's outer
level, row pointers, columns and left-fold values bit-exact."""
import numpy as np
import pytest

import oracle as O
import workloads as W
from tests.conftest import gpu_available
from tests.util import random_dcsr

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
    zo, zp, zc, zv = N.dcsr_spadd_k(dops, parts)
    ro, rp, rc, rv = O.dcsr_spadd_k(ops)
    assert np.array_equal(zo.cpu().numpy(), ro), "Z outer"
    assert np.array_equal(zp.cpu().numpy(), rp), "Z.pos"
    assert np.array_equal(zc.cpu().numpy(), rc), "Z.crd"
    assert np.array_equal(zv.cpu().numpy().view(np.uint8), rv.view(np.uint8)), "Z.val bits"


def test_fig3a_dcsr_on_gpu(golden):
    g = golden("fig3a_dcsr_add.json")

    def dcsr(entries, v0):
        return W.from_coo([e[0] for e in entries], [e[1] for e in entries],
                          np.arange(v0, v0 + len(entries), dtype=np.float32), 5, 8, fmt=W.DCSR)
    _check([dcsr(g["A"], 1), dcsr(g["B"], 101)], g["P"])


@pytest.mark.parametrize("k", [2, 3, 4])
def test_dcsr_add_random(k):
    rng = np.random.default_rng(700 + k)
    for trial in range(5):
        M, Nc = int(rng.integers(2, 5000)), int(rng.integers(2, 3000))
        ops = [random_dcsr(rng, M, Nc, int(rng.integers(1, M + 1)), float(rng.uniform(0.001, 0.03)))
               for _ in range(k)]
        for P in (1, 4, 97, 2000):
            _check(ops, P)


def test_dcsr_add_fp64_dense_row_and_hypersparse():
    rng = np.random.default_rng(12)
    A = random_dcsr(rng, 300, 4000, 100, 0.01, dtype=np.float64)
    rows = np.concatenate([np.repeat(7, 4000), rng.integers(0, 300, 50)])
    cols = np.concatenate([np.arange(4000), rng.integers(0, 4000, 50)])
    key = np.unique(rows.astype(np.int64) * 4000 + cols)
    B = W.from_coo(key // 4000, key % 4000, rng.uniform(-1, 1, len(key)), 300, 4000, fmt=W.DCSR, dtype=np.float64)
    for P in (3, 31, 400):
        _check([A, B], P)
    wl = W.build("c3", 0.01)
    C3 = wl.ops[0]
    rows = np.repeat(C3.outer_crd, np.diff(C3.pos))
    sel = rng.random(C3.nnz) < 0.4
    D = W.from_coo(rows[sel], (C3.crd[sel] + 1) % C3.ncols, C3.val[sel], C3.nrows, C3.ncols, fmt=W.DCSR)
    _check([C3, D], 300)
