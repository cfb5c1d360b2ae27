"""GPU parity of the recursive partitioning path (nacho_dcsr_hadamard: Alg. 2 on the DCSR Hadamard
product) against the oracle of Listing emul-dcsr2-rewritten: the surviving rows, the remapped
partition (every field bit-exact), Z's structure and product values bit-exact."""
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
    parts, zo, zp, zc, zv = N.dcsr_hadamard(dops, P)
    rm = O.dcsr_rows_intersect(ops)
    assert np.array_equal(zo.cpu().numpy(), rm.rows.astype(np.int32)), "surviving rows"
    op = O.partition_remapped(ops, rm, P)
    for f in ("query", "row", "row_pos", "col", "pos"):
        assert np.array_equal(getattr(parts, f).cpu().numpy(), getattr(op, f)), f
    ro, rp, rc, rv = O.dcsr_hadamard(ops, rm)
    assert np.array_equal(zp.cpu().numpy(), rp), "Z.pos"
    assert np.array_equal(zc.cpu().numpy(), rc), "Z.crd"
    assert np.array_equal(zv.cpu().numpy().view(np.uint8), rv.view(np.uint8)), "Z.val bits"


def test_fig3b_on_gpu(golden):
    g = golden("fig3b_dcsr_mul_partition.json")

    def dcsr(entries):
        return W.from_coo([e[0] for e in entries], [e[1] for e in entries],
                          np.arange(1, len(entries) + 1, dtype=np.float32), 5, 8, fmt=W.DCSR)
    A, B = dcsr(g["A"]), dcsr(g["B"])
    _check([A, B], g["P"])
    parts, zo, zp, zc, zv = N.dcsr_hadamard([A.to(DEV), B.to(DEV)], g["P"])
    assert [[int(r), int(c)] for r, c in zip(parts.row.cpu(), parts.col.cpu())] == g["boundaries_row_col"]
    assert zo.cpu().tolist() == g["Z_outer"] and zp.cpu().tolist() == g["Z_pos"]


@pytest.mark.parametrize("k", [2, 3, 4])
def test_recursive_random(k):
    rng = np.random.default_rng(500 + k)
    for trial in range(6):
        M, Nc = int(rng.integers(2, 3000)), int(rng.integers(2, 2000))
        ops = [random_dcsr(rng, M, Nc, int(rng.integers(1, M + 1)), float(rng.uniform(0.001, 0.05)))
               for _ in range(k)]
        for P in (1, 3, 64, 1000):
            _check(ops, P)


def test_recursive_fp64_and_disjoint():
    rng = np.random.default_rng(9)
    A = random_dcsr(rng, 500, 800, 200, 0.02, dtype=np.float64)
    B = random_dcsr(rng, 500, 800, 200, 0.02, dtype=np.float64)
    _check([A, B], 17)
    # disjoint stored rows: nothing survives
    C = W.from_coo([1, 3], [0, 1], np.ones(2, np.float32), 6, 4, fmt=W.DCSR)
    D = W.from_coo([2, 4], [0, 1], np.ones(2, np.float32), 6, 4, fmt=W.DCSR)
    _check([C, D], 4)


def test_recursive_hypersparse_scaled():
    """C3-shaped operands (10^6 stored rows of 10^8 at scale 0.01 -> 10^4 of 10^6): two DCSR matrices
    sharing about half of their stored rows."""
    wl = W.build("c3", 0.01)
    A = wl.ops[0]
    rng = np.random.default_rng(3)
    keep = rng.random(A.nouter) < 0.5
    rows = np.repeat(A.outer_crd, np.diff(A.pos))
    sel = np.repeat(keep, np.diff(A.pos))
    B = W.from_coo(rows[sel], A.crd[sel], (A.val[sel] * 2).astype(np.float32), A.nrows, A.ncols, fmt=W.DCSR)
    _check([A, B], 200)
