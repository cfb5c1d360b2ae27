"""Pins of the DCSR k-way SpAdd oracle (Listing 2, lst:eadd-dcsr2-cfir): fig:dcsr-add-partition
in its DCSR form (A stores rows {0, 2, 4}, B rows {0, 2, 3}), the partition of DCSR
operands against the same matrices in CSR (the lexicographic definition does not depend on the
format), and dense brute force."""
import numpy as np
import pytest

import oracle as O
import workloads as W
from tests.util import random_dcsr


def _dcsr(entries, shape, vals):
    return W.from_coo([e[0] for e in entries], [e[1] for e in entries], np.asarray(vals, np.float32), shape[0],
                      shape[1], fmt=W.DCSR)


def _to_csr(A):
    rows = np.repeat(A.outer_crd.astype(np.int64), np.diff(A.pos))
    return W.from_coo(rows, A.crd, A.val, A.nrows, A.ncols, dtype=A.val.dtype)


def test_fig3a_dcsr_form(golden):
    g = golden("fig3a_dcsr_add.json")
    A = _dcsr(g["A"], g["shape"], np.arange(1, 13))
    B = _dcsr(g["B"], g["shape"], np.arange(101, 113))
    assert A.outer_crd.tolist() == [0, 2, 4] and B.outer_crd.tolist() == [0, 2, 3]
    parts = O.partition_rank([A, B], g["P"])
    assert [[int(r), int(c)] for r, c in zip(parts.row, parts.col)] == g["boundaries_row_col"]
    assert parts.pos2().tolist() == g["boundary_positions_AB"]
    assert parts.row_pos.tolist() == [0, 0, 1, 2, 3]   # lower bound of the row in A's outer level
    ent, rows = O.dcsr_spadd_counts([A, B], parts)
    assert ent.tolist() == g["spadd_counts"] and rows.tolist() == [1, 1, 1, 1]
    zo, zp, zc, zv = O.dcsr_spadd_k([A, B])
    assert zo.tolist() == [0, 2, 3, 4]                  # the union of the stored rows
    assert zp.tolist() == [z for z, r in zip(g["Z_pos"], [None] + list(range(5))) if r != 1] and zp[-1] == g["nnz_Z"]


@pytest.mark.parametrize("k", [2, 3, 4])
def test_dcsr_spadd_against_dense(k):
    rng = np.random.default_rng(60 + k)
    for _ in range(20):
        M, N = int(rng.integers(1, 50)), int(rng.integers(1, 40))
        ops = [random_dcsr(rng, M, N, int(rng.integers(1, M + 1)), float(rng.uniform(0.05, 0.5))) for _ in range(k)]
        zo, zp, zc, zv = O.dcsr_spadd_k(ops)
        dense = [W.to_dense(A).astype(np.float32) for A in ops]
        mask = np.logical_or.reduce([d != 0 for d in dense])
        rows = np.nonzero(mask.any(axis=1))[0]
        assert zo.tolist() == rows.tolist()
        # left fold in operand order over the operands that store the coordinate (values are nonzero)
        fold = np.zeros((M, N), np.float32)
        have = np.zeros((M, N), bool)
        for d in dense:
            fold = np.where(d != 0, np.where(have, (fold + d).astype(np.float32), d), fold)
            have |= d != 0
        got = [(int(zo[s]), int(c)) for s in range(len(zo)) for c in zc[zp[s]:zp[s + 1]]]
        r, c = np.nonzero(mask)
        assert got == list(zip(r.tolist(), c.tolist()))
        assert np.array_equal(zv.view(np.uint8), fold[r, c].view(np.uint8))
        # the DCSR partition is the CSR partition of the same matrices (format-independent definition)
        csr = [_to_csr(A) for A in ops]
        for P in (1, 3, 9):
            pd, pc = O.partition_rank(ops, P), O.partition_rank(csr, P)
            assert np.array_equal(pd.row, pc.row) and np.array_equal(pd.col, pc.col)
            assert np.array_equal(pd.pos, pc.pos)
            ent, nrs = O.dcsr_spadd_counts(ops, pd)
            assert ent.sum() == len(zc) and nrs.sum() == len(zo)
            assert np.array_equal(ent, O.spadd_counts(csr, pc))
