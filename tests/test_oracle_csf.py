"""Pins of the third-order CSF oracle (3-level Alg. 1 and the 3-level union):
fig:coordinate-tree's cost functions and a worked partition, dense brute force, and the
special case of one slice, which is the CSR (two-level) algorithm."""
import numpy as np
import pytest

import oracle as O
import workloads as W
from tests.util import random_csr


def _csf(entries, shape, vals):
    e = np.asarray(entries)
    return W.csf_from_coo(e[:, 0], e[:, 1], e[:, 2], vals, shape)


def test_fig_coordinate_tree(golden):
    g = golden("fig_coordinate_tree_csf.json")
    A = _csf(g["A"], g["shape"], np.arange(1, 7))
    B = _csf(g["B"], g["shape"], np.arange(11, 18))
    c = g["cost_at_1_2_1"]
    assert O.csf_cost([A, B], 1, 2, 1) == (c["C_i"], c["C_j"], c["C_k"])
    parts = O.csf_partition_rank([A, B], g["P"])
    b = g["boundary_1"]
    assert [int(parts.row[1]), int(parts.row_pos[1]), int(parts.col[1])] == b["ijk"]
    assert parts.pos2()[1].tolist() == b["pos_AB"]
    assert parts.pos2()[2].tolist() == [6, 7]
    z = O.csf_spadd_k([A, B])
    assert len(z[4]) == g["union_nnz"] and z[0].tolist() == g["union_slices"]
    assert np.diff(z[1]).tolist() == g["union_fibers_per_slice"]


def _dense(T):
    D = np.zeros(T.shape)
    for s in range(len(T.crd0)):
        for f in range(T.pos1[s], T.pos1[s + 1]):
            for q in range(T.pos2[f], T.pos2[f + 1]):
                D[T.crd0[s], T.crd1[f], T.crd2[q]] = T.val[q]
    return D


@pytest.mark.parametrize("k", [2, 3])
def test_csf_against_dense(k):
    rng = np.random.default_rng(90 + k)
    for _ in range(15):
        shape = tuple(int(x) for x in rng.integers(1, 9, 3))
        ops = [W.random_csf(rng, shape, float(rng.uniform(0.05, 0.5))) for _ in range(k)]
        # every boundary is the entry number Q_p of the lexicographic multiset, its costs sum to Q_p
        E = sorted((i, j, kk) for T in ops for i, j, kk in zip(*np.nonzero(_dense(T))))
        for P in (1, 2, 5):
            parts = O.csf_partition_rank(ops, P)
            for p in range(1, P):
                Q = (p * len(E)) // P
                if Q >= len(E):
                    continue
                ijk = (int(parts.row[p]), int(parts.row_pos[p]), int(parts.col[p]))
                assert ijk == tuple(int(x) for x in E[Q])
                assert sum(O.csf_cost(ops, *ijk)) == sum(1 for e in E if e < E[Q])
                assert parts.pos2()[p].sum() == sum(1 for e in E if e < E[Q])
        # the union: structure = the stored coordinates of any operand, values the left fold
        c0, p1, c1, p2, c2, v = O.csf_spadd_k(ops)
        dense = [_dense(T).astype(np.float32) for T in ops]
        mask = np.logical_or.reduce([d != 0 for d in dense])
        fold = np.zeros(shape, np.float32)
        have = np.zeros(shape, bool)
        for d in dense:
            fold = np.where(d != 0, np.where(have, (fold + d).astype(np.float32), d), fold)
            have |= d != 0
        got = [(int(c0[s]), int(c1[f]), int(c2[q])) for s in range(len(c0)) for f in range(p1[s], p1[s + 1])
               for q in range(p2[f], p2[f + 1])]
        want = list(zip(*[x.tolist() for x in np.nonzero(mask)]))
        assert got == want
        assert np.array_equal(v.view(np.uint8), fold[mask].view(np.uint8))


def test_one_slice_is_the_csr_algorithm():
    rng = np.random.default_rng(5)
    base = random_csr(rng, 30, 40, 0.2)
    mats = [base, random_csr(rng, 30, 40, 0.15, base=base, share=0.5)]
    tens = []
    for A in mats:
        rows = np.repeat(np.arange(30), np.diff(A.pos))
        tens.append(W.csf_from_coo(np.zeros(len(rows), np.int64), rows, A.crd, A.val, (1, 30, 40)))
    for P in (1, 3, 17):
        pt, pc = O.csf_partition_rank(tens, P), O.partition_rank(mats, P)
        assert np.array_equal(pt.pos, pc.pos)
        assert np.array_equal(pt.row_pos[1:P], pc.row[1:P]) and np.array_equal(pt.col[1:P], pc.col[1:P])
    c0, p1, c1, p2, c2, v = O.csf_spadd_k(tens)
    zp, zc, zv = O.spadd_k(mats)
    assert np.array_equal(c2, zc) and np.array_equal(v.view(np.uint8), zv.view(np.uint8))
