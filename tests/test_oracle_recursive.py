"""Pins of the recursive-partitioning oracle (Alg. 2 on the DCSR Hadamard product, Listing
emul-dcsr2-rewritten): fig:dcsr-mul-partition's worked example, brute force
on tiny random DCSR operands (surviving rows, T, T', the rank of every boundary in the remapped
space, Z against the CSR intersection of the same matrices), and the balance bound."""
import numpy as np
import pytest

import oracle as O
import workloads as W
from tests.util import random_dcsr


def _dcsr(entries, shape, vals=None):
    r = [e[0] for e in entries]
    c = [e[1] for e in entries]
    v = np.asarray(vals if vals is not None else np.arange(1, len(entries) + 1), np.float32)
    return W.from_coo(r, c, v, shape[0], shape[1], fmt=W.DCSR)


def test_fig3b_recursive_partition(golden):
    g = golden("fig3b_dcsr_mul_partition.json")
    A, B = _dcsr(g["A"], g["shape"]), _dcsr(g["B"], g["shape"])
    rm = O.dcsr_rows_intersect([A, B])
    assert rm.rows.tolist() == g["surviving_rows"]
    assert rm.T.tolist() == g["T"] and rm.Tp.tolist() == g["T_prime"]
    parts = O.partition_remapped([A, B], rm, g["P"])
    assert [[int(r), int(c)] for r, c in zip(parts.row, parts.col)] == g["boundaries_row_col"]
    assert parts.row_pos.tolist() == g["boundary_row_pos"]
    assert parts.pos2().tolist() == g["boundary_positions_AB"]
    assert np.diff(parts.pos2().sum(axis=1)).tolist() == g["work_per_partition"]
    zo, zp, zc, zv = O.dcsr_hadamard([A, B], rm)
    assert zo.tolist() == g["Z_outer"] and zp.tolist() == g["Z_pos"]
    assert [[int(zo[s]), int(c)] for s in range(len(zo)) for c in zc[zp[s]:zp[s + 1]]] == g["Z"]


def _entries(A):
    out = []
    for ip in range(A.nouter):
        r = int(A.outer_crd[ip])
        for q in range(int(A.pos[ip]), int(A.pos[ip + 1])):
            out.append((r, int(A.crd[q]), q))
    return out


@pytest.mark.parametrize("k", [2, 3])
def test_recursive_against_brute_force(k):
    rng = np.random.default_rng(40 + k)
    for _ in range(25):
        M, N = int(rng.integers(2, 60)), int(rng.integers(2, 40))
        ops = [random_dcsr(rng, M, N, int(rng.integers(1, M + 1)), float(rng.uniform(0.05, 0.6))) for _ in range(k)]
        rm = O.dcsr_rows_intersect(ops)
        stored = [set(int(r) for r in A.outer_crd) for A in ops]
        surv = sorted(set.intersection(*stored))
        assert rm.rows.tolist() == surv
        for s, r in enumerate(surv):
            ips = [int(np.searchsorted(A.outer_crd, r)) for A in ops]
            assert rm.ip[:, s].tolist() == ips
            assert rm.T[s] == sum(int(A.pos[i + 1] - A.pos[i]) for A, i in zip(ops, ips))
        assert rm.Tp.tolist() == np.concatenate([[0], np.cumsum(rm.T)]).tolist()
        # the remapped multiset: every surviving row's entries, lexicographic (row, col)
        E = sorted((r, c) for A in ops for (r, c, q) in _entries(A) if r in set(surv))
        assert len(E) == rm.Tp[-1]
        for P in (1, 2, 5, 11):
            parts = O.partition_remapped(ops, rm, P)
            for p in range(1, P):
                Q = (p * len(E)) // P
                if Q >= len(E):
                    assert parts.row_pos[p] == rm.S
                    continue
                r, c = E[Q]
                assert (parts.row[p], parts.col[p]) == (r, c)
                assert parts.row_pos[p] == surv.index(r)
                for o, A in enumerate(ops):   # operand o's first entry at or after (r, c) in row r
                    ip = int(rm.ip[o, parts.row_pos[p]])
                    seg = A.crd[A.pos[ip]:A.pos[ip + 1]]
                    assert parts.pos[p * k + o] == A.pos[ip] + int(np.searchsorted(seg, c))
            # Theorem 1 bound with Delta = k: every partition's work within k of T'/P
            w = np.diff([0] + [int(x) for x in parts.query[1:P]] + [len(E)])
            assert (np.abs(w - len(E) / P) <= k).all()
        # Z: the CSR intersection of the same matrices, restricted to the surviving rows
        zo, zp, zc, zv = O.dcsr_hadamard(ops, rm)
        csr = [W.from_coo([r for (r, c, q) in _entries(A)], [c for (r, c, q) in _entries(A)],
                          np.asarray([A.val[q] for (r, c, q) in _entries(A)], np.float32), M, N) for A in ops]
        cp, cc, cv = O.hadamard_k(csr)
        got = [(int(zo[s]), int(c)) for s in range(len(zo)) for c in zc[zp[s]:zp[s + 1]]]
        want = [(r, int(c)) for r in range(M) for c in cc[cp[r]:cp[r + 1]]]
        assert got == want
        assert np.array_equal(zv.view(np.uint8), cv.view(np.uint8))
