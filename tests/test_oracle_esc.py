"""Pins of the ESC scatter-kernel oracle (oracle_spgemm_work, oracle_esc_partition, oracle_spgemm,
oracle_sssmm; P:2063-2074 expand-sort-contract, Listing 6's broadcast-scaled cost P:1714-1727,
SSSMM P:2540-2559) against what the mathematics fixes: the dense product on small integers (exact)
and in fp64, the structural (boolean) product, a different closed form of the expansion size,
explicit enumeration of the expansion on tiny inputs, identities, a hand-worked example, and an fp32
case whose value depends on the summation order (reading R23: left fold over k ascending)."""
import numpy as np
import pytest

import oracle as O
import workloads as W
from tests.util import random_csr


def _csr(rows, cols, vals, M, N, dtype=np.float32):
    return W.from_coo(rows, cols, np.asarray(vals, dtype=dtype), M, N, dtype=dtype)


def _dense_from(pos, crd, val, M, N):
    D = np.zeros((M, N), np.float64)
    S = np.zeros((M, N), bool)
    for i in range(M):
        for q in range(int(pos[i]), int(pos[i + 1])):
            D[i, int(crd[q])] = val[q]
            S[i, int(crd[q])] = True
    return D, S


def _expansion(A, B):
    """Every product of the expansion T in its order: (i, A position q, B position r, j)."""
    T = []
    for i in range(A.nrows):
        for q in range(int(A.pos[i]), int(A.pos[i + 1])):
            k = int(A.crd[q])
            for r in range(int(B.pos[k]), int(B.pos[k + 1])):
                T.append((i, q, r, int(B.crd[r])))
    return T


# ---------------------------------------------------------------- a hand-worked example
# A (2 x 3): row 0 = {k0: 1, k2: 2}, row 1 = {k1: 3}.  B (3 x 4): row 0 = {j1: 1, j3: 2},
# row 1 = {j0: 4}, row 2 = {j1: 5, j2: 6}.
# Costs nnz(B_k) of A's entries (q = 0, 1, 2 -> k = 0, 2, 1): 2, 2, 1 -> W = [0, 2, 4, 5], Q* = 5.
# T = (0,q0,r0,j1) (0,q0,r1,j3) (0,q1,r3,j1) (0,q1,r4,j2) (1,q2,r2,j0).
# C row 0: j1 = 1*1 + 2*5 = 11, j2 = 2*6 = 12, j3 = 1*2 = 2; row 1: j0 = 3*4 = 12.
# P = 2: Q = [0, 2, 5]; b_1 = product 2 = (row 0, q 1, r 3, j 1).  P = 3: Q = [0, 1, 3, 5];
# b_1 = product 1 = (0, q0, r1, j3), b_2 = product 3 = (0, q1, r4, j2).
def _worked():
    A = _csr([0, 0, 1], [0, 2, 1], [1, 2, 3], 2, 3)
    B = _csr([0, 0, 1, 2, 2], [1, 3, 0, 1, 2], [1, 2, 4, 5, 6], 3, 4)
    return A, B


def test_worked_example_work_and_product():
    A, B = _worked()
    assert O.spgemm_work(A, B).tolist() == [0, 2, 4, 5]
    c_pos, c_crd, c_val = O.spgemm(A, B)
    assert c_pos.tolist() == [0, 3, 4]
    assert c_crd.tolist() == [1, 2, 3, 0]
    assert c_val.tolist() == [11.0, 12.0, 2.0, 12.0]


def test_worked_example_partitions():
    A, B = _worked()
    p2 = O.esc_partition(A, B, 2)
    assert p2.query.tolist() == [0, 2, 5]
    assert p2.row.tolist() == [0, 0, 2]
    assert p2.pos2().tolist() == [[0, 0], [1, 3], [3, 5]]
    assert p2.col.tolist() == [1, 1, 0]
    p3 = O.esc_partition(A, B, 3)
    assert p3.query.tolist() == [0, 1, 3, 5]
    assert p3.pos2().tolist() == [[0, 0], [0, 1], [1, 4], [3, 5]]
    assert p3.col.tolist() == [1, 3, 2, 0]


# ---------------------------------------------------------------- work: a second closed form
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_work_equals_column_count_times_row_length(seed):
    rng = np.random.default_rng(seed)
    A = random_csr(rng, 23, 17, 0.2)
    B = random_csr(rng, 17, 29, 0.25, dense_rows=(3,))
    W_ = O.spgemm_work(A, B)
    colcount = np.bincount(A.crd, minlength=17)                   # nnz of A's column k
    rowlen = np.diff(B.pos)                                       # nnz of B's row k
    assert W_[-1] == int(np.dot(colcount, rowlen))
    assert W_[-1] == len(_expansion(A, B))
    assert np.all(np.diff(W_) == rowlen[A.crd])


# ---------------------------------------------------------------- partition: explicit enumeration
@pytest.mark.parametrize("seed,P", [(3, 1), (4, 5), (5, 16), (6, 64), (7, 200)])
def test_partition_locates_product_Qp(seed, P):
    rng = np.random.default_rng(seed)
    A = random_csr(rng, 19, 13, 0.25, empty_frac=0.3)
    B = random_csr(rng, 13, 21, 0.2, dense_rows=(2,), empty_frac=0.3)
    T = _expansion(A, B)
    parts = O.esc_partition(A, B, P)
    Q = parts.query
    assert Q[0] == 0 and Q[-1] == len(T)
    assert np.all(np.diff(Q) >= len(T) // P) and np.all(np.diff(Q) <= -(-len(T) // P))   # equal work
    pp = parts.pos2()
    for p in range(P + 1):
        if Q[p] >= len(T):
            assert (parts.row[p], pp[p, 0], pp[p, 1], parts.col[p]) == (A.nrows, A.nnz, B.nnz, 0)
        else:
            i, q, r, j = T[Q[p]]
            assert (parts.row[p], pp[p, 0], pp[p, 1], parts.col[p]) == (i, q, r, j)


def test_empty_expansion():
    A = _csr([0, 1], [2, 2], [1, 1], 3, 4)
    B = _csr([0, 1], [1, 3], [1, 1], 4, 5)      # row 2 of B is empty: no product
    assert O.spgemm_work(A, B)[-1] == 0
    parts = O.esc_partition(A, B, 4)
    assert parts.row.tolist() == [3] * 5
    c_pos, c_crd, c_val = O.spgemm(A, B)
    assert c_pos.tolist() == [0, 0, 0, 0] and len(c_crd) == 0


# ---------------------------------------------------------------- the product
@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_spgemm_small_integers_exact_and_structural(seed):
    rng = np.random.default_rng(seed)
    A = random_csr(rng, 31, 22, 0.2, ints=True, dense_rows=(5,))
    B = random_csr(rng, 22, 27, 0.2, ints=True, dense_rows=(1,))
    c_pos, c_crd, c_val = O.spgemm(A, B)
    D, S = _dense_from(c_pos, c_crd, c_val, 31, 27)
    DA, DB = W.to_dense(A), W.to_dense(B)
    assert np.array_equal(D, DA @ DB)                               # exact: small integers
    assert np.array_equal(S, ((DA != 0).astype(int) @ (DB != 0).astype(int)) > 0)   # structure
    assert all(np.all(np.diff(c_crd[c_pos[i]:c_pos[i + 1]]) > 0) for i in range(31))


def test_structural_zero_is_stored():
    A = _csr([0, 0], [0, 1], [1, 1], 1, 2)
    B = _csr([0, 1], [0, 0], [1, -1], 2, 1)
    c_pos, c_crd, c_val = O.spgemm(A, B)
    assert c_pos.tolist() == [0, 1] and c_crd.tolist() == [0] and c_val.tolist() == [0.0]


def test_spgemm_fp64_against_dense():
    rng = np.random.default_rng(11)
    A = random_csr(rng, 40, 30, 0.15, dtype=np.float64, dense_rows=(7,))
    B = random_csr(rng, 30, 35, 0.15, dtype=np.float64, dense_rows=(4,))
    c_pos, c_crd, c_val = O.spgemm(A, B)
    D, _ = _dense_from(c_pos, c_crd, c_val, 40, 35)
    ref = W.to_dense(A) @ W.to_dense(B)
    assert np.max(np.abs(D - ref)) <= 1e-12 * np.max(np.abs(ref))


def test_fp32_fold_is_left_to_right_over_k():
    # products 1e8, -1e8, 1 at k = 0, 1, 2: (1e8 + -1e8) + 1 = 1; the reverse order gives 0 in fp32
    A = _csr([0, 0, 0], [0, 1, 2], [1, 1, 1], 1, 3)
    B = _csr([0, 1, 2], [0, 0, 0], [1e8, -1e8, 1], 3, 1)
    assert O.spgemm(A, B)[2].tolist() == [1.0]
    B2 = _csr([0, 1, 2], [0, 0, 0], [1, -1e8, 1e8], 3, 1)
    assert O.spgemm(A, B2)[2].tolist() == [0.0]                     # (1 + -1e8) + 1e8 = 0 in fp32


def test_identities():
    rng = np.random.default_rng(5)
    B = random_csr(rng, 12, 15, 0.3)
    I = _csr(range(12), range(12), np.ones(12), 12, 12)
    c_pos, c_crd, c_val = O.spgemm(I, B)
    assert np.array_equal(c_pos, B.pos) and np.array_equal(c_crd, B.crd) and np.array_equal(c_val, B.val)
    I2 = _csr(range(15), range(15), np.ones(15), 15, 15)
    c_pos, c_crd, c_val = O.spgemm(B, I2)
    assert np.array_equal(c_pos, B.pos) and np.array_equal(c_crd, B.crd) and np.array_equal(c_val, B.val)


# ---------------------------------------------------------------- sampled SpGEMM
@pytest.mark.parametrize("seed", [0, 1])
def test_sssmm_small_integers(seed):
    rng = np.random.default_rng(seed)
    A = random_csr(rng, 25, 18, 0.2, ints=True)
    B = random_csr(rng, 18, 21, 0.2, ints=True, dense_rows=(2,))
    S = random_csr(rng, 25, 21, 0.3, ints=True)
    z_pos, z_crd, z_val = O.sssmm(S, A, B)
    D, Sz = _dense_from(z_pos, z_crd, z_val, 25, 21)
    DA, DB, DS = W.to_dense(A), W.to_dense(B), W.to_dense(S)
    struct = (((DA != 0).astype(int) @ (DB != 0).astype(int)) > 0) & (DS != 0)
    assert np.array_equal(Sz, struct)
    assert np.array_equal(D, np.where(struct, DS * (DA @ DB), 0.0))


def test_sssmm_fp64_against_dense():
    rng = np.random.default_rng(9)
    A = random_csr(rng, 30, 20, 0.2, dtype=np.float64)
    B = random_csr(rng, 20, 26, 0.2, dtype=np.float64)
    S = random_csr(rng, 30, 26, 0.4, dtype=np.float64)
    z_pos, z_crd, z_val = O.sssmm(S, A, B)
    D, Sz = _dense_from(z_pos, z_crd, z_val, 30, 26)
    DA, DB, DS = W.to_dense(A), W.to_dense(B), W.to_dense(S)
    ref = np.where(Sz, DS * (DA @ DB), 0.0)
    assert np.max(np.abs(D - ref)) <= 1e-12 * max(np.max(np.abs(ref)), 1.0)
