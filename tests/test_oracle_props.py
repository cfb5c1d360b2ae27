"""Oracle pinned to brute force, closed forms, textbook special cases and the paper's invariants.

Invariants: I1 monotone boundaries, I2 exact cover, I3 Theorem 1,
I4 the 2-Delta balance corollary, I5 equal coordinates in one partition,
I6 positions are lower bounds, I7 probe budget, I8 single writer.
"""
import bisect
import math

import numpy as np
import pytest

import oracle as O
import workloads as W
from tests.util import brute_force_boundary, entries, random_csr, random_dcsr


def _instances(seed, n, kmax=4, dcsr=False):
    rng = np.random.default_rng(seed)
    for _ in range(n):
        M = int(rng.integers(1, 7))
        N = int(rng.integers(1, 9))
        k = int(rng.integers(1, kmax + 1))
        dens = float(rng.uniform(0.0, 0.8))
        base = random_csr(rng, M, N, dens)
        ops = [base] + [random_csr(rng, M, N, dens * 0.5, base=base, share=0.5) for _ in range(k - 1)]
        yield rng, ops


def _check_parts_eq(a, b):
    assert a.row.tolist() == b.row.tolist()
    assert a.col.tolist() == b.col.tolist()
    assert a.row_pos.tolist() == b.row_pos.tolist()
    assert a.pos.tolist() == b.pos.tolist()
    assert a.query.tolist() == b.query.tolist()


def test_rank_equals_alg1_equals_brute_force():
    for rng, ops in _instances(11, 300):
        qstar = sum(A.nnz for A in ops)
        for P in (1, 2, 3, 5, max(1, qstar + 3)):
            pr = O.partition_rank(ops, P)
            pa = O.partition_alg1(ops, P)
            _check_parts_eq(pr, pa)
            for p in range(1, P):
                (bi, bj), bpos = brute_force_boundary(ops, int(pr.query[p]))
                assert (int(pr.row[p]), int(pr.col[p])) == (bi, bj)
                assert pr.pos2()[p].tolist() == bpos


def test_queries_floor_and_total_cost():
    for qstar, P in [(0, 4), (12, 4), (13, 4), (4_000_000_000, 999_983), (7, 10)]:
        Q = O.queries(qstar, P)
        assert Q.tolist() == [p * qstar // P for p in range(P + 1)]


def _invariants(ops, P, parts, probes=None):
    k = len(ops)
    pos = parts.pos2()
    nnz = np.array([A.nnz for A in ops])
    qstar = int(nnz.sum())
    # I1: lexicographically non-decreasing boundaries, monotone positions
    keys = list(zip(parts.row.tolist(), parts.col.tolist()))
    assert all(keys[p] <= keys[p + 1] for p in range(P))
    assert (np.diff(pos, axis=0) >= 0).all()
    # I2: exact cover of every operand's positions
    assert pos[0].tolist() == [0] * k and pos[P].tolist() == nnz.tolist()
    # I3 (Theorem 1): 0 <= Q - C(b) < Delta for interior p; Delta = max multiplicity of a coordinate
    ents = [entries(A) for A in ops]
    allk = sorted(e for es in ents for e in es)
    mult = max([allk.count(e) for e in set(allk)] or [1])
    cost = pos.sum(axis=1)
    for p in range(1, P):
        d = int(parts.query[p]) - int(cost[p])
        assert 0 <= d < max(mult, 1)
    # I4: balance |work_p - Q*/P| < Delta + 1
    work = np.diff(cost)
    assert (np.abs(work - qstar / P) < mult + 1).all()
    # I5/I6: positions are lower bounds of the boundary coordinate in every operand
    for p in range(1, P):
        key = (int(parts.row[p]), int(parts.col[p]))
        if key[0] >= ops[0].nrows:
            continue
        for o in range(k):
            assert pos[p, o] == bisect.bisect_left(ents[o], key)
    # I7: probe budget ceil(log2(M+1)) + ceil(log2 N) cost evaluations per boundary
    if probes is not None:
        M, N = ops[0].nrows, ops[0].ncols
        bound = math.ceil(math.log2(M + 1)) + math.ceil(math.log2(max(N, 1)))
        assert probes.max() <= bound


def test_invariants_random():
    for rng, ops in _instances(12, 200):
        qstar = sum(A.nnz for A in ops)
        for P in (1, 2, 4, 7, qstar + 5):
            parts, probes = O.partition_alg1(ops, P, with_probes=True)
            _invariants(ops, P, parts, probes)


def test_single_operand_closed_form():
    """k = 1: the cut is a plain nnz split -- pos = Q_p, row = upper_bound(pos, Q_p) - 1, col = crd[Q_p]."""
    rng = np.random.default_rng(3)
    for _ in range(100):
        A = random_csr(rng, int(rng.integers(1, 40)), int(rng.integers(1, 40)), 0.2, empty_frac=0.4)
        for P in (1, 3, 8, A.nnz + 2):
            parts = O.partition_rank([A], P)
            for p in range(1, P):
                q = int(parts.query[p])
                if q >= A.nnz:
                    assert parts.row[p] == A.nrows
                    continue
                assert parts.pos[p] == q
                assert parts.row[p] == np.searchsorted(A.pos, q, side="right") - 1
                assert parts.col[p] == A.crd[q]


def test_dcsr_closed_form_and_alg1():
    rng = np.random.default_rng(4)
    for _ in range(60):
        A = random_dcsr(rng, int(rng.integers(2, 200)), int(rng.integers(1, 30)), int(rng.integers(1, 12)), 0.3)
        assert O.validate(A) == 0
        for P in (1, 2, 5, A.nnz + 3):
            pr = O.partition_rank([A], P)
            pa = O.partition_alg1([A], P)
            _check_parts_eq(pr, pa)
            for p in range(1, P):
                q = int(pr.query[p])
                rp = np.searchsorted(A.pos, q, side="right") - 1
                assert pr.row_pos[p] == rp and pr.row[p] == A.outer_crd[rp] and pr.col[p] == A.crd[q]


def test_two_operand_one_row_is_merge_path():
    """k = 2 on one row with disjoint coordinates reduces to the merge-path diagonal split."""
    rng = np.random.default_rng(5)
    for _ in range(100):
        N = 64
        perm = rng.permutation(N)
        na, nb = int(rng.integers(0, 20)), int(rng.integers(0, 20))
        a, b = np.sort(perm[:na]), np.sort(perm[na:na + nb])
        ops = [W.from_coo([0] * len(v), v, np.ones(len(v)), 1, N) for v in (a, b)]
        merged = sorted([(x, 0) for x in a] + [(x, 1) for x in b])
        P = 5
        parts = O.partition_rank(ops, P)
        for p in range(1, P):
            d = int(parts.query[p])
            if d >= na + nb:
                continue
            i = sum(1 for x, s in merged[:d] if s == 0)   # textbook merge path: #a in the first d merged
            assert parts.pos2()[p].tolist() == [i, d - i]


def _dense_spmv(A, x):
    return W.to_dense(A) @ x.astype(np.float64)


@pytest.mark.parametrize("dtype,tol", [(np.float32, 1e-5), (np.float64, 1e-12)])
def test_spmv_against_dense(dtype, tol):
    rng = np.random.default_rng(6)
    for _ in range(40):
        M, N = int(rng.integers(1, 60)), int(rng.integers(1, 60))
        A = random_csr(rng, M, N, 0.2, dtype=dtype, dense_rows=[0] if rng.random() < 0.3 else ())
        x = rng.uniform(0.5, 1.5, N).astype(dtype)
        y = O.spmv(A, x)
        ref = _dense_spmv(A, x)
        scale = np.abs(W.to_dense(A)) @ np.abs(x.astype(np.float64))
        assert (np.abs(y - ref) <= tol * np.maximum(scale, 1e-300) + 0).all()


def test_spmv_special_cases():
    rng = np.random.default_rng(7)
    n = 50
    I = W.from_coo(np.arange(n), np.arange(n), np.ones(n), n, n, dtype=np.float64)
    x = rng.uniform(-2, 2, n)
    assert np.array_equal(O.spmv(I, x), x)                               # A = I -> y = x exactly
    A = random_csr(rng, 40, 30, 0.3, dtype=np.float64)
    A.val[:] = 1.0
    assert np.array_equal(O.spmv(A, np.ones(30)), np.diff(A.pos).astype(np.float64))   # row lengths
    B = random_csr(rng, 40, 30, 0.4, dtype=np.float64, ints=True)
    xi = rng.integers(-4, 5, 30).astype(np.float64)
    assert np.array_equal(O.spmv(B, xi), W.to_dense(B) @ xi)           # exact small-integer sums


def test_dcsr_spmv_compressed_y():
    rng = np.random.default_rng(8)
    A = random_dcsr(rng, 500, 40, 20, 0.3, dtype=np.float64)
    x = rng.uniform(0.5, 1.5, 40)
    y = O.spmv(A, x)
    ref = (W.to_dense(A) @ x)[A.outer_crd]
    assert np.allclose(y, ref, rtol=1e-12, atol=0)


def test_spmm_against_dense():
    rng = np.random.default_rng(9)
    A = random_csr(rng, 50, 40, 0.2, dtype=np.float32, dense_rows=[3])
    B = rng.uniform(0.5, 1.5, (40, 64)).astype(np.float32)
    C = O.spmm(A, B)
    ref = W.to_dense(A) @ B.astype(np.float64)
    scale = np.abs(W.to_dense(A)) @ np.abs(B.astype(np.float64))
    assert (np.abs(C - ref) <= 1e-5 * scale).all()
    Ai = W.from_coo(np.arange(40), np.arange(40), np.ones(40), 40, 40)
    assert np.array_equal(O.spmm(Ai, B), B)                             # A = I -> C = B


@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_spadd_against_dense(k):
    rng = np.random.default_rng(10 + k)
    for trial in range(20):
        M, N = int(rng.integers(1, 30)), int(rng.integers(1, 30))
        base = random_csr(rng, M, N, 0.3)
        ops = [base] + [random_csr(rng, M, N, 0.2, base=base, share=0.5) for _ in range(k - 1)]
        z_pos, z_crd, z_val = O.spadd_k(ops)
        mask = np.zeros((M, N), bool)
        dense = np.zeros((M, N), np.float32)
        for A in ops:
            D = W.to_dense(A).astype(np.float32)
            mask |= np.array([[False] * N for _ in range(M)]) if A.nnz == 0 else (D != 0)
            dense = dense + D                               # (a + b) + c in fp32, absent terms are +0
        rows, cols = np.nonzero(mask)
        assert z_pos.tolist() == np.concatenate([[0], np.cumsum(mask.sum(axis=1))]).tolist()
        assert z_crd.tolist() == cols.tolist()
        assert np.array_equal(z_val, dense[rows, cols])     # bit-exact fold
        # per-partition counts = brute-force count of union coordinates in [b_p, b_{p+1})
        for P in (1, 3, 6):
            parts = O.partition_rank(ops, P)
            cnt = O.spadd_counts(ops, parts)
            keys = list(zip(rows.tolist(), cols.tolist()))
            b = list(zip(parts.row.tolist(), parts.col.tolist()))
            bf = [sum(1 for c in keys if b[p] <= c < b[p + 1]) for p in range(P)]
            assert cnt.tolist() == bf


# ---------------------------------------------------------------- fp64 branches and validation codes
def _spread_values(rng, n):
    """fp64 values over ~30 binades with random signs: the order of a three-term sum then changes the
    rounded result for many entries, so a fold in any other order than the left fold fails the pin."""
    return rng.uniform(1.0, 2.0, n) * np.exp2(rng.integers(-15, 15, n)) * rng.choice([-1.0, 1.0], n)


@pytest.mark.parametrize("k", [2, 3, 4])
def test_spadd_f64_left_fold_against_dense(k):
    """oracle_spadd_k's fp64 branch (R9 left fold in operand order) against a dense fp64 evaluation
    ((0 + a_0) + a_1) + ... with absent terms +0 (x + 0 = x exactly for x != -0): bit-exact."""
    rng = np.random.default_rng(40 + k)
    order_matters = 0
    for trial in range(15):
        M, N = int(rng.integers(1, 30)), int(rng.integers(1, 30))
        base = random_csr(rng, M, N, 0.35, dtype=np.float64)
        ops = [base] + [random_csr(rng, M, N, 0.25, dtype=np.float64, base=base, share=0.6) for _ in range(k - 1)]
        for A in ops:
            A.val[:] = _spread_values(rng, A.nnz)
        z_pos, z_crd, z_val = O.spadd_k(ops)
        mask = np.zeros((M, N), bool)
        dense = np.zeros((M, N), np.float64)
        rdense = np.zeros((M, N), np.float64)
        Ds = [W.to_dense(A) for A in ops]
        for A, D in zip(ops, Ds):
            mask |= D != 0
            dense = dense + D                              # left fold in operand order
        for D in reversed(Ds):
            rdense = rdense + D                            # right-to-left fold, for discrimination only
        rows, cols = np.nonzero(mask)
        assert z_val.dtype == np.float64
        assert z_pos.tolist() == np.concatenate([[0], np.cumsum(mask.sum(axis=1))]).tolist()
        assert z_crd.tolist() == cols.tolist()
        assert np.array_equal(z_val, dense[rows, cols])
        order_matters += int((dense[rows, cols] != rdense[rows, cols]).sum())
    if k >= 3:
        assert order_matters > 0, "inputs do not discriminate the fold order"


def test_spmm_f64_against_dense():
    """oracle_spmm's fp64 branch: within 1e-12 of a dense fp64 product (relative to sum|a b|), which an
    fp32 read of A or B (~1e-8) would fail; and exact on small integers (all partial sums < 2^53)."""
    rng = np.random.default_rng(41)
    for nb in (1, 7, 64):
        A = random_csr(rng, 45, 37, 0.25, dtype=np.float64, dense_rows=[2])
        A.val[:] = rng.uniform(0.5, 1.5, A.nnz) + rng.uniform(0, 1e-9, A.nnz)   # fp64-only digits
        B = (rng.uniform(0.5, 1.5, (37, nb)) + rng.uniform(0, 1e-9, (37, nb))).astype(np.float64)
        C = O.spmm(A, B)
        assert C.dtype == np.float64
        D = W.to_dense(A)
        ref = D @ B
        scale = np.abs(D) @ np.abs(B)
        assert (np.abs(C - ref) <= 1e-12 * scale).all()
        Bf = B.astype(np.float32).astype(np.float64)       # what an fp32 read would see
        assert (np.abs(D @ Bf - ref) > 1e-12 * scale).any()
        Ai = random_csr(rng, 30, 37, 0.3, dtype=np.float64, ints=True)
        Bi = rng.integers(-4, 5, (37, nb)).astype(np.float64)
        assert np.array_equal(O.spmm(Ai, Bi), W.to_dense(Ai) @ Bi)


def _malformed_cases():
    """One malformed operand per oracle_validate reject code (oracle.c, P:1675-1684 sorted levels; R10)."""
    def csr(M, N, pos, crd):
        crd = np.asarray(crd, np.int32)
        return W.SparseMatrix(W.CSR, M, N, np.asarray(pos, np.int64), crd, np.ones(len(crd), np.float32))

    def dcsr(M, N, outer, pos, crd):
        crd = np.asarray(crd, np.int32)
        return W.SparseMatrix(W.DCSR, M, N, np.asarray(pos, np.int64), crd, np.ones(len(crd), np.float32),
                              np.asarray(outer, np.int32))
    cases = {
        1: csr(-1, 3, [0], []),                                  # negative size
        3: csr(2, 3, [1, 1, 1], [0]),                            # pos[0] != 0
        4: csr(2, 3, [0, 1, 1], [0, 2]),                         # pos[nouter] != nnz
        5: csr(3, 3, [0, 2, 1, 2], [0, 1]),                      # pos decreasing
        6: csr(2, 3, [0, 1, 2], [0, 3]),                         # crd >= ncols
        7: csr(2, 3, [0, 2, 2], [1, 1]),                         # crd not strictly increasing in a row
        8: dcsr(4, 3, [5], [0, 1], [0]),                         # stored row coordinate >= nrows
        9: dcsr(4, 3, [2, 2], [0, 1, 2], [0, 1]),                # stored rows not strictly increasing
        10: dcsr(4, 3, [1, 2], [0, 0, 1], [0]),                  # empty stored row (R10)
    }
    bad_nouter = csr(3, 3, [0, 1, 2], [0, 1])                    # CSR with nouter != nrows
    cases[2] = bad_nouter
    neg = csr(2, 3, [0, 1, 2], [0, -1])                          # negative crd -> also code 6
    return cases, neg


def test_validate_reject_codes():
    cases, neg = _malformed_cases()
    assert sorted(cases) == list(range(1, 11))
    for code, A in cases.items():
        assert O.validate(A) == code, (code, O.validate(A))
    assert O.validate(neg) == 6
    ok = W.from_coo([0, 0, 2], [1, 2, 0], [1.0, 2.0, 3.0], 3, 3)
    assert O.validate(ok) == 0
    okd = W.from_coo([0, 0, 2], [1, 2, 0], [1.0, 2.0, 3.0], 3, 3, fmt=W.DCSR)
    assert O.validate(okd) == 0
