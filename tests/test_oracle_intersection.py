"""Pins of the k-way intersection oracle (oracle_hadamard_k, oracle_hadamard_counts, oracle_inner_k)
against what the paper and the mathematics fix: Listing 1's worked vectors (P:333-344 with
fig:sparse-vec-rep), fig:vec_lb_example's partition, dense brute force on tiny
inputs, closed forms (k = 1, A (.) A, the Frobenius norm) and the count invariants."""
import numpy as np
import pytest

import oracle as O
import workloads as W
from tests.util import random_csr


def _vec_row(cols, N, vals):
    return W.from_coo([0] * len(cols), cols, np.asarray(vals), 1, N, dtype=np.asarray(vals).dtype)


def test_listing1_three_finger_product(golden):
    g = golden("listing1_vec3_mul.json")
    N = g["N"]
    base = {"a": 2.0, "b": 10.0, "c": 100.0}   # value of position q: base + q (distinct, exact in fp64)
    ops = [_vec_row(g["vectors"][v], N, base[v] + np.arange(len(g["vectors"][v]), dtype=np.float64))
           for v in "abc"]
    z_pos, z_crd, z_val = O.hadamard_k(ops)
    assert z_crd.tolist() == g["intersection"]
    assert z_pos.tolist() == [0, len(g["intersection"])]
    expect = [(base["a"] + pa) * (base["b"] + pb) * (base["c"] + pc) for pa, pb, pc in g["positions_abc"]]
    assert z_val.tolist() == expect


def test_fig2_intersection_counts_per_partition(golden):
    g = golden("listing1_vec3_mul.json")["fig2_vec_lb"]
    f2 = golden("fig2_vec_lb.json")
    ops = [_vec_row(f2["vectors"][v], f2["N"], np.ones(len(f2["vectors"][v]), np.float32)) for v in "abc"]
    parts = O.partition_rank(ops, f2["P"])
    assert parts.row.tolist() == [b[0] for b in f2["boundaries_row_col"]]
    assert O.hadamard_counts(ops, parts).tolist() == g["intersection_counts_per_partition"]
    assert O.hadamard_k(ops)[1].tolist() == g["intersection"]


@pytest.mark.parametrize("k", [2, 3, 4])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_hadamard_against_dense(k, dtype):
    rng = np.random.default_rng(70 + k)
    for _ in range(20):
        M, N = int(rng.integers(1, 25)), int(rng.integers(1, 30))
        base = random_csr(rng, M, N, float(rng.uniform(0.1, 0.8)), dtype=dtype)
        ops = [base] + [random_csr(rng, M, N, float(rng.uniform(0.1, 0.8)), dtype=dtype, base=base, share=0.7)
                        for _ in range(k - 1)]
        masks = [W.to_dense(A) != 0 for A in ops]   # values in [0.5, 1.5): stored == nonzero
        both = np.logical_and.reduce(masks)
        dense = W.to_dense(ops[0]).astype(dtype)
        for A in ops[1:]:
            dense = (dense * W.to_dense(A).astype(dtype)).astype(dtype)   # left fold, rounded per step
        z_pos, z_crd, z_val = O.hadamard_k(ops)
        rows, cols = np.nonzero(both)
        assert np.array_equal(z_pos, np.concatenate([[0], np.cumsum(both.sum(axis=1))]))
        assert np.array_equal(z_crd, cols.astype(np.int32))
        assert np.array_equal(z_val.view(np.uint8), dense[rows, cols].astype(dtype).view(np.uint8))


def test_special_cases():
    rng = np.random.default_rng(9)
    A = random_csr(rng, 30, 40, 0.3)
    # k = 1: Z = A
    zp, zc, zv = O.hadamard_k([A])
    assert np.array_equal(zp, A.pos) and np.array_equal(zc, A.crd) and np.array_equal(zv, A.val)
    # A (.) A: same structure, squares (fp32 products)
    zp, zc, zv = O.hadamard_k([A, A])
    assert np.array_equal(zp, A.pos) and np.array_equal(zc, A.crd)
    assert np.array_equal(zv, (A.val * A.val).astype(np.float32))
    # with an empty operand: empty Z
    E = W.from_coo([], [], np.zeros(0, np.float32), 30, 40)
    zp, zc, zv = O.hadamard_k([A, E, A])
    assert zp.tolist() == [0] * 31 and len(zc) == 0
    # inner product: <A, A> = ||A||_F^2, k = 1 sums the values, with an empty operand 0
    assert O.inner_k([A, A]) == pytest.approx(float(np.sum(A.val.astype(np.float64) ** 2)), rel=1e-12)
    assert O.inner_k([A]) == pytest.approx(float(np.sum(A.val.astype(np.float64))), rel=1e-12)
    assert O.inner_k([A, E]) == 0.0


@pytest.mark.parametrize("k", [2, 3])
def test_inner_against_dense(k):
    rng = np.random.default_rng(30 + k)
    for _ in range(10):
        M, N = int(rng.integers(1, 40)), int(rng.integers(1, 40))
        base = random_csr(rng, M, N, 0.4, dtype=np.float64)
        ops = [base] + [random_csr(rng, M, N, 0.4, dtype=np.float64, base=base, share=0.6) for _ in range(k - 1)]
        prod = np.ones((M, N))
        for A in ops:
            prod = prod * W.to_dense(A)
        assert O.inner_k(ops) == pytest.approx(float(prod.sum()), rel=1e-12, abs=1e-300)


@pytest.mark.parametrize("k", [2, 3])
def test_counts_sum_to_nnz_and_respect_cuts(k):
    rng = np.random.default_rng(50 + k)
    base = random_csr(rng, 60, 80, 0.2, dense_rows=[7])
    ops = [base] + [random_csr(rng, 60, 80, 0.15, base=base, share=0.6) for _ in range(k - 1)]
    zp, zc, _ = O.hadamard_k(ops)
    rows = np.repeat(np.arange(60), np.diff(zp))
    for P in (1, 3, 17, 200):
        parts = O.partition_rank(ops, P)
        cnt = O.hadamard_counts(ops, parts)
        assert cnt.sum() == len(zc)
        # brute force: coordinates in [b_p, b_{p+1}) lexicographically
        for p in range(P):
            lo = (parts.row[p], parts.col[p])
            hi = (parts.row[p + 1], parts.col[p + 1]) if p + 1 < P else (60, 0)
            n = sum(1 for r, c in zip(rows, zc) if lo <= (r, c) < hi)
            assert n == cnt[p]
