"""GPU parity of the ESC scatter kernels (nacho_spgemm_work, nacho_partition_esc, nacho_spgemm_esc,
nacho_sssmm_esc_count / nacho_sssmm_esc) against the oracle, through the C ABI: the work prefix, every
boundary field and the whole output (pos, crd, val) bit-exact -- the products and their k-ordered
left fold are the same operations in the same order on both sides (reading R23 / R24)."""
import numpy as np
import pytest
import torch

import oracle as O
import workloads as W
from tests.util import random_csr

pytestmark = pytest.mark.gpu


def _csr(rows, cols, vals, M, N, dtype=np.float32):
    return W.from_coo(rows, cols, np.asarray(vals, dtype=dtype), M, N, dtype=dtype)


def _gpu(A):
    return A.to("cuda")


def _check_partition(A, B, P):
    import paper_2604_17198_b200 as N
    dA, dB = _gpu(A), _gpu(B)
    Wd = N.spgemm_work(dA, dB)
    Wr = O.spgemm_work(A, B)
    assert np.array_equal(Wd.cpu().numpy(), Wr)
    qstar = int(Wr[-1])
    parts = N.partition_esc(dA, dB, Wd, qstar, P)
    ref = O.esc_partition(A, B, P)
    assert np.array_equal(parts.query.cpu().numpy(), ref.query)
    assert np.array_equal(parts.row.cpu().numpy(), ref.row)
    assert np.array_equal(parts.row_pos.cpu().numpy(), ref.row_pos)
    assert np.array_equal(parts.col.cpu().numpy(), ref.col)
    assert np.array_equal(parts.pos.cpu().numpy(), ref.pos)


def _check_spgemm(A, B, P=None):
    import paper_2604_17198_b200 as N
    c_pos, c_crd, c_val = N.spgemm(_gpu(A), _gpu(B), P=P)
    r_pos, r_crd, r_val = O.spgemm(A, B)
    assert np.array_equal(c_pos.cpu().numpy(), r_pos)
    assert np.array_equal(c_crd.cpu().numpy(), r_crd)
    assert np.array_equal(c_val.cpu().numpy(), r_val)     # bit-exact (same products, same fold order)


def _check_sssmm(S, A, B, P=None):
    import paper_2604_17198_b200 as N
    z_pos, z_crd, z_val = N.sssmm(_gpu(S), _gpu(A), _gpu(B), P=P)
    r_pos, r_crd, r_val = O.sssmm(S, A, B)
    assert np.array_equal(z_pos.cpu().numpy(), r_pos)
    assert np.array_equal(z_crd.cpu().numpy(), r_crd)
    assert np.array_equal(z_val.cpu().numpy(), r_val)


@pytest.mark.parametrize("seed,P", [(0, 1), (1, 3), (2, 17), (3, 256), (4, 5000)])
def test_work_and_partition(seed, P):
    rng = np.random.default_rng(seed)
    A = random_csr(rng, 57, 41, 0.12, empty_frac=0.3, dense_rows=(9,))
    B = random_csr(rng, 41, 63, 0.1, empty_frac=0.3, dense_rows=(5,))
    _check_partition(A, B, P)


def test_worked_example():
    A = _csr([0, 0, 1], [0, 2, 1], [1, 2, 3], 2, 3)
    B = _csr([0, 0, 1, 2, 2], [1, 3, 0, 1, 2], [1, 2, 4, 5, 6], 3, 4)
    for P in (1, 2, 3, 5, 9):
        _check_partition(A, B, P)
        _check_spgemm(A, B, P)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("seed,P", [(0, None), (1, 7), (2, 1), (3, 997)])
def test_spgemm_random(dtype, seed, P):
    rng = np.random.default_rng(seed)
    A = random_csr(rng, 300, 200, 0.03, dtype=dtype, dense_rows=(17,))
    B = random_csr(rng, 200, 250, 0.04, dtype=dtype, dense_rows=(3, 150))
    _check_spgemm(A, B, P)


def test_spgemm_edge_cases():
    # no product at all (B's row 2 empty), then a single product, then a structural zero
    _check_spgemm(_csr([0, 1], [2, 2], [1, 1], 3, 4), _csr([0, 1], [1, 3], [1, 1], 4, 5))
    _check_spgemm(_csr([1], [0], [2], 3, 1), _csr([0], [4], [3], 1, 6))
    _check_spgemm(_csr([0, 0], [0, 1], [1, 1], 1, 2), _csr([0, 1], [0, 0], [1, -1], 2, 1))
    # the fp32 order-dependent fold: (1e8 + -1e8) + 1 = 1
    A = _csr([0, 0, 0], [0, 1, 2], [1, 1, 1], 1, 3)
    B = _csr([0, 1, 2], [0, 0, 0], [1e8, -1e8, 1], 3, 1)
    _check_spgemm(A, B)
    # one dense row times a dense-row B: long runs of one (i, j)
    rng = np.random.default_rng(7)
    A = random_csr(rng, 40, 60, 0.02, dense_rows=(0, 39))
    B = random_csr(rng, 60, 70, 0.05, dense_rows=tuple(range(0, 60, 2)))
    _check_spgemm(A, B, 13)


def test_spgemm_c2_operands_scaled():
    wl = W.build("c2", 0.01)
    A, B = wl.ops[0], wl.ops[1]
    _check_spgemm(A, B)
    _check_spgemm(A, B, 4096)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("seed,P", [(0, None), (1, 11), (2, 1)])
def test_sssmm_random(dtype, seed, P):
    rng = np.random.default_rng(seed)
    A = random_csr(rng, 200, 150, 0.04, dtype=dtype, dense_rows=(7,))
    B = random_csr(rng, 150, 180, 0.04, dtype=dtype, dense_rows=(2,))
    S = random_csr(rng, 200, 180, 0.1, dtype=dtype, dense_rows=(7,))
    _check_sssmm(S, A, B, P)


def test_sssmm_edge_cases():
    rng = np.random.default_rng(3)
    A = random_csr(rng, 30, 20, 0.2)
    B = random_csr(rng, 20, 25, 0.2)
    empty = _csr([], [], [], 30, 25)
    _check_sssmm(empty, A, B)                           # nothing sampled
    _check_sssmm(random_csr(rng, 30, 25, 1.0, empty_frac=0.0), A, B, 7)   # all sampled = SpGEMM scaled


def test_sssmm_c2_operands_scaled():
    wl = W.build("c2", 0.01)
    A, B, S = wl.ops
    _check_sssmm(S, A, B)


def test_esc_rejects_bad_arguments():
    import paper_2604_17198_b200 as N
    rng = np.random.default_rng(1)
    A = _gpu(random_csr(rng, 10, 8, 0.3))
    B = _gpu(random_csr(rng, 9, 8, 0.3))   # A.ncols != B.nrows
    with pytest.raises(N.NachoError):
        N.spgemm_work(A, B)
