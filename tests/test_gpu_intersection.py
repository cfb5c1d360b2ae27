"""GPU parity of the k-way intersection kernels (nacho_hadamard_k, nacho_inner_k) against the CPU
oracle (oracle_hadamard_k / _counts / _inner_k, Listing 1's k-finger merge per row): Z structure,
per-partition offsets and product values bit-exact; the inner product within 1e-5 (fp32) / 1e-12
(fp64) of sum |products|."""
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


def _ops(rng, k, M, Nc, dens, dtype=np.float32, dense_rows=()):
    base = random_csr(rng, M, Nc, dens, dtype=dtype, dense_rows=dense_rows)
    return [base] + [random_csr(rng, M, Nc, dens * 0.7, dtype=dtype, base=base, share=0.6, dense_rows=dense_rows)
                     for _ in range(k - 1)]


def _check(ops, P=None, tol=None):
    dops = [A.to(DEV) for A in ops]
    k = len(ops)
    if P and -(-sum(A.nnz for A in ops) // P) + k - 1 > N.lib.nacho_spadd_tile(k):
        parts = N.partition(dops, P)   # partitions larger than a stage: rejected, never overrun
        with pytest.raises(N.NachoError):
            N.hadamard_k(dops, parts)
        return
    P = P or N.auto_partitions(dops, "spadd")
    parts = N.partition(dops, P)
    off = torch.full((P + 1,), -1, dtype=torch.int64, device=DEV)
    zp, zc, zv = N.hadamard_k(dops, parts, part_off=off)
    rp, rc, rv = O.hadamard_k(ops)
    n = int(zp[-1].item())
    assert n == len(rc)
    assert np.array_equal(zp.cpu().numpy(), rp), "Z.pos"
    assert np.array_equal(zc[:n].cpu().numpy(), rc), "Z.crd"
    assert np.array_equal(zv[:n].cpu().numpy().view(np.uint8), rv.view(np.uint8)), "Z.val bits"
    cnt = O.hadamard_counts(ops, O.partition_rank(ops, P))
    assert np.array_equal(off.cpu().numpy(), np.concatenate([[0], np.cumsum(cnt)])), "part_off"
    s = float(N.inner_k(dops, parts).item())
    ref = O.inner_k(ops)
    absum = O.inner_k([W.SparseMatrix(A.format, A.nrows, A.ncols, A.pos, A.crd, np.abs(A.val)) for A in ops])
    tol = tol or (1e-5 if ops[0].val.dtype == np.float32 else 1e-12)
    assert abs(s - ref) <= tol * max(absum, 1e-300), (s, ref)


@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_intersection_random(k):
    rng = np.random.default_rng(300 + k)
    for trial in range(6):
        M, Nc = int(rng.integers(1, 1500)), int(rng.integers(1, 4000))
        ops = _ops(rng, k, M, Nc, float(rng.uniform(0.001, 0.02)),
                   dense_rows=[int(rng.integers(M))] if trial % 2 == 0 else ())
        for P in (None, 7, 301):
            if -(-sum(A.nnz for A in ops) // P if P else 0) + k > N.lib.nacho_spadd_tile(k):
                continue   # partitions must fit the stage
            _check(ops, P)


@pytest.mark.parametrize("k", [2, 3])
def test_intersection_fp64(k):
    rng = np.random.default_rng(90 + k)
    ops = _ops(rng, k, 600, 3000, 0.006, dtype=np.float64, dense_rows=[5, 300])
    for P in (None, 50):
        _check(ops, P)


def test_intersection_edge_cases():
    z = W.from_coo([], [], np.zeros(0, np.float32), 6, 9)
    one = W.from_coo([2], [3], np.array([1.5], np.float32), 6, 9)
    dense = W.from_coo([1] * 5000, list(range(5000)), np.full(5000, 0.5, np.float32), 4, 5000)
    dense2 = W.from_coo([1] * 2500, list(range(0, 5000, 2)), np.full(2500, 3.0, np.float32), 4, 5000)
    for ops in ([z, z], [one, z], [one, one, one], [dense, dense2], [dense, dense2, dense], [dense]):
        for P in (None, 3, 40):
            _check(ops, P)


@pytest.mark.parametrize("values", ["int", "uniform"])
def test_intersection_c2_scaled(values):
    """The C2 operands (B reuses 30 % of A's coordinates, C 30 % of A's or B's): one-row bitmap
    partitions and merge-path partitions."""
    wl = W.build("c2", 0.05, values=values, kmax=8)
    _check(wl.ops)
    _check(wl.ops[:2])


def test_intersection_subtiles():
    """Hypersparse operands whose partitions span more rows than a stage's row-pointer pool: the
    count-then-emit sub-tile path (and one pass of sub-tile sums for the inner product)."""
    rng = np.random.default_rng(11)
    M, Nc = 400_000, 1000
    rows = np.sort(rng.choice(M, 3000, replace=False))
    ops = []
    for o in range(3):
        keep = rows[rng.random(len(rows)) < 0.8]
        cols = rng.integers(0, 4, len(keep))
        ops.append(W.from_coo(keep, cols, rng.integers(1, 4, len(keep)).astype(np.float32), M, Nc))
    _check(ops, None)


def test_k5_rejected():
    rng = np.random.default_rng(1)
    ops = [A.to(DEV) for A in _ops(rng, 5, 50, 50, 0.1)]
    parts = N.partition(ops, N.auto_partitions(ops, "spadd"))
    with pytest.raises(N.NachoError):
        N.hadamard_k(ops, parts)
