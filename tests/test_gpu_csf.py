"""GPU parity of the third-order CSF path (nacho_partition_csf, nacho_csf_spadd_k)
against the CPU oracle (oracle_csf_partition_rank, oracle_csf_spadd_k): every boundary (x_i, x_j, x_k,
pos) and Z's five arrays bit-exact, values bit-exact (left fold in operand order on both sides)."""
import numpy as np
import pytest

import oracle as O
import workloads as W
from tests.conftest import gpu_available

pytestmark = pytest.mark.gpu

if gpu_available():
    import torch
    import paper_2604_17198_b200 as N
    DEV = torch.device("cuda:0")


def _dev(T):
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(DEV)
    return W.Tensor3(tuple(T.shape), t(T.crd0), t(T.pos1), t(T.crd1), t(T.pos2), t(T.crd2), t(T.val))


def _sparse_ops(rng, k, shape, nnz, share=0.5, dtype=np.float32, hot_slice=None):
    """k CSF operands with ~nnz entries each; operands 1.. reuse `share` of operand 0's coordinates so
    the union merges at every level; `hot_slice` adds a slice holding a large block of entries."""
    n0, n1, n2 = shape
    size = n0 * n1 * n2

    def draw(n):
        lin = np.unique(rng.integers(0, size, n))
        if hot_slice is not None:
            blk = hot_slice * n1 * n2 + rng.integers(0, n1 * n2, n // 4)
            lin = np.unique(np.concatenate([lin, blk]))
        return lin

    base = draw(nnz)
    ops = []
    for o in range(k):
        lin = base if o == 0 else np.unique(np.concatenate([rng.choice(base, int(len(base) * share), replace=False)
                                                            if len(base) else base, draw(nnz // 2)]))
        i, r = np.divmod(lin, n1 * n2)
        j, kk = np.divmod(r, n2)
        vals = rng.integers(-8, 9, len(lin)) * 0.25 if o % 2 else rng.uniform(-1, 1, len(lin))
        ops.append(W.csf_from_coo(i, j, kk, vals, shape, dtype))
    return ops


def _check(ops, P):
    d = [_dev(T) for T in ops]
    k = len(ops)
    parts = N.partition_csf(d, P)
    ref = O.csf_partition_rank(ops, P)
    assert np.array_equal(parts.query.cpu().numpy(), ref.query), "query"
    assert np.array_equal(parts.row.cpu().numpy(), ref.row), "x_i"
    assert np.array_equal(parts.row_pos.cpu().numpy(), ref.row_pos), "x_j"
    assert np.array_equal(parts.col.cpu().numpy(), ref.col), "x_k"
    assert np.array_equal(parts.pos.cpu().numpy().reshape(P + 1, k), ref.pos2()), "pos"
    z = N.csf_spadd_k(d, parts)
    r = O.csf_spadd_k(ops)
    for name, a, b in zip(("crd0", "pos1", "crd1", "pos2", "crd2"), z[:5], r[:5]):
        assert np.array_equal(a.cpu().numpy(), b), name
    assert np.array_equal(z[5].cpu().numpy().view(np.uint8), r[5].view(np.uint8)), "val bits"


def test_csf_fig_coordinate_tree(golden):
    g = golden("fig_coordinate_tree_csf.json")
    e = [np.asarray(g[n]) for n in ("A", "B")]
    A = W.csf_from_coo(e[0][:, 0], e[0][:, 1], e[0][:, 2], np.arange(1, 7), g["shape"])
    B = W.csf_from_coo(e[1][:, 0], e[1][:, 1], e[1][:, 2], np.arange(11, 18), g["shape"])
    for P in range(1, 16):
        _check([A, B], P)
    parts = N.partition_csf([_dev(A), _dev(B)], g["P"])
    assert [int(parts.row[1]), int(parts.row_pos[1]), int(parts.col[1])] == g["boundary_1"]["ijk"]


@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_csf_random_small(k):
    rng = np.random.default_rng(700 + k)
    for _ in range(8):
        shape = tuple(int(x) for x in rng.integers(1, 12, 3))
        ops = [W.random_csf(rng, shape, float(rng.uniform(0.02, 0.6))) for _ in range(k)]
        for P in (1, 2, 7, 64):
            _check(ops, P)


@pytest.mark.parametrize("k", [2, 3, 4])
def test_csf_random_tiles(k):
    """Several thousand partitions over ~10^5 entries per operand, one hot slice, ragged tails."""
    rng = np.random.default_rng(800 + k)
    ops = _sparse_ops(rng, k, (3000, 400, 2000), 120_000, hot_slice=17)
    for P in (1, 999, 4096):
        _check(ops, P)


def test_csf_fp64_and_one_slice():
    rng = np.random.default_rng(5)
    _check(_sparse_ops(rng, 3, (50, 60, 70), 20_000, dtype=np.float64), 333)
    # one slice: the CSR (two-level) case one level down
    _check(_sparse_ops(rng, 2, (1, 500, 800), 30_000), 257)


def test_csf_edge_cases():
    empty = W.csf_from_coo([], [], [], np.zeros(0, np.float32), (4, 5, 6))
    one = W.csf_from_coo([3], [4], [5], np.array([2.5], np.float32), (4, 5, 6))
    first = W.csf_from_coo([0], [0], [0], np.array([1.0], np.float32), (4, 5, 6))
    for ops in ([empty], [empty, empty], [one, empty], [empty, one, one], [first, one], [one, first, one, first]):
        for P in (1, 3, 10):
            _check(ops, P)


def test_csf_rejects():
    rng = np.random.default_rng(1)
    ops = [_dev(W.random_csf(rng, (4, 4, 4), 0.3)) for _ in range(5)]
    with pytest.raises(N.NachoError):
        N.partition_csf(ops, 4)
    bad = _dev(W.random_csf(rng, (4, 4, 5), 0.3))
    with pytest.raises(N.NachoError):
        N.partition_csf(ops[:1] + [bad], 4)
