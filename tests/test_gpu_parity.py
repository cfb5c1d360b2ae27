"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on identical seeded inputs.

Bit-exact: partition boundaries, SpAdd structure (Z.pos, Z.crd), SpAdd values (left fold), per-partition
offsets; SpMV/SpMM within 1e-5 (fp32) / 1e-12 (fp64) of sum|a*x| (BASELINE north_star).
"""
import numpy as np
import pytest

import oracle as O
import workloads as W
from tests.conftest import gpu_available
from tests.util import random_csr, random_dcsr

pytestmark = pytest.mark.gpu

if gpu_available():
    import torch
    import paper_2604_17198_b200 as N
    DEV = torch.device("cuda:0")


def _dev(A):
    return A.to(DEV)


def _parts_equal(gp, op):
    assert np.array_equal(gp.query.cpu().numpy(), op.query), "query"
    assert np.array_equal(gp.pos.cpu().numpy(), op.pos), "pos"
    assert np.array_equal(gp.row.cpu().numpy(), op.row), "row"
    assert np.array_equal(gp.row_pos.cpu().numpy(), op.row_pos), "row_pos"
    assert np.array_equal(gp.col.cpu().numpy(), op.col), "col"


def _random_ops(rng, k, M, N, dens, dense_rows=(), empty_frac=0.3):
    base = random_csr(rng, M, N, dens, dense_rows=dense_rows, empty_frac=empty_frac)
    return [base] + [random_csr(rng, M, N, dens * 0.6, base=base, share=0.5, empty_frac=empty_frac)
                     for _ in range(k - 1)]


# ---------------------------------------------------------------- partition
@pytest.mark.parametrize("k", [1, 2, 3, 4, 8])
def test_partition_random_bit_exact(k):
    rng = np.random.default_rng(100 + k)
    for trial in range(12):
        M, Nc = int(rng.integers(1, 300)), int(rng.integers(1, 3000))
        ops = _random_ops(rng, k, M, Nc, float(rng.uniform(0.001, 0.05)),
                          dense_rows=[int(rng.integers(M))] if trial % 3 == 0 else ())
        qstar = sum(A.nnz for A in ops)
        for P in (1, 2, 7, 8, 64, max(1, qstar + 5)):
            gp = N.partition([_dev(A) for A in ops], P)
            _parts_equal(gp, O.partition_rank(ops, P))


def test_partition_dcsr_bit_exact():
    rng = np.random.default_rng(7)
    for _ in range(10):
        A = random_dcsr(rng, int(rng.integers(10, 100000)), int(rng.integers(1, 500)), int(rng.integers(1, 300)), 0.05)
        for P in (1, 3, 64, A.nnz + 2):
            _parts_equal(N.partition([_dev(A)], P), O.partition_rank([A], P))


@pytest.mark.parametrize("name,scale,P", [("c1", 1.0, 8), ("c2", 0.05, 4096), ("c2", 0.05, 131072),
                                          ("c3", 0.01, 1000), ("c5", 2e-4, 777)])
def test_partition_configs(name, scale, P):
    wl = W.build(name, scale, device="cuda")
    gp = N.partition(wl.ops, P)
    _parts_equal(gp, O.partition_rank([A.numpy() for A in wl.ops], P))


def test_partition_long_row_segments():
    """One row whose segments total >= 2^26 entries: the k-way select's 64-bit window path (the
    32-bit path serves shorter segments); boundaries bit-exact against the oracle."""
    rng = np.random.default_rng(2026)
    n = 3 << 23                                        # 3 * 2^23 per operand, 3 operands: 1.125 * 2^26
    ops = []
    for o in range(3):
        crd = np.cumsum(rng.integers(1, 40, n)).astype(np.int64)
        pos = np.array([0, 0, n, n], np.int64)         # rows 0 and 2 empty, row 1 holds everything
        ops.append(W.SparseMatrix(W.CSR, 3, 40 * n, pos, crd.astype(np.int32), np.ones(n, np.float32)))
    for P in (1, 5, 64):
        _parts_equal(N.partition([_dev(A) for A in ops], P), O.partition_rank(ops, P))


def test_partition_many_rows():
    """More than 2^26 rows: the outer search's 64-bit index path (32-bit below 2^26 rows), k = 1 and
    k = 2, boundaries bit-exact against the oracle."""
    rng = np.random.default_rng(2027)
    M, Nc = (1 << 26) + 1000, 5000
    ops = []
    for o in range(2):
        rows = np.sort(rng.choice(M, size=6000, replace=False))
        rows[-1] = M - 1                                  # reach the last rows
        cnt = np.zeros(M + 1, np.int64)
        per = rng.integers(1, 4, len(rows))
        cnt[rows + 1] = per
        pos = np.cumsum(cnt)
        crd = np.concatenate([np.sort(rng.choice(Nc, size=c, replace=False)) for c in per]).astype(np.int32)
        ops.append(W.SparseMatrix(W.CSR, M, Nc, pos, crd, np.ones(len(crd), np.float32)))
    for k in (1, 2):
        for P in (1, 7, 300):
            _parts_equal(N.partition([_dev(A) for A in ops[:k]], P), O.partition_rank(ops[:k], P))
    # SpMV over the same rows: few partitions, so chunks search their rows (64-bit outer indices)
    A = ops[0]
    x = rng.uniform(-1, 1, Nc).astype(np.float32)
    dA = _dev(A)
    for P in (1, 3):
        y = N.spmv(dA, torch.from_numpy(x).to(DEV), N.partition([dA], P)).cpu().numpy()
        _spmv_check(A, x, y, 1e-5)


def test_device_generator_matches_numpy_recipe():
    for name, scale in [("c1", 1.0), ("c2", 0.01), ("c3", 0.002), ("c4", 1e-4), ("c5", 2e-5)]:
        d = W.build(name, scale, device="cuda")
        h = W.build(name, scale)
        for A, B in zip(d.ops, h.ops):
            A = A.numpy()
            for f in ("pos", "crd", "val", "outer_crd"):
                a, b = getattr(A, f), getattr(B, f)
                assert (a is None and b is None) or np.array_equal(a, b), (name, f)
        if h.x is not None:
            assert np.array_equal(d.x.cpu().numpy(), h.x)


# ---------------------------------------------------------------- SpMV
def _spmv_check(A, x, y, tol):
    ref = O.spmv(A, x)
    scale = np.abs(O.spmv(W.SparseMatrix(A.format, A.nrows, A.ncols, A.pos, A.crd, np.abs(A.val), A.outer_crd),
                          np.abs(x))).astype(np.float64)
    err = np.abs(y.astype(np.float64) - ref.astype(np.float64))
    bad = err > tol * np.maximum(scale, 1e-300)
    assert not bad.any(), f"{bad.sum()} rows off; max err {err.max()}"


@pytest.mark.parametrize("dtype,tol", [(np.float32, 1e-5), (np.float64, 1e-12)])
def test_spmv_random(dtype, tol):
    rng = np.random.default_rng(11)
    for trial in range(15):
        M, Nc = int(rng.integers(1, 5000)), int(rng.integers(1, 3000))
        A = random_csr(rng, M, Nc, float(rng.uniform(0.0005, 0.01)), dtype=dtype,
                       dense_rows=[int(rng.integers(M))] if trial % 2 == 0 else (), empty_frac=0.4)
        x = rng.uniform(0.5, 1.5, Nc).astype(dtype)
        Ad, xd = _dev(A), torch.from_numpy(x).to(DEV)
        for P in (None, 1, 3, 64, A.nnz + 5):
            parts = N.partition([Ad], P) if P else None
            y = N.spmv(Ad, xd, parts).cpu().numpy()
            _spmv_check(A, x, y, tol)


def test_spmv_integer_exact_any_P():
    rng = np.random.default_rng(12)
    A = random_csr(rng, 3000, 2000, 0.01, dtype=np.float64, ints=True, dense_rows=[5, 6])
    x = rng.integers(-4, 5, 2000).astype(np.float64)
    ref = O.spmv(A, x)
    Ad, xd = _dev(A), torch.from_numpy(x).to(DEV)
    for P in (None, 1, 2, 17, 1000):
        y = N.spmv(Ad, xd, N.partition([Ad], P) if P else None).cpu().numpy()
        assert np.array_equal(y, ref)


@pytest.mark.parametrize("dense_y", [False, True])
def test_spmv_dcsr(dense_y):
    rng = np.random.default_rng(13)
    for _ in range(6):
        A = random_dcsr(rng, int(rng.integers(100, 100000)), 400, int(rng.integers(1, 500)), 0.05)
        x = rng.uniform(0.5, 1.5, 400).astype(np.float32)
        Ad, xd = _dev(A), torch.from_numpy(x).to(DEV)
        for P in (None, 1, 9):
            y = N.spmv(Ad, xd, N.partition([Ad], P) if P else None, dense_y=dense_y).cpu().numpy()
            yc = y[A.outer_crd] if dense_y else y
            _spmv_check(A, x, yc, 1e-5)
            if dense_y:
                mask = np.ones(A.nrows, bool)
                mask[A.outer_crd] = False
                assert (y[mask] == 0).all()


def test_spmv_edge_cases():
    # empty matrix, all rows empty but one, single dense row straddling many partitions, N = 1
    cases = [W.from_coo([], [], [], 10, 7), W.from_coo([4] * 3, [0, 2, 5], [1.0, 2.0, 3.0], 9, 6),
             W.from_coo([3] * 5000, list(range(5000)), np.ones(5000), 7, 5000),
             W.from_coo(list(range(50)), [0] * 50, np.ones(50), 60, 1)]
    for A in cases:
        A.val = A.val.astype(np.float32)
        x = np.linspace(0.5, 1.5, A.ncols).astype(np.float32)
        Ad, xd = _dev(A), torch.from_numpy(x).to(DEV)
        for P in (None, 1, 3, 100, 4099):
            y = N.spmv(Ad, xd, N.partition([Ad], P) if P else None).cpu().numpy()
            _spmv_check(A, x, y, 1e-5)


@pytest.mark.parametrize("name,scale", [("c1", 1.0), ("c3", 0.02), ("c5", 1e-3)])
def test_spmv_configs(name, scale):
    wl = W.build(name, scale, device="cuda")
    A = wl.ops[0]
    parts = N.partition([A], wl.P) if wl.P else None
    y = N.spmv(A, wl.x, parts).cpu().numpy()
    _spmv_check(A.numpy(), wl.x.cpu().numpy(), y, 1e-12 if y.dtype == np.float64 else 1e-5)


# ---------------------------------------------------------------- SpAdd
def _spadd_check(ops, P=None):
    dops = [_dev(A) for A in ops]
    parts = N.partition(dops, P or N.auto_partitions(dops, "spadd"))
    part_off = N.spadd_k_count(dops, parts)
    op = O.partition_rank(ops, parts.P)
    cnt = O.spadd_counts(ops, op)
    assert np.array_equal(part_off.cpu().numpy(), np.concatenate([[0], np.cumsum(cnt)])), "part_off"
    nnz_z = int(part_off[-1].item())
    z_pos, z_crd, z_val = N.spadd_k_fill(dops, parts, part_off, nnz_z)
    rp, rc, rv = O.spadd_k(ops)
    assert np.array_equal(z_pos.cpu().numpy(), rp), "Z.pos"
    assert np.array_equal(z_crd.cpu().numpy(), rc), "Z.crd"
    assert np.array_equal(z_val.cpu().numpy().view(np.uint8), rv.view(np.uint8)), "Z.val bits"
    # staged single-read variant: any P (partitions larger than a tile run as Alg.-1-cut chunks)
    so = torch.full((parts.P + 1,), -1, dtype=torch.int64, device=DEV)
    sz_pos, sz_crd, sz_val = N.spadd_k_staged(dops, parts, part_off=so)
    n = int(sz_pos[-1].item())
    assert n == len(rc)
    assert np.array_equal(so.cpu().numpy(), np.concatenate([[0], np.cumsum(cnt)])), "staged part_off"
    assert np.array_equal(sz_pos.cpu().numpy(), rp), "staged Z.pos"
    assert np.array_equal(sz_crd[:n].cpu().numpy(), rc), "staged Z.crd"
    assert np.array_equal(sz_val[:n].cpu().numpy().view(np.uint8), rv.view(np.uint8)), "staged Z.val bits"
    # single-pass (look-back) variant, when the partitions fit its tile
    qstar = sum(A.nnz for A in ops)
    if -(-qstar // parts.P) + len(ops) - 1 <= N.lib.nacho_spadd_tile(len(ops)):
        po = torch.full((parts.P + 1,), -1, dtype=torch.int64, device=DEV)
        fz_pos, fz_crd, fz_val = N.spadd_k_fused(dops, parts, part_off=po)
        n = int(fz_pos[-1].item())
        assert n == len(rc)
        assert np.array_equal(po.cpu().numpy(), np.concatenate([[0], np.cumsum(cnt)])), "fused part_off"
        assert np.array_equal(fz_pos.cpu().numpy(), rp), "fused Z.pos"
        assert np.array_equal(fz_crd[:n].cpu().numpy(), rc), "fused Z.crd"
        assert np.array_equal(fz_val[:n].cpu().numpy().view(np.uint8), rv.view(np.uint8)), "fused Z.val bits"



@pytest.mark.parametrize("k", [1, 2, 3, 4, 8])
def test_spadd_random(k):
    rng = np.random.default_rng(200 + k)
    for trial in range(8):
        M, Nc = int(rng.integers(1, 2000)), int(rng.integers(1, 5000))
        ops = _random_ops(rng, k, M, Nc, float(rng.uniform(0.0005, 0.01)),
                          dense_rows=[int(rng.integers(M))] if trial % 2 == 0 else ())
        for P in (None, 1, 5, 300):
            _spadd_check(ops, P)


def test_spadd_edge_cases():
    z = W.from_coo([], [], [], 5, 5)
    one = W.from_coo([2], [3], [1.5], 5, 5)
    dense = W.from_coo([1] * 6000, list(range(6000)), np.full(6000, 0.25), 4, 6000)
    one_w = W.from_coo([1, 3], [17, 5999], [1.5, -2.0], 4, 6000)
    for ops in ([z, z], [z, one, z], [one, one, one], [dense, dense, one_w], [one_w, dense], [dense]):
        for P in (None, 1, 2, 8, 20000):
            _spadd_check([W.SparseMatrix(A.format, A.nrows, A.ncols, A.pos, A.crd, A.val.astype(np.float32))
                          for A in ops], P)


def test_spadd_fp64():
    """fp64 values through every SpAdd path (count / fill, fused, staged; bitmap and merge-path
    partitions): bit-exact left folds against the oracle."""
    rng = np.random.default_rng(91)
    for k in (2, 3, 5):
        ops32 = _random_ops(rng, k, 700, 3000, 0.004, dense_rows=[11, 500])
        ops = [W.SparseMatrix(A.format, A.nrows, A.ncols, A.pos, A.crd,
                              rng.uniform(-2, 2, A.nnz).astype(np.float64)) for A in ops32]
        for P in (None, 4, 97):
            _spadd_check(ops, P)


def test_spadd_wide_keys():
    """Hypersparse operands whose partitions span more rows than 32-bit (row, column) keys can hold
    next to a wide column range: the 64-bit key path (index-only merge buffers) of spadd4."""
    rng = np.random.default_rng(77)
    M, Nc = 3_000_000, 2_000_000
    ops = []
    base_rows = np.sort(rng.choice(M, size=4000, replace=False))
    for o in range(3):
        keep = base_rows[rng.random(len(base_rows)) < 0.7]
        extra = np.sort(rng.choice(M, size=1500, replace=False))
        rows = np.concatenate([np.repeat(keep, 2), extra])
        cols = np.concatenate([np.stack([rng.integers(0, Nc // 2, len(keep)),
                                         rng.integers(Nc // 2, Nc, len(keep))], 1).ravel(),
                               rng.integers(0, Nc, len(extra))])
        key = np.unique(rows.astype(np.int64) * Nc + cols)
        r, c = key // Nc, key % Nc
        vals = rng.integers(-4, 5, len(r)).astype(np.float32)
        ops.append(W.from_coo(r, c, vals, M, Nc))
    for P in (None, 3, 40):
        _spadd_check(ops, P)


@pytest.mark.parametrize("values", ["int", "uniform"])
def test_spadd_c2_scaled(values):
    wl = W.build("c2", 0.05, values=values, kmax=8)
    _spadd_check(wl.ops)
    _spadd_check(wl.ops, 131)


# ---------------------------------------------------------------- SpMM
@pytest.mark.parametrize("nb,dtype", [(64, np.float32), (1, np.float32), (40, np.float32), (128, np.float32),
                                      (256, np.float32), (64, np.float64)])
def test_spmm_random(nb, dtype):
    rng = np.random.default_rng(300 + nb)
    A = random_csr(rng, 1500, 800, 0.01, dtype=dtype, dense_rows=[7], empty_frac=0.4)
    B = rng.uniform(0.5, 1.5, (800, nb)).astype(dtype)
    ref = O.spmm(A, B)
    absA = W.SparseMatrix("csr", A.nrows, A.ncols, A.pos, A.crd, np.abs(A.val))
    scale = O.spmm(absA, np.abs(B)).astype(np.float64)
    Ad, Bd = _dev(A), torch.from_numpy(B).to(DEV)
    tol = 1e-5 if dtype == np.float32 else 1e-12
    for P in (None, 1, 7, 2000):
        C = N.spmm(Ad, Bd, N.partition([Ad], P) if P else None).cpu().numpy()
        err = np.abs(C.astype(np.float64) - ref)
        assert (err <= tol * np.maximum(scale, 1e-300)).all(), f"P={P} max err {err.max()}"


def test_spmm_c4_scaled():
    wl = W.build("c4", 2e-4, device="cuda")
    A = wl.ops[0]
    C = N.spmm(A, wl.x).cpu().numpy()
    Ah, Bh = A.numpy(), wl.x.cpu().numpy()
    ref = O.spmm(Ah, Bh)
    assert np.allclose(C, ref, rtol=1e-5, atol=0)


# ---------------------------------------------------------------- ABI errors
def test_abi_errors_raise():
    A = _dev(W.from_coo([0], [0], np.ones(1, np.float32), 2, 2))
    with pytest.raises(N.NachoError):
        N.partition([A], 0)
    with pytest.raises(N.NachoError):
        N.partition([A] * 9, 4)
    B = _dev(W.from_coo([0], [0], np.ones(1, np.float32), 3, 2))
    with pytest.raises(N.NachoError):
        N.partition([A, B], 4)
    bad = _dev(W.SparseMatrix("csr", 2, 2, np.array([0, 2, 2], np.int64), np.array([1, 0], np.int32),
                              np.ones(2, np.float32)))
    with pytest.raises(N.NachoError):
        N.validate(bad)
    N.validate(A)
