"""GPU parity at the benchmark's own sizes and launch configurations (nnz >= 2^31).

C5 is the 4e9-nonzero CSR SpMV that bench.py times (auto P = 976,563 partitions, positions above
2^31, up to 4e9).  The oracle cannot sweep 4e9 entries in seconds, so the checks are
  * every boundary p = 0..P against the k = 1 closed form of SURVEY 8(c) C3 (pos = Q_p,
    row = upper_bound(pos, Q_p) - 1, col = crd[Q_p]; the end boundary (M, 0, nnz)), computed here
    from the host copy of `pos` -- the mathematics of Theorem 1 with one operand, not the kernel;
  * y on sampled rows: >= 1e4 random rows, the rows cut by a sample of boundaries (all of them
    above 2^31), the rows holding positions 2^31 - 1, 2^31 and 3 * 2^30, and the three heaviest (dense) rows --
    each against oracle_spmv run on the CSR slice of exactly those rows (rows are independent in
    y = A x), within 1e-5 of sum|a x| (north_star).
C2 (3 x 1e7 nnz) is small enough for the oracle in full: every SpAdd path bit-exact at auto P.
"""
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


def _rows_slice(A, rows):
    """CSR of the given rows of device matrix A (host numpy arrays), gathered on the device."""
    rows_t = torch.as_tensor(np.asarray(rows, np.int64), device=DEV)
    st, en = A.pos[rows_t], A.pos[rows_t + 1]
    ln = en - st
    tot = int(ln.sum().item())
    base = torch.repeat_interleave(st - torch.cumsum(ln, 0) + ln, ln, output_size=tot)
    idx = base + torch.arange(tot, device=DEV, dtype=torch.int64)
    pos = torch.zeros(len(rows) + 1, dtype=torch.int64, device=DEV)
    torch.cumsum(ln, 0, out=pos[1:])
    return W.SparseMatrix(W.CSR, len(rows), A.ncols, pos.cpu().numpy(), A.crd[idx].cpu().numpy(),
                          A.val[idx].cpu().numpy())


@pytest.fixture(scope="module")
def c5():
    wl = W.build("c5", 1.0, device="cuda")
    yield wl
    del wl
    torch.cuda.empty_cache()


def test_c5_fullscale_partition_closed_form(c5):
    A = c5.ops[0]
    nnz, M = A.nnz, A.nrows
    assert nnz > 2 ** 31 + 2 ** 30, nnz
    P = N.auto_partitions([A], "spmv")
    parts = N.partition([A], P)
    torch.cuda.synchronize()
    pos = A.pos.cpu().numpy()
    p = np.arange(P + 1, dtype=np.int64)
    Q = (p.astype(object) * nnz // P).astype(np.int64)            # exact floor(p Q* / P) (R4)
    q_in = Q[:P].copy()
    col = np.empty(P + 1, np.int64)
    col[:P] = A.crd[torch.as_tensor(q_in, device=DEV)].cpu().numpy()
    col[0] = 0                                                     # b_0 = origin (R1)
    col[P] = 0
    row = np.searchsorted(pos, Q, side="right") - 1
    row[0] = 0
    row[P] = M
    ppos = Q.copy()
    ppos[P] = nnz
    assert np.array_equal(parts.query.cpu().numpy(), Q), "query"
    assert np.array_equal(parts.pos.cpu().numpy(), ppos), "pos"
    assert np.array_equal(parts.row.cpu().numpy(), row), "row"
    assert np.array_equal(parts.row_pos.cpu().numpy(), row), "row_pos"
    assert np.array_equal(parts.col.cpu().numpy().astype(np.int64), col), "col"
    assert (Q > 2 ** 31).sum() > P // 3                             # int64 positions exercised


def test_c5_fullscale_spmv_sampled_rows(c5):
    A = c5.ops[0]
    nnz, M = A.nnz, A.nrows
    P = N.auto_partitions([A], "spmv")          # the launch configuration bench.py times
    parts = N.partition([A], P)
    y = N.spmv(A, c5.x, parts)
    torch.cuda.synchronize()
    pos = A.pos.cpu().numpy()
    deg = np.diff(pos)
    rng = np.random.default_rng(5)
    rows = set(rng.integers(0, M, 12000).tolist())
    brow = parts.row.cpu().numpy()[1:-1]
    bq = parts.pos.cpu().numpy()[1:-1]
    cut = brow[(bq > pos[brow]) & (bq > 2 ** 31)]                 # rows cut by a boundary above 2^31
    rows |= set(rng.choice(np.unique(cut), 4000, replace=False).tolist())
    cut_lo = brow[(bq > pos[brow]) & (bq < 2 ** 31)]
    rows |= set(rng.choice(np.unique(cut_lo), 1000, replace=False).tolist())
    for q in (2 ** 31 - 1, 2 ** 31, 3 * 2 ** 30, nnz - 1):
        r = int(np.searchsorted(pos, q, side="right") - 1)
        rows |= {r - 1, r, r + 1} & set(range(M))
    heavy = np.argsort(deg)[-3:]
    rows |= set(heavy.tolist())
    rows = np.array(sorted(rows), np.int64)
    assert deg[heavy].min() > 5 * 10 ** 7
    sub = _rows_slice(A, rows)
    x = c5.x.cpu().numpy()
    ref = O.spmv(sub, x)
    absA = W.SparseMatrix(W.CSR, sub.nrows, sub.ncols, sub.pos, sub.crd, np.abs(sub.val))
    scale = O.spmv(absA, np.abs(x)).astype(np.float64)
    got = y[torch.as_tensor(rows, device=DEV)].cpu().numpy().astype(np.float64)
    err = np.abs(got - ref.astype(np.float64))
    bad = err > 1e-5 * np.maximum(scale, 1e-300)
    assert not bad.any(), f"{bad.sum()} of {len(rows)} sampled rows off; max rel {(err / np.maximum(scale, 1e-300)).max()}"


def test_c2_fullscale_spadd_all_paths():
    """The bench workload (C2, auto P) through every single-read SpAdd path and the two-pass path:
    part_off, Z.pos, Z.crd and Z.val bit-exact against the oracle on the whole output."""
    wl = W.build("c2", 1.0, device="cuda")
    ops = wl.ops
    host = [A.numpy() for A in ops]
    rp, rc, rv = O.spadd_k(host)
    P = N.auto_partitions(ops, "spadd")
    parts = N.partition(ops, P)
    op = O.partition_rank(host, P)
    for f in ("query", "row", "row_pos", "col", "pos"):
        assert np.array_equal(getattr(parts, f).cpu().numpy(), getattr(op, f)), f
    off_ref = np.concatenate([[0], np.cumsum(O.spadd_counts(host, op))])
    for name, fn in (("fused", N.spadd_k_fused), ("staged", N.spadd_k_staged)):
        po = torch.full((P + 1,), -1, dtype=torch.int64, device=DEV)
        z_pos, z_crd, z_val = fn(ops, parts, part_off=po)
        n = int(z_pos[-1].item())
        assert n == len(rc), name
        assert np.array_equal(po.cpu().numpy(), off_ref), name + " part_off"
        assert np.array_equal(z_pos.cpu().numpy(), rp), name + " Z.pos"
        assert np.array_equal(z_crd[:n].cpu().numpy(), rc), name + " Z.crd"
        assert np.array_equal(z_val[:n].cpu().numpy().view(np.uint32), rv.view(np.uint32)), name + " Z.val"
    part_off = N.spadd_k_count(ops, parts)
    assert np.array_equal(part_off.cpu().numpy(), off_ref)
    z_pos, z_crd, z_val = N.spadd_k_fill(ops, parts, part_off, len(rc))
    assert np.array_equal(z_pos.cpu().numpy(), rp)
    assert np.array_equal(z_crd.cpu().numpy(), rc)
    assert np.array_equal(z_val.cpu().numpy().view(np.uint32), rv.view(np.uint32))


def test_esc_spgemm_bench_scale():
    """The ESC SpGEMM line of bench.py at its own size (C2's operands A B, ~1e8 products, auto P):
    W, every boundary and the whole of C bit-exact against the oracle."""
    wl = W.build("c2", 1.0, device="cuda")
    A, B = wl.ops[0], wl.ops[1]
    hA, hB = A.numpy(), B.numpy()
    Wd = N.spgemm_work(A, B)
    Wr = O.spgemm_work(hA, hB)
    assert np.array_equal(Wd.cpu().numpy(), Wr)
    qstar = int(Wr[-1])
    P = N.esc_auto_partitions(qstar)
    parts = N.partition_esc(A, B, Wd, qstar, P)
    ref = O.esc_partition(hA, hB, P)
    for f in ("query", "row", "col", "pos"):
        assert np.array_equal(getattr(parts, f).cpu().numpy(), getattr(ref, f)), f
    c_pos, c_crd, c_val, nnz_c = N.spgemm_esc(A, B, Wd, parts, qstar)
    n = int(nnz_c.item())
    r_pos, r_crd, r_val = O.spgemm(hA, hB)
    assert n == len(r_crd)
    assert np.array_equal(c_pos.cpu().numpy(), r_pos)
    assert np.array_equal(c_crd[:n].cpu().numpy(), r_crd)
    assert np.array_equal(c_val[:n].cpu().numpy(), r_val)


def test_esc_sssmm_bench_scale():
    """The ESC SSSMM line of bench.py at its own size (Z = C (.) (A B) on C2's operands, ~1e8 products
    expanded, the sampled ones kept): Z bit-exact against the oracle."""
    wl = W.build("c2", 1.0, device="cuda")
    A, B, S = wl.ops
    z_pos, z_crd, z_val = N.sssmm(S, A, B)
    r_pos, r_crd, r_val = O.sssmm(S.numpy(), A.numpy(), B.numpy())
    assert np.array_equal(z_pos.cpu().numpy(), r_pos)
    assert np.array_equal(z_crd.cpu().numpy(), r_crd)
    assert np.array_equal(z_val.cpu().numpy(), r_val)
