"""The CUDA kernels run on a device slice of partitions (what each rank of paper_2604_17198_b200.dist
executes) and the per-slice results combine into the oracle's full result -- emulating D ranks on one
GPU (the driver gives one B200)."""
import numpy as np
import pytest
import torch

import oracle as O
import workloads as W
from tests.conftest import gpu_available
from tests.util import random_csr

pytestmark = pytest.mark.gpu

if gpu_available():
    import paper_2604_17198_b200 as N
    from paper_2604_17198_b200 import dist as D


@pytest.mark.parametrize("ndev", [2, 4, 8])
def test_spmv_device_slices(ndev):
    wl = W.build("c5", 2e-4, device="cuda")
    A = wl.ops[0]
    P = ndev * 16
    parts = N.partition([A], P)
    rp = parts.row_pos.cpu()
    pieces = []
    for d in range(ndev):
        lo, hi = D.rank_range(P, ndev, d)
        y = torch.zeros(A.nrows, dtype=A.val.dtype, device="cuda")
        N.spmv(A, wl.x, D.slice_parts(parts, lo, hi), y=y)
        own_lo, own_hi, seam = D.spmv_rank_rows(rp, lo, hi, A.nrows)
        pieces.append((y, own_lo, own_hi, seam))
    y = D.spmv_combine(pieces, A.nrows, A.val.dtype, "cuda").cpu().numpy()
    ref = O.spmv(A.numpy(), wl.x.cpu().numpy())
    assert np.allclose(y, ref, rtol=1e-5, atol=0)


@pytest.mark.parametrize("ndev", [2, 8])
@pytest.mark.parametrize("path", ["fused", "staged"])
def test_spadd_device_slices(ndev, path):
    wl = W.build("c2", 0.02, device="cuda", values="int", kmax=8)
    ops = wl.ops
    P = ndev * ((N.auto_partitions(ops, "spadd") + ndev - 1) // ndev)
    parts = N.partition(ops, P)
    pieces = []
    for d in range(ndev):
        lo, hi = D.rank_range(P, ndev, d)
        view = D.slice_parts(parts, lo, hi)
        off = torch.empty(view.P + 1, dtype=torch.int64, device="cuda")
        run = N.spadd_k_staged if path == "staged" else N.spadd_k_fused
        zp, zc, zv = run(ops, view, part_off=off)
        pieces.append((zp, zc, zv, int(off[-1].item()), int(parts.row[lo].item()), int(parts.row[hi].item())))
    zp, zc, zv = D.spadd_combine(pieces, ops[0].nrows, "cuda")
    rp, rc, rv = O.spadd_k([A.numpy() for A in ops])
    assert np.array_equal(zp.cpu().numpy(), rp)
    assert np.array_equal(zc.cpu().numpy(), rc)
    assert np.array_equal(zv.cpu().numpy(), rv)


@pytest.mark.parametrize("k", [1, 3])
def test_partition_slice_equals_full(k):
    """nacho_partition_slice writes exactly the boundaries nacho_partition writes at those indices."""
    wl = W.build("c2", 0.02, device="cuda", values="int", kmax=8)
    ops = wl.ops[:k]
    P = 8 * (N.auto_partitions(ops, "spadd") // 8 + 1)
    full = N.partition(ops, P)
    for lo, hi in ((0, P // 8), (3 * P // 8, P // 2), (7 * P // 8, P), (0, P)):
        sl = N.partition_slice(ops, P, lo, hi)
        for f in ("query", "row", "row_pos", "col"):
            assert torch.equal(getattr(sl, f), getattr(full, f)[lo:hi + 1]), f
        assert torch.equal(sl.pos, full.pos[lo * k:(hi + 1) * k])
