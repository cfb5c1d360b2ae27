"""Multi-rank host logic of paper_2604_17198_b200.dist on CPU: world_size 2 (and 3) over gloo.

The per-rank local results are emulated from the definition of what a rank's kernels produce for its
slice of partitions (owned rows exact on the slice, one seam carry; the union of the slice's coordinate
range); the exchange and assembly code under test is the one the NCCL path runs.  The assembled y / Z
must equal the oracle's full result (I9: device cuts are a subset of the fine cuts)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import workloads as W
from paper_2604_17198_b200 import dist as D
from tests.util import random_csr


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _emulated_spmv_local(A, x, parts, lo, hi):
    """What the kernels leave in a zeroed y for partitions [lo, hi) of a one-operand partition."""
    s, e = int(parts.pos[lo]), int(parts.pos[hi])
    own_lo, own_hi, seam = D.spmv_rank_rows(torch.from_numpy(parts.row_pos), lo, hi, A.nouter)
    y = np.zeros(A.nouter, dtype=np.float64)
    rows = list(range(own_lo, own_hi)) + ([seam] if seam >= 0 else [])
    for r in rows:
        a, b = max(int(A.pos[r]), s), min(int(A.pos[r + 1]), e)
        y[r] = sum(float(A.val[q]) * float(x[A.crd[q]]) for q in range(a, b))
    return torch.from_numpy(y), own_lo, own_hi, seam


def _emulated_spadd_local(ops, parts, lo, hi, z):
    """The union of the coordinate range [b_lo, b_hi) with local row pointers on the owned rows."""
    z_pos, z_crd, z_val = z
    M = ops[0].nrows
    rows = np.repeat(np.arange(M), np.diff(z_pos))
    keys = list(zip(rows.tolist(), z_crd.tolist()))
    b_lo = (int(parts.row[lo]), int(parts.col[lo]))
    b_hi = (int(parts.row[hi]), int(parts.col[hi]))
    sel = np.array([b_lo <= kk < b_hi for kk in keys], dtype=bool) if keys else np.zeros(0, bool)
    l_crd, l_val, l_rows = z_crd[sel], z_val[sel], rows[sel]
    own_lo, own_hi = int(parts.row[lo]), int(parts.row[hi])
    lp = np.zeros(M + 1, np.int64)
    for r in range(own_lo, own_hi):
        lp[r + 1] = int((l_rows <= r).sum())
    return (torch.from_numpy(lp), torch.from_numpy(l_crd.astype(np.int32)), torch.from_numpy(l_val),
            int(sel.sum()), own_lo, own_hi)


def _worker(rank, world, port, seed, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(seed)
        # ---- SpMV with a dense row that straddles the device cuts
        A = random_csr(rng, 40, 60, 0.15, dtype=np.float64, dense_rows=[17], empty_frac=0.3)
        x = rng.uniform(0.5, 1.5, 60)
        P_total = 4 * world
        parts = O.partition_rank([A], P_total)
        lo, hi = D.rank_range(P_total, world, rank)
        y_local, own_lo, own_hi, seam = _emulated_spmv_local(A, x, parts, lo, hi)
        y = D.spmv_assemble(y_local, own_lo, own_hi, seam, A.nouter).numpy()
        ref = O.spmv(A, x)
        ok_spmv = np.allclose(y, ref, rtol=1e-12, atol=1e-12)
        # ---- 3-way SpAdd: exact structure and values
        base = random_csr(rng, 30, 50, 0.2, dtype=np.float32)
        ops = [base] + [random_csr(rng, 30, 50, 0.1, dtype=np.float32, base=base, share=0.5) for _ in range(2)]
        parts3 = O.partition_rank(ops, P_total)
        z = O.spadd_k(ops)
        lp, lc, lv, nl, olo, ohi = _emulated_spadd_local(ops, parts3, lo, hi, z)
        zp, zc, zv = D.spadd_assemble(ops[0].nrows, lp, lc, lv, nl, olo, ohi)
        ok_spadd = (np.array_equal(zp.numpy(), z[0]) and np.array_equal(zc.numpy(), z[1])
                    and np.array_equal(zv.numpy(), z[2]))
        q.put((rank, bool(ok_spmv), bool(ok_spadd)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,seed", [(2, 1), (2, 2), (3, 3)])
def test_distributed_assembly_gloo(world, seed):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, seed, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(r[1] for r in res), f"SpMV assembly mismatch: {res}"
    assert all(r[2] for r in res), f"SpAdd assembly mismatch: {res}"


def test_device_cuts_are_fine_cuts():
    """I9: the device cuts of P = D are boundaries of P = D * P_l (floor(d*P_l*Q/(D*P_l)) = floor(d*Q/D))."""
    rng = np.random.default_rng(4)
    base = random_csr(rng, 50, 80, 0.2)
    ops = [base, random_csr(rng, 50, 80, 0.1, base=base, share=0.5)]
    for Dn, Pl in [(2, 3), (4, 5), (8, 2)]:
        coarse = O.partition_rank(ops, Dn)
        fine = O.partition_rank(ops, Dn * Pl)
        assert np.array_equal(coarse.pos2(), fine.pos2()[::Pl])
        assert np.array_equal(coarse.row, fine.row[::Pl]) and np.array_equal(coarse.col, fine.col[::Pl])


def test_slice_parts_views_share_storage():
    class P_:
        pass
    p = P_()
    p.k = 2
    p.query = torch.arange(9)
    p.row = torch.arange(9) * 10
    p.row_pos = torch.arange(9) * 10
    p.col = torch.arange(9, dtype=torch.int32)
    p.pos = torch.arange(18)
    v = D.slice_parts(p, 2, 6)
    assert v.P == 4 and v.row.tolist() == [20, 30, 40, 50, 60] and v.pos.tolist() == list(range(4, 14))
    assert D.rank_range(16, 4, 2) == (8, 12)
