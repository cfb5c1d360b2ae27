"""Multi-GPU path on one B200 (the driver gives one GPU): the real sharding kernels
(nacho_device_cuts, nacho_shard_rows), the shard generator, the local kernels on each device's shard
and the seam fix-up (nacho_dist_seam) for D emulated devices, compared with the CPU oracle; the NCCL
calls (nacho_dist_spmv, nacho_dist_spadd_gather, nacho_dist_broadcast) at world size 1; and a
2-process run on the one GPU whose exchange goes through torch.distributed (gloo) instead of NCCL
(NCCL refuses two ranks on one device)."""
import os
import socket

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


def _cuts_match_oracle(A_host, cuts, ndev):
    p = O.partition_rank([A_host], ndev)
    ref = [[int(p.row_pos[d]), int(p.pos[d])] for d in range(ndev + 1)]
    assert cuts == ref, "device cuts differ from Alg. 1 (oracle) with P = D"


def _emulate_spmv(A_full, x, ndev, crd_vals=None):
    """Every device's shard through the real kernels; carries all-gathered by stacking."""
    cuts = N.device_cuts(A_full, ndev).cpu().tolist()
    plans = D.shard_plans(cuts, A_full.nrows)
    ys, carries = [], []
    for p in plans:
        if crd_vals is None:
            crd, val = A_full.crd[p.pos_lo:p.pos_hi].clone(), A_full.val[p.pos_lo:p.pos_hi].clone()
        else:
            crd, val = crd_vals(p)
        A_loc = D.build_shard(p, A_full.pos, crd, val, A_full.ncols)
        y = torch.zeros(max(p.nloc, 1), dtype=A_full.val.dtype, device="cuda")
        if p.nloc > 0:
            N.spmv(A_loc, x, N.partition([A_loc], N.auto_partitions([A_loc], "spmv")), y=y[:p.nloc])
        r, b = D.carry_of(p, y)
        carries.append(torch.cat([r, b]))
        ys.append(y)
    allc = torch.stack(carries).contiguous()
    for p, y in zip(plans, ys):
        if p.nloc > 0:
            N.dist_seam(allc, ndev, p.d, p.row_lo, p.own > 0, y)
    return cuts, D.spmv_combine(list(zip(ys, plans)), A_full.nrows, A_full.val.dtype, "cuda")


@pytest.mark.parametrize("ndev", [2, 4, 8])
def test_spmv_device_shards(ndev):
    wl = W.build("c5", 2e-4, device="cuda")
    A = wl.ops[0]
    cuts, y = _emulate_spmv(A, wl.x, ndev)
    Ah = A.numpy()
    _cuts_match_oracle(Ah, cuts, ndev)
    ref = O.spmv(Ah, wl.x.cpu().numpy())
    assert np.allclose(y.cpu().numpy(), ref, rtol=1e-5, atol=0)


@pytest.mark.parametrize("dtype,tol", [(np.float32, 1e-5), (np.float64, 1e-12)])
def test_spmv_dense_row_spanning_devices(dtype, tol):
    """A dense row longer than several device shares: chained seam carries, devices owning no row."""
    rng = np.random.default_rng(5)
    Ah = random_csr(rng, 50, 3000, 0.002, dtype=dtype, dense_rows=[7, 31], empty_frac=0.2)
    A = Ah.to("cuda")
    x = torch.from_numpy(rng.uniform(0.5, 1.5, 3000).astype(dtype)).cuda()
    cuts, y = _emulate_spmv(A, x, 8)
    _cuts_match_oracle(Ah, cuts, 8)
    plans = D.shard_plans(cuts, A.nrows)
    assert any(p.own == 0 for p in plans)
    ref = O.spmv(Ah, x.cpu().numpy())
    scale = np.abs(W.to_dense(Ah)) @ np.abs(x.cpu().numpy())
    assert (np.abs(y.cpu().numpy() - ref) <= tol * np.maximum(scale, 1e-300)).all()


def test_shard_generator_matches_full_build():
    """workloads.shard_entries (a device generates only its slice) is bit-identical to the slice of
    the full matrix, and the shards built from it give the oracle's y."""
    wl = W.build("c5", 2e-4, device="cuda")
    A = wl.ops[0]
    ndev = 4

    def gen(p):
        return W.shard_entries("c5", A.pos, p.pos_lo, p.pos_hi, 2e-4)
    cuts = N.device_cuts(A, ndev).cpu().tolist()
    for p in D.shard_plans(cuts, A.nrows):
        c, v = gen(p)
        assert torch.equal(c, A.crd[p.pos_lo:p.pos_hi]) and torch.equal(v, A.val[p.pos_lo:p.pos_hi])
    _, y = _emulate_spmv(A, wl.x, ndev, crd_vals=gen)
    ref = O.spmv(A.numpy(), wl.x.cpu().numpy())
    assert np.allclose(y.cpu().numpy(), ref, rtol=1e-5, atol=0)


@pytest.mark.parametrize("ndev", [2, 8])
def test_spadd_device_shards(ndev):
    wl = W.build("c2", 0.02, device="cuda", values="int", kmax=8)
    ops = wl.ops
    dparts = N.partition(ops, ndev)   # device cuts: Alg. 1 with P = D
    pieces = []
    for d in range(ndev):
        sh, row_lo, own = D.spadd_shard_ops(ops, dparts, d)
        P = N.auto_partitions(sh, "spadd")
        off = torch.empty(P + 1, dtype=torch.int64, device="cuda")
        zp, zc, zv = N.spadd_k_fused(sh, N.partition(sh, P), part_off=off)
        pieces.append((zp, zc, zv, int(off[-1].item()), row_lo, own))
    zp, zc, zv = D.spadd_combine(pieces, ops[0].nrows, "cuda")
    rp, rc, rv = O.spadd_k([A.numpy() for A in ops])
    assert np.array_equal(zp.cpu().numpy(), rp)
    assert np.array_equal(zc.cpu().numpy(), rc)
    assert np.array_equal(zv.cpu().numpy(), rv)


def _dist1():
    return N.Dist(1, 0, N.Dist.unique_id())


def test_nccl_world1_spmv_and_broadcast():
    """nacho_dist_init / _broadcast / _spmv / _destroy through real NCCL (one rank)."""
    comm = _dist1()
    try:
        wl = W.build("c5", 2e-4, device="cuda")
        A = wl.ops[0]
        x = wl.x.clone()
        comm.broadcast(x, 0)
        assert torch.equal(x, wl.x)
        cuts = N.device_cuts(A, 1).cpu().tolist()
        plans = D.shard_plans(cuts, A.nrows)
        A_loc = D.build_shard(plans[0], A.pos, A.crd.clone(), A.val.clone(), A.ncols)
        y_loc = torch.empty(plans[0].nloc, dtype=A.val.dtype, device="cuda")
        y_full = torch.full((A.nrows,), float("nan"), dtype=A.val.dtype, device="cuda")
        comm.spmv(A_loc, None, x, y_loc, D.cut_rows(plans, A.nrows), y_full=y_full)
        ref = O.spmv(A.numpy(), wl.x.cpu().numpy())
        assert np.allclose(y_full.cpu().numpy(), ref, rtol=1e-5, atol=0)
        assert torch.equal(y_full, y_loc)
    finally:
        comm.close()


def test_nccl_world1_spadd_gather():
    comm = _dist1()
    try:
        wl = W.build("c2", 0.02, device="cuda", values="int", kmax=8)
        ops = wl.ops
        P = N.auto_partitions(ops, "spadd")
        off = torch.empty(P + 1, dtype=torch.int64, device="cuda")
        zp, zc, zv = N.spadd_k_fused(ops, N.partition(ops, P), part_off=off)
        M = ops[0].nrows
        cap = sum(A.nnz for A in ops)
        z_pos = torch.full((M + 1,), -1, dtype=torch.int64, device="cuda")
        z_crd = torch.empty(cap, dtype=torch.int32, device="cuda")
        z_val = torch.empty(cap, dtype=zv.dtype, device="cuda")
        n = comm.spadd_gather(zp, zc, zv, off[-1:], [0, M], z_pos, z_crd, z_val)
        rp, rc, rv = O.spadd_k([A.numpy() for A in ops])
        assert n == len(rc)
        assert np.array_equal(z_pos.cpu().numpy(), rp)
        assert np.array_equal(z_crd[:n].cpu().numpy(), rc) and np.array_equal(z_val[:n].cpu().numpy(), rv)
    finally:
        comm.close()


# ------------------------------------------------------------------ two processes on the one GPU
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _mp_worker(rank, world, port, q):
    import torch.distributed as td
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    td.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2604_17198_b200 as N_
        from paper_2604_17198_b200 import dist as D_
        torch.cuda.set_device(0)
        scale = 2e-4
        # the rank's real setup: full row pointers, device cuts, only its own entries generated
        A_loc, plans, cuts = D_.spmv_setup("c5", scale, world, rank)
        p = plans[rank]
        x = W.dense_x("c5", scale) if rank == 0 else torch.empty(W.scaled(W.CONFIGS["c5"], scale)["m"],
                                                                dtype=torch.float32, device="cuda")
        xc = x.cpu()
        td.broadcast(xc, src=0)   # x replicated (gloo here; nacho_dist_broadcast over NCCL in the product)
        x = xc.cuda()
        y = torch.zeros(max(p.nloc, 1), dtype=torch.float32, device="cuda")
        if p.nloc > 0:
            N_.spmv(A_loc, x, N_.partition([A_loc], N_.auto_partitions([A_loc], "spmv")), y=y[:p.nloc])
        r, b = D_.carry_of(p, y)
        mine = torch.cat([r, b]).cpu()
        allc = [torch.empty_like(mine) for _ in range(world)]
        td.all_gather(allc, mine)
        if p.nloc > 0:
            N_.dist_seam(torch.stack(allc).cuda().contiguous(), world, rank, p.row_lo, p.own > 0, y)
        segs = [None] * world
        td.all_gather_object(segs, (p.row_lo, y[:p.own].cpu().numpy()))
        q.put((rank, segs if rank == 0 else None))
    except Exception as e:   # report instead of leaving the parent waiting
        q.put((rank, ("error", repr(e))))
        raise
    finally:
        td.destroy_process_group()


def test_two_processes_one_gpu_spmv():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_mp_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=120)
    for r in res.values():
        assert not (isinstance(r, tuple) and r and r[0] == "error"), r
    wl = W.build("c5", 2e-4)
    A = wl.ops[0]
    y = np.zeros(A.nrows, np.float32)
    for lo, seg in res[0]:
        y[lo:lo + len(seg)] = seg
    ref = O.spmv(A, wl.x)
    assert np.allclose(y, ref, rtol=1e-5, atol=0)
