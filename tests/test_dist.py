"""Multi-GPU host logic on CPU: the shard plan the device cuts give, and the NCCL
unique-id handoff of nacho_dist_init over a world-size-2 gloo group.

The device cuts are Alg. 1 with P = D; the plan must tile the rows exactly once (R7
ownership), hold every position exactly once, and leave one seam row per device whose row continues
on the next one (a dense row may span several devices).  The cuts are taken from the ORACLE here
(partition_rank with P = D), so the plan logic is checked against the paper's definition; the GPU
tests check nacho_device_cuts against the same oracle and run the kernels on the shards."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2604_17198_b200 import dist as D
from tests.util import random_csr


def _oracle_cuts(A, ndev):
    p = O.partition_rank([A], ndev)
    return [(int(p.row_pos[d]), int(p.pos[d])) for d in range(ndev + 1)]


def _check_plans(A, ndev):
    plans = D.shard_plans(_oracle_cuts(A, ndev), A.nrows)
    M = A.nrows
    owned = np.zeros(M, np.int64)
    held = 0
    for p in plans:
        owned[p.row_lo:p.row_lo + p.own] += 1
        held += p.pos_hi - p.pos_lo
        assert p.pos_lo <= p.pos_hi
        # every held position lies in the held rows
        if p.pos_hi > p.pos_lo:
            r_first = int(np.searchsorted(A.pos, p.pos_lo, side="right") - 1)
            r_last = int(np.searchsorted(A.pos, p.pos_hi - 1, side="right") - 1)
            assert p.row_lo <= r_first and r_last < p.row_lo + max(p.nloc, 1)
        # the seam row is the row the next device starts in
        if p.has_carry:
            assert p.row_lo + p.nloc - 1 == plans[p.d + 1].row_lo
    assert (owned == 1).all(), "rows owned exactly once (R7)"
    assert held == A.nnz, "positions held exactly once"
    # work balance (Theorem 1 with Delta = 1 for one operand): floor / ceil of nnz / D
    w = [p.pos_hi - p.pos_lo for p in plans]
    assert max(w) - min(w) <= 1
    return plans


@pytest.mark.parametrize("ndev", [1, 2, 3, 8])
def test_shard_plans_tile_rows_and_positions(ndev):
    rng = np.random.default_rng(10 + ndev)
    for trial in range(6):
        M, N = int(rng.integers(5, 80)), int(rng.integers(5, 90))
        A = random_csr(rng, M, N, float(rng.uniform(0.02, 0.3)), dense_rows=[int(rng.integers(M))] if trial % 2 else ())
        _check_plans(A, ndev)


def test_dense_row_spans_devices():
    """A dense row longer than a device share: the devices inside it own no rows and pass carries on."""
    rng = np.random.default_rng(3)
    A = random_csr(rng, 12, 400, 0.01, dense_rows=[5], empty_frac=0.0)
    plans = _check_plans(A, 8)
    inside = [p for p in plans if p.own == 0]
    assert inside, "some device lies entirely inside the dense row"
    assert all(p.row_lo == 5 and p.has_carry for p in inside)


def test_more_devices_than_entries():
    A = random_csr(np.random.default_rng(1), 6, 6, 0.0, empty_frac=1.0)   # nnz = 0
    plans = D.shard_plans(_oracle_cuts(A, 4), A.nrows)
    assert plans[0].own == 6 and all(p.own == 0 and p.nloc == 0 for p in plans[1:])
    assert D.cut_rows(plans, 6) == [0, 6, 6, 6, 6]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _id_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2604_17198_b200 as N
        obj = [N.Dist.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        q.put((rank, obj[0]))
    finally:
        dist.destroy_process_group()


def test_unique_id_handoff_gloo():
    """nacho_dist_unique_id on rank 0, handed to every rank by torch.distributed (the only role torch
    has in the multi-GPU path): every rank receives the same NACHO_DIST_UNIQUE_ID_SIZE bytes."""
    import paper_2604_17198_b200 as N
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_id_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    assert res[0] == res[1] and len(res[0]) == N.lib.nacho_dist_unique_id_size()


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
