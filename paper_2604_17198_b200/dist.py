"""Device-level sharding of the hot path over D GPUs of one box.

The partition IS the device decomposition: with P_total = D * P_l partitions, rank d runs partitions
[d*P_l, (d+1)*P_l) -- its device cut is the Q = floor(d*Q*/D) cut of Alg. 1, so every
rank gets Q*/D +- Delta work and the result is identical to the single-GPU one for the same P_total
(invariant I9).  The paper is shared-memory only; the exchange step is new:

  SpMV   every rank computes the rows its partitions own (R7) into a zeroed y, which leaves at most one
         non-owned "seam" row holding the rank's trailing carry.  Exchange = all-gather of the owned row
         segments + all-gather of the D seam (row, value) pairs, added in rank order.
  SpAdd  every rank unions its coordinate range [b_{d*P_l}, b_{(d+1)*P_l}) into a local Z.  Equal
         coordinates never straddle a cut, so no values merge at seams: exchange =
         all-gather of the D union counts -> global offsets, all-gather of the Z segments, rebasing of
         the locally owned Z.pos rows.

Transport is torch.distributed (NCCL over NVLink on GPUs, gloo in the CPU tests); the local compute is
a callable, so the same assembly code runs on the CUDA kernels and, in tests, on emulated slices.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist


@dataclass
class PartsView:
    """A contiguous slice [lo, hi) of a Parts record (boundaries lo..hi), sharing its storage."""
    P: int
    k: int
    query: torch.Tensor
    row: torch.Tensor
    row_pos: torch.Tensor
    col: torch.Tensor
    pos: torch.Tensor
    max_work: int = 0

    def c(self):
        from . import PartsC
        s = PartsC()
        s.P, s.k = self.P, self.k
        s.query, s.row, s.row_pos = self.query.data_ptr(), self.row.data_ptr(), self.row_pos.data_ptr()
        s.col, s.pos = self.col.data_ptr(), self.pos.data_ptr()
        s.max_work = self.max_work
        return s


def slice_parts(parts, lo: int, hi: int) -> PartsView:
    """Partitions [lo, hi) of `parts` (boundaries lo..hi inclusive) without copying."""
    k = parts.k
    return PartsView(hi - lo, k, parts.query[lo:hi + 1], parts.row[lo:hi + 1], parts.row_pos[lo:hi + 1],
                     parts.col[lo:hi + 1], parts.pos[lo * k:(hi + 1) * k], getattr(parts, "max_work", 0))


def rank_range(P_total: int, world: int, rank: int):
    """Rank `rank`'s partitions: [rank*P_l, (rank+1)*P_l) with P_total = world * P_l."""
    assert P_total % world == 0, "P_total must be a multiple of the world size"
    P_l = P_total // world
    return rank * P_l, (rank + 1) * P_l


def _all_gather_v(t: torch.Tensor, counts, group=None) -> torch.Tensor:
    """Variable-size all-gather along dim 0 (pads to the largest chunk)."""
    world = len(counts)
    mx = max(max(counts), 1)
    buf = torch.zeros((mx,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    if t.shape[0]:
        buf[:t.shape[0]] = t
    out = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(out, buf, group=group)
    return torch.cat([o[:c] for o, c in zip(out, counts)], dim=0)


def _all_gather_scalars(vals, device, dtype=torch.int64, group=None):
    t = torch.tensor(vals, dtype=dtype, device=device)
    out = [torch.empty_like(t) for _ in range(dist.get_world_size(group))]
    dist.all_gather(out, t, group=group)
    return torch.stack(out)


# ------------------------------------------------------------------ local (single-process) combination
def spmv_combine(pieces, nrows: int, dtype, device):
    """pieces[d] = (y_local_d, own_lo, own_hi, seam_row): owned segments, then seams in rank order."""
    y = torch.zeros(nrows, dtype=dtype, device=device)
    for yl, lo, hi, _ in pieces:
        y[lo:hi] = yl[lo:hi]
    for yl, _, _, seam in pieces:
        if 0 <= seam < nrows:
            y[seam] += yl[seam]
    return y


def spadd_combine(pieces, nrows: int, device):
    """pieces[d] = (z_pos_local, z_crd_local, z_val_local, nnz_local, own_lo, own_hi)."""
    base = 0
    z_pos = torch.zeros(nrows + 1, dtype=torch.int64, device=device)
    crds, vals = [], []
    for zp, zc, zv, nl, lo, hi in pieces:
        z_pos[lo + 1:hi + 1] = zp[lo + 1:hi + 1] + base
        crds.append(zc[:nl])
        vals.append(zv[:nl])
        base += nl
    return z_pos, torch.cat(crds), torch.cat(vals)


# ------------------------------------------------------------------ SpMV
def spmv_assemble(y_local: torch.Tensor, own_lo: int, own_hi: int, seam_row: int, nrows: int, group=None):
    """Full y from every rank's zero-initialised local y.

    y_local : this rank's y (length nrows); exact on its owned rows [own_lo, own_hi) and holding the
              rank's trailing carry on `seam_row` (== own_hi, or -1 when the rank has no carry).
    """
    world = dist.get_world_size(group)
    seg = y_local[own_lo:own_hi]
    meta = _all_gather_scalars([own_lo, own_hi, seam_row], y_local.device, group=group)
    counts = [int(m[1] - m[0]) for m in meta]
    segs = _all_gather_v(seg, counts, group=group)
    sv = y_local[seam_row:seam_row + 1] if 0 <= seam_row < nrows else torch.zeros(1, dtype=y_local.dtype,
                                                                                   device=y_local.device)
    seams = _all_gather_v(sv, [1] * world, group=group)
    y = torch.zeros(nrows, dtype=y_local.dtype, device=y_local.device)
    off = 0
    for d in range(world):
        lo, hi = int(meta[d][0]), int(meta[d][1])
        y[lo:hi] = segs[off:off + (hi - lo)]
        off += hi - lo
    for d in range(world):  # seam carries in rank (= partition) order
        r = int(meta[d][2])
        if 0 <= r < nrows:
            y[r] += seams[d]
    return y


def spmv_rank_rows(parts_row_pos: torch.Tensor, lo: int, hi: int, nouter: int):
    """Owned outer rows [own_lo, own_hi) of partitions [lo, hi) and the seam row (R7)."""
    own_lo = int(parts_row_pos[lo])
    own_hi = int(parts_row_pos[hi])
    seam = own_hi if own_hi < nouter else -1
    return own_lo, own_hi, seam


def spmv(A, x, parts, group=None):
    """Distributed y = A x on the CUDA kernels: local slice, then the exchange above."""
    from . import spmv as local_spmv
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    lo, hi = rank_range(parts.P, world, rank)
    view = slice_parts(parts, lo, hi)
    n_y = int(A.pos.shape[0]) - 1
    y_local = torch.zeros(n_y, dtype=A.val.dtype, device=x.device)
    local_spmv(A, x, view, y=y_local)
    rp = parts.row_pos.cpu()
    own_lo, own_hi, seam = spmv_rank_rows(rp, lo, hi, n_y)
    return spmv_assemble(y_local, own_lo, own_hi, seam, n_y, group=group)


# ------------------------------------------------------------------ SpAdd
def spadd_assemble(nrows: int, z_pos_local: torch.Tensor, z_crd_local: torch.Tensor, z_val_local: torch.Tensor,
                   nnz_local: int, own_lo: int, own_hi: int, group=None):
    """Global Z from every rank's local union.

    z_pos_local : local row pointers, valid on the owned rows: z_pos_local[r+1] for r in [own_lo, own_hi)
                  counts the local entries up to the end of row r (relative to this rank's segment).
    """
    world = dist.get_world_size(group)
    meta = _all_gather_scalars([nnz_local, own_lo, own_hi], z_crd_local.device, group=group)
    counts = [int(m[0]) for m in meta]
    base = [0]
    for c in counts:
        base.append(base[-1] + c)
    rank = dist.get_rank(group)
    z_crd = _all_gather_v(z_crd_local[:nnz_local], counts, group=group)
    z_val = _all_gather_v(z_val_local[:nnz_local], counts, group=group)
    rows = _all_gather_v(z_pos_local[own_lo + 1:own_hi + 1] + base[rank], [int(m[2] - m[1]) for m in meta],
                         group=group)
    z_pos = torch.zeros(nrows + 1, dtype=torch.int64, device=z_crd_local.device)
    off = 0
    for d in range(world):
        lo, hi = int(meta[d][1]), int(meta[d][2])
        z_pos[lo + 1:hi + 1] = rows[off:off + (hi - lo)]
        off += hi - lo
    return z_pos, z_crd, z_val


class ShardedZ:
    """One device's share of Z = sum_o A_o under a device-level cut: the union entries of partitions
    [lo, hi) of the global P-partition (local CSR pieces: z_pos is valid on the owned rows
    [own_lo, own_hi), relative to this shard's first entry)."""

    def __init__(self, z_pos, z_crd, z_val, nnz, own_lo, own_hi, part_off):
        self.z_pos, self.z_crd, self.z_val = z_pos, z_crd, z_val
        self.nnz, self.own_lo, self.own_hi, self.part_off = nnz, own_lo, own_hi, part_off


def spadd_shard(ops, P_total: int, world: int, rank: int, out=None, ws=None, sync=True) -> ShardedZ:
    """This device's share of the k-way SpAdd: it searches only its own P_l + 1 boundaries
    (nacho_partition_slice) and runs the staged single-read kernels on them; no communication.
    sync=False skips the one device->host read (nnz of the shard) for timed loops."""
    from . import partition_slice, spadd_k_staged
    lo, hi = rank_range(P_total, world, rank)
    parts = partition_slice(ops, P_total, lo, hi)
    dev = ops[0].pos.device
    part_off = torch.empty(parts.P + 1, dtype=torch.int64, device=dev)
    z_pos, z_crd, z_val = spadd_k_staged(ops, parts, *(out or ()), part_off=part_off, ws=ws)
    nnz = int(part_off[-1].item()) if sync else -1
    own_lo, own_hi = (int(parts.row[0].item()), int(parts.row[-1].item())) if sync else (-1, -1)
    return ShardedZ(z_pos, z_crd, z_val, nnz, own_lo, own_hi, part_off)


def spadd(ops, P_total: int, group=None):
    """Distributed k-way SpAdd: every rank computes its shard (spadd_shard), then the Z segments are
    all-gathered and rebased (spadd_assemble) -- equal coordinates never straddle a cut."""
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    sh = spadd_shard(ops, P_total, world, rank)
    return spadd_assemble(ops[0].nrows, sh.z_pos, sh.z_crd, sh.z_val, sh.nnz, sh.own_lo, sh.own_hi, group=group)
