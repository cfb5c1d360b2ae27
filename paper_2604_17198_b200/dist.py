"""Device-level sharding of the hot path over D GPUs of one box.

The partition IS the device decomposition: device d owns the coordinate range [b_d, b_{d+1}) of
Alg. 1 run with P = D (one partition per processor; the boundaries are saved
positions), so every device does Q*/D +- Delta work (Theorem 1) and holds only
that shard of A.  The paper is shared-memory only; the exchange step is this build's:

  SpMV   x is replicated (nacho_dist_broadcast at setup).  Device d holds rows
         [row_lo, row_lo + nloc) of A restricted to its positions [pos_lo, pos_hi): every row it owns
         (R7: rows [cut_d, cut_{d+1})) plus, for d < D-1, the row cut by b_{d+1}, whose partial sum is
         the device's seam carry.  nacho_dist_spmv = local partitions + SpMV, an NCCL all-gather of
         one (row, value) pair per device, the seam fix-up (carries added in device order by the
         owner), and optionally the gather of the owned y segments.
  SpAdd  every device unions its coordinate range; equal coordinates never straddle a cut
         (P:2635-2637), so no values merge: nacho_dist_spadd_gather all-gathers the D union sizes
         (global offsets) and gathers the Z segments.

All of it runs in libnacho.so (kernels + NCCL); this module is host-side bookkeeping: the shard plan
from the device cuts, building a device's shard, and the single-process helpers the one-GPU tests
use to emulate D devices with the same kernels.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch


@dataclass
class ShardPlan:
    """Device d's share of a one-operand matrix under the device cuts."""
    d: int
    D: int
    row_lo: int      # first row held (cut_d)
    nloc: int        # rows held: owned rows + the row cut by b_{d+1} (d < D-1)
    own: int         # rows owned (R7): [row_lo, row_lo + own)
    pos_lo: int      # positions [pos_lo, pos_hi) of A held by the device
    pos_hi: int

    @property
    def has_carry(self) -> bool:
        return self.nloc > self.own


def shard_plans(cuts, nrows: int):
    """Plans of every device from the D+1 device cuts (host array [(row, pos)] * (D+1))."""
    D = len(cuts) - 1
    plans = []
    for d in range(D):
        row_lo, pos_lo = int(cuts[d][0]), int(cuts[d][1])
        row_hi, pos_hi = int(cuts[d + 1][0]), int(cuts[d + 1][1])
        own = row_hi - row_lo
        nloc = own + 1 if d < D - 1 else nrows - row_lo
        if d < D - 1 and row_hi >= nrows:   # empty tail shards (P > Q*): no row past the end
            nloc = own
        plans.append(ShardPlan(d, D, row_lo, nloc, own, pos_lo, pos_hi))
    return plans


def cut_rows(plans, nrows: int):
    """Host int64[D+1]: each device's first row, then nrows (the nacho_dist_* cut_rows argument)."""
    return [p.row_lo for p in plans] + [nrows]


def build_shard(plan: ShardPlan, pos_full: torch.Tensor, crd: torch.Tensor, val: torch.Tensor, ncols: int):
    """Device d's CSR shard: nacho_shard_rows on the full row pointers, crd / val of its positions
    (already sliced by the caller: a shard generator, or a slice of a full matrix)."""
    from . import shard_rows
    import workloads as W
    lp = shard_rows(pos_full, plan.row_lo, plan.nloc, plan.pos_lo, plan.pos_hi)
    return W.SparseMatrix("csr", plan.nloc, ncols, lp, crd, val)


def spmv_setup(name: str, scale: float, D: int, d: int, device="cuda"):
    """Setup of device d for SpMV on configuration `name`: full row pointers (degrees only), the device
    cuts (nacho_device_cuts), and only this device's entries generated (workloads.shard_entries)."""
    import workloads as W
    from . import device_cuts
    pos, cfg = W.full_pos(name, scale, device)
    M = cfg["m"]
    full = W.SparseMatrix("csr", M, M, pos, torch.empty(0, dtype=torch.int32, device=device),
                          torch.empty(0, dtype=torch.float32, device=device))
    cuts = device_cuts(_PosOnly(full, int(pos[-1].item())), D).cpu().tolist()
    plans = shard_plans(cuts, M)
    p = plans[d]
    crd, val = W.shard_entries(name, pos, p.pos_lo, p.pos_hi, scale, device)
    A_local = build_shard(p, pos, crd, val, M)
    del pos
    return A_local, plans, cuts


class _PosOnly:
    """Descriptor source for nacho_device_cuts: pos and sizes only."""

    def __init__(self, A, nnz):
        self.pos, self.nrows, self.ncols, self.nnz = A.pos, A.nrows, A.ncols, nnz


# ------------------------------------------------------------------ one-GPU emulation helpers (tests)
def carry_of(plan: ShardPlan, y_local: torch.Tensor):
    """(row, value-bits) pair nacho_dist_spmv all-gathers for this device."""
    if plan.has_carry and plan.nloc > 0:
        v = y_local[plan.nloc - 1:plan.nloc].clone()
        bits = v.view(torch.int32).to(torch.int64) if v.dtype == torch.float32 else v.view(torch.int64)
        if v.dtype == torch.float32:
            bits = bits & 0xFFFFFFFF
        return torch.tensor([plan.row_lo + plan.nloc - 1], dtype=torch.int64, device=y_local.device), bits
    z = torch.zeros(1, dtype=torch.int64, device=y_local.device)
    return z - 1, z


def spmv_combine(pieces, nrows: int, dtype, device):
    """pieces[d] = (y_local_d after the seam fix-up, plan_d): the owned segments of every device."""
    y = torch.zeros(nrows, dtype=dtype, device=device)
    for yl, p in pieces:
        y[p.row_lo:p.row_lo + p.own] = yl[:p.own]
    return y


# ------------------------------------------------------------------ partition slices (SpAdd shards)
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


def spadd_shard_ops(ops, dparts, d: int):
    """Device d's operand shards for the k-way SpAdd: rows [b_d.row, b_{d+1}.row] of every operand,
    restricted to that operand's cut positions b_d.pos[o], b_{d+1}.pos[o] (nacho_shard_rows), crd / val
    copied (16-byte-aligned bases for the bulk copies)."""
    import workloads as W
    from . import shard_rows
    k = len(ops)
    M = ops[0].nrows
    D = dparts.P
    row_lo = int(dparts.row[d].item())
    row_hi = int(dparts.row[d + 1].item())
    nloc = (row_hi - row_lo + 1) if d < D - 1 and row_hi < M else (M - row_lo if d == D - 1 else row_hi - row_lo)
    out = []
    for o, A in enumerate(ops):
        lo = int(dparts.pos[d * k + o].item())
        hi = int(dparts.pos[(d + 1) * k + o].item())
        lp = shard_rows(A.pos, row_lo, nloc, lo, hi)
        out.append(W.SparseMatrix("csr", nloc, A.ncols, lp, A.crd[lo:hi].clone(), A.val[lo:hi].clone()))
    own = (row_hi if d < D - 1 else M) - row_lo
    return out, row_lo, own


def spadd_combine(pieces, nrows: int, device):
    """pieces[d] = (z_pos_local, z_crd_local, z_val_local, nnz_local, row_lo, own): one-GPU emulation of
    nacho_dist_spadd_gather (device d's Z.pos rows row_lo + 1 .. row_lo + own, its entries at its offset)."""
    base = 0
    z_pos = torch.zeros(nrows + 1, dtype=torch.int64, device=device)
    crds, vals = [], []
    for zp, zc, zv, nl, lo, own in pieces:
        z_pos[lo + 1:lo + own + 1] = zp[1:own + 1] + base
        crds.append(zc[:nl])
        vals.append(zv[:nl])
        base += nl
    return z_pos, torch.cat(crds), torch.cat(vals)
