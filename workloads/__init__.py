"""Seeded synthetic workloads for the paper's hot path (inputs only -- no method arithmetic).

`SparseMatrix` is a plain container of CSR / DCSR arrays (numpy on the host or torch on a device).
`build(cfg, scale, device)` manufactures the operands of a configuration C1..C5 of BASELINE.json
(SURVEY.md 8(d)); on "cpu" the numpy recipe is used, on "cuda" the bit-identical CUDA twin.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import recipe as R

HERE = os.path.dirname(os.path.abspath(__file__))

CSR, DCSR, COO = "csr", "dcsr", "coo"


@dataclass
class SparseMatrix:
    format: str
    nrows: int
    ncols: int
    pos: object            # int64 [nouter+1]
    crd: object            # int32 [nnz]
    val: object            # float32/float64 [nnz]
    outer_crd: object = None   # int32 [nouter] (DCSR); COO: the row of every entry [nnz], pos = [0, nnz]

    @property
    def nnz(self) -> int:
        return int(self.crd.shape[0])

    @property
    def nouter(self) -> int:
        return int(self.pos.shape[0]) - 1

    def numpy(self) -> "SparseMatrix":
        def cv(a):
            if a is None:
                return None
            if isinstance(a, np.ndarray):
                return a
            return a.detach().cpu().numpy()
        return SparseMatrix(self.format, self.nrows, self.ncols, cv(self.pos), cv(self.crd), cv(self.val), cv(self.outer_crd))

    def to(self, device) -> "SparseMatrix":
        import torch

        def cv(a):
            if a is None:
                return None
            t = torch.from_numpy(a) if isinstance(a, np.ndarray) else a
            return t.to(device).contiguous()
        return SparseMatrix(self.format, self.nrows, self.ncols, cv(self.pos), cv(self.crd), cv(self.val), cv(self.outer_crd))


@dataclass
class Workload:
    name: str
    kind: str                      # spmv | spmv_dcsr | spadd | spmm
    ops: list
    x: object = None               # dense x (spmv) or B (spmm, row-major [N, nb])
    nb: int = 0
    P: int = 0                     # fixed partition count (0 = auto)
    meta: dict = field(default_factory=dict)


def from_coo(rows, cols, vals, nrows, ncols, fmt=CSR, dtype=np.float32) -> SparseMatrix:
    """Builds a sorted CSR/DCSR operand from coordinate lists (fixtures; duplicates not allowed)."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    vals = np.asarray(vals, dtype=dtype)
    order = np.lexsort((cols, rows))
    rows, cols, vals = rows[order], cols[order], vals[order]
    if fmt == CSR:
        pos = np.zeros(nrows + 1, dtype=np.int64)
        np.add.at(pos, rows + 1, 1)
        pos = np.cumsum(pos).astype(np.int64)
        return SparseMatrix(CSR, nrows, ncols, pos, cols.astype(np.int32), vals)
    outer, counts = np.unique(rows, return_counts=True)
    pos = np.zeros(len(outer) + 1, dtype=np.int64)
    pos[1:] = np.cumsum(counts)
    return SparseMatrix(DCSR, nrows, ncols, pos, cols.astype(np.int32), vals, outer.astype(np.int32))


def to_dense(A: SparseMatrix) -> np.ndarray:
    A = A.numpy()
    D = np.zeros((A.nrows, A.ncols), dtype=np.float64)
    if A.format == COO:
        for q in range(A.nnz):
            D[int(A.outer_crd[q]), int(A.crd[q])] = A.val[q]
        return D
    for ip in range(A.nouter):
        r = ip if A.format == CSR else int(A.outer_crd[ip])
        for q in range(int(A.pos[ip]), int(A.pos[ip + 1])):
            D[r, int(A.crd[q])] = A.val[q]
    return D


# ------------------------------------------------------------------ configurations
# (M = N, target nnz, dtype, seed, column kind) -- BASELINE.json "configs", SURVEY.md 8(d).
CONFIGS = {
    "c1": dict(kind="spmv", m=4096, target=36_900, dtype=np.float64, seed=1, cols="local", dense_row=2049, P=8),
    "c2": dict(kind="spadd", m=1_000_000, target=10_000_000, dtype=np.float32, seed=2, cols="local", k=3),
    "c3": dict(kind="spmv_dcsr", m=100_000_000, nouter=1_000_000, target=50_000_000, dtype=np.float32, seed=3, cols="uniform"),
    "c4": dict(kind="spmm", m=50_000_000, target=1_000_000_000, dtype=np.float32, seed=4, cols="web", nb=64),
    "c5": dict(kind="spmv", m=200_000_000, target=4_000_000_000, dtype=np.float32, seed=5, cols="local"),
}

STREAM_OP = [R.S_COL, R.S_COL + 16, R.S_COL + 32]  # own column stream of C2 operands A, B, C


def scaled(cfg: dict, scale: float) -> dict:
    c = dict(cfg)
    if scale != 1.0:
        c["m"] = max(64, int(round(c["m"] * scale)))
        c["target"] = max(16, int(round(c["target"] * scale)))
        if "nouter" in c:
            c["nouter"] = max(8, int(round(c["nouter"] * scale)))
        if c.get("dense_row") is not None:
            c["dense_row"] = min(c["dense_row"], c["m"] - 1)
    return c


def _cdiv(m, target, cap, min_deg=0):
    return R.find_cdiv(m, target, cap, min_deg)


def build(name: str, scale: float = 1.0, device: str = "cpu", values: str = "uniform", kmax: int = 4,
          column_kind: Optional[str] = None) -> Workload:
    """Manufactures configuration `name` (c1..c5), optionally scaled down by `scale`."""
    cfg = scaled(CONFIGS[name], scale)
    if column_kind:
        cfg["cols"] = column_kind
    dev = device if device != "cpu" else None
    gen = _HostGen(cfg, values, kmax) if dev is None else _DeviceGen(cfg, values, kmax, device)
    kind = cfg["kind"]
    m = cfg["m"]
    if kind == "spadd":
        pos = gen.pos(m, cfg["target"], cap=m)
        ops = []
        for o in range(cfg["k"]):
            crd = gen.cols(pos, o, mode=0 if o == 0 else o)
            val = gen.vals(1000 + o, pos)
            ops.append(SparseMatrix(CSR, m, m, pos, crd, val))
        return Workload(name, kind, ops, meta=cfg)
    if kind == "spmv_dcsr":
        nouter = cfg["nouter"]
        outer = gen.outer(m, nouter)
        pos = gen.pos(nouter, cfg["target"], cap=m, min_deg=1)
        crd = gen.cols_rows(pos, outer, m)
        val = gen.vals(1000, pos)
        A = SparseMatrix(DCSR, m, m, pos, crd, val, outer)
        return Workload(name, kind, [A], x=gen.dense(R.S_X, m, 1), meta=cfg)
    pos = gen.pos(m, cfg["target"], cap=m, dense_row=cfg.get("dense_row"))
    crd = gen.cols(pos, 0, mode=0)
    val = gen.vals(1000, pos)
    A = SparseMatrix(CSR, m, m, pos, crd, val)
    if kind == "spmm":
        return Workload(name, kind, [A], x=gen.dense(R.S_B, m, cfg["nb"]), nb=cfg["nb"], meta=cfg)
    return Workload(name, kind, [A], x=gen.dense(R.S_X, m, 1), P=cfg.get("P", 0), meta=cfg)


class _HostGen:
    def __init__(self, cfg, values, kmax):
        self.cfg, self.values, self.kmax = cfg, values, kmax
        self.dtype = cfg["dtype"]

    def pos(self, m, target, cap, min_deg=0, dense_row=None):
        cd = _cdiv(m, target, cap, min_deg)
        deg = R.degrees(m, cd, cap, self.cfg["seed"], min_deg)
        if dense_row is not None:
            deg[dense_row] = cap
        return R.pos_from_degrees(deg)

    def cols(self, pos, o, mode):
        cfg = self.cfg
        m = cfg["m"]
        rows = R.entry_rows(pos)
        own = R.columns(cfg["cols"], m, m, cfg["seed"], pos, STREAM_OP[o], rows)
        if mode == 0:
            return own
        k = np.arange(pos[-1], dtype=np.int64) - pos[rows]
        a = R.columns(cfg["cols"], m, m, cfg["seed"], pos, STREAM_OP[0], rows)
        if mode == 1:
            reuse = (R.hash4(cfg["seed"], R.S_REUSE_B, rows, k) % np.uint64(10)) < np.uint64(3)
            return np.where(reuse, a, own).astype(np.int32)
        b = R.columns(cfg["cols"], m, m, cfg["seed"], pos, STREAM_OP[1], rows)
        reuse = (R.hash4(cfg["seed"], R.S_REUSE_C, rows, k) % np.uint64(10)) < np.uint64(3)
        pickb = (R.hash4(cfg["seed"], R.S_PICK_C, rows, k) & np.uint64(1)) == np.uint64(1)
        return np.where(reuse, np.where(pickb, b, a), own).astype(np.int32)

    def cols_rows(self, pos, outer, m):
        # DCSR: column pattern generated with the stored row *coordinate* as the row counter
        cfg = self.cfg
        ip = R.entry_rows(pos)
        rows = outer.astype(np.int64)[ip]
        k = np.arange(pos[-1], dtype=np.int64) - pos[ip]
        d = (pos[ip + 1] - pos[ip]).astype(np.int64)
        return _columns_rkd(cfg["cols"], m, m, cfg["seed"], R.S_COL, rows, k, d)

    def vals(self, stream, pos):
        n = int(pos[-1])
        return R.values(self.cfg["seed"], stream, np.arange(n, dtype=np.int64), self.dtype, self.values, self.kmax)

    def outer(self, m, nouter):
        return R.outer_rows(m, nouter, self.cfg["seed"])

    def dense(self, stream, n, nb):
        v = R.values(self.cfg["seed"], stream, np.arange(n * nb, dtype=np.int64), self.dtype, "uniform")
        return v if nb == 1 else v.reshape(n, nb)


def _columns_rkd(kind, m, n, seed, stream, r, k, d):
    """Column rule of recipe.columns expressed on explicit (row, k, deg) arrays."""
    if kind == "uniform":
        w = np.full_like(d, n)
        w0 = np.zeros_like(d)
    else:
        w = np.minimum(n, np.maximum(4 * d, 4096))
        w0 = np.clip((r * n) // m - w // 2, 0, n - w)
    lo = w0 + (k * w) // d
    hi = w0 + ((k + 1) * w) // d
    col = lo + (R.hash4(seed, stream, r, k) % (hi - lo).astype(np.uint64)).astype(np.int64)
    return np.where(d >= n, k, col).astype(np.int32)


# ------------------------------------------------------------------ device generator
_LIB = None


def _lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(HERE, "libnacho_gen.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run __graft_entry__.build()")
        L = ctypes.CDLL(path)
        i64, u64, vp, ci = ctypes.c_int64, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_int
        L.wl_degrees.argtypes = [i64, i64, i64, i64, u64, i64, i64, vp, vp]
        L.wl_columns.argtypes = [ci, ci, i64, i64, u64, vp, i64, u64, u64, u64, vp, vp]
        L.wl_columns_rows.argtypes = [ci, i64, i64, u64, vp, vp, i64, i64, u64, vp, vp]
        L.wl_values.argtypes = [u64, u64, i64, ci, ci, ci, vp, vp]
        L.wl_outer.argtypes = [i64, i64, u64, vp, vp]
        L.wl_columns_range.argtypes = [ci, ci, i64, i64, u64, vp, i64, i64, u64, u64, u64, vp, vp]
        L.wl_values_range.argtypes = [u64, u64, i64, i64, ci, ci, ci, vp, vp]
        _LIB = L
    return _LIB


KIND_ID = {"local": 0, "uniform": 1, "web": 2}


class _DeviceGen:
    def __init__(self, cfg, values, kmax, device):
        import torch
        self.torch = torch
        self.cfg, self.values, self.kmax = cfg, values, kmax
        self.device = torch.device(device)
        self.f64 = cfg["dtype"] == np.float64
        self.tdtype = torch.float64 if self.f64 else torch.float32
        self.stream = torch.cuda.current_stream(self.device).cuda_stream

    def _chk(self, rc):
        if rc != 0:
            raise RuntimeError(f"workload generator CUDA error {rc}")

    def pos(self, m, target, cap, min_deg=0, dense_row=None):
        t = self.torch
        cd = _cdiv(m, target, cap, min_deg)
        deg = t.empty(m, dtype=t.int64, device=self.device)
        self._chk(_lib().wl_degrees(m, cd, cap, min_deg, self.cfg["seed"], -1 if dense_row is None else dense_row,
                                    cap, deg.data_ptr(), self.stream))
        pos = t.zeros(m + 1, dtype=t.int64, device=self.device)
        t.cumsum(deg, 0, out=pos[1:])
        del deg
        return pos

    def cols(self, pos, o, mode):
        t = self.torch
        nnz = int(pos[-1].item())
        crd = t.empty(nnz, dtype=t.int32, device=self.device)
        m = self.cfg["m"]
        self._chk(_lib().wl_columns(KIND_ID[self.cfg["cols"]], mode, m, m, self.cfg["seed"], pos.data_ptr(), nnz,
                                    STREAM_OP[o], STREAM_OP[0], STREAM_OP[1], crd.data_ptr(), self.stream))
        return crd

    def cols_rows(self, pos, outer, m):
        t = self.torch
        nnz = int(pos[-1].item())
        crd = t.empty(nnz, dtype=t.int32, device=self.device)
        self._chk(_lib().wl_columns_rows(KIND_ID[self.cfg["cols"]], m, m, self.cfg["seed"], pos.data_ptr(),
                                         outer.data_ptr(), outer.shape[0], nnz, R.S_COL, crd.data_ptr(), self.stream))
        return crd

    def vals(self, stream, pos):
        t = self.torch
        n = int(pos[-1].item())
        v = t.empty(n, dtype=self.tdtype, device=self.device)
        self._chk(_lib().wl_values(self.cfg["seed"], stream, n, 0 if self.values == "uniform" else 1, self.kmax,
                                   int(self.f64), v.data_ptr(), self.stream))
        return v

    def outer(self, m, nouter):
        t = self.torch
        o = t.empty(nouter, dtype=t.int32, device=self.device)
        self._chk(_lib().wl_outer(m, nouter, self.cfg["seed"], o.data_ptr(), self.stream))
        return o

    def dense(self, stream, n, nb):
        t = self.torch
        v = t.empty(n * nb, dtype=self.tdtype, device=self.device)
        self._chk(_lib().wl_values(self.cfg["seed"], stream, n * nb, 0, 4, int(self.f64), v.data_ptr(), self.stream))
        return v if nb == 1 else v.view(n, nb)


# ------------------------------------------------------------------ device shards (multi-GPU setup)
def full_pos(name: str, scale: float = 1.0, device: str = "cuda"):
    """The full row-pointer array of a one-operand configuration (cheap: degrees only)."""
    cfg = scaled(CONFIGS[name], scale)
    gen = _DeviceGen(cfg, "uniform", 4, device)
    return gen.pos(cfg["m"], cfg["target"], cap=cfg["m"], dense_row=cfg.get("dense_row")), cfg


def shard_entries(name: str, pos, e_lo: int, e_hi: int, scale: float = 1.0, device: str = "cuda"):
    """crd / val of entries [e_lo, e_hi) of configuration `name` -- bit-identical to the slice of the
    full matrix build() makes (counter-based generator), so a device holds only its shard."""
    import torch
    cfg = scaled(CONFIGS[name], scale)
    gen = _DeviceGen(cfg, "uniform", 4, device)
    n = e_hi - e_lo
    crd = torch.empty(n, dtype=torch.int32, device=gen.device)
    m = cfg["m"]
    gen._chk(_lib().wl_columns_range(KIND_ID[cfg["cols"]], 0, m, m, cfg["seed"], pos.data_ptr(), e_lo, e_hi,
                                     STREAM_OP[0], STREAM_OP[0], STREAM_OP[1], crd.data_ptr(), gen.stream))
    val = torch.empty(n, dtype=gen.tdtype, device=gen.device)
    gen._chk(_lib().wl_values_range(cfg["seed"], 1000, e_lo, n, 0, 4, int(gen.f64), val.data_ptr(), gen.stream))
    return crd, val


def dense_x(name: str, scale: float = 1.0, device: str = "cuda"):
    cfg = scaled(CONFIGS[name], scale)
    gen = _DeviceGen(cfg, "uniform", 4, device)
    return gen.dense(R.S_X, cfg["m"], 1)


def to_coo(A: SparseMatrix) -> SparseMatrix:
    """The COO form of a CSR operand (TACO's Compressed(non-unique) o Singleton: pos = [0, nnz], the
    row level one coordinate per entry).  Test fixtures and setup only."""
    if A.format != CSR:
        raise ValueError("to_coo takes a CSR operand")
    if isinstance(A.pos, np.ndarray):
        rows = np.repeat(np.arange(A.nrows, dtype=np.int32), np.diff(A.pos))
        pos = np.array([0, A.nnz], np.int64)
    else:
        import torch
        rows = torch.repeat_interleave(torch.arange(A.nrows, dtype=torch.int32, device=A.pos.device),
                                       A.pos[1:] - A.pos[:-1])
        pos = torch.tensor([0, A.nnz], dtype=torch.int64, device=A.pos.device)
    return SparseMatrix(COO, A.nrows, A.ncols, pos, A.crd, A.val, rows)


@dataclass
class Tensor3:
    """A third-order tensor in CSF (Compressed o Compressed o Compressed): slices crd0 (i), fibers
    pos1 / crd1 (j), entries pos2 / crd2 (k), val."""
    shape: tuple
    crd0: object
    pos1: object
    crd1: object
    pos2: object
    crd2: object
    val: object

    @property
    def nnz(self) -> int:
        return int(self.crd2.shape[0])

    def to(self, device) -> "Tensor3":
        import torch

        def cv(a):
            return a if isinstance(a, torch.Tensor) and a.device == torch.device(device) else torch.as_tensor(a).to(device)
        return Tensor3(self.shape, cv(self.crd0), cv(self.pos1), cv(self.crd1), cv(self.pos2), cv(self.crd2), cv(self.val))


def csf_from_coo(i, j, k, vals, shape, dtype=np.float32) -> Tensor3:
    """A CSF tensor from coordinate lists (fixtures; duplicates not allowed)."""
    i, j, k = (np.asarray(x, dtype=np.int64) for x in (i, j, k))
    vals = np.asarray(vals, dtype=dtype)
    order = np.lexsort((k, j, i))
    i, j, k, vals = i[order], j[order], k[order], vals[order]
    fib = np.ones(len(i), bool)
    fib[1:] = (i[1:] != i[:-1]) | (j[1:] != j[:-1])
    fstart = np.nonzero(fib)[0]
    pos2 = np.concatenate([fstart, [len(i)]]).astype(np.int64)
    fi, fj = i[fstart], j[fstart]
    sl = np.ones(len(fi), bool)
    sl[1:] = fi[1:] != fi[:-1]
    sstart = np.nonzero(sl)[0]
    pos1 = np.concatenate([sstart, [len(fi)]]).astype(np.int64)
    return Tensor3(tuple(int(x) for x in shape), fi[sstart].astype(np.int32), pos1, fj.astype(np.int32), pos2,
                   k.astype(np.int32), vals)


def random_csf(rng, shape, density, dtype=np.float32) -> Tensor3:
    mask = rng.random(shape) < density
    i, j, k = np.nonzero(mask)
    return csf_from_coo(i, j, k, rng.uniform(0.5, 1.5, len(i)), shape, dtype)

