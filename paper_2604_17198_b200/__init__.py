"""paper_2604_17198_b200 -- thin Python binding of libnacho.so (include/nacho.h).

Argument marshalling only: torch CUDA tensors -> raw device pointers and sizes.  Every step of the
hot path (partition search, SpMV, SpAdd, SpMM, scans, fix-ups) runs in the library's sm_100a
kernels.  There is no CPU fallback: importing without the built library raises.

Operands are any objects with the attributes of workloads.SparseMatrix (format, nrows, ncols, pos,
crd, val, outer_crd) holding contiguous CUDA tensors (pos int64, crd/outer_crd int32, val fp32/fp64).
"""
from __future__ import annotations

import ctypes
import os

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("NACHO_LIB", os.path.join(HERE, "libnacho.so"))

NACHO_CSR, NACHO_DCSR = 0, 1
NACHO_F32, NACHO_F64 = 0, 1
MAX_K = 8
STATUS = {0: "SUCCESS", 1: "INVALID_ARG", 2: "SHAPE", 3: "FORMAT", 4: "OVERFLOW", 5: "WORKSPACE", 6: "CUDA"}


class NachoError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"nacho {STATUS.get(status, status)}: {msg}")
        self.status = status


class Matrix(ctypes.Structure):
    _fields_ = [("format", ctypes.c_int32), ("dtype", ctypes.c_int32),
                ("nrows", ctypes.c_int64), ("ncols", ctypes.c_int64), ("nnz", ctypes.c_int64),
                ("nouter", ctypes.c_int64), ("outer_crd", ctypes.c_void_p), ("pos", ctypes.c_void_p),
                ("crd", ctypes.c_void_p), ("val", ctypes.c_void_p)]


class PartsC(ctypes.Structure):
    _fields_ = [("P", ctypes.c_int32), ("k", ctypes.c_int32), ("query", ctypes.c_void_p),
                ("row", ctypes.c_void_p), ("row_pos", ctypes.c_void_p), ("col", ctypes.c_void_p),
                ("pos", ctypes.c_void_p), ("max_work", ctypes.c_int64)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is not built; run __graft_entry__.build() (no CPU fallback exists)")
    L = ctypes.CDLL(LIB_PATH)
    vp, i32, i64, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
    L.nacho_partition.argtypes = [vp, i32, i32, vp, vp]
    L.nacho_partition_slice.argtypes = [vp, i32, i32, i32, vp, vp]
    L.nacho_auto_partitions.argtypes = [vp, i32, i32]
    L.nacho_auto_partitions.restype = i32
    L.nacho_spmv_workspace_size.argtypes = [vp, i32]
    L.nacho_spmv_workspace_size.restype = sz
    L.nacho_spmv.argtypes = [vp, vp, vp, vp, i32, vp, sz, vp]
    L.nacho_spadd_k_workspace_size.argtypes = [vp, i32, i32]
    L.nacho_spadd_k_workspace_size.restype = sz
    L.nacho_spadd_k_count.argtypes = [vp, i32, vp, vp, vp, sz, vp]
    L.nacho_spadd_k_fill.argtypes = [vp, i32, vp, vp, vp, vp, vp, vp, sz, vp]
    L.nacho_spadd_k.argtypes = [vp, i32, vp, vp, vp, vp, vp, vp, sz, vp]
    L.nacho_spadd_k_staged.argtypes = [vp, i32, vp, vp, vp, vp, vp, vp, sz, vp]
    L.nacho_spadd_k_staged_workspace_size.argtypes = [vp, i32, i32]
    L.nacho_spadd_k_staged_workspace_size.restype = sz
    L.nacho_spmm_workspace_size.argtypes = [vp, i32, i32]
    L.nacho_spmm_workspace_size.restype = sz
    L.nacho_spmm.argtypes = [vp, vp, vp, i64, i32, vp, i64, vp, sz, vp]
    L.nacho_validate.argtypes = [vp, vp]
    L.nacho_last_error.restype = ctypes.c_char_p
    L.nacho_launch_count.argtypes = [i32]
    L.nacho_launch_count.restype = i64
    return L


lib = _load()

EXPORTS = ["nacho_partition", "nacho_partition_slice", "nacho_auto_partitions", "nacho_spmv_workspace_size", "nacho_spmv",
           "nacho_spadd_k_workspace_size", "nacho_spadd_k_count", "nacho_spadd_k_fill", "nacho_spadd_k",
           "nacho_spadd_k_staged_workspace_size", "nacho_spadd_k_staged",
           "nacho_spmm_workspace_size", "nacho_spmm", "nacho_validate", "nacho_last_error",
           "nacho_launch_count"]


def _check(status):
    if status != 0:
        raise NachoError(status, lib.nacho_last_error().decode())


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream):
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def _require(t, dtype, name):
    if not (isinstance(t, torch.Tensor) and t.is_cuda):
        raise TypeError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")


def matrix(A) -> Matrix:
    """nacho_matrix descriptor of a workloads.SparseMatrix-like object (no copies)."""
    _require(A.pos, torch.int64, "pos")
    _require(A.crd, torch.int32, "crd")
    if A.val.dtype not in (torch.float32, torch.float64):
        raise TypeError("val must be float32 or float64")
    _require(A.val, A.val.dtype, "val")
    m = Matrix()
    m.format = NACHO_CSR if A.format == "csr" else NACHO_DCSR
    m.dtype = NACHO_F64 if A.val.dtype == torch.float64 else NACHO_F32
    m.nrows, m.ncols = int(A.nrows), int(A.ncols)
    m.nnz = int(A.crd.shape[0])
    m.nouter = int(A.pos.shape[0]) - 1
    if A.outer_crd is not None:
        _require(A.outer_crd, torch.int32, "outer_crd")
        m.outer_crd = A.outer_crd.data_ptr()
    m.pos, m.crd, m.val = A.pos.data_ptr(), A.crd.data_ptr(), A.val.data_ptr()
    return m


def _matrices(ops):
    arr = (Matrix * len(ops))()
    for i, A in enumerate(ops):
        arr[i] = matrix(A)
    return arr


class Parts:
    """Device partition record (nacho_parts): P+1 boundaries of k operands."""

    def __init__(self, P, k, device):
        self.P, self.k = P, k
        self.query = torch.empty(P + 1, dtype=torch.int64, device=device)
        self.row = torch.empty(P + 1, dtype=torch.int64, device=device)
        self.row_pos = torch.empty(P + 1, dtype=torch.int64, device=device)
        self.col = torch.empty(P + 1, dtype=torch.int32, device=device)
        self.pos = torch.empty((P + 1) * k, dtype=torch.int64, device=device)
        self.max_work = 0   # set by partition() / partition_slice() (host-side bound, no device read)

    def c(self) -> PartsC:
        s = PartsC()
        s.P, s.k = self.P, self.k
        s.query, s.row, s.row_pos = self.query.data_ptr(), self.row.data_ptr(), self.row_pos.data_ptr()
        s.col, s.pos = self.col.data_ptr(), self.pos.data_ptr()
        s.max_work = self.max_work
        return s


def _workspace(nbytes, device):
    if nbytes == 0:
        return None, 0
    return torch.empty(nbytes, dtype=torch.uint8, device=device), nbytes


def auto_partitions(ops, op: str) -> int:
    code = {"spmv": 0, "spadd": 1, "spmm": 2}[op]
    arr = _matrices(ops)
    return lib.nacho_auto_partitions(arr, len(ops), code)


def partition(ops, P: int, out: Parts = None, stream=None) -> Parts:
    """nacho_partition: Alg. 1 boundaries for P partitions of the k = len(ops) operands."""
    arr = _matrices(ops)
    out = out or Parts(P, len(ops), ops[0].pos.device)
    pc = out.c()
    _check(lib.nacho_partition(arr, len(ops), P, ctypes.byref(pc), _stream(stream)))
    out.max_work = pc.max_work
    return out


def partition_slice(ops, P: int, p_begin: int, p_end: int, out: Parts = None, stream=None) -> Parts:
    """nacho_partition_slice: boundaries p_begin .. p_end of the P-partition (a device's share)."""
    arr = _matrices(ops)
    out = out or Parts(p_end - p_begin, len(ops), ops[0].pos.device)
    pc = out.c()
    _check(lib.nacho_partition_slice(arr, len(ops), P, p_begin, ctypes.byref(pc), _stream(stream)))
    out.max_work = pc.max_work
    return out


def spmv(A, x, parts: Parts = None, dense_y: bool = False, y=None, ws=None, stream=None):
    """nacho_spmv: y = A x (CSR y[nrows]; DCSR compressed y[nouter], or y[nrows] with dense_y)."""
    m = matrix(A)
    _require(x, A.val.dtype, "x")
    n_y = A.nrows if (A.format == "csr" or dense_y) else int(A.pos.shape[0]) - 1
    if y is None:
        y = torch.empty(n_y, dtype=A.val.dtype, device=x.device)
    need = lib.nacho_spmv_workspace_size(ctypes.byref(m), parts.P if parts else 0)
    if ws is None or ws.numel() < need:
        ws, _ = _workspace(need, x.device)
    pc = ctypes.byref(parts.c()) if parts else None
    _check(lib.nacho_spmv(ctypes.byref(m), pc, _ptr(x), _ptr(y), int(dense_y), _ptr(ws), need, _stream(stream)))
    return y


def spadd_k_count(ops, parts: Parts, part_off=None, ws=None, stream=None):
    """nacho_spadd_k_count: per-partition union counts and their exclusive prefix sum."""
    arr = _matrices(ops)
    dev = ops[0].pos.device
    if part_off is None:
        part_off = torch.empty(parts.P + 1, dtype=torch.int64, device=dev)
    need = lib.nacho_spadd_k_workspace_size(arr, len(ops), parts.P)
    if ws is None or ws.numel() < need:
        ws, _ = _workspace(need, dev)
    pc = parts.c()
    _check(lib.nacho_spadd_k_count(arr, len(ops), ctypes.byref(pc), _ptr(part_off), _ptr(ws), need, _stream(stream)))
    return part_off


def spadd_k_fill(ops, parts: Parts, part_off, nnz_z: int, z_pos=None, z_crd=None, z_val=None, stream=None):
    arr = _matrices(ops)
    dev = ops[0].pos.device
    if z_pos is None:
        z_pos = torch.empty(ops[0].nrows + 1, dtype=torch.int64, device=dev)
    if z_crd is None:
        z_crd = torch.empty(max(nnz_z, 1), dtype=torch.int32, device=dev)
    if z_val is None:
        z_val = torch.empty(max(nnz_z, 1), dtype=ops[0].val.dtype, device=dev)
    pc = parts.c()
    _check(lib.nacho_spadd_k_fill(arr, len(ops), ctypes.byref(pc), _ptr(part_off), _ptr(z_pos), _ptr(z_crd),
                                  _ptr(z_val), None, 0, _stream(stream)))
    return z_pos, z_crd[:nnz_z], z_val[:nnz_z]


def spadd_k_fused(ops, parts: Parts, z_pos=None, z_crd=None, z_val=None, part_off=None, ws=None, stream=None):
    """nacho_spadd_k: single-pass SpAdd (decoupled look-back); Z buffers sized Q* (an upper bound).
    Returns (z_pos, z_crd, z_val) with z_crd / z_val at full capacity; nnz_Z = z_pos[-1]."""
    arr = _matrices(ops)
    dev = ops[0].pos.device
    cap = max(1, sum(int(A.crd.shape[0]) for A in ops))
    if z_pos is None:
        z_pos = torch.empty(ops[0].nrows + 1, dtype=torch.int64, device=dev)
    if z_crd is None:
        z_crd = torch.empty(cap, dtype=torch.int32, device=dev)
    if z_val is None:
        z_val = torch.empty(cap, dtype=ops[0].val.dtype, device=dev)
    need = lib.nacho_spadd_k_workspace_size(arr, len(ops), parts.P)
    if ws is None or ws.numel() < need:
        ws, _ = _workspace(need, dev)
    pc = parts.c()
    _check(lib.nacho_spadd_k(arr, len(ops), ctypes.byref(pc), _ptr(part_off), _ptr(z_pos), _ptr(z_crd), _ptr(z_val),
                             _ptr(ws), need, _stream(stream)))
    return z_pos, z_crd, z_val


def spadd_k_staged(ops, parts: Parts, z_pos=None, z_crd=None, z_val=None, part_off=None, ws=None, stream=None):
    """nacho_spadd_k_staged: one read of the operands, no look-back (staged union -> scan -> placement).
    Returns (z_pos, z_crd, z_val) with z_crd / z_val at capacity Q*; nnz_Z = z_pos[-1]."""
    arr = _matrices(ops)
    dev = ops[0].pos.device
    cap = max(1, sum(int(A.crd.shape[0]) for A in ops))
    if z_pos is None:
        z_pos = torch.empty(ops[0].nrows + 1, dtype=torch.int64, device=dev)
    if z_crd is None:
        z_crd = torch.empty(cap, dtype=torch.int32, device=dev)
    if z_val is None:
        z_val = torch.empty(cap, dtype=ops[0].val.dtype, device=dev)
    if part_off is None:
        part_off = torch.empty(parts.P + 1, dtype=torch.int64, device=dev)
    need = lib.nacho_spadd_k_staged_workspace_size(arr, len(ops), parts.P)
    if ws is None or ws.numel() < need:
        ws, _ = _workspace(need, dev)
    pc = parts.c()
    _check(lib.nacho_spadd_k_staged(arr, len(ops), ctypes.byref(pc), _ptr(part_off), _ptr(z_pos), _ptr(z_crd),
                                    _ptr(z_val), _ptr(ws), need, _stream(stream)))
    return z_pos, z_crd, z_val


def spadd_k(ops, parts: Parts = None, P: int = None, stream=None):
    """Two-pass k-way SpAdd (partition -> count/scan -> host reads nnz_Z -> fill)."""
    if parts is None:
        parts = partition(ops, P or auto_partitions(ops, "spadd"), stream=stream)
    part_off = spadd_k_count(ops, parts, stream=stream)
    nnz_z = int(part_off[-1].item())           # the one device->host read of the two-pass scheme
    return spadd_k_fill(ops, parts, part_off, nnz_z, stream=stream)


def spmm(A, B, parts: Parts = None, C=None, ws=None, stream=None):
    """nacho_spmm: C = A B with B row-major [ncols, nb]."""
    m = matrix(A)
    _require(B, A.val.dtype, "B")
    nb = int(B.shape[1])
    if C is None:
        C = torch.empty(A.nrows, nb, dtype=A.val.dtype, device=B.device)
    need = lib.nacho_spmm_workspace_size(ctypes.byref(m), parts.P if parts else 0, nb)
    if ws is None or ws.numel() < need:
        ws, _ = _workspace(need, B.device)
    pc = ctypes.byref(parts.c()) if parts else None
    _check(lib.nacho_spmm(ctypes.byref(m), pc, _ptr(B), B.stride(0), nb, _ptr(C), C.stride(0), _ptr(ws), need,
                          _stream(stream)))
    return C


def validate(A, stream=None):
    m = matrix(A)
    _check(lib.nacho_validate(ctypes.byref(m), _stream(stream)))


def launch_count(reset: bool = False) -> int:
    return lib.nacho_launch_count(int(reset))
