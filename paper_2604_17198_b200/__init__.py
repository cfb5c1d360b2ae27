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

NACHO_CSR, NACHO_DCSR, NACHO_COO = 0, 1, 2
NACHO_F32, NACHO_F64 = 0, 1
MAX_K = 8
STATUS = {0: "SUCCESS", 1: "INVALID_ARG", 2: "SHAPE", 3: "FORMAT", 4: "OVERFLOW", 5: "WORKSPACE", 6: "CUDA",
          7: "NCCL"}


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


class Tensor3C(ctypes.Structure):
    _fields_ = [("dtype", ctypes.c_int32), ("n0", ctypes.c_int64), ("n1", ctypes.c_int64), ("n2", ctypes.c_int64),
                ("nnz", ctypes.c_int64), ("n_slices", ctypes.c_int64), ("n_fibers", ctypes.c_int64),
                ("crd0", ctypes.c_void_p), ("pos1", ctypes.c_void_p), ("crd1", ctypes.c_void_p),
                ("pos2", ctypes.c_void_p), ("crd2", ctypes.c_void_p), ("val", ctypes.c_void_p)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is not built; run __graft_entry__.build() (no CPU fallback exists)")
    L = ctypes.CDLL(LIB_PATH)
    vp, i32, i64, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
    L.nacho_partition.argtypes = [vp, i32, i32, vp, vp]
    L.nacho_partition_slice.argtypes = [vp, i32, i32, i32, vp, vp]
    L.nacho_auto_partitions.argtypes = [vp, i32, i32]
    L.nacho_auto_partitions.restype = i32
    L.nacho_spadd_tile.argtypes = [i32]
    L.nacho_spadd_tile.restype = i32
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
    L.nacho_hadamard_k.argtypes = [vp, i32, vp, vp, vp, vp, vp, vp, sz, vp]
    L.nacho_inner_k_workspace_size.argtypes = [vp, i32, i32]
    L.nacho_inner_k_workspace_size.restype = sz
    L.nacho_inner_k.argtypes = [vp, i32, vp, vp, vp, sz, vp]
    L.nacho_dcsr_hadamard_workspace_size.argtypes = [vp, i32, i32]
    L.nacho_dcsr_hadamard_workspace_size.restype = sz
    L.nacho_dcsr_hadamard.argtypes = [vp, i32, vp, vp, vp, vp, vp, vp, vp, sz, vp]
    L.nacho_dcsr_spadd_k_workspace_size.argtypes = [vp, i32, i32]
    L.nacho_dcsr_spadd_k_workspace_size.restype = sz
    L.nacho_dcsr_spadd_k.argtypes = [vp, i32, vp, vp, vp, vp, vp, vp, vp, sz, vp]
    L.nacho_mixed_spadd_k_workspace_size.argtypes = [vp, i32, i32]
    L.nacho_mixed_spadd_k_workspace_size.restype = sz
    L.nacho_mixed_spadd_k.argtypes = [vp, i32, vp, vp, vp, vp, vp, vp, sz, vp]
    L.nacho_partition_csf.argtypes = [vp, i32, i32, vp, vp]
    L.nacho_csf_spadd_k_workspace_size.argtypes = [vp, i32, i32]
    L.nacho_csf_spadd_k_workspace_size.restype = sz
    L.nacho_csf_spadd_k.argtypes = [vp, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp, sz, vp]
    # ESC scatter kernels (esc.cu)
    L.nacho_spgemm_work_workspace_size.argtypes = [vp]
    L.nacho_spgemm_work_workspace_size.restype = sz
    L.nacho_spgemm_work.argtypes = [vp, vp, vp, vp, sz, vp]
    L.nacho_esc_auto_partitions.argtypes = [i64]
    L.nacho_esc_auto_partitions.restype = i32
    L.nacho_partition_esc.argtypes = [vp, vp, vp, i64, i32, vp, vp]
    L.nacho_spgemm_esc_workspace_size.argtypes = [vp, vp, i64]
    L.nacho_spgemm_esc_workspace_size.restype = sz
    L.nacho_spgemm_esc.argtypes = [vp, vp, vp, vp, i64, vp, vp, vp, vp, vp, sz, vp]
    L.nacho_sssmm_count_workspace_size.argtypes = [i32]
    L.nacho_sssmm_count_workspace_size.restype = sz
    L.nacho_sssmm_mask_bytes.argtypes = [i64, i32]
    L.nacho_sssmm_mask_bytes.restype = sz
    L.nacho_sssmm_esc_count.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp, sz, vp]
    L.nacho_sssmm_esc_workspace_size.argtypes = [vp, vp, i64]
    L.nacho_sssmm_esc_workspace_size.restype = sz
    L.nacho_sssmm_esc.argtypes = [vp, vp, vp, vp, vp, vp, vp, i64, vp, vp, vp, vp, vp, sz, vp]
    # multi-GPU (dist.cuh)
    L.nacho_dist_unique_id_size.restype = sz
    L.nacho_dist_unique_id.argtypes = [vp]
    L.nacho_dist_init.argtypes = [ctypes.POINTER(vp), vp, i32, i32]
    L.nacho_dist_destroy.argtypes = [vp]
    L.nacho_dist_broadcast.argtypes = [vp, vp, sz, i32, vp]
    L.nacho_device_cuts.argtypes = [vp, i32, vp, vp]
    L.nacho_shard_rows.argtypes = [vp, i64, i64, i64, i64, vp, vp]
    L.nacho_dist_seam.argtypes = [vp, i32, i32, i64, i32, i32, vp, vp]
    L.nacho_dist_spmv_workspace_size.argtypes = [vp, i32, i32]
    L.nacho_dist_spmv_workspace_size.restype = sz
    L.nacho_dist_spmv.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp, sz, vp]
    L.nacho_dist_spadd_workspace_size.argtypes = [i32]
    L.nacho_dist_spadd_workspace_size.restype = sz
    L.nacho_dist_spadd_gather.argtypes = [vp, vp, vp, vp, i32, vp, vp, vp, vp, vp, ctypes.POINTER(i64), vp, sz, vp]
    return L


lib = _load()

EXPORTS = ["nacho_partition", "nacho_partition_slice", "nacho_auto_partitions", "nacho_spadd_tile", "nacho_spmv_workspace_size", "nacho_spmv",
           "nacho_spadd_k_workspace_size", "nacho_spadd_k_count", "nacho_spadd_k_fill", "nacho_spadd_k",
           "nacho_spadd_k_staged_workspace_size", "nacho_spadd_k_staged",
           "nacho_spmm_workspace_size", "nacho_spmm", "nacho_validate", "nacho_last_error",
           "nacho_launch_count", "nacho_hadamard_k", "nacho_inner_k_workspace_size", "nacho_inner_k",
           "nacho_dcsr_hadamard_workspace_size", "nacho_dcsr_hadamard", "nacho_dcsr_spadd_k_workspace_size",
           "nacho_dcsr_spadd_k", "nacho_mixed_spadd_k_workspace_size", "nacho_mixed_spadd_k",
           "nacho_partition_csf", "nacho_csf_spadd_k_workspace_size", "nacho_csf_spadd_k",
           "nacho_spgemm_work_workspace_size", "nacho_spgemm_work", "nacho_esc_auto_partitions",
           "nacho_partition_esc", "nacho_spgemm_esc_workspace_size", "nacho_spgemm_esc",
           "nacho_sssmm_mask_bytes", "nacho_sssmm_count_workspace_size", "nacho_sssmm_esc_count", "nacho_sssmm_esc_workspace_size",
           "nacho_sssmm_esc",
           "nacho_dist_unique_id_size", "nacho_dist_unique_id", "nacho_dist_init",
           "nacho_dist_destroy", "nacho_dist_broadcast", "nacho_device_cuts", "nacho_shard_rows", "nacho_dist_seam",
           "nacho_dist_spmv_workspace_size", "nacho_dist_spmv", "nacho_dist_spadd_workspace_size",
           "nacho_dist_spadd_gather"]


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
    m.format = {"csr": NACHO_CSR, "dcsr": NACHO_DCSR, "coo": NACHO_COO}[A.format]
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


# ------------------------------------------------------------------ k-way intersection
def hadamard_k(ops, parts: Parts, z_pos=None, z_crd=None, z_val=None, part_off=None, ws=None, stream=None):
    """nacho_hadamard_k: Z = ops[0] (.) ... (.) ops[k-1] in one pass.  z_crd / z_val at capacity
    min_o nnz_o; nnz_Z = z_pos[-1]."""
    arr = _matrices(ops)
    dev = ops[0].pos.device
    cap = max(1, min(int(A.crd.shape[0]) for A in ops))
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
    _check(lib.nacho_hadamard_k(arr, len(ops), ctypes.byref(pc), _ptr(part_off), _ptr(z_pos), _ptr(z_crd), _ptr(z_val),
                                _ptr(ws), need, _stream(stream)))
    return z_pos, z_crd, z_val


def inner_k(ops, parts: Parts, out=None, ws=None, stream=None) -> torch.Tensor:
    """nacho_inner_k: sum over the intersection of the products (device double[1])."""
    arr = _matrices(ops)
    dev = ops[0].pos.device
    out = out if out is not None else torch.empty(1, dtype=torch.float64, device=dev)
    need = lib.nacho_inner_k_workspace_size(arr, len(ops), parts.P)
    if ws is None or ws.numel() < need:
        ws, _ = _workspace(need, dev)
    pc = parts.c()
    _check(lib.nacho_inner_k(arr, len(ops), ctypes.byref(pc), _ptr(out), _ptr(ws), need, _stream(stream)))
    return out


def dcsr_hadamard(ops, P: int = None, stream=None):
    """nacho_dcsr_hadamard: recursive partitioning (Alg. 2) + the DCSR Hadamard product.  Returns
    (parts, z_outer, z_pos, z_crd, z_val) trimmed to S surviving rows and nnz_Z (one host read)."""
    arr = _matrices(ops)
    dev = ops[0].pos.device
    k = len(ops)
    P = P or max(1, -(-sum(int(A.crd.shape[0]) for A in ops) // 512))
    parts = Parts(P, k, dev)
    cap_r = max(1, min(int(A.pos.shape[0]) - 1 for A in ops))
    cap_z = max(1, min(int(A.crd.shape[0]) for A in ops))
    counts = torch.zeros(2, dtype=torch.int64, device=dev)
    z_outer = torch.empty(cap_r, dtype=torch.int32, device=dev)
    z_pos = torch.zeros(cap_r + 1, dtype=torch.int64, device=dev)
    z_crd = torch.empty(cap_z, dtype=torch.int32, device=dev)
    z_val = torch.empty(cap_z, dtype=ops[0].val.dtype, device=dev)
    need = lib.nacho_dcsr_hadamard_workspace_size(arr, k, P)
    ws, _ = _workspace(need, dev)
    pc = parts.c()
    _check(lib.nacho_dcsr_hadamard(arr, k, ctypes.byref(pc), _ptr(counts), _ptr(z_outer), _ptr(z_pos), _ptr(z_crd),
                                   _ptr(z_val), _ptr(ws), need, _stream(stream)))
    S, nnz = (int(v) for v in counts.cpu().tolist())
    return parts, z_outer[:S], z_pos[:S + 1], z_crd[:nnz], z_val[:nnz]


def dcsr_spadd_k(ops, parts: Parts, stream=None):
    """nacho_dcsr_spadd_k: Z = sum of DCSR operands over `parts` (nacho_partition on the same operands).
    Returns (z_outer, z_pos, z_crd, z_val) trimmed to Z's stored rows and nnz_Z (one host read)."""
    arr = _matrices(ops)
    dev = ops[0].pos.device
    k = len(ops)
    cap_r = max(1, sum(int(A.pos.shape[0]) - 1 for A in ops))
    cap_z = max(1, sum(int(A.crd.shape[0]) for A in ops))
    counts = torch.zeros(2, dtype=torch.int64, device=dev)
    z_outer = torch.empty(cap_r, dtype=torch.int32, device=dev)
    z_pos = torch.zeros(cap_r + 1, dtype=torch.int64, device=dev)
    z_crd = torch.empty(cap_z, dtype=torch.int32, device=dev)
    z_val = torch.empty(cap_z, dtype=ops[0].val.dtype, device=dev)
    need = lib.nacho_dcsr_spadd_k_workspace_size(arr, k, parts.P)
    ws, _ = _workspace(need, dev)
    pc = parts.c()
    _check(lib.nacho_dcsr_spadd_k(arr, k, ctypes.byref(pc), _ptr(counts), _ptr(z_outer), _ptr(z_pos), _ptr(z_crd),
                                  _ptr(z_val), _ptr(ws), need, _stream(stream)))
    nr, nnz = (int(v) for v in counts.cpu().tolist())
    return z_outer[:nr], z_pos[:nr + 1], z_crd[:nnz], z_val[:nnz]


def mixed_spadd_k(ops, parts: Parts, stream=None):
    """nacho_mixed_spadd_k: Z (CSR) = sum of CSR / COO operands over `parts`.  Returns (z_pos, z_crd,
    z_val) trimmed to nnz_Z (one host read)."""
    arr = _matrices(ops)
    dev = ops[0].pos.device
    k = len(ops)
    cap = max(1, sum(int(A.crd.shape[0]) for A in ops))
    nnz = torch.zeros(1, dtype=torch.int64, device=dev)
    z_pos = torch.empty(ops[0].nrows + 1, dtype=torch.int64, device=dev)
    z_crd = torch.empty(cap, dtype=torch.int32, device=dev)
    z_val = torch.empty(cap, dtype=ops[0].val.dtype, device=dev)
    need = lib.nacho_mixed_spadd_k_workspace_size(arr, k, parts.P)
    ws, _ = _workspace(need, dev)
    pc = parts.c()
    _check(lib.nacho_mixed_spadd_k(arr, k, ctypes.byref(pc), _ptr(nnz), _ptr(z_pos), _ptr(z_crd), _ptr(z_val),
                                   _ptr(ws), need, _stream(stream)))
    n = int(nnz.item())
    return z_pos, z_crd[:n], z_val[:n]


# ------------------------------------------------------------------ third-order CSF (include/nacho.h, csf.cuh)
def tensor3(T) -> Tensor3C:
    """nacho_tensor3 descriptor of a workloads.Tensor3-like object on the device (no copies)."""
    for name, dt in (("crd0", torch.int32), ("pos1", torch.int64), ("crd1", torch.int32), ("pos2", torch.int64),
                     ("crd2", torch.int32)):
        _require(getattr(T, name), dt, name)
    if T.val.dtype not in (torch.float32, torch.float64):
        raise TypeError("val must be float32 or float64")
    _require(T.val, T.val.dtype, "val")
    s = Tensor3C()
    s.dtype = NACHO_F64 if T.val.dtype == torch.float64 else NACHO_F32
    s.n0, s.n1, s.n2 = (int(x) for x in T.shape)
    s.nnz, s.n_slices, s.n_fibers = int(T.crd2.shape[0]), int(T.crd0.shape[0]), int(T.crd1.shape[0])
    s.crd0, s.pos1, s.crd1 = T.crd0.data_ptr(), T.pos1.data_ptr(), T.crd1.data_ptr()
    s.pos2, s.crd2, s.val = T.pos2.data_ptr(), T.crd2.data_ptr(), T.val.data_ptr()
    return s


def _tensors3(ops):
    arr = (Tensor3C * len(ops))()
    for i, T in enumerate(ops):
        arr[i] = tensor3(T)
    return arr


def partition_csf(ops, P: int, stream=None) -> Parts:
    """nacho_partition_csf: Alg. 1 at d = 3 (row = x_i, row_pos = x_j, col = x_k)."""
    arr = _tensors3(ops)
    out = Parts(P, len(ops), ops[0].pos1.device)
    pc = out.c()
    _check(lib.nacho_partition_csf(arr, len(ops), P, ctypes.byref(pc), _stream(stream)))
    out.max_work = pc.max_work
    return out


def csf_spadd_k(ops, parts: Parts, stream=None):
    """nacho_csf_spadd_k: Z = sum of CSF operands over `parts`.  Returns (crd0, pos1, crd1, pos2, crd2,
    val) trimmed to Z's slices / fibers / nnz (one host read)."""
    arr = _tensors3(ops)
    dev = ops[0].pos1.device
    k = len(ops)
    cs = max(1, sum(int(T.crd0.shape[0]) for T in ops))
    cf = max(1, sum(int(T.crd1.shape[0]) for T in ops))
    ce = max(1, sum(int(T.crd2.shape[0]) for T in ops))
    counts = torch.zeros(3, dtype=torch.int64, device=dev)
    z = [torch.empty(cs, dtype=torch.int32, device=dev), torch.zeros(cs + 1, dtype=torch.int64, device=dev),
         torch.empty(cf, dtype=torch.int32, device=dev), torch.zeros(cf + 1, dtype=torch.int64, device=dev),
         torch.empty(ce, dtype=torch.int32, device=dev), torch.empty(ce, dtype=ops[0].val.dtype, device=dev)]
    need = lib.nacho_csf_spadd_k_workspace_size(arr, k, parts.P)
    ws, _ = _workspace(need, dev)
    pc = parts.c()
    _check(lib.nacho_csf_spadd_k(arr, k, ctypes.byref(pc), _ptr(counts), *(_ptr(x) for x in z), _ptr(ws), need,
                                 _stream(stream)))
    ns, nf, ne = (int(v) for v in counts.cpu().tolist())
    return z[0][:ns], z[1][:ns + 1], z[2][:nf], z[3][:nf + 1], z[4][:ne], z[5][:ne]


# ------------------------------------------------------------------ ESC scatter kernels (esc.cu)
def spgemm_work(A, B, W=None, stream=None):
    """nacho_spgemm_work: W[q] = sum_{q' < q} nnz(B_{A.crd[q']}) (device int64[nnz(A)+1])."""
    a, b = matrix(A), matrix(B)
    dev = A.pos.device
    if W is None:
        W = torch.empty(A.nnz + 1, dtype=torch.int64, device=dev)
    need = lib.nacho_spgemm_work_workspace_size(ctypes.byref(a))
    ws, _ = _workspace(need, dev)
    _check(lib.nacho_spgemm_work(ctypes.byref(a), ctypes.byref(b), _ptr(W), _ptr(ws), need, _stream(stream)))
    return W


def partition_esc(A, B, W, qstar: int, P: int, out: Parts = None, stream=None) -> Parts:
    """nacho_partition_esc: b_p locates product number Q_p of the expansion (k = 2 record)."""
    a, b = matrix(A), matrix(B)
    out = out or Parts(P, 2, A.pos.device)
    pc = out.c()
    _check(lib.nacho_partition_esc(ctypes.byref(a), ctypes.byref(b), _ptr(W), qstar, P, ctypes.byref(pc),
                                   _stream(stream)))
    out.max_work = pc.max_work
    return out


def esc_auto_partitions(qstar: int) -> int:
    return lib.nacho_esc_auto_partitions(qstar)


def spgemm_esc(A, B, W, parts: Parts, qstar: int, c_pos=None, c_crd=None, c_val=None, nnz_c=None, ws=None,
               stream=None):
    """nacho_spgemm_esc: C = A B by expand - sort - contract.  Returns (c_pos, c_crd, c_val, nnz_c) with
    c_crd / c_val of capacity Q* (nnz_c a device int64[1]; the caller trims)."""
    a, b = matrix(A), matrix(B)
    dev = A.pos.device
    if c_pos is None:
        c_pos = torch.empty(A.nrows + 1, dtype=torch.int64, device=dev)
        c_crd = torch.empty(max(qstar, 1), dtype=torch.int32, device=dev)
        c_val = torch.empty(max(qstar, 1), dtype=A.val.dtype, device=dev)
        nnz_c = torch.empty(1, dtype=torch.int64, device=dev)
    need = lib.nacho_spgemm_esc_workspace_size(ctypes.byref(a), ctypes.byref(b), qstar)
    if ws is None or ws.numel() < need:
        ws, _ = _workspace(need, dev)
    pc = parts.c()
    _check(lib.nacho_spgemm_esc(ctypes.byref(a), ctypes.byref(b), _ptr(W), ctypes.byref(pc), qstar, _ptr(c_pos),
                                _ptr(c_crd), _ptr(c_val), _ptr(nnz_c), _ptr(ws), need, _stream(stream)))
    return c_pos, c_crd, c_val, nnz_c


def spgemm(A, B, P: int = None, stream=None):
    """C = A B (ESC): work -> host reads Q* -> partition -> expand / sort / contract -> trimmed C."""
    W = spgemm_work(A, B, stream=stream)
    qstar = int(W[-1].item())
    P = P or esc_auto_partitions(qstar)
    parts = partition_esc(A, B, W, qstar, P, stream=stream)
    c_pos, c_crd, c_val, nnz_c = spgemm_esc(A, B, W, parts, qstar, stream=stream)
    n = int(nnz_c.item())
    return c_pos, c_crd[:n], c_val[:n]


def sssmm(S, A, B, P: int = None, stream=None):
    """Z = S (.) (A B) (ESC over the sampled expansion): work -> partition -> count -> host reads the kept
    count -> fill / sort / contract -> trimmed Z."""
    s, a, b = matrix(S), matrix(A), matrix(B)
    dev = A.pos.device
    W = spgemm_work(A, B, stream=stream)
    qstar = int(W[-1].item())
    P = P or esc_auto_partitions(qstar)
    parts = partition_esc(A, B, W, qstar, P, stream=stream)
    part_off = torch.empty(P + 1, dtype=torch.int64, device=dev)
    mask = torch.empty(lib.nacho_sssmm_mask_bytes(qstar, P), dtype=torch.uint8, device=dev)
    need = lib.nacho_sssmm_count_workspace_size(P)
    ws, _ = _workspace(need, dev)
    pc = parts.c()
    _check(lib.nacho_sssmm_esc_count(ctypes.byref(s), ctypes.byref(a), ctypes.byref(b), _ptr(W), ctypes.byref(pc),
                                     _ptr(part_off), _ptr(mask), _ptr(ws), need, _stream(stream)))
    n_kept = int(part_off[-1].item())
    z_pos = torch.empty(A.nrows + 1, dtype=torch.int64, device=dev)
    z_crd = torch.empty(max(n_kept, 1), dtype=torch.int32, device=dev)
    z_val = torch.empty(max(n_kept, 1), dtype=A.val.dtype, device=dev)
    nnz_z = torch.empty(1, dtype=torch.int64, device=dev)
    need = lib.nacho_sssmm_esc_workspace_size(ctypes.byref(a), ctypes.byref(b), n_kept)
    ws, _ = _workspace(need, dev)
    _check(lib.nacho_sssmm_esc(ctypes.byref(s), ctypes.byref(a), ctypes.byref(b), _ptr(W), ctypes.byref(pc),
                               _ptr(part_off), _ptr(mask), n_kept, _ptr(z_pos), _ptr(z_crd), _ptr(z_val), _ptr(nnz_z),
                               _ptr(ws), need, _stream(stream)))
    n = int(nnz_z.item())
    return z_pos, z_crd[:n], z_val[:n]


# ------------------------------------------------------------------ multi-GPU (include/nacho.h, dist.cuh)
def device_cuts(A, D: int, stream=None) -> torch.Tensor:
    """nacho_device_cuts: the D+1 device cuts (row, position) of Alg. 1 with P = D on one CSR operand
    (reads only A.pos).  Returns a device int64 tensor [D+1, 2]."""
    cuts = torch.empty((D + 1, 2), dtype=torch.int64, device=A.pos.device)
    m = matrix_pos_only(A)
    _check(lib.nacho_device_cuts(ctypes.byref(m), D, _ptr(cuts), _stream(stream)))
    return cuts


def matrix_pos_only(A) -> Matrix:
    """Descriptor of an operand of which only pos (and the sizes) are resident (device cuts)."""
    _require(A.pos, torch.int64, "pos")
    m = Matrix()
    m.format, m.dtype = NACHO_CSR, NACHO_F32
    m.nrows, m.ncols = int(A.nrows), int(A.ncols)
    m.nouter = int(A.pos.shape[0]) - 1
    m.nnz = int(A.nnz)
    m.pos = A.pos.data_ptr()
    return m


def shard_rows(pos: torch.Tensor, row_lo: int, nloc: int, pos_lo: int, pos_hi: int, stream=None) -> torch.Tensor:
    """nacho_shard_rows: rebased row pointers of rows [row_lo, row_lo + nloc) within [pos_lo, pos_hi)."""
    out = torch.empty(nloc + 1, dtype=torch.int64, device=pos.device)
    _check(lib.nacho_shard_rows(_ptr(pos), row_lo, nloc, pos_lo, pos_hi, _ptr(out), _stream(stream)))
    return out


def dist_seam(carries: torch.Tensor, D: int, d: int, row_lo: int, owns_first: bool, y_local: torch.Tensor, stream=None):
    """nacho_dist_seam: add the seam carries of devices < d ending in row_lo to y_local[0]."""
    dt = NACHO_F64 if y_local.dtype == torch.float64 else NACHO_F32
    _check(lib.nacho_dist_seam(_ptr(carries), D, d, row_lo, int(bool(owns_first)), dt, _ptr(y_local), _stream(stream)))


class Dist:
    """nacho_dist communicator (NCCL inside libnacho.so).  torch.distributed only moves the unique id."""

    def __init__(self, nranks: int, rank: int, id_bytes: bytes):
        self.nranks, self.rank = nranks, rank
        h = ctypes.c_void_p()
        buf = ctypes.create_string_buffer(id_bytes, len(id_bytes))
        _check(lib.nacho_dist_init(ctypes.byref(h), buf, nranks, rank))
        self.h = h

    @staticmethod
    def unique_id() -> bytes:
        n = lib.nacho_dist_unique_id_size()
        buf = ctypes.create_string_buffer(n)
        _check(lib.nacho_dist_unique_id(buf))
        return buf.raw

    @classmethod
    def from_process_group(cls):
        """Rank 0 creates the NCCL unique id; a torch.distributed broadcast hands it to every rank."""
        import torch.distributed as td
        n = lib.nacho_dist_unique_id_size()
        obj = [cls.unique_id() if td.get_rank() == 0 else None]
        td.broadcast_object_list(obj, src=0)
        assert len(obj[0]) == n
        return cls(td.get_world_size(), td.get_rank(), obj[0])

    def broadcast(self, t: torch.Tensor, root: int = 0, stream=None):
        _check(lib.nacho_dist_broadcast(self.h, _ptr(t), t.numel() * t.element_size(), root, _stream(stream)))

    def spmv(self, A_local, parts, x, y_local, cut_rows, y_full=None, ws=None, stream=None):
        """nacho_dist_spmv: local partitions + seam carries (+ gather of the owned y segments)."""
        m = matrix(A_local)
        P = parts.P if parts is not None else 0
        need = lib.nacho_dist_spmv_workspace_size(ctypes.byref(m), P, self.nranks)
        if ws is None or ws.numel() < need:
            ws, _ = _workspace(need, x.device)
        cr = (ctypes.c_int64 * (self.nranks + 1))(*[int(c) for c in cut_rows])
        pc = ctypes.byref(parts.c()) if parts is not None else None
        _check(lib.nacho_dist_spmv(self.h, ctypes.byref(m), pc, _ptr(x), _ptr(y_local), cr, _ptr(y_full), _ptr(ws),
                                   need, _stream(stream)))
        return y_local

    def spadd_gather(self, z_pos_local, z_crd_local, z_val_local, nnz_local, cut_rows, z_pos, z_crd, z_val, ws=None,
                     stream=None):
        """nacho_dist_spadd_gather: global offsets from the device union sizes, Z segments gathered."""
        need = lib.nacho_dist_spadd_workspace_size(self.nranks)
        if ws is None or ws.numel() < need:
            ws, _ = _workspace(need, z_pos.device)
        cr = (ctypes.c_int64 * (self.nranks + 1))(*[int(c) for c in cut_rows])
        tot = ctypes.c_int64(0)
        dt = NACHO_F64 if z_val_local.dtype == torch.float64 else NACHO_F32
        _check(lib.nacho_dist_spadd_gather(self.h, _ptr(z_pos_local), _ptr(z_crd_local), _ptr(z_val_local), dt,
                                           _ptr(nnz_local), cr, _ptr(z_pos), _ptr(z_crd), _ptr(z_val),
                                           ctypes.byref(tot), _ptr(ws), need, _stream(stream)))
        return int(tot.value)

    def close(self):
        if self.h:
            _check(lib.nacho_dist_destroy(self.h))
            self.h = None
