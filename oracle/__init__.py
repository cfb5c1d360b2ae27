"""ctypes front-end of the CPU oracle (oracle.c) -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may import
this package.  It never imports the CUDA product package and the product never imports it.
Functions accept any object with the attributes of workloads.SparseMatrix holding numpy arrays.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")


def build(force: bool = False) -> str:
    src = os.path.join(HERE, "oracle.c")
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-Wall", "-shared", "-fPIC", "-o", LIB_PATH, src])
    return LIB_PATH


class _Matrix(ctypes.Structure):
    _fields_ = [("format", ctypes.c_int32), ("dtype", ctypes.c_int32),
                ("nrows", ctypes.c_int64), ("ncols", ctypes.c_int64), ("nnz", ctypes.c_int64),
                ("nouter", ctypes.c_int64), ("outer_crd", ctypes.c_void_p), ("pos", ctypes.c_void_p),
                ("crd", ctypes.c_void_p), ("val", ctypes.c_void_p)]


class _Parts(ctypes.Structure):
    _fields_ = [("P", ctypes.c_int32), ("k", ctypes.c_int32), ("query", ctypes.c_void_p),
                ("row", ctypes.c_void_p), ("row_pos", ctypes.c_void_p), ("col", ctypes.c_void_p),
                ("pos", ctypes.c_void_p)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        L = _lib
        vp = ctypes.c_void_p
        L.oracle_validate.argtypes = [vp]
        L.oracle_total_cost.argtypes = [ctypes.c_int32, vp]
        L.oracle_total_cost.restype = ctypes.c_int64
        L.oracle_queries.argtypes = [ctypes.c_int64, ctypes.c_int32, vp]
        L.oracle_partition_rank.argtypes = [ctypes.c_int32, vp, ctypes.c_int32, vp]
        L.oracle_partition_alg1.argtypes = [ctypes.c_int32, vp, ctypes.c_int32, vp, vp]
        L.oracle_lb_search.argtypes = [vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64]
        L.oracle_lb_search.restype = ctypes.c_int64
        L.oracle_spmv.argtypes = [vp, vp, vp]
        L.oracle_spmm.argtypes = [vp, vp, ctypes.c_int64, ctypes.c_int32, vp, ctypes.c_int64]
        L.oracle_spadd_k.argtypes = [ctypes.c_int32, vp, vp, vp, vp, ctypes.c_int64]
        L.oracle_spadd_k.restype = ctypes.c_int64
        L.oracle_spadd_counts.argtypes = [ctypes.c_int32, vp, vp, vp]
        L.oracle_hadamard_k.argtypes = [ctypes.c_int32, vp, vp, vp, vp, ctypes.c_int64]
        L.oracle_hadamard_k.restype = ctypes.c_int64
        L.oracle_hadamard_counts.argtypes = [ctypes.c_int32, vp, vp, vp]
        L.oracle_inner_k.argtypes = [ctypes.c_int32, vp, vp]
        i64 = ctypes.c_int64
        L.oracle_dcsr_rows_intersect.argtypes = [ctypes.c_int32, vp, vp, vp, vp, i64]
        L.oracle_dcsr_rows_intersect.restype = i64
        L.oracle_exclusive_prefix.argtypes = [vp, i64, vp]
        L.oracle_partition_remapped.argtypes = [ctypes.c_int32, vp, i64, vp, vp, i64, vp, ctypes.c_int32, vp]
        L.oracle_dcsr_hadamard.argtypes = [ctypes.c_int32, vp, i64, vp, i64, vp, vp, vp, i64]
        L.oracle_dcsr_hadamard.restype = i64
        L.oracle_dcsr_spadd_k.argtypes = [ctypes.c_int32, vp, vp, vp, vp, vp, vp, i64, i64]
        L.oracle_dcsr_spadd_k.restype = i64
        L.oracle_dcsr_spadd_counts.argtypes = [ctypes.c_int32, vp, vp, vp, vp]
        L.oracle_mixed_spadd_k.argtypes = [ctypes.c_int32, vp, vp, vp, vp, i64]
        L.oracle_mixed_spadd_k.restype = i64
        L.oracle_csf_cost.argtypes = [ctypes.c_int32, vp, i64, i64, i64, vp, vp, vp]
        L.oracle_csf_partition_rank.argtypes = [ctypes.c_int32, vp, ctypes.c_int32, vp]
        L.oracle_csf_spadd_k.argtypes = [ctypes.c_int32, vp, vp, vp, vp, vp, vp, vp, i64, i64, i64, vp]
        L.oracle_csf_spadd_k.restype = i64
        L.oracle_spgemm_work.argtypes = [vp, vp, vp]
        L.oracle_spgemm_work.restype = i64
        L.oracle_esc_partition.argtypes = [vp, vp, ctypes.c_int32, vp]
        L.oracle_spgemm.argtypes = [vp, vp, vp, vp, vp, i64]
        L.oracle_spgemm.restype = i64
        L.oracle_sssmm.argtypes = [vp, vp, vp, vp, vp, vp, i64]
        L.oracle_sssmm.restype = i64
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data


def _matrices(ops):
    keep = []
    arr = (_Matrix * len(ops))()
    for i, A in enumerate(ops):
        pos = np.ascontiguousarray(A.pos, dtype=np.int64)
        crd = np.ascontiguousarray(A.crd, dtype=np.int32)
        val = np.ascontiguousarray(A.val)
        outer = None if A.outer_crd is None else np.ascontiguousarray(A.outer_crd, dtype=np.int32)
        keep += [pos, crd, val, outer]
        arr[i].format = {"csr": 0, "dcsr": 1, "coo": 2}[A.format]
        arr[i].dtype = 1 if val.dtype == np.float64 else 0
        arr[i].nrows, arr[i].ncols = A.nrows, A.ncols
        arr[i].nnz = crd.shape[0]
        arr[i].nouter = pos.shape[0] - 1
        arr[i].outer_crd, arr[i].pos, arr[i].crd, arr[i].val = _p(outer), _p(pos), _p(crd), _p(val)
    return arr, keep


class Parts:
    """Partition record (Listing 7 `Parts`): SoA arrays of length P+1."""

    def __init__(self, P, k):
        self.P, self.k = P, k
        self.query = np.zeros(P + 1, np.int64)
        self.row = np.zeros(P + 1, np.int64)
        self.row_pos = np.zeros(P + 1, np.int64)
        self.col = np.zeros(P + 1, np.int32)
        self.pos = np.zeros((P + 1) * k, np.int64)

    def c(self):
        s = _Parts()
        s.P, s.k = self.P, self.k
        s.query, s.row, s.row_pos, s.col, s.pos = (_p(self.query), _p(self.row), _p(self.row_pos),
                                                   _p(self.col), _p(self.pos))
        return s

    def pos2(self):
        return self.pos.reshape(self.P + 1, self.k)


def validate(A) -> int:
    arr, keep = _matrices([A])
    return lib().oracle_validate(ctypes.byref(arr[0]))


def total_cost(ops) -> int:
    arr, keep = _matrices(ops)
    return lib().oracle_total_cost(len(ops), arr)


def queries(qstar: int, P: int) -> np.ndarray:
    Q = np.zeros(P + 1, np.int64)
    lib().oracle_queries(qstar, P, _p(Q))
    return Q


def partition_rank(ops, P) -> Parts:
    arr, keep = _matrices(ops)
    out = Parts(P, len(ops))
    s = out.c()
    if lib().oracle_partition_rank(len(ops), arr, P, ctypes.byref(s)) != 0:
        raise ValueError("oracle_partition_rank failed")
    return out


def partition_alg1(ops, P, with_probes=False):
    arr, keep = _matrices(ops)
    out = Parts(P, len(ops))
    probes = np.zeros(P + 1, np.int64)
    s = out.c()
    if lib().oracle_partition_alg1(len(ops), arr, P, ctypes.byref(s), _p(probes)) != 0:
        raise ValueError("oracle_partition_alg1 failed")
    return (out, probes) if with_probes else out


def lb_search(crd, lo, hi, x) -> int:
    crd = np.ascontiguousarray(crd, dtype=np.int32)
    return lib().oracle_lb_search(_p(crd) if crd.size else None, lo, hi, x)


def spmv(A, x) -> np.ndarray:
    arr, keep = _matrices([A])
    x = np.ascontiguousarray(x, dtype=A.val.dtype)
    y = np.zeros(A.pos.shape[0] - 1, dtype=A.val.dtype)
    lib().oracle_spmv(ctypes.byref(arr[0]), _p(x), _p(y))
    return y


def spmm(A, B) -> np.ndarray:
    arr, keep = _matrices([A])
    B = np.ascontiguousarray(B, dtype=A.val.dtype)
    nb = B.shape[1]
    C = np.zeros((A.nrows, nb), dtype=A.val.dtype)
    if lib().oracle_spmm(ctypes.byref(arr[0]), _p(B), nb, nb, _p(C), nb) != 0:
        raise ValueError("oracle_spmm: CSR only")
    return C


def spadd_k(ops):
    """Returns (z_pos, z_crd, z_val) of the k-way structural union with left-fold values."""
    arr, keep = _matrices(ops)
    cap = int(sum(int(A.crd.shape[0]) for A in ops))
    M = ops[0].nrows
    z_pos = np.zeros(M + 1, np.int64)
    z_crd = np.zeros(max(cap, 1), np.int32)
    z_val = np.zeros(max(cap, 1), dtype=ops[0].val.dtype)
    n = lib().oracle_spadd_k(len(ops), arr, _p(z_pos), _p(z_crd), _p(z_val), cap)
    if n < 0:
        raise ValueError("oracle_spadd_k failed")
    return z_pos, z_crd[:n].copy(), z_val[:n].copy()


def spadd_counts(ops, parts: Parts) -> np.ndarray:
    arr, keep = _matrices(ops)
    cnt = np.zeros(parts.P, np.int64)
    s = parts.c()
    if lib().oracle_spadd_counts(len(ops), arr, ctypes.byref(s), _p(cnt)) != 0:
        raise ValueError("oracle_spadd_counts failed")
    return cnt


def hadamard_k(ops):
    """(z_pos, z_crd, z_val) of the k-way structural intersection (Listing 1 per row), product values."""
    arr, keep = _matrices(ops)
    cap = int(min(int(A.crd.shape[0]) for A in ops))
    M = ops[0].nrows
    z_pos = np.zeros(M + 1, np.int64)
    z_crd = np.zeros(max(cap, 1), np.int32)
    z_val = np.zeros(max(cap, 1), dtype=ops[0].val.dtype)
    n = lib().oracle_hadamard_k(len(ops), arr, _p(z_pos), _p(z_crd), _p(z_val), cap)
    if n < 0:
        raise ValueError("oracle_hadamard_k failed")
    return z_pos, z_crd[:n].copy(), z_val[:n].copy()


def hadamard_counts(ops, parts: Parts) -> np.ndarray:
    arr, keep = _matrices(ops)
    cnt = np.zeros(parts.P, np.int64)
    s = parts.c()
    if lib().oracle_hadamard_counts(len(ops), arr, ctypes.byref(s), _p(cnt)) != 0:
        raise ValueError("oracle_hadamard_counts failed")
    return cnt


def inner_k(ops) -> float:
    arr, keep = _matrices(ops)
    out = ctypes.c_double(0.0)
    if lib().oracle_inner_k(len(ops), arr, ctypes.byref(out)) != 0:
        raise ValueError("oracle_inner_k failed")
    return float(out.value)


class Remap:
    """Lines 2-4 of Listing emul-dcsr2-rewritten: surviving rows, T, T', outer positions ip[o][s]."""

    def __init__(self, rows, T, Tp, ip):
        self.rows, self.T, self.Tp, self.ip = rows, T, Tp, ip
        self.S = len(rows)


def dcsr_rows_intersect(ops) -> Remap:
    arr, keep = _matrices(ops)
    k = len(ops)
    cap = max(1, min(int(A.nouter) for A in ops))
    rows = np.zeros(cap, np.int64)
    T = np.zeros(cap, np.int64)
    ip = np.zeros(k * cap, np.int64)
    S = lib().oracle_dcsr_rows_intersect(k, arr, _p(rows), _p(T), _p(ip), cap)
    if S < 0:
        raise ValueError("oracle_dcsr_rows_intersect failed (DCSR operands only)")
    Tp = np.zeros(S + 1, np.int64)
    lib().oracle_exclusive_prefix(_p(T), S, _p(Tp))
    ipm = ip.reshape(k, cap)[:, :S].copy()
    return Remap(rows[:S].copy(), T[:S].copy(), Tp, ipm)


def _ip_flat(rm):
    k = rm.ip.shape[0]
    cap = max(1, rm.S)
    flat = np.zeros(k * cap, np.int64)
    for o in range(k):
        flat[o * cap:o * cap + rm.S] = rm.ip[o]
    return flat, cap


def partition_remapped(ops, rm: Remap, P) -> Parts:
    arr, keep = _matrices(ops)
    out = Parts(P, len(ops))
    flat, cap = _ip_flat(rm)
    rows = np.ascontiguousarray(rm.rows, np.int64) if rm.S else np.zeros(1, np.int64)
    s = out.c()
    if lib().oracle_partition_remapped(len(ops), arr, rm.S, _p(rows), _p(flat), cap, _p(rm.Tp), P,
                                       ctypes.byref(s)) != 0:
        raise ValueError("oracle_partition_remapped failed")
    return out


def dcsr_hadamard(ops, rm: Remap):
    """(z_outer, z_pos, z_crd, z_val): Z over the surviving rows (every one stored, R21)."""
    arr, keep = _matrices(ops)
    flat, cap = _ip_flat(rm)
    zcap = max(1, min(int(A.crd.shape[0]) for A in ops))
    z_pos = np.zeros(rm.S + 1, np.int64)
    z_crd = np.zeros(zcap, np.int32)
    z_val = np.zeros(zcap, dtype=ops[0].val.dtype)
    n = lib().oracle_dcsr_hadamard(len(ops), arr, rm.S, _p(flat), cap, _p(z_pos), _p(z_crd), _p(z_val), zcap)
    if n < 0:
        raise ValueError("oracle_dcsr_hadamard failed")
    return rm.rows.astype(np.int32), z_pos, z_crd[:n].copy(), z_val[:n].copy()


def dcsr_spadd_k(ops):
    """(z_outer, z_pos, z_crd, z_val) of the DCSR k-way union (Listing 2)."""
    arr, keep = _matrices(ops)
    rcap = max(1, sum(int(A.nouter) for A in ops))
    zcap = max(1, sum(int(A.crd.shape[0]) for A in ops))
    z_outer = np.zeros(rcap, np.int32)
    z_pos = np.zeros(rcap + 1, np.int64)
    z_crd = np.zeros(zcap, np.int32)
    z_val = np.zeros(zcap, dtype=ops[0].val.dtype)
    nr = ctypes.c_int64(0)
    n = lib().oracle_dcsr_spadd_k(len(ops), arr, _p(z_outer), _p(z_pos), _p(z_crd), _p(z_val), ctypes.byref(nr),
                                  rcap, zcap)
    if n < 0:
        raise ValueError("oracle_dcsr_spadd_k failed (DCSR operands only)")
    r = nr.value
    return z_outer[:r].copy(), z_pos[:r + 1].copy(), z_crd[:n].copy(), z_val[:n].copy()


def dcsr_spadd_counts(ops, parts: Parts):
    arr, keep = _matrices(ops)
    ent = np.zeros(parts.P, np.int64)
    rows = np.zeros(parts.P, np.int64)
    s = parts.c()
    if lib().oracle_dcsr_spadd_counts(len(ops), arr, ctypes.byref(s), _p(ent), _p(rows)) != 0:
        raise ValueError("oracle_dcsr_spadd_counts failed")
    return ent, rows


def mixed_spadd_k(ops):
    """(z_pos, z_crd, z_val): CSR Z of CSR and COO operands mixed (the union per row, left fold)."""
    arr, keep = _matrices(ops)
    cap = max(1, sum(int(A.crd.shape[0]) for A in ops))
    z_pos = np.zeros(ops[0].nrows + 1, np.int64)
    z_crd = np.zeros(cap, np.int32)
    z_val = np.zeros(cap, dtype=ops[0].val.dtype)
    n = lib().oracle_mixed_spadd_k(len(ops), arr, _p(z_pos), _p(z_crd), _p(z_val), cap)
    if n < 0:
        raise ValueError("oracle_mixed_spadd_k failed (CSR / COO operands only)")
    return z_pos, z_crd[:n].copy(), z_val[:n].copy()


# ------------------------------------------------------------------ third-order CSF
class _Tensor3(ctypes.Structure):
    _fields_ = [("dtype", ctypes.c_int32), ("n0", ctypes.c_int64), ("n1", ctypes.c_int64), ("n2", ctypes.c_int64),
                ("nnz", ctypes.c_int64), ("n_slices", ctypes.c_int64), ("n_fibers", ctypes.c_int64),
                ("crd0", ctypes.c_void_p), ("pos1", ctypes.c_void_p), ("crd1", ctypes.c_void_p),
                ("pos2", ctypes.c_void_p), ("crd2", ctypes.c_void_p), ("val", ctypes.c_void_p)]


def _tensors(ops):
    keep = []
    arr = (_Tensor3 * len(ops))()
    for i, T in enumerate(ops):
        a = [np.ascontiguousarray(x, dtype=d) for x, d in
             ((T.crd0, np.int32), (T.pos1, np.int64), (T.crd1, np.int32), (T.pos2, np.int64), (T.crd2, np.int32))]
        val = np.ascontiguousarray(T.val)
        keep += a + [val]
        arr[i].dtype = 1 if val.dtype == np.float64 else 0
        arr[i].n0, arr[i].n1, arr[i].n2 = T.shape
        arr[i].nnz, arr[i].n_slices, arr[i].n_fibers = a[4].shape[0], a[0].shape[0], a[2].shape[0]
        arr[i].crd0, arr[i].pos1, arr[i].crd1, arr[i].pos2, arr[i].crd2 = (_p(x) for x in a)
        arr[i].val = _p(val)
    return arr, keep


def csf_cost(ops, xi, xj, xk):
    arr, keep = _tensors(ops)
    c = [ctypes.c_int64(0) for _ in range(3)]
    lib().oracle_csf_cost(len(ops), arr, xi, xj, xk, *(ctypes.byref(x) for x in c))
    return tuple(int(x.value) for x in c)


def csf_partition_rank(ops, P) -> Parts:
    arr, keep = _tensors(ops)
    out = Parts(P, len(ops))
    s = out.c()
    if lib().oracle_csf_partition_rank(len(ops), arr, P, ctypes.byref(s)) != 0:
        raise ValueError("oracle_csf_partition_rank failed")
    return out


def csf_spadd_k(ops):
    """(crd0, pos1, crd1, pos2, crd2, val) of the 3-level union Z = sum_o ops[o] in CSF."""
    arr, keep = _tensors(ops)
    cs = max(1, sum(len(T.crd0) for T in ops))
    cf = max(1, sum(len(T.crd1) for T in ops))
    ce = max(1, sum(len(T.crd2) for T in ops))
    z = [np.zeros(cs, np.int32), np.zeros(cs + 1, np.int64), np.zeros(cf, np.int32), np.zeros(cf + 1, np.int64),
         np.zeros(ce, np.int32), np.zeros(ce, dtype=np.asarray(ops[0].val).dtype)]
    counts = np.zeros(3, np.int64)
    n = lib().oracle_csf_spadd_k(len(ops), arr, *(_p(x) for x in z), cs, cf, ce, _p(counts))
    if n < 0:
        raise ValueError("oracle_csf_spadd_k overflow")
    ns, nf, ne = (int(x) for x in counts)
    return z[0][:ns], z[1][:ns + 1], z[2][:nf], z[3][:nf + 1], z[4][:ne], z[5][:ne]



# ------------------------------------------------------------------ ESC scatter kernels
def spgemm_work(A, B) -> np.ndarray:
    """W[q] = sum_{q' < q} nnz(B_{A.crd[q']}) for q in [0, nnz(A)] (Listing 6's broadcast-scaled cost)."""
    arr, keep = _matrices([A, B])
    W = np.zeros(A.crd.shape[0] + 1, np.int64)
    if lib().oracle_spgemm_work(ctypes.byref(arr[0]), ctypes.byref(arr[1]), _p(W)) < 0:
        raise ValueError("oracle_spgemm_work: CSR x CSR with A.ncols == B.nrows")
    return W


def esc_partition(A, B, P) -> Parts:
    """Boundaries of the expansion: b_p = location of product number Q_p (pos = (A position, B position))."""
    arr, keep = _matrices([A, B])
    out = Parts(P, 2)
    s = out.c()
    if lib().oracle_esc_partition(ctypes.byref(arr[0]), ctypes.byref(arr[1]), P, ctypes.byref(s)) != 0:
        raise ValueError("oracle_esc_partition failed")
    return out


def spgemm(A, B):
    """(c_pos, c_crd, c_val) of C = A B: structural product, left fold over k ascending."""
    arr, keep = _matrices([A, B])
    W = spgemm_work(A, B)
    cap = max(int(W[-1]), 1)
    c_pos = np.zeros(A.nrows + 1, np.int64)
    c_crd = np.zeros(cap, np.int32)
    c_val = np.zeros(cap, dtype=A.val.dtype)
    n = lib().oracle_spgemm(ctypes.byref(arr[0]), ctypes.byref(arr[1]), _p(c_pos), _p(c_crd), _p(c_val), cap)
    if n < 0:
        raise ValueError("oracle_spgemm failed")
    return c_pos, c_crd[:n].copy(), c_val[:n].copy()


def sssmm(S, A, B):
    """(z_pos, z_crd, z_val) of Z = S (.) (A B): Z_ij = S_ij * C_ij on the coordinates S and C both store."""
    arr, keep = _matrices([S, A, B])
    cap = max(int(S.crd.shape[0]), 1)
    z_pos = np.zeros(S.nrows + 1, np.int64)
    z_crd = np.zeros(cap, np.int32)
    z_val = np.zeros(cap, dtype=S.val.dtype)
    n = lib().oracle_sssmm(ctypes.byref(arr[0]), ctypes.byref(arr[1]), ctypes.byref(arr[2]), _p(z_pos), _p(z_crd),
                           _p(z_val), cap)
    if n < 0:
        raise ValueError("oracle_sssmm failed")
    return z_pos, z_crd[:n].copy(), z_val[:n].copy()
