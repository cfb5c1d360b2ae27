"""The C-ABI library loads on a CPU-only box and exports every symbol include/nacho.h declares;
host-only entry points (sizes, auto partition counts) behave as documented."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "nacho.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(nacho_\w+)\s*\(", src)))


def test_header_symbols_exported():
    import paper_2604_17198_b200 as N
    names = _declared()
    assert len(names) >= 12
    for n in names:
        assert hasattr(N.lib, n), f"libnacho.so does not export {n}"
    assert sorted(N.EXPORTS) == names


def test_header_compiles_as_c():
    import subprocess
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "t.c")
        open(c, "w").write('#include "nacho.h"\nint main(void){return (int)sizeof(nacho_matrix);}\n')
        subprocess.check_call(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                               "-c", c, "-o", os.path.join(d, "t.o")])


def _desc(nnz, dtype=0, nrows=100, ncols=100):
    import paper_2604_17198_b200 as N
    m = N.Matrix()
    m.format, m.dtype, m.nrows, m.ncols, m.nnz, m.nouter = 0, dtype, nrows, ncols, nnz, nrows
    return m


def test_auto_partitions_and_workspace_host_only():
    import paper_2604_17198_b200 as N
    L = N.lib
    # SpMV tiles: 256 threads x 16 (fp32) / x 8 (fp64) positions per partition
    for nnz, dt, tile in [(0, 0, 4096), (1, 0, 4096), (4096, 0, 4096), (4097, 0, 4096), (10**9, 0, 4096),
                          (5000, 1, 2048)]:
        m = _desc(nnz, dt)
        assert L.nacho_auto_partitions(ctypes.byref(m), 1, 0) == max(1, -(-nnz // tile))
    ops = (N.Matrix * 3)(*[_desc(10**7) for _ in range(3)])
    # SpAdd: a 256 x 8-slot stage minus the bulk-copy pad (7 per operand) and Theorem 1's slack k - 1
    assert L.nacho_spadd_tile(3) == 256 * 8 - 7 * 3 and L.nacho_spadd_tile(0) == 0
    assert L.nacho_auto_partitions(ops, 3, 1) == -(-3 * 10**7 // (256 * 8 - 7 * 3 - 2))
    assert L.nacho_auto_partitions(ctypes.byref(_desc(10**6)), 1, 2) == -(-10**6 // 1024)
    m = _desc(10**6)
    assert L.nacho_spmv_workspace_size(ctypes.byref(m), 10) >= 10 * 12
    assert L.nacho_spmm_workspace_size(ctypes.byref(m), 10, 64) >= 10 * (8 + 64 * 4)


def test_invalid_arguments_rejected_before_launch():
    import paper_2604_17198_b200 as N
    L = N.lib
    m = _desc(10)
    parts = N.PartsC()
    # k out of range / P < 1 / null parts: host-side errors, no GPU touched
    assert L.nacho_partition(ctypes.byref(m), 0, 4, ctypes.byref(parts), None) == 1
    assert L.nacho_partition(ctypes.byref(m), 1, 0, ctypes.byref(parts), None) in (1,)
    m.ncols = 2**31
    assert L.nacho_spmv(ctypes.byref(m), None, None, None, 0, None, 0, None) in (1, 4)
    m = _desc(10, nrows=2**31)   # partition-local row spans are 32-bit
    assert L.nacho_partition(ctypes.byref(m), 1, 4, ctypes.byref(parts), None) == 4
    assert b"" != L.nacho_last_error()
