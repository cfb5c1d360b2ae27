"""Synthetic input recipe (workloads/): valid sorted formats, determinism, the intended shape."""
import numpy as np
import pytest

import oracle as O
import workloads as W
from workloads import recipe as R


def test_feistel_is_a_bijection():
    for n in (1, 2, 3, 17, 1000, 4097):
        p = R.feistel_perm(np.arange(n, dtype=np.uint64), n, seed=9)
        assert sorted(p.tolist()) == list(range(n))


def test_sum_floor_div_matches_direct():
    for cdiv, m, cap, mn in [(1000, 50, 100, 0), (12345, 20000, 500, 1), (7, 3, 10, 0)]:
        q = np.arange(m)
        direct = int(np.clip(cdiv // (q + 1), mn, cap).sum())
        assert R.sum_floor_div(cdiv, m, cap, mn) == direct


@pytest.mark.parametrize("name,scale", [("c1", 1.0), ("c2", 0.02), ("c3", 0.002), ("c4", 1e-4), ("c5", 2e-5)])
def test_configs_valid_and_deterministic(name, scale):
    a = W.build(name, scale)
    b = W.build(name, scale)
    for A, B in zip(a.ops, b.ops):
        assert O.validate(A) == 0
        assert np.array_equal(A.crd, B.crd) and np.array_equal(A.val, B.val) and np.array_equal(A.pos, B.pos)
    cfg = a.meta
    nnz = a.ops[0].nnz
    extra = cfg["m"] if cfg.get("dense_row") is not None else 0
    assert abs(nnz - cfg["target"] - extra) <= max(0.02 * cfg["target"], 64)


def test_c1_has_the_dense_row_and_skew():
    wl = W.build("c1")
    A = wl.ops[0]
    deg = np.diff(A.pos)
    assert deg[2049] == 4096 and A.val.dtype == np.float64
    assert np.median(deg) < 10 and np.sort(deg)[-2] > 100      # heavy power-law head besides the dense row
    assert abs(A.nnz - (36_900 + 4096)) < 200


def test_c2_operands_share_rows_and_overlap():
    wl = W.build("c2", 0.02)
    A, B, C = wl.ops
    assert np.array_equal(A.pos, B.pos) and np.array_equal(A.pos, C.pos)
    ka = set(zip(np.repeat(np.arange(A.nrows), np.diff(A.pos)).tolist(), A.crd.tolist()))
    kb = set(zip(np.repeat(np.arange(B.nrows), np.diff(B.pos)).tolist(), B.crd.tolist()))
    frac = len(ka & kb) / len(kb)
    assert 0.25 < frac < 0.45          # 30% reused + chance collisions
    assert (np.diff(A.pos) == 0).any()  # empty rows present
    z_pos, z_crd, _ = O.spadd_k(wl.ops)
    assert 2.0 * A.nnz < len(z_crd) < 2.7 * A.nnz


def test_dcsr_stored_rows_nonempty():
    wl = W.build("c3", 0.002)
    A = wl.ops[0]
    assert A.format == "dcsr" and (np.diff(A.pos) >= 1).all()
    assert (np.diff(A.outer_crd.astype(np.int64)) > 0).all()


def test_integer_values_mode():
    wl = W.build("c2", 0.01, values="int", kmax=8)
    for A in wl.ops:
        assert np.array_equal(A.val, np.round(A.val)) and np.abs(A.val).max() <= 8 and (A.val != 0).all()
