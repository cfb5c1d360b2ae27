"""Pins of the mixed CSR / COO oracle (the COO + CSR addition the paper evaluates; COO =
TACO's Compressed(non-unique) o Singleton levels): the partition of COO operands is the
partition of the same matrices in CSR (the lexicographic rank does not depend on the format), the
mixed union equals the CSR union bit for bit, and dense brute force."""
import numpy as np
import pytest

import oracle as O
import workloads as W
from tests.util import random_csr


@pytest.mark.parametrize("k", [2, 3])
def test_mixed_against_csr_and_dense(k):
    rng = np.random.default_rng(80 + k)
    for trial in range(20):
        M, N = int(rng.integers(1, 60)), int(rng.integers(1, 50))
        base = random_csr(rng, M, N, float(rng.uniform(0.02, 0.4)), dense_rows=[int(rng.integers(M))] if trial % 3 == 0 else ())
        csr = [base] + [random_csr(rng, M, N, float(rng.uniform(0.02, 0.4)), base=base, share=0.5) for _ in range(k - 1)]
        fmts = [rng.random() < 0.5 for _ in range(k)]
        if not any(fmts):
            fmts[0] = True
        mixed = [W.to_coo(A) if f else A for A, f in zip(csr, fmts)]
        zp, zc, zv = O.mixed_spadd_k(mixed)
        rp, rc, rv = O.spadd_k(csr)
        assert np.array_equal(zp, rp) and np.array_equal(zc, rc)
        assert np.array_equal(zv.view(np.uint8), rv.view(np.uint8))
        dense = sum(W.to_dense(A) for A in mixed)
        mask = np.logical_or.reduce([W.to_dense(A) != 0 for A in mixed])
        r, c = np.nonzero(mask)
        assert np.array_equal(zc, c.astype(np.int32))
        assert np.allclose(zv, dense[r, c], rtol=1e-6)
        for P in (1, 4, 13):
            pm, pc = O.partition_rank(mixed, P), O.partition_rank(csr, P)
            for f in ("query", "row", "row_pos", "col", "pos"):
                assert np.array_equal(getattr(pm, f), getattr(pc, f)), f
