"""Small seeded random instances for tests (inputs only)."""
import numpy as np

import workloads as W


def random_csr(rng, M, N, density, dtype=np.float32, dense_rows=(), empty_frac=0.3, ints=False, base=None,
               share=0.0):
    """Random CSR with empty rows; optionally shares a fraction of coordinates with `base`."""
    mask = rng.random((M, N)) < density
    mask[rng.random(M) < empty_frac, :] = False
    for r in dense_rows:
        mask[r, :] = True
    if base is not None and share > 0:
        bm = W.to_dense(base) != 0
        mask |= bm & (rng.random((M, N)) < share)
    rows, cols = np.nonzero(mask)
    if ints:
        vals = rng.integers(1, 5, size=len(rows)) * rng.choice([-1, 1], size=len(rows))
    else:
        vals = rng.uniform(0.5, 1.5, size=len(rows))
    A = W.from_coo(rows, cols, vals.astype(dtype), M, N, dtype=dtype)
    return A


def random_dcsr(rng, M, N, nstored, density, dtype=np.float32):
    rows_sel = np.sort(rng.choice(M, size=min(nstored, M), replace=False))
    rr, cc = [], []
    for r in rows_sel:
        cols = np.nonzero(rng.random(N) < density)[0]
        if len(cols) == 0:
            cols = np.array([rng.integers(N)])
        rr += [r] * len(cols)
        cc += list(cols)
    vals = rng.uniform(0.5, 1.5, size=len(rr)).astype(dtype)
    return W.from_coo(rr, cc, vals, M, N, fmt=W.DCSR, dtype=dtype)


def entries(A):
    """Sorted list of (row, col) of a CSR/DCSR operand."""
    A = A.numpy()
    out = []
    for ip in range(A.nouter):
        r = ip if A.format == "csr" else int(A.outer_crd[ip])
        for q in range(int(A.pos[ip]), int(A.pos[ip + 1])):
            out.append((r, int(A.crd[q])))
    return out


def brute_force_boundary(ops, Q):
    """Lexicographic argmax over all cut points x = (xi, xj), xi in [0, M), xj in [0, N), plus the end (M, 0),
    of {C(x) <= Q} with C(x) = #entries (over all operands) lexicographically before x (Theorem 1's C)."""
    M, N = ops[0].nrows, ops[0].ncols
    ents = [entries(A) for A in ops]
    allk = sorted(e for es in ents for e in es)
    best = (0, 0)
    cands = [(i, j) for i in range(M) for j in range(N)] + [(M, 0)]
    import bisect
    for x in cands:
        c = bisect.bisect_left(allk, x)
        if c <= Q and x > best:
            best = x
    pos = [bisect.bisect_left(es, best) for es in ents]
    return best, pos
