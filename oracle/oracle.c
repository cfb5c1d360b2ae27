/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY (see oracle.h).  Plain, slow, single-threaded.
 *
 * Every function follows a definition or an algorithm of the paper (PAPER.md line cited)
 * step by step, without blocking, fusion or reordering.  Where the paper is silent the
 * reading taken is named "R<n>" and listed in DESIGN.md ("Readings of the paper").
 *
 * Nothing here is shared with the CUDA path.
 */
#include "oracle.h"
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ helpers */

static long double vget_ld(const or_matrix *A, int64_t q) {
    return A->dtype == OR_F64 ? (long double)((const double *)A->val)[q]
                              : (long double)((const float *)A->val)[q];
}
/* row coordinate of outer position ip (P:1679 CSR dense row level; P:562 DCSR compressed row level) */
static int64_t row_of(const or_matrix *A, int64_t ip) {
    return A->format == OR_CSR ? ip : (int64_t)A->outer_crd[ip];   /* COO: ip is the entry */
}

/* lb_search of Listing 7: "Find least ipA in [lA, hA] s.t. A[ipA] >= i".
 * Returns hi+1 when every crd in [lo, hi] is < x (and lo when the window is empty). */
int64_t oracle_lb_search(const int32_t *crd, int64_t lo, int64_t hi, int64_t x) {
    int64_t a = lo, b = hi + 1;            /* answer in [a, b] */
    while (a < b) {
        int64_t m = a + (b - a) / 2;
        if ((int64_t)crd[m] >= x) b = m; else a = m + 1;
    }
    return a;
}

/* ------------------------------------------------------------- validation */
/* Sorted-level invariants ("These are sorted formats") and DCSR canonical
 * form (R10: stored rows are non-empty). */
int oracle_validate(const or_matrix *A) {
    if (A->nrows < 0 || A->ncols < 0 || A->nnz < 0) return 1;
    if (A->format == OR_CSR && A->nouter != A->nrows) return 2;
    if (A->pos[0] != 0) return 3;
    if (A->pos[A->nouter] != A->nnz) return 4;
    for (int64_t i = 0; i < A->nouter; i++) {
        if (A->pos[i + 1] < A->pos[i]) return 5;
        for (int64_t q = A->pos[i]; q < A->pos[i + 1]; q++) {
            if (A->crd[q] < 0 || (int64_t)A->crd[q] >= A->ncols) return 6;
            if (q > A->pos[i] && A->crd[q] <= A->crd[q - 1]) return 7;
        }
    }
    if (A->format == OR_DCSR) {
        for (int64_t i = 0; i < A->nouter; i++) {
            if (A->outer_crd[i] < 0 || (int64_t)A->outer_crd[i] >= A->nrows) return 8;
            if (i > 0 && A->outer_crd[i] <= A->outer_crd[i - 1]) return 9;
            if (A->pos[i + 1] == A->pos[i]) return 10;
        }
    }
    return 0;
}

/* ------------------------------------------------- total cost and queries */
/* Q* = sum of non-zeros of every sparse operand ("sum of the number of non-zeros
 * contained in each sparse tensor"); dense operands cost nothing (R5). */
int64_t oracle_total_cost(int32_t k, const or_matrix *ops) {
    int64_t q = 0;
    for (int32_t o = 0; o < k; o++) q += ops[o].nnz;
    return q;
}

/* Q_p = p * Q* / P, rounded down (R4), computed in 128-bit. */
void oracle_queries(int64_t qstar, int32_t P, int64_t *Q) {
    for (int32_t p = 0; p <= P; p++) Q[p] = (int64_t)(((__int128)p * (__int128)qstar) / (__int128)P);
}

static void set_origin(int32_t k, or_parts *out, int32_t p) {
    out->row[p] = 0; out->row_pos[p] = 0; out->col[p] = 0;
    for (int32_t o = 0; o < k; o++) out->pos[(int64_t)p * k + o] = 0;
}
static void set_end(int32_t k, const or_matrix *ops, or_parts *out, int32_t p) {
    out->row[p] = ops[0].nrows;
    out->row_pos[p] = ops[0].format == OR_DCSR ? ops[0].nouter : ops[0].nrows;   /* COO: the dense row index */
    out->col[p] = 0;
    for (int32_t o = 0; o < k; o++) out->pos[(int64_t)p * k + o] = ops[o].nnz;
}
/* number of stored rows of operand 0 with coordinate < row (CSR: row itself) */
static int64_t outer_lb(const or_matrix *A, int64_t row) {
    if (A->format != OR_DCSR) return row;   /* CSR and COO: the dense row index */
    int64_t a = 0, b = A->nouter;
    while (a < b) { int64_t m = a + (b - a) / 2; if ((int64_t)A->outer_crd[m] >= row) b = m; else a = m + 1; }
    return a;
}

/* --------------------------------------- partition: the plain definition (rank) */
/*
 * The cost of coiterating from the origin to coordinate x (Theorem 1's C(x)) with the
 * nnz-count cost functions is the number of stored entries, over all operands, that come
 * lexicographically before x.  The highest coordinate whose cost is <= Q is therefore the
 * coordinate of entry number Q (0-indexed) of the lexicographically sorted multiset E of all stored
 * entries, and the positions are the per-operand counts of entries strictly before it.
 * One sweep enumerates E in order (the k-finger merge of Listing 1, in union form).
 * b_0 = origin and b_P = end (R1); an interior query with Q_p >= Q* (only when Q* = 0) is the end.
 */
int oracle_partition_rank(int32_t k, const or_matrix *ops, int32_t P, or_parts *out) {
    if (k < 1 || P < 1) return 1;
    int64_t qstar = oracle_total_cost(k, ops);
    oracle_queries(qstar, P, out->query);
    int64_t *q  = (int64_t *)calloc((size_t)k, sizeof(int64_t));   /* cursor position per operand */
    int64_t *ip = (int64_t *)calloc((size_t)k, sizeof(int64_t));   /* outer position per operand */
    int64_t c = 0;                                                   /* entries enumerated so far */
    int32_t p = 1;
    while (p < P) {
        int64_t best_r = -1, best_c = -1;
        for (int32_t o = 0; o < k; o++) {
            if (q[o] >= ops[o].nnz) continue;
            if (ops[o].format == OR_COO) ip[o] = q[o];                  /* COO: the row level is per entry */
            else while (ops[o].pos[ip[o] + 1] <= q[o]) ip[o]++;      /* outer position holding q[o] */
            int64_t r = row_of(&ops[o], ip[o]), cc = ops[o].crd[q[o]];
            if (best_r < 0 || r < best_r || (r == best_r && cc < best_c)) { best_r = r; best_c = cc; }
        }
        if (best_r < 0) break;                                       /* E exhausted */
        int32_t g = 0;                                               /* entries with this coordinate */
        for (int32_t o = 0; o < k; o++)
            if (q[o] < ops[o].nnz && row_of(&ops[o], ip[o]) == best_r && ops[o].crd[q[o]] == best_c) g++;
        while (p < P && out->query[p] < c + g) {                      /* E[Q_p] has this coordinate */
            out->row[p] = best_r;
            out->row_pos[p] = outer_lb(&ops[0], best_r);
            out->col[p] = (int32_t)best_c;
            for (int32_t o = 0; o < k; o++) out->pos[(int64_t)p * k + o] = q[o];
            p++;
        }
        for (int32_t o = 0; o < k; o++)
            if (q[o] < ops[o].nnz && row_of(&ops[o], ip[o]) == best_r && ops[o].crd[q[o]] == best_c) q[o]++;
        c += g;
    }
    for (; p < P; p++) set_end(k, ops, out, p);
    set_origin(k, out, 0);
    set_end(k, ops, out, P);
    free(q); free(ip);
    return 0;
}

/* ------------------------------------- partition: literal Alg. 1 (Listing 7 form) */
/*
 * FindPartition (Alg. 1) over the loop order i -> j with the CSR cost functions of
 * Listing 5 -- or, for a DCSR row level, the compressed-level query of P:1735-1737 --
 * searched as in Listing 7: an outer binary search with midpoint low+(high-low+1)/2
 * (P:1783), an inner lb_search per operand, and windows [l, h] that narrow as the search proceeds
 * (P:1790-1793).  The window update on a rejected midpoint uses h = ip - 1 (Listing 7 writes
 * hA = ipA, which can probe one past the window; the result is identical -- reading R15).
 * Domains: x_i in [0, M], x_j in [0, N) (R2).  If x_i = M the boundary is the end.
 */
static void find_partition_alg1(int32_t k, const or_matrix *ops, int64_t Q, or_parts *out, int32_t p,
                                int64_t *probes) {
    int64_t n_probe = 0;
    int64_t R = Q;
    const int64_t M = ops[0].nrows, N = ops[0].ncols;
    int64_t *lo = (int64_t *)malloc(sizeof(int64_t) * (size_t)k);
    int64_t *hi = (int64_t *)malloc(sizeof(int64_t) * (size_t)k);
    int64_t *ipv = (int64_t *)malloc(sizeof(int64_t) * (size_t)k);
    int64_t *rp = (int64_t *)malloc(sizeof(int64_t) * (size_t)k);

    /* ---- level m = i : HighestCoordinateLeqQuery over x_i in [0, M] (Alg. 1 line 7) ---- */
    for (int32_t o = 0; o < k; o++) {        /* outer windows (used for DCSR compressed rows) */
        lo[o] = 0; hi[o] = ops[o].nouter - 1; rp[o] = 0;
    }
    int64_t low = 0, high = M, cost_low = 0;  /* C_i(0) = 0 */
    while (low < high) {
        int64_t x = low + (high - low + 1) / 2;
        int64_t cost = 0;
        for (int32_t o = 0; o < k; o++) {
            if (ops[o].format == OR_CSR) {
                ipv[o] = x;                                               /* dense level: position == coordinate */
                cost += ops[o].pos[x] - ops[o].pos[0];                    /* Listing 5: C_i = A.pos[x_i] - A.pos[0] */
            } else {
                ipv[o] = oracle_lb_search(ops[o].outer_crd, lo[o], hi[o], x);  /* stored rows with coordinate < x */
                cost += ops[o].pos[ipv[o]] - ops[o].pos[0];
            }
        }
        n_probe++;
        if (cost <= R) { low = x; cost_low = cost; for (int32_t o = 0; o < k; o++) { lo[o] = ipv[o]; rp[o] = ipv[o]; } }
        else           { high = x - 1; for (int32_t o = 0; o < k; o++) hi[o] = ipv[o] - 1; }
    }
    int64_t xi = low;
    R -= cost_low;                                                   /* Alg. 1 line 8 */
    if (xi >= M) {
        set_end(k, ops, out, p);
    } else {
        /* ---- level m = j : HighestCoordinateLeqQuery over x_j in [0, N) within row xi ---- */
        int64_t *seg = (int64_t *)malloc(sizeof(int64_t) * (size_t)k);
        for (int32_t o = 0; o < k; o++) {
            int64_t r = (ops[o].format == OR_CSR) ? xi : rp[o];     /* outer position of row xi (if stored) */
            if (ops[o].format == OR_DCSR) {
                /* rp[o] = #stored rows with coordinate < xi (window start after the outer search) */
                r = oracle_lb_search(ops[o].outer_crd, 0, ops[o].nouter - 1, xi);
            }
            int stored = (ops[o].format == OR_CSR) || (r < ops[o].nouter && ops[o].outer_crd[r] == xi);
            seg[o] = ops[o].pos[r];
            lo[o] = ops[o].pos[r];
            hi[o] = stored ? ops[o].pos[r + 1] - 1 : ops[o].pos[r] - 1;
            rp[o] = r;
        }
        int64_t jlow = 0, jhigh = N - 1;
        while (jlow < jhigh) {
            int64_t x = jlow + (jhigh - jlow + 1) / 2;
            int64_t cost = 0;
            for (int32_t o = 0; o < k; o++) {
                ipv[o] = oracle_lb_search(ops[o].crd, lo[o], hi[o], x);    /* Listing 7 line 8-10 */
                cost += ipv[o] - seg[o];                                    /* Listing 5: C_j = x_jp - A.pos[x_i] */
            }
            n_probe++;
            if (cost <= R) { jlow = x; for (int32_t o = 0; o < k; o++) lo[o] = ipv[o]; }
            else           { jhigh = x - 1; for (int32_t o = 0; o < k; o++) hi[o] = ipv[o] - 1; }
        }
        out->row[p] = xi;
        out->row_pos[p] = rp[0];
        out->col[p] = (int32_t)jlow;
        for (int32_t o = 0; o < k; o++) out->pos[(int64_t)p * k + o] = lo[o];   /* Listing 7 line 20: p.ipA = lA */
        free(seg);
    }
    if (probes) probes[p] = n_probe;
    free(lo); free(hi); free(ipv); free(rp);
}

int oracle_partition_alg1(int32_t k, const or_matrix *ops, int32_t P, or_parts *out, int64_t *probes) {
    if (k < 1 || P < 1) return 1;
    int64_t qstar = oracle_total_cost(k, ops);
    oracle_queries(qstar, P, out->query);
    for (int32_t p = 1; p < P; p++) find_partition_alg1(k, ops, out->query[p], out, p, probes);
    set_origin(k, out, 0);  if (probes) probes[0] = 0;      /* R1 */
    set_end(k, ops, out, P); if (probes) probes[P] = 0;
    return 0;
}

/* ---------------------------------------------------------------- SpMV */
/* y_i = sum_j A_ij x_j (the broadcast example y = A x of P:1742-1744).  Products and sums in long
 * double (exact products for fp32 inputs), rounded once to the value type (R13). */
int oracle_spmv(const or_matrix *A, const void *x, void *y) {
    for (int64_t ip = 0; ip < A->nouter; ip++) {
        long double acc = 0.0L;
        for (int64_t q = A->pos[ip]; q < A->pos[ip + 1]; q++) {
            long double xv = A->dtype == OR_F64 ? (long double)((const double *)x)[A->crd[q]]
                                                : (long double)((const float *)x)[A->crd[q]];
            acc += vget_ld(A, q) * xv;
        }
        if (A->dtype == OR_F64) ((double *)y)[ip] = (double)acc;
        else                    ((float *)y)[ip]  = (float)acc;
    }
    return 0;
}

/* ---------------------------------------------------------------- SpMM */
/* C_ik = sum_j A_ij B_jk, loop order i -> j -> k (Listing 6 broadcast; R6). */
int oracle_spmm(const or_matrix *A, const void *B, int64_t ldb, int32_t nb, void *C, int64_t ldc) {
    if (A->format != OR_CSR) return 1;
    long double *acc = (long double *)malloc(sizeof(long double) * (size_t)(nb > 0 ? nb : 1));
    for (int64_t i = 0; i < A->nrows; i++) {
        for (int32_t c = 0; c < nb; c++) acc[c] = 0.0L;
        for (int64_t q = A->pos[i]; q < A->pos[i + 1]; q++) {
            long double a = vget_ld(A, q);
            int64_t j = A->crd[q];
            for (int32_t c = 0; c < nb; c++) {
                long double b = A->dtype == OR_F64 ? (long double)((const double *)B)[j * ldb + c]
                                                   : (long double)((const float *)B)[j * ldb + c];
                acc[c] += a * b;
            }
        }
        for (int32_t c = 0; c < nb; c++) {
            if (A->dtype == OR_F64) ((double *)C)[i * ldc + c] = (double)acc[c];
            else                    ((float *)C)[i * ldc + c]  = (float)acc[c];
        }
    }
    free(acc);
    return 0;
}

/* -------------------------------------------------------------- k-way SpAdd */
/*
 * Z = A_0 + ... + A_{k-1}: coiteration over the union (Listing 2, in CSR form), one
 * k-finger merge per row.  Structure is the structural union (TACO assembly is symbolic).
 * Z.val(i,j) = left fold in operand order over the operands that store (i,j), starting from the
 * first present value (R9), in the value type's own arithmetic.
 */
int64_t oracle_spadd_k(int32_t k, const or_matrix *ops, int64_t *z_pos, int32_t *z_crd, void *z_val,
                       int64_t capacity) {
    for (int32_t o = 0; o < k; o++) if (ops[o].format != OR_CSR) return -1;
    const int64_t M = ops[0].nrows;
    const int f64 = ops[0].dtype == OR_F64;
    int64_t *q = (int64_t *)malloc(sizeof(int64_t) * (size_t)k);
    int64_t nz = 0;
    z_pos[0] = 0;
    for (int64_t i = 0; i < M; i++) {
        for (int32_t o = 0; o < k; o++) q[o] = ops[o].pos[i];
        for (;;) {
            int64_t j = -1;
            for (int32_t o = 0; o < k; o++)
                if (q[o] < ops[o].pos[i + 1] && (j < 0 || ops[o].crd[q[o]] < j)) j = ops[o].crd[q[o]];
            if (j < 0) break;
            double vd = 0.0; float vf = 0.0f; int have = 0;
            for (int32_t o = 0; o < k; o++) {
                if (q[o] < ops[o].pos[i + 1] && ops[o].crd[q[o]] == j) {
                    if (f64) { double a = ((const double *)ops[o].val)[q[o]]; vd = have ? vd + a : a; }
                    else     { float  a = ((const float *)ops[o].val)[q[o]];  vf = have ? vf + a : a; }
                    have = 1;
                    q[o]++;
                }
            }
            if (nz >= capacity) { free(q); return -1; }
            z_crd[nz] = (int32_t)j;
            if (f64) ((double *)z_val)[nz] = vd; else ((float *)z_val)[nz] = vf;
            nz++;
        }
        z_pos[i + 1] = nz;
    }
    free(q);
    return nz;
}

/* Per-partition assembly counts: the number of union coordinates c with
 * b_p <=lex c <lex b_{p+1}; matching coordinates of different operands fall in one partition
 * because the cut is in coordinate space. */
int oracle_spadd_counts(int32_t k, const or_matrix *ops, const or_parts *parts, int64_t *cnt) {
    for (int32_t o = 0; o < k; o++) if (ops[o].format != OR_CSR) return 1;
    const int32_t P = parts->P;
    const int64_t M = ops[0].nrows;
    int64_t *q = (int64_t *)malloc(sizeof(int64_t) * (size_t)k);
    for (int32_t p = 0; p < P; p++) cnt[p] = 0;
    int32_t p = 0;
    for (int64_t i = 0; i < M; i++) {
        for (int32_t o = 0; o < k; o++) q[o] = ops[o].pos[i];
        for (;;) {
            int64_t j = -1;
            for (int32_t o = 0; o < k; o++)
                if (q[o] < ops[o].pos[i + 1] && (j < 0 || ops[o].crd[q[o]] < j)) j = ops[o].crd[q[o]];
            if (j < 0) break;
            /* advance p while c >= b_{p+1} (lexicographic on (row, col)) */
            while (p + 1 < P && (i > parts->row[p + 1] || (i == parts->row[p + 1] && j >= parts->col[p + 1]))) p++;
            cnt[p]++;
            for (int32_t o = 0; o < k; o++)
                if (q[o] < ops[o].pos[i + 1] && ops[o].crd[q[o]] == j) q[o]++;
        }
    }
    free(q);
    return 0;
}

/* ------------------------------------------------------ k-way intersection */
/*
 * Z = A_0 (.) ... (.) A_{k-1} (element-wise product): the k-finger merge of Listing 1 (P:333-344,
 * "z_i = a_i * b_i * c_i via a three-finger merge") applied to every CSR row, which is the loop body of
 * the partitioned CSR Hadamard product of Listing 8 run with one partition.  A
 * coordinate is emitted when every operand's head equals the minimum head (Listing 1 line "if i ==
 * i_a && i == i_b && i == i_c"); every finger whose head equals the minimum advances.  Z.val is the
 * product in operand order, left to right, in the value type's own arithmetic (Listing 1 evaluates
 * a.v * b.v * c.v as (a.v * b.v) * c.v).  Structure is the structural intersection (stored entries,
 * whatever their values).
 */
int64_t oracle_hadamard_k(int32_t k, const or_matrix *ops, int64_t *z_pos, int32_t *z_crd, void *z_val,
                          int64_t capacity) {
    for (int32_t o = 0; o < k; o++) if (ops[o].format != OR_CSR) return -1;
    const int64_t M = ops[0].nrows;
    const int f64 = ops[0].dtype == OR_F64;
    int64_t *q = (int64_t *)malloc(sizeof(int64_t) * (size_t)k);
    int64_t nz = 0;
    z_pos[0] = 0;
    for (int64_t i = 0; i < M; i++) {
        for (int32_t o = 0; o < k; o++) q[o] = ops[o].pos[i];
        for (;;) {
            /* while p_a < nnz(a) && p_b < nnz(b) && ... (all fingers inside their row segments) */
            int inside = 1;
            for (int32_t o = 0; o < k; o++) if (q[o] >= ops[o].pos[i + 1]) inside = 0;
            if (!inside) break;
            int64_t j = ops[0].crd[q[0]];
            for (int32_t o = 1; o < k; o++) if (ops[o].crd[q[o]] < j) j = ops[o].crd[q[o]];
            int all = 1;
            for (int32_t o = 0; o < k; o++) if (ops[o].crd[q[o]] != j) all = 0;
            if (all) {
                if (nz >= capacity) { free(q); return -1; }
                if (f64) {
                    double v = ((const double *)ops[0].val)[q[0]];
                    for (int32_t o = 1; o < k; o++) v = v * ((const double *)ops[o].val)[q[o]];
                    ((double *)z_val)[nz] = v;
                } else {
                    float v = ((const float *)ops[0].val)[q[0]];
                    for (int32_t o = 1; o < k; o++) v = v * ((const float *)ops[o].val)[q[o]];
                    ((float *)z_val)[nz] = v;
                }
                z_crd[nz++] = (int32_t)j;
            }
            for (int32_t o = 0; o < k; o++) if (ops[o].crd[q[o]] == j) q[o]++;
        }
        z_pos[i + 1] = nz;
    }
    free(q);
    return nz;
}

/* Per-partition assembly counts of the intersection (P:2051-2056 with the intersection predicate):
 * cnt[p] = #coordinates c stored by every operand with b_p <=lex c <lex b_{p+1}. */
int oracle_hadamard_counts(int32_t k, const or_matrix *ops, const or_parts *parts, int64_t *cnt) {
    for (int32_t o = 0; o < k; o++) if (ops[o].format != OR_CSR) return 1;
    const int32_t P = parts->P;
    const int64_t M = ops[0].nrows;
    int64_t *q = (int64_t *)malloc(sizeof(int64_t) * (size_t)k);
    for (int32_t p = 0; p < P; p++) cnt[p] = 0;
    int32_t p = 0;
    for (int64_t i = 0; i < M; i++) {
        for (int32_t o = 0; o < k; o++) q[o] = ops[o].pos[i];
        for (;;) {
            int inside = 1;
            for (int32_t o = 0; o < k; o++) if (q[o] >= ops[o].pos[i + 1]) inside = 0;
            if (!inside) break;
            int64_t j = ops[0].crd[q[0]];
            for (int32_t o = 1; o < k; o++) if (ops[o].crd[q[o]] < j) j = ops[o].crd[q[o]];
            int all = 1;
            for (int32_t o = 0; o < k; o++) if (ops[o].crd[q[o]] != j) all = 0;
            if (all) {
                while (p + 1 < P && (i > parts->row[p + 1] || (i == parts->row[p + 1] && j >= parts->col[p + 1]))) p++;
                cnt[p]++;
            }
            for (int32_t o = 0; o < k; o++) if (ops[o].crd[q[o]] == j) q[o]++;
        }
    }
    free(q);
    return 0;
}

/* The intersect-reduce inner product s = sum_(i,j) prod_o A_o(i,j) (the fused (.) + reduction of
 * the paper's inner-product evaluation, on CSR operands): the same k-finger merge, every
 * product and the sum accumulated wide (long double), rounded once (reading R13: summation order
 * free within tolerance). */
int oracle_inner_k(int32_t k, const or_matrix *ops, double *out) {
    for (int32_t o = 0; o < k; o++) if (ops[o].format != OR_CSR) return 1;
    const int64_t M = ops[0].nrows;
    int64_t *q = (int64_t *)malloc(sizeof(int64_t) * (size_t)k);
    long double s = 0.0L;
    for (int64_t i = 0; i < M; i++) {
        for (int32_t o = 0; o < k; o++) q[o] = ops[o].pos[i];
        for (;;) {
            int inside = 1;
            for (int32_t o = 0; o < k; o++) if (q[o] >= ops[o].pos[i + 1]) inside = 0;
            if (!inside) break;
            int64_t j = ops[0].crd[q[0]];
            for (int32_t o = 1; o < k; o++) if (ops[o].crd[q[o]] < j) j = ops[o].crd[q[o]];
            int all = 1;
            for (int32_t o = 0; o < k; o++) if (ops[o].crd[q[o]] != j) all = 0;
            if (all) {
                long double v = 1.0L;
                for (int32_t o = 0; o < k; o++) v *= vget_ld(&ops[o], q[o]);
                s += v;
            }
            for (int32_t o = 0; o < k; o++) if (ops[o].crd[q[o]] == j) q[o]++;
        }
    }
    free(q);
    *out = (double)s;
    return 0;
}

/* --------------------------------------------- recursive partitioning (Alg. 2) */
/*
 * The DCSR Hadamard product Z = A_0 (.) ... (.) A_{k-1} of Listing emul-dcsr2-cfir has an
 * outer sparse intersection, so Alg. 2 remaps the row cost before partitioning.  These
 * functions follow Listing emul-dcsr2-rewritten line by line:
 *   line 2-3  while i <- rows(A_0) cap ... cap rows(A_{k-1}):  T[i] = C_j(N_j | i)
 *             (C_j(N_j | i) = the non-zeros of row i over the operands, the nnz cost of P:1689),
 *   line 4    T' = exclusive_prefix_sum(T),
 *   line 5    C'_i(x_i) = T'[x_i]  (the remapped cost),
 *   line 7-9  for i <- i_T:  while j <- cols(A_0[i]) cap ...:  Z[i, j] = prod_o A_o[i, j].
 */

/* Lines 2-3: the surviving rows (k-finger intersection of the outer levels, Listing 1's predicate)
 * with T and every operand's outer position of the row.  rows / T / ip (ip[o * cap + s]) need
 * capacity >= min_o nouter_o.  Returns S, the number of surviving rows, or -1. */
int64_t oracle_dcsr_rows_intersect(int32_t k, const or_matrix *ops, int64_t *rows, int64_t *T, int64_t *ip,
                                   int64_t cap) {
    for (int32_t o = 0; o < k; o++) if (ops[o].format != OR_DCSR) return -1;
    int64_t *q = (int64_t *)calloc((size_t)k, sizeof(int64_t));
    int64_t S = 0;
    for (;;) {
        int inside = 1;
        for (int32_t o = 0; o < k; o++) if (q[o] >= ops[o].nouter) inside = 0;
        if (!inside) break;
        int64_t r = ops[0].outer_crd[q[0]];
        for (int32_t o = 1; o < k; o++) if (ops[o].outer_crd[q[o]] < r) r = ops[o].outer_crd[q[o]];
        int all = 1;
        for (int32_t o = 0; o < k; o++) if (ops[o].outer_crd[q[o]] != r) all = 0;
        if (all) {
            if (S >= cap) { free(q); return -1; }
            int64_t t = 0;
            for (int32_t o = 0; o < k; o++) {
                t += ops[o].pos[q[o] + 1] - ops[o].pos[q[o]];
                ip[(int64_t)o * cap + S] = q[o];
            }
            rows[S] = r;
            T[S] = t;
            S++;
        }
        for (int32_t o = 0; o < k; o++) if (ops[o].outer_crd[q[o]] == r) q[o]++;
    }
    free(q);
    return S;
}

/* Line 4: T' = exclusive prefix sum of T (S + 1 entries, T'[S] = the remapped total cost). */
void oracle_exclusive_prefix(const int64_t *T, int64_t S, int64_t *Tp) {
    int64_t acc = 0;
    for (int64_t s = 0; s < S; s++) { Tp[s] = acc; acc += T[s]; }
    Tp[S] = acc;
}

/*
 * Line 5-6: partition the remapped loop nest (i' over the surviving rows, j over the row's columns)
 * with C'_i = T' and the inner nnz cost -- the plain definition of oracle_partition_rank applied to
 * the remapped space: Q_p = floor(p * T'[S] / P) (R4), b_p = the coordinate of entry number Q_p of
 * the lexicographic multiset of the surviving rows' entries (ties between operands irrelevant).
 * row_pos = i' (index of the surviving row), row = rows[i'], col, pos[o] = absolute position in crd_o
 * of operand o's first entry at or after b_p within row i'.  b_0: i' = 0, col 0, pos[o] = start of
 * row 0's segment; b_P (and Q_p >= T'[S]): i' = S, row = nrows, col 0, pos[o] = end of the last
 * surviving row's segment (0 when S = 0).
 */
int oracle_partition_remapped(int32_t k, const or_matrix *ops, int64_t S, const int64_t *rows, const int64_t *ip,
                              int64_t cap, const int64_t *Tp, int32_t P, or_parts *out) {
    if (k < 1 || P < 1) return 1;
    oracle_queries(Tp[S], P, out->query);
    for (int32_t p = 0; p <= P; p++) {
        const int64_t Q = out->query[p];
        if (p == 0 && S > 0) {                    /* origin (R1): the first surviving row, column 0 */
            out->row[p] = rows[0]; out->row_pos[p] = 0; out->col[p] = 0;
            for (int32_t o = 0; o < k; o++) out->pos[(int64_t)p * k + o] = ops[o].pos[ip[(int64_t)o * cap]];
            continue;
        }
        if (p == P || Q >= Tp[S] || S == 0) {   /* end */
            out->row[p] = ops[0].nrows; out->row_pos[p] = S; out->col[p] = 0;
            for (int32_t o = 0; o < k; o++)
                out->pos[(int64_t)p * k + o] = S > 0 ? ops[o].pos[ip[(int64_t)o * cap + S - 1] + 1] : 0;
            continue;
        }
        /* the surviving row holding entry Q: highest s with T'[s] <= Q */
        int64_t s = 0;
        while (s + 1 < S && Tp[s + 1] <= Q) s++;
        int64_t R = Q - Tp[s];            /* entry number R of row s's merged multiset */
        int64_t *q = (int64_t *)malloc(sizeof(int64_t) * (size_t)k);
        for (int32_t o = 0; o < k; o++) q[o] = ops[o].pos[ip[(int64_t)o * cap + s]];
        int64_t c = 0, col = 0;
        for (;;) {                         /* k-finger union merge of row s until entry R */
            int64_t j = -1;
            for (int32_t o = 0; o < k; o++) {
                const int64_t e = ops[o].pos[ip[(int64_t)o * cap + s] + 1];
                if (q[o] < e && (j < 0 || ops[o].crd[q[o]] < j)) j = ops[o].crd[q[o]];
            }
            int64_t g = 0;
            for (int32_t o = 0; o < k; o++) {
                const int64_t e = ops[o].pos[ip[(int64_t)o * cap + s] + 1];
                if (q[o] < e && ops[o].crd[q[o]] == j) g++;
            }
            if (R < c + g) { col = j; break; }
            for (int32_t o = 0; o < k; o++) {
                const int64_t e = ops[o].pos[ip[(int64_t)o * cap + s] + 1];
                if (q[o] < e && ops[o].crd[q[o]] == j) q[o]++;
            }
            c += g;
        }
        out->row[p] = rows[s]; out->row_pos[p] = s; out->col[p] = (int32_t)col;
        for (int32_t o = 0; o < k; o++) out->pos[(int64_t)p * k + o] = q[o];
        free(q);
    }
    return 0;
}

/* Lines 7-9: Z over the surviving rows (DCSR: z_outer = the surviving rows, every one stored, with
 * possibly empty segments -- reading R21), values the product in operand order (R17).  Returns nnz_Z. */
int64_t oracle_dcsr_hadamard(int32_t k, const or_matrix *ops, int64_t S, const int64_t *ip, int64_t cap,
                             int64_t *z_pos, int32_t *z_crd, void *z_val, int64_t zcap) {
    const int f64 = ops[0].dtype == OR_F64;
    int64_t *q = (int64_t *)malloc(sizeof(int64_t) * (size_t)k);
    int64_t nz = 0;
    z_pos[0] = 0;
    for (int64_t s = 0; s < S; s++) {
        for (int32_t o = 0; o < k; o++) q[o] = ops[o].pos[ip[(int64_t)o * cap + s]];
        for (;;) {
            int inside = 1;
            for (int32_t o = 0; o < k; o++) if (q[o] >= ops[o].pos[ip[(int64_t)o * cap + s] + 1]) inside = 0;
            if (!inside) break;
            int64_t j = ops[0].crd[q[0]];
            for (int32_t o = 1; o < k; o++) if (ops[o].crd[q[o]] < j) j = ops[o].crd[q[o]];
            int all = 1;
            for (int32_t o = 0; o < k; o++) if (ops[o].crd[q[o]] != j) all = 0;
            if (all) {
                if (nz >= zcap) { free(q); return -1; }
                if (f64) {
                    double v = ((const double *)ops[0].val)[q[0]];
                    for (int32_t o = 1; o < k; o++) v = v * ((const double *)ops[o].val)[q[o]];
                    ((double *)z_val)[nz] = v;
                } else {
                    float v = ((const float *)ops[0].val)[q[0]];
                    for (int32_t o = 1; o < k; o++) v = v * ((const float *)ops[o].val)[q[o]];
                    ((float *)z_val)[nz] = v;
                }
                z_crd[nz++] = (int32_t)j;
            }
            for (int32_t o = 0; o < k; o++) if (ops[o].crd[q[o]] == j) q[o]++;
        }
        z_pos[s + 1] = nz;
    }
    free(q);
    return nz;
}

/* ---------------------------------------------------------- DCSR k-way SpAdd */
/*
 * Z = A_0 + ... + A_{k-1} on DCSR operands: Listing 2 (lst:eadd-dcsr2-cfir) literally --
 *   while i <- rows(A_0) cup ... :  while j <- cols(A_0[i]) cup ... :  Z[i, j] = sum_o A_o[i, j]
 * with the k-finger merges of Listing 1 in union form at both levels; values the left fold in operand
 * order from the first present value (R9).  Z is DCSR: its outer level is the union of the operands'
 * stored rows, all non-empty (R10).  Capacities: z_outer >= sum nouter, z_pos >= that + 1, z_crd /
 * z_val >= sum nnz.  Returns nnz_Z (z_nrows receives the number of stored rows), or -1.
 */
int64_t oracle_dcsr_spadd_k(int32_t k, const or_matrix *ops, int32_t *z_outer, int64_t *z_pos, int32_t *z_crd,
                            void *z_val, int64_t *z_nrows, int64_t rcap, int64_t zcap) {
    for (int32_t o = 0; o < k; o++) if (ops[o].format != OR_DCSR) return -1;
    const int f64 = ops[0].dtype == OR_F64;
    int64_t *qi = (int64_t *)calloc((size_t)k, sizeof(int64_t));   /* outer cursors */
    int64_t *q = (int64_t *)calloc((size_t)k, sizeof(int64_t));    /* inner cursors */
    int64_t *e = (int64_t *)calloc((size_t)k, sizeof(int64_t));
    int64_t nz = 0, nr = 0;
    z_pos[0] = 0;
    for (;;) {
        int64_t r = -1;
        for (int32_t o = 0; o < k; o++)
            if (qi[o] < ops[o].nouter && (r < 0 || ops[o].outer_crd[qi[o]] < r)) r = ops[o].outer_crd[qi[o]];
        if (r < 0) break;
        for (int32_t o = 0; o < k; o++) {
            if (qi[o] < ops[o].nouter && ops[o].outer_crd[qi[o]] == r) { q[o] = ops[o].pos[qi[o]]; e[o] = ops[o].pos[qi[o] + 1]; }
            else { q[o] = 0; e[o] = 0; }
        }
        for (;;) {
            int64_t j = -1;
            for (int32_t o = 0; o < k; o++) if (q[o] < e[o] && (j < 0 || ops[o].crd[q[o]] < j)) j = ops[o].crd[q[o]];
            if (j < 0) break;
            double vd = 0.0; float vf = 0.0f; int have = 0;
            for (int32_t o = 0; o < k; o++) {
                if (q[o] < e[o] && ops[o].crd[q[o]] == j) {
                    if (f64) { double a = ((const double *)ops[o].val)[q[o]]; vd = have ? vd + a : a; }
                    else     { float  a = ((const float *)ops[o].val)[q[o]];  vf = have ? vf + a : a; }
                    have = 1;
                    q[o]++;
                }
            }
            if (nz >= zcap) { free(qi); free(q); free(e); return -1; }
            z_crd[nz] = (int32_t)j;
            if (f64) ((double *)z_val)[nz] = vd; else ((float *)z_val)[nz] = vf;
            nz++;
        }
        if (nr >= rcap) { free(qi); free(q); free(e); return -1; }
        z_outer[nr] = (int32_t)r;
        z_pos[nr + 1] = nz;
        nr++;
        for (int32_t o = 0; o < k; o++) if (qi[o] < ops[o].nouter && ops[o].outer_crd[qi[o]] == r) qi[o]++;
    }
    free(qi); free(q); free(e);
    *z_nrows = nr;
    return nz;
}

/* Per-partition assembly counts of the DCSR union for given boundaries: ent[p] = #union coordinates c
 * with b_p <=lex c <lex b_{p+1}; rows[p] = #union rows whose first union coordinate lies there (the
 * partition that appends the row to Z's outer level). */
int oracle_dcsr_spadd_counts(int32_t k, const or_matrix *ops, const or_parts *parts, int64_t *ent, int64_t *rows) {
    for (int32_t o = 0; o < k; o++) if (ops[o].format != OR_DCSR) return 1;
    const int32_t P = parts->P;
    int64_t *qi = (int64_t *)calloc((size_t)k, sizeof(int64_t));
    int64_t *q = (int64_t *)calloc((size_t)k, sizeof(int64_t));
    int64_t *e = (int64_t *)calloc((size_t)k, sizeof(int64_t));
    for (int32_t p = 0; p < P; p++) { ent[p] = 0; rows[p] = 0; }
    int32_t p = 0;
    for (;;) {
        int64_t r = -1;
        for (int32_t o = 0; o < k; o++)
            if (qi[o] < ops[o].nouter && (r < 0 || ops[o].outer_crd[qi[o]] < r)) r = ops[o].outer_crd[qi[o]];
        if (r < 0) break;
        for (int32_t o = 0; o < k; o++) {
            if (qi[o] < ops[o].nouter && ops[o].outer_crd[qi[o]] == r) { q[o] = ops[o].pos[qi[o]]; e[o] = ops[o].pos[qi[o] + 1]; }
            else { q[o] = 0; e[o] = 0; }
        }
        int first = 1;
        for (;;) {
            int64_t j = -1;
            for (int32_t o = 0; o < k; o++) if (q[o] < e[o] && (j < 0 || ops[o].crd[q[o]] < j)) j = ops[o].crd[q[o]];
            if (j < 0) break;
            while (p + 1 < P && (r > parts->row[p + 1] || (r == parts->row[p + 1] && j >= parts->col[p + 1]))) p++;
            ent[p]++;
            if (first) { rows[p]++; first = 0; }
            for (int32_t o = 0; o < k; o++) if (q[o] < e[o] && ops[o].crd[q[o]] == j) q[o]++;
        }
        for (int32_t o = 0; o < k; o++) if (qi[o] < ops[o].nouter && ops[o].outer_crd[qi[o]] == r) qi[o]++;
    }
    free(qi); free(q); free(e);
    return 0;
}

/* ------------------------------------------------------ mixed CSR / COO k-way SpAdd */
/* The row segment of operand o: CSR [pos[i], pos[i+1]); COO the entries whose row is i (a cursor that
 * moves forward over the sorted row level). */
int64_t oracle_mixed_spadd_k(int32_t k, const or_matrix *ops, int64_t *z_pos, int32_t *z_crd, void *z_val,
                             int64_t capacity) {
    for (int32_t o = 0; o < k; o++) if (ops[o].format == OR_DCSR) return -1;
    const int64_t M = ops[0].nrows;
    const int f64 = ops[0].dtype == OR_F64;
    int64_t *q = (int64_t *)calloc((size_t)k, sizeof(int64_t));
    int64_t *e = (int64_t *)calloc((size_t)k, sizeof(int64_t));
    int64_t *cc = (int64_t *)calloc((size_t)k, sizeof(int64_t));   /* COO cursors */
    int64_t nz = 0;
    z_pos[0] = 0;
    for (int64_t i = 0; i < M; i++) {
        for (int32_t o = 0; o < k; o++) {
            if (ops[o].format == OR_CSR) { q[o] = ops[o].pos[i]; e[o] = ops[o].pos[i + 1]; }
            else {
                q[o] = cc[o];
                while (cc[o] < ops[o].nnz && ops[o].outer_crd[cc[o]] == i) cc[o]++;
                e[o] = cc[o];
            }
        }
        for (;;) {
            int64_t j = -1;
            for (int32_t o = 0; o < k; o++) if (q[o] < e[o] && (j < 0 || ops[o].crd[q[o]] < j)) j = ops[o].crd[q[o]];
            if (j < 0) break;
            double vd = 0.0; float vf = 0.0f; int have = 0;
            for (int32_t o = 0; o < k; o++) {
                if (q[o] < e[o] && ops[o].crd[q[o]] == j) {
                    if (f64) { double a = ((const double *)ops[o].val)[q[o]]; vd = have ? vd + a : a; }
                    else     { float  a = ((const float *)ops[o].val)[q[o]];  vf = have ? vf + a : a; }
                    have = 1;
                    q[o]++;
                }
            }
            if (nz >= capacity) { free(q); free(e); free(cc); return -1; }
            z_crd[nz] = (int32_t)j;
            if (f64) ((double *)z_val)[nz] = vd; else ((float *)z_val)[nz] = vf;
            nz++;
        }
        z_pos[i + 1] = nz;
    }
    free(q); free(e); free(cc);
    return nz;
}

/* ------------------------------------------------------ third-order CSF (3-level Alg. 1) */
static int64_t lb32(const int32_t *a, int64_t lo, int64_t hi, int64_t x) {   /* least i in [lo, hi] with a[i] >= x */
    while (lo < hi) { int64_t m = lo + (hi - lo) / 2; if ((int64_t)a[m] >= x) hi = m; else lo = m + 1; }
    return lo;
}

/* C_i(x_i) = entries of slices i < x_i; C_j(x_j | x_i) = entries of slice x_i in fibers j < x_j;
 * C_k(x_k | x_i, x_j) = entries of fiber (x_i, x_j) with k < x_k -- summed over the operands
 * (the nnz cost functions of P:1689 on the levels of fig:coordinate-tree). */
void oracle_csf_cost(int32_t k, const or_tensor3 *ops, int64_t xi, int64_t xj, int64_t xk, int64_t *ci, int64_t *cj,
                     int64_t *ck) {
    *ci = *cj = *ck = 0;
    for (int32_t o = 0; o < k; o++) {
        const or_tensor3 *T = &ops[o];
        const int64_t s = lb32(T->crd0, 0, T->n_slices, xi);
        *ci += T->pos2[T->pos1[s]];
        if (s < T->n_slices && T->crd0[s] == xi) {
            const int64_t f = lb32(T->crd1, T->pos1[s], T->pos1[s + 1], xj);
            *cj += T->pos2[f] - T->pos2[T->pos1[s]];
            if (f < T->pos1[s + 1] && T->crd1[f] == xj)
                *ck += lb32(T->crd2, T->pos2[f], T->pos2[f + 1], xk) - T->pos2[f];
        }
    }
}

/* The entries of every operand enumerated in lexicographic (i, j, k) order by a 3-level k-finger
 * merge (Listing 1's union form); b_p = entry number Q_p (R1-R4 as in oracle_partition_rank). */
int oracle_csf_partition_rank(int32_t k, const or_tensor3 *ops, int32_t P, or_parts *out) {
    if (k < 1 || P < 1) return 1;
    int64_t qstar = 0;
    for (int32_t o = 0; o < k; o++) qstar += ops[o].nnz;
    oracle_queries(qstar, P, out->query);
    int64_t *q = (int64_t *)calloc((size_t)k, sizeof(int64_t));
    int64_t *f = (int64_t *)calloc((size_t)k, sizeof(int64_t));
    int64_t *sl = (int64_t *)calloc((size_t)k, sizeof(int64_t));
    int64_t c = 0;
    int32_t p = 1;
    while (p < P) {
        int64_t bi = -1, bj = -1, bk = -1;
        for (int32_t o = 0; o < k; o++) {
            if (q[o] >= ops[o].nnz) continue;
            while (ops[o].pos2[f[o] + 1] <= q[o]) f[o]++;
            while (ops[o].pos1[sl[o] + 1] <= f[o]) sl[o]++;
            const int64_t i = ops[o].crd0[sl[o]], j = ops[o].crd1[f[o]], kk = ops[o].crd2[q[o]];
            if (bi < 0 || i < bi || (i == bi && (j < bj || (j == bj && kk < bk)))) { bi = i; bj = j; bk = kk; }
        }
        if (bi < 0) break;
        int32_t g = 0;
        for (int32_t o = 0; o < k; o++)
            if (q[o] < ops[o].nnz && ops[o].crd0[sl[o]] == bi && ops[o].crd1[f[o]] == bj && ops[o].crd2[q[o]] == bk) g++;
        while (p < P && out->query[p] < c + g) {
            out->row[p] = bi; out->row_pos[p] = bj; out->col[p] = (int32_t)bk;
            for (int32_t o = 0; o < k; o++) out->pos[(int64_t)p * k + o] = q[o];
            p++;
        }
        for (int32_t o = 0; o < k; o++)
            if (q[o] < ops[o].nnz && ops[o].crd0[sl[o]] == bi && ops[o].crd1[f[o]] == bj && ops[o].crd2[q[o]] == bk) q[o]++;
        c += g;
    }
    for (; p <= P; p++) {   /* end: (n0, 0, 0), every operand exhausted */
        out->row[p] = ops[0].n0; out->row_pos[p] = 0; out->col[p] = 0;
        for (int32_t o = 0; o < k; o++) out->pos[(int64_t)p * k + o] = ops[o].nnz;
    }
    out->row[0] = 0; out->row_pos[0] = 0; out->col[0] = 0;
    for (int32_t o = 0; o < k; o++) out->pos[o] = 0;
    free(q); free(f); free(sl);
    return 0;
}

/* Z = sum_o A_o, three nested union loops (Listing 2 with one more level), left fold (R9). */
int64_t oracle_csf_spadd_k(int32_t k, const or_tensor3 *ops, int32_t *z_crd0, int64_t *z_pos1, int32_t *z_crd1,
                           int64_t *z_pos2, int32_t *z_crd2, void *z_val, int64_t cap_s, int64_t cap_f, int64_t cap_e,
                           int64_t *counts) {
    const int f64 = ops[0].dtype == OR_F64;
    int64_t *s = (int64_t *)calloc((size_t)k, sizeof(int64_t));   /* slice cursors */
    int64_t *f = (int64_t *)calloc((size_t)k, sizeof(int64_t)), *fe = (int64_t *)calloc((size_t)k, sizeof(int64_t));
    int64_t *q = (int64_t *)calloc((size_t)k, sizeof(int64_t)), *qe = (int64_t *)calloc((size_t)k, sizeof(int64_t));
    int64_t ns = 0, nf = 0, ne = 0;
    z_pos1[0] = 0; z_pos2[0] = 0;
    for (;;) {
        int64_t i = -1;
        for (int32_t o = 0; o < k; o++) if (s[o] < ops[o].n_slices && (i < 0 || ops[o].crd0[s[o]] < i)) i = ops[o].crd0[s[o]];
        if (i < 0) break;
        for (int32_t o = 0; o < k; o++) {
            if (s[o] < ops[o].n_slices && ops[o].crd0[s[o]] == i) { f[o] = ops[o].pos1[s[o]]; fe[o] = ops[o].pos1[s[o] + 1]; }
            else { f[o] = fe[o] = 0; }
        }
        for (;;) {
            int64_t j = -1;
            for (int32_t o = 0; o < k; o++) if (f[o] < fe[o] && (j < 0 || ops[o].crd1[f[o]] < j)) j = ops[o].crd1[f[o]];
            if (j < 0) break;
            for (int32_t o = 0; o < k; o++) {
                if (f[o] < fe[o] && ops[o].crd1[f[o]] == j) { q[o] = ops[o].pos2[f[o]]; qe[o] = ops[o].pos2[f[o] + 1]; }
                else { q[o] = qe[o] = 0; }
            }
            for (;;) {
                int64_t kk = -1;
                for (int32_t o = 0; o < k; o++) if (q[o] < qe[o] && (kk < 0 || ops[o].crd2[q[o]] < kk)) kk = ops[o].crd2[q[o]];
                if (kk < 0) break;
                double vd = 0.0; float vf = 0.0f; int have = 0;
                for (int32_t o = 0; o < k; o++) {
                    if (q[o] < qe[o] && ops[o].crd2[q[o]] == kk) {
                        if (f64) { double a = ((const double *)ops[o].val)[q[o]]; vd = have ? vd + a : a; }
                        else     { float  a = ((const float *)ops[o].val)[q[o]];  vf = have ? vf + a : a; }
                        have = 1; q[o]++;
                    }
                }
                if (ne >= cap_e) goto overflow;
                z_crd2[ne] = (int32_t)kk;
                if (f64) ((double *)z_val)[ne] = vd; else ((float *)z_val)[ne] = vf;
                ne++;
            }
            if (nf >= cap_f) goto overflow;
            z_crd1[nf] = (int32_t)j;
            z_pos2[nf + 1] = ne;
            nf++;
            for (int32_t o = 0; o < k; o++) if (f[o] < fe[o] && ops[o].crd1[f[o]] == j) f[o]++;
        }
        if (ns >= cap_s) goto overflow;
        z_crd0[ns] = (int32_t)i;
        z_pos1[ns + 1] = nf;
        ns++;
        for (int32_t o = 0; o < k; o++) if (s[o] < ops[o].n_slices && ops[o].crd0[s[o]] == i) s[o]++;
    }
    counts[0] = ns; counts[1] = nf; counts[2] = ne;
    free(s); free(f); free(fe); free(q); free(qe);
    return ne;
overflow:
    free(s); free(f); free(fe); free(q); free(qe);
    return -1;
}


/* ---------------------------------------------------------------- ESC scatter kernels (SpGEMM, SSSMM) */
/* Appends versus scatters: a kernel that scatters into a sparse output (SpGEMM
 * C_ij = sum_k A_ik B_kj over the loop order i -> k -> j) is run as expand-sort-contract (ESC):
 * the expansion T materialises every product A_ik * B_kj with its coordinate (i, j) -- rows i
 * ascending, A positions q ascending within a row, B positions ascending within row k of B --, a
 * sort by (i, j) turns the reduction into a segmented reduction, and the contraction folds every
 * run of equal coordinates.  The load balancing applies to the expansion only. */

/* The cost of the expansion, the broadcast-scaled cost of Listing 6:
 * A's entry q at (i, k) is coiterated with the whole row k of B (B's j level is not indexed by A),
 * so it costs nnz(B_k).  W[q] = sum_{q' < q} nnz(B_{A.crd[q']}) for q in [0, nnz(A)]; returns
 * Q* = W[nnz(A)] (the number of products), or -1 if the shapes disagree. */
int64_t oracle_spgemm_work(const or_matrix *A, const or_matrix *B, int64_t *W) {
    if (A->format != OR_CSR || B->format != OR_CSR || A->ncols != B->nrows) return -1;
    int64_t w = 0;
    for (int64_t q = 0; q < A->nnz; q++) {
        W[q] = w;
        const int64_t k = A->crd[q];
        w += B->pos[k + 1] - B->pos[k];
    }
    W[A->nnz] = w;
    return w;
}

/* Partition of the expansion by its definition (Q_p of P:1089-1093 over the cost W): b_p locates
 * product number Q_p of T -- row[p] = its row i, pos[2p] = the A position q that produces it,
 * pos[2p+1] = its B position, col[p] = its column j, row_pos[p] = row[p] (CSR).  A query at or past
 * Q* gives the end (nrows, nnz(A), nnz(B), col 0).  k = 2 in the record.  Returns 0, or 1 on a bad
 * argument. */
int oracle_esc_partition(const or_matrix *A, const or_matrix *B, int32_t P, or_parts *out) {
    if (P < 1 || A->format != OR_CSR || B->format != OR_CSR || A->ncols != B->nrows) return 1;
    int64_t *W = (int64_t *)malloc(sizeof(int64_t) * (size_t)(A->nnz + 1));
    const int64_t qstar = oracle_spgemm_work(A, B, W);
    oracle_queries(qstar, P, out->query);
    int64_t q = 0, i = 0;
    for (int32_t p = 0; p <= P; p++) {
        const int64_t Q = out->query[p];
        if (Q >= qstar) {
            out->row[p] = A->nrows; out->row_pos[p] = A->nrows; out->col[p] = 0;
            out->pos[2 * (int64_t)p] = A->nnz; out->pos[2 * (int64_t)p + 1] = B->nnz;
            continue;
        }
        while (W[q + 1] <= Q) q++;               /* the entry with W[q] <= Q < W[q + 1] */
        while (A->pos[i + 1] <= q) i++;          /* its row */
        const int64_t bp = B->pos[A->crd[q]] + (Q - W[q]);
        out->row[p] = i; out->row_pos[p] = i; out->col[p] = B->crd[bp];
        out->pos[2 * (int64_t)p] = q; out->pos[2 * (int64_t)p + 1] = bp;
    }
    free(W);
    return 0;
}

static int cmp_i32(const void *a, const void *b) {
    const int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    return (x > y) - (x < y);
}

/* C = A B, CSR x CSR -> CSR, with ESC's result: C stores (i, j) iff some k has A_ik and B_kj stored
 * (structurally, whatever the sum); the value is the left fold over k ascending (the order a stable
 * sort of T by (i, j) keeps) of the products A_ik * B_kj, each rounded in the value type, starting
 * from the first product (reading R23).  Row by row with a dense accumulator (Gustavson's order,
 * the same fold).  Returns nnz(C), or -1 (shape / capacity). */
int64_t oracle_spgemm(const or_matrix *A, const or_matrix *B, int64_t *c_pos, int32_t *c_crd, void *c_val,
                      int64_t cap) {
    if (A->format != OR_CSR || B->format != OR_CSR || A->ncols != B->nrows) return -1;
    const int f64 = A->dtype == OR_F64;
    const int64_t N = B->ncols;
    int64_t *stamp = (int64_t *)malloc(sizeof(int64_t) * (size_t)(N > 0 ? N : 1));
    double *accd = (double *)malloc(sizeof(double) * (size_t)(N > 0 ? N : 1));
    float *accf = (float *)malloc(sizeof(float) * (size_t)(N > 0 ? N : 1));
    int32_t *cols = (int32_t *)malloc(sizeof(int32_t) * (size_t)(N > 0 ? N : 1));
    for (int64_t j = 0; j < N; j++) stamp[j] = -1;
    int64_t nz = 0;
    c_pos[0] = 0;
    for (int64_t i = 0; i < A->nrows; i++) {
        int64_t nc = 0;
        for (int64_t q = A->pos[i]; q < A->pos[i + 1]; q++) {
            const int64_t k = A->crd[q];
            for (int64_t r = B->pos[k]; r < B->pos[k + 1]; r++) {
                const int64_t j = B->crd[r];
                const int first = stamp[j] != i;
                if (first) { stamp[j] = i; cols[nc++] = (int32_t)j; }
                if (f64) {
                    const double t = ((const double *)A->val)[q] * ((const double *)B->val)[r];
                    accd[j] = first ? t : accd[j] + t;
                } else {
                    const float t = ((const float *)A->val)[q] * ((const float *)B->val)[r];
                    accf[j] = first ? t : accf[j] + t;
                }
            }
        }
        qsort(cols, (size_t)nc, sizeof(int32_t), cmp_i32);
        if (nz + nc > cap) { nz = -1; break; }
        for (int64_t u = 0; u < nc; u++) {
            const int32_t j = cols[u];
            c_crd[nz] = j;
            if (f64) ((double *)c_val)[nz] = accd[j]; else ((float *)c_val)[nz] = accf[j];
            nz++;
        }
        c_pos[i + 1] = nz;
    }
    free(stamp); free(accd); free(accf); free(cols);
    return nz;
}

/* Sampled SpGEMM (SSSMM): Z = S (.) (A B).  Z stores (i, j) iff S stores it and C = A B
 * stores it structurally; Z_ij = S_ij * C_ij with C_ij the ESC fold of oracle_spgemm (reading R24:
 * the sampling restricts the expansion to j in S_i, which leaves the products of every kept (i, j)
 * and their order unchanged, and the sampled value scales the contracted sum).  Returns nnz(Z) or
 * -1. */
int64_t oracle_sssmm(const or_matrix *S, const or_matrix *A, const or_matrix *B, int64_t *z_pos, int32_t *z_crd,
                     void *z_val, int64_t cap) {
    if (S->format != OR_CSR || S->nrows != A->nrows || S->ncols != B->ncols || S->dtype != A->dtype) return -1;
    int64_t cap_c = 0;
    for (int64_t q = 0; q < A->nnz; q++) cap_c += B->pos[A->crd[q] + 1] - B->pos[A->crd[q]];
    const int f64 = A->dtype == OR_F64;
    int64_t *c_pos = (int64_t *)malloc(sizeof(int64_t) * (size_t)(A->nrows + 1));
    int32_t *c_crd = (int32_t *)malloc(sizeof(int32_t) * (size_t)(cap_c > 0 ? cap_c : 1));
    void *c_val = malloc((f64 ? 8 : 4) * (size_t)(cap_c > 0 ? cap_c : 1));
    int64_t nz = oracle_spgemm(A, B, c_pos, c_crd, c_val, cap_c);
    if (nz < 0) goto out;
    nz = 0;
    z_pos[0] = 0;
    for (int64_t i = 0; i < S->nrows; i++) {
        int64_t s = S->pos[i], c = c_pos[i];
        while (s < S->pos[i + 1] && c < c_pos[i + 1]) {
            if (S->crd[s] < c_crd[c]) { s++; continue; }
            if (S->crd[s] > c_crd[c]) { c++; continue; }
            if (nz >= cap) { nz = -1; goto out; }
            z_crd[nz] = S->crd[s];
            if (f64) ((double *)z_val)[nz] = ((const double *)S->val)[s] * ((const double *)c_val)[c];
            else     ((float *)z_val)[nz]  = ((const float *)S->val)[s] * ((const float *)c_val)[c];
            nz++; s++; c++;
        }
        z_pos[i + 1] = nz;
    }
out:
    free(c_pos); free(c_crd); free(c_val);
    return nz;
}
