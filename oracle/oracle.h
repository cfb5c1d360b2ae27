/*
 * oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, single-threaded CPU oracle for the data-parallel hot path of
 * Chougule et al., "Partitioning Unstructured Sparse Tensor Algebra for
 * Load-Balanced Parallel Execution" (arXiv 2604.17198, "Nacho").  Citations
 * "P:<line>" refer to /root/reference/PAPER.md.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library.  It shares no code, header, helper or constant with the
 * CUDA path (paper_2604_17198_b200/); it defines its own types below.
 *
 * Conventions:
 *   positions (pos) int64, coordinates in crd int32, row coordinates int64,
 *   values fp32 (dtype 0) or fp64 (dtype 1).
 */
#ifndef NACHO_ORACLE_H
#define NACHO_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OR_CSR  0
#define OR_DCSR 1
#define OR_COO  2   /* Compressed(non-unique) o Singleton: pos = [0, nnz], outer_crd = row of every entry */
#define OR_F32  0
#define OR_F64  1

typedef struct {
    int32_t        format;     /* OR_CSR (Dense o Compressed) or OR_DCSR (Compressed o Compressed) */
    int32_t        dtype;      /* OR_F32 / OR_F64 */
    int64_t        nrows, ncols, nnz;
    int64_t        nouter;     /* CSR: nrows; DCSR: number of stored rows */
    const int32_t *outer_crd;  /* DCSR only: [nouter] stored row coordinates, strictly increasing */
    const int64_t *pos;        /* [nouter+1] */
    const int32_t *crd;        /* [nnz] */
    const void    *val;        /* [nnz] */
} or_matrix;

typedef struct {
    int32_t  P, k;
    int64_t *query;    /* [P+1] Q_p */
    int64_t *row;      /* [P+1] boundary row coordinate */
    int64_t *row_pos;  /* [P+1] outer-level position of the boundary (CSR: == row) */
    int32_t *col;      /* [P+1] boundary column coordinate */
    int64_t *pos;      /* [(P+1)*k] per-operand positions */
} or_parts;

/* 0 if the operand satisfies the format invariants of P:1675-1684 (sorted levels), else a code > 0 */
int     oracle_validate(const or_matrix *A);
int64_t oracle_total_cost(int32_t k, const or_matrix *ops);
void    oracle_queries(int64_t qstar, int32_t P, int64_t *Q);

/* Partition boundaries by the plain definition (rank of the Q-th entry of the lexicographic
 * multiset of all stored entries).  Returns 0 on success. */
int     oracle_partition_rank(int32_t k, const or_matrix *ops, int32_t P, or_parts *out);
/* Partition boundaries by literal Alg. 1 in the Listing 7 form.
 * probes[p] (optional) receives the number of cost-function evaluations for boundary p. */
int     oracle_partition_alg1(int32_t k, const or_matrix *ops, int32_t P, or_parts *out, int64_t *probes);
/* lb_search of Listing 7: least position in [lo, hi] with crd[pos] >= x, or hi+1. */
int64_t oracle_lb_search(const int32_t *crd, int64_t lo, int64_t hi, int64_t x);

/* y = A x.  CSR: y[nrows]; DCSR: compressed y[nouter] aligned with outer_crd.  Wide accumulation. */
int     oracle_spmv(const or_matrix *A, const void *x, void *y);
/* C = A B, B [ncols x nb] with leading dimension ldb, C [nrows x nb] with ldc (CSR only). */
int     oracle_spmm(const or_matrix *A, const void *B, int64_t ldb, int32_t nb, void *C, int64_t ldc);
/* Z = sum_o ops[o] (k-way structural union, CSR).  Z.pos[nrows+1]; z_crd/z_val need capacity >= nnz_Z.
 * Values: left fold in operand order starting from the first present value.  Returns nnz_Z, or -1. */
int64_t oracle_spadd_k(int32_t k, const or_matrix *ops, int64_t *z_pos, int32_t *z_crd, void *z_val, int64_t capacity);
/* Per-partition union counts for given boundaries: cnt[p] = #union coordinates c with b_p <=lex c <lex b_{p+1}. */
int     oracle_spadd_counts(int32_t k, const or_matrix *ops, const or_parts *parts, int64_t *cnt);

/* Z = ops[0] (.) ... (.) ops[k-1] (k-way structural intersection, CSR; Listing 1's k-finger merge per
 * row).  Values: product in operand order, left to right, in the value type.  Returns nnz_Z, or -1. */
int64_t oracle_hadamard_k(int32_t k, const or_matrix *ops, int64_t *z_pos, int32_t *z_crd, void *z_val,
                          int64_t capacity);
/* Per-partition intersection counts for given boundaries. */
int     oracle_hadamard_counts(int32_t k, const or_matrix *ops, const or_parts *parts, int64_t *cnt);
/* s = sum over the intersection of the products (wide accumulation, rounded once to double). */
int     oracle_inner_k(int32_t k, const or_matrix *ops, double *out);

/* Recursive partitioning (Alg. 2) of the DCSR Hadamard product, Listing emul-dcsr2-rewritten: */
/* lines 2-3: surviving rows, T, outer positions ip[o * cap + s]; returns S or -1 */
int64_t oracle_dcsr_rows_intersect(int32_t k, const or_matrix *ops, int64_t *rows, int64_t *T, int64_t *ip,
                                   int64_t cap);
/* line 4: T' (S + 1 entries) */
void    oracle_exclusive_prefix(const int64_t *T, int64_t S, int64_t *Tp);
/* lines 5-6: the remapped partition (row_pos = surviving-row index) */
int     oracle_partition_remapped(int32_t k, const or_matrix *ops, int64_t S, const int64_t *rows, const int64_t *ip,
                                  int64_t cap, const int64_t *Tp, int32_t P, or_parts *out);
/* lines 7-9: Z over the surviving rows (z_pos[S + 1]); returns nnz_Z or -1 */
int64_t oracle_dcsr_hadamard(int32_t k, const or_matrix *ops, int64_t S, const int64_t *ip, int64_t cap,
                             int64_t *z_pos, int32_t *z_crd, void *z_val, int64_t zcap);

/* Z = sum_o ops[o] on DCSR operands (Listing 2): Z DCSR over the union of the stored rows; returns
 * nnz_Z (z_nrows = stored rows of Z) or -1 */
int64_t oracle_dcsr_spadd_k(int32_t k, const or_matrix *ops, int32_t *z_outer, int64_t *z_pos, int32_t *z_crd,
                            void *z_val, int64_t *z_nrows, int64_t rcap, int64_t zcap);
/* per-partition union entries and rows started, DCSR operands */
int     oracle_dcsr_spadd_counts(int32_t k, const or_matrix *ops, const or_parts *parts, int64_t *ent, int64_t *rows);

/* Z = sum_o ops[o] for CSR and COO operands mixed (the COO + CSR addition of P:2449-2470): the
 * union per row, left fold; Z is CSR (z_pos[nrows + 1]).  Returns nnz_Z or -1. */
int64_t oracle_mixed_spadd_k(int32_t k, const or_matrix *ops, int64_t *z_pos, int32_t *z_crd, void *z_val,
                             int64_t capacity);

/* A third-order tensor in CSF (Compressed o Compressed o Compressed, P:846-1030 coordinate tree):
 * slices crd0[n_slices] (i), fibers pos1[n_slices+1] / crd1[n_fibers] (j), entries pos2[n_fibers+1] /
 * crd2[nnz] (k), val[nnz]. */
typedef struct {
    int32_t        dtype;
    int64_t        n0, n1, n2, nnz, n_slices, n_fibers;
    const int32_t *crd0;
    const int64_t *pos1;
    const int32_t *crd1;
    const int64_t *pos2;
    const int32_t *crd2;
    const void    *val;
} or_tensor3;

/* The cost of coordinate (x_i, x_j, x_k) over k CSF operands: entries lexicographically before it,
 * split as C_i(x_i) + C_j(x_j | x_i) + C_k(x_k | x_i, x_j) (fig:coordinate-tree). */
void    oracle_csf_cost(int32_t k, const or_tensor3 *ops, int64_t xi, int64_t xj, int64_t xk, int64_t *ci, int64_t *cj,
                        int64_t *ck);
/* Partition boundaries of k CSF operands by the rank definition: row = i, row_pos = j, col = k,
 * pos[o] = level-2 positions (entries of operand o before the boundary). */
int     oracle_csf_partition_rank(int32_t k, const or_tensor3 *ops, int32_t P, or_parts *out);
/* Z = sum_o ops[o] (3-level union, left fold) in CSF; counts[0..2] = slices, fibers, nnz.  -1 on
 * capacity overflow. */
int64_t oracle_csf_spadd_k(int32_t k, const or_tensor3 *ops, int32_t *z_crd0, int64_t *z_pos1, int32_t *z_crd1,
                           int64_t *z_pos2, int32_t *z_crd2, void *z_val, int64_t cap_s, int64_t cap_f, int64_t cap_e,
                           int64_t *counts);

/* ESC scatter kernels: SpGEMM C = A B over i -> k -> j and sampled SpGEMM Z = S (.) (A B).
 * W[nnz(A)+1]: exclusive prefix of nnz(B_{A.crd[q]}) (Listing 6's broadcast-scaled cost); returns Q*. */
int64_t oracle_spgemm_work(const or_matrix *A, const or_matrix *B, int64_t *W);
/* b_p = location of product number Q_p of the expansion (k = 2 record: pos = A position, B position). */
int     oracle_esc_partition(const or_matrix *A, const or_matrix *B, int32_t P, or_parts *out);
/* C = A B (CSR): structural product, left fold over k ascending in the value type; nnz(C) or -1. */
int64_t oracle_spgemm(const or_matrix *A, const or_matrix *B, int64_t *c_pos, int32_t *c_crd, void *c_val,
                      int64_t cap);
/* Z = S (.) (A B): Z_ij = S_ij * C_ij on the stored coordinates of both; nnz(Z) or -1. */
int64_t oracle_sssmm(const or_matrix *S, const or_matrix *A, const or_matrix *B, int64_t *z_pos, int32_t *z_crd,
                     void *z_val, int64_t cap);

#ifdef __cplusplus
}
#endif
#endif
