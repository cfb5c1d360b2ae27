/*
 * nacho.h -- C ABI of libnacho.so: load-balanced partitioning of sparse tensor algebra and the
 * partitioned kernels that execute over it, on NVIDIA B200 (sm_100a).
 *
 * Paper: Chougule, Root, Lacouture, Yan, Yadav, Kjolstad, "Partitioning Unstructured Sparse Tensor
 * Algebra for Load-Balanced Parallel Execution" (arXiv 2604.17198).  P:<n> = PAPER.md line n.
 *
 * Conventions for every entry point
 *   - All array pointers are DEVICE pointers, borrowed: the caller allocates and owns them (e.g.
 *     torch tensors).  Inputs are read-only during the call; outputs must not alias inputs.
 *   - Calls are asynchronous on `stream` (a cudaStream_t passed as void*); none synchronises the host.
 *   - The library holds no device allocations; scratch space is the caller's `ws` of at least
 *     *_workspace_size() bytes (pass NULL/0 when the size is 0).
 *   - Argument errors are detected on the host before any launch and return a status != 0; the
 *     message is available from nacho_last_error() (thread-local).  Launch failures return
 *     NACHO_ERR_CUDA.  No C++ exception crosses this ABI.
 *   - Types (reading R11): positions int64, column coordinates int32, row coordinates int64, values
 *     fp32 or fp64.
 */
#ifndef NACHO_H
#define NACHO_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  NACHO_SUCCESS = 0,
  NACHO_ERR_INVALID_ARG = 1, /* null pointer, P < 1, k outside [1, NACHO_MAX_K], unsupported dtype/format */
  NACHO_ERR_SHAPE = 2,       /* operand shapes disagree (k-way ops), or x / B do not match A */
  NACHO_ERR_FORMAT = 3,      /* nacho_validate found a violated sorted-level invariant */
  NACHO_ERR_OVERFLOW = 4,    /* nrows or ncols > INT32_MAX, or a count does not fit the index types */
  NACHO_ERR_WORKSPACE = 5,   /* ws_bytes smaller than the *_workspace_size() result */
  NACHO_ERR_CUDA = 6,        /* a launch or CUDA runtime call failed */
  NACHO_ERR_NCCL = 7         /* NCCL not loadable, or an NCCL call failed (multi-GPU calls only) */
} nacho_status;

typedef enum { NACHO_CSR = 0, NACHO_DCSR = 1, NACHO_COO = 2 } nacho_format;
typedef enum { NACHO_F32 = 0, NACHO_F64 = 1 } nacho_dtype;

#define NACHO_MAX_K 8

/* A sparse matrix in a TACO level format:
 *   CSR  = Dense(rows) o Compressed(cols)       -- pos[nrows+1], crd[nnz]
 *   DCSR = Compressed(rows) o Compressed(cols)  -- outer_crd[nouter], pos[nouter+1]
 * pos[0] = 0, pos non-decreasing, pos[nouter] = nnz; crd strictly increasing within each row
 * segment and < ncols; DCSR outer_crd strictly increasing and every stored row non-empty (R10).
 *   COO  = Compressed(non-unique)(rows) o Singleton(cols): nouter = 1, pos = [0, nnz],
 *          outer_crd[nnz] = the row of every entry (sorted by (row, col), no duplicates).  COO operands
 *          are taken by nacho_partition and nacho_mixed_spadd_k (mixed with CSR operands) only. */
typedef struct {
  int32_t format;            /* nacho_format */
  int32_t dtype;             /* nacho_dtype of val */
  int64_t nrows, ncols, nnz;
  int64_t nouter;            /* CSR: == nrows; DCSR: number of stored rows */
  const int32_t* outer_crd;  /* DCSR: [nouter]; CSR: NULL */
  const int64_t* pos;        /* [nouter + 1] */
  const int32_t* crd;        /* [nnz] */
  const void* val;           /* [nnz] */
} nacho_matrix;

/* The partition record `Parts` of Listing 7 and Listing 8 (p.i, p.jpA, p.jpB;
 * P:2120-2126), as structure-of-arrays of P+1 boundaries.  Partition p covers the lexicographic
 * coordinate range [b_p, b_{p+1}).  b_0 is the origin (row 0, col 0, pos 0) and b_P the end
 * (row nrows, row_pos nouter, col 0, pos[o] = nnz_o) -- reading R1.  All arrays caller-allocated. */
typedef struct {
  int32_t P;         /* number of partitions (>= 1) */
  int32_t k;         /* number of sparse operands coiterated */
  int64_t* query;    /* [P+1]  Q_p = floor(p * Q* / P)                                (R4) */
  int64_t* row;      /* [P+1]  boundary row coordinate x_i                             (Alg. 1) */
  int64_t* row_pos;  /* [P+1]  outer-level position of x_i (CSR: == row; DCSR: index into outer_crd) */
  int32_t* col;      /* [P+1]  boundary column coordinate x_j                          (Alg. 1) */
  int64_t* pos;      /* [(P+1)*k] pos[p*k+o] = #entries of operand o before b_p        (P:1795 p.ipA) */
  int64_t max_work;  /* host-side bound on any partition's work (entries over the operands): written by
                        nacho_partition / nacho_partition_slice as ceil(Q* / P) + k - 1 (Theorem 1,
                        P:1146-1161); 0 = unknown -- calls that need it then read the record's first and
                        last query (a synchronising 16-byte copy) */
} nacho_parts;

/* ------------------------------------------------------------------------------------------------
 * nacho_partition -- Alg. 1 "FindPartition" run for every boundary p = 0..P with the
 * query Q_p = floor(p*Q* /P), Q* = sum_o nnz_o, using the CSR / DCSR
 * cost functions of Listing 5 and the position-space specialisation of Listing 7
 * (P:1752-1799).  One warp per boundary performs a 32-ary search over the row level and, for k > 1,
 * a k-way order-statistic search over the row's column segments (matching coordinates of different
 * operands always land on the same side of a cut).  Result: the unique highest
 * coordinate with cost <= Q_p (Theorem 1: 0 <= Q_p - C(b_p) < k).
 *   ops   host array of k operand descriptors (device arrays inside); all must share format, nrows
 *         and ncols.  DCSR requires k == 1.
 *   out   caller-allocated device arrays for P+1 boundaries; out->P and out->k must equal P and k.
 * Errors: INVALID_ARG (k, P, nulls, DCSR with k > 1), SHAPE (mismatched operands), OVERFLOW. */
nacho_status nacho_partition(const nacho_matrix* ops, int32_t k, int32_t P, nacho_parts* out, void* stream);

/* nacho_partition_slice -- the boundaries p_begin .. p_begin + out->P of the P-partition (the same
 * values nacho_partition writes at those indices), into out[0 .. out->P]: a device's share of a
 * device-level cut (device d runs partitions [d P_l, (d+1) P_l) of P = D P_l), so each
 * device searches only its own P_l + 1 boundaries.  The queries stay Q_p = floor(p Q* / P).
 * Errors: as nacho_partition; INVALID_ARG when [p_begin, p_begin + out->P] leaves [0, P]. */
nacho_status nacho_partition_slice(const nacho_matrix* ops, int32_t k, int32_t P, int32_t p_begin, nacho_parts* out,
                                   void* stream);

/* Partition count the kernels below pick when the caller does not fix P: ceil(Q* / tile), tile being
 * the per-CTA work of the kernel for that operation (op: 0 spmv, 1 spadd, 2 spmm). */
int32_t nacho_auto_partitions(const nacho_matrix* ops, int32_t k, int32_t op);
/* The largest partition (entries summed over the k operands) the single-read SpAdd / intersection
 * kernels take: a stage of 256 x 8 slots minus the bulk-copy pads (7 per operand); 0 for a bad k. */
int32_t nacho_spadd_tile(int32_t k);

/* ------------------------------------------------------------------------------------------------
 * nacho_spmv -- y = A x over a partition of A (SpMV is the broadcast example of P:1742-1744; the
 * per-partition loop bounds follow Listing 8).  Partition p streams the positions
 * [parts.pos[p], parts.pos[p+1]); rows finished inside p are written by p (ownership rule R7: p
 * owns rows [b_p.row, b_{p+1}.row - 1], empty rows are written as 0); a row cut by a boundary
 * leaves a carry that a fix-up kernel adds in partition order.
 *   A       CSR or DCSR, fp32 or fp64.
 *   parts   a partition of A with k == 1 (from nacho_partition), or NULL: the library then computes
 *           one with nacho_auto_partitions(A, 1, 0) partitions inside `ws`.
 *   x       [ncols] dense, dtype of A.
 *   y       CSR: [nrows].  DCSR: [nouter] compressed y aligned with outer_crd (R12), or [nrows]
 *           when dense_y != 0 (then rows not stored are written as 0).
 *   ws      >= nacho_spmv_workspace_size(A, parts ? parts->P : 0) bytes (carries [+ parts]).
 * Numerics: products and sums in the value type; summation order differs from the sequential one
 * (R13), so results agree with the oracle to 1e-5 (fp32) / 1e-12 (fp64) relative to sum|a*x|. */
size_t nacho_spmv_workspace_size(const nacho_matrix* A, int32_t P);
nacho_status nacho_spmv(const nacho_matrix* A, const nacho_parts* parts, const void* x, void* y, int32_t dense_y,
                        void* ws, size_t ws_bytes, void* stream);

/* ------------------------------------------------------------------------------------------------
 * k-way SpAdd Z = A_0 + ... + A_{k-1} (CSR, union coiteration of Listing 2), assembled in
 * the paper's two passes (Fig. 7a):
 *   nacho_spadd_k_count : per partition, symbolic k-way union merge -> cnt_p; exclusive prefix sum
 *                         -> part_off[0..P] with part_off[P] = nnz_Z.
 *   (caller reads part_off[P], allocates z_crd / z_val of nnz_Z entries -- the one host sync)
 *   nacho_spadd_k_fill  : re-merge, write (col, value) at part_off[p] and the Z.pos entries of the
 *                         rows partition p owns (guarded single writer, R7).
 * Z.pos[0] = 0.  Values: left fold in operand order of the present values (R9), in the value type --
 * bit-identical to the oracle.  Structural zeros are kept (symbolic assembly).
 *   ops      k CSR operands of identical shape and dtype.   parts: k-operand partition of ops.
 *   part_off [P+1] int64 (device).   z_pos [nrows+1] int64.   z_crd [nnz_Z] int32, z_val [nnz_Z].
 *   ws       >= nacho_spadd_k_workspace_size(ops, k, P). */
size_t nacho_spadd_k_workspace_size(const nacho_matrix* ops, int32_t k, int32_t P);
/* nacho_spadd_k -- the same Z in ONE pass: every partition merges its staged operand ranges once,
 * obtains its write offset from a decoupled look-back over the partitions (single-pass prefix
 * sum) and writes Z immediately, so assembly and compute share one read of the operands
 * and no host round trip separates them.  z_crd / z_val must hold Q* = sum_o nnz_o entries (an
 * upper bound of nnz_Z, reading "Allocation" of Fig. 7a as an upper-bound allocation); nnz_Z is
 * z_pos[nrows] (and part_off[P] when part_off != NULL, which then receives every partition's
 * offset).  Partitions must hold at most 2048 entries (nacho_auto_partitions(ops, k, 1) does);
 * larger ones return NACHO_ERR_INVALID_ARG -- use the two-pass calls.
 *   ws  >= nacho_spadd_k_workspace_size(ops, k, P) bytes (look-back flags). */
nacho_status nacho_spadd_k(const nacho_matrix* ops, int32_t k, const nacho_parts* parts, int64_t* part_off,
                           int64_t* z_pos, int32_t* z_crd, void* z_val, void* ws, size_t ws_bytes, void* stream);
/* nacho_spadd_k_staged -- the same Z with one read of the operands and no look-back: every partition
 * merges once and writes its union at the provisional offset sum_o b_p.pos[o] (an upper bound of its
 * final offset, the cost C(b_p) of Theorem 1) of a workspace staging buffer, with
 * partition-local Z.pos counts; an exclusive prefix sum of the union sizes and a placement
 * pass then move every union to part_off[p] and add part_off[p] to the Z.pos entries it owns (R7).
 *   Partitions of any size: one larger than the 2048-entry tile runs as chunks whose cuts are
 *   further Alg. 1 searches (queries C(b_p) + c (2048 - k + 1)), so every coordinate still lies in
 *   one chunk and a caller's coarse P (e.g. one partition per worker) stays fast.
 *   part_off [P+1] int64 (required; part_off[P] = nnz_Z).  z_crd / z_val: capacity >= nnz_Z (Q* is
 *   always enough).
 *   ws  >= nacho_spadd_k_staged_workspace_size(ops, k, P) bytes: per-chunk counts, offsets and rows +
 *   Q* staged (col, value) pairs (sized for partitions from nacho_partition; a record whose max_work
 *   exceeds ceil(Q* / P) + k - 1 may need more: WORKSPACE).  Errors as nacho_spadd_k. */
size_t nacho_spadd_k_staged_workspace_size(const nacho_matrix* ops, int32_t k, int32_t P);
nacho_status nacho_spadd_k_staged(const nacho_matrix* ops, int32_t k, const nacho_parts* parts, int64_t* part_off,
                                  int64_t* z_pos, int32_t* z_crd, void* z_val, void* ws, size_t ws_bytes,
                                  void* stream);
nacho_status nacho_spadd_k_count(const nacho_matrix* ops, int32_t k, const nacho_parts* parts, int64_t* part_off,
                                 void* ws, size_t ws_bytes, void* stream);
nacho_status nacho_spadd_k_fill(const nacho_matrix* ops, int32_t k, const nacho_parts* parts,
                                const int64_t* part_off, int64_t* z_pos, int32_t* z_crd, void* z_val, void* ws,
                                size_t ws_bytes, void* stream);

/* ------------------------------------------------------------------------------------------------
 * nacho_spmm -- C = A B with loop order i -> j -> k (Listing 6): A is broadcast over k,
 * whose cost factor N_k is uniform, so the cuts are A's one-operand cuts and k is never cut (R6).
 *   A      CSR, fp32 or fp64.       parts: k == 1 partition of A, or NULL (auto, inside ws).
 *   B      [ncols x nb] row-major with leading dimension ldb >= nb.   C: [nrows x nb], ldc >= nb.
 *   nb     1..256 (64 is the tuned case).
 *   ws     >= nacho_spmm_workspace_size(A, P, nb). */
size_t nacho_spmm_workspace_size(const nacho_matrix* A, int32_t P, int32_t nb);
nacho_status nacho_spmm(const nacho_matrix* A, const nacho_parts* parts, const void* B, int64_t ldb, int32_t nb,
                        void* C, int64_t ldc, void* ws, size_t ws_bytes, void* stream);

/* ------------------------------------------------------------------------------------------------
 * k-way intersection kernels on the same partitioner (a1-a5): Alg. 1 over the
 * operands' entries is exact for a coiteration that walks every operand's entries, and
 * equal coordinates never straddle a cut, so every output coordinate is produced
 * inside one partition.  The merge predicate is Listing 1's (emit when every head equals
 * the minimum) instead of the union's.  CSR operands, k <= 4, partitions of at most
 * nacho_auto_partitions(ops, k, 1)'s size.
 *
 * nacho_hadamard_k -- Z = ops[0] (.) ... (.) ops[k-1], the partitioned CSR Hadamard product of
 * Listing 8 in one pass (assembly count, decoupled look-back offsets, fill): Z.pos
 * [nrows+1]; Z.crd / Z.val with capacity >= min_o nnz_o (nnz_Z = z_pos[nrows]); values are the product
 * in operand order, left to right, in the value type (bit-identical to Listing 1's a.v * b.v * c.v).
 * part_off (optional, [P+1]) receives the per-partition offsets.  Workspace:
 * nacho_spadd_k_workspace_size. */
nacho_status nacho_hadamard_k(const nacho_matrix* ops, int32_t k, const nacho_parts* parts, int64_t* part_off,
                              int64_t* z_pos, int32_t* z_crd, void* z_val, void* ws, size_t ws_bytes, void* stream);

/* nacho_inner_k -- the intersect-reduce inner product s = sum_(i,j) prod_o ops[o](i,j) (the fused
 * (.) + reduction of the paper's inner-product evaluation, on CSR operands): products as
 * in nacho_hadamard_k, summed in fp64 per partition and then over partitions in a fixed order
 * (deterministic).  result: device double[1]. */
size_t nacho_inner_k_workspace_size(const nacho_matrix* ops, int32_t k, int32_t P);
nacho_status nacho_inner_k(const nacho_matrix* ops, int32_t k, const nacho_parts* parts, double* result, void* ws,
                           size_t ws_bytes, void* stream);

/* ------------------------------------------------------------------------------------------------
 * nacho_dcsr_hadamard -- recursive partitioning (Alg. 2) of the DCSR
 * Hadamard product Z = ops[0] (.) ... (.) ops[k-1] (Listing emul-dcsr2-cfir), whose outer
 * sparse intersection skips whole rows.  The flow of P:1815-1825 / Listing emul-dcsr2-rewritten
 * (P:1478-1496): (1) Alg. 1 partitions the outer intersection (the outer levels as one-row operands);
 * (2) its assembly / prefix sum / compute give the surviving rows rows(A_0) cap ... and
 * T[i] = C_j(N_j | i), the row's non-zeros over the operands; (3) T' = exclusive prefix sum of T, the
 * remapped cost C'_i; (4) Alg. 1 with C'_i and the inner nnz cost partitions the
 * remapped loop nest into `parts` (caller-allocated, parts->P partitions: row_pos = index of the
 * surviving row, row = its coordinate, pos[o] = absolute positions in crd_o); (5) assembly / prefix
 * sum / compute of Listing 8's loop body over those partitions.  Output Z in DCSR over the surviving
 * rows, every one stored even when its column intersection is empty (reading R21): counts[0] = S
 * (device int64[2]; counts[1] = nnz_Z), z_outer[S] (capacity >= min_o nouter_o), z_pos[S + 1],
 * z_crd / z_val (capacity >= min_o nnz_o), values the product in operand order (R17).  DCSR operands,
 * k <= 4; one thread per partition in the assembly / compute kernels (Listing 8's shape). */
size_t nacho_dcsr_hadamard_workspace_size(const nacho_matrix* ops, int32_t k, int32_t P);
nacho_status nacho_dcsr_hadamard(const nacho_matrix* ops, int32_t k, nacho_parts* parts, int64_t* counts,
                                 int32_t* z_outer, int64_t* z_pos, int32_t* z_crd, void* z_val, void* ws,
                                 size_t ws_bytes, void* stream);

/* ------------------------------------------------------------------------------------------------
 * nacho_dcsr_spadd_k -- Z = ops[0] + ... + ops[k-1] on DCSR operands (Listing 2, lst:eadd-dcsr2-cfir,
 * P:568-574) over the partition `parts` made by nacho_partition on the same DCSR
 * operands (Alg. 1 with k compressed outer levels: the row cost sum_o pos_o[lb_o(x)], P:1670-1672;
 * row_pos = the boundary row's lower bound in operand 0's outer level).  Assembly (union entries and
 * rows started per partition), prefix sums, compute (one thread per partition, Listing 8's shape):
 * Z is DCSR over the union of the stored rows: counts[0] = its stored rows, counts[1] = nnz_Z (device
 * int64[2]); z_outer / z_pos capacity >= sum_o nouter_o (+1), z_crd / z_val >= sum_o nnz_o; values fold
 * left in operand order (R9).  k <= 4. */
size_t nacho_dcsr_spadd_k_workspace_size(const nacho_matrix* ops, int32_t k, int32_t P);
nacho_status nacho_dcsr_spadd_k(const nacho_matrix* ops, int32_t k, const nacho_parts* parts, int64_t* counts,
                                int32_t* z_outer, int64_t* z_pos, int32_t* z_crd, void* z_val, void* ws,
                                size_t ws_bytes, void* stream);

/* ------------------------------------------------------------------------------------------------
 * nacho_mixed_spadd_k -- Z = ops[0] + ... + ops[k-1] for CSR and COO operands mixed (the COO + CSR
 * addition the paper evaluates without a format conversion) over the
 * partition nacho_partition made of the same operands (Alg. 1 with the COO row level: C_i(x) counts
 * the entries whose row is < x, a binary search per probe).  One thread per partition (Listing 8's
 * shape): count, prefix sum, fill.  Z is CSR: z_pos[nrows + 1], z_crd / z_val capacity >= sum_o nnz_o,
 * nnz_z (device int64[1]).  Values fold left in operand order (R9).  k <= 4. */
size_t nacho_mixed_spadd_k_workspace_size(const nacho_matrix* ops, int32_t k, int32_t P);
nacho_status nacho_mixed_spadd_k(const nacho_matrix* ops, int32_t k, const nacho_parts* parts, int64_t* nnz_z,
                                 int64_t* z_pos, int32_t* z_crd, void* z_val, void* ws, size_t ws_bytes, void* stream);

/* ------------------------------------------------------------------------------------------------
 * Third-order tensors in CSF = Compressed(i) o Compressed(j) o Compressed(k): the coordinate tree of
 * fig:coordinate-tree.  crd0[n_slices] strictly increasing slice coordinates;
 * pos1[n_slices + 1] fiber ranges, crd1[n_fibers] increasing within a slice; pos2[n_fibers + 1]
 * entry ranges, crd2[nnz] increasing within a fiber; val[nnz].  Every stored slice / fiber non-empty,
 * pos1[0] = pos2[0] = 0.  All arrays device memory, owned by the caller. */
typedef struct {
  int32_t dtype;   /* nacho_dtype of val */
  int64_t n0, n1, n2;
  int64_t nnz, n_slices, n_fibers;
  const int32_t* crd0;
  const int64_t* pos1;
  const int32_t* crd1;
  const int64_t* pos2;
  const int32_t* crd2;
  const void* val;
} nacho_tensor3;

/* nacho_partition_csf -- Alg. 1 at d = 3 for k CSF operands of one shape: boundary p is
 * the highest coordinate (x_i, x_j, x_k) whose cost C_i(x_i) + C_j(x_j | x_i) + C_k(x_k | x_i, x_j)
 * (the entries lexicographically before it, summed over the operands; the coordinate-tree cost
 * functions) is <= Q_p = floor(p Q* / P), Q* = sum_o nnz_o.  One warp per
 * boundary: a 32-ary search per level (i over [0, n0], j inside slice x_i) and the k-way select of
 * the CSR path over the fibers' crd2 segments.  out->row = x_i, out->row_pos = x_j, out->col = x_k,
 * out->pos[p k + o] = entries of operand o before b_p; b_0 = (0, 0, 0), b_P = (n0, 0, 0) with
 * pos = nnz.  k <= 4.  Errors: INVALID_ARG (k, P, nulls), SHAPE (shapes differ). */
nacho_status nacho_partition_csf(const nacho_tensor3* ops, int32_t k, int32_t P, nacho_parts* out, void* stream);

/* nacho_csf_spadd_k -- Z = ops[0] + ... + ops[k-1] in CSF (the paper's third-order tensor addition,
 * P:2403-2441) over the partition nacho_partition_csf made: assembly (entries, fibers
 * and slices started per partition), three prefix sums, compute (one thread per partition, Listing 8's
 * shape, the union at three levels; pos1 / pos2 written by the partition that completes the slice /
 * fiber).  counts (device int64[3]) = Z's slices, fibers, nnz.  Capacities: z_crd0 / z_pos1 >= sum_o
 * n_slices_o (+1), z_crd1 / z_pos2 >= sum_o n_fibers_o (+1), z_crd2 / z_val >= sum_o nnz_o.  Values fold
 * left in operand order (R9).  k <= 4. */
size_t nacho_csf_spadd_k_workspace_size(const nacho_tensor3* ops, int32_t k, int32_t P);
nacho_status nacho_csf_spadd_k(const nacho_tensor3* ops, int32_t k, const nacho_parts* parts, int64_t* counts,
                               int32_t* z_crd0, int64_t* z_pos1, int32_t* z_crd1, int64_t* z_pos2, int32_t* z_crd2,
                               void* z_val, void* ws, size_t ws_bytes, void* stream);

/* ------------------------------------------------------------------------------------------------
 * ESC scatter kernels: a kernel that scatters into a sparse output runs as
 * expand - sort - contract, with the load balancing applied to the expansion only
 * (P:2073-2074).  SpGEMM C = A B over i -> k -> j; sampled SpGEMM Z = S (.) (A B)
 * (SSSMM).  A, B, S CSR of one dtype; A.ncols == B.nrows; S is A.nrows x B.ncols.
 * ------------------------------------------------------------------------------------------------ */

/* nacho_spgemm_work -- the expansion's cost, Listing 6's broadcast-scaled cost (P:1714-1727,
 * P:1742-1749): W[q] = sum_{q' < q} nnz(B_{A.crd[q']}) for q in [0, nnz(A)] (device int64[nnz(A)+1]);
 * W[nnz(A)] = Q*, the number of products (the caller reads it to size the expansion). */
size_t nacho_spgemm_work_workspace_size(const nacho_matrix* A);
nacho_status nacho_spgemm_work(const nacho_matrix* A, const nacho_matrix* B, int64_t* W, void* ws, size_t ws_bytes,
                               void* stream);
/* P for about 8192 products per partition. */
int32_t nacho_esc_auto_partitions(int64_t qstar);

/* nacho_partition_esc -- Alg. 1 over i -> k -> j with the cost W: Q_p = floor(p Q* / P)
 * (P:1089-1093); b_p locates product number Q_p of the expansion (rows ascending, A positions, B
 * positions): row[p] = row_pos[p] = its row i, pos[2p] = the A position q producing it, pos[2p+1] = its
 * B position, col[p] = its column j.  A query at or past Q* gives (nrows, nnz(A), nnz(B), col 0).  out
 * must have k == 2 and P == P; max_work is set to floor(Q* / P) + 1. */
nacho_status nacho_partition_esc(const nacho_matrix* A, const nacho_matrix* B, const int64_t* W, int64_t qstar,
                                 int32_t P, nacho_parts* out, void* stream);

/* nacho_spgemm_esc -- C = A B: expand (one CTA per partition writes the products [Q_p, Q_{p+1}) at
 * their expansion index: key (i, j), value A_ik * B_kj), stable radix sort by (i, j), contract (every
 * run of one (i, j) folded left to right, i.e. k ascending -- reading R23).  C stores (i, j) iff some
 * product has that coordinate.  c_pos[A.nrows+1], c_crd / c_val capacity >= Q*; *nnz_c (device int64)
 * receives nnz(C).  The workspace holds the expansion twice (sort buffers) and the run indices. */
size_t nacho_spgemm_esc_workspace_size(const nacho_matrix* A, const nacho_matrix* B, int64_t qstar);
nacho_status nacho_spgemm_esc(const nacho_matrix* A, const nacho_matrix* B, const int64_t* W, const nacho_parts* parts,
                              int64_t qstar, int64_t* c_pos, int32_t* c_crd, void* c_val, int64_t* nnz_c, void* ws,
                              size_t ws_bytes, void* stream);

/* nacho_sssmm_esc_count / nacho_sssmm_esc -- Z = S (.) (A B) (reading R24: Z_ij = S_ij * C_ij on the
 * coordinates S and C both store).  The expansion over the same W / partition keeps the products whose
 * j is stored in S_i: count per partition -> part_off (device int64[P+1], exclusive prefix; part_off[P]
 * = kept products, which the caller reads) -> fill in expansion order -> sort -> contract.  Z
 * capacity >= part_off[P].  keep_mask (device, nacho_sssmm_mask_bytes(Q*, P) bytes, caller-owned) carries
 * the count pass's membership bits to the fill (the assembly records the predicate, the compute reuses
 * it: no second search in S). */
size_t nacho_sssmm_mask_bytes(int64_t qstar, int32_t P);
size_t nacho_sssmm_count_workspace_size(int32_t P);
nacho_status nacho_sssmm_esc_count(const nacho_matrix* S, const nacho_matrix* A, const nacho_matrix* B, const int64_t* W,
                                   const nacho_parts* parts, int64_t* part_off, uint8_t* keep_mask, void* ws,
                                   size_t ws_bytes, void* stream);
size_t nacho_sssmm_esc_workspace_size(const nacho_matrix* A, const nacho_matrix* B, int64_t n_kept);
nacho_status nacho_sssmm_esc(const nacho_matrix* S, const nacho_matrix* A, const nacho_matrix* B, const int64_t* W,
                             const nacho_parts* parts, const int64_t* part_off, const uint8_t* keep_mask, int64_t n_kept,
                             int64_t* z_pos, int32_t* z_crd, void* z_val, int64_t* nnz_z, void* ws, size_t ws_bytes,
                             void* stream);

/* ------------------------------------------------------------------------------------------------
 * nacho_validate -- full structural check of an operand (sorted levels; R10) on the device.
 * Synchronous on `stream` (it reads one flag back).  Returns NACHO_ERR_FORMAT on a violation.  The one
 * exception to "no device allocations": a 4-byte result flag, cudaMallocAsync'd and freed on `stream`
 * inside the call. */
nacho_status nacho_validate(const nacho_matrix* A, void* stream);

/* ------------------------------------------------------------------------------------------------
 * Multi-GPU (one process per GPU).  The paper's partition is the device decomposition:
 * with D devices, device d owns [b_d, b_{d+1}) of Alg. 1 run with P = D (one partition
 * per processor; saved positions P:1795), so its work is Q* / D +- Delta (Theorem 1).  The
 * paper is shared-memory only: the exchange below is this library's addition.  NCCL is
 * loaded at run time (libnccl.so.2, the copy torch already loaded if any); failures -> NACHO_ERR_NCCL.
 * torch (or any launcher) only moves the unique id between processes. */
typedef struct nacho_dist_s nacho_dist;

/* Size of the opaque NCCL unique id (bytes); nacho_dist_unique_id fills a HOST buffer of that size on
 * one process, which hands it to every rank (e.g. a torch.distributed broadcast). */
size_t nacho_dist_unique_id_size(void);
nacho_status nacho_dist_unique_id(void* id);

/* Communicator of `nranks` processes, this one `rank` (the current CUDA device is used).  Collective:
 * every rank calls it.  Destroy with nacho_dist_destroy. */
nacho_status nacho_dist_init(nacho_dist** comm, const void* id, int32_t nranks, int32_t rank);
nacho_status nacho_dist_destroy(nacho_dist* comm);

/* In-place broadcast of `bytes` of a device buffer from `root` (the x / B replication at setup). */
nacho_status nacho_dist_broadcast(nacho_dist* comm, void* buf, size_t bytes, int32_t root, void* stream);

/* Device cuts of one CSR operand for D devices: cuts[2d] = row, cuts[2d+1] = position of Alg. 1 at
 * Q_d = floor(d Q* / D) (k = 1 closed form: position Q_d, row = highest x with pos[x] <= Q_d; cut 0 is
 * the origin and cut D the end, R1).  `cuts`: device int64[2(D+1)].  Reads only A->pos. */
nacho_status nacho_device_cuts(const nacho_matrix* A, int32_t D, int64_t* cuts, void* stream);

/* Row pointers of a shard: rows [row_lo, row_lo + nloc) of `pos` restricted to positions
 * [pos_lo, pos_hi) and rebased to 0 (first / last row possibly partial).  local_pos: device
 * int64[nloc + 1].  A k-operand SpAdd shard calls it once per operand with that operand's cut
 * positions b_d.pos[o], b_{d+1}.pos[o]. */
nacho_status nacho_shard_rows(const int64_t* pos, int64_t row_lo, int64_t nloc, int64_t pos_lo, int64_t pos_hi,
                              int64_t* local_pos, void* stream);

/* Seam fix-up of device d (Listing 8's carry rule, at device level): if the device owns
 * its first row (owns_first), add the carries of the devices before it that end in that row
 * (carries: device int64[2D] of (row, value bits), row -1 = none), in device order, to y_local[0]. */
nacho_status nacho_dist_seam(const int64_t* carries, int32_t D, int32_t d, int64_t row_lo, int32_t owns_first,
                             int32_t dtype, void* y_local, void* stream);

/* y = A x on D devices: this device's shard A_local (rows cut_rows[d] .. cut_rows[d+1] of A, the last
 * one partial when d < D-1; nacho_device_cuts + nacho_shard_rows), its partitions `parts` (or NULL:
 * auto P), the replicated x.  y_local[nrows_local] receives the rows the device owns (R7: rows
 * [cut_rows[d], cut_rows[d+1]); its last slot is the outgoing seam carry when d < D-1), after the seam
 * carries of earlier devices are added (an NCCL all-gather of one (row, value) pair per device).  If
 * y_full (device, [nrows of A]) is not NULL every device's owned segment is gathered into it (one
 * NCCL broadcast per device).  cut_rows: HOST int64[D+1] (cut D = nrows).  Collective. */
size_t nacho_dist_spmv_workspace_size(const nacho_matrix* A_local, int32_t P, int32_t D);
nacho_status nacho_dist_spmv(nacho_dist* comm, const nacho_matrix* A_local, const nacho_parts* parts, const void* x,
                             void* y_local, const int64_t* cut_rows, void* y_full, void* ws, size_t ws_bytes,
                             void* stream);

/* Exchange step of a k-way SpAdd on D devices: every device has run nacho_spadd_k on its operand
 * shards (rows cut_rows[d] .. cut_rows[d+1]); z_*_local is its union and nnz_local (device int64[1])
 * its size.  Equal coordinates never straddle a cut, so no values merge: an NCCL
 * all-gather of the D sizes gives the global offsets (the host reads them: variable-size collectives
 * need host counts -- the call synchronises `stream`), then Z.crd / Z.val / Z.pos segments are
 * gathered into z_pos[nrows+1] / z_crd / z_val (capacity >= the total, returned in *nnz_total). */
size_t nacho_dist_spadd_workspace_size(int32_t D);
nacho_status nacho_dist_spadd_gather(nacho_dist* comm, const int64_t* z_pos_local, const int32_t* z_crd_local,
                                     const void* z_val_local, int32_t dtype, const int64_t* nnz_local,
                                     const int64_t* cut_rows, int64_t* z_pos, int32_t* z_crd, void* z_val,
                                     int64_t* nnz_total, void* ws, size_t ws_bytes, void* stream);

/* Message for the last non-success status on this thread ("" if none). */
const char* nacho_last_error(void);

/* Number of kernel launches issued by this library on this thread since the last reset (for the
 * benchmark's gpu_launches claim). */
int64_t nacho_launch_count(int32_t reset);

#ifdef __cplusplus
}
#endif
#endif /* NACHO_H */
