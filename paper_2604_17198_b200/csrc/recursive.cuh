// recursive.cuh -- recursive partitioning (Alg. 2) of the DCSR Hadamard product
// Z = A_0 (.) ... (.) A_{k-1} (Listing emul-dcsr2-cfir).  The outer sparse
// intersection skips whole rows, so the row cost is remapped before partitioning: the kernel flow of
// P:1815-1825 (one partitioning kernel per sparse intersection), i.e. Listing emul-dcsr2-rewritten
// with every loop load-balanced:
//   1. partition the outer intersection: Alg. 1 over the outer levels viewed as k one-row operands
//      (the existing k-way partition kernel), P1 partitions;
//   2. assembly of the outer intersection (surviving rows per partition), prefix sum, and compute:
//      every surviving row with T[i] = C_j(N_j | i) (its non-zeros over the operands) and its outer
//      position in every operand (lines 2-3);
//   3. T' = exclusive_prefix_sum(T) (line 4): the remapped cost C'_i = T' (line 5);
//   4. partition the remapped loop nest (i' over the surviving rows, j over their columns) with C'_i
//      and the inner nnz cost (Alg. 1: a 32-ary search over T', the k-way select in the row);
//   5. assembly (intersection count per partition), prefix sum, compute (Listing 8's loop body with
//      the intersection predicate, its Z.pos guard) -- lines 7-9.
// The per-partition loops are Listing 8's: one thread per partition walks its range with a k-finger
// merge (the paper's GPU code shape; this path is not performance-tuned).  Z is DCSR over the
// surviving rows, every one stored (possibly with an empty segment, reading R21).
#pragma once
#include "common.cuh"

namespace nacho {

constexpr int kRecThreads = 128;

// Views of the k outer levels as one-row CSR operands (crd = outer_crd): pos_views[2o] = 0,
// pos_views[2o + 1] = nouter_o.
__global__ void rec_outer_views_kernel(OpsArg in, int64_t* pos_views) {
  const int o = threadIdx.x;
  if (o < in.k) {
    pos_views[2 * o] = 0;
    pos_views[2 * o + 1] = in.op[o].nouter;
  }
}

// Step 2, assembly (MODE 0: count) and compute (MODE 1: fill) of the outer intersection over outer
// partition p: entries [b_p.pos[o], b_{p+1}.pos[o]) of every outer level.
template <int MODE>
__global__ void __launch_bounds__(kRecThreads) rec_rows_kernel(OpsArg in, PartsArg op, int64_t* cnt, const int64_t* off,
                                                               int32_t* rows, int64_t* T, int64_t* ip, int64_t cap) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= op.P) return;
  const int k = in.k;
  int64_t q[NACHO_MAX_K], e[NACHO_MAX_K];
#pragma unroll
  for (int o = 0; o < NACHO_MAX_K; ++o)
    if (o < k) { q[o] = op.pos[p * k + o]; e[o] = op.pos[(p + 1) * k + o]; }
  int64_t n = 0, w = MODE ? off[p] : 0;
  for (;;) {
    bool inside = true;
    for (int o = 0; o < k; ++o) inside = inside && q[o] < e[o];
    if (!inside) break;
    int64_t r = INT64_MAX;
    for (int o = 0; o < k; ++o) r = min(r, (int64_t)ldg(in.op[o].outer + q[o]));
    bool all = true;
    for (int o = 0; o < k; ++o) all = all && (int64_t)ldg(in.op[o].outer + q[o]) == r;
    if (all) {
      if (MODE) {
        int64_t t = 0;
        for (int o = 0; o < k; ++o) {
          t += ldg(in.op[o].pos + q[o] + 1) - ldg(in.op[o].pos + q[o]);
          ip[(int64_t)o * cap + w] = q[o];
        }
        rows[w] = (int32_t)r;
        T[w] = t;
        ++w;
      }
      ++n;
    }
    for (int o = 0; o < k; ++o) if ((int64_t)ldg(in.op[o].outer + q[o]) == r) ++q[o];
  }
  if (!MODE) cnt[p] = n;
}

// Exclusive prefix sum of n = *n_dev int64 values (one CTA, a running carry over tiles); out[n] = total.
template <int THREADS>
__global__ void __launch_bounds__(THREADS) rec_scan_kernel(const int64_t* __restrict__ in, const int64_t* n_dev,
                                                           int64_t n_host, int64_t* __restrict__ out) {
  constexpr int IT = 8;
  __shared__ int64_t red[THREADS / 32 + 1];
  const int64_t n = n_dev ? *n_dev : n_host;
  int64_t carry = 0;
  for (int64_t base = 0; base < n; base += (int64_t)THREADS * IT) {
    int64_t v[IT];
    int64_t s = 0;
#pragma unroll
    for (int i = 0; i < IT; ++i) {
      const int64_t j = base + (int64_t)threadIdx.x * IT + i;
      v[i] = j < n ? in[j] : 0;
      s += v[i];
    }
    int64_t tot;
    int64_t ex = block_excl_sum<THREADS, int64_t>(s, red, &tot) + carry;
#pragma unroll
    for (int i = 0; i < IT; ++i) {
      const int64_t j = base + (int64_t)threadIdx.x * IT + i;
      if (j < n) out[j] = ex;
      ex += v[i];
    }
    carry += tot;
  }
  if (threadIdx.x == 0) out[n] = carry;
}

// Step 4: boundary p of the remapped partition, one warp each.  Q_p = floor(p T'[S] / P) (R4);
// outer level: highest s with T'[s] <= Q (32-ary search over T'); inner level: the (R+1)-th smallest
// entry of the k column segments of surviving row s (the k-way select of the CSR partition).
// Origin / end as in oracle_partition_remapped (R1).
template <int KM>
__global__ void __launch_bounds__(128) rec_partition_kernel(OpsArg in, PartsArg out, const int64_t* S_dev,
                                                            const int32_t* rows, const int64_t* Tp, const int64_t* ip,
                                                            int64_t cap) {
  const int64_t p = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
  if (p > out.P) return;
  const int lane = threadIdx.x & 31;
  const int k = in.k;
  const int64_t S = *S_dev;
  const int64_t total = S > 0 ? Tp[S] : 0;
  const int64_t Q = query_of(total, out.P, p);
  int64_t rowv, rp;
  int32_t col = 0;
  int64_t pos[KM];
  if (p == 0 && S > 0) {
    rowv = rows[0]; rp = 0;
#pragma unroll
    for (int o = 0; o < KM; ++o) if (o < k) pos[o] = ldg(in.op[o].pos + ip[(int64_t)o * cap]);
  } else if (p == out.P || Q >= total || S == 0) {
    rowv = in.nrows; rp = S;
#pragma unroll
    for (int o = 0; o < KM; ++o) if (o < k) pos[o] = S > 0 ? ldg(in.op[o].pos + ip[(int64_t)o * cap + S - 1] + 1) : 0;
  } else {
    const int64_t s = warp_highest_true(0, S - 1, [&](int64_t x) { return ldg(Tp + x) <= Q; });
    rowv = rows[s]; rp = s;
    int64_t lo[KM], hi[KM];
#pragma unroll
    for (int o = 0; o < KM; ++o) {
      if (o < k) {
        const int64_t i = ip[(int64_t)o * cap + s];
        lo[o] = ldg(in.op[o].pos + i);
        hi[o] = ldg(in.op[o].pos + i + 1);
      }
    }
    Boundary b;
    warp_kway_select<KM>(in, k, lo, hi, Q - ldg(Tp + s), b);
    col = b.col;
#pragma unroll
    for (int o = 0; o < KM; ++o) if (o < k) pos[o] = b.pos[o];
  }
  if (lane == 0) {
    out.query[p] = Q;
    out.row[p] = rowv;
    out.row_pos[p] = rp;
    out.col[p] = col;
  }
  if (lane < k) {
    int64_t v = 0;
#pragma unroll
    for (int o = 0; o < KM; ++o) if (o == lane) v = pos[o];
    out.pos[p * k + lane] = v;
  }
}

// Step 5, Listing 8 over the remapped rows: partition p walks surviving rows
// [b_p.row_pos, b_{p+1}.row_pos] (the last one only up to b_{p+1}.pos, R7's clamp), intersecting the
// k column segments.  MODE 0 counts; MODE 1 writes Z at off[p] and Z.pos[s + 1] of every row it
// completes (Listing 8's guard: the partition's range reaches the row's end in every operand).
template <typename V, int MODE>
__global__ void __launch_bounds__(kRecThreads) rec_hadamard_kernel(OpsArg in, PartsArg pa, const int64_t* S_dev,
                                                                   const int64_t* ip, int64_t cap, int64_t* cnt,
                                                                   const int64_t* off, int64_t* z_pos, int32_t* z_crd,
                                                                   V* z_val) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= pa.P) return;
  const int k = in.k;
  const int64_t S = *S_dev;
  const int64_t s0 = pa.row_pos[p], s1 = pa.row_pos[p + 1];
  int64_t jz = MODE ? off[p] : 0, n = 0;
  if (MODE && p == 0) z_pos[0] = 0;
  for (int64_t s = s0; s <= s1 && s < S; ++s) {
    int64_t q[NACHO_MAX_K], e[NACHO_MAX_K];
    bool ends_row = true;
    for (int o = 0; o < k; ++o) {
      const int64_t i = ip[(int64_t)o * cap + s];
      const int64_t rs = ldg(in.op[o].pos + i), re = ldg(in.op[o].pos + i + 1);
      q[o] = s == s0 ? pa.pos[p * k + o] : rs;
      e[o] = s == s1 ? pa.pos[(p + 1) * k + o] : re;
      if (q[o] < rs) q[o] = rs;
      if (e[o] > re) e[o] = re;
      ends_row = ends_row && e[o] == re;
    }
    for (;;) {
      bool inside = true;
      for (int o = 0; o < k; ++o) inside = inside && q[o] < e[o];
      if (!inside) break;
      int32_t j = INT32_MAX;
      for (int o = 0; o < k; ++o) j = min(j, ldg(in.op[o].crd + q[o]));
      bool all = true;
      for (int o = 0; o < k; ++o) all = all && ldg(in.op[o].crd + q[o]) == j;
      if (all) {
        if (MODE) {
          V v = static_cast<const V*>(in.op[0].val)[q[0]];
          for (int o = 1; o < k; ++o) v = v * static_cast<const V*>(in.op[o].val)[q[o]];
          z_crd[jz] = j;
          z_val[jz] = v;
          ++jz;
        }
        ++n;
      }
      for (int o = 0; o < k; ++o) if (ldg(in.op[o].crd + q[o]) == j) ++q[o];
    }
    if (MODE && ends_row) z_pos[s + 1] = jz;   // the row is complete in this partition
  }
  if (!MODE) cnt[p] = n;
}

// The output sizes: counts[0] = S (surviving rows = Z's stored rows), counts[1] = nnz_Z.
__global__ void rec_counts_kernel(const int64_t* S_dev, const int64_t* nnz_dev, int64_t* counts) {
  if (threadIdx.x == 0) { counts[0] = *S_dev; counts[1] = *nnz_dev; }
}

}  // namespace nacho
