// spmv.cuh -- partitioned CSR / DCSR SpMV y = A x and its carry fix-up.
#pragma once
#include "common.cuh"

namespace nacho {

template <typename T>
struct SpmvArgs {
  const int64_t* pos;
  const int32_t* crd;
  const T* val;
  const int32_t* outer;   // DCSR row coordinates (only used for a dense y)
  int64_t nouter;
  int64_t ncols;
  const T* x;
  T* y;
  int32_t dense_y;        // DCSR: write y[outer[rp]] instead of y[rp]
  int32_t P;
  const int64_t* ppos;    // parts.pos   (k == 1): [P+1]
  const int64_t* prow;    // parts.row_pos:        [P+1]
  int64_t* carry_row;     // [P] outer position receiving partition p's carry (-1: none)
  T* carry_val;           // [P]
};

template <typename T>
__device__ __forceinline__ int64_t y_index(const SpmvArgs<T>& a, int64_t rp) {
  return (a.dense_y && a.outer) ? (int64_t)ldg(a.outer + rp) : rp;
}

// Keyed (segmented) sum: (k1,v1) (+) (k2,v2) = (k2, k1 == k2 ? v1 + v2 : v2).  Keys are outer
// positions, non-decreasing along the partition, so this is the reduce-by-row of partial sums.
template <typename T>
struct KV { int64_t k; T v; };
template <typename T>
__device__ __forceinline__ KV<T> kv_op(KV<T> a, KV<T> b) { return KV<T>{b.k, a.k == b.k ? a.v + b.v : b.v}; }

// One CTA per partition p.  The partition's positions [s, e) are processed in chunks of TILE items;
// thread t of a chunk owns the IPT consecutive positions [a_t, b_t).  Each thread walks its items
// row by row (Listing 8's loop bounds): rows that end inside [a_t, b_t) are "finished";
// the first finished row may have started earlier (its partial needs the carry from the preceding
// threads), later ones are complete and written directly.  Ownership (R7): CTA p writes exactly
// the rows [b_p.row_pos, b_{p+1}.row_pos - 1], including empty ones (written as 0).  The row cut by
// b_{p+1} leaves a carry (row, partial) that spmv_fixup adds in partition order.
template <typename T, int THREADS, int IPT>
__global__ void __launch_bounds__(THREADS) spmv_kernel(SpmvArgs<T> a) {
  constexpr int TILE = THREADS * IPT;
  constexpr int W = THREADS / 32;
  __shared__ int32_t s_crd[TILE + TILE / 32];
  __shared__ T s_val[TILE + TILE / 32];
  __shared__ KV<T> s_agg[W];
  __shared__ KV<T> s_carry;

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int p = blockIdx.x;
  const int64_t s = ldg(a.ppos + p), e = ldg(a.ppos + p + 1);
  const int64_t rp0 = ldg(a.prow + p), rpE = ldg(a.prow + p + 1);
  if (tid == 0) s_carry = KV<T>{rp0, T(0)};

  for (int64_t cs = s;; cs += TILE) {
    const int64_t ce = (e - cs < TILE) ? e : cs + TILE;
    const int n = (int)(ce - cs);
    __syncthreads();  // s_carry written / previous chunk's smem reads done
    for (int j = tid; j < n; j += THREADS) {
      s_crd[j + (j >> 5)] = ldg(a.crd + cs + j);
      s_val[j + (j >> 5)] = ldg(a.val + cs + j);
    }
    const KV<T> chunk_carry = s_carry;
    __syncthreads();

    const int i0 = tid * IPT;
    const bool active = (i0 < n) || tid == 0;
    const int cnt = active ? ((n - i0 < IPT) ? (n - i0 > 0 ? n - i0 : 0) : IPT) : 0;
    const int64_t at = cs + i0, bt = at + cnt;

    bool head = true, head_done = false;
    int64_t head_row = 0;
    T head_val = T(0), acc = T(0);
    int64_t rp = 0;
    if (active) {
      if (tid == 0 && cs == s) {
        rp = rp0;
      } else {  // largest rp in [rp0, rpE] with pos[rp] <= at
        int64_t lo = rp0, hi = rpE < a.nouter ? rpE : a.nouter;
        while (lo < hi) {
          const int64_t m = lo + ((hi - lo + 1) >> 1);
          if (ldg(a.pos + m) <= at) lo = m; else hi = m - 1;
        }
        rp = lo;
      }
      int64_t next_end = rp < a.nouter ? ldg(a.pos + rp + 1) : INT64_MAX;
      for (int i = 0; i < cnt; ++i) {
        const int64_t q = at + i;
        while (next_end <= q) {  // row rp finished before item q
          if (head) { head_done = true; head_row = rp; head_val = acc; head = false; }
          else a.y[y_index(a, rp)] = acc;
          acc = T(0);
          ++rp;
          next_end = ldg(a.pos + rp + 1);
        }
        const int j = i0 + i;
        const int sj = j + (j >> 5);
        acc += s_val[sj] * ldg(a.x + s_crd[sj]);
      }
      while (rp < a.nouter && next_end <= bt) {  // rows ending exactly at b_t (and empty ones) are ours
        if (head) { head_done = true; head_row = rp; head_val = acc; head = false; }
        else a.y[y_index(a, rp)] = acc;
        acc = T(0);
        ++rp;
        next_end = rp < a.nouter ? ldg(a.pos + rp + 1) : INT64_MAX;
      }
    }
    // ---- keyed scan of the tails (rp, acc) across the chunk's threads
    KV<T> mine = active ? KV<T>{rp, acc} : KV<T>{INT64_MAX, T(0)};
    KV<T> inc = mine;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      KV<T> u;
      u.k = __shfl_up_sync(kFull, inc.k, d);
      u.v = __shfl_up_sync(kFull, inc.v, d);
      if (lane >= d) inc = kv_op(u, inc);
    }
    if (lane == 31) s_agg[w] = inc;
    __syncthreads();
    KV<T> pre = chunk_carry;
    for (int ww = 0; ww < w; ++ww) pre = kv_op(pre, s_agg[ww]);
    KV<T> excl;
    excl.k = __shfl_up_sync(kFull, inc.k, 1);
    excl.v = __shfl_up_sync(kFull, inc.v, 1);
    excl = (lane == 0) ? pre : kv_op(pre, excl);
    if (head_done) {
      const T c = (excl.k == head_row) ? excl.v : T(0);
      a.y[y_index(a, head_row)] = c + head_val;
    }
    // new chunk carry = inclusive value of the last active thread
    const int last = n > 0 ? (n - 1) / IPT : 0;
    if (tid == last) s_carry = kv_op(pre, inc);
    if (ce >= e) break;
  }
  __syncthreads();
  if (tid == 0) {
    const KV<T> c = s_carry;
    const bool has = c.k < a.nouter && c.k == rpE;
    a.carry_row[p] = has ? c.k : -1;
    a.carry_val[p] = has ? c.v : T(0);
  }
}

// Adds every partition's carry to the row it belongs to, in partition order (deterministic for a
// given P).  The partitions whose carries go to one row form a contiguous run; the warp holding the
// run's last carry sums the run (lanes strided, tree reduction) and adds it to y.
template <typename T>
__global__ void spmv_fixup_kernel(SpmvArgs<T> a) {
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t idx = gw * 32 + lane;
  const int64_t key = idx < a.P ? a.carry_row[idx] : -1;
  const bool is_end = key >= 0 && (idx == a.P - 1 || a.carry_row[idx + 1] != key);
  unsigned m = __ballot_sync(kFull, is_end);
  while (m) {
    const int l = __ffs(m) - 1;
    m &= m - 1;
    const int64_t row = __shfl_sync(kFull, key, l);
    const int64_t end = gw * 32 + l;
    const int64_t start = warp_run_start(a.carry_row, end, row);
    T sum = T(0);
    for (int64_t j = start + lane; j <= end; j += 32) sum += a.carry_val[j];
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) sum += __shfl_xor_sync(kFull, sum, d);
    if (lane == 0) a.y[y_index(a, row)] += sum;
  }
}

}  // namespace nacho
