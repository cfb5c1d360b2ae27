// common.cuh -- device-side types and warp/block primitives shared by the libnacho kernels.
// (Nothing here is shared with the oracle.)
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/nacho.h"

namespace nacho {

constexpr int kWarp = 32;
constexpr unsigned kFull = 0xffffffffu;

// One sparse operand as the kernels see it: pos in the outer-position space
// [0, nouter], crd/val in position space.  outer != nullptr <=> DCSR.
struct OpView {
  int32_t fmt;            // nacho_format: CSR, DCSR (outer = stored rows), COO (outer = row of every entry)
  const int64_t* pos;
  const int32_t* crd;
  const void* val;
  const int32_t* outer;
  int64_t nouter;
  int64_t nnz;
};

// Up to NACHO_MAX_K operands passed by value to kernels.
struct OpsArg {
  OpView op[NACHO_MAX_K];
  int32_t k;
  int32_t dtype;
  int64_t nrows, ncols;
  int32_t pos_shared;   // every operand's pos is one array (same row profile): C_i(x) = k * pos[x]
};

// Partition record (device pointers), see nacho_parts.
struct PartsArg {
  int32_t P, k;
  int64_t* query;
  int64_t* row;
  int64_t* row_pos;
  int32_t* col;
  int64_t* pos;
  int64_t max_work;   // host-side bound (nacho_parts.max_work), 0 = unknown
};

// Q_p = floor(p * Q* / P) without 128-bit arithmetic: (Q*/P)*p + ((Q*%P)*p)/P is exact because
// (Q*%P)*p < P*P <= 2^62 (reading R4).
__host__ __device__ __forceinline__ int64_t query_of(int64_t qstar, int64_t P, int64_t p) {
  const int64_t r = qstar % P;   // (r p) / P: 32-bit when r p < 2^32 (P < 2^16), the usual case
  const int64_t t = (P < 65536) ? (int64_t)((uint32_t)(r * p) / (uint32_t)P) : (r * p) / P;
  return (qstar / P) * p + t;
}

template <typename T>
__device__ __forceinline__ T ldg(const T* p) { return __ldg(p); }

// ------------------------------------------------------------------ warp 32-ary search
// Largest x in [lo, hi] with pred(x) true, given pred(lo) true and pred monotone (true...false).
// Each round probes 32 evenly spaced candidates (one per lane) and keeps the bracket between the
// last accepted and the first rejected probe: ceil(log32(hi-lo+1)) rounds of one probe per lane.
template <typename Pred>
__device__ __forceinline__ int64_t warp_highest_true(int64_t lo, int64_t hi, Pred pred) {
  const int lane = threadIdx.x & 31;
  if (hi < ((int64_t)1 << 26)) {   // 32-bit index arithmetic ((lane + 1) * span < 2^31)
    int32_t l = (int32_t)lo, h = (int32_t)hi;
    while (h > l) {
      const int32_t span = h - l;
      int32_t x = (span <= 32) ? l + lane + 1 : l + (((lane + 1) * span + 31) >> 5);
      if (x > h) x = h;
      const bool ok = pred((int64_t)x);
      const unsigned m = __ballot_sync(kFull, ok);
      const int32_t x0 = __shfl_sync(kFull, x, 0);
      if (m == 0) { h = x0 - 1; continue; }
      const int j = 31 - __clz(m);
      const int32_t xj = __shfl_sync(kFull, x, j);
      const int32_t xn = __shfl_sync(kFull, x, j < 31 ? j + 1 : 31);
      l = xj;
      if (j < 31 && xn > xj) h = xn - 1;
    }
    return l;
  }
  while (hi > lo) {
    const int64_t span = hi - lo;
    int64_t x = (span <= 32) ? lo + lane + 1 : lo + (((int64_t)(lane + 1) * span + 31) >> 5);
    if (x > hi) x = hi;
    const bool ok = pred(x);
    const unsigned m = __ballot_sync(kFull, ok);
    const int64_t x0 = __shfl_sync(kFull, x, 0);
    if (m == 0) { hi = x0 - 1; continue; }
    const int j = 31 - __clz(m);
    const int64_t xj = __shfl_sync(kFull, x, j);
    const int64_t xn = __shfl_sync(kFull, x, j < 31 ? j + 1 : 31);
    lo = xj;
    if (j < 31 && xn > xj) hi = xn - 1;
  }
  return lo;
}

// lower bound: least p in [lo, hi+1] with crd[p] >= v (lb_search of Listing 7).
__device__ __forceinline__ int64_t lb_search(const int32_t* __restrict__ crd, int64_t lo, int64_t hi, int64_t v) {
  int64_t a = lo, b = hi + 1;
  while (a < b) {
    const int64_t m = a + ((b - a) >> 1);
    if ((int64_t)ldg(crd + m) >= v) b = m; else a = m + 1;
  }
  return a;
}

// ------------------------------------------------------------------ boundary search
struct Boundary {
  int64_t row;       // row coordinate
  int64_t row_pos;   // outer position
  int32_t col;
  int64_t pos[NACHO_MAX_K];
};

__device__ __forceinline__ void set_end(const OpsArg& a, Boundary& b) {
  b.row = a.nrows;
  b.row_pos = a.op[0].nouter;
  b.col = 0;
#pragma unroll
  for (int o = 0; o < NACHO_MAX_K; ++o) if (o < a.k) b.pos[o] = a.op[o].nnz;
}

__device__ __forceinline__ void set_origin(const OpsArg& a, Boundary& b) {
  b.row = 0; b.row_pos = 0; b.col = 0;
#pragma unroll
  for (int o = 0; o < NACHO_MAX_K; ++o) if (o < a.k) b.pos[o] = 0;
}

// #lanes c in [0, n) (n <= 32) with v(c) < x, for a per-lane value v non-decreasing over lanes and a
// per-lane query x (binary search over lanes with shuffles; all lanes execute every shuffle).
template <typename V>
__device__ __forceinline__ int lanes_less(V v, V x, int n) {
  int lo = 0, hi = n;
#pragma unroll
  for (int it = 0; it < 6; ++it) {
    const int mid = (lo + hi) >> 1;
    const V vm = __shfl_sync(kFull, v, mid & 31);
    if (lo < hi) { if (vm < x) lo = mid + 1; else hi = mid; }
  }
  return lo;
}

// The (R+1)-th smallest column of the multiset union of the windows crd_o[lo_o, hi_o) (one row
// segment per operand) and its lower-bound position in every operand -- the inner level of
// FindPartition for k operands.  Invariant: entries left of lo_o are smaller than the answer v*,
// entries at or after hi_o are larger, and v* is the R-th (0-based) of the windows' union.
// Each round samples 32 positions of every window (one load per lane and operand, all in flight
// at once); the samples of the largest window are candidate values whose rank is bracketed from
// the other windows' samples; the bracket that provably contains v* becomes the new windows
// (shrinking them ~33/(k+1)-fold).  Once every window holds <= 32 entries the answer is resolved
// exactly with lane shuffles.
// KM: compile-time bound on k (register arrays sized KM).  Column values are int32 (crd < ncols <=
// INT32_MAX), so INT32_MAX is a safe "past the window" value.
// I: window index type.  The windows are offsets from cp[o] (the row segment's first entry); the
// caller takes I = int32_t when the segments' total length is below 2^26 (every product and rank
// below fits 32 bits: half the instructions of the 64-bit form), int64_t otherwise.
template <int KM, typename I>
__device__ __forceinline__ void warp_kway_select_t(const int32_t* const (&cp)[KM], int k, I (&lo)[KM], I (&hi)[KM], I R,
                                                int32_t& col, I (&pos)[KM]) {
  const int lane = threadIdx.x & 31;
  constexpr int32_t INF = INT32_MAX;
  for (;;) {
    int m = 0;
    I lmax = -1;
#pragma unroll
    for (int o = 0; o < KM; ++o)
      if (o < k && hi[o] - lo[o] > lmax) { lmax = hi[o] - lo[o]; m = o; }
    if (lmax <= 32) break;
    I sp[KM];
    int32_t u[KM];
#pragma unroll
    for (int o = 0; o < KM; ++o) {
      if (o < k) {
        const I len = hi[o] - lo[o];
        if (len > 0) {
          if constexpr (sizeof(I) == 4) sp[o] = lo[o] + (I)(((uint32_t)(lane + 1) * (uint32_t)len) / 33u);
          else sp[o] = lo[o] + ((int64_t)(lane + 1) * len) / 33;
          u[o] = (int32_t)ldg(cp[o] + sp[o]);
        } else { sp[o] = lo[o]; u[o] = INF; }
      }
    }
    int32_t cand = 0;
    I own = 0, spm = 0;
#pragma unroll
    for (int o = 0; o < KM; ++o)
      if (o == m) { cand = u[o]; spm = sp[o]; own = sp[o] - lo[o]; }
    I L = own, U = own;
    I Lo[KM], Uo[KM];
#pragma unroll
    for (int o = 0; o < KM; ++o) {
      Lo[o] = Uo[o] = 0;
      if (o < k && o != m) {   // (the candidates' own window m brackets itself: no rank search)
        const I len = hi[o] - lo[o];
        const int j = lanes_less(u[o], cand, len > 0 ? 32 : 0);
        const I sjm = __shfl_sync(kFull, sp[o], j > 0 ? j - 1 : 0);
        const I sj = __shfl_sync(kFull, sp[o], j < 32 ? j : 31);
        Lo[o] = j > 0 ? sjm - lo[o] + 1 : 0;
        Uo[o] = j < 32 ? sj - lo[o] : len;
        L += Lo[o];
        U += Uo[o];
      }
    }
    const unsigned below = __ballot_sync(kFull, U <= R);   // candidates <= v*
    const unsigned above = __ballot_sync(kFull, L > R);    // candidates >  v*
    const int ia = below ? 31 - __clz(below) : -1;
    const int ib = above ? __ffs(above) - 1 : 32;
    I drop = 0;
#pragma unroll
    for (int o = 0; o < KM; ++o) {
      if (o < k) {
        const I la = __shfl_sync(kFull, o == m ? spm - lo[o] : Lo[o], ia >= 0 ? ia : 0);
        const I ub = __shfl_sync(kFull, o == m ? spm - lo[o] : Uo[o], ib < 32 ? ib : 0);
        const I nlo = ia >= 0 ? lo[o] + la : lo[o];
        const I nhi = ib < 32 ? lo[o] + ub : hi[o];
        drop += nlo - lo[o];
        lo[o] = nlo;
        hi[o] = nhi;
      }
    }
    R -= drop;
  }
  // ---- exact resolution: every window holds <= 32 entries, lane l holds entry l of each
  int32_t e[KM];
#pragma unroll
  for (int o = 0; o < KM; ++o)
    if (o < k) e[o] = (lane < hi[o] - lo[o]) ? (int32_t)ldg(cp[o] + lo[o] + lane) : INF;
  // rank of lane l's entry of window o in the multiset union ordered by (column, operand):
  // entries of lower operands with a column <= it, of higher operands with a column < it, and the l
  // entries before it in its own window -- unique ranks, so exactly one entry has rank R
  int32_t vstar = INF;
  bool found = false;   // warp-uniform: the one entry of rank R is found, the other windows are skipped
#pragma unroll
  for (int o = 0; o < KM; ++o) {
    if (o < k && !found && hi[o] > lo[o]) {
      const int32_t x = e[o];
      int rank = lane;
#pragma unroll
      for (int o2 = 0; o2 < KM; ++o2) {
        if (o2 < k && o2 != o && hi[o2] > lo[o2]) {
          const int n2 = (int)(hi[o2] - lo[o2]);
          rank += lanes_less(e[o2], (o2 < o && x != INF) ? x + 1 : x, n2);
        }
      }
      const unsigned hm = __ballot_sync(kFull, x != INF && (I)rank == R);
      if (hm) { vstar = __shfl_sync(kFull, x, __ffs(hm) - 1); found = true; }
    }
  }
  col = vstar;
#pragma unroll
  for (int o = 0; o < KM; ++o)
    if (o < k) pos[o] = lo[o] + __popc(__ballot_sync(kFull, e[o] < vstar));
}

template <int KM>
__device__ __noinline__ void warp_kway_select64(const OpsArg& a, int k, int64_t (&lo)[KM], int64_t (&hi)[KM], int64_t R,
                                               Boundary& b) {
  const int32_t* cp[KM];
  int64_t l64[KM], h64[KM], p64[KM];
#pragma unroll
  for (int o = 0; o < KM; ++o)
    if (o < k) { cp[o] = a.op[o].crd + lo[o]; l64[o] = 0; h64[o] = hi[o] - lo[o]; }
  warp_kway_select_t<KM, int64_t>(cp, k, l64, h64, R, b.col, p64);
#pragma unroll
  for (int o = 0; o < KM; ++o)
    if (o < k) b.pos[o] = lo[o] + p64[o];
}

// The (R+1)-th smallest column of the multiset union of the row segments crd_o[lo_o, hi_o) (absolute
// positions) and its lower-bound position in every operand: the inner level of FindPartition.
template <int KM>
__device__ __forceinline__ void warp_kway_select(const OpsArg& a, int k, int64_t (&lo)[KM], int64_t (&hi)[KM], int64_t R,
                                              Boundary& b) {
  const int32_t* cp[KM];
  int64_t tot = 0;
#pragma unroll
  for (int o = 0; o < KM; ++o)
    if (o < k) { cp[o] = a.op[o].crd + lo[o]; tot += hi[o] - lo[o]; }
  if (tot < ((int64_t)1 << 26)) {
    int32_t l32[KM], h32[KM], p32[KM];
#pragma unroll
    for (int o = 0; o < KM; ++o)
      if (o < k) { l32[o] = 0; h32[o] = (int32_t)(hi[o] - lo[o]); }
    warp_kway_select_t<KM, int32_t>(cp, k, l32, h32, (int32_t)R, b.col, p32);
#pragma unroll
    for (int o = 0; o < KM; ++o)
      if (o < k) b.pos[o] = lo[o] + p32[o];
  } else {
    warp_kway_select64<KM>(a, k, lo, hi, R, b);   // segments of 2^26 entries or more: out of line
  }
}

// FindPartition (Alg. 1) for query Q, executed by one full warp; every lane returns
// the same boundary.  Level i (rows): highest outer position x with sum_o pos_o[x] <= Q (Listing 5
// C_i; for DCSR the compressed row level is searched in its position space).  Level j:
// residual R = Q - C_i(x); one operand -> the position is Q itself (position space);
// k operands -> the highest column v with sum_o (lb_o(v) - seg_o) <= R, found by a 32-ary search
// over column values in which every lane runs the per-operand lb_search of Listing 7 inside windows
// that narrow round by round.
template <int KM = NACHO_MAX_K>
__device__ __forceinline__ Boundary warp_find_boundary(const OpsArg& a, int64_t Q, int64_t outer_lo, int64_t outer_hi) {
  Boundary b;
  const int k = a.k;
  // ---- level i
  auto outer_ok = [&](int64_t x) {
    if (a.pos_shared) return (int64_t)k * ldg(a.op[0].pos + x) <= Q;   // one load instead of k
    int64_t s = 0;
#pragma unroll
    for (int o = 0; o < KM; ++o) if (o < k) s += ldg(a.op[o].pos + x);
    return s <= Q;
  };
  const int64_t x = warp_highest_true(outer_lo, outer_hi, outer_ok);
  if (x >= a.op[0].nouter) { set_end(a, b); return b; }
  b.row_pos = x;
  b.row = a.op[0].outer ? (int64_t)ldg(a.op[0].outer + x) : x;
  if (k == 1) {
    b.pos[0] = Q;
    b.col = ldg(a.op[0].crd + Q);
    return b;
  }
  // ---- level j: the (R+1)-th smallest column of the multiset union of the row's k segments
  int64_t lo[KM], hi[KM];
  int64_t R = Q;
#pragma unroll
  for (int o = 0; o < KM; ++o) {
    if (o < k) {
      lo[o] = ldg((a.pos_shared ? a.op[0].pos : a.op[o].pos) + x);
      hi[o] = ldg((a.pos_shared ? a.op[0].pos : a.op[o].pos) + x + 1);
      R -= lo[o];
    }
  }
  warp_kway_select<KM>(a, k, lo, hi, R, b);
  return b;
}


// First index of the run of `row` that ends at `end` in a carry-row array (the run is contiguous:
// entries before it hold other rows or -1).  Warp-cooperative: exponential probes end - 2^lane
// bracket the start, then 32-ary search -- O(log32 run) rounds of loads instead of a 32-per-round
// walk (a dense row spans ~10^4..10^5 partitions).
__device__ __forceinline__ int64_t warp_run_start(const int64_t* keys, int64_t end, int64_t row) {
  const int lane = threadIdx.x & 31;
  const int64_t probe = end - ((int64_t)1 << lane);
  const bool in = probe >= 0 && lane < 62 && keys[probe < 0 ? 0 : probe] == row;
  const unsigned m = __ballot_sync(kFull, in);
  const int L = __ffs(~m) - 1;   // first lane whose probe left the run (m == kFull cannot happen below 2^31)
  if (L < 0) return 0;
  // the start lies in (end - 2^L, end - 2^(L-1)]  (L = 0: the start is end itself)
  if (L == 0) return end;
  int64_t hi = end - ((int64_t)1 << (L - 1));            // in the run
  int64_t lo = end - ((int64_t)1 << L) + 1;              // first candidate
  if (lo < 0) lo = 0;
  // least j in [lo, hi] with keys[j] == row (a monotone predicate on this interval)
  while (lo < hi) {
    const int64_t span = hi - lo;
    const int64_t x = lo + ((int64_t)lane * span) / 32;   // lane 0 probes lo
    const bool ok = keys[x] == row;
    const unsigned mm = __ballot_sync(kFull, ok);
    const int f = __ffs(mm) - 1;                          // first lane inside the run
    if (f < 0) { lo = __shfl_sync(kFull, x, 31) + 1; continue; }   // all probes before the start
    const int64_t xf = __shfl_sync(kFull, x, f);
    const int64_t xp = __shfl_sync(kFull, x, f > 0 ? f - 1 : 0);
    if (f == 0) { hi = xf; break; }
    lo = xp + 1;
    hi = xf;
  }
  return hi;
}

// ------------------------------------------------------------------ scans
template <typename T>
__device__ __forceinline__ T warp_incl_sum(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const T u = __shfl_up_sync(kFull, v, d);
    if (lane >= d) v += u;
  }
  return v;
}

// Block-wide exclusive sum of one value per thread; returns the exclusive prefix and writes the
// block total to *total.  `red` must hold >= THREADS/32 elements of shared memory.
template <int THREADS, typename T>
__device__ __forceinline__ T block_excl_sum(T v, T* red, T* total) {
  constexpr int W = THREADS / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const T inc = warp_incl_sum(v);
  if (lane == 31) red[w] = inc;
  __syncthreads();
  if (w == 0) {
    T t = lane < W ? red[lane] : T(0);
    const T ti = warp_incl_sum(t);
    if (lane < W) red[lane] = ti - t;  // exclusive warp offsets
    if (lane == W - 1) red[W] = ti;
  }
  __syncthreads();
  const T res = red[w] + inc - v;
  *total = red[W];
  __syncthreads();
  return res;
}

}  // namespace nacho
