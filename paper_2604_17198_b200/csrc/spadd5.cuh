// spadd5.cuh -- single-read k-way SpAdd Z = A_0 + ... + A_{k-1} (CSR) over a k-operand partition:
// the assembly (union count), the prefix sum of the counts and
// the compute (fill) of Fig. 7a in ONE pass over the operands, one CTA per partition.
//
// Per partition p (rows [b_p.row, b_{p+1}.row], positions [b_p.pos[o], b_{p+1}.pos[o]) of operand o):
//   1. one thread issues 1-D bulk copies (cp.async.bulk -> UBLKCP, completion on an mbarrier) of
//      every operand's crd and val range into shared memory (16-byte-aligned slot runs; the < 4
//      unaligned tail entries by plain loads), while all threads mark the first entry of every row
//      that starts inside the partition (Listing 8's row loop bounds) and record the
//      per-row merged offsets ML[l] = sum_o (pos_o[row0 + l] - b_p.pos[o]);
//   2. a block max-scan of the marks gives every entry its partition-local row; the crd words are
//      turned into 32-bit keys (local row << cb) | col in place;
//   3. k - 1 stable merge-path stages (ties keep operand order) merge the operand runs; the last
//      stage folds equal keys left to right in operand order from the first present value (R9)
//      and counts the union -- the assembly count cnt_p;
//   4. the count is published at once (decoupled look-back state "aggregate"), the union is
//      compacted in shared memory, and warp 0 resolves the exclusive prefix of the counts of
//      partitions < p (the look-back) -- the write offset off_p;
//   5. Z.crd / Z.val are written coalesced at off_p, and Z.pos[r] = off_p + U[ML[r - row0]] for the
//      rows the partition owns (R7: rows (b_p.row, b_{p+1}.row]), U being the exclusive count of
//      union entries before each merged position.
// A partition spanning more rows than a sub-tile holds (lmax: the key's row bits, the ML capacity)
// runs as row-aligned sub-tiles, counted first and emitted after the look-back (two reads; rare).
#pragma once
#include "common.cuh"
#include "tma.cuh"

namespace nacho {

#ifndef NACHO_S5_THREADS   // tuning override (CTA size; the tile is kS5Threads * kS5VT slots)
#define NACHO_S5_THREADS 256
#endif
#ifndef NACHO_S5_MINB      // tuning override (__launch_bounds__ min blocks per SM)
#define NACHO_S5_MINB 4
#endif
constexpr int kS5Threads = NACHO_S5_THREADS;
constexpr int kS5VT = 8;
constexpr int kS5Slots = kS5Threads * kS5VT;   // shared-memory slots per (sub-)tile
constexpr int kS5LMax = 1024;                 // rows per sub-tile (ML capacity)
constexpr uint32_t kS5Inf = 0xffffffffu;      // larger than every key (keys < 2^32 - 2^cb)

// Entries (summed over the k operands) a partition may hold: the slots minus the pad of the bulk
// copies (<= 3 head slots per operand, and 1..4 tail slots: a sentinel key after every run).
__host__ __device__ constexpr int s5_max_entries(int k) { return kS5Slots - 7 * k; }

template <typename V>
struct S5Args {
  OpsArg ops;
  PartsArg parts;
  int32_t cb;         // column bits of the keys
  int32_t lmax;       // rows per sub-tile: <= kS5LMax and < 2^(32 - cb)
  int32_t use_bulk;   // crd / val bases 16-byte aligned: bulk copies; else plain loads
  unsigned long long* state;   // [P] look-back states, [P] = ticket counter (zeroed by the host)
  int64_t* part_off;           // [P+1] or null
  int64_t* z_pos;
  int32_t* z_crd;
  V* z_val;
};

template <typename V, int K>
struct S5Smem {
  uint32_t key0[kS5Slots + 16];   // crd (bulk copy) -> keys in place (+ read-past-end room)
  V val[kS5Slots];                 // values (bulk copy) -> compacted union values
  uint32_t key1[kS5Slots + 16];   // row marks -> merge output -> compacted union columns
  uint16_t src1[kS5Slots + 16];
  uint32_t key2[K >= 4 ? kS5Slots + 16 : 1];
  uint16_t src2[K >= 4 ? kS5Slots + 16 : 1];
  int32_t U[kS5Slots + 1];     // union entries before each merged position
  int32_t ML[kS5LMax + 1];     // merged position of each owned row's first entry
  int64_t s[K], e[K];          // positions of the current (sub-)tile per operand
  int32_t soff[K], n[K], base[K + 1];
  int64_t tile, r0, r1, a0, off;
  int32_t lrows;               // owned rows of the current sub-tile: l = 1 .. lrows
  int32_t wred[kS5Threads / 32];
  int32_t total;
  uint64_t bar;
};

// ------------------------------------------------------------------ block scans
// Exclusive sum over the CTA (every thread calls); *total receives the sum.  Two __syncthreads;
// every warp scans the per-warp sums with shuffles.
__device__ __forceinline__ int s5_block_excl(int v, int32_t* wred, int* total) {
  constexpr int NW = kS5Threads / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int y = __shfl_up_sync(kFull, x, d);
    if (lane >= d) x += y;
  }
  if (lane == 31) wred[w] = x;
  __syncthreads();
  int ws = lane < NW ? wred[lane] : 0;
#pragma unroll
  for (int d = 1; d < NW; d <<= 1) {
    const int y = __shfl_up_sync(kFull, ws, d);
    if (lane >= d) ws += y;
  }
  const int pre = __shfl_sync(kFull, ws, (w + 31) & 31);   // inclusive sum of warps < w (lane w - 1)
  *total = __shfl_sync(kFull, ws, NW - 1);
  __syncthreads();
  return (w ? pre : 0) + x - v;
}

// Exclusive max over the CTA (values >= 0; 0 for thread 0).
__device__ __forceinline__ uint32_t s5_block_excl_max(uint32_t v, int32_t* wred) {
  constexpr int NW = kS5Threads / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, x, d);
    if (lane >= d) x = max(x, y);
  }
  if (lane == 31) wred[w] = (int32_t)x;
  __syncthreads();
  uint32_t ws = lane < NW ? (uint32_t)wred[lane] : 0u;
#pragma unroll
  for (int d = 1; d < NW; d <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, ws, d);
    if (lane >= d) ws = max(ws, y);
  }
  const uint32_t pre = __shfl_sync(kFull, ws, (w + 31) & 31);
  __syncthreads();
  const uint32_t ex = __shfl_up_sync(kFull, x, 1);
  return max(w ? pre : 0u, lane ? ex : 0u);
}

// ------------------------------------------------------------------ merge path
// Split of output diagonal d of the stable merge of X[0,a) and Y[0,b) (ties: X first).
__device__ __forceinline__ int s5_split(const uint32_t* X, int a, const uint32_t* Y, int b, int d) {
  int lo = d > b ? d - b : 0, hi = d < a ? d : a;
  while (lo < hi) {
    const int m = (lo + hi) >> 1;
    if (X[m] <= Y[d - 1 - m]) lo = m + 1; else hi = m;
  }
  return lo;
}

// One merge step: the smaller head (X on ties: stable, lower operands first) and its value slot.
// Every run ends in a sentinel key kS5Inf, so the heads are re-read without bounds checks (items
// past the merged length read slack slots and are discarded by the caller).
template <bool XSRC>
__device__ __forceinline__ void s5_step(const uint32_t* X, const uint16_t* XS, int xs0, const uint32_t* Y, int ys0,
                                        int& i, int& j, uint32_t& xk, uint32_t& yk, uint32_t& key, int& slot) {
  const bool px = xk <= yk;
  key = px ? xk : yk;
  slot = px ? (XSRC ? (int)XS[i] : xs0 + i) : ys0 + j;
  i += px ? 1 : 0;
  j += px ? 0 : 1;
  xk = X[i];
  yk = Y[j];
}

// One intermediate stage: items [d, d + VT) of merge(X, Y) with their value slots into (OK, OS),
// and the sentinel after the merged run.  X's slots: XSRC ? xs[i] : xs0 + i; Y's: ys0 + j.
template <bool XSRC>
__device__ __forceinline__ void s5_merge_stage(const uint32_t* X, const uint16_t* xs, int xs0, int a,
                                               const uint32_t* Y, int ys0, int b, uint32_t* OK, uint16_t* OS) {
  const int n = a + b;
  const int d = threadIdx.x * kS5VT;
  if (d >= n) {
    if (d == 0) OK[0] = kS5Inf;   // empty merge: the sentinel alone
    return;
  }
  int i = s5_split(X, a, Y, b, d), j = d - i;
  uint32_t xk = X[i], yk = Y[j];
  uint32_t ko[kS5VT];
  int so[kS5VT];
#pragma unroll
  for (int v = 0; v < kS5VT; ++v) s5_step<XSRC>(X, xs, xs0, Y, ys0, i, j, xk, yk, ko[v], so[v]);
  uint4* ok4 = reinterpret_cast<uint4*>(OK + d);
  ok4[0] = make_uint4(ko[0], ko[1], ko[2], ko[3]);
  ok4[1] = make_uint4(ko[4], ko[5], ko[6], ko[7]);
  *reinterpret_cast<uint4*>(OS + d) = make_uint4(so[0] | (so[1] << 16), so[2] | (so[3] << 16), so[4] | (so[5] << 16),
                                                  so[6] | (so[7] << 16));
  if (d + kS5VT >= n) OK[n] = kS5Inf;
}

// ------------------------------------------------------------------ decoupled look-back
constexpr unsigned long long kS5Agg = 1ull << 62, kS5Incl = 2ull << 62, kS5Val = (1ull << 62) - 1;
#ifndef NACHO_LB_SLEEP_MAX   // look-back polling back-off cap (ns)
#define NACHO_LB_SLEEP_MAX 256
#endif

// Warp 0: exclusive prefix of the counts of tiles < t, after the aggregate of t was published.
__device__ __forceinline__ int64_t s5_lookback(unsigned long long* st, int64_t t) {
  const int lane = threadIdx.x & 31;
  unsigned long long excl = 0;
  int64_t base = t - 1;
  for (;;) {
    const int64_t q = base - lane;
    unsigned long long v = q >= 0 ? ld_acquire(st + q) : kS5Incl;
    int first;
    unsigned ns = 32;
    for (;;) {
      const unsigned ready = __ballot_sync(kFull, (v >> 62) != 0);
      const unsigned incl = __ballot_sync(kFull, (v >> 62) == 2);
      first = incl ? __ffs(incl) - 1 : 32;   // nearest predecessor with an inclusive prefix
      const unsigned need = first >= 31 ? kFull : ((2u << first) - 1);
      if ((ready & need) == need) break;
      if ((v >> 62) == 0) { __nanosleep(ns); ns = ns < NACHO_LB_SLEEP_MAX ? 2 * ns : ns; v = ld_acquire(st + q); }
    }
    unsigned long long s = lane <= first ? (v & kS5Val) : 0ull;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) s += __shfl_xor_sync(kFull, s, d);
    excl += s;
    if (first < 32) break;
    base -= 32;
  }
  return (int64_t)excl;
}

// ------------------------------------------------------------------ one (sub-)tile
// mode 0: count only (returns the union size).  mode 1: count, publish, look-back, emit.
// mode 2: emit at the known offset sh.off (fallback second pass).
template <typename V, int K>
__device__ __forceinline__ int s5_subtile(const S5Args<V>& a, S5Smem<V, K>& sh, int j, int nsub, int mode, uint32_t& phase) {
  const int tid = threadIdx.x;
  const int lmax = a.lmax;
  // ---- (sub-)tile bounds: rows [a0, a0 + lmax) (the last one up to r1), owned Z.pos rows a0 + 1 ..
#pragma unroll
  for (int o = 0; o < K; ++o) {   // static operand index: no local copy of the kernel parameters
    if (tid == o) {
      const OpView& op = a.ops.op[o];
      const int64_t a0 = sh.r0 + (int64_t)j * lmax;
      const int64_t L = sh.r1 - sh.r0;
      int64_t s = a.parts.pos[sh.tile * K + o], e = a.parts.pos[(sh.tile + 1) * K + o];
      if (j > 0) s = ldg(op.pos + a0);
      if (j < nsub - 1) e = ldg(op.pos + a0 + lmax);
      sh.s[o] = s;
      sh.e[o] = e;
      if (o == 0) {
        sh.a0 = a0;
        sh.lrows = (int32_t)(j < nsub - 1 ? lmax : L - (int64_t)j * lmax);
      }
    }
  }
  __syncthreads();
  if (tid == 0) {   // slot layout: operand o's run at soff[o], 16-byte-aligned region base[o]
    int b = 0;
#pragma unroll
    for (int o = 0; o < K; ++o) {
      const int n = (int)(sh.e[o] - sh.s[o]);
      sh.base[o] = b;
      sh.soff[o] = b + (int)(sh.s[o] & 3);
      sh.n[o] = n;
      b = (sh.soff[o] + n + 4) & ~3;   // >= 1 pad slot: the run's sentinel
    }
    sh.base[K] = b;
    // bulk copies of the aligned middle [s & ~3, e & ~3) of every run
    uint32_t bytes = 0;
    int64_t lo[K], hi[K];
#pragma unroll
    for (int o = 0; o < K; ++o) {
      lo[o] = sh.s[o] & ~int64_t(3);
      hi[o] = sh.e[o] & ~int64_t(3);
      if (!a.use_bulk || hi[o] <= sh.s[o]) hi[o] = lo[o];
      bytes += (uint32_t)(hi[o] - lo[o]) * (4u + (uint32_t)sizeof(V));
    }
    fence_proxy_async();   // earlier generic accesses of these buffers before the async writes
    if (bytes) {
      mbar_arrive_expect_tx(&sh.bar, bytes);
#pragma unroll
      for (int o = 0; o < K; ++o) {
        if (hi[o] > lo[o]) {
          const OpView& op = a.ops.op[o];
          const uint32_t nb = (uint32_t)(hi[o] - lo[o]);
          bulk_g2s(sh.key0 + sh.base[o], op.crd + lo[o], nb * 4u, &sh.bar);
          bulk_g2s(sh.val + sh.base[o], static_cast<const V*>(op.val) + lo[o], nb * (uint32_t)sizeof(V), &sh.bar);
        }
      }
    } else {
      mbar_arrive(&sh.bar);
    }
  }
  __syncthreads();
  const int S = sh.base[K];
  // ---- entries the bulk copies do not cover (plain loads), and the row-mark initialisation:
  // every slot of operand o's region starts at mark (o << 16) | 0 (local row 0)
#pragma unroll
  for (int o = 0; o < K; ++o) {
    const int64_t s = sh.s[o], e = sh.e[o];
    int64_t from = e & ~int64_t(3);
    if (!a.use_bulk || from < s) from = s;
    const OpView& op = a.ops.op[o];
    for (int64_t q = from + tid; q < e; q += kS5Threads) {
      const int slot = sh.soff[o] + (int)(q - s);
      sh.key0[slot] = (uint32_t)ldg(op.crd + q);
      sh.val[slot] = ldg(static_cast<const V*>(op.val) + q);
    }
  }
  for (int c = tid; c < (S >> 2); c += kS5Threads) {
    const int slot = c << 2;
    uint32_t o = 0;
#pragma unroll
    for (int oo = 1; oo < K; ++oo) o += slot >= sh.base[oo] ? 1u : 0u;
    const uint32_t m = o << 16;
    reinterpret_cast<uint4*>(sh.key1)[c] = make_uint4(m, m, m, m);
  }
  __syncthreads();
  // ---- row marks: the first entry of every row l in [1, lrows] of each operand (Listing 8 bounds)
  const int lrows = sh.lrows;
  for (int l = tid + 1; l <= lrows; l += kS5Threads) {
    int msum = 0;
#pragma unroll
    for (int o = 0; o < K; ++o) {
      const OpView& op = a.ops.op[o];
      const int64_t p = min(ldg(op.pos + sh.a0 + l), sh.e[o]);
      const int64_t pn = l < lrows ? min(ldg(op.pos + sh.a0 + l + 1), sh.e[o]) : sh.e[o];
      const int rel = (int)(p - sh.s[o]);
      msum += rel;
      if (pn > p) sh.key1[sh.soff[o] + rel] = ((uint32_t)o << 16) | (uint32_t)l;
    }
    sh.ML[l] = msum;
  }
  __syncthreads();
  // ---- local row of every slot (max-scan of the marks), keys in place
  {
    const int d = tid * kS5VT;
    uint32_t m[kS5VT];
    const uint4 m0 = reinterpret_cast<const uint4*>(sh.key1 + d)[0];
    const uint4 m1 = reinterpret_cast<const uint4*>(sh.key1 + d)[1];
    m[0] = m0.x; m[1] = m0.y; m[2] = m0.z; m[3] = m0.w; m[4] = m1.x; m[5] = m1.y; m[6] = m1.z; m[7] = m1.w;
#pragma unroll
    for (int v = 1; v < kS5VT; ++v) m[v] = max(m[v], m[v - 1]);
    const uint32_t pre = s5_block_excl_max(m[kS5VT - 1], sh.wred);
    while (!mbar_try_wait(&sh.bar, phase)) {
    }
    if (d < S) {
      uint4* k4 = reinterpret_cast<uint4*>(sh.key0 + d);
      uint4 c0 = k4[0], c1 = k4[1];
      const int cb = a.cb;
      auto mk = [&](uint32_t c, uint32_t mm) { return ((max(mm, pre) & 0xffffu) << cb) | c; };
      c0.x = mk(c0.x, m[0]); c0.y = mk(c0.y, m[1]); c0.z = mk(c0.z, m[2]); c0.w = mk(c0.w, m[3]);
      c1.x = mk(c1.x, m[4]); c1.y = mk(c1.y, m[5]); c1.z = mk(c1.z, m[6]); c1.w = mk(c1.w, m[7]);
      k4[0] = c0;
      k4[1] = c1;
#pragma unroll
      for (int o = 0; o < K; ++o) {   // the sentinel after each run (a pad slot)
        const int z = sh.soff[o] + sh.n[o];
        if (z >= d && z < d + kS5VT) sh.key0[z] = kS5Inf;
      }
    }
  }
  phase ^= 1u;
  __syncthreads();
  // ---- merge stages 1 .. K-2 (operand runs folded into a growing sorted prefix)
  const uint32_t* X = sh.key0 + sh.soff[0];
  const uint16_t* XS = sh.src1;
  const int xs0 = sh.soff[0];
  int na = sh.n[0];
#pragma unroll
  for (int st = 1; st + 1 < K; ++st) {
    uint32_t* OK = (st & 1) ? sh.key1 : sh.key2;
    uint16_t* OS = (st & 1) ? sh.src1 : sh.src2;
    if (st == 1) s5_merge_stage<false>(X, XS, xs0, na, sh.key0 + sh.soff[st], sh.soff[st], sh.n[st], OK, OS);
    else s5_merge_stage<true>(X, XS, xs0, na, sh.key0 + sh.soff[st], sh.soff[st], sh.n[st], OK, OS);
    __syncthreads();
    X = OK;
    XS = OS;
    na += sh.n[st];
  }
  // ---- last stage: merge, fold equal keys, count
  constexpr bool XSRC = K >= 3;
  const uint32_t* Y = K > 1 ? sh.key0 + sh.soff[K - 1] : sh.key0 + sh.soff[0] + sh.n[0];   // K = 1: the sentinel
  const int ys0 = K > 1 ? sh.soff[K - 1] : 0;
  const int nb = K > 1 ? sh.n[K - 1] : 0;
  const int n = na + nb;
  const int d = tid * kS5VT;
  const uint32_t cmask = (1u << a.cb) - 1u;
  V res[kS5VT];
  uint32_t col[kS5VT];
  uint32_t em = 0;   // bit v: item v ends a run this thread owns (one union entry)
  if (d < n) {
    int i = s5_split(X, na, Y, nb, d), jj = d - i;
    uint32_t pk = kS5Inf;
    if (d > 0) {
      const bool tx = i > 0 && (jj == 0 || X[i - 1] >= Y[jj - 1]);
      pk = tx ? X[i - 1] : Y[jj - 1];
    }
    uint32_t xk = X[i], yk = Y[jj];
    bool own = false;
    V acc = V(0);
#pragma unroll
    for (int v = 0; v < kS5VT; ++v) {
      uint32_t key;
      int slot;
      s5_step<XSRC>(X, XS, xs0, Y, ys0, i, jj, xk, yk, key, slot);
      const bool valid = d + v < n;
      const bool start = valid && key != pk;
      if (v > 0 && own && (start || !valid) && d + v - 1 < n) em |= 1u << (v - 1);
      own = own || start;
      if (own && valid) {
        const V x = sh.val[slot];
        acc = start ? x : acc + x;
      }
      res[v] = acc;
      col[v] = key & cmask;
      pk = key;
    }
    // the run holding the last item may continue past this thread's items (at most K - 1 more)
    if (own && d + kS5VT <= n) {
      em |= 1u << (kS5VT - 1);
#pragma unroll
      for (int r = 0; r < K - 1; ++r) {
        if (d + kS5VT + r >= n || (xk <= yk ? xk : yk) != pk) break;
        uint32_t key;
        int slot;
        s5_step<XSRC>(X, XS, xs0, Y, ys0, i, jj, xk, yk, key, slot);
        acc = acc + sh.val[slot];
      }
      res[kS5VT - 1] = acc;
    }
  }
  int total;
  const int cnt = __popc(em);
  const int ex = s5_block_excl(cnt, sh.wred, &total);   // syncs: every fold has read sh.val
  if (mode == 0) return total;
  if (mode == 1 && tid < 32) {   // publish the count at once, then resolve the offset
    const int64_t t = sh.tile;
    if (t == 0) {
      if (tid == 0) { st_release(a.state, kS5Incl | (unsigned long long)total); sh.off = 0; }
    } else {
      if (tid == 0) st_release(a.state + t, kS5Agg | (unsigned long long)total);
    }
  }
  // compacted union (columns in key1, values in val) and the union prefix U at merged positions
  if (d < n) {
    int e = ex;
#pragma unroll
    for (int v = 0; v < kS5VT; ++v) {
      if (d + v < n) sh.U[d + v] = e;
      if (em & (1u << v)) { sh.key1[e] = col[v]; sh.val[e] = res[v]; ++e; }
    }
  }
  if (tid == 0) sh.U[n] = total;
  if (mode == 1 && sh.tile > 0 && tid < 32) {
#ifdef NACHO_S5_NOLB   // timing experiment only: provisional offsets, no look-back (wrong output)
    int64_t excl = 0;
    for (int o = 0; o < K; ++o) excl += a.parts.pos[sh.tile * K + o];
#else
    const int64_t excl = s5_lookback(a.state, sh.tile);
#endif
    if (tid == 0) {
      st_release(a.state + sh.tile, kS5Incl | (unsigned long long)(excl + total));
      sh.off = excl;
    }
  }
  __syncthreads();
  const int64_t off = sh.off;
  for (int q = tid; q < total; q += kS5Threads) {
    a.z_crd[off + q] = (int32_t)sh.key1[q];
    a.z_val[off + q] = sh.val[q];
  }
  for (int l = tid + 1; l <= lrows; l += kS5Threads) a.z_pos[sh.a0 + l] = off + sh.U[sh.ML[l]];
  __syncthreads();   // buffers are reused by the next sub-tile
  return total;
}

template <typename V, int K>
__global__ void __launch_bounds__(kS5Threads, NACHO_S5_MINB) spadd5_kernel(const S5Args<V> a) {
  extern __shared__ __align__(128) unsigned char s5_raw[];
  S5Smem<V, K>& sh = *reinterpret_cast<S5Smem<V, K>*>(s5_raw);
  const int tid = threadIdx.x;
  const int P = a.parts.P;
  if (tid == 0) {
    sh.tile = (int64_t)atomicAdd(a.state + P, 1ull);   // ticket order: predecessors already run
    sh.r0 = a.parts.row[sh.tile];
    sh.r1 = a.parts.row[sh.tile + 1];
    mbar_init(&sh.bar, 1);
    fence_barrier_init();
  }
  __syncthreads();
  const int64_t t = sh.tile;
  const int64_t L = sh.r1 - sh.r0;
  const int lmax = a.lmax;
  uint32_t phase = 0;
  // one (sub-)tile in one pass (mode 1); or, spanning more rows than a sub-tile holds: count every
  // sub-tile (mode 0), publish + look-back, then emit every sub-tile at the known offset (mode 2)
  const bool single = L < lmax;
  const int nsub = single ? 1 : (int)((L + lmax) / lmax);
  const int niter = single ? 1 : 2 * nsub;
  int64_t total = 0, off = 0;
  for (int it = 0; it < niter; ++it) {   // one call site: the sub-tile body is inlined once
    if (!single && it == nsub) {
      if (tid < 32) {
        int64_t excl = 0;
        if (t == 0) {
          if (tid == 0) st_release(a.state, kS5Incl | (unsigned long long)total);
        } else {
          if (tid == 0) st_release(a.state + t, kS5Agg | (unsigned long long)total);
          excl = s5_lookback(a.state, t);
          if (tid == 0) st_release(a.state + t, kS5Incl | (unsigned long long)(excl + total));
        }
        if (tid == 0) sh.off = excl;
      }
      __syncthreads();
    }
    const int mode = single ? 1 : (it < nsub ? 0 : 2);
    if (mode == 2 && it == nsub) off = sh.off;
    const int c = s5_subtile<V, K>(a, sh, single ? 0 : it % nsub, nsub, mode, phase);
    if (mode == 1) { total = c; off = sh.off; }
    else if (mode == 0) total += c;
    else {
      if (tid == 0) sh.off += c;
      __syncthreads();
    }
  }
  if (tid == 0) {
    if (t == 0) a.z_pos[0] = 0;
    if (a.part_off) {
      a.part_off[t] = off;
      if (t == P - 1) a.part_off[P] = off + total;
    }
  }
}

}  // namespace nacho
