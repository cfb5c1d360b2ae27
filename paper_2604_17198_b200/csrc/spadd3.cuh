// spadd3.cuh -- the B200 k-way SpAdd kernel.
//
// Persistent CTAs, three per SM.  A CTA claims partitions in increasing order from a ticket counter,
// stages the partition's k operand ranges (crd, val) and row pointers into shared memory with 1-D
// TMA bulk copies (cp.async.bulk, one mbarrier) and computes their union:
//   1. row id of every entry: row starts scattered as marks, one max-scan (no per-entry search);
//   2. key = (local row, column) packed in 32 bits when the partition's row span and column range
//      fit 31 bits (else 64-bit keys on sub-chunks of half size, see sa_partition64);
//   3. k-1 plain merge-path stages (duplicates kept, ties in operand order, so every stage's output
//      positions are known and no scan is needed: merge path);
//   4. one pass folds each run of equal keys left-to-right (R9) and compacts it (one block scan).
// Every array that threads access in blocked order is padded (one word per 32) so the accesses are
// free of shared-memory bank conflicts.
// Modes:
//   kCount : assembly -- union size of every partition            -> cnt[p]
//   kFill  : compute  -- writes Z at part_off[p] and the owned Z.pos entries     (R7)
//   kFused : both in one pass; the write offset comes from a decoupled look-back over the partitions
//            (Merrill & Garland's single-pass prefix scan, cited by the paper at P:1475).  Tickets are
//            claimed when a CTA starts a partition, so a partition's predecessors started earlier.
// Requires every partition to hold <= TILE entries (true for nacho_auto_partitions); the generic
// chunking kernel of spadd.cuh covers larger partitions.
#pragma once
#include "common.cuh"
#include "spadd.cuh"
#include "tma.cuh"

namespace nacho {

enum SpaddMode { kCount = 0, kFill = 1, kFused = 2 };

// Optional phase timer (compile with -DNACHO_PROF): thread 0 of CTA 0 accumulates clock64 deltas.
#ifdef NACHO_PROF
__device__ unsigned long long g_phase[16];
#define NACHO_PHASE(id, last)                                            \
  do {                                                                   \
    if (blockIdx.x == 0 && threadIdx.x == 0) {                           \
      const unsigned long long _t = clock64();                           \
      g_phase[id] += _t - (last);                                        \
      (last) = _t;                                                       \
    }                                                                    \
  } while (0)
#else
#define NACHO_PHASE(id, last) do { } while (0)
#endif

#ifndef SA_MINB
#define SA_MINB 3
#endif

template <typename T>
struct Spadd2Args {
  OpsArg ops;
  PartsArg parts;
  int64_t* part_cnt;              // kCount: [P]
  int64_t* part_off;              // kFill: read [P+1]; kFused: written [P+1] (may be null)
  unsigned long long* lb_state;   // kFused: [P], zeroed before launch
  unsigned long long* ticket;     // partition ticket counter, zeroed before launch (null: static order)
  int64_t* z_pos;
  int32_t* z_crd;
  T* z_val;
};

constexpr int kSaThreads = 256;              // 8 warps
constexpr int kSaTile = 2048;                // entries per partition (sum over operands)
constexpr int kSaSpt = kSaTile / kSaThreads; // merged steps per thread
constexpr int kSaPosCap = 128;               // staged row pointers per operand
constexpr int kSaCrdCap = kSaTile + 8 * NACHO_MAX_K;
constexpr int kSaK0Cap = kSaTile + NACHO_MAX_K + 16;       // operand keys (32-bit words)
constexpr int kSaBufCap = 2176;                            // padded merge buffer (32-bit words)
constexpr int kSaChunk64 = 1016;                           // entries of a 64-bit sub-chunk

// Padded index of element i in a thread-blocked buffer (one pad element per 32 words).
template <typename KT>
__device__ __forceinline__ int pd(int i) { return sizeof(KT) == 4 ? i + (i >> 5) : i + (i >> 4); }

struct SaHeader {
  Boundary b0, b1;
  int64_t p;                     // partition id, -1: no more work
  int64_t pos_base;              // row of pos slot 0 (b0.row + 1)
  int32_t crd_off[NACHO_MAX_K];  // smem element offset of operand o's first entry (b0.pos[o])
  int32_t off[NACHO_MAX_K + 1];  // entry offsets of the operands in the concatenation
  int32_t pos_n;                 // staged rows per operand (0: none needed, -1: read pos from global)
  int32_t pos_shift;             // row pos_base sits at slot pos_shift (16-byte aligned copies)
};

template <typename T>
struct SaShared {
  uint64_t full;
  SaHeader h;
  Boundary cb0, cb1;             // current sub-chunk (64-bit path)
  int64_t red[kSaThreads / 32 + 1];
  uint32_t redu[kSaThreads / 32 + 1];
  int32_t redmin[kSaThreads / 32], redmax[kSaThreads / 32];
  int64_t bcast;
  alignas(16) int32_t crd[kSaCrdCap];
  alignas(16) T val[kSaCrdCap];
};

template <typename T>
__host__ __device__ constexpr size_t sa_smem_bytes(int k, bool vals) {
  // SaShared + pos slices + operand keys + 2 padded key buffers + 2 padded value buffers
  return ((sizeof(SaShared<T>) + 15) & ~size_t(15)) + size_t(k) * (kSaPosCap + 4) * 8 + size_t(kSaK0Cap) * 4 +
         2 * size_t(kSaBufCap) * 4 + 2 * size_t(kSaBufCap) * (vals ? sizeof(T) : 0) + 64;
}

// Exclusive sum over the CTA.
__device__ __forceinline__ int64_t sa_excl_sum(int64_t v, int64_t* red, int64_t* total) {
  constexpr int W = kSaThreads / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t inc = warp_incl_sum(v);
  if (lane == 31) red[w] = inc;
  __syncthreads();
  if (w == 0) {
    const int64_t t = lane < W ? red[lane] : 0;
    const int64_t ti = warp_incl_sum(t);
    if (lane < W) red[lane] = ti - t;
    if (lane == W - 1) red[W] = ti;
  }
  __syncthreads();
  const int64_t res = red[w] + inc - v;
  *total = red[W];
  __syncthreads();
  return res;
}

// Decoupled look-back (warp 0): exclusive prefix of the union sizes of partitions < p.
__device__ __forceinline__ int64_t sa_lookback(unsigned long long* st, int64_t p, int64_t nu) {
  constexpr unsigned long long INCL = 1ull << 63, AGG = 1ull << 62, VAL = (1ull << 62) - 1;
  const int lane = threadIdx.x & 31;
  unsigned long long excl = 0;
  if (p == 0) {
    if (lane == 0) st_release(st, INCL | (unsigned long long)nu);
    return 0;
  }
  if (lane == 0) st_release(st + p, AGG | (unsigned long long)nu);
  int64_t base = p - 1;
  for (;;) {
    const int64_t q = base - lane;
    unsigned long long v = q >= 0 ? ld_acquire(st + q) : INCL;
    int first;
    for (;;) {
      const unsigned ready = __ballot_sync(kFull, (v & (INCL | AGG)) != 0);
      const unsigned incl = __ballot_sync(kFull, (v & INCL) != 0);
      first = incl ? __ffs(incl) - 1 : 32;  // nearest inclusive predecessor
      const unsigned need = first >= 31 ? kFull : ((2u << first) - 1);
      if ((ready & need) == need) break;
      if (!(v & (INCL | AGG))) { __nanosleep(20); v = ld_acquire(st + q); }
    }
    unsigned long long s = (lane <= first) ? (v & VAL) : 0ull;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) s += __shfl_xor_sync(kFull, s, d);
    excl += s;
    if (first < 32) break;
    base -= 32;
  }
  if (lane == 0) st_release(st + p, INCL | (excl + (unsigned long long)nu));
  return (int64_t)excl;
}

// Inclusive max-scan of n (<= kSaTile) padded uint32 marks, in place.
__device__ __forceinline__ void sa_max_scan(uint32_t* v, int n, uint32_t* red) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  uint32_t loc[kSaSpt];
  uint32_t run = 0;
#pragma unroll
  for (int s = 0; s < kSaSpt; ++s) {
    const int j = tid * kSaSpt + s;
    const uint32_t x = j < n ? v[pd<uint32_t>(j)] : 0u;
    run = x > run ? x : run;
    loc[s] = run;
  }
  uint32_t inc = run;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t u = __shfl_up_sync(kFull, inc, d);
    if (lane >= d && u > inc) inc = u;
  }
  if (lane == 31) red[w] = inc;
  __syncthreads();
  uint32_t pre = 0;
  for (int ww = 0; ww < w; ++ww) pre = red[ww] > pre ? red[ww] : pre;
  uint32_t ex = __shfl_up_sync(kFull, inc, 1);
  if (lane == 0) ex = 0;
  pre = ex > pre ? ex : pre;
#pragma unroll
  for (int s = 0; s < kSaSpt; ++s) {
    const int j = tid * kSaSpt + s;
    if (j < n) v[pd<uint32_t>(j)] = loc[s] > pre ? loc[s] : pre;
  }
  __syncthreads();
}

// Keys of the entries [cs_o, ce_o) (offsets inside operand o's staged range) of every operand, rows
// counted from row0 (rows (row0, row_end] can start inside the ranges).  K0 holds operand o's keys
// at koff[o] .. koff[o] + (ce_o - cs_o) followed by an all-ones sentinel.
template <typename T, typename KT>
__device__ __forceinline__ void sa_keys(const Spadd2Args<T>& a, SaShared<T>& sh, const int64_t* pb, int k,
                                        const int* cs, const int* ce, const int* koff, KT* K0, uint32_t* rid,
                                        int rsh, int32_t cmin, int64_t row0, int64_t row_end) {
  const int tid = threadIdx.x;
  const SaHeader& h = sh.h;
  int n = 0;
  if (row_end - row0 >= (int64_t(1) << 28)) {
    // enormous row span (hypersparse CSR): row of every entry by binary search over pos
    for (int o = 0; o < k; ++o) {
      const int no = ce[o] - cs[o];
      const int32_t* c = sh.crd + h.crd_off[o] + cs[o];
      KT* d = K0 + koff[o];
      for (int j = tid; j < no; j += kSaThreads) {
        const int64_t gq = h.b0.pos[o] + cs[o] + j;
        int64_t lo = row0, hi = row_end;
        while (lo < hi) {
          const int64_t m = lo + ((hi - lo + 1) >> 1);
          if (ldg(a.ops.op[o].pos + m) <= gq) lo = m; else hi = m - 1;
        }
        d[j] = ((KT)(uint64_t)(lo - row0) << rsh) | (KT)(uint32_t)(c[j] - cmin);
      }
      if (tid == 0) d[no] = ~KT(0);
    }
    __syncthreads();
    return;
  }
  // marks: (o << 28) by default = "row0" of operand o; then the row starts inside the ranges
  for (int o = 0; o < k; ++o) {
    const int no = ce[o] - cs[o];
    for (int j = tid; j < no; j += kSaThreads) rid[pd<uint32_t>(n + j)] = (uint32_t)o << 28;
    n += no;
  }
  __syncthreads();
  {
    int base = 0;
    for (int o = 0; o < k; ++o) {
      const int64_t s = h.b0.pos[o] + cs[o], e = h.b0.pos[o] + ce[o];
      for (int64_t r = row0 + 1 + tid; r <= row_end; r += kSaThreads) {
        int64_t ps, pe;
        const int64_t slot = r - h.pos_base;
        if (h.pos_n > 0 && slot >= 0 && slot + 1 < h.pos_n) {
          const int64_t* po = pb + o * (kSaPosCap + 4) + h.pos_shift + slot;
          ps = po[0];
          pe = po[1];
        } else {
          ps = ldg(a.ops.op[o].pos + r);
          pe = ldg(a.ops.op[o].pos + r + 1);
        }
        if (ps >= s && ps < e && pe > ps) rid[pd<uint32_t>(base + (int)(ps - s))] = ((uint32_t)o << 28) | (uint32_t)(r - row0);
      }
      base += ce[o] - cs[o];
    }
  }
  __syncthreads();
  sa_max_scan(rid, n, sh.redu);
  int base = 0;
  for (int o = 0; o < k; ++o) {
    const int no = ce[o] - cs[o];
    const int32_t* c = sh.crd + h.crd_off[o] + cs[o];
    KT* d = K0 + koff[o];
    for (int j = tid; j < no; j += kSaThreads) {
      const uint32_t lr = rid[pd<uint32_t>(base + j)] & ((1u << 28) - 1);
      d[j] = ((KT)lr << rsh) | (KT)(uint32_t)(c[j] - cmin);
    }
    if (tid == 0) d[no] = ~KT(0);
    base += no;
  }
  __syncthreads();
}

// Key/value access to a merge input: operand keys (contiguous) or a padded stage output.
template <typename KT, typename T, bool PAD>
struct SaSrc {
  const KT* k;
  const T* v;
  __device__ __forceinline__ int ix(int i) const { return PAD ? pd<KT>(i) : i; }
  __device__ __forceinline__ KT key(int i) const { return k[ix(i)]; }
  __device__ __forceinline__ T val(int i) const { return v[ix(i)]; }
};

// Merge-path split of diagonal d0 of merge(X, Y) (ties take X first): the number of X entries among
// the first d0 merged ones.  4-ary steps (three independent probes per round).
template <class SX, class SY>
__device__ __forceinline__ int sa_split(const SX& X, int nx, const SY& Y, int ny, int d0) {
  int lo = max(0, d0 - ny), hi = min(d0, nx);
  while (lo < hi) {
    const int q1 = lo + ((hi - lo) >> 2), q2 = lo + ((hi - lo) >> 1), q3 = lo + 3 * ((hi - lo) >> 2);
    const bool c1 = X.key(q1) <= Y.key(d0 - 1 - q1);
    const bool c2 = X.key(q2) <= Y.key(d0 - 1 - q2);
    const bool c3 = X.key(q3) <= Y.key(d0 - 1 - q3);
    if (c3) lo = q3 + 1;
    else if (c2) { lo = q2 + 1; hi = q3; }
    else if (c1) { lo = q1 + 1; hi = q2; }
    else hi = q1;
  }
  return lo;
}

// One merge step: consumes the smaller head (X on ties), returns its key (and value), and refills
// the consumed head with a single shared-memory load.
template <typename T, bool VALS, typename KT, class SX, class SY>
__device__ __forceinline__ KT sa_step(const SX& X, const SY& Y, int& i, int& j, KT& xk, KT& yk, T& v) {
  const bool tx = xk <= yk;
  const KT key = tx ? xk : yk;
  if (VALS) v = *(tx ? X.v + X.ix(i) : Y.v + Y.ix(j));
  i += tx ? 1 : 0;
  j += tx ? 0 : 1;
  const KT nk = *(tx ? X.k + X.ix(i) : Y.k + Y.ix(j));
  xk = tx ? nk : xk;
  yk = tx ? yk : nk;
  return key;
}

// Plain merge path Z = merge(X, Y) keeping duplicates; ties take X first, so equal keys stay in
// operand order.  X[nx] and Y[ny] are all-ones sentinels.  Z (padded) gets its sentinel at nx + ny.
template <typename T, bool VALS, typename KT, class SX, class SY>
__device__ __forceinline__ void sa_pmerge(const SX& X, int nx, const SY& Y, int ny, KT* __restrict__ Z,
                                          T* __restrict__ Zv) {
  const int tid = threadIdx.x;
  const int total = nx + ny;
  const int d0 = min(total, tid * kSaSpt);
  const int d1 = min(total, d0 + kSaSpt);
  int i = sa_split(X, nx, Y, ny, d0), j = d0 - i;
  KT xk = X.key(i), yk = Y.key(j);
#pragma unroll
  for (int s = 0; s < kSaSpt; ++s) {
    if (d0 + s < d1) {
      T v;
      const int zi = pd<KT>(d0 + s);
      Z[zi] = sa_step<T, VALS>(X, Y, i, j, xk, yk, v);
      if (VALS) Zv[zi] = v;
    }
  }
  if (d0 < d1 && d1 == total) Z[pd<KT>(total)] = ~KT(0);
  if (total == 0 && tid == 0) Z[pd<KT>(0)] = ~KT(0);
}

// The last merge stage fused with the fold: merges the diagonal range [d0, d1) of merge(X, Y) in
// registers and folds every run of equal keys left to right in operand order (R9).  A run belongs to
// the thread holding its first entry; that thread reads past d1 while the run continues (a run has
// <= k entries, one per operand, so it never spans more than the next thread's range).  The runs are
// compacted into U (padded) with one block scan; returns the union size.
template <typename T, bool VALS, typename KT, class SX, class SY>
__device__ __forceinline__ int sa_pmerge_fold(const SX& X, int nx, const SY& Y, int ny, KT* __restrict__ Uk,
                                              T* __restrict__ Uv, int64_t* red) {
  const int tid = threadIdx.x;
  const int total = nx + ny;
  const int d0 = min(total, tid * kSaSpt);
  const int d1 = min(total, d0 + kSaSpt);
  int i = sa_split(X, nx, Y, ny, d0), j = d0 - i;
  KT xk = X.key(i), yk = Y.key(j);
  KT prev = ~KT(0);  // key of merged entry d0 - 1 (all-ones: none; never a key)
  if (d0 > 0) {
    const KT xp = i > 0 ? X.key(i - 1) : KT(0), yp = j > 0 ? Y.key(j - 1) : KT(0);
    prev = xp > yp ? xp : yp;
  }
  KT ok[kSaSpt];
  T ov[kSaSpt];
  unsigned em = 0;
  bool mine = false;
  T acc = T(0);
#pragma unroll
  for (int s = 0; s < kSaSpt; ++s) {
    if (d0 + s < d1) {
      T v;
      const KT key = sa_step<T, VALS>(X, Y, i, j, xk, yk, v);
      const bool fresh = key != prev;
      mine = fresh || mine;
      if (VALS) acc = fresh ? v : acc + v;
      prev = key;
      ok[s] = key;
      if (VALS) ov[s] = acc;
      const KT nxt = xk < yk ? xk : yk;
      if (mine && nxt != key) em |= 1u << s;
    }
  }
  if (d1 - d0 == kSaSpt && mine && (xk < yk ? xk : yk) == prev) {
    while ((xk < yk ? xk : yk) == prev) {  // finish my last run past d1
      T v;
      sa_step<T, VALS>(X, Y, i, j, xk, yk, v);
      if (VALS) acc = acc + v;
    }
    if (VALS) ov[kSaSpt - 1] = acc;
    em |= 1u << (kSaSpt - 1);
  }
  int64_t tot;
  int64_t idx = sa_excl_sum((int64_t)__popc(em), red, &tot);
#pragma unroll
  for (int s = 0; s < kSaSpt; ++s) {
    if ((em >> s) & 1u) { Uk[pd<KT>(idx)] = ok[s]; if (VALS) Uv[pd<KT>(idx)] = ov[s]; ++idx; }
  }
  __syncthreads();
  return (int)tot;
}

// Union of the keyed operands.  Returns nu; *Uk/*Uv point at the result (padded iff *upad).
template <typename T, bool VALS, typename KT>
__device__ __forceinline__ int sa_union(SaShared<T>& sh, int k, const int* cs, const int* ce, const int* koff,
                                        KT* K0, KT* B1, KT* B2, T* V1, T* V2, const KT** Uk, const T** Uv,
                                        bool* upad) {
  const SaHeader& h = sh.h;
  auto opsrc = [&](int o) { return SaSrc<KT, T, false>{K0 + koff[o], sh.val + h.crd_off[o] + cs[o]}; };
  if (k == 1) {
    *Uk = K0 + koff[0];
    *Uv = sh.val + h.crd_off[0] + cs[0];
    *upad = false;
    return ce[0] - cs[0];
  }
  if (k == 2) {
    *upad = true;
    *Uk = B1;
    *Uv = V1;
    return sa_pmerge_fold<T, VALS, KT>(opsrc(0), ce[0] - cs[0], opsrc(1), ce[1] - cs[1], B1, V1, sh.red);
  }
  int n = (ce[0] - cs[0]) + (ce[1] - cs[1]);
  sa_pmerge<T, VALS, KT>(opsrc(0), ce[0] - cs[0], opsrc(1), ce[1] - cs[1], B1, V1);
  __syncthreads();
  KT* Xk = B1; T* Xv = V1;
  KT* Dk = B2; T* Dv = V2;
  for (int o = 2; o < k - 1; ++o) {
    sa_pmerge<T, VALS, KT>(SaSrc<KT, T, true>{Xk, Xv}, n, opsrc(o), ce[o] - cs[o], Dk, Dv);
    __syncthreads();
    n += ce[o] - cs[o];
    KT* tk = Xk; Xk = Dk; Dk = tk;
    T* tv = Xv; Xv = Dv; Dv = tv;
  }
  const int nu = sa_pmerge_fold<T, VALS, KT>(SaSrc<KT, T, true>{Xk, Xv}, n, opsrc(k - 1), ce[k - 1] - cs[k - 1], Dk,
                                             Dv, sh.red);
  *Uk = Dk;
  *Uv = Dv;
  *upad = true;
  return nu;
}

// Writes U (nu entries) at `off` and Z.pos[r+1] for the owned rows r in [row_lo, row_hi], whose keys
// are (r - key_row0) << rsh.
template <typename T, typename KT, bool PAD>
__device__ __forceinline__ void sa_write(const Spadd2Args<T>& a, const KT* Uk, const T* Uv, int nu, int64_t off,
                                         int rsh, int32_t cmin, int64_t row_lo, int64_t row_hi, int64_t key_row0) {
  const int tid = threadIdx.x;
  const SaSrc<KT, T, PAD> U{Uk, Uv};
  const KT cmask = rsh >= 32 ? (KT)0xffffffffu : (KT)((1u << rsh) - 1u);
  for (int j = tid; j < nu; j += kSaThreads) {
    a.z_crd[off + j] = (int32_t)(U.key(j) & cmask) + cmin;
    a.z_val[off + j] = U.val(j);
  }
  for (int64_t r = row_lo + tid; r <= row_hi; r += kSaThreads) {
    const KT key = (KT)((KT)(r - key_row0 + 1) << rsh);  // first key of the next row
    int lo = 0, hi = nu;
    while (lo < hi) { const int m = (lo + hi) >> 1; if (U.key(m) < key) lo = m + 1; else hi = m; }
    a.z_pos[r + 1] = off + lo;
  }
}

template <typename T, typename KT>
__device__ __forceinline__ void sa_write_any(const Spadd2Args<T>& a, const KT* Uk, const T* Uv, bool upad, int nu,
                                             int64_t off, int rsh, int32_t cmin, int64_t row_lo, int64_t row_hi,
                                             int64_t key_row0) {
  if (upad) sa_write<T, KT, true>(a, Uk, Uv, nu, off, rsh, cmin, row_lo, row_hi, key_row0);
  else sa_write<T, KT, false>(a, Uk, Uv, nu, off, rsh, cmin, row_lo, row_hi, key_row0);
}

// Offset of partition p's output (kFill: given; kFused: look-back).  All threads return it.
template <typename T, int MODE>
__device__ __forceinline__ int64_t sa_offset(const Spadd2Args<T>& a, SaShared<T>& sh, int64_t p, int64_t nu) {
  if (MODE == kFill) return a.part_off[p];
  const int P = a.parts.P;
  if ((threadIdx.x >> 5) == 0) {
    const int64_t ex = sa_lookback(a.lb_state, p, nu);
    if ((threadIdx.x & 31) == 0) {
      sh.bcast = ex;
      if (a.part_off) { a.part_off[p] = ex; if (p == P - 1) a.part_off[P] = ex + nu; }
    }
  }
  __syncthreads();
  return sh.bcast;
}

// The rare path: a partition whose (row span, column range) does not fit 32-bit keys is processed as
// sub-chunks of <= kSaChunk64 entries cut by FindPartition, with 64-bit keys.  Kept out of line so its
// register needs do not burden the 32-bit fast path.
template <typename T, int MODE>
__device__ __noinline__ void sa_partition64(const Spadd2Args<T>& a, SaShared<T>& sh, const int64_t* pb,
                                            unsigned char* kbuf, T* V1, T* V2, int64_t p) {
  const int tid = threadIdx.x;
  const int k = a.ops.k;
  const int64_t M = a.ops.nrows;
  const SaHeader& h = sh.h;
  int cs[NACHO_MAX_K], ce[NACHO_MAX_K], koff[NACHO_MAX_K];
  uint64_t* K0 = reinterpret_cast<uint64_t*>(kbuf);
  uint64_t* B1 = reinterpret_cast<uint64_t*>(kbuf + kSaK0Cap * 4);
  uint64_t* B2 = reinterpret_cast<uint64_t*>(kbuf + kSaK0Cap * 4 + kSaBufCap * 4);
  uint32_t* rid = reinterpret_cast<uint32_t*>(B2);
  int64_t cB = 0, cPE = 0;
  for (int o = 0; o < k; ++o) { cB += h.b0.pos[o]; cPE += h.b1.pos[o]; }
  int64_t count = 0;
  int64_t off = 0;
  // fused needs the partition's union size before any write: pass 0 counts, pass 1 writes
  for (int pass = (MODE == kFused) ? 0 : 1; pass < 2; ++pass) {
    if (pass == 1 && MODE != kCount) {
      off = sa_offset<T, MODE>(a, sh, p, count);
      if (p == 0 && tid == 0) a.z_pos[0] = 0;
    }
    if (tid == 0) sh.cb0 = h.b0;
    __syncthreads();
    int64_t cb = cB;
    int64_t written = 0;
    for (;;) {
      const bool last = cPE - cb <= kSaChunk64;
      if (!last) {
        if (tid < 32) {
          const Boundary f = warp_find_boundary(a.ops, cb + (kSaChunk64 - (k - 1)), sh.cb0.row_pos, h.b1.row_pos);
          if (tid == 0) sh.cb1 = f;
        }
      } else if (tid == 0) {
        sh.cb1 = h.b1;
      }
      __syncthreads();
      for (int o = 0, acc = 0; o < k; ++o) {
        cs[o] = (int)(sh.cb0.pos[o] - h.b0.pos[o]);
        ce[o] = (int)(sh.cb1.pos[o] - h.b0.pos[o]);
        koff[o] = acc;
        acc += ce[o] - cs[o] + 1;
      }
      const int64_t row0 = sh.cb0.row;
      const int64_t row_end = sh.cb1.row < M - 1 ? sh.cb1.row : M - 1;
      sa_keys<T, uint64_t>(a, sh, pb, k, cs, ce, koff, K0, rid, 32, 0, row0, row_end);
      const uint64_t* Uk;
      const T* Uv;
      bool upad;
      const int nu = (pass == 0 || MODE == kCount)
                         ? sa_union<T, false, uint64_t>(sh, k, cs, ce, koff, K0, B1, B2, V1, V2, &Uk, &Uv, &upad)
                         : sa_union<T, true, uint64_t>(sh, k, cs, ce, koff, K0, B1, B2, V1, V2, &Uk, &Uv, &upad);
      if (pass == 1 && MODE != kCount)
        sa_write_any<T, uint64_t>(a, Uk, Uv, upad, nu, off + written, 32, 0, row0, (sh.cb1.row < M ? sh.cb1.row : M) - 1,
                                  row0);
      written += nu;
      __syncthreads();
      if (last) break;
      cb = 0;
      for (int o = 0; o < k; ++o) cb += sh.cb1.pos[o];
      if (tid == 0) sh.cb0 = sh.cb1;
      __syncthreads();
    }
    count = written;
  }
  if (MODE == kCount && tid == 0) a.part_cnt[p] = count;
}

template <typename T, int MODE>
__global__ void __launch_bounds__(kSaThreads, SA_MINB) spadd2_kernel(const __grid_constant__ Spadd2Args<T> a) {
  constexpr bool VALS = MODE != kCount;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  SaShared<T>& sh = *reinterpret_cast<SaShared<T>*>(smem_raw);
  const int k = a.ops.k;
  unsigned char* dyn = smem_raw + ((sizeof(SaShared<T>) + 15) & ~size_t(15));
  int64_t* pb = reinterpret_cast<int64_t*>(dyn);                        // [k][cap+4]
  dyn += size_t(k) * (kSaPosCap + 4) * 8;
  unsigned char* kbuf = dyn;                                            // K0 | B1 | B2
  dyn += size_t(kSaK0Cap) * 4 + 2 * size_t(kSaBufCap) * 4;
  T* V1 = reinterpret_cast<T*>(dyn);
  T* V2 = V1 + (VALS ? kSaBufCap : 0);

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t M = a.ops.nrows;
  const int P = a.parts.P;
  const SaHeader& h = sh.h;
  if (tid == 0) {
    mbar_init(&sh.full, 1);
    fence_barrier_init();
  }
  __syncthreads();
  unsigned long long tlast = clock64();
  (void)tlast;
  int64_t ps = blockIdx.x;
  for (int it = 0;; ++it, ps += gridDim.x) {
    // ---- claim a partition, stage its operand ranges and row pointers (thread 0)
    if (tid == 0) {
      SaHeader& hw = sh.h;
      const int64_t p = a.ticket ? (int64_t)atomicAdd(a.ticket, 1ull) : ps;
      hw.p = p < P ? p : -1;
      if (p < P) {
        load_boundary<T>(a.parts, k, p, hw.b0);
        load_boundary<T>(a.parts, k, p + 1, hw.b1);
        int acc = 0, co = 0;
        hw.off[0] = 0;
        uint32_t bytes = 0;
        for (int o = 0; o < k; ++o) {
          const int64_t s = hw.b0.pos[o], e = hw.b1.pos[o];
          acc += (int)(e - s);
          hw.off[o + 1] = acc;
          const int64_t s0 = s & ~int64_t(3);
          hw.crd_off[o] = co + (int)(s - s0);
          const int64_t lim = a.ops.op[o].nnz & ~int64_t(3);
          int64_t c = (e + 3) & ~int64_t(3);
          if (c > lim) c = lim;
          if (c < s0) c = s0;
          for (int64_t q = (c > s ? c : s); q < e; ++q) {  // unaligned tail at the array end
            sh.crd[co + (int)(q - s0)] = ldg(a.ops.op[o].crd + q);
            if (VALS) sh.val[co + (int)(q - s0)] = ldg(reinterpret_cast<const T*>(a.ops.op[o].val) + q);
          }
          bytes += (uint32_t)(c - s0) * (VALS ? 4 + sizeof(T) : 4);
          co += (int)(((e + 3) & ~int64_t(3)) - s0);
        }
        const int64_t r_hi = hw.b1.row < M - 1 ? hw.b1.row : M - 1;
        const int64_t span = r_hi - hw.b0.row;  // rows b0.row+1 .. r_hi (+1 for the end pointer)
        hw.pos_base = hw.b0.row + 1;
        hw.pos_n = (span >= 1 && span + 1 <= kSaPosCap) ? (int)(span + 1) : (span < 1 ? 0 : -1);
        hw.pos_shift = (int)(hw.pos_base & 1);
        if (hw.pos_n > 0) {
          for (int o = 0; o < k; ++o) {
            const int64_t s = hw.pos_base, e = s + hw.pos_n, s0 = s & ~int64_t(1);
            const int64_t lim = (a.ops.op[o].nouter + 1) & ~int64_t(1);
            int64_t c = (e + 1) & ~int64_t(1);
            if (c > lim) c = lim;
            if (c < s0) c = s0;
            for (int64_t q = (c > s ? c : s); q < e; ++q) pb[o * (kSaPosCap + 4) + (int)(q - s0)] = ldg(a.ops.op[o].pos + q);
            bytes += (uint32_t)(c - s0) * 8;
          }
        }
        fence_proxy_async();
        mbar_arrive_expect_tx(&sh.full, bytes);
        co = 0;
        for (int o = 0; o < k; ++o) {
          const int64_t s = hw.b0.pos[o], e = hw.b1.pos[o];
          const int64_t s0 = s & ~int64_t(3);
          const int64_t lim = a.ops.op[o].nnz & ~int64_t(3);
          int64_t c = (e + 3) & ~int64_t(3);
          if (c > lim) c = lim;
          if (c > s0) {
            bulk_g2s(&sh.crd[co], a.ops.op[o].crd + s0, (uint32_t)(c - s0) * 4, &sh.full);
            if (VALS)
              bulk_g2s(&sh.val[co], reinterpret_cast<const T*>(a.ops.op[o].val) + s0, (uint32_t)(c - s0) * sizeof(T),
                       &sh.full);
          }
          co += (int)(((e + 3) & ~int64_t(3)) - s0);
          if (hw.pos_n > 0) {
            const int64_t q0 = hw.pos_base, q1 = q0 + hw.pos_n, qs0 = q0 & ~int64_t(1);
            const int64_t plim = (a.ops.op[o].nouter + 1) & ~int64_t(1);
            int64_t pc = (q1 + 1) & ~int64_t(1);
            if (pc > plim) pc = plim;
            if (pc > qs0) bulk_g2s(pb + o * (kSaPosCap + 4), a.ops.op[o].pos + qs0, (uint32_t)(pc - qs0) * 8, &sh.full);
          }
        }
      }
    }
    __syncthreads();
    const int64_t p = h.p;
    if (p < 0) break;
    mbar_wait(&sh.full, it & 1);
    NACHO_PHASE(0, tlast);
    const int64_t brow = h.b0.row;
    const int64_t r_hi = h.b1.row < M - 1 ? h.b1.row : M - 1;

    // ---- column range and key width
    int32_t cmn = INT32_MAX, cmx = -1;
    for (int o = 0; o < k; ++o) {
      const int32_t* c = sh.crd + h.crd_off[o];
      const int no = h.off[o + 1] - h.off[o];
      for (int j = tid; j < no; j += kSaThreads) { const int32_t v = c[j]; cmn = min(cmn, v); cmx = max(cmx, v); }
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      cmn = min(cmn, __shfl_xor_sync(kFull, cmn, d));
      cmx = max(cmx, __shfl_xor_sync(kFull, cmx, d));
    }
    if (lane == 0) { sh.redmin[w] = cmn; sh.redmax[w] = cmx; }
    __syncthreads();
    int32_t cmin = INT32_MAX, cmaxv = -1;
#pragma unroll
    for (int ww = 0; ww < kSaThreads / 32; ++ww) { cmin = min(cmin, sh.redmin[ww]); cmaxv = max(cmaxv, sh.redmax[ww]); }
    if (cmaxv < cmin) { cmin = 0; cmaxv = 0; }
    const int rbits = 64 - __clzll((unsigned long long)(r_hi - brow + 1));
    const int cbits = 32 - __clz((unsigned)(cmaxv - cmin) | 1u);
    const bool k32 = rbits + cbits <= 31 && r_hi - brow < (int64_t(1) << 28);
    NACHO_PHASE(1, tlast);

    if (k32) {
      // ======== whole partition, 32-bit keys
      int cs[NACHO_MAX_K], ce[NACHO_MAX_K], koff[NACHO_MAX_K];
      uint32_t* K0 = reinterpret_cast<uint32_t*>(kbuf);
      uint32_t* B1 = K0 + kSaK0Cap;
      uint32_t* B2 = B1 + kSaBufCap;
      for (int o = 0, acc = 0; o < k; ++o) {
        cs[o] = 0;
        ce[o] = h.off[o + 1] - h.off[o];
        koff[o] = acc;
        acc += ce[o] + 1;
      }
      sa_keys<T, uint32_t>(a, sh, pb, k, cs, ce, koff, K0, B2, cbits, cmin, brow, r_hi);
      NACHO_PHASE(2, tlast);
      const uint32_t* Uk;
      const T* Uv;
      bool upad;
      const int nu = sa_union<T, VALS, uint32_t>(sh, k, cs, ce, koff, K0, B1, B2, V1, V2, &Uk, &Uv, &upad);
      NACHO_PHASE(3, tlast);
      if (MODE == kCount) {
        if (tid == 0) a.part_cnt[p] = nu;
      } else {
        const int64_t off = sa_offset<T, MODE>(a, sh, p, nu);
        NACHO_PHASE(4, tlast);
        if (p == 0 && tid == 0) a.z_pos[0] = 0;
        sa_write_any<T, uint32_t>(a, Uk, Uv, upad, nu, off, cbits, cmin, brow, (h.b1.row < M ? h.b1.row : M) - 1, brow);
      }
    } else {
      sa_partition64<T, MODE>(a, sh, pb, kbuf, V1, V2, p);
    }
    __syncthreads();
    NACHO_PHASE(5, tlast);
  }
}

}  // namespace nacho
