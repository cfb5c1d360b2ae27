// spadd4.cuh -- k-way union SpAdd Z = A_0 + ... + A_{k-1} over equal-work partitions (SURVEY 8(a)
// rows a9-a11): one CTA per partition of <= kS4Tile entries (summed over the operands).
//
// Every output coordinate lies wholly inside one partition (the coordinate-space cut of Alg. 1,
// P:2635-2639), so a CTA computes its partition's union without looking at its neighbours:
//   1. all threads load the k operand ranges [b_p.pos[o], b_{p+1}.pos[o]) with coalesced loads
//      (entries concatenated in operand order; no single-thread staging, no serial setup);
//   2. row of every entry: the rows starting inside a range mark their first entry, every range's
//      first entry carries row b_p.row, and a "last mark wins" scan spreads the marks; the key is
//      (local row << cb) | (column - cmin), 32-bit when the partition's row span and column range
//      fit 31 bits, else 64-bit (then the merge stages carry entry indices only, keys are re-read);
//   3. k-1 stable merge-path stages (ties keep the lower operand first, so equal keys stay in
//      operand order); the last stage is fused with the fold: each run of equal keys is folded left
//      to right from its first value (R9) by the thread holding its first entry, and the runs are
//      compacted with one block scan;
//   4. the partition's output offset: part_off[p] (two-pass, Fig. 7a) or a decoupled
//      look-back over the partitions (single pass; partition ids are tickets taken in launch order,
//      so a partition's predecessors have always started);
//   5. Z.crd / Z.val at that offset and Z.pos[r+1] for the rows the partition completes (R7: rows
//      [b_p.row, b_{p+1}.row)).
#pragma once
#include "common.cuh"
#include "tma.cuh"

namespace nacho {

// kS4Stage: single read of the operands without a look-back -- the union goes to a staging buffer at
// the partition's provisional offset sum_o b_p.pos[o] (>= its final one), Z.pos gets partition-local
// counts, cnt[p] = union size (and per-block sums); s4_place_kernel then places it.
enum S4Mode { kS4Count = 0, kS4Fill = 1, kS4Fused = 2, kS4Stage = 3 };

// Phase timers (debug build -DNACHO_PROF): thread 0 of every 16th partition adds its clock64 deltas.
#ifdef NACHO_PROF
__device__ unsigned long long g_phase[16];
#define S4PH(id)                                                           \
  do {                                                                     \
    if (threadIdx.x == 0 && (p & 15) == 0) {                               \
      const unsigned long long _t = clock64();                             \
      atomicAdd(&g_phase[id], _t - s4t);                                   \
      s4t = _t;                                                            \
    }                                                                      \
  } while (0)
#define S4PH_INIT unsigned long long s4t = clock64()
#else
#define S4PH(id) do { } while (0)
#define S4PH_INIT unsigned long long s4t = 0
#endif

#ifndef NACHO_S4_THREADS   // tuning override
#define NACHO_S4_THREADS 256
#endif
constexpr int kS4Threads = NACHO_S4_THREADS;
#ifndef NACHO_S4_VT   // tuning override
#define NACHO_S4_VT 8
#endif
#ifndef NACHO_S4_MINB
#define NACHO_S4_MINB 4
#endif
constexpr int kS4Vt = NACHO_S4_VT;                // merged entries per thread and stage
constexpr int kS4Tile = kS4Threads * kS4Vt;       // entries per partition
constexpr int kS4Buf = kS4Tile + kS4Tile / 16 + 8;   // padded stage-buffer capacity (elements)
constexpr int kS4BlkShift = 8;                    // kS4Stage: partitions per block sum = 256
static_assert(kS4Threads >= (1 << kS4BlkShift), "s4_place_kernel sums a block's predecessors with one load per thread");
constexpr int kS4DenseWords = 2048;               // widest column range of the bitmap path (x 32 columns)
constexpr int kS4PosRound = 8;                    // row pointers loaded per thread and round

template <typename T>
struct Spadd4Args {
  OpsArg ops;
  PartsArg parts;
  int64_t* part_cnt;              // kS4Count: [P]
  int64_t* part_off;              // kS4Fill: read [P+1]; kS4Fused: written [P+1] (may be null)
  unsigned long long* lb_state;   // kS4Fused: [P], zeroed before launch
  unsigned long long* ticket;     // kS4Fused: zeroed before launch
  int64_t* z_pos;
  int32_t* z_crd;
  T* z_val;
  unsigned long long* blk_cnt;    // kS4Stage: union sizes summed per block of 2^kS4BlkShift chunks
                                  // (placement: their exclusive prefix)
  int32_t chunks;                 // kS4Stage: CTAs (chunks) per partition; 1 unless partitions exceed a tile
  int64_t* ch_prov;               // kS4Stage: per chunk, provisional offset sum_o b.pos[o]
  int64_t* ch_row;                // kS4Stage: per chunk, [2*c] first row, [2*c+1] end row
};

// Padded slot of element i of a thread-blocked stage buffer (conflict-free blocked accesses).
template <typename KT>
__device__ __forceinline__ int s4pd(int i) { return sizeof(KT) == 4 ? i + (i >> 5) : i + (i >> 4); }

// Shared memory.  SMALL (fill / stage modes with k <= 3): one stage buffer and no union buffers, so
// five CTAs fit an SM; the 64-bit operand keys then span zk + uv (uv must follow zk).  Otherwise two
// stage key buffers (the 64-bit keys alias them) and three source buffers.
template <typename T, bool SMALL = false>
struct S4Shared {
  int64_t b0pos[NACHO_MAX_K];
  int32_t off[NACHO_MAX_K + 1];           // concatenation offsets; off[o] = INT32_MAX for o > k
  const int32_t* crdp[NACHO_MAX_K];       // crd of entry j of operand o = crdp[o][j] (j concatenated)
  const void* valp[NACHO_MAX_K];
  const int64_t* posp[NACHO_MAX_K];       // pos_o + row0 + 1
  int64_t p;
  int64_t bcast;
  int64_t cpos[2][NACHO_MAX_K];           // chunked staged mode: the chunk's start / end positions
  int64_t crow[2];
  int32_t ired[kS4Threads / 32];
  int32_t fred_f[kS4Threads / 32], fred_v[kS4Threads / 32];
  int32_t cmn[kS4Threads / 32], cmx[kS4Threads / 32];
  alignas(16) T val[kS4Tile];                     // operand values (concatenated)
  alignas(16) int32_t col[kS4Buf];                // columns (padded slots); 32-bit path: the keys in place
  alignas(16) uint32_t zk[(SMALL ? 1 : 2) * kS4Buf];   // 32-bit path: stage keys | 64-bit: operand keys
  alignas(16) T uv[kS4Buf];                       // union values; before that: the row marks
  alignas(16) uint16_t zs[(SMALL ? 1 : 3) * kS4Buf];   // stage sources (+ union sources)
  static constexpr int kPosCap = SMALL ? kS4Threads * kS4PosRound : 2 * kS4Threads * kS4PosRound;
};
static_assert(sizeof(uint32_t) * kS4Buf % 16 == 0, "uv must start right after zk");

// The SMALL layout serves the emitting modes with at most three operands.
__host__ __device__ constexpr bool s4_small(int mode, int km) { return (mode == kS4Fill || mode == kS4Stage) && km <= 3; }

// "Last mark wins" combine for the row scan: (f, v) . (f2, v2) = (f | f2, f2 ? v2 : v).
__device__ __forceinline__ void s4_mark_op(int& f, int& v, int f2, int v2) {
  v = f2 ? v2 : v;
  f = f | f2;
}

// Merge input Y: operand keys, stored at padded slots of the concatenation (base = operand offset).
template <typename KT>
struct S4Y {
  const KT* K;
  int base;
  __device__ __forceinline__ KT operator[](int j) const { return K[s4pd<KT>(base + j)]; }
};

// Merge input X: operand 0's keys (KIND 0, unpadded, source = index), a keyed stage buffer
// (KIND 1: keys and sources at padded slots) or an index-only stage buffer (KIND 2: key = K[source]).
template <typename KT, int KIND>
struct S4X {
  const KT* K;
  const KT* zk;
  const uint16_t* zs;
  __device__ __forceinline__ KT key(int i) const {
    if constexpr (KIND == 0) return K[s4pd<KT>(i)];
    else if constexpr (KIND == 1) return zk[s4pd<KT>(i)];
    else return K[s4pd<KT>(zs[s4pd<KT>(i)])];
  }
  __device__ __forceinline__ int src(int i) const {
    if constexpr (KIND == 0) return i;
    else return zs[s4pd<KT>(i)];
  }
};

// Merge-path split of diagonal d of merge(X, Y) (ties: X first): #X entries among the first d.
template <typename KT, class XS>
__device__ __forceinline__ int s4_split(const XS& X, int nx, const S4Y<KT>& Y, int ny, int d) {
  int lo = max(0, d - ny), hi = min(d, nx);
  while (lo < hi) {
    const int m = (lo + hi) >> 1;
    if (X.key(m) <= Y[d - 1 - m]) lo = m + 1; else hi = m;
  }
  return lo;
}

// One plain merge stage Z = merge(X, Y) keeping duplicates (ties: X first).  Y = an operand's keys,
// sources ybase + j.  Z gets sources (and, if ZK, keys) at padded slots.
template <typename KT, class XS>
__device__ __forceinline__ void s4_merge(const XS& X, int nx, const S4Y<KT>& Y, int ybase, int ny, KT* ZK, uint16_t* ZS) {
  const int total = nx + ny;
  const int d0 = min(total, (int)threadIdx.x * kS4Vt), d1 = min(total, d0 + kS4Vt);
  if (d0 >= d1) return;
  int i = s4_split<KT>(X, nx, Y, ny, d0), j = d0 - i;
  constexpr KT INF = ~KT(0);
  KT xk = i < nx ? X.key(i) : INF, yk = j < ny ? Y[j] : INF;
#pragma unroll
  for (int s = 0; s < kS4Vt; ++s) {
    if (d0 + s < d1) {
      const bool tx = xk <= yk && i < nx;
      const int zi = s4pd<KT>(d0 + s);
      if (ZK) ZK[zi] = tx ? xk : yk;
      ZS[zi] = (uint16_t)(tx ? X.src(i) : ybase + j);
      if (tx) { ++i; xk = i < nx ? X.key(i) : INF; }
      else { ++j; yk = j < ny ? Y[j] : INF; }
    }
  }
}

// The last merge stage fused with the fold and the compaction.  Runs of equal keys (<= k entries,
// one per operand, in operand order) belong to the thread holding their first entry, which reads
// past its range while the run continues.  Writes the source of every run's first entry to US and
// the folded value to UV (padded slots); returns the union size.
template <typename T, typename KT, bool VALS, class XS>
__device__ __forceinline__ int s4_merge_fold(const XS& X, int nx, const S4Y<KT>& Y, int ybase, int ny, const T* val,
                                             uint16_t* US, T* UV, int32_t* ired) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  constexpr KT INF = ~KT(0);
  const int total = nx + ny;
  const int d0 = min(total, tid * kS4Vt), d1 = min(total, d0 + kS4Vt);
  int os[kS4Vt];
  T ov[kS4Vt];
  unsigned em = 0;
  if (d0 < d1) {
    int i = s4_split<KT>(X, nx, Y, ny, d0), j = d0 - i;
    KT xk = i < nx ? X.key(i) : INF, yk = j < ny ? Y[j] : INF;
    KT prev = INF;   // key of merged entry d0 - 1 (INF: none; never a key)
    if (d0 > 0) {
      const KT xp = i > 0 ? X.key(i - 1) : KT(0), yp = j > 0 ? Y[j - 1] : KT(0);
      prev = xp > yp ? xp : yp;
    }
    bool mine = false;
    T acc = T(0);
    int first = 0;
#pragma unroll
    for (int s = 0; s < kS4Vt; ++s) {
      if (d0 + s < d1) {
        const bool tx = xk <= yk && i < nx;
        const KT key = tx ? xk : yk;
        const int src = tx ? X.src(i) : ybase + j;
        if (tx) { ++i; xk = i < nx ? X.key(i) : INF; }
        else { ++j; yk = j < ny ? Y[j] : INF; }
        const bool fresh = key != prev;
        mine = mine || fresh;
        if (VALS) { const T v = val[src]; acc = fresh ? v : acc + v; }
        first = fresh ? src : first;
        prev = key;
        os[s] = first;
        ov[s] = acc;
        const KT nxt = (xk <= yk && i < nx) ? xk : yk;
        if (mine && nxt != key) em |= 1u << s;
      }
    }
    if (d1 - d0 == kS4Vt && mine) {   // my last run continues past d1: finish it
      KT nxt = (xk <= yk && i < nx) ? xk : yk;
      if (nxt == prev) {
        while (nxt == prev) {
          const bool tx = xk <= yk && i < nx;
          if (VALS) acc = acc + val[tx ? X.src(i) : ybase + j];
          if (tx) { ++i; xk = i < nx ? X.key(i) : INF; }
          else { ++j; yk = j < ny ? Y[j] : INF; }
          nxt = (xk <= yk && i < nx) ? xk : yk;
        }
        ov[kS4Vt - 1] = acc;
        em |= 1u << (kS4Vt - 1);
      }
    }
  }
  // compaction: exclusive block sum of the emitted counts
  const int cnt = __popc(em);
  int inc = cnt;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int u = __shfl_up_sync(kFull, inc, d);
    if (lane >= d) inc += u;
  }
  if (lane == 31) ired[w] = inc;
  __syncthreads();
  int pre = 0, tot = 0;
#pragma unroll
  for (int ww = 0; ww < kS4Threads / 32; ++ww) {
    const int v = ired[ww];
    pre += ww < w ? v : 0;
    tot += v;
  }
  int idx = pre + inc - cnt;
#pragma unroll
  for (int s = 0; s < kS4Vt; ++s) {
    if ((em >> s) & 1u) {
      US[s4pd<KT>(idx)] = (uint16_t)os[s];
      if (VALS) UV[s4pd<KT>(idx)] = ov[s];
      ++idx;
    }
  }
  return tot;
}

// Where a directly emitting final stage writes (kS4Fill / kS4Stage: the offset is known up front).
template <typename T>
struct S4Out {
  int32_t* z_crd;
  T* z_val;
  int64_t* z_pos;
  int64_t off;       // Z index of the partition's first union entry
  int64_t pos_off;   // added to the Z.pos values
  int64_t row0, L;   // owned rows: row0 + [0, L)
  int cb;
  int32_t cmin;
};

// The last merge stage fused with the fold and the output: like s4_merge_fold, but every run is
// written straight from registers at off + its union index (one block scan), together with Z.pos for
// the rows it ends: run key -> row r0, the next merged key (the next union entry) -> row r1, rows
// [r0, r1) end after this entry.  Rows before the first union entry are written by its emitter.
template <typename T, typename KT, class XS>
__device__ __forceinline__ int s4_merge_fold_emit(const XS& X, int nx, const S4Y<KT>& Y, int ybase, int ny, const T* val,
                                                  int32_t* ired, const S4Out<T>& out) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  constexpr KT INF = ~KT(0);
  const int total = nx + ny;
  const int d0 = min(total, tid * kS4Vt), d1 = min(total, d0 + kS4Vt);
  KT ok[kS4Vt], nk[kS4Vt];
  T ov[kS4Vt];
  unsigned em = 0;
  if (d0 < d1) {
    int i = s4_split<KT>(X, nx, Y, ny, d0), j = d0 - i;
    KT xk = i < nx ? X.key(i) : INF, yk = j < ny ? Y[j] : INF;
    KT prev = INF;
    if (d0 > 0) {
      const KT xp = i > 0 ? X.key(i - 1) : KT(0), yp = j > 0 ? Y[j - 1] : KT(0);
      prev = xp > yp ? xp : yp;
    }
    bool mine = false;
    T acc = T(0);
#pragma unroll
    for (int s = 0; s < kS4Vt; ++s) {
      if (d0 + s < d1) {
        const bool tx = xk <= yk && i < nx;
        const KT key = tx ? xk : yk;
        const int src = tx ? X.src(i) : ybase + j;
        if (tx) { ++i; xk = i < nx ? X.key(i) : INF; }
        else { ++j; yk = j < ny ? Y[j] : INF; }
        const bool fresh = key != prev;
        mine = mine || fresh;
        const T v = val[src];
        acc = fresh ? v : acc + v;
        prev = key;
        const KT nxt = (xk <= yk && i < nx) ? xk : yk;
        ok[s] = key;
        ov[s] = acc;
        nk[s] = nxt;
        if (mine && nxt != key) em |= 1u << s;
      }
    }
    if (d1 - d0 == kS4Vt && mine) {   // my last run continues past d1: finish it
      KT nxt = (xk <= yk && i < nx) ? xk : yk;
      if (nxt == prev) {
        while (nxt == prev) {
          const bool tx = xk <= yk && i < nx;
          acc = acc + val[tx ? X.src(i) : ybase + j];
          if (tx) { ++i; xk = i < nx ? X.key(i) : INF; }
          else { ++j; yk = j < ny ? Y[j] : INF; }
          nxt = (xk <= yk && i < nx) ? xk : yk;
        }
        ov[kS4Vt - 1] = acc;
        nk[kS4Vt - 1] = nxt;
        em |= 1u << (kS4Vt - 1);
      }
    }
  }
  const int cnt = __popc(em);
  int inc = cnt;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int u = __shfl_up_sync(kFull, inc, d);
    if (lane >= d) inc += u;
  }
  if (lane == 31) ired[w] = inc;
  __syncthreads();
  int pre = 0, tot = 0;
#pragma unroll
  for (int ww = 0; ww < kS4Threads / 32; ++ww) {
    const int v = ired[ww];
    pre += ww < w ? v : 0;
    tot += v;
  }
  int idx = pre + inc - cnt;
  const KT cmask = (KT)(((KT)1 << out.cb) - 1);
  bool first = idx == 0;
#pragma unroll
  for (int s = 0; s < kS4Vt; ++s) {
    if ((em >> s) & 1u) {
      out.z_crd[out.off + idx] = (int32_t)(ok[s] & cmask) + out.cmin;
      out.z_val[out.off + idx] = ov[s];
      // local rows fit 32 bits (key bits); L may not (trailing rows of the last partition)
      const int r0 = (int)(ok[s] >> out.cb);
      const int64_t r1 = nk[s] == INF ? out.L : min((int64_t)(nk[s] >> out.cb), out.L);
      if (first) {   // rows before the first union entry end empty
        const int64_t lead = r0 < out.L ? r0 : out.L;
        for (int64_t r = 0; r < lead; ++r) out.z_pos[out.row0 + r + 1] = out.pos_off;
        first = false;
      }
      if (r0 < r1) {
        int64_t* zp = out.z_pos + out.row0 + 1;
        const int64_t v = out.pos_off + idx + 1;
        zp[r0] = v;
        for (int64_t r = r0 + 1; r < r1; ++r) zp[r] = v;   // empty rows after it
      }
      ++idx;
    }
  }
  if (tot == 0)
    for (int64_t r = tid; r < out.L; r += kS4Threads) out.z_pos[out.row0 + r + 1] = out.pos_off;
  return tot;
}

// Decoupled look-back (warp 0): exclusive prefix of the union sizes of partitions < p.
__device__ __forceinline__ int64_t s4_lookback(unsigned long long* st, int64_t p, int64_t nu) {
  constexpr unsigned long long INCL = 1ull << 63, AGG = 1ull << 62, VAL = (1ull << 62) - 1;
  const int lane = threadIdx.x & 31;
  if (p == 0) {
    if (lane == 0) st_release(st, INCL | (unsigned long long)nu);
    return 0;
  }
  if (lane == 0) st_release(st + p, AGG | (unsigned long long)nu);
  unsigned long long excl = 0;
  int64_t base = p - 1;
  for (;;) {
    const int64_t q = base - lane;
    unsigned long long v = q >= 0 ? ld_acquire(st + q) : INCL;
    int first;
    unsigned ns = 64;
    for (;;) {
      const unsigned ready = __ballot_sync(kFull, (v & (INCL | AGG)) != 0);
      const unsigned incl = __ballot_sync(kFull, (v & INCL) != 0);
      first = incl ? __ffs(incl) - 1 : 32;   // nearest inclusive predecessor
      const unsigned need = first >= 31 ? kFull : ((2u << first) - 1);
      if ((ready & need) == need) break;
      if (!(v & (INCL | AGG))) { __nanosleep(ns); ns = ns < 512 ? 2 * ns : ns; v = ld_acquire(st + q); }
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

// Union of the keyed operands (K: concatenated operand keys).  KIND of the stage buffers: 1 (keyed,
// 32-bit) or 2 (index-only, 64-bit).  Returns nu; US / UV hold the union.
template <typename T, typename KT, bool VALS, int KIND, class SH>
__device__ __forceinline__ int s4_union(SH& sh, int k, const KT* K, KT* Z1, KT* Z2, uint16_t* S1,
                                        uint16_t* S2, uint16_t* US, T* UV) {
  const int* off = sh.off;
  if (k == 1) {
    const S4X<KT, 0> X{K, nullptr, nullptr};
    return s4_merge_fold<T, KT, VALS>(X, off[1], S4Y<KT>{K, 0}, 0, 0, sh.val, US, UV, sh.ired);
  }
  if (k == 2) {
    const S4X<KT, 0> X{K, nullptr, nullptr};
    return s4_merge_fold<T, KT, VALS>(X, off[1], S4Y<KT>{K, off[1]}, off[1], off[2] - off[1], sh.val, US, UV, sh.ired);
  }
  {
    const S4X<KT, 0> X{K, nullptr, nullptr};
    s4_merge<KT>(X, off[1], S4Y<KT>{K, off[1]}, off[1], off[2] - off[1], KIND == 1 ? Z1 : nullptr, S1);
  }
  __syncthreads();
  KT* xk = Z1;
  uint16_t* xs = S1;
  KT* zk = Z2;
  uint16_t* zs = S2;
  for (int o = 2; o < k - 1; ++o) {
    const S4X<KT, KIND> X{K, xk, xs};
    s4_merge<KT>(X, off[o], S4Y<KT>{K, off[o]}, off[o], off[o + 1] - off[o], KIND == 1 ? zk : nullptr, zs);
    __syncthreads();
    KT* tk = xk; xk = zk; zk = tk;
    uint16_t* ts = xs; xs = zs; zs = ts;
  }
  const S4X<KT, KIND> X{K, xk, xs};
  return s4_merge_fold<T, KT, VALS>(X, off[k - 1], S4Y<KT>{K, off[k - 1]}, off[k - 1], off[k] - off[k - 1], sh.val, US, UV,
                                    sh.ired);
}

// s4_union with a directly emitting final stage.
template <typename T, typename KT, int KIND, class SH>
__device__ __forceinline__ int s4_union_emit(SH& sh, int k, const KT* K, KT* Z1, KT* Z2, uint16_t* S1,
                                             uint16_t* S2, const S4Out<T>& out) {
  const int* off = sh.off;
  if (k <= 2) {
    const S4X<KT, 0> X{K, nullptr, nullptr};
    const int ny = k == 2 ? off[2] - off[1] : 0;
    return s4_merge_fold_emit<T, KT>(X, off[1], S4Y<KT>{K, off[1]}, off[1], ny, sh.val, sh.ired, out);
  }
  {
    const S4X<KT, 0> X{K, nullptr, nullptr};
    s4_merge<KT>(X, off[1], S4Y<KT>{K, off[1]}, off[1], off[2] - off[1], KIND == 1 ? Z1 : nullptr, S1);
  }
  __syncthreads();
  KT* xk = Z1;
  uint16_t* xs = S1;
  KT* zk = Z2;
  uint16_t* zs = S2;
  for (int o = 2; o < k - 1; ++o) {
    const S4X<KT, KIND> X{K, xk, xs};
    s4_merge<KT>(X, off[o], S4Y<KT>{K, off[o]}, off[o], off[o + 1] - off[o], KIND == 1 ? zk : nullptr, zs);
    __syncthreads();
    KT* tk = xk; xk = zk; zk = tk;
    uint16_t* ts = xs; xs = zs; zs = ts;
  }
  const S4X<KT, KIND> X{K, xk, xs};
  return s4_merge_fold_emit<T, KT>(X, off[k - 1], S4Y<KT>{K, off[k - 1]}, off[k - 1], off[k] - off[k - 1], sh.val, sh.ired,
                                   out);
}

// Single-row partitions with a narrow column range (the bulk of a power-law matrix's heavy rows):
// the union is a bitmap.  Each operand's columns set bits of its bitmap, the union bitmap's prefix
// popcounts give every column its union index, values fold into that slot operand by operand (left
// fold in operand order, R9), and the set bits of the union bitmap are the output columns.  No keys,
// no merge-path stages: a handful of instructions per entry.
template <typename T, int MODE, int KM, class SH>
__device__ __forceinline__ void s4_dense(const Spadd4Args<T>& a, SH& sh, int64_t p, int n, int64_t row0,
                                         int64_t row1, int32_t cmin, int nw) {
  constexpr bool VALS = MODE != kS4Count;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int k = KM < NACHO_MAX_K ? KM : a.ops.k;
  uint32_t* bm = sh.zk;                 // [k][nw] operand bitmaps
  uint32_t* U = bm + k * nw;            // [nw] union bitmap
  int32_t* pre = reinterpret_cast<int32_t*>(U + nw);   // [nw] union entries before word w
  T* ov = sh.uv;                        // [nu] folded union values
  for (int i = tid; i < (k + 1) * nw; i += kS4Threads) bm[i] = 0u;
  __syncthreads();
  int ob[KM > 1 ? KM - 1 : 1];
#pragma unroll
  for (int o = 0; o < KM - 1; ++o) ob[o] = sh.off[o + 1];
  for (int j = tid; j < n; j += kS4Threads) {
    int o = 0;
#pragma unroll
    for (int oo = 0; oo < KM - 1; ++oo) o += j >= ob[oo] ? 1 : 0;
    const int c = sh.col[s4pd<uint32_t>(j)] - cmin;
    atomicOr(&bm[o * nw + (c >> 5)], 1u << (c & 31));
  }
  __syncthreads();
  // union bitmap and its exclusive prefix popcount (block scan over the words)
  constexpr int WPT = 4;                // words per thread and round
  int carry = 0;
  for (int w0 = 0; w0 < nw; w0 += kS4Threads * WPT) {
    uint32_t u[WPT];
    int c = 0;
#pragma unroll
    for (int q = 0; q < WPT; ++q) {
      const int ww = w0 + tid * WPT + q;
      u[q] = 0u;
      if (ww < nw) {
#pragma unroll
        for (int o = 0; o < KM; ++o) if (o < k) u[q] |= bm[o * nw + ww];
        U[ww] = u[q];
      }
      c += __popc(u[q]);
    }
    int inc = c;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int v = __shfl_up_sync(kFull, inc, d);
      if (lane >= d) inc += v;
    }
    if (lane == 31) sh.ired[w] = inc;
    __syncthreads();
    int before = carry, tot = 0;
#pragma unroll
    for (int ww = 0; ww < kS4Threads / 32; ++ww) {
      const int v = sh.ired[ww];
      before += ww < w ? v : 0;
      tot += v;
    }
    int x = before + inc - c;
#pragma unroll
    for (int q = 0; q < WPT; ++q) {
      const int ww = w0 + tid * WPT + q;
      if (ww < nw) pre[ww] = x;
      x += __popc(u[q]);
    }
    carry += tot;
    __syncthreads();
  }
  const int nu = carry;
  // values: operand by operand, each entry into its union slot (= if no lower operand has the column)
  if (VALS) {
    for (int o = 0; o < k; ++o) {
      for (int j = sh.off[o] + tid; j < sh.off[o + 1]; j += kS4Threads) {
        const int c = sh.col[s4pd<uint32_t>(j)] - cmin;
        const int ww = c >> 5;
        const uint32_t bit = 1u << (c & 31);
        const int r = pre[ww] + __popc(U[ww] & (bit - 1u));
        bool prior = false;
#pragma unroll
        for (int o2 = 0; o2 < KM; ++o2) if (o2 < o) prior = prior || (bm[o2 * nw + ww] & bit) != 0u;
        const T v = sh.val[j];
        ov[r] = prior ? ov[r] + v : v;
      }
      __syncthreads();
    }
  }
  if (MODE == kS4Count) {
    if (tid == 0) a.part_cnt[p] = nu;
    return;
  }
  int64_t off, pos_off;
  if (MODE == kS4Fill) {
    off = ldg(a.part_off + p);
    pos_off = off;
  } else if (MODE == kS4Stage) {
    off = 0;
#pragma unroll
    for (int o = 0; o < KM; ++o) if (o < k) off += sh.b0pos[o];
    pos_off = 0;
    if (tid == 0) {
      a.part_cnt[p] = nu;
      atomicAdd(a.blk_cnt + (p >> kS4BlkShift), (unsigned long long)nu);
      a.ch_prov[p] = off;
      a.ch_row[2 * p] = row0;
      a.ch_row[2 * p + 1] = row1;
    }
  } else {
    if (w == 0) {
      const int64_t ex = s4_lookback(a.lb_state, p, nu);
      if (lane == 0) {
        sh.bcast = ex;
        if (a.part_off) { a.part_off[p] = ex; if (p == a.parts.P - 1) a.part_off[a.parts.P] = ex + nu; }
      }
    }
    __syncthreads();
    off = sh.bcast;
    pos_off = off;
  }
  if (p == 0 && tid == 0) a.z_pos[0] = 0;
  // output: the set bits of the union bitmap, word by word
  for (int ww = tid; ww < nw; ww += kS4Threads) {
    uint32_t bits = U[ww];
    int idx = pre[ww];
    while (bits) {
      const int b = __ffs(bits) - 1;
      bits &= bits - 1u;
      a.z_crd[off + idx] = cmin + 32 * ww + b;
      a.z_val[off + idx] = ov[idx];
      ++idx;
    }
  }
  // the partition's one row completes here iff b_{p+1} lies in a later row (R7); trailing empty rows
  // of the last partition follow it
  for (int64_t r = tid; r < row1 - row0; r += kS4Threads) a.z_pos[row0 + r + 1] = pos_off + nu;
}

// Keys (32- or 64-bit), union, offset and writes of one partition.
template <typename T, typename KT, int MODE, int KM, class SH>
__device__ __forceinline__ void s4_body(const Spadd4Args<T>& a, SH& sh, int64_t p, int n, int64_t row0,
                                        int64_t row1, int cb, int32_t cmin, unsigned long long& s4t) {
  (void)s4t;
  constexpr bool VALS = MODE != kS4Count;
  constexpr int KIND = sizeof(KT) == 4 ? 1 : 2;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int k = KM < NACHO_MAX_K ? KM : a.ops.k;
  const int32_t* mark = reinterpret_cast<const int32_t*>(sh.uv);
  KT* K = sizeof(KT) == 4 ? reinterpret_cast<KT*>(sh.col) : reinterpret_cast<KT*>(sh.zk);

  // ---- row of every entry ("last mark wins" scan), then its key
  {
    const int j0 = tid * kS4Vt;
    int mv[kS4Vt], mk[kS4Vt];
    int f = 0, v = 0;
#pragma unroll
    for (int s = 0; s < kS4Vt; ++s) {
      const int j = j0 + s;
      mk[s] = j < n ? mark[s4pd<uint32_t>(j)] : -1;
      s4_mark_op(f, v, mk[s] >= 0, mk[s]);
      mv[s] = v;
    }
    int fi = f, vi = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int fu = __shfl_up_sync(kFull, fi, d), vu = __shfl_up_sync(kFull, vi, d);
      if (lane >= d) { int ff = fu, vv = vu; s4_mark_op(ff, vv, fi, vi); fi = ff; vi = vv; }
    }
    if (lane == 31) { sh.fred_f[w] = fi; sh.fred_v[w] = vi; }
    __syncthreads();
    int pf = 0, pv = 0;
    for (int ww = 0; ww < w; ++ww) s4_mark_op(pf, pv, sh.fred_f[ww], sh.fred_v[ww]);
    int ef = __shfl_up_sync(kFull, fi, 1), ev = __shfl_up_sync(kFull, vi, 1);
    if (lane == 0) { ef = 0; ev = 0; }
    s4_mark_op(pf, pv, ef, ev);   // the row flowing into my first entry
    bool seen = false;
#pragma unroll
    for (int s = 0; s < kS4Vt; ++s) {
      const int j = j0 + s;
      if (j < n) {
        seen = seen || mk[s] >= 0;
        const int lr = seen ? mv[s] : pv;
        K[s4pd<KT>(j)] = ((KT)(uint32_t)lr << cb) | (KT)(uint32_t)(sh.col[s4pd<uint32_t>(j)] - cmin);
      }
    }
  }
  __syncthreads();

  // ---- union
  KT* Z1 = reinterpret_cast<KT*>(sh.zk);
  KT* Z2 = Z1 + kS4Buf;
  uint16_t* S1 = sh.zs;
  uint16_t* S2 = S1 + kS4Buf;
  uint16_t* US = S2 + kS4Buf;
  S4PH(3);
  if (MODE == kS4Fill || MODE == kS4Stage) {   // offset known up front: emit from the fold directly
    S4Out<T> out;
    out.z_crd = a.z_crd;
    out.z_val = a.z_val;
    out.z_pos = a.z_pos;
    out.row0 = row0;
    out.L = row1 - row0;
    out.cb = cb;
    out.cmin = cmin;
    if (MODE == kS4Fill) {
      out.off = ldg(a.part_off + p);
      out.pos_off = out.off;
    } else {
      out.off = 0;
#pragma unroll
      for (int o = 0; o < KM; ++o) if (o < k) out.off += sh.b0pos[o];   // provisional: sum_o b_p.pos[o]
      out.pos_off = 0;
    }
    if (p == 0 && tid == 0) a.z_pos[0] = 0;
    const int nu = s4_union_emit<T, KT, KIND, SH>(sh, k, K, Z1, Z2, S1, S2, out);
    if (MODE == kS4Stage && tid == 0) {
      a.part_cnt[p] = nu;
      atomicAdd(a.blk_cnt + (p >> kS4BlkShift), (unsigned long long)nu);
      a.ch_prov[p] = out.off;
      a.ch_row[2 * p] = row0;
      a.ch_row[2 * p + 1] = row1;
    }
    S4PH(4);
    return;
  }
  const int nu = s4_union<T, KT, VALS, KIND, SH>(sh, k, K, Z1, Z2, S1, S2, US, sh.uv);
  S4PH(4);
  if (MODE == kS4Count) {
    if (tid == 0) a.part_cnt[p] = nu;
    return;
  }
  // ---- output offset (kS4Fused: decoupled look-back)
  int64_t off;
  int64_t pos_off = 0;
  {
    if (w == 0) {
      const int64_t ex = s4_lookback(a.lb_state, p, nu);
      if (lane == 0) {
        sh.bcast = ex;
        if (a.part_off) { a.part_off[p] = ex; if (p == a.parts.P - 1) a.part_off[a.parts.P] = ex + nu; }
      }
    }
    __syncthreads();
    off = sh.bcast;
    pos_off = off;
  }
  S4PH(5);
  // ---- Z.crd / Z.val, then Z.pos[r+1] for the owned rows [row0, row1) (local [0, L))
  const KT cmask = (KT)(((KT)1 << cb) - 1);
  for (int j = tid; j < nu; j += kS4Threads) {
    const int src = US[s4pd<KT>(j)];
    a.z_crd[off + j] = (int32_t)(K[s4pd<KT>(src)] & cmask) + cmin;
    a.z_val[off + j] = sh.uv[s4pd<KT>(j)];
  }
  const int64_t L = row1 - row0;
  if (p == 0 && tid == 0) a.z_pos[0] = 0;
  auto row_of = [&](int j) -> int64_t { return (int64_t)(K[s4pd<KT>(US[s4pd<KT>(j)])] >> cb); };
  {
    const int64_t lead = nu > 0 ? (row_of(0) < L ? row_of(0) : L) : L;   // rows before the first entry
    for (int64_t r = tid; r < lead; r += kS4Threads) a.z_pos[row0 + r + 1] = pos_off;
  }
  // entry j ends rows [row(j), row(j+1)) (clipped to the owned rows); row(j+1) from the next lane
  for (int jb = 0; jb < nu; jb += kS4Threads) {
    const int j = jb + tid;
    const int64_t r0 = j < nu ? row_of(j) : L;
    int64_t r1 = __shfl_down_sync(kFull, r0, 1);
    if (lane == 31) r1 = j + 1 < nu ? row_of(j + 1) : L;
    if (j + 1 >= nu) r1 = L;
    r1 = r1 < L ? r1 : L;
    for (int64_t r = r0; r < r1; ++r) a.z_pos[row0 + r + 1] = pos_off + j + 1;
  }
  __syncthreads();
  S4PH(6);
}

// KM: compile-time operand count (1..4), or NACHO_MAX_K for any k (read from a.ops.k).
// The 64-bit key path is rare (very wide partitions); kept out of line so it does not crowd the
// instruction cache of the hot 32-bit and bitmap paths.
template <typename T, int MODE, int KM, class SH>
__device__ __noinline__ void s4_body64(const Spadd4Args<T>& a, SH& sh, int64_t p, int n, int64_t row0, int64_t row1,
                                       int32_t cmin, unsigned long long& s4t) {
  s4_body<T, uint64_t, MODE, KM, SH>(a, sh, p, n, row0, row1, 32, cmin, s4t);
}

template <typename T, int MODE, int KM, bool CHK>   // CHK: staged mode, partitions larger than a tile
__global__ void __launch_bounds__(kS4Threads, s4_small(MODE, KM) ? 1280 / kS4Threads : NACHO_S4_MINB) spadd4_kernel(const __grid_constant__ Spadd4Args<T> a) {
  constexpr bool VALS = MODE != kS4Count;
  extern __shared__ __align__(16) unsigned char s4raw[];
  using SH = S4Shared<T, s4_small(MODE, KM)>;
  SH& sh = *reinterpret_cast<SH*>(s4raw);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int k = KM < NACHO_MAX_K ? KM : a.ops.k;
  int64_t p;
  S4PH_INIT;
  if (MODE == kS4Fused) {
    if (tid == 0) sh.p = (int64_t)atomicAdd(a.ticket, 1ull);
    __syncthreads();
    p = sh.p;
  } else {
    p = blockIdx.x;
  }
  // ---- staged mode, partitions larger than a tile: CTA p is chunk c of partition pp, the part of it
  //      between the queries C(b_pp) + c Tq and C(b_pp) + (c+1) Tq -- two more FindPartition (Alg. 1)
  //      searches, whose cuts coincide with the global partition's for those queries, so chunks tile
  //      the partition and every coordinate lies in one chunk (work <= Tq + k - 1 = kS4Tile)
  constexpr bool chunked = MODE == kS4Stage && CHK;
  if constexpr (chunked) {
    if (w < 2) {
      const int64_t pp = p / a.chunks, c = p - pp * a.chunks;
      int64_t C0 = 0, C1 = 0;
      for (int o = 0; o < k; ++o) { C0 += ldg(a.parts.pos + pp * k + o); C1 += ldg(a.parts.pos + (pp + 1) * k + o); }
      const int64_t Tq = kS4Tile - (k - 1);
      const int64_t Q = C0 + (c + w) * Tq;
      int64_t row, pos[KM];
      if ((w == 0 && c == 0) || Q >= C1) {   // the partition's own boundary
        const int64_t q = (w == 0 && c == 0) ? pp : pp + 1;
        row = ldg(a.parts.row + q);
#pragma unroll
        for (int o = 0; o < KM; ++o) pos[o] = o < k ? ldg(a.parts.pos + q * k + o) : 0;
      } else {
        const Boundary b = warp_find_boundary<KM>(a.ops, Q, ldg(a.parts.row_pos + pp), ldg(a.parts.row_pos + pp + 1));
        row = b.row;
#pragma unroll
        for (int o = 0; o < KM; ++o) pos[o] = b.pos[o];
      }
      if (lane == 0) sh.crow[w] = row;
#pragma unroll
      for (int o = 0; o < KM; ++o) if (lane == o && o < k) sh.cpos[w][o] = pos[o];
    }
    __syncthreads();
  }
  // ---- boundaries and operand ranges (warp 0: lane o < k holds operand o; sizes scanned by shuffles)
  const int64_t row0 = chunked ? sh.crow[0] : ldg(a.parts.row + p);
  const int64_t row1 = chunked ? sh.crow[1] : ldg(a.parts.row + p + 1);
  if (w == 0) {
    int64_t b0 = 0;
    int sz = 0;
    if (lane < k) {
      b0 = chunked ? sh.cpos[0][lane] : ldg(a.parts.pos + p * k + lane);
      sz = (int)((chunked ? sh.cpos[1][lane] : ldg(a.parts.pos + (p + 1) * k + lane)) - b0);
    }
    int inc = sz;
#pragma unroll
    for (int d = 1; d < NACHO_MAX_K; d <<= 1) {
      const int u = __shfl_up_sync(kFull, inc, d);
      if (lane >= d) inc += u;
    }
    if (lane < k) {
      const int ex = inc - sz;
      sh.b0pos[lane] = b0;
      sh.off[lane + 1] = inc;
      sh.crdp[lane] = a.ops.op[lane].crd + (b0 - ex);
      sh.valp[lane] = reinterpret_cast<const T*>(a.ops.op[lane].val) + (b0 - ex);
      sh.posp[lane] = a.ops.op[lane].pos + row0 + 1;
    } else if (lane < NACHO_MAX_K) {
      sh.off[lane + 1] = INT32_MAX;
    }
    if (lane == 0) sh.off[0] = 0;
  }
  const int64_t M = a.ops.nrows;
  const int64_t rlast = row1 < M ? row1 : M - 1;
  const int64_t span = rlast > row0 ? rlast - row0 : 0;   // rows (row0, row0 + span] may start inside
  __syncthreads();
  const int n = sh.off[k];
  S4PH(0);

  // ---- one round of loads: the k ranges (entry j of the concatenation -> operand o(j)) and, when
  //      they fit, the row pointers pos_o[row0 + 1 .. row0 + span + 1] as local offsets (smem)
  int32_t* mark = reinterpret_cast<int32_t*>(sh.uv);
  int32_t* spos = reinterpret_cast<int32_t*>(sh.zk);   // [k][span + 1], free until the merges
  const int np = (int)span + 1;
  const bool pre = span > 0 && (int64_t)k * np <= SH::kPosCap;
  int32_t cmn = INT32_MAX, cmx = -1;
  {
    int32_t c[kS4Vt];
    T v[kS4Vt];
    int ob[KM > 1 ? KM - 1 : 1];   // concatenation offsets 1..KM-1 (INT32_MAX past k): o(j) = #{ob <= j}
#pragma unroll
    for (int o = 0; o < KM - 1; ++o) ob[o] = sh.off[o + 1];
#pragma unroll
    for (int i = 0; i < kS4Vt; ++i) {
      const int j = tid + kS4Threads * i;
      if (j < n) {
        int o = 0;
#pragma unroll
        for (int oo = 0; oo < KM - 1; ++oo) o += j >= ob[oo] ? 1 : 0;
        c[i] = ldg(sh.crdp[o] + j);
        if (VALS) v[i] = ldg(reinterpret_cast<const T*>(sh.valp[o]) + j);
        mark[s4pd<uint32_t>(j)] = (j == sh.off[o]) ? 0 : -1;   // a range's first entry belongs to row0 unless marked
      }
    }
    if (pre) {
      // flattened (operand, pointer) index f = tid + 256 m -> (po, pi) = (f / np, f % np)
#pragma unroll
      for (int half = 0; half < SH::kPosCap / (kS4Threads * kS4PosRound); ++half) {
        int64_t pv[kS4PosRound];
#pragma unroll
        for (int m = 0; m < kS4PosRound; ++m) {
          const int f = tid + (half * kS4PosRound + m) * kS4Threads;
          int po = 0;
#pragma unroll
          for (int oo = 1; oo < KM; ++oo) po += (oo < k && f >= oo * np) ? 1 : 0;
          const int pi = f - po * np;
          pv[m] = f < k * np ? ldg(sh.posp[po] + pi) - sh.b0pos[po] : 0;
        }
#pragma unroll
        for (int m = 0; m < kS4PosRound; ++m) {
          const int f = tid + (half * kS4PosRound + m) * kS4Threads;
          if (f < k * np) spos[f] = (int32_t)(pv[m] < INT32_MAX ? pv[m] : INT32_MAX);
        }
      }
    }
#pragma unroll
    for (int i = 0; i < kS4Vt; ++i) {
      const int j = tid + kS4Threads * i;
      if (j < n) {
        sh.col[s4pd<uint32_t>(j)] = c[i];
        if (VALS) sh.val[j] = v[i];
        cmn = min(cmn, c[i]);
        cmx = max(cmx, c[i]);
      }
    }
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    cmn = min(cmn, __shfl_xor_sync(kFull, cmn, d));
    cmx = max(cmx, __shfl_xor_sync(kFull, cmx, d));
  }
  if (lane == 0) { sh.cmn[w] = cmn; sh.cmx[w] = cmx; }
  __syncthreads();
  S4PH(1);
  int32_t cmin = INT32_MAX, cmax = -1;
#pragma unroll
  for (int ww = 0; ww < kS4Threads / 32; ++ww) { cmin = min(cmin, sh.cmn[ww]); cmax = max(cmax, sh.cmx[ww]); }
  if (cmax < cmin) { cmin = 0; cmax = 0; }
  // ---- one row, narrow column range: bitmap union (s4_dense)
  {
    const int nw = (int)(((int64_t)cmax - cmin) / 32 + 1);
    if (span == 0 && (int64_t)nw * (k + 2) <= (int64_t)(sizeof(sh.zk) / 4) && nw <= kS4DenseWords) {
      s4_dense<T, MODE, KM, SH>(a, sh, p, n, row0, row1, cmin, nw);
      S4PH(5);   // phase-timer slot 5: bitmap partitions
#ifdef NACHO_PROF
      if (tid == 0 && (p & 15) == 0) atomicAdd(&g_phase[7], 1ull);
#endif
      return;
    }
  }
  // ---- rows (row0, row0 + span] starting inside operand o's range mark their first entry (non-empty)
  for (int o = 0; o < k; ++o) {
    const int base = sh.off[o], no = sh.off[o + 1] - base;
    if (pre) {
      const int32_t* sp = spos + o * np;
      for (int r = tid; r < (int)span; r += kS4Threads) {
        const int ps = sp[r], pe = sp[r + 1];
        if (ps < no && pe > ps) mark[s4pd<uint32_t>(base + ps)] = r + 1;
      }
    } else {
      const int64_t s = sh.b0pos[o];
      const int64_t* __restrict__ pos = a.ops.op[o].pos + row0;
#pragma unroll 2
      for (int64_t r = 1 + tid; r <= span; r += kS4Threads) {
        const int64_t ps = ldg(pos + r) - s, pe = ldg(pos + r + 1) - s;
        if (ps >= 0 && ps < no && pe > ps) mark[s4pd<uint32_t>(base + (int)ps)] = (int)r;
      }
    }
  }
  __syncthreads();
  S4PH(2);
  const int cb = 32 - __clz((unsigned)(cmax - cmin));                       // column bits (0 if one column)
  const int rb = span > 0 ? 64 - __clzll((unsigned long long)span) : 0;      // local row bits
  if (rb + cb <= 31) s4_body<T, uint32_t, MODE, KM, SH>(a, sh, p, n, row0, row1, cb, cmin, s4t);
  else s4_body64<T, MODE, KM, SH>(a, sh, p, n, row0, row1, cmin, s4t);
}

// Places the staged unions (kS4Stage): partition p's union moves from its provisional offset
// sum_o b_p.pos[o] to its final offset, and its owned Z.pos entries (rows [b_p.row, b_{p+1}.row)) get
// that offset added.  The offset -- the exclusive prefix of the union sizes -- is computed
// here from the per-256-partition block sums the stage kernel accumulated plus the sizes of p's
// predecessors inside its block (no separate scan kernel).  One CTA per partition.
template <typename T>
__global__ void __launch_bounds__(kS4Threads, 6) s4_place_kernel(const __grid_constant__ Spadd4Args<T> a,
                                                               const int32_t* __restrict__ t_crd,
                                                               const T* __restrict__ t_val) {
  __shared__ unsigned long long s_red[kS4Threads / 32];
  const int64_t p = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  // every load that does not depend on the offset is issued before the offset's reduction, so a
  // CTA waits on about two DRAM round trips instead of four
  const int64_t nu = ldg(a.part_cnt + p), prov = ldg(a.ch_prov + p);
  const int64_t r0 = ldg(a.ch_row + 2 * p), r1 = ldg(a.ch_row + 2 * p + 1);
  const int64_t b = p >> kS4BlkShift;
  unsigned long long v = tid == 0 ? a.blk_cnt[b] : 0ull;   // exclusive prefix of the block sums (run_spadd_staged)
  const int64_t q = (b << kS4BlkShift) + tid;
  if (q < p) v += (unsigned long long)ldg(a.part_cnt + q);
  constexpr int U = kS4Tile / kS4Threads;   // a chunk's union fits one round (nu <= kS4Tile)
  int32_t c[U];
  T vv[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t j = u * kS4Threads + tid;
    if (j < nu) { c[u] = __ldcs(t_crd + prov + j); vv[u] = __ldcs(t_val + prov + j); }
  }
  const int64_t rr = r0 + tid;
  const int64_t zp0 = rr < r1 ? a.z_pos[rr + 1] : 0;
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(kFull, v, d);
  if (lane == 0) s_red[w] = v;
  __syncthreads();
  unsigned long long tot = 0;
#pragma unroll
  for (int ww = 0; ww < kS4Threads / 32; ++ww) tot += s_red[ww];
  const int64_t off = (int64_t)tot;
  if (tid == 0) {   // p is a chunk; partition pp's offset is that of its first chunk
    const int64_t pp = p / a.chunks;
    if (p == pp * a.chunks) a.part_off[pp] = off;
    if (p == (int64_t)a.parts.P * a.chunks - 1) a.part_off[a.parts.P] = off + nu;
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t j = u * kS4Threads + tid;
    if (j < nu) { a.z_crd[off + j] = c[u]; a.z_val[off + j] = vv[u]; }
  }
  for (int64_t j = U * kS4Threads + tid; j < nu; j += kS4Threads) {   // not reached (nu <= kS4Tile)
    a.z_crd[off + j] = t_crd[prov + j];
    a.z_val[off + j] = t_val[prov + j];
  }
  if (rr < r1) a.z_pos[rr + 1] = zp0 + off;
  for (int64_t r = rr + kS4Threads; r < r1; r += kS4Threads) a.z_pos[r + 1] += off;
}

}  // namespace nacho
