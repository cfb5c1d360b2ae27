// spadd7.cuh -- single-read k-way SpAdd Z = A_0 + ... + A_{k-1} (CSR), persistent and software-
// pipelined: the assembly (union count), the prefix sum of the counts (P:1475,
// P:1897-1898) and the compute (fill) of Fig. 7a in ONE pass over the operands, with
// the partition p's global-memory latency (ticket, Parts record, operand ranges, row pointers) off
// the critical path of the warps that merge.
//
// One CTA = three roles over a ring of NS shared-memory stages (one partition, or one row-aligned
// sub-tile of a partition, per stage):
//   producer warp (8): takes partitions in ticket order (atomic counter: every predecessor of a
//     partition is already owned by a running CTA, so the look-back always progresses), reads its
//     Parts record (b_p, b_{p+1}: P:1795), and fills a free stage with 1-D bulk copies
//     (cp.async.bulk -> UBLKCP, completion on the stage's mbarrier) of every operand's crd / val
//     range [b_p.pos[o], b_{p+1}.pos[o]) and of the row pointers pos_o[row0 + 1 .. row1] of the
//     partition's rows (Listing 8's row loop bounds; operands sharing one pos array
//     are copied once); the next partition's ticket and record are fetched while it waits for the
//     following stage to free up;
//   compute warps (0-7): row marks -> partition-local rows -> 32-bit keys (local row << cb | col),
//     k - 1 stable merge-path stages (ties keep operand order), the last one folding equal keys
//     left to right in operand order from the first present value (R9) and counting the union
//     (the assembly count cnt_p), publication of cnt_p at once (decoupled look-back state
//     "aggregate"), the compacted union written back into the stage, and the union count before
//     each owned row (for Z.pos);
//   emission warp (9): resolves the exclusive prefix of the counts of partitions < p (the
//     look-back) -- the write offset off_p -- publishes the inclusive prefix, writes Z.crd / Z.val
//     at off_p and Z.pos of the rows p owns (R7: rows (b_p.row, b_{p+1}.row]), frees the stage.
// A partition spanning more rows than a stage's row-pointer pool holds runs as row-aligned
// sub-tiles: every sub-tile counted, then (after the look-back, done by compute warp 0) emitted
// at the known offset (two reads; rare: C2's partitions span at most 337 rows).
#pragma once
#include "spadd6.cuh"

namespace nacho {

constexpr int kS7Compute = kS5Threads;       // compute threads: warps 0 .. 7
constexpr int kS7Threads = kS7Compute + 64;  // + producer warp 8 + emission warp 9
constexpr int kS7Slots = kS5Slots;           // shared-memory slots per stage (entries + pads)
constexpr int kS7PosPool = 384;              // row-pointer pool per stage (int64 words)
constexpr int kS7LMax = kS7PosPool - 2;      // rows per (sub-)tile, one distinct pos array

// The coiteration the kernel runs over a partition (P:2051-2061 assembly, P:2145-2150 compute):
constexpr int kS7Union = 0;      // k-way SpAdd: union of coordinates, values summed (Listing 2)
constexpr int kS7Inter = 1;      // k-way Hadamard: intersection, values multiplied (Listings 1 and 8)
constexpr int kS7InterSum = 2;   // intersect-reduce inner product: sum of the intersection's products

template <typename V, int K>
struct S7Cfg {
#ifdef NACHO_S7_NS   // tuning / debugging override
  static constexpr int NS = NACHO_S7_NS;
#else
  static constexpr int NS = sizeof(V) == 4 && K <= 3 ? 3 : 2;     // stages
#endif
#ifdef NACHO_S7_MINB   // tuning override
  static constexpr int MINB = NACHO_S7_MINB;
#else
  static constexpr int MINB = sizeof(V) == 4 && K <= 3 ? 3 : 2;   // CTAs / SM (64 registers at 3)
#endif
};

template <typename V>
struct S7Args {
  OpsArg ops;
  PartsArg parts;
  int32_t cb;          // column bits of the keys
  int32_t lmax;        // rows per (sub-)tile: <= sp - 2, < 2^(32 - cb) - 1, <= kS7LMax
  int32_t use_bulk;    // crd / val / pos bases 16-byte aligned: bulk copies; else plain loads
  int32_t ndist;       // distinct pos arrays among the operands
  int32_t sp;          // pool words per distinct pos array (even)
  int32_t pd[NACHO_MAX_K];              // operand -> distinct pos array index
  const int64_t* dpos[NACHO_MAX_K];     // distinct pos arrays
  unsigned long long* state;            // [P] look-back states, [P] ticket, [P+1] error flag
  int64_t* part_off;                    // [P+1] or null
  int64_t* z_pos;
  int32_t* z_crd;
  V* z_val;
  double* partial;                      // kS7InterSum: [P] per-partition sums of products
};

template <typename V, int K>
struct alignas(16) S7Stage {
  uint32_t key[kS7Slots + 16];   // crd (bulk copy) -> keys in place -> union columns
  V val[kS7Slots];                // values (bulk copy) -> union values
  int64_t pos[kS7PosPool];        // row pointers (bulk copy) -> union count before each owned row
  // job record (producer -> compute -> emission)
  int64_t tile;                   // partition p; -1: stop
  int64_t a0;                     // first row: owned Z.pos rows a0 + 1 .. a0 + lrows
  int64_t ps;                     // first row held in the pos pool
  int64_t off;                    // mode 2: known write offset
  int64_t s[K], e[K];             // operand ranges
  int32_t soff[K], n[K], base[K + 1];
  int32_t lrows, mode, last, total;   // mode 1: one pass; 0: count a sub-tile; 2: emit a sub-tile
};

template <typename V, int K>
struct S7Smem {
  S7Stage<V, K> st[S7Cfg<V, K>::NS];
  alignas(16) uint32_t key1[kS7Slots + 16];   // row marks -> merge output -> union prefix U
  uint16_t src1[kS7Slots + 16];
  uint32_t key2[K >= 4 ? kS7Slots + 16 : 1];
  uint16_t src2[K >= 4 ? kS7Slots + 16 : 1];
  int32_t ML[kS7LMax + 1];        // merged position of each owned row's first entry
  int32_t wred[kS7Compute / 32];
  double wsum[kS7Compute / 32];
  int64_t run_off;
  int64_t excl[S7Cfg<V, K>::NS];     // emission -> compute: exclusive prefix of the stage's job
  int32_t excl_ok[S7Cfg<V, K>::NS];  // ... once resolved (reset by the emission after the job)
  uint64_t full[S7Cfg<V, K>::NS], done[S7Cfg<V, K>::NS], empty[S7Cfg<V, K>::NS];
};

#ifdef NACHO_S7_PROF   // dev builds: cycles per role and wait, accumulated at state[P + 2 + i]
#define S7_T0() const long long _t0 = clock64()
#define S7_ACC(i) atomicAdd(a.state + a.parts.P + 2 + (i), (unsigned long long)(clock64() - _t0))
#else
#define S7_T0()
#define S7_ACC(i)
#endif

__device__ __forceinline__ void s7_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// Waits of the producer / emission warps: back off between polls so that a warp running ahead of
// the compute warps does not take their issue slots.
#ifndef NACHO_S7_SLEEP_P   // back-off of the waits (ns): producer (free stage), emission (loaded / computed
#define NACHO_S7_SLEEP_P 256  // stage), compute warps (loaded stage)
#define NACHO_S7_SLEEP_EF 64
#define NACHO_S7_SLEEP_ED 256
#define NACHO_S7_SLEEP_C 128
#endif
__device__ __forceinline__ void s7_wait_sleep(uint64_t* bar, uint32_t parity, unsigned ns) {
  while (!mbar_try_wait(bar, parity)) __nanosleep(ns);
}

// ------------------------------------------------------------------ producer warp
template <typename V, int K, int OP>
__device__ __forceinline__ void s7_produce(const S7Args<V>& a, S7Smem<V, K>& sh) {
  constexpr int NS = S7Cfg<V, K>::NS;
  const int lane = threadIdx.x & 31;
  const int P = a.parts.P;
  const int lmax = a.lmax;
  int njob = 0;
  // the next partition's ticket and Parts record (issued before the stage wait)
  int64_t t, r0 = 0, r1 = 0, ps_o = 0, pe_o = 0;   // lane o < K: operand o's positions
  auto fetch = [&]() {
    unsigned long long tk = 0;
    if (lane == 0) tk = atomicAdd(a.state + P, 1ull);
    t = (int64_t)__shfl_sync(kFull, tk, 0);
    if (t < P) {
      r0 = a.parts.row[t];
      r1 = a.parts.row[t + 1];
      if (lane < K) {
        ps_o = a.parts.pos[t * K + lane];
        pe_o = a.parts.pos[(t + 1) * K + lane];
      }
      if (t == 0 && lane == 0 && a.z_pos) a.z_pos[0] = 0;
    }
  };
  // one job: (sub-)tile rows (a0, a0 + lrows], operand o's range [so, eo) held by lane o
  auto job = [&](int64_t tile, int mode, int last, int64_t a0, int lrows, int64_t so, int64_t eo) {
    const int s = njob % NS;
    const uint32_t ph = (uint32_t)(njob / NS) & 1u;
    ++njob;
    {
      S7_T0();
      s7_wait_sleep(&sh.empty[s], ph ^ 1u, NACHO_S7_SLEEP_P);
      if (lane == 0) S7_ACC(0);   // producer: waiting for a free stage
    }
    S7Stage<V, K>& g = sh.st[s];
    int64_t sv[K], ev[K];
    int soff[K], nn[K], base[K + 1];
    int b = 0;
#pragma unroll
    for (int o = 0; o < K; ++o) {
      sv[o] = __shfl_sync(kFull, so, o);
      ev[o] = __shfl_sync(kFull, eo, o);
      nn[o] = (int)(ev[o] - sv[o]);
      base[o] = b;
      soff[o] = b + (int)(sv[o] & 3);
      b = (soff[o] + nn[o] + 4) & ~3;   // >= 1 pad slot: the run's sentinel
    }
    base[K] = b;
    if (b > kS7Slots) {   // a record whose partitions exceed the stage (not from nacho_partition)
      if (lane == 0) atomicOr(a.state + P + 1, 1ull);
      b = 0;
#pragma unroll
      for (int o = 0; o < K; ++o) { ev[o] = sv[o]; nn[o] = 0; base[o] = b; soff[o] = b + (int)(sv[o] & 3); b = (soff[o] + 4) & ~3; }
      base[K] = b;
    }
    const int64_t ps = (a0 + 1) & ~int64_t(1);        // pool: rows [ps, ...) of every distinct pos array
    const int64_t pneed = a0 + lrows + 1;             // rows a0 + 1 .. a0 + lrows are read
    // bulk ranges: crd / val [s & ~3, ceil4(e)) -- the <= 3 slots past e land in the run's pad --
    // unless ceil4(e) passes the array end (then [.., e & ~3) and plain loads of the rest); pos
    // [ps, ceil2(pneed)) likewise
    const int64_t pe_up = (pneed + 1) & ~int64_t(1);
    const bool pos_up = pe_up <= a.ops.op[0].nouter + 1;
    const int64_t pe = lrows > 0 ? (pos_up ? pe_up : (pneed & ~int64_t(1))) : ps;
    if (lane == 0) {
      g.tile = tile; g.a0 = a0; g.ps = ps; g.lrows = lrows; g.mode = mode; g.last = last;
#pragma unroll
      for (int o = 0; o < K; ++o) { g.s[o] = sv[o]; g.e[o] = ev[o]; g.soff[o] = soff[o]; g.n[o] = nn[o]; }
#pragma unroll
      for (int o = 0; o <= K; ++o) g.base[o] = base[o];
    }
    int64_t hi[K];
    uint32_t bytes = 0;
#pragma unroll
    for (int o = 0; o < K; ++o) {
      const int64_t lo = sv[o] & ~int64_t(3);
      const int64_t up = (ev[o] + 3) & ~int64_t(3);
      hi[o] = up <= a.ops.op[o].nnz ? up : (ev[o] & ~int64_t(3));
      if (!a.use_bulk || hi[o] <= sv[o]) hi[o] = lo;
      bytes += (uint32_t)(hi[o] - lo) * (4u + (uint32_t)sizeof(V));
    }
    const bool pcopy = a.use_bulk && lrows > 0 && pe > ps;
    if (pcopy) bytes += (uint32_t)(pe - ps) * 8u * (uint32_t)a.ndist;
    // 1. the transaction bytes, then the copies (one per lane: crd of operand o at lane o, val at
    //    lane K + o, pos of distinct array d at lane 2K + d) -- nothing waits on global memory first
    if (lane == 0 && bytes) mbar_expect_tx(&sh.full[s], bytes);
    __syncwarp();
    if (lane < 2 * K) {
      const int o = lane < K ? lane : lane - K;
      int64_t so2 = 0, hi2 = 0;
      int bo = 0;
#pragma unroll
      for (int oo = 0; oo < K; ++oo) if (oo == o) { so2 = sv[oo]; hi2 = hi[oo]; bo = base[oo]; }
      const int64_t lo = so2 & ~int64_t(3);
      if (hi2 > lo) {
        const OpView& op = a.ops.op[o];
        const uint32_t nb = (uint32_t)(hi2 - lo);
        if (lane < K) bulk_g2s(g.key + bo, op.crd + lo, nb * 4u, &sh.full[s]);
        else bulk_g2s(g.val + bo, static_cast<const V*>(op.val) + lo, nb * (uint32_t)sizeof(V), &sh.full[s]);
      }
    } else if (lane < 2 * K + a.ndist) {
      const int d = lane - 2 * K;
      if (pcopy) bulk_g2s(g.pos + d * a.sp, a.dpos[d] + ps, (uint32_t)(pe - ps) * 8u, &sh.full[s]);
    }
    // 2. entries the copies do not cover (array ends, unaligned bases): plain loads
#pragma unroll
    for (int o = 0; o < K; ++o) {
      const int64_t from = hi[o] > (sv[o] & ~int64_t(3)) ? hi[o] : sv[o];
      if (from < ev[o]) {
        const OpView& op = a.ops.op[o];
        for (int64_t q = from + lane; q < ev[o]; q += 32) {
          const int slot = soff[o] + (int)(q - sv[o]);
          g.key[slot] = (uint32_t)ldg(op.crd + q);
          g.val[slot] = ldg(static_cast<const V*>(op.val) + q);
        }
      }
    }
    if (lrows > 0 && (!pcopy || pe < pneed)) {
      for (int d = 0; d < a.ndist; ++d)
        for (int64_t r = (pcopy ? pe : ps) + lane; r < pneed; r += 32) g.pos[d * a.sp + (int)(r - ps)] = ldg(a.dpos[d] + r);
    }
    // 3. the arrival: releases the record and the plain stores; the phase completes with the copies
    __syncwarp();
    if (lane == 0) mbar_arrive(&sh.full[s]);
  };
  fetch();
  for (;;) {
    if (t >= P) {   // no partitions left: a stop record
      job(-1, 1, 1, 0, 0, 0, 0);
      break;
    }
    const int64_t tile = t, row0 = r0, L = r1 - r0;
    const int64_t so = ps_o, eo = pe_o;
    if (L < lmax) {
      job(tile, 1, 1, row0, (int)L, so, eo);
      fetch();
      continue;
    }
    const int nsub = (int)((L + lmax) / lmax);
    for (int pass = 0; pass < (OP == kS7InterSum ? 1 : 2); ++pass) {
      for (int j = 0; j < nsub; ++j) {
        const int64_t a0 = row0 + (int64_t)j * lmax;
        const int lrows = (int)(j < nsub - 1 ? lmax : L - (int64_t)j * lmax);
        int64_t s_j = so, e_j = eo;
        if (lane < K) {
          if (j > 0) s_j = ldg(a.dpos[a.pd[lane]] + a0);
          if (j < nsub - 1) e_j = ldg(a.dpos[a.pd[lane]] + a0 + lmax);
        }
        job(tile, pass == 0 ? 0 : 2, j == nsub - 1, a0, lrows, s_j, e_j);
      }
    }
    fetch();
  }
}

// ------------------------------------------------------------------ emission warp
template <typename V, int K, int OP>
__device__ __forceinline__ void s7_emit(const S7Args<V>& a, S7Smem<V, K>& sh) {
  constexpr int NS = S7Cfg<V, K>::NS;
  const int lane = threadIdx.x & 31;
  const int P = a.parts.P;
  for (int njob = 0;; ++njob) {
    const int s = njob % NS;
    const uint32_t ph = (uint32_t)(njob / NS) & 1u;
    // the look-back of a one-pass job runs while the compute warps merge it: it needs only the
    // predecessors' states, so it starts as soon as the job record is in the stage
    s7_wait_sleep(&sh.full[s], ph, NACHO_S7_SLEEP_EF);
    S7Stage<V, K>& g = sh.st[s];
    const int64_t t = g.tile;
    const int mode = g.mode;
    int64_t excl = 0;
    if (OP != kS7InterSum && t > 0 && mode == 1) {
      S7_T0();
      excl = s5_lookback(a.state, t);
      if (lane == 0) S7_ACC(2);   // emission: look-back
    }
    if (lane == 0) {   // the compute warps publish the inclusive prefix at once if it is known
      sh.excl[s] = excl;
      __threadfence_block();
      *reinterpret_cast<volatile int*>(&sh.excl_ok[s]) = 1;
    }
    {
      S7_T0();
      s7_wait_sleep(&sh.done[s], ph, NACHO_S7_SLEEP_ED);
      if (lane == 0) S7_ACC(1);   // emission: waiting for a computed stage
    }
    if (lane == 0) sh.excl_ok[s] = 0;
    if (t < 0) break;
    if (OP != kS7InterSum && mode != 0) {
      const int total = g.total, lrows = g.lrows;
      const int64_t a0 = g.a0;
      int64_t off;
      if (mode == 2) {
        off = g.off;
      } else {
        off = excl;
        if (lane == 0) {
          if (t > 0) st_release(a.state + t, kS5Incl | (unsigned long long)(off + total));
          if (a.part_off) {
            a.part_off[t] = off;
            if (t == P - 1) a.part_off[P] = off + total;
          }
        }
      }
      S7_T0();
      int32_t* zc = a.z_crd + off;
      V* zv = a.z_val + off;
#pragma unroll 4
      for (int q = lane; q < total; q += 32) {
        zc[q] = (int32_t)g.key[q];
        zv[q] = g.val[q];
      }
      const int32_t* zrel = reinterpret_cast<const int32_t*>(g.pos);
      for (int l = lane + 1; l <= lrows; l += 32) a.z_pos[a0 + l] = off + zrel[l];
      if (lane == 0) S7_ACC(8);   // emission: writing Z (dev builds)
    }
    fence_proxy_async();   // generic accesses of the stage before the producer's bulk copies
    __syncwarp();
    if (lane == 0) mbar_arrive(&sh.empty[s]);
  }
}

// ------------------------------------------------------------------ one-row jobs: bitmap union
// A job inside one row whose columns span at most s7_bw<K>() words (most partitions of a power-law
// matrix's heavy rows): per-operand column bitmaps (one atomic OR per entry), the union bitmap's
// exclusive popcount prefix gives every union column its output index, and the values fold into
// that slot operand by operand -- the left fold in operand order from the first present value
// (R9) -- so no keys and no merge stages.  Returns the union size; with `emit` the union (column,
// value) is written at [0, total) of the stage's key / val arrays (inputs are held in registers).
template <int K>
__host__ __device__ constexpr int s7_bw() { return (3 * (kS7Slots + 16) / 2 - 8) / (K + 2); }

template <typename V, int K, int OP>
__device__ __forceinline__ int s7_bitmap(S7Stage<V, K>& g, S7Smem<V, K>& sh, int cmin, int nw, int S, bool emit) {
  const int tid = threadIdx.x;
  uint32_t* bm = sh.key1;              // [K][nw] operand bitmaps, then U[nw] union, pre[nw + 1]
  uint32_t* U = bm + K * nw;
  uint32_t* pre = U + nw;
  for (int w = tid; w < K * nw; w += kS7Compute) bm[w] = 0;
  if (tid < 8 * K) {   // pad slots of every run (<= 3 before, <= 4 after it) -> ~0u: not an entry
    const int o = tid >> 3, j = tid & 7;
    const int z = j < 4 ? g.base[o] + j : g.soff[o] + g.n[o] + (j - 4);
    if ((j < 4 && z < g.soff[o]) || (j >= 4 && z < g.base[o + 1])) g.key[z] = ~0u;
  }
  s6_sync();   // bitmaps zeroed, pads marked
  // slots d .. d + 7 (consecutive: mostly one operand, sorted columns): the bits of one word are
  // combined in registers, one atomic OR per distinct word (1-2 per thread on dense rows)
  const int d = tid * kS5VT;
  uint32_t c[kS5VT];
  V v[kS5VT];
  int oo[kS5VT];   // operand of the slot, -1: not an entry
  {
    const uint4 c0 = reinterpret_cast<const uint4*>(g.key + d)[0];
    const uint4 c1 = reinterpret_cast<const uint4*>(g.key + d)[1];
    c[0] = c0.x; c[1] = c0.y; c[2] = c0.z; c[3] = c0.w; c[4] = c1.x; c[5] = c1.y; c[6] = c1.z; c[7] = c1.w;
  }
  uint32_t cw = ~0u, cbits = 0;
#pragma unroll
  for (int i = 0; i < kS5VT; ++i) {
    const int slot = d + i;
    int o = 0;
#pragma unroll
    for (int q = 1; q < K; ++q) o += slot >= g.base[q] ? 1 : 0;
    const bool ok = slot < S && c[i] != ~0u;
    oo[i] = ok ? o : -1;
    v[i] = ok ? g.val[slot] : V(0);
    c[i] -= (uint32_t)cmin;
    if (ok) {
      const uint32_t w = (uint32_t)(o * nw) + (c[i] >> 5);
      if (w != cw) {
        if (cw != ~0u) atomicOr(&bm[cw], cbits);
        cw = w;
        cbits = 0;
      }
      cbits |= 1u << (c[i] & 31);
    }
  }
  if (cw != ~0u) atomicOr(&bm[cw], cbits);
  s6_sync();
  // union words and their exclusive popcount prefix (each thread a contiguous run of words)
  const int wpt = (nw + kS7Compute - 1) / kS7Compute;
  const int w0 = tid * wpt;
  int cnt = 0;
  for (int w = w0; w < w0 + wpt && w < nw; ++w) {
    uint32_t u = OP == kS7Union ? 0u : ~0u;
#pragma unroll
    for (int q = 0; q < K; ++q) u = OP == kS7Union ? (u | bm[q * nw + w]) : (u & bm[q * nw + w]);
    U[w] = u;
    cnt += __popc(u);
  }
  int total;
  int run = s6_block_excl(cnt, sh.wred, &total);
  for (int w = w0; w < w0 + wpt && w < nw; ++w) {
    pre[w] = (uint32_t)run;
    run += __popc(U[w]);
  }
  if (!emit) return total;
  s6_sync();
  // values fold operand by operand (one phase per operand: distinct output slots within a phase)
#pragma unroll
  for (int o = 0; o < K; ++o) {
#pragma unroll
    for (int i = 0; i < kS5VT; ++i) {
      if (oo[i] == o) {
        const int w = (int)(c[i] >> 5);
        const uint32_t bit = c[i] & 31;
        const uint32_t uw = U[w];
        const int idx = (int)pre[w] + __popc(uw & ((1u << bit) - 1u));
        if (OP == kS7Union) {
          uint32_t lower = 0;
#pragma unroll
          for (int q = 0; q < K; ++q) if (q < o) lower |= bm[q * nw + w];
          if ((lower >> bit) & 1u) {
            g.val[idx] = g.val[idx] + v[i];
          } else {
            g.key[idx] = c[i] + (uint32_t)cmin;
            g.val[idx] = v[i];
          }
        } else if ((uw >> bit) & 1u) {   // in every operand: the product, left to right
          if (o == 0) {
            g.key[idx] = c[i] + (uint32_t)cmin;
            g.val[idx] = v[i];
          } else {
            g.val[idx] = g.val[idx] * v[i];
          }
        }
      }
    }
    if (o + 1 < K) s6_sync();
  }
  return total;
}

// ------------------------------------------------------------------ compute warps
template <typename V, int K, int OP>
__device__ __forceinline__ void s7_compute(const S7Args<V>& a, S7Smem<V, K>& sh) {
  constexpr int NS = S7Cfg<V, K>::NS;
  const int tid = threadIdx.x;
  const int P = a.parts.P;
  int64_t cnt_total = 0, run_off = 0;
  double sum_run = 0.0;   // kS7InterSum: the current partition's sum over its sub-tiles (thread 0)
  for (int njob = 0;; ++njob) {
    const int s = njob % NS;
    {
      S7_T0();
      s7_wait_sleep(&sh.full[s], (uint32_t)(njob / NS) & 1u, NACHO_S7_SLEEP_C);
      if (tid == 0) S7_ACC(3);   // compute: waiting for a loaded stage
    }
    S7Stage<V, K>& g = sh.st[s];
    const int64_t t = g.tile;
    if (t < 0) {
      if (tid == 0) mbar_arrive(&sh.done[s]);   // forwards the stop record to the emission warp
      break;
    }
    const int mode = g.mode;
    const int last = g.last;   // read before the union count: tid 0 may free the stage right after it
    const int S = g.base[K];
    const int lrows = g.lrows;
    // ---- one-row job with a narrow column span: the bitmap union
    int cmin = INT32_MAX, cmax = -1;
    if (lrows == 0) {
#pragma unroll
      for (int o = 0; o < K; ++o) {
        if (g.n[o] > 0) {
          cmin = min(cmin, (int)g.key[g.soff[o]]);
          cmax = max(cmax, (int)g.key[g.soff[o] + g.n[o] - 1]);
        }
      }
    }
    const int nw = cmax >= cmin ? ((cmax - cmin) >> 5) + 1 : 0;
    const bool bmp = lrows == 0 && nw > 0 && nw <= s7_bw<K>();
    const int d = tid * kS5VT;
    V res[kS5VT];
    uint32_t col[kS5VT];
    uint32_t em = 0;   // merge path: bit v -- item v ends a run this thread owns (one union entry)
    int n = 0, ex = 0, total = 0;
#ifdef NACHO_S7_PROF
    const long long _tc = clock64();
#endif
    if (bmp) {
      total = s7_bitmap<V, K, OP>(g, sh, cmin, nw, S, mode != 0 || OP == kS7InterSum);
    } else {
      // ---- partition-local row of every slot (multi-row jobs only), keys in place, run sentinels
      if (lrows > 0) {
        for (int c = tid; c < (S >> 2); c += kS7Compute) {   // mark (o << 16) | 0: operand o, local row 0
          const int slot = c << 2;
          uint32_t o = 0;
  #pragma unroll
          for (int oo = 1; oo < K; ++oo) o += slot >= g.base[oo] ? 1u : 0u;
          const uint32_t m = o << 16;
          reinterpret_cast<uint4*>(sh.key1)[c] = make_uint4(m, m, m, m);
        }
        s6_sync();
        const int64_t pb = g.a0 - g.ps;
        for (int l = tid + 1; l <= lrows; l += kS7Compute) {   // first entry of rows 1 .. lrows
          int msum = 0;
  #pragma unroll
          for (int o = 0; o < K; ++o) {
            const int64_t* pp = g.pos + a.pd[o] * a.sp + (pb + l);
            const int64_t so = g.s[o], eo = g.e[o];
            const int64_t p = min(pp[0], eo);
            const int64_t pn = l < lrows ? min(pp[1], eo) : eo;
            const int rel = (int)(p - so);
            msum += rel;
            if (pn > p) sh.key1[g.soff[o] + rel] = ((uint32_t)o << 16) | (uint32_t)l;
          }
          sh.ML[l] = msum;
        }
        s6_sync();
        const int d = tid * kS5VT;
        uint32_t m[kS5VT];
        const uint4 m0 = reinterpret_cast<const uint4*>(sh.key1 + d)[0];
        const uint4 m1 = reinterpret_cast<const uint4*>(sh.key1 + d)[1];
        m[0] = m0.x; m[1] = m0.y; m[2] = m0.z; m[3] = m0.w; m[4] = m1.x; m[5] = m1.y; m[6] = m1.z; m[7] = m1.w;
  #pragma unroll
        for (int v = 1; v < kS5VT; ++v) m[v] = max(m[v], m[v - 1]);
        const uint32_t pre = s6_block_excl_max(m[kS5VT - 1], sh.wred);
        if (d < S) {
          uint4* k4 = reinterpret_cast<uint4*>(g.key + d);
          uint4 c0 = k4[0], c1 = k4[1];
          const int cb = a.cb;
          auto mk = [&](uint32_t c, uint32_t mm) { return ((max(mm, pre) & 0xffffu) << cb) | c; };
          c0.x = mk(c0.x, m[0]); c0.y = mk(c0.y, m[1]); c0.z = mk(c0.z, m[2]); c0.w = mk(c0.w, m[3]);
          c1.x = mk(c1.x, m[4]); c1.y = mk(c1.y, m[5]); c1.z = mk(c1.z, m[6]); c1.w = mk(c1.w, m[7]);
          k4[0] = c0;
          k4[1] = c1;
  #pragma unroll
          for (int o = 0; o < K; ++o) {   // the sentinel after every run, by the slot's owner
            const int z = g.soff[o] + g.n[o];
            if (z >= d && z < d + kS5VT) g.key[z] = kS5Inf;
          }
        }
      } else if (tid < K) {
        g.key[g.soff[tid] + g.n[tid]] = kS5Inf;   // the sentinel after every run (keys are the columns)
      }
      s6_sync();
      // ---- merge stages 1 .. K-2
      const uint32_t* X = g.key + g.soff[0];
      const uint16_t* XS = sh.src1;
      const int xs0 = g.soff[0];
      int na = g.n[0];
  #pragma unroll
      for (int st = 1; st + 1 < K; ++st) {
        uint32_t* OK = (st & 1) ? sh.key1 : sh.key2;
        uint16_t* OS = (st & 1) ? sh.src1 : sh.src2;
        if (st == 1) s5_merge_stage<false>(X, XS, xs0, na, g.key + g.soff[st], g.soff[st], g.n[st], OK, OS);
        else s5_merge_stage<true>(X, XS, xs0, na, g.key + g.soff[st], g.soff[st], g.n[st], OK, OS);
        s6_sync();
        X = OK;
        XS = OS;
        na += g.n[st];
      }
      // ---- last stage: merge, fold equal keys (R9), count
      constexpr bool XSRC = K >= 3;
      const uint32_t* Y = K > 1 ? g.key + g.soff[K - 1] : g.key + g.soff[0] + g.n[0];
      const int ys0 = K > 1 ? g.soff[K - 1] : 0;
      const int nb = K > 1 ? g.n[K - 1] : 0;
      n = na + nb;
      const uint32_t cmask = (1u << a.cb) - 1u;
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
        int rl = 0;   // operands storing the current key (the run length)
  #pragma unroll
        for (int v = 0; v < kS5VT; ++v) {
          uint32_t key;
          int slot;
          s5_step<XSRC>(X, XS, xs0, Y, ys0, i, jj, xk, yk, key, slot);
          const bool valid = d + v < n;
          const bool start = valid && key != pk;
          // a run ends: one union entry; an intersection entry only if every operand stores the key
          if (v > 0 && own && (start || !valid) && d + v - 1 < n && (OP == kS7Union || rl == K)) em |= 1u << (v - 1);
          own = own || start;
          if (own && valid) {
            const V x = g.val[slot];
            acc = start ? x : (OP == kS7Union ? acc + x : acc * x);
            rl = start ? 1 : rl + 1;
          }
          res[v] = acc;
          col[v] = key & cmask;
          pk = key;
        }
        if (own && d + kS5VT <= n) {   // the last run may continue past this thread's items
  #pragma unroll
          for (int r = 0; r < K - 1; ++r) {
            if (d + kS5VT + r >= n || (xk <= yk ? xk : yk) != pk) break;
            uint32_t key;
            int slot;
            s5_step<XSRC>(X, XS, xs0, Y, ys0, i, jj, xk, yk, key, slot);
            acc = OP == kS7Union ? acc + g.val[slot] : acc * g.val[slot];
            ++rl;
          }
          if (OP == kS7Union || rl == K) em |= 1u << (kS5VT - 1);
          res[kS5VT - 1] = acc;
        }
      }
      ex = s6_block_excl(__popc(em), sh.wred, &total);   // syncs: every merge / fold is done
    }
#ifdef NACHO_S7_PROF
    if (tid == 0) atomicAdd(a.state + a.parts.P + 2 + (bmp ? 4 : 5), (unsigned long long)(clock64() - _tc));
    if (tid == 0) atomicAdd(a.state + a.parts.P + 2 + (bmp ? 6 : 7), 1ull);
#endif
    if (OP == kS7InterSum) {   // the partition's sum of products (deterministic order), no output
      double ps = 0.0;
      if (bmp) {
        s6_sync();   // the last operand phase's products
        for (int q = tid; q < total; q += kS7Compute) ps += (double)g.val[q];
      } else {
#pragma unroll
        for (int v = 0; v < kS5VT; ++v) if (em & (1u << v)) ps += (double)res[v];
      }
#pragma unroll
      for (int o2 = 16; o2 > 0; o2 >>= 1) ps += __shfl_xor_sync(kFull, ps, o2);
      if ((tid & 31) == 0) sh.wsum[tid >> 5] = ps;
      s6_sync();
      if (tid == 0) {
        double js = 0.0;
        for (int w = 0; w < kS7Compute / 32; ++w) js += sh.wsum[w];
        sum_run += js;
        if (mode == 1 || last) {
          a.partial[t] = sum_run;
          sum_run = 0.0;
        }
        g.total = total;
      }
      s6_sync();
      if (tid == 0) mbar_arrive(&sh.done[s]);
      continue;
    }
    if (mode == 0) {   // count a sub-tile; after the last one: publish, look back, known offset
      cnt_total += total;
      if (last) {
        if (tid < 32) {
          int64_t excl = 0;
          if (t == 0) {
            if (tid == 0) st_release(a.state, kS5Incl | (unsigned long long)cnt_total);
          } else {
            if (tid == 0) st_release(a.state + t, kS5Agg | (unsigned long long)cnt_total);
            excl = s5_lookback(a.state, t);
            if (tid == 0) st_release(a.state + t, kS5Incl | (unsigned long long)(excl + cnt_total));
          }
          if (tid == 0) {
            sh.run_off = excl;
            if (a.part_off) {
              a.part_off[t] = excl;
              if (t == P - 1) a.part_off[P] = excl + cnt_total;
            }
          }
        }
        s6_sync();
        run_off = sh.run_off;
        cnt_total = 0;
      }
      if (tid == 0) mbar_arrive(&sh.done[s]);
      continue;
    }
    if (tid == 0) {
      if (mode == 1) {   // inclusive prefix if the early look-back is done, else the aggregate
        const bool known = t == 0 || *reinterpret_cast<volatile int*>(&sh.excl_ok[s]) != 0;
        __threadfence_block();
        const unsigned long long v = known ? kS5Incl | (unsigned long long)(sh.excl[s] + total)
                                           : kS5Agg | (unsigned long long)total;
        st_release(a.state + t, t == 0 ? kS5Incl | (unsigned long long)total : v);
      }
      else g.off = run_off;
      g.total = total;
    }
    if (mode == 2) run_off += total;
    // ---- the compacted union into the stage, and the union count before each owned row
    if (!bmp && d < n) {
      int e = ex;
#pragma unroll
      for (int v = 0; v < kS5VT; ++v) {
        if (d + v < n) sh.key1[d + v] = (uint32_t)e;   // U: union entries before merged position d + v
        if (em & (1u << v)) { g.key[e] = col[v]; g.val[e] = res[v]; ++e; }
      }
    }
    if (tid == 0 && !bmp) sh.key1[n] = (uint32_t)total;
    s6_sync();
    int32_t* zrel = reinterpret_cast<int32_t*>(g.pos);
    for (int l = tid + 1; l <= lrows; l += kS7Compute) zrel[l] = (int32_t)sh.key1[sh.ML[l]];
    fence_proxy_async();
    s6_sync();   // key1 / ML are reused by the next job
    if (tid == 0) mbar_arrive(&sh.done[s]);
  }
}

template <typename V, int K, int OP>
__global__ void __launch_bounds__(kS7Threads, S7Cfg<V, K>::MINB) spadd7_kernel(const S7Args<V> a) {
  extern __shared__ __align__(128) unsigned char s7_raw[];
  S7Smem<V, K>& sh = *reinterpret_cast<S7Smem<V, K>*>(s7_raw);
  constexpr int NS = S7Cfg<V, K>::NS;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&sh.full[s], 1);
      mbar_init(&sh.done[s], 1);
      mbar_init(&sh.empty[s], 1);
      sh.excl_ok[s] = 0;
    }
    fence_barrier_init();
  }
  __syncthreads();
  const int w = threadIdx.x >> 5;
  if (w == kS7Compute / 32) s7_produce<V, K, OP>(a, sh);
  else if (w == kS7Compute / 32 + 1) s7_emit<V, K, OP>(a, sh);
  else s7_compute<V, K, OP>(a, sh);
}

// Sum of the per-partition partials in a fixed order (one CTA): the inner product's final reduction.
__global__ void __launch_bounds__(1024) s7_sum_partials_kernel(const double* __restrict__ partial, int64_t P,
                                                               double* __restrict__ out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int64_t p = threadIdx.x; p < P; p += blockDim.x) s += partial[p];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    *out = t;
  }
}

}  // namespace nacho
