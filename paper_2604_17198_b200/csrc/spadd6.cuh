// spadd6.cuh -- the single-read k-way SpAdd of spadd5.cuh as a persistent, warp-specialised kernel:
// the write-offset resolution (decoupled look-back over the union counts) and the output
// writes (Z.crd / Z.val / Z.pos) move from the CTA's critical path to a dedicated
// emission warp, so the eight compute warps go on to the next partition while the offset of the
// previous one resolves.
//
//   compute warps 0-7 (per partition, ticket order): bulk-copy the operand ranges, row marks, keys,
//     k - 1 merge-path stages with the fold, union count -> publish the count ("aggregate") ->
//     wait until the emission slot is free -> compacted union + per-row union offsets into the slot
//     -> hand the slot to the emission warp (mbarrier `full`) -> next partition;
//   emission warp 8: wait `full` -> look-back (exclusive prefix of the counts of the partitions
//     before this one) -> publish the inclusive prefix -> write Z.crd / Z.val at the offset and
//     Z.pos of the rows the partition owns (R7) -> free the slot (mbarrier `empty`).
// A partition spanning more rows than a sub-tile holds runs its sub-tiles twice (count, then
// emit at the offset the compute warps resolve themselves), as in spadd5.cuh.
#pragma once
#include "spadd5.cuh"

namespace nacho {

constexpr int kS6Compute = kS5Threads;            // compute threads (warps 0 .. 7)
constexpr int kS6Threads = kS6Compute + 32;       // + the emission warp
constexpr int kS6Slots = kS5Slots;

__device__ __forceinline__ void s6_sync() { named_sync(1, kS6Compute); }

template <typename V, int K>
struct S6Smem {
  uint32_t key0[kS6Slots + 16];   // crd (bulk copy) -> keys in place
  V val[kS6Slots];                 // values (bulk copy)
  uint32_t key1[kS6Slots + 16];   // row marks -> merge output -> union prefix U
  uint16_t src1[kS6Slots + 16];
  uint32_t key2[K >= 4 ? kS6Slots + 16 : 1];
  uint16_t src2[K >= 4 ? kS6Slots + 16 : 1];
  int32_t ML[kS5LMax + 1];        // merged position of each owned row's first entry
  // emission slot: compute warps -> emission warp
  int32_t outc[kS6Slots];
  V outv[kS6Slots];
  int32_t zrel[kS5LMax + 1];      // union entries of the slot's rows before each owned row
  int64_t j_tile, j_a0, j_off;
  int32_t j_total, j_lrows, j_known;
  // compute-side state of the current (sub-)tile
  int64_t s[K], e[K];
  int32_t soff[K], n[K], base[K + 1];
  int64_t tile, r0, r1, a0, off;
  int32_t lrows;
  int32_t wred[kS6Compute / 32];
  uint64_t bar_load, bar_full, bar_empty;
};

__device__ __forceinline__ bool s6_try(uint64_t* bar, uint32_t parity) { return mbar_try_wait(bar, parity); }
__device__ __forceinline__ void s6_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// Exclusive sum / max over the compute threads (named barrier 1).
__device__ __forceinline__ int s6_block_excl(int v, int32_t* wred, int* total) {
  constexpr int NW = kS6Compute / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int y = __shfl_up_sync(kFull, x, d);
    if (lane >= d) x += y;
  }
  if (lane == 31) wred[w] = x;
  s6_sync();
  int ws = lane < NW ? wred[lane] : 0;
#pragma unroll
  for (int d = 1; d < NW; d <<= 1) {
    const int y = __shfl_up_sync(kFull, ws, d);
    if (lane >= d) ws += y;
  }
  const int pre = __shfl_sync(kFull, ws, (w + 31) & 31);
  *total = __shfl_sync(kFull, ws, NW - 1);
  s6_sync();
  return (w ? pre : 0) + x - v;
}

__device__ __forceinline__ uint32_t s6_block_excl_max(uint32_t v, int32_t* wred) {
  constexpr int NW = kS6Compute / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, x, d);
    if (lane >= d) x = max(x, y);
  }
  if (lane == 31) wred[w] = (int32_t)x;
  s6_sync();
  uint32_t ws = lane < NW ? (uint32_t)wred[lane] : 0u;
#pragma unroll
  for (int d = 1; d < NW; d <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, ws, d);
    if (lane >= d) ws = max(ws, y);
  }
  const uint32_t pre = __shfl_sync(kFull, ws, (w + 31) & 31);
  s6_sync();
  const uint32_t ex = __shfl_up_sync(kFull, x, 1);
  return max(w ? pre : 0u, lane ? ex : 0u);
}

// ------------------------------------------------------------------ compute warps: one (sub-)tile
// mode 0: count only.  mode 1: count, publish the aggregate, hand the union to the emission warp
// (which resolves the offset).  mode 2: hand the union over at the known offset sh.off.
template <typename V, int K>
__device__ __forceinline__ int s6_tile(const S5Args<V>& a, S6Smem<V, K>& sh, int j, int nsub, int mode,
                                       uint32_t& ph_load, uint32_t& ph_empty) {
  const int tid = threadIdx.x;
  const int lmax = a.lmax;
  // ---- bounds, slot layout and the bulk copies (one thread: its loads issue back to back)
  if (tid == 0) {
    const int64_t a0 = sh.r0 + (int64_t)j * lmax;
    const int64_t L = sh.r1 - sh.r0;
    sh.a0 = a0;
    sh.lrows = (int32_t)(j < nsub - 1 ? lmax : L - (int64_t)j * lmax);
    int64_t s[K], e[K];
#pragma unroll
    for (int o = 0; o < K; ++o) {
      s[o] = j > 0 ? ldg(a.ops.op[o].pos + a0) : a.parts.pos[sh.tile * K + o];
      e[o] = j < nsub - 1 ? ldg(a.ops.op[o].pos + a0 + lmax) : a.parts.pos[(sh.tile + 1) * K + o];
    }
    int b = 0;
    uint32_t bytes = 0;
    int64_t lo[K], hi[K];
#pragma unroll
    for (int o = 0; o < K; ++o) {
      const int n = (int)(e[o] - s[o]);
      sh.s[o] = s[o];
      sh.e[o] = e[o];
      sh.base[o] = b;
      sh.soff[o] = b + (int)(s[o] & 3);
      sh.n[o] = n;
      b = (sh.soff[o] + n + 4) & ~3;   // >= 1 pad slot: the run's sentinel
      lo[o] = s[o] & ~int64_t(3);
      hi[o] = e[o] & ~int64_t(3);
      if (!a.use_bulk || hi[o] <= s[o]) hi[o] = lo[o];
      bytes += (uint32_t)(hi[o] - lo[o]) * (4u + (uint32_t)sizeof(V));
    }
    sh.base[K] = b;
    fence_proxy_async();   // earlier generic accesses of these buffers before the async writes
    if (bytes) {
      mbar_arrive_expect_tx(&sh.bar_load, bytes);
#pragma unroll
      for (int o = 0; o < K; ++o) {
        if (hi[o] > lo[o]) {
          const OpView& op = a.ops.op[o];
          const uint32_t nb = (uint32_t)(hi[o] - lo[o]);
          bulk_g2s(sh.key0 + sh.base[o], op.crd + lo[o], nb * 4u, &sh.bar_load);
          bulk_g2s(sh.val + sh.base[o], static_cast<const V*>(op.val) + lo[o], nb * (uint32_t)sizeof(V),
                   &sh.bar_load);
        }
      }
    } else {
      mbar_arrive(&sh.bar_load);
    }
  }
  s6_sync();
  const int S = sh.base[K];
  // ---- entries the bulk copies do not cover (< 4 per operand; warp 1), row-mark initialisation:
  // every slot of operand o's region starts at mark (o << 16) | 0 (local row 0)
  if (a.use_bulk) {
    if (tid >= 32 && tid < 32 + 4 * K) {
      const int o = (tid - 32) >> 2;
#pragma unroll
      for (int oo = 0; oo < K; ++oo) {
        if (oo == o) {
          const int64_t s = sh.s[oo], e = sh.e[oo];
          const int64_t from = max(e & ~int64_t(3), s);
          const int64_t q = from + ((tid - 32) & 3);
          if (q < e) {
            const int slot = sh.soff[oo] + (int)(q - s);
            sh.key0[slot] = (uint32_t)ldg(a.ops.op[oo].crd + q);
            sh.val[slot] = ldg(static_cast<const V*>(a.ops.op[oo].val) + q);
          }
        }
      }
    }
  } else {
#pragma unroll
    for (int o = 0; o < K; ++o) {
      const int64_t s = sh.s[o], e = sh.e[o];
      for (int64_t q = s + tid; q < e; q += kS6Compute) {
        const int slot = sh.soff[o] + (int)(q - s);
        sh.key0[slot] = (uint32_t)ldg(a.ops.op[o].crd + q);
        sh.val[slot] = ldg(static_cast<const V*>(a.ops.op[o].val) + q);
      }
    }
  }
  for (int c = tid; c < (S >> 2); c += kS6Compute) {
    const int slot = c << 2;
    uint32_t o = 0;
#pragma unroll
    for (int oo = 1; oo < K; ++oo) o += slot >= sh.base[oo] ? 1u : 0u;
    const uint32_t m = o << 16;
    reinterpret_cast<uint4*>(sh.key1)[c] = make_uint4(m, m, m, m);
  }
  s6_sync();
  // ---- row marks: the first entry of every row l in [1, lrows] of each operand (Listing 8 bounds)
  const int lrows = sh.lrows;
  for (int l = tid + 1; l <= lrows; l += kS6Compute) {
    int msum = 0;
#pragma unroll
    for (int o = 0; o < K; ++o) {
      const int64_t* pp = a.ops.op[o].pos + sh.a0 + l;
      const int64_t eo = sh.e[o];
      const int64_t p = min(ldg(pp), eo);
      const int64_t pn = l < lrows ? min(ldg(pp + 1), eo) : eo;
      const int rel = (int)(p - sh.s[o]);
      msum += rel;
      if (pn > p) sh.key1[sh.soff[o] + rel] = ((uint32_t)o << 16) | (uint32_t)l;
    }
    sh.ML[l] = msum;
  }
  s6_sync();
  // ---- local row of every slot (max-scan of the marks), keys in place, run sentinels
  {
    const int d = tid * kS5VT;
    uint32_t m[kS5VT];
    const uint4 m0 = reinterpret_cast<const uint4*>(sh.key1 + d)[0];
    const uint4 m1 = reinterpret_cast<const uint4*>(sh.key1 + d)[1];
    m[0] = m0.x; m[1] = m0.y; m[2] = m0.z; m[3] = m0.w; m[4] = m1.x; m[5] = m1.y; m[6] = m1.z; m[7] = m1.w;
#pragma unroll
    for (int v = 1; v < kS5VT; ++v) m[v] = max(m[v], m[v - 1]);
    const uint32_t pre = s6_block_excl_max(m[kS5VT - 1], sh.wred);
    s6_wait(&sh.bar_load, ph_load);
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
      for (int o = 0; o < K; ++o) {
        const int z = sh.soff[o] + sh.n[o];
        if (z >= d && z < d + kS5VT) sh.key0[z] = kS5Inf;
      }
    }
  }
  ph_load ^= 1u;
  s6_sync();
  // ---- merge stages 1 .. K-2
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
    s6_sync();
    X = OK;
    XS = OS;
    na += sh.n[st];
  }
  // ---- last stage: merge, fold equal keys (R9), count
  constexpr bool XSRC = K >= 3;
  const uint32_t* Y = K > 1 ? sh.key0 + sh.soff[K - 1] : sh.key0 + sh.soff[0] + sh.n[0];
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
    if (own && d + kS5VT <= n) {   // the last run may continue past this thread's items
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
  const int ex = s6_block_excl(__popc(em), sh.wred, &total);   // syncs: every merge / fold is done
  if (mode == 0) return total;
  if (mode == 1 && tid == 0)   // the count is public at once (look-back state "aggregate")
    st_release(a.state + sh.tile, (sh.tile == 0 ? kS5Incl : kS5Agg) | (unsigned long long)total);
  // ---- hand the union to the emission warp
  s6_wait(&sh.bar_empty, ph_empty);
  ph_empty ^= 1u;
  if (d < n) {
    int e = ex;
#pragma unroll
    for (int v = 0; v < kS5VT; ++v) {
      if (d + v < n) sh.key1[d + v] = (uint32_t)e;   // U: union entries before merged position d + v
      if (em & (1u << v)) { sh.outc[e] = (int32_t)col[v]; sh.outv[e] = res[v]; ++e; }
    }
  }
  if (tid == 0) sh.key1[n] = (uint32_t)total;
  s6_sync();
  for (int l = tid + 1; l <= lrows; l += kS6Compute) sh.zrel[l] = (int32_t)sh.key1[sh.ML[l]];
  if (tid == 0) {
    sh.j_tile = sh.tile;
    sh.j_a0 = sh.a0;
    sh.j_total = total;
    sh.j_lrows = lrows;
    sh.j_known = mode == 2;
    sh.j_off = sh.off;
  }
  s6_sync();
  if (tid == 0) mbar_arrive(&sh.bar_full);
  return total;
}

// ------------------------------------------------------------------ emission warp
template <typename V, int K>
__device__ __forceinline__ void s6_emit(const S5Args<V>& a, S6Smem<V, K>& sh) {
  const int lane = threadIdx.x & 31;
  const int P = a.parts.P;
  uint32_t ph = 0;
  if (lane == 0) mbar_arrive(&sh.bar_empty);   // the slot starts free
  for (;;) {
    s6_wait(&sh.bar_full, ph);
    ph ^= 1u;
    const int64_t t = sh.j_tile;
    if (t < 0) break;
    const int total = sh.j_total, lrows = sh.j_lrows;
    const int64_t a0 = sh.j_a0;
    int64_t off;
    if (sh.j_known) {
      off = sh.j_off;
    } else {
      off = t > 0 ? s5_lookback(a.state, t) : 0;
      if (lane == 0) {
        if (t > 0) st_release(a.state + t, kS5Incl | (unsigned long long)(off + total));
        if (a.part_off) {
          a.part_off[t] = off;
          if (t == P - 1) a.part_off[P] = off + total;
        }
      }
    }
    for (int q = lane; q < total; q += 32) {
      a.z_crd[off + q] = sh.outc[q];
      a.z_val[off + q] = sh.outv[q];
    }
    for (int l = lane + 1; l <= lrows; l += 32) a.z_pos[a0 + l] = off + sh.zrel[l];
    __syncwarp();
    if (lane == 0) mbar_arrive(&sh.bar_empty);
  }
}

template <typename V, int K>
__global__ void __launch_bounds__(kS6Threads, 4) spadd6_kernel(const S5Args<V> a) {
  extern __shared__ __align__(128) unsigned char s6_raw[];
  S6Smem<V, K>& sh = *reinterpret_cast<S6Smem<V, K>*>(s6_raw);
  const int tid = threadIdx.x;
  const int P = a.parts.P;
  if (tid == 0) {
    mbar_init(&sh.bar_load, 1);
    mbar_init(&sh.bar_full, 1);
    mbar_init(&sh.bar_empty, 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (tid >= kS6Compute) {
    s6_emit<V, K>(a, sh);
    return;
  }
  const int lmax = a.lmax;
  uint32_t ph_load = 0, ph_empty = 0;
  for (;;) {
    if (tid == 0) {
      const int64_t t = (int64_t)atomicAdd(a.state + P, 1ull);   // ticket order: predecessors already run
      sh.tile = t;
      if (t < P) {
        sh.r0 = a.parts.row[t];
        sh.r1 = a.parts.row[t + 1];
        if (t == 0) a.z_pos[0] = 0;
      }
    }
    s6_sync();
    const int64_t t = sh.tile;
    if (t >= P) break;
    const int64_t L = sh.r1 - sh.r0;
    if (L < lmax) {
      s6_tile<V, K>(a, sh, 0, 1, 1, ph_load, ph_empty);
      continue;
    }
    // more rows than a sub-tile: count every sub-tile, resolve the offset here, then emit
    const int nsub = (int)((L + lmax) / lmax);
    int64_t total = 0;
    for (int j = 0; j < nsub; ++j) total += s6_tile<V, K>(a, sh, j, nsub, 0, ph_load, ph_empty);
    if (tid < 32) {
      int64_t excl = 0;
      if (t == 0) {
        if (tid == 0) st_release(a.state, kS5Incl | (unsigned long long)total);
      } else {
        if (tid == 0) st_release(a.state + t, kS5Agg | (unsigned long long)total);
        excl = s5_lookback(a.state, t);
        if (tid == 0) st_release(a.state + t, kS5Incl | (unsigned long long)(excl + total));
      }
      if (tid == 0) {
        sh.off = excl;
        if (a.part_off) {
          a.part_off[t] = excl;
          if (t == P - 1) a.part_off[P] = excl + total;
        }
      }
    }
    s6_sync();
    for (int j = 0; j < nsub; ++j) {
      const int c = s6_tile<V, K>(a, sh, j, nsub, 2, ph_load, ph_empty);
      if (tid == 0) sh.off += c;
      s6_sync();
    }
  }
  // no more partitions: stop the emission warp once the slot is free
  if (tid == 0) {
    s6_wait(&sh.bar_empty, ph_empty);
    sh.j_tile = -1;
    mbar_arrive(&sh.bar_full);
  }
}

}  // namespace nacho
