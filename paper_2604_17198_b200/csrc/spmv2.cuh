// spmv2.cuh -- the B200 partitioned CSR / DCSR SpMV, one CTA per partition
// of <= kSvTileMax positions (nacho_auto_partitions; larger partitions use spmv_kernel's chunk loop).
//
//   1. thread 0 stages the partition's crd / val range (from a 16-byte aligned start s0) and its row
//      pointers into shared memory with 1-D TMA bulk copies (cp.async.bulk, SASS UBLKCP);
//   2. thread t owns the 16-byte aligned slots [8t, 8t+8) of the staged range (positions s0 + slot
//      inside [s, e)) and reads them with vector loads; the CTA reduces its column range and, when
//      it spans <= XCAP columns, stages that x window with a second bulk copy, so the gathers x[crd]
//      are shared-memory reads (local / banded / dense-row tiles) instead of global ones;
//   3. row walk, keyed segmented scan and carries exactly as spmv_kernel (Listing 8 bounds,
//      ownership rule R7, carry fix-up in partition order).
#pragma once
#include "common.cuh"
#include "spmv.cuh"
#include "tma.cuh"

namespace nacho {

template <typename T>
struct Sv2Cfg;
template <>
struct Sv2Cfg<float> { static constexpr int XCAP = 5120; };
template <>
struct Sv2Cfg<double> { static constexpr int XCAP = 2560; };

constexpr int kSvThreads = 256;
constexpr int kSvIpt = 8;
constexpr int kSvSlots = kSvThreads * kSvIpt;   // 2048 staged slots
constexpr int kSvTileMax = kSvSlots - 8;        // positions per partition (room for the alignment shift)
constexpr int kSvPosCap = 256;
constexpr int kSvFewRows = 16;                  // tiles spanning <= this many rows take the row path

template <typename T>
struct Sv2Shared {
  uint64_t bar;
  int64_t s, e, s0, rp0, rpE;
  int32_t cmin_w[kSvThreads / 32], cmax_w[kSvThreads / 32];
  int32_t xlo;       // first column of the staged x window
  int32_t xmode;     // 1: x window staged
  int32_t pos_n;     // staged row pointers (rows rp0 .. rp0+pos_n-1), 0: read global
  int32_t pos_off;   // slot of row rp0 inside pos
  KV<T> agg[kSvThreads / 32];
  KV<T> wpre[kSvThreads / 32];
  T part[kSvFewRows + 1][kSvThreads / 32];
  alignas(16) int32_t crd[kSvSlots + 8];
  alignas(16) T val[kSvSlots + 8];
  alignas(16) T x[Sv2Cfg<T>::XCAP + 8];
  alignas(16) int64_t pos[kSvPosCap + 4];
};

template <typename T>
__global__ void __launch_bounds__(kSvThreads, 5) spmv2_kernel(const __grid_constant__ SpmvArgs<T> a) {
  constexpr int XCAP = Sv2Cfg<T>::XCAP;
  constexpr int W = kSvThreads / 32;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Sv2Shared<T>& sh = *reinterpret_cast<Sv2Shared<T>*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int p = blockIdx.x;

  if (tid == 0) {
    mbar_init(&sh.bar, 1);
    fence_barrier_init();
    const int64_t s = ldg(a.ppos + p), e = ldg(a.ppos + p + 1);
    const int64_t rp0 = ldg(a.prow + p), rpE = ldg(a.prow + p + 1);
    const int64_t nnz = ldg(a.ppos + a.P);
    const int64_t s0 = s & ~int64_t(3);
    sh.s = s; sh.e = e; sh.s0 = s0; sh.rp0 = rp0; sh.rpE = rpE;
    // crd / val: 16-byte aligned bulk copy of [s0, c); positions past c (array end only) by hand
    int64_t c = (e + 3) & ~int64_t(3);
    const int64_t lim = nnz & ~int64_t(3);
    if (c > lim) c = lim;
    if (c < s0) c = s0;
    for (int64_t q = (c > s ? c : s); q < e; ++q) {
      sh.crd[q - s0] = ldg(a.crd + q);
      sh.val[q - s0] = ldg(a.val + q);
    }
    uint32_t bytes = (uint32_t)(c - s0) * (4 + sizeof(T));
    // row pointers of rows rp0 .. min(rpE, nouter-1)+1
    const int64_t r_last = (rpE < a.nouter ? rpE : a.nouter - 1) + 1;
    const int64_t pn = r_last - rp0 + 1;
    const int64_t ps0 = rp0 & ~int64_t(1);
    int64_t pc = 0;
    if (pn <= kSvPosCap) {
      sh.pos_n = (int)pn;
      sh.pos_off = (int)(rp0 - ps0);
      pc = (r_last + 2) & ~int64_t(1);
      const int64_t plim = (a.nouter + 1) & ~int64_t(1);
      if (pc > plim) pc = plim;
      if (pc < ps0) pc = ps0;
      for (int64_t q = (pc > rp0 ? pc : rp0); q <= r_last; ++q) sh.pos[q - ps0] = ldg(a.pos + q);
      bytes += (uint32_t)(pc - ps0) * 8;
    } else {
      sh.pos_n = 0;
    }
    fence_proxy_async();
    mbar_arrive_expect_tx(&sh.bar, bytes);
    if (c > s0) {
      bulk_g2s(sh.crd, a.crd + s0, (uint32_t)(c - s0) * 4, &sh.bar);
      bulk_g2s(sh.val, a.val + s0, (uint32_t)(c - s0) * sizeof(T), &sh.bar);
    }
    if (pn <= kSvPosCap && pc > ps0) bulk_g2s(sh.pos, a.pos + ps0, (uint32_t)(pc - ps0) * 8, &sh.bar);
  }
  __syncthreads();
  mbar_wait(&sh.bar, 0);
  const int64_t s = sh.s, e = sh.e, s0 = sh.s0, rp0 = sh.rp0, rpE = sh.rpE;
  const int lo_slot = (int)(s - s0), hi_slot = (int)(e - s0);
  const int64_t r_end = rpE < a.nouter ? rpE : a.nouter - 1;   // last row with positions in [s, e)

  if (sh.pos_n && r_end - rp0 + 1 <= kSvFewRows) {
    // ======== few-row tile (heavy rows, dense rows): every row's slice is reduced by the whole CTA
    // with consecutive threads on consecutive positions, so the x gathers of a row are coalesced.
    const int64_t* PP = sh.pos + sh.pos_off - rp0;
    const int nr = (int)(r_end - rp0 + 1);
    for (int r = 0; r < nr; ++r) {
      const int64_t rs = PP[rp0 + r] > s ? PP[rp0 + r] : s;
      const int64_t re = PP[rp0 + r + 1] < e ? PP[rp0 + r + 1] : e;
      T acc = T(0);
      for (int j = (int)(rs - s0) + tid; j < (int)(re - s0); j += kSvThreads) acc += sh.val[j] * ldg(a.x + sh.crd[j]);
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) acc += __shfl_xor_sync(kFull, acc, d);
      if (lane == 0) sh.part[r][w] = acc;
    }
    __syncthreads();
    if (tid < nr) {
      T tot = T(0);
#pragma unroll
      for (int ww = 0; ww < W; ++ww) tot += sh.part[tid][ww];
      const int64_t r = rp0 + tid;
      if (PP[r + 1] <= e) a.y[y_index(a, r)] = tot;          // row finished here: owned (R7)
      else { a.carry_row[p] = r; a.carry_val[p] = tot; }     // row continues: carry
    }
    if (tid == 0 && (r_end < rp0 || PP[r_end + 1] <= e)) { a.carry_row[p] = -1; a.carry_val[p] = T(0); }
    return;
  }

  // ======== many-row tile: thread t owns the 16-byte aligned slots [8t, 8t+8) (positions s0 + slot
  // inside [s, e)), products from a staged x window when the tile's columns fit it
  const int j0 = tid * kSvIpt;
  int32_t cr[kSvIpt];
  T vv[kSvIpt];
  {
    const int4* c4 = reinterpret_cast<const int4*>(sh.crd + j0);
    const int4 ca = c4[0], cb = c4[1];
    cr[0] = ca.x; cr[1] = ca.y; cr[2] = ca.z; cr[3] = ca.w;
    cr[4] = cb.x; cr[5] = cb.y; cr[6] = cb.z; cr[7] = cb.w;
    if constexpr (sizeof(T) == 4) {
      const float4* v4 = reinterpret_cast<const float4*>(sh.val + j0);
      const float4 va = v4[0], vb = v4[1];
      vv[0] = va.x; vv[1] = va.y; vv[2] = va.z; vv[3] = va.w;
      vv[4] = vb.x; vv[5] = vb.y; vv[6] = vb.z; vv[7] = vb.w;
    } else {
      const double2* v2 = reinterpret_cast<const double2*>(sh.val + j0);
#pragma unroll
      for (int i = 0; i < 4; ++i) { const double2 t = v2[i]; vv[2 * i] = t.x; vv[2 * i + 1] = t.y; }
    }
  }
  const int ia = max(0, lo_slot - j0), ib = min(kSvIpt, hi_slot - j0);  // valid item range [ia, ib)
  int32_t cmn = INT32_MAX, cmx = -1;
#pragma unroll
  for (int i = 0; i < kSvIpt; ++i) if (i >= ia && i < ib) { cmn = min(cmn, cr[i]); cmx = max(cmx, cr[i]); }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    cmn = min(cmn, __shfl_xor_sync(kFull, cmn, d));
    cmx = max(cmx, __shfl_xor_sync(kFull, cmx, d));
  }
  if (lane == 0) { sh.cmin_w[w] = cmn; sh.cmax_w[w] = cmx; }
  __syncthreads();
  if (tid == 0) {
    int32_t lo = INT32_MAX, hi = -1;
    for (int ww = 0; ww < W; ++ww) { lo = min(lo, sh.cmin_w[ww]); hi = max(hi, sh.cmax_w[ww]); }
    const int32_t xlo = lo & ~3;
    sh.xmode = 0;
    if (hi >= lo && (int64_t)hi - xlo + 8 <= XCAP) {
      int64_t xc = ((int64_t)hi + 4) & ~int64_t(3);
      const int64_t xlim = a.ncols & ~int64_t(3);
      if (xc > xlim) xc = xlim;
      if (xc < xlo) xc = xlo;
      sh.xmode = 1;
      sh.xlo = xlo;
      for (int64_t q = xc; q <= hi; ++q) sh.x[q - xlo] = ldg(a.x + q);  // tail at the end of x
      fence_proxy_async();
      mbar_arrive_expect_tx(&sh.bar, (uint32_t)(xc - xlo) * sizeof(T));
      if (xc > xlo) bulk_g2s(sh.x, a.x + xlo, (uint32_t)(xc - xlo) * sizeof(T), &sh.bar);
    }
  }
  __syncthreads();
  const bool xs = sh.xmode != 0;
  if (xs) mbar_wait(&sh.bar, 1);
  const int32_t xlo = sh.xlo;

  // ---- products and row walk over my valid items
  const bool active = ib > ia || tid == 0;
  const int64_t at = s0 + j0 + ia;                  // first position of mine
  const int64_t bt = s0 + j0 + (ib > ia ? ib : ia); // one past my last
  const int64_t* PP = sh.pos_n ? sh.pos + sh.pos_off - rp0 : a.pos;   // PP[r] = pos[r]
  bool head = true, head_done = false;
  int64_t head_row = 0, rp = 0;
  T head_val = T(0), acc = T(0);
  if (active) {
    if (tid == 0) {
      rp = rp0;
    } else {  // largest rp in [rp0, min(rpE, nouter)] with pos[rp] <= at
      int64_t lo = rp0, hi = rpE < a.nouter ? rpE : a.nouter;
      while (lo < hi) {
        const int64_t m = lo + ((hi - lo + 1) >> 1);
        if (PP[m] <= at) lo = m; else hi = m - 1;
      }
      rp = lo;
    }
    int64_t next_end = rp < a.nouter ? PP[rp + 1] : INT64_MAX;
    // 32-bit local view of the row ends (position - s0)
    int32_t nend = (int32_t)min(next_end - s0, (int64_t)INT32_MAX);
#pragma unroll
    for (int i = 0; i < kSvIpt; ++i) {
      if (i >= ia && i < ib) {
        const int32_t q = j0 + i;
        while (nend <= q) {  // row rp finished before position q
          if (head) { head_done = true; head_row = rp; head_val = acc; head = false; }
          else a.y[y_index(a, rp)] = acc;
          acc = T(0);
          ++rp;
          nend = (int32_t)min(PP[rp + 1] - s0, (int64_t)INT32_MAX);
        }
        const T xv = xs ? sh.x[cr[i] - xlo] : ldg(a.x + cr[i]);
        acc += vv[i] * xv;
      }
    }
    next_end = (int64_t)nend + s0;
    if (nend == INT32_MAX) next_end = rp < a.nouter ? PP[rp + 1] : INT64_MAX;
    while (rp < a.nouter && next_end <= bt) {  // rows ending exactly at b_t (and empty ones) are ours
      if (head) { head_done = true; head_row = rp; head_val = acc; head = false; }
      else a.y[y_index(a, rp)] = acc;
      acc = T(0);
      ++rp;
      next_end = rp < a.nouter ? PP[rp + 1] : INT64_MAX;
    }
  }
  // ---- keyed scan of the tails (rp, acc) across the CTA
  KV<T> inc = active ? KV<T>{rp, acc} : KV<T>{INT64_MAX, T(0)};
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    KV<T> u;
    u.k = __shfl_up_sync(kFull, inc.k, d);
    u.v = __shfl_up_sync(kFull, inc.v, d);
    if (lane >= d) inc = kv_op(u, inc);
  }
  if (lane == 31) sh.agg[w] = inc;
  __syncthreads();
  if (tid < 32) {  // exclusive prefix of the warp aggregates, seeded with (rp0, 0)
    KV<T> run = KV<T>{rp0, T(0)};
    for (int ww = 0; ww < W; ++ww) {
      if (lane == ww) sh.wpre[ww] = run;
      run = kv_op(run, sh.agg[ww]);
    }
  }
  __syncthreads();
  const KV<T> pre = sh.wpre[w];
  KV<T> excl;
  excl.k = __shfl_up_sync(kFull, inc.k, 1);
  excl.v = __shfl_up_sync(kFull, inc.v, 1);
  excl = (lane == 0) ? pre : kv_op(pre, excl);
  if (head_done) {
    const T c = (excl.k == head_row) ? excl.v : T(0);
    a.y[y_index(a, head_row)] = c + head_val;
  }
  // CTA carry: inclusive value of the last active thread
  const int last = hi_slot > lo_slot ? (hi_slot - 1) / kSvIpt : lo_slot / kSvIpt;
  if (tid == (last < kSvThreads ? last : 0)) {
    const KV<T> c = kv_op(pre, inc);
    const bool has = c.k < a.nouter && c.k == rpE;
    a.carry_row[p] = has ? c.k : -1;
    a.carry_val[p] = has ? c.v : T(0);
  }
}

template <typename T>
constexpr size_t sv2_smem_bytes() { return sizeof(Sv2Shared<T>) + 128; }

}  // namespace nacho
