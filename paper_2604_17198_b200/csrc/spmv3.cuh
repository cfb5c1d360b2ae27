// spmv3.cuh -- partitioned CSR / DCSR SpMV: one CTA per tile of at most
// sv3_tile<T>() positions (nacho_auto_partitions sizes P so that a partition is one tile; a larger
// user partition runs as tile-sized chunks, one CTA each, cut in position space).
//
// Design (an HBM stream plus an x gather; no tensor cores).  Two limiters besides DRAM shape it:
//   * the L1TEX wavefronts of the x gather: a warp-wide load costs one wavefront per distinct
//     128-byte line (~1/cycle/SM), so a gather touching 32 lines moves one nonzero per cycle per SM
//     (~290 GNNZ/s chip-wide).  Warp w owns a chunk of 32*V consecutive positions and reads crd /
//     val / x lane-strided (instruction i touches positions 32i + lane): 128 contiguous bytes of crd
//     / val per instruction, and the gathers of a long row (columns a few apart) touch ~4 lines;
//   * instruction issue: no per-item branches.  Products go to shared memory; each thread then runs
//     a segmented inclusive scan over V consecutive products (128-bit smem accesses, row starts
//     flagged in a byte map), the threads' trailing runs are combined by a (flag, sum) scan, and one
//     thread per owned row reads its sum at the row's last item.  Rows owned (R7: rows
//     [b_p.row, b_{p+1}.row)) are written once; the row cut by b_{p+1} leaves a carry that
//     spmv_fixup_kernel adds in partition order (Listing 8's bounds).
#pragma once
#include "common.cuh"
#include "spmv.cuh"

namespace nacho {

constexpr int kSv3Threads = 256;
template <typename T> struct Sv3Cfg;
#ifndef NACHO_SV3_V   // tuning override (-DNACHO_SV3_V=.. -DNACHO_SV3_MINB=..)
#define NACHO_SV3_V 16
#define NACHO_SV3_MINB 3
#endif
template <> struct Sv3Cfg<float> { static constexpr int V = NACHO_SV3_V, MINB = NACHO_SV3_MINB; };
template <> struct Sv3Cfg<double> { static constexpr int V = 8, MINB = 3; };

// positions per partition
template <typename T>
__host__ __device__ constexpr int sv3_tile() { return kSv3Threads * Sv3Cfg<T>::V; }

template <typename T>
struct KVl { int k; T v; };
template <typename T>
__device__ __forceinline__ KVl<T> kvl_op(KVl<T> a, KVl<T> b) { return KVl<T>{b.k, a.k == b.k ? a.v + b.v : b.v}; }

// Shared-memory slot of item q.  fp32: 4 pad words per 32 items, so the lane-strided writes
// (32 consecutive items) and the per-thread 128-bit reads of V consecutive items are both
// conflict-free; fp64: one pad slot per 32 (scalar accesses).
template <typename T>
__device__ __forceinline__ int sv3_slot(int q) { return sizeof(T) == 4 ? q + 4 * (q >> 5) : q + (q >> 5); }
template <typename T>
__host__ __device__ constexpr int sv3_stride32() { return sizeof(T) == 4 ? 36 : 33; }

// Gather phase: products of the warp chunk into sprod (lane-strided).  FULL: all SLOTS positions
// valid (no predicates, immediate offsets).
template <typename T, int V, bool FULL>
__device__ __forceinline__ void sv3_products(const SpmvArgs<T>& a, int64_t s, int n, int wb, int lane, T* sprod) {
  const int32_t* __restrict__ crd = a.crd + s + wb + lane;
  const T* __restrict__ val = a.val + s + wb + lane;
  const T* __restrict__ x = a.x;
  int32_t cr[V];
  T vv[V];
#pragma unroll
  for (int i = 0; i < V; ++i) {
    if (FULL || wb + 32 * i + lane < n) { cr[i] = __ldcs(crd + 32 * i); vv[i] = __ldcs(val + 32 * i); }
    else { cr[i] = 0; vv[i] = T(0); }
  }
  T* sp = sprod + sv3_slot<T>(wb) + lane;   // slot of position wb + 32i + lane
#pragma unroll
  for (int i = 0; i < V; ++i)
    if (FULL || wb + 32 * i + lane < n) sp[sv3_stride32<T>() * i] = vv[i] * ldg(x + (uint32_t)cr[i]);
}

// Segmented-scan combine: (f1, v1) . (f2, v2) = (f1 | f2, f2 ? v2 : v1 + v2).
template <typename T>
struct FV { int f; T v; };
template <typename T>
__device__ __forceinline__ FV<T> fv_op(FV<T> a, FV<T> b) { return FV<T>{a.f | b.f, b.f ? b.v : a.v + b.v}; }

// Steps 2-5 of a tile (after the products are in sprod and the row ends in send, and a barrier):
// row-start marks, segmented scan, row sums, carry.  Ends with every smem read done (barrier).
// BAR 0: __syncthreads (one tile per CTA); 1: named barrier 1 of the kSv3Threads compute threads
// (spmv7.cuh's persistent CTAs, whose producer warp does not take part).
template <int BAR>
__device__ __forceinline__ void sv3_sync() {
  if constexpr (BAR == 0) __syncthreads();
  else asm volatile("bar.sync 1, %0;" ::"r"(kSv3Threads) : "memory");
}

template <typename T, int V, bool DY, int BAR = 0>
__device__ __forceinline__ void sv3_tail(const SpmvArgs<T>& a, int64_t p, int64_t s, int n, int64_t rp0, int64_t rpE,
                                         int lim_r, bool smem_rows, const int32_t* send, T* sprod, uint8_t* mark,
                                         FV<T>* s_wagg, T* s_cin, int32_t* s_ffl) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t* __restrict__ gend = a.pos + rp0 + 1;
  auto row_end = [&](int r) -> int32_t { return smem_rows ? send[r] : (int32_t)(ldg(gend + r) - s); };
  // 2. mark the row starts inside the tile: row r + 1 starts at E[r] (empty rows mark the same item)
  for (int r = tid; r < lim_r; r += kSv3Threads) {
    const int q = row_end(r);
    if (q < n) mark[q] = 1;
  }
  sv3_sync<BAR>();

  // 3. segmented inclusive scan over my V consecutive items (in place), then across threads
  const int j0 = tid * V;
  int ffl = j0 + V;
  T acc = T(0);
  if constexpr (sizeof(T) == 4 && V % 4 == 0) {   // 128-bit smem accesses
    float4* sp4 = reinterpret_cast<float4*>(sprod + sv3_slot<T>(j0));
    const uint32_t* mw = reinterpret_cast<const uint32_t*>(mark + j0);
#pragma unroll
    for (int k = 0; k < V / 4; ++k) {
      float4 v = sp4[k];
      const uint32_t m = mw[k];
      float* vs = reinterpret_cast<float*>(&v);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int q = j0 + 4 * k + c;
        const bool f = ((m >> (8 * c)) & 0xffu) != 0 && q < n;
        const float pv = q < n ? vs[c] : 0.f;
        acc = f ? pv : acc + pv;
        vs[c] = acc;
        if (f && ffl == j0 + V) ffl = q;
      }
      sp4[k] = v;
    }
  } else {
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const int q = j0 + i;
      if (q < n) {
        const bool f = mark[q] != 0;
        T& slot = sprod[sv3_slot<T>(q)];
        acc = f ? slot : acc + slot;
        slot = acc;
        if (f && ffl == j0 + V) ffl = q;
      }
    }
  }
  FV<T> inc = FV<T>{ffl < j0 + V ? 1 : 0, acc};
#pragma unroll
  for (int dd = 1; dd < 32; dd <<= 1) {
    FV<T> u;
    u.f = __shfl_up_sync(kFull, inc.f, dd);
    u.v = __shfl_up_sync(kFull, inc.v, dd);
    if (lane >= dd) inc = fv_op(u, inc);
  }
  if (lane == 31) s_wagg[w] = inc;
  sv3_sync<BAR>();
  FV<T> pre = FV<T>{0, T(0)};
  for (int ww = 0; ww < w; ++ww) pre = fv_op(pre, s_wagg[ww]);
  FV<T> excl;
  excl.f = __shfl_up_sync(kFull, inc.f, 1);
  excl.v = __shfl_up_sync(kFull, inc.v, 1);
  excl = (lane == 0) ? pre : fv_op(pre, excl);
  s_cin[tid] = excl.v;
  s_ffl[tid] = ffl;
  sv3_sync<BAR>();

  // 4. row sums: the segmented prefix at the row's last item (+ the carry-in when that item lies in
  //    its thread's leading run); empty rows are 0.  One thread per owned row.
  auto seg_at = [&](int q) -> T {   // full in-tile segmented sum ending at item q
    const int t = q / V;
    const T v = sprod[sv3_slot<T>(q)];
    return q < s_ffl[t] ? v + s_cin[t] : v;
  };
  for (int r = tid; r < lim_r; r += kSv3Threads) {
    const int q1 = row_end(r);
    const int q0 = r > 0 ? row_end(r - 1) : 0;
    const T v = q1 > q0 ? seg_at(q1 - 1) : T(0);
    if constexpr (DY) a.y[ldg(a.outer + rp0 + r)] = v;
    else a.y[rp0 + r] = v;
  }
  // 5. CTA carry: row lim_r (cut by b_{p+1}) holds the items [E[lim_r - 1], n).  A partition that
  //    owns no row passes a (possibly zero) carry even when empty, so the carries of one row stay one
  //    contiguous run for spmv_fixup_kernel (one writer per row).
  if (tid == kSv3Threads - 1) {
    const int q0 = lim_r > 0 ? row_end(lim_r - 1) : 0;
    const bool has = rpE < a.nouter && (n > q0 || lim_r == 0);
    a.carry_row[p] = has ? rpE : -1;
    a.carry_val[p] = (has && n > q0) ? seg_at(n - 1) : T(0);
  }
}

template <typename T, bool DY>
__global__ void __launch_bounds__(kSv3Threads, Sv3Cfg<T>::MINB) spmv3_kernel(const __grid_constant__ SpmvArgs<T> a) {
  constexpr int V = Sv3Cfg<T>::V;
  constexpr int WCH = 32 * V;                  // positions per warp chunk
  constexpr int SLOTS = kSv3Threads * V;
  constexpr int W = kSv3Threads / 32;
  constexpr int ROWCAP = SLOTS + 256;          // row ends staged (more, i.e. empty rows: global reads)
  __shared__ int32_t send[ROWCAP];             // local row ends E[r] of the owned rows
  __shared__ __align__(16) T sprod[SLOTS + SLOTS / 8 + 4];   // products, then segmented sums
  __shared__ __align__(16) uint8_t mark[SLOTS + 16];   // mark[q] = 1: a row starts at item q
  __shared__ FV<T> s_wagg[W];
  __shared__ T s_cin[kSv3Threads];             // sum flowing into thread t's leading run
  __shared__ int32_t s_ffl[kSv3Threads];       // thread t's first flagged item (or its end)

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  // CTA = chunk c of partition p: a partition larger than a tile is processed as tile-sized chunks,
  // each a sub-partition cut in position space (the single-operand cut of P:1735-1737), so the
  // carries of consecutive chunks chain exactly like those of partitions
  const int64_t cid = blockIdx.x;
  const int64_t p = a.chunks == 1 ? cid : cid / a.chunks;
  const int c = (int)(cid - p * a.chunks);
  const int64_t sp = ldg(a.ppos + p), ep = ldg(a.ppos + p + 1);
  const int64_t rp0p = ldg(a.prow + p), rpEp = ldg(a.prow + p + 1);
  const int64_t s = sp + (int64_t)c * SLOTS;
  if (c > 0 && s >= ep) {   // past the partition: a zero carry keeps row rpEp's run contiguous
    if (tid == 0) {
      a.carry_row[cid] = rpEp < a.nouter ? rpEp : -1;
      a.carry_val[cid] = T(0);
    }
    return;
  }
  const int64_t e = ep - s < SLOTS ? ep : s + SLOTS;
  int64_t rp0 = rp0p, rpE = rpEp;
  if (a.chunks > 1) {   // rows containing the chunk's cuts: 32-ary warp searches over the partition's rows
    __shared__ int64_t s_rows[2];
    const int64_t hi = rpEp < a.nouter ? rpEp : a.nouter;
    if (w < 2) {
      const int64_t q = w == 0 ? s : e;
      const bool need = w == 0 ? c > 0 : e < ep;
      int64_t r = w == 0 ? rp0p : rpEp;
      if (need) r = warp_highest_true(rp0p, hi, [&](int64_t x) { return ldg(a.pos + x) <= q; });
      if (lane == 0) s_rows[w] = r;
    }
    __syncthreads();
    rp0 = s_rows[0];
    rpE = s_rows[1];
  }
  const int n = (int)(e - s);  const int wb = w * WCH;                      // warp chunk [wb, wb + WCH) in local positions
  // owned rows [0, lim_r) (R7): local ends E[r] = pos[rp0 + r + 1] - s, in [0, n]
  const int lim_r = (int)((rpE < a.nouter ? rpE : a.nouter) - rp0);
  const bool smem_rows = lim_r <= ROWCAP;
  const int64_t* __restrict__ gend = a.pos + rp0 + 1;

  // 0. clear the row-start marks (V bytes per thread)
  if constexpr (V == 16) reinterpret_cast<uint4*>(mark)[tid] = make_uint4(0, 0, 0, 0);
  else if constexpr (V == 8) reinterpret_cast<uint2*>(mark)[tid] = make_uint2(0, 0);
  else for (int i = 0; i < V; ++i) mark[tid * V + i] = 0;
  // 1. products (crd / val read lane-strided: 128 contiguous bytes per warp instruction; the x
  //    gathers of a long row touch a few lines instead of 32), staged row ends
  if (n == SLOTS) sv3_products<T, V, true>(a, s, n, wb, lane, sprod);
  else sv3_products<T, V, false>(a, s, n, wb, lane, sprod);
  if (smem_rows)
    for (int i = tid; i < lim_r; i += kSv3Threads) send[i] = (int32_t)(ldg(gend + i) - s);
  __syncthreads();
  sv3_tail<T, V, DY>(a, cid, s, n, rp0, rpE, lim_r, smem_rows, send, sprod, mark, s_wagg, s_cin, s_ffl);
}

}  // namespace nacho
