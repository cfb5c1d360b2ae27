// spmm.cuh -- partitioned CSR x skinny-dense SpMM C = A B, loop order i -> j -> k.
#pragma once
#include "common.cuh"

namespace nacho {

template <typename T>
struct SpmmArgs {
  const int64_t* pos;
  const int32_t* crd;
  const T* val;
  int64_t nrows;
  const T* B;
  int64_t ldb;
  int32_t nb;
  T* C;
  int64_t ldc;
  int32_t P;           // carries (the fix-up's count): partitions x chunks
  int32_t chunks;      // spmm64: CTAs per partition (tile-sized chunks of larger partitions)
  const int64_t* ppos;
  const int64_t* prow;
  int64_t* carry_row;  // [P]
  T* carry_val;        // [P * nb]
};

template <typename T, int CPL>
struct Vec { T v[CPL]; };

template <typename T, int CPL, bool VEC>
__device__ __forceinline__ void load_brow(const SpmmArgs<T>& a, int64_t c, int lane, T (&b)[CPL]) {
  const int c0 = lane * CPL;
  const T* src = a.B + c * a.ldb + c0;
  if (VEC && c0 + CPL <= a.nb) {
    if constexpr (CPL * sizeof(T) == 8) {
      const float2 t = __ldg(reinterpret_cast<const float2*>(src));
      const T* tt = reinterpret_cast<const T*>(&t);
#pragma unroll
      for (int j = 0; j < CPL; ++j) b[j] = tt[j];
      return;
    } else if constexpr (CPL * sizeof(T) == 16) {
      const float4 t = __ldg(reinterpret_cast<const float4*>(src));
      const T* tt = reinterpret_cast<const T*>(&t);
#pragma unroll
      for (int j = 0; j < CPL; ++j) b[j] = tt[j];
      return;
    }
  }
#pragma unroll
  for (int j = 0; j < CPL; ++j) b[j] = (c0 + j < a.nb) ? __ldg(src + j) : T(0);
}

template <typename T, int CPL>
__device__ __forceinline__ void store_crow(const SpmmArgs<T>& a, int64_t r, int lane, const T (&v)[CPL]) {
  const int c0 = lane * CPL;
  T* dst = a.C + r * a.ldc + c0;
#pragma unroll
  for (int j = 0; j < CPL; ++j) if (c0 + j < a.nb) dst[j] = v[j];
}

// CTA per partition, WARPS warps; warp w walks WITEMS consecutive positions of the chunk.  Lane l
// owns the columns [l*CPL, (l+1)*CPL) of the row accumulators; one B-row gather per non-zero is a
// single coalesced nb*sizeof(T)-byte request.  Row ownership, heads, tails and carries follow
// spmv_kernel with warps in place of threads (R6: k is never cut, so A's cuts are the cuts).
template <typename T, int CPL, bool VEC, int WARPS, int WITEMS>
__global__ void __launch_bounds__(WARPS * 32) spmm_kernel(SpmmArgs<T> a) {
  constexpr int TILE = WARPS * WITEMS;
  constexpr int NBMAX = 32 * CPL;
  __shared__ T s_tail[WARPS][NBMAX];
  __shared__ int64_t s_tkey[WARPS];
  __shared__ T s_carry[NBMAX];
  __shared__ int64_t s_ckey;

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int p = blockIdx.x;
  const int64_t s = ldg(a.ppos + p), e = ldg(a.ppos + p + 1);
  const int64_t rp0 = ldg(a.prow + p), rpE = ldg(a.prow + p + 1);
  if (tid == 0) s_ckey = rp0;
  for (int c = tid; c < NBMAX; c += WARPS * 32) s_carry[c] = T(0);

  for (int64_t cs = s;; cs += TILE) {
    const int64_t ce = (e - cs < TILE) ? e : cs + TILE;
    const int n = (int)(ce - cs);
    __syncthreads();
    const int i0 = w * WITEMS;
    const bool active = i0 < n || w == 0;
    const int cnt = active ? max(0, min(WITEMS, n - i0)) : 0;
    const int64_t at = cs + i0, bt = at + cnt;

    T acc[CPL], hv[CPL];
#pragma unroll
    for (int j = 0; j < CPL; ++j) { acc[j] = T(0); hv[j] = T(0); }
    bool head = true, head_done = false;
    int64_t head_row = 0, rp = 0;
    if (active) {
      if (w == 0 && cs == s) rp = rp0;
      else {
        int64_t lo = rp0, hi = rpE < a.nrows ? rpE : a.nrows;
        lo = warp_highest_true(lo, hi, [&](int64_t m) { return ldg(a.pos + m) <= at; });
        rp = lo;
      }
      int64_t next_end = rp < a.nrows ? ldg(a.pos + rp + 1) : INT64_MAX;
      for (int base = 0; base < cnt; base += 32) {
        const int nn = min(32, cnt - base);
        int32_t mc = 0;
        T mv = T(0);
        if (lane < nn) { mc = ldg(a.crd + at + base + lane); mv = ldg(a.val + at + base + lane); }
        constexpr int U = CPL <= 2 ? 8 : 4;  // B rows in flight per warp
        for (int i = 0; i < nn; i += U) {
          T bb[U][CPL];
          T vv[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int32_t c = __shfl_sync(kFull, mc, (i + u) & 31);
            vv[u] = __shfl_sync(kFull, mv, (i + u) & 31);
            if (i + u < nn) load_brow<T, CPL, VEC>(a, c, lane, bb[u]);
          }
#pragma unroll
          for (int u = 0; u < U; ++u) {
            if (i + u < nn) {
              const int64_t q = at + base + i + u;
              while (next_end <= q) {
                if (head) {
                  head_done = true; head_row = rp; head = false;
#pragma unroll
                  for (int j = 0; j < CPL; ++j) hv[j] = acc[j];
                } else store_crow<T, CPL>(a, rp, lane, acc);
#pragma unroll
                for (int j = 0; j < CPL; ++j) acc[j] = T(0);
                ++rp;
                next_end = ldg(a.pos + rp + 1);
              }
#pragma unroll
              for (int j = 0; j < CPL; ++j) acc[j] += vv[u] * bb[u][j];
            }
          }
        }
      }
      while (rp < a.nrows && next_end <= bt) {
        if (head) {
          head_done = true; head_row = rp; head = false;
#pragma unroll
          for (int j = 0; j < CPL; ++j) hv[j] = acc[j];
        } else store_crow<T, CPL>(a, rp, lane, acc);
#pragma unroll
        for (int j = 0; j < CPL; ++j) acc[j] = T(0);
        ++rp;
        next_end = rp < a.nrows ? ldg(a.pos + rp + 1) : INT64_MAX;
      }
    }
    // ---- tails to shared memory
    if (lane == 0) s_tkey[w] = active ? rp : INT64_MAX;
#pragma unroll
    for (int j = 0; j < CPL; ++j) s_tail[w][lane * CPL + j] = acc[j];
    __syncthreads();
    // carry into warp w's head row: tails of the run of preceding warps with that key (+ chunk carry)
    if (head_done) {
      T c[CPL];
#pragma unroll
      for (int j = 0; j < CPL; ++j) c[j] = T(0);
      int ww = w - 1;
      for (; ww >= 0 && s_tkey[ww] == head_row; --ww)
#pragma unroll
        for (int j = 0; j < CPL; ++j) c[j] += s_tail[ww][lane * CPL + j];
      if (ww < 0 && s_ckey == head_row)
#pragma unroll
        for (int j = 0; j < CPL; ++j) c[j] += s_carry[lane * CPL + j];
#pragma unroll
      for (int j = 0; j < CPL; ++j) c[j] += hv[j];
      store_crow<T, CPL>(a, head_row, lane, c);
    }
    // new chunk carry: last active warp's tail + preceding run (+ old carry)
    const int lastw = n > 0 ? (n - 1) / WITEMS : 0;
    T nc[CPL];
    const int64_t key = s_tkey[lastw];
    if (w == 0) {
#pragma unroll
      for (int j = 0; j < CPL; ++j) nc[j] = T(0);
      int ww = lastw;
      for (; ww >= 0 && s_tkey[ww] == key; --ww)
#pragma unroll
        for (int j = 0; j < CPL; ++j) nc[j] += s_tail[ww][lane * CPL + j];
      if (ww < 0 && s_ckey == key)
#pragma unroll
        for (int j = 0; j < CPL; ++j) nc[j] += s_carry[lane * CPL + j];
    }
    __syncthreads();
    if (w == 0) {
#pragma unroll
      for (int j = 0; j < CPL; ++j) s_carry[lane * CPL + j] = nc[j];
      if (lane == 0) s_ckey = key;
    }
    if (ce >= e) break;
  }
  __syncthreads();
  const bool has = s_ckey < a.nrows && s_ckey == rpE;
  if (tid == 0) a.carry_row[p] = has ? s_ckey : -1;
  for (int c = tid; c < a.nb; c += WARPS * 32) a.carry_val[(int64_t)p * a.nb + c] = has ? s_carry[c] : T(0);
}

// nb == 64 fp32 fast path: eight-lane groups, each lane owns 8 columns (two float4), so a warp
// instruction advances four nonzeros (one per group) instead of one.  Group g of the CTA walks the
// 32 consecutive positions [s + 32g, s + 32g + 32); heads, tails and the CTA carry combine across
// the 32 groups in position order exactly like spmm_kernel's warps.
constexpr int kSm2Groups = 32;       // 8-lane groups per CTA (256 threads)
constexpr int kSm2Items = 32;        // positions per group
constexpr int kSm2Tile = kSm2Groups * kSm2Items;
#ifndef NACHO_SM2_BATCH   // nonzeros whose B rows a lane group loads before using them (registers: 8 per nonzero)
#define NACHO_SM2_BATCH 8  // C4: batch 8 / 2 CTAs per SM 65.0 ms, batch 4 / 3 CTAs 67.1, 4 / 4 72.1, 2 / 5 84.5
#define NACHO_SM2_MINB 2
#endif
constexpr int kSm2Batch = NACHO_SM2_BATCH;

template <bool CHUNKED>
__global__ void __launch_bounds__(256, NACHO_SM2_MINB) spmm64_kernel(const __grid_constant__ SpmmArgs<float> a) {
  __shared__ float4 s_tail[kSm2Groups][16];   // 64 floats per group
  __shared__ int64_t s_tkey[kSm2Groups];
  const int tid = threadIdx.x, g = tid >> 3, gl = tid & 7;
  const unsigned gmask = 0xffu << (tid & 24);
  // CTA = chunk c of partition p (partitions larger than a tile run as tile-sized chunks, cut in
  // position space; their carries chain like those of partitions)
  const int64_t p = blockIdx.x;   // carry index
  const int64_t pp = CHUNKED ? p / a.chunks : p;
  const int c = (int)(p - pp * a.chunks);
  const int64_t sp = ldg(a.ppos + pp), ep = ldg(a.ppos + pp + 1);
  const int64_t rp0p = ldg(a.prow + pp), rpEp = ldg(a.prow + pp + 1);
  const int64_t s = sp + (int64_t)c * kSm2Tile;
  if (CHUNKED && c > 0 && s >= ep) {   // past the partition: a zero carry keeps row rpEp's run contiguous
    if (tid == 0) a.carry_row[p] = rpEp < a.nrows ? rpEp : -1;
    if (tid < 16) reinterpret_cast<float4*>(a.carry_val + p * 64)[tid] = make_float4(0, 0, 0, 0);
    return;
  }
  const int64_t e = ep - s < kSm2Tile ? ep : s + kSm2Tile;
  int64_t rp0 = rp0p, rpE = rpEp;
  if (CHUNKED) {
    __shared__ int64_t s_rows[2];
    const int w = tid >> 5, lane = tid & 31;
    const int64_t hi = rpEp < a.nrows ? rpEp : a.nrows;
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
  const int i0 = g * kSm2Items;
  const int n = (int)(e - s);
  const bool active = i0 < n || g == 0;
  const int cnt = active ? max(0, min(kSm2Items, n - i0)) : 0;
  const int64_t at = s + i0, bt = at + cnt;
  float4 acc0 = make_float4(0, 0, 0, 0), acc1 = acc0, hv0 = acc0, hv1 = acc0;
  bool head = true, head_done = false;
  int64_t head_row = 0, rp = 0;
  auto store_row = [&](int64_t r, const float4& u0, const float4& u1) {
    float4* dst = reinterpret_cast<float4*>(a.C + r * a.ldc) + 2 * gl;
    dst[0] = u0;
    dst[1] = u1;
  };
  if (active) {
    if (g == 0) {
      rp = rp0;
    } else {
      int64_t lo = rp0, hi = rpE < a.nrows ? rpE : a.nrows;
      while (lo < hi) {
        const int64_t m = lo + ((hi - lo + 1) >> 1);
        if (ldg(a.pos + m) <= at) lo = m; else hi = m - 1;
      }
      rp = lo;
    }
    int64_t next_end = rp < a.nrows ? ldg(a.pos + rp + 1) : INT64_MAX;
    // the group's positions: lane gl holds positions gl, gl+8, gl+16, gl+24
    int32_t mc[4];
    float mv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = gl + 8 * u;
      mc[u] = j < cnt ? ldg(a.crd + at + j) : 0;
      mv[u] = j < cnt ? ldg(a.val + at + j) : 0.f;
    }
#pragma unroll
    for (int ib = 0; ib < kSm2Items / kSm2Batch; ++ib) {   // batches of positions (static register indices)
      if (kSm2Batch * ib >= cnt) break;
      float4 b0[kSm2Batch], b1[kSm2Batch];
      float vv[kSm2Batch];
#pragma unroll
      for (int u = 0; u < kSm2Batch; ++u) {
        const int j = kSm2Batch * ib + u;
        const int32_t c = __shfl_sync(gmask, mc[j >> 3], j & 7, 8);
        vv[u] = __shfl_sync(gmask, mv[j >> 3], j & 7, 8);
        if (j < cnt) {
          const float4* src = reinterpret_cast<const float4*>(a.B + (int64_t)c * a.ldb) + 2 * gl;
          b0[u] = __ldg(src);
          b1[u] = __ldg(src + 1);
        }
      }
#pragma unroll
      for (int u = 0; u < kSm2Batch; ++u) {
        const int j = kSm2Batch * ib + u;
        if (j < cnt) {
          const int64_t q = at + j;
          while (next_end <= q) {
            if (head) { head_done = true; head_row = rp; hv0 = acc0; hv1 = acc1; head = false; }
            else store_row(rp, acc0, acc1);
            acc0 = make_float4(0, 0, 0, 0); acc1 = acc0;
            ++rp;
            next_end = ldg(a.pos + rp + 1);
          }
          const float v = vv[u];
          acc0.x += v * b0[u].x; acc0.y += v * b0[u].y; acc0.z += v * b0[u].z; acc0.w += v * b0[u].w;
          acc1.x += v * b1[u].x; acc1.y += v * b1[u].y; acc1.z += v * b1[u].z; acc1.w += v * b1[u].w;
        }
      }
    }
    while (rp < a.nrows && next_end <= bt) {
      if (head) { head_done = true; head_row = rp; hv0 = acc0; hv1 = acc1; head = false; }
      else store_row(rp, acc0, acc1);
      acc0 = make_float4(0, 0, 0, 0); acc1 = acc0;
      ++rp;
      next_end = rp < a.nrows ? ldg(a.pos + rp + 1) : INT64_MAX;
    }
  }
  if (gl == 0) s_tkey[g] = active ? rp : INT64_MAX;
  s_tail[g][2 * gl] = acc0;
  s_tail[g][2 * gl + 1] = acc1;
  __syncthreads();
  auto add4 = [](float4& x, const float4& y) { x.x += y.x; x.y += y.y; x.z += y.z; x.w += y.w; };
  if (head_done) {  // carry into my head row: tails of the run of preceding groups with that key
    float4 c0 = hv0, c1 = hv1;
    for (int gg = g - 1; gg >= 0 && s_tkey[gg] == head_row; --gg) {
      add4(c0, s_tail[gg][2 * gl]);
      add4(c1, s_tail[gg][2 * gl + 1]);
    }
    store_row(head_row, c0, c1);
  }
  // CTA carry: the last active group's tail plus the run of groups before it with the same key
  const int lastg = n > 0 ? (n - 1) / kSm2Items : 0;
  if (g == lastg) {
    const int64_t key = s_tkey[lastg];
    float4 c0 = acc0, c1 = acc1;
    for (int gg = lastg - 1; gg >= 0 && s_tkey[gg] == key; --gg) {
      add4(c0, s_tail[gg][2 * gl]);
      add4(c1, s_tail[gg][2 * gl + 1]);
    }
    const bool has = key < a.nrows && key == rpE;
    if (gl == 0) a.carry_row[p] = has ? key : -1;
    float4* dst = reinterpret_cast<float4*>(a.carry_val + (int64_t)p * 64) + 2 * gl;
    dst[0] = has ? c0 : make_float4(0, 0, 0, 0);
    dst[1] = has ? c1 : make_float4(0, 0, 0, 0);
  }
}

template <typename T>
__global__ void spmm_fixup_kernel(SpmmArgs<T> a) {
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
    if (end - start >= 64) {
      // long run (a dense row's carries): lanes stride over the partitions, each summing 8 columns at
      // a time, then a shuffle tree per column -- a fixed order, so deterministic for a given P
      for (int c0 = 0; c0 < a.nb; c0 += 8) {
        T acc[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) acc[u] = T(0);
        for (int64_t j = start + lane; j <= end; j += 32) {
          const T* cv = a.carry_val + j * a.nb + c0;
#pragma unroll
          for (int u = 0; u < 8; ++u) if (c0 + u < a.nb) acc[u] += cv[u];
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
#pragma unroll
          for (int d = 16; d > 0; d >>= 1) acc[u] += __shfl_xor_sync(kFull, acc[u], d);
        }
        if (lane < 8 && c0 + lane < a.nb) {
          T v = acc[0];
#pragma unroll
          for (int u = 1; u < 8; ++u) v = lane == u ? acc[u] : v;
          a.C[row * a.ldc + c0 + lane] += v;
        }
      }
      continue;
    }
    for (int c = lane; c < a.nb; c += 32) {   // four independent partial sums per lane (ILP)
      T s0 = T(0), s1 = T(0), s2 = T(0), s3 = T(0);
      int64_t j = start;
      for (; j + 3 <= end; j += 4) {
        s0 += a.carry_val[j * a.nb + c];
        s1 += a.carry_val[(j + 1) * a.nb + c];
        s2 += a.carry_val[(j + 2) * a.nb + c];
        s3 += a.carry_val[(j + 3) * a.nb + c];
      }
      for (; j <= end; ++j) s0 += a.carry_val[j * a.nb + c];
      a.C[row * a.ldc + c] += (s0 + s1) + (s2 + s3);
    }
  }
}

}  // namespace nacho
