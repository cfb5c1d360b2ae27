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
  int32_t P;
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
        for (int i = 0; i < nn; i += 4) {
          T bb[4][CPL];
          T vv[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int32_t c = __shfl_sync(kFull, mc, (i + u) & 31);
            vv[u] = __shfl_sync(kFull, mv, (i + u) & 31);
            if (i + u < nn) load_brow<T, CPL, VEC>(a, c, lane, bb[u]);
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
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
    int64_t start = end;
    for (;;) {
      const int64_t j = start - 1 - lane;
      const bool match = j >= 0 && a.carry_row[j] == row;
      const unsigned mm = __ballot_sync(kFull, match);
      if (mm == kFull) { start -= 32; continue; }
      start -= __ffs(~mm) - 1;
      break;
    }
    for (int c = lane; c < a.nb; c += 32) {
      T sum = T(0);
      for (int64_t j = start; j <= end; ++j) sum += a.carry_val[j * a.nb + c];
      a.C[row * a.ldc + c] += sum;
    }
  }
}

}  // namespace nacho
