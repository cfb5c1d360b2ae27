// spadd.cuh -- k-way union SpAdd Z = sum_o A_o over partitions:
// assembly (count) -> exclusive prefix sum -> compute (fill), the paper's Fig. 7a.
#pragma once
#include "common.cuh"

namespace nacho {

template <typename T>
struct SpaddArgs {
  OpsArg ops;
  PartsArg parts;
  int64_t qstar;
  int64_t* part_cnt;        // count pass: [P]
  const int64_t* part_off;  // fill pass:  [P+1]
  int64_t* z_pos;
  int32_t* z_crd;
  T* z_val;
};

template <int THREADS>
struct SpaddShared {
  Boundary B, E, PE;        // chunk start, chunk end, partition end
  int off[NACHO_MAX_K + 1]; // operand offsets inside the staged chunk
  int64_t red[THREADS / 32 + 1];
  uint64_t redu[THREADS / 32 + 1];
};

// Inclusive max-scan of n (<= THREADS*SPT) uint64 values in shared memory, in place.
template <int THREADS, int SPT>
__device__ __forceinline__ void block_max_scan(uint64_t* v, int n, uint64_t* red) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  uint64_t loc[SPT];
  uint64_t run = 0;
#pragma unroll
  for (int s = 0; s < SPT; ++s) {
    const int j = tid * SPT + s;
    const uint64_t x = j < n ? v[j] : 0;
    run = x > run ? x : run;
    loc[s] = run;
  }
  uint64_t inc = run;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint64_t u = __shfl_up_sync(kFull, inc, d);
    if (lane >= d && u > inc) inc = u;
  }
  if (lane == 31) red[w] = inc;
  __syncthreads();
  uint64_t pre = 0;
  for (int ww = 0; ww < w; ++ww) pre = red[ww] > pre ? red[ww] : pre;
  uint64_t ex = __shfl_up_sync(kFull, inc, 1);
  if (lane == 0) ex = 0;
  pre = ex > pre ? ex : pre;
#pragma unroll
  for (int s = 0; s < SPT; ++s) {
    const int j = tid * SPT + s;
    if (j < n) v[j] = loc[s] > pre ? loc[s] : pre;
  }
  __syncthreads();
}

// One merge-path stage of the union (P:314 merge path, generalised in the paper to coordinate
// space): Z = X (u) Y over sorted unique (row, col) keys; equal keys are emitted once with the
// value X + Y (left fold: X carries operands 0..o-1, Y is operand o -- reading R9).  Thread t takes
// the SPT merged steps starting at diagonal t*SPT; a step that takes Y[j] equal to the previous X
// is skipped (it was folded into that X).  Returns |Z|.
template <typename T, bool VALS, int THREADS, int SPT>
__device__ __forceinline__ int merge_stage(const uint64_t* __restrict__ Xk, const T* __restrict__ Xv, int nx,
                                           const uint64_t* __restrict__ Yk, const T* __restrict__ Yv, int ny,
                                           uint64_t* __restrict__ Zk, T* __restrict__ Zv, int64_t* red) {
  const int tid = threadIdx.x;
  const int total = nx + ny;
  const int d0 = min(total, tid * SPT);
  const int d1 = min(total, d0 + SPT);
  int lo = max(0, d0 - ny), hi = min(d0, nx);
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (Xk[mid] <= Yk[d0 - 1 - mid]) lo = mid + 1; else hi = mid;
  }
  int i = lo, j = d0 - lo;
  uint64_t ok[SPT];
  T ov[SPT];
  bool emit[SPT];
  int cnt = 0;
#pragma unroll
  for (int s = 0; s < SPT; ++s) {
    emit[s] = false;
    if (d0 + s < d1) {
      const bool takeX = i < nx && (j >= ny || Xk[i] <= Yk[j]);
      if (takeX) {
        const uint64_t key = Xk[i];
        T v = T(0);
        if (VALS) v = Xv[i];
        if (j < ny && Yk[j] == key) { if (VALS) v = v + Yv[j]; }
        ok[s] = key; ov[s] = v; emit[s] = true; ++i;
      } else {
        const uint64_t key = Yk[j];
        if (!(i > 0 && Xk[i - 1] == key)) { ok[s] = key; if (VALS) ov[s] = Yv[j]; emit[s] = true; }
        ++j;
      }
      cnt += emit[s] ? 1 : 0;
    }
  }
  int64_t tot;
  int64_t idx = block_excl_sum<THREADS, int64_t>((int64_t)cnt, red, &tot);
#pragma unroll
  for (int s = 0; s < SPT; ++s) {
    if (emit[s]) { Zk[idx] = ok[s]; if (VALS) Zv[idx] = ov[s]; ++idx; }
  }
  __syncthreads();
  return (int)tot;
}

template <typename T>
__device__ __forceinline__ void load_boundary(const PartsArg& P, int k, int64_t p, Boundary& b) {
  b.row = P.row[p];
  b.row_pos = P.row_pos[p];
  b.col = P.col[p];
#pragma unroll
  for (int o = 0; o < NACHO_MAX_K; ++o) if (o < k) b.pos[o] = P.pos[p * k + o];
}

// CTA per partition.  FILL = false: assembly -- the union size of the partition.
// FILL = true: compute -- writes Z.crd / Z.val at part_off[p] and Z.pos[r+1] for the rows the
// partition owns (rows [b_p.row, b_{p+1}.row - 1], the guarded single writer of Listing 8, R7).
// A partition holding more than TILE entries is processed in chunks whose ends are found by the
// same FindPartition search (the hierarchy of P:1089-1093 applied inside the partition).
template <typename T, bool FILL, int THREADS, int TILE>
__global__ void __launch_bounds__(THREADS, 2) spadd_kernel(const __grid_constant__ SpaddArgs<T> a) {
  constexpr int SPT = TILE / THREADS;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SpaddShared<THREADS>& sh = *reinterpret_cast<SpaddShared<THREADS>*>(smem_raw);
  uint64_t* K0 = reinterpret_cast<uint64_t*>(smem_raw + ((sizeof(SpaddShared<THREADS>) + 15) & ~size_t(15)));
  uint64_t* K1 = K0 + TILE;
  uint64_t* K2 = K1 + TILE;
  T* V0 = reinterpret_cast<T*>(K2 + TILE);
  T* V1 = V0 + (FILL ? TILE : 0);
  T* V2 = V1 + (FILL ? TILE : 0);

  const int tid = threadIdx.x;
  const int k = a.ops.k;
  const int64_t p = blockIdx.x;
  const int64_t M = a.ops.nrows;

  if (tid == 0) {
    load_boundary<T>(a.parts, k, p, sh.B);
    load_boundary<T>(a.parts, k, p + 1, sh.PE);
  }
  __syncthreads();
  int64_t cPE = 0, cB = 0;
  for (int o = 0; o < k; ++o) { cPE += sh.PE.pos[o]; cB += sh.B.pos[o]; }
  int64_t out_off = FILL ? a.part_off[p] : 0;
  int64_t count = 0;
  if (FILL && p == 0 && tid == 0) a.z_pos[0] = 0;

  for (;;) {
    // ---- chunk end E (partition end, or the FindPartition cut TILE-(k-1) entries further)
    const bool last = (cPE - cB) <= TILE;
    if (last) {
      if (tid == 0) sh.E = sh.PE;
    } else if (tid < 32) {
      const Boundary f = warp_find_boundary(a.ops, cB + (TILE - (k - 1)), sh.B.row_pos, sh.PE.row_pos);
      if (tid == 0) sh.E = f;
    }
    __syncthreads();
    if (tid == 0) {
      sh.off[0] = 0;
      for (int o = 0; o < k; ++o) sh.off[o + 1] = sh.off[o] + (int)(sh.E.pos[o] - sh.B.pos[o]);
    }
    __syncthreads();
    const int n = sh.off[k];
    const int64_t Brow = sh.B.row, Erow = sh.E.row;

    // ---- 1. stage crd (and val) of every operand's contiguous range into K0/V0;
    //         row marks (o << 32 | local row) default to the chunk's first row
    for (int o = 0; o < k; ++o) {
      const int64_t base = sh.B.pos[o];
      const int oo = sh.off[o], no = sh.off[o + 1] - oo;
      const int32_t* crd = a.ops.op[o].crd;
      const T* val = reinterpret_cast<const T*>(a.ops.op[o].val);
      for (int j = tid; j < no; j += THREADS) {
        K0[oo + j] = (uint64_t)(uint32_t)ldg(crd + base + j);
        if (FILL) V0[oo + j] = ldg(val + base + j);
        K1[oo + j] = (uint64_t)o << 32;
      }
    }
    __syncthreads();
    // ---- 2. row id of every entry: scatter the row starts that fall inside the range, max-scan
    const int64_t r_hi = Erow < M - 1 ? Erow : M - 1;
    for (int64_t r = Brow + 1 + tid; r <= r_hi; r += THREADS) {
      for (int o = 0; o < k; ++o) {
        const int64_t ps = ldg(a.ops.op[o].pos + r);
        const int64_t b0 = sh.B.pos[o];
        if (ps >= b0 && ps < sh.E.pos[o] && ldg(a.ops.op[o].pos + r + 1) > ps)
          K1[sh.off[o] + (int)(ps - b0)] = ((uint64_t)o << 32) | (uint64_t)(r - Brow);
      }
    }
    __syncthreads();
    block_max_scan<THREADS, SPT>(K1, n, sh.redu);
    for (int j = tid; j < n; j += THREADS) K0[j] |= (K1[j] & 0xffffffffull) << 32;
    __syncthreads();

    // ---- 3. union by k-1 merge-path stages (operand order = fold order)
    const uint64_t* Uk = K0;
    const T* Uv = V0;
    int nu = sh.off[1];
    uint64_t* Dk = K1;
    T* Dv = V1;
    for (int o = 1; o < k; ++o) {
      const int oo = sh.off[o];
      nu = merge_stage<T, FILL, THREADS, SPT>(Uk, Uv, nu, K0 + oo, V0 + oo, sh.off[o + 1] - oo, Dk, Dv, sh.red);
      Uk = Dk; Uv = Dv;
      Dk = (Dk == K1) ? K2 : K1;
      Dv = (Dv == V1) ? V2 : V1;
    }

    // ---- 4. outputs
    if (FILL) {
      for (int j = tid; j < nu; j += THREADS) {
        a.z_crd[out_off + j] = (int32_t)(Uk[j] & 0xffffffffull);
        a.z_val[out_off + j] = Uv[j];
      }
      const int64_t own_hi = (Erow < M ? Erow : M) - 1;
      for (int64_t r = Brow + tid; r <= own_hi; r += THREADS) {
        const uint64_t key = (uint64_t)(r - Brow + 1) << 32;  // first key of the next row
        int lo = 0, hi = nu;
        while (lo < hi) { const int m = (lo + hi) >> 1; if (Uk[m] < key) lo = m + 1; else hi = m; }
        a.z_pos[r + 1] = out_off + lo;
      }
    }
    out_off += nu;
    count += nu;
    if (last) break;
    int64_t cE = 0;
    for (int o = 0; o < k; ++o) cE += sh.E.pos[o];
    cB = cE;
    __syncthreads();
    if (tid == 0) sh.B = sh.E;
    __syncthreads();
  }
  if (!FILL && tid == 0) a.part_cnt[p] = count;
}

// Exclusive prefix sum of the P partition counts -> part_off[0..P] (Merrill's scan is
// cited at P:1475).  One CTA walks the array in tiles of THREADS*8 with a running carry.
template <int THREADS>
__global__ void __launch_bounds__(THREADS) scan_counts_kernel(const int64_t* __restrict__ cnt, int64_t n,
                                                              int64_t* __restrict__ off) {
  constexpr int IT = 16;   // 16 K counts in one round (P of a 2.6e7-entry SpAdd)
  __shared__ int64_t red[THREADS / 32 + 1];
  int64_t carry = 0;
  for (int64_t base = 0; base < n; base += (int64_t)THREADS * IT) {
    int64_t v[IT];
    int64_t s = 0;
#pragma unroll
    for (int i = 0; i < IT; ++i) {
      const int64_t j = base + (int64_t)threadIdx.x * IT + i;
      v[i] = j < n ? cnt[j] : 0;
      s += v[i];
    }
    int64_t tot;
    int64_t ex = block_excl_sum<THREADS, int64_t>(s, red, &tot) + carry;
#pragma unroll
    for (int i = 0; i < IT; ++i) {
      const int64_t j = base + (int64_t)threadIdx.x * IT + i;
      if (j < n) off[j] = ex;
      ex += v[i];
    }
    carry += tot;
  }
  if (threadIdx.x == 0) off[n] = carry;
}

}  // namespace nacho
