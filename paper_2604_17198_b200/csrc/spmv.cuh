// spmv.cuh -- partitioned CSR / DCSR SpMV y = A x and its carry fix-up.
#pragma once
#include "common.cuh"

namespace nacho {

template <typename T>
struct SpmvArgs {
  const int64_t* pos;
  const int32_t* crd;
  const T* val;
  const int32_t* outer;   // DCSR row coordinates (only used for a dense y)
  int64_t nouter;
  int64_t ncols;
  const T* x;
  T* y;
  int32_t dense_y;        // DCSR: write y[outer[rp]] instead of y[rp]
  int32_t P;              // carries (the fix-up's count): partitions x chunks
  int32_t chunks;         // spmv3: CTAs per partition (tile-sized chunks of larger partitions)
  const int64_t* ppos;    // parts.pos   (k == 1): [P+1]
  const int64_t* prow;    // parts.row_pos:        [P+1]
  int64_t* carry_row;     // [P] outer position receiving partition p's carry (-1: none)
  T* carry_val;           // [P]
};

template <typename T>
__device__ __forceinline__ int64_t y_index(const SpmvArgs<T>& a, int64_t rp) {
  return (a.dense_y && a.outer) ? (int64_t)ldg(a.outer + rp) : rp;
}

// Adds every partition's carry to the row it belongs to, in partition order (deterministic for a
// given P).  The partitions whose carries go to one row form a contiguous run; the warp holding the
// run's last carry sums the run (lanes strided, tree reduction) and adds it to y.
template <typename T>
__global__ void spmv_fixup_kernel(SpmvArgs<T> a) {
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
    T sum = T(0);
    for (int64_t j = start + lane; j <= end; j += 32) sum += a.carry_val[j];
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) sum += __shfl_xor_sync(kFull, sum, d);
    if (lane == 0) a.y[y_index(a, row)] += sum;
  }
}

}  // namespace nacho
