// partition.cuh -- the partitioning kernel.
#pragma once
#include "common.cuh"

namespace nacho {

// One warp per boundary p in [0, P]: Q_p = floor(p Q* / P), b_0 = origin, b_P = end
// (reading R1), interior boundaries by FindPartition (Alg. 1).  The P+1 searches are independent
// ("computed independently, and thus in parallel").
template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32) partition_kernel(const __grid_constant__ OpsArg a, PartsArg out, int64_t qstar) {
  const int64_t p = (int64_t)blockIdx.x * WARPS + (threadIdx.x >> 5);
  if (p > out.P) return;  // warp-uniform
  Boundary b;
  if (p == 0) set_origin(a, b);
  else if (p == out.P) set_end(a, b);
  else b = warp_find_boundary(a, query_of(qstar, out.P, p), 0, a.op[0].nouter);
  const int lane = threadIdx.x & 31;
  if (lane == 0) {
    out.query[p] = query_of(qstar, out.P, p);
    out.row[p] = b.row;
    out.row_pos[p] = b.row_pos;
    out.col[p] = b.col;
  }
  if (lane < a.k) {
    int64_t v = 0;
#pragma unroll
    for (int o = 0; o < NACHO_MAX_K; ++o) if (o == lane) v = b.pos[o];
    out.pos[p * a.k + lane] = v;
  }
}

}  // namespace nacho
