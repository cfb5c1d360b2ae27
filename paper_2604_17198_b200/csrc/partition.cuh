// partition.cuh -- the partitioning kernel.
#pragma once
#include "common.cuh"

namespace nacho {

// One warp per boundary p in [0, P]: Q_p = floor(p Q* / P), b_0 = origin, b_P = end
// (reading R1), interior boundaries by FindPartition (Alg. 1).  The P+1 searches are independent
// ("computed independently, and thus in parallel").
// KM: compile-time bound on k (sizes the per-lane register arrays of the k-way search).
template <int WARPS, int KM>
// Boundaries p0 .. p0 + out.P of the Ptot-partition go to out[0 .. out.P] (a whole partition: p0 = 0,
// Ptot = out.P; a device slice otherwise).
#ifndef NACHO_PART_MINB   // tuning override: CTAs per SM the register allocation must allow
#define NACHO_PART_MINB 8   // 64 registers: 50 % occupancy (47 vs 51 us on C2; a few spilled bytes)
#endif
__global__ void __launch_bounds__(WARPS * 32, NACHO_PART_MINB) partition_kernel(const __grid_constant__ OpsArg a, PartsArg out, int64_t qstar,
                                                               int64_t Ptot, int64_t p0) {
  const int64_t i = (int64_t)blockIdx.x * WARPS + (threadIdx.x >> 5);
  if (i > out.P) return;  // warp-uniform
  const int64_t p = p0 + i;
  const int64_t Q = query_of(qstar, Ptot, p);   // one 64-bit division pair per boundary
  Boundary b;
  if (p == 0) set_origin(a, b);
  else if (p == Ptot) set_end(a, b);
  else b = warp_find_boundary<KM>(a, Q, 0, a.op[0].nouter);
  const int lane = threadIdx.x & 31;
  if (lane == 0) {
    out.query[i] = Q;
    out.row[i] = b.row;
    out.row_pos[i] = b.row_pos;
    out.col[i] = b.col;
  }
  if (lane < a.k) {
    int64_t v = 0;
#pragma unroll
    for (int o = 0; o < NACHO_MAX_K; ++o) if (o == lane) v = b.pos[o];
    out.pos[i * a.k + lane] = v;
  }
}

// One operand (SpMV, SpMM, DCSR SpMV): the cut is a plain position split (Listing 7 specialised to
// a single compressed operand: pos = Q_p), so only the row level needs a search --
// one thread per boundary, binary search for the largest outer position x with pos[x] <= Q_p.
__global__ void __launch_bounds__(256) partition1_kernel(const __grid_constant__ OpsArg a, PartsArg out,
                                                         int64_t qstar, int64_t Ptot, int64_t p0) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i > out.P) return;
  const int64_t p = p0 + i;
  const OpView& A = a.op[0];
  const int64_t Q = query_of(qstar, Ptot, p);
  int64_t row, rp, pos;
  int32_t col = 0;
  if (p == 0) {
    row = 0; rp = 0; pos = 0;                                         // origin (R1)
  } else if (p == Ptot || Q >= A.nnz) {
    row = a.nrows; rp = A.nouter; pos = A.nnz;                        // end (R1, R2)
  } else {
    int64_t lo = 0, hi = A.nouter;                                    // pos[lo] <= Q < pos[hi+1]
    while (lo < hi) {
      const int64_t m = lo + ((hi - lo + 1) >> 1);
      if (ldg(A.pos + m) <= Q) lo = m; else hi = m - 1;
    }
    rp = lo;
    row = A.outer ? (int64_t)ldg(A.outer + lo) : lo;
    pos = Q;
    col = ldg(A.crd + Q);
  }
  out.query[i] = Q;
  out.row[i] = row;
  out.row_pos[i] = rp;
  out.col[i] = col;
  out.pos[i] = pos;
}

}  // namespace nacho
