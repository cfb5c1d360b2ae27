// dcsr_add.cuh -- k-way SpAdd of DCSR operands (Listing 2, lst:eadd-dcsr2-cfir; SURVEY 8(f)
// #3): Alg. 1 with a compressed outer level for k operands, and the partitioned union.
//   dcsr_partition_kernel: boundary p, one warp each.  Level i: the highest row coordinate x in
//     [0, nrows] with C_i(x) = sum_o pos_o[lb_o(x)] <= Q_p (lb_o: lower bound of x in operand o's
//     outer level -- the DCSR row cost), a 32-ary search over x whose probes each run k
//     binary searches; level j: the k-way select of the CSR path in the row's k segments (an operand
//     that does not store row x contributes an empty segment).  row_pos = lb_0(x).
//   dcsr_spadd_kernel: one thread per partition (Listing 8's shape): the union of the k operands'
//     entries [b_p.pos[o], b_{p+1}.pos[o]) in (row, col) order -- k-finger merges at both levels --
//     counted (MODE 0: entries and rows whose first union entry lies in the partition) or written
//     (MODE 1: Z.crd / Z.val at the entry offset, Z's outer coordinate of every row started here, and
//     Z.pos of every row completed here, Listing 8's guard).  Values fold left in operand order (R9).
// Not performance-tuned: a coverage path.
#pragma once
#include "common.cuh"

namespace nacho {

__device__ __forceinline__ int64_t dcsr_lb(const int32_t* outer, int64_t n, int64_t x) {
  int64_t a = 0, b = n;
  while (a < b) {
    const int64_t m = a + ((b - a) >> 1);
    if ((int64_t)ldg(outer + m) >= x) b = m; else a = m + 1;
  }
  return a;
}

template <int KM>
__global__ void __launch_bounds__(128) dcsr_partition_kernel(const __grid_constant__ OpsArg a, PartsArg out,
                                                             int64_t qstar) {
  const int64_t p = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
  if (p > out.P) return;
  const int lane = threadIdx.x & 31;
  const int k = a.k;
  const int64_t Q = query_of(qstar, out.P, p);
  Boundary b;
  if (p == 0) {
    set_origin(a, b);
  } else if (p == out.P || Q >= qstar) {
    set_end(a, b);
    if (a.op[0].fmt != NACHO_DCSR) b.row_pos = a.nrows;   // CSR / COO: the dense row index
  } else {
    auto cost_ok = [&](int64_t x) {   // C_i(x): entries of rows < x over the operands (per level type)
      int64_t s = 0;
#pragma unroll
      for (int o = 0; o < KM; ++o) {
        if (o < k) {
          const OpView& op = a.op[o];
          s += op.fmt == NACHO_CSR ? ldg(op.pos + x)
             : op.fmt == NACHO_DCSR ? ldg(op.pos + dcsr_lb(op.outer, op.nouter, x))
                                    : dcsr_lb(op.outer, op.nnz, x);   // COO: the row level per entry
        }
      }
      return s <= Q;
    };
    const int64_t x = warp_highest_true(0, a.nrows, cost_ok);
    int64_t lo[KM], hi[KM];
    int64_t R = Q;
#pragma unroll
    for (int o = 0; o < KM; ++o) {
      if (o < k) {
        const OpView& op = a.op[o];
        if (op.fmt == NACHO_CSR) {
          lo[o] = ldg(op.pos + x);
          hi[o] = ldg(op.pos + x + 1);
        } else if (op.fmt == NACHO_DCSR) {
          const int64_t i = dcsr_lb(op.outer, op.nouter, x);
          const bool present = i < op.nouter && (int64_t)ldg(op.outer + i) == x;
          lo[o] = ldg(op.pos + i);
          hi[o] = present ? ldg(op.pos + i + 1) : lo[o];
        } else {
          lo[o] = dcsr_lb(op.outer, op.nnz, x);
          hi[o] = dcsr_lb(op.outer, op.nnz, x + 1);
        }
        R -= lo[o];
      }
    }
    warp_kway_select<KM>(a, k, lo, hi, R, b);
    b.row = x;
    b.row_pos = a.op[0].fmt == NACHO_DCSR ? dcsr_lb(a.op[0].outer, a.op[0].nouter, x) : x;
  }
  if (lane == 0) {
    out.query[p] = Q;
    out.row[p] = b.row;
    out.row_pos[p] = b.row_pos;
    out.col[p] = b.col;
  }
  if (lane < k) {
    int64_t v = 0;
#pragma unroll
    for (int o = 0; o < NACHO_MAX_K; ++o) if (o == lane) v = b.pos[o];
    out.pos[p * k + lane] = v;
  }
}

template <typename V, int MODE>
__global__ void __launch_bounds__(128) dcsr_spadd_kernel(const __grid_constant__ OpsArg a, PartsArg pa, int64_t* ent,
                                                         int64_t* rst, const int64_t* off_e, const int64_t* off_r,
                                                         int32_t* z_outer, int64_t* z_pos, int32_t* z_crd, V* z_val) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= pa.P) return;
  const int k = a.k;
  int64_t q[NACHO_MAX_K], e[NACHO_MAX_K], ip[NACHO_MAX_K];
  for (int o = 0; o < k; ++o) {
    q[o] = pa.pos[p * k + o];
    e[o] = pa.pos[(p + 1) * k + o];
    // outer position holding entry q[o]: the highest i with pos[i] <= q[o] (and a non-empty row)
    int64_t lo = 0, hi = a.op[o].nouter > 0 ? a.op[o].nouter - 1 : 0;
    while (lo < hi) {
      const int64_t m = lo + ((hi - lo + 1) >> 1);
      if (ldg(a.op[o].pos + m) <= q[o]) lo = m; else hi = m - 1;
    }
    ip[o] = lo;
  }
  int64_t ne = 0, nr = 0;
  const int64_t e0 = MODE ? off_e[p] : 0, r0 = MODE ? off_r[p] : 0;
  if (MODE && p == 0) z_pos[0] = 0;
  int64_t cur_row = -1, ri = -1;
  for (;;) {
    int64_t br = INT64_MAX;
    int32_t bc = INT32_MAX;
    for (int o = 0; o < k; ++o) {
      if (q[o] >= e[o]) continue;
      while (ldg(a.op[o].pos + ip[o] + 1) <= q[o]) ++ip[o];
      const int64_t r = ldg(a.op[o].outer + ip[o]);
      const int32_t c = ldg(a.op[o].crd + q[o]);
      if (r < br || (r == br && c < bc)) { br = r; bc = c; }
    }
    if (br == INT64_MAX) break;
    if (br != cur_row) {   // a new union row inside the partition
      if (MODE && cur_row >= 0) z_pos[ri + 1] = e0 + ne;   // the previous one completed here
      bool started = true;
      if (cur_row < 0) {   // the partition's first row: did an earlier partition hold entries of it?
        for (int o = 0; o < k; ++o) {
          const int64_t i = dcsr_lb(a.op[o].outer, a.op[o].nouter, br);
          if (i < a.op[o].nouter && ldg(a.op[o].outer + i) == br && ldg(a.op[o].pos + i) < pa.pos[p * k + o])
            started = false;
        }
      }
      if (started) {
        ri = r0 + nr;
        ++nr;
        if (MODE) z_outer[ri] = (int32_t)br;
      } else {
        ri = r0 - 1;
      }
      cur_row = br;
    }
    V acc = V(0);
    bool have = false;
    for (int o = 0; o < k; ++o) {
      if (q[o] < e[o] && ldg(a.op[o].outer + ip[o]) == br && ldg(a.op[o].crd + q[o]) == bc) {
        const V x = static_cast<const V*>(a.op[o].val)[q[o]];
        acc = have ? acc + x : x;
        have = true;
        ++q[o];
      }
    }
    if (MODE) {
      z_crd[e0 + ne] = bc;
      z_val[e0 + ne] = acc;
    }
    ++ne;
  }
  if (MODE && cur_row >= 0) {   // the last row: completed here unless an operand holds more of it
    bool done = true;
    for (int o = 0; o < k; ++o) {
      const int64_t i = dcsr_lb(a.op[o].outer, a.op[o].nouter, cur_row);
      if (i < a.op[o].nouter && ldg(a.op[o].outer + i) == cur_row && ldg(a.op[o].pos + i + 1) > e[o]) done = false;
    }
    if (done) z_pos[ri + 1] = e0 + ne;
  }
  if (!MODE) { ent[p] = ne; rst[p] = nr; }
}

// k-way union of CSR and COO operands mixed (the COO + CSR addition), Z in CSR: one
// thread per partition walks its rows [b_p.row, b_{p+1}.row] (the last one up to the cut): an
// operand's entries of row r inside the partition are [max(pos[r], s_o), min(pos[r + 1], e_o)) for
// CSR and the run of its row level equal to r from its cursor for COO.  MODE 0 counts; MODE 1 writes
// Z at off[p] and Z.pos[r + 1] of every row the partition owns (R7: r < b_{p+1}.row).
template <typename V, int MODE>
__global__ void __launch_bounds__(128) mixed_spadd_kernel(const __grid_constant__ OpsArg a, PartsArg pa, int64_t* cnt,
                                                          const int64_t* off, int64_t* z_pos, int32_t* z_crd,
                                                          V* z_val) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= pa.P) return;
  const int k = a.k;
  const int64_t M = a.nrows;
  const int64_t r0 = pa.row[p], r1 = pa.row[p + 1];
  int64_t q[NACHO_MAX_K], e[NACHO_MAX_K];
  for (int o = 0; o < k; ++o) { q[o] = pa.pos[p * k + o]; e[o] = pa.pos[(p + 1) * k + o]; }
  int64_t n = 0;
  const int64_t w0 = MODE ? off[p] : 0;
  if (MODE && p == 0) z_pos[0] = 0;
  for (int64_t r = r0; r <= r1 && r < M; ++r) {
    int64_t hi[NACHO_MAX_K];
    for (int o = 0; o < k; ++o) {
      const OpView& op = a.op[o];
      if (op.fmt == NACHO_CSR) {
        const int64_t rs = ldg(op.pos + r), re = ldg(op.pos + r + 1);
        if (q[o] < rs) q[o] = rs;
        hi[o] = re < e[o] ? re : e[o];
      } else {
        int64_t h = q[o];
        while (h < e[o] && (int64_t)ldg(op.outer + h) == r) ++h;
        hi[o] = h;
      }
    }
    for (;;) {
      int32_t j = INT32_MAX;
      for (int o = 0; o < k; ++o) if (q[o] < hi[o]) j = min(j, ldg(a.op[o].crd + q[o]));
      if (j == INT32_MAX) break;
      V acc = V(0);
      bool have = false;
      for (int o = 0; o < k; ++o) {
        if (q[o] < hi[o] && ldg(a.op[o].crd + q[o]) == j) {
          const V x = static_cast<const V*>(a.op[o].val)[q[o]];
          acc = have ? acc + x : x;
          have = true;
          ++q[o];
        }
      }
      if (MODE) { z_crd[w0 + n] = j; z_val[w0 + n] = acc; }
      ++n;
    }
    if (MODE && r < r1) z_pos[r + 1] = w0 + n;   // owned row (R7)
  }
  if (!MODE) cnt[p] = n;
}

}  // namespace nacho
