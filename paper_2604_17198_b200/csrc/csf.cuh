// csf.cuh -- third-order CSF tensors (Compressed o Compressed o Compressed; the coordinate tree of
// P:846-1030): Alg. 1 at d = 3 for k operands and the partitioned k-way addition (the
// paper's third-order tensor addition).
//   csf_partition_kernel: boundary p, one warp each.  Level i: the highest x_i in [0, n0] with
//     C_i(x_i) = sum_o pos2_o[pos1_o[lb(crd0_o, x_i)]] <= Q_p; level j inside slice x_i: the highest x_j
//     in [0, n1] with C_i(x_i) + C_j(x_j | x_i) <= Q_p, C_j summing the entries of the slice's fibers
//     j < x_j; level k inside fiber (x_i, x_j): the k-way select of the CSR path on the fibers' crd2
//     segments (operands without the slice / fiber contribute empty segments).  32-ary searches whose
//     probes run one binary search per operand (the cost functions of P:1689 on each level).
//   csf_spadd_kernel: one thread per partition (Listing 8's shape): the union of the operands'
//     entries [b_p.pos[o], b_{p+1}.pos[o]) in (i, j, k) order (k-finger merges at three levels),
//     counted (entries, fibers and slices whose first union entry lies in the partition) or written
//     (Z's crd2 / val at the entry offset, crd1 / crd0 of the fibers / slices started here, pos2 /
//     pos1 of those completed here -- Listing 8's guard, one level up).  Left fold (R9).
// Not performance-tuned: a coverage path.
#pragma once
#include "common.cuh"

namespace nacho {

struct Csf3View {
  int64_t n0, n1, n2, nnz, ns, nf;
  const int32_t* crd0;
  const int64_t* pos1;
  const int32_t* crd1;
  const int64_t* pos2;
  const int32_t* crd2;
  const void* val;
};

struct Csf3Args {
  Csf3View op[4];
  int32_t k;
  int64_t n0;
};

// least i in [lo, hi] with a[i] >= x
__device__ __forceinline__ int64_t csf_lb(const int32_t* a, int64_t lo, int64_t hi, int64_t x) {
  while (lo < hi) {
    const int64_t m = lo + ((hi - lo) >> 1);
    if ((int64_t)ldg(a + m) >= x) hi = m; else lo = m + 1;
  }
  return lo;
}

template <int KM>
__global__ void __launch_bounds__(128) csf_partition_kernel(const __grid_constant__ Csf3Args a, PartsArg out,
                                                            int64_t qstar) {
  const int64_t p = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
  if (p > out.P) return;
  const int lane = threadIdx.x & 31;
  const int k = a.k;
  const int64_t Q = query_of(qstar, out.P, p);
  int64_t xi = 0, xj = 0;
  int32_t col = 0;
  int64_t pos[KM];
  if (p == 0) {
#pragma unroll
    for (int o = 0; o < KM; ++o) pos[o] = 0;
  } else if (p == out.P || Q >= qstar) {
    xi = a.n0;
#pragma unroll
    for (int o = 0; o < KM; ++o) pos[o] = o < k ? a.op[o].nnz : 0;
  } else {
    // level i
    xi = warp_highest_true(0, a.n0, [&](int64_t x) {
      int64_t s = 0;
#pragma unroll
      for (int o = 0; o < KM; ++o)
        if (o < k) {
          const Csf3View& T = a.op[o];
          s += ldg(T.pos2 + ldg(T.pos1 + csf_lb(T.crd0, 0, T.ns, x)));
        }
      return s <= Q;
    });
    int64_t flo[KM], fhi[KM];
    int64_t base = 0;
#pragma unroll
    for (int o = 0; o < KM; ++o) {
      if (o < k) {
        const Csf3View& T = a.op[o];
        const int64_t s = csf_lb(T.crd0, 0, T.ns, xi);
        const bool present = s < T.ns && (int64_t)ldg(T.crd0 + s) == xi;
        flo[o] = ldg(T.pos1 + s);
        fhi[o] = present ? ldg(T.pos1 + s + 1) : flo[o];
        base += ldg(T.pos2 + flo[o]);
      }
    }
    // level j inside slice xi
    xj = warp_highest_true(0, a.op[0].n1, [&](int64_t y) {
      int64_t s = base;
#pragma unroll
      for (int o = 0; o < KM; ++o)
        if (o < k && fhi[o] > flo[o]) {
          const Csf3View& T = a.op[o];
          s += ldg(T.pos2 + csf_lb(T.crd1, flo[o], fhi[o], y)) - ldg(T.pos2 + flo[o]);
        }
      return s <= Q;
    });
    // level k inside fiber (xi, xj)
    const int32_t* cp[KM];
    int64_t lo[KM], len[KM], sel[KM];
    int64_t R = Q;
#pragma unroll
    for (int o = 0; o < KM; ++o) {
      if (o < k) {
        const Csf3View& T = a.op[o];
        const int64_t f = csf_lb(T.crd1, flo[o], fhi[o], xj);
        const bool present = f < fhi[o] && (int64_t)ldg(T.crd1 + f) == xj;
        lo[o] = ldg(T.pos2 + f);
        len[o] = present ? ldg(T.pos2 + f + 1) - lo[o] : 0;
        R -= lo[o];
        cp[o] = T.crd2 + lo[o];
        sel[o] = 0;
      }
    }
    int64_t zero[KM];
#pragma unroll
    for (int o = 0; o < KM; ++o) zero[o] = 0;
    warp_kway_select_t<KM, int64_t>(cp, k, zero, len, R, col, sel);
#pragma unroll
    for (int o = 0; o < KM; ++o) pos[o] = o < k ? lo[o] + sel[o] : 0;
  }
  if (lane == 0) {
    out.query[p] = Q;
    out.row[p] = xi;
    out.row_pos[p] = xj;
    out.col[p] = col;
  }
  if (lane < k) {
    int64_t w = 0;
#pragma unroll
    for (int o = 0; o < KM; ++o) if (o == lane) w = pos[o];
    out.pos[p * k + lane] = w;
  }
}

// fiber holding entry q (highest f with pos2[f] <= q) and slice holding fiber f
__device__ __forceinline__ int64_t csf_fiber_of(const Csf3View& T, int64_t q) {
  int64_t lo = 0, hi = T.nf > 0 ? T.nf - 1 : 0;
  while (lo < hi) {
    const int64_t m = lo + ((hi - lo + 1) >> 1);
    if (ldg(T.pos2 + m) <= q) lo = m; else hi = m - 1;
  }
  return lo;
}
__device__ __forceinline__ int64_t csf_slice_of(const Csf3View& T, int64_t f) {
  int64_t lo = 0, hi = T.ns > 0 ? T.ns - 1 : 0;
  while (lo < hi) {
    const int64_t m = lo + ((hi - lo + 1) >> 1);
    if (ldg(T.pos1 + m) <= f) lo = m; else hi = m - 1;
  }
  return lo;
}

template <typename V, int MODE>
__global__ void __launch_bounds__(128) csf_spadd_kernel(const __grid_constant__ Csf3Args a, PartsArg pa, int64_t* cnt,
                                                        const int64_t* off, int32_t* z_crd0, int64_t* z_pos1,
                                                        int32_t* z_crd1, int64_t* z_pos2, int32_t* z_crd2, V* z_val) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= pa.P) return;
  const int k = a.k;
  const int64_t P = pa.P;
  // off: [0, P] entry offsets, [P+1, 2P+1] fiber offsets, [2P+2, 3P+2] slice offsets (exclusive scans)
  int64_t q[4], e[4], f[4], s[4];
  for (int o = 0; o < k; ++o) {
    q[o] = pa.pos[p * k + o];
    e[o] = pa.pos[(p + 1) * k + o];
    f[o] = csf_fiber_of(a.op[o], q[o]);
    s[o] = csf_slice_of(a.op[o], f[o]);
  }
  const int64_t e0 = MODE ? off[p] : 0, f0 = MODE ? off[P + 1 + p] : 0, s0 = MODE ? off[2 * P + 2 + p] : 0;
  if (MODE && p == 0) { z_pos1[0] = 0; z_pos2[0] = 0; }
  int64_t ne = 0, nfb = 0, nsl = 0, ci = -1, cj = -1, fi = -1, si = -1;
  auto before_start = [&](int64_t i, int64_t j, bool fiber) {   // an earlier partition holds entries of it
    for (int o = 0; o < k; ++o) {
      const Csf3View& T = a.op[o];
      const int64_t sl = csf_lb(T.crd0, 0, T.ns, i);
      if (sl >= T.ns || (int64_t)ldg(T.crd0 + sl) != i) continue;
      int64_t first = ldg(T.pos2 + ldg(T.pos1 + sl));
      if (fiber) {
        const int64_t fb = csf_lb(T.crd1, ldg(T.pos1 + sl), ldg(T.pos1 + sl + 1), j);
        if (fb >= ldg(T.pos1 + sl + 1) || (int64_t)ldg(T.crd1 + fb) != j) continue;
        first = ldg(T.pos2 + fb);
      }
      if (first < pa.pos[p * k + o]) return true;
    }
    return false;
  };
  auto after_end = [&](int64_t i, int64_t j, bool fiber) {   // a later partition holds entries of it
    for (int o = 0; o < k; ++o) {
      const Csf3View& T = a.op[o];
      const int64_t sl = csf_lb(T.crd0, 0, T.ns, i);
      if (sl >= T.ns || (int64_t)ldg(T.crd0 + sl) != i) continue;
      int64_t last = ldg(T.pos2 + ldg(T.pos1 + sl + 1));
      if (fiber) {
        const int64_t fb = csf_lb(T.crd1, ldg(T.pos1 + sl), ldg(T.pos1 + sl + 1), j);
        if (fb >= ldg(T.pos1 + sl + 1) || (int64_t)ldg(T.crd1 + fb) != j) continue;
        last = ldg(T.pos2 + fb + 1);
      }
      if (last > e[o]) return true;
    }
    return false;
  };
  for (;;) {
    int64_t bi = INT64_MAX, bj = INT64_MAX, bk = INT64_MAX;
    for (int o = 0; o < k; ++o) {
      if (q[o] >= e[o]) continue;
      const Csf3View& T = a.op[o];
      while (ldg(T.pos2 + f[o] + 1) <= q[o]) ++f[o];
      while (ldg(T.pos1 + s[o] + 1) <= f[o]) ++s[o];
      const int64_t i = ldg(T.crd0 + s[o]), j = ldg(T.crd1 + f[o]), kk = ldg(T.crd2 + q[o]);
      if (i < bi || (i == bi && (j < bj || (j == bj && kk < bk)))) { bi = i; bj = j; bk = kk; }
    }
    if (bi == INT64_MAX) break;
    if (bi != ci || bj != cj) {   // a new fiber (maybe a new slice)
      if (MODE && fi >= 0) z_pos2[fi + 1] = e0 + ne;   // the previous fiber completed here
      if (bi != ci) {
        if (MODE && si >= 0) z_pos1[si + 1] = fi + 1;    // the previous slice completed here
        const bool started = ci >= 0 || !before_start(bi, 0, false);
        si = started ? s0 + nsl : s0 - 1;
        if (started) { ++nsl; if (MODE) z_crd0[si] = (int32_t)bi; }
      }
      const bool fstarted = cj >= 0 || ci >= 0 ? true : !before_start(bi, bj, true);
      fi = fstarted ? f0 + nfb : f0 - 1;
      if (fstarted) { ++nfb; if (MODE) z_crd1[fi] = (int32_t)bj; }
      ci = bi;
      cj = bj;
    }
    V acc = V(0);
    bool have = false;
    for (int o = 0; o < k; ++o) {
      if (q[o] < e[o]) {
        const Csf3View& T = a.op[o];
        if ((int64_t)ldg(T.crd0 + s[o]) == bi && (int64_t)ldg(T.crd1 + f[o]) == bj && (int64_t)ldg(T.crd2 + q[o]) == bk) {
          const V x = static_cast<const V*>(T.val)[q[o]];
          acc = have ? acc + x : x;
          have = true;
          ++q[o];
        }
      }
    }
    if (MODE) { z_crd2[e0 + ne] = (int32_t)bk; z_val[e0 + ne] = acc; }
    ++ne;
  }
  if (MODE && ci >= 0) {
    if (!after_end(ci, cj, true)) z_pos2[fi + 1] = e0 + ne;
    if (!after_end(ci, 0, false)) z_pos1[si + 1] = fi + 1;
  }
  if (!MODE) { cnt[p] = ne; cnt[P + 1 + p] = nfb; cnt[2 * P + 2 + p] = nsl; }
}

// counts = (slices, fibers, nnz) of Z from the three scans' totals
__global__ void csf_counts_kernel(const int64_t* off, int64_t P, int64_t* counts) {
  if (threadIdx.x == 0) { counts[0] = off[3 * P + 2]; counts[1] = off[2 * P + 1]; counts[2] = off[P]; }
}

}  // namespace nacho
