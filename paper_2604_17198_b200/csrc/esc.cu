// esc.cu -- the ESC scatter kernels: SpGEMM C = A B over the loop order i -> k -> j and
// sampled SpGEMM Z = S (.) (A B) as expand - sort - contract, with Nacho's load
// balancing applied to the expansion only.
//
//   work      W[q] = sum_{q' < q} nnz(B_{A.crd[q']}): the broadcast-scaled cost of Listing 6
//              -- A's entry (i, k) is coiterated with all of B's row k
//             (one length per entry, then a device-wide exclusive scan);
//   partition Alg. 1 over i -> k -> j with that cost: C_i(x) = W[A.pos[x]] (outer
//             search), C_k(q | x) = W[q] (search in row x's positions), C_j = the offset inside
//             B's row k, solved directly: b_p locates product number Q_p;
//   expand    one CTA per partition materialises its products [Q_p, Q_{p+1}) -- coordinate key
//             (i << jbits) | j and value A_ik * B_kj -- at their expansion index (append-only:
//             the offsets are the queries themselves); SSSMM keeps the products whose j is stored
//             in S_i (count per partition, exclusive scan, order-preserving fill);
//   sort      a stable radix sort by key (CUB, a library primitive as SURVEY A24 / K6 allow) keeps
//             the products of one (i, j) in expansion order, i.e. k ascending (reading R23);
//   contract  run heads -> exclusive scan -> one thread per run folds it left to right in the value
//             type and writes C.crd / C.val / the row pointers (SSSMM: times S_ij, reading R24).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <cstring>

#include "common.cuh"

// status plumbing shared with api.cu (the thread-local last error and the launch counter)
nacho_status nacho_internal_fail(nacho_status s, const char* msg);
nacho_status nacho_internal_launched(const char* what);

namespace nacho {

constexpr int kEscThreads = 256;
constexpr int64_t kEscTile = 8192;   // products per partition of the automatic P

struct EscOps {
  const int64_t* a_pos;
  const int32_t* a_crd;
  const void* a_val;
  int64_t a_rows, a_nnz;
  const int64_t* b_pos;
  const int32_t* b_crd;
  const void* b_val;
  int64_t b_nnz;
  const int64_t* s_pos;   // SSSMM sampling matrix S (null for SpGEMM)
  const int32_t* s_crd;
  const void* s_val;
  const int64_t* W;       // [a_nnz + 1]
  int32_t jbits;          // key = (i << jbits) | j
};

// ------------------------------------------------------------------ work
__global__ void esc_len_kernel(const EscOps o, int64_t* W) {
  const int64_t n = o.a_nnz;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q <= n; q += (int64_t)gridDim.x * blockDim.x) {
    int64_t len = 0;
    if (q < n) {
      const int64_t k = ldg(o.a_crd + q);
      len = ldg(o.b_pos + k + 1) - ldg(o.b_pos + k);
    }
    W[q] = len;
  }
}

// ------------------------------------------------------------------ partition (Alg. 1, i -> k -> j)
__global__ void __launch_bounds__(128) esc_partition_kernel(const EscOps o, int64_t qstar, int32_t P, PartsArg out) {
  const int64_t p = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (p > P) return;
  const int64_t Q = query_of(qstar, P, p);
  int64_t x = o.a_rows, q = o.a_nnz, bp = o.b_nnz;
  int32_t col = 0;
  if (Q < qstar) {
    // level i: the largest row x with C_i(x) = W[A.pos[x]] <= Q (x < nrows: C_i(nrows) = Q* > Q)
    x = warp_highest_true(0, o.a_rows, [&](int64_t xx) { return ldg(o.W + ldg(o.a_pos + xx)) <= Q; });
    // level k: the largest position q of row x with W[q] <= Q (q < A.pos[x + 1] by the maximality of x)
    q = warp_highest_true(ldg(o.a_pos + x), ldg(o.a_pos + x + 1), [&](int64_t qq) { return ldg(o.W + qq) <= Q; });
    // level j: the offset Q - W[q] inside row k of B
    const int64_t k = ldg(o.a_crd + q);
    bp = ldg(o.b_pos + k) + (Q - ldg(o.W + q));
    col = ldg(o.b_crd + bp);
  }
  if (lane == 0) {
    out.query[p] = Q;
    out.row[p] = x;
    out.row_pos[p] = x;
    out.col[p] = col;
    out.pos[2 * p] = q;
    out.pos[2 * p + 1] = bp;
  }
}

// ------------------------------------------------------------------ expand
constexpr int kEscAll = 0;     // SpGEMM: every product at its expansion index
constexpr int kEscCount = 1;   // SSSMM: kept products per partition
constexpr int kEscFill = 2;    // SSSMM: kept products at part_off[p] + rank, in expansion order

template <typename V>
struct EscExpandArgs {
  EscOps o;
  PartsArg parts;
  int64_t* cnt;             // kEscCount: [P]; kEscFill: part_off [P + 1]
  unsigned long long* key;  // kEscAll / kEscFill
  V* val;
  uint8_t* mask;            // SSSMM: the count pass's keep bits (8 products per byte), read by the fill
};

// Byte offset of partition p's keep bits in the SSSMM mask (floor(Q_p / 8) + p: monotone, and
// partition p's ceil((Q_{p+1} - Q_p) / 8) bytes never reach partition p + 1's).
__device__ __forceinline__ int64_t esc_mask_base(int64_t Qp, int64_t p) { return (Qp >> 3) + p; }

// One CTA per partition, in chunks of kEscChunk products: thread t walks products
// [c0 + 8t, c0 + 8t + 8) sequentially -- one search for the first product's A entry q and row i,
// then q / i advance as the product index passes W[q + 1] / A.pos[i + 1] (zero-cost entries and empty
// rows are stepped over) and B's row k is read in order -- and the chunk is staged in shared memory
// so that the expansion is written with coalesced stores.
constexpr int kEscVT = 8;
constexpr int kEscChunk = kEscThreads * kEscVT;

// CTAs per SM the registers are sized for (pinned: left free, ptxas picked 47-55 registers for the
// count pass from one build to the next, 1.1-1.5 ms)
template <int MODE>
constexpr int esc_minb() { return MODE == kEscCount ? 5 : 3; }

template <typename V, int MODE>
__global__ void __launch_bounds__(kEscThreads, esc_minb<MODE>()) esc_expand_kernel(const EscExpandArgs<V> a) {
  __shared__ unsigned long long skey[MODE == kEscCount ? 1 : kEscChunk];
  __shared__ V sval[MODE == kEscCount ? 1 : kEscChunk];
  __shared__ int32_t wsum[kEscThreads / 32 + 1];
  const EscOps& o = a.o;
  const int64_t p = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t Q0 = a.parts.query[p], Q1 = a.parts.query[p + 1];
  const int64_t q0 = a.parts.pos[2 * p];
  const int64_t q1 = min(a.parts.pos[2 * (p + 1)], o.a_nnz - 1);
  const int64_t x0 = a.parts.row[p];
  const int64_t x1 = min(a.parts.row[p + 1], o.a_rows - 1);
  const V* av = static_cast<const V*>(o.a_val);
  const V* bv = static_cast<const V*>(o.b_val);
  int64_t run = MODE == kEscFill ? a.cnt[p] : 0;   // kept products written so far
  int64_t kept = 0;
  for (int64_t c0 = Q0; c0 < Q1; c0 += kEscChunk) {
    const int64_t wb = c0 + (int64_t)tid * kEscVT;
    const int64_t we = min(wb + kEscVT, Q1);
    unsigned long long kk[kEscVT];
    V vv[kEscVT];
    uint32_t keep = 0;
    if (wb < we) {
      // the A entry producing product wb: the largest q in [q0, q1] with W[q] <= wb; its row i
      int64_t q = q0, hi = q1;
      while (q < hi) {
        const int64_t mid = (q + hi + 1) >> 1;
        if (ldg(o.W + mid) <= wb) q = mid; else hi = mid - 1;
      }
      int64_t i = x0, rh = x1;
      while (i < rh) {
        const int64_t mid = (i + rh + 1) >> 1;
        if (ldg(o.a_pos + mid) <= q) i = mid; else rh = mid - 1;
      }
      int64_t wq = ldg(o.W + q), wn = ldg(o.W + q + 1);
      int64_t apn = ldg(o.a_pos + i + 1);
      int64_t bs = ldg(o.b_pos + ldg(o.a_crd + q));
      V a_iq = ldg(av + q);
      int64_t sp = 0, se = 0;   // sampled: cursor in S_i (valid for the current q)
      bool fresh = true;
#pragma unroll
      for (int v = 0; v < kEscVT; ++v) {
        const int64_t w = wb + v;
        if (w < we) {
          if (w >= wn) {   // next A entry with a product (entries without one are stepped over)
            do {
              ++q;
              wq = wn;
              wn = ldg(o.W + q + 1);
            } while (w >= wn);
            while (apn <= q) apn = ldg(o.a_pos + (++i) + 1);
            bs = ldg(o.b_pos + ldg(o.a_crd + q));
            a_iq = ldg(av + q);
            fresh = true;
          }
          const int64_t r = bs + (w - wq);
          const int32_t j = ldg(o.b_crd + r);
          bool kp = true;
          if (MODE == kEscFill) {   // sampled: the count pass recorded the membership
            kp = (a.mask[esc_mask_base(Q0, p) + ((wb - Q0) >> 3)] >> v) & 1u;
          } else if (MODE != kEscAll) {   // sampled: is j stored in S_i?  (j rises along B's row: gallop)
            if (fresh) {
              sp = ldg(o.s_pos + i);
              se = ldg(o.s_pos + i + 1);
              fresh = false;
            }
            int g = 0;
            while (sp < se && ldg(o.s_crd + sp) < j && g < 4) { ++sp; ++g; }
            if (sp < se && ldg(o.s_crd + sp) < j) {
              int64_t lo = sp + 1, h2 = se;
              while (lo < h2) {
                const int64_t mid = (lo + h2) >> 1;
                if (ldg(o.s_crd + mid) < j) lo = mid + 1; else h2 = mid;
              }
              sp = lo;
            }
            kp = sp < se && ldg(o.s_crd + sp) == j;
          }
          if (kp) {
            keep |= 1u << v;
            if (MODE != kEscCount) {
              kk[v] = ((unsigned long long)i << o.jbits) | (unsigned long long)(uint32_t)j;
              vv[v] = a_iq * ldg(bv + r);
            }
          }
        }
      }
    }
    if (MODE == kEscCount && wb < we) a.mask[esc_mask_base(Q0, p) + ((wb - Q0) >> 3)] = (uint8_t)keep;
    const int n_chunk = (int)min((int64_t)kEscChunk, Q1 - c0);
    if (MODE == kEscAll) {   // every product at its expansion index
#pragma unroll
      for (int v = 0; v < kEscVT; ++v)
        if (keep & (1u << v)) { skey[tid * kEscVT + v] = kk[v]; sval[tid * kEscVT + v] = vv[v]; }
      __syncthreads();
      for (int u = tid; u < n_chunk; u += kEscThreads) {
        a.key[c0 + u] = skey[u];
        a.val[c0 + u] = sval[u];
      }
      __syncthreads();
      continue;
    }
    // kept products: rank in expansion order (block exclusive scan of the per-thread counts)
    const int cnt = __popc(keep);
    int x = cnt;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int y = __shfl_up_sync(kFull, x, d);
      if (lane >= d) x += y;
    }
    if (lane == 31) wsum[wid] = x;
    __syncthreads();
    int before = 0, tot = 0;
#pragma unroll
    for (int u = 0; u < kEscThreads / 32; ++u) {
      const int c = wsum[u];
      before += u < wid ? c : 0;
      tot += c;
    }
    if (MODE == kEscFill) {
      int z = before + x - cnt;
#pragma unroll
      for (int v = 0; v < kEscVT; ++v)
        if (keep & (1u << v)) { skey[z] = kk[v]; sval[z] = vv[v]; ++z; }
      __syncthreads();
      for (int u = tid; u < tot; u += kEscThreads) {
        a.key[run + u] = skey[u];
        a.val[run + u] = sval[u];
      }
    }
    __syncthreads();
    run += tot;
    kept += tot;
  }
  if (MODE == kEscCount && tid == 0) a.cnt[p] = kept;
}

// ------------------------------------------------------------------ contract
__global__ void esc_heads_kernel(const unsigned long long* __restrict__ key, int64_t n, int64_t* __restrict__ head) {
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < n; w += (int64_t)gridDim.x * blockDim.x)
    head[w] = (w == 0 || key[w] != key[w - 1]) ? 1 : 0;
}

template <typename V, bool SAMPLE>
struct EscContractArgs {
  EscOps o;
  const unsigned long long* key;
  const V* val;
  const int64_t* idx;   // exclusive scan of the run heads
  int64_t n;            // products (sorted)
  int64_t* c_pos;
  int32_t* c_crd;
  V* c_val;
  int64_t* nnz;
};

template <typename V, bool SAMPLE>
__global__ void __launch_bounds__(kEscThreads) esc_contract_kernel(const EscContractArgs<V, SAMPLE> a) {
  const uint64_t jmask = (1ull << a.o.jbits) - 1ull;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < a.n; w += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long kw = a.key[w];
    const int64_t iprev = w == 0 ? -1 : (int64_t)(a.key[w - 1] >> a.o.jbits);
    if (w > 0 && a.key[w - 1] == kw) continue;   // not a run head
    const int64_t out = a.idx[w];
    // the run's products in expansion order (k ascending): a left fold in the value type
    V acc = a.val[w];
    int64_t e = w + 1;
    for (; e < a.n && a.key[e] == kw; ++e) acc = acc + a.val[e];
    const int64_t i = (int64_t)(kw >> a.o.jbits);
    const int32_t j = (int32_t)(kw & jmask);
    if (SAMPLE) {   // Z_ij = S_ij * C_ij (j is stored in S_i: the expansion kept only those)
      int64_t sl = ldg(a.o.s_pos + i), sh = ldg(a.o.s_pos + i + 1);
      while (sl < sh) {
        const int64_t mid = (sl + sh) >> 1;
        if (ldg(a.o.s_crd + mid) < j) sl = mid + 1; else sh = mid;
      }
      acc = ldg(static_cast<const V*>(a.o.s_val) + sl) * acc;
    }
    a.c_crd[out] = j;
    a.c_val[out] = acc;
    // row pointers: the rows after the previous entry's row up to i start at this entry
    for (int64_t rr = iprev + 1; rr <= i; ++rr) a.c_pos[rr] = out;
    if (e == a.n) {   // the last entry: the remaining rows end at nnz
      for (int64_t rr = i + 1; rr <= a.o.a_rows; ++rr) a.c_pos[rr] = out + 1;
      *a.nnz = out + 1;
    }
  }
}

__global__ void esc_empty_kernel(int64_t* c_pos, int64_t rows, int64_t* nnz) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r <= rows; r += (int64_t)gridDim.x * blockDim.x)
    c_pos[r] = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) *nnz = 0;
}

}  // namespace nacho

using namespace nacho;

namespace {

#define ESC_TRY(x)                          \
  do {                                      \
    const nacho_status _s = (x);            \
    if (_s != NACHO_SUCCESS) return _s;     \
  } while (0)

nacho_status efail(nacho_status s, const char* msg) { return nacho_internal_fail(s, msg); }

size_t al(size_t x) { return (x + 255) & ~size_t(255); }

int bits_for(int64_t n) {   // bits to hold 0 .. n - 1 (at least 1: a radix sort over 0 bits is no sort)
  int b = 1;
  while (b < 63 && (int64_t(1) << b) < n) ++b;
  return b;
}

int grid_for(int64_t n) {
  const int64_t g = (n + kEscThreads - 1) / kEscThreads;
  return (int)(g < 1 ? 1 : (g > 148 * 32 ? 148 * 32 : g));
}

nacho_status check_csr(const nacho_matrix* A, const char* nm) {
  if (!A) return efail(NACHO_ERR_INVALID_ARG, "null matrix descriptor");
  if (A->format != NACHO_CSR || A->nouter != A->nrows)
    return efail(NACHO_ERR_INVALID_ARG, nm);
  if (A->dtype != NACHO_F32 && A->dtype != NACHO_F64) return efail(NACHO_ERR_INVALID_ARG, "bad dtype");
  if (!A->pos || (A->nnz > 0 && (!A->crd || !A->val))) return efail(NACHO_ERR_INVALID_ARG, "null pos / crd / val");
  if (A->nrows > INT32_MAX || A->ncols > INT32_MAX) return efail(NACHO_ERR_OVERFLOW, "nrows / ncols > INT32_MAX");
  return NACHO_SUCCESS;
}

nacho_status check_pair(const nacho_matrix* A, const nacho_matrix* B) {
  ESC_TRY(check_csr(A, "ESC SpGEMM: A must be CSR"));
  ESC_TRY(check_csr(B, "ESC SpGEMM: B must be CSR"));
  if (A->ncols != B->nrows) return efail(NACHO_ERR_SHAPE, "ESC SpGEMM: A.ncols != B.nrows");
  if (A->dtype != B->dtype) return efail(NACHO_ERR_INVALID_ARG, "ESC SpGEMM: A and B dtypes differ");
  if (bits_for(A->nrows) + bits_for(B->ncols) > 64) return efail(NACHO_ERR_OVERFLOW, "ESC keys need > 64 bits");
  return NACHO_SUCCESS;
}

EscOps make_esc(const nacho_matrix* A, const nacho_matrix* B, const nacho_matrix* S, const int64_t* W) {
  EscOps o;
  memset(&o, 0, sizeof(o));
  o.a_pos = A->pos; o.a_crd = A->crd; o.a_val = A->val; o.a_rows = A->nrows; o.a_nnz = A->nnz;
  o.b_pos = B->pos; o.b_crd = B->crd; o.b_val = B->val; o.b_nnz = B->nnz;
  if (S) { o.s_pos = S->pos; o.s_crd = S->crd; o.s_val = S->val; }
  o.W = W;
  o.jbits = bits_for(B->ncols);
  return o;
}

PartsArg esc_parts(const nacho_parts* p) {
  PartsArg a;
  memset(&a, 0, sizeof(a));
  a.P = p->P; a.k = p->k; a.query = p->query; a.row = p->row; a.row_pos = p->row_pos; a.col = p->col; a.pos = p->pos;
  return a;
}

nacho_status check_esc_parts(const nacho_parts* p) {
  if (!p || p->P < 1 || p->k != 2 || !p->query || !p->row || !p->row_pos || !p->col || !p->pos)
    return efail(NACHO_ERR_INVALID_ARG, "ESC partition record: P >= 1, k == 2, all arrays");
  return NACHO_SUCCESS;
}

// sort + contract workspace: keys in / out, values in / out, run heads -> indices, CUB scratch
template <typename V>
size_t sort_bytes(int64_t n, int ebits) {
  size_t s1 = 0, s2 = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, s1, (const unsigned long long*)nullptr, (unsigned long long*)nullptr,
                                  (const V*)nullptr, (V*)nullptr, n, 0, ebits);
  cub::DeviceScan::ExclusiveSum(nullptr, s2, (const int64_t*)nullptr, (int64_t*)nullptr, n);
  return std::max(s1, s2);
}

template <typename V>
size_t esc_ws(int64_t n, int ebits) {
  const size_t nn = (size_t)(n > 0 ? n : 1);
  return 2 * al(nn * 8) + 2 * al(nn * sizeof(V)) + al(nn * 8) + al(sort_bytes<V>(n, ebits));
}

// sort the n products in ws's first key / value buffers and contract them into C
template <typename V, bool SAMPLE>
nacho_status sort_contract(const EscOps& o, int64_t n, int ebits, unsigned char* ws, int64_t* c_pos, int32_t* c_crd,
                           V* c_val, int64_t* nnz, cudaStream_t st) {
  const size_t nn = (size_t)(n > 0 ? n : 1);
  auto* k_in = reinterpret_cast<unsigned long long*>(ws);
  auto* k_out = reinterpret_cast<unsigned long long*>(ws + al(nn * 8));
  V* v_in = reinterpret_cast<V*>(ws + 2 * al(nn * 8));
  V* v_out = reinterpret_cast<V*>(ws + 2 * al(nn * 8) + al(nn * sizeof(V)));
  int64_t* idx = reinterpret_cast<int64_t*>(ws + 2 * al(nn * 8) + 2 * al(nn * sizeof(V)));
  void* tmp = ws + 2 * al(nn * 8) + 2 * al(nn * sizeof(V)) + al(nn * 8);
  size_t tb = al(sort_bytes<V>(n, ebits));
  if (n == 0) {
    esc_empty_kernel<<<grid_for(o.a_rows + 1), kEscThreads, 0, st>>>(c_pos, o.a_rows, nnz);
    return nacho_internal_launched("esc_empty_kernel");
  }
  if (cub::DeviceRadixSort::SortPairs(tmp, tb, k_in, k_out, v_in, v_out, n, 0, ebits, st) != cudaSuccess)
    return efail(NACHO_ERR_CUDA, "ESC: radix sort");
  ESC_TRY(nacho_internal_launched("esc_sort (cub onesweep)"));
  esc_heads_kernel<<<grid_for(n), kEscThreads, 0, st>>>(k_out, n, idx);
  ESC_TRY(nacho_internal_launched("esc_heads_kernel"));
  tb = al(sort_bytes<V>(n, ebits));
  if (cub::DeviceScan::ExclusiveSum(tmp, tb, idx, idx, n, st) != cudaSuccess) return efail(NACHO_ERR_CUDA, "ESC: scan");
  ESC_TRY(nacho_internal_launched("esc_scan (cub)"));
  EscContractArgs<V, SAMPLE> ca{o, k_out, v_out, idx, n, c_pos, c_crd, c_val, nnz};
  esc_contract_kernel<V, SAMPLE><<<grid_for(n), kEscThreads, 0, st>>>(ca);
  return nacho_internal_launched("esc_contract_kernel");
}

}  // namespace

extern "C" {

size_t nacho_spgemm_work_workspace_size(const nacho_matrix* A) {
  size_t t = 0;
  const int64_t n = A ? A->nnz + 1 : 1;
  cub::DeviceScan::ExclusiveSum(nullptr, t, (const int64_t*)nullptr, (int64_t*)nullptr, n);
  return al(t);
}

nacho_status nacho_spgemm_work(const nacho_matrix* A, const nacho_matrix* B, int64_t* W, void* ws, size_t ws_bytes,
                               void* stream) {
  ESC_TRY(check_pair(A, B));
  if (!W) return efail(NACHO_ERR_INVALID_ARG, "null W");
  const size_t need = nacho_spgemm_work_workspace_size(A);
  if (!ws || ws_bytes < need) return efail(NACHO_ERR_WORKSPACE, "nacho_spgemm_work: workspace too small");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const EscOps o = make_esc(A, B, nullptr, W);
  esc_len_kernel<<<grid_for(A->nnz + 1), kEscThreads, 0, st>>>(o, W);
  ESC_TRY(nacho_internal_launched("esc_len_kernel"));
  size_t tb = need;
  if (cub::DeviceScan::ExclusiveSum(ws, tb, W, W, A->nnz + 1, st) != cudaSuccess)
    return efail(NACHO_ERR_CUDA, "nacho_spgemm_work: scan");
  return nacho_internal_launched("esc_work_scan (cub)");
}

int32_t nacho_esc_auto_partitions(int64_t qstar) {
  int64_t P = (qstar + kEscTile - 1) / kEscTile;
  if (P < 1) P = 1;
  if (P > INT32_MAX - 1) P = INT32_MAX - 1;
  return (int32_t)P;
}

nacho_status nacho_partition_esc(const nacho_matrix* A, const nacho_matrix* B, const int64_t* W, int64_t qstar,
                                 int32_t P, nacho_parts* out, void* stream) {
  ESC_TRY(check_pair(A, B));
  if (!W || qstar < 0) return efail(NACHO_ERR_INVALID_ARG, "null W or negative Q*");
  ESC_TRY(check_esc_parts(out));
  if (out->P != P) return efail(NACHO_ERR_INVALID_ARG, "nacho_partition_esc: out->P != P");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const EscOps o = make_esc(A, B, nullptr, W);
  const int64_t threads = (int64_t)(P + 1) * 32;
  esc_partition_kernel<<<(unsigned)((threads + 127) / 128), 128, 0, st>>>(o, qstar, P, esc_parts(out));
  out->max_work = qstar / P + 1;
  return nacho_internal_launched("esc_partition_kernel");
}

size_t nacho_spgemm_esc_workspace_size(const nacho_matrix* A, const nacho_matrix* B, int64_t qstar) {
  if (!A || !B) return 0;
  const int eb = bits_for(A->nrows) + bits_for(B->ncols);
  return A->dtype == NACHO_F64 ? esc_ws<double>(qstar, eb) : esc_ws<float>(qstar, eb);
}

nacho_status nacho_spgemm_esc(const nacho_matrix* A, const nacho_matrix* B, const int64_t* W, const nacho_parts* parts,
                              int64_t qstar, int64_t* c_pos, int32_t* c_crd, void* c_val, int64_t* nnz_c, void* ws,
                              size_t ws_bytes, void* stream) {
  ESC_TRY(check_pair(A, B));
  ESC_TRY(check_esc_parts(parts));
  if (!W || !c_pos || !nnz_c || (qstar > 0 && (!c_crd || !c_val))) return efail(NACHO_ERR_INVALID_ARG, "null output");
  const size_t need = nacho_spgemm_esc_workspace_size(A, B, qstar);
  if (!ws || ws_bytes < need) return efail(NACHO_ERR_WORKSPACE, "nacho_spgemm_esc: workspace too small");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const EscOps o = make_esc(A, B, nullptr, W);
  const int eb = bits_for(A->nrows) + o.jbits;
  auto* w8 = static_cast<unsigned char*>(ws);
  const size_t nn = (size_t)(qstar > 0 ? qstar : 1);
  if (A->dtype == NACHO_F64) {
    EscExpandArgs<double> ea{o, esc_parts(parts), nullptr, reinterpret_cast<unsigned long long*>(w8),
                             reinterpret_cast<double*>(w8 + 2 * al(nn * 8))};
    if (qstar > 0) {
      esc_expand_kernel<double, kEscAll><<<parts->P, kEscThreads, 0, st>>>(ea);
      ESC_TRY(nacho_internal_launched("esc_expand_kernel"));
    }
    return sort_contract<double, false>(o, qstar, eb, w8, c_pos, c_crd, static_cast<double*>(c_val), nnz_c, st);
  }
  EscExpandArgs<float> ea{o, esc_parts(parts), nullptr, reinterpret_cast<unsigned long long*>(w8),
                          reinterpret_cast<float*>(w8 + 2 * al(nn * 8))};
  if (qstar > 0) {
    esc_expand_kernel<float, kEscAll><<<parts->P, kEscThreads, 0, st>>>(ea);
    ESC_TRY(nacho_internal_launched("esc_expand_kernel"));
  }
  return sort_contract<float, false>(o, qstar, eb, w8, c_pos, c_crd, static_cast<float*>(c_val), nnz_c, st);
}

// ---- sampled SpGEMM
static nacho_status check_sample(const nacho_matrix* S, const nacho_matrix* A, const nacho_matrix* B) {
  ESC_TRY(check_pair(A, B));
  ESC_TRY(check_csr(S, "SSSMM: S must be CSR"));
  if (S->nrows != A->nrows || S->ncols != B->ncols) return efail(NACHO_ERR_SHAPE, "SSSMM: S is not nrows(A) x ncols(B)");
  if (S->dtype != A->dtype) return efail(NACHO_ERR_INVALID_ARG, "SSSMM: S dtype differs");
  return NACHO_SUCCESS;
}

size_t nacho_sssmm_mask_bytes(int64_t qstar, int32_t P) { return (size_t)(qstar > 0 ? qstar : 0) / 8 + (size_t)P + 2; }

size_t nacho_sssmm_count_workspace_size(int32_t P) {
  size_t t = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, t, (const int64_t*)nullptr, (int64_t*)nullptr, (int64_t)P + 1);
  return al(t);
}

nacho_status nacho_sssmm_esc_count(const nacho_matrix* S, const nacho_matrix* A, const nacho_matrix* B, const int64_t* W,
                                   const nacho_parts* parts, int64_t* part_off, uint8_t* keep_mask, void* ws,
                                   size_t ws_bytes, void* stream) {
  ESC_TRY(check_sample(S, A, B));
  ESC_TRY(check_esc_parts(parts));
  if (!W || !part_off || !keep_mask) return efail(NACHO_ERR_INVALID_ARG, "null W / part_off / keep_mask");
  const size_t need = nacho_sssmm_count_workspace_size(parts->P);
  if (!ws || ws_bytes < need) return efail(NACHO_ERR_WORKSPACE, "nacho_sssmm_esc_count: workspace too small");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const EscOps o = make_esc(A, B, S, W);
  if (cudaMemsetAsync(part_off + parts->P, 0, 8, st) != cudaSuccess) return efail(NACHO_ERR_CUDA, "memset");
  if (A->dtype == NACHO_F64) {
    EscExpandArgs<double> ea{o, esc_parts(parts), part_off, nullptr, nullptr, keep_mask};
    esc_expand_kernel<double, kEscCount><<<parts->P, kEscThreads, 0, st>>>(ea);
  } else {
    EscExpandArgs<float> ea{o, esc_parts(parts), part_off, nullptr, nullptr, keep_mask};
    esc_expand_kernel<float, kEscCount><<<parts->P, kEscThreads, 0, st>>>(ea);
  }
  ESC_TRY(nacho_internal_launched("esc_expand_kernel (count)"));
  size_t tb = need;
  if (cub::DeviceScan::ExclusiveSum(ws, tb, part_off, part_off, (int64_t)parts->P + 1, st) != cudaSuccess)
    return efail(NACHO_ERR_CUDA, "SSSMM: scan of the partition counts");
  return nacho_internal_launched("esc_count_scan (cub)");
}

size_t nacho_sssmm_esc_workspace_size(const nacho_matrix* A, const nacho_matrix* B, int64_t n_kept) {
  return nacho_spgemm_esc_workspace_size(A, B, n_kept);
}

nacho_status nacho_sssmm_esc(const nacho_matrix* S, const nacho_matrix* A, const nacho_matrix* B, const int64_t* W,
                             const nacho_parts* parts, const int64_t* part_off, const uint8_t* keep_mask, int64_t n_kept,
                             int64_t* z_pos, int32_t* z_crd, void* z_val, int64_t* nnz_z, void* ws, size_t ws_bytes,
                             void* stream) {
  ESC_TRY(check_sample(S, A, B));
  ESC_TRY(check_esc_parts(parts));
  if (!W || !part_off || !keep_mask || !z_pos || !nnz_z || n_kept < 0 || (n_kept > 0 && (!z_crd || !z_val)))
    return efail(NACHO_ERR_INVALID_ARG, "null argument");
  const size_t need = nacho_sssmm_esc_workspace_size(A, B, n_kept);
  if (!ws || ws_bytes < need) return efail(NACHO_ERR_WORKSPACE, "nacho_sssmm_esc: workspace too small");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const EscOps o = make_esc(A, B, S, W);
  const int eb = bits_for(A->nrows) + o.jbits;
  auto* w8 = static_cast<unsigned char*>(ws);
  const size_t nn = (size_t)(n_kept > 0 ? n_kept : 1);
  if (A->dtype == NACHO_F64) {
    EscExpandArgs<double> ea{o, esc_parts(parts), const_cast<int64_t*>(part_off),
                             reinterpret_cast<unsigned long long*>(w8), reinterpret_cast<double*>(w8 + 2 * al(nn * 8)),
                             const_cast<uint8_t*>(keep_mask)};
    if (n_kept > 0) {
      esc_expand_kernel<double, kEscFill><<<parts->P, kEscThreads, 0, st>>>(ea);
      ESC_TRY(nacho_internal_launched("esc_expand_kernel (fill)"));
    }
    return sort_contract<double, true>(o, n_kept, eb, w8, z_pos, z_crd, static_cast<double*>(z_val), nnz_z, st);
  }
  EscExpandArgs<float> ea{o, esc_parts(parts), const_cast<int64_t*>(part_off), reinterpret_cast<unsigned long long*>(w8),
                          reinterpret_cast<float*>(w8 + 2 * al(nn * 8)), const_cast<uint8_t*>(keep_mask)};
  if (n_kept > 0) {
    esc_expand_kernel<float, kEscFill><<<parts->P, kEscThreads, 0, st>>>(ea);
    ESC_TRY(nacho_internal_launched("esc_expand_kernel (fill)"));
  }
  return sort_contract<float, true>(o, n_kept, eb, w8, z_pos, z_crd, static_cast<float*>(z_val), nnz_z, st);
}

}  // extern "C"
