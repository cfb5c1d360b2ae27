// api.cu -- the C ABI of libnacho.so (include/nacho.h): host-side validation, workspace carving
// and kernel launches.  Every numeric step runs in the kernels of the included headers.
#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "partition.cuh"
#include "spadd.cuh"
#include "spadd4.cuh"
#include "spadd5.cuh"
#include "spadd6.cuh"
#include "spadd7.cuh"
#include "dist.cuh"
#include "recursive.cuh"
#include "dcsr_add.cuh"
#include "csf.cuh"
#include "spmm.cuh"
#include "spmv.cuh"
#include "spmv3.cuh"
#include "spmv7.cuh"

using namespace nacho;

namespace {

thread_local std::string g_err;
thread_local int64_t g_launches = 0;

nacho_status fail(nacho_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

nacho_status launched(const char* what) {
  ++g_launches;
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(NACHO_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return NACHO_SUCCESS;
}

#define NACHO_TRY(x)                          \
  do {                                        \
    const nacho_status _s = (x);              \
    if (_s != NACHO_SUCCESS) return _s;       \
  } while (0)

constexpr int kSpaddThreads = 256;
constexpr int kSpaddTile = 2048;  // entries (summed over operands) per CTA chunk
constexpr int kSpmmWarps = 8;
constexpr int kSpmmWitems = 128;  // 1024 positions per CTA
#ifndef NACHO_PART_WARPS   // tuning override
#define NACHO_PART_WARPS 4
#endif
constexpr int kPartWarps = NACHO_PART_WARPS;

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

// The > 48 KB dynamic shared-memory opt-in is a per-device function attribute: set it once per
// device (bit d of `done`), race-free across host threads (setting it twice is harmless).
template <typename F>
nacho_status smem_optin(F kern, size_t smem, std::atomic<uint64_t>& done, const char* name) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return fail(NACHO_ERR_CUDA, "cudaGetDevice");
  const uint64_t bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return NACHO_SUCCESS;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return fail(NACHO_ERR_CUDA, "cudaFuncSetAttribute(%s)", name);
  done.fetch_or(bit, std::memory_order_acq_rel);
  return NACHO_SUCCESS;
}

int spmv_impl() {   // 3: one tile per CTA (spmv3.cuh, default); 7: the experimental pipelined spmv7.cuh
  static const int impl = [] {
    const char* e = getenv("NACHO_SPMV_IMPL");
    return e && e[0] == '7' ? 7 : 3;
  }();
  return impl;
}
int64_t spmv_tile(int dtype) {   // positions per tile of the SpMV kernel in use (= the auto partition size)
  if (spmv_impl() == 7) return dtype == NACHO_F64 ? sv7_tile<double>() : sv7_tile<float>();
  return dtype == NACHO_F64 ? sv3_tile<double>() : sv3_tile<float>();
}

nacho_status check_matrix(const nacho_matrix* A, const char* name) {
  if (!A) return fail(NACHO_ERR_INVALID_ARG, "%s: null descriptor", name);
  if (A->format != NACHO_CSR && A->format != NACHO_DCSR && A->format != NACHO_COO)
    return fail(NACHO_ERR_INVALID_ARG, "%s: bad format %d", name, A->format);
  if (A->format == NACHO_COO && (A->nouter != 1 || (A->nnz > 0 && !A->outer_crd)))
    return fail(NACHO_ERR_SHAPE, "%s: COO needs nouter == 1 (pos = [0, nnz]) and a row level", name);
  if (A->dtype != NACHO_F32 && A->dtype != NACHO_F64) return fail(NACHO_ERR_INVALID_ARG, "%s: bad dtype %d", name, A->dtype);
  if (A->nrows < 0 || A->ncols < 0 || A->nnz < 0 || A->nouter < 0) return fail(NACHO_ERR_SHAPE, "%s: negative size", name);
  if (A->ncols > INT32_MAX) return fail(NACHO_ERR_OVERFLOW, "%s: ncols %lld > INT32_MAX", name, (long long)A->ncols);
  if (A->nrows > INT32_MAX) return fail(NACHO_ERR_OVERFLOW, "%s: nrows > INT32_MAX (local row spans are 32-bit)", name);
  if (A->format == NACHO_CSR && A->nouter != A->nrows) return fail(NACHO_ERR_SHAPE, "%s: CSR needs nouter == nrows", name);
  if (A->format == NACHO_DCSR && A->nouter > A->nrows) return fail(NACHO_ERR_SHAPE, "%s: DCSR nouter > nrows", name);
  if (!A->pos) return fail(NACHO_ERR_INVALID_ARG, "%s: null pos", name);
  if (A->nnz > 0 && (!A->crd || !A->val)) return fail(NACHO_ERR_INVALID_ARG, "%s: null crd/val", name);
  if (A->format == NACHO_DCSR && A->nouter > 0 && !A->outer_crd) return fail(NACHO_ERR_INVALID_ARG, "%s: null outer_crd", name);
  return NACHO_SUCCESS;
}

nacho_status check_ops(const nacho_matrix* ops, int32_t k) {
  if (!ops) return fail(NACHO_ERR_INVALID_ARG, "null operand array");
  if (k < 1 || k > NACHO_MAX_K) return fail(NACHO_ERR_INVALID_ARG, "k = %d outside [1, %d]", k, NACHO_MAX_K);
  for (int o = 0; o < k; ++o) {
    NACHO_TRY(check_matrix(ops + o, "operand"));
    const bool dense_rows = ops[o].format != NACHO_DCSR && ops[0].format != NACHO_DCSR;   // CSR / COO mix
    if ((ops[o].format != ops[0].format && !dense_rows) || ops[o].nrows != ops[0].nrows ||
        ops[o].ncols != ops[0].ncols || ops[o].dtype != ops[0].dtype)
      return fail(NACHO_ERR_SHAPE, "operand %d disagrees with operand 0 in format/shape/dtype", o);
  }
  if (ops[0].format == NACHO_DCSR && k > 4) return fail(NACHO_ERR_INVALID_ARG, "DCSR partitioning supports k <= 4");
  return NACHO_SUCCESS;
}

bool all_csr(const nacho_matrix* ops, int32_t k) {
  for (int o = 0; o < k; ++o) if (ops[o].format != NACHO_CSR) return false;
  return true;
}

OpsArg make_ops(const nacho_matrix* ops, int32_t k) {
  OpsArg a;
  memset(&a, 0, sizeof(a));
  a.k = k;
  a.dtype = ops[0].dtype;
  a.nrows = ops[0].nrows;
  a.ncols = ops[0].ncols;
  for (int o = 0; o < k; ++o) {
    a.op[o].pos = ops[o].pos;
    a.op[o].crd = ops[o].crd;
    a.op[o].val = ops[o].val;
    a.op[o].fmt = ops[o].format;
    a.op[o].outer = ops[o].format != NACHO_CSR ? ops[o].outer_crd : nullptr;
    a.op[o].nouter = ops[o].nouter;
    a.op[o].nnz = ops[o].nnz;
  }
  a.pos_shared = 1;
  for (int o = 1; o < k; ++o)
    if (ops[o].pos != ops[0].pos) a.pos_shared = 0;
  return a;
}

int64_t total_cost(const nacho_matrix* ops, int32_t k) {  // a1: Q* = sum_o nnz_o
  int64_t q = 0;
  for (int o = 0; o < k; ++o) q += ops[o].nnz;
  return q;
}

size_t parts_bytes(int64_t P, int k) {
  return align_up((P + 1) * 8) * 3 + align_up((P + 1) * 4) + align_up((P + 1) * 8 * k);
}

PartsArg carve_parts(void* ws, int64_t P, int k) {
  char* c = static_cast<char*>(ws);
  PartsArg pa;
  pa.P = (int32_t)P;
  pa.k = k;
  pa.max_work = 0;
  pa.query = reinterpret_cast<int64_t*>(c); c += align_up((P + 1) * 8);
  pa.row = reinterpret_cast<int64_t*>(c); c += align_up((P + 1) * 8);
  pa.row_pos = reinterpret_cast<int64_t*>(c); c += align_up((P + 1) * 8);
  pa.col = reinterpret_cast<int32_t*>(c); c += align_up((P + 1) * 4);
  pa.pos = reinterpret_cast<int64_t*>(c);
  return pa;
}

PartsArg parts_arg(const nacho_parts* p) {
  PartsArg pa;
  pa.P = p->P; pa.k = p->k; pa.query = p->query; pa.row = p->row; pa.row_pos = p->row_pos;
  pa.col = p->col; pa.pos = p->pos; pa.max_work = p->max_work;
  return pa;
}

int64_t max_part_work(const nacho_matrix* ops, int32_t k, const PartsArg& pa, int64_t limit, cudaStream_t st);

nacho_status check_parts(const nacho_parts* p, int32_t k) {
  if (!p) return fail(NACHO_ERR_INVALID_ARG, "null parts");
  if (p->P < 1) return fail(NACHO_ERR_INVALID_ARG, "parts.P = %d < 1", p->P);
  if (p->k != k) return fail(NACHO_ERR_INVALID_ARG, "parts.k = %d, expected %d", p->k, k);
  if (!p->query || !p->row || !p->row_pos || !p->col || !p->pos) return fail(NACHO_ERR_INVALID_ARG, "parts: null array");
  return NACHO_SUCCESS;
}

// Boundaries p0 .. p0 + pa.P of the Ptot-partition into pa (whole partition: p0 = 0, Ptot = pa.P).
nacho_status launch_partition(const nacho_matrix* ops, int32_t k, const PartsArg& pa, cudaStream_t st,
                              int64_t Ptot = -1, int64_t p0 = 0) {
  const OpsArg a = make_ops(ops, k);
  if (Ptot < 0) Ptot = pa.P;
  const int64_t q = total_cost(ops, k);
  bool levels = ops[0].format == NACHO_DCSR && k > 1;
  for (int o = 0; o < k; ++o) levels = levels || ops[o].format == NACHO_COO;
  if (levels) {   // k compressed / COO outer levels (dcsr_add.cuh)
    if (Ptot != pa.P || p0 != 0) return fail(NACHO_ERR_INVALID_ARG, "partition slices take CSR (or one DCSR) operands");
    if (k > 4) return fail(NACHO_ERR_INVALID_ARG, "DCSR / COO partitioning takes k <= 4 operands");
    const unsigned g = (unsigned)((int64_t(pa.P) + 4) / 4);
    if (k <= 2) dcsr_partition_kernel<2><<<g, 128, 0, st>>>(a, pa, q);
    else dcsr_partition_kernel<4><<<g, 128, 0, st>>>(a, pa, q);
    return launched("dcsr_partition_kernel");
  }
  if (k == 1) {
    partition1_kernel<<<(unsigned)((int64_t(pa.P) + 256) / 256), 256, 0, st>>>(a, pa, q, Ptot, p0);
    return launched("partition1_kernel");
  }
  const int64_t nb = (int64_t(pa.P) + 1 + kPartWarps - 1) / kPartWarps;
  if (k == 2) partition_kernel<kPartWarps, 2><<<(unsigned)nb, kPartWarps * 32, 0, st>>>(a, pa, q, Ptot, p0);
  else if (k == 3) partition_kernel<kPartWarps, 3><<<(unsigned)nb, kPartWarps * 32, 0, st>>>(a, pa, q, Ptot, p0);
  else if (k == 4) partition_kernel<kPartWarps, 4><<<(unsigned)nb, kPartWarps * 32, 0, st>>>(a, pa, q, Ptot, p0);
  else partition_kernel<kPartWarps, NACHO_MAX_K><<<(unsigned)nb, kPartWarps * 32, 0, st>>>(a, pa, q, Ptot, p0);
  return launched("partition_kernel");
}

// Carries of an SpMV over P partitions made by nacho_partition (work <= ceil(nnz / P)): one per
// tile-sized chunk.
int64_t spmv_carry_cap(const nacho_matrix* A, int64_t P) {
  const int64_t tile = spmv_tile(A->dtype);
  const int64_t w = (A->nnz + P - 1) / P;
  return P * (w <= tile ? 1 : (w + tile - 1) / tile);
}

int32_t auto_p(int64_t work, int64_t tile) {
  int64_t P = (work + tile - 1) / tile;
  if (P < 1) P = 1;
  if (P > INT32_MAX - 1) P = INT32_MAX - 1;
  return (int32_t)P;
}

template <typename T, bool DY>
nacho_status launch_spmv7(const SpmvArgs<T>& a, cudaStream_t st) {
  auto kern = spmv7_kernel<T, DY>;
  const size_t smem = sizeof(Sv7Smem<T>);
  static std::atomic<uint64_t> done{0};   // per instantiation: the opt-in is per kernel and device
  NACHO_TRY(smem_optin(kern, smem, done, "spmv7_kernel"));
  int dev = 0, sms = 0, per = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, kSv7Threads, smem) != cudaSuccess || per < 1)
    return fail(NACHO_ERR_CUDA, "spmv7 occupancy query");
  const int64_t grid = std::min<int64_t>(a.P, (int64_t)sms * per);
  kern<<<(unsigned)grid, kSv7Threads, smem, st>>>(a, (int64_t)a.P);
  return launched("spmv7_kernel");
}

template <typename T>
nacho_status run_spmv(const nacho_matrix* A, const PartsArg& pa, const void* x, void* y, int32_t dense_y,
                      char* ws_carry, int64_t carry_cap, cudaStream_t st) {
  SpmvArgs<T> a;
  a.pos = A->pos; a.crd = A->crd; a.val = static_cast<const T*>(A->val);
  a.outer = A->format == NACHO_DCSR ? A->outer_crd : nullptr;
  a.nouter = A->nouter;
  a.ncols = A->ncols;
  a.x = static_cast<const T*>(x); a.y = static_cast<T*>(y);
  a.dense_y = (A->format == NACHO_DCSR && dense_y) ? 1 : 0;
  a.ppos = pa.pos; a.prow = pa.row_pos;
  // partitions larger than a tile run as tile-sized chunks (one CTA each, spmv3.cuh)
  const bool aligned = reinterpret_cast<uintptr_t>(A->crd) % 16 == 0 && reinterpret_cast<uintptr_t>(A->val) % 16 == 0 &&
                       reinterpret_cast<uintptr_t>(A->pos) % 16 == 0;
  const bool use7 = spmv_impl() == 7 && aligned && A->nnz > 0;
  const int64_t tile = use7 ? sv7_tile<T>() : sv3_tile<T>();
  const int64_t maxpart = max_part_work(A, 1, pa, tile, st);
  const int64_t chunks = maxpart <= tile ? 1 : (maxpart + tile - 1) / tile;
  if (int64_t(pa.P) * chunks > carry_cap)
    return fail(NACHO_ERR_WORKSPACE, "partitions of up to %lld positions need %lld carries, workspace holds %lld",
                (long long)maxpart, (long long)(int64_t(pa.P) * chunks), (long long)carry_cap);
  a.chunks = (int32_t)chunks;
  a.P = (int32_t)(int64_t(pa.P) * chunks);
  a.carry_row = reinterpret_cast<int64_t*>(ws_carry);
  a.carry_val = reinterpret_cast<T*>(ws_carry + align_up(carry_cap * 8));
  if (a.dense_y) {
    if (cudaMemsetAsync(y, 0, sizeof(T) * A->nrows, st) != cudaSuccess) return fail(NACHO_ERR_CUDA, "memset y");
  }
  if (use7) {   // persistent, bulk-copy pipelined (spmv7.cuh)
    NACHO_TRY((a.dense_y ? launch_spmv7<T, true>(a, st) : launch_spmv7<T, false>(a, st)));
  } else {
    if (a.dense_y) spmv3_kernel<T, true><<<(unsigned)a.P, kSv3Threads, 0, st>>>(a);
    else spmv3_kernel<T, false><<<(unsigned)a.P, kSv3Threads, 0, st>>>(a);
    NACHO_TRY(launched("spmv3_kernel"));
  }
  const int64_t warps = (int64_t(a.P) + 31) / 32;
  spmv_fixup_kernel<T><<<(unsigned)((warps + 7) / 8), 256, 0, st>>>(a);
  return launched("spmv_fixup_kernel");
}

template <typename T, bool FILL>
nacho_status launch_spadd(const SpaddArgs<T>& a, cudaStream_t st) {
  auto kern = spadd_kernel<T, FILL, kSpaddThreads, kSpaddTile>;
  const size_t smem = ((sizeof(SpaddShared<kSpaddThreads>) + 15) & ~size_t(15)) + 3 * kSpaddTile * 8 +
                      (FILL ? 3 * kSpaddTile * sizeof(T) : 0);
  static std::atomic<uint64_t> done{0};
  NACHO_TRY(smem_optin(kern, smem, done, "spadd_kernel"));
  kern<<<a.parts.P, kSpaddThreads, smem, st>>>(a);
  return launched(FILL ? "spadd_fill_kernel" : "spadd_count_kernel");
}

template <typename T, int MODE, int KM, bool CHK>
nacho_status launch_spadd4_k(const Spadd4Args<T>& a, cudaStream_t st, int64_t grid) {
  auto kern = spadd4_kernel<T, MODE, KM, CHK>;
  const size_t smem = sizeof(S4Shared<T, s4_small(MODE, KM)>);
  static std::atomic<uint64_t> done{0};
  NACHO_TRY(smem_optin(kern, smem, done, "spadd4_kernel"));
  kern<<<(unsigned)grid, kS4Threads, smem, st>>>(a);
  return launched(MODE == kS4Count ? "spadd4_count" : MODE == kS4Fill ? "spadd4_fill" : MODE == kS4Fused ? "spadd4_fused" : "spadd4_stage");
}

// One CTA per partition (spadd4.cuh); shared memory is dynamic (> 48 KB).  k = 2, 3 (and 1) get
// compile-time operand loops; other k the generic instantiation.
template <typename T, int MODE>
nacho_status launch_spadd4(const Spadd4Args<T>& a, cudaStream_t st, int64_t grid = -1) {
  if (grid < 0) grid = a.parts.P;
  if (MODE == kS4Stage && a.chunks > 1) {
    switch (a.ops.k) {
      case 1: return launch_spadd4_k<T, MODE, 1, true>(a, st, grid);
      case 2: return launch_spadd4_k<T, MODE, 2, true>(a, st, grid);
      case 3: return launch_spadd4_k<T, MODE, 3, true>(a, st, grid);
      default: return launch_spadd4_k<T, MODE, NACHO_MAX_K, true>(a, st, grid);
    }
  }
  switch (a.ops.k) {
    case 1: return launch_spadd4_k<T, MODE, 1, false>(a, st, grid);
    case 2: return launch_spadd4_k<T, MODE, 2, false>(a, st, grid);
    case 3: return launch_spadd4_k<T, MODE, 3, false>(a, st, grid);
    default: return launch_spadd4_k<T, MODE, NACHO_MAX_K, false>(a, st, grid);
  }
}

// Largest possible partition of a k-operand partition with P parts (Theorem 1 slack k-1).
// Upper bound of the work of one partition of a k-operand partition record: ceil(span/P) + k - 1
// (Theorem 1 slack), span = Q* for a whole record.  A record that is a slice of a finer one (the
// device cuts of dist.py) has a smaller span: when the cheap bound fails, the span is read from the
// record's first and last query (a synchronising 16-byte copy).
int64_t max_part_work(const nacho_matrix* ops, int32_t k, const PartsArg& pa, int64_t limit, cudaStream_t st) {
  if (pa.max_work > 0) return pa.max_work;   // recorded by the partition call: no device read
  const int64_t q = total_cost(ops, k);
  int64_t w = (q + pa.P - 1) / pa.P + (k - 1);
  if (w <= limit || pa.P < 1) return w;
  int64_t ends[2] = {0, q};
  if (cudaMemcpyAsync(&ends[0], pa.query, 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaMemcpyAsync(&ends[1], pa.query + pa.P, 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return w;
  return (ends[1] - ends[0] + pa.P - 1) / pa.P + (k - 1);
}

bool fits_sa_tile(const nacho_matrix* ops, int32_t k, const nacho_parts* parts, cudaStream_t st) {
  return max_part_work(ops, k, parts_arg(parts), kS4Tile, st) <= kS4Tile;
}

template <typename T, int CPL, bool VEC>
nacho_status launch_spmm(const SpmmArgs<T>& a, cudaStream_t st) {
  spmm_kernel<T, CPL, VEC, kSpmmWarps, kSpmmWitems><<<a.P, kSpmmWarps * 32, 0, st>>>(a);
  NACHO_TRY(launched("spmm_kernel"));
  const int64_t warps = (a.P + 31) / 32;
  spmm_fixup_kernel<T><<<(unsigned)((warps + 7) / 8), 256, 0, st>>>(a);
  return launched("spmm_fixup_kernel");
}

template <typename T>
nacho_status run_spmm(SpmmArgs<T> a, cudaStream_t st, int64_t maxpart, int64_t carry_cap) {
  a.chunks = 1;
  if constexpr (sizeof(T) == 4) {
    const bool al = reinterpret_cast<uintptr_t>(a.B) % 16 == 0 && reinterpret_cast<uintptr_t>(a.C) % 16 == 0 &&
                    a.ldb % 4 == 0 && a.ldc % 4 == 0;
    if (a.nb == 64 && al) {  // eight-lane-group fast path; larger partitions as tile-sized chunks
      const int64_t chunks = maxpart <= kSm2Tile ? 1 : (maxpart + kSm2Tile - 1) / kSm2Tile;
      if (int64_t(a.P) * chunks <= carry_cap) {
        a.chunks = (int32_t)chunks;
        a.P = (int32_t)(int64_t(a.P) * chunks);
        if (chunks > 1) spmm64_kernel<true><<<(unsigned)a.P, 256, 0, st>>>(a);
        else spmm64_kernel<false><<<(unsigned)a.P, 256, 0, st>>>(a);
        NACHO_TRY(launched("spmm64_kernel"));
        const int64_t warps = (int64_t(a.P) + 31) / 32;
        spmm_fixup_kernel<T><<<(unsigned)((warps + 7) / 8), 256, 0, st>>>(a);
        return launched("spmm_fixup_kernel");
      }
    }
  }
  const int cpl = a.nb <= 32 ? 1 : a.nb <= 64 ? 2 : a.nb <= 128 ? 4 : 8;
  const bool vec = (reinterpret_cast<uintptr_t>(a.B) % (cpl * sizeof(T)) == 0) && (a.ldb % cpl == 0);
  switch (cpl) {
    case 1: return launch_spmm<T, 1, false>(a, st);
    case 2: return vec ? launch_spmm<T, 2, true>(a, st) : launch_spmm<T, 2, false>(a, st);
    case 4:
      if (sizeof(T) == 4) return vec ? launch_spmm<T, 4, true>(a, st) : launch_spmm<T, 4, false>(a, st);
      return launch_spmm<T, 4, false>(a, st);
    default: return launch_spmm<T, 8, false>(a, st);
  }
}

__global__ void validate_kernel(nacho_matrix A, int* flag) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i > A.nouter) return;
  int bad = 0;
  if (i == 0 && A.pos[0] != 0) bad = 1;
  if (i == A.nouter && A.pos[A.nouter] != A.nnz) bad = 2;
  if (i < A.nouter) {
    const int64_t s = A.pos[i], e = A.pos[i + 1];
    if (e < s || s < 0 || e > A.nnz) bad = 3;
    else {
      for (int64_t q = s; q < e && !bad; ++q) {
        const int32_t c = A.crd[q];
        if (c < 0 || c >= A.ncols) bad = 4;
        if (q > s && c <= A.crd[q - 1]) bad = 5;
      }
    }
    if (A.format == NACHO_DCSR) {
      const int32_t r = A.outer_crd[i];
      if (r < 0 || r >= A.nrows) bad = 6;
      if (i > 0 && r <= A.outer_crd[i - 1]) bad = 7;
      if (e == s) bad = 8;
    }
  }
  if (bad) atomicMax(flag, bad);
}

// Chunks per partition of the staged SpAdd: 1 when every partition fits a tile, else enough
// kS4Tile - (k - 1) query-wide chunks for the largest partition (work <= max_work).
int64_t staged_chunks(int64_t max_work, int32_t k) {
  if (max_work <= kS4Tile) return 1;
  const int64_t tq = kS4Tile - (k - 1);
  return (max_work + tq - 1) / tq;
}

struct StagedWs {   // carving of the staged workspace for nchunk chunks
  int64_t* cnt; unsigned long long* blk; int64_t* blk_off; int64_t* prov; int64_t* rows; char* stage;
};
size_t staged_ws_layout(int64_t nchunk, char* ws, StagedWs* out) {
  size_t o = 0;
  auto take = [&](size_t bytes) { const size_t at = o; o += align_up(bytes); return at; };
  const size_t c = take((size_t)(nchunk + 1) * 8), b = take((size_t)((nchunk >> kS4BlkShift) + 1) * 8),
               bo = take((size_t)((nchunk >> kS4BlkShift) + 2) * 8),
               pv = take((size_t)nchunk * 8), r = take((size_t)nchunk * 16);
  if (out) {
    out->cnt = reinterpret_cast<int64_t*>(ws + c);
    out->blk = reinterpret_cast<unsigned long long*>(ws + b);
    out->blk_off = reinterpret_cast<int64_t*>(ws + bo);
    out->prov = reinterpret_cast<int64_t*>(ws + pv);
    out->rows = reinterpret_cast<int64_t*>(ws + r);
    out->stage = ws + o;
  }
  return o;
}

template <typename T>
nacho_status run_spadd_staged(const nacho_matrix* ops, int32_t k, const nacho_parts* parts, int64_t* part_off,
                              int64_t* z_pos, int32_t* z_crd, T* z_val, char* ws, int64_t chunks, cudaStream_t st) {
  const int64_t q = total_cost(ops, k);
  const int64_t nchunk = (int64_t)parts->P * chunks;
  StagedWs w;
  staged_ws_layout(nchunk, ws, &w);
  int32_t* t_crd = reinterpret_cast<int32_t*>(w.stage);
  T* t_val = reinterpret_cast<T*>(w.stage + align_up((size_t)q * 4));
  if (cudaMemsetAsync(w.blk, 0, sizeof(unsigned long long) * ((nchunk >> kS4BlkShift) + 1), st) != cudaSuccess)
    return fail(NACHO_ERR_CUDA, "memset block sums");
  Spadd4Args<T> a{make_ops(ops, k), parts_arg(parts), w.cnt, part_off, nullptr, nullptr, z_pos, t_crd, t_val, w.blk,
                  (int32_t)chunks, w.prov, w.rows};
  NACHO_TRY((launch_spadd4<T, kS4Stage>(a, st, nchunk)));
  // the block sums -> their exclusive prefix (one small scan: every placement CTA then reads one value
  // instead of summing all preceding blocks, O(nchunk) instead of O(nchunk^2 / 512) loads)
  const int64_t nblk = ((nchunk - 1) >> kS4BlkShift) + 1;
  scan_counts_kernel<1024><<<1, 1024, 0, st>>>(reinterpret_cast<const int64_t*>(w.blk), nblk, w.blk_off);
  NACHO_TRY(launched("scan_counts_kernel (block sums)"));
  Spadd4Args<T> c = a;
  c.blk_cnt = reinterpret_cast<unsigned long long*>(w.blk_off);   // the placement reads the prefix
  c.z_crd = z_crd;
  c.z_val = z_val;
  s4_place_kernel<T><<<(unsigned)nchunk, kS4Threads, 0, st>>>(c, t_crd, t_val);
  return launched("s4_place_kernel");
}

// Single-read SpAdd (spadd5.cuh): key column bits and the rows per sub-tile.
int s5_cb(int64_t ncols) {
  int cb = 1;
  while (cb < 31 && (int64_t(1) << cb) < ncols) ++cb;
  return cb;
}

bool spadd5_applies(const nacho_matrix* ops, int32_t k, const PartsArg& pa, cudaStream_t st) {
  if (s5_cb(ops[0].ncols) > 24) return false;   // < 256 rows per sub-tile: the spadd4 path
  return max_part_work(ops, k, pa, s5_max_entries(k), st) <= s5_max_entries(k);
}

template <typename T, int K>
nacho_status launch_spadd5_k(const S5Args<T>& a, cudaStream_t st) {
#ifdef NACHO_SPADD5   // one CTA per partition (spadd5.cuh)
  auto kern = spadd5_kernel<T, K>;
  const size_t smem = sizeof(S5Smem<T, K>);
  static std::atomic<uint64_t> done{0};
  NACHO_TRY(smem_optin(kern, smem, done, "spadd5_kernel"));
  kern<<<(unsigned)a.parts.P, kS5Threads, smem, st>>>(a);
  return launched("spadd5_kernel");
#else                 // persistent, warp-specialised (spadd6.cuh): grid = resident CTAs
  auto kern = spadd6_kernel<T, K>;
  const size_t smem = sizeof(S6Smem<T, K>);
  static std::atomic<uint64_t> done{0};
  NACHO_TRY(smem_optin(kern, smem, done, "spadd6_kernel"));
  int dev = 0, sms = 0, per = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, kS6Threads, smem) != cudaSuccess || per < 1)
    return fail(NACHO_ERR_CUDA, "spadd6 occupancy query");
  const int64_t grid = std::min<int64_t>(a.parts.P, (int64_t)sms * per);
  kern<<<(unsigned)grid, kS6Threads, smem, st>>>(a);
  return launched("spadd6_kernel");
#endif
}

template <typename T>
nacho_status run_spadd5(const nacho_matrix* ops, int32_t k, const nacho_parts* parts, int64_t* part_off, int64_t* z_pos,
                        int32_t* z_crd, T* z_val, unsigned long long* state, cudaStream_t st) {
  S5Args<T> a;
  a.ops = make_ops(ops, k);
  a.parts = parts_arg(parts);
  a.cb = s5_cb(ops[0].ncols);
  const int64_t lm = (int64_t(1) << (32 - a.cb)) - 1;
  a.lmax = (int32_t)(lm < kS5LMax ? lm : kS5LMax);
  a.use_bulk = 1;
  for (int o = 0; o < k; ++o)
    if (reinterpret_cast<uintptr_t>(ops[o].crd) % 16 || reinterpret_cast<uintptr_t>(ops[o].val) % 16) a.use_bulk = 0;
  a.state = state;
  a.part_off = part_off;
  a.z_pos = z_pos;
  a.z_crd = z_crd;
  a.z_val = z_val;
  if (cudaMemsetAsync(state, 0, sizeof(unsigned long long) * (parts->P + 1), st) != cudaSuccess)
    return fail(NACHO_ERR_CUDA, "memset look-back states");
  switch (k) {
    case 1: return launch_spadd5_k<T, 1>(a, st);
    case 2: return launch_spadd5_k<T, 2>(a, st);
    case 3: return launch_spadd5_k<T, 3>(a, st);
    case 4: return launch_spadd5_k<T, 4>(a, st);
    case 5: return launch_spadd5_k<T, 5>(a, st);
    case 6: return launch_spadd5_k<T, 6>(a, st);
    case 7: return launch_spadd5_k<T, 7>(a, st);
    default: return launch_spadd5_k<T, 8>(a, st);
  }
}

// Pipelined single-read SpAdd (spadd7.cuh): producer / compute / emission warps over NS stages.
template <typename T, int K, int OP = kS7Union>
nacho_status launch_spadd7_k(const S7Args<T>& a, cudaStream_t st) {
  auto kern = spadd7_kernel<T, K, OP>;
  const size_t smem = sizeof(S7Smem<T, K>);
  static std::atomic<uint64_t> done{0};
  NACHO_TRY(smem_optin(kern, smem, done, "spadd7_kernel"));
  int dev = 0, sms = 0, per = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, kS7Threads, smem) != cudaSuccess || per < 1)
    return fail(NACHO_ERR_CUDA, "spadd7 occupancy query");
  const int64_t grid = std::min<int64_t>(a.parts.P, (int64_t)sms * per);
  kern<<<(unsigned)grid, kS7Threads, smem, st>>>(a);
  return launched("spadd7_kernel");
}

template <typename T, int OP = kS7Union>
nacho_status run_spadd7(const nacho_matrix* ops, int32_t k, const nacho_parts* parts, int64_t* part_off, int64_t* z_pos,
                        int32_t* z_crd, T* z_val, unsigned long long* state, cudaStream_t st, double* partial = nullptr) {
  S7Args<T> a;
  memset(&a, 0, sizeof(a));
  a.ops = make_ops(ops, k);
  a.parts = parts_arg(parts);
  a.cb = s5_cb(ops[0].ncols);
  a.ndist = 0;
  a.use_bulk = 1;
  for (int o = 0; o < k; ++o) {
    int d = 0;
    while (d < a.ndist && a.dpos[d] != ops[o].pos) ++d;   // operands sharing one pos array: one copy
    if (d == a.ndist) a.dpos[a.ndist++] = ops[o].pos;
    a.pd[o] = d;
    if (reinterpret_cast<uintptr_t>(ops[o].crd) % 16 || reinterpret_cast<uintptr_t>(ops[o].val) % 16 ||
        reinterpret_cast<uintptr_t>(ops[o].pos) % 16)
      a.use_bulk = 0;
  }
  a.sp = (kS7PosPool / a.ndist) & ~1;
  int64_t lm = (int64_t(1) << (32 - a.cb)) - 2;
  if (lm > a.sp - 2) lm = a.sp - 2;
  if (lm > kS7LMax) lm = kS7LMax;
  a.lmax = (int32_t)lm;
  a.state = state;
  a.part_off = part_off;
  a.z_pos = z_pos;
  a.z_crd = z_crd;
  a.z_val = z_val;
  a.partial = partial;
#ifdef NACHO_S7_PROF
  const int nclear = parts->P + 2 + 16;
#else
  const int nclear = parts->P + 2;
#endif
  if (cudaMemsetAsync(state, 0, sizeof(unsigned long long) * nclear, st) != cudaSuccess)
    return fail(NACHO_ERR_CUDA, "memset look-back states");
  if constexpr (OP != kS7Union) {   // intersections: k <= 4 instantiated
    switch (k) {
      case 1: return launch_spadd7_k<T, 1, OP>(a, st);
      case 2: return launch_spadd7_k<T, 2, OP>(a, st);
      case 3: return launch_spadd7_k<T, 3, OP>(a, st);
      case 4: return launch_spadd7_k<T, 4, OP>(a, st);
      default: return fail(NACHO_ERR_INVALID_ARG, "intersection kernels take k <= 4 operands (k = %d)", k);
    }
  } else {
    switch (k) {
      case 1: return launch_spadd7_k<T, 1>(a, st);
      case 2: return launch_spadd7_k<T, 2>(a, st);
      case 3: return launch_spadd7_k<T, 3>(a, st);
      case 4: return launch_spadd7_k<T, 4>(a, st);
      case 5: return launch_spadd7_k<T, 5>(a, st);
      case 6: return launch_spadd7_k<T, 6>(a, st);
      case 7: return launch_spadd7_k<T, 7>(a, st);
      default: return launch_spadd7_k<T, 8>(a, st);
    }
  }
}

// Which single-read kernel nacho_spadd_k runs: 7 (pipelined, default) or 6 (NACHO_SPADD_IMPL=6;
// A/B comparisons only).
int spadd_impl() {
  static const int impl = [] {
    const char* e = getenv("NACHO_SPADD_IMPL");
    return e && e[0] == '6' ? 6 : 7;
  }();
  return impl;
}

}  // namespace

// status plumbing for the other translation units of the library (esc.cu)
nacho_status nacho_internal_fail(nacho_status s, const char* msg) { return fail(s, "%s", msg); }
nacho_status nacho_internal_launched(const char* what) { return launched(what); }

extern "C" {

/* ------------------------------------------------------------------ k-way intersection (spadd7, OP) */
static nacho_status check_intersection(const nacho_matrix* ops, int32_t k, const nacho_parts* parts, cudaStream_t st) {
  NACHO_TRY(check_ops(ops, k));
  if (!all_csr(ops, k)) return fail(NACHO_ERR_INVALID_ARG, "intersection kernels take CSR operands");
  if (k > 4) return fail(NACHO_ERR_INVALID_ARG, "intersection kernels take k <= 4 operands (k = %d)", k);
  NACHO_TRY(check_parts(parts, k));
  if (!spadd5_applies(ops, k, parts_arg(parts), st))
    return fail(NACHO_ERR_INVALID_ARG, "partitions larger than %d entries (or > 2^24 columns): use P >= "
                "nacho_auto_partitions(ops, k, 1)", s5_max_entries(k));
  return NACHO_SUCCESS;
}

nacho_status nacho_hadamard_k(const nacho_matrix* ops, int32_t k, const nacho_parts* parts, int64_t* part_off,
                              int64_t* z_pos, int32_t* z_crd, void* z_val, void* ws, size_t ws_bytes, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  NACHO_TRY(check_intersection(ops, k, parts, st));
  if (!z_pos) return fail(NACHO_ERR_INVALID_ARG, "null z_pos");
  if (total_cost(ops, k) > 0 && (!z_crd || !z_val)) return fail(NACHO_ERR_INVALID_ARG, "null z_crd / z_val");
  const size_t need = nacho_spadd_k_workspace_size(ops, k, parts->P);
  if (ws_bytes < need || !ws) return fail(NACHO_ERR_WORKSPACE, "workspace %zu < %zu bytes", ws_bytes, need);
  auto* flags = static_cast<unsigned long long*>(ws);
  if (ops[0].dtype == NACHO_F64)
    return run_spadd7<double, kS7Inter>(ops, k, parts, part_off, z_pos, z_crd, static_cast<double*>(z_val), flags, st);
  return run_spadd7<float, kS7Inter>(ops, k, parts, part_off, z_pos, z_crd, static_cast<float*>(z_val), flags, st);
}

size_t nacho_inner_k_workspace_size(const nacho_matrix* ops, int32_t k, int32_t P) {
  return nacho_spadd_k_workspace_size(ops, k, P) + align_up((size_t)(P > 0 ? P : 1) * 8);
}

nacho_status nacho_inner_k(const nacho_matrix* ops, int32_t k, const nacho_parts* parts, double* result, void* ws,
                           size_t ws_bytes, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  NACHO_TRY(check_intersection(ops, k, parts, st));
  if (!result) return fail(NACHO_ERR_INVALID_ARG, "null result");
  const size_t need = nacho_inner_k_workspace_size(ops, k, parts->P);
  if (ws_bytes < need || !ws) return fail(NACHO_ERR_WORKSPACE, "workspace %zu < %zu bytes", ws_bytes, need);
  auto* flags = static_cast<unsigned long long*>(ws);
  double* partial = reinterpret_cast<double*>(static_cast<char*>(ws) + nacho_spadd_k_workspace_size(ops, k, parts->P));
  nacho_status r = ops[0].dtype == NACHO_F64
                       ? run_spadd7<double, kS7InterSum>(ops, k, parts, nullptr, nullptr, nullptr, nullptr, flags, st, partial)
                       : run_spadd7<float, kS7InterSum>(ops, k, parts, nullptr, nullptr, nullptr, nullptr, flags, st, partial);
  NACHO_TRY(r);
  s7_sum_partials_kernel<<<1, 1024, 0, st>>>(partial, parts->P, result);
  return launched("s7_sum_partials_kernel");
}

/* ------------------------------------------------------------------ recursive partitioning (Alg. 2) */
namespace {
struct RecLayout {
  int64_t P1, cap;
  size_t pos_views, parts1, cnt1, off1, T, ip, Tp, cnt2, off2, total;
};

RecLayout rec_layout(const nacho_matrix* ops, int32_t k, int32_t P) {
  RecLayout L;
  int64_t nouter = 0, cap = INT64_MAX;
  for (int o = 0; o < k; ++o) { nouter += ops[o].nouter; cap = std::min<int64_t>(cap, ops[o].nouter); }
  L.cap = cap > 0 ? cap : 1;
  L.P1 = std::max<int64_t>(1, (nouter + 255) / 256);   // 256 outer entries per partition (one thread each)
  size_t o = 0;
  L.pos_views = o; o += align_up((size_t)2 * k * 8);
  L.parts1 = o; o += parts_bytes(L.P1, k);
  L.cnt1 = o; o += align_up((size_t)(L.P1 + 1) * 8);
  L.off1 = o; o += align_up((size_t)(L.P1 + 2) * 8);
  L.T = o; o += align_up((size_t)L.cap * 8);
  L.ip = o; o += align_up((size_t)k * L.cap * 8);
  L.Tp = o; o += align_up((size_t)(L.cap + 2) * 8);
  L.cnt2 = o; o += align_up((size_t)(P + 1) * 8);
  L.off2 = o; o += align_up((size_t)(P + 2) * 8);
  L.total = o;
  return L;
}
}  // namespace

size_t nacho_dcsr_hadamard_workspace_size(const nacho_matrix* ops, int32_t k, int32_t P) {
  if (!ops || k < 1 || k > NACHO_MAX_K) return 0;
  return rec_layout(ops, k, P > 0 ? P : 1).total;
}

nacho_status nacho_dcsr_hadamard(const nacho_matrix* ops, int32_t k, nacho_parts* parts, int64_t* counts,
                                 int32_t* z_outer, int64_t* z_pos, int32_t* z_crd, void* z_val, void* ws,
                                 size_t ws_bytes, void* stream) {
  if (!ops || k < 1 || k > 4) return fail(NACHO_ERR_INVALID_ARG, "k = %d outside [1, 4]", k);
  for (int o = 0; o < k; ++o) {
    NACHO_TRY(check_matrix(ops + o, "operand"));
    if (ops[o].format != NACHO_DCSR) return fail(NACHO_ERR_INVALID_ARG, "recursive partitioning takes DCSR operands");
    if (ops[o].nrows != ops[0].nrows || ops[o].ncols != ops[0].ncols || ops[o].dtype != ops[0].dtype)
      return fail(NACHO_ERR_SHAPE, "operand %d disagrees with operand 0", o);
  }
  NACHO_TRY(check_parts(parts, k));
  if (!counts || !z_outer || !z_pos) return fail(NACHO_ERR_INVALID_ARG, "null output");
  const RecLayout L = rec_layout(ops, k, parts->P);
  if (!ws || ws_bytes < L.total) return fail(NACHO_ERR_WORKSPACE, "workspace %zu < %zu bytes", ws_bytes, L.total);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  char* w = static_cast<char*>(ws);
  int64_t* pos_views = reinterpret_cast<int64_t*>(w + L.pos_views);
  int64_t* cnt1 = reinterpret_cast<int64_t*>(w + L.cnt1);
  int64_t* off1 = reinterpret_cast<int64_t*>(w + L.off1);
  int64_t* T = reinterpret_cast<int64_t*>(w + L.T);
  int64_t* ip = reinterpret_cast<int64_t*>(w + L.ip);
  int64_t* Tp = reinterpret_cast<int64_t*>(w + L.Tp);
  int64_t* cnt2 = reinterpret_cast<int64_t*>(w + L.cnt2);
  int64_t* off2 = reinterpret_cast<int64_t*>(w + L.off2);
  const int64_t* S_dev = off1 + L.P1;   // the scan's total
  const OpsArg in = make_ops(ops, k);
  // 1. the outer intersection partitioned: Alg. 1 over the outer levels as one-row operands
  rec_outer_views_kernel<<<1, 32, 0, st>>>(in, pos_views);
  NACHO_TRY(launched("rec_outer_views_kernel"));
  nacho_matrix views[4];
  for (int o = 0; o < k; ++o) {
    views[o] = ops[o];
    views[o].format = NACHO_CSR;
    views[o].nrows = 1;
    views[o].ncols = ops[o].nrows;
    views[o].nouter = 1;
    views[o].nnz = ops[o].nouter;
    views[o].outer_crd = nullptr;
    views[o].pos = pos_views + 2 * o;
    views[o].crd = ops[o].outer_crd;
  }
  PartsArg p1 = carve_parts(w + L.parts1, L.P1, k);
  NACHO_TRY(launch_partition(views, k, p1, st));
  // 2. surviving rows: count, prefix sum (-> S), fill rows / T / outer positions
  const unsigned g1 = (unsigned)((L.P1 + kRecThreads - 1) / kRecThreads);
  rec_rows_kernel<0><<<g1, kRecThreads, 0, st>>>(in, p1, cnt1, nullptr, nullptr, nullptr, nullptr, L.cap);
  NACHO_TRY(launched("rec_rows_kernel<0>"));
  rec_scan_kernel<1024><<<1, 1024, 0, st>>>(cnt1, nullptr, L.P1, off1);
  NACHO_TRY(launched("rec_scan_kernel"));
  rec_rows_kernel<1><<<g1, kRecThreads, 0, st>>>(in, p1, nullptr, off1, z_outer, T, ip, L.cap);
  NACHO_TRY(launched("rec_rows_kernel<1>"));
  // 3. T' = exclusive prefix sum of T
  rec_scan_kernel<1024><<<1, 1024, 0, st>>>(T, S_dev, 0, Tp);
  NACHO_TRY(launched("rec_scan_kernel"));
  // 4. the remapped partition
  const PartsArg p2 = parts_arg(parts);
  if (k == 1) rec_partition_kernel<1><<<(unsigned)((p2.P + 4) / 4), 128, 0, st>>>(in, p2, S_dev, z_outer, Tp, ip, L.cap);
  else if (k == 2) rec_partition_kernel<2><<<(unsigned)((p2.P + 4) / 4), 128, 0, st>>>(in, p2, S_dev, z_outer, Tp, ip, L.cap);
  else rec_partition_kernel<4><<<(unsigned)((p2.P + 4) / 4), 128, 0, st>>>(in, p2, S_dev, z_outer, Tp, ip, L.cap);
  NACHO_TRY(launched("rec_partition_kernel"));
  // 5. Z: count, prefix sum, fill (Listing 8 over the remapped rows)
  const unsigned g2 = (unsigned)((p2.P + kRecThreads - 1) / kRecThreads);
  const bool f64 = ops[0].dtype == NACHO_F64;
  if (f64) rec_hadamard_kernel<double, 0><<<g2, kRecThreads, 0, st>>>(in, p2, S_dev, ip, L.cap, cnt2, nullptr, nullptr, nullptr, nullptr);
  else rec_hadamard_kernel<float, 0><<<g2, kRecThreads, 0, st>>>(in, p2, S_dev, ip, L.cap, cnt2, nullptr, nullptr, nullptr, nullptr);
  NACHO_TRY(launched("rec_hadamard_kernel<0>"));
  rec_scan_kernel<1024><<<1, 1024, 0, st>>>(cnt2, nullptr, p2.P, off2);
  NACHO_TRY(launched("rec_scan_kernel"));
  if (f64)
    rec_hadamard_kernel<double, 1><<<g2, kRecThreads, 0, st>>>(in, p2, S_dev, ip, L.cap, nullptr, off2, z_pos, z_crd,
                                                               static_cast<double*>(z_val));
  else
    rec_hadamard_kernel<float, 1><<<g2, kRecThreads, 0, st>>>(in, p2, S_dev, ip, L.cap, nullptr, off2, z_pos, z_crd,
                                                              static_cast<float*>(z_val));
  NACHO_TRY(launched("rec_hadamard_kernel<1>"));
  rec_counts_kernel<<<1, 32, 0, st>>>(S_dev, off2 + p2.P, counts);
  return launched("rec_counts_kernel");
}

/* ------------------------------------------------------------------ DCSR k-way SpAdd (Listing 2) */
size_t nacho_dcsr_spadd_k_workspace_size(const nacho_matrix* ops, int32_t k, int32_t P) {
  (void)ops; (void)k;
  const size_t Pe = P > 0 ? P : 1;
  return 2 * align_up((Pe + 1) * 8) + 2 * align_up((Pe + 2) * 8);
}

nacho_status nacho_dcsr_spadd_k(const nacho_matrix* ops, int32_t k, const nacho_parts* parts, int64_t* counts,
                                int32_t* z_outer, int64_t* z_pos, int32_t* z_crd, void* z_val, void* ws,
                                size_t ws_bytes, void* stream) {
  NACHO_TRY(check_ops(ops, k));
  if (ops[0].format != NACHO_DCSR) return fail(NACHO_ERR_INVALID_ARG, "nacho_dcsr_spadd_k takes DCSR operands");
  NACHO_TRY(check_parts(parts, k));
  if (!counts || !z_outer || !z_pos) return fail(NACHO_ERR_INVALID_ARG, "null output");
  if (total_cost(ops, k) > 0 && (!z_crd || !z_val)) return fail(NACHO_ERR_INVALID_ARG, "null z_crd / z_val");
  const int64_t P = parts->P;
  const size_t need = nacho_dcsr_spadd_k_workspace_size(ops, k, parts->P);
  if (!ws || ws_bytes < need) return fail(NACHO_ERR_WORKSPACE, "workspace %zu < %zu bytes", ws_bytes, need);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  char* w = static_cast<char*>(ws);
  int64_t* ent = reinterpret_cast<int64_t*>(w);
  int64_t* rst = reinterpret_cast<int64_t*>(w + align_up((P + 1) * 8));
  int64_t* off_e = reinterpret_cast<int64_t*>(w + 2 * align_up((P + 1) * 8));
  int64_t* off_r = reinterpret_cast<int64_t*>(w + 2 * align_up((P + 1) * 8) + align_up((P + 2) * 8));
  const OpsArg a = make_ops(ops, k);
  const PartsArg pa = parts_arg(parts);
  const unsigned g = (unsigned)((P + 127) / 128);
  const bool f64 = ops[0].dtype == NACHO_F64;
  if (f64) dcsr_spadd_kernel<double, 0><<<g, 128, 0, st>>>(a, pa, ent, rst, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr);
  else dcsr_spadd_kernel<float, 0><<<g, 128, 0, st>>>(a, pa, ent, rst, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr);
  NACHO_TRY(launched("dcsr_spadd_kernel<0>"));
  rec_scan_kernel<1024><<<1, 1024, 0, st>>>(ent, nullptr, P, off_e);
  NACHO_TRY(launched("rec_scan_kernel"));
  rec_scan_kernel<1024><<<1, 1024, 0, st>>>(rst, nullptr, P, off_r);
  NACHO_TRY(launched("rec_scan_kernel"));
  if (f64)
    dcsr_spadd_kernel<double, 1><<<g, 128, 0, st>>>(a, pa, nullptr, nullptr, off_e, off_r, z_outer, z_pos, z_crd,
                                                     static_cast<double*>(z_val));
  else
    dcsr_spadd_kernel<float, 1><<<g, 128, 0, st>>>(a, pa, nullptr, nullptr, off_e, off_r, z_outer, z_pos, z_crd,
                                                    static_cast<float*>(z_val));
  NACHO_TRY(launched("dcsr_spadd_kernel<1>"));
  rec_counts_kernel<<<1, 32, 0, st>>>(off_r + P, off_e + P, counts);
  return launched("rec_counts_kernel");
}

/* ------------------------------------------------------------------ mixed CSR / COO k-way SpAdd */
size_t nacho_mixed_spadd_k_workspace_size(const nacho_matrix* ops, int32_t k, int32_t P) {
  (void)ops; (void)k;
  const size_t Pe = P > 0 ? P : 1;
  return align_up((Pe + 1) * 8) + align_up((Pe + 2) * 8);
}

nacho_status nacho_mixed_spadd_k(const nacho_matrix* ops, int32_t k, const nacho_parts* parts, int64_t* nnz_z,
                                 int64_t* z_pos, int32_t* z_crd, void* z_val, void* ws, size_t ws_bytes, void* stream) {
  NACHO_TRY(check_ops(ops, k));
  if (k > 4) return fail(NACHO_ERR_INVALID_ARG, "nacho_mixed_spadd_k takes k <= 4 operands");
  for (int o = 0; o < k; ++o)
    if (ops[o].format == NACHO_DCSR) return fail(NACHO_ERR_INVALID_ARG, "nacho_mixed_spadd_k takes CSR / COO operands");
  NACHO_TRY(check_parts(parts, k));
  if (!nnz_z || !z_pos) return fail(NACHO_ERR_INVALID_ARG, "null output");
  if (total_cost(ops, k) > 0 && (!z_crd || !z_val)) return fail(NACHO_ERR_INVALID_ARG, "null z_crd / z_val");
  const int64_t P = parts->P;
  const size_t need = nacho_mixed_spadd_k_workspace_size(ops, k, parts->P);
  if (!ws || ws_bytes < need) return fail(NACHO_ERR_WORKSPACE, "workspace %zu < %zu bytes", ws_bytes, need);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int64_t* cnt = static_cast<int64_t*>(ws);
  int64_t* off = reinterpret_cast<int64_t*>(static_cast<char*>(ws) + align_up((P + 1) * 8));
  const OpsArg a = make_ops(ops, k);
  const PartsArg pa = parts_arg(parts);
  const unsigned g = (unsigned)((P + 127) / 128);
  const bool f64 = ops[0].dtype == NACHO_F64;
  if (f64) mixed_spadd_kernel<double, 0><<<g, 128, 0, st>>>(a, pa, cnt, nullptr, nullptr, nullptr, nullptr);
  else mixed_spadd_kernel<float, 0><<<g, 128, 0, st>>>(a, pa, cnt, nullptr, nullptr, nullptr, nullptr);
  NACHO_TRY(launched("mixed_spadd_kernel<0>"));
  rec_scan_kernel<1024><<<1, 1024, 0, st>>>(cnt, nullptr, P, off);
  NACHO_TRY(launched("rec_scan_kernel"));
  if (f64) mixed_spadd_kernel<double, 1><<<g, 128, 0, st>>>(a, pa, nullptr, off, z_pos, z_crd, static_cast<double*>(z_val));
  else mixed_spadd_kernel<float, 1><<<g, 128, 0, st>>>(a, pa, nullptr, off, z_pos, z_crd, static_cast<float*>(z_val));
  NACHO_TRY(launched("mixed_spadd_kernel<1>"));
  if (cudaMemcpyAsync(nnz_z, off + P, 8, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
    return fail(NACHO_ERR_CUDA, "nnz_Z copy");
  return NACHO_SUCCESS;
}

/* ------------------------------------------------------------------ third-order CSF (csf.cuh) */
namespace {
nacho_status check_tensors(const nacho_tensor3* ops, int32_t k, Csf3Args& a) {
  if (!ops) return fail(NACHO_ERR_INVALID_ARG, "null operand array");
  if (k < 1 || k > 4) return fail(NACHO_ERR_INVALID_ARG, "k = %d outside [1, 4] (CSF)", k);
  for (int o = 0; o < k; ++o) {
    const nacho_tensor3& T = ops[o];
    if (T.n0 < 0 || T.n1 < 0 || T.n2 < 0 || T.nnz < 0 || T.n_slices < 0 || T.n_fibers < 0)
      return fail(NACHO_ERR_SHAPE, "tensor %d: negative size", o);
    if (T.n0 > INT32_MAX || T.n1 > INT32_MAX || T.n2 > INT32_MAX)
      return fail(NACHO_ERR_OVERFLOW, "tensor %d: a dimension > INT32_MAX", o);
    if (T.n0 != ops[0].n0 || T.n1 != ops[0].n1 || T.n2 != ops[0].n2 || T.dtype != ops[0].dtype)
      return fail(NACHO_ERR_SHAPE, "tensor %d disagrees with tensor 0 in shape/dtype", o);
    if (T.dtype != NACHO_F32 && T.dtype != NACHO_F64) return fail(NACHO_ERR_INVALID_ARG, "tensor %d: dtype", o);
    if (!T.pos1 || !T.pos2) return fail(NACHO_ERR_INVALID_ARG, "tensor %d: null pos1 / pos2", o);
    if ((T.n_slices > 0 && !T.crd0) || (T.n_fibers > 0 && !T.crd1) || (T.nnz > 0 && (!T.crd2 || !T.val)))
      return fail(NACHO_ERR_INVALID_ARG, "tensor %d: null crd / val", o);
    Csf3View& v = a.op[o];
    v.n0 = T.n0; v.n1 = T.n1; v.n2 = T.n2; v.nnz = T.nnz; v.ns = T.n_slices; v.nf = T.n_fibers;
    v.crd0 = T.crd0; v.pos1 = T.pos1; v.crd1 = T.crd1; v.pos2 = T.pos2; v.crd2 = T.crd2; v.val = T.val;
  }
  a.k = k;
  a.n0 = ops[0].n0;
  return NACHO_SUCCESS;
}
}  // namespace

nacho_status nacho_partition_csf(const nacho_tensor3* ops, int32_t k, int32_t P, nacho_parts* out, void* stream) {
  Csf3Args a;
  NACHO_TRY(check_tensors(ops, k, a));
  if (P < 1) return fail(NACHO_ERR_INVALID_ARG, "P = %d < 1", P);
  NACHO_TRY(check_parts(out, k));
  if (out->P != P) return fail(NACHO_ERR_INVALID_ARG, "parts.P = %d != P = %d", out->P, P);
  int64_t qstar = 0;
  for (int o = 0; o < k; ++o) qstar += ops[o].nnz;
  out->max_work = (qstar + P - 1) / P + (k - 1);
  const unsigned g = (unsigned)((P + 1 + 3) / 4);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const PartsArg pa = parts_arg(out);
  if (k <= 2) csf_partition_kernel<2><<<g, 128, 0, st>>>(a, pa, qstar);
  else csf_partition_kernel<4><<<g, 128, 0, st>>>(a, pa, qstar);
  return launched("csf_partition_kernel");
}

size_t nacho_csf_spadd_k_workspace_size(const nacho_tensor3* ops, int32_t k, int32_t P) {
  (void)ops; (void)k;
  const size_t Pe = P > 0 ? P : 1;
  return 2 * align_up(3 * (Pe + 1) * 8);
}

nacho_status nacho_csf_spadd_k(const nacho_tensor3* ops, int32_t k, const nacho_parts* parts, int64_t* counts,
                               int32_t* z_crd0, int64_t* z_pos1, int32_t* z_crd1, int64_t* z_pos2, int32_t* z_crd2,
                               void* z_val, void* ws, size_t ws_bytes, void* stream) {
  Csf3Args a;
  NACHO_TRY(check_tensors(ops, k, a));
  NACHO_TRY(check_parts(parts, k));
  if (!counts || !z_pos1 || !z_pos2) return fail(NACHO_ERR_INVALID_ARG, "null output");
  int64_t qstar = 0;
  for (int o = 0; o < k; ++o) qstar += ops[o].nnz;
  if (qstar > 0 && (!z_crd0 || !z_crd1 || !z_crd2 || !z_val)) return fail(NACHO_ERR_INVALID_ARG, "null z_crd / z_val");
  const int64_t P = parts->P;
  const size_t need = nacho_csf_spadd_k_workspace_size(ops, k, parts->P);
  if (!ws || ws_bytes < need) return fail(NACHO_ERR_WORKSPACE, "workspace %zu < %zu bytes", ws_bytes, need);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int64_t* cnt = static_cast<int64_t*>(ws);
  int64_t* off = reinterpret_cast<int64_t*>(static_cast<char*>(ws) + align_up(3 * (P + 1) * 8));
  const PartsArg pa = parts_arg(parts);
  const unsigned g = (unsigned)((P + 127) / 128);
  const bool f64 = ops[0].dtype == NACHO_F64;
  if (f64) csf_spadd_kernel<double, 0><<<g, 128, 0, st>>>(a, pa, cnt, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr);
  else csf_spadd_kernel<float, 0><<<g, 128, 0, st>>>(a, pa, cnt, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr);
  NACHO_TRY(launched("csf_spadd_kernel<0>"));
  for (int l = 0; l < 3; ++l) {
    rec_scan_kernel<1024><<<1, 1024, 0, st>>>(cnt + l * (P + 1), nullptr, P, off + l * (P + 1));
    NACHO_TRY(launched("rec_scan_kernel"));
  }
  if (f64)
    csf_spadd_kernel<double, 1><<<g, 128, 0, st>>>(a, pa, nullptr, off, z_crd0, z_pos1, z_crd1, z_pos2, z_crd2,
                                                    static_cast<double*>(z_val));
  else
    csf_spadd_kernel<float, 1><<<g, 128, 0, st>>>(a, pa, nullptr, off, z_crd0, z_pos1, z_crd1, z_pos2, z_crd2,
                                                   static_cast<float*>(z_val));
  NACHO_TRY(launched("csf_spadd_kernel<1>"));
  csf_counts_kernel<<<1, 32, 0, st>>>(off, P, counts);
  return launched("csf_counts_kernel");
}

/* ------------------------------------------------------------------ multi-GPU (dist.cuh) */
#define NACHO_NCCL(call)                                                                              \
  do {                                                                                                \
    const ncclResult_t _r = (call);                                                                   \
    if (_r != ncclSuccess) return fail(NACHO_ERR_NCCL, "%s: %s", #call, nccl().GetErrorString(_r));  \
  } while (0)

size_t nacho_dist_unique_id_size(void) { return sizeof(ncclUniqueId); }

nacho_status nacho_dist_unique_id(void* id) {
  if (!id) return fail(NACHO_ERR_INVALID_ARG, "null id buffer");
  if (!nccl().ok) return fail(NACHO_ERR_NCCL, "libnccl.so.2 not loadable");
  NACHO_NCCL(nccl().GetUniqueId(static_cast<ncclUniqueId*>(id)));
  return NACHO_SUCCESS;
}

nacho_status nacho_dist_init(nacho_dist** comm, const void* id, int32_t nranks, int32_t rank) {
  if (!comm || !id) return fail(NACHO_ERR_INVALID_ARG, "null comm / id");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(NACHO_ERR_INVALID_ARG, "rank %d of %d", rank, nranks);
  if (!nccl().ok) return fail(NACHO_ERR_NCCL, "libnccl.so.2 not loadable");
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof(uid));
  ncclComm_t c;
  NACHO_NCCL(nccl().CommInitRank(&c, nranks, uid, rank));
  *comm = new nacho_dist_s{c, nranks, rank};
  return NACHO_SUCCESS;
}

nacho_status nacho_dist_destroy(nacho_dist* comm) {
  if (!comm) return NACHO_SUCCESS;
  const ncclResult_t r = nccl().CommDestroy(comm->comm);
  delete comm;
  if (r != ncclSuccess) return fail(NACHO_ERR_NCCL, "ncclCommDestroy: %s", nccl().GetErrorString(r));
  return NACHO_SUCCESS;
}

nacho_status nacho_dist_broadcast(nacho_dist* comm, void* buf, size_t bytes, int32_t root, void* stream) {
  if (!comm || (!buf && bytes)) return fail(NACHO_ERR_INVALID_ARG, "null comm / buffer");
  if (root < 0 || root >= comm->nranks) return fail(NACHO_ERR_INVALID_ARG, "root %d", root);
  NACHO_NCCL(nccl().Broadcast(buf, buf, bytes, ncclChar, root, comm->comm, static_cast<cudaStream_t>(stream)));
  return NACHO_SUCCESS;
}

nacho_status nacho_device_cuts(const nacho_matrix* A, int32_t D, int64_t* cuts, void* stream) {
  if (!A || !A->pos) return fail(NACHO_ERR_INVALID_ARG, "A: null descriptor / pos");   // crd / val not read
  if (A->format != NACHO_CSR || A->nouter < 0 || A->nnz < 0) return fail(NACHO_ERR_INVALID_ARG, "A: CSR sizes");
  if (D < 1 || !cuts) return fail(NACHO_ERR_INVALID_ARG, "D = %d / null cuts", D);
  device_cuts_kernel<<<(D + 1 + 127) / 128, 128, 0, static_cast<cudaStream_t>(stream)>>>(A->pos, A->nouter, A->nnz, D,
                                                                                          cuts);
  return launched("device_cuts_kernel");
}

nacho_status nacho_shard_rows(const int64_t* pos, int64_t row_lo, int64_t nloc, int64_t pos_lo, int64_t pos_hi,
                              int64_t* local_pos, void* stream) {
  if (!pos || !local_pos) return fail(NACHO_ERR_INVALID_ARG, "null pos / local_pos");
  if (row_lo < 0 || nloc < 0 || pos_lo < 0 || pos_hi < pos_lo) return fail(NACHO_ERR_INVALID_ARG, "bad shard range");
  const int64_t g = std::min<int64_t>((nloc + 256) / 256, 148 * 16);
  shard_rows_kernel<<<(unsigned)std::max<int64_t>(g, 1), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      pos, row_lo, nloc, pos_lo, pos_hi, local_pos);
  return launched("shard_rows_kernel");
}

nacho_status nacho_dist_seam(const int64_t* carries, int32_t D, int32_t d, int64_t row_lo, int32_t owns_first,
                             int32_t dtype, void* y_local, void* stream) {
  if (!carries || !y_local) return fail(NACHO_ERR_INVALID_ARG, "null carries / y_local");
  if (D < 1 || d < 0 || d >= D) return fail(NACHO_ERR_INVALID_ARG, "device %d of %d", d, D);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dtype == NACHO_F64) seam_kernel<double><<<1, 32, 0, st>>>(carries, D, d, row_lo, owns_first, static_cast<double*>(y_local));
  else seam_kernel<float><<<1, 32, 0, st>>>(carries, D, d, row_lo, owns_first, static_cast<float*>(y_local));
  return launched("seam_kernel");
}

size_t nacho_dist_spmv_workspace_size(const nacho_matrix* A_local, int32_t P, int32_t D) {
  return nacho_spmv_workspace_size(A_local, P) + align_up(2 * 8) + align_up((size_t)(D > 0 ? D : 1) * 2 * 8);
}

nacho_status nacho_dist_spmv(nacho_dist* comm, const nacho_matrix* A_local, const nacho_parts* parts, const void* x,
                             void* y_local, const int64_t* cut_rows, void* y_full, void* ws, size_t ws_bytes,
                             void* stream) {
  if (!comm || !cut_rows) return fail(NACHO_ERR_INVALID_ARG, "null comm / cut_rows");
  NACHO_TRY(check_matrix(A_local, "A_local"));
  if (A_local->format != NACHO_CSR) return fail(NACHO_ERR_INVALID_ARG, "dist SpMV shards CSR operands");
  const int D = comm->nranks, d = comm->rank;
  const size_t need = nacho_dist_spmv_workspace_size(A_local, parts ? parts->P : 0, D);
  if (ws_bytes < need || !ws) return fail(NACHO_ERR_WORKSPACE, "workspace %zu < %zu bytes", ws_bytes, need);
  const size_t sw = nacho_spmv_workspace_size(A_local, parts ? parts->P : 0);
  char* w = static_cast<char*>(ws);
  int64_t* send = reinterpret_cast<int64_t*>(w + sw);
  int64_t* carries = reinterpret_cast<int64_t*>(w + sw + align_up(2 * 8));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t nloc = A_local->nrows;
  const int64_t row_lo = cut_rows[d];
  const int64_t own = cut_rows[d + 1] - row_lo;   // rows this device owns (R7)
  // + the row cut by b_{d+1} (its seam carry), unless the cut is the end of the rows
  const bool has_carry = d < D - 1 && cut_rows[d + 1] < cut_rows[D];
  const int64_t expect = own + (has_carry ? 1 : 0);
  if (nloc != expect)
    return fail(NACHO_ERR_SHAPE, "shard holds %lld rows, the cut %lld", (long long)nloc, (long long)expect);
  // 1. the device's partitions (P:1089-1093 on the shard)
  NACHO_TRY(nacho_spmv(A_local, parts, x, y_local, 0, w, sw, stream));
  // 2. seam carries: all-gather of (row, partial) pairs, added in device order by the owner
  const bool f64 = A_local->dtype == NACHO_F64;
  if (f64) carry_pack_kernel<double><<<1, 32, 0, st>>>(static_cast<double*>(y_local), nloc, row_lo, has_carry, send);
  else carry_pack_kernel<float><<<1, 32, 0, st>>>(static_cast<float*>(y_local), nloc, row_lo, has_carry, send);
  NACHO_TRY(launched("carry_pack_kernel"));
  NACHO_NCCL(nccl().AllGather(send, carries, 2, ncclInt64, comm->comm, st));
  NACHO_TRY(nacho_dist_seam(carries, D, d, row_lo, own > 0, A_local->dtype, y_local, stream));
  // 3. optional gather of the owned y segments (one broadcast per device, grouped)
  if (y_full) {
    const size_t es = f64 ? 8 : 4;
    NACHO_NCCL(nccl().GroupStart());
    for (int r = 0; r < D; ++r) {
      const int64_t own_r = cut_rows[r + 1] - cut_rows[r];
      if (own_r <= 0) continue;
      void* dst = static_cast<char*>(y_full) + (size_t)cut_rows[r] * es;
      NACHO_NCCL(nccl().Broadcast(r == d ? y_local : dst, dst, (size_t)own_r, f64 ? ncclFloat64 : ncclFloat32, r,
                                  comm->comm, st));
    }
    NACHO_NCCL(nccl().GroupEnd());
  }
  return NACHO_SUCCESS;
}

size_t nacho_dist_spadd_workspace_size(int32_t D) {
  const size_t De = D > 0 ? D : 1;
  return align_up(8) + align_up(De * 8) + align_up((De + 1) * 8);
}

nacho_status nacho_dist_spadd_gather(nacho_dist* comm, const int64_t* z_pos_local, const int32_t* z_crd_local,
                                     const void* z_val_local, int32_t dtype, const int64_t* nnz_local,
                                     const int64_t* cut_rows, int64_t* z_pos, int32_t* z_crd, void* z_val,
                                     int64_t* nnz_total, void* ws, size_t ws_bytes, void* stream) {
  if (!comm || !cut_rows || !z_pos_local || !nnz_local || !z_pos) return fail(NACHO_ERR_INVALID_ARG, "null argument");
  const int D = comm->nranks, d = comm->rank;
  const size_t need = nacho_dist_spadd_workspace_size(D);
  if (ws_bytes < need || !ws) return fail(NACHO_ERR_WORKSPACE, "workspace %zu < %zu bytes", ws_bytes, need);
  char* w = static_cast<char*>(ws);
  int64_t* counts = reinterpret_cast<int64_t*>(w + align_up(8));
  int64_t* off = reinterpret_cast<int64_t*>(w + align_up(8) + align_up((size_t)D * 8));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // 1. device union sizes -> global offsets (P:1475 at device level)
  NACHO_NCCL(nccl().AllGather(nnz_local, counts, 1, ncclInt64, comm->comm, st));
  offsets_kernel<<<1, 32, 0, st>>>(counts, D, off);
  NACHO_TRY(launched("offsets_kernel"));
  std::vector<int64_t> h(D + 1);
  if (cudaMemcpyAsync(h.data(), off, (D + 1) * 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)   // variable-size collectives need the counts on the host
    return fail(NACHO_ERR_CUDA, "reading the device offsets");
  if (nnz_total) *nnz_total = h[D];
  if ((!z_crd || !z_val) && h[D] > 0) return fail(NACHO_ERR_INVALID_ARG, "null z_crd / z_val");
  // 2. this device's Z.pos rows (row_lo, row_hi] at its offset, then every segment gathered
  const int64_t M = cut_rows[D];
  const int64_t own = (d < D - 1 ? cut_rows[d + 1] : M) - cut_rows[d];
  if (own > 0) {
    zpos_segment_kernel<<<(unsigned)std::min<int64_t>((own + 255) / 256, 148 * 16), 256, 0, st>>>(
        z_pos_local, own, off + d, z_pos + cut_rows[d] + 1);
    NACHO_TRY(launched("zpos_segment_kernel"));
  }
  if (d == 0 && cudaMemsetAsync(z_pos, 0, 8, st) != cudaSuccess) return fail(NACHO_ERR_CUDA, "z_pos[0]");
  const size_t es = dtype == NACHO_F64 ? 8 : 4;
  NACHO_NCCL(nccl().GroupStart());
  for (int r = 0; r < D; ++r) {
    const int64_t own_r = (r < D - 1 ? cut_rows[r + 1] : M) - cut_rows[r];
    const int64_t cnt = h[r + 1] - h[r];
    if (cnt > 0) {
      NACHO_NCCL(nccl().Broadcast(r == d ? (const void*)z_crd_local : z_crd + h[r], z_crd + h[r], (size_t)cnt, ncclInt32, r,
                                  comm->comm, st));
      void* vdst = static_cast<char*>(z_val) + (size_t)h[r] * es;
      NACHO_NCCL(nccl().Broadcast(r == d ? z_val_local : vdst, vdst, (size_t)cnt, es == 8 ? ncclFloat64 : ncclFloat32,
                                  r, comm->comm, st));
    }
    if (own_r > 0)
      NACHO_NCCL(nccl().Broadcast(z_pos + cut_rows[r] + 1, z_pos + cut_rows[r] + 1, (size_t)own_r, ncclInt64, r,
                                  comm->comm, st));
  }
  NACHO_NCCL(nccl().GroupEnd());
  if (D > 1) NACHO_NCCL(nccl().Broadcast(z_pos, z_pos, 1, ncclInt64, 0, comm->comm, st));
  return NACHO_SUCCESS;
}

const char* nacho_last_error(void) { return g_err.c_str(); }

// Debug only (not part of nacho.h): the spadd2 phase timers of a -DNACHO_PROF build.
int nacho_debug_phases(unsigned long long* out, int reset) {
#ifdef NACHO_PROF
  cudaMemcpyFromSymbol(out, g_phase, sizeof(g_phase));
  if (reset) { unsigned long long z[16] = {0}; cudaMemcpyToSymbol(g_phase, z, sizeof(z)); }
  return 1;
#else
  (void)out; (void)reset;
  return 0;
#endif
}

int64_t nacho_launch_count(int32_t reset) {
  const int64_t v = g_launches;
  if (reset) g_launches = 0;
  return v;
}

nacho_status nacho_partition(const nacho_matrix* ops, int32_t k, int32_t P, nacho_parts* out, void* stream) {
  NACHO_TRY(check_ops(ops, k));
  if (P < 1) return fail(NACHO_ERR_INVALID_ARG, "P = %d < 1", P);
  NACHO_TRY(check_parts(out, k));
  if (out->P != P) return fail(NACHO_ERR_INVALID_ARG, "parts.P = %d != P = %d", out->P, P);
  out->max_work = (total_cost(ops, k) + P - 1) / P + (k - 1);
  return launch_partition(ops, k, parts_arg(out), static_cast<cudaStream_t>(stream));
}

nacho_status nacho_partition_slice(const nacho_matrix* ops, int32_t k, int32_t P, int32_t p_begin, nacho_parts* out,
                                   void* stream) {
  NACHO_TRY(check_ops(ops, k));
  if (P < 1) return fail(NACHO_ERR_INVALID_ARG, "P = %d < 1", P);
  NACHO_TRY(check_parts(out, k));
  if (p_begin < 0 || (int64_t)p_begin + out->P > P)
    return fail(NACHO_ERR_INVALID_ARG, "slice [%d, %lld] outside [0, %d]", p_begin, (long long)p_begin + out->P, P);
  out->max_work = (total_cost(ops, k) + P - 1) / P + (k - 1);
  return launch_partition(ops, k, parts_arg(out), static_cast<cudaStream_t>(stream), P, p_begin);
}

int32_t nacho_spadd_tile(int32_t k) { return k < 1 || k > NACHO_MAX_K ? 0 : s5_max_entries(k); }

int32_t nacho_auto_partitions(const nacho_matrix* ops, int32_t k, int32_t op) {
  if (!ops || k < 1) return 1;
  const int64_t work = total_cost(ops, k);
  if (op == 0) return auto_p(work, spmv_tile(ops[0].dtype));
  if (op == 1) return auto_p(work, s5_max_entries(k) - (k - 1));
  return auto_p(work, kSpmmWarps * kSpmmWitems);
}

size_t nacho_spmv_workspace_size(const nacho_matrix* A, int32_t P) {
  if (!A) return 0;
  const bool auto_parts = P <= 0;
  const int64_t Pe = auto_parts ? nacho_auto_partitions(A, 1, 0) : P;
  const size_t vs = A->dtype == NACHO_F64 ? 8 : 4;
  const int64_t nc = spmv_carry_cap(A, Pe);
  return align_up(nc * 8) + align_up(nc * vs) + (auto_parts ? parts_bytes(Pe, 1) : 0);
}

nacho_status nacho_spmv(const nacho_matrix* A, const nacho_parts* parts, const void* x, void* y, int32_t dense_y,
                        void* ws, size_t ws_bytes, void* stream) {
  NACHO_TRY(check_matrix(A, "A"));
  if (A->format == NACHO_COO) return fail(NACHO_ERR_INVALID_ARG, "SpMV takes CSR / DCSR operands");
  if (!x && A->ncols > 0) return fail(NACHO_ERR_INVALID_ARG, "null x");
  if (!y && (A->nouter > 0 || (dense_y && A->nrows > 0))) return fail(NACHO_ERR_INVALID_ARG, "null y");
  if (parts) NACHO_TRY(check_parts(parts, 1));
  const size_t need = nacho_spmv_workspace_size(A, parts ? parts->P : 0);
  if (ws_bytes < need || (need > 0 && !ws)) return fail(NACHO_ERR_WORKSPACE, "workspace %zu < %zu bytes", ws_bytes, need);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  char* c = static_cast<char*>(ws);
  PartsArg pa;
  const int64_t P = parts ? parts->P : nacho_auto_partitions(A, 1, 0);
  const int64_t cap = spmv_carry_cap(A, P);
  if (parts) {
    pa = parts_arg(parts);
  } else {
    const size_t vs = A->dtype == NACHO_F64 ? 8 : 4;
    pa = carve_parts(c + align_up(cap * 8) + align_up(cap * vs), P, 1);
    NACHO_TRY(launch_partition(A, 1, pa, st));
  }
  if (A->dtype == NACHO_F64) return run_spmv<double>(A, pa, x, y, dense_y, c, cap, st);
  return run_spmv<float>(A, pa, x, y, dense_y, c, cap, st);
}

size_t nacho_spadd_k_workspace_size(const nacho_matrix* ops, int32_t k, int32_t P) {
  (void)ops; (void)k;
#ifdef NACHO_S7_PROF
  return align_up((size_t)((P > 0 ? P : 1) + 2 + 16) * 8);   // + profiling counters (dev builds)
#endif
  return align_up((size_t)((P > 0 ? P : 1) + 2) * 8);   // look-back states, ticket, error flag
}

nacho_status nacho_spadd_k_count(const nacho_matrix* ops, int32_t k, const nacho_parts* parts, int64_t* part_off,
                                 void* ws, size_t ws_bytes, void* stream) {
  NACHO_TRY(check_ops(ops, k));
  if (!all_csr(ops, k)) return fail(NACHO_ERR_INVALID_ARG, "SpAdd supports CSR operands (COO: nacho_mixed_spadd_k)");
  NACHO_TRY(check_parts(parts, k));
  if (!part_off) return fail(NACHO_ERR_INVALID_ARG, "null part_off");
  const size_t need = nacho_spadd_k_workspace_size(ops, k, parts->P);
  if (ws_bytes < need || !ws) return fail(NACHO_ERR_WORKSPACE, "workspace %zu < %zu bytes", ws_bytes, need);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int64_t* cnt = static_cast<int64_t*>(ws);
  if (fits_sa_tile(ops, k, parts, st)) {
    if (ops[0].dtype == NACHO_F64) {
      Spadd4Args<double> a{make_ops(ops, k), parts_arg(parts), cnt, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
      NACHO_TRY((launch_spadd4<double, kS4Count>(a, st)));
    } else {
      Spadd4Args<float> a{make_ops(ops, k), parts_arg(parts), cnt, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
      NACHO_TRY((launch_spadd4<float, kS4Count>(a, st)));
    }
  } else if (ops[0].dtype == NACHO_F64) {
    SpaddArgs<double> a{make_ops(ops, k), parts_arg(parts), total_cost(ops, k), cnt, nullptr, nullptr, nullptr, nullptr};
    NACHO_TRY((launch_spadd<double, false>(a, st)));
  } else {
    SpaddArgs<float> a{make_ops(ops, k), parts_arg(parts), total_cost(ops, k), cnt, nullptr, nullptr, nullptr, nullptr};
    NACHO_TRY((launch_spadd<float, false>(a, st)));
  }
  scan_counts_kernel<1024><<<1, 1024, 0, st>>>(cnt, parts->P, part_off);
  return launched("scan_counts_kernel");
}

nacho_status nacho_spadd_k_fill(const nacho_matrix* ops, int32_t k, const nacho_parts* parts,
                                const int64_t* part_off, int64_t* z_pos, int32_t* z_crd, void* z_val, void* ws,
                                size_t ws_bytes, void* stream) {
  (void)ws; (void)ws_bytes;
  NACHO_TRY(check_ops(ops, k));
  if (!all_csr(ops, k)) return fail(NACHO_ERR_INVALID_ARG, "SpAdd supports CSR operands (COO: nacho_mixed_spadd_k)");
  NACHO_TRY(check_parts(parts, k));
  if (!part_off || !z_pos) return fail(NACHO_ERR_INVALID_ARG, "null part_off / z_pos");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (fits_sa_tile(ops, k, parts, st)) {
    if (ops[0].dtype == NACHO_F64) {
      Spadd4Args<double> a{make_ops(ops, k), parts_arg(parts), nullptr, const_cast<int64_t*>(part_off), nullptr, nullptr,
                           z_pos, z_crd, static_cast<double*>(z_val)};
      return launch_spadd4<double, kS4Fill>(a, st);
    }
    Spadd4Args<float> a{make_ops(ops, k), parts_arg(parts), nullptr, const_cast<int64_t*>(part_off), nullptr, nullptr,
                        z_pos, z_crd, static_cast<float*>(z_val)};
    return launch_spadd4<float, kS4Fill>(a, st);
  }
  if (ops[0].dtype == NACHO_F64) {
    SpaddArgs<double> a{make_ops(ops, k), parts_arg(parts), total_cost(ops, k), nullptr, part_off, z_pos, z_crd,
                        static_cast<double*>(z_val)};
    return launch_spadd<double, true>(a, st);
  }
  SpaddArgs<float> a{make_ops(ops, k), parts_arg(parts), total_cost(ops, k), nullptr, part_off, z_pos, z_crd,
                     static_cast<float*>(z_val)};
  return launch_spadd<float, true>(a, st);
}

nacho_status nacho_spadd_k(const nacho_matrix* ops, int32_t k, const nacho_parts* parts, int64_t* part_off,
                           int64_t* z_pos, int32_t* z_crd, void* z_val, void* ws, size_t ws_bytes, void* stream) {
  NACHO_TRY(check_ops(ops, k));
  if (!all_csr(ops, k)) return fail(NACHO_ERR_INVALID_ARG, "SpAdd supports CSR operands (COO: nacho_mixed_spadd_k)");
  NACHO_TRY(check_parts(parts, k));
  if (!z_pos) return fail(NACHO_ERR_INVALID_ARG, "null z_pos");
  if (total_cost(ops, k) > 0 && (!z_crd || !z_val)) return fail(NACHO_ERR_INVALID_ARG, "null z_crd / z_val");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t need = nacho_spadd_k_workspace_size(ops, k, parts->P);
  if (ws_bytes < need || !ws) return fail(NACHO_ERR_WORKSPACE, "workspace %zu < %zu bytes", ws_bytes, need);
  auto* flags = static_cast<unsigned long long*>(ws);
  if (spadd5_applies(ops, k, parts_arg(parts), st)) {
    if (spadd_impl() == 7) {
      if (ops[0].dtype == NACHO_F64)
        return run_spadd7<double>(ops, k, parts, part_off, z_pos, z_crd, static_cast<double*>(z_val), flags, st);
      return run_spadd7<float>(ops, k, parts, part_off, z_pos, z_crd, static_cast<float*>(z_val), flags, st);
    }
    if (ops[0].dtype == NACHO_F64)
      return run_spadd5<double>(ops, k, parts, part_off, z_pos, z_crd, static_cast<double*>(z_val), flags, st);
    return run_spadd5<float>(ops, k, parts, part_off, z_pos, z_crd, static_cast<float*>(z_val), flags, st);
  }
  if (!fits_sa_tile(ops, k, parts, st))
    return fail(NACHO_ERR_INVALID_ARG, "partitions larger than %d entries: use the two-pass calls", kS4Tile);
  if (cudaMemsetAsync(flags, 0, sizeof(unsigned long long) * (parts->P + 1), st) != cudaSuccess)
    return fail(NACHO_ERR_CUDA, "memset look-back flags");
  if (ops[0].dtype == NACHO_F64) {
    Spadd4Args<double> a{make_ops(ops, k), parts_arg(parts), nullptr, part_off, flags, flags + parts->P, z_pos, z_crd,
                         static_cast<double*>(z_val)};
    return launch_spadd4<double, kS4Fused>(a, st);
  }
  Spadd4Args<float> a{make_ops(ops, k), parts_arg(parts), nullptr, part_off, flags, flags + parts->P, z_pos, z_crd,
                      static_cast<float*>(z_val)};
  return launch_spadd4<float, kS4Fused>(a, st);
}

size_t nacho_spadd_k_staged_workspace_size(const nacho_matrix* ops, int32_t k, int32_t P) {
  if (!ops || k < 1) return 0;
  const int64_t q = total_cost(ops, k);
  const size_t vs = ops[0].dtype == NACHO_F64 ? 8 : 4;
  const int64_t Pe = P > 0 ? P : 1;
  const int64_t nchunk = Pe * staged_chunks((q + Pe - 1) / Pe + (k - 1), k);   // partitions of nacho_partition
  return staged_ws_layout(nchunk, nullptr, nullptr) + align_up((size_t)q * 4) + align_up((size_t)q * vs);
}

/* Single read of the operands, no look-back: staged union + scan + placement (spadd4.cuh). */
nacho_status nacho_spadd_k_staged(const nacho_matrix* ops, int32_t k, const nacho_parts* parts, int64_t* part_off,
                                  int64_t* z_pos, int32_t* z_crd, void* z_val, void* ws, size_t ws_bytes,
                                  void* stream) {
  NACHO_TRY(check_ops(ops, k));
  if (!all_csr(ops, k)) return fail(NACHO_ERR_INVALID_ARG, "SpAdd supports CSR operands (COO: nacho_mixed_spadd_k)");
  NACHO_TRY(check_parts(parts, k));
  if (!z_pos || !part_off) return fail(NACHO_ERR_INVALID_ARG, "null z_pos / part_off");
  if (total_cost(ops, k) > 0 && (!z_crd || !z_val)) return fail(NACHO_ERR_INVALID_ARG, "null z_crd / z_val");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t chunks = staged_chunks(max_part_work(ops, k, parts_arg(parts), kS4Tile, st), k);
  const int64_t q = total_cost(ops, k);
  const size_t vs = ops[0].dtype == NACHO_F64 ? 8 : 4;
  const size_t need = staged_ws_layout((int64_t)parts->P * chunks, nullptr, nullptr) + align_up((size_t)q * 4) +
                      align_up((size_t)q * vs);
  if (ws_bytes < need || !ws) return fail(NACHO_ERR_WORKSPACE, "workspace %zu < %zu bytes", ws_bytes, need);
  if (ops[0].dtype == NACHO_F64)
    return run_spadd_staged<double>(ops, k, parts, part_off, z_pos, z_crd, static_cast<double*>(z_val),
                                    static_cast<char*>(ws), chunks, st);
  return run_spadd_staged<float>(ops, k, parts, part_off, z_pos, z_crd, static_cast<float*>(z_val),
                                 static_cast<char*>(ws), chunks, st);
}

// Carries of an SpMM over P partitions made by nacho_partition: one per tile-sized chunk.
int64_t spmm_carry_cap(const nacho_matrix* A, int64_t P) {
  const int64_t w = (A->nnz + P - 1) / P;
  return P * (w <= kSm2Tile ? 1 : (w + kSm2Tile - 1) / kSm2Tile);
}

size_t nacho_spmm_workspace_size(const nacho_matrix* A, int32_t P, int32_t nb) {
  if (!A) return 0;
  const bool auto_parts = P <= 0;
  const int64_t Pe = auto_parts ? nacho_auto_partitions(A, 1, 2) : P;
  const size_t vs = A->dtype == NACHO_F64 ? 8 : 4;
  const int64_t nc = spmm_carry_cap(A, Pe);
  return align_up(nc * 8) + align_up(nc * vs * (nb > 0 ? nb : 1)) + (auto_parts ? parts_bytes(Pe, 1) : 0);
}

nacho_status nacho_spmm(const nacho_matrix* A, const nacho_parts* parts, const void* B, int64_t ldb, int32_t nb,
                        void* C, int64_t ldc, void* ws, size_t ws_bytes, void* stream) {
  NACHO_TRY(check_matrix(A, "A"));
  if (A->format != NACHO_CSR) return fail(NACHO_ERR_INVALID_ARG, "SpMM supports CSR");
  if (nb < 1 || nb > 256) return fail(NACHO_ERR_INVALID_ARG, "nb = %d outside [1, 256]", nb);
  if (ldb < nb || ldc < nb) return fail(NACHO_ERR_SHAPE, "ldb/ldc < nb");
  if ((!B && A->ncols > 0) || (!C && A->nrows > 0)) return fail(NACHO_ERR_INVALID_ARG, "null B/C");
  if (parts) NACHO_TRY(check_parts(parts, 1));
  const size_t need = nacho_spmm_workspace_size(A, parts ? parts->P : 0, nb);
  if (ws_bytes < need || !ws) return fail(NACHO_ERR_WORKSPACE, "workspace %zu < %zu bytes", ws_bytes, need);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  char* c = static_cast<char*>(ws);
  const int64_t P = parts ? parts->P : nacho_auto_partitions(A, 1, 2);
  const size_t vs = A->dtype == NACHO_F64 ? 8 : 4;
  const int64_t cap = spmm_carry_cap(A, P);
  PartsArg pa;
  if (parts) pa = parts_arg(parts);
  else {
    pa = carve_parts(c + align_up(cap * 8) + align_up(cap * vs * nb), P, 1);
    NACHO_TRY(launch_partition(A, 1, pa, st));
  }
  const int64_t maxpart = max_part_work(A, 1, pa, kSm2Tile, st);
  if (A->dtype == NACHO_F64) {
    SpmmArgs<double> a{A->pos, A->crd, static_cast<const double*>(A->val), A->nrows, static_cast<const double*>(B), ldb,
                       nb, static_cast<double*>(C), ldc, pa.P, 1, pa.pos, pa.row_pos,
                       reinterpret_cast<int64_t*>(c), reinterpret_cast<double*>(c + align_up(cap * 8))};
    return run_spmm<double>(a, st, maxpart, cap);
  }
  SpmmArgs<float> a{A->pos, A->crd, static_cast<const float*>(A->val), A->nrows, static_cast<const float*>(B), ldb,
                    nb, static_cast<float*>(C), ldc, pa.P, 1, pa.pos, pa.row_pos,
                    reinterpret_cast<int64_t*>(c), reinterpret_cast<float*>(c + align_up(cap * 8))};
  return run_spmm<float>(a, st, maxpart, cap);
}

nacho_status nacho_validate(const nacho_matrix* A, void* stream) {
  NACHO_TRY(check_matrix(A, "A"));
  if (A->format == NACHO_COO) return fail(NACHO_ERR_INVALID_ARG, "nacho_validate takes CSR / DCSR operands");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int* flag = nullptr;
  if (cudaMallocAsync(&flag, sizeof(int), st) != cudaSuccess) return fail(NACHO_ERR_CUDA, "cudaMallocAsync");
  cudaMemsetAsync(flag, 0, sizeof(int), st);
  const int64_t n = A->nouter + 1;
  validate_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(*A, flag);
  nacho_status s = launched("validate_kernel");
  int h = 0;
  cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(flag, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return fail(NACHO_ERR_CUDA, "validate sync");
  if (s != NACHO_SUCCESS) return s;
  if (h) return fail(NACHO_ERR_FORMAT, "format invariant %d violated", h);
  return NACHO_SUCCESS;
}

}  // extern "C"
