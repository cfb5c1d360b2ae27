// dist.cuh -- device-level sharding and the exchange step of the multi-GPU path: the
// paper's partition is the device decomposition.  With D devices, device d owns the coordinate range
// [b_d, b_{d+1}) of Alg. 1 run with P = D (one partition per processor; the boundaries
// are saved positions), so every device does Q*/D +- Delta work (Theorem 1).
// The paper itself is shared-memory only; the exchange is this build's addition:
//   SpMV  -- x replicated (broadcast at setup); device d computes the rows it holds, the row cut by
//            b_{d+1} leaves a partial sum ("seam carry") that is added, in device order, to the
//            device that owns the row (R7: the device holding the row's last entry); the owned y
//            segments are gathered with one broadcast per device.
//   SpAdd -- equal coordinates never straddle a cut, so no values merge at seams:
//            the device union sizes give global offsets; Z.crd / Z.val / Z.pos segments are gathered.
// NCCL is loaded at run time (dlopen of libnccl.so.2: the copy torch already loaded, else the
// system one), so libnacho.so has no link-time NCCL dependency.
#pragma once
#include <dlfcn.h>

#include <cstdint>
#include <mutex>

#include <nccl.h>

#include "common.cuh"

namespace nacho {

// ------------------------------------------------------------------ kernels
// Device cuts of a single-operand matrix for D devices: cut d = Alg. 1 at Q_d = floor(d Q*/D) in
// closed form (k = 1: position Q_d, row = highest x with pos[x] <= Q_d); cut 0 is the
// origin, cut D the end (R1).  One thread per cut, binary search over pos.
__global__ void device_cuts_kernel(const int64_t* __restrict__ pos, int64_t nouter, int64_t nnz, int32_t D,
                                   int64_t* __restrict__ cuts) {
  const int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d > D) return;
  if (d == 0) { cuts[0] = 0; cuts[1] = 0; return; }
  if (d == D) { cuts[2 * D] = nouter; cuts[2 * D + 1] = nnz; return; }
  const int64_t Q = query_of(nnz, D, d);
  int64_t lo = 0, hi = nouter;   // highest x in [0, nouter] with pos[x] <= Q
  while (lo < hi) {
    const int64_t mid = lo + (hi - lo + 1) / 2;
    if (__ldg(pos + mid) <= Q) lo = mid; else hi = mid - 1;
  }
  cuts[2 * d] = lo;
  cuts[2 * d + 1] = Q;
}

// Row pointers of a shard: rows [row_lo, row_lo + nloc) of the full matrix restricted to the
// positions [pos_lo, pos_hi) (first / last row possibly partial), rebased to start at 0.
__global__ void shard_rows_kernel(const int64_t* __restrict__ pos, int64_t row_lo, int64_t nloc, int64_t pos_lo,
                                  int64_t pos_hi, int64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= nloc; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t p = i == 0 ? pos_lo : (i == nloc ? pos_hi : __ldg(pos + row_lo + i));
    p = p < pos_lo ? pos_lo : (p > pos_hi ? pos_hi : p);
    out[i] = p - pos_lo;
  }
}

// The device's outgoing seam carry: (row, value bits) of its last local row when that row is owned
// by a later device, else (-1, 0).
template <typename T>
__global__ void carry_pack_kernel(const T* __restrict__ y_local, int64_t nloc, int64_t row_lo, int32_t has_carry,
                                  int64_t* __restrict__ out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (has_carry && nloc > 0) {
    T v = y_local[nloc - 1];
    int64_t bits = 0;
    memcpy(&bits, &v, sizeof(T));
    out[0] = row_lo + nloc - 1;
    out[1] = bits;
  } else {
    out[0] = -1;
    out[1] = 0;
  }
}

// Seam fix-up (Listing 8's carry rule at device level): the owner of its first row adds the carries
// of the devices before it that end in that row, in device order (a dense row may span several
// devices: the chain walks back while the carry row matches).
template <typename T>
__global__ void seam_kernel(const int64_t* __restrict__ carries, int32_t D, int32_t d, int64_t row_lo,
                            int32_t owns_first, T* __restrict__ y_local) {
  if (threadIdx.x != 0 || blockIdx.x != 0 || !owns_first) return;
  int q = d - 1;
  while (q >= 0 && carries[2 * q] == row_lo) --q;
  T acc = y_local[0];
  T s = T(0);
  for (int r = q + 1; r < d; ++r) {   // device order: the earliest carry first
    T v;
    memcpy(&v, carries + 2 * r + 1, sizeof(T));
    s = r == q + 1 ? v : s + v;
  }
  if (q + 1 < d) y_local[0] = s + acc;
}

// Z.pos segment of a device's SpAdd shard: rows row_lo + 1 .. row_lo + nown of the global Z.pos are
// off + local_zpos[1 .. nown].
__global__ void zpos_segment_kernel(const int64_t* __restrict__ local_zpos, int64_t nown, const int64_t* __restrict__ off,
                                    int64_t* __restrict__ out) {
  const int64_t o = *off;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nown; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = o + local_zpos[i + 1];
}

// Exclusive prefix of the D gathered union sizes (one thread; D <= a few hundred).
__global__ void offsets_kernel(const int64_t* __restrict__ counts, int32_t D, int64_t* __restrict__ off) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  int64_t s = 0;
  for (int r = 0; r < D; ++r) { off[r] = s; s += counts[r]; }
  off[D] = s;
}

// ------------------------------------------------------------------ NCCL (loaded at run time)
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  const char* (*GetErrorString)(ncclResult_t);
  bool ok = false;
};

inline NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);   // torch's copy, if already loaded
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
#define NACHO_SYM(f, n) api.f = reinterpret_cast<decltype(api.f)>(dlsym(h, n))
    NACHO_SYM(GetUniqueId, "ncclGetUniqueId");
    NACHO_SYM(CommInitRank, "ncclCommInitRank");
    NACHO_SYM(CommDestroy, "ncclCommDestroy");
    NACHO_SYM(Broadcast, "ncclBroadcast");
    NACHO_SYM(AllGather, "ncclAllGather");
    NACHO_SYM(GroupStart, "ncclGroupStart");
    NACHO_SYM(GroupEnd, "ncclGroupEnd");
    NACHO_SYM(GetErrorString, "ncclGetErrorString");
#undef NACHO_SYM
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.Broadcast && api.AllGather &&
             api.GroupStart && api.GroupEnd && api.GetErrorString;
  });
  return api;
}

}  // namespace nacho

// The opaque communicator of the C ABI.
struct nacho_dist_s {
  ncclComm_t comm;
  int32_t nranks, rank;
};
