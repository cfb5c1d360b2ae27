// spmv7.cuh -- EXPERIMENTAL (NACHO_SPMV_IMPL=7; the default is spmv3.cuh, faster on B200: C5 9.9 ms
// against 13.2 ms for this kernel -- two CTAs per SM of one compute group each cannot hide the x
// gathers and scans that spmv3's three independent CTAs per SM overlap).
// The partitioned CSR / DCSR SpMV of spmv3.cuh as a
// persistent, software-pipelined kernel: the crd / val stream of every tile (and the row pointers of
// its rows) reach shared memory by 1-D bulk copies (cp.async.bulk -> UBLKCP) issued by a producer
// warp one tile ahead, so the compute warps never wait on HBM for the stream; their only global
// latency is the x gather, whose addresses they read from shared memory.
//
// One CTA = producer warp (8) + compute warps (0-7) over a ring of NS stages; job j = tile (partition
// p, chunk c) of spmv3's numbering, taken round-robin (j = blockIdx.x + i * gridDim.x: tiles are
// independent -- the row cut by a tile's end leaves a carry that spmv_fixup_kernel adds in partition
// order, Listing 8's bounds, P:2118-2150 -- so no ordering between CTAs is needed).
//   producer: tile bounds [s, e) (Parts positions; chunks of a large partition are cut in position
//     space) and rows [rp0, rpE]; bulk copies of crd / val [s, e) and of the row ends
//     pos[rp0 + 1 .. rpE] (int64, when at most kSv7Pool of them; else the compute warps read them
//     from global memory);
//   compute: local row ends, products a_ij * x_j (x gathered by crd from shared memory), the stage
//     is released, then spmv3's segmented scan / row sums / carry (sv3_tail).
#pragma once
#include "spmv3.cuh"
#include "tma.cuh"

namespace nacho {

constexpr int kSv7Compute = kSv3Threads;        // compute threads: warps 0 .. 7
constexpr int kSv7Threads = kSv7Compute + 32;   // + the producer warp
constexpr int kSv7Pool = 1024;                  // row ends staged per tile (int64)
constexpr int kSv7Stages = 2;
// positions per thread: spmv3's (tiles of 4096 fp32 / 2048 fp64 positions; two CTAs per SM).  Tried:
// half tiles with three stages and three CTAs per SM -- 15.2 ms on C5 against 13.2 ms.
template <typename T> struct Sv7Cfg { static constexpr int V = Sv3Cfg<T>::V; };
template <typename T>
__host__ __device__ constexpr int sv7_tile() { return kSv7Compute * Sv7Cfg<T>::V; }

template <typename T>
struct alignas(16) Sv7Stage {
  int32_t crd[sv7_tile<T>() + 8];
  T val[sv7_tile<T>() + 8];
  alignas(16) int64_t pos[kSv7Pool + 4];
  alignas(16) T xs[sizeof(T) == 4 ? 4 : sv7_tile<T>() + 8];   // fp64: x[crd] gathered by cp.async (fp32: into crd)
  int64_t job, s, rp0, rpE, ps;   // job -1: stop
  int32_t n, lim_r, pooled, skip, head;   // head: slots before position s (bulk copies start at s & ~3)
};

template <typename T>
struct Sv7Smem {
  Sv7Stage<T> st[kSv7Stages];
  int32_t send[kSv7Pool + 4];
  alignas(16) T sprod[sv7_tile<T>() + sv7_tile<T>() / 8 + 4];
  alignas(16) uint8_t mark[sv7_tile<T>() + 16];
  FV<T> s_wagg[kSv7Compute / 32];
  T s_cin[kSv7Compute];
  int32_t s_ffl[kSv7Compute];
  uint64_t full[kSv7Stages], empty[kSv7Stages];
};

template <typename T>
__device__ __forceinline__ void sv7_produce(const SpmvArgs<T>& a, Sv7Smem<T>& sh, int64_t njobs) {
  constexpr int SLOTS = sv7_tile<T>();
  const int lane = threadIdx.x & 31;
  int it = 0;
  const int64_t nnz = ldg(a.pos + a.nouter);
  // the next job's Parts record is read before waiting for its stage
  auto rec = [&](int64_t jj, int64_t& sp_, int64_t& ep_, int64_t& r0_, int64_t& r1_) {
    if (jj >= njobs) return;
    const int64_t pp = a.chunks == 1 ? jj : jj / a.chunks;
    sp_ = ldg(a.ppos + pp); ep_ = ldg(a.ppos + pp + 1);
    r0_ = ldg(a.prow + pp); r1_ = ldg(a.prow + pp + 1);
  };
  int64_t nsp = 0, nep = 0, nr0 = 0, nr1 = 0;
  rec(blockIdx.x, nsp, nep, nr0, nr1);
  for (int64_t j = blockIdx.x;; j += gridDim.x, ++it) {
    const int s_ = it % kSv7Stages;
    const uint32_t ph = (uint32_t)(it / kSv7Stages) & 1u;
    const int64_t sp = nsp, ep = nep, rp0p = nr0, rpEp = nr1;
    rec(j + gridDim.x, nsp, nep, nr0, nr1);
    while (!mbar_try_wait(&sh.empty[s_], ph ^ 1u)) __nanosleep(64);
    Sv7Stage<T>& g = sh.st[s_];
    if (j >= njobs) {
      if (lane == 0) { g.job = -1; mbar_arrive(&sh.full[s_]); }
      return;
    }
    const int64_t p = a.chunks == 1 ? j : j / a.chunks;
    const int c = (int)(j - p * a.chunks);
    const int64_t s = sp + (int64_t)c * SLOTS;
    if (c > 0 && s >= ep) {   // past the partition: a zero carry (spmv3's rule)
      if (lane == 0) { g.job = j; g.skip = 1; g.rpE = rpEp; mbar_arrive(&sh.full[s_]); }
      continue;
    }
    const int64_t e = ep - s < SLOTS ? ep : s + SLOTS;
    int64_t rp0 = rp0p, rpE = rpEp;
    if (a.chunks > 1) {   // rows holding the chunk's cuts: 32-ary searches over the partition's rows
      const int64_t hi = rpEp < a.nouter ? rpEp : a.nouter;
      if (c > 0) rp0 = warp_highest_true(rp0p, hi, [&](int64_t x) { return ldg(a.pos + x) <= s; });
      if (e < ep) rpE = warp_highest_true(rp0p, hi, [&](int64_t x) { return ldg(a.pos + x) <= e; });
    }
    const int n = (int)(e - s);
    const int lim_r = (int)((rpE < a.nouter ? rpE : a.nouter) - rp0);
    // crd / val: [s & ~3, ceil4(e)) when in bounds (the <= 3 slots either side land in the pads),
    // else [.., e & ~3) and plain loads of the rest
    const int64_t lo = s & ~int64_t(3);
    int64_t hi = (e + 3) & ~int64_t(3);
    if (hi > nnz) hi = e & ~int64_t(3);
    if (hi < lo) hi = lo;
    const int head = (int)(s - lo);
    // row ends pos[rp0 + 1 .. rp0 + lim_r]: [ps, ceil2(rp0 + lim_r + 1)) clamped to the array
    const int64_t ps = (rp0 + 1) & ~int64_t(1);
    const int64_t pneed = rp0 + lim_r + 1;
    const bool pooled = lim_r > 0 && pneed - ps <= kSv7Pool;
    int64_t pe = (pneed + 1) & ~int64_t(1);
    if (pe > a.nouter + 1) pe = pneed & ~int64_t(1);
    if (!pooled || pe < ps) pe = ps;
    const uint32_t bytes = (uint32_t)(hi - lo) * (4u + (uint32_t)sizeof(T)) + (uint32_t)(pe - ps) * 8u;
    if (lane == 0) {
      g.job = j; g.skip = 0; g.s = s; g.rp0 = rp0; g.rpE = rpE; g.ps = ps;
      g.n = n; g.lim_r = lim_r; g.pooled = pooled; g.head = head;
      if (bytes) mbar_expect_tx(&sh.full[s_], bytes);
    }
    __syncwarp();
    if (lane == 0 && hi > lo) bulk_g2s(g.crd, a.crd + lo, (uint32_t)(hi - lo) * 4u, &sh.full[s_]);
    if (lane == 1 && hi > lo) bulk_g2s(g.val, a.val + lo, (uint32_t)(hi - lo) * (uint32_t)sizeof(T), &sh.full[s_]);
    if (lane == 2 && pe > ps) bulk_g2s(g.pos, a.pos + ps, (uint32_t)(pe - ps) * 8u, &sh.full[s_]);
    for (int64_t q = (hi > lo ? hi : lo) + lane; q < e; q += 32) {   // the array's last < 4 entries
      g.crd[q - lo] = ldg(a.crd + q);
      g.val[q - lo] = ldg(a.val + q);
    }
    if (pooled)
      for (int64_t r = pe + lane; r < pneed; r += 32) g.pos[r - ps] = ldg(a.pos + r);
    __syncwarp();
    if (lane == 0) mbar_arrive(&sh.full[s_]);
  }
}

// Slots receiving x[crd]: fp32 overwrites the column indices in place (each thread reads its index
// before its cp.async writes the slot), fp64 needs 8-byte slots.
template <typename T>
__device__ __forceinline__ T* sv7_xs(Sv7Stage<T>& g) {
  if constexpr (sizeof(T) == 4) return reinterpret_cast<T*>(g.crd);
  else return g.xs;
}

// The x gathers of a tile: every compute thread reads the column indices of its lane-strided slots
// and issues one cp.async per slot that overwrites the slot's crd with x[crd] -- no registers held, so
// the gathers of tile n + 1 are in flight while tile n's scan and row sums run.
template <typename T>
__device__ __forceinline__ void sv7_gather(const SpmvArgs<T>& a, Sv7Stage<T>& g, int wb, int lane) {
  constexpr int V = Sv7Cfg<T>::V;
  const int n = g.n, head = g.head;
  if (g.skip) return;
  int32_t* cs = g.crd + head + wb + lane;
#pragma unroll
  for (int i = 0; i < V; ++i) {
    if (wb + 32 * i + lane < n) {
      const uint32_t c = (uint32_t)cs[32 * i];
      cp_async_ca<sizeof(T)>(sv7_xs(g) + head + wb + lane + 32 * i, a.x + c);
    }
  }
}

// Tile metadata the scan of a tile needs after its stage has been handed back.
struct Sv7Job {
  int64_t j, s, rp0, rpE;
  int n, lim_r;
  bool pooled, skip;
};

template <typename T, bool DY>
__device__ __forceinline__ void sv7_compute(const SpmvArgs<T>& a, Sv7Smem<T>& sh) {
  constexpr int V = Sv7Cfg<T>::V;
  constexpr int WCH = 32 * V;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int wb = w * WCH;
  Sv7Job prev;
  prev.j = -1;
  // iteration it: the gathers of tile it go out, tile it - 1's scan and row sums run while they fly,
  // then tile it's products are formed and its stage is handed back (one sprod buffer)
  auto tail = [&](const Sv7Job& q) {
    if (q.skip) {
      if (tid == 0) {
        a.carry_row[q.j] = q.rpE < a.nouter ? q.rpE : -1;
        a.carry_val[q.j] = T(0);
      }
      return;
    }
    sv3_tail<T, V, DY, 1>(a, q.j, q.s, q.n, q.rp0, q.rpE, q.lim_r, q.pooled && q.lim_r <= kSv7Pool, sh.send, sh.sprod,
                          sh.mark, sh.s_wagg, sh.s_cin, sh.s_ffl);
  };
  for (int it = 0;; ++it) {
    const int s_ = it % kSv7Stages;
    while (!mbar_try_wait(&sh.full[s_], (uint32_t)(it / kSv7Stages) & 1u)) {
    }
    Sv7Stage<T>& g = sh.st[s_];
    Sv7Job cur;
    cur.j = g.job;
    if (cur.j >= 0) {
      cur.skip = g.skip != 0;
      cur.s = g.s; cur.rp0 = g.rp0; cur.rpE = g.rpE;
      cur.n = g.n; cur.lim_r = g.lim_r; cur.pooled = g.pooled != 0;
      sv7_gather<T>(a, g, wb, lane);
    }
    cp_async_commit();
    if (prev.j >= 0) tail(prev);
    named_sync(1, kSv7Compute);   // sprod / send / mark of the previous tile are free
    if (cur.j < 0) return;
    if (!cur.skip) {
      // clear the row-start marks; local row ends from the staged row pointers
      if constexpr (V == 16) reinterpret_cast<uint4*>(sh.mark)[tid] = make_uint4(0, 0, 0, 0);
      else if constexpr (V == 8) reinterpret_cast<uint2*>(sh.mark)[tid] = make_uint2(0, 0);
      else for (int i = 0; i < V; ++i) sh.mark[tid * V + i] = 0;
      if (cur.pooled) {
        const int64_t pb = cur.rp0 + 1 - g.ps;
        for (int r = tid; r < cur.lim_r; r += kSv7Compute) sh.send[r] = (int32_t)(g.pos[pb + r] - cur.s);
      }
      // products from this thread's own slots (its cp.async gathers)
      cp_async_wait<0>();
      const int head = g.head, n = cur.n;
      const T* xs = sv7_xs(g) + head + wb + lane;
      const T* vs = g.val + head + wb + lane;
      T* sp = sh.sprod + sv3_slot<T>(wb) + lane;
#pragma unroll
      for (int i = 0; i < V; ++i)
        if (wb + 32 * i + lane < n) sp[sv3_stride32<T>() * i] = vs[32 * i] * xs[32 * i];
    }
    fence_proxy_async();          // the stage's generic / cp.async writes before the next bulk copies
    named_sync(1, kSv7Compute);   // products and row ends in place; the stage is consumed
    if (tid == 0) mbar_arrive(&sh.empty[s_]);
    prev = cur;
  }
}

template <typename T, bool DY>
__global__ void __launch_bounds__(kSv7Threads, 2) spmv7_kernel(const __grid_constant__ SpmvArgs<T> a, int64_t njobs) {
  extern __shared__ __align__(128) unsigned char sv7_raw[];
  Sv7Smem<T>& sh = *reinterpret_cast<Sv7Smem<T>*>(sv7_raw);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kSv7Stages; ++s) {
      mbar_init(&sh.full[s], 1);
      mbar_init(&sh.empty[s], 1);
    }
    fence_barrier_init();
  }
  __syncthreads();
  if ((threadIdx.x >> 5) == kSv7Compute / 32) sv7_produce<T>(a, sh, njobs);
  else sv7_compute<T, DY>(a, sh);
}

}  // namespace nacho
