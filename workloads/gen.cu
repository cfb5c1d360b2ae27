// gen.cu -- device twin of workloads/recipe.py (input generator only; none of the method's
// arithmetic lives here).  Every function reproduces the numpy recipe bit for bit: integer
// arithmetic on (seed, stream, a, b) counters; values use 24 random bits so fp32/fp64 are exact.
// Built into workloads/libnacho_gen.so; it shares no code with the oracle or with libnacho.
#include <cstdint>
#include <cuda_runtime.h>

namespace {

constexpr uint64_t K_SEED = 0x9E3779B97F4A7C15ull, K_STREAM = 0xD1B54A32D192ED03ull;
constexpr uint64_t K_A = 0xABC98388FB8FAC03ull, K_B = 0x8CB92BA72F3D8DD7ull;
enum { S_PERM = 1, S_COL, S_VAL, S_X, S_B, S_KIND, S_OUTER, S_REUSE_B, S_REUSE_C, S_PICK_C };

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27; z *= 0x94D049BB133111EBull;
  z ^= z >> 31; return z;
}
__device__ __forceinline__ uint64_t hash4(uint64_t seed, uint64_t stream, uint64_t a, uint64_t b) {
  return mix64(seed * K_SEED + stream * K_STREAM + a * K_A + b * K_B);
}
__device__ __forceinline__ int feistel_bits(int64_t n) {
  int b = 64 - __clzll((unsigned long long)(n - 1));
  if (b < 2) b = 2;
  return (b + 1) / 2;
}
__device__ uint64_t feistel_perm(uint64_t x, int64_t n, uint64_t seed) {
  if (n <= 1) return 0;
  const int h = feistel_bits(n);
  const uint64_t mask = (1ull << h) - 1;
  do {
    for (int rnd = 0; rnd < 4; ++rnd) {
      uint64_t L = x >> h, R = x & mask;
      uint64_t F = hash4(seed, S_PERM, R, (uint64_t)rnd) & mask;
      x = (R << h) | (L ^ F);
    }
  } while (x >= (uint64_t)n);
  return x;
}

__global__ void k_degrees(int64_t m, int64_t cdiv, int64_t cap, int64_t min_deg, uint64_t seed,
                          int64_t dense_row, int64_t dense_deg, int64_t* __restrict__ deg) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < m; r += (int64_t)gridDim.x * blockDim.x) {
    int64_t rank = (int64_t)feistel_perm((uint64_t)r, m, seed);
    int64_t d = cdiv / (rank + 1);
    d = d < min_deg ? min_deg : d;
    d = d > cap ? cap : d;
    if (r == dense_row) d = dense_deg;
    deg[r] = d;
  }
}

__device__ __forceinline__ int64_t pick(uint64_t seed, uint64_t stream, int64_t r, int64_t k, int64_t lo, int64_t hi) {
  return lo + (int64_t)(hash4(seed, stream, (uint64_t)r, (uint64_t)k) % (uint64_t)(hi - lo));
}

// kind: 0 local, 1 uniform, 2 web
__device__ int64_t column_of(int kind, int64_t m, int64_t n, uint64_t seed, uint64_t stream,
                             int64_t r, int64_t k, int64_t d) {
  if (d >= n) return k;
  int64_t w, w0;
  if (kind == 1) { w = n; w0 = 0; }
  else {
    w = 4 * d > 4096 ? 4 * d : 4096;
    if (w > n) w = n;
    int64_t centre = (r * n) / m;
    w0 = centre - w / 2;
    if (w0 > n - w) w0 = n - w;
    if (w0 < 0) w0 = 0;
  }
  int64_t lo = w0 + (k * w) / d, hi = w0 + ((k + 1) * w) / d;
  int64_t col = pick(seed, stream, r, k, lo, hi);
  if (kind == 2) {
    int64_t npop = n / 64 > 1 ? n / 64 : 1;
    int64_t d1 = d / 2;
    bool web = ((hash4(seed, S_KIND, (uint64_t)r, 0) & 1ull) == 1ull) && d1 <= npop && (d - d1) <= n - npop && d1 > 0;
    if (web) {
      int64_t lw, hw;
      if (k < d1) { lw = (k * npop) / d1; hw = ((k + 1) * npop) / d1; }
      else { int64_t kk = k - d1, dd = d - d1; lw = npop + (kk * (n - npop)) / dd; hw = npop + ((kk + 1) * (n - npop)) / dd; }
      if (hw < lw + 1) hw = lw + 1;
      col = pick(seed, stream, r, k, lw, hw);
    }
  }
  return col;
}

__device__ __forceinline__ int64_t row_of_entry(const int64_t* __restrict__ pos, int64_t m, int64_t e) {
  int64_t a = 0, b = m;  // largest r with pos[r] <= e  (pos[0] = 0 <= e)
  while (a < b) { int64_t mid = a + (b - a + 1) / 2; if (pos[mid] <= e) a = mid; else b = mid - 1; }
  return a;
}

// mode: 0 plain (stream_own), 1 C2 operand B (reuse A 30%), 2 C2 operand C (reuse A or B 30%)
__global__ void k_columns(int kind, int mode, int64_t m, int64_t n, uint64_t seed, const int64_t* __restrict__ pos,
                          int64_t e_lo, int64_t e_hi, uint64_t stream_own, uint64_t stream_a, uint64_t stream_b,
                          int32_t* __restrict__ crd) {
  for (int64_t e = e_lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < e_hi; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = row_of_entry(pos, m, e);
    int64_t k = e - pos[r], d = pos[r + 1] - pos[r];
    int64_t c;
    if (mode == 1 && (hash4(seed, S_REUSE_B, r, k) % 10ull) < 3ull) c = column_of(kind, m, n, seed, stream_a, r, k, d);
    else if (mode == 2 && (hash4(seed, S_REUSE_C, r, k) % 10ull) < 3ull)
      c = column_of(kind, m, n, seed, (hash4(seed, S_PICK_C, r, k) & 1ull) ? stream_b : stream_a, r, k, d);
    else c = column_of(kind, m, n, seed, stream_own, r, k, d);
    crd[e - e_lo] = (int32_t)c;
  }
}

__global__ void k_columns_rows(int kind, int64_t m, int64_t n, uint64_t seed, const int64_t* __restrict__ pos,
                               const int32_t* __restrict__ outer, int64_t nouter, int64_t nnz, uint64_t stream,
                               int32_t* __restrict__ crd) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t ip = row_of_entry(pos, nouter, e);
    int64_t k = e - pos[ip], d = pos[ip + 1] - pos[ip];
    crd[e] = (int32_t)column_of(kind, m, n, seed, stream, (int64_t)outer[ip], k, d);
  }
}

__device__ __forceinline__ double value_of(uint64_t seed, uint64_t stream, uint64_t idx, int mode, int kmax) {
  uint64_t h = hash4(seed, stream, idx, 0);
  int64_t bits = (int64_t)(h >> 40);
  if (mode == 0) return 0.5 + (double)bits * 5.9604644775390625e-08;  // 2^-24
  double mag = (double)(1 + bits % kmax);
  return (h >> 63) ? -mag : mag;
}

__global__ void k_values(uint64_t seed, uint64_t stream, int64_t i0, int64_t n, int mode, int kmax, int f64, void* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double v = value_of(seed, stream, (uint64_t)(i0 + i), mode, kmax);
    if (f64) ((double*)out)[i] = v; else ((float*)out)[i] = (float)v;
  }
}

__global__ void k_outer(int64_t m, int64_t nouter, uint64_t seed, int32_t* __restrict__ out) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nouter; k += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = (k * m) / nouter, hi = ((k + 1) * m) / nouter;
    out[k] = (int32_t)pick(seed, S_OUTER, k, 0, lo, hi);
  }
}

inline int grid_for(int64_t n) {
  int64_t g = (n + 255) / 256;
  if (g > 148 * 64) g = 148 * 64;
  if (g < 1) g = 1;
  return (int)g;
}

}  // namespace

extern "C" {
int wl_degrees(int64_t m, int64_t cdiv, int64_t cap, int64_t min_deg, uint64_t seed, int64_t dense_row,
               int64_t dense_deg, int64_t* deg, void* stream) {
  k_degrees<<<grid_for(m), 256, 0, (cudaStream_t)stream>>>(m, cdiv, cap, min_deg, seed, dense_row, dense_deg, deg);
  return (int)cudaGetLastError();
}
int wl_columns(int kind, int mode, int64_t m, int64_t n, uint64_t seed, const int64_t* pos, int64_t nnz,
               uint64_t stream_own, uint64_t stream_a, uint64_t stream_b, int32_t* crd, void* stream) {
  k_columns<<<grid_for(nnz), 256, 0, (cudaStream_t)stream>>>(kind, mode, m, n, seed, pos, 0, nnz, stream_own, stream_a,
                                                             stream_b, crd);
  return (int)cudaGetLastError();
}
// entries [e_lo, e_hi) only (a device shard's slice; pos is the full row-pointer array)
int wl_columns_range(int kind, int mode, int64_t m, int64_t n, uint64_t seed, const int64_t* pos, int64_t e_lo,
                     int64_t e_hi, uint64_t stream_own, uint64_t stream_a, uint64_t stream_b, int32_t* crd,
                     void* stream) {
  k_columns<<<grid_for(e_hi - e_lo), 256, 0, (cudaStream_t)stream>>>(kind, mode, m, n, seed, pos, e_lo, e_hi, stream_own,
                                                                     stream_a, stream_b, crd);
  return (int)cudaGetLastError();
}
int wl_columns_rows(int kind, int64_t m, int64_t n, uint64_t seed, const int64_t* pos, const int32_t* outer,
                    int64_t nouter, int64_t nnz, uint64_t cstream, int32_t* crd, void* stream) {
  k_columns_rows<<<grid_for(nnz), 256, 0, (cudaStream_t)stream>>>(kind, m, n, seed, pos, outer, nouter, nnz, cstream, crd);
  return (int)cudaGetLastError();
}
int wl_values(uint64_t seed, uint64_t vstream, int64_t n, int mode, int kmax, int f64, void* out, void* stream) {
  k_values<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(seed, vstream, 0, n, mode, kmax, f64, out);
  return (int)cudaGetLastError();
}
int wl_values_range(uint64_t seed, uint64_t vstream, int64_t i0, int64_t n, int mode, int kmax, int f64, void* out,
                    void* stream) {
  k_values<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(seed, vstream, i0, n, mode, kmax, f64, out);
  return (int)cudaGetLastError();
}
int wl_outer(int64_t m, int64_t nouter, uint64_t seed, int32_t* out, void* stream) {
  k_outer<<<grid_for(nouter), 256, 0, (cudaStream_t)stream>>>(m, nouter, seed, out);
  return (int)cudaGetLastError();
}
}
