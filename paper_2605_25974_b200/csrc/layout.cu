// §8(f) f4 — packed AoS records <-> SoA planes on the device.
//
// The reference keeps a PauliSum as packed records `x[W] u64 | z[W] u64 |
// flags u8 | coeff c128` (sums.py:48-57, 16W + 17 bytes, unaligned) and
// transposes to the SoA planes on the host (sums.py:417-426, :469-477).  Here
// the records cross PCIe as they are and the transpose runs on the GPU: a CTA
// stages a tile of whole records in shared memory with 16-byte accesses
// (tiles start at a multiple of 16 records, hence 16-byte aligned), then
// every thread moves one 64-bit field of one record; consecutive threads take
// consecutive records, so the plane side is coalesced.  Unaligned fields are
// assembled from aligned 32-bit shared-memory words (loads) or written as
// bytes (stores).
#include "common.cuh"

namespace plb {

constexpr int kLayTile = 128;     // records per tile (multiple of 16)
constexpr int kLayThreads = 256;

__device__ __forceinline__ u64 lds_u64_unaligned(const uint32_t* S, uint32_t off) {
  const uint32_t w = off >> 2, sh = (off & 3u) * 8u;
  const uint32_t a = S[w], b = S[w + 1], c = S[w + 2];
  const uint32_t lo = __funnelshift_r(a, b, sh), hi = __funnelshift_r(b, c, sh);
  return ((u64)hi << 32) | lo;
}

__device__ __forceinline__ void sts_u64_bytes(uint8_t* S, uint32_t off, u64 v) {
#pragma unroll
  for (int b = 0; b < 8; ++b) S[off + b] = (uint8_t)(v >> (8 * b));
}

template <int W>
__global__ void __launch_bounds__(kLayThreads)
k_aos_to_soa(const uint8_t* __restrict__ rec, int64_t M, u64* __restrict__ x, u64* __restrict__ z,
             uint8_t* __restrict__ k, u64* __restrict__ c, int64_t ld) {
  constexpr int RB = 16 * W + 17;
  constexpr int NF = 2 * W + 2;  // 64-bit fields per record: x[W], z[W], re, im
  __shared__ __align__(16) uint32_t S[(kLayTile * RB + 15) / 16 * 4 + 4];
  const int tid = threadIdx.x;
  for (int64_t t0 = (int64_t)blockIdx.x * kLayTile; t0 < M; t0 += (int64_t)gridDim.x * kLayTile) {
    const int nrec = (int)min((int64_t)kLayTile, M - t0);
    const uint32_t bytes = (uint32_t)nrec * RB;
    const uint8_t* src = rec + t0 * RB;
    for (uint32_t i = tid; i < bytes / 16; i += kLayThreads)
      reinterpret_cast<uint4*>(S)[i] = reinterpret_cast<const uint4*>(src)[i];
    for (uint32_t i = (bytes & ~15u) + tid; i < bytes; i += kLayThreads)
      reinterpret_cast<uint8_t*>(S)[i] = src[i];
    __syncthreads();
    for (int e = tid; e < nrec * NF; e += kLayThreads) {
      const int r = e % nrec, q = e / nrec;
      const uint32_t off = (uint32_t)r * RB + (q < 2 * W ? 8u * q : 16u * W + 1u + 8u * (q - 2 * W));
      const u64 v = lds_u64_unaligned(S, off);
      if (q < W) x[q * ld + t0 + r] = v;
      else if (q < 2 * W) z[(q - W) * ld + t0 + r] = v;
      else c[2 * (t0 + r) + (q - 2 * W)] = v;
    }
    for (int r = tid; r < nrec; r += kLayThreads)
      k[t0 + r] = reinterpret_cast<const uint8_t*>(S)[(uint32_t)r * RB + 16 * W];
    __syncthreads();
  }
}

template <int W>
__global__ void __launch_bounds__(kLayThreads)
k_soa_to_aos(const u64* __restrict__ x, const u64* __restrict__ z, const uint8_t* __restrict__ k,
             const u64* __restrict__ c, int64_t ld, int64_t M, uint8_t* __restrict__ rec) {
  constexpr int RB = 16 * W + 17;
  constexpr int NF = 2 * W + 2;
  __shared__ __align__(16) uint8_t S[(kLayTile * RB + 15) / 16 * 16];
  const int tid = threadIdx.x;
  for (int64_t t0 = (int64_t)blockIdx.x * kLayTile; t0 < M; t0 += (int64_t)gridDim.x * kLayTile) {
    const int nrec = (int)min((int64_t)kLayTile, M - t0);
    const uint32_t bytes = (uint32_t)nrec * RB;
    for (int e = tid; e < nrec * NF; e += kLayThreads) {
      const int r = e % nrec, q = e / nrec;
      u64 v;
      if (q < W) v = x[q * ld + t0 + r];
      else if (q < 2 * W) v = z[(q - W) * ld + t0 + r];
      else v = c[2 * (t0 + r) + (q - 2 * W)];
      const uint32_t off = (uint32_t)r * RB + (q < 2 * W ? 8u * q : 16u * W + 1u + 8u * (q - 2 * W));
      sts_u64_bytes(S, off, v);
    }
    for (int r = tid; r < nrec; r += kLayThreads) S[(uint32_t)r * RB + 16 * W] = k ? k[t0 + r] : 0;
    __syncthreads();
    uint8_t* dst = rec + t0 * RB;
    for (uint32_t i = tid; i < bytes / 16; i += kLayThreads)
      reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(S)[i];
    for (uint32_t i = (bytes & ~15u) + tid; i < bytes; i += kLayThreads) dst[i] = S[i];
    __syncthreads();
  }
}

template <int W>
static int launch_a2s(const uint8_t* rec, int64_t M, u64* x, u64* z, uint8_t* k, u64* c, int64_t ld,
                      cudaStream_t st) {
  const int64_t tiles = ceil_div(M, (int64_t)kLayTile);
  const unsigned grid = (unsigned)std::min<int64_t>(tiles, 8 * (int64_t)num_sms());
  k_aos_to_soa<W><<<grid, kLayThreads, 0, st>>>(rec, M, x, z, k, c, ld);
  PLB_CHECK_LAUNCH("k_aos_to_soa");
  return PL_OK;
}

template <int W>
static int launch_s2a(const u64* x, const u64* z, const uint8_t* k, const u64* c, int64_t ld,
                      int64_t M, uint8_t* rec, cudaStream_t st) {
  const int64_t tiles = ceil_div(M, (int64_t)kLayTile);
  const unsigned grid = (unsigned)std::min<int64_t>(tiles, 8 * (int64_t)num_sms());
  k_soa_to_aos<W><<<grid, kLayThreads, 0, st>>>(x, z, k, c, ld, M, rec);
  PLB_CHECK_LAUNCH("k_soa_to_aos");
  return PL_OK;
}

}  // namespace plb

using namespace plb;

extern "C" int pl_aos_to_soa(int W, int64_t M, const void* records, uint64_t* x, uint64_t* z,
                             uint8_t* k, double* c, int64_t ld, void* stream) {
  if (!valid_words(W)) {
    set_error("unsupported word count W=%d", W);
    return PL_ERR_TIER;
  }
  if (M < 0 || ld < M || (M > 0 && (!records || !x || !z || !k || !c)) ||
      (reinterpret_cast<uintptr_t>(records) & 15)) {
    set_error("pl_aos_to_soa: bad argument (records must be 16-byte aligned, ld >= M)");
    return PL_ERR_ARG;
  }
  if (M == 0) return PL_OK;
  return PLB_DISPATCH_W(W, launch_a2s, (const uint8_t*)records, M, (u64*)x, (u64*)z, k, (u64*)c, ld,
                        (cudaStream_t)stream);
}

extern "C" int pl_soa_to_aos(int W, int64_t M, const uint64_t* x, const uint64_t* z,
                             const uint8_t* k, const double* c, int64_t ld, void* records,
                             void* stream) {
  if (!valid_words(W)) {
    set_error("unsupported word count W=%d", W);
    return PL_ERR_TIER;
  }
  if (M < 0 || ld < M || (M > 0 && (!records || !x || !z || !c)) ||
      (reinterpret_cast<uintptr_t>(records) & 15)) {
    set_error("pl_soa_to_aos: bad argument (records must be 16-byte aligned, ld >= M)");
    return PL_ERR_ARG;
  }
  if (M == 0) return PL_OK;
  return PLB_DISPATCH_W(W, launch_s2a, (const u64*)x, (const u64*)z, k, (const u64*)c, ld, M,
                        (uint8_t*)records,
                        (cudaStream_t)stream);
}
