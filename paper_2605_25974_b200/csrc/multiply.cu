// K1 batched pair multiply, batched commutation parity, raw outer product.
//
// K1 replaces bench.py:168-177 (_batch_pair_multiply) over the SoA planes:
// HBM-bound streaming (read 2x(16W+1) B, write 16W+1 B per pair = 387 B at
// W=8).  Each thread owns two adjacent pairs so every plane access is one
// 128-bit load/store, coalesced across the warp.
#include "common.cuh"
#include <cstring>
#include <mutex>

namespace plb {

__device__ __forceinline__ ulonglong2 ld2(const u64* p) {
  return __ldg(reinterpret_cast<const ulonglong2*>(p));
}
__device__ __forceinline__ void st2(u64* p, u64 a, u64 b) {
  *reinterpret_cast<ulonglong2*>(p) = make_ulonglong2(a, b);
}

template <int W, bool VEC>
__global__ void __launch_bounds__(256)
k_batch_multiply(int64_t P, const u64* __restrict__ ax, const u64* __restrict__ az,
                 const uint8_t* __restrict__ ak, int64_t lda,
                 const u64* __restrict__ bx, const u64* __restrict__ bz,
                 const uint8_t* __restrict__ bk, int64_t ldb,
                 u64* __restrict__ ox, u64* __restrict__ oz, uint8_t* __restrict__ ok,
                 int64_t ldo) {
  const int64_t units = VEC ? (P >> 1) : P;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < units; g += stride) {
    if (VEC) {
      const int64_t p = 2 * g;
      int k0 = 0, k1 = 0;
#pragma unroll
      for (int w = 0; w < W; ++w) {
        const ulonglong2 a_x = ld2(ax + w * lda + p), a_z = ld2(az + w * lda + p);
        const ulonglong2 b_x = ld2(bx + w * ldb + p), b_z = ld2(bz + w * ldb + p);
        k0 += phase_word(a_x.x, a_z.x, b_x.x, b_z.x);
        k1 += phase_word(a_x.y, a_z.y, b_x.y, b_z.y);
        st2(ox + w * ldo + p, a_x.x ^ b_x.x, a_x.y ^ b_x.y);
        st2(oz + w * ldo + p, a_z.x ^ b_z.x, a_z.y ^ b_z.y);
      }
      if (ak) { k0 += ak[p]; k1 += ak[p + 1]; }
      if (bk) { k0 += bk[p]; k1 += bk[p + 1]; }
      *reinterpret_cast<uchar2*>(ok + p) = make_uchar2((uint8_t)(k0 & 3), (uint8_t)(k1 & 3));
    } else {
      const int64_t p = g;
      int k = 0;
#pragma unroll
      for (int w = 0; w < W; ++w) {
        const u64 a_x = __ldg(ax + w * lda + p), a_z = __ldg(az + w * lda + p);
        const u64 b_x = __ldg(bx + w * ldb + p), b_z = __ldg(bz + w * ldb + p);
        k += phase_word(a_x, a_z, b_x, b_z);
        ox[w * ldo + p] = a_x ^ b_x;
        oz[w * ldo + p] = a_z ^ b_z;
      }
      if (ak) k += ak[p];
      if (bk) k += bk[p];
      ok[p] = (uint8_t)(k & 3);
    }
  }
  // odd tail of the vector path
  if (VEC && (P & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const int64_t p = P - 1;
    int k = 0;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const u64 a_x = ax[w * lda + p], a_z = az[w * lda + p];
      const u64 b_x = bx[w * ldb + p], b_z = bz[w * ldb + p];
      k += phase_word(a_x, a_z, b_x, b_z);
      ox[w * ldo + p] = a_x ^ b_x;
      oz[w * ldo + p] = a_z ^ b_z;
    }
    if (ak) k += ak[p];
    if (bk) k += bk[p];
    ok[p] = (uint8_t)(k & 3);
  }
}

static inline bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

template <int W>
static int launch_batch_multiply(int64_t P, const u64* ax, const u64* az, const uint8_t* ak,
                                 int64_t lda, const u64* bx, const u64* bz, const uint8_t* bk,
                                 int64_t ldb, u64* ox, u64* oz, uint8_t* ok, int64_t ldo,
                                 cudaStream_t st) {
  const bool vec = al16(ax) && al16(az) && al16(bx) && al16(bz) && al16(ox) && al16(oz) &&
                   !(lda & 1) && !(ldb & 1) && !(ldo & 1) && ((uintptr_t)ok % 2 == 0) &&
                   (!ak || (uintptr_t)ak % 2 == 0) && (!bk || (uintptr_t)bk % 2 == 0);
  const int64_t units = vec ? (P >> 1) : P;
  const int threads = 256;
  int64_t blocks = ceil_div(units > 0 ? units : 1, threads);
  const int64_t cap = (int64_t)num_sms() * 16;
  if (blocks > cap) blocks = cap;
  if (vec)
    k_batch_multiply<W, true><<<(unsigned)blocks, threads, 0, st>>>(P, ax, az, ak, lda, bx, bz, bk,
                                                                    ldb, ox, oz, ok, ldo);
  else
    k_batch_multiply<W, false><<<(unsigned)blocks, threads, 0, st>>>(P, ax, az, ak, lda, bx, bz,
                                                                     bk, ldb, ox, oz, ok, ldo);
  PLB_CHECK_LAUNCH("k_batch_multiply");
  return PL_OK;
}

// ------------------------------------------------------------ batched sip
template <int W>
__global__ void __launch_bounds__(256)
k_batch_sip(int64_t P, const u64* __restrict__ ax, const u64* __restrict__ az, int64_t lda,
            const u64* __restrict__ bx, const u64* __restrict__ bz, int64_t ldb,
            uint8_t* __restrict__ anti) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < P; p += stride) {
    u64 acc = 0;
#pragma unroll
    for (int w = 0; w < W; ++w)
      acc ^= sip_word(__ldg(ax + w * lda + p), __ldg(az + w * lda + p), __ldg(bx + w * ldb + p),
                      __ldg(bz + w * ldb + p));
    anti[p] = (uint8_t)(popc64(acc) & 1);
  }
}

template <int W>
static int launch_batch_sip(int64_t P, const u64* ax, const u64* az, int64_t lda, const u64* bx,
                            const u64* bz, int64_t ldb, uint8_t* anti, cudaStream_t st) {
  int64_t blocks = ceil_div(P > 0 ? P : 1, 256);
  const int64_t cap = (int64_t)num_sms() * 16;
  if (blocks > cap) blocks = cap;
  k_batch_sip<W><<<(unsigned)blocks, 256, 0, st>>>(P, ax, az, lda, bx, bz, ldb, anti);
  PLB_CHECK_LAUNCH("k_batch_sip");
  return PL_OK;
}

// ------------------------------------------------------- raw outer product
// Complex product rounded exactly like numpy's complex128 multiply on
// FMA-capable x86 hosts (the reference's sums.py:141):
//   re = fma(ar, br, -(ai*bi)),  im = fma(ar, bi, ai*br)
// (verified bit-for-bit against numpy 2.3.5).
__device__ __forceinline__ double2 cmul_np(double2 a, double2 b) {
  return make_double2(__fma_rn(a.x, b.x, -__dmul_rn(a.y, b.y)),
                      __fma_rn(a.x, b.y, __dmul_rn(a.y, b.x)));
}

template <int W>
__global__ void __launch_bounds__(256)
k_outer_raw(int64_t Ma, int64_t Mb, const u64* __restrict__ ax, const u64* __restrict__ az,
            const uint8_t* __restrict__ ak, const double2* __restrict__ ac, int64_t lda,
            const u64* __restrict__ bx, const u64* __restrict__ bz,
            const uint8_t* __restrict__ bk, const double2* __restrict__ bc, int64_t ldb,
            u64* __restrict__ ox, u64* __restrict__ oz, uint8_t* __restrict__ ok,
            double2* __restrict__ oc, int64_t ldo) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= Ma) return;
  u64 a_x[W], a_z[W];
#pragma unroll
  for (int w = 0; w < W; ++w) {
    a_x[w] = __ldg(ax + w * lda + i);
    a_z[w] = __ldg(az + w * lda + i);
  }
  const int ka = ak ? ak[i] : 0;
  const double2 ca = ac[i];
  for (int64_t j = blockIdx.y; j < Mb; j += gridDim.y) {
    const int64_t r = j * Ma + i;  // j-major rows, sums.py:137
    int k = ka + (bk ? bk[j] : 0);
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const u64 b_x = __ldg(bx + w * ldb + j), b_z = __ldg(bz + w * ldb + j);
      k += phase_word(a_x[w], a_z[w], b_x, b_z);
      ox[w * ldo + r] = a_x[w] ^ b_x;
      oz[w * ldo + r] = a_z[w] ^ b_z;
    }
    ok[r] = (uint8_t)(k & 3);
    oc[r] = cmul_np(ca, bc[j]);
  }
}

template <int W>
static int launch_outer_raw(int64_t Ma, int64_t Mb, const u64* ax, const u64* az,
                            const uint8_t* ak, const double* ac, int64_t lda, const u64* bx,
                            const u64* bz, const uint8_t* bk, const double* bc, int64_t ldb,
                            u64* ox, u64* oz, uint8_t* ok, double* oc, int64_t ldo,
                            cudaStream_t st) {
  dim3 grid((unsigned)ceil_div(Ma, 256), (unsigned)(Mb < 65535 ? Mb : 65535));
  k_outer_raw<W><<<grid, 256, 0, st>>>(Ma, Mb, ax, az, ak, (const double2*)ac, lda, bx, bz, bk,
                                       (const double2*)bc, ldb, ox, oz, ok, (double2*)oc, ldo);
  PLB_CHECK_LAUNCH("k_outer_raw");
  return PL_OK;
}

}  // namespace plb

using namespace plb;

extern "C" int pl_batch_multiply(int W, int64_t P, const uint64_t* ax, const uint64_t* az,
                                 const uint8_t* ak, int64_t lda, const uint64_t* bx,
                                 const uint64_t* bz, const uint8_t* bk, int64_t ldb, uint64_t* ox,
                                 uint64_t* oz, uint8_t* ok, int64_t ldo, void* stream) {
  if (P < 0 || lda < P || ldb < P || ldo < P) {
    set_error("pl_batch_multiply: bad sizes P=%lld lda=%lld ldb=%lld ldo=%lld", (long long)P,
              (long long)lda, (long long)ldb, (long long)ldo);
    return PL_ERR_ARG;
  }
  if (P == 0) return PL_OK;
  if (!ax || !az || !bx || !bz || !ox || !oz || !ok) {
    set_error("pl_batch_multiply: null pointer");
    return PL_ERR_ARG;
  }
  return PLB_DISPATCH_W(W, launch_batch_multiply, P, (const u64*)ax, (const u64*)az, ak, lda,
                        (const u64*)bx, (const u64*)bz, bk, ldb, (u64*)ox, (u64*)oz, ok, ldo,
                        (cudaStream_t)stream);
}

extern "C" int pl_batch_sip(int W, int64_t P, const uint64_t* ax, const uint64_t* az,
                            int64_t lda, const uint64_t* bx, const uint64_t* bz, int64_t ldb,
                            uint8_t* anti, void* stream) {
  if (P < 0 || lda < P || ldb < P) {
    set_error("pl_batch_sip: bad sizes");
    return PL_ERR_ARG;
  }
  if (P == 0) return PL_OK;
  return PLB_DISPATCH_W(W, launch_batch_sip, P, (const u64*)ax, (const u64*)az, lda,
                        (const u64*)bx, (const u64*)bz, ldb, anti, (cudaStream_t)stream);
}

extern "C" int pl_outer_multiply_raw(int W, int64_t Ma, int64_t Mb, const uint64_t* ax,
                                     const uint64_t* az, const uint8_t* ak, const double* ac,
                                     int64_t lda, const uint64_t* bx, const uint64_t* bz,
                                     const uint8_t* bk, const double* bc, int64_t ldb,
                                     uint64_t* ox, uint64_t* oz, uint8_t* ok, double* oc,
                                     int64_t ldo, void* stream) {
  if (Ma < 0 || Mb < 0 || lda < Ma || ldb < Mb || ldo < Ma * Mb) {
    set_error("pl_outer_multiply_raw: bad sizes");
    return PL_ERR_ARG;
  }
  if (Ma == 0 || Mb == 0) return PL_OK;
  return PLB_DISPATCH_W(W, launch_outer_raw, Ma, Mb, (const u64*)ax, (const u64*)az, ak, ac, lda,
                        (const u64*)bx, (const u64*)bz, bk, bc, ldb, (u64*)ox, (u64*)oz, ok, oc,
                        ldo, (cudaStream_t)stream);
}

// ------------------------------------------------------------------------
// One pair from HOST memory: product and symplectic parity in one launch.
// The scalar API (PauliString.multiply / commutes, strings.py:133-147) used to
// move six one-element tensors to the device per call (~100 us); here the
// operands sit in a mapped pinned buffer the kernel reads and writes directly
// (zero-copy), so a call costs one launch and one stream synchronisation.
namespace plb {

constexpr int kPairMaxW = 16;
// mapped buffer layout (u64 words): in ax | az | bx | bz | ka, kb ; out x | z | k, sip
constexpr int kPairIn = 4 * kPairMaxW + 2, kPairOut = 2 * kPairMaxW + 2;

__global__ void __launch_bounds__(32) k_pair_host(int W, const u64* __restrict__ in,
                                                  u64* __restrict__ out) {
  const int lane = threadIdx.x;
  const bool on = lane < W;
  const u64 ax = on ? in[lane] : 0ull, az = on ? in[kPairMaxW + lane] : 0ull;
  const u64 bx = on ? in[2 * kPairMaxW + lane] : 0ull, bz = on ? in[3 * kPairMaxW + lane] : 0ull;
  int ph = phase_word(ax, az, bx, bz);
  int sp = popc64(sip_word(ax, az, bx, bz));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ph += __shfl_xor_sync(0xffffffffu, ph, o);
    sp += __shfl_xor_sync(0xffffffffu, sp, o);
  }
  if (on) {
    out[lane] = ax ^ bx;
    out[kPairMaxW + lane] = az ^ bz;
  }
  if (lane == 0) {
    out[2 * kPairMaxW] = (u64)(((int)in[4 * kPairMaxW] + (int)in[4 * kPairMaxW + 1] + ph) & 3);
    out[2 * kPairMaxW + 1] = (u64)(sp & 1);
  }
}

}  // namespace plb

extern "C" int pl_pair_host(int W, const uint64_t* ax, const uint64_t* az, int ak,
                            const uint64_t* bx, const uint64_t* bz, int bk, uint64_t* ox,
                            uint64_t* oz, int* ok, int* anti, void* stream) {
  using namespace plb;
  if (!valid_words(W)) {
    set_error("unsupported word count W=%d", W);
    return PL_ERR_TIER;
  }
  if (!ax || !az || !bx || !bz) {
    set_error("pl_pair_host: operand pointers must not be NULL");
    return PL_ERR_ARG;
  }
  static std::mutex mtx;
  static u64* hbuf[64] = {nullptr};
  static u64* dbuf[64] = {nullptr};
  int dev = 0;
  PLB_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) {
    set_error("device index %d out of range", dev);
    return PL_ERR_ARG;
  }
  std::lock_guard<std::mutex> lock(mtx);
  if (!hbuf[dev]) {
    PLB_CUDA(cudaHostAlloc((void**)&hbuf[dev], (kPairIn + kPairOut) * sizeof(u64), cudaHostAllocMapped));
    PLB_CUDA(cudaHostGetDevicePointer((void**)&dbuf[dev], hbuf[dev], 0));
  }
  u64* h = hbuf[dev];
  memcpy(h, ax, 8 * W);
  memcpy(h + kPairMaxW, az, 8 * W);
  memcpy(h + 2 * kPairMaxW, bx, 8 * W);
  memcpy(h + 3 * kPairMaxW, bz, 8 * W);
  h[4 * kPairMaxW] = (u64)(ak & 3);
  h[4 * kPairMaxW + 1] = (u64)(bk & 3);
  cudaStream_t st = (cudaStream_t)stream;
  k_pair_host<<<1, 32, 0, st>>>(W, dbuf[dev], dbuf[dev] + kPairIn);
  PLB_CHECK_LAUNCH("k_pair_host");
  PLB_CUDA(cudaStreamSynchronize(st));
  const u64* o = h + kPairIn;
  if (ox) memcpy(ox, o, 8 * W);
  if (oz) memcpy(oz, o + kPairMaxW, 8 * W);
  if (ok) *ok = (int)o[2 * kPairMaxW];
  if (anti) *anti = (int)o[2 * kPairMaxW + 1];
  return PL_OK;
}
