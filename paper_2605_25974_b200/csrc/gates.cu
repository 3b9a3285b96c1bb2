// §8(f) rows f1/f2: Clifford conjugation in place and the Pauli-rotation split
// on SoA planes.
//
// f2  pl_apply_clifford  restates gates.py:31-102 (apply_clifford_inplace):
//     U P U^dagger for H, S, CNOT, CZ over every term; only the plane words
//     holding the touched qubits are read and written (the SoA layout makes
//     each a coalesced stream of M words), and the phase byte takes the
//     tableau sign flip (flags ^= 2).
// f1  pl_rotation_split  restates _rotation_columns (sums.py:177-223): terms
//     commuting with the generator pass through, an anti-commuting term Q of
//     coefficient c becomes (c*cos, Q) followed by
//     (c*(-i sin)*i^k, letters of P*Q) with k = flags + phase(P, Q)
//     (strings.py:32-44); with sin == 0 only the coefficients scale, with
//     cos == 0 the anti-commuting terms are replaced in place.  Output order
//     is the reference's interleaving: term i at i + #anti(< i), its partner
//     right after it.  Coefficient arithmetic reproduces numpy's complex128
//     products bit for bit (cmul_np).
#include "common.cuh"
#include "scan.cuh"

namespace plb {

// numpy complex128 multiply on FMA hosts
__device__ __forceinline__ double2 cmul_fma(double2 a, double2 b) {
  return make_double2(__fma_rn(a.x, b.x, -__dmul_rn(a.y, b.y)),
                      __fma_rn(a.x, b.y, __dmul_rn(a.y, b.x)));
}

// gate codes of the C ABI
enum { kGateH = 0, kGateS = 1, kGateCNOT = 2, kGateCZ = 3 };

template <int GATE>
__global__ void k_clifford(u64* __restrict__ x, u64* __restrict__ z, uint8_t* __restrict__ k,
                           int64_t ld, int64_t M, int wc, int pc, int wt, int pt) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < M;
       t += (int64_t)gridDim.x * blockDim.x) {
    if (GATE == kGateH) {  // gates.py:31-38
      const u64 mask = 1ull << pc;
      const u64 xw = x[wc * ld + t], zw = z[wc * ld + t];
      const u64 xb = xw & mask, zb = zw & mask;
      if ((xb & zb) != 0) k[t] ^= 2;
      x[wc * ld + t] = (xw & ~mask) | zb;
      z[wc * ld + t] = (zw & ~mask) | xb;
    } else if (GATE == kGateS) {  // gates.py:41-45
      const u64 mask = 1ull << pc;
      const u64 xb = x[wc * ld + t] & mask;
      const u64 zw = z[wc * ld + t];
      if ((xb & zw) != 0) k[t] ^= 2;
      z[wc * ld + t] = zw ^ xb;
    } else {
      const u64 xcw = x[wc * ld + t], zcw = z[wc * ld + t];
      const u64 xtw = wt == wc ? xcw : x[wt * ld + t];
      const u64 ztw = wt == wc ? zcw : z[wt * ld + t];
      const u64 xc = (xcw >> pc) & 1, zc = (zcw >> pc) & 1;
      const u64 xt = (xtw >> pt) & 1, zt = (ztw >> pt) & 1;
      if (GATE == kGateCNOT) {  // gates.py:48-57
        if (xc & zt & (xt ^ zc ^ 1)) k[t] ^= 2;
        x[wt * ld + t] = xtw ^ (xc << pt);  // (x and z are separate planes: same-word safe)
        z[wc * ld + t] = zcw ^ (zt << pc);
      } else {  // CZ, gates.py:60-69
        if (xc & xt & (zc ^ zt)) k[t] ^= 2;
        if (wt == wc) {
          z[wc * ld + t] = zcw ^ (xt << pc) ^ (xc << pt);
        } else {
          z[wc * ld + t] = zcw ^ (xt << pc);
          z[wt * ld + t] = ztw ^ (xc << pt);
        }
      }
    }
  }
}

static unsigned grid_for(int64_t m, int threads) {
  int64_t b = ceil_div(m, threads);
  const int64_t cap = 8LL * num_sms();
  return (unsigned)(b < 1 ? 1 : b > cap ? cap : b);
}

// ------------------------------------------------------------- rotation
struct RotGen {
  u64 x[16], z[16];
  int base;  // popc(gx & gz) over all words
};

template <int W>
__device__ __forceinline__ bool rot_anti(const RotGen& G, const u64* x, const u64* z, int64_t ld,
                                         int64_t t) {
  u64 acc = 0;
#pragma unroll
  for (int w = 0; w < W; ++w) acc ^= (G.x[w] & z[w * ld + t]) ^ (G.z[w] & x[w * ld + t]);
  return popc64(acc) & 1;
}

template <int W>
__global__ void k_rot_anti(RotGen G, const u64* __restrict__ x, const u64* __restrict__ z,
                           int64_t ld, int64_t M, uint32_t* __restrict__ anti) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < M;
       t += (int64_t)gridDim.x * blockDim.x)
    anti[t] = rot_anti<W>(G, x, z, ld, t) ? 1u : 0u;
}

// MODE 0: sin == 0 (scale), 1: cos == 0 (replace), 2: split (interleave)
template <int W, int MODE>
__global__ void k_rot_write(RotGen G, const u64* __restrict__ x, const u64* __restrict__ z,
                            const uint8_t* __restrict__ k, const double2* __restrict__ c,
                            int64_t ld, int64_t M, const uint32_t* __restrict__ anti,
                            const uint32_t* __restrict__ before, double cos_t, double2 msin,
                            u64* __restrict__ ox, u64* __restrict__ oz, uint8_t* __restrict__ ok,
                            double2* __restrict__ oc, int64_t ldo) {
  const double2 pf[4] = {make_double2(1.0, 0.0), make_double2(0.0, 1.0),
                         make_double2(-1.0, 0.0), make_double2(-0.0, -1.0)};
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < M;
       t += (int64_t)gridDim.x * blockDim.x) {
    const bool a = anti[t] != 0;
    const double2 ct = c[t];
    const int64_t o = MODE == 2 ? t + before[t] : t;
    // product P*Q: letters, phase (sums.py:194-196 with P as the left operand)
    int pk = 0;
    if (a && MODE != 0) {
      pk = G.base + k[t];
#pragma unroll
      for (int w = 0; w < W; ++w) {
        const u64 bx = x[w * ld + t], bz = z[w * ld + t];
        pk += popc64(bx & bz) + 2 * popc64(G.z[w] & bx) - popc64((G.x[w] ^ bx) & (G.z[w] ^ bz));
      }
      pk &= 3;
    }
    const double2 prod = cmul_fma(cmul_fma(ct, msin), pf[pk]);
    if (MODE == 1 && a) {
#pragma unroll
      for (int w = 0; w < W; ++w) {
        ox[w * ldo + o] = x[w * ld + t] ^ G.x[w];
        oz[w * ldo + o] = z[w * ld + t] ^ G.z[w];
      }
      ok[o] = 0;
      oc[o] = prod;
      continue;
    }
#pragma unroll
    for (int w = 0; w < W; ++w) {
      ox[w * ldo + o] = x[w * ld + t];
      oz[w * ldo + o] = z[w * ld + t];
    }
    ok[o] = k[t];
    oc[o] = (a && MODE != 1) ? cmul_fma(ct, make_double2(cos_t, 0.0)) : ct;
    if (MODE == 2 && a) {
#pragma unroll
      for (int w = 0; w < W; ++w) {
        ox[w * ldo + o + 1] = x[w * ld + t] ^ G.x[w];
        oz[w * ldo + o + 1] = z[w * ld + t] ^ G.z[w];
      }
      ok[o + 1] = 0;
      oc[o + 1] = prod;
    }
  }
}

static __global__ void k_rot_count(int64_t M, const uint32_t* total, int64_t* out) {
  *out = M + (total ? (int64_t)*total : 0);
}

template <int W>
static int run_rotation(const RotGen& G, const u64* x, const u64* z, const uint8_t* k,
                        const double2* c, int64_t ld, int64_t M, double cos_t, double2 msin,
                        void* ws, u64* ox, u64* oz, uint8_t* ok, double2* oc, int64_t ldo,
                        int64_t* out_count, cudaStream_t st) {
  uint32_t* anti = (uint32_t*)ws;
  uint32_t* before = anti + M;
  uint32_t* scratch = before + M;
  uint32_t* total = scratch + scan_scratch_words(M);
  const unsigned g = grid_for(M, 256);
  StageTimer t_(st, "k_rotation");
  k_rot_anti<W><<<g, 256, 0, st>>>(G, x, z, ld, M, anti);
  PLB_CHECK_LAUNCH("k_rot_anti");
  const int mode = msin.x == 0.0 && msin.y == 0.0 ? 0 : cos_t == 0.0 ? 1 : 2;
  if (mode == 2) {
    int rc = exclusive_scan_u32(anti, before, M, scratch, total, st);
    if (rc) return rc;
  }
  switch (mode) {
    case 0: k_rot_write<W, 0><<<g, 256, 0, st>>>(G, x, z, k, c, ld, M, anti, before, cos_t, msin,
                                                 ox, oz, ok, oc, ldo); break;
    case 1: k_rot_write<W, 1><<<g, 256, 0, st>>>(G, x, z, k, c, ld, M, anti, before, cos_t, msin,
                                                 ox, oz, ok, oc, ldo); break;
    default: k_rot_write<W, 2><<<g, 256, 0, st>>>(G, x, z, k, c, ld, M, anti, before, cos_t,
                                                  msin, ox, oz, ok, oc, ldo); break;
  }
  PLB_CHECK_LAUNCH("k_rot_write");
  // out_count = M (+ anti-commuting terms when split), on the device
  k_rot_count<<<1, 1, 0, st>>>(M, mode == 2 ? total : nullptr, out_count);
  PLB_CHECK_LAUNCH("k_rot_count");
  return PL_OK;
}

}  // namespace plb

using namespace plb;

extern "C" int pl_apply_clifford(int W, int64_t M, uint64_t* x, uint64_t* z, uint8_t* k, int64_t ld,
                                 int gate, int q0, int q1, void* stream) {
  const int nq = 64 * W;
  const bool two = gate == kGateCNOT || gate == kGateCZ;
  if (!valid_words(W) || M < 0 || ld < M || gate < 0 || gate > 3 || q0 < 0 || q0 >= nq ||
      (two && (q1 < 0 || q1 >= nq || q1 == q0))) {
    set_error("pl_apply_clifford: bad arguments (W=%d gate=%d q=(%d,%d))", W, gate, q0, q1);
    return valid_words(W) ? PL_ERR_ARG : PL_ERR_TIER;
  }
  if (M == 0) return PL_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const unsigned g = grid_for(M, 256);
  const int wc = q0 >> 6, pc = q0 & 63, wt = two ? q1 >> 6 : 0, pt = two ? q1 & 63 : 0;
  u64 *X = (u64*)x, *Z = (u64*)z;
  StageTimer t_(st, "k_clifford");
  switch (gate) {
    case kGateH: k_clifford<kGateH><<<g, 256, 0, st>>>(X, Z, k, ld, M, wc, pc, wt, pt); break;
    case kGateS: k_clifford<kGateS><<<g, 256, 0, st>>>(X, Z, k, ld, M, wc, pc, wt, pt); break;
    case kGateCNOT: k_clifford<kGateCNOT><<<g, 256, 0, st>>>(X, Z, k, ld, M, wc, pc, wt, pt); break;
    default: k_clifford<kGateCZ><<<g, 256, 0, st>>>(X, Z, k, ld, M, wc, pc, wt, pt); break;
  }
  PLB_CHECK_LAUNCH("k_clifford");
  return PL_OK;
}

extern "C" int64_t pl_rotation_workspace_bytes(int64_t M) {
  return 4 * (2 * (M > 0 ? M : 1) + scan_scratch_words(M) + 2);
}

extern "C" int pl_rotation_split(int W, int64_t M, const uint64_t* x, const uint64_t* z,
                                 const uint8_t* k, const double* c, int64_t ld,
                                 const uint64_t* gen_x, const uint64_t* gen_z, double cos_t,
                                 double msin_re, double msin_im, void* workspace,
                                 size_t workspace_bytes, uint64_t* ox, uint64_t* oz, uint8_t* ok,
                                 double* oc, int64_t ldo, int64_t* out_count, void* stream) {
  if (!valid_words(W) || M < 0 || ld < M || !gen_x || !gen_z || !out_count) {
    set_error("pl_rotation_split: bad arguments");
    return valid_words(W) ? PL_ERR_ARG : PL_ERR_TIER;
  }
  const bool split = !(msin_re == 0.0 && msin_im == 0.0) && cos_t != 0.0;
  if (ldo < (split ? 2 * M : M)) {
    set_error("pl_rotation_split: output leading dimension %lld < %lld", (long long)ldo,
              (long long)(split ? 2 * M : M));
    return PL_ERR_ARG;
  }
  if ((int64_t)workspace_bytes < pl_rotation_workspace_bytes(M) || !workspace) {
    set_error("pl_rotation_split: workspace too small");
    return PL_ERR_WORKSPACE;
  }
  cudaStream_t st = (cudaStream_t)stream;
  if (M == 0) {
    PLB_CUDA(cudaMemsetAsync(out_count, 0, sizeof(int64_t), st));
    return PL_OK;
  }
  RotGen G{};
  G.base = 0;
  for (int w = 0; w < W; ++w) {  // generator words are host arrays (a single string)
    G.x[w] = gen_x[w];
    G.z[w] = gen_z[w];
    G.base += __builtin_popcountll(gen_x[w] & gen_z[w]);
  }
  const double2 ms = make_double2(msin_re, msin_im);
#define PLB_ROT(WW)                                                                              \
  run_rotation<WW>(G, (const u64*)x, (const u64*)z, k, (const double2*)c, ld, M, cos_t, ms,     \
                   workspace, (u64*)ox, (u64*)oz, ok, (double2*)oc, ldo, out_count, st)
  switch (W) {
    case 1: return PLB_ROT(1);
    case 2: return PLB_ROT(2);
    case 4: return PLB_ROT(4);
    case 8: return PLB_ROT(8);
    default: return PLB_ROT(16);
  }
#undef PLB_ROT
}
