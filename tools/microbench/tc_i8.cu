// tcgen05.mma kind::i8 on B200 (sm_100a): a functional check of the
// descriptors (D = A * B^T for 0/1 int8 operands, exact) and a throughput
// microbenchmark (one CTA per SM issuing back-to-back 128x256x32 MMAs).
// This is the tensor-core formulation of the commutation bitmatrix
// (grouping.py:136-140): parity(popc(x_r & z_c) + popc(z_r & x_c)) =
// (A_r . B_c) & 1 with A_r = [x_r | z_r], B_c = [z_c | x_c] as 0/1 bytes,
// K = 2 * 64W.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tc_i8 tc_i8.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e = (x);                                                       \
    if (e != cudaSuccess) {                                                    \
      printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__);              \
      exit(1);                                                                 \
    }                                                                          \
  } while (0)

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// K-major, no swizzle: core matrix = 8 rows x 16 bytes (128 B contiguous);
// lbo / sbo = byte distances between K-adjacent core matrices and between
// 8-row groups (which field is which is checked at run time below).
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
  return d;               // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
}

__host__ __device__ constexpr uint32_t idesc_i8(int M, int N) {
  return (2u << 4)            // D format S32
         | (0u << 7)          // A unsigned 8-bit
         | (0u << 10)         // B unsigned 8-bit
         | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);  // K-major A and B
}

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t ad, uint64_t bd, uint32_t idesc,
                                       uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   sa(bar))
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}\n" ::"r"(sa(bar)),
      "r"(phase)
      : "memory");
}

template <int M, int N, int KB>
__global__ void __launch_bounds__(128) k_tc(const uint8_t* A, const uint8_t* B, int32_t* D,
                                            int reps, int lbo_is_k) {
  constexpr int KT = 32 * KB;  // bytes per row
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;           // M x KT
  uint8_t* sB = smem + M * KT;  // N x KT
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // core-matrix layout: element (r, k) at (r/8)*SBO + (k/16)*128 + (r%8)*16 + k%16
  constexpr uint32_t SBO = (KT / 16) * 128;
  for (int e = tid; e < M * KT; e += blockDim.x) {
    const int r = e / KT, k = e % KT;
    sA[(r / 8) * SBO + (k / 16) * 128 + (r % 8) * 16 + k % 16] = A[e];
  }
  for (int e = tid; e < N * KT; e += blockDim.x) {
    const int r = e / KT, k = e % KT;
    sB[(r / 8) * SBO + (k / 16) * 128 + (r % 8) * 16 + k % 16] = B[e];
  }
  if (tid == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     sa(&tbase)),
                 "r"(N));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tbase;
  const uint32_t lbo = lbo_is_k ? 128u : SBO, sbo = lbo_is_k ? SBO : 128u;
  if (tid == 0) {
    constexpr uint32_t idesc = idesc_i8(M, N);
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int kb = 0; kb < KB; ++kb) {
        const uint64_t ad = smem_desc(sa(sA) + kb * 256, lbo, sbo);
        const uint64_t bd = smem_desc(sa(sB) + kb * 256, lbo, sbo);
        mma_i8(tmem, ad, bd, idesc, (r | kb) ? 1u : 0u);
      }
    }
    commit(&bar);
  }
  __syncwarp();
  mbar_wait(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // D row (32*warp + lane), columns c..c+7
  for (int c = 0; c < N; c += 8) {
    uint32_t v[8];
    const uint32_t taddr = tmem + ((uint32_t)(32 * warp) << 16) + c;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                   "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (D) {
      int32_t* out = D + ((int64_t)blockIdx.x * M + 32 * warp + lane) * N + c;
#pragma unroll
      for (int i = 0; i < 8; ++i) out[i] = (int32_t)v[i];
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(N));
}

int main() {
  constexpr int M = 128, N = 256, KB = 4, KT = 32 * KB;
  std::vector<uint8_t> hA(M * KT), hB(N * KT);
  srand(7);
  for (auto& v : hA) v = rand() & 1;
  for (auto& v : hB) v = rand() & 1;
  uint8_t *dA, *dB;
  int32_t* dD;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  CK(cudaMalloc(&dA, M * KT));
  CK(cudaMalloc(&dB, N * KT));
  CK(cudaMalloc(&dD, (size_t)sms * M * N * 4));
  CK(cudaMemcpy(dA, hA.data(), M * KT, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, hB.data(), N * KT, cudaMemcpyHostToDevice));
  const size_t sm = (size_t)(M + N) * KT;
  auto kern = k_tc<M, N, KB>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  for (int lbo_is_k = 1; lbo_is_k >= 0; --lbo_is_k) {
    kern<<<1, 128, sm>>>(dA, dB, dD, 1, lbo_is_k);
    CK(cudaDeviceSynchronize());
    std::vector<int32_t> hD(M * N);
    CK(cudaMemcpy(hD.data(), dD, M * N * 4, cudaMemcpyDeviceToHost));
    int bad = 0;
    for (int i = 0; i < M; ++i)
      for (int j = 0; j < N; ++j) {
        int s = 0;
        for (int k = 0; k < KT; ++k) s += hA[i * KT + k] * hB[j * KT + k];
        bad += hD[i * N + j] != s;
      }
    printf("{\"check\": \"D = A*B^T (u8 0/1, M=%d N=%d K=%d)\", \"lbo_is_k\": %d, \"mismatches\": %d}\n",
           M, N, KT, lbo_is_k, bad);
    if (bad == 0) {
      const int reps = 20000;
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      kern<<<sms, 128, sm>>>(dA, dB, nullptr, 100, lbo_is_k);
      CK(cudaDeviceSynchronize());
      cudaEventRecord(a);
      kern<<<sms, 128, sm>>>(dA, dB, nullptr, reps, lbo_is_k);
      cudaEventRecord(b);
      CK(cudaEventSynchronize(b));
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double ops = 2.0 * M * N * 32 * (double)KB * reps * sms;
      printf("{\"kernel\": \"tcgen05.mma.kind::i8 128x256x32, 1 CTA/SM\", \"ms\": %.3f, "
             "\"ops_per_s\": %.4e}\n",
             ms, ops / (ms * 1e-3));
      break;
    }
  }
  return 0;
}
