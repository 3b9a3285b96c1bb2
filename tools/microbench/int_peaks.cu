// Integer-pipe peaks on B200 for the commutation bitmatrix pipe choice (K5,
// grouping.py:136-140 restated; strings.py:47-51):
//   * LOP3 (32-bit, 3-input logic), POPC, and IADD3 throughput per SM;
//   * legacy mma.sync m16n8k256 b1 AND.POPC (the binary-MMA formulation of
//     popc(x_r & z_c) + popc(z_r & x_c)) throughput.
// Each kernel runs long chains of independent operations per thread; the
// reported rate is operations / second over the whole GPU (CUDA events).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o int_peaks int_peaks.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kIters = 4096;
constexpr int kChains = 8;

__global__ void k_lop3(uint32_t* out, uint32_t seed) {
  uint32_t a[kChains], b = seed * 0x9E3779B9u + threadIdx.x, c = seed ^ 0x85EBCA6Bu;
#pragma unroll
  for (int i = 0; i < kChains; ++i) a[i] = threadIdx.x * (i + 1);
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < kChains; ++i) {
      // (a & b) ^ c : one LOP3 each
      asm volatile("lop3.b32 %0, %0, %1, %2, 0x78;" : "+r"(a[i]) : "r"(b), "r"(c));
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < kChains; ++i) s ^= a[i];
  if (s == 0x12345678u) out[0] = s;
}

__global__ void k_popc(uint32_t* out, uint32_t seed) {
  uint32_t a[kChains];
#pragma unroll
  for (int i = 0; i < kChains; ++i) a[i] = threadIdx.x * (i + 7) + seed;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < kChains; ++i) {
      uint32_t p;
      asm volatile("popc.b32 %0, %1;" : "=r"(p) : "r"(a[i]));
      a[i] += p;  // keeps the chain dependent (adds one IADD per POPC)
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < kChains; ++i) s ^= a[i];
  if (s == 0x12345678u) out[0] = s;
}

// popc only (no dependent add): independent POPCs from rotating inputs
__global__ void k_popc_only(uint32_t* out, uint32_t seed) {
  uint32_t a[kChains], acc[kChains];
#pragma unroll
  for (int i = 0; i < kChains; ++i) {
    a[i] = threadIdx.x * (i + 7) + seed;
    acc[i] = 0;
  }
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < kChains; ++i) {
      uint32_t p;
      asm volatile("popc.b32 %0, %1;" : "=r"(p) : "r"(a[i] ^ it));
      acc[i] ^= p;
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < kChains; ++i) s ^= acc[i];
  if (s == 0x12345678u) out[0] = s;
}

// binary MMA: D(16x8, s32) += popc(A(16x256 b1) & B(256x8 b1))
__global__ void k_bmma(uint32_t* out, uint32_t seed) {
  uint32_t a[4], b[2];
  int32_t d[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i) a[i] = seed * (threadIdx.x + i);
  b[0] = seed ^ threadIdx.x;
  b[1] = seed + threadIdx.x;
#pragma unroll
  for (int c = 0; c < 4; ++c)
#pragma unroll
    for (int i = 0; i < 4; ++i) d[c][i] = 0;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {  // 4 independent accumulators
      asm volatile(
          "mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.and.popc "
          "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
          : "+r"(d[c][0]), "+r"(d[c][1]), "+r"(d[c][2]), "+r"(d[c][3])
          : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
    }
  }
  int32_t s = 0;
#pragma unroll
  for (int c = 0; c < 4; ++c)
#pragma unroll
    for (int i = 0; i < 4; ++i) s ^= d[c][i];
  if (s == 0x12345678) out[0] = s;
}

template <typename K>
static double run(K kern, int blocks, int threads, const char* name, double ops_per_thread) {
  uint32_t* out;
  cudaMalloc(&out, 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  kern<<<blocks, threads>>>(out, 1);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    kern<<<blocks, threads>>>(out, r + 2);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  const double ops = ops_per_thread * (double)blocks * threads;
  const double rate = ops / (best * 1e-3);
  printf("{\"kernel\": \"%s\", \"ms\": %.4f, \"ops\": %.4e, \"ops_per_s\": %.4e}\n", name, best, ops,
         rate);
  cudaFree(out);
  return rate;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaSetDevice(dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("{\"sms\": %d, \"clock_khz\": %d}\n", sms, clk);
  const int blocks = sms * 8, threads = 256;
  const double lop3 = run(k_lop3, blocks, threads, "lop3.b32", (double)kIters * kChains);
  const double popc = run(k_popc, blocks, threads, "popc.b32 (+iadd chain)", (double)kIters * kChains);
  const double popc2 = run(k_popc_only, blocks, threads, "popc.b32 (independent)", (double)kIters * kChains);
  // per warp: 4 MMAs per iteration, each 16*8 outputs * 256 bit-ANDs; count per thread /32
  const double bmma_bitops = run(k_bmma, blocks, threads, "mma.m16n8k256.b1.and.popc (bit-and ops)",
                                 (double)kIters * 4 * 16 * 8 * 256 / 32.0);
  printf("{\"per_sm_per_clk\": {\"lop3\": %.1f, \"popc\": %.1f, \"bmma_bitops\": %.1f}}\n",
         lop3 / sms / (clk * 1e3), popc2 / sms / (clk * 1e3), bmma_bitops / sms / (clk * 1e3));
  return 0;
}
