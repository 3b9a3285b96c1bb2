// K5 — all-pairs commutation bitmatrix (restates grouping.py:136-140, the
// parity popc(x_r & z_c) + popc(z_r & x_c) of strings.py:47-51).
//
// Method 1 (row-list XOR over transposed letter slices, the default for
// sparse rows).  A CTA owns a block of 1024 columns and transposes it in
// shared memory into three bit slices per qubit q: the columns' z bits at q,
// their x bits at q, and the XOR of both.  A row letter X at q pairs with the
// z slice, Z with the x slice and Y with the z^x slice, so
//   sip(r, c) = XOR over the letters of r of the matching slice bit of c,
// one 64-bit shared load + XOR per letter per 64 columns (a half-warp per
// row, 16 lanes x 64 columns).  The rows' letter lists (CSR, built once per
// call) are staged per warp 16 rows at a time and prefetched one block
// ahead.  Cost per 1024 checks is proportional to the row weight (config 5:
// weight 2-12), far below the 4W LOP3 + POPC per check of method 2 and the
// 256 W int8 tensor ops per check of method 3.
//
// Method 2 (direct).  One thread per row, the row's 2W words in registers,
// columns broadcast from shared memory: 4W LOP3 + POPC per check.  Used for
// dense rows and W = 16 (whose slices exceed shared memory).
//
// Method 3 (tensor, bitmatrix_tc.cuh): the int8 GEMM formulation on
// tcgen05.mma.kind::i8 for dense rows, W <= 8: 1.4-1.5x method 2 on uniform
// random strings (W=8: 6.4e11 vs 4.5e11 checks/s; the LOP3 roofline of method
// 2 is 5.4e11), chosen by "auto" above ~24 W letters per row.  The legacy
// binary MMA (mma.sync m16n8k256 b1 AND.POPC) compiles to an int8 emulation
// on sm_100a (MOVM.U4TO8 + IMMA) and is not used.
#include "common.cuh"
#include "scan.cuh"
#include "bitmatrix_kernels.cuh"
#include "bitmatrix_tc.cuh"

namespace plb {

// ------------------------------------------------------------- launchers
static inline int64_t list_capacity_entries(int64_t rows) { return rows * 64; }

template <int W>
static int launch_bitmatrix(int64_t M, const u64* x, const u64* z, int64_t ld, int64_t row0,
                            int64_t rows, int64_t col0, int64_t cols, uint32_t* bits,
                            int64_t ld_bits, int method, void* ws, size_t ws_bytes,
                            cudaStream_t st) {
  if (W == 16 && (method == 1 || method == 3)) {
    set_error("bitmatrix methods 1 and 3 support W <= 8");
    return PL_ERR_ARG;
  }
  if constexpr (W <= 8) if (method == 3) {
    const size_t smem = TcSmem<W>::BYTES;
    auto kern = k_bitmatrix_tc<W>;
    PLB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int64_t colblocks = ceil_div(cols, kTcCols);
    const int64_t rowblocks = ceil_div(rows, kTcRows);
    for (int64_t rb = 0; rb < rowblocks; rb += 65535) {
      const int64_t nrb = rowblocks - rb < 65535 ? rowblocks - rb : 65535;
      StageTimer t_(st, "k_bitmatrix_tc");
      kern<<<dim3((unsigned)colblocks, (unsigned)nrb), kTcThreads, smem, st>>>(
          x, z, ld, M, row0 + rb * kTcRows, rows - rb * kTcRows, col0, cols,
          bits + rb * kTcRows * ld_bits, ld_bits);
      PLB_CHECK_LAUNCH("k_bitmatrix_tc");
    }
    return PL_OK;
  }
  if (method != 2 && W <= 8) {
    // CSR row lists: off (rows+1) u32 | scan scratch | list u16
    const int64_t need_min = (rows + 1) * 4 + scan_scratch_words(rows) * 4 + 16;
    if (ws == nullptr || (int64_t)ws_bytes < need_min) {
      if (method == 1) {
        set_error("bitmatrix: workspace too small (%lld < %lld)", (long long)ws_bytes,
                  (long long)need_min);
        return PL_ERR_WORKSPACE;
      }
      method = 2;
    }
  }
  if constexpr (W <= 8) if (method != 2) {
    uint8_t* p = (uint8_t*)ws;
    uint32_t* off = (uint32_t*)p;
    p += (rows + 1) * 4;
    uint32_t* scratch = (uint32_t*)p;
    p += scan_scratch_words(rows) * 4;
    p = (uint8_t*)(((uintptr_t)p + 15) & ~(uintptr_t)15);
    uint32_t* list = (uint32_t*)p;
    const int64_t cap = ((int64_t)ws_bytes - (p - (uint8_t*)ws)) / 4;
    const unsigned nb = (unsigned)ceil_div(rows, 256);
    k_row_weight<W, 2><<<nb, 256, 0, st>>>(x, z, ld, row0, rows, off);
    PLB_CHECK_LAUNCH("k_row_weight");
    int rc = exclusive_scan_u32(off, off, rows, scratch, off + rows, st);
    if (rc) return rc;
    uint32_t total = 0;
    PLB_CUDA(cudaMemcpyAsync(&total, off + rows, 4, cudaMemcpyDeviceToHost, st));
    PLB_CUDA(cudaStreamSynchronize(st));
    const double avg = rows ? (double)total / (double)rows : 0.0;
    // method 1 costs ~1 shared load per letter per 64 checks; method 3 (tensor)
    // 256 W int8 ops per check whatever the density.  Measured crossover on
    // B200 (profiles/r2/bitmatrix_pipes.json): ~24 W letters per row
    const bool dense = avg > 24.0 * W;
    if ((int64_t)total > cap || (method == 0 && dense)) {
      if (method == 1) {
        set_error("bitmatrix: list workspace too small (%u entries > %lld)", total,
                  (long long)cap);
        return PL_ERR_WORKSPACE;
      }
      return launch_bitmatrix<W>(M, x, z, ld, row0, rows, col0, cols, bits, ld_bits, 3, ws,
                                 ws_bytes, st);
    } else {
      k_row_fill<W, 2><<<nb, 256, 0, st>>>(x, z, ld, row0, rows, off, list);
      PLB_CHECK_LAUNCH("k_row_fill");
      const int64_t colblocks = ceil_div(cols, kColsY);
      int64_t splits = ceil_div(2 * num_sms(), colblocks);
      const int64_t max_splits = ceil_div(rows, 256);
      if (splits > max_splits) splits = max_splits;
      if (splits < 1) splits = 1;
      if (splits > 65535) splits = 65535;
      const int64_t rps = ceil_div(rows, splits);
      const size_t smem = letters_smem_bytes<W>();
      auto kern = k_bitmatrix_letters<W>;
      PLB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      for (int64_t cbase = 0; cbase < colblocks; cbase += 65535) {
        const int64_t nblk = colblocks - cbase < 65535 ? colblocks - cbase : 65535;
        dim3 grid((unsigned)nblk, (unsigned)splits);
        StageTimer t_(st, "k_bitmatrix_letters");
        kern<<<grid, 1024, smem, st>>>(x, z, ld, M, row0, rows, col0 + cbase * kColsY,
                                       cols - cbase * kColsY, off, list,
                                       bits + cbase * (kColsY / 32), ld_bits, rps);
        PLB_CHECK_LAUNCH("k_bitmatrix_lists");
      }
      return PL_OK;
    }
  }
  // method 2
  constexpr int kDirectCols = DirectCols<W>::value;
  const int64_t colblocks = ceil_div(cols, kDirectCols);
  const int64_t rowblocks = ceil_div(rows, kDirectRows);
  for (int64_t rb = 0; rb < rowblocks; rb += 65535) {
    const int64_t nrb = rowblocks - rb < 65535 ? rowblocks - rb : 65535;
    dim3 grid((unsigned)colblocks, (unsigned)nrb);
    StageTimer t_(st, "k_bitmatrix_direct");
    k_bitmatrix_direct<W><<<grid, kDirectRows, 0, st>>>(
        x, z, ld, M, row0 + rb * kDirectRows, rows - rb * kDirectRows, col0, cols,
        bits + rb * kDirectRows * ld_bits, ld_bits);
    PLB_CHECK_LAUNCH("k_bitmatrix_direct");
  }
  return PL_OK;
}

}  // namespace plb

using namespace plb;

extern "C" int64_t pl_bitmatrix_workspace_bytes(int W, int64_t rows) {
  (void)W;
  if (rows < 0) return 0;
  return (rows + 1) * 4 + scan_scratch_words(rows) * 4 + 16 + list_capacity_entries(rows) * 4;
}

extern "C" int pl_commutation_bitmatrix(int W, int64_t M, const uint64_t* x, const uint64_t* z,
                                        int64_t ld, int64_t row0, int64_t rows, int64_t col0,
                                        int64_t cols, uint32_t* bits, int64_t ld_bits, int method,
                                        void* workspace, size_t workspace_bytes, void* stream) {
  if (M < 0 || ld < M || row0 < 0 || rows < 0 || row0 + rows > M || col0 < 0 || cols < 0 ||
      col0 + cols > M || (col0 % 32) != 0 || ld_bits < ceil_div(cols, 32) || method < 0 ||
      method > 3) {
    set_error("pl_commutation_bitmatrix: bad arguments");
    return PL_ERR_ARG;
  }
  if (rows * 128LL * (W > 0 ? W : 1) >= 0xFFFFFFFFLL) {
    set_error("pl_commutation_bitmatrix: too many rows per call (split the row range)");
    return PL_ERR_CAPACITY;
  }
  if (rows == 0 || cols == 0) return PL_OK;
  return PLB_DISPATCH_W(W, launch_bitmatrix, M, (const u64*)x, (const u64*)z, ld, row0, rows,
                        col0, cols, bits, ld_bits, method, workspace, workspace_bytes,
                        (cudaStream_t)stream);
}
