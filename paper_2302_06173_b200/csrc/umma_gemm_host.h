// Host helpers for umma_gemm.cuh: TMA tensor maps (driver entry point fetched
// through the runtime, so nothing links libcuda directly) and the launcher.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "internal.h"  // DeviceOnce
#include "umma_gemm.cuh"

namespace rwb {
namespace gemm {

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                   CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                   CUtensorMapFloatOOBfill);

inline EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// 2-D bf16 row-major matrix [rows, cols] (cols contiguous, row pitch ld
// elements), box {box_cols cols, box_rows rows}, OOB -> zeros; the swizzle
// follows the box row (128 B -> 128-byte swizzle, 64 B -> 64-byte swizzle).
inline int make_map(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint64_t ld,
                    uint32_t box_rows, uint32_t box_cols = 64) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return static_cast<int>(cudaErrorNotSupported);
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * 2};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, box_cols * 2 == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                                                       : CU_TENSOR_MAP_SWIZZLE_64B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : static_cast<int>(cudaErrorInvalidValue);
}

// MN-major operand [K rows, MN cols] (MN contiguous, pitch ld) as a 3-D tensor
// {64 MN, K, MN / 64 chunks} (strides: ld x 2 bytes per K row, 128 bytes per
// chunk), box {64, box_k, chunks}: one TMA instruction per stage lays the
// chunks out 64 x box_k x 2 bytes apart, exactly as `chunks` 2-D boxes would.
inline int make_map_mn3(CUtensorMap* map, const void* base, uint64_t k_rows, uint64_t mn_cols, uint64_t ld,
                        uint32_t box_k, uint32_t chunks) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return static_cast<int>(cudaErrorNotSupported);
  cuuint64_t dims[3] = {64, k_rows, (mn_cols + 63) / 64};
  cuuint64_t strides[2] = {ld * 2, 128};
  cuuint32_t box[3] = {64, box_k, chunks};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : static_cast<int>(cudaErrorInvalidValue);
}

// Epilogue staging box map: [rows, cols] row-major, element size esize, box
// {128 bytes of columns, 32 rows}, 128-byte swizzle.  Fails (non-zero) when
// the matrix cannot be a TMA operand (base not 16-byte aligned, pitch not a
// multiple of 16 bytes); the launcher then keeps the register epilogue.
inline int make_epi_map(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint64_t ld, int esize) {
  EncodeTiledFn fn = encode_fn();
  if (!fn || !base || (reinterpret_cast<uintptr_t>(base) & 15u) || ((ld * esize) & 15u)) return 1;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * esize};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(128 / esize), 32};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, esize == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                  const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : 1;
}

// RW_GEMM_TMA_EPI=0 keeps the register epilogue (A/B measurements)
inline int& tma_epi_override() {  // -1: environment / default; 0 / 1 forced (tests)
  static int v = -1;
  return v;
}
inline bool tma_epi_enabled() {
  if (tma_epi_override() >= 0) return tma_epi_override() != 0;
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("RW_GEMM_TMA_EPI");
    v = (e && *e) ? (std::atoi(e) != 0) : 1;
  }
  return v != 0;
}

// C[M,N] (+)= A . B^T with A given as [M,K] (K_MAJOR) or [K,M] (MN_MAJOR) and
// B as [N,K] (K_MAJOR) or [K,N] (MN_MAJOR); lda/ldb = row pitch in elements.
template <int BN, int AMAJ, int BMAJ, int EPI>
int launch(const void* A, int64_t lda, const void* B, int64_t ldb, int M, int N, int K, const EpiArgs& ep,
           cudaStream_t stream, int max_ctas = 0) {
  CUtensorMap ma, mb;
  // K-major: box {BK of K, rows}; MN-major: box {64 of M/N, BK K-rows}, or the
  // whole tile's chunks as one 3-D box (RWB_TMA3D, M/N a multiple of 64 so no
  // chunk reads past the matrix)
  const bool a3 = RWB_TMA3D && AMAJ == MN_MAJOR && M % 64 == 0;
  const bool b3 = RWB_TMA3D && BMAJ == MN_MAJOR && N % 64 == 0;
  int e = AMAJ == K_MAJOR ? make_map(&ma, A, M, K, lda, BM, BK)
          : a3            ? make_map_mn3(&ma, A, K, M, lda, BK, BM / 64)
                          : make_map(&ma, A, K, M, lda, BK);
  if (e) return e;
  e = BMAJ == K_MAJOR ? make_map(&mb, B, N, K, ldb, BN, BK)
      : b3            ? make_map_mn3(&mb, B, K, N, ldb, BK, BN / 64)
                      : make_map(&mb, B, K, N, ldb, BK);
  if (e) return e;
  EpiArgs epx = ep;
  epx.mn3 = (a3 ? 1 : 0) | (b3 ? 2 : 0);
  CUtensorMap mo{}, mi{};
  {
    constexpr int es = epi_f32(EPI) ? 4 : 2;
    bool ok = tma_epi_enabled() && make_epi_map(&mo, ep.out, M, N, ep.ldo, es) == 0;
    if (ok && uses_y(EPI)) ok = make_epi_map(&mi, ep.y, M, N, ep.ldy, 2) == 0;
    if (ok && EPI == EPI_F32_ACC) mi = mo;
    epx.tma_epi = ok ? 1 : 0;
    // fused column sums exist only in the TMA epilogue (float2 stores: even ldc, 8-byte base)
    if (ep.colsum && (!ok || !uses_y(EPI) || (ep.ldc & 1) || (reinterpret_cast<uintptr_t>(ep.colsum) & 7)))
      return static_cast<int>(cudaErrorNotSupported);
  }
  auto kern = umma_gemm_kernel<BN, AMAJ, BMAJ, EPI>;
  static DeviceOnce once;  // the attribute is per device
  const int se = once.run([&](int) {
    return static_cast<int>(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 static_cast<int>(Cfg<BN>::kSmem)));
  });
  if (se) return se;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int tiles = ((M + BM - 1) / BM) * ((N + BN - 1) / BN);
  int grid = tiles < sms ? tiles : sms;
  if (max_ctas > 0 && grid > max_ctas) grid = max_ctas;
  kern<<<grid, kThreads, Cfg<BN>::kSmem, stream>>>(ma, mb, mo, mi, M, N, K, epx);
  return static_cast<int>(cudaGetLastError());
}

// CTA-pair (cta_group::2) variant: same contract, M tiles of 256 (MH = 1) or
// 512 (MH = 2: 256 rows per CTA) per pair.
template <int BN, int AMAJ, int BMAJ, int EPI, int MH = 1>
int launch2(const void* A, int64_t lda, const void* B, int64_t ldb, int M, int N, int K, const EpiArgs& ep,
            cudaStream_t stream, int max_ctas = 0) {
  CUtensorMap ma, mb;
  int e = AMAJ == K_MAJOR ? make_map(&ma, A, M, K, lda, MH * BM, BK) : make_map(&ma, A, K, M, lda, BK);
  if (e) return e;
  e = BMAJ == K_MAJOR ? make_map(&mb, B, N, K, ldb, BN / 2, BK) : make_map(&mb, B, K, N, ldb, BK);
  if (e) return e;
  EpiArgs epx = ep;
  CUtensorMap mo{}, mi{};
  {
    constexpr int es = epi_f32(EPI) ? 4 : 2;
    bool ok = tma_epi_enabled() && make_epi_map(&mo, ep.out, M, N, ep.ldo, es) == 0;
    if (ok && uses_y(EPI)) ok = make_epi_map(&mi, ep.y, M, N, ep.ldy, 2) == 0;
    if (ok && EPI == EPI_F32_ACC) mi = mo;
    epx.tma_epi = ok ? 1 : 0;
    if (ep.colsum && (!ok || !uses_y(EPI) || (ep.ldc & 1) || (reinterpret_cast<uintptr_t>(ep.colsum) & 7)))
      return static_cast<int>(cudaErrorNotSupported);
  }
  auto kern = umma_gemm2_kernel<BN, AMAJ, BMAJ, EPI, MH>;
  static DeviceOnce once;  // the attribute is per device
  const int se = once.run([&](int) {
    return static_cast<int>(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 static_cast<int>(Cfg2<BN, MH>::kSmem)));
  });
  if (se) return se;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int tiles = ((M + 2 * MH * BM - 1) / (2 * MH * BM)) * ((N + BN - 1) / BN);
  int pairs = sms / 2;
  if (tiles < pairs) pairs = tiles;
  if (max_ctas > 0 && pairs * 2 > max_ctas) pairs = max_ctas / 2 > 0 ? max_ctas / 2 : 1;
  kern<<<pairs * 2, Cfg2<BN, MH>::kThreads, Cfg2<BN, MH>::kSmem, stream>>>(ma, mb, mo, mi, M, N, K, epx);
  return static_cast<int>(cudaGetLastError());
}

}  // namespace gemm
}  // namespace rwb
