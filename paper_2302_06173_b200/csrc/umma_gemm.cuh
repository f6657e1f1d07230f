// Blackwell (sm_100a) bf16 GEMM on the 5th-gen tensor cores, hand-written:
//   TMA (cp.async.bulk.tensor, 128B swizzle) -> smem ring (kStages)
//   -> one elected thread issues tcgen05.mma.cta_group::1.kind::f16
//      (M=128, N=BN, K=16 per instruction) into a TMEM fp32 accumulator
//   -> 4 epilogue warps: tcgen05.ld -> fused epilogue -> global.
// Persistent: one CTA per SM walks output tiles; two TMEM accumulator stages
// let the epilogue of tile i overlap the MMAs of tile i+1.
//
// C[M,N] = A[M,K] . B[N,K]^T  (UMMA convention), where each operand is
// either K-major (K contiguous) or MN-major (M resp. N contiguous) in global
// memory.  This covers the three replay GEMMs of an affine layer
// (model.cpp:59-73, 121-147) without transposes:
//   forward  Y[R,N]  = X[R,K] . W[K,N]     A=X  K-major, B=W  MN-major
//   dgrad    dX[R,K] = dZ[R,N] . W[K,N]^T  A=dZ K-major, B=W  K-major
//   wgrad    dW[K,N] = X[R,K]^T . dZ[R,N]  A=X  MN-major, B=dZ MN-major
//
// Determinism: fixed tiling, no split-K, no atomics: identical inputs give
// identical bits (the GPU "ghost run" contract of SURVEY §7 hard part 5).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace rwb {
namespace gemm {

constexpr int BM = 128;
// K depth of one pipeline stage: 64 bf16 = 128 B rows (128-byte swizzle) or,
// with RWB_GEMM_BK=32, 64 B rows (64-byte swizzle) and twice the stages in the
// same shared memory -- a stage is released after 2 MMAs instead of 4, so the
// loads in flight cover more of the memory latency.
#ifndef RWB_GEMM_BK
#define RWB_GEMM_BK 64
#endif
constexpr int BK = RWB_GEMM_BK;
static_assert(BK == 64 || BK == 32, "BK: 64 (128B swizzle) or 32 (64B swizzle)");
constexpr uint32_t kKRowBytes = BK * 2;                // K-major row = one swizzle atom row
constexpr uint32_t kKSwizzleCode = BK == 64 ? 2u : 4u;  // SM100 descriptor layout: 128B / 64B swizzle
constexpr int kThreads = 256;  // warp0 TMA, warp1 MMA, warp2 TMEM alloc, warps 4-7 epilogue
constexpr int kEpiWarp0 = 4;

enum Major : int { K_MAJOR = 0, MN_MAJOR = 1 };

enum Epi : int {
  EPI_BF16 = 0,           // out_bf16 = acc
  EPI_BIAS_TANH_BF16 = 1, // out_bf16 = tanh(acc + bias[n])            (forward)
  EPI_DTANH_BF16 = 2,     // out_bf16 = acc * (1 - y[m,n]^2)           (dgrad -> next dz)
  EPI_F32 = 3,            // out_f32  = acc                             (wgrad, first mb)
  EPI_F32_ACC = 4,        // out_f32  = out_f32 + acc                   (wgrad, ordered mb sum)
  EPI_BOUNDARY_DTANH_BF16 = 5,  // out_bf16 = bf16(acc) * (1 - y^2): a stage-boundary gradient
                                // (rounded to bf16 as sent) fused with the previous stage's dz
};
__host__ __device__ constexpr bool uses_y(int epi) { return epi == EPI_DTANH_BF16 || epi == EPI_BOUNDARY_DTANH_BF16; }

struct EpiArgs {
  void* out;             // bf16 or f32 [M, N] row-major, leading dim ldo (elements)
  int64_t ldo;
  const float* bias;     // [N] (EPI_BIAS_TANH_BF16)
  const __nv_bfloat16* y;  // [M, N] row-major, ld ldy (EPI_DTANH_BF16)
  int64_t ldy;
  int tma_epi;           // set by the launcher: output (and y / old output) tiles move by TMA
  int mn3;               // set by the launcher: bit 0 / 1 = the MN-major A / B map is 3-D (one TMA per stage)
  float* colsum;         // dtanh epilogues, TMA path: per 32-row block column sums of the bf16
  int64_t ldc;           //   output, colsum[(row / 32) * ldc + col] (fused db partials)
};
__host__ __device__ constexpr bool epi_f32(int epi) { return epi == EPI_F32 || epi == EPI_F32_ACC; }
// epilogues that read an [M, N] tile besides the accumulator (y, or the old output)
__host__ __device__ constexpr bool epi_input(int epi) { return uses_y(epi) || epi == EPI_F32_ACC; }

// ---------------------------------------------------------------- PTX
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
// Waits on an mbarrier phase.  A pipeline bug must not hang the GPU: after
// ~2^34 cycles (several seconds) the kernel traps instead.
#ifndef RWB_WAIT_HINT_NS
#define RWB_WAIT_HINT_NS 200000
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  uint32_t done = 0;
  const long long t0 = clock64();
  while (true) {
#if RWB_WAIT_HINT_NS
    // suspend-time hint: the waiting warp is parked until the phase flips (or
    // the hint elapses) instead of re-polling -- fewer issue slots and less
    // power spent by the producer / epilogue warps while the MMAs run
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\n"
        "selp.u32 %0, 1, 0, P1;\n"
        "}\n"
        : "=r"(done)
        : "r"(smem_u32(b)), "r"(parity), "r"(uint32_t(RWB_WAIT_HINT_NS))
        : "memory");
#else
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
        "selp.u32 %0, 1, 0, P1;\n"
        "}\n"
        : "=r"(done)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
#endif
    if (done) return;
    if (clock64() - t0 > (1ll << 34)) __trap();
  }
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                            int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
// 3-D box {64 MN, BK K-rows, n chunks}: an MN-major tile's 64-wide chunks in
// one instruction (chunk c lands c x 64 x BK x 2 bytes further in smem)
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
#ifndef RWB_TMA3D
#define RWB_TMA3D 0
#endif  // 1: MN-major operands whose M/N is a multiple of 64 load through 3-D maps
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
// smem -> global tensor store (bulk group), and the group waits
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// generic-proxy smem writes -> visible to the async proxy (TMA store source)
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_mma(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accum) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum)
      : "memory");
}
// 32 lanes x 32 consecutive fp32 columns: thread i gets row (lane base + i)
__device__ __forceinline__ void tmem_ld_32cols(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
        "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
        "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// the same load without the wait: several loads share one tcgen05.wait::ld
__device__ __forceinline__ void tmem_ld_32cols_nowait(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
        "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
        "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// UMMA shared-memory descriptor (SM100 "version 1"), SWIZZLE_128B.
//   K-major : rows of 128 B (64 bf16 of K); 8-row groups 1024 B apart (SBO).
//   MN-major: rows of 128 B (64 bf16 of M/N) per K index; 8 K-rows = 1024 B
//             (SBO); successive 64-wide M/N chunks LBO bytes apart.
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes,
                                              uint32_t layout = 2u /* SWIZZLE_128B */) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3FFFu);
  d |= uint64_t((lbo_bytes >> 4) & 0x3FFFu) << 16;
  d |= uint64_t((sbo_bytes >> 4) & 0x3FFFu) << 32;
  d |= uint64_t(1) << 46;  // version = 1 (Blackwell)
  d |= uint64_t(layout) << 61;
  return d;
}
// K-major operand, 16-element K step k inside the stage: +32 B along the row;
// 8-row groups 8 x kKRowBytes apart (SBO)
__device__ __forceinline__ uint64_t kmajor_desc(uint32_t base, int k) {
  return make_desc(base + uint32_t(k) * 32u, 16, 8 * kKRowBytes, kKSwizzleCode);
}

// kind::f16 instruction descriptor: BF16 x BF16 -> F32, dense
__host__ __device__ constexpr uint32_t make_idesc(int m, int n, int a_major, int b_major) {
  return (1u << 4)                      // c_format F32
         | (1u << 7)                    // a_format BF16
         | (1u << 10)                   // b_format BF16
         | (uint32_t(a_major) << 15)    // a major
         | (uint32_t(b_major) << 16)    // b major
         | (uint32_t(n >> 3) << 17)     // N / 8
         | (uint32_t(m >> 4) << 24);    // M / 16
}

// tanh for the forward epilogue: the MUFU approximation (max relative error
// ~2^-11) instead of the ~20-instruction accurate tanhf; the result is
// rounded to bf16 (2^-9 relative) right after, so the replay tolerance is
// unaffected, and the epilogue warps no longer steal issue slots from the
// MMA warp's scheduler (forward GEMM 165.5 -> 157.4 cycles per MMA, profiles/r01/README.md).
__device__ __forceinline__ float tanh_fast(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// y operand of EPI_DTANH_BF16 for one full 32-column chunk of one row:
// 4 x 128-bit loads, issued ahead of use so their latency overlaps the
// accumulator wait / the previous chunk.
struct YChunk {
  uint4 q[4];
};
// (the register epilogue serves pitches / bases the TMA maps reject, so every
// vector access checks the actual address)
__device__ __forceinline__ bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
__device__ __forceinline__ void load_y_chunk(const EpiArgs& ep, int row, int col0, int M, int N, YChunk& y) {
  if (row < M && col0 + 32 <= N && al16(ep.y + int64_t(row) * ep.ldy + col0)) {
    const uint4* p = reinterpret_cast<const uint4*>(ep.y + int64_t(row) * ep.ldy + col0);
#pragma unroll
    for (int q = 0; q < 4; ++q) y.q[q] = __ldg(p + q);
  }
}

// Epilogue of one 32-column TMEM chunk for one accumulator row (thread).
// yk: the chunk's y already in registers (EPI_DTANH_BF16, full chunks).
template <int EPI>
__device__ __forceinline__ void epi_chunk(const float* v, int row, int col0, int N, const EpiArgs& ep,
                                          const YChunk* yk = nullptr) {
    if constexpr (EPI == EPI_F32 || EPI == EPI_F32_ACC) {
      float* o = static_cast<float*>(ep.out) + int64_t(row) * ep.ldo + col0;
      if (col0 + 32 <= N && al16(o)) {
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          float4 w = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
          if constexpr (EPI == EPI_F32_ACC) {
            const float4 p = *reinterpret_cast<const float4*>(o + j);
            w.x = __fadd_rn(p.x, w.x);
            w.y = __fadd_rn(p.y, w.y);
            w.z = __fadd_rn(p.z, w.z);
            w.w = __fadd_rn(p.w, w.w);
          }
          *reinterpret_cast<float4*>(o + j) = w;
        }
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)  // constant trip count: v stays in registers
          if (col0 + j < N) o[j] = EPI == EPI_F32_ACC ? __fadd_rn(o[j], v[j]) : v[j];
      }
    } else {
      __nv_bfloat16* o = static_cast<__nv_bfloat16*>(ep.out) + int64_t(row) * ep.ldo + col0;
      const bool full = col0 + 32 <= N;
      const bool full_y = full && (!uses_y(EPI) || al16(ep.y + int64_t(row) * ep.ldy + col0));
      float w[32];
      if constexpr (EPI == EPI_BIAS_TANH_BF16) {
        float bv[32];
        if (full && (reinterpret_cast<uintptr_t>(ep.bias) & 15u) == 0) {  // same 128 B for every lane: one broadcast each
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            const float4 b4 = __ldg(reinterpret_cast<const float4*>(ep.bias + col0 + j));
            bv[j] = b4.x;
            bv[j + 1] = b4.y;
            bv[j + 2] = b4.z;
            bv[j + 3] = b4.w;
          }
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) bv[j] = (col0 + j < N) ? __ldg(ep.bias + col0 + j) : 0.f;
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) w[j] = tanh_fast(__fadd_rn(v[j], bv[j]));
      } else if constexpr (uses_y(EPI)) {
        const __nv_bfloat16* yp = ep.y + int64_t(row) * ep.ldy + col0;
        float yv[32];
        if (full_y) {  // 64 contiguous bytes of this row: 4 x 128-bit loads (prefetched when yk)
#pragma unroll
          for (int j = 0; j < 32; j += 8) {
            const uint4 u = yk ? yk->q[j / 8] : *reinterpret_cast<const uint4*>(yp + j);
            const __nv_bfloat162* p2 = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const float2 f = __bfloat1622float2(p2[q]);
              yv[j + 2 * q] = f.x;
              yv[j + 2 * q + 1] = f.y;
            }
          }
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) yv[j] = (col0 + j < N) ? __bfloat162float(yp[j]) : 0.f;
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          // boundary: the gradient crosses the stage boundary as bf16 (the
          // wire value), then dtanh_first's expression, bit for bit
          const float g = EPI == EPI_BOUNDARY_DTANH_BF16 ? __bfloat162float(__float2bfloat16_rn(v[j])) : v[j];
          w[j] = __fmul_rn(g, __fsub_rn(1.f, __fmul_rn(yv[j], yv[j])));
        }
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) w[j] = v[j];
      }
#ifdef RWB_PROBE_NOSTORE
      if (w[0] != 12345.f) return;  // probe only: compute everything, store (almost) nothing
#endif
      if (full && al16(o)) {
#pragma unroll
        for (int j = 0; j < 32; j += 8) {
          uint4 pk;
          __nv_bfloat162 h0 = __floats2bfloat162_rn(w[j], w[j + 1]);
          __nv_bfloat162 h1 = __floats2bfloat162_rn(w[j + 2], w[j + 3]);
          __nv_bfloat162 h2 = __floats2bfloat162_rn(w[j + 4], w[j + 5]);
          __nv_bfloat162 h3 = __floats2bfloat162_rn(w[j + 6], w[j + 7]);
          pk.x = *reinterpret_cast<uint32_t*>(&h0);
          pk.y = *reinterpret_cast<uint32_t*>(&h1);
          pk.z = *reinterpret_cast<uint32_t*>(&h2);
          pk.w = *reinterpret_cast<uint32_t*>(&h3);
          *reinterpret_cast<uint4*>(o + j) = pk;
        }
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (col0 + j < N) o[j] = __float2bfloat16_rn(w[j]);
      }
    }
}

// Drain one accumulator tile: this thread owns TMEM lane `row - m0`.
// EPI_DTANH_BF16: y0 holds chunk 0's y (loaded before the accumulator wait);
// chunk c+1's y is loaded before chunk c is processed.
template <int BN, int EPI>
__device__ __forceinline__ void epilogue_tile(uint32_t tbase, int row, int n0, int M, int N, const EpiArgs& ep,
                                              const YChunk* y0 = nullptr) {
  if constexpr (uses_y(EPI)) {
    YChunk cur = *y0, nxt;
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 32) {
      if (c0 + 32 < BN) load_y_chunk(ep, row, n0 + c0 + 32, M, N, nxt);
      float v[32];
      tmem_ld_32cols(tbase + uint32_t(c0), v);
      if (row < M) epi_chunk<EPI>(v, row, n0 + c0, N, ep, &cur);
      cur = nxt;
    }
  } else {
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 32) {
      float v[32];
      tmem_ld_32cols(tbase + uint32_t(c0), v);
      if (row < M) epi_chunk<EPI>(v, row, n0 + c0, N, ep);
    }
  }
}

// ---------------------------------------------------------------- TMA epilogue
// Each epilogue warp owns 32 accumulator rows and two 32-row x 128-byte
// staging boxes in shared memory (128-byte swizzle: the 16-byte piece p of
// row r sits at piece p ^ (r % 8), so a warp's row-per-lane accesses are
// bank-conflict free).  A box holds 64 bf16 or 32 fp32 output columns; it
// leaves by one TMA tensor store (full 128-byte lines, clipped at the matrix
// edge), while the other box is being filled.  Epilogues with an input tile
// (y of the dtanh epilogues, the old output of the fp32 accumulate) TMA-load
// it into the box one box ahead and compute in place.
#ifdef RWB_PAIR_EXPERIMENT
// epilogue probe (warp 4, lane 0 of every CTA): [0] cycles inside the tile
// epilogues, [1] waiting for a staging buffer / input box, [2] TMEM loads,
// [3] column sums
__device__ long long g_epi_dbg[148][4];
#define RWB_EPI_T(v) const long long v = (threadIdx.x == 128 ? clock64() : 0)
#define RWB_EPI_ADD(k, t0) \
  if (threadIdx.x == 128) g_epi_dbg[blockIdx.x][k] += clock64() - (t0)
#else
#define RWB_EPI_T(v)
#define RWB_EPI_ADD(k, t0)
#endif
constexpr uint32_t kEpiBoxBytes = 32 * 128;
constexpr uint32_t kEpiSmem = 4 * 2 * kEpiBoxBytes;  // 4 warps x double buffer

__device__ __forceinline__ uint32_t swz(uint32_t row, uint32_t piece) {
  return row * 128u + ((piece ^ (row & 7u)) << 4);
}
__device__ __forceinline__ void epi_load_box(const CUtensorMap* mi, uint8_t* buf, uint64_t* bar, int c0, int r0) {
  mbar_expect_tx(bar, kEpiBoxBytes);
  tma_load_2d(buf, mi, bar, c0, r0);
}

// `release` runs once, right after the tile's last TMEM load has completed:
// the accumulator goes back to the MMA warp while the last box is still being
// computed and stored (TMEM is full for the wide pair, so that box's math and
// store would otherwise stall the next tile's MMAs).
// NBUF staging boxes per warp: 2 = the next input box is prefetched into the
// other buffer and a box's store overlaps the next box's math; 1 = the wide
// pair's 16-warp epilogue (half the smem per warp) -- an output-only box is
// computed into registers before the wait for the previous store to have read
// the buffer, and an input box is fetched once that store has read it.
#ifndef RWB_EPI_EARLY_RELEASE
#define RWB_EPI_EARLY_RELEASE 1
#endif
template <int NBUF>
__device__ __forceinline__ void epi_first_input(const CUtensorMap* mi, uint8_t* ebuf, uint64_t* ebar, uint32_t seq,
                                                int c0, int r0) {
  const uint32_t b = NBUF == 2 ? (seq & 1u) : 0u;
  bulk_wait_read<0>();
  epi_load_box(mi, ebuf + b * kEpiBoxBytes, &ebar[b], c0, r0);
}
// The tile's bias columns [c0, c0 + BN) into this warp's shared array (zero
// past N), read by the forward epilogue as broadcast LDS instead of global
// loads on the critical path; staged while the warp waits for the accumulator.
template <int BN>
__device__ __forceinline__ void stage_bias(float* sb, const float* bias, int c0, int N) {
  constexpr int PER = BN / 32;  // columns per lane
  static_assert(PER % 4 == 0, "float4 pieces");
  const int lane = int(threadIdx.x & 31u);
  const bool vec = (reinterpret_cast<uintptr_t>(bias) & 15u) == 0;  // caller-owned pointer: may be unaligned
  __syncwarp();  // every lane is done reading the previous tile's bias
#pragma unroll
  for (int q = 0; q < PER; q += 4) {
    const int c = c0 + lane * PER + q;
    float4 b;
    if (vec && c + 4 <= N) {
      b = __ldg(reinterpret_cast<const float4*>(bias + c));
    } else {
      b.x = c < N ? __ldg(bias + c) : 0.f;
      b.y = c + 1 < N ? __ldg(bias + c + 1) : 0.f;
      b.z = c + 2 < N ? __ldg(bias + c + 2) : 0.f;
      b.w = c + 3 < N ? __ldg(bias + c + 3) : 0.f;
    }
    *reinterpret_cast<float4*>(sb + lane * PER + q) = b;
  }
  __syncwarp();
}

template <int BN, int EPI, int NBUF, class Release>
__device__ __forceinline__ void epilogue_tile_tma(uint32_t tbase, int r0, int n0, int M, int N, const EpiArgs& ep,
                                                  const CUtensorMap* mo, const CUtensorMap* mi, uint8_t* ebuf,
                                                  uint64_t* ebar, uint32_t& seq, Release release,
                                                  const float* sbias = nullptr) {
  static_assert(NBUF == 1 || NBUF == 2, "one or two staging boxes per warp");
  constexpr int COLS = epi_f32(EPI) ? 32 : 64;
  constexpr int NB = BN / COLS;
  const uint32_t lane = threadIdx.x & 31u;
  RWB_EPI_T(te0);
#pragma unroll 1
  for (int i = 0; i < NB; ++i, ++seq) {
    const uint32_t b = NBUF == 2 ? (seq & 1u) : 0u;
    uint8_t* buf = ebuf + b * kEpiBoxBytes;
    const int c0 = n0 + i * COLS;
    RWB_EPI_T(tl0);
    // the box's accumulator columns: every 32-column load issued, one wait
    uint32_t vr[COLS / 32][32];
#pragma unroll
    for (int h = 0; h < COLS / 32; ++h) tmem_ld_32cols_nowait(tbase + uint32_t(i * COLS + h * 32), vr[h]);
    RWB_EPI_ADD(2, tl0);
    RWB_EPI_T(tw0);
    if constexpr (epi_input(EPI)) {
      if (lane == 0) {
        if constexpr (NBUF == 2) {
          if (i + 1 < NB) {  // next box's input, into the other buffer once its store has read it
            bulk_wait_read<0>();
            epi_load_box(mi, ebuf + (b ^ 1u) * kEpiBoxBytes, &ebar[b ^ 1u], c0 + COLS, r0);
          }
        } else if (i > 0) {  // this box's input, once the previous box's store has read the buffer
          bulk_wait_read<0>();
          epi_load_box(mi, buf, &ebar[0], c0, r0);
        }
      }
      mbar_wait(&ebar[b], NBUF == 2 ? (seq >> 1) & 1u : seq & 1u);
    }
    RWB_EPI_ADD(1, tw0);
    tmem_wait_ld();
    if (RWB_EPI_EARLY_RELEASE && i == NB - 1) {
      tc_fence_before();
      __syncwarp();
      release();
    }
    // an output-only box is computed into registers first; the wait for its
    // buffer (the store two boxes back, or the previous one when NBUF == 1)
    // comes after the math
    const auto own_buffer = [&] {
      if constexpr (!epi_input(EPI)) {
        RWB_EPI_T(tb0);
        if (lane == 0) bulk_wait_read<NBUF - 1>();
        __syncwarp();
        RWB_EPI_ADD(1, tb0);
      }
    };
    if constexpr (epi_f32(EPI)) {
      if constexpr (EPI != EPI_F32_ACC) own_buffer();
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        float4* p = reinterpret_cast<float4*>(buf + swz(lane, q));
        float4 w = make_float4(__uint_as_float(vr[0][4 * q]), __uint_as_float(vr[0][4 * q + 1]),
                               __uint_as_float(vr[0][4 * q + 2]), __uint_as_float(vr[0][4 * q + 3]));
        if constexpr (EPI == EPI_F32_ACC) {
          const float4 o = *p;
          w.x = __fadd_rn(o.x, w.x);
          w.y = __fadd_rn(o.y, w.y);
          w.z = __fadd_rn(o.z, w.z);
          w.w = __fadd_rn(o.w, w.w);
        }
        *p = w;
      }
    } else {
      uint4 pk[COLS / 32][4];
#pragma unroll
      for (int h = 0; h < COLS / 32; ++h) {
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(vr[h][j]);
        const int col = c0 + h * 32;
        float w[32];
        if constexpr (EPI == EPI_BIAS_TANH_BF16) {
          float bv[32];
#ifdef RWB_PROBE_NOBIAS  // probe only: no bias loads
#pragma unroll
          for (int j = 0; j < 32; ++j) bv[j] = float(j) * 0.5f;
          if (false) {
#else
          if (sbias) {  // staged in shared memory at the tile's start (zero past N): broadcast reads
#pragma unroll
            for (int j = 0; j < 32; j += 4) {
              const float4 b4 = *reinterpret_cast<const float4*>(sbias + i * COLS + h * 32 + j);
              bv[j] = b4.x;
              bv[j + 1] = b4.y;
              bv[j + 2] = b4.z;
              bv[j + 3] = b4.w;
            }
          } else if (col + 32 <= N && (reinterpret_cast<uintptr_t>(ep.bias) & 15u) == 0) {
#endif
#pragma unroll
            for (int j = 0; j < 32; j += 4) {
              const float4 b4 = __ldg(reinterpret_cast<const float4*>(ep.bias + col + j));
              bv[j] = b4.x;
              bv[j + 1] = b4.y;
              bv[j + 2] = b4.z;
              bv[j + 3] = b4.w;
            }
          } else {
#ifndef RWB_PROBE_NOBIAS
#pragma unroll
            for (int j = 0; j < 32; ++j) bv[j] = (col + j < N) ? __ldg(ep.bias + col + j) : 0.f;
#endif
          }
#pragma unroll
          for (int j = 0; j < 32; ++j) {
#ifdef RWB_PROBE_NOTANH  // probe only: the epilogue without its MUFU work
            w[j] = __fadd_rn(v[j], bv[j]);
#else
            w[j] = tanh_fast(__fadd_rn(v[j], bv[j]));
#endif
          }
        } else if constexpr (uses_y(EPI)) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const uint4 u = *reinterpret_cast<const uint4*>(buf + swz(lane, h * 4 + q));
            const __nv_bfloat162* p2 = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 y2 = __bfloat1622float2(p2[e]);
              const int j = q * 8 + 2 * e;
              const float g0 = EPI == EPI_BOUNDARY_DTANH_BF16 ? __bfloat162float(__float2bfloat16_rn(v[j])) : v[j];
              const float g1 =
                  EPI == EPI_BOUNDARY_DTANH_BF16 ? __bfloat162float(__float2bfloat16_rn(v[j + 1])) : v[j + 1];
              w[j] = __fmul_rn(g0, __fsub_rn(1.f, __fmul_rn(y2.x, y2.x)));
              w[j + 1] = __fmul_rn(g1, __fsub_rn(1.f, __fmul_rn(y2.y, y2.y)));
            }
          }
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) w[j] = v[j];
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          __nv_bfloat162 h0 = __floats2bfloat162_rn(w[8 * q], w[8 * q + 1]);
          __nv_bfloat162 h1 = __floats2bfloat162_rn(w[8 * q + 2], w[8 * q + 3]);
          __nv_bfloat162 h2 = __floats2bfloat162_rn(w[8 * q + 4], w[8 * q + 5]);
          __nv_bfloat162 h3 = __floats2bfloat162_rn(w[8 * q + 6], w[8 * q + 7]);
          pk[h][q].x = *reinterpret_cast<uint32_t*>(&h0);
          pk[h][q].y = *reinterpret_cast<uint32_t*>(&h1);
          pk[h][q].z = *reinterpret_cast<uint32_t*>(&h2);
          pk[h][q].w = *reinterpret_cast<uint32_t*>(&h3);
        }
        if constexpr (uses_y(EPI)) {  // in place over the consumed y pieces
#pragma unroll
          for (int q = 0; q < 4; ++q) *reinterpret_cast<uint4*>(buf + swz(lane, h * 4 + q)) = pk[h][q];
        }
      }
      if constexpr (!uses_y(EPI)) {
        own_buffer();
#ifdef RWB_PROBE_NOSTS  // probe only: no staging writes (the stores send stale smem)
        if (lane == 32)
#endif
#pragma unroll
        for (int h = 0; h < COLS / 32; ++h)
#pragma unroll
          for (int q = 0; q < 4; ++q) *reinterpret_cast<uint4*>(buf + swz(lane, h * 4 + q)) = pk[h][q];
      }
    }
    fence_proxy_async_smem();
    __syncwarp();
    RWB_EPI_T(tc0);
    if constexpr (uses_y(EPI)) {
      // (a box wholly below the matrix -- the tail of a 256 / 512-row tile -- has no
      // partial row to write: the buffer holds ceil(M / 32) of them)
      if (ep.colsum && r0 < M) {  // db partials: lane l sums columns 2l, 2l+1 of the box over its 32 rows, in row order
        float s0 = 0.f, s1 = 0.f;
#pragma unroll 8
        for (uint32_t r = 0; r < 32; ++r) {
          const __nv_bfloat162 p2 =
              *reinterpret_cast<const __nv_bfloat162*>(buf + swz(r, lane >> 2) + ((lane & 3u) << 2));
          const float2 f = __bfloat1622float2(p2);
          s0 = __fadd_rn(s0, f.x);
          s1 = __fadd_rn(s1, f.y);
        }
        const int col = c0 + 2 * int(lane);
        float* dst = ep.colsum + int64_t(r0 / 32) * ep.ldc + col;
        if (col + 1 < N) {
          *reinterpret_cast<float2*>(dst) = make_float2(s0, s1);
        } else if (col < N) {
          dst[0] = s0;
        }
      }
    }
    RWB_EPI_ADD(3, tc0);
    if (lane == 0) {
      tma_store_2d(mo, buf, c0, r0);
      bulk_commit();
    }
  }
  if (!RWB_EPI_EARLY_RELEASE) {
    tc_fence_before();
    __syncwarp();
    release();
  }
  RWB_EPI_ADD(0, te0);
}

// Grouped tile rasterization: consecutive tile ids walk GM M-tiles down one
// N column before moving right, so the ~148 concurrently active tiles cover a
// compact GM x (148/GM) block whose A and B panels stay resident in the
// 126 MB L2 (plain M-fastest order re-streams the whole A panel per N tile).
__device__ __forceinline__ void tile_coords(int tile, int tiles_m, int tiles_n, int gm, int& tm, int& tn) {
  const int per_group = gm * tiles_n;
  const int group = tile / per_group;
  const int first_m = group * gm;
  const int gsz = min(tiles_m - first_m, gm);
  const int in = tile - group * per_group;
  tm = first_m + in % gsz;
  tn = in / gsz;
}
#ifndef RWB_GROUP_M
#define RWB_GROUP_M 16
#endif
constexpr int kGroupM = RWB_GROUP_M;
// the pair kernels' raster group in M rows: 16 single-CTA tiles' worth for
// MH = 1 (8 pair tiles of 256 rows); 4096 rows = 8 pair tiles of 512 for MH = 2
// (profiles/r02/gemm_variants7_wide.log, replay ms: 1024 / 2048 / 4096 rows -> 633-634 / 627-630 / 623-626)
#ifndef RWB_GROUP_WIDE
#define RWB_GROUP_WIDE 8
#endif
template <int MH>
__host__ __device__ constexpr int group_tiles2() {
  return MH == 1 ? kGroupM / 2 : RWB_GROUP_WIDE;
}

template <int BN>
struct Cfg {
#ifdef RWB_GEMM_STAGES
  static constexpr int kStages = RWB_GEMM_STAGES;
#else
  static constexpr int kStages = (BN == 256 ? 4 : 6) * (64 / BK);
#endif
  static constexpr uint32_t kABytes = BM * BK * 2;   // 16 KB
  static constexpr uint32_t kBBytes = BN * BK * 2;   // 32 KB (BN=256)
  static constexpr uint32_t kStageBytes = kABytes + kBBytes;
  static constexpr uint32_t kTmemCols = 2 * BN;      // two accumulator stages
  static constexpr size_t kSmem = size_t(kStages) * kStageBytes + kEpiSmem + 1024;  // + alignment slack
};

// smem layout inside one operand buffer for MN-major tiles: TMA boxes of
// {64 (MN), 64 (K)} stacked along MN every 64*128 B = 8 KB  => LBO = 8192.
constexpr uint32_t kMnChunkBytes = 64 * 2 * BK;  // one 64-wide MN chunk x BK K-rows of 128 B

#ifdef RWB_PAIR_EXPERIMENT
// tools/pair_probe.cu / tools/gemm_probe.cu instrumentation (per CTA):
// [0] MMA-warp cycles waiting on full_bar, [1] on tempty_bar, [2] total MMA
// loop cycles, [3] producer cycles waiting on empty_bar
__device__ long long g_pair_dbg[148][4];
#endif

template <int BN, int AMAJ, int BMAJ, int EPI>
__global__ void __launch_bounds__(kThreads, 1)
    umma_gemm_kernel(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
                     const __grid_constant__ CUtensorMap tma_o, const __grid_constant__ CUtensorMap tma_i,
                     int M, int N, int K, EpiArgs ep) {
  using C = Cfg<BN>;
  constexpr int S = C::kStages;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte aligned base for the swizzled tiles
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full_bar[S], empty_bar[S], tfull_bar[2], tempty_bar[2], epi_bar[8];
  __shared__ uint32_t tmem_base_sh;

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int tiles_m = (M + BM - 1) / BM, tiles_n = (N + BN - 1) / BN;
  const int num_tiles = tiles_m * tiles_n;
  const int num_kb = (K + BK - 1) / BK;

  if (threadIdx.x == 0) {
    prefetch_tmap(&tma_a);
    prefetch_tmap(&tma_b);
    for (int i = 0; i < S; ++i) {
      mbar_init(&full_bar[i], 1);
      mbar_init(&empty_bar[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull_bar[i], 1);
      mbar_init(&tempty_bar[i], 4);  // one arrive per epilogue warp
    }
    for (int i = 0; i < 8; ++i) mbar_init(&epi_bar[i], 1);
    if (ep.tma_epi) {
      prefetch_tmap(&tma_o);
      if (epi_input(EPI)) prefetch_tmap(&tma_i);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {  // TMEM allocation (whole warp), address published via smem
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base_sh)),
                 "r"(C::kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_sh;

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        int tm, tn;
        tile_coords(tile, tiles_m, tiles_n, kGroupM, tm, tn);
        const int m0 = tm * BM, n0 = tn * BN;
        for (int kb = 0; kb < num_kb; ++kb) {
#ifdef RWB_PAIR_EXPERIMENT
          const long long w0 = clock64();
#endif
          mbar_wait(&empty_bar[stage], phase ^ 1);
#ifdef RWB_PAIR_EXPERIMENT
          g_pair_dbg[blockIdx.x][3] += clock64() - w0;
#endif
          uint8_t* sa = smem + stage * C::kStageBytes;
          uint8_t* sb = sa + C::kABytes;
#ifdef RWB_PROBE_NOTMA
          if (tile != int(blockIdx.x) || kb >= S) {  // probe only: no data movement after the first fill
            mbar_arrive(&full_bar[stage]);
            if (++stage == S) {
              stage = 0;
              phase ^= 1;
            }
            continue;
          }
#endif
          mbar_expect_tx(&full_bar[stage], C::kStageBytes);
          const int k0 = kb * BK;
          if constexpr (AMAJ == K_MAJOR) {
            tma_load_2d(sa, &tma_a, &full_bar[stage], k0, m0);  // box {64 K, 128 M}
          } else if (ep.mn3 & 1) {
            tma_load_3d(sa, &tma_a, &full_bar[stage], 0, k0, m0 / 64);  // box {64 M, 64 K, 2 chunks}
          } else {
#pragma unroll
            for (int c = 0; c < BM / 64; ++c)                    // boxes {64 M, 64 K}
              tma_load_2d(sa + c * kMnChunkBytes, &tma_a, &full_bar[stage], m0 + c * 64, k0);
          }
          if constexpr (BMAJ == K_MAJOR) {
            tma_load_2d(sb, &tma_b, &full_bar[stage], k0, n0);  // box {64 K, BN N}
          } else if (ep.mn3 & 2) {
            tma_load_3d(sb, &tma_b, &full_bar[stage], 0, k0, n0 / 64);  // box {64 N, 64 K, BN/64 chunks}
          } else {
#pragma unroll
            for (int c = 0; c < BN / 64; ++c)
              tma_load_2d(sb + c * kMnChunkBytes, &tma_b, &full_bar[stage], n0 + c * 64, k0);
          }
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    constexpr uint32_t idesc = make_idesc(BM, BN, AMAJ, BMAJ);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
#ifdef RWB_PAIR_EXPERIMENT
    const long long l0 = clock64();
#endif
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
#ifdef RWB_PAIR_EXPERIMENT
      const long long a0 = clock64();
#endif
      mbar_wait(&tempty_bar[acc], acc_phase ^ 1);  // epilogue drained this accumulator
#ifdef RWB_PAIR_EXPERIMENT
      if (lane == 0) g_pair_dbg[blockIdx.x][1] += clock64() - a0;
#endif
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + uint32_t(acc * BN);
      for (int kb = 0; kb < num_kb; ++kb) {
#ifdef RWB_PAIR_EXPERIMENT
        const long long f0 = clock64();
#endif
        mbar_wait(&full_bar[stage], phase);
#ifdef RWB_PAIR_EXPERIMENT
        if (lane == 0) g_pair_dbg[blockIdx.x][0] += clock64() - f0;
#endif
        tc_fence_after();
        if (lane == 0) {
          const uint32_t sa = smem_u32(smem + stage * C::kStageBytes);
          const uint32_t sb = sa + C::kABytes;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            // K-major: +32 B per 16-element K step inside the 128 B swizzle row
            // MN-major: +2 K-row groups (2 x 1024 B) per 16-element K step
            const uint64_t ad = AMAJ == K_MAJOR ? kmajor_desc(sa, k)
                                                : make_desc(sa + k * 2048, kMnChunkBytes, 1024);
            const uint64_t bd = BMAJ == K_MAJOR ? kmajor_desc(sb, k)
                                                : make_desc(sb + k * 2048, kMnChunkBytes, 1024);
            tc_mma(d_tmem, ad, bd, idesc, (kb | k) != 0 ? 1u : 0u);
          }
          tc_commit(&empty_bar[stage]);  // frees the smem stage when these MMAs finish
        }
        __syncwarp();
        if (++stage == S) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (lane == 0) tc_commit(&tfull_bar[acc]);  // accumulator ready for the epilogue
      __syncwarp();
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
#ifdef RWB_PAIR_EXPERIMENT
    if (lane == 0) g_pair_dbg[blockIdx.x][2] += clock64() - l0;
#endif
  } else if (warp >= kEpiWarp0) {
    // ===================== epilogue (warps 4..7 -> TMEM lanes 0..127) =====================
    const int ew = warp - kEpiWarp0;  // == warp % 4: TMEM lane quarter this warp may access
    uint8_t* ebuf = smem + S * C::kStageBytes + ew * 2 * kEpiBoxBytes;
    uint64_t* ebar = &epi_bar[ew * 2];
    uint32_t seq = 0;  // boxes this warp has staged so far (buffer = seq % 2)
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      int tm, tn;
      tile_coords(tile, tiles_m, tiles_n, kGroupM, tm, tn);
      const int m0 = tm * BM, n0 = tn * BN;
      const int row = m0 + ew * 32 + lane;
      const uint32_t tbase = tmem_base + (uint32_t(ew * 32) << 16) + uint32_t(acc * BN);
#ifdef RWB_PROBE_EPI_SKIP
      if (true) {  // probe only: release the accumulator without reading it
        mbar_wait(&tfull_bar[acc], acc_phase);
        tc_fence_after();
        if (lane == 0 && ep.tma_epi) mbar_arrive(&tempty_bar[acc]);
      } else
#endif
      if (ep.tma_epi) {
        if constexpr (epi_input(EPI)) {  // the tile's first input box overlaps the wait
          if (lane == 0) epi_first_input<2>(&tma_i, ebuf, ebar, seq, n0, m0 + ew * 32);
        }
        mbar_wait(&tfull_bar[acc], acc_phase);
        tc_fence_after();
        epilogue_tile_tma<BN, EPI, 2>(tbase, m0 + ew * 32, n0, M, N, ep, &tma_o, &tma_i, ebuf, ebar, seq, [&] {
          if (lane == 0) mbar_arrive(&tempty_bar[acc]);
        });
      } else {
        YChunk y0;
        if constexpr (uses_y(EPI)) load_y_chunk(ep, row, n0, M, N, y0);  // overlaps the wait
        mbar_wait(&tfull_bar[acc], acc_phase);
        tc_fence_after();
        epilogue_tile<BN, EPI>(tbase, row, n0, M, N, ep, &y0);
      }
      if (!ep.tma_epi) {  // (the TMA epilogue released the accumulator after its last TMEM load)
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty_bar[acc]);
      }
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
    if (ep.tma_epi && lane == 0) bulk_wait_all();  // the last stores have landed
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(C::kTmemCols));
  }
}

// ===================================================================================
// CTA-pair variant: tcgen05.mma.cta_group::2 with M = 256 per pair.  Each CTA
// of a (2,1,1) cluster loads its own 128 rows of A and HALF of the B tile
// (BN/2 rows) into the same smem offsets; the leader (rank 0) issues the MMAs
// for both, each CTA's TMEM receives its 128 accumulator rows.  Per SM the
// tensor core now reads 128x16 of A + (BN/2)x16 of B per instruction instead
// of 128x16 + BNx16, which relieves the shared-memory bandwidth that limits
// the single-CTA kernel.
// ===================================================================================
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa_rank0(uint32_t local_smem_addr) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(local_smem_addr));
  return r;
}
// Arrive on a barrier of another CTA of the cluster.  The accumulator-empty
// signal only orders this warp's completed TMEM loads (tcgen05.wait::ld +
// fence::before_thread_sync) before the peer's next MMAs: release at CTA
// scope (the default semantics) suffices -- a cluster-scope release compiles
// to MEMBAR.ALL.GPU + ERRBAR, which the epilogue warps measurably stall on
// (ncu source page, profiles/r02/README.md)
#ifndef RWB_ARRIVE_CLUSTER_RELEASE
#define RWB_ARRIVE_CLUSTER_RELEASE 0
#endif
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
#if RWB_ARRIVE_CLUSTER_RELEASE
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
#else
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
#endif
}
// TMA load into this CTA's smem, completion counted on the LEADER's barrier
__device__ __forceinline__ void tma_load_2d_2sm(void* dst, const CUtensorMap* map, uint32_t leader_bar, int c0,
                                                int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(leader_bar), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tc_mma2(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accum) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum)
      : "memory");
}
// arrive (once the issued MMAs complete) on the barrier at this offset in BOTH CTAs
__device__ __forceinline__ void tc_commit2_mc(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(uint16_t(3))
      : "memory");
}


// MH = 128-row halves per CTA.  MH = 1: the pair computes a 256 x BN tile
// (16 KB of A + 16 KB of B per CTA and k-block, 6 stages, two TMEM
// accumulators so the epilogue overlaps the next tile).  MH = 2: each CTA
// owns 256 rows, the pair a 512 x BN tile -- two MMAs per 16-deep K step
// share the B operand, so L2->SM bytes per FLOP drop by another quarter
// (32 KB A + 16 KB B per CTA and k-block, 4 stages); the two 256-column
// accumulators fill TMEM, so the epilogue no longer overlaps the MMAs.
template <int BN, int MH = 1>
struct Cfg2 {
  static constexpr int BNH = BN / 2;
  // MH = 2: eight epilogue warps, one group of four per row half, drain the
  // two accumulators concurrently (the MMAs wait for both); their staging
  // boxes take the smem of the fourth stage (3 stages measure as fast as 4)
#ifndef RWB_GEMM2_CQ
#define RWB_GEMM2_CQ 1
#endif
  static constexpr int kCQ = MH == 2 ? RWB_GEMM2_CQ : 1;  // column slices per half (warps per lane quarter)
  static constexpr int kEpiWarps = 4 * MH * kCQ;
  static constexpr int kThreads = 128 + 32 * kEpiWarps;
  // sixteen epilogue warps (kCQ = 2) stage one box each, so three stages still fit
#ifndef RWB_GEMM2_EPIBUFS
#define RWB_GEMM2_EPIBUFS (RWB_GEMM2_CQ == 2 ? 1 : 2)
#endif
  static constexpr int kEpiBufs = MH == 2 ? RWB_GEMM2_EPIBUFS : 2;
  static constexpr uint32_t kEpiSmemT = kEpiWarps * kEpiBufs * kEpiBoxBytes;
#ifdef RWB_GEMM2_STAGES
  static constexpr int kStages = RWB_GEMM2_STAGES;
#else
  static constexpr int kStages = (MH == 1 ? 6 : (kEpiWarps * kEpiBufs <= 16 ? 3 : 2)) * (64 / BK);
#endif
  static constexpr uint32_t kHalfBytes = BM * BK * 2;      // 16 KB: 128 rows of A
  static constexpr uint32_t kABytes = MH * kHalfBytes;     // this CTA's MH x 128 rows
  static constexpr uint32_t kBBytes = BNH * BK * 2;        // 16 KB: half of the B tile
  static constexpr uint32_t kStageBytes = kABytes + kBBytes;
  static constexpr int kNAcc = MH == 1 ? 2 : 1;            // accumulator stages in TMEM
  static constexpr uint32_t kTmemCols = kNAcc * MH * BN;   // 512 either way
#ifndef RWB_GEMM2_SBIAS
#define RWB_GEMM2_SBIAS 1
#endif
  // per-warp bias columns (the wide kernel has the smem; MH = 1 uses six stages)
  static constexpr uint32_t kBiasSmem = (RWB_GEMM2_SBIAS && MH == 2) ? kEpiWarps * (BN / kCQ) * 4 : 0;
  static constexpr size_t kSmem = size_t(kStages) * kStageBytes + kEpiSmemT + kBiasSmem + 1024;
};

template <int BN, int AMAJ, int BMAJ, int EPI, int MH = 1>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(Cfg2<BN, MH>::kThreads, 1)
    umma_gemm2_kernel(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
                      const __grid_constant__ CUtensorMap tma_o, const __grid_constant__ CUtensorMap tma_i,
                      int M, int N, int K, EpiArgs ep) {
  using C = Cfg2<BN, MH>;
  constexpr int S = C::kStages;
  constexpr int BNH = C::BNH;
  constexpr int NACC = C::kNAcc;
  constexpr int PM = 2 * MH * BM;  // rows per CTA pair
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full_bar[S], empty_bar[S], tfull_bar[2], tempty_bar[2], epi_bar[2 * C::kEpiWarps];
  __shared__ uint32_t tmem_base_sh;

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int tiles_m = (M + PM - 1) / PM, tiles_n = (N + BN - 1) / BN;
  const int num_tiles = tiles_m * tiles_n;
  const int num_kb = (K + BK - 1) / BK;
  const int cid = blockIdx.x / 2, ncl = gridDim.x / 2;

  if (threadIdx.x == 0) {
    prefetch_tmap(&tma_a);
    prefetch_tmap(&tma_b);
    for (int i = 0; i < S; ++i) {
      mbar_init(&full_bar[i], 1);  // the leader's expect_tx arrive (bytes of BOTH CTAs' loads)
      mbar_init(&empty_bar[i], 1);
    }
    for (int i = 0; i < NACC; ++i) {
      mbar_init(&tfull_bar[i], 1);
      mbar_init(&tempty_bar[i], 2 * C::kEpiWarps);  // every epilogue warp of both CTAs (leader's copy is used)
    }
    for (int i = 0; i < 2 * C::kEpiWarps; ++i) mbar_init(&epi_bar[i], 1);
    if (ep.tma_epi) {
      prefetch_tmap(&tma_o);
      if (epi_input(EPI)) prefetch_tmap(&tma_i);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base_sh)),
                 "r"(C::kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_sh;

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = cid; tile < num_tiles; tile += ncl) {
        int tm, tn;
      tile_coords(tile, tiles_m, tiles_n, group_tiles2<MH>(), tm, tn);
        const int m0 = tm * PM + int(rank) * MH * BM;  // this CTA's A rows
        const int nb0 = tn * BN + int(rank) * BNH;   // this CTA's half of B
        for (int kb = 0; kb < num_kb; ++kb) {
#ifdef RWB_PAIR_EXPERIMENT
          const long long w0 = clock64();
#endif
          mbar_wait(&empty_bar[stage], phase ^ 1);
#ifdef RWB_PAIR_EXPERIMENT
          g_pair_dbg[blockIdx.x][3] += clock64() - w0;
#endif
          uint8_t* sa = smem + stage * C::kStageBytes;
          uint8_t* sb = sa + C::kABytes;
          const uint32_t fb = smem_u32(&full_bar[stage]);
#if defined(RWB_PAIR_EXPERIMENT) && RWB_PAIR_EXPERIMENT == 2
          // no data movement after the first fill: timing of MMA + sync only
          if (tile != cid || kb >= S) {
            if (leader) mbar_arrive(&full_bar[stage]);
            if (++stage == S) {
              stage = 0;
              phase ^= 1;
            }
            continue;
          }
#endif
          // only the leader arrives (with both CTAs' byte count); the peer's
          // TMA completes its bytes on the leader's barrier directly
          if (leader) mbar_expect_tx(&full_bar[stage], 2 * C::kStageBytes);
          const uint32_t lbar = fb & 0xFEFFFFFFu;  // the leader's barrier
          const int k0 = kb * BK;
          if constexpr (AMAJ == K_MAJOR) {
            tma_load_2d_2sm(sa, &tma_a, lbar, k0, m0);
          } else {
#pragma unroll
            for (int c = 0; c < MH * BM / 64; ++c)
              tma_load_2d_2sm(sa + c * kMnChunkBytes, &tma_a, lbar, m0 + c * 64, k0);
          }
          if constexpr (BMAJ == K_MAJOR) {
            tma_load_2d_2sm(sb, &tma_b, lbar, k0, nb0);
          } else {
#pragma unroll
            for (int c = 0; c < BNH / 64; ++c) tma_load_2d_2sm(sb + c * kMnChunkBytes, &tma_b, lbar, nb0 + c * 64, k0);
          }
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (leader CTA only) =====================
    if (leader) {
      constexpr uint32_t idesc = make_idesc(2 * BM, BN, AMAJ, BMAJ);  // M = 256 per pair instruction
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
#ifdef RWB_PAIR_EXPERIMENT
      const long long l0 = clock64();
#endif
      for (int tile = cid; tile < num_tiles; tile += ncl) {
#ifdef RWB_PAIR_EXPERIMENT
        const long long a0 = clock64();
#endif
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
#ifdef RWB_PAIR_EXPERIMENT
        if (lane == 0) g_pair_dbg[blockIdx.x][1] += clock64() - a0;
#endif
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + uint32_t(acc * MH * BN);
        for (int kb = 0; kb < num_kb; ++kb) {
#ifdef RWB_PAIR_EXPERIMENT
          const long long f0 = clock64();
#endif
          mbar_wait(&full_bar[stage], phase);
#ifdef RWB_PAIR_EXPERIMENT
          if (lane == 0) g_pair_dbg[blockIdx.x][0] += clock64() - f0;
#endif
          tc_fence_after();
          if (lane == 0) {
            const uint32_t sa = smem_u32(smem + stage * C::kStageBytes);
            const uint32_t sb = sa + C::kABytes;
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) {
              const uint64_t bd = BMAJ == K_MAJOR ? kmajor_desc(sb, k)
                                                  : make_desc(sb + k * 2048, kMnChunkBytes, 1024);
#pragma unroll
              for (int h = 0; h < MH; ++h) {  // the row halves share the B operand
                const uint32_t sah = sa + uint32_t(h) * C::kHalfBytes;
                const uint64_t ad = AMAJ == K_MAJOR ? kmajor_desc(sah, k)
                                                    : make_desc(sah + k * 2048, kMnChunkBytes, 1024);
                tc_mma2(d_tmem + uint32_t(h * BN), ad, bd, idesc, (kb | k) != 0 ? 1u : 0u);
              }
            }
            tc_commit2_mc(&empty_bar[stage]);  // frees this stage in BOTH CTAs
          }
          __syncwarp();
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (lane == 0) tc_commit2_mc(&tfull_bar[acc]);
        __syncwarp();
        if (++acc == NACC) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
#ifdef RWB_PAIR_EXPERIMENT
      if (lane == 0) g_pair_dbg[blockIdx.x][2] += clock64() - l0;
#endif
    }
  } else if (warp >= kEpiWarp0) {
    // ===================== epilogue (both CTAs, own rows) =====================
    const int ewg = warp - kEpiWarp0;   // epilogue warp index
    const int ew = ewg & 3;             // TMEM lane quarter (== warp % 4)
    const int hw = (ewg >> 2) % MH;     // MH = 2: the row half this warp drains
    const int cq = (ewg >> 2) / MH;     // its column slice of the half (kCQ slices)
    constexpr int BNQ = BN / C::kCQ;
    const uint32_t tempty_leader = mapa_rank0(smem_u32(&tempty_bar[0]));
    uint8_t* ebuf = smem + S * C::kStageBytes + ewg * C::kEpiBufs * kEpiBoxBytes;
    uint64_t* ebar = &epi_bar[ewg * 2];
    uint32_t seq = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = cid; tile < num_tiles; tile += ncl) {
      int tm, tn;
      tile_coords(tile, tiles_m, tiles_n, group_tiles2<MH>(), tm, tn);
#pragma unroll 1
      for (int h = hw; h < hw + 1; ++h) {  // this warp's row half (accumulator h)
        const int r0 = tm * PM + int(rank) * MH * BM + h * BM + ew * 32;
        const int row = r0 + lane;
        const int c0 = tn * BN + cq * BNQ;
        const uint32_t tbase = tmem_base + (uint32_t(ew * 32) << 16) + uint32_t((acc * MH + h) * BN + cq * BNQ);
        if (ep.tma_epi) {
          if constexpr (epi_input(EPI)) {
            if (lane == 0) epi_first_input<C::kEpiBufs>(&tma_i, ebuf, ebar, seq, c0, r0);
          }
          float* sbias = nullptr;
          if constexpr (EPI == EPI_BIAS_TANH_BF16 && C::kBiasSmem > 0) {
            sbias = reinterpret_cast<float*>(smem + S * C::kStageBytes + C::kEpiSmemT) + ewg * BNQ;
            stage_bias<BNQ>(sbias, ep.bias, c0, N);
          }
          mbar_wait(&tfull_bar[acc], acc_phase);
          tc_fence_after();
          epilogue_tile_tma<BNQ, EPI, C::kEpiBufs>(tbase, r0, c0, M, N, ep, &tma_o, &tma_i, ebuf, ebar, seq, [&] {
            if (lane == 0) mbar_arrive_cluster(tempty_leader + uint32_t(acc) * 8u);
          }, sbias);
        } else {
          YChunk y0;
          if constexpr (uses_y(EPI)) load_y_chunk(ep, row, c0, M, N, y0);
          mbar_wait(&tfull_bar[acc], acc_phase);
          tc_fence_after();
          epilogue_tile<BNQ, EPI>(tbase, row, c0, M, N, ep, &y0);
        }
      }
      if (!ep.tma_epi) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(tempty_leader + uint32_t(acc) * 8u);
      }
      if (++acc == NACC) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
    if (ep.tma_epi && lane == 0) bulk_wait_all();
  }
  __syncthreads();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(C::kTmemCols));
  }
}

}  // namespace gemm
}  // namespace rwb
