// CRC32 (IEEE 802.3, reflected, poly 0xEDB88320, init/xorout 0xFFFFFFFF) of a
// device buffer — the per-record payload checksum of the log format
// (wire.cpp:31-38), computed on the GPU so the logging capture
// path never touches payload bytes on the CPU.
//
// CRC is affine over GF(2): with raw(M) the register after processing M from
// state 0 and S^n the linear map "advance the register through n zero bytes",
//   raw(A || B) = S^|B|(raw(A)) ^ raw(B),   crc(M) = ~(S^|M|(~0) ^ raw(M)).
// Level 1 (crc_chunks_kernel): 64 KB chunks, lane pieces of 128 bytes read
// with 256-bit loads, slice-by-4 bank-sliced smem tables, shuffle + smem fold.
// Level 2 (crc_final_kernel): one CTA folds the unit raws and the tail as
// trees and applies the init/xorout conditioning.  Operators are 32x32 GF(2)
// matrices (32 uint32 columns) built on the host, applied on the device by
// bit loop or through byte tables.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <mutex>
#include <vector>

#include "internal.h"

namespace rwb {
namespace {

constexpr uint32_t kPiece = 128;                        // bytes per lane
constexpr uint32_t kChunk = 65536;                      // bytes per chunk (16 warps)
constexpr int kWarpsPerChunk = int(kChunk / (kPiece * 32));  // 16
constexpr int kLevels = 9;                              // S^(128 * 2^l): 5 in-warp + 4 across warps
constexpr int kChunkThreads = 1024;                     // 2 chunks per CTA pass
constexpr int kChunksPerPass = kChunkThreads / 32 / kWarpsPerChunk;
constexpr int kFinThreads = 256;
constexpr int kFinLevels = 8;                           // log2(256)
constexpr uint32_t kTailPiece = kChunk / kFinThreads;   // 256 bytes per thread of the tail

struct Mat {
  uint32_t c[32];
};

__host__ __device__ inline uint32_t mat_apply(const Mat& m, uint32_t v) {
  uint32_t r = 0;
#pragma unroll
  for (int i = 0; i < 32; ++i)
    if (v & (1u << i)) r ^= m.c[i];
  return r;
}
__host__ __device__ inline Mat mat_mul(const Mat& a, const Mat& b) {  // a o b
  Mat r;
  for (int i = 0; i < 32; ++i) r.c[i] = mat_apply(a, b.c[i]);
  return r;
}
__host__ __device__ inline Mat mat_identity() {
  Mat r;
  for (int i = 0; i < 32; ++i) r.c[i] = 1u << i;
  return r;
}
// S^(8 bits): one zero byte through the reflected register
__host__ __device__ inline uint32_t crc_table_entry(uint32_t i) {
  uint32_t c = i;
  for (int k = 0; k < 8; ++k) c = (c & 1u) ? 0xEDB88320u ^ (c >> 1) : (c >> 1);
  return c;
}
__host__ __device__ inline Mat op_one_byte() {
  Mat m;
  for (int i = 0; i < 32; ++i) {
    const uint32_t v = 1u << i;
    m.c[i] = crc_table_entry(v & 0xFFu) ^ (v >> 8);
  }
  return m;
}
__host__ __device__ inline Mat op_pow(Mat base, uint64_t n) {  // S^n
  Mat r = mat_identity();
  while (n) {
    if (n & 1) r = mat_mul(base, r);
    base = mat_mul(base, base);
    n >>= 1;
  }
  return r;
}

struct TreeOps {
  Mat op[kLevels];  // S^(128 * 2^l)
};

// Level 1, persistent: one 1024-thread CTA per SM, two 64 KB chunks per pass
// (16 warps per chunk; lane L of warp w owns the 128-byte piece 32 w + L).
// A lane reads its piece straight from global memory with four 256-bit loads
// (LDG.256), all issued before the first lookup.  The slice-by-4 tables are BANK-SLICED: entry b of
// table k for lane L sits at word (k * 256 + b) * 32 + L, i.e. in bank L, so
// a warp's 32 random lookups never conflict (a shared 256-entry table costs
// ~3.5 wavefronts per lookup): 128 KB.  The pieces fold into the chunk's raw
// CRC with S^(128 * 2^l) applied through byte tables (4 lookups each):
// levels 0-4 by warp shuffles, 5-8 across the chunk's 16 warps.
constexpr uint32_t kSliceWords = 4 * 256 * 32;
constexpr uint32_t kOpWords = kLevels * 4 * 256;
constexpr uint32_t kChunkSmem = (kSliceWords + kOpWords + kChunkThreads / 32) * 4;

__device__ __forceinline__ uint32_t op_apply_tab(const uint32_t* ot, uint32_t v) {
  return ot[v & 0xFFu] ^ ot[256 + ((v >> 8) & 0xFFu)] ^ ot[512 + ((v >> 16) & 0xFFu)] ^ ot[768 + (v >> 24)];
}
// byte tables of an operator: ot[j * 256 + b] = m(b << 8j)
__device__ __forceinline__ uint32_t op_tab_entry(const Mat& m, uint32_t i) {
  const uint32_t j = i >> 8, b = i & 0xFFu;
  uint32_t r = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q)
    if (b & (1u << q)) r ^= m.c[8 * j + q];
  return r;
}

template <bool ALIGNED32>
__global__ void __launch_bounds__(kChunkThreads, 1) crc_chunks_kernel(const uint8_t* __restrict__ data, uint64_t nchunks,
                                                                      TreeOps ops, uint32_t* __restrict__ chunk_raw,
                                                                      uint32_t zero) {
  extern __shared__ __align__(16) uint32_t sm[];
  uint32_t* slice = sm;                  // [4][256][32]
  uint32_t* optab = sm + kSliceWords;    // [kLevels][4][256]
  uint32_t* wraw = optab + kOpWords;     // [warps]
  const uint32_t t = threadIdx.x, lane = t & 31u, warp = t >> 5;
  // tables: the 1024 distinct entries once (table k = k extra zero bytes),
  // staged in the first 4 KB of the op-table area, then replicated per bank
  // (conflict-free stores: lane L writes bank L)
  for (uint32_t i = t; i < 256u; i += kChunkThreads) {
    uint32_t e = crc_table_entry(i);
    optab[i] = e;
#pragma unroll
    for (int k = 1; k < 4; ++k) {
      e = (e >> 8) ^ crc_table_entry(e & 0xFFu);
      optab[k * 256 + i] = e;
    }
  }
  __syncthreads();
  for (uint32_t i = warp; i < 4u * 256u; i += kChunkThreads / 32) slice[i * 32u + lane] = optab[i];
  __syncthreads();
  for (uint32_t i = t; i < kOpWords; i += kChunkThreads) optab[i] = op_tab_entry(ops.op[i >> 10], i & 1023u);
  __syncthreads();
  const uint32_t* tl = slice + lane;
  const uint32_t wic = warp % kWarpsPerChunk, cip = warp / kWarpsPerChunk;
  const uint64_t passes = (nchunks + kChunksPerPass - 1) / kChunksPerPass;
  for (uint64_t pass = blockIdx.x; pass < passes; pass += gridDim.x) {
    const uint64_t chunk = pass * kChunksPerPass + cip;
    uint32_t c = 0;
    if (chunk < nchunks) {
      const uint8_t* piece = data + chunk * kChunk + (uint64_t(wic) * 32u + lane) * kPiece;
      uint32_t w[kPiece / 4];
#pragma unroll
      for (int s = 0; s < int(kPiece / 32); ++s) {
        uint32_t* r = w + 8 * s;
        if constexpr (ALIGNED32) {
          asm("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
              : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
              : "l"(piece + 32 * s));
        } else {  // any alignment: bytes (records are 256 B aligned in practice)
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const uint8_t* b = piece + 32 * s + 4 * k;
            r[k] = uint32_t(b[0]) | (uint32_t(b[1]) << 8) | (uint32_t(b[2]) << 16) | (uint32_t(b[3]) << 24);
          }
        }
      }
      // every load in flight before the first lookup: ptxas otherwise sinks each
      // load to its first use (one 32-byte load in flight per lane); `zero` (a
      // kernel argument, always 0) makes the first word depend on all of them
      uint32_t dep = 0;
#pragma unroll
      for (int s = 1; s < int(kPiece / 32); ++s) dep |= w[8 * s];
      c = w[0] ^ (dep & zero);
      c = tl[(3 * 256 + (c & 0xFFu)) << 5] ^ tl[(2 * 256 + ((c >> 8) & 0xFFu)) << 5] ^
          tl[(256 + ((c >> 16) & 0xFFu)) << 5] ^ tl[(c >> 24) << 5];
#pragma unroll
      for (int k = 1; k < int(kPiece / 4); ++k) {  // 4 bytes per step, little-endian byte order
        c ^= w[k];
        c = tl[(3 * 256 + (c & 0xFFu)) << 5] ^ tl[(2 * 256 + ((c >> 8) & 0xFFu)) << 5] ^
            tl[(256 + ((c >> 16) & 0xFFu)) << 5] ^ tl[(c >> 24) << 5];
      }
    }
    // level l pairs runs of 2^l pieces: left' = S^(128 * 2^l)(left) ^ right
#pragma unroll
    for (int l = 0; l < 5; ++l) {
      const uint32_t o = __shfl_down_sync(0xFFFFFFFFu, c, 1u << l);
      const uint32_t f = op_apply_tab(optab + l * 1024, c) ^ o;
      if ((lane & ((2u << l) - 1u)) == 0) c = f;
    }
    if (lane == 0) wraw[warp] = c;
    __syncthreads();
    if (wic == 0) {  // the chunk's 16 warp raws, levels 5..8
      uint32_t v = lane < uint32_t(kWarpsPerChunk) ? wraw[warp + lane] : 0u;
#pragma unroll
      for (int l = 5; l < kLevels; ++l) {
        const uint32_t o = __shfl_down_sync(0xFFFFFFFFu, v, 1u << (l - 5));
        const uint32_t f = op_apply_tab(optab + l * 1024, v) ^ o;
        if ((lane & ((2u << (l - 5)) - 1u)) == 0) v = f;
      }
      if (lane == 0 && chunk < nchunks) chunk_raw[chunk] = v;
    }
    __syncthreads();
  }
}

// Level 2, one CTA, as trees (no serial chain):
// (1) the chunk raws, front-padded with virtual zero chunks to 256 x per
//     (raw(0^k || M) = raw(M): leading zeros are free): thread t loads its
//     `per` consecutive raws, folds them with S^65536, then an 8-level tree
//     with S^(per * 64 KB * 2^l);
// (2) the tail (< 64 KB) as one front-padded virtual chunk: thread t's
//     256-byte piece by table, then the 8-level S^(256 * 2^l) tree;
// (3) raw = S^|tail|(chunks) ^ tail, crc = ~(S^n(~0) ^ raw).
// Operators depend on n only: precomputed on the host, cached per n.
struct FinalOps {
  Mat unit;                  // S^65536
  Mat range[kFinLevels];     // S^(per * 65536 * 2^l)
  Mat tailtree[kFinLevels];  // S^(256 * 2^l)
  Mat tail;                  // S^|tail|
  Mat total;                 // S^n
};
__global__ void __launch_bounds__(kFinThreads) crc_final_kernel(const uint8_t* __restrict__ data, uint64_t n,
                                                                uint64_t nchunks, uint64_t per,
                                                                const uint32_t* __restrict__ chunk_raw, FinalOps ops,
                                                                uint32_t* out) {
  __shared__ uint32_t table[256];
  __shared__ uint32_t utab[1024];
  __shared__ uint32_t rng[kFinThreads];
  __shared__ uint32_t part[kFinThreads];
  const uint32_t t = threadIdx.x;
  table[t] = crc_table_entry(t);
  for (uint32_t i = t; i < 1024u; i += kFinThreads) utab[i] = op_tab_entry(ops.unit, i);
  __syncthreads();
  {
    const uint64_t pad = uint64_t(kFinThreads) * per - nchunks;  // virtual zero chunks in front
    uint32_t r = 0;
    constexpr int kBatch = 16;  // independent loads in flight, then the dependent fold
    for (uint64_t v0 = uint64_t(t) * per; v0 < uint64_t(t + 1) * per; v0 += kBatch) {
      uint32_t x[kBatch];
#pragma unroll
      for (int j = 0; j < kBatch; ++j) {
        const uint64_t v = v0 + j;
        x[j] = (v < uint64_t(t + 1) * per && v >= pad) ? chunk_raw[v - pad] : 0u;
      }
#pragma unroll
      for (int j = 0; j < kBatch; ++j)
        if (v0 + j < uint64_t(t + 1) * per && v0 + j >= pad) r = op_apply_tab(utab, r) ^ x[j];
    }
    rng[t] = r;
  }
  const uint64_t tail0 = nchunks * kChunk;
  const uint32_t start = kChunk - static_cast<uint32_t>(n - tail0);  // first real byte of the virtual tail chunk
  {
    uint32_t c = 0;
    const uint32_t b0 = t * kTailPiece;
    for (uint32_t i = (b0 > start ? b0 : start); i < b0 + kTailPiece; ++i)
      c = table[(c ^ data[tail0 + (i - start)]) & 0xFFu] ^ (c >> 8);
    part[t] = c;
  }
  __syncthreads();
  for (int l = 0; l < kFinLevels; ++l) {  // both trees, level by level
    const uint32_t stride = 1u << l;
    if ((t & ((stride << 1) - 1)) == 0) {
      rng[t] = mat_apply(ops.range[l], rng[t]) ^ rng[t + stride];
      part[t] = mat_apply(ops.tailtree[l], part[t]) ^ part[t + stride];
    }
    __syncthreads();
  }
  if (t == 0) *out = ~(mat_apply(ops.total, 0xFFFFFFFFu) ^ mat_apply(ops.tail, rng[0]) ^ part[0]);
}

struct CrcOps {
  TreeOps tree;
  Mat pow2[48];  // S^(2^k bytes)
};
CrcOps make_crc_ops() {
  CrcOps ops;
  const Mat b = op_one_byte();
  for (int l = 0; l < kLevels; ++l) ops.tree.op[l] = op_pow(b, uint64_t(kPiece) << l);
  ops.pow2[0] = b;
  for (int k = 1; k < 48; ++k) ops.pow2[k] = mat_mul(ops.pow2[k - 1], ops.pow2[k - 1]);
  return ops;
}
const CrcOps& crc_ops() {
  static const CrcOps ops = make_crc_ops();  // thread-safe one-time init
  return ops;
}
// S^n from the power-of-two table: <= 48 products of 32x32 GF(2) matrices
Mat op_pow_fast(uint64_t n) {
  const CrcOps& ops = crc_ops();
  Mat r = mat_identity();
  for (int k = 0; n; ++k, n >>= 1)
    if (n & 1) r = mat_mul(ops.pow2[k], r);
  return r;
}

}  // namespace

// scratch: >= crc32_scratch_words(n) uint32 device words
int launch_crc32(const void* data, uint64_t n, uint32_t* out_dev, uint32_t* scratch, void* stream) {
  auto st = static_cast<cudaStream_t>(stream);
  const CrcOps& ops = crc_ops();
  const uint64_t nchunks = n / kChunk;
  static DeviceOnce once;
  static int num_sms = 0;
  const int se = once.run([](int dev) {
    cudaError_t e = cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(crc_chunks_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(kChunkSmem));
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(crc_chunks_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(kChunkSmem));
    return static_cast<int>(e);
  });
  if (se) return se;
  if (nchunks) {
    const uint64_t passes = (nchunks + kChunksPerPass - 1) / kChunksPerPass;
    const unsigned grid = static_cast<unsigned>(passes < uint64_t(num_sms) ? passes : uint64_t(num_sms));
    // 256-bit loads need 32-byte aligned pieces (records are cudaMalloc'd or
    // pool-allocated, 256 B aligned); any other address takes the byte-load variant
    auto* d8 = static_cast<const uint8_t*>(data);
    if ((reinterpret_cast<uintptr_t>(data) & 31u) == 0)
      crc_chunks_kernel<true><<<grid, kChunkThreads, kChunkSmem, st>>>(d8, nchunks, ops.tree, scratch, 0u);
    else
      crc_chunks_kernel<false><<<grid, kChunkThreads, kChunkSmem, st>>>(d8, nchunks, ops.tree, scratch, 0u);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return static_cast<int>(e);
  }
  const uint64_t per = (nchunks + kFinThreads - 1) / kFinThreads;
  // the operators depend on n only: one cached set per length (records repeat their size)
  static std::mutex mu;
  static uint64_t cached_n = ~uint64_t(0);
  static FinalOps cached;
  FinalOps fo;
  {
    std::lock_guard<std::mutex> lk(mu);
    if (cached_n != n) {
      cached.unit = op_pow_fast(kChunk);
      Mat r = op_pow_fast(per * kChunk), q = op_pow_fast(kTailPiece);
      for (int l = 0; l < kFinLevels; ++l) {
        cached.range[l] = r;
        cached.tailtree[l] = q;
        r = mat_mul(r, r);
        q = mat_mul(q, q);
      }
      cached.tail = op_pow_fast(n - nchunks * kChunk);
      cached.total = op_pow_fast(n);
      cached_n = n;
    }
    fo = cached;
  }
  crc_final_kernel<<<1, kFinThreads, 0, st>>>(static_cast<const uint8_t*>(data), n, nchunks, per, scratch, fo,
                                               out_dev);
  return static_cast<int>(cudaGetLastError());
}

uint64_t crc32_scratch_words(uint64_t n) { return n / kChunk + 1; }

}  // namespace rwb
