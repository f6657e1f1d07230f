// CRC32 (IEEE 802.3, reflected, poly 0xEDB88320, init/xorout 0xFFFFFFFF) of a
// device buffer — the per-record payload checksum of the log format
// (wire.cpp:31-38), computed on the GPU so the logging capture
// path never touches payload bytes on the CPU.
//
// CRC is affine over GF(2): with raw(M) the register after processing M from
// state 0 and S^n the linear map "advance the register through n zero bytes",
//   raw(A || B) = S^|B|(raw(A)) ^ raw(B),   crc(M) = ~(S^|M|(~0) ^ raw(M)).
// Level 1: each CTA stages a 64 KB chunk in smem (coalesced 16-byte loads),
// 256 threads compute raw CRCs of 256-byte pieces with a smem table, and the
// pieces are folded with a log-depth tree using S^256, S^512, ... operators.
// Level 2: one thread folds the chunk CRCs with S^65536 and the tail, and
// applies the init/xorout conditioning.  Operators are 32x32 GF(2) matrices
// (32 uint32 columns) built on the host.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <vector>

#include "internal.h"

namespace rwb {
namespace {

constexpr int kCrcThreads = 256;
constexpr uint32_t kPiece = 256;                      // bytes per thread
constexpr uint32_t kChunk = kPiece * kCrcThreads;     // 64 KB per CTA
constexpr int kLevels = 8;                            // log2(256) tree levels

struct Mat {
  uint32_t c[32];
};
struct TreeOps {
  Mat op[kLevels];  // S^(256 * 2^l)
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

__global__ void __launch_bounds__(kCrcThreads) crc_chunks_kernel(const uint8_t* __restrict__ data, uint64_t n,
                                                                 TreeOps ops, uint32_t* __restrict__ chunk_raw) {
  __shared__ uint32_t table[256];
  extern __shared__ __align__(16) uint8_t buf[];  // kChunk bytes (dynamic, opt-in > 48 KB)
  __shared__ uint32_t part[kCrcThreads];
  const uint32_t t = threadIdx.x;
  table[t] = crc_table_entry(t);
  const uint64_t base = uint64_t(blockIdx.x) * kChunk;  // full chunks only
  const uint4* src = reinterpret_cast<const uint4*>(data + base);
  const bool aligned16 = (reinterpret_cast<uintptr_t>(data) & 15u) == 0;
  if (aligned16) {
#pragma unroll 4
    for (uint32_t i = t; i < kChunk / 16; i += kCrcThreads) reinterpret_cast<uint4*>(buf)[i] = __ldg(src + i);
  } else {
    for (uint32_t i = t; i < kChunk; i += kCrcThreads) buf[i] = data[base + i];
  }
  __syncthreads();
  uint32_t c = 0;
  const uint8_t* p = buf + t * kPiece;
#pragma unroll 8
  for (uint32_t i = 0; i < kPiece; ++i) c = table[(c ^ p[i]) & 0xFFu] ^ (c >> 8);
  part[t] = c;
  __syncthreads();
  // tree fold: at level l, piece pairs of 256*2^l bytes: left' = S^len(right)(left) ^ right
  for (int l = 0; l < kLevels; ++l) {
    const uint32_t stride = 1u << l;
    if ((t & ((stride << 1) - 1)) == 0) part[t] = mat_apply(ops.op[l], part[t]) ^ part[t + stride];
    __syncthreads();
  }
  if (t == 0) chunk_raw[blockIdx.x] = part[0];
  (void)n;
}

// one CTA: pieces of the tail (< 64 KB) in parallel, then thread 0 folds the
// chunk CRCs and the tail pieces in order and applies the conditioning.
__global__ void __launch_bounds__(kCrcThreads) crc_final_kernel(const uint8_t* __restrict__ data, uint64_t n,
                                                                uint64_t nchunks, const uint32_t* __restrict__ chunk_raw,
                                                                Mat s_chunk, Mat s_piece, uint32_t* out) {
  __shared__ uint32_t table[256];
  __shared__ uint32_t part[kCrcThreads];
  const uint32_t t = threadIdx.x;
  table[t] = crc_table_entry(t);
  __syncthreads();
  const uint64_t tail0 = nchunks * kChunk;
  const uint64_t tail = n - tail0;  // < kChunk
  const uint64_t b0 = tail0 + uint64_t(t) * kPiece;
  uint32_t c = 0;
  for (uint64_t i = b0; i < b0 + kPiece && i < n; ++i) c = table[(c ^ data[i]) & 0xFFu] ^ (c >> 8);
  part[t] = c;
  __syncthreads();
  if (t != 0) return;
  uint32_t r = 0;
  for (uint64_t i = 0; i < nchunks; ++i) r = mat_apply(s_chunk, r) ^ chunk_raw[i];
  const uint32_t npieces = static_cast<uint32_t>((tail + kPiece - 1) / kPiece);
  for (uint32_t i = 0; i < npieces; ++i) {
    const uint64_t len = (i + 1 == npieces) ? tail - uint64_t(i) * kPiece : kPiece;
    const Mat s = len == kPiece ? s_piece : op_pow(op_one_byte(), len);
    r = mat_apply(s, r) ^ part[i];
  }
  const Mat sn = op_pow(op_one_byte(), n);
  *out = ~(mat_apply(sn, 0xFFFFFFFFu) ^ r);
}

struct CrcOps {
  TreeOps tree;
  Mat chunk;
};
CrcOps make_crc_ops() {
  CrcOps ops;
  const Mat b = op_one_byte();
  for (int l = 0; l < kLevels; ++l) ops.tree.op[l] = op_pow(b, uint64_t(kPiece) << l);
  ops.chunk = op_pow(b, kChunk);
  return ops;
}
const CrcOps& crc_ops() {
  static const CrcOps ops = make_crc_ops();  // thread-safe one-time init
  return ops;
}

}  // namespace

// scratch: >= max(1, n / 64 KB) uint32 device words
int launch_crc32(const void* data, uint64_t n, uint32_t* out_dev, uint32_t* scratch, void* stream) {
  auto st = static_cast<cudaStream_t>(stream);
  const CrcOps& ops = crc_ops();
  const uint64_t nchunks = n / kChunk;
  static unsigned long long dev_mask = 0;
  if (first_on_device(dev_mask)) {
    const cudaError_t e = cudaFuncSetAttribute(crc_chunks_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               static_cast<int>(kChunk));
    if (e != cudaSuccess) return static_cast<int>(e);
  }
  if (nchunks) {
    crc_chunks_kernel<<<static_cast<unsigned>(nchunks), kCrcThreads, kChunk, st>>>(
        static_cast<const uint8_t*>(data), n, ops.tree, scratch);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return static_cast<int>(e);
  }
  crc_final_kernel<<<1, kCrcThreads, 0, st>>>(static_cast<const uint8_t*>(data), n, nchunks, scratch, ops.chunk,
                                              ops.tree.op[0], out_dev);
  return static_cast<int>(cudaGetLastError());
}

uint64_t crc32_scratch_words(uint64_t n) { return n / kChunk + 1; }

}  // namespace rwb
