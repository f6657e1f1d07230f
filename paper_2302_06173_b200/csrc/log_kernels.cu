// CRC32 (IEEE 802.3, reflected, poly 0xEDB88320, init/xorout 0xFFFFFFFF) of a
// device buffer — the per-record payload checksum of the log format
// (wire.cpp:31-38), computed on the GPU so the logging capture
// path never touches payload bytes on the CPU.
//
// CRC is affine over GF(2): with raw(M) the register after processing M from
// state 0 and S^n the linear map "advance the register through n zero bytes",
//   raw(A || B) = S^|B|(raw(A)) ^ raw(B),   crc(M) = ~(S^|M|(~0) ^ raw(M)).
// Level 1: each CTA stages a 64 KB chunk in smem (coalesced 16-byte loads, one
// padding word per 256-byte piece against bank conflicts), 256 threads compute
// raw CRCs of 256-byte pieces 4 bytes at a time (slice-by-4 smem tables), and the
// pieces are folded with a log-depth tree using S^256, S^512, ... operators.
// Level 2: one thread folds the chunk CRCs with S^65536 and the tail, and
// applies the init/xorout conditioning.  Operators are 32x32 GF(2) matrices
// (32 uint32 columns) built on the host.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <mutex>
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

// smem layout of a staged chunk: piece t (256 bytes) at word t * kPieceWords,
// one padding word per piece, so that thread t reading word k of its piece
// hits bank (t + k) % 32 -- conflict free (an unpadded 256-byte stride puts
// all 32 lanes in one bank)
constexpr uint32_t kPieceWords = kPiece / 4 + 1;
constexpr uint32_t kChunkSmem = kCrcThreads * kPieceWords * 4;

__global__ void __launch_bounds__(kCrcThreads) crc_chunks_kernel(const uint8_t* __restrict__ data, uint64_t n,
                                                                 TreeOps ops, uint32_t* __restrict__ chunk_raw) {
  __shared__ uint32_t table[4][256];  // slice-by-4
  extern __shared__ __align__(16) uint32_t wbuf[];  // kChunkSmem bytes (dynamic, opt-in > 48 KB)
  __shared__ uint32_t part[kCrcThreads];
  const uint32_t t = threadIdx.x;
  {
    uint32_t e = crc_table_entry(t);
    table[0][t] = e;
#pragma unroll
    for (int k = 1; k < 4; ++k) {
      e = (e >> 8) ^ crc_table_entry(e & 0xFFu);
      table[k][t] = e;
    }
  }
  const uint64_t base = uint64_t(blockIdx.x) * kChunk;  // full chunks only
  const uint4* src = reinterpret_cast<const uint4*>(data + base);
  const bool aligned16 = (reinterpret_cast<uintptr_t>(data) & 15u) == 0;
  if (aligned16) {
#pragma unroll 4
    for (uint32_t i = t; i < kChunk / 16; i += kCrcThreads) {
      const uint4 v = __ldg(src + i);
      uint32_t* d = wbuf + (i >> 4) * kPieceWords + (i & 15u) * 4;  // 16 uint4 per piece
      d[0] = v.x;
      d[1] = v.y;
      d[2] = v.z;
      d[3] = v.w;
    }
  } else {
    uint8_t* b = reinterpret_cast<uint8_t*>(wbuf);
    for (uint32_t i = t; i < kChunk; i += kCrcThreads) b[(i >> 8) * kPieceWords * 4 + (i & 255u)] = data[base + i];
  }
  __syncthreads();
  uint32_t c = 0;
  const uint32_t* p = wbuf + t * kPieceWords;
#pragma unroll 8
  for (uint32_t k = 0; k < kPiece / 4; ++k) {  // 4 bytes per step (little-endian byte order)
    c ^= p[k];
    c = table[3][c & 0xFFu] ^ table[2][(c >> 8) & 0xFFu] ^ table[1][(c >> 16) & 0xFFu] ^ table[0][c >> 24];
  }
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

// one CTA: (1) thread t folds chunk CRCs [t*per, (t+1)*per) in order, (2) the
// tail (< 64 KB) in 256-byte pieces in parallel, (3) thread 0 folds the range
// CRCs and the tail pieces in order and applies the conditioning.  Every
// operator is precomputed on the host (S^n for the record length included).
struct FinalOps {
  Mat chunk;       // S^65536
  Mat range;       // S^(per * 65536)
  Mat last_range;  // S^(len of the last range)
  Mat piece;       // S^256
  Mat tail_last;   // S^(len of the last tail piece)
  Mat total;       // S^n
};
__global__ void __launch_bounds__(kCrcThreads) crc_final_kernel(const uint8_t* __restrict__ data, uint64_t n,
                                                                uint64_t nchunks, uint64_t per,
                                                                const uint32_t* __restrict__ chunk_raw, FinalOps ops,
                                                                uint32_t* out) {
  __shared__ uint32_t table[256];
  __shared__ uint32_t part[kCrcThreads];
  __shared__ uint32_t rng[kCrcThreads];
  const uint32_t t = threadIdx.x;
  table[t] = crc_table_entry(t);
  {
    uint32_t r = 0;
    const uint64_t c0 = uint64_t(t) * per, c1 = c0 + per < nchunks ? c0 + per : nchunks;
    for (uint64_t i = c0; i < c1; ++i) r = mat_apply(ops.chunk, r) ^ chunk_raw[i];
    rng[t] = r;
  }
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
  const uint64_t nranges = per ? (nchunks + per - 1) / per : 0;
  for (uint64_t i = 0; i + 1 < nranges; ++i) r = mat_apply(ops.range, r) ^ rng[i];
  if (nranges) r = mat_apply(ops.last_range, r) ^ rng[nranges - 1];
  const uint32_t npieces = static_cast<uint32_t>((tail + kPiece - 1) / kPiece);
  for (uint32_t i = 0; i + 1 < npieces; ++i) r = mat_apply(ops.piece, r) ^ part[i];
  if (npieces) r = mat_apply(ops.tail_last, r) ^ part[npieces - 1];
  *out = ~(mat_apply(ops.total, 0xFFFFFFFFu) ^ r);
}

struct CrcOps {
  TreeOps tree;
  Mat chunk;
  Mat pow2[48];  // S^(2^k bytes)
};
CrcOps make_crc_ops() {
  CrcOps ops;
  const Mat b = op_one_byte();
  for (int l = 0; l < kLevels; ++l) ops.tree.op[l] = op_pow(b, uint64_t(kPiece) << l);
  ops.chunk = op_pow(b, kChunk);
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

// scratch: >= max(1, n / 64 KB) uint32 device words
int launch_crc32(const void* data, uint64_t n, uint32_t* out_dev, uint32_t* scratch, void* stream) {
  auto st = static_cast<cudaStream_t>(stream);
  const CrcOps& ops = crc_ops();
  const uint64_t nchunks = n / kChunk;
  static DeviceOnce once;
  const int se = once.run([](int) {
    return static_cast<int>(cudaFuncSetAttribute(crc_chunks_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 static_cast<int>(kChunkSmem)));
  });
  if (se) return se;
  if (nchunks) {
    crc_chunks_kernel<<<static_cast<unsigned>(nchunks), kCrcThreads, kChunkSmem, st>>>(
        static_cast<const uint8_t*>(data), n, ops.tree, scratch);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return static_cast<int>(e);
  }
  const uint64_t per = (nchunks + kCrcThreads - 1) / kCrcThreads;
  const uint64_t nranges = per ? (nchunks + per - 1) / per : 0;
  const uint64_t tail = n - nchunks * kChunk;
  // the operators depend on n only: one cached set per length (records repeat their size)
  static std::mutex mu;
  static uint64_t cached_n = ~uint64_t(0);
  static FinalOps cached;
  FinalOps fo;
  {
    std::lock_guard<std::mutex> lk(mu);
    if (cached_n != n) {
      cached.chunk = ops.chunk;
      cached.range = op_pow_fast(per * kChunk);
      cached.last_range = nranges ? op_pow_fast((nchunks - (nranges - 1) * per) * kChunk) : mat_identity();
      cached.piece = ops.tree.op[0];
      cached.tail_last = tail ? op_pow_fast(tail - (tail - 1) / kPiece * kPiece) : mat_identity();
      cached.total = op_pow_fast(n);
      cached_n = n;
    }
    fo = cached;
  }
  crc_final_kernel<<<1, kCrcThreads, 0, st>>>(static_cast<const uint8_t*>(data), n, nchunks, per, scratch, fo,
                                              out_dev);
  return static_cast<int>(cudaGetLastError());
}

uint64_t crc32_scratch_words(uint64_t n) { return n / kChunk + 1; }

}  // namespace rwb
