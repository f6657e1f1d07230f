// Microbenchmark: variants of the fp32 Adam undo elementwise body on a flat
// 1B-element state, to separate the memory-pattern ceiling (4 reads, 3
// writes per element) from the cost of the IEEE arithmetic.  Not product
// code; the product kernel lives in paper_2302_06173_b200/csrc.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -fmad=false -lineinfo \
//        -o tools/undo_variants tools/undo_variants.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#define CK(x)                                                                    \
  do {                                                                           \
    cudaError_t e = (x);                                                         \
    if (e != cudaSuccess) {                                                      \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);   \
      exit(1);                                                                   \
    }                                                                            \
  } while (0)

struct Sc {
  float eta, c1, c2, eps, wd, omb1, omb2, b1, b2;
  float r1, r2, rb1, rb2;  // RN(1/c) for the constant divisors
};

// IEEE a/b for a constant b with precomputed r = RN(1/b): Markstein
// q = RN(a r); e = a - b q (exact); q' = RN(q + e r).  Fast path only when a
// is comfortably normal; otherwise the IEEE division.
__device__ __forceinline__ float div_const(float a, float b, float r) {
  const uint32_t ex = (__float_as_uint(a) >> 23) & 0xffu;
  if (ex - 24u < 200u) {
    float q = __fmul_rn(a, r);
    float e = __fmaf_rn(-q, b, a);
    return __fmaf_rn(e, r, q);
  }
  return __fdiv_rn(a, b);
}

template <int MODE>
__device__ __forceinline__ void undo_elem(const Sc& s, float& x, float g, float& m, float& v,
                                          bool& bad) {
  if constexpr (MODE == 2) {  // memory ceiling: trivial math, same traffic
    float xt = __fadd_rn(x, g);
    m = __fadd_rn(m, g);
    v = __fadd_rn(v, g);
    x = xt;
    return;
  } else {
    float mhat, vhat;
    if constexpr (MODE == 1) {
      mhat = div_const(m, s.c1, s.r1);
      vhat = div_const(v, s.c2, s.r2);
    } else {
      mhat = __fdiv_rn(m, s.c1);
      vhat = __fdiv_rn(v, s.c2);
    }
    float xt = __fadd_rn(x, __fdiv_rn(__fmul_rn(s.eta, mhat), __fadd_rn(__fsqrt_rn(vhat), s.eps)));
    float gd = __fadd_rn(g, __fmul_rn(s.wd, xt));
    float mn = __fsub_rn(m, __fmul_rn(s.omb1, gd));
    float vn = __fsub_rn(v, __fmul_rn(__fmul_rn(s.omb2, gd), gd));
    if constexpr (MODE == 1) {
      m = div_const(mn, s.b1, s.rb1);
      v = div_const(vn, s.b2, s.rb2);
    } else {
      m = __fdiv_rn(mn, s.b1);
      v = __fdiv_rn(vn, s.b2);
    }
    x = xt;
    if constexpr (MODE != 3) {
      bad |= ((__float_as_uint(x) & 0x7f800000u) == 0x7f800000u) |
             ((__float_as_uint(m) & 0x7f800000u) == 0x7f800000u) |
             ((__float_as_uint(v) & 0x7f800000u) == 0x7f800000u);
    }
  }
}

struct F8 {
  float4 a, b;
};

template <int LDMODE>
__device__ __forceinline__ float4 ld(const float4* p) {
  if constexpr (LDMODE == 0) return __ldcs(p);
  else return *p;
}
template <int LDMODE>
__device__ __forceinline__ void st(float4* p, const float4& v) {
  if constexpr (LDMODE == 0) __stcs(p, v);
  else *p = v;
}
// 256-bit (sm_100) vector access
template <int LDMODE>
__device__ __forceinline__ F8 ld8(const F8* p) {
  uint32_t r[8];
  if constexpr (LDMODE == 2)
    asm volatile("ld.global.L1::no_allocate.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                   "=r"(r[7]) : "l"(p));
  else
    asm volatile("ld.global.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                   "=r"(r[7]) : "l"(p));
  F8 o;
  o.a = make_float4(__uint_as_float(r[0]), __uint_as_float(r[1]), __uint_as_float(r[2]), __uint_as_float(r[3]));
  o.b = make_float4(__uint_as_float(r[4]), __uint_as_float(r[5]), __uint_as_float(r[6]), __uint_as_float(r[7]));
  return o;
}
template <int LDMODE>
__device__ __forceinline__ void st8(F8* p, const F8& v) {
  if constexpr (LDMODE == 2)
    asm volatile("st.global.L1::no_allocate.L2::evict_first.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                 :: "l"(p), "r"(__float_as_uint(v.a.x)), "r"(__float_as_uint(v.a.y)), "r"(__float_as_uint(v.a.z)),
                    "r"(__float_as_uint(v.a.w)), "r"(__float_as_uint(v.b.x)), "r"(__float_as_uint(v.b.y)),
                    "r"(__float_as_uint(v.b.z)), "r"(__float_as_uint(v.b.w)) : "memory");
  else
    asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                 :: "l"(p), "r"(__float_as_uint(v.a.x)), "r"(__float_as_uint(v.a.y)), "r"(__float_as_uint(v.a.z)),
                    "r"(__float_as_uint(v.a.w)), "r"(__float_as_uint(v.b.x)), "r"(__float_as_uint(v.b.y)),
                    "r"(__float_as_uint(v.b.z)), "r"(__float_as_uint(v.b.w)) : "memory");
}

template <int MODE>
__device__ __forceinline__ void undo4(const Sc& s, float4& x, const float4& g, float4& m, float4& v, bool& bad) {
  undo_elem<MODE>(s, x.x, g.x, m.x, v.x, bad);
  undo_elem<MODE>(s, x.y, g.y, m.y, v.y, bad);
  undo_elem<MODE>(s, x.z, g.z, m.z, v.z, bad);
  undo_elem<MODE>(s, x.w, g.w, m.w, v.w, bad);
}

// flat grid-stride over float4 with U float4 per thread per iteration
template <int MODE, int U, int LDMODE, int MINB>
__global__ void __launch_bounds__(256, MINB) undo_flat(float* __restrict__ x, const float* __restrict__ g,
                                                       float* __restrict__ m, float* __restrict__ v,
                                                       uint64_t n4, Sc s, int* flag) {
  bool bad = false;
  if constexpr (LDMODE >= 2) {  // 256-bit accesses: n8 = n4/2 units
    const uint64_t n8 = n4 / 2;
    const uint64_t stride = uint64_t(gridDim.x) * 256 * U;
    for (uint64_t base = uint64_t(blockIdx.x) * 256 * U + threadIdx.x; base < n8; base += stride) {
      F8 xr[U], gr[U], mr[U], vr[U];
#pragma unroll
      for (int k = 0; k < U; ++k) {
        uint64_t i = base + uint64_t(k) * 256;
        if (i < n8) {
          xr[k] = ld8<LDMODE>(reinterpret_cast<const F8*>(x) + i);
          gr[k] = ld8<LDMODE>(reinterpret_cast<const F8*>(g) + i);
          mr[k] = ld8<LDMODE>(reinterpret_cast<const F8*>(m) + i);
          vr[k] = ld8<LDMODE>(reinterpret_cast<const F8*>(v) + i);
        }
      }
#pragma unroll
      for (int k = 0; k < U; ++k) {
        uint64_t i = base + uint64_t(k) * 256;
        if (i < n8) {
          undo4<MODE>(s, xr[k].a, gr[k].a, mr[k].a, vr[k].a, bad);
          undo4<MODE>(s, xr[k].b, gr[k].b, mr[k].b, vr[k].b, bad);
          st8<LDMODE>(reinterpret_cast<F8*>(x) + i, xr[k]);
          st8<LDMODE>(reinterpret_cast<F8*>(m) + i, mr[k]);
          st8<LDMODE>(reinterpret_cast<F8*>(v) + i, vr[k]);
        }
      }
    }
  } else {
    const uint64_t stride = uint64_t(gridDim.x) * 256 * U;
    for (uint64_t base = uint64_t(blockIdx.x) * 256 * U + threadIdx.x; base < n4; base += stride) {
      float4 xr[U], gr[U], mr[U], vr[U];
#pragma unroll
      for (int k = 0; k < U; ++k) {
        uint64_t i = base + uint64_t(k) * 256;
        if (i < n4) {
          xr[k] = ld<LDMODE>(reinterpret_cast<const float4*>(x) + i);
          gr[k] = ld<LDMODE>(reinterpret_cast<const float4*>(g) + i);
          mr[k] = ld<LDMODE>(reinterpret_cast<const float4*>(m) + i);
          vr[k] = ld<LDMODE>(reinterpret_cast<const float4*>(v) + i);
        }
      }
#pragma unroll
      for (int k = 0; k < U; ++k) {
        uint64_t i = base + uint64_t(k) * 256;
        if (i < n4) {
          undo4<MODE>(s, xr[k], gr[k], mr[k], vr[k], bad);
          st<LDMODE>(reinterpret_cast<float4*>(x) + i, xr[k]);
          st<LDMODE>(reinterpret_cast<float4*>(m) + i, mr[k]);
          st<LDMODE>(reinterpret_cast<float4*>(v) + i, vr[k]);
        }
      }
    }
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

// ---- TMA bulk (cp.async.bulk) variant: smem-staged, persistent ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(b)), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" :: "r"(smem_u32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
               :: "l"(dst), "r"(smem_u32(src)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" :: "n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" :: "n"(N) : "memory");
}

// TILE floats per array per stage; S stages; T threads.  DEFER: refill the
// stage of the PREVIOUS tile after wait_group<1> (its stores are complete)
// instead of waiting for the just-issued stores to read smem.
template <int MODE, int TILE, int S, int T, int DEFER>
__global__ void __launch_bounds__(T, 1) undo_tma(float* __restrict__ x, const float* __restrict__ g,
                                                 float* __restrict__ m, float* __restrict__ v,
                                                 uint64_t n4, Sc s, int* flag) {
  extern __shared__ __align__(128) unsigned char smem[];
  float* buf = reinterpret_cast<float*>(smem);  // [S][4][TILE]
  __shared__ uint64_t full[S];
  const uint64_t n = n4 * 4;
  const uint64_t ntiles = n / TILE;  // assume divisible for the bench
  const uint32_t tid = threadIdx.x;
  if (tid == 0) {
    for (int i = 0; i < S; ++i) mbar_init(&full[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](uint64_t tile, int st) {
    float* b = buf + size_t(st) * 4 * TILE;
    const uint64_t off = tile * TILE;
    mbar_expect_tx(&full[st], 4 * TILE * 4);
    bulk_load(b + 0 * TILE, x + off, TILE * 4, &full[st]);
    bulk_load(b + 1 * TILE, g + off, TILE * 4, &full[st]);
    bulk_load(b + 2 * TILE, m + off, TILE * 4, &full[st]);
    bulk_load(b + 3 * TILE, v + off, TILE * 4, &full[st]);
  };
  const uint64_t per = (ntiles + gridDim.x - 1) / gridDim.x;
  uint64_t first = DEFER == 2 ? blockIdx.x * per : blockIdx.x;
  const uint64_t step = DEFER == 2 ? 1 : gridDim.x;
  const uint64_t tend = DEFER == 2 ? (first + per < ntiles ? first + per : ntiles) : ntiles;
  if (tid == 0) {
    for (int k = 0; k < S; ++k) {
      uint64_t t = first + k * step;
      if (t < tend) issue(t, k);
    }
  }
  bool bad = false;
  int it = 0;
  for (uint64_t t = first; t < tend; t += step, ++it) {
    const int st = it % S;
    const uint32_t par = (it / S) & 1;
    mbar_wait(&full[st], par);
    float* b = buf + size_t(st) * 4 * TILE;
#pragma unroll 2
    for (int e = tid * 4; e < TILE; e += T * 4) {
      float4 xr = *reinterpret_cast<float4*>(b + e);
      float4 gr = *reinterpret_cast<float4*>(b + TILE + e);
      float4 mr = *reinterpret_cast<float4*>(b + 2 * TILE + e);
      float4 vr = *reinterpret_cast<float4*>(b + 3 * TILE + e);
      undo4<MODE>(s, xr, gr, mr, vr, bad);
      *reinterpret_cast<float4*>(b + e) = xr;
      *reinterpret_cast<float4*>(b + 2 * TILE + e) = mr;
      *reinterpret_cast<float4*>(b + 3 * TILE + e) = vr;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      const uint64_t off = t * TILE;
      bulk_store(x + off, b, TILE * 4);
      bulk_store(m + off, b + 2 * TILE, TILE * 4);
      bulk_store(v + off, b + 3 * TILE, TILE * 4);
      bulk_commit();
      if constexpr (DEFER) {
        if (it > 0) {
          bulk_wait<1>();  // previous tile's stores complete
          const int ps = (it - 1) % S;
          uint64_t nt = t - step + uint64_t(S) * step;
          if (nt < tend) issue(nt, ps);
        }
      } else {
        uint64_t nt = t + uint64_t(S) * step;
        if (nt < ntiles) {
          bulk_wait_read<0>();
          issue(nt, st);
        }
      }
    }
  }
  if (tid == 0) bulk_wait<0>();
  if (__syncthreads_or(bad) && tid == 0) atomicOr(flag, 1);
}

__global__ void fill(float* p, uint64_t n, float scale, float off, uint32_t seed) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    uint32_t h = uint32_t(i) * 2654435761u ^ seed;
    h ^= h >> 15;
    h *= 2246822519u;
    h ^= h >> 13;
    p[i] = off + scale * (float(h & 0xffffff) / 16777216.0f);
  }
}

__global__ void copy_kernel(const float4* __restrict__ a, float4* __restrict__ b, uint64_t n4) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n4;
       i += uint64_t(gridDim.x) * blockDim.x)
    __stcs(b + i, __ldcs(a + i));
}

static size_t g_dyn_smem = 0;
static int g_threads = 256;
template <typename K>
int occ(K k) {
  int b = 0;
  if (g_dyn_smem) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g_dyn_smem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k, g_threads, g_dyn_smem);
  return b;
}

int main(int argc, char** argv) {
  setvbuf(stdout, NULL, _IONBF, 0);
  uint64_t n = argc > 1 ? strtoull(argv[1], 0, 10) : 1000000000ull;
  int reps = argc > 2 ? atoi(argv[2]) : 10;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  float *x, *g, *m, *v, *x0, *m0, *v0;
  int* flag;
  CK(cudaMalloc(&x, n * 4));
  CK(cudaMalloc(&g, n * 4));
  CK(cudaMalloc(&m, n * 4));
  CK(cudaMalloc(&v, n * 4));
  CK(cudaMalloc(&x0, n * 4));
  CK(cudaMalloc(&m0, n * 4));
  CK(cudaMalloc(&v0, n * 4));
  CK(cudaMalloc(&flag, 4));
  fill<<<sms * 8, 256>>>(x0, n, 0.2f, -0.1f, 1);
  fill<<<sms * 8, 256>>>(g, n, 0.2f, -0.1f, 2);
  fill<<<sms * 8, 256>>>(m0, n, 0.002f, -0.001f, 3);
  fill<<<sms * 8, 256>>>(v0, n, 1e-4f, 1e-6f, 4);
  CK(cudaDeviceSynchronize());
  Sc s;
  const double b1 = 0.9, b2 = 0.999, t = 11;
  s.eta = 1e-4f;
  s.c1 = float(1.0 - pow(b1, t));
  s.c2 = float(1.0 - pow(b2, t));
  s.eps = 1e-8f;
  s.wd = 0.01f;
  s.omb1 = float(1.0 - b1);
  s.omb2 = float(1.0 - b2);
  s.b1 = float(b1);
  s.b2 = float(b2);
  s.r1 = 1.0f / s.c1;
  s.r2 = 1.0f / s.c2;
  s.rb1 = 1.0f / s.b1;
  s.rb2 = 1.0f / s.b2;
  const uint64_t n4 = n / 4;
  const double bytes = double(n) * 28.0;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  std::vector<float> ref_x, ref_m, ref_v;

  auto reset = [&]() {
    CK(cudaMemcpy(x, x0, n * 4, cudaMemcpyDeviceToDevice));
    CK(cudaMemcpy(m, m0, n * 4, cudaMemcpyDeviceToDevice));
    CK(cudaMemcpy(v, v0, n * 4, cudaMemcpyDeviceToDevice));
  };
  auto sample = [&](std::vector<float>& ox, std::vector<float>& om, std::vector<float>& ov) {
    const int S = 1 << 20;
    ox.resize(S);
    om.resize(S);
    ov.resize(S);
    CK(cudaMemcpy(ox.data(), x + (n - S), S * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(om.data(), m + (n - S), S * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(ov.data(), v + (n - S), S * 4, cudaMemcpyDeviceToHost));
  };

  auto run = [&](const char* name, auto kern, int blocks_per_sm_override, bool check_ref) {
    int bps = occ(kern);
    if (blocks_per_sm_override > 0) bps = blocks_per_sm_override;
    int grid = sms * bps;
    reset();
    kern<<<grid, g_threads, g_dyn_smem>>>(x, g, m, v, n4, s, flag);  // one pass for the parity sample
    CK(cudaDeviceSynchronize());
    std::vector<float> ox, om, ov;
    sample(ox, om, ov);
    bool same = true;
    if (check_ref) {
      if (ref_x.empty()) {
        ref_x = ox;
        ref_m = om;
        ref_v = ov;
      } else {
        same = !memcmp(ox.data(), ref_x.data(), ox.size() * 4) &&
               !memcmp(om.data(), ref_m.data(), om.size() * 4) &&
               !memcmp(ov.data(), ref_v.data(), ov.size() * 4);
      }
    }
    float best = 1e30f, tot = 0;
    for (int r = 0; r < reps; ++r) {
      reset();
      CK(cudaEventRecord(e0));
      kern<<<grid, g_threads, g_dyn_smem>>>(x, g, m, v, n4, s, flag);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      best = ms < best ? ms : best;
      tot += ms;
    }
    printf("%-44s occ=%d grid=%6d  best %.4f ms  %.1f GB/s  mean %.1f GB/s  %s\n", name, bps, grid,
           best, bytes / best / 1e6, bytes / (tot / reps) / 1e6,
           check_ref ? (same ? "bitwise==IEEE" : "MISMATCH") : "");
  };

  // copy ceiling (same as MEASURED_PEAKS: 1 read + 1 write)
  {
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
      CK(cudaEventRecord(e0));
      copy_kernel<<<sms * 8, 256>>>(reinterpret_cast<const float4*>(x0), reinterpret_cast<float4*>(x), n4);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      best = ms < best ? ms : best;
    }
    printf("%-44s best %.4f ms  %.1f GB/s\n", "copy 4B/elem r+w (ldcs/stcs)", best, n * 8.0 / best / 1e6);
  }
  run("IEEE   U2 cs       (product-like)", undo_flat<0, 2, 0, 1>, 0, true);
  run("IEEE   U1 cs", undo_flat<0, 1, 0, 1>, 0, true);
  run("IEEE   U4 cs", undo_flat<0, 4, 0, 1>, 0, true);
  run("IEEE   U2 cs minb4", undo_flat<0, 2, 0, 4>, 0, true);
  run("IEEE   U2 plain", undo_flat<0, 2, 1, 1>, 0, true);
  run("IEEE   V8(256b) U1 evict_first", undo_flat<0, 1, 2, 1>, 0, true);
  run("IEEE   V8(256b) U1 plain", undo_flat<0, 1, 3, 1>, 0, true);
  run("IEEE   V8(256b) U2 evict_first", undo_flat<0, 2, 2, 1>, 0, true);
  run("IEEE   U2 cs nocheck", undo_flat<3, 2, 0, 1>, 0, true);
  run("CDIV   U2 cs", undo_flat<1, 2, 0, 1>, 0, true);
  run("CDIV   U1 cs", undo_flat<1, 1, 0, 1>, 0, true);
  run("CDIV   U2 cs minb4", undo_flat<1, 2, 0, 4>, 0, true);
  run("CDIV   U4 cs", undo_flat<1, 4, 0, 1>, 0, true);
  run("CDIV   V8 U1 evict_first", undo_flat<1, 1, 2, 1>, 0, true);
  run("CDIV   V8 U2 evict_first", undo_flat<1, 2, 2, 1>, 0, true);
  run("TRIV   U2 cs       (memory ceiling)", undo_flat<2, 2, 0, 1>, 0, false);
  run("TRIV   U1 cs", undo_flat<2, 1, 0, 1>, 0, false);
  run("TRIV   U4 cs", undo_flat<2, 4, 0, 1>, 0, false);
  run("TRIV   U2 plain", undo_flat<2, 2, 1, 1>, 0, false);
  run("TRIV   V8 U1 evict_first", undo_flat<2, 1, 2, 1>, 0, false);
  run("TRIV   V8 U2 evict_first", undo_flat<2, 2, 2, 1>, 0, false);
  run("TRIV   V8 U1 plain", undo_flat<2, 1, 3, 1>, 0, false);
  run("TRIV   U2 cs grid x2", undo_flat<2, 2, 0, 1>, 16, false);
  run("IEEE   V8 U2 plain", undo_flat<0, 2, 3, 1>, 0, true);
  run("IEEE   V8 U3 evict_first", undo_flat<0, 3, 2, 1>, 0, true);
  run("IEEE   V8 U2 evict_first grid x1.5", undo_flat<0, 2, 2, 1>, 3, true);
  auto tma = [&](const char* nm, auto k, int tile, int S, int T) {
    g_dyn_smem = size_t(S) * tile * 16;
    g_threads = T;
    run(nm, k, 0, true);
    g_dyn_smem = 0;
    g_threads = 256;
  };
  tma("TMA t2048 S3 T256 imm", undo_tma<0, 2048, 3, 256, 0>, 2048, 3, 256);
  tma("TMA t2048 S3 T256 defer", undo_tma<0, 2048, 3, 256, 1>, 2048, 3, 256);
  tma("TMA t2048 S3 T256 defer CONTIG", undo_tma<0, 2048, 3, 256, 2>, 2048, 3, 256);
  tma("TRIV-TMA t2048 S3 T256 defer", undo_tma<2, 2048, 3, 256, 1>, 2048, 3, 256);
  tma("TRIV-TMA t2048 S3 T256 CONTIG", undo_tma<2, 2048, 3, 256, 2>, 2048, 3, 256);
  tma("TMA t2048 S4 T256 defer (1/SM?)", undo_tma<0, 2048, 4, 256, 1>, 2048, 4, 256);
  tma("TMA t1024 S6 T256 defer", undo_tma<0, 1024, 6, 256, 1>, 1024, 6, 256);
  tma("TMA t2048 S3 T384 imm", undo_tma<0, 2048, 3, 384, 0>, 2048, 3, 384);
  tma("TMA t2048 S3 T512 imm", undo_tma<0, 2048, 3, 512, 0>, 2048, 3, 512);
  tma("TMA t2048 S3 T512 defer", undo_tma<0, 2048, 3, 512, 1>, 2048, 3, 512);
  tma("TMA t1536 S4 T256 defer", undo_tma<0, 1536, 4, 256, 1>, 1536, 4, 256);
  tma("TMA t1536 S4 T384 defer", undo_tma<0, 1536, 4, 384, 1>, 1536, 4, 384);
  tma("TMA t2048 S2 T256 imm (3/SM)", undo_tma<0, 2048, 2, 256, 0>, 2048, 2, 256);
  tma("TMA t2048 S2 T384 imm (3/SM)", undo_tma<0, 2048, 2, 384, 0>, 2048, 2, 384);
  tma("TMA t1024 S4 T256 defer (3/SM)", undo_tma<0, 1024, 4, 256, 1>, 1024, 4, 256);
  tma("TMA t1024 S3 T256 imm (4/SM)", undo_tma<0, 1024, 3, 256, 0>, 1024, 3, 256);
  tma("TMA t4096 S3 T512 imm (1/SM)", undo_tma<0, 4096, 3, 512, 0>, 4096, 3, 512);
  tma("TMA t3072 S2 T512 imm (2/SM)", undo_tma<0, 3072, 2, 512, 0>, 3072, 2, 512);
  g_dyn_smem = 0;
  return 0;
}
