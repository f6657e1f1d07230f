// LAMB step, first pass and trust ratio (optim.cpp:273-295).
//
// Pass 1 (per group): advance m, v exactly as step_lamb does, compute the
// update r + lambda x and accumulate ||x||^2 and ||update||^2 in fp64
// (the reference accumulates in double too).  The reduction order is fixed
// (per-thread strided sums, a fixed block tree, a fixed final tree), so the
// result is deterministic, but it is not the reference's left-to-right
// sequential sum: the trust ratio agrees to ~1e-15 relative (tolerance-matched;
// everything elementwise is bit-exact).  The trust kernel then stores the
// ratio (the LAMB "saved scalar", optim.cpp:294) and writes scaled = eta *
// trust into the group's ScalarSet for the elementwise pass 2 (x update),
// which runs through the fused TMA kernel.
#include <cuda_runtime.h>

#include <cstdint>

#include "internal.h"

namespace rwb {
namespace {

constexpr int kLT = 256;

template <typename T>
struct LA;
template <>
struct LA<float> {
  __device__ static float mul(float a, float b) { return __fmul_rn(a, b); }
  __device__ static float add(float a, float b) { return __fadd_rn(a, b); }
  __device__ static float div(float a, float b) { return __fdiv_rn(a, b); }
  __device__ static float sqrt(float a) { return __fsqrt_rn(a); }
};
template <>
struct LA<double> {
  __device__ static double mul(double a, double b) { return __dmul_rn(a, b); }
  __device__ static double add(double a, double b) { return __dadd_rn(a, b); }
  __device__ static double div(double a, double b) { return __ddiv_rn(a, b); }
  __device__ static double sqrt(double a) { return __dsqrt_rn(a); }
};

template <typename T>
__global__ void __launch_bounds__(kLT) lamb_pass1_kernel(const T* __restrict__ x, T* __restrict__ g,
                                                         const T* __restrict__ grad, T* __restrict__ m,
                                                         T* __restrict__ v, uint64_t off, uint64_t len,
                                                         ScalarSet ss, Uniform u, double* __restrict__ partial) {
  using A = LA<T>;
  const T c1 = T(ss.c1), c2 = T(ss.c2), b1 = T(u.b1), b2 = T(u.b2), omb1 = T(u.one_m_b1), omb2 = T(u.one_m_b2),
          eps = T(u.eps), wd = T(u.wd);
  double sx = 0.0, su = 0.0;
  for (uint64_t i = blockIdx.x * uint64_t(kLT) + threadIdx.x; i < len; i += uint64_t(gridDim.x) * kLT) {
    const uint64_t k = off + i;
    const T gd = grad ? grad[k] : g[k];
    if (grad) g[k] = gd;  // block.g = grad (optim.cpp:349)
    const T mk = A::add(A::mul(b1, m[k]), A::mul(omb1, gd));
    const T vk = A::add(A::mul(b2, v[k]), A::mul(A::mul(omb2, gd), gd));
    m[k] = mk;
    v[k] = vk;
    const T mhat = A::div(mk, c1);
    const T vhat = A::div(vk, c2);
    const T xk = x[k];
    const T upd = A::add(A::div(mhat, A::add(A::sqrt(vhat), eps)), A::mul(wd, xk));
    const double xd = double(xk), ud = double(upd);
    sx = __dadd_rn(sx, __dmul_rn(xd, xd));
    su = __dadd_rn(su, __dmul_rn(ud, ud));
  }
  __shared__ double shx[kLT], shu[kLT];
  shx[threadIdx.x] = sx;
  shu[threadIdx.x] = su;
  __syncthreads();
  for (int s = kLT / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      shx[threadIdx.x] = __dadd_rn(shx[threadIdx.x], shx[threadIdx.x + s]);
      shu[threadIdx.x] = __dadd_rn(shu[threadIdx.x], shu[threadIdx.x + s]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    partial[2 * blockIdx.x] = shx[0];
    partial[2 * blockIdx.x + 1] = shu[0];
  }
}

// one CTA: fixed-order tree over the pass-1 partials -> trust ratio
__global__ void __launch_bounds__(kLT) lamb_trust_kernel(const double* __restrict__ partial, int nparts, double eta,
                                                         double wd, double* __restrict__ trust_out,
                                                         ScalarSet* __restrict__ set) {
  __shared__ double shx[kLT], shu[kLT];
  double sx = 0.0, su = 0.0;
  for (int i = threadIdx.x; i < nparts; i += kLT) {
    sx = __dadd_rn(sx, partial[2 * i]);
    su = __dadd_rn(su, partial[2 * i + 1]);
  }
  shx[threadIdx.x] = sx;
  shu[threadIdx.x] = su;
  __syncthreads();
  for (int s = kLT / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      shx[threadIdx.x] = __dadd_rn(shx[threadIdx.x], shx[threadIdx.x + s]);
      shu[threadIdx.x] = __dadd_rn(shu[threadIdx.x], shu[threadIdx.x + s]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double xn = __dsqrt_rn(shx[0]), un = __dsqrt_rn(shu[0]);
    const double trust = (xn > 0.0 && un > 0.0) ? __ddiv_rn(xn, un) : 1.0;  // optim.cpp:290
    *trust_out = trust;
    set->eta = __dmul_rn(eta, trust);  // (eta * trust) * update, optim.cpp:292
    set->denom = __dsub_rn(1.0, __dmul_rn(set->eta, wd));
  }
}

}  // namespace

int lamb_parts_for(uint64_t len) {
  uint64_t b = (len + kLT * 16 - 1) / (kLT * 16);
  return static_cast<int>(b < 1 ? 1 : (b > 1184 ? 1184 : b));
}

int launch_lamb_pass1(int dtype, void* x, void* g, const void* grad, void* m, void* v, uint64_t off, uint64_t len,
                      const ScalarSet& ss, const Uniform& u, double* partial, double* trust_out,
                      ScalarSet* set_dev, void* stream) {
  auto st = static_cast<cudaStream_t>(stream);
  const int parts = lamb_parts_for(len);
  if (dtype == RW_F64)
    lamb_pass1_kernel<double><<<parts, kLT, 0, st>>>(static_cast<const double*>(x), static_cast<double*>(g),
                                                     static_cast<const double*>(grad), static_cast<double*>(m),
                                                     static_cast<double*>(v), off, len, ss, u, partial);
  else
    lamb_pass1_kernel<float><<<parts, kLT, 0, st>>>(static_cast<const float*>(x), static_cast<float*>(g),
                                                    static_cast<const float*>(grad), static_cast<float*>(m),
                                                    static_cast<float*>(v), off, len, ss, u, partial);
  lamb_trust_kernel<<<1, kLT, 0, st>>>(partial, parts, ss.eta, u.wd, trust_out, set_dev);
  return static_cast<int>(cudaGetLastError());
}

}  // namespace rwb
