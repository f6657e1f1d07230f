// LAMB step, first pass and trust ratio (optim.cpp:195-217).
//
// Pass 1 (all groups, one launch): advance m, v exactly as step_lamb does,
// compute the update r + lambda x and accumulate ||x||^2 and ||update||^2 in
// fp64 (the reference accumulates in double too).  The reduction order is
// fixed (per-lane strided sums, a warp xor tree per chunk, per-thread strided
// sums over a group's chunks, a block tree), so the result is deterministic,
// but it is not the reference's left-to-right sequential sum: the trust ratio
// agrees to ~1e-15 relative (tolerance-matched; everything elementwise is
// bit-exact).  The trust kernel (one CTA per group) stores the ratio (the LAMB
// "saved scalar", optim.cpp:216) and writes scaled = eta * trust into the
// group's ScalarSet for the elementwise pass 2 (x update), which runs through
// the fused TMA kernel.
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

// vector type for 16-byte accesses
template <typename T>
struct V16;
template <>
struct V16<float> {
  using type = float4;
  static constexpr int n = 4;
};
template <>
struct V16<double> {
  using type = double2;
  static constexpr int n = 2;
};

// m, v advance and the two squared-norm contributions of one element
template <typename T>
__device__ __forceinline__ void lamb_math(const T xk, const T gd, T& mk, T& vk, const T c1, const T c2,
                                          const Uniform& u, double& sx, double& su) {
  using A = LA<T>;
  mk = A::add(A::mul(T(u.b1), mk), A::mul(T(u.one_m_b1), gd));
  vk = A::add(A::mul(T(u.b2), vk), A::mul(A::mul(T(u.one_m_b2), gd), gd));
  const T mhat = A::div(mk, c1);
  const T vhat = A::div(vk, c2);
  const T upd = A::add(A::div(mhat, A::add(A::sqrt(vhat), T(u.eps))), A::mul(T(u.wd), xk));
  const double xd = double(xk), ud = double(upd);
  sx = __dadd_rn(sx, __dmul_rn(xd, xd));
  su = __dadd_rn(su, __dmul_rn(ud, ud));
}

template <typename T>
__device__ __forceinline__ void lamb_elem(const T* __restrict__ x, T* __restrict__ g, const T* __restrict__ grad,
                                          T* __restrict__ m, T* __restrict__ v, uint64_t k, const T c1, const T c2,
                                          const Uniform& u, double& sx, double& su) {
  const T gd = grad ? grad[k] : g[k];
  if (grad) g[k] = gd;  // block.g = grad (optim.cpp:271)
  T mk = m[k], vk = v[k];
  lamb_math<T>(x[k], gd, mk, vk, c1, c2, u, sx, su);
  m[k] = mk;
  v[k] = vk;
}

// Pass 1 over ALL selected groups in one launch: one warp per chunk (the same
// chunk decomposition as the fused TMA kernel's work list), the chunk's
// (||x||^2, ||update||^2) partial reduced by a fixed xor tree and stored at
// its chunk index, so the result does not depend on scheduling.
template <typename T>
__global__ void __launch_bounds__(kLT) lamb_pass1_kernel(const T* __restrict__ x, T* __restrict__ g,
                                                         const T* __restrict__ grad, T* __restrict__ m,
                                                         T* __restrict__ v, const WorkItem* __restrict__ work,
                                                         uint32_t n_work, uint32_t total_chunks, uint32_t chunk_elems,
                                                         const ScalarSet* __restrict__ sets, Uniform u,
                                                         double2* __restrict__ partial) {
  const int lane = threadIdx.x & 31;
  const uint32_t warps = gridDim.x * (kLT / 32);
  for (uint32_t c = blockIdx.x * (kLT / 32) + (threadIdx.x >> 5); c < total_chunks; c += warps) {
    uint32_t lo = 0, hi = n_work - 1;  // last item with chunk_begin <= c
    while (lo < hi) {
      const uint32_t mid = (lo + hi + 1) >> 1;
      if (work[mid].chunk_begin <= c) lo = mid;
      else hi = mid - 1;
    }
    const WorkItem w = work[lo];
    const ScalarSet ss = sets[w.sidx];
    const T c1 = T(ss.c1), c2 = T(ss.c2);
    const uint64_t begin = w.off + uint64_t(c - w.chunk_begin) * chunk_elems;
    const uint64_t end = min(begin + chunk_elems, w.off + w.len);
    double sx = 0.0, su = 0.0;
    // unaligned head, 16-byte vector body (4 fp32 / 2 fp64 per lane), tail
    constexpr int EV = V16<T>::n;
    using VT = typename V16<T>::type;
    uint64_t a16 = (begin + EV - 1) / EV * EV;
    if (a16 > end) a16 = end;
    const uint64_t b16 = a16 + (end - a16) / EV * EV;
    for (uint64_t k = begin + lane; k < a16; k += 32) lamb_elem<T>(x, g, grad, m, v, k, c1, c2, u, sx, su);
#pragma unroll 4
    for (uint64_t k = a16 + uint64_t(lane) * EV; k < b16; k += 32 * EV) {
      const VT xv = *reinterpret_cast<const VT*>(x + k);
      VT gv = *reinterpret_cast<const VT*>((grad ? grad : g) + k);
      VT mv = *reinterpret_cast<const VT*>(m + k);
      VT vv = *reinterpret_cast<const VT*>(v + k);
      const T* xp = reinterpret_cast<const T*>(&xv);
      const T* gp = reinterpret_cast<const T*>(&gv);
      T* mp = reinterpret_cast<T*>(&mv);
      T* vp = reinterpret_cast<T*>(&vv);
#pragma unroll
      for (int e = 0; e < EV; ++e) lamb_math<T>(xp[e], gp[e], mp[e], vp[e], c1, c2, u, sx, su);
      *reinterpret_cast<VT*>(m + k) = mv;
      *reinterpret_cast<VT*>(v + k) = vv;
      if (grad) *reinterpret_cast<VT*>(g + k) = gv;  // block.g = grad (optim.cpp:271)
    }
    for (uint64_t k = b16 + lane; k < end; k += 32) lamb_elem<T>(x, g, grad, m, v, k, c1, c2, u, sx, su);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      sx = __dadd_rn(sx, __shfl_xor_sync(0xffffffffu, sx, o));
      su = __dadd_rn(su, __shfl_xor_sync(0xffffffffu, su, o));
    }
    if (lane == 0) partial[c] = make_double2(sx, su);
  }
}

// One CTA per group: fixed-order reduction of its chunk partials -> trust
// ratio (optim.cpp:210-212), saved (:216) and folded into the group's
// ScalarSet as scaled = eta * trust for the x pass (:214).
__global__ void __launch_bounds__(kLT) lamb_trust_kernel(const WorkItem* __restrict__ work,
                                                         const double2* __restrict__ partial, double wd,
                                                         double* __restrict__ trust_table, uint32_t depth,
                                                         ScalarSet* __restrict__ sets) {
  const WorkItem w = work[blockIdx.x];
  __shared__ double shx[kLT], shu[kLT];
  double sx = 0.0, su = 0.0;
  for (uint32_t i = threadIdx.x; i < w.nchunks; i += kLT) {
    const double2 p = partial[w.chunk_begin + i];
    sx = __dadd_rn(sx, p.x);
    su = __dadd_rn(su, p.y);
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
    const double trust = (xn > 0.0 && un > 0.0) ? __ddiv_rn(xn, un) : 1.0;  // optim.cpp:212
    trust_table[uint64_t(w.gid) * depth + w.pad] = trust;
    ScalarSet* set = sets + w.sidx;
    set->eta = __dmul_rn(set->eta, trust);  // (eta * trust) * update
    set->denom = __dsub_rn(1.0, __dmul_rn(set->eta, wd));
  }
}

// Reference-order norms (rw_state_set_flags(RW_STATE_LAMB_SEQUENTIAL_NORMS),
// used by the host-block drop-in): one thread per group re-forms each
// element's update from the m, v pass 1 just wrote (the same expression, so
// the same bits) and accumulates ||x||^2 and ||update||^2 left to right in
// fp64 exactly as step_lamb's loop does (optim.cpp:199-208).  The sums land in
// the group's first chunk partial, zeros in the others, so the trust kernel's
// tree adds only exact zeros and the ratio equals the reference's bit for bit.
// O(n) on one thread: a parity path for host-resident blocks, not the batch path.
template <typename T>
__global__ void lamb_seq_norms_kernel(const T* __restrict__ x, const T* __restrict__ m, const T* __restrict__ v,
                                      const WorkItem* __restrict__ work, const ScalarSet* __restrict__ sets,
                                      Uniform u, double2* __restrict__ partial) {
  using A = LA<T>;
  const WorkItem w = work[blockIdx.x];
  if (threadIdx.x != 0) return;
  const ScalarSet ss = sets[w.sidx];
  const T c1 = T(ss.c1), c2 = T(ss.c2);
  double sx = 0.0, su = 0.0;
  for (uint64_t k = w.off; k < w.off + w.len; ++k) {
    const T xk = x[k];
    const T mhat = A::div(m[k], c1);
    const T vhat = A::div(v[k], c2);
    const T upd = A::add(A::div(mhat, A::add(A::sqrt(vhat), T(u.eps))), A::mul(T(u.wd), xk));
    const double xd = double(xk), ud = double(upd);
    sx = __dadd_rn(sx, __dmul_rn(xd, xd));
    su = __dadd_rn(su, __dmul_rn(ud, ud));
  }
  partial[w.chunk_begin] = make_double2(sx, su);
  for (uint32_t i = 1; i < w.nchunks; ++i) partial[w.chunk_begin + i] = make_double2(0.0, 0.0);
}

}  // namespace

int launch_lamb_pass1(int dtype, void* x, void* g, const void* grad, void* m, void* v, const WorkItem* work,
                      uint32_t n_work, uint32_t total_chunks, uint32_t chunk_elems, ScalarSet* sets,
                      const Uniform& u, double* partial, double* trust_table, uint32_t depth, bool sequential,
                      void* stream) {
  auto st = static_cast<cudaStream_t>(stream);
  if (n_work == 0 || total_chunks == 0) return 0;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint32_t want = (total_chunks + kLT / 32 - 1) / (kLT / 32);
  const uint32_t grid = want < uint32_t(sms) * 8 ? want : uint32_t(sms) * 8;
  auto* p2 = reinterpret_cast<double2*>(partial);
  if (dtype == RW_F64)
    lamb_pass1_kernel<double><<<grid, kLT, 0, st>>>(
        static_cast<const double*>(x), static_cast<double*>(g), static_cast<const double*>(grad),
        static_cast<double*>(m), static_cast<double*>(v), work, n_work, total_chunks, chunk_elems, sets, u, p2);
  else
    lamb_pass1_kernel<float><<<grid, kLT, 0, st>>>(
        static_cast<const float*>(x), static_cast<float*>(g), static_cast<const float*>(grad),
        static_cast<float*>(m), static_cast<float*>(v), work, n_work, total_chunks, chunk_elems, sets, u, p2);
  if (sequential) {
    if (dtype == RW_F64)
      lamb_seq_norms_kernel<double><<<n_work, 32, 0, st>>>(static_cast<const double*>(x), static_cast<const double*>(m),
                                                           static_cast<const double*>(v), work, sets, u, p2);
    else
      lamb_seq_norms_kernel<float><<<n_work, 32, 0, st>>>(static_cast<const float*>(x), static_cast<const float*>(m),
                                                          static_cast<const float*>(v), work, sets, u, p2);
  }
  lamb_trust_kernel<<<n_work, kLT, 0, st>>>(work, p2, u.wd, trust_table, depth, sets);
  return static_cast<int>(cudaGetLastError());
}

}  // namespace rwb
