// Fused optimizer step / inverse-step ("update-undo") kernels for sm_100a.
//
// One launch covers a whole list of parameter groups (multi-tensor apply over
// the flat state).  Per element it performs exactly the IEEE operation
// sequence of the reference loops in optim.cpp (cited per kind below), with
// every operation an explicit round-to-nearest intrinsic so no FMA
// contraction can occur regardless of -fmad (the library is also built with
// -fmad=false).  The same pass:
//   * caches the incoming gradient into g (optim.cpp:349, `block.g = grad`),
//   * evaluates check_finite on x, m, v (optim.cpp:361-363 / :382-384) as a
//     per-group non-finite flag (no extra HBM pass),
//   * rewrites the group's update-progress marker (t, updated;
//     optim.cpp:359-360 / :380-381) after the group's last element is stored
//     (last-CTA-done counter behind a gpu-scope fence).
//
// HBM layout: x, g, m, v are separate flat arrays (SoA), groups padded to
// 64-element (256 B) boundaries by the host layout builder, so the body uses
// 128-bit loads/stores (float4 / double2) with streaming cache hints.
// Work unit = one chunk of `chunk_elems` elements of one group; a persistent
// grid of (#SMs x resident CTAs) walks the chunk space with a static stride.
#include <cuda_runtime.h>

#include <cstdint>

#include "internal.h"

namespace rwb {
namespace {

template <typename T>
struct Arith;

template <>
struct Arith<float> {
  using V = float4;
  static constexpr int EV = 4;
  __device__ __forceinline__ static float mul(float a, float b) { return __fmul_rn(a, b); }
  __device__ __forceinline__ static float add(float a, float b) { return __fadd_rn(a, b); }
  __device__ __forceinline__ static float sub(float a, float b) { return __fsub_rn(a, b); }
  __device__ __forceinline__ static float div(float a, float b) { return __fdiv_rn(a, b); }
  __device__ __forceinline__ static float sqrt(float a) { return __fsqrt_rn(a); }
  __device__ __forceinline__ static bool nonfinite(float a) {
    return (__float_as_uint(a) & 0x7f800000u) == 0x7f800000u;
  }
  __device__ __forceinline__ static float cvt(double d) { return static_cast<float>(d); }
};

template <>
struct Arith<double> {
  using V = double2;
  static constexpr int EV = 2;
  __device__ __forceinline__ static double mul(double a, double b) { return __dmul_rn(a, b); }
  __device__ __forceinline__ static double add(double a, double b) { return __dadd_rn(a, b); }
  __device__ __forceinline__ static double sub(double a, double b) { return __dsub_rn(a, b); }
  __device__ __forceinline__ static double div(double a, double b) { return __ddiv_rn(a, b); }
  __device__ __forceinline__ static double sqrt(double a) { return __dsqrt_rn(a); }
  __device__ __forceinline__ static bool nonfinite(double a) {
    return (static_cast<unsigned long long>(__double_as_longlong(a)) & 0x7ff0000000000000ull) ==
           0x7ff0000000000000ull;
  }
  __device__ __forceinline__ static double cvt(double d) { return d; }
};

template <typename T>
struct Sc {
  T eta, c1, c2, denom, wd, mu, omd, b1, b2, omb1, omb2, eps;
};

// ---- the per-element expression trees (Appendix A of SURVEY.md) ----
template <int KIND, bool UNDO, typename T>
__device__ __forceinline__ void elem(const Sc<T>& s, T& x, T g, T& m, T& v, T& vmax) {
  using A = Arith<T>;
  if constexpr (KIND == RW_SGD) {
    if constexpr (!UNDO) {
      // optim.cpp:179  x -= eta * (g + wd * x)
      x = A::sub(x, A::mul(s.eta, A::add(g, A::mul(s.wd, x))));
    } else {
      // optim.cpp:187  x = (x + eta * g) / denom
      x = A::div(A::add(x, A::mul(s.eta, g)), s.denom);
    }
  } else if constexpr (KIND == RW_SGDM) {
    if constexpr (!UNDO) {
      // optim.cpp:193-195
      T gd = A::add(g, A::mul(s.wd, x));
      m = A::add(A::mul(s.mu, m), A::mul(s.omd, gd));
      x = A::sub(x, A::mul(s.eta, m));
    } else {
      // optim.cpp:202-205
      T xt = A::add(x, A::mul(s.eta, m));
      T gd = A::add(g, A::mul(s.wd, xt));
      m = A::div(A::sub(m, A::mul(s.omd, gd)), s.mu);
      x = xt;
    }
  } else if constexpr (KIND == RW_ADAM || KIND == RW_AMSGRAD) {
    if constexpr (!UNDO) {
      // optim.cpp:212-217 (Adam) / :326-332 (AMSGrad)
      T gd = A::add(g, A::mul(s.wd, x));
      m = A::add(A::mul(s.b1, m), A::mul(s.omb1, gd));
      v = A::add(A::mul(s.b2, v), A::mul(A::mul(s.omb2, gd), gd));
      T den_src = v;
      if constexpr (KIND == RW_AMSGRAD) {
        vmax = (vmax < v) ? v : vmax;  // std::max(vmax, v)
        den_src = vmax;
      }
      T mhat = A::div(m, s.c1);
      T vhat = A::div(den_src, s.c2);
      x = A::sub(x, A::div(A::mul(s.eta, mhat), A::add(A::sqrt(vhat), s.eps)));
    } else {
      // optim.cpp:227-233 (Adam only; AMSGrad undo is refused on the host)
      T mhat = A::div(m, s.c1);
      T vhat = A::div(v, s.c2);
      T xt = A::add(x, A::div(A::mul(s.eta, mhat), A::add(A::sqrt(vhat), s.eps)));
      T gd = A::add(g, A::mul(s.wd, xt));
      m = A::div(A::sub(m, A::mul(s.omb1, gd)), s.b1);
      v = A::div(A::sub(v, A::mul(A::mul(s.omb2, gd), gd)), s.b2);
      x = xt;
    }
  } else if constexpr (KIND == RW_ADAMW) {
    if constexpr (!UNDO) {
      // optim.cpp:241-247
      T gd = g;
      m = A::add(A::mul(s.b1, m), A::mul(s.omb1, gd));
      v = A::add(A::mul(s.b2, v), A::mul(A::mul(s.omb2, gd), gd));
      T mhat = A::div(m, s.c1);
      T vhat = A::div(v, s.c2);
      x = A::sub(x, A::mul(s.eta, A::add(A::div(mhat, A::add(A::sqrt(vhat), s.eps)),
                                         A::mul(s.wd, x))));
    } else {
      // optim.cpp:259-265
      T mhat = A::div(m, s.c1);
      T vhat = A::div(v, s.c2);
      T xt = A::div(A::add(x, A::div(A::mul(s.eta, mhat), A::add(A::sqrt(vhat), s.eps))),
                    s.denom);
      T gd = g;
      m = A::div(A::sub(m, A::mul(s.omb1, gd)), s.b1);
      v = A::div(A::sub(v, A::mul(A::mul(s.omb2, gd), gd)), s.b2);
      x = xt;
    }
  }
}

template <int KIND>
struct Uses {
  static constexpr bool m = KIND != RW_SGD;
  static constexpr bool v = KIND == RW_ADAM || KIND == RW_ADAMW || KIND == RW_AMSGRAD;
  static constexpr bool vmax = KIND == RW_AMSGRAD;
};

// streaming 128-bit accesses (read-once / write-once data, footprint >> L2)
template <typename V>
__device__ __forceinline__ V ld_stream(const V* p) {
  return __ldcs(p);
}
template <typename V>
__device__ __forceinline__ void st_stream(V* p, const V& v) {
  __stcs(p, v);
}

template <typename T>
__device__ __forceinline__ T comp(const typename Arith<T>::V& v, int i);
template <>
__device__ __forceinline__ float comp<float>(const float4& v, int i) {
  return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
}
template <>
__device__ __forceinline__ double comp<double>(const double2& v, int i) {
  return i == 0 ? v.x : v.y;
}
template <typename T>
__device__ __forceinline__ void set_comp(typename Arith<T>::V& v, int i, T val);
template <>
__device__ __forceinline__ void set_comp<float>(float4& v, int i, float val) {
  if (i == 0) v.x = val;
  else if (i == 1) v.y = val;
  else if (i == 2) v.z = val;
  else v.w = val;
}
template <>
__device__ __forceinline__ void set_comp<double>(double2& v, int i, double val) {
  if (i == 0) v.x = val;
  else v.y = val;
}

constexpr int kThreads = 256;
constexpr int kUnroll = 2;

template <typename T, int KIND, bool UNDO, bool COPY_GRAD>
__global__ void __launch_bounds__(kThreads) optim_kernel(
    T* __restrict__ x, T* __restrict__ g, T* __restrict__ m, T* __restrict__ v,
    T* __restrict__ vmax, const T* __restrict__ grad, const WorkItem* __restrict__ work,
    uint32_t n_work, uint32_t total_chunks, uint32_t chunk_elems,
    const ScalarSet* __restrict__ sets, Uniform u, rw_group* __restrict__ groups,
    uint32_t* __restrict__ done) {
  using A = Arith<T>;
  using V = typename A::V;
  constexpr int EV = A::EV;
  using U = Uses<KIND>;

  Sc<T> s;
  s.wd = A::cvt(u.wd);
  s.mu = A::cvt(u.mu);
  s.omd = A::cvt(u.one_m_damp);
  s.b1 = A::cvt(u.b1);
  s.b2 = A::cvt(u.b2);
  s.omb1 = A::cvt(u.one_m_b1);
  s.omb2 = A::cvt(u.one_m_b2);
  s.eps = A::cvt(u.eps);

  for (uint32_t chunk = blockIdx.x; chunk < total_chunks; chunk += gridDim.x) {
    // locate the work item owning this chunk (items sorted by chunk_begin)
    uint32_t lo = 0, hi = n_work;
    while (hi - lo > 1) {
      uint32_t mid = (lo + hi) >> 1;
      if (__ldg(&work[mid].chunk_begin) <= chunk) lo = mid;
      else hi = mid;
    }
    const WorkItem& it = work[lo];
    const ScalarSet ss = sets[it.sidx];
    s.eta = A::cvt(ss.eta);
    s.c1 = A::cvt(ss.c1);
    s.c2 = A::cvt(ss.c2);
    s.denom = A::cvt(ss.denom);

    const uint64_t cbeg = it.off + uint64_t(chunk - it.chunk_begin) * chunk_elems;
    uint64_t cend = cbeg + chunk_elems;
    const uint64_t gend = it.off + it.len;
    if (cend > gend) cend = gend;
    // aligned vector body [vb, ve)
    uint64_t vb = (cbeg + EV - 1) / EV * EV;
    if (vb > cend) vb = cend;
    const uint64_t ve = vb + (cend - vb) / EV * EV;

    bool bad = false;
    T dummy_v = T(0), dummy_vm = T(0), dummy_m = T(0);

    for (uint64_t base = vb + uint64_t(threadIdx.x) * EV; base < ve;
         base += uint64_t(kThreads) * EV * kUnroll) {
      V xr[kUnroll], gr[kUnroll], mr[kUnroll], vr[kUnroll], wr[kUnroll];
#pragma unroll
      for (int k = 0; k < kUnroll; ++k) {
        const uint64_t i = base + uint64_t(k) * kThreads * EV;
        if (i < ve) {
          xr[k] = ld_stream(reinterpret_cast<const V*>(x + i));
          if constexpr (COPY_GRAD) gr[k] = ld_stream(reinterpret_cast<const V*>(grad + i));
          else gr[k] = ld_stream(reinterpret_cast<const V*>(g + i));
          if constexpr (U::m) mr[k] = ld_stream(reinterpret_cast<const V*>(m + i));
          if constexpr (U::v) vr[k] = ld_stream(reinterpret_cast<const V*>(v + i));
          if constexpr (U::vmax) wr[k] = ld_stream(reinterpret_cast<const V*>(vmax + i));
        }
      }
#pragma unroll
      for (int k = 0; k < kUnroll; ++k) {
        const uint64_t i = base + uint64_t(k) * kThreads * EV;
        if (i < ve) {
#pragma unroll
          for (int e = 0; e < EV; ++e) {
            T xe = comp<T>(xr[k], e), ge = comp<T>(gr[k], e);
            T me = U::m ? comp<T>(mr[k], e) : dummy_m;
            T ve_ = U::v ? comp<T>(vr[k], e) : dummy_v;
            T we = U::vmax ? comp<T>(wr[k], e) : dummy_vm;
            elem<KIND, UNDO, T>(s, xe, ge, me, ve_, we);
            bad |= A::nonfinite(xe);
            set_comp<T>(xr[k], e, xe);
            if constexpr (U::m) {
              bad |= A::nonfinite(me);
              set_comp<T>(mr[k], e, me);
            }
            if constexpr (U::v) {
              bad |= A::nonfinite(ve_);
              set_comp<T>(vr[k], e, ve_);
            }
            if constexpr (U::vmax) set_comp<T>(wr[k], e, we);
          }
          st_stream(reinterpret_cast<V*>(x + i), xr[k]);
          if constexpr (COPY_GRAD) st_stream(reinterpret_cast<V*>(g + i), gr[k]);
          if constexpr (U::m) st_stream(reinterpret_cast<V*>(m + i), mr[k]);
          if constexpr (U::v) st_stream(reinterpret_cast<V*>(v + i), vr[k]);
          if constexpr (U::vmax) st_stream(reinterpret_cast<V*>(vmax + i), wr[k]);
        }
      }
    }
    // unaligned head [cbeg, vb) and tail [ve, cend): scalar
    {
      const uint64_t nh = vb - cbeg, nt = cend - ve;
      for (uint64_t j = threadIdx.x; j < nh + nt; j += kThreads) {
        const uint64_t i = j < nh ? cbeg + j : ve + (j - nh);
        T xe = x[i];
        T ge = COPY_GRAD ? grad[i] : g[i];
        T me = U::m ? m[i] : T(0);
        T ve_ = U::v ? v[i] : T(0);
        T we = U::vmax ? vmax[i] : T(0);
        elem<KIND, UNDO, T>(s, xe, ge, me, ve_, we);
        bad |= A::nonfinite(xe);
        x[i] = xe;
        if constexpr (COPY_GRAD) g[i] = ge;
        if constexpr (U::m) {
          bad |= A::nonfinite(me);
          m[i] = me;
        }
        if constexpr (U::v) {
          bad |= A::nonfinite(ve_);
          v[i] = ve_;
        }
        if constexpr (U::vmax) vmax[i] = we;
      }
    }

    // chunk done: publish the non-finite flag and, for the group's last
    // chunk, the update-progress marker.
    const int any_bad = __syncthreads_or(bad ? 1 : 0);
    if (threadIdx.x == 0) {
      if (any_bad) atomicOr(&groups[it.gid].flags, 1u);
      __threadfence();
      const uint32_t prev = atomicAdd(&done[lo], 1u);
      if (prev == it.nchunks - 1) {
        groups[it.gid].t = it.new_t;
        groups[it.gid].updated = UNDO ? 0u : 1u;
        done[lo] = 0u;
        __threadfence();
      }
    }
  }
}

template <typename T, int KIND, bool UNDO, bool COPY_GRAD>
int launch_t(const LaunchArgs& a, cudaStream_t st) {
  auto kern = optim_kernel<T, KIND, UNDO, COPY_GRAD>;
  static int blocks_per_sm = -1;  // per instantiation
  static int num_sms = -1;
  if (blocks_per_sm < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, kern, kThreads, 0);
    if (blocks_per_sm < 1) blocks_per_sm = 1;
  }
  uint32_t grid = static_cast<uint32_t>(num_sms * blocks_per_sm);
  if (grid > a.total_chunks) grid = a.total_chunks;
  if (grid == 0) return 0;
  kern<<<grid, kThreads, 0, st>>>(static_cast<T*>(a.x), static_cast<T*>(a.g), static_cast<T*>(a.m),
                                  static_cast<T*>(a.v), static_cast<T*>(a.vmax),
                                  static_cast<const T*>(a.grad), a.work, a.n_work, a.total_chunks,
                                  a.chunk_elems, a.sets, a.u, a.groups, a.done);
  return static_cast<int>(cudaGetLastError());
}

template <typename T, int KIND>
int launch_kind(const LaunchArgs& a, cudaStream_t st) {
  const bool copy = a.grad != nullptr && a.grad != a.g;
  if (a.undo) {
    if constexpr (KIND == RW_AMSGRAD || KIND == RW_LAMB) {
      return static_cast<int>(cudaErrorInvalidValue);
    } else {
      return launch_t<T, KIND, true, false>(a, st);
    }
  }
  if constexpr (KIND == RW_LAMB) {
    return static_cast<int>(cudaErrorInvalidValue);
  } else {
    return copy ? launch_t<T, KIND, false, true>(a, st) : launch_t<T, KIND, false, false>(a, st);
  }
}

template <typename T>
int launch_dtype(const LaunchArgs& a, cudaStream_t st) {
  switch (a.kind) {
    case RW_SGD: return launch_kind<T, RW_SGD>(a, st);
    case RW_SGDM: return launch_kind<T, RW_SGDM>(a, st);
    case RW_ADAM: return launch_kind<T, RW_ADAM>(a, st);
    case RW_ADAMW: return launch_kind<T, RW_ADAMW>(a, st);
    case RW_AMSGRAD: return launch_kind<T, RW_AMSGRAD>(a, st);
    default: return static_cast<int>(cudaErrorInvalidValue);
  }
}

// ---- seeded_fill on the device (tensor.cpp:69-103) ----
__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

template <typename T>
__global__ void seeded_fill_kernel(T* __restrict__ out, uint64_t n, uint64_t seed_mixed,
                                   uint64_t offset) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t idx = offset + i;
    const uint64_t r = mix64(seed_mixed ^ (idx * 0x9E3779B97F4A7C15ull + 1));
    // unit = (r >> 11) * 2^-53 exactly; (unit * 2 - 1) exact; * 0.1 one rounding
    const double unit = __dmul_rn(static_cast<double>(r >> 11), 0x1.0p-53);
    const double val = __dmul_rn(__dsub_rn(__dmul_rn(unit, 2.0), 1.0), 0.1);
    out[i] = static_cast<T>(val);
  }
}

// ---- ordered_sum (tensor.cpp:105-117) ----
constexpr int kMaxSum = 64;
struct SumPtrs {
  const void* p[kMaxSum];
};
template <typename T>
__global__ void ordered_sum_kernel(SumPtrs ptrs, uint32_t count, uint64_t n, T* __restrict__ out,
                                   bool accumulate) {
  using A = Arith<T>;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    T acc = accumulate ? out[i] : static_cast<const T*>(ptrs.p[0])[i];
    for (uint32_t k = accumulate ? 0u : 1u; k < count; ++k)
      acc = A::add(acc, static_cast<const T*>(ptrs.p[k])[i]);
    out[i] = acc;
  }
}

constexpr int kMaxClear = 1024;
struct ClearIds {
  uint32_t id[kMaxClear];
};
__global__ void clear_updated_kernel(rw_group* groups, ClearIds ids, uint32_t n) {
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) groups[ids.id[i]].updated = 0u;
}

int grid_for(uint64_t n, int threads) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  uint64_t want = (n + threads - 1) / threads;
  uint64_t cap = uint64_t(sms) * 8;
  return static_cast<int>(want < cap ? (want ? want : 1) : cap);
}

}  // namespace

uint32_t chunk_elems_for(int dtype) { return dtype == RW_F64 ? 4096u : 8192u; }

int launch_optim(const LaunchArgs& a, void* stream) {
  auto st = static_cast<cudaStream_t>(stream);
  if (a.total_chunks == 0) return 0;
  return a.dtype == RW_F64 ? launch_dtype<double>(a, st) : launch_dtype<float>(a, st);
}

int launch_seeded_fill(int dtype, void* out, uint64_t n, uint64_t seed, uint64_t offset,
                       void* stream) {
  if (n == 0) return 0;
  auto st = static_cast<cudaStream_t>(stream);
  const uint64_t sm = [&] {
    uint64_t x = seed;
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
  }();
  const int grid = grid_for(n, 256);
  if (dtype == RW_F64)
    seeded_fill_kernel<double><<<grid, 256, 0, st>>>(static_cast<double*>(out), n, sm, offset);
  else
    seeded_fill_kernel<float><<<grid, 256, 0, st>>>(static_cast<float*>(out), n, sm, offset);
  return static_cast<int>(cudaGetLastError());
}

int launch_ordered_sum(int dtype, const void* const* tensors, uint32_t count, uint64_t n, void* out,
                       void* stream) {
  if (n == 0 || count == 0) return 0;
  auto st = static_cast<cudaStream_t>(stream);
  const int grid = grid_for(n, 256);
  for (uint32_t base = 0; base < count; base += kMaxSum) {
    SumPtrs p{};
    const uint32_t c = count - base < kMaxSum ? count - base : kMaxSum;
    for (uint32_t k = 0; k < c; ++k) p.p[k] = tensors[base + k];
    if (dtype == RW_F64)
      ordered_sum_kernel<double><<<grid, 256, 0, st>>>(p, c, n, static_cast<double*>(out), base > 0);
    else
      ordered_sum_kernel<float><<<grid, 256, 0, st>>>(p, c, n, static_cast<float*>(out), base > 0);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return static_cast<int>(e);
  }
  return 0;
}

int launch_clear_updated(rw_group* groups, const uint32_t* ids, uint32_t n, void* stream) {
  auto st = static_cast<cudaStream_t>(stream);
  for (uint32_t base = 0; base < n; base += kMaxClear) {
    ClearIds c;
    const uint32_t k = n - base < kMaxClear ? n - base : kMaxClear;
    for (uint32_t i = 0; i < k; ++i) c.id[i] = ids[base + i];
    clear_updated_kernel<<<1, 256, 0, st>>>(groups, c, k);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return static_cast<int>(e);
  }
  return 0;
}

}  // namespace rwb
