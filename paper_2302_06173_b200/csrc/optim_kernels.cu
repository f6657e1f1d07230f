// Fused optimizer step / inverse-step ("update-undo") kernels for sm_100a.
//
// One launch covers a whole list of parameter groups (multi-tensor apply over
// the flat state).  Per element it performs exactly the IEEE operation
// sequence of the reference loops in optim.cpp (cited per kind below), every
// operation an explicit round-to-nearest intrinsic so no FMA contraction can
// occur regardless of -fmad (the library is also built with -fmad=false).
// The same pass:
//   * caches the incoming gradient into g (optim.cpp:271, `block.g = grad`),
//   * evaluates check_finite on x, m, v (optim.cpp:283-285 / :304-306) as a
//     per-group non-finite flag (no extra HBM pass),
//   * rewrites the group's update-progress marker (t, updated;
//     optim.cpp:281-282 / :302-303) once the group's last tile is stored.
//
// Data movement (the kernel is HBM-bound: 28 B/param for Adam fp32):
//   x, g, m, v are separate flat arrays (SoA).  The state is cut into tiles
//   of 8 KB per stream (2048 fp32 / 1024 fp64 elements, never crossing a
//   group boundary).  A persistent grid of 2 CTAs/SM walks the tiles; each
//   CTA runs a 3-stage TMA bulk-copy pipeline:
//     cp.async.bulk global->smem (mbarrier complete_tx) for x, g, m, v
//     -> 256 threads compute in smem (128-bit ld/st.shared)
//     -> cp.async.bulk smem->global for x, (g), m, v (bulk_group)
//   The refill of a stage is deferred one tile (cp.async.bulk.wait_group 1),
//   so the producer never waits for the stores it just issued.  Measured on
//   B200 (tools/undo_variants.cu): 6.63 TB/s for the 1B-param Adam undo vs
//   6.0-6.3 TB/s for register-staged 128/256-bit LDG/STG variants.
// Ragged tile ends (groups are 256 B aligned by the layout builder, but the C
// ABI accepts any offset) are handled element-wise from global memory.
#include <cuda_bf16.h>
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
#ifdef RW_OPTIM_PROBE_NODIV  // probe only (wrong math): how much do the IEEE divides cost?
  __device__ __forceinline__ static float div(float a, float b) { return __fmul_rn(a, b); }
#else
  __device__ __forceinline__ static float div(float a, float b) { return __fdiv_rn(a, b); }
#endif
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
      // optim.cpp:101  x -= eta * (g + wd * x)
      x = A::sub(x, A::mul(s.eta, A::add(g, A::mul(s.wd, x))));
    } else {
      // optim.cpp:109  x = (x + eta * g) / denom
      x = A::div(A::add(x, A::mul(s.eta, g)), s.denom);
    }
  } else if constexpr (KIND == RW_SGDM) {
    if constexpr (!UNDO) {
      // optim.cpp:115-117
      T gd = A::add(g, A::mul(s.wd, x));
      m = A::add(A::mul(s.mu, m), A::mul(s.omd, gd));
      x = A::sub(x, A::mul(s.eta, m));
    } else {
      // optim.cpp:124-127
      T xt = A::add(x, A::mul(s.eta, m));
      T gd = A::add(g, A::mul(s.wd, xt));
      m = A::div(A::sub(m, A::mul(s.omd, gd)), s.mu);
      x = xt;
    }
  } else if constexpr (KIND == RW_ADAM || KIND == RW_AMSGRAD) {
    if constexpr (!UNDO) {
      // optim.cpp:134-139 (Adam) / :248-254 (AMSGrad)
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
      // optim.cpp:149-155 (Adam only; AMSGrad undo is refused on the host)
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
      // optim.cpp:163-169
      T gd = g;
      m = A::add(A::mul(s.b1, m), A::mul(s.omb1, gd));
      v = A::add(A::mul(s.b2, v), A::mul(A::mul(s.omb2, gd), gd));
      T mhat = A::div(m, s.c1);
      T vhat = A::div(v, s.c2);
      x = A::sub(x, A::mul(s.eta, A::add(A::div(mhat, A::add(A::sqrt(vhat), s.eps)),
                                         A::mul(s.wd, x))));
    } else {
      // optim.cpp:181-187
      T mhat = A::div(m, s.c1);
      T vhat = A::div(v, s.c2);
      T xt = A::div(A::add(x, A::div(A::mul(s.eta, mhat), A::add(A::sqrt(vhat), s.eps))),
                    s.denom);
      T gd = g;
      m = A::div(A::sub(m, A::mul(s.omb1, gd)), s.b1);
      v = A::div(A::sub(v, A::mul(A::mul(s.omb2, gd), gd)), s.b2);
      x = xt;
    }
  } else if constexpr (KIND == RW_LAMB) {
    // s.eta carries scaled = eta * trust (the saved ratio) for LAMB.
    if constexpr (!UNDO) {
      // second pass of step_lamb, optim.cpp:204-215: m, v already advanced
      // by lamb_pass1_kernel; x -= (eta * trust) * update
      T mhat = A::div(m, s.c1);
      T vhat = A::div(v, s.c2);
      T u = A::add(A::div(mhat, A::add(A::sqrt(vhat), s.eps)), A::mul(s.wd, x));
      x = A::sub(x, A::mul(s.eta, u));
    } else {
      // optim.cpp:231-240 with scaled = eta * trust, denom = 1 - scaled * wd
      T mhat = A::div(m, s.c1);
      T vhat = A::div(v, s.c2);
      T r = A::div(mhat, A::add(A::sqrt(vhat), s.eps));
      T xt = A::div(A::add(x, A::mul(s.eta, r)), s.denom);
      T gd = g;
      m = A::div(A::sub(m, A::mul(s.omb1, gd)), s.b1);
      v = A::div(A::sub(v, A::mul(A::mul(s.omb2, gd), gd)), s.b2);
      x = xt;
    }
  }
}

template <int KIND>
struct Uses {
  // g is read by every pass except LAMB's step x-pass (its gradient was
  // consumed by the norm pass)
  template <bool UNDO>
  static constexpr bool g = !(KIND == RW_LAMB && !UNDO);
  static constexpr bool m = KIND != RW_SGD;
  static constexpr bool v = KIND == RW_ADAM || KIND == RW_ADAMW || KIND == RW_AMSGRAD || KIND == RW_LAMB;
  static constexpr bool vmax = KIND == RW_AMSGRAD;
  static constexpr int slots = vmax ? 5 : 4;
};

// ---- PTX wrappers: mbarrier + bulk async copies (TMA, non-tensor) ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
               "r"(bytes)
               : "memory");
}
#ifndef RW_OPTIM_WAIT_HINT_NS
#define RW_OPTIM_WAIT_HINT_NS 0
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
#if RW_OPTIM_WAIT_HINT_NS
  // suspend-time hint: waiting warps are parked until the tile lands
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity), "r"(uint32_t(RW_OPTIM_WAIT_HINT_NS))
      : "memory");
#else
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
#endif
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(b))
      : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
// the same with an L2 eviction-priority policy (createpolicy)
__device__ __forceinline__ void bulk_load_hint(void* dst, const void* src, uint32_t bytes, uint64_t* b,
                                               uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(b)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void bulk_store_hint(void* dst, const void* src, uint32_t bytes, uint64_t pol) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes), "l"(pol)
               : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
// ... only until their shared-memory sources have been read (the stage can be
// refilled; the global writes may still be in flight)
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

#ifndef RW_OPTIM_THREADS
#define RW_OPTIM_THREADS 256
#endif
constexpr int kThreads = RW_OPTIM_THREADS;
#ifndef RW_OPTIM_STAGES
#define RW_OPTIM_STAGES 3
#endif
#ifndef RW_OPTIM_SLOT_BYTES
#define RW_OPTIM_SLOT_BYTES 8192
#endif
#ifndef RW_OPTIM_WAIT_READ
#define RW_OPTIM_WAIT_READ 0
#endif
#ifndef RW_OPTIM_INTERLEAVE
#define RW_OPTIM_INTERLEAVE 0
#endif
#ifndef RW_OPTIM_L2HINT
#define RW_OPTIM_L2HINT 0
#endif
#ifndef RW_OPTIM_MIN_BLOCKS
#define RW_OPTIM_MIN_BLOCKS 1
#endif
constexpr int kStages = RW_OPTIM_STAGES;  // smem stages (3 x 8 KB slots: 2 CTAs per SM)
// fused NVLink push: 4 stages (2 tiles of stores in flight, 1 CTA per SM)
// measured no faster than 3 (GPT-2 XL push 29.8 vs 29.9 ms), so 3
constexpr int kStagesPush = 3;
constexpr int kStagesMax = kStages > 4 ? kStages : 4;
constexpr uint32_t kSlotBytes = RW_OPTIM_SLOT_BYTES;  // per stream per stage

// per-stage tile descriptor, written by the producer thread before it arms
// the stage's mbarrier (release) and read by all threads after the wait
// (acquire)
struct StageMeta {
  uint64_t a;      // first element of the tile
  uint64_t a16;    // first element of the 16-byte-aligned bulk part
  uint32_t nbulk;  // elements moved by TMA
  uint32_t nhead;  // unaligned elements before a16 (global access)
  uint32_t ntail;  // unaligned elements after the bulk part
  uint32_t item;   // work item index
  uint32_t gid;    // group (marker table index)
  uint32_t bad;    // non-finite seen in this tile
  uint32_t copy;   // copy-only tile (fused push of an untouched group)
  uint32_t pad;
  ScalarSet ss;    // eta, c1, c2, denom of the tile's group
};

template <bool PUSH>
constexpr int stages_for() {
  return PUSH ? kStagesPush : kStages;
}
template <typename T, int KIND, bool PUSH>
constexpr size_t dyn_smem_bytes() {
  return size_t(stages_for<PUSH>()) * Uses<KIND>::slots * kSlotBytes;
}

// PUSH: the resolved tiles are also written to a peer replica (NVLink stores
// from the same bulk-copy engine), and copy-only work items pass untouched
// groups through to the peer: recover_replication fused with apply_undo.
template <typename T, int KIND, bool UNDO, bool COPY_GRAD, bool PUSH>
__global__ void __launch_bounds__(kThreads, RW_OPTIM_MIN_BLOCKS) optim_kernel(
    T* __restrict__ x, T* __restrict__ g, T* __restrict__ m, T* __restrict__ v,
    T* __restrict__ vmax, const T* __restrict__ grad, const WorkItem* __restrict__ work,
    uint32_t n_work, uint32_t total_chunks, const ScalarSet* __restrict__ sets, Uniform u,
    rw_group* __restrict__ groups, uint32_t* __restrict__ done, T* __restrict__ px,
    T* __restrict__ pg, T* __restrict__ pm, T* __restrict__ pv, const __grid_constant__ InlineMeta inl) {
  if (work == nullptr) {  // small call: metadata in the parameter space
    work = inl.work;
    sets = inl.sets;
  }
  using A = Arith<T>;
  using V = typename A::V;
  constexpr int EV = A::EV;
  using U = Uses<KIND>;
  constexpr int NS = U::slots;
  constexpr uint32_t TILE = kSlotBytes / sizeof(T);
  constexpr int SX = 0, SG = 1, SM = 2, SV = 3, SW = 4;

  extern __shared__ __align__(128) unsigned char smem_raw[];
  constexpr int S = stages_for<PUSH>();
  constexpr int D = S - 2;  // tiles whose stores may still be in flight
  __shared__ uint64_t full[kStagesMax];
  __shared__ StageMeta meta[kStagesMax];
  T* const buf = reinterpret_cast<T*>(smem_raw);
  auto slot = [&](int st, int k) { return buf + (size_t(st) * NS + k) * TILE; };
  const T* gsrc = COPY_GRAD ? grad : g;
  const uint32_t tid = threadIdx.x;

  Sc<T> s;
  s.wd = A::cvt(u.wd);
  s.mu = A::cvt(u.mu);
  s.omd = A::cvt(u.one_m_damp);
  s.b1 = A::cvt(u.b1);
  s.b2 = A::cvt(u.b2);
  s.omb1 = A::cvt(u.one_m_b1);
  s.omb2 = A::cvt(u.one_m_b2);
  s.eps = A::cvt(u.eps);

  // The chunks a CTA visits increase monotonically, so the producer walks the
  // work list with a cursor and only touches global metadata when it
  // crosses into the next group.  Contiguous: each CTA owns one range of
  // chunks.  Interleaved: CTA b visits b, b + grid, b + 2 grid, ... so the
  // whole grid sweeps one compact window of every stream at a time.
#if RW_OPTIM_INTERLEAVE
  const uint32_t n_mine = total_chunks > blockIdx.x ? (total_chunks - blockIdx.x + gridDim.x - 1) / gridDim.x : 0u;
  auto chunk_of = [&](uint32_t j) { return blockIdx.x + j * gridDim.x; };
#else
  const uint32_t per_cta = (total_chunks + gridDim.x - 1) / gridDim.x;
  const uint32_t c_begin = min(total_chunks, blockIdx.x * per_cta);
  const uint32_t n_mine = min(total_chunks, c_begin + per_cta) - c_begin;
  auto chunk_of = [&](uint32_t j) { return c_begin + j; };
#endif

  // producer-only state (thread 0): cached current work item
  uint32_t cur = 0, cur_cb = 0, cur_nc = 0, cur_gid = 0, cur_flags = 0;
  uint64_t cur_off = 0, cur_len = 0;
  ScalarSet cur_ss{};
  auto load_item = [&](uint32_t i) {
    const WorkItem& it = work[i];
    cur = i;
    cur_cb = it.chunk_begin;
    cur_nc = it.nchunks;
    cur_off = it.off;
    cur_len = it.len;
    cur_gid = it.gid;
    cur_flags = it.flags;
    cur_ss = sets[it.sidx];
  };

  if (tid == 0) {
    for (int i = 0; i < S; ++i) mbar_init(&full[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (n_mine) {
      const uint32_t c0 = chunk_of(0);
      uint32_t lo = 0, hi = n_work;
      while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (work[mid].chunk_begin <= c0) lo = mid;
        else hi = mid;
      }
      load_item(lo);
    }
  }
  __syncthreads();

  // L2 policy of the streaming traffic (build option RW_OPTIM_L2HINT:
  // 1 = loads evict-first, 2 = loads and stores, 3 = stores only)
#if RW_OPTIM_L2HINT
  const uint64_t l2pol = policy_evict_first();
#if RW_OPTIM_L2HINT <= 2
  auto bulk_load = [&](void* dst, const void* src, uint32_t bytes, uint64_t* b) {
    bulk_load_hint(dst, src, bytes, b, l2pol);
  };
#endif
#if RW_OPTIM_L2HINT >= 2
  auto bulk_store = [&](void* dst, const void* src, uint32_t bytes) { bulk_store_hint(dst, src, bytes, l2pol); };
#endif
#endif
  // producer (thread 0): locate the tile, publish its descriptor, arm the
  // stage barrier with the byte count and launch the bulk loads
  auto issue = [&](uint32_t chunk, int st) {
    while (chunk >= cur_cb + cur_nc) load_item(cur + 1);
    const uint64_t a = cur_off + uint64_t(chunk - cur_cb) * TILE;
    uint64_t b = a + TILE;
    if (b > cur_off + cur_len) b = cur_off + cur_len;
    uint64_t a16 = (a + EV - 1) / EV * EV;
    if (a16 > b) a16 = b;
    const uint64_t b16 = a16 + (b - a16) / EV * EV;
    StageMeta& mt = meta[st];
    mt.a = a;
    mt.a16 = a16;
    mt.nbulk = static_cast<uint32_t>(b16 - a16);
    mt.nhead = static_cast<uint32_t>(a16 - a);
    mt.ntail = static_cast<uint32_t>(b - b16);
    mt.item = cur;
    mt.gid = cur_gid;
    mt.bad = 0;
    mt.copy = (PUSH && (cur_flags & kWorkCopyOnly)) ? 1u : 0u;
    mt.ss = cur_ss;
    const uint32_t bytes = mt.nbulk * sizeof(T);
    constexpr bool kG = U::template g<UNDO> || PUSH;
    constexpr int nload = 1 + (kG ? 1 : 0) + (U::m ? 1 : 0) + (U::v ? 1 : 0) + (U::vmax ? 1 : 0);
    mbar_expect_tx(&full[st], bytes * nload);
    if (bytes) {
      bulk_load(slot(st, SX), x + a16, bytes, &full[st]);
      if constexpr (kG) bulk_load(slot(st, SG), gsrc + a16, bytes, &full[st]);
      if constexpr (U::m) bulk_load(slot(st, SM), m + a16, bytes, &full[st]);
      if constexpr (U::v) bulk_load(slot(st, SV), v + a16, bytes, &full[st]);
      if constexpr (U::vmax) bulk_load(slot(st, SW), vmax + a16, bytes, &full[st]);
    }
  };
  // marker bookkeeping once tiles' stores are complete: completed tiles are
  // counted per item in a register and published with one atomic per
  // (CTA, group); the CTA that completes a group rewrites its marker.
  uint32_t acc_item = 0xFFFFFFFFu, acc_cnt = 0;
  auto flush = [&]() {
    if (acc_cnt == 0) return;
    const WorkItem& it = work[acc_item];
    if (PUSH && (it.flags & kWorkCopyOnly)) {  // untouched group: marker unchanged
      acc_cnt = 0;
      return;
    }
#if RW_OPTIM_WAIT_READ
    bulk_wait<0>();  // stages were recycled on read-out: the writes themselves must be complete
#endif
    __threadfence();
    const uint32_t prev = atomicAdd(&done[acc_item], acc_cnt);
    if (prev + acc_cnt == it.nchunks) {
      groups[it.gid].t = it.new_t;
      groups[it.gid].updated = UNDO ? 0u : 1u;
      done[acc_item] = 0u;
      __threadfence();
    }
    acc_cnt = 0;
  };
  auto account = [&](uint32_t item) {
    if (item != acc_item) {
      flush();
      acc_item = item;
    }
    ++acc_cnt;
  };

  if (tid == 0) {
    for (int k = 0; k < S; ++k)
      if (uint32_t(k) < n_mine) issue(chunk_of(uint32_t(k)), k);
  }

  uint32_t ring_item[D];  // the last D tiles' work items (thread 0)
  uint32_t iter = 0;
  for (; iter < n_mine; ++iter) {
    const int st = static_cast<int>(iter % S);
    mbar_wait(&full[st], (iter / S) & 1u);
    const StageMeta& mt = meta[st];
    s.eta = A::cvt(mt.ss.eta);
    s.c1 = A::cvt(mt.ss.c1);
    s.c2 = A::cvt(mt.ss.c2);
    s.denom = A::cvt(mt.ss.denom);
    const uint32_t nbulk = mt.nbulk, nhead = mt.nhead, ntail = mt.ntail;
    const uint64_t ma = mt.a, ma16 = mt.a16;

    bool bad = false;
    T* xs = slot(st, SX);
    T* gs = slot(st, SG);
    T* ms = slot(st, SM);
    T* vs = slot(st, SV);
    T* ws = slot(st, SW);
    T zero_m = T(0), zero_v = T(0), zero_w = T(0);
    auto body = [&](uint32_t e) {
      V xr = *reinterpret_cast<const V*>(xs + e);
      V gr{};
      if constexpr (U::template g<UNDO> || PUSH) gr = *reinterpret_cast<const V*>(gs + e);
      V mr, vr, wr;
      if constexpr (U::m) mr = *reinterpret_cast<const V*>(ms + e);
      if constexpr (U::v) vr = *reinterpret_cast<const V*>(vs + e);
      if constexpr (U::vmax) wr = *reinterpret_cast<const V*>(ws + e);
      T* xp = reinterpret_cast<T*>(&xr);
      const T* gp = reinterpret_cast<const T*>(&gr);
      T* mp = reinterpret_cast<T*>(&mr);
      T* vp = reinterpret_cast<T*>(&vr);
      T* wp = reinterpret_cast<T*>(&wr);
#pragma unroll
      for (int k = 0; k < EV; ++k) {
        T& me = U::m ? mp[k] : zero_m;
        T& ve = U::v ? vp[k] : zero_v;
        T& we = U::vmax ? wp[k] : zero_w;
        elem<KIND, UNDO, T>(s, xp[k], gp[k], me, ve, we);
        bad |= A::nonfinite(xp[k]);
        if constexpr (U::m) bad |= A::nonfinite(me);
        if constexpr (U::v) bad |= A::nonfinite(ve);
      }
      *reinterpret_cast<V*>(xs + e) = xr;
      if constexpr (U::m) *reinterpret_cast<V*>(ms + e) = mr;
      if constexpr (U::v) *reinterpret_cast<V*>(vs + e) = vr;
      if constexpr (U::vmax) *reinterpret_cast<V*>(ws + e) = wr;
    };
    const bool copy_only = PUSH && mt.copy;
    if (copy_only) {
      // untouched group: the loaded tile goes to the peer unchanged
    } else if (nbulk == TILE) {  // full tile: compile-time trip count, unrolled for ILP
      constexpr uint32_t kIters = TILE / (kThreads * EV);
#pragma unroll
      for (uint32_t k = 0; k < kIters; ++k) body(tid * EV + k * kThreads * EV);
    } else {
      for (uint32_t e = tid * EV; e < nbulk; e += kThreads * EV) body(e);
    }
    // unaligned head/tail elements straight from global memory
    if (copy_only && tid < nhead + ntail) {
      const uint64_t i = tid < nhead ? ma + tid : ma16 + nbulk + (tid - nhead);
      px[i] = x[i];
      if (pg) pg[i] = g[i];
      if constexpr (U::m) pm[i] = m[i];
      if constexpr (U::v) pv[i] = v[i];
    } else if (tid < nhead + ntail) {
      const uint64_t i = tid < nhead ? ma + tid : ma16 + nbulk + (tid - nhead);
      T xe = x[i];
      const T ge = gsrc[i];
      T me = U::m ? m[i] : T(0);
      T ve = U::v ? v[i] : T(0);
      T we = U::vmax ? vmax[i] : T(0);
      elem<KIND, UNDO, T>(s, xe, ge, me, ve, we);
      bad |= A::nonfinite(xe);
      x[i] = xe;
      if constexpr (COPY_GRAD) g[i] = ge;
      if constexpr (U::m) {
        bad |= A::nonfinite(me);
        m[i] = me;
      }
      if constexpr (U::v) {
        bad |= A::nonfinite(ve);
        v[i] = ve;
      }
      if constexpr (U::vmax) vmax[i] = we;
      if constexpr (PUSH) {
        px[i] = xe;
        if (pg) pg[i] = ge;
        if constexpr (U::m) pm[i] = me;
        if constexpr (U::v) pv[i] = ve;
      }
    }
    if (bad) atomicOr(&meta[st].bad, 1u);
    fence_proxy_async_smem();  // generic smem writes -> visible to the bulk stores
    __syncthreads();
    if (tid == 0) {
      if (nbulk) {
        const uint32_t bytes = nbulk * sizeof(T);
        if (!copy_only) {
          bulk_store(x + ma16, xs, bytes);
          if constexpr (COPY_GRAD) bulk_store(g + ma16, gs, bytes);
          if constexpr (U::m) bulk_store(m + ma16, ms, bytes);
          if constexpr (U::v) bulk_store(v + ma16, vs, bytes);
          if constexpr (U::vmax) bulk_store(vmax + ma16, ws, bytes);
        }
        if constexpr (PUSH) {  // NVLink: the peer replica receives the resolved tile
          bulk_store(px + ma16, xs, bytes);
          if (pg) bulk_store(pg + ma16, gs, bytes);
          if constexpr (U::m) bulk_store(pm + ma16, ms, bytes);
          if constexpr (U::v) bulk_store(pv + ma16, vs, bytes);
        }
      }
      bulk_commit();
      if (mt.bad) atomicOr(&groups[mt.gid].flags, 1u);
      const uint32_t this_item = mt.item;
      if (iter >= uint32_t(D)) {
#if RW_OPTIM_WAIT_READ
        bulk_wait_read<D>();  // tile iter-D's stores have read their stage: refill it
#else
        bulk_wait<D>();  // tile iter-D's stores are complete: its stage can be refilled
#endif
        const uint32_t r = (iter - D) % D;
        account(ring_item[r]);
        const uint32_t nj = iter - D + uint32_t(S);  // the stage's next tile
        if (nj < n_mine) issue(chunk_of(nj), static_cast<int>((iter - D) % S));
      }
      ring_item[iter % D] = this_item;
    }
  }
  if (tid == 0 && iter > 0) {
    bulk_wait<0>();
    for (uint32_t j = iter > uint32_t(D) ? iter - D : 0; j < iter; ++j) account(ring_item[j % D]);
    flush();
  }
}

const InlineMeta kNoInline{};

template <typename T, int KIND, bool UNDO, bool COPY_GRAD, bool PUSH = false>
int launch_t(const LaunchArgs& a, cudaStream_t st) {
  auto kern = optim_kernel<T, KIND, UNDO, COPY_GRAD, PUSH>;
  constexpr size_t smem = dyn_smem_bytes<T, KIND, PUSH>();
  static int blocks_per_sm = -1;  // per instantiation (same on every B200)
  static int num_sms = -1;
  static DeviceOnce once;
  const int se = once.run([&](int dev) {
    int sms = 0, bps = 0;
    cudaError_t e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, kThreads, smem);
    if (e != cudaSuccess) return static_cast<int>(e);
    num_sms = sms;
    blocks_per_sm = bps < 1 ? 1 : bps;
    return 0;
  });
  if (se) return se;
  uint32_t grid = static_cast<uint32_t>(num_sms * blocks_per_sm);
  if (grid > a.total_chunks) grid = a.total_chunks;
  if (grid == 0) return 0;
  kern<<<grid, kThreads, smem, st>>>(static_cast<T*>(a.x), static_cast<T*>(a.g),
                                     static_cast<T*>(a.m), static_cast<T*>(a.v),
                                     static_cast<T*>(a.vmax), static_cast<const T*>(a.grad), a.work,
                                     a.n_work, a.total_chunks, a.sets, a.u, a.groups, a.done,
                                     static_cast<T*>(a.px), static_cast<T*>(a.pg), static_cast<T*>(a.pm),
                                     static_cast<T*>(a.pv), a.inl ? *a.inl : kNoInline);
  return static_cast<int>(cudaGetLastError());
}

template <typename T, int KIND>
int launch_kind(const LaunchArgs& a, cudaStream_t st) {
  const bool copy = a.grad != nullptr && a.grad != a.g;
  if (a.undo) {
    if constexpr (KIND == RW_AMSGRAD) {
      return static_cast<int>(cudaErrorInvalidValue);
    } else {
      if (a.px) return launch_t<T, KIND, true, false, true>(a, st);
      return launch_t<T, KIND, true, false>(a, st);
    }
  }
  if constexpr (KIND == RW_LAMB) {
    // LAMB step pass 2 (x only); the gradient was cached by lamb_pass1_kernel
    return launch_t<T, KIND, false, false>(a, st);
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
    case RW_LAMB: return launch_kind<T, RW_LAMB>(a, st);
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
    if constexpr (sizeof(T) == 2) out[i] = __double2bfloat16(val);  // one rounding
    else out[i] = static_cast<T>(val);
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

uint32_t chunk_elems_for(int dtype) { return kSlotBytes / (dtype == RW_F64 ? 8u : 4u); }


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
  else if (dtype == RW_BF16)
    seeded_fill_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>(static_cast<__nv_bfloat16*>(out), n, sm, offset);
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
