// Host side of the C ABI (include/rewind_b200.h): guards, scalar derivation,
// marker bookkeeping and launch of the fused kernels.  Mirrors the control
// flow of optimizer_step / optimizer_undo (optim.cpp:260-307) group by group.
//
// Build note: compiled with -ffp-contract=off so the double scalars below are
// the same IEEE expressions the reference evaluates (optim.cpp:94-97, :106,
// :177) — glibc pow for the bias corrections, exactly as the reference.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "internal.h"

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  return fail(RW_CUDA_ERROR, "CUDA error in %s: %s", what, cudaGetErrorString(e));
}

#define RW_CUDA(call)                                   \
  do {                                                  \
    cudaError_t e_ = (call);                            \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
  } while (0)

const char* kErrNames[] = {"OK",           "InvalidShape",     "ShapeMismatch",  "EmptyInput",
                           "NumericalError", "NonInvertibleHyper", "NotInvertible", "NothingToUndo",
                           "AlreadyUpdated", "MissingActivation", "ChannelBroken", "InvalidInjection",
                           "NotFailed",    "StorageError",     "MissingLogData", "CorruptLog",
                           "NoCheckpoint", "NoReplica",        "InvalidConfig",  "TooLarge"};

const char* kind_name(int k) {
  switch (k) {
    case RW_SGD: return "sgd";
    case RW_SGDM: return "sgdm";
    case RW_ADAM: return "adam";
    case RW_ADAMW: return "adamw";
    case RW_LAMB: return "lamb";
    case RW_AMSGRAD: return "amsgrad";
  }
  return "?";
}

// OptimizerHyper::lr_at, optim.cpp:50-57
int lr_at(const rw_hyper* h, uint64_t t, double* out) {
  double v = h->lr;
  for (uint32_t i = 0; i < h->lr_table_len; ++i)
    if (t >= h->lr_table_from[i]) v = h->lr_table_value[i];
  if (!(v > 0.0)) return fail(RW_INVALID_CONFIG, "InvalidConfig: learning rate must be positive");
  *out = v;
  return RW_OK;
}

// Ring of per-launch metadata slots so back-to-back asynchronous calls never
// overwrite a work list that a queued copy/kernel still reads.
// The work list and the scalar sets of one launch sit back to back in one
// pinned and one device buffer, so a launch uploads its metadata with one copy.
struct Slot {
  uint8_t* h_buf = nullptr;  // pinned
  uint8_t* d_buf = nullptr;
  size_t buf_cap = 0;
  rwb::WorkItem* h_work = nullptr;   // views into h_buf / d_buf for the current launch
  rwb::ScalarSet* h_sets = nullptr;
  rwb::WorkItem* d_work = nullptr;
  rwb::ScalarSet* d_sets = nullptr;
  size_t meta_bytes = 0;             // work + sets of the current launch
  uint32_t* d_done = nullptr;
  uint32_t cap = 0;
  cudaEvent_t ev = nullptr;
  bool used = false;
};
constexpr int kSlots = 8;
constexpr uint32_t kTrustDepth = RW_LAMB_TRUST_DEPTH;

}  // namespace

namespace rwb {
void set_error(const char* msg) { g_err = msg; }
}  // namespace rwb

struct rw_state {
  int dtype = RW_F32;
  int device = 0;
  void* x = nullptr;
  void* g = nullptr;
  void* m = nullptr;
  void* v = nullptr;
  void* vmax = nullptr;
  uint64_t total = 0;
  std::vector<rw_group> mirror;  // host mirror of the marker table
  rw_group* d_groups = nullptr;
  Slot slots[kSlots];
  int next_slot = 0;
  // LAMB saved scalars (ParamBlock::saved_scalars, optim.cpp:216): a per-group
  // ring of the last kTrustDepth trust ratios, written by lamb_trust_kernel;
  // head/count are host-side so the stack top is known without a sync.
  double* d_trust = nullptr;       // [G * kTrustDepth]
  double* d_partial = nullptr;     // pass-1 scratch, 2 doubles per chunk
  uint64_t partial_cap = 0;
  std::vector<uint64_t> trust_head;
  std::vector<uint32_t> trust_count;
  uint32_t flags = 0;  // RW_STATE_* (rw_state_set_flags)
  // host-resident undo pipeline (rw_optimizer_undo_host)
  cudaStream_t h2d = nullptr;
  cudaStream_t d2h = nullptr;
  std::vector<cudaEvent_t> evs;
  // its staging ring: kHostRing slots of x, g, m, v slices (device memory
  // of its own, so the host-resident state may exceed HBM)
  void* ring[3][4] = {};
  uint64_t ring_cap = 0;  // elements per buffer
  bool host_resident = false;  // created by rw_state_create_host: no device x, g, m, v
};

namespace {

int ensure_slot(rw_state* s, Slot& sl, uint32_t n_items, uint32_t n_sets) {
  if (sl.used) RW_CUDA(cudaEventSynchronize(sl.ev));
  if (!sl.ev) RW_CUDA(cudaEventCreateWithFlags(&sl.ev, cudaEventDisableTiming));
  if (n_items > sl.cap) {
    cudaFree(sl.d_done);
    sl.d_done = nullptr;
    uint32_t cap = std::max<uint32_t>(n_items, 256);
    RW_CUDA(cudaMalloc(&sl.d_done, sizeof(uint32_t) * cap));
    RW_CUDA(cudaMemset(sl.d_done, 0, sizeof(uint32_t) * cap));
    sl.cap = cap;
  }
  static_assert(sizeof(rwb::WorkItem) % alignof(rwb::ScalarSet) == 0, "sets follow the work items");
  const size_t need = sizeof(rwb::WorkItem) * n_items + sizeof(rwb::ScalarSet) * n_sets;
  if (need > sl.buf_cap) {
    cudaFreeHost(sl.h_buf);
    cudaFree(sl.d_buf);
    sl.h_buf = nullptr;
    sl.d_buf = nullptr;
    const size_t cap = std::max<size_t>(need, 16384);
    RW_CUDA(cudaMallocHost(&sl.h_buf, cap));
    RW_CUDA(cudaMalloc(&sl.d_buf, cap));
    sl.buf_cap = cap;
  }
  sl.h_work = reinterpret_cast<rwb::WorkItem*>(sl.h_buf);
  sl.d_work = reinterpret_cast<rwb::WorkItem*>(sl.d_buf);
  sl.h_sets = reinterpret_cast<rwb::ScalarSet*>(sl.h_buf + sizeof(rwb::WorkItem) * n_items);
  sl.d_sets = reinterpret_cast<rwb::ScalarSet*>(sl.d_buf + sizeof(rwb::WorkItem) * n_items);
  sl.meta_bytes = need;
  (void)s;
  return RW_OK;
}

rwb::Uniform uniform_of(const rw_hyper* h) {
  rwb::Uniform u;
  u.wd = h->weight_decay;
  u.mu = h->momentum;
  u.one_m_damp = 1.0 - h->dampening;
  u.b1 = h->beta1;
  u.b2 = h->beta2;
  u.one_m_b1 = 1.0 - h->beta1;
  u.one_m_b2 = 1.0 - h->beta2;
  u.eps = h->eps;
  return u;
}

// Build the scalar set for the step/undo index tt (the t the reference feeds
// lr_at and bias_correction).
rwb::ScalarSet scalars_at(const rw_hyper* h, uint64_t tt, double eta) {
  rwb::ScalarSet ss;
  ss.eta = eta;
  ss.c1 = 1.0 - std::pow(h->beta1, static_cast<double>(tt));
  ss.c2 = 1.0 - std::pow(h->beta2, static_cast<double>(tt));
  ss.denom = 1.0 - eta * h->weight_decay;
  return ss;
}

int launch_groups(rw_state* s, const rw_hyper* h, const uint32_t* ids, uint32_t n, bool undo,
                  const void* grad, const std::vector<double>& etas, void* stream,
                  const uint8_t* copy_only = nullptr, void* const* peers = nullptr) {
  if (n == 0) return RW_OK;
  if (s->host_resident)
    return fail(RW_INVALID_ARGUMENT, "state was created by rw_state_create_host: it has no device buffers "
                                     "(use rw_optimizer_undo_host)");
  RW_CUDA(cudaSetDevice(s->device));
  Slot& sl = s->slots[s->next_slot];
  s->next_slot = (s->next_slot + 1) % kSlots;

  // distinct scalar sets by tt; LAMB: one set per item (eta = eta * trust)
  const bool lamb = h->kind == RW_LAMB;
  std::map<uint64_t, uint32_t> set_of;
  for (uint32_t i = 0; i < n; ++i) {
    const rw_group& gr = s->mirror[ids[i]];
    const uint64_t tt = undo ? gr.t : gr.t + 1;
    set_of.emplace(tt, 0);
  }
  const uint32_t n_sets = lamb ? n : static_cast<uint32_t>(set_of.size());
  int st = ensure_slot(s, sl, n, n_sets);
  if (st) return st;
  {
    uint32_t k = 0;
    for (auto& kv : set_of) kv.second = k++;
  }
  for (uint32_t i = 0; i < n; ++i) {
    if (copy_only && copy_only[i]) continue;  // pass-through groups use no scalars
    const rw_group& gr = s->mirror[ids[i]];
    const uint64_t tt = undo ? gr.t : gr.t + 1;
    sl.h_sets[lamb ? i : set_of[tt]] = scalars_at(h, tt, etas[i]);
  }
  const uint32_t ce = rwb::chunk_elems_for(s->dtype);
  uint64_t chunk = 0;
  uint32_t n_items = 0;
  for (uint32_t i = 0; i < n; ++i) {
    const rw_group& gr = s->mirror[ids[i]];
    rwb::WorkItem& w = sl.h_work[n_items++];
    w.off = gr.offset;
    w.len = gr.len;
    w.gid = ids[i];
    w.new_t = undo ? gr.t - 1 : gr.t + 1;
    w.nchunks = static_cast<uint32_t>((gr.len + ce - 1) / ce);
    w.chunk_begin = static_cast<uint32_t>(chunk);
    w.sidx = lamb ? i : set_of[undo ? gr.t : gr.t + 1];
    w.flags = (copy_only && copy_only[i]) ? rwb::kWorkCopyOnly : 0u;
    w.pad = lamb && !undo ? static_cast<uint32_t>(s->trust_head[ids[i]] % kTrustDepth) : 0u;  // trust slot
    chunk += w.nchunks;
  }
  if (chunk > 0xFFFFFFF0ull) return fail(RW_TOO_LARGE, "TooLarge: too many chunks in one call");
  auto cs = static_cast<cudaStream_t>(stream);
  // small non-LAMB calls: metadata in the kernel parameters, no H2D copy
  const bool inline_meta = !lamb && n_items <= rwb::kInlineItems && n_sets <= rwb::kInlineSets;
  rwb::InlineMeta im;
  if (n_items > 0) {
    if (inline_meta) {
      std::memcpy(im.work, sl.h_work, sizeof(rwb::WorkItem) * n_items);
      std::memcpy(im.sets, sl.h_sets, sizeof(rwb::ScalarSet) * n_sets);
    } else {
      RW_CUDA(cudaMemcpyAsync(sl.d_buf, sl.h_buf, sl.meta_bytes, cudaMemcpyHostToDevice, cs));  // work + sets
    }
    if (lamb && !undo) {
      // step_lamb first pass over every group: m, v, both norms, trust
      if (s->partial_cap < chunk) {
        cudaFree(s->d_partial);
        s->d_partial = nullptr;
        RW_CUDA(cudaMalloc(&s->d_partial, sizeof(double) * 2 * chunk));
        s->partial_cap = chunk;
      }
      int e = rwb::launch_lamb_pass1(s->dtype, s->x, s->g, grad == s->g ? nullptr : grad, s->m, s->v, sl.d_work,
                                     n_items, static_cast<uint32_t>(chunk), ce, sl.d_sets, uniform_of(h),
                                     s->d_partial, s->d_trust, kTrustDepth,
                                     (s->flags & RW_STATE_LAMB_SEQUENTIAL_NORMS) != 0, stream);
      if (e) return cuda_fail(static_cast<cudaError_t>(e), "lamb pass 1");
      grad = nullptr;  // pass 1 cached it in g
    }
    rwb::LaunchArgs a;
    a.dtype = s->dtype;
    a.kind = h->kind;
    a.undo = undo;
    a.x = s->x;
    a.g = s->g;
    a.m = s->m;
    a.v = s->v;
    a.vmax = s->vmax;
    a.grad = grad;
    a.work = sl.d_work;
    a.n_work = n_items;
    a.total_chunks = static_cast<uint32_t>(chunk);
    a.chunk_elems = ce;
    a.sets = sl.d_sets;
    a.u = uniform_of(h);
    a.groups = s->d_groups;
    a.done = sl.d_done;
    if (inline_meta) {
      a.work = nullptr;
      a.sets = nullptr;
      a.inl = &im;
    }
    if (peers) {
      a.px = peers[0];
      a.pg = peers[1];
      a.pm = peers[2];
      a.pv = peers[3];
    }
    int e = rwb::launch_optim(a, stream);
    if (e) return cuda_fail(static_cast<cudaError_t>(e), "optim kernel launch");
  }
  // host mirror follows what the kernel writes at group completion
  for (uint32_t i = 0; i < n; ++i) {
    if (copy_only && copy_only[i]) continue;
    rw_group& gr = s->mirror[ids[i]];
    gr.t = undo ? gr.t - 1 : gr.t + 1;
    gr.updated = undo ? 0u : 1u;
    if (lamb) {  // push / pop the saved trust ratio (optim.cpp:216 / :241)
      const uint32_t g = ids[i];
      if (undo) {
        s->trust_head[g] -= 1;
        s->trust_count[g] -= 1;
      } else {
        s->trust_head[g] += 1;
        s->trust_count[g] = std::min(s->trust_count[g] + 1, kTrustDepth);
      }
    }
  }
  RW_CUDA(cudaEventRecord(sl.ev, cs));
  sl.used = true;
  return RW_OK;
}

size_t elem_size(int dtype) { return dtype == RW_F64 ? 8 : 4; }

// undo_lamb guards (optim.cpp:219-230) for the groups ids[0..n): the saved
// trust ratio must exist; etas[i] (lr_at(t)) becomes scaled = eta * trust and
// denom = 1 - scaled * wd must not vanish.  One D2H read of the trust table.
int lamb_undo_scalars(rw_state* s, const rw_hyper* h, const uint32_t* ids, uint32_t n, std::vector<double>& etas,
                      void* stream) {
  if (h->beta1 == 0.0 || h->beta2 == 0.0)
    return fail(RW_NON_INVERTIBLE_HYPER, "NonInvertibleHyper: beta1*beta2 == 0 for lamb");
  for (uint32_t i = 0; i < n; ++i)
    if (s->trust_count[ids[i]] == 0)
      return fail(RW_NOTHING_TO_UNDO, "NothingToUndo: no saved trust ratio for lamb undo (group %u)", ids[i]);
  if (n == 0) return RW_OK;
  std::vector<double> tr(s->mirror.size() * kTrustDepth);
  RW_CUDA(cudaSetDevice(s->device));
  auto cs = static_cast<cudaStream_t>(stream);
  RW_CUDA(cudaMemcpyAsync(tr.data(), s->d_trust, sizeof(double) * tr.size(), cudaMemcpyDeviceToHost, cs));
  RW_CUDA(cudaStreamSynchronize(cs));
  for (uint32_t i = 0; i < n; ++i) {
    const uint32_t g = ids[i];
    const double trust = tr[uint64_t(g) * kTrustDepth + (s->trust_head[g] - 1) % kTrustDepth];
    const double scaled = etas[i] * trust;
    if (1.0 - scaled * h->weight_decay == 0.0)
      return fail(RW_NON_INVERTIBLE_HYPER, "NonInvertibleHyper: trust*lr*weight_decay == 1 for lamb (group %u)", g);
    etas[i] = scaled;
  }
  return RW_OK;
}

}  // namespace

extern "C" {

int rw_abi_version(void) { return RW_ABI_VERSION; }
const char* rw_last_error_message(void) { return g_err.c_str(); }
const char* rw_status_name(int status) {
  if (status >= 0 && status <= 19) return kErrNames[status];
  if (status == RW_CUDA_ERROR) return "CudaError";
  if (status == RW_INVALID_ARGUMENT) return "InvalidArgument";
  return "Unknown";
}
int rw_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int rw_invertibility_check(int32_t kind) {
  switch (kind) {
    case RW_SGD:
    case RW_SGDM:
    case RW_ADAM:
    case RW_ADAMW: return RW_INVERTIBLE;
    case RW_LAMB: return RW_INVERTIBLE_WITH_SAVED_SCALARS;
    default: return RW_NOT_INVERTIBLE_KIND;
  }
}

// OptimizerHyper::validate, optim.cpp:59-71 (same checks, same order)
int rw_hyper_validate(const rw_hyper* h) {
  if (!h) return fail(RW_INVALID_ARGUMENT, "null hyper");
  if (!(h->lr > 0.0)) return fail(RW_INVALID_CONFIG, "InvalidConfig: optimizer.lr must be > 0");
  if (h->weight_decay < 0.0) return fail(RW_INVALID_CONFIG, "InvalidConfig: optimizer.weight_decay must be >= 0");
  if (h->momentum < 0.0 || h->momentum > 1.0) return fail(RW_INVALID_CONFIG, "InvalidConfig: optimizer.momentum must be in [0,1]");
  if (h->dampening < 0.0 || h->dampening > 1.0) return fail(RW_INVALID_CONFIG, "InvalidConfig: optimizer.dampening must be in [0,1]");
  if (h->beta1 < 0.0 || h->beta1 >= 1.0) return fail(RW_INVALID_CONFIG, "InvalidConfig: optimizer.beta1 must be in [0,1)");
  if (h->beta2 < 0.0 || h->beta2 >= 1.0) return fail(RW_INVALID_CONFIG, "InvalidConfig: optimizer.beta2 must be in [0,1)");
  if (!(h->eps > 0.0)) return fail(RW_INVALID_CONFIG, "InvalidConfig: optimizer.eps must be > 0");
  for (uint32_t i = 0; i < h->lr_table_len; ++i)
    if (!(h->lr_table_value[i] > 0.0)) return fail(RW_INVALID_CONFIG, "InvalidConfig: optimizer.lr_table entries must be > 0");
  return RW_OK;
}

int rw_lr_at(const rw_hyper* h, uint64_t t, double* out) {
  if (!h || !out) return fail(RW_INVALID_ARGUMENT, "null argument");
  return lr_at(h, t, out);
}

static int state_create(rw_state** out, int32_t dtype, void* x, void* g, void* m, void* v, void* vmax,
                        uint64_t total, const rw_group* groups, uint32_t n_groups, int32_t device,
                        bool host_resident) {
  rwb::DeviceScope dev_scope(device);
  if (!out) return fail(RW_INVALID_ARGUMENT, "null out");
  *out = nullptr;
  if (dtype != RW_F32 && dtype != RW_F64) return fail(RW_INVALID_ARGUMENT, "dtype must be RW_F32 or RW_F64");
  if (!host_resident && (!x || !g)) return fail(RW_INVALID_ARGUMENT, "x and g are required");
  for (void* p : {x, g, m, v, vmax})
    if (p && (reinterpret_cast<uintptr_t>(p) & 15u))
      return fail(RW_INVALID_ARGUMENT, "state buffers must be 16-byte aligned");
  if (n_groups > 0 && !groups) return fail(RW_INVALID_ARGUMENT, "null groups");
  for (uint32_t i = 0; i < n_groups; ++i) {
    // shape_elements (tensor.cpp:125-133): a zero extent is InvalidShape
    if (groups[i].len == 0) return fail(RW_INVALID_SHAPE, "InvalidShape: zero extent (group %u)", i);
    if (groups[i].offset + groups[i].len > total || groups[i].offset + groups[i].len < groups[i].offset)
      return fail(RW_INVALID_SHAPE, "InvalidShape: group %u [%llu, +%llu) exceeds the state (%llu)", i,
                  (unsigned long long)groups[i].offset, (unsigned long long)groups[i].len,
                  (unsigned long long)total);
  }
  int ndev = rw_device_count();
  if (ndev == 0) return fail(RW_CUDA_ERROR, "no CUDA device visible: the B200 path has no CPU fallback");
  if (device < 0 || device >= ndev) return fail(RW_INVALID_ARGUMENT, "bad device %d", device);
  auto* s = new rw_state();
  s->dtype = dtype;
  s->device = device;
  s->x = x;
  s->g = g;
  s->m = m;
  s->v = v;
  s->vmax = vmax;
  s->host_resident = host_resident;
  s->total = total;
  s->mirror.assign(groups, groups + n_groups);
  for (auto& gr : s->mirror) gr.flags = 0;
  s->trust_head.assign(n_groups, 0);
  s->trust_count.assign(n_groups, 0);
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess && n_groups) e = cudaMalloc(&s->d_groups, sizeof(rw_group) * n_groups);
  if (e == cudaSuccess && n_groups) e = cudaMalloc(&s->d_trust, sizeof(double) * n_groups * kTrustDepth);
  if (e == cudaSuccess && n_groups) e = cudaMemset(s->d_trust, 0, sizeof(double) * n_groups * kTrustDepth);
  if (e == cudaSuccess && n_groups)
    e = cudaMemcpy(s->d_groups, s->mirror.data(), sizeof(rw_group) * n_groups, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    rw_state_destroy(s);
    return cuda_fail(e, "rw_state_create");
  }
  // Size every launch slot for a call over all groups now: growing one later
  // means cudaFreeHost / cudaFree (device-wide synchronisations) inside the
  // call -- e.g. inside the first recovery of a job, the one that matters.
  {
    const uint32_t pre = std::min<uint32_t>(std::max<uint32_t>(n_groups, 1), 4096);
    for (auto& sl : s->slots) {
      const int st = ensure_slot(s, sl, pre, pre);
      if (st) {
        rw_state_destroy(s);
        return st;
      }
    }
  }
  *out = s;
  return RW_OK;
}

int rw_state_create(rw_state** out, int32_t dtype, void* x, void* g, void* m, void* v, void* vmax,
                    uint64_t total, const rw_group* groups, uint32_t n_groups, int32_t device) {
  return state_create(out, dtype, x, g, m, v, vmax, total, groups, n_groups, device, false);
}

int rw_state_create_host(rw_state** out, int32_t dtype, uint64_t total, const rw_group* groups,
                         uint32_t n_groups, int32_t device) {
  return state_create(out, dtype, nullptr, nullptr, nullptr, nullptr, nullptr, total, groups, n_groups, device,
                      true);
}

void rw_state_destroy(rw_state* s) {
  rwb::DeviceScope dev_scope(s ? s->device : -1);
  if (!s) return;
  cudaSetDevice(s->device);
  for (auto& sl : s->slots) {
    if (sl.ev) {
      cudaEventSynchronize(sl.ev);
      cudaEventDestroy(sl.ev);
    }
    cudaFreeHost(sl.h_buf);
    cudaFree(sl.d_buf);
    cudaFree(sl.d_done);
  }
  for (auto& r : s->ring)
    for (void* p : r) cudaFree(p);
  cudaFree(s->d_groups);
  cudaFree(s->d_trust);
  cudaFree(s->d_partial);
  if (s->h2d) cudaStreamSynchronize(s->h2d), cudaStreamDestroy(s->h2d);
  if (s->d2h) cudaStreamSynchronize(s->d2h), cudaStreamDestroy(s->d2h);
  for (cudaEvent_t e : s->evs) cudaEventDestroy(e);
  delete s;
}

int rw_state_set_flags(rw_state* s, uint32_t flags) {
  if (!s) return fail(RW_INVALID_ARGUMENT, "null state");
  if (flags & ~uint32_t(RW_STATE_LAMB_SEQUENTIAL_NORMS)) return fail(RW_INVALID_ARGUMENT, "unknown state flag");
  s->flags = flags;
  return RW_OK;
}

int rw_state_info(const rw_state* s, int32_t* dtype, uint64_t* total, int32_t* device) {
  if (!s) return fail(RW_INVALID_ARGUMENT, "null state");
  if (dtype) *dtype = s->dtype;
  if (total) *total = s->total;
  if (device) *device = s->device;
  return RW_OK;
}

uint32_t rw_state_num_groups(const rw_state* s) { return s ? static_cast<uint32_t>(s->mirror.size()) : 0; }

void* rw_state_ptr(rw_state* s, int which) {
  if (!s) return nullptr;
  switch (which) {
    case 0: return s->x;
    case 1: return s->g;
    case 2: return s->m;
    case 3: return s->v;
    case 4: return s->vmax;
  }
  return nullptr;
}

int rw_state_saved_scalars(rw_state* s, uint32_t group, double* out, uint32_t cap, uint32_t* count,
                           void* stream) {
  rwb::DeviceScope dev_scope(s ? s->device : -1);
  if (!s || !count || (cap && !out)) return fail(RW_INVALID_ARGUMENT, "null argument");
  if (group >= s->mirror.size()) return fail(RW_INVALID_ARGUMENT, "group id %u out of range", group);
  const uint32_t c = s->trust_count[group];
  *count = c;
  if (c == 0 || cap == 0) return RW_OK;
  double ring[kTrustDepth];
  RW_CUDA(cudaSetDevice(s->device));
  auto cs = static_cast<cudaStream_t>(stream);
  RW_CUDA(cudaMemcpyAsync(ring, s->d_trust + uint64_t(group) * kTrustDepth, sizeof(ring), cudaMemcpyDeviceToHost, cs));
  RW_CUDA(cudaStreamSynchronize(cs));
  const uint64_t head = s->trust_head[group];
  for (uint32_t k = 0; k < c && k < cap; ++k) out[k] = ring[(head - c + k) % kTrustDepth];
  return RW_OK;
}

int rw_state_set_saved_scalars(rw_state* s, uint32_t group, const double* in, uint32_t count, void* stream) {
  rwb::DeviceScope dev_scope(s ? s->device : -1);
  if (!s || (count && !in)) return fail(RW_INVALID_ARGUMENT, "null argument");
  if (group >= s->mirror.size()) return fail(RW_INVALID_ARGUMENT, "group id %u out of range", group);
  if (count > kTrustDepth) return fail(RW_TOO_LARGE, "TooLarge: at most %u saved scalars per group", kTrustDepth);
  double ring[kTrustDepth] = {};
  for (uint32_t k = 0; k < count; ++k) ring[k] = in[k];
  RW_CUDA(cudaSetDevice(s->device));
  auto cs = static_cast<cudaStream_t>(stream);
  RW_CUDA(cudaMemcpyAsync(s->d_trust + uint64_t(group) * kTrustDepth, ring, sizeof(ring), cudaMemcpyHostToDevice, cs));
  RW_CUDA(cudaStreamSynchronize(cs));
  s->trust_head[group] = count;
  s->trust_count[group] = count;
  return RW_OK;
}

int rw_state_read_groups(rw_state* s, rw_group* out, void* stream) {
  rwb::DeviceScope dev_scope(s ? s->device : -1);
  if (!s || !out) return fail(RW_INVALID_ARGUMENT, "null argument");
  if (s->mirror.empty()) return RW_OK;
  RW_CUDA(cudaSetDevice(s->device));
  auto cs = static_cast<cudaStream_t>(stream);
  RW_CUDA(cudaMemcpyAsync(out, s->d_groups, sizeof(rw_group) * s->mirror.size(), cudaMemcpyDeviceToHost, cs));
  RW_CUDA(cudaStreamSynchronize(cs));
  // device table is authoritative
  for (size_t i = 0; i < s->mirror.size(); ++i) {
    s->mirror[i].t = out[i].t;
    s->mirror[i].updated = out[i].updated;
  }
  return RW_OK;
}

int rw_state_write_groups(rw_state* s, const rw_group* in, void* stream) {
  rwb::DeviceScope dev_scope(s ? s->device : -1);
  if (!s || !in) return fail(RW_INVALID_ARGUMENT, "null argument");
  if (s->mirror.empty()) return RW_OK;
  for (size_t i = 0; i < s->mirror.size(); ++i) {
    if (in[i].offset != s->mirror[i].offset || in[i].len != s->mirror[i].len)
      return fail(RW_SHAPE_MISMATCH, "ShapeMismatch: group %zu layout differs", i);
  }
  RW_CUDA(cudaSetDevice(s->device));
  s->mirror.assign(in, in + s->mirror.size());
  auto cs = static_cast<cudaStream_t>(stream);
  RW_CUDA(cudaMemcpyAsync(s->d_groups, s->mirror.data(), sizeof(rw_group) * s->mirror.size(),
                          cudaMemcpyHostToDevice, cs));
  RW_CUDA(cudaStreamSynchronize(cs));
  return RW_OK;
}

int rw_state_check(rw_state* s, void* stream) {
  rwb::DeviceScope dev_scope(s ? s->device : -1);
  if (!s) return fail(RW_INVALID_ARGUMENT, "null state");
  if (s->mirror.empty()) return RW_OK;
  std::vector<rw_group> dev(s->mirror.size());
  int st = rw_state_read_groups(s, dev.data(), stream);
  if (st) return st;
  bool bad = false;
  uint32_t first = 0;
  for (size_t i = 0; i < dev.size(); ++i)
    if (dev[i].flags & 1u) {
      if (!bad) first = static_cast<uint32_t>(i);
      bad = true;
      dev[i].flags &= ~1u;
    }
  if (!bad) return RW_OK;
  auto cs = static_cast<cudaStream_t>(stream);
  RW_CUDA(cudaMemcpyAsync(s->d_groups, dev.data(), sizeof(rw_group) * dev.size(), cudaMemcpyHostToDevice, cs));
  RW_CUDA(cudaStreamSynchronize(cs));
  return fail(RW_NUMERICAL_ERROR, "NumericalError: non-finite value in optimizer state (group %u)", first);
}

int rw_clear_updated(rw_state* s, const uint32_t* ids, uint32_t n, void* stream) {
  rwb::DeviceScope dev_scope(s ? s->device : -1);
  if (!s) return fail(RW_INVALID_ARGUMENT, "null state");
  for (uint32_t i = 0; i < n; ++i) {
    if (ids[i] >= s->mirror.size()) return fail(RW_INVALID_ARGUMENT, "group id %u out of range", ids[i]);
    s->mirror[ids[i]].updated = 0;
  }
  RW_CUDA(cudaSetDevice(s->device));
  int e = rwb::launch_clear_updated(s->d_groups, ids, n, stream);
  if (e) return cuda_fail(static_cast<cudaError_t>(e), "clear_updated");
  return RW_OK;
}

// optimizer_step, optim.cpp:260-286
int rw_optimizer_step(rw_state* s, const rw_hyper* h, const uint32_t* ids, uint32_t n,
                      const void* grad, uint32_t stop_after, void* stream) {
  rwb::DeviceScope dev_scope(s ? s->device : -1);
  if (!s || !h || (n && !ids)) return fail(RW_INVALID_ARGUMENT, "null argument");
  if (n > stop_after) n = stop_after;  // MidUpdate(k): the crash hits after k groups
  std::vector<double> etas(n);
  std::vector<uint8_t> seen(s->mirror.size(), 0);
  for (uint32_t i = 0; i < n; ++i) {
    if (ids[i] >= s->mirror.size()) return fail(RW_INVALID_ARGUMENT, "group id %u out of range", ids[i]);
    if (seen[ids[i]]) return fail(RW_INVALID_ARGUMENT, "group id %u listed twice", ids[i]);
    seen[ids[i]] = 1;
    const rw_group& gr = s->mirror[ids[i]];
    // require_same_shape (:340) holds by construction: grad shares the flat layout.
    if (gr.updated) return fail(RW_ALREADY_UPDATED, "AlreadyUpdated: block already stepped this iteration (group %u)", ids[i]);
    if (h->require_invertible && rw_invertibility_check(h->kind) == RW_NOT_INVERTIBLE_KIND)
      return fail(RW_NOT_INVERTIBLE, "NotInvertible: %s cannot be undone", kind_name(h->kind));
    // :349 caches the gradient BEFORE :350 lr_at may raise; reproduce that
    // partial mutation for the failing group only.
    int st = lr_at(h, gr.t + 1, &etas[i]);
    if (st) {
      if (grad && grad != s->g) {
        const size_t es = elem_size(s->dtype);
        auto cs = static_cast<cudaStream_t>(stream);
        RW_CUDA(cudaMemcpyAsync(static_cast<char*>(s->g) + gr.offset * es,
                                static_cast<const char*>(grad) + gr.offset * es, gr.len * es,
                                cudaMemcpyDeviceToDevice, cs));
      }
      return st;
    }
  }
  if (h->kind == RW_AMSGRAD && !s->vmax) return fail(RW_INVALID_ARGUMENT, "amsgrad needs a vmax buffer");
  if ((h->kind != RW_SGD && !s->m) ||
      ((h->kind == RW_ADAM || h->kind == RW_ADAMW || h->kind == RW_AMSGRAD) && !s->v))
    return fail(RW_INVALID_ARGUMENT, "%s needs m%s buffers", kind_name(h->kind),
                h->kind == RW_SGDM ? "" : " and v");
  return launch_groups(s, h, ids, n, false, grad, etas, stream);
}

}  // extern "C"

namespace {
// The guards of optimizer_undo (optim.cpp:288-307) and of undo_<kind>, for
// every group, before anything is launched; fills the per-group eta (LAMB:
// eta * saved trust ratio).
int undo_prepare(rw_state* s, const rw_hyper* h, const uint32_t* ids, uint32_t n, std::vector<double>& etas,
                 void* stream) {
  if (!s || !h || (n && !ids)) return fail(RW_INVALID_ARGUMENT, "null argument");
  etas.assign(n, 0.0);
  std::vector<uint8_t> seen(s->mirror.size(), 0);
  for (uint32_t i = 0; i < n; ++i) {
    if (ids[i] >= s->mirror.size()) return fail(RW_INVALID_ARGUMENT, "group id %u out of range", ids[i]);
    if (seen[ids[i]]) return fail(RW_INVALID_ARGUMENT, "group id %u listed twice", ids[i]);
    seen[ids[i]] = 1;
    const rw_group& gr = s->mirror[ids[i]];
    if (!gr.updated) return fail(RW_NOTHING_TO_UNDO, "NothingToUndo: block has no pending update (group %u)", ids[i]);
    if (h->kind == RW_AMSGRAD) return fail(RW_NOT_INVERTIBLE, "NotInvertible: amsgrad element-wise max has no inverse");
    int st = lr_at(h, gr.t, &etas[i]);
    if (st) return st;
    const double eta = etas[i];
    switch (h->kind) {
      case RW_SGD:  // optim.cpp:106-107
        if (1.0 - eta * h->weight_decay == 0.0)
          return fail(RW_NON_INVERTIBLE_HYPER, "NonInvertibleHyper: lr*weight_decay == 1 for sgd");
        break;
      case RW_SGDM:  // :200
        if (h->momentum == 0.0) return fail(RW_NON_INVERTIBLE_HYPER, "NonInvertibleHyper: momentum == 0 for sgdm");
        break;
      case RW_ADAM:  // :222-224
        if (h->beta1 == 0.0 || h->beta2 == 0.0)
          return fail(RW_NON_INVERTIBLE_HYPER, "NonInvertibleHyper: beta1*beta2 == 0 for adam");
        break;
      case RW_ADAMW:  // :252-256
        if (h->beta1 == 0.0 || h->beta2 == 0.0)
          return fail(RW_NON_INVERTIBLE_HYPER, "NonInvertibleHyper: beta1*beta2 == 0 for adamw");
        if (1.0 - eta * h->weight_decay == 0.0)
          return fail(RW_NON_INVERTIBLE_HYPER, "NonInvertibleHyper: lr*weight_decay == 1 for adamw");
        break;
      case RW_LAMB:  // optim.cpp:219-225; the trust read + denom check follow the loop
        if (h->beta1 == 0.0 || h->beta2 == 0.0)
          return fail(RW_NON_INVERTIBLE_HYPER, "NonInvertibleHyper: beta1*beta2 == 0 for lamb");
        if (s->trust_count[ids[i]] == 0)
          return fail(RW_NOTHING_TO_UNDO, "NothingToUndo: no saved trust ratio for lamb undo (group %u)", ids[i]);
        break;
      default: return fail(RW_INVALID_ARGUMENT, "unknown optimizer kind %d", h->kind);
    }
  }
  if (!s->host_resident && ((h->kind != RW_SGD && !s->m) ||
                            ((h->kind == RW_ADAM || h->kind == RW_ADAMW || h->kind == RW_LAMB) && !s->v)))
    return fail(RW_INVALID_ARGUMENT, "%s needs m/v buffers", kind_name(h->kind));
  if (h->kind == RW_LAMB) return lamb_undo_scalars(s, h, ids, n, etas, stream);
  return RW_OK;
}
}  // namespace

extern "C" {

// optimizer_undo, optim.cpp:288-307 and the per-kind guards of undo_<kind>
int rw_optimizer_undo(rw_state* s, const rw_hyper* h, const uint32_t* ids, uint32_t n, void* stream) {
  rwb::DeviceScope dev_scope(s ? s->device : -1);
  std::vector<double> etas;
  int st = undo_prepare(s, h, ids, n, etas, stream);
  if (st) return st;
  return launch_groups(s, h, ids, n, true, nullptr, etas, stream);
}

// optimizer_undo over a state whose bytes live in HOST memory (same flat
// layout): the device buffers of `s` are the staging area.  The groups are
// cut into slices of ~slice_elems elements in layout order; slice k's H2D
// (copy stream 1), undo (the caller's stream) and D2H (copy stream 2) run as a
// three-stage pipeline, so the two PCIe directions and the kernel overlap.
int rw_optimizer_undo_host(rw_state* s, const rw_hyper* h, const uint32_t* ids, uint32_t n, const void* hx,
                           const void* hg, const void* hm, const void* hv, void* ox, void* om, void* ov,
                           uint64_t slice_elems, void* stream) {
  rwb::DeviceScope dev_scope(s ? s->device : -1);
  std::vector<double> etas;
  int st = undo_prepare(s, h, ids, n, etas, stream);
  if (st) return st;
  const bool um = h->kind != RW_SGD, uv = h->kind == RW_ADAM || h->kind == RW_ADAMW || h->kind == RW_LAMB;
  if (!hx || !hg || !ox || (um && (!hm || !om)) || (uv && (!hv || !ov)))
    return fail(RW_INVALID_ARGUMENT, "host x, g (and m, v as the kind needs) in and out buffers required");
  if (n == 0) return RW_OK;
  if (slice_elems == 0) slice_elems = 16ull << 20;
  RW_CUDA(cudaSetDevice(s->device));
  auto cs = static_cast<cudaStream_t>(stream);
  if (!s->h2d) RW_CUDA(cudaStreamCreateWithFlags(&s->h2d, cudaStreamNonBlocking));
  if (!s->d2h) RW_CUDA(cudaStreamCreateWithFlags(&s->d2h, cudaStreamNonBlocking));
  // groups in layout order -> slices
  std::vector<uint32_t> order(n);
  for (uint32_t i = 0; i < n; ++i) order[i] = i;
  std::sort(order.begin(), order.end(),
            [&](uint32_t a, uint32_t b) { return s->mirror[ids[a]].offset < s->mirror[ids[b]].offset; });
  struct SliceDesc {
    uint64_t begin, end;
    std::vector<uint32_t> gids;
    std::vector<double> etas;
  };
  std::vector<SliceDesc> slices;
  for (uint32_t k : order) {
    const rw_group& gr = s->mirror[ids[k]];
    if (slices.empty() || slices.back().end - slices.back().begin >= slice_elems) {
      // slices tile the span contiguously: unselected groups inside it pass through
      const uint64_t b = slices.empty() ? gr.offset : slices.back().end;
      slices.push_back(SliceDesc{b, b, {}, {}});
    }
    SliceDesc& sd = slices.back();
    sd.end = std::max<uint64_t>(sd.end, gr.offset + gr.len);
    sd.gids.push_back(ids[k]);
    sd.etas.push_back(etas[k]);
  }
  // staging ring: slice k lives in slot k % kRing at offset 0 (its work
  // items are slice-relative), so device memory is bounded by kRing slices
  // whatever the size of the host-resident state
  constexpr size_t kRing = 3;
  uint64_t cap = 0;
  for (const SliceDesc& sd : slices) cap = std::max<uint64_t>(cap, sd.end - sd.begin);
  const size_t es = elem_size(s->dtype);
  if (cap > s->ring_cap) {
    RW_CUDA(cudaDeviceSynchronize());  // earlier calls may still read the old ring
    for (auto& r : s->ring)
      for (void*& q : r) {
        cudaFree(q);
        q = nullptr;
      }
    s->ring_cap = 0;
    for (auto& r : s->ring)
      for (void*& q : r) RW_CUDA(cudaMalloc(&q, cap * es));
    s->ring_cap = cap;
  }
  while (s->evs.size() < 3 * slices.size() + 1) {
    cudaEvent_t e;
    RW_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    s->evs.push_back(e);
  }
  // One work list for every slice, uploaded before the first bulk H2D so no
  // small metadata copy queues behind the slice copies on the H2D engine.
  // Each slice's items are contiguous, their chunk_begin relative to it.
  Slot& sl = s->slots[s->next_slot];
  s->next_slot = (s->next_slot + 1) % kSlots;
  const bool lamb = h->kind == RW_LAMB;
  std::map<uint64_t, uint32_t> set_of;
  for (uint32_t i = 0; i < n; ++i) set_of.emplace(s->mirror[ids[i]].t, 0);
  const uint32_t n_sets = lamb ? n : static_cast<uint32_t>(set_of.size());
  st = ensure_slot(s, sl, n, n_sets);
  if (st) return st;
  {
    uint32_t k = 0;
    for (auto& kv : set_of) kv.second = k++;
  }
  const uint32_t ce = rwb::chunk_elems_for(s->dtype);
  std::vector<uint32_t> first(slices.size()), chunks(slices.size());
  uint32_t item = 0;
  for (size_t k = 0; k < slices.size(); ++k) {
    first[k] = item;
    uint64_t chunk = 0;
    for (size_t j = 0; j < slices[k].gids.size(); ++j) {
      const uint32_t gid = slices[k].gids[j];
      const rw_group& gr = s->mirror[gid];
      const uint32_t sidx = lamb ? item : set_of[gr.t];
      sl.h_sets[sidx] = scalars_at(h, gr.t, slices[k].etas[j]);
      rwb::WorkItem& w = sl.h_work[item++];
      w.off = gr.offset - slices[k].begin;  // slice-relative: the ring slot holds the slice at 0
      w.len = gr.len;
      w.new_t = gr.t - 1;
      w.gid = gid;
      w.nchunks = static_cast<uint32_t>((gr.len + ce - 1) / ce);
      w.chunk_begin = static_cast<uint32_t>(chunk);
      w.sidx = sidx;
      w.flags = 0;
      w.pad = 0;
      chunk += w.nchunks;
    }
    if (chunk > 0xFFFFFFF0ull) return fail(RW_TOO_LARGE, "TooLarge: too many chunks in one slice");
    chunks[k] = static_cast<uint32_t>(chunk);
  }
  RW_CUDA(cudaMemcpyAsync(sl.d_buf, sl.h_buf, sl.meta_bytes, cudaMemcpyHostToDevice, cs));  // work + sets
  cudaEvent_t start = s->evs[3 * slices.size()];
  RW_CUDA(cudaEventRecord(start, cs));  // prior work + the metadata upload first
  RW_CUDA(cudaStreamWaitEvent(s->h2d, start, 0));
  RW_CUDA(cudaStreamWaitEvent(s->d2h, start, 0));
  const void* hin[4] = {hx, hg, um ? hm : nullptr, uv ? hv : nullptr};
  void* hout[3] = {ox, um ? om : nullptr, uv ? ov : nullptr};
  // out != in: the parts of the layout outside the span pass through too
  {
    const uint64_t span_b = slices.front().begin, span_e = slices.back().end;
    const int in_of_out[3] = {0, 2, 3};
    for (int b = 0; b < 3; ++b) {
      if (!hout[b] || hout[b] == hin[in_of_out[b]]) continue;
      auto* o = static_cast<char*>(hout[b]);
      auto* i = static_cast<const char*>(hin[in_of_out[b]]);
      if (span_b) RW_CUDA(cudaMemcpyAsync(o, i, span_b * es, cudaMemcpyHostToHost, s->d2h));
      if (span_e < s->total)
        RW_CUDA(cudaMemcpyAsync(o + span_e * es, i + span_e * es, (s->total - span_e) * es, cudaMemcpyHostToHost,
                                s->d2h));
    }
  }
  for (size_t k = 0; k < slices.size(); ++k) {
    const SliceDesc& sd = slices[k];
    const uint64_t off = sd.begin * es, bytes = (sd.end - sd.begin) * es;
    void* const* slot_buf = s->ring[k % kRing];
    void* din[4] = {slot_buf[0], slot_buf[1], slot_buf[2], slot_buf[3]};
    void* dout[3] = {slot_buf[0], slot_buf[2], slot_buf[3]};
    // the slot's previous slice must have left for the host before it is refilled
    if (k >= kRing) RW_CUDA(cudaStreamWaitEvent(s->h2d, s->evs[3 * (k - kRing) + 2], 0));
    for (int b = 0; b < 4; ++b)
      if (hin[b])
        RW_CUDA(cudaMemcpyAsync(din[b], static_cast<const char*>(hin[b]) + off, bytes, cudaMemcpyHostToDevice,
                                s->h2d));
    RW_CUDA(cudaEventRecord(s->evs[3 * k], s->h2d));
    RW_CUDA(cudaStreamWaitEvent(cs, s->evs[3 * k], 0));
    rwb::LaunchArgs a;
    a.dtype = s->dtype;
    a.kind = h->kind;
    a.undo = true;
    a.x = din[0];
    a.g = din[1];
    a.m = din[2];
    a.v = din[3];
    a.vmax = nullptr;
    a.grad = nullptr;
    a.work = sl.d_work + first[k];
    a.n_work = static_cast<uint32_t>(sd.gids.size());
    a.total_chunks = chunks[k];
    a.chunk_elems = ce;
    a.sets = sl.d_sets;
    a.u = uniform_of(h);
    a.groups = s->d_groups;
    a.done = sl.d_done + first[k];
    int e = rwb::launch_optim(a, stream);
    if (e) {
      cudaStreamSynchronize(s->h2d);
      return cuda_fail(static_cast<cudaError_t>(e), "optim kernel launch");
    }
    RW_CUDA(cudaEventRecord(s->evs[3 * k + 1], cs));
    RW_CUDA(cudaStreamWaitEvent(s->d2h, s->evs[3 * k + 1], 0));
    for (int b = 0; b < 3; ++b)
      if (hout[b])
        RW_CUDA(cudaMemcpyAsync(static_cast<char*>(hout[b]) + off, dout[b], bytes, cudaMemcpyDeviceToHost, s->d2h));
    RW_CUDA(cudaEventRecord(s->evs[3 * k + 2], s->d2h));
  }
  for (uint32_t i = 0; i < n; ++i) {  // host mirror follows the kernels' marker writes
    rw_group& gr = s->mirror[ids[i]];
    gr.t -= 1;
    gr.updated = 0;
    if (lamb) {
      s->trust_head[ids[i]] -= 1;
      s->trust_count[ids[i]] -= 1;
    }
  }
  // the call is ordered on `stream`: it completes when the last D2H lands
  RW_CUDA(cudaStreamWaitEvent(cs, s->evs[3 * (slices.size() - 1) + 2], 0));
  RW_CUDA(cudaEventRecord(sl.ev, cs));
  sl.used = true;
  return RW_OK;
}

// ---------------- numerics ----------------
static uint64_t mix64(uint64_t x) {  // tensor.cpp:69-74
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
uint64_t rw_derive_seed(uint64_t base, const uint64_t* parts, uint32_t n) {  // tensor.cpp:76-83
  uint64_t h = mix64(base);
  for (uint32_t i = 0; i < n; ++i) h = mix64(h ^ mix64(parts[i]));
  return h;
}
int rw_seeded_fill(int32_t dtype, void* out, uint64_t n, uint64_t seed, uint64_t offset, void* stream) {
  rwb::DeviceScope dev_scope(rwb::DeviceScope::device_of(out));
  if (!out && n) return fail(RW_INVALID_ARGUMENT, "null out");
  int e = rwb::launch_seeded_fill(dtype, out, n, seed, offset, stream);
  if (e) return cuda_fail(static_cast<cudaError_t>(e), "seeded_fill");
  return RW_OK;
}
int rw_ordered_sum(int32_t dtype, const void* const* tensors, uint32_t count, uint64_t n, void* out,
                   void* stream) {
  rwb::DeviceScope dev_scope(rwb::DeviceScope::device_of(out));
  if (count == 0) return fail(RW_EMPTY_INPUT, "EmptyInput: ordered_sum of nothing");
  int e = rwb::launch_ordered_sum(dtype, tensors, count, n, out, stream);
  if (e) return cuda_fail(static_cast<cudaError_t>(e), "ordered_sum");
  return RW_OK;
}

}  // extern "C"

// ---------------- host-buffer ParamBlock entry points ----------------
namespace {

// Per-thread staging area: device copies of one block + a one-group rw_state.
struct HostStage {
  int dtype = -1;
  uint64_t n = 0;
  int device = -1;
  void* d[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};  // x g m v vmax
  rw_state* st = nullptr;
  cudaStream_t stream = nullptr;
  void release() {
    if (st) rw_state_destroy(st);
    st = nullptr;
    for (auto& p : d) {
      cudaFree(p);
      p = nullptr;
    }
    n = 0;
  }
  ~HostStage() {
    release();
    if (stream) cudaStreamDestroy(stream);
  }
};
thread_local HostStage g_stage;

int stage_prepare(int dtype, uint64_t n) {
  if (rw_device_count() == 0) return fail(RW_CUDA_ERROR, "no CUDA device visible: the B200 path has no CPU fallback");
  int dev = 0;
  RW_CUDA(cudaGetDevice(&dev));
  HostStage& S = g_stage;
  if (S.st && S.dtype == dtype && S.n == n && S.device == dev) return RW_OK;
  S.release();
  S.dtype = dtype;
  S.n = n;
  S.device = dev;
  if (!S.stream) RW_CUDA(cudaStreamCreateWithFlags(&S.stream, cudaStreamNonBlocking));
  const size_t bytes = n * elem_size(dtype);
  for (auto& p : S.d) RW_CUDA(cudaMalloc(&p, bytes));
  rw_group gr{0, n, 0, 0, 0};
  const int st = rw_state_create(&S.st, dtype, S.d[0], S.d[1], S.d[2], S.d[3], S.d[4], n, &gr, 1, dev);
  // the host-block drop-in reproduces step_lamb's left-to-right norms (bit-exact trust ratio)
  return st ? st : rw_state_set_flags(S.st, RW_STATE_LAMB_SEQUENTIAL_NORMS);
}

int block_guards_step(const rw_hyper* h, uint64_t t, uint32_t updated, double* eta) {
  if (updated) return fail(RW_ALREADY_UPDATED, "AlreadyUpdated: block already stepped this iteration");
  if (h->require_invertible && rw_invertibility_check(h->kind) == RW_NOT_INVERTIBLE_KIND)
    return fail(RW_NOT_INVERTIBLE, "NotInvertible: %s cannot be undone", kind_name(h->kind));
  return lr_at(h, t + 1, eta);
}

}  // namespace

extern "C" {

// optimizer_step on a host ParamBlock (optim.cpp:260-286)
int rw_host_block_step(int32_t dtype, void* x, void* g, void* m, void* v, void* vmax, uint64_t n,
                       uint64_t* t, uint32_t* updated, const void* grad, const rw_hyper* h) {
  if (!x || !g || !t || !updated || !h || !grad) return fail(RW_INVALID_ARGUMENT, "null argument");
  if (dtype != RW_F32 && dtype != RW_F64) return fail(RW_INVALID_ARGUMENT, "bad dtype");
  if (n == 0) return fail(RW_INVALID_SHAPE, "InvalidShape: zero extent");
  const size_t bytes = n * elem_size(dtype);
  double eta = 0;
  int st = block_guards_step(h, *t, *updated, &eta);
  if (st) {
    if (st == RW_INVALID_CONFIG) std::memcpy(g, grad, bytes);  // :349 runs before :350 raises
    return st;
  }
  const bool um = h->kind != RW_SGD, uv = h->kind == RW_ADAM || h->kind == RW_ADAMW || h->kind == RW_AMSGRAD;
  if ((um && !m) || (uv && !v) || (h->kind == RW_AMSGRAD && !vmax))
    return fail(RW_INVALID_ARGUMENT, "%s needs its m/v/vmax buffers", kind_name(h->kind));
  if (h->kind == RW_LAMB)
    return fail(RW_INVALID_ARGUMENT, "lamb needs the saved-scalar stack: use rw_host_block_lamb_step");
  st = stage_prepare(dtype, n);
  if (st) return st;
  HostStage& S = g_stage;
  void* hs[5] = {x, const_cast<void*>(grad), m, v, vmax};
  const bool use[5] = {true, true, um, uv, h->kind == RW_AMSGRAD};
  for (int i = 0; i < 5; ++i)
    if (use[i]) RW_CUDA(cudaMemcpyAsync(S.d[i], hs[i], bytes, cudaMemcpyHostToDevice, S.stream));
  rw_group gr{0, n, *t, 0, 0};
  st = rw_state_write_groups(S.st, &gr, S.stream);
  if (st) return st;
  const uint32_t id = 0;
  st = rw_optimizer_step(S.st, h, &id, 1, nullptr, UINT32_MAX, S.stream);
  if (st) return st;
  void* outs[5] = {x, g, m, v, vmax};
  for (int i = 0; i < 5; ++i)
    if (use[i]) RW_CUDA(cudaMemcpyAsync(outs[i], S.d[i], bytes, cudaMemcpyDeviceToHost, S.stream));
  *t += 1;  // optim.cpp:281-282
  *updated = 1;
  return rw_state_check(S.st, S.stream);  // :361-363, after mutation
}

// optimizer_undo on a host ParamBlock (optim.cpp:288-307)
int rw_host_block_undo(int32_t dtype, void* x, void* g, void* m, void* v, uint64_t n, uint64_t* t,
                       uint32_t* updated, const rw_hyper* h) {
  if (!x || !g || !t || !updated || !h) return fail(RW_INVALID_ARGUMENT, "null argument");
  if (dtype != RW_F32 && dtype != RW_F64) return fail(RW_INVALID_ARGUMENT, "bad dtype");
  if (n == 0) return fail(RW_INVALID_SHAPE, "InvalidShape: zero extent");
  // the guards (NothingToUndo, AMSGrad, lr_at, per-kind hyper) run inside
  // rw_optimizer_undo before any launch; check the flag first so a refused
  // call never touches the device.
  if (!*updated) return fail(RW_NOTHING_TO_UNDO, "NothingToUndo: block has no pending update");
  if (h->kind == RW_AMSGRAD) return fail(RW_NOT_INVERTIBLE, "NotInvertible: amsgrad element-wise max has no inverse");
  if (h->kind == RW_LAMB)
    return fail(RW_INVALID_ARGUMENT, "lamb needs the saved-scalar stack: use rw_host_block_lamb_undo");
  const bool um = h->kind != RW_SGD, uv = h->kind == RW_ADAM || h->kind == RW_ADAMW;
  if ((um && !m) || (uv && !v)) return fail(RW_INVALID_ARGUMENT, "%s needs its m/v buffers", kind_name(h->kind));
  int st = stage_prepare(dtype, n);
  if (st) return st;
  HostStage& S = g_stage;
  const size_t bytes = n * elem_size(dtype);
  rw_group gr{0, n, *t, 1, 0};
  st = rw_state_write_groups(S.st, &gr, S.stream);
  if (st) return st;
  void* hs[4] = {x, g, m, v};
  const bool use[4] = {true, true, um, uv};
  const uint32_t id = 0;
  for (int i = 0; i < 4; ++i)
    if (use[i]) RW_CUDA(cudaMemcpyAsync(S.d[i], hs[i], bytes, cudaMemcpyHostToDevice, S.stream));
  st = rw_optimizer_undo(S.st, h, &id, 1, S.stream);
  if (st) return st;
  const bool out[4] = {true, false, um, uv};
  for (int i = 0; i < 4; ++i)
    if (out[i]) RW_CUDA(cudaMemcpyAsync(hs[i], S.d[i], bytes, cudaMemcpyDeviceToHost, S.stream));
  *t -= 1;  // optim.cpp:302-303
  *updated = 0;
  return rw_state_check(S.st, S.stream);  // :382-384, after mutation
}

int rw_host_block_lamb_step(int32_t dtype, void* x, void* g, void* m, void* v, uint64_t n, uint64_t* t,
                            uint32_t* updated, const void* grad, const rw_hyper* h, double* trust_out) {
  if (!x || !g || !m || !v || !t || !updated || !h || !grad || !trust_out)
    return fail(RW_INVALID_ARGUMENT, "null argument");
  if (h->kind != RW_LAMB) return fail(RW_INVALID_ARGUMENT, "rw_host_block_lamb_step needs kind RW_LAMB");
  if (dtype != RW_F32 && dtype != RW_F64) return fail(RW_INVALID_ARGUMENT, "bad dtype");
  if (n == 0) return fail(RW_INVALID_SHAPE, "InvalidShape: zero extent");
  const size_t bytes = n * elem_size(dtype);
  double eta = 0;
  int st = block_guards_step(h, *t, *updated, &eta);
  if (st) {
    if (st == RW_INVALID_CONFIG) std::memcpy(g, grad, bytes);
    return st;
  }
  st = stage_prepare(dtype, n);
  if (st) return st;
  HostStage& S = g_stage;
  void* hs[4] = {x, const_cast<void*>(grad), m, v};
  for (int i = 0; i < 4; ++i) RW_CUDA(cudaMemcpyAsync(S.d[i], hs[i], bytes, cudaMemcpyHostToDevice, S.stream));
  rw_group gr{0, n, *t, 0, 0};
  st = rw_state_write_groups(S.st, &gr, S.stream);
  if (st) return st;
  st = rw_state_set_saved_scalars(S.st, 0, nullptr, 0, S.stream);
  if (st) return st;
  const uint32_t id = 0;
  st = rw_optimizer_step(S.st, h, &id, 1, nullptr, UINT32_MAX, S.stream);
  if (st) return st;
  void* outs[4] = {x, g, m, v};
  for (int i = 0; i < 4; ++i) RW_CUDA(cudaMemcpyAsync(outs[i], S.d[i], bytes, cudaMemcpyDeviceToHost, S.stream));
  uint32_t cnt = 0;
  st = rw_state_saved_scalars(S.st, 0, trust_out, 1, &cnt, S.stream);
  if (st) return st;
  *t += 1;
  *updated = 1;
  return rw_state_check(S.st, S.stream);
}

int rw_host_block_lamb_undo(int32_t dtype, void* x, void* g, void* m, void* v, uint64_t n, uint64_t* t,
                            uint32_t* updated, const rw_hyper* h, uint32_t have_saved, double trust) {
  if (!x || !g || !m || !v || !t || !updated || !h) return fail(RW_INVALID_ARGUMENT, "null argument");
  if (h->kind != RW_LAMB) return fail(RW_INVALID_ARGUMENT, "rw_host_block_lamb_undo needs kind RW_LAMB");
  if (dtype != RW_F32 && dtype != RW_F64) return fail(RW_INVALID_ARGUMENT, "bad dtype");
  if (n == 0) return fail(RW_INVALID_SHAPE, "InvalidShape: zero extent");
  if (!*updated) return fail(RW_NOTHING_TO_UNDO, "NothingToUndo: block has no pending update");
  double eta = 0;
  int st = lr_at(h, *t, &eta);
  if (st) return st;
  if (h->beta1 == 0.0 || h->beta2 == 0.0)
    return fail(RW_NON_INVERTIBLE_HYPER, "NonInvertibleHyper: beta1*beta2 == 0 for lamb");
  if (!have_saved) return fail(RW_NOTHING_TO_UNDO, "NothingToUndo: no saved trust ratio for lamb undo");
  st = stage_prepare(dtype, n);
  if (st) return st;
  HostStage& S = g_stage;
  const size_t bytes = n * elem_size(dtype);
  rw_group gr{0, n, *t, 1, 0};
  st = rw_state_write_groups(S.st, &gr, S.stream);
  if (st) return st;
  st = rw_state_set_saved_scalars(S.st, 0, &trust, 1, S.stream);
  if (st) return st;
  void* hs[4] = {x, g, m, v};
  for (int i = 0; i < 4; ++i) RW_CUDA(cudaMemcpyAsync(S.d[i], hs[i], bytes, cudaMemcpyHostToDevice, S.stream));
  const uint32_t id = 0;
  st = rw_optimizer_undo(S.st, h, &id, 1, S.stream);
  if (st) return st;
  const bool out[4] = {true, false, true, true};
  for (int i = 0; i < 4; ++i)
    if (out[i]) RW_CUDA(cudaMemcpyAsync(hs[i], S.d[i], bytes, cudaMemcpyDeviceToHost, S.stream));
  *t -= 1;
  *updated = 0;
  return rw_state_check(S.st, S.stream);
}

}  // extern "C"

// ---------------- peer memory (CUDA IPC over NVLink) ----------------
#include <cuda.h>

namespace {
using AddrRangeFn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
AddrRangeFn addr_range_fn() {
  static AddrRangeFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<AddrRangeFn>(p);
  }
  return fn;
}
}  // namespace

extern "C" {

int rw_ipc_export(const void* ptr, void* handle_out, uint64_t* offset_out) {
  rwb::DeviceScope dev_scope(rwb::DeviceScope::device_of(ptr));
  if (!ptr || !handle_out || !offset_out) return fail(RW_INVALID_ARGUMENT, "null argument");
  AddrRangeFn fn = addr_range_fn();
  if (!fn) return fail(RW_CUDA_ERROR, "cuMemGetAddressRange unavailable");
  CUdeviceptr base = 0;
  size_t size = 0;
  if (fn(&base, &size, reinterpret_cast<CUdeviceptr>(ptr)) != CUDA_SUCCESS)
    return fail(RW_CUDA_ERROR, "cuMemGetAddressRange failed");
  cudaIpcMemHandle_t h;
  RW_CUDA(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
  std::memcpy(handle_out, &h, sizeof(h));
  *offset_out = reinterpret_cast<uint64_t>(ptr) - static_cast<uint64_t>(base);
  return RW_OK;
}

int rw_ipc_import(const void* handle, void** base_out) {
  if (!handle || !base_out) return fail(RW_INVALID_ARGUMENT, "null argument");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  RW_CUDA(cudaIpcOpenMemHandle(base_out, h, cudaIpcMemLazyEnablePeerAccess));
  return RW_OK;
}

int rw_ipc_close(void* base) {
  RW_CUDA(cudaIpcCloseMemHandle(base));
  return RW_OK;
}

// apply_undo fused with recover_replication:
// one launch undoes `undo_ids` in place AND streams every group of the
// resolved state (x, m, v; g when peer_g) into a peer replica over NVLink.
int rw_undo_and_push(rw_state* s, const rw_hyper* h, const uint32_t* undo_ids, uint32_t n_undo, void* peer_x,
                     void* peer_g, void* peer_m, void* peer_v, void* stream) {
  rwb::DeviceScope dev_scope(s ? s->device : -1);
  if (!s || !h || !peer_x || (n_undo && !undo_ids)) return fail(RW_INVALID_ARGUMENT, "null argument");
  const bool um = h->kind != RW_SGD, uv = h->kind == RW_ADAM || h->kind == RW_ADAMW || h->kind == RW_LAMB;
  if ((um && !peer_m) || (uv && !peer_v)) return fail(RW_INVALID_ARGUMENT, "peer m/v buffers required");
  const uint32_t G = static_cast<uint32_t>(s->mirror.size());
  std::vector<uint8_t> is_undo(G, 0);
  std::vector<double> etas_u(n_undo);
  for (uint32_t i = 0; i < n_undo; ++i) {
    if (undo_ids[i] >= G) return fail(RW_INVALID_ARGUMENT, "group id %u out of range", undo_ids[i]);
    if (is_undo[undo_ids[i]]) return fail(RW_INVALID_ARGUMENT, "group id %u listed twice", undo_ids[i]);
    is_undo[undo_ids[i]] = 1;
  }
  // the undo guards of rw_optimizer_undo, same order, before any launch
  for (uint32_t i = 0; i < n_undo; ++i) {
    const rw_group& gr = s->mirror[undo_ids[i]];
    if (!gr.updated) return fail(RW_NOTHING_TO_UNDO, "NothingToUndo: block has no pending update (group %u)", undo_ids[i]);
    if (h->kind == RW_AMSGRAD) return fail(RW_NOT_INVERTIBLE, "NotInvertible: amsgrad element-wise max has no inverse");
    int st = lr_at(h, gr.t, &etas_u[i]);
    if (st) return st;
    if (h->kind == RW_SGDM && h->momentum == 0.0)
      return fail(RW_NON_INVERTIBLE_HYPER, "NonInvertibleHyper: momentum == 0 for sgdm");
    if ((h->kind == RW_ADAM || h->kind == RW_ADAMW) && (h->beta1 == 0.0 || h->beta2 == 0.0))
      return fail(RW_NON_INVERTIBLE_HYPER, "NonInvertibleHyper: beta1*beta2 == 0");
    if ((h->kind == RW_SGD || h->kind == RW_ADAMW) && 1.0 - etas_u[i] * h->weight_decay == 0.0)
      return fail(RW_NON_INVERTIBLE_HYPER, "NonInvertibleHyper: lr*weight_decay == 1");
  }
  if (h->kind == RW_LAMB) {
    int st = lamb_undo_scalars(s, h, undo_ids, n_undo, etas_u, stream);
    if (st) return st;
  }
  // every group, in layout order: undo groups flagged, the rest copy-only
  std::vector<uint32_t> ids(G);
  std::vector<uint8_t> copy(G);
  std::vector<double> etas(G, 0.0);
  uint32_t k = 0;
  for (uint32_t gi = 0; gi < G; ++gi) {
    ids[gi] = gi;
    copy[gi] = is_undo[gi] ? 0 : 1;
  }
  for (uint32_t i = 0; i < n_undo; ++i) etas[undo_ids[i]] = etas_u[i];
  (void)k;
  void* peers[4] = {peer_x, peer_g, peer_m, peer_v};
  return launch_groups(s, h, ids.data(), G, true, nullptr, etas, stream, copy.data(), peers);
}

}  // extern "C"
