// Internal declarations shared by the CUDA kernels and the C-ABI host code.
// Not part of the public boundary (see include/rewind_b200.h).
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <mutex>

#include "rewind_b200.h"

namespace rwb {

// Per selected group, per launch.  Built on the host in update order.
struct WorkItem {
  uint64_t off;          // element offset of the group in the flat buffers
  uint64_t len;          // elements
  uint64_t new_t;        // marker value written when the group completes
  uint32_t gid;          // index into the device marker table
  uint32_t chunk_begin;  // first global chunk index of this group
  uint32_t nchunks;
  uint32_t sidx;         // index into the ScalarSet table
  uint32_t flags;        // kWorkCopyOnly: pass the group through (push only)
  uint32_t pad;
};
constexpr uint32_t kWorkCopyOnly = 1u;

// t-dependent scalars of one call, derived in double on the host exactly as
// optim.cpp does (lr_at :50-57, bias_correction :94-97, denom :106/:177).
struct ScalarSet {
  double eta, c1, c2, denom;
};

// t-independent scalars (optim.cpp: 1.0 - h.beta1 etc. are double
// expressions evaluated per element in the reference; they are loop
// invariant so one host evaluation is the same value).
struct Uniform {
  double wd, mu, one_m_damp, b1, b2, one_m_b1, one_m_b2, eps;
};

// Small calls carry their work list and scalar sets in the kernel's
// parameter space (__grid_constant__) instead of a pinned H2D copy: no copy
// on the stream ahead of the kernel, so a 50-group undo costs one launch.
#ifndef RW_INLINE_ITEMS
#define RW_INLINE_ITEMS 128
#endif
constexpr uint32_t kInlineItems = RW_INLINE_ITEMS;
constexpr uint32_t kInlineSets = 16;
struct InlineMeta {
  WorkItem work[kInlineItems];
  ScalarSet sets[kInlineSets];
};

struct LaunchArgs {
  int dtype;     // RW_F32 / RW_F64
  int kind;      // RW_SGD..RW_AMSGRAD
  bool undo;
  void* x;
  void* g;
  void* m;
  void* v;
  void* vmax;
  const void* grad;  // step only; nullptr or == g means "g already holds it"
  const WorkItem* work;
  uint32_t n_work;
  uint32_t total_chunks;
  uint32_t chunk_elems;
  const ScalarSet* sets;
  Uniform u;
  rw_group* groups;
  uint32_t* done;
  // fused replica push (rw_undo_and_push): peer buffers, same layout; null = off
  void* px = nullptr;
  void* pg = nullptr;
  void* pm = nullptr;
  void* pv = nullptr;
  // work == nullptr: the work list and sets are in *inl (host memory, copied
  // into the launch's parameters)
  const InlineMeta* inl = nullptr;
};

// One-time per-device setup of a call site (kernel attributes such as the
// max dynamic smem, occupancy queries): `setup(device)` runs under a lock, and
// the device's bit is published only after it succeeded, so a failed setup is
// retried by the next call and no concurrent caller sees half-written values.
class DeviceOnce {
 public:
  template <class F>
  int run(F&& setup) {
    int d = 0;
    cudaGetDevice(&d);
    const unsigned long long b = 1ull << (d & 63);
    if (mask_.load(std::memory_order_acquire) & b) return 0;
    std::lock_guard<std::mutex> lk(mu_);
    if (mask_.load(std::memory_order_relaxed) & b) return 0;
    const int e = setup(d);
    if (e == 0) mask_.fetch_or(b, std::memory_order_release);
    return e;
  }

 private:
  std::mutex mu_;
  std::atomic<unsigned long long> mask_{0};
};

// The CUDA runtime is shared with the caller (PyTorch), whose current device
// may differ from the memory an entry point works on (PyTorch sets devices
// lazily).  Every entry point that launches work binds the device of the state
// / the caller's memory for its duration and restores the caller's device.
class DeviceScope {
 public:
  explicit DeviceScope(int dev) { bind(dev); }
  ~DeviceScope() {
    if (changed_) cudaSetDevice(prev_);
  }
  DeviceScope(const DeviceScope&) = delete;
  DeviceScope& operator=(const DeviceScope&) = delete;
  // device of a device pointer, or -1 for host / unknown memory
  static int device_of(const void* p) {
    if (!p) return -1;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
      cudaGetLastError();
      return -1;
    }
    return (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) ? a.device : -1;
  }

 private:
  void bind(int dev) {
    if (dev < 0 || cudaGetDevice(&prev_) != cudaSuccess || prev_ == dev) return;
    changed_ = cudaSetDevice(dev) == cudaSuccess;
  }
  int prev_ = 0;
  bool changed_ = false;
};

// record the thread-local last-error message (rw_last_error_message)
void set_error(const char* msg);
// elements per chunk for a dtype (one chunk = one CTA work unit)
uint32_t chunk_elems_for(int dtype);
// launch the fused step/undo kernel; returns cudaError_t as int
int launch_optim(const LaunchArgs& a, void* stream);
int launch_seeded_fill(int dtype, void* out, uint64_t n, uint64_t seed, uint64_t offset, void* stream);
int launch_ordered_sum(int dtype, const void* const* tensors, uint32_t count, uint64_t n, void* out,
                       void* stream);
int launch_clear_updated(rw_group* groups, const uint32_t* ids, uint32_t n, void* stream);

// lamb_kernels.cu: LAMB step pass 1 (m, v and both norms) over the work list
// + one trust CTA per item: trust -> trust_table[gid * depth + item.pad],
// sets[item.sidx].eta *= trust (scaled), .denom = 1 - scaled * wd.
// partial: 2 doubles per chunk.
int launch_lamb_pass1(int dtype, void* x, void* g, const void* grad, void* m, void* v, const WorkItem* work,
                      uint32_t n_work, uint32_t total_chunks, uint32_t chunk_elems, ScalarSet* sets,
                      const Uniform& u, double* partial, double* trust_table, uint32_t depth, bool sequential,
                      void* stream);

// log_kernels.cu: CRC32 (wire.cpp:31-38) of a device buffer into *out_dev;
// scratch = crc32_scratch_words(n) device uint32 words
int launch_crc32(const void* data, uint64_t n, uint32_t* out_dev, uint32_t* scratch, void* stream);
uint64_t crc32_scratch_words(uint64_t n);

// replay_kernels.cu (all return cudaError_t as int)
int replay_forward_layer(const void* x, int64_t rows, int64_t in, int64_t out, const void* w, const float* b,
                         void* y, void* stream);
// colsum (optional, y_prev != NULL): the epilogue also writes the per-32-row column
// sums of dst, [ceil(rows/32), in] fp32 (fused db partials); *fused reports whether
// it did (it cannot when the output is not a TMA operand or the engine is the
// register epilogue), and then replay_colsum must run instead
int replay_dgrad_layer(const void* dz, int64_t rows, int64_t in, int64_t out, const void* w,
                       const void* y_prev, void* dst, void* stream, float* colsum = nullptr,
                       int* fused = nullptr);
// db (+)= the nsplit partial rows of part [nsplit, cols], summed in row order
int replay_colsum_final(const float* part, int64_t nsplit, int64_t cols, float* db, int accumulate, void* stream);
int replay_wgrad_layer(const void* x, const void* dz, int64_t rows, int64_t in, int64_t out, float* dw,
                       int accumulate, void* stream);
int replay_set_sm_reserve(int n);
int replay_set_gemm_engine(int epilogue, int pair);
// first-layer dgrad of stage k fused with stage k-1's dz: bf16(dX) * (1 - y^2)
int replay_dgrad_boundary(const void* dz, int64_t rows, int64_t in, int64_t out, const void* w,
                          const void* y_prev_stage, void* dz_prev_stage, void* stream);
int replay_dtanh_first(const void* g, const void* y, void* dz, uint64_t n, void* stream);
int replay_colsum(const void* dz, int64_t rows, int64_t cols, float* db, float* scratch, int accumulate,
                  void* stream);
int replay_cast_bf16(const float* in, void* out, uint64_t n, void* stream);
int replay_mse_grad(const void* pred, const float* target, uint64_t n, uint64_t micro_batches, void* grad,
                    double* loss, double* scratch, void* stream);

}  // namespace rwb
