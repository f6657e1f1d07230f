// C ABI of the replay compute (include/rewind_b200.h, "replay compute").
// Mirrors forward_stage / backward_stage / accumulate_grads / mse_loss
// (model.cpp:77-188) on device buffers; the layer loop order, the cached
// activations and the gradient flow are the reference's.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <string>

#include "internal.h"

namespace {
int rfail(int code, const char* msg) {
  rwb::set_error(msg);
  return code;
}
int cfail(int e, const char* what) {
  std::string m = std::string("CUDA error in ") + what + ": " + cudaGetErrorString(static_cast<cudaError_t>(e));
  rwb::set_error(m.c_str());
  return RW_CUDA_ERROR;
}
int check_desc(const rw_stage_desc* st, int64_t rows) {
  if (!st || !st->dims || !st->w || !st->b) return rfail(RW_INVALID_ARGUMENT, "null stage descriptor");
  if (st->num_layers < 1) return rfail(RW_INVALID_CONFIG, "InvalidConfig: stage needs >= 1 layer");
  if (rows < 1) return rfail(RW_INVALID_SHAPE, "InvalidShape: zero extent");
  for (int l = 0; l <= st->num_layers; ++l)
    if (st->dims[l] < 1 || (st->dims[l] % 8) != 0)
      return rfail(RW_INVALID_SHAPE, "InvalidShape: stage widths must be positive multiples of 8 (16-byte rows)");
  if (rw_device_count() == 0) return rfail(RW_CUDA_ERROR, "no CUDA device visible: the B200 path has no CPU fallback");
  return RW_OK;
}
}  // namespace

extern "C" {

int rw_stage_forward(const rw_stage_desc* st, int64_t rows, void* const* acts, void* stream) {
  rwb::DeviceScope dev_scope(rwb::DeviceScope::device_of(acts ? acts[0] : nullptr));
  int s = check_desc(st, rows);
  if (s) return s;
  if (!acts) return rfail(RW_INVALID_ARGUMENT, "null activations");
  for (int l = 0; l < st->num_layers; ++l) {  // model.cpp:84-87, layer order
    if (!acts[l] || !acts[l + 1]) return rfail(RW_MISSING_ACTIVATION, "MissingActivation: null activation buffer");
    int e = rwb::replay_forward_layer(acts[l], rows, st->dims[l], st->dims[l + 1], st->w[l], st->b[l], acts[l + 1],
                                      stream);
    if (e) return cfail(e, "stage forward GEMM");
  }
  return RW_OK;
}

int rw_stage_backward(const rw_stage_desc* st, int64_t rows, void* const* acts, const void* grad_in,
                      void* grad_out, float* const* dw, float* const* db, int32_t accumulate, void* dz0, void* dz1,
                      float* scratch, void* stream) {
  return rw_stage_backward_ex(st, rows, acts, grad_in, 0, grad_out, nullptr, dw, db, accumulate, dz0, dz1, scratch,
                              stream);
}

int rw_stage_backward_ex(const rw_stage_desc* st, int64_t rows, void* const* acts, const void* grad_in,
                         int32_t grad_in_is_dz, void* grad_out, const void* prev_y, float* const* dw,
                         float* const* db, int32_t accumulate, void* dz0, void* dz1, float* scratch, void* stream) {
  int s = check_desc(st, rows);
  if (s) return s;
  int64_t mx = 0;
  for (int l = 0; l <= st->num_layers; ++l) mx = st->dims[l] > mx ? st->dims[l] : mx;
  return rw_stage_backward_ex2(st, rows, acts, grad_in, grad_in_is_dz, grad_out, prev_y, dw, db, accumulate, dz0,
                               dz1, scratch, uint64_t(64) * uint64_t(mx), stream);
}

int rw_stage_backward_ex2(const rw_stage_desc* st, int64_t rows, void* const* acts, const void* grad_in,
                          int32_t grad_in_is_dz, void* grad_out, const void* prev_y, float* const* dw,
                          float* const* db, int32_t accumulate, void* dz0, void* dz1, float* scratch,
                          uint64_t scratch_elems, void* stream) {
  rwb::DeviceScope dev_scope(rwb::DeviceScope::device_of(grad_in));
  int s = check_desc(st, rows);
  if (s) return s;
  if (!acts || !grad_in || !dw || !db || !dz0 || !dz1 || !scratch)
    return rfail(RW_INVALID_ARGUMENT, "null argument");
  if (prev_y && !grad_out) return rfail(RW_INVALID_ARGUMENT, "prev_y needs grad_out");
  for (int l = 0; l <= st->num_layers; ++l)
    if (!acts[l]) return rfail(RW_MISSING_ACTIVATION, "MissingActivation: no cached forward for micro-batch");
  const int L = st->num_layers;
  // dz of the last layer: dL/dy * (1 - y^2)  (model.cpp:113-120) -- or
  // already fused into the next stage's first-layer dgrad (grad_in_is_dz)
  void* cur = dz0;
  void* nxt = dz1;
  int e = 0;
  if (grad_in_is_dz) {
    cur = const_cast<void*>(grad_in);
  } else {
    e = rwb::replay_dtanh_first(grad_in, acts[L], cur, uint64_t(rows) * uint64_t(st->dims[L]), stream);
    if (e) return cfail(e, "dtanh");
  }
  // db partials of the dz in `cur` already written by the GEMM that produced it
  // (per 32-row block, into scratch) when the scratch holds ceil(rows/32) rows
  const int64_t nsplit = (rows + 31) / 32;
  bool cur_fused = false;
  for (int li = L - 1; li >= 0; --li) {  // reverse layer order (model.cpp:107)
    const int64_t in = st->dims[li], out = st->dims[li + 1];
    // dW = x^T dz (:193-203), accumulated over micro-batches in order
    e = rwb::replay_wgrad_layer(acts[li], cur, rows, in, out, dw[li], accumulate, stream);
    if (e) return cfail(e, "wgrad GEMM");
    // db = column sums of dz (:204-209)
    e = cur_fused ? rwb::replay_colsum_final(scratch, nsplit, out, db[li], accumulate, stream)
                  : rwb::replay_colsum(cur, rows, out, db[li], scratch, accumulate, stream);
    if (e) return cfail(e, "db colsum");
    // dx = dz W^T (:210-219); for li > 0 fuse the next layer's (1 - y^2)
    // (and the column sums of the dz it produces)
    if (li > 0) {
      int fused = 0;
      float* part = uint64_t(nsplit) * uint64_t(in) <= scratch_elems ? scratch : nullptr;
      e = rwb::replay_dgrad_layer(cur, rows, in, out, st->w[li], acts[li], nxt, stream, part, &fused);
      if (e) return cfail(e, "dgrad GEMM");
      cur_fused = fused != 0;
      std::swap(cur, nxt);
    } else if (grad_out && prev_y) {  // dz of the previous stage (same GPU), bit-identical
      e = rwb::replay_dgrad_boundary(cur, rows, in, out, st->w[li], prev_y, grad_out, stream);
      if (e) return cfail(e, "dgrad GEMM");
    } else if (grad_out) {
      e = rwb::replay_dgrad_layer(cur, rows, in, out, st->w[li], nullptr, grad_out, stream);
      if (e) return cfail(e, "dgrad GEMM");
    }
  }
  return RW_OK;
}

int rw_mse_grad(const void* pred, const float* target, uint64_t n, uint64_t micro_batches, void* grad, double* loss,
                double* scratch, void* stream) {
  rwb::DeviceScope dev_scope(rwb::DeviceScope::device_of(pred));
  if (micro_batches == 0) return rfail(RW_INVALID_CONFIG, "InvalidConfig: micro_batches must be >= 1");
  if (!pred || !target || !grad || !scratch) return rfail(RW_INVALID_ARGUMENT, "null argument");
  int e = rwb::replay_mse_grad(pred, target, n, micro_batches, grad, loss, scratch, stream);
  if (e) return cfail(e, "mse");
  return RW_OK;
}

int rw_replay_set_sm_reserve(int32_t n) { return rwb::replay_set_sm_reserve(n); }
int rw_replay_set_gemm_engine(int32_t epilogue, int32_t pair) { return rwb::replay_set_gemm_engine(epilogue, pair); }

int rw_cast_f32_to_bf16(const float* in, void* out, uint64_t n, void* stream) {
  rwb::DeviceScope dev_scope(rwb::DeviceScope::device_of(in));
  if (!in || !out) return rfail(RW_INVALID_ARGUMENT, "null argument");
  int e = rwb::replay_cast_bf16(in, out, n, stream);
  if (e) return cfail(e, "cast");
  return RW_OK;
}

}  // extern "C"
