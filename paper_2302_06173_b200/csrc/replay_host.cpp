// C++ replay drivers (recovery.cpp is absent from the reference):
// recover_replay of a contiguous group of stages on one GPU and
// recover_parallel over the helpers of an rw_comm, both composed from the
// replay compute of replay_capi.cpp (forward_stage / backward_stage /
// accumulate_grads / mse_loss, model.cpp:77-188) and the fused optimizer step.
// Same arithmetic and order as the Python drivers (replay.py), so a replay is
// bit-identical to the GPU ghost run and parallel == sequential bit for bit.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <vector>

#include "internal.h"

namespace {

int pfail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  rwb::set_error(buf);
  return code;
}

#define PCK(call)                \
  do {                           \
    const int s_ = (call);       \
    if (s_) return s_;           \
  } while (0)

constexpr uint64_t kAlign = 256;
uint64_t up(uint64_t b) { return (b + kAlign - 1) / kAlign * kAlign; }

struct StageView {
  const rw_replay_stage* s;
  int L;
  std::vector<int64_t> dims;
  std::vector<uint64_t> off;  // element offsets of blocks W0, b0, W1, b1, ... in the state
  std::vector<uint64_t> len;
  uint64_t grad_elems = 0;    // flat gradient length (the state's total)
};

int view_stages(const rw_replay_stage* stages, uint32_t n, std::vector<StageView>& out) {
  out.clear();
  for (uint32_t k = 0; k < n; ++k) {
    const rw_replay_stage& s = stages[k];
    if (!s.state || !s.grad || !s.desc.dims || !s.desc.w || !s.desc.b || s.desc.num_layers < 1)
      return pfail(RW_INVALID_ARGUMENT, "stage %u: incomplete rw_replay_stage", k);
    StageView v;
    v.s = &s;
    v.L = s.desc.num_layers;
    v.dims.assign(s.desc.dims, s.desc.dims + v.L + 1);
    const uint32_t G = rw_state_num_groups(s.state);
    if (G != uint32_t(2 * v.L)) return pfail(RW_SHAPE_MISMATCH, "ShapeMismatch: stage %u state has %u blocks", k, G);
    std::vector<rw_group> g(G);
    PCK(rw_state_read_groups(s.state, g.data(), nullptr));
    for (int l = 0; l < v.L; ++l) {
      if (g[2 * l].len != uint64_t(v.dims[l] * v.dims[l + 1]) || g[2 * l + 1].len != uint64_t(v.dims[l + 1]))
        return pfail(RW_SHAPE_MISMATCH, "ShapeMismatch: stage %u layer %d blocks", k, l);
    }
    for (auto& r : g) v.off.push_back(r.offset), v.len.push_back(r.len);
    PCK(rw_state_info(s.state, nullptr, &v.grad_elems, nullptr));
    if (k > 0 && v.dims[0] != out.back().dims.back())
      return pfail(RW_SHAPE_MISMATCH, "ShapeMismatch: stage %u input width differs from stage %u output", k, k - 1);
    out.push_back(std::move(v));
  }
  return RW_OK;
}

// Workspace carve-up (everything 256-byte aligned), shared by both drivers.
struct Work {
  std::vector<std::vector<void*>> acts;  // per stage: L + 1 activation pointers (acts[0] set per mb)
  void* input = nullptr;                  // synth_inputs of the first stage (bf16)
  float* target = nullptr;                // synth_targets (fp32)
  void* loss_grad = nullptr;              // mse gradient (bf16)
  double* mse_scratch = nullptr;
  void* gbuf[2] = {nullptr, nullptr};     // stage-boundary gradients (ping-pong)
  void* dz0 = nullptr;
  void* dz1 = nullptr;
  float* f32 = nullptr;
  uint64_t f32_elems = 0;
  std::vector<std::vector<float*>> mb_grads;  // parallel: [my mb index][stage] flat partials
  std::vector<float*> merged;                 // parallel: per stage, rw_ordered_reduce_out_elems
  float* reduce_scratch = nullptr;
  uint64_t reduce_scratch_elems = 0;
  uint64_t bytes = 0;
};

int carve(const std::vector<StageView>& sv, int64_t rows, uint32_t my_mbs, int32_t d, int32_t rank, uint32_t m,
          bool parallel, char* base, Work& w) {
  uint64_t at = 0;
  auto take = [&](uint64_t bytes) -> void* {
    void* p = base ? base + at : nullptr;
    at += up(bytes);
    return p;
  };
  const uint64_t R = uint64_t(rows);
  int64_t mx = 0;
  for (auto& v : sv)
    for (int64_t x : v.dims) mx = std::max(mx, x);
  w = Work{};
  w.acts.assign(sv.size(), {});
  for (size_t k = 0; k < sv.size(); ++k) {
    w.acts[k].assign(sv[k].L + 1, nullptr);
    for (int l = 1; l <= sv[k].L; ++l) w.acts[k][l] = take(R * uint64_t(sv[k].dims[l]) * 2);
  }
  const int64_t din = sv.front().dims.front(), dout = sv.back().dims.back();
  w.input = take(R * uint64_t(din) * 2);
  w.target = static_cast<float*>(take(R * uint64_t(dout) * 4));
  w.loss_grad = take(R * uint64_t(dout) * 2);
  w.mse_scratch = static_cast<double*>(take(256 * 8));
  w.gbuf[0] = take(R * uint64_t(mx) * 2);
  w.gbuf[1] = take(R * uint64_t(mx) * 2);
  w.dz0 = take(R * uint64_t(mx) * 2);
  w.dz1 = take(R * uint64_t(mx) * 2);
  w.f32_elems = std::max<uint64_t>(64, (R + 31) / 32) * uint64_t(mx);
  w.f32 = static_cast<float*>(take(w.f32_elems * 4));
  if (parallel) {
    w.mb_grads.assign(my_mbs, {});
    for (uint32_t i = 0; i < my_mbs; ++i)
      for (auto& v : sv) w.mb_grads[i].push_back(static_cast<float*>(take(v.grad_elems * 4)));
    uint64_t scr = 0;
    for (auto& v : sv) {
      w.merged.push_back(static_cast<float*>(take(rw_ordered_reduce_out_elems(v.grad_elems, d) * 4)));
      scr = std::max(scr, rw_ordered_reduce_scratch_elems(v.grad_elems, m, d, rank));
    }
    w.reduce_scratch_elems = scr;
    w.reduce_scratch = static_cast<float*>(take(std::max<uint64_t>(scr, 1) * 4));
  }
  w.bytes = at;
  return RW_OK;
}

// forward of one micro-batch through every stage (acts[k][0] = the input)
int forward_mb(const std::vector<StageView>& sv, Work& w, int64_t rows, const void* x, void* stream) {
  for (size_t k = 0; k < sv.size(); ++k) {
    w.acts[k][0] = const_cast<void*>(x);
    PCK(rw_stage_forward(&sv[k].s->desc, rows, w.acts[k].data(), stream));
    x = w.acts[k][sv[k].L];
  }
  return RW_OK;
}

// backward of one micro-batch through every stage in reverse, group-internal
// boundaries fused (stage k's first-layer dgrad emits stage k-1's dz directly,
// rw_stage_backward_ex); gradients into dw/db of `grads[k]` (accumulate: +=)
int backward_mb(const std::vector<StageView>& sv, Work& w, int64_t rows, const void* g,
                const std::vector<float*>& grads, int accumulate, void* stream) {
  const int n = static_cast<int>(sv.size());
  int pp = 0;
  for (int k = n - 1; k >= 0; --k) {
    const StageView& v = sv[size_t(k)];
    std::vector<float*> dw(v.L), db(v.L);
    for (int l = 0; l < v.L; ++l) {
      dw[l] = grads[size_t(k)] + v.off[2 * l];
      db[l] = grads[size_t(k)] + v.off[2 * l + 1];
    }
    void* gout = k > 0 ? w.gbuf[pp] : nullptr;
    const void* prev_y = k > 0 ? w.acts[size_t(k) - 1][sv[size_t(k) - 1].L] : nullptr;
    PCK(rw_stage_backward_ex2(&v.s->desc, rows, w.acts[size_t(k)].data(), g, k < n - 1, gout, prev_y, dw.data(),
                              db.data(), accumulate, w.dz0, w.dz1, w.f32, w.f32_elems, stream));
    g = gout;
    pp ^= 1;
  }
  return RW_OK;
}

int inputs_of(const rw_replay_log* log, const std::vector<StageView>& sv, Work& w, int64_t rows, uint32_t m,
              uint64_t it, uint64_t it0, uint32_t mb, const void** x, void* stream) {
  const uint64_t slot = (it - it0) * m + mb;
  if (!log->acts) {  // the group starts the pipeline: synth_inputs (model.cpp:190-193), never logged
    const uint64_t parts[3] = {1, it, mb};
    PCK(rw_seeded_fill(RW_BF16, w.input, uint64_t(rows) * uint64_t(sv.front().dims.front()),
                       rw_derive_seed(log->seed, parts, 3), 0, stream));
    *x = w.input;
    return RW_OK;
  }
  *x = log->acts[slot];
  if (!*x) return pfail(RW_MISSING_LOG_DATA, "MissingLogData: activation (%llu, %u)", (unsigned long long)it, mb);
  return RW_OK;
}

int grad_in_of(const rw_replay_log* log, const std::vector<StageView>& sv, Work& w, int64_t rows, uint32_t m,
               uint64_t it, uint64_t it0, uint32_t mb, const void** g, void* stream) {
  const uint64_t slot = (it - it0) * m + mb;
  if (!log->grads) {  // the group ends the pipeline: mse_loss vs synth_targets (model.cpp:174-198)
    const uint64_t parts[3] = {2, it, mb};
    const uint64_t n = uint64_t(rows) * uint64_t(sv.back().dims.back());
    PCK(rw_seeded_fill(RW_F32, w.target, n, rw_derive_seed(log->seed, parts, 3), 0, stream));
    PCK(rw_mse_grad(w.acts.back()[sv.back().L], w.target, n, m, w.loss_grad, nullptr, w.mse_scratch, stream));
    *g = w.loss_grad;
    return RW_OK;
  }
  *g = log->grads[slot];
  if (!*g) return pfail(RW_MISSING_LOG_DATA, "MissingLogData: gradient (%llu, %u)", (unsigned long long)it, mb);
  return RW_OK;
}

// apply_layerwise_updates over the group (stages and blocks in reverse layer
// order), the iteration-end flag clear, the bf16 shadow refresh
int step_stages(const std::vector<StageView>& sv, const rw_hyper* h, const std::vector<float*>& grads, void* stream) {
  for (size_t k = sv.size(); k-- > 0;) {
    const StageView& v = sv[k];
    const uint32_t G = uint32_t(2 * v.L);
    std::vector<uint32_t> ids(G);
    for (uint32_t i = 0; i < G; ++i) ids[i] = G - 1 - i;
    PCK(rw_optimizer_step(v.s->state, h, ids.data(), G, grads[k], UINT32_MAX, stream));
    PCK(rw_clear_updated(v.s->state, ids.data(), G, stream));
    const float* x = static_cast<const float*>(rw_state_ptr(v.s->state, 0));
    for (int l = 0; l < v.L; ++l)
      PCK(rw_cast_f32_to_bf16(x + v.off[2 * l], const_cast<void*>(v.s->desc.w[l]), v.len[2 * l], stream));
  }
  return RW_OK;
}

uint32_t my_count(uint32_t m, int32_t d, int32_t rank) {
  uint32_t c = 0;
  for (uint32_t mb = 0; mb < m; ++mb) c += int32_t(mb % uint32_t(d)) == rank;
  return c;
}

}  // namespace

extern "C" {

uint64_t rw_replay_workspace_bytes(const rw_replay_stage* stages, uint32_t n_stages, int64_t rows,
                                   uint32_t micro_batches, rw_comm* comm) {
  std::vector<StageView> sv;
  if (!stages || !n_stages || rows < 1 || view_stages(stages, n_stages, sv)) return 0;
  const int32_t d = comm ? rw_comm_size(comm) : 1, rank = comm ? rw_comm_rank(comm) : 0;
  Work w;
  const bool parallel = micro_batches > 0 && comm;
  carve(sv, rows, parallel ? my_count(micro_batches, d, rank) : 0, d, rank, micro_batches, parallel, nullptr, w);
  return w.bytes;
}

int rw_replay_group(const rw_replay_stage* stages, uint32_t n_stages, int64_t rows, uint32_t micro_batches,
                    uint64_t it0, uint64_t it1, const rw_hyper* h, const rw_replay_log* log, void* workspace,
                    uint64_t workspace_bytes, void* stream) {
  if (!stages || !n_stages || !h || !log || rows < 1 || micro_batches == 0 || it1 < it0)
    return pfail(RW_INVALID_ARGUMENT, "bad replay arguments");
  std::vector<StageView> sv;
  PCK(view_stages(stages, n_stages, sv));
  Work w;
  carve(sv, rows, 0, 1, 0, micro_batches, false, nullptr, w);
  if (!workspace || workspace_bytes < w.bytes)
    return pfail(RW_INVALID_ARGUMENT, "workspace of %llu bytes needed (rw_replay_workspace_bytes)",
                 (unsigned long long)w.bytes);
  carve(sv, rows, 0, 1, 0, micro_batches, false, static_cast<char*>(workspace), w);
  std::vector<float*> grads;
  for (auto& v : sv) grads.push_back(v.s->grad);
  for (uint64_t it = it0; it < it1; ++it) {
    for (uint32_t mb = 0; mb < micro_batches; ++mb) {  // timestamp order
      const void* x = nullptr;
      const void* g = nullptr;
      PCK(inputs_of(log, sv, w, rows, micro_batches, it, it0, mb, &x, stream));
      PCK(forward_mb(sv, w, rows, x, stream));
      PCK(grad_in_of(log, sv, w, rows, micro_batches, it, it0, mb, &g, stream));
      PCK(backward_mb(sv, w, rows, g, grads, mb > 0, stream));  // accumulate_grads in ascending mb order
    }
    PCK(step_stages(sv, h, grads, stream));
  }
  return RW_OK;
}

int rw_recover_parallel(const rw_replay_stage* stages, uint32_t n_stages, int64_t rows, uint32_t micro_batches,
                        uint64_t it0, uint64_t it1, const rw_hyper* h, const rw_replay_log* log, rw_comm* comm,
                        void* workspace, uint64_t workspace_bytes, void* stream) {
  if (!stages || !n_stages || !h || !log || !comm || rows < 1 || micro_batches == 0 || it1 < it0)
    return pfail(RW_INVALID_ARGUMENT, "bad recover_parallel arguments");
  std::vector<StageView> sv;
  PCK(view_stages(stages, n_stages, sv));
  const int32_t d = rw_comm_size(comm), rank = rw_comm_rank(comm);
  const uint32_t mine = my_count(micro_batches, d, rank);
  Work w;
  carve(sv, rows, mine, d, rank, micro_batches, true, nullptr, w);
  if (!workspace || workspace_bytes < w.bytes)
    return pfail(RW_INVALID_ARGUMENT, "workspace of %llu bytes needed (rw_replay_workspace_bytes)",
                 (unsigned long long)w.bytes);
  carve(sv, rows, mine, d, rank, micro_batches, true, static_cast<char*>(workspace), w);
  for (uint64_t it = it0; it < it1; ++it) {
    // this helper's micro-batches {mb : mb mod d == rank}, each into its own partials
    std::vector<std::vector<const float*>> parts(sv.size(), std::vector<const float*>(micro_batches, nullptr));
    uint32_t i = 0;
    for (uint32_t mb = 0; mb < micro_batches; ++mb) {
      if (int32_t(mb % uint32_t(d)) != rank) continue;
      const void* x = nullptr;
      const void* g = nullptr;
      PCK(inputs_of(log, sv, w, rows, micro_batches, it, it0, mb, &x, stream));
      PCK(forward_mb(sv, w, rows, x, stream));
      PCK(grad_in_of(log, sv, w, rows, micro_batches, it, it0, mb, &g, stream));
      PCK(backward_mb(sv, w, rows, g, w.mb_grads[i], 0, stream));
      for (size_t k = 0; k < sv.size(); ++k) parts[k][mb] = w.mb_grads[i][k];
      ++i;
    }
    // ascending-mb ordered merge of every stage, then the same step on every helper
    for (size_t k = sv.size(); k-- > 0;)
      PCK(rw_ordered_reduce(comm, parts[k].data(), micro_batches, sv[k].grad_elems, w.merged[k], w.reduce_scratch,
                            w.reduce_scratch_elems, stream));
    PCK(step_stages(sv, h, w.merged, stream));
  }
  return RW_OK;
}

}  // extern "C"
