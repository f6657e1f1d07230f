// A C++ host driving the whole single-survivor repair through the C ABI only
// (no Python): the reference's own ParamBlocks (rewind_ref, oracle/_ref) and
// a flat fp64 device state hold the same model; both take a layer-wise Adam
// update that is torn after k blocks (MidUpdate(k), reverse layer order,
// SPEC:229-231, 334-342); the device side then reads its markers, resolves
// (rw_resolve_summarize x2 + rw_resolve_plan) and undoes the updated groups
// in one launch, the reference side runs optimizer_undo on the same blocks.
// Every value and marker must agree bit for bit after each phase.
//
//   resolve_undo_test   (B200; prints "<n> failure(s)")
#include <bits/stdc++.h>
#define rewind rewind_ref
#include "rewind/errors.hpp"
#include "rewind/optim.hpp"
#include "rewind/tensor.hpp"
#undef rewind

#include <cuda_runtime.h>

#include "rewind_b200.h"

namespace R = rewind_ref;

static int g_fail = 0;
#define EXPECT(cond, what)                                       \
  do {                                                           \
    if (!(cond)) {                                               \
      std::printf("FAIL %s (%s:%d)\n", what, __FILE__, __LINE__); \
      ++g_fail;                                                  \
    }                                                            \
  } while (0)
#define CK(call)                                                                   \
  do {                                                                             \
    int st_ = (call);                                                              \
    if (st_) {                                                                     \
      std::printf("FAIL %s -> %d (%s)\n", #call, st_, rw_last_error_message());    \
      return 1;                                                                    \
    }                                                                              \
  } while (0)

int main() {
  if (rw_device_count() == 0) {
    std::printf("resolve_undo_test: no GPU\n");
    return 1;
  }
  const std::vector<size_t> sizes = {1000, 37, 4096, 70001, 5, 2048, 999, 12345};
  const uint32_t G = static_cast<uint32_t>(sizes.size()), k_crash = 5;
  R::OptimizerHyper h;
  h.kind = R::OptimizerKind::Adam;
  h.lr = 1e-3;
  h.weight_decay = 0.01;
  h.lr_table = {{1, 1e-3}, {30, 5e-4}};

  // reference blocks and the flat device layout (64-element aligned groups)
  std::vector<R::ParamBlock> ref;
  std::vector<R::Tensor> grads;
  std::vector<rw_group> groups(G);
  uint64_t total = 0;
  for (uint32_t i = 0; i < G; ++i) {
    R::ParamBlock b = R::ParamBlock::make({sizes[i]}, 100 + i);
    b.m = R::seeded_fill({sizes[i]}, 200 + i);
    b.v = R::seeded_fill({sizes[i]}, 300 + i);
    for (double& x : b.v.data) x = std::fabs(x) * 1e-3;
    b.t = 20;
    ref.push_back(b);
    grads.push_back(R::seeded_fill({sizes[i]}, 400 + i));
    groups[i] = rw_group{total, sizes[i], 20, 0, 0};
    total += (sizes[i] + 63) / 64 * 64;
  }
  auto upload = [&](std::vector<double>& flat, auto get) {
    flat.assign(total, 0.0);
    for (uint32_t i = 0; i < G; ++i) {
      const auto& d = get(i);
      std::copy(d.begin(), d.end(), flat.begin() + groups[i].offset);
    }
  };
  std::vector<double> hx, hm, hv, hg;
  upload(hx, [&](uint32_t i) -> const std::vector<double>& { return ref[i].x.data; });
  upload(hm, [&](uint32_t i) -> const std::vector<double>& { return ref[i].m.data; });
  upload(hv, [&](uint32_t i) -> const std::vector<double>& { return ref[i].v.data; });
  upload(hg, [&](uint32_t i) -> const std::vector<double>& { return grads[i].data; });
  double *dx, *dg, *dm, *dv, *dgrad;
  const size_t bytes = total * sizeof(double);
  for (double** p : {&dx, &dg, &dm, &dv, &dgrad}) cudaMalloc(p, bytes);
  cudaMemcpy(dx, hx.data(), bytes, cudaMemcpyHostToDevice);
  cudaMemcpy(dm, hm.data(), bytes, cudaMemcpyHostToDevice);
  cudaMemcpy(dv, hv.data(), bytes, cudaMemcpyHostToDevice);
  cudaMemcpy(dgrad, hg.data(), bytes, cudaMemcpyHostToDevice);
  cudaMemset(dg, 0, bytes);
  rw_state* s = nullptr;
  CK(rw_state_create(&s, RW_F64, dx, dg, dm, dv, nullptr, total, groups.data(), G, 0));

  std::vector<uint64_t> from = {1, 30};
  std::vector<double> value = {1e-3, 5e-4};
  rw_hyper hc{};
  hc.kind = RW_ADAM;
  hc.lr = h.lr;
  hc.weight_decay = h.weight_decay;
  hc.momentum = h.momentum;
  hc.dampening = h.dampening;
  hc.beta1 = h.beta1;
  hc.beta2 = h.beta2;
  hc.eps = h.eps;
  hc.lr_table_from = from.data();
  hc.lr_table_value = value.data();
  hc.lr_table_len = 2;

  // torn layer-wise update: reverse layer order, crash after k_crash blocks
  std::vector<uint32_t> order(G);
  for (uint32_t i = 0; i < G; ++i) order[i] = G - 1 - i;
  CK(rw_optimizer_step(s, &hc, order.data(), G, dgrad, k_crash, nullptr));
  for (uint32_t j = 0; j < k_crash; ++j) R::optimizer_step(ref[order[j]], grads[order[j]], h);

  auto compare = [&](const char* phase) {
    std::vector<double> cx(total), cm(total), cv(total);
    cudaMemcpy(cx.data(), dx, bytes, cudaMemcpyDeviceToHost);
    cudaMemcpy(cm.data(), dm, bytes, cudaMemcpyDeviceToHost);
    cudaMemcpy(cv.data(), dv, bytes, cudaMemcpyDeviceToHost);
    std::vector<rw_group> mk(G);
    rw_state_read_groups(s, mk.data(), nullptr);
    for (uint32_t i = 0; i < G; ++i) {
      const size_t o = groups[i].offset, n = sizes[i];
      const bool same = std::memcmp(cx.data() + o, ref[i].x.data.data(), n * 8) == 0 &&
                        std::memcmp(cm.data() + o, ref[i].m.data.data(), n * 8) == 0 &&
                        std::memcmp(cv.data() + o, ref[i].v.data.data(), n * 8) == 0;
      if (!same) std::printf("  %s: group %u differs\n", phase, i);
      EXPECT(same, phase);
      EXPECT(mk[i].t == ref[i].t && (mk[i].updated != 0) == ref[i].updated, "marker");
    }
  };
  compare("torn step");

  // resolve (one survivor: the global summary is the local one) and undo
  std::vector<rw_group> mk(G);
  CK(rw_state_read_groups(s, mk.data(), nullptr));
  rw_resolve_summary loc{}, glob{};
  CK(rw_resolve_summarize(mk.data(), G, nullptr, &hc, UINT64_MAX, &loc));
  CK(rw_resolve_summarize(mk.data(), G, nullptr, &hc, loc.t_min, &glob));
  glob.t_max = loc.t_max;
  std::vector<uint8_t> acts(G);
  uint64_t target = 0;
  int32_t strategy = -1;
  CK(rw_resolve_plan(&glob, RW_POLICY_UNDO, mk.data(), G, acts.data(), &target, &strategy));
  EXPECT(strategy == RW_STRATEGY_UNDO && target == 20, "plan: undo to 20");
  std::vector<uint32_t> undo;
  for (uint32_t i = 0; i < G; ++i)
    if (acts[i] == RW_ACT_UNDO) undo.push_back(i);
  EXPECT(undo.size() == k_crash, "undo set = the stepped blocks");
  CK(rw_optimizer_undo(s, &hc, undo.data(), static_cast<uint32_t>(undo.size()), nullptr));
  CK(rw_state_check(s, nullptr));
  for (uint32_t i : undo) R::optimizer_undo(ref[i], h);
  compare("resolved");

  rw_state_destroy(s);
  for (double* p : {dx, dg, dm, dv, dgrad}) cudaFree(p);
  std::printf("resolve_undo_test: %d failure(s)\n", g_fail);
  return g_fail ? 1 : 0;
}
