// Drop-in test (test infrastructure): the SAME reference objects
// (rewind::ParamBlock / Tensor / OptimizerHyper from the reference headers,
// renamed rewind_ref by the oracle shim) are driven through
//   (a) the reference library (oracle/_ref/librewind_ref.so), and
//   (b) rewind_b200::optimizer_step / optimizer_undo (include/rewind_b200.hpp
//       over librewind_b200.so),
// and must agree bit for bit, including the exceptions (rewind::Error with
// the same Err code, thrown by the drop-in through REWIND_B200_ERROR).
//
//   dropin_test --cpu   : guard paths only (no GPU needed; the device path
//                         must fail loudly with CudaError)
//   dropin_test         : full parity on a B200
#include <cstring>
#include <bits/stdc++.h>
#define rewind rewind_ref
#include "rewind/errors.hpp"
#include "rewind/optim.hpp"
#include "rewind/tensor.hpp"
#undef rewind

#define REWIND_B200_ERROR(code, msg) throw rewind_ref::Error(static_cast<rewind_ref::Err>(code), msg)
#include "rewind_b200.hpp"

namespace R = rewind_ref;
namespace B = rewind_b200;

static int g_fail = 0;
#define EXPECT(cond, what)                                       \
  do {                                                           \
    if (!(cond)) {                                               \
      std::printf("FAIL %s (%s:%d)\n", what, __FILE__, __LINE__); \
      ++g_fail;                                                  \
    }                                                            \
  } while (0)

template <class F>
std::string err_of(F&& f) {
  try {
    f();
  } catch (const R::Error& e) {
    return R::err_name(e.code());
  } catch (const B::Error& e) {
    return "B200:" + std::to_string(static_cast<int>(e.code()));
  } catch (const std::exception& e) {
    return std::string("other:") + e.what();
  }
  return "OK";
}

static bool same_bits(const R::Tensor& a, const R::Tensor& b) {
  return a.data.size() == b.data.size() &&
         std::memcmp(a.data.data(), b.data.data(), a.data.size() * sizeof(double)) == 0;
}

static R::OptimizerHyper hyper(R::OptimizerKind k) {
  R::OptimizerHyper h;
  h.kind = k;
  h.lr = k == R::OptimizerKind::Adam || k == R::OptimizerKind::AdamW ? 1e-3 : 0.05;
  h.weight_decay = 0.01;
  h.momentum = 0.9;
  h.dampening = 0.1;
  h.lr_table = {{1, h.lr}, {20, h.lr * 0.5}};
  return h;
}

int cpu_checks() {
  // invertibility_check mirrors optim.cpp:35-48
  for (int k = 0; k < 6; ++k)
    EXPECT(static_cast<int>(B::invertibility_check(static_cast<R::OptimizerKind>(k))) ==
               static_cast<int>(R::invertibility_check(static_cast<R::OptimizerKind>(k))),
           "invertibility");
  // guards that fire before any device work give the reference's Err
  R::ParamBlock a = R::ParamBlock::make({5}, 1), b = a;
  R::Tensor g = R::seeded_fill({5}, 2);
  R::OptimizerHyper h = hyper(R::OptimizerKind::Adam);
  EXPECT(err_of([&] { R::optimizer_undo(a, h); }) == err_of([&] { B::optimizer_undo(b, h); }),
         "NothingToUndo");
  a.updated = b.updated = true;
  EXPECT(err_of([&] { R::optimizer_step(a, g, h); }) == err_of([&] { B::optimizer_step(b, g, h); }),
         "AlreadyUpdated");
  a.updated = b.updated = false;
  R::OptimizerHyper ams = hyper(R::OptimizerKind::AmsGrad);
  ams.require_invertible = true;
  EXPECT(err_of([&] { R::optimizer_step(a, g, ams); }) == err_of([&] { B::optimizer_step(b, g, ams); }),
         "NotInvertible");
  R::Tensor bad = R::seeded_fill({6}, 2);
  EXPECT(err_of([&] { R::optimizer_step(a, bad, h); }) == err_of([&] { B::optimizer_step(b, bad, h); }),
         "ShapeMismatch");
  R::OptimizerHyper neg = h;
  neg.lr_table = {{1, -1.0}};
  EXPECT(err_of([&] { R::optimizer_step(a, g, neg); }) == err_of([&] { B::optimizer_step(b, g, neg); }),
         "InvalidConfig");
  EXPECT(same_bits(a.g, b.g), "grad cached before lr_at raises (optim.cpp:271-272)");
  // LAMB undo with an empty saved-scalar stack (optim.cpp:227-229)
  R::OptimizerHyper lamb = hyper(R::OptimizerKind::Lamb);
  a.updated = b.updated = true;
  a.t = b.t = 2;
  EXPECT(err_of([&] { R::optimizer_undo(a, lamb); }) == err_of([&] { B::optimizer_undo(b, lamb); }),
         "lamb NothingToUndo without a saved ratio");
  return 0;
}


int gpu_checks() {
  std::mt19937_64 rng(7);
  for (int k : {0, 1, 2, 3}) {
    const auto kind = static_cast<R::OptimizerKind>(k);
    for (int trial = 0; trial < 4; ++trial) {
      const std::size_t n = 1 + rng() % 9000;
      R::ParamBlock a = R::ParamBlock::make({n}, rng());
      a.m = R::seeded_fill({n}, rng());
      a.v = R::seeded_fill({n}, rng());
      for (double& x : a.v.data) x = std::fabs(x) * 1e-3;
      a.t = rng() % 40;
      R::ParamBlock b = a;
      R::Tensor g = R::seeded_fill({n}, rng());
      R::OptimizerHyper h = hyper(kind);
      R::optimizer_step(a, g, h);
      B::optimizer_step(b, g, h);
      EXPECT(same_bits(a.x, b.x) && same_bits(a.m, b.m) && same_bits(a.v, b.v) && same_bits(a.g, b.g),
             "step bit-exact");
      EXPECT(a.t == b.t && a.updated == b.updated, "step marker");
      R::optimizer_undo(a, h);
      B::optimizer_undo(b, h);
      EXPECT(same_bits(a.x, b.x) && same_bits(a.m, b.m) && same_bits(a.v, b.v), "undo bit-exact");
      EXPECT(a.t == b.t && a.updated == b.updated, "undo marker");
      EXPECT(err_of([&] { R::optimizer_undo(a, h); }) == err_of([&] { B::optimizer_undo(b, h); }),
             "double undo");
    }
  }
  // AMSGrad step (vmax), and its undo refusal
  {
    R::ParamBlock a = R::ParamBlock::make({777}, 3), b = a;
    R::Tensor g = R::seeded_fill({777}, 4);
    R::OptimizerHyper h = hyper(R::OptimizerKind::AmsGrad);
    R::optimizer_step(a, g, h);
    B::optimizer_step(b, g, h);
    EXPECT(same_bits(a.x, b.x) && same_bits(a.vmax, b.vmax), "amsgrad step");
    EXPECT(err_of([&] { R::optimizer_undo(a, h); }) == err_of([&] { B::optimizer_undo(b, h); }),
           "amsgrad undo");
  }
  // LAMB: the host-block path forms both norms in step_lamb's left-to-right
  // order, so m, v, g, the trust ratio pushed to saved_scalars and x are all
  // bit-exact
  for (int trial = 0; trial < 4; ++trial) {
    const std::size_t n = 1 + rng() % 20000;
    R::ParamBlock a = R::ParamBlock::make({n}, rng());
    a.m = R::seeded_fill({n}, rng());
    a.v = R::seeded_fill({n}, rng());
    for (double& x : a.v.data) x = std::fabs(x) * 1e-3;
    a.t = rng() % 40;
    R::ParamBlock b = a;
    R::Tensor g = R::seeded_fill({n}, rng());
    R::OptimizerHyper h = hyper(R::OptimizerKind::Lamb);
    R::optimizer_step(a, g, h);
    B::optimizer_step(b, g, h);
    EXPECT(same_bits(a.m, b.m) && same_bits(a.v, b.v) && same_bits(a.g, b.g), "lamb step m/v/g bit-exact");
    EXPECT(b.saved_scalars.size() == 1 && a.saved_scalars.size() == 1 &&
               std::memcmp(&a.saved_scalars[0], &b.saved_scalars[0], sizeof(double)) == 0,
           "lamb trust ratio bit-exact");
    EXPECT(same_bits(a.x, b.x), "lamb step x bit-exact");
    EXPECT(a.t == b.t && a.updated == b.updated, "lamb step marker");
    R::optimizer_undo(a, h);
    B::optimizer_undo(b, h);
    EXPECT(same_bits(a.m, b.m) && same_bits(a.v, b.v), "lamb undo m/v bit-exact");
    EXPECT(same_bits(a.x, b.x), "lamb undo x bit-exact");
    EXPECT(a.saved_scalars.empty() && b.saved_scalars.empty(), "lamb undo pops the ratio");
    EXPECT(a.t == b.t && a.updated == b.updated, "lamb undo marker");
  }
  // NumericalError after mutation
  {
    R::ParamBlock a = R::ParamBlock::make({16}, 5), b = a;
    R::Tensor g = R::seeded_fill({16}, 6);
    g.data[3] = std::numeric_limits<double>::infinity();
    R::OptimizerHyper h = hyper(R::OptimizerKind::Adam);
    std::string ea = err_of([&] { R::optimizer_step(a, g, h); });
    std::string eb = err_of([&] { B::optimizer_step(b, g, h); });
    EXPECT(ea == "NumericalError" && ea == eb, "NumericalError");
    EXPECT(a.t == b.t && a.updated == b.updated, "mutation happened before the raise");
  }
  return 0;
}

int main(int argc, char** argv) {
  const bool cpu_only = argc > 1 && std::string(argv[1]) == "--cpu";
  cpu_checks();
  if (cpu_only) {
    // the device path must refuse loudly when no GPU is visible
    if (rw_device_count() == 0) {
      R::ParamBlock b = R::ParamBlock::make({4}, 1);
      R::Tensor g = R::seeded_fill({4}, 2);
      std::string e = err_of([&] { B::optimizer_step(b, g, hyper(R::OptimizerKind::Adam)); });
      EXPECT(e == "B200:99", "no-GPU step must fail with CudaError");
    }
  } else {
    gpu_checks();
  }
  std::printf("%s: %d failure(s)\n", cpu_only ? "dropin_test --cpu" : "dropin_test", g_fail);
  return g_fail ? 1 : 0;
}
