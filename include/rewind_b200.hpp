// rewind_b200.hpp — header-only C++ drop-in for the reference optimizer API.
//
// Re-exposes the reference signatures (/root/reference/proj/core/include/rewind/optim.hpp)
//
//   void optimizer_step(ParamBlock&, const Tensor& grad, const OptimizerHyper&);  // optim.hpp:71-72
//   void optimizer_undo(ParamBlock&, const OptimizerHyper&);                      // optim.hpp:76
//   Invertibility invertibility_check(OptimizerKind);                             // optim.hpp:32
//
// on top of the C ABI in rewind_b200.h.  The functions are templates over the
// block / tensor / hyper types, so they accept the reference's OWN
// rewind::ParamBlock, rewind::Tensor and rewind::OptimizerHyper unchanged
// (anything with the same member names), and they throw the reference's own
// exception type when the integrator says which one it is:
//
//   #include "rewind/errors.hpp"          // the reference
//   #define REWIND_B200_ERROR(code, msg) throw rewind::Error(static_cast<rewind::Err>(code), msg)
//   #include "rewind_b200.hpp"
//   ...
//   rewind_b200::optimizer_undo(block, hyper);   // was rewind::optimizer_undo
//
// Without the macro, rewind_b200::Error (same Err numbering) is thrown.
// State stays fp64 as in the reference, so results are bit-identical to
// rewind::optimizer_step / optimizer_undo for every optimizer (the kernel
// evaluates the same IEEE operation sequence; for LAMB the host-block path
// forms the two norms in the reference's left-to-right order, so the trust
// ratio pushed to saved_scalars is the reference's too);
// tests/cpp/dropin_test.cpp checks it.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "rewind_b200.h"

namespace rewind_b200 {

// errors.hpp:11-33 (same order => same numeric codes)
enum class Err {
  InvalidShape, ShapeMismatch, EmptyInput, NumericalError, NonInvertibleHyper, NotInvertible,
  NothingToUndo, AlreadyUpdated, MissingActivation, ChannelBroken, InvalidInjection, NotFailed,
  StorageError, MissingLogData, CorruptLog, NoCheckpoint, NoReplica, InvalidConfig, TooLarge,
  // B200-side failures with no reference twin
  CudaError = 99, InvalidArgument = 100,
};

class Error : public std::runtime_error {
 public:
  Error(Err code, const std::string& msg) : std::runtime_error(msg), code_(code) {}
  Err code() const { return code_; }

 private:
  Err code_;
};

namespace detail {
[[noreturn]] inline void raise_status(int status) {
  const char* m = rw_last_error_message();
  std::string msg = m ? m : "";
  const int code = status - 1;  // status = 1 + (int)Err
#ifdef REWIND_B200_ERROR
  if (status >= 1 && status <= 19) {
    REWIND_B200_ERROR(code, msg);
  }
#endif
  throw Error(static_cast<Err>(code), msg);
}
inline void check(int status) {
  if (status != RW_OK) raise_status(status);
}

template <class Hyper>
struct HyperC {
  rw_hyper c{};
  std::vector<uint64_t> from;
  std::vector<double> value;
  explicit HyperC(const Hyper& h) {
    c.kind = static_cast<int32_t>(h.kind);
    c.require_invertible = h.require_invertible ? 1 : 0;
    c.lr = h.lr;
    c.weight_decay = h.weight_decay;
    c.momentum = h.momentum;
    c.dampening = h.dampening;
    c.beta1 = h.beta1;
    c.beta2 = h.beta2;
    c.eps = h.eps;
    for (const auto& [f, v] : h.lr_table) {
      from.push_back(static_cast<uint64_t>(f));
      value.push_back(v);
    }
    c.lr_table_from = from.data();
    c.lr_table_value = value.data();
    c.lr_table_len = static_cast<uint32_t>(from.size());
  }
};

template <class T>
double* ptr_or_null(T& t) {
  return t.data.empty() ? nullptr : t.data.data();
}
}  // namespace detail

// optim.hpp:16-23
enum class OptimizerKind : std::uint8_t { Sgd, SgdMomentum, Adam, AdamW, Lamb, AmsGrad };
// optim.hpp:28
enum class Invertibility { Invertible, InvertibleWithSavedScalars, NotInvertible };

template <class Kind>
Invertibility invertibility_check(Kind kind) {
  return static_cast<Invertibility>(rw_invertibility_check(static_cast<int32_t>(kind)));
}

// optimizer_step(ParamBlock&, const Tensor& grad, const OptimizerHyper&), optim.cpp:260-286.
// ShapeMismatch is checked first (:262), then the C ABI applies the same
// guards in the same order and runs the fused kernel on the block.
template <class Block, class Tensor, class Hyper>
void optimizer_step(Block& block, const Tensor& grad, const Hyper& hyper) {
  if (block.x.shape != grad.shape) {
#ifdef REWIND_B200_ERROR
    REWIND_B200_ERROR(RW_SHAPE_MISMATCH - 1, std::string("ShapeMismatch: gradient shape does not match block"));
#endif
    throw Error(Err::ShapeMismatch, "ShapeMismatch: gradient shape does not match block");
  }
  detail::HyperC<Hyper> h(hyper);
  const uint64_t n = block.x.data.size();
  // zero-initialised moments exist for every kind in the reference (ParamBlock::make)
  if (block.g.data.size() != n) block.g.data.assign(n, 0.0);
  if (block.m.data.size() != n) block.m.data.assign(n, 0.0);
  if (block.v.data.size() != n) block.v.data.assign(n, 0.0);
  if (h.c.kind == RW_AMSGRAD && block.vmax.data.size() != n) {  // optim.cpp:245
    block.vmax.shape = block.x.shape;
    block.vmax.data.assign(n, 0.0);
  }
  block.g.shape = block.x.shape;
  uint64_t t = block.t;
  uint32_t upd = block.updated ? 1u : 0u;
  if (h.c.kind == RW_LAMB) {  // step_lamb pushes its trust ratio (optim.cpp:216)
    double trust = 0.0;
    const int sl = rw_host_block_lamb_step(RW_F64, block.x.data.data(), block.g.data.data(), block.m.data.data(),
                                           block.v.data.data(), n, &t, &upd, grad.data.data(), &h.c, &trust);
    block.t = t;
    block.updated = upd != 0;
    if (sl == RW_OK || sl == RW_NUMERICAL_ERROR) block.saved_scalars.push_back(trust);  // before check_finite
    detail::check(sl);
    return;
  }
  const int st = rw_host_block_step(RW_F64, block.x.data.data(), block.g.data.data(),
                                    block.m.data.data(), block.v.data.data(),
                                    h.c.kind == RW_AMSGRAD ? block.vmax.data.data() : nullptr, n, &t,
                                    &upd, grad.data.data(), &h.c);
  block.t = t;
  block.updated = upd != 0;
  detail::check(st);
}

// optimizer_undo(ParamBlock&, const OptimizerHyper&), optim.cpp:288-307.
template <class Block, class Hyper>
void optimizer_undo(Block& block, const Hyper& hyper) {
  detail::HyperC<Hyper> h(hyper);
  const uint64_t n = block.x.data.size();
  uint64_t t = block.t;
  uint32_t upd = block.updated ? 1u : 0u;
  if (h.c.kind == RW_LAMB) {  // undo_lamb consumes the top ratio (optim.cpp:227-241)
    const bool have = !block.saved_scalars.empty();
    const int sl = rw_host_block_lamb_undo(RW_F64, block.x.data.data(), detail::ptr_or_null(block.g),
                                           detail::ptr_or_null(block.m), detail::ptr_or_null(block.v), n, &t, &upd,
                                           &h.c, have ? 1u : 0u, have ? block.saved_scalars.back() : 0.0);
    block.t = t;
    block.updated = upd != 0;
    if (sl == RW_OK || sl == RW_NUMERICAL_ERROR) block.saved_scalars.pop_back();
    detail::check(sl);
    return;
  }
  const int st = rw_host_block_undo(RW_F64, block.x.data.data(), detail::ptr_or_null(block.g),
                                    detail::ptr_or_null(block.m), detail::ptr_or_null(block.v), n,
                                    &t, &upd, &h.c);
  block.t = t;
  block.updated = upd != 0;
  detail::check(st);
}

}  // namespace rewind_b200
