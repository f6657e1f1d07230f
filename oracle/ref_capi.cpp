// ORACLE — test infrastructure, not product code.
//
// extern "C" wrappers around the UNMODIFIED reference library (built from
// /root/reference/proj/core/src/*.cpp through oracle/shim/*.cpp) so pytest can
// drive it with ctypes.  Nothing here computes: every function forwards to the
// reference symbol it names and converts `rewind::Error` into a status code
// 1 + (int)Err (errors.hpp:11-33), with the message kept in a thread-local
// buffer.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs may load the resulting oracle/_ref/librewind_ref.so.
#include <bits/stdc++.h>
#define rewind rewind_ref
#include "rewind/errors.hpp"
#include "rewind/model.hpp"
#include "rewind/optim.hpp"
#include "rewind/schedule.hpp"
#include "rewind/tensor.hpp"
#include "rewind/wire.hpp"
#undef rewind

namespace R = rewind_ref;

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    g_err.clear();
    return 0;
  } catch (const R::Error& e) {
    g_err = e.what();
    return 1 + static_cast<int>(e.code());
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1000;
  }
}

std::vector<std::size_t> shape_of(const std::size_t* shape, int ndim) {
  return std::vector<std::size_t>(shape, shape + ndim);
}
}  // namespace

extern "C" {

struct ref_hyper_c {
  int kind;
  double lr;
  double weight_decay;
  double momentum;
  double dampening;
  double beta1;
  double beta2;
  double eps;
  int require_invertible;
  int n_lr_table;
  const std::uint64_t* lr_from;
  const double* lr_value;
};

static R::OptimizerHyper to_hyper(const ref_hyper_c* h) {
  R::OptimizerHyper o;
  o.kind = static_cast<R::OptimizerKind>(h->kind);
  o.lr = h->lr;
  o.weight_decay = h->weight_decay;
  o.momentum = h->momentum;
  o.dampening = h->dampening;
  o.beta1 = h->beta1;
  o.beta2 = h->beta2;
  o.eps = h->eps;
  o.require_invertible = h->require_invertible != 0;
  for (int i = 0; i < h->n_lr_table; ++i) o.lr_table.emplace_back(h->lr_from[i], h->lr_value[i]);
  return o;
}

const char* ref_last_error(void) { return g_err.c_str(); }
const char* ref_err_name(int code) { return R::err_name(static_cast<R::Err>(code)); }

// ---------------- optimizers (optim.hpp / optim.cpp) ----------------
void* ref_block_make(const std::size_t* shape, int ndim, std::uint64_t seed) {
  auto* b = new R::ParamBlock();
  int st = guarded([&] { *b = R::ParamBlock::make(shape_of(shape, ndim), seed); });
  if (st) {
    delete b;
    return nullptr;
  }
  return b;
}
void ref_block_free(void* b) { delete static_cast<R::ParamBlock*>(b); }
std::size_t ref_block_size(void* b) { return static_cast<R::ParamBlock*>(b)->x.size(); }

// Overwrite any of x/g/m/v (NULL = keep) plus t and the updated flag.
void ref_block_set(void* vb, const double* x, const double* g, const double* m,
                   const double* v, std::uint64_t t, int updated) {
  auto* b = static_cast<R::ParamBlock*>(vb);
  std::size_t n = b->x.size();
  if (x) std::copy(x, x + n, b->x.data.begin());
  if (g) std::copy(g, g + n, b->g.data.begin());
  if (m) std::copy(m, m + n, b->m.data.begin());
  if (v) std::copy(v, v + n, b->v.data.begin());
  b->t = t;
  b->updated = updated != 0;
}
void ref_block_get(void* vb, double* x, double* g, double* m, double* v,
                   std::uint64_t* t, int* updated) {
  auto* b = static_cast<R::ParamBlock*>(vb);
  if (x) std::copy(b->x.data.begin(), b->x.data.end(), x);
  if (g) std::copy(b->g.data.begin(), b->g.data.end(), g);
  if (m) std::copy(b->m.data.begin(), b->m.data.end(), m);
  if (v) std::copy(b->v.data.begin(), b->v.data.end(), v);
  if (t) *t = b->t;
  if (updated) *updated = b->updated ? 1 : 0;
}
int ref_block_saved_scalars(void* vb, double* out, int cap) {
  auto* b = static_cast<R::ParamBlock*>(vb);
  int n = static_cast<int>(b->saved_scalars.size());
  for (int i = 0; i < n && i < cap; ++i) out[i] = b->saved_scalars[static_cast<std::size_t>(i)];
  return n;
}
void ref_block_push_scalar(void* vb, double s) { static_cast<R::ParamBlock*>(vb)->saved_scalars.push_back(s); }

int ref_optimizer_step(void* vb, const double* grad, const std::size_t* shape, int ndim,
                       const ref_hyper_c* h) {
  auto* b = static_cast<R::ParamBlock*>(vb);
  return guarded([&] {
    auto shp = shape_of(shape, ndim);
    R::Tensor g(shp, std::vector<double>(grad, grad + R::shape_elements(shp)));
    R::optimizer_step(*b, g, to_hyper(h));
  });
}
int ref_optimizer_undo(void* vb, const ref_hyper_c* h) {
  auto* b = static_cast<R::ParamBlock*>(vb);
  return guarded([&] { R::optimizer_undo(*b, to_hyper(h)); });
}
int ref_invertibility_check(int kind) {
  return static_cast<int>(R::invertibility_check(static_cast<R::OptimizerKind>(kind)));
}
int ref_lr_at(const ref_hyper_c* h, std::uint64_t t, double* out) {
  return guarded([&] { *out = to_hyper(h).lr_at(t); });
}
int ref_validate(const ref_hyper_c* h) {
  return guarded([&] { to_hyper(h).validate(); });
}
int ref_optimizer_from_name(const char* name) {
  auto k = R::optimizer_from_name(name);
  return k ? static_cast<int>(*k) : -1;
}

// ---------------- numerics (tensor.hpp / tensor.cpp) ----------------
std::uint64_t ref_mix64(std::uint64_t x) { return R::mix64(x); }
std::uint64_t ref_derive_seed(std::uint64_t base, const std::uint64_t* parts, int n) {
  // derive_seed takes an initializer_list; replay its definition shape by
  // calling it with the exact arity used in the reference (1..4 parts).
  switch (n) {
    case 0: return R::derive_seed(base, {});
    case 1: return R::derive_seed(base, {parts[0]});
    case 2: return R::derive_seed(base, {parts[0], parts[1]});
    case 3: return R::derive_seed(base, {parts[0], parts[1], parts[2]});
    case 4: return R::derive_seed(base, {parts[0], parts[1], parts[2], parts[3]});
    default: return 0;
  }
}
std::uint64_t ref_rng_value_at(std::uint64_t seed, std::uint64_t i) { return R::Rng::value_at(seed, i); }
double ref_rng_unit_at(std::uint64_t seed, std::uint64_t i) { return R::Rng::unit_at(seed, i); }
int ref_seeded_fill(const std::size_t* shape, int ndim, std::uint64_t seed, double* out) {
  return guarded([&] {
    R::Tensor t = R::seeded_fill(shape_of(shape, ndim), seed);
    std::copy(t.data.begin(), t.data.end(), out);
  });
}
// tensors: count pointers, each n doubles, all shape [n] unless shapes differ
// (lens[i] gives each length so ShapeMismatch is reachable).
int ref_ordered_sum(const double* const* tensors, const std::size_t* lens, int count, double* out) {
  return guarded([&] {
    std::vector<R::Tensor> ts;
    for (int i = 0; i < count; ++i) {
      ts.emplace_back(std::vector<std::size_t>{lens[i]},
                      std::vector<double>(tensors[i], tensors[i] + lens[i]));
    }
    R::Tensor s = R::ordered_sum(ts);
    std::copy(s.data.begin(), s.data.end(), out);
  });
}
int ref_l2_norm(const double* x, std::size_t n, double* out) {
  return guarded([&] {
    R::Tensor t;
    t.shape = {n};
    t.data.assign(x, x + n);
    *out = R::l2_norm(t);
  });
}
int ref_check_finite(const double* x, std::size_t n) {
  return guarded([&] {
    R::Tensor t;
    t.shape = {n};
    t.data.assign(x, x + n);
    R::check_finite(t, "oracle");
  });
}

// ---------------- wire ----------------
std::uint32_t ref_crc32(const unsigned char* p, std::size_t n) {
  return R::crc32(std::span<const std::byte>(reinterpret_cast<const std::byte*>(p), n));
}
std::uint64_t ref_fnv1a64(const unsigned char* p, std::size_t n) {
  return R::fnv1a64(std::span<const std::byte>(reinterpret_cast<const std::byte*>(p), n));
}

// ---------------- schedule ----------------
int ref_bubble_ratio(int p, int m, long long* num, long long* den) {
  return guarded([&] {
    R::Ratio r = R::bubble_ratio(p, m);
    *num = r.num;
    *den = r.den;
  });
}
// kinds/mbs: p * cap entries, row-major; returns slots per row via *slots.
int ref_build_1f1b_schedule(int p, int m, int* kinds, int* mbs, int cap, int* slots) {
  return guarded([&] {
    R::Schedule s = R::build_1f1b_schedule(p, m);
    R::validate_schedule(s);
    int len = static_cast<int>(s.slots_per_iteration());
    *slots = len;
    if (len > cap) return;
    for (int st = 0; st < p; ++st) {
      for (int i = 0; i < len; ++i) {
        const auto& a = s.rows[static_cast<std::size_t>(st)][static_cast<std::size_t>(i)];
        kinds[st * cap + i] = static_cast<int>(a.kind);
        mbs[st * cap + i] = static_cast<int>(a.mb);
      }
    }
  });
}
int ref_schedule_grid(int p, int m, char* buf, std::size_t cap) {
  return guarded([&] {
    std::string g = R::schedule_grid(R::build_1f1b_schedule(p, m));
    std::snprintf(buf, cap, "%s", g.c_str());
  });
}
long long ref_count_bubbles(int p, int m) {
  return static_cast<long long>(R::count_bubbles(R::build_1f1b_schedule(p, m)));
}

// ---------------- model ----------------
void* ref_stage_make(int stage_id, std::size_t in, std::size_t hidden, std::size_t out,
                     int layers, std::uint64_t seed) {
  auto* s = new R::Stage();
  int st = guarded([&] { *s = R::make_stage(stage_id, in, hidden, out, layers, seed); });
  if (st) {
    delete s;
    return nullptr;
  }
  return s;
}
void ref_stage_free(void* s) { delete static_cast<R::Stage*>(s); }
int ref_stage_nblocks(void* s) { return static_cast<int>(static_cast<R::Stage*>(s)->blocks().size()); }
void* ref_stage_block(void* s, int i) { return static_cast<R::Stage*>(s)->blocks()[static_cast<std::size_t>(i)]; }
int ref_forward_stage(void* vs, const double* act, std::size_t rows, std::size_t cols,
                      std::uint32_t mb, double* out) {
  auto* s = static_cast<R::Stage*>(vs);
  return guarded([&] {
    R::Tensor a({rows, cols}, std::vector<double>(act, act + rows * cols));
    R::Tensor y = R::forward_stage(*s, a, mb);
    std::copy(y.data.begin(), y.data.end(), out);
  });
}
// param_grads: array of nblocks output pointers, sized like the blocks.
int ref_backward_stage(void* vs, const double* grad_in, std::size_t rows, std::size_t cols,
                       std::uint32_t mb, double* grad_out, double** param_grads) {
  auto* s = static_cast<R::Stage*>(vs);
  return guarded([&] {
    R::Tensor g({rows, cols}, std::vector<double>(grad_in, grad_in + rows * cols));
    R::StageBackward b = R::backward_stage(*s, g, mb);
    std::copy(b.grad_out.data.begin(), b.grad_out.data.end(), grad_out);
    for (std::size_t i = 0; i < b.param_grads.size(); ++i) {
      std::copy(b.param_grads[i].data.begin(), b.param_grads[i].data.end(), param_grads[i]);
    }
  });
}
int ref_mse_loss(const double* pred, const double* tgt, std::size_t rows, std::size_t cols,
                 std::size_t micro_batches, double* loss, double* grad) {
  return guarded([&] {
    R::Tensor p({rows, cols}, std::vector<double>(pred, pred + rows * cols));
    R::Tensor t({rows, cols}, std::vector<double>(tgt, tgt + rows * cols));
    R::LossGrad lg = R::mse_loss(p, t, micro_batches);
    *loss = lg.loss;
    std::copy(lg.grad.data.begin(), lg.grad.data.end(), grad);
  });
}
int ref_synth_inputs(std::uint64_t seed, std::uint64_t it, std::uint64_t stream,
                     std::size_t rows, std::size_t dim, double* out) {
  return guarded([&] {
    R::Tensor t = R::synth_inputs(seed, it, stream, rows, dim);
    std::copy(t.data.begin(), t.data.end(), out);
  });
}
int ref_synth_targets(std::uint64_t seed, std::uint64_t it, std::uint64_t stream,
                      std::size_t rows, std::size_t dim, double* out) {
  return guarded([&] {
    R::Tensor t = R::synth_targets(seed, it, stream, rows, dim);
    std::copy(t.data.begin(), t.data.end(), out);
  });
}

}  // extern "C"
