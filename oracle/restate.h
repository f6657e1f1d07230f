/* ORACLE — test infrastructure, not product code.
 *
 * Plain-C restatement of the reference optimizer arithmetic
 * (/root/reference/proj/core/src/optim.cpp) in fp64 AND fp32.
 *
 *  - fp64 functions must equal the reference library (oracle/_ref) bit for bit;
 *    tests/test_oracle.py pins that on randomised blocks.
 *  - fp32 functions are the "reference operation order reproduced in fp32"
 *    oracle the CUDA fp32 kernels must match bit for bit (north_star: no FMA
 *    contraction).  Scalars are derived in double exactly as optim.cpp does and
 *    rounded to float ONCE (oracle_scalars()).
 *
 * Compiled with -ffp-contract=off so every C operator is one IEEE operation.
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg) load it.
 */
#ifndef REWIND_ORACLE_RESTATE_H
#define REWIND_ORACLE_RESTATE_H
#include <stddef.h>
#include <stdint.h>

/* OptimizerKind order of optim.hpp:16-23 */
enum { OR_SGD = 0, OR_SGDM = 1, OR_ADAM = 2, OR_ADAMW = 3, OR_LAMB = 4, OR_AMSGRAD = 5 };

typedef struct {
  int kind;
  double lr;
  double weight_decay, momentum, dampening, beta1, beta2, eps;
  int n_lr_table;
  const uint64_t* lr_from;
  const double* lr_value;
} or_hyper;

/* Every per-call scalar the loops use, derived in double as optim.cpp does. */
typedef struct {
  double eta;         /* lr_at(t+1) for step (optim.cpp:272), lr_at(t) for undo (:293) */
  double c1, c2;      /* bias_correction (optim.cpp:94-97) at t+1 (step) / t (undo) */
  double wd, mu, one_m_damp, b1, b2, one_m_b1, one_m_b2, eps;
  double denom;       /* 1 - eta*wd (undo_sgd :184, undo_adamw :255) */
} or_scalars;

/* returns 0 or 1+Err (InvalidConfig=17 -> 18) when lr_at would raise */
int oracle_scalars(const or_hyper* h, uint64_t t_before, int is_undo, or_scalars* out);
double oracle_lr_at(const or_hyper* h, uint64_t t);

/* Element loops.  Return 1 if any of x, m, v is non-finite afterwards
 * (check_finite at optim.cpp:283-285 / :304-306), else 0. */
int oracle_step_f64(int kind, const or_scalars* s, double* x, const double* g, double* m, double* v, size_t n);
int oracle_undo_f64(int kind, const or_scalars* s, double* x, const double* g, double* m, double* v, size_t n);
int oracle_step_f32(int kind, const or_scalars* s, float* x, const float* g, float* m, float* v, size_t n);
int oracle_undo_f32(int kind, const or_scalars* s, float* x, const float* g, float* m, float* v, size_t n);

/* AMSGrad step (optim.cpp:244-256) with its running max. */
int oracle_step_amsgrad_f64(const or_scalars* s, double* x, const double* g, double* m, double* v, double* vmax, size_t n);
int oracle_step_amsgrad_f32(const or_scalars* s, float* x, const float* g, float* m, float* v, float* vmax, size_t n);

/* LAMB (optim.cpp:195-242): step returns the trust ratio through *trust. */
int oracle_step_lamb_f64(const or_scalars* s, double* x, const double* g, double* m, double* v, size_t n, double* trust);
int oracle_undo_lamb_f64(const or_scalars* s, double trust, double* x, const double* g, double* m, double* v, size_t n);

/* ordered_sum (tensor.cpp:105-117): out = ((t0 + t1) + t2) + ... */
void oracle_ordered_sum_f32(const float* const* ts, int count, size_t n, float* out);
void oracle_ordered_sum_f64(const double* const* ts, int count, size_t n, double* out);

/* seeded_fill (tensor.cpp:94-103) and its helpers (tensor.cpp:69-92). */
uint64_t oracle_mix64(uint64_t x);
uint64_t oracle_derive_seed(uint64_t base, const uint64_t* parts, int n);
void oracle_seeded_fill_f64(uint64_t seed, size_t n, double* out);
void oracle_seeded_fill_f32(uint64_t seed, size_t n, float* out);

#endif
