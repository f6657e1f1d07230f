/* ORACLE — test infrastructure, not product code.  See restate.h.
 * Every loop cites the optim.cpp / tensor.cpp lines it restates; the C
 * expressions keep the reference's association order operator by operator
 * (C and C++ share left-to-right evaluation of * and + chains). */
#include "restate.h"

#include <math.h>
#include <string.h>

/* optim.cpp:50-57 (last breakpoint with t >= from wins). */
double oracle_lr_at(const or_hyper* h, uint64_t t) {
  double out = h->lr;
  for (int i = 0; i < h->n_lr_table; ++i)
    if (t >= h->lr_from[i]) out = h->lr_value[i];
  return out;
}

int oracle_scalars(const or_hyper* h, uint64_t t_before, int is_undo, or_scalars* s) {
  memset(s, 0, sizeof(*s));
  /* step uses lr_at(t+1) and bias_correction(t+1) (optim.cpp:272, :132);
   * undo uses lr_at(t) and bias_correction(t) (optim.cpp:293, :147). */
  uint64_t tt = is_undo ? t_before : t_before + 1;
  s->eta = oracle_lr_at(h, tt);
  if (!(s->eta > 0.0)) return 1 + 17; /* Err::InvalidConfig */
  s->c1 = 1.0 - pow(h->beta1, (double)tt);
  s->c2 = 1.0 - pow(h->beta2, (double)tt);
  s->wd = h->weight_decay;
  s->mu = h->momentum;
  s->one_m_damp = 1.0 - h->dampening;
  s->b1 = h->beta1;
  s->b2 = h->beta2;
  s->one_m_b1 = 1.0 - h->beta1;
  s->one_m_b2 = 1.0 - h->beta2;
  s->eps = h->eps;
  s->denom = 1.0 - s->eta * h->weight_decay;
  return 0;
}

#define FIN_ACC(T, fin, x, m, v) \
  fin |= !(isfinite(x) && isfinite(m) && isfinite(v))

/* One template, instantiated for double and float.  For float every scalar is
 * rounded once from its double value. */
#define DEFINE_LOOPS(T, SUF, SQRT)                                                        \
  int oracle_step_##SUF(int kind, const or_scalars* S, T* x, const T* g, T* m, T* v,      \
                        size_t n) {                                                        \
    const T eta = (T)S->eta, c1 = (T)S->c1, c2 = (T)S->c2, wd = (T)S->wd, mu = (T)S->mu;  \
    const T omd = (T)S->one_m_damp, b1 = (T)S->b1, b2 = (T)S->b2;                         \
    const T omb1 = (T)S->one_m_b1, omb2 = (T)S->one_m_b2, eps = (T)S->eps;                \
    int fin = 0;                                                                           \
    for (size_t i = 0; i < n; ++i) {                                                       \
      switch (kind) {                                                                      \
        case OR_SGD: /* optim.cpp:99-103 */                                               \
          x[i] = x[i] - eta * (g[i] + wd * x[i]);                                          \
          break;                                                                           \
        case OR_SGDM: { /* optim.cpp:113-119 */                                            \
          T gd = g[i] + wd * x[i];                                                         \
          m[i] = mu * m[i] + omd * gd;                                                     \
          x[i] = x[i] - eta * m[i];                                                        \
          break;                                                                           \
        }                                                                                  \
        case OR_ADAM: { /* optim.cpp:131-141 */                                            \
          T gd = g[i] + wd * x[i];                                                         \
          m[i] = b1 * m[i] + omb1 * gd;                                                    \
          v[i] = b2 * v[i] + omb2 * gd * gd;                                               \
          T mhat = m[i] / c1;                                                              \
          T vhat = v[i] / c2;                                                              \
          x[i] = x[i] - eta * mhat / (SQRT(vhat) + eps);                                   \
          break;                                                                           \
        }                                                                                  \
        case OR_ADAMW: { /* optim.cpp:160-171 */                                           \
          T gd = g[i];                                                                     \
          m[i] = b1 * m[i] + omb1 * gd;                                                    \
          v[i] = b2 * v[i] + omb2 * gd * gd;                                               \
          T mhat = m[i] / c1;                                                              \
          T vhat = v[i] / c2;                                                              \
          x[i] = x[i] - eta * (mhat / (SQRT(vhat) + eps) + wd * x[i]);                     \
          break;                                                                           \
        }                                                                                  \
        default:                                                                           \
          return -1;                                                                       \
      }                                                                                    \
      FIN_ACC(T, fin, x[i], m[i], v[i]);                                                   \
    }                                                                                      \
    return fin;                                                                            \
  }                                                                                        \
  int oracle_undo_##SUF(int kind, const or_scalars* S, T* x, const T* g, T* m, T* v,      \
                        size_t n) {                                                        \
    const T eta = (T)S->eta, c1 = (T)S->c1, c2 = (T)S->c2, wd = (T)S->wd, mu = (T)S->mu;  \
    const T omd = (T)S->one_m_damp, b1 = (T)S->b1, b2 = (T)S->b2;                         \
    const T omb1 = (T)S->one_m_b1, omb2 = (T)S->one_m_b2, eps = (T)S->eps;                \
    const T denom = (T)S->denom;                                                           \
    int fin = 0;                                                                           \
    for (size_t i = 0; i < n; ++i) {                                                       \
      switch (kind) {                                                                      \
        case OR_SGD: /* optim.cpp:105-111 */                                               \
          x[i] = (x[i] + eta * g[i]) / denom;                                              \
          break;                                                                           \
        case OR_SGDM: { /* optim.cpp:121-129 */                                            \
          T xt = x[i] + eta * m[i];                                                        \
          T gd = g[i] + wd * xt;                                                           \
          m[i] = (m[i] - omd * gd) / mu;                                                   \
          x[i] = xt;                                                                       \
          break;                                                                           \
        }                                                                                  \
        case OR_ADAM: { /* optim.cpp:143-157 */                                            \
          T mhat = m[i] / c1;                                                              \
          T vhat = v[i] / c2;                                                              \
          T xt = x[i] + eta * mhat / (SQRT(vhat) + eps);                                   \
          T gd = g[i] + wd * xt;                                                           \
          m[i] = (m[i] - omb1 * gd) / b1;                                                  \
          v[i] = (v[i] - omb2 * gd * gd) / b2;                                             \
          x[i] = xt;                                                                       \
          break;                                                                           \
        }                                                                                  \
        case OR_ADAMW: { /* optim.cpp:173-189 */                                           \
          T mhat = m[i] / c1;                                                              \
          T vhat = v[i] / c2;                                                              \
          T xt = (x[i] + eta * mhat / (SQRT(vhat) + eps)) / denom;                         \
          T gd = g[i];                                                                     \
          m[i] = (m[i] - omb1 * gd) / b1;                                                  \
          v[i] = (v[i] - omb2 * gd * gd) / b2;                                             \
          x[i] = xt;                                                                       \
          break;                                                                           \
        }                                                                                  \
        default:                                                                           \
          return -1;                                                                       \
      }                                                                                    \
      FIN_ACC(T, fin, x[i], m[i], v[i]);                                                   \
    }                                                                                      \
    return fin;                                                                            \
  }                                                                                        \
  int oracle_step_amsgrad_##SUF(const or_scalars* S, T* x, const T* g, T* m, T* v,        \
                                T* vmax, size_t n) {                                       \
    const T eta = (T)S->eta, c1 = (T)S->c1, c2 = (T)S->c2, wd = (T)S->wd;                 \
    const T b1 = (T)S->b1, b2 = (T)S->b2, omb1 = (T)S->one_m_b1;                          \
    const T omb2 = (T)S->one_m_b2, eps = (T)S->eps;                                       \
    int fin = 0;                                                                           \
    for (size_t i = 0; i < n; ++i) { /* optim.cpp:244-256 */                               \
      T gd = g[i] + wd * x[i];                                                             \
      m[i] = b1 * m[i] + omb1 * gd;                                                        \
      v[i] = b2 * v[i] + omb2 * gd * gd;                                                   \
      vmax[i] = vmax[i] < v[i] ? v[i] : vmax[i]; /* std::max(vmax, v) */                   \
      T mhat = m[i] / c1;                                                                  \
      T vhat = vmax[i] / c2;                                                               \
      x[i] = x[i] - eta * mhat / (SQRT(vhat) + eps);                                       \
      FIN_ACC(T, fin, x[i], m[i], v[i]);                                                   \
    }                                                                                      \
    return fin;                                                                            \
  }                                                                                        \
  void oracle_ordered_sum_##SUF(const T* const* ts, int count, size_t n, T* out) {        \
    /* tensor.cpp:105-117: acc = t0; acc += tk for k = 1.. in order */                     \
    for (size_t i = 0; i < n; ++i) out[i] = ts[0][i];                                      \
    for (int k = 1; k < count; ++k)                                                        \
      for (size_t i = 0; i < n; ++i) out[i] = out[i] + ts[k][i];                           \
  }

DEFINE_LOOPS(double, f64, sqrt)
DEFINE_LOOPS(float, f32, sqrtf)

/* LAMB step, optim.cpp:195-217 (fp64 only: the trust-ratio norms are
 * sequential left-to-right sums). */
int oracle_step_lamb_f64(const or_scalars* S, double* x, const double* g, double* m, double* v,
                         size_t n, double* trust_out) {
  double xnorm_sq = 0.0, unorm_sq = 0.0;
  /* Pass 2 recomputes update[i] from the same (already-updated) m, v and the
   * not-yet-updated x[i], so it equals the reference's stored update[i]. */
  for (size_t i = 0; i < n; ++i) {
    double gd = g[i];
    m[i] = S->b1 * m[i] + S->one_m_b1 * gd;
    v[i] = S->b2 * v[i] + S->one_m_b2 * gd * gd;
    double mhat = m[i] / S->c1;
    double vhat = v[i] / S->c2;
    double u = mhat / (sqrt(vhat) + S->eps) + S->wd * x[i];
    xnorm_sq += x[i] * x[i];
    unorm_sq += u * u;
  }
  double xnorm = sqrt(xnorm_sq), unorm = sqrt(unorm_sq);
  double trust = (xnorm > 0.0 && unorm > 0.0) ? xnorm / unorm : 1.0;
  int fin = 0;
  for (size_t i = 0; i < n; ++i) {
    double mhat = m[i] / S->c1;
    double vhat = v[i] / S->c2;
    double u = mhat / (sqrt(vhat) + S->eps) + S->wd * x[i];
    x[i] = x[i] - S->eta * trust * u;
    FIN_ACC(double, fin, x[i], m[i], v[i]);
  }
  *trust_out = trust;
  return fin;
}

/* LAMB undo, optim.cpp:219-242. */
int oracle_undo_lamb_f64(const or_scalars* S, double trust, double* x, const double* g, double* m,
                         double* v, size_t n) {
  double scaled = S->eta * trust;
  double denom = 1.0 - scaled * S->wd;
  int fin = 0;
  for (size_t i = 0; i < n; ++i) {
    double mhat = m[i] / S->c1;
    double vhat = v[i] / S->c2;
    double r = mhat / (sqrt(vhat) + S->eps);
    double xt = (x[i] + scaled * r) / denom;
    double gd = g[i];
    m[i] = (m[i] - S->one_m_b1 * gd) / S->b1;
    v[i] = (v[i] - S->one_m_b2 * gd * gd) / S->b2;
    x[i] = xt;
    FIN_ACC(double, fin, x[i], m[i], v[i]);
  }
  return fin;
}

/* tensor.cpp:69-74 */
uint64_t oracle_mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
/* tensor.cpp:76-83 */
uint64_t oracle_derive_seed(uint64_t base, const uint64_t* parts, int n) {
  uint64_t h = oracle_mix64(base);
  for (int i = 0; i < n; ++i) h = oracle_mix64(h ^ oracle_mix64(parts[i]));
  return h;
}
/* tensor.cpp:85-103 */
static double unit_at(uint64_t seed, uint64_t i) {
  uint64_t v = oracle_mix64(oracle_mix64(seed) ^ (i * 0x9E3779B97F4A7C15ull + 1));
  return (double)(v >> 11) * 0x1.0p-53;
}
void oracle_seeded_fill_f64(uint64_t seed, size_t n, double* out) {
  for (size_t i = 0; i < n; ++i) out[i] = (unit_at(seed, i) * 2.0 - 1.0) * 0.1;
}
void oracle_seeded_fill_f32(uint64_t seed, size_t n, float* out) {
  for (size_t i = 0; i < n; ++i) out[i] = (float)((unit_at(seed, i) * 2.0 - 1.0) * 0.1);
}
