// Host-only pieces of the recovery path that have no reference source file
// (recovery.cpp and planner.cpp are absent, P/core/CMakeLists.txt:11-17), so
// they are built from their SPEC contracts:
//   * consistency resolver — consensus_iteration + apply_undo
//     (SPEC:484-492), extended with the north_star's per-group "redo";
//   * selective-logging policy — group_machines,
//     recovery_time_estimate, logging_worthwhile;
//   * bubble_ratio (schedule.cpp:86-93), which the policy consumes.
// Pure C++: O(groups) and O(N^2) with N <= a few hundred, so not kernels.
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <numeric>
#include <string>
#include <vector>

#include "internal.h"

namespace {
int fail2(int code, const char* msg) {
  rwb::set_error(msg);
  return code;
}
}  // namespace

extern "C" {

// ---------------- resolver ----------------
//
// Markers: group t = completed steps, updated = stepped in the in-flight
// iteration.  A rank's groups can only be at t_lo or t_lo+1 after a crash in
// synchronous training (one gradient version is cached).  The
// consensus target is t_lo = min over survivors when
// rolling back, or t_lo+1 when every group still at t_lo holds its
// synchronised gradient (north_star "undo or redo").
//
// Spec gap: SPEC:487 undoes blocks whose flag is set OR
// whose t is beyond the target, but optimizer_undo refuses !updated blocks
// (optim.cpp:289).  We decide on t alone and re-arm the flag before undoing
// (rw_apply in the Python/C++ drivers), allowing at most one step of undo.
int rw_resolve_summarize(const rw_group* groups, uint32_t n, const uint8_t* grad_ready,
                         const rw_hyper* h, uint64_t t_floor, rw_resolve_summary* out) {
  if (!out || (n && !groups) || !h) return fail2(RW_INVALID_ARGUMENT, "null argument");
  rw_resolve_summary s{};
  s.t_min = UINT64_MAX;
  s.t_max = 0;
  for (uint32_t i = 0; i < n; ++i) {
    if (groups[i].t < s.t_min) s.t_min = groups[i].t;
    if (groups[i].t > s.t_max) s.t_max = groups[i].t;
  }
  // n == 0 (a replacement with no state yet): t_min stays UINT64_MAX and
  // t_max 0, the identities of the MIN / MAX all-reduces, so a joining rank
  // never drags the consensus down.
  // phase 1: t_floor == UINT64_MAX -> relative to the local minimum;
  // phase 2: relative to the all-reduced (global MIN) t_floor.
  const uint64_t lo = t_floor == UINT64_MAX ? s.t_min : t_floor;
  for (uint32_t i = 0; i < n; ++i) {
    if (groups[i].t == lo + 1) s.undo_elems += groups[i].len;
    if (groups[i].t == lo) {
      s.redo_elems += groups[i].len;
      if (!grad_ready || !grad_ready[i]) s.redo_blocked += 1;
    }
  }
  // undo_<kind> hyper guards (optim.cpp:106, :122, :144, :174-178) and the
  // AMSGrad refusal (:290-292).  LAMB undoes with its saved trust ratio
  // (:297-320); a group whose ratio is missing fails at apply time.
  bool blocked = rw_invertibility_check(h->kind) == RW_NOT_INVERTIBLE_KIND;
  if (h->kind == RW_SGDM && h->momentum == 0.0) blocked = true;
  if ((h->kind == RW_ADAM || h->kind == RW_ADAMW || h->kind == RW_LAMB) && (h->beta1 == 0.0 || h->beta2 == 0.0))
    blocked = true;
  s.undo_blocked = blocked ? 1 : 0;
  s.t_min = lo;
  *out = s;
  return RW_OK;
}

int rw_resolve_plan(const rw_resolve_summary* gs, int32_t policy, const rw_group* groups, uint32_t n,
                    uint8_t* actions, uint64_t* target, int32_t* strategy) {
  if (!gs || !target || !strategy || (n && (!groups || !actions)))
    return fail2(RW_INVALID_ARGUMENT, "null argument");
  const uint64_t lo = gs->t_min;
  for (uint32_t i = 0; i < n; ++i) actions[i] = RW_ACT_NONE;
  if (gs->t_max == lo) {  // already consistent
    *target = lo;
    *strategy = RW_STRATEGY_NONE;
    return RW_OK;
  }
  if (gs->t_max > lo + 1) {  // more than one step apart: only one g version cached
    *target = lo;
    *strategy = RW_STRATEGY_GLOBAL_ROLLBACK;
    return RW_OK;
  }
  const bool can_undo = gs->undo_blocked == 0;
  const bool can_redo = gs->redo_blocked == 0;
  int32_t st;
  if (policy == RW_POLICY_MIN_COST && can_undo && can_redo)
    st = gs->redo_elems < gs->undo_elems ? RW_STRATEGY_REDO : RW_STRATEGY_UNDO;
  else if (can_undo)
    st = RW_STRATEGY_UNDO;
  else if (can_redo)
    st = RW_STRATEGY_REDO;
  else
    st = RW_STRATEGY_GLOBAL_ROLLBACK;
  *strategy = st;
  *target = st == RW_STRATEGY_REDO ? lo + 1 : lo;
  for (uint32_t i = 0; i < n; ++i) {
    if (st == RW_STRATEGY_UNDO && groups[i].t == lo + 1) actions[i] = RW_ACT_UNDO;
    if (st == RW_STRATEGY_REDO && groups[i].t == lo) actions[i] = RW_ACT_REDO;
  }
  return RW_OK;
}

// ---------------- schedule ----------------
// bubble_ratio, schedule.cpp:86-93: exact reduced (p-1)/(m+p-1)
int rw_bubble_ratio(int32_t p, int32_t m, int64_t* num, int64_t* den) {
  if (p < 1 || m < 1) return fail2(RW_INVALID_CONFIG, "InvalidConfig: p and m must be >= 1");
  int64_t a = p - 1, b = static_cast<int64_t>(m) + p - 1;
  int64_t g = std::gcd(a, b);
  if (g == 0) {
    *num = 0;
    *den = 1;
    return RW_OK;
  }
  *num = a / g;
  *den = b / g;
  return RW_OK;
}

// ---------------- selective-logging planner ----------------
namespace {
struct Plan {
  std::vector<uint32_t> start;  // first machine of each group
  std::vector<uint32_t> size;
  std::vector<double> R;        // R(G_i), seconds per iteration
};

double group_weighted(const Plan& p, uint32_t i, uint32_t N, bool parallel) {
  // (|G|/N) * R(G), with R divided by floor(N/|G|) under parallel recovery
  double r = p.R[i];
  if (parallel) r /= std::floor(static_cast<double>(N) / p.size[i]);
  return (static_cast<double>(p.size[i]) / N) * r;
}
}  // namespace

int rw_group_machines(uint32_t N, const double* R, const double* M, double B, double T, double M_max,
                      int32_t parallel, uint32_t* group_of, uint32_t* n_groups, double* storage,
                      double* recovery) {
  if (N == 0 || !R || (N > 1 && !M) || !group_of || !n_groups)
    return fail2(RW_INVALID_CONFIG, "InvalidConfig: empty profile");
  if (!(B > 0.0) || !(T >= 1.0)) return fail2(RW_INVALID_CONFIG, "InvalidConfig: B > 0 and T >= 1 required");
  for (uint32_t i = 0; i < N; ++i)
    if (!(R[i] > 0.0)) return fail2(RW_INVALID_CONFIG, "InvalidConfig: R must be > 0");
  for (uint32_t i = 0; i + 1 < N; ++i)
    if (M[i] < 0.0) return fail2(RW_INVALID_CONFIG, "InvalidConfig: M must be >= 0");
  Plan p;
  for (uint32_t i = 0; i < N; ++i) {
    p.start.push_back(i);
    p.size.push_back(1);
    p.R.push_back(R[i]);
  }
  // boundary between group i and i+1 is machine boundary start[i+1]-1
  auto bM = [&](uint32_t i) { return M[p.start[i + 1] - 1]; };
  auto stor = [&]() {
    double s = 0.0;
    for (uint32_t i = 0; i + 1 < p.start.size(); ++i) s += bM(i);
    return T * s;
  };
  const bool par = parallel != 0;
  while (stor() > M_max && p.start.size() > 1) {
    // greedy: adjacent pair with the smallest dR/dM; ties -> lowest left index
    // (SPEC:570, :611); zero-M boundaries only if no positive-M merge exists.
    int best = -1;
    double best_ratio = 0.0;
    bool best_pos = false;
    for (uint32_t i = 0; i + 1 < p.start.size(); ++i) {
      const double m = bM(i);
      Plan q;
      q.size = {p.size[i] + p.size[i + 1]};
      q.R = {p.R[i] + p.R[i + 1] + m / B};
      const double dR = group_weighted(q, 0, N, par) - group_weighted(p, i, N, par) -
                        group_weighted(p, i + 1, N, par);
      const double dM = T * m;
      const bool pos = dM > 0.0;
      const double ratio = pos ? dR / dM : 0.0;
      if (best < 0 || (pos && !best_pos) || (pos == best_pos && pos && ratio < best_ratio)) {
        best = static_cast<int>(i);
        best_ratio = ratio;
        best_pos = pos;
      }
    }
    const uint32_t i = static_cast<uint32_t>(best);
    const double m = bM(i);
    p.R[i] = p.R[i] + p.R[i + 1] + m / B;  // SPEC:570 R(G_i,G_{i+1})
    p.size[i] += p.size[i + 1];
    p.start.erase(p.start.begin() + i + 1);
    p.size.erase(p.size.begin() + i + 1);
    p.R.erase(p.R.begin() + i + 1);
  }
  for (uint32_t gi = 0; gi < p.start.size(); ++gi)
    for (uint32_t k = 0; k < p.size[gi]; ++k) group_of[p.start[gi] + k] = gi;
  *n_groups = static_cast<uint32_t>(p.start.size());
  if (storage) *storage = stor();
  if (recovery) {
    double r = 0.0;
    for (uint32_t gi = 0; gi < p.start.size(); ++gi) r += group_weighted(p, gi, N, par);
    *recovery = r;
  }
  return RW_OK;
}

int rw_recovery_time_estimate(uint32_t N, const double* R, const double* M, double B, int32_t parallel,
                              const uint32_t* group_of, double lost_iterations, double* out) {
  if (N == 0 || !R || !group_of || !out || (N > 1 && !M)) return fail2(RW_INVALID_ARGUMENT, "null argument");
  if (!(B > 0.0)) return fail2(RW_INVALID_CONFIG, "InvalidConfig: B must be > 0");
  Plan p;
  for (uint32_t i = 0; i < N; ++i) {
    if (i > 0 && group_of[i] != group_of[i - 1] && group_of[i] != group_of[i - 1] + 1)
      return fail2(RW_INVALID_CONFIG, "InvalidConfig: groups must be contiguous and ordered");
    if (i == 0 && group_of[0] != 0) return fail2(RW_INVALID_CONFIG, "InvalidConfig: first group must be 0");
    if (i == 0 || group_of[i] != group_of[i - 1]) {
      p.start.push_back(i);
      p.size.push_back(1);
      p.R.push_back(R[i]);
    } else {
      p.size.back() += 1;
      p.R.back() += R[i] + M[i - 1] / B;  // internal boundary becomes replay work
    }
  }
  double r = 0.0;
  for (uint32_t gi = 0; gi < p.start.size(); ++gi) r += group_weighted(p, gi, N, parallel != 0);
  *out = lost_iterations * r;
  return RW_OK;
}

int rw_logging_worthwhile(double bytes_per_iteration, double pcie_bytes_per_s, int32_t p, int32_t m,
                          double iteration_time_s, int32_t* worthwhile, double* transfer_s,
                          double* bubble_s) {
  if (!(pcie_bytes_per_s > 0.0) || !(iteration_time_s > 0.0) || !worthwhile)
    return fail2(RW_INVALID_CONFIG, "InvalidConfig: positive bandwidth and iteration time required");
  int64_t num = 0, den = 1;
  int st = rw_bubble_ratio(p, m, &num, &den);
  if (st) return st;
  const double tr = bytes_per_iteration / pcie_bytes_per_s;
  const double bub = (static_cast<double>(num) / static_cast<double>(den)) * iteration_time_s;
  *worthwhile = tr <= bub ? 1 : 0;
  if (bytes_per_iteration > 0.0 && num == 0) *worthwhile = 0;
  if (transfer_s) *transfer_s = tr;
  if (bubble_s) *bubble_s = bub;
  return RW_OK;
}

}  // extern "C"
