// mixedstep_b200.hpp — C++ host mirror of the reference solver/model API over
// the C-ABI (include/mixedstep_b200.h). Header-only; link libmixedstep_b200.so.
//
// Names, argument meaning and error behaviour follow the reference:
//   precision.hpp:11-80   FloatFormat, StagePrecision, PrecisionPolicy, policy_for
//   systems.hpp:60-119    CoupledSystem (here: System, device-resident), factories
//   solver.hpp:39-163     SolverConfig, SolveStatus, StepRecord, StepOutcome,
//                         SolveResult, estimate_error, adjust_step, initial_step,
//                         bs32_step, solve, dp54_reference
// Config errors throw std::invalid_argument (MS_EINVAL); CUDA failures throw
// std::runtime_error (MS_ECUDA); numerical failure is SolveResult::status.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "mixedstep_b200.h"

namespace mixedstep_b200 {

using Vector = std::vector<double>;

enum class FloatFormat : std::uint8_t { Binary32 = MS_BINARY32, Binary64 = MS_BINARY64 };
enum class PolicyVariant : std::uint8_t { Single = MS_SINGLE, Mixed1 = MS_MIXED1, Mixed2 = MS_MIXED2,
                                          Double = MS_DOUBLE, Custom = MS_CUSTOM };
enum class SolveStatus : std::uint8_t { Completed, MaxIterations, MaxFailedSteps, WallClock, SlowSolver,
                                        StepTooSmall, NonFinite };

inline void check(int rc, const char* what) {
  if (rc == MS_OK) return;
  const std::string msg = std::string(what) + ": " + ms_last_error();
  if (rc == MS_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

struct StagePrecision {
  FloatFormat f_prec, sum_prec, g_prec;
  ms_stage_prec c() const {
    return ms_stage_prec{static_cast<uint8_t>(f_prec), static_cast<uint8_t>(sum_prec),
                         static_cast<uint8_t>(g_prec), 0};
  }
};
inline constexpr StagePrecision kAllBinary64{FloatFormat::Binary64, FloatFormat::Binary64, FloatFormat::Binary64};
inline constexpr StagePrecision kAllBinary32{FloatFormat::Binary32, FloatFormat::Binary32, FloatFormat::Binary32};

struct PrecisionPolicy {
  PolicyVariant variant = PolicyVariant::Custom;
  StagePrecision per_stage[3] = {kAllBinary64, kAllBinary64, kAllBinary64};
  StagePrecision first_step_k1 = kAllBinary64;
  FloatFormat storage = FloatFormat::Binary64;
  const StagePrecision& stage(int ell) const { return per_stage[ell - 2]; }
  ms_policy c() const {
    ms_policy p{};
    for (int l = 0; l < 3; ++l) p.per_stage[l] = per_stage[l].c();
    p.first_step_k1 = first_step_k1.c();
    p.storage = static_cast<uint8_t>(storage);
    p.variant = static_cast<uint8_t>(variant);
    return p;
  }
  FloatFormat lowest_format() const {
    const ms_policy p = c();
    return static_cast<FloatFormat>(ms_policy_lowest_format(&p));
  }
};

inline PrecisionPolicy policy_for(PolicyVariant v) {
  ms_policy p{};
  check(ms_policy_for(static_cast<int>(v), &p), "policy_for");
  PrecisionPolicy o;
  o.variant = v;
  for (int l = 0; l < 3; ++l)
    o.per_stage[l] = {static_cast<FloatFormat>(p.per_stage[l].f_prec), static_cast<FloatFormat>(p.per_stage[l].sum_prec),
                      static_cast<FloatFormat>(p.per_stage[l].g_prec)};
  o.first_step_k1 = o.per_stage[2];
  o.storage = static_cast<FloatFormat>(p.storage);
  return o;
}

struct SolverConfig {  // solver.hpp:39-61
  double rel_tol = 1e-6;
  double abs_tol = 1e-8;
  double h_min_factor = 100.0;
  std::int64_t max_iterations = 100000;
  std::int64_t max_failed_steps = 85000;
  bool time_limits_enabled = true;
  double wall_clock_limit = 5400.0;
  double slow_solver_elapsed = 2700.0;
  double slow_solver_progress = 0.10;
  double safety = 0.9;
  double fac_min = 0.2;
  double fac_max = 5.0;
  double controller_exponent = 1.0 / 3.0;
  bool record_step_log = true;
  bool record_snapshots = false;
  ms_solver_config c() const {
    ms_solver_config o{};
    o.rel_tol = rel_tol; o.abs_tol = abs_tol; o.h_min_factor = h_min_factor;
    o.max_iterations = max_iterations; o.max_failed_steps = max_failed_steps;
    o.time_limits_enabled = time_limits_enabled; o.record_step_log = record_step_log;
    o.wall_clock_limit = wall_clock_limit; o.slow_solver_elapsed = slow_solver_elapsed;
    o.slow_solver_progress = slow_solver_progress; o.safety = safety; o.fac_min = fac_min;
    o.fac_max = fac_max; o.controller_exponent = controller_exponent;
    o.record_snapshots = record_snapshots;
    return o;
  }
};

struct StepRecord { double t, h, err; bool accepted; };
struct FlopTally { std::int64_t low = 0, high = 0, rhs_evals = 0; };
struct StepSnapshot { Vector x_before, x_after; double h; };  // solver.hpp:96-100
struct SolveResult {
  SolveStatus status = SolveStatus::Completed;
  Vector final_state;
  double t_reached = 0.0;
  std::int64_t n_accepted = 0, n_failed = 0;
  std::vector<StepRecord> step_log;
  std::vector<StepSnapshot> snapshots;
  std::vector<Vector> y_eval;  // dense output (D6 extension): one row per reached t_eval
  FlopTally flops;
  double device_ms = 0.0;
  std::int64_t total_steps() const { return n_accepted + n_failed; }
};
struct StepOutcome {
  Vector x_next, x_tilde;
  double err = 0.0;
  bool accepted = false;
  Vector k4, x_store;
  double h_used = 0.0, h_next = 0.0;
};

// A coupled system resident on one B200 (the CoupledSystem of systems.hpp:60-103).
class System {
 public:
  explicit System(const ms_system_desc& d) { check(ms_system_create(&d, &h_), "ms_system_create"); }
  ~System() { if (h_) ms_system_destroy(h_); }
  System(const System&) = delete;
  System& operator=(const System&) = delete;
  int dim() const { return ms_system_dim(h_); }
  int agents() const { return ms_system_agents(h_); }
  std::size_t size() const { return static_cast<std::size_t>(dim()) * agents(); }
  void fill_k_uniform(std::uint64_t seed, std::uint64_t stream, double lo, double hi) {
    check(ms_system_fill_k_uniform(h_, seed, stream, lo, hi), "fill_k_uniform");
  }
  void eval_rhs(double t, const Vector& x, const StagePrecision& sp, Vector& out) const {
    if (x.size() != size()) throw std::invalid_argument("eval_rhs: state length must be d*N");
    out.resize(x.size());
    check(ms_eval_rhs(h_, t, x.data(), sp.c(), out.data()), "eval_rhs");
  }
  Vector eval_rhs(double t, const Vector& x, const StagePrecision& sp) const {
    Vector out;
    eval_rhs(t, x, sp, out);
    return out;
  }
  ms_system_t handle() const { return h_; }

 private:
  ms_system_t h_ = nullptr;
};

inline double estimate_error(const Vector& x_n, const Vector& x_next, const Vector& x_tilde, double ab, double rel) {
  if (x_n.size() != x_next.size() || x_n.size() != x_tilde.size())
    throw std::invalid_argument("estimate_error: length mismatch");
  double e = 0.0;
  check(ms_estimate_error(static_cast<int64_t>(x_n.size()), x_n.data(), x_next.data(), x_tilde.data(), ab, rel, &e),
        "estimate_error");
  return e;
}

inline double adjust_step(double h, double err, double rel_tol, const SolverConfig& cfg) {
  const ms_solver_config c = cfg.c();
  double o = 0.0;
  check(ms_adjust_step(h, err, rel_tol, &c, &o), "adjust_step");
  return o;
}

inline double initial_step(const System& sys, double t0, double t_final, const Vector& x0, const SolverConfig& cfg,
                           int order = 3) {
  const ms_solver_config c = cfg.c();
  double h0 = 0.0;
  check(ms_initial_step(sys.handle(), t0, t_final, x0.data(), &c, order, &h0, nullptr), "initial_step");
  return h0;
}

inline StepOutcome bs32_step(const System& sys, double t, const Vector& x_n, double h, const Vector& k1,
                             const PrecisionPolicy& policy, const SolverConfig& cfg) {
  StepOutcome o;
  o.x_next.resize(x_n.size());
  o.x_tilde.resize(x_n.size());
  o.k4.resize(x_n.size());
  o.x_store.resize(x_n.size());
  ms_step_outcome r{};
  r.x_next = o.x_next.data();
  r.x_tilde = o.x_tilde.data();
  r.k4 = o.k4.data();
  r.x_store = o.x_store.data();
  const ms_policy p = policy.c();
  const ms_solver_config c = cfg.c();
  check(ms_bs32_step(sys.handle(), t, x_n.data(), h, k1.data(), &p, &c, &r), "bs32_step");
  o.err = r.err;
  o.accepted = r.accepted != 0;
  o.h_used = r.h_used;
  o.h_next = r.h_next;
  return o;
}

namespace detail {
template <class F>
SolveResult run(F&& call, std::size_t dn, const SolverConfig& cfg, const std::vector<double>* t_eval = nullptr) {
  SolveResult out;
  out.final_state.resize(dn);
  std::vector<ms_step_record> log(cfg.record_step_log ? static_cast<std::size_t>(cfg.max_iterations) : 0);
  ms_solve_result r{};
  r.final_state = out.final_state.data();
  r.step_log = log.empty() ? nullptr : log.data();
  r.step_log_capacity = static_cast<int64_t>(log.size());
  // snapshots: as many accepted steps as 256 MiB of rows hold
  std::int64_t scap = 0;
  if (cfg.record_snapshots) {
    const std::int64_t fit = static_cast<std::int64_t>((std::size_t(256) << 20) / (8 * (dn ? dn : 1))) - 1;
    scap = std::max<std::int64_t>(1, std::min<std::int64_t>(cfg.max_iterations, fit));
  }
  std::vector<double> rows(scap ? static_cast<std::size_t>(scap + 1) * dn : 0), hs(static_cast<std::size_t>(scap));
  if (scap) {
    r.snapshots = rows.data();
    r.snapshot_h = hs.data();
    r.snapshot_capacity = scap;
  }
  std::vector<double> dense(t_eval ? t_eval->size() * dn : 0);
  if (t_eval && !t_eval->empty()) {
    r.t_eval = t_eval->data();
    r.n_eval = static_cast<int64_t>(t_eval->size());
    r.y_eval = dense.data();
  }
  call(r);
  out.status = static_cast<SolveStatus>(r.status);
  out.t_reached = r.t_reached;
  out.n_accepted = r.n_accepted;
  out.n_failed = r.n_failed;
  out.flops = {r.flops_low, r.flops_high, r.rhs_evals};
  out.device_ms = r.device_ms;
  const int64_t m = r.step_log_count < r.step_log_capacity ? r.step_log_count : r.step_log_capacity;
  for (int64_t i = 0; i < m; ++i)
    out.step_log.push_back({log[i].t, log[i].h, log[i].err, log[i].accepted != 0});
  for (int64_t q = 0; q < r.n_eval_done; ++q)
    out.y_eval.emplace_back(dense.begin() + q * dn, dense.begin() + (q + 1) * dn);
  const int64_t ns = std::min<int64_t>(scap, r.snapshot_count);
  for (int64_t k = 0; k < ns; ++k) {
    const double* b = rows.data() + static_cast<std::size_t>(k) * dn;
    out.snapshots.push_back({Vector(b, b + dn), Vector(b + dn, b + 2 * dn), hs[static_cast<std::size_t>(k)]});
  }
  return out;
}
}  // namespace detail

inline SolveResult solve(const System& sys, const Vector& x0, double t0, double t_final, const PrecisionPolicy& policy,
                         const SolverConfig& cfg) {
  const ms_policy p = policy.c();
  const ms_solver_config c = cfg.c();
  return detail::run([&](ms_solve_result& r) {
    check(ms_solve(sys.handle(), x0.data(), t0, t_final, &p, &c, &r), "solve");
  }, x0.size(), cfg);
}

// solve with dense output at the sorted times t_eval in [t0, t_final] (D6 extension)
inline SolveResult solve(const System& sys, const Vector& x0, double t0, double t_final, const PrecisionPolicy& policy,
                         const SolverConfig& cfg, const std::vector<double>& t_eval) {
  const ms_policy p = policy.c();
  const ms_solver_config c = cfg.c();
  return detail::run([&](ms_solve_result& r) {
    check(ms_solve(sys.handle(), x0.data(), t0, t_final, &p, &c, &r), "solve");
  }, x0.size(), cfg, &t_eval);
}

inline SolveResult dp54_reference(const System& sys, const Vector& x0, double t0, double t_final,
                                  const SolverConfig& cfg = SolverConfig{}) {
  const ms_solver_config c = cfg.c();
  return detail::run([&](ms_solve_result& r) {
    check(ms_dp54_reference(sys.handle(), x0.data(), t0, t_final, &c, &r), "dp54_reference");
  }, x0.size(), cfg);
}

// Concurrent solves of one system under up to four policies (the harness's
// variants, harness.cpp:113-121): one K sweep per stage for all of them where the
// model allows, each result bit-identical to its own solve().
inline std::vector<SolveResult> solve_variants(const System& sys, const Vector& x0, double t0, double t_final,
                                               const std::vector<PrecisionPolicy>& policies,
                                               const SolverConfig& cfg) {
  const std::size_t nv = policies.size(), dn = x0.size();
  ms_variants_t vh = nullptr;
  check(ms_variants_create(sys.handle(), static_cast<int32_t>(nv), &vh), "variants_create");
  std::vector<ms_policy> pols(nv);
  for (std::size_t i = 0; i < nv; ++i) pols[i] = policies[i].c();
  const ms_solver_config c = cfg.c();
  std::vector<SolveResult> out(nv);
  std::vector<std::vector<ms_step_record>> logs(nv);
  std::vector<ms_solve_result> rs(nv);
  for (std::size_t i = 0; i < nv; ++i) {
    out[i].final_state.resize(dn);
    logs[i].resize(cfg.record_step_log ? static_cast<std::size_t>(cfg.max_iterations) : 0);
    rs[i] = ms_solve_result{};
    rs[i].final_state = out[i].final_state.data();
    rs[i].step_log = logs[i].empty() ? nullptr : logs[i].data();
    rs[i].step_log_capacity = static_cast<int64_t>(logs[i].size());
  }
  const int rc = ms_variants_solve(vh, x0.data(), t0, t_final, pols.data(), &c, rs.data());
  ms_variants_destroy(vh);
  check(rc, "variants_solve");
  for (std::size_t i = 0; i < nv; ++i) {
    const ms_solve_result& r = rs[i];
    out[i].status = static_cast<SolveStatus>(r.status);
    out[i].t_reached = r.t_reached;
    out[i].n_accepted = r.n_accepted;
    out[i].n_failed = r.n_failed;
    out[i].flops = {r.flops_low, r.flops_high, r.rhs_evals};
    out[i].device_ms = r.device_ms;
    const int64_t m = std::min(r.step_log_count, r.step_log_capacity);
    for (int64_t k = 0; k < m; ++k)
      out[i].step_log.push_back({logs[i][k].t, logs[i][k].h, logs[i][k].err, logs[i][k].accepted != 0});
  }
  return out;
}

// ---- host metrics over device results (metrics.hpp / metrics.cpp) ------------

// Analytic propagator of the reference LCO at time t (systems.cpp:270-306):
// the agent mean rotates, deviations decay through exp(tA), A = [[-1,1],[-1,0]].
inline Vector lco_analytic(const Vector& x0, double t) {
  if (x0.size() % 2 != 0) throw std::invalid_argument("lco_analytic: state length must be 2N");
  const std::size_t n = x0.size() / 2;
  double xm0 = 0.0, vm0 = 0.0;
  for (std::size_t i = 0; i < n; ++i) {
    xm0 += x0[2 * i];
    vm0 += x0[2 * i + 1];
  }
  xm0 /= static_cast<double>(n);
  vm0 /= static_cast<double>(n);
  const double ct = std::cos(t), st = std::sin(t);
  const double xm = xm0 * ct + vm0 * st, vm = -xm0 * st + vm0 * ct;
  const double w = std::sqrt(3.0) / 2.0, decay = std::exp(-0.5 * t);
  const double cw = std::cos(w * t), sw = std::sin(w * t) / w;
  const double p00 = decay * (cw - 0.5 * sw), p01 = decay * sw, p10 = decay * -sw, p11 = decay * (cw + 0.5 * sw);
  Vector out(x0.size());
  for (std::size_t i = 0; i < n; ++i) {
    const double du = x0[2 * i] - xm0, dv = x0[2 * i + 1] - vm0;
    out[2 * i] = xm + p00 * du + p01 * dv;
    out[2 * i + 1] = vm + p10 * du + p11 * dv;
  }
  return out;
}

// ||x_ref - x||_2 / sqrt(N) (metrics.cpp:10-17), squares summed in index order
inline double normalized_final_error(const Vector& x_ref, const Vector& x, std::int64_t n_agents) {
  if (x_ref.size() != x.size()) throw std::invalid_argument("normalized_final_error: length mismatch");
  if (n_agents < 1) throw std::invalid_argument("normalized_final_error: N must be >= 1");
  double s = 0.0;
  for (std::size_t k = 0; k < x.size(); ++k) s += (x_ref[k] - x[k]) * (x_ref[k] - x[k]);
  return std::sqrt(s) / std::sqrt(static_cast<double>(n_agents));
}

// one-step error against the analytic LCO propagator re-anchored at x_n (metrics.cpp:42-52)
inline double real_local_error(const Vector& x_n, const Vector& x_next, double h_n, double ab, double rel) {
  const Vector x_ex = lco_analytic(x_n, h_n);
  const double delta = ab / rel;
  double err = 0.0;
  for (std::size_t k = 0; k < x_next.size(); ++k)
    err = std::max(err, std::abs(x_next[k] - x_ex[k]) / std::max(std::abs(x_ex[k]), delta));
  return err;
}

struct ErrorReport {  // metrics.hpp:31-35
  double normalized_final_error = 0.0;
  double mean_e_bs = 0.0;
  bool has_mean_e_analytic = false;
  double mean_e_analytic = 0.0;
};

// metrics.cpp:19-40
inline ErrorReport error_report(const SolveResult& run, const Vector& x_ref_final, std::int64_t n_agents, double ab,
                                double rel) {
  ErrorReport er;
  er.normalized_final_error = normalized_final_error(x_ref_final, run.final_state, n_agents);
  double sum = 0.0;
  std::int64_t n = 0;
  for (const StepRecord& r : run.step_log)
    if (r.accepted) {
      sum += r.err;
      ++n;
    }
  er.mean_e_bs = n > 0 ? sum / static_cast<double>(n) : 0.0;
  if (!run.snapshots.empty()) {
    double a = 0.0;
    for (const StepSnapshot& q : run.snapshots) a += real_local_error(q.x_before, q.x_after, q.h, ab, rel);
    er.has_mean_e_analytic = true;
    er.mean_e_analytic = a / static_cast<double>(run.snapshots.size());
  }
  return er;
}

}  // namespace mixedstep_b200
