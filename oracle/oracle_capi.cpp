// oracle_capi.cpp — C entry points of the CPU oracle (orc_*), shaped like the
// product ABI (include/mixedstep_b200.h) so tests drive both with the same
// structs. TEST INFRASTRUCTURE ONLY: loaded by tests/, __graft_entry__.smoke()
// and bench.py's CPU legs, never by the product package.
#include <cstring>
#include <string>

#include "../include/mixedstep_b200.h"
#include "mixedstep_oracle.hpp"

using namespace orc;

namespace {

thread_local std::string g_err;

struct OrcSystem {
  ModelParams p;
  int k_storage = MS_K_SCALAR;
  std::unique_ptr<CoupledSystem> sys;
  void rebuild() { sys = std::make_unique<CoupledSystem>(p); }
};

template <class F>
int guard(F&& f) {
  try {
    f();
    return MS_OK;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return MS_EINVAL;
  } catch (const std::exception& e) {
    g_err = e.what();
    return MS_ECUDA;
  }
}

FloatFormat fmt(uint8_t v) { return v == MS_BINARY32 ? FloatFormat::Binary32 : FloatFormat::Binary64; }
StagePrecision sp_of(const ms_stage_prec& s) { return {fmt(s.f_prec), fmt(s.sum_prec), fmt(s.g_prec)}; }
ms_stage_prec ms_of(const StagePrecision& s) {
  ms_stage_prec o{};
  o.f_prec = s.f_prec == FloatFormat::Binary32 ? MS_BINARY32 : MS_BINARY64;
  o.sum_prec = s.sum_prec == FloatFormat::Binary32 ? MS_BINARY32 : MS_BINARY64;
  o.g_prec = s.g_prec == FloatFormat::Binary32 ? MS_BINARY32 : MS_BINARY64;
  return o;
}
PrecisionPolicy policy_of(const ms_policy& p) {
  PrecisionPolicy o;
  o.variant = static_cast<PolicyVariant>(p.variant);
  for (int l = 0; l < 3; ++l) o.per_stage[static_cast<size_t>(l)] = sp_of(p.per_stage[l]);
  o.first_step_k1 = sp_of(p.first_step_k1);
  o.storage = fmt(p.storage);
  return o;
}
SolverConfig cfg_of(const ms_solver_config& c) {
  SolverConfig o;
  o.rel_tol = c.rel_tol;
  o.abs_tol = c.abs_tol;
  o.h_min_factor = c.h_min_factor;
  o.max_iterations = c.max_iterations;
  o.max_failed_steps = c.max_failed_steps;
  o.time_limits_enabled = c.time_limits_enabled != 0;
  o.record_step_log = c.record_step_log != 0;
  o.wall_clock_limit = c.wall_clock_limit;
  o.slow_solver_elapsed = c.slow_solver_elapsed;
  o.slow_solver_progress = c.slow_solver_progress;
  o.safety = c.safety;
  o.fac_min = c.fac_min;
  o.fac_max = c.fac_max;
  o.controller_exponent = c.controller_exponent;
  o.record_snapshots = c.record_snapshots != 0;
  return o;
}

// K storage rounding: one RNE rounding from binary64 straight to the format
// (GCC's _Float16 / __bf16 conversions), held exactly in a float.
float round_k(double v, int k_storage) {
  switch (k_storage) {
    case MS_K_F16: return static_cast<float>(static_cast<_Float16>(v));
    case MS_K_BF16: return static_cast<float>(static_cast<__bf16>(v));
    default: return static_cast<float>(v);
  }
}

int dim_of(int model) {
  switch (model) {
    case MS_MODEL_LCO: return 2;
    case MS_MODEL_CC: return 4;
    default: return 1;
  }
}

Vec copy_vec(const double* p, int n) {
  if (!p) return {};
  return Vec(p, p + n);
}

void fill_result(const SolveResult& r, int dn, ms_solve_result* out) {
  out->status = static_cast<int32_t>(r.status);
  out->t_reached = r.t_reached;
  out->n_accepted = r.n_accepted;
  out->n_failed = r.n_failed;
  out->rhs_evals = r.flops.rhs_evals;
  out->flops_low = r.flops.low;
  out->flops_high = r.flops.high;
  if (out->final_state) std::memcpy(out->final_state, r.final_state.data(), sizeof(double) * static_cast<size_t>(dn));
  out->step_log_count = static_cast<int64_t>(r.step_log.size());
  if (out->step_log) {
    const int64_t m = std::min<int64_t>(out->step_log_capacity, out->step_log_count);
    for (int64_t i = 0; i < m; ++i) {
      const StepRecord& s = r.step_log[static_cast<size_t>(i)];
      out->step_log[i].t = s.t;
      out->step_log[i].h = s.h;
      out->step_log[i].err = s.err;
      out->step_log[i].accepted = s.accepted ? 1 : 0;
    }
  }
  out->device_ms = 0.0;
  // StepSnapshots in the C-ABI layout: row 0 = x_before of the first, row k+1
  // = x_after of snapshot k (consecutive snapshots chain, solver.cpp:324-327)
  out->n_eval_done = static_cast<int64_t>(r.y_eval.size());
  if (out->y_eval)
    for (std::size_t q = 0; q < r.y_eval.size() && static_cast<int64_t>(q) < out->n_eval; ++q)
      std::memcpy(out->y_eval + q * static_cast<size_t>(dn), r.y_eval[q].data(), sizeof(double) * static_cast<size_t>(dn));
  out->snapshot_count = static_cast<int64_t>(r.snapshots.size());
  if (out->snapshots && out->snapshot_h && !r.snapshots.empty()) {
    const int64_t m = std::min<int64_t>(out->snapshot_capacity, out->snapshot_count);
    const size_t row = static_cast<size_t>(dn);
    std::memcpy(out->snapshots, r.snapshots[0].x_before.data(), sizeof(double) * row);
    for (int64_t k = 0; k < m; ++k) {
      const StepSnapshot& q = r.snapshots[static_cast<size_t>(k)];
      std::memcpy(out->snapshots + (size_t)(k + 1) * row, q.x_after.data(), sizeof(double) * row);
      out->snapshot_h[k] = q.h;
    }
  }
}

}  // namespace

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }
void orc_set_threads(int n) { set_threads(n); }
int orc_get_threads(void) { return get_threads(); }
double orc_round_to(double x, int f) { return round_to(x, fmt(static_cast<uint8_t>(f))); }
double orc_machine_epsilon(int f) { return machine_epsilon(fmt(static_cast<uint8_t>(f))); }
double orc_round_k(double v, int k_storage) { return round_k(v, k_storage); }

int orc_policy_for(int variant, ms_policy* out) {
  return guard([&] {
    if (variant < 0 || variant > MS_DOUBLE) throw std::invalid_argument("policy_for: unknown variant");
    const PrecisionPolicy p = policy_for(static_cast<PolicyVariant>(variant));
    std::memset(out, 0, sizeof(*out));
    for (int l = 0; l < 3; ++l) out->per_stage[l] = ms_of(p.per_stage[static_cast<size_t>(l)]);
    out->first_step_k1 = ms_of(p.first_step_k1);
    out->storage = p.storage == FloatFormat::Binary32 ? MS_BINARY32 : MS_BINARY64;
    out->variant = static_cast<uint8_t>(variant);
  });
}
int orc_policy_lowest_format(const ms_policy* p) {
  return policy_of(*p).lowest_format() == FloatFormat::Binary32 ? MS_BINARY32 : MS_BINARY64;
}

uint64_t orc_rng_next(uint64_t seed, uint64_t stream, int64_t skip) {
  SplitMix64 r(seed, stream);
  for (int64_t i = 0; i < skip; ++i) r.next();
  return r.next();
}
int orc_rng_uniform(uint64_t seed, uint64_t stream, int64_t n, double lo, double hi, double* out) {
  SplitMix64 r(seed, stream);
  for (int64_t i = 0; i < n; ++i) out[i] = r.uniform(lo, hi);
  return MS_OK;
}
int orc_rng_normal(uint64_t seed, uint64_t stream, int64_t n, double* out) {
  SplitMix64 r(seed, stream);
  for (int64_t i = 0; i < n; ++i) out[i] = r.normal();
  return MS_OK;
}

int orc_system_create(const ms_system_desc* d, void** out) {
  return guard([&] {
    auto s = std::make_unique<OrcSystem>();
    ModelParams& p = s->p;
    const int n = d->n_agents;
    if (n < 1) throw std::invalid_argument("system: N must be >= 1");
    switch (d->model) {
      case MS_MODEL_LCO: p.kind = ModelKind::LCO; break;
      case MS_MODEL_KURAMOTO: p.kind = ModelKind::Kuramoto; break;
      case MS_MODEL_CC: p.kind = ModelKind::CC; break;
      case MS_MODEL_SCALAR_EXP: p.kind = ModelKind::ScalarExp; break;
      case MS_MODEL_SCALAR_ZERO: p.kind = ModelKind::ScalarZero; break;
      case MS_MODEL_SCALAR_NAN: p.kind = ModelKind::ScalarNan; break;
      default: throw std::invalid_argument("system: unknown model");
    }
    p.n = n;
    p.d = dim_of(d->model);
    p.coupled_slot = d->model == MS_MODEL_LCO ? d->coupled_slot : 0;
    if (p.coupled_slot < 0 || p.coupled_slot >= p.d) throw std::invalid_argument("system: bad coupled slot");
    if (d->m) p.m = copy_vec(d->m, p.d);
    else {
      p.m.assign(static_cast<size_t>(p.d), 0.0);
      if (d->model < MS_MODEL_SCALAR_EXP) p.m[static_cast<size_t>(p.coupled_slot)] = 1.0 / n;
    }
    p.coupling_k = d->coupling_k;
    p.stimulus_i0 = d->stimulus_i0;
    p.omega = copy_vec(d->omega, n);
    p.w2 = copy_vec(d->w2, n);
    p.k1 = copy_vec(d->cc_k1, n);
    p.theta_h = copy_vec(d->cc_theta_h, n);
    p.k0 = copy_vec(d->cc_k0, n);
    p.k2 = copy_vec(d->cc_k2, n);
    p.a = copy_vec(d->cc_a, n);
    p.b = copy_vec(d->cc_b, n);
    p.c = copy_vec(d->cc_c, n);
    p.eps = copy_vec(d->cc_eps, n);
    if (p.kind == ModelKind::Kuramoto && p.omega.empty()) throw std::invalid_argument("kuramoto: omega required");
    if (p.kind == ModelKind::CC && (p.k1.empty() || p.theta_h.empty()))
      throw std::invalid_argument("cc: k1 and theta_h required");
    // the split form for the fast and ordered modes;
    // the oracle always sums in ascending j (the device's ordered mode)
    p.split = p.kind == ModelKind::Kuramoto && (d->rhs_mode == MS_RHS_FAST || d->rhs_mode == MS_RHS_ORDERED);
    s->k_storage = d->k_storage;
    if (d->k_storage != MS_K_SCALAR && d->K) {
      auto K = std::make_shared<std::vector<float>>(static_cast<size_t>(n) * static_cast<size_t>(n));
      const size_t nn = K->size();
      if (d->k_host_dtype == MS_HOST_F32) {
        const float* src = static_cast<const float*>(d->K);
        for (size_t q = 0; q < nn; ++q) (*K)[q] = round_k(static_cast<double>(src[q]), d->k_storage);
      } else {
        const double* src = static_cast<const double*>(d->K);
        for (size_t q = 0; q < nn; ++q) (*K)[q] = round_k(src[q], d->k_storage);
      }
      p.K = K;
    }
    s->rebuild();
    *out = s.release();
  });
}

int orc_system_destroy(void* h) {
  delete static_cast<OrcSystem*>(h);
  return MS_OK;
}

int orc_system_fill_k_uniform(void* h, uint64_t seed, uint64_t stream, double lo, double hi) {
  return guard([&] {
    auto* s = static_cast<OrcSystem*>(h);
    if (s->k_storage == MS_K_SCALAR) throw std::invalid_argument("fill_k: system has scalar coupling");
    const size_t nn = static_cast<size_t>(s->p.n) * static_cast<size_t>(s->p.n);
    auto K = std::make_shared<std::vector<float>>(nn);
    SplitMix64 r(seed, stream);
    for (size_t q = 0; q < nn; ++q) (*K)[q] = round_k(r.uniform(lo, hi), s->k_storage);
    s->p.K = K;
    s->rebuild();
  });
}

// batched tensor-core semantics for this system: 0 off, MS_K_F16 / MS_K_BF16
int orc_system_set_op_round(void* h, int ks) {
  return guard([&] {
    auto* s = static_cast<OrcSystem*>(h);
    s->p.op_round = ks;
    s->rebuild();
  });
}
// per-trajectory frequencies (ensemble members share K)
int orc_system_set_omega(void* h, const double* omega) {
  return guard([&] {
    auto* s = static_cast<OrcSystem*>(h);
    s->p.omega.assign(omega, omega + s->p.n);
    s->rebuild();
  });
}

int orc_system_get_k(void* h, double* out) {
  auto* s = static_cast<OrcSystem*>(h);
  if (!s->p.K) return MS_EINVAL;
  for (size_t q = 0; q < s->p.K->size(); ++q) out[q] = (*s->p.K)[q];
  return MS_OK;
}

// Reference factories (systems.cpp:209-268), for the D1 bridge tests.
int orc_make_lco(int n, uint64_t seed, void** out) {
  return guard([&] {
    auto s = std::make_unique<OrcSystem>();
    s->sys = make_lco(n, seed);
    s->p = s->sys->params();
    *out = s.release();
  });
}
int orc_make_kuramoto(int n, double sigma, double k, uint64_t seed, void** out) {
  return guard([&] {
    auto s = std::make_unique<OrcSystem>();
    s->sys = make_kuramoto(n, sigma, k, seed);
    s->p = s->sys->params();
    *out = s.release();
  });
}
int orc_make_cc(int n, double k, double i0, uint64_t seed, void** out) {
  return guard([&] {
    auto s = std::make_unique<OrcSystem>();
    s->sys = make_cc(n, k, i0, seed);
    s->p = s->sys->params();
    *out = s.release();
  });
}
// read back per-agent parameter arrays (0 omega, 1 k1, 2 theta_h, 3 m)
int orc_system_get_param(void* h, int which, double* out) {
  auto* s = static_cast<OrcSystem*>(h);
  const Vec* v = nullptr;
  switch (which) {
    case 0: v = &s->p.omega; break;
    case 1: v = &s->p.k1; break;
    case 2: v = &s->p.theta_h; break;
    case 3: v = &s->p.m; break;
    default: return MS_EINVAL;
  }
  std::memcpy(out, v->data(), sizeof(double) * v->size());
  return static_cast<int>(v->size());
}
int orc_system_dim(void* h) { return static_cast<OrcSystem*>(h)->sys->dim(); }
int orc_system_agents(void* h) { return static_cast<OrcSystem*>(h)->sys->agents(); }
int orc_system_flop_profile(void* h, int64_t out[4]) {
  const FlopProfile fp = static_cast<OrcSystem*>(h)->sys->flop_profile();
  out[0] = fp.theta_f;
  out[1] = fp.theta_g;
  out[2] = fp.theta_w;
  out[3] = fp.d;
  return MS_OK;
}

int orc_eval_rhs(void* h, double t, const double* x, ms_stage_prec sp, double* out) {
  return guard([&] {
    auto* s = static_cast<OrcSystem*>(h);
    const Vec xv(x, x + s->sys->size());
    Vec o;
    s->sys->eval_rhs(t, xv, sp_of(sp), o);
    std::memcpy(out, o.data(), sizeof(double) * o.size());
  });
}

int orc_estimate_error(int64_t n, const double* a, const double* b, const double* c, double ab,
                       double rel, double* err) {
  return guard([&] {
    *err = estimate_error(Vec(a, a + n), Vec(b, b + n), Vec(c, c + n), ab, rel);
  });
}
int orc_adjust_step(double h, double err, double rel, const ms_solver_config* cfg, double* out) {
  return guard([&] { *out = adjust_step(h, err, rel, cfg_of(*cfg)); });
}
int orc_initial_step(void* h, double t0, double tf, const double* x0, const ms_solver_config* cfg,
                     int order, double* h0, int64_t* evals) {
  return guard([&] {
    auto* s = static_cast<OrcSystem*>(h);
    FlopTally tally;
    *h0 = initial_step(*s->sys, t0, tf, Vec(x0, x0 + s->sys->size()), cfg_of(*cfg), order, &tally);
    if (evals) *evals = tally.rhs_evals;
  });
}

int orc_bs32_step(void* h, double t, const double* x_n, double hh, const double* k1,
                  const ms_policy* pol, const ms_solver_config* cfg, ms_step_outcome* out) {
  return guard([&] {
    auto* s = static_cast<OrcSystem*>(h);
    const size_t dn = s->sys->size();
    FlopTally tally;
    const StepOutcome o = bs32_step(*s->sys, t, Vec(x_n, x_n + dn), hh, Vec(k1, k1 + dn),
                                    policy_of(*pol), cfg_of(*cfg), &tally);
    auto put = [&](double* dst, const Vec& v) {
      if (!dst) return;
      if (v.empty()) {
        for (size_t i = 0; i < dn; ++i) dst[i] = std::numeric_limits<double>::quiet_NaN();
      } else {
        std::memcpy(dst, v.data(), sizeof(double) * dn);
      }
    };
    put(out->x_next, o.x_next);
    put(out->x_tilde, o.x_tilde);
    put(out->k4, o.k4);
    put(out->x_store, o.x_store);
    out->err = o.err;
    out->accepted = o.accepted ? 1 : 0;
    out->h_used = o.h_used;
    out->h_next = o.h_next;
    out->rhs_evals = tally.rhs_evals;
    out->flops_low = tally.low;
    out->flops_high = tally.high;
  });
}

int orc_solve(void* h, const double* x0, double t0, double tf, const ms_policy* pol,
              const ms_solver_config* cfg, ms_solve_result* res) {
  return guard([&] {
    auto* s = static_cast<OrcSystem*>(h);
    const size_t dn = s->sys->size();
    SolverConfig c = cfg_of(*cfg);
    if (res->t_eval && res->n_eval > 0) c.t_eval.assign(res->t_eval, res->t_eval + res->n_eval);
    const SolveResult r = solve(*s->sys, Vec(x0, x0 + dn), t0, tf, policy_of(*pol), c);
    fill_result(r, static_cast<int>(dn), res);
  });
}

int orc_dp54_reference(void* h, const double* x0, double t0, double tf, const ms_solver_config* cfg,
                       ms_solve_result* res) {
  return guard([&] {
    auto* s = static_cast<OrcSystem*>(h);
    const size_t dn = s->sys->size();
    const SolveResult r = dp54_reference(*s->sys, Vec(x0, x0 + dn), t0, tf, cfg_of(*cfg));
    fill_result(r, static_cast<int>(dn), res);
  });
}

int orc_lco_analytic(int64_t n2, const double* x0, double t, double* out) {
  return guard([&] {
    const Vec o = lco_analytic(Vec(x0, x0 + n2), t);
    std::memcpy(out, o.data(), sizeof(double) * o.size());
  });
}

int orc_scheme_flops_bs32(void) { return scheme_flops_per_component(ButcherTableau::bs32()); }

}  // extern "C"
