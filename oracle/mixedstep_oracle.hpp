// mixedstep_oracle.hpp — CPU restatement of the reference hot path.
//
// TEST INFRASTRUCTURE ONLY. This file is the parity oracle for the B200
// kernels: it is built into oracle/liborc.so and may be loaded only by
// tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
// reference legs. Nothing in paper_2605_23727_b200/ links or calls it.
//
// Why a restatement: the reference (proj/, C++20) cannot be built here —
// every header includes <Eigen/Core> (systems.hpp:3) and Eigen3 is absent, as
// are the vendored doctest/CLI11/json.hpp (CMakeLists.txt:5,12). The code
// below restates, function by function and operation by operation, the hot
// path of the reference; each function cites the file:line it follows
// (paths relative to /root/reference/proj/). Eigen is replaced by
// std::vector<double> loops with identical per-element rounding. The two
// Eigen reductions whose order the reference leaves to Eigen
// (initial_step's .sum(), solver.cpp:430-444) are fixed to ascending
// sequential order here; that order is the contract.
//
// Build flags: -O3 -ffp-contract=off, no -march (the reference's x86-64
// baseline build, src/CMakeLists.txt:12, has no FMA contraction).
//
// Extensions beyond the reference, each applied only where the reference
// multiplies by coupling_k:
//   * dense K_ij (stored as float values that are exact in the storage
//     format: f32, or f16/bf16 pre-rounded), G_ij <- K_ij * g(x_i, x_j);
//   * LCO config-1 form: coupling on slot 1, per-agent w_i^2 (D2);
//   * CC per-cell constants (D4);
//   * Kuramoto "split" semantics, the formula the
//     device fast path evaluates, here in ascending sequential order.
#pragma once

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <limits>
#include <memory>
#include <stdexcept>
#include <vector>

namespace orc {

using Vec = std::vector<double>;

// ---- precision.hpp:11-80 / precision.cpp:9-42 -----------------------------
enum class FloatFormat : std::uint8_t { Binary32, Binary64 };

constexpr double machine_epsilon(FloatFormat p) noexcept {  // precision.hpp:14-16
  return p == FloatFormat::Binary32 ? 0x1p-23 : 0x1p-52;
}
inline double round_to(double x, FloatFormat p) noexcept {  // precision.hpp:21-24
  if (p == FloatFormat::Binary64) return x;
  return static_cast<double>(static_cast<float>(x));
}
constexpr FloatFormat wider_of(FloatFormat a, FloatFormat b) noexcept {  // precision.hpp:26-30
  return (a == FloatFormat::Binary64 || b == FloatFormat::Binary64) ? FloatFormat::Binary64
                                                                     : FloatFormat::Binary32;
}

struct StagePrecision {  // precision.hpp:36-42
  FloatFormat f_prec;
  FloatFormat sum_prec;
  FloatFormat g_prec;
  friend bool operator==(const StagePrecision&, const StagePrecision&) = default;
};
inline constexpr StagePrecision kAllBinary64{FloatFormat::Binary64, FloatFormat::Binary64,
                                             FloatFormat::Binary64};
inline constexpr StagePrecision kAllBinary32{FloatFormat::Binary32, FloatFormat::Binary32,
                                             FloatFormat::Binary32};

enum class PolicyVariant : std::uint8_t { Single, Mixed1, Mixed2, Double, Custom };

struct PrecisionPolicy {  // precision.hpp:61-74
  PolicyVariant variant = PolicyVariant::Custom;
  std::array<StagePrecision, 3> per_stage{kAllBinary64, kAllBinary64, kAllBinary64};
  StagePrecision first_step_k1 = kAllBinary64;
  FloatFormat storage = FloatFormat::Binary64;
  const StagePrecision& stage(int ell) const { return per_stage[static_cast<size_t>(ell - 2)]; }
  FloatFormat lowest_format() const noexcept {  // precision.cpp:9-20
    if (storage == FloatFormat::Binary32) return FloatFormat::Binary32;
    for (const StagePrecision& sp : {per_stage[0], per_stage[1], per_stage[2], first_step_k1})
      if (sp.f_prec == FloatFormat::Binary32 || sp.sum_prec == FloatFormat::Binary32 ||
          sp.g_prec == FloatFormat::Binary32)
        return FloatFormat::Binary32;
    return FloatFormat::Binary64;
  }
};

inline PrecisionPolicy policy_for(PolicyVariant v) {  // precision.cpp:22-42
  constexpr StagePrecision sss = kAllBinary32;
  constexpr StagePrecision dds{FloatFormat::Binary64, FloatFormat::Binary64, FloatFormat::Binary32};
  constexpr StagePrecision ddd = kAllBinary64;
  PrecisionPolicy p;
  p.variant = v;
  switch (v) {
    case PolicyVariant::Single: p.per_stage = {sss, sss, sss}; break;
    case PolicyVariant::Mixed1: p.per_stage = {sss, sss, dds}; break;
    case PolicyVariant::Mixed2: p.per_stage = {dds, dds, dds}; break;
    case PolicyVariant::Double: p.per_stage = {ddd, ddd, ddd}; break;
    case PolicyVariant::Custom: throw std::invalid_argument("policy_for: custom has no table row");
  }
  p.first_step_k1 = p.per_stage[2];  // precision.cpp:37
  p.storage = v == PolicyVariant::Single ? FloatFormat::Binary32 : FloatFormat::Binary64;
  return p;
}

// ---- rng.hpp:13-52 ----------------------------------------------------------
class SplitMix64 {
 public:
  explicit SplitMix64(std::uint64_t seed, std::uint64_t stream = 0) noexcept
      : state_(seed + stream * 0xD1342543DE82EF95ull) {}
  std::uint64_t next() noexcept {
    std::uint64_t z = (state_ += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  double uniform01() noexcept { return static_cast<double>(next() >> 11) * 0x1p-53; }
  double uniform(double lo, double hi) noexcept { return lo + (hi - lo) * uniform01(); }
  double normal() noexcept {
    if (has_cached_) {
      has_cached_ = false;
      return cached_;
    }
    double u1 = uniform01();
    if (u1 <= 0.0) u1 = 0x1p-53;
    const double u2 = uniform01();
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double a = 6.283185307179586476925286766559 * u2;
    cached_ = r * std::sin(a);
    has_cached_ = true;
    return r * std::cos(a);
  }

 private:
  std::uint64_t state_;
  double cached_ = 0.0;
  bool has_cached_ = false;
};

// ---- systems.hpp / systems.cpp -----------------------------------------------
enum class ModelKind { LCO, Kuramoto, CC, ScalarExp, ScalarZero, ScalarNan };

struct FlopProfile {  // systems.hpp:24-29
  std::int64_t theta_f, theta_g, theta_w;
  int d;
};

struct CcConstants {  // systems.hpp:32-43
  static constexpr double k0 = 2.0;
  static constexpr double k2 = 0.144832;
  static constexpr double k3 = 2.0;
  static constexpr double a = 2.0;
  static constexpr double b = 0.7;
  static constexpr double c = 0.8;
  static constexpr double eps = 0.228249;
  static constexpr double k1_mean = 0.339278;
  static constexpr double k1_sdev = 0.090909;
};

struct ModelParams {
  ModelKind kind = ModelKind::Kuramoto;
  int n = 1;
  int d = 1;
  int coupled_slot = 0;
  Vec m;  // [d]
  Vec omega, w2, k1, theta_h, k0, k2, a, b, c, eps;
  double coupling_k = 1.0;
  double stimulus_i0 = 0.0;
  std::shared_ptr<const std::vector<float>> K;  // row-major n x n; null = scalar coupling_k
  bool split = false;
  int op_round = 0;  // batched tensor-core semantics: binary32 sin/cos GEMM operands rounded to f16 (2) / bf16 (3)
};

void set_threads(int n);
int get_threads();

class CoupledSystem {  // systems.hpp:60-103
 public:
  explicit CoupledSystem(ModelParams p);
  int dim() const noexcept { return p_.d; }
  int agents() const noexcept { return p_.n; }
  std::size_t size() const noexcept { return static_cast<std::size_t>(p_.d) * p_.n; }
  const Vec& weights() const noexcept { return p_.m; }
  const ModelParams& params() const noexcept { return p_; }
  FlopProfile flop_profile() const noexcept { return flops_; }
  void eval_rhs(double t, const Vec& x, const StagePrecision& sp, Vec& out) const;
  Vec eval_rhs(double t, const Vec& x, const StagePrecision& sp) const {
    Vec out(x.size());
    eval_rhs(t, x, sp, out);
    return out;
  }

 private:
  ModelParams p_;
  FlopProfile flops_;
};

// Factories: systems.cpp:209-268 (reference forms, scalar coupling).
std::unique_ptr<CoupledSystem> make_lco(int n_agents, std::uint64_t seed);
std::unique_ptr<CoupledSystem> make_kuramoto(int n_agents, double sigma, double coupling_k,
                                             std::uint64_t seed);
std::unique_ptr<CoupledSystem> make_cc(int n_agents, double coupling_k, double stimulus_i0,
                                       std::uint64_t seed);
Vec lco_analytic(const Vec& x0, double t);  // systems.cpp:270-306

// ---- solver.hpp / solver.cpp -------------------------------------------------
struct ButcherTableau {  // solver.hpp:15-30
  Vec c;
  std::vector<Vec> a;
  Vec b, b_tilde;
  int order_high = 0, order_low = 0;
  bool fsal = false;
  int stages() const { return static_cast<int>(c.size()); }
  static const ButcherTableau& bs32();
  static const ButcherTableau& dp54();
};
int scheme_flops_per_component(const ButcherTableau& tab);  // solver.cpp:361-384

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
  std::vector<double> t_eval;  // dense output times (D6 extension, not in the reference)
};

enum class SolveStatus : std::uint8_t {  // solver.hpp:63-71
  Completed, MaxIterations, MaxFailedSteps, WallClock, SlowSolver, StepTooSmall, NonFinite
};

struct StepOutcome {  // solver.hpp:75-86
  Vec x_next, x_tilde;
  double err = 0.0;
  bool accepted = false;
  Vec k4, x_store;
  double h_used = 0.0, h_next = 0.0;
};
struct StepRecord { double t, h, err; bool accepted; };     // solver.hpp:88-93
struct StepSnapshot { Vec x_before, x_after; double h; };  // solver.hpp:96-100
struct FlopTally {                                         // solver.hpp:104-113
  std::int64_t low = 0, high = 0, rhs_evals = 0;
};
struct SolveResult {  // solver.hpp:115-126
  SolveStatus status = SolveStatus::Completed;
  Vec final_state;
  double t_reached = 0.0;
  std::int64_t n_accepted = 0, n_failed = 0;
  std::vector<StepRecord> step_log;
  std::vector<StepSnapshot> snapshots;
  std::vector<Vec> y_eval;  // dense output rows, one per t_eval reached
  FlopTally flops;
  std::int64_t total_steps() const { return n_accepted + n_failed; }
};

double estimate_error(const Vec& x_n, const Vec& x_next, const Vec& x_tilde, double ab, double rel);
double adjust_step(double h, double err, double rel_tol, const SolverConfig& cfg);
double initial_step(const CoupledSystem& sys, double t0, double t_final, const Vec& x0,
                    const SolverConfig& cfg, int order = 3, FlopTally* tally = nullptr);
StepOutcome bs32_step(const CoupledSystem& sys, double t, const Vec& x_n, double h, const Vec& k1,
                      const PrecisionPolicy& policy, const SolverConfig& cfg,
                      FlopTally* tally = nullptr);
SolveResult solve(const CoupledSystem& sys, const Vec& x0, double t0, double t_final,
                  const PrecisionPolicy& policy, const SolverConfig& cfg);
SolveResult dp54_reference(const CoupledSystem& sys, const Vec& x0, double t0, double t_final,
                           const SolverConfig& cfg = SolverConfig{});

}  // namespace orc
