// C++ host API (include/mixedstep_b200.hpp) on the device: reference KATs of
// proj/tests/test_solver.cpp:111-168 through the C++ mirror. Exit 0 = pass.
#include <cmath>
#include <cstdio>

#include "mixedstep_b200.hpp"

using namespace mixedstep_b200;

#define REQUIRE(c)                                              \
  do {                                                          \
    if (!(c)) {                                                 \
      std::fprintf(stderr, "FAILED %s (line %d)\n", #c, __LINE__); \
      return 1;                                                 \
    }                                                           \
  } while (0)

int main() {
  ms_system_desc d{};
  d.model = MS_MODEL_SCALAR_EXP;
  d.n_agents = 1;
  System exp_sys(d);
  SolverConfig cfg;
  cfg.rel_tol = 1e-2;
  cfg.abs_tol = 1e-2;
  const auto dbl = policy_for(PolicyVariant::Double);
  StepOutcome o = bs32_step(exp_sys, 0.0, {1.0}, 0.1, {1.0}, dbl, cfg);
  REQUIRE(std::fabs(o.x_next[0] - 1.1051666666666666) <= 1e-15 * 2.11);  // doctest Approx scale
  REQUIRE(std::fabs(o.x_tilde[0] - 1.1051895833333334) <= 1e-15 * 2.11);
  REQUIRE(std::fabs(o.err - 2.073593726436435e-05) <= 1e-12 * (1.0 + 2.1e-5));
  REQUIRE(o.k4[0] == o.x_next[0] && o.accepted);

  SolverConfig c2;
  c2.rel_tol = 1e-8;
  c2.abs_tol = 1e-10;
  SolveResult r = solve(exp_sys, {1.0}, 0.0, 1.0, dbl, c2);
  REQUIRE(r.status == SolveStatus::Completed && r.t_reached == 1.0);
  REQUIRE(std::fabs(r.final_state[0] - std::exp(1.0)) / std::exp(1.0) <= 1e-6);
  for (const auto& rec : r.step_log) REQUIRE(rec.accepted ? rec.err <= c2.rel_tol : !(rec.err <= c2.rel_tol));

  // invalid configuration throws like the reference (solver.cpp:217-224)
  bool threw = false;
  try {
    SolverConfig bad;
    bad.abs_tol = 1.0;
    solve(exp_sys, {1.0}, 0.0, 1.0, dbl, bad);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  REQUIRE(threw);
  // snapshots + dense output (solver.cpp:324-327; D6 extension) and the metrics over them
  SolverConfig c3;
  c3.rel_tol = 1e-6;
  c3.abs_tol = 1e-8;
  c3.record_snapshots = true;
  ms_system_desc ld{};
  ld.model = MS_MODEL_LCO;
  ld.n_agents = 4;
  ld.coupling_k = 1.0;
  System lco(ld);
  Vector x0 = {0.1, 0.2, 0.3, 0.4, 0.5, 0.6, 0.7, 0.8};
  SolveResult rs = solve(lco, x0, 0.0, 2.0, dbl, c3, std::vector<double>{0.0, 1.0, 2.0});
  REQUIRE(rs.status == SolveStatus::Completed);
  REQUIRE(static_cast<int64_t>(rs.snapshots.size()) == rs.n_accepted && rs.snapshots.front().x_before == x0);
  REQUIRE(rs.y_eval.size() == 3 && rs.y_eval.back() == rs.final_state && rs.y_eval.front() == x0);
  const ErrorReport er = error_report(rs, lco_analytic(x0, 2.0), 4, c3.abs_tol, c3.rel_tol);
  REQUIRE(er.has_mean_e_analytic && er.mean_e_analytic < c3.rel_tol && er.normalized_final_error < 1e-5);
  // the four named variants concurrently, each equal to its own solve
  std::vector<PrecisionPolicy> pols = {policy_for(PolicyVariant::Single), policy_for(PolicyVariant::Mixed1),
                                       policy_for(PolicyVariant::Mixed2), policy_for(PolicyVariant::Double)};
  SolverConfig c4 = c3;
  c4.record_snapshots = false;
  const std::vector<SolveResult> vr = solve_variants(lco, x0, 0.0, 2.0, pols, c4);
  for (std::size_t i = 0; i < pols.size(); ++i) {
    const SolveResult one = solve(lco, x0, 0.0, 2.0, pols[i], c4);
    REQUIRE(vr[i].final_state == one.final_state && vr[i].n_accepted == one.n_accepted);
  }
  std::printf("cpp api ok: %lld accepted, %lld evals\n", (long long)r.n_accepted, (long long)r.flops.rhs_evals);
  return 0;
}
