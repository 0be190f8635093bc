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
  std::printf("cpp api ok: %lld accepted, %lld evals\n", (long long)r.n_accepted, (long long)r.flops.rhs_evals);
  return 0;
}
