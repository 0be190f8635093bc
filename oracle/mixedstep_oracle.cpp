// mixedstep_oracle.cpp — CPU restatement of the reference hot path.
// TEST INFRASTRUCTURE ONLY (see mixedstep_oracle.hpp for scope and rules).
// Compiled with -O3 -ffp-contract=off and no -march, like the reference.
#include "mixedstep_oracle.hpp"

#include <cstddef>

#ifdef _OPENMP
#include <omp.h>
#endif

namespace orc {

namespace {
int g_threads = 1;
}  // namespace

void set_threads(int n) { g_threads = n < 1 ? 1 : n; }
int get_threads() { return g_threads; }

namespace {

constexpr double kNaN = std::numeric_limits<double>::quiet_NaN();

// wider<A,B>, systems.cpp:16-25
template <class A, class B> struct wider { using type = double; };
template <> struct wider<float, float> { using type = float; };
template <class A, class B> using wider_t = typename wider<A, B>::type;

// ---- model kernels (systems.cpp:112-189 + dense-K extension) --------------

// Coupling value in precision S: RN_S(K_ij) for dense K, RN_S(coupling_k)
// otherwise — exactly where the reference writes static_cast<S>(coupling_k).
template <class S, bool HasK>
inline S kij(const ModelParams& p, const float* K, int i, int j) {
  if constexpr (HasK) {
    return static_cast<S>(K[static_cast<std::size_t>(i) * static_cast<std::size_t>(p.n) + j]);
  } else {
    (void)K; (void)i; (void)j;
    return static_cast<S>(p.coupling_k);
  }
}

struct LcoKernel {  // systems.cpp:112-127 (+ D2 config-1 form)
  static constexpr int kDim = 2;
  const ModelParams& p;
  template <class S> void f(int i, const S* xi, S* out) const {
    out[0] = xi[1];
    if (p.w2.empty()) out[1] = -xi[0];
    else out[1] = -(static_cast<S>(p.w2[static_cast<std::size_t>(i)]) * xi[0]);
  }
  template <class S, bool HasK>
  void g(int i, int j, const float* K, const S* xi, const S* xj, S* out) const {
    const S diff = xj[0] - xi[0];
    out[0] = S(0);
    out[1] = S(0);
    out[p.coupled_slot] = kij<S, HasK>(p, K, i, j) * diff;
  }
};

struct KuramotoKernel {  // systems.cpp:129-144
  static constexpr int kDim = 1;
  const ModelParams& p;
  template <class S> void f(int i, const S*, S* out) const {
    out[0] = static_cast<S>(p.omega[static_cast<std::size_t>(i)]);
  }
  template <class S, bool HasK>
  void g(int i, int j, const float* K, const S* xi, const S* xj, S* out) const {
    out[0] = kij<S, HasK>(p, K, i, j) * std::sin(xj[0] - xi[0]);
  }
};

struct CcKernel {  // systems.cpp:146-189 (+ D4 per-cell constants)
  static constexpr int kDim = 4;
  const ModelParams& p;
  template <class S> S cst(const Vec& v, double dflt, int i) const {
    return static_cast<S>(v.empty() ? dflt : v[static_cast<std::size_t>(i)]);
  }
  template <class S> void f(int i, const S* xi, S* out) const {
    using C = CcConstants;
    const S x1 = xi[0], x2 = xi[1], x3 = xi[2], x4 = xi[3];
    const S th = static_cast<S>(p.theta_h[static_cast<std::size_t>(i)]);
    const S x2sq = x2 * x2;
    const S x2h = x2sq * x2sq;
    out[0] = cst<S>(p.k0, C::k0, i) * th / (th + x2h) * (cst<S>(p.a, C::a, i) * x1 * x1 + S(1)) -
             static_cast<S>(p.k1[static_cast<std::size_t>(i)]) * x1;
    out[1] = cst<S>(p.k2, C::k2, i) * (x1 - x2);
    const S x1sq = x1 * x1;
    out[2] = x3 * (S(1) - x3 * x3 / S(3)) - x4 +
             static_cast<S>(p.stimulus_i0) * (S(1) - S(4) / (S(4) + x1sq));
    out[3] = cst<S>(p.eps, C::eps, i) * (x3 + cst<S>(p.b, C::b, i) - cst<S>(p.c, C::c, i) * x4);
  }
  template <class S, bool HasK>
  void g(int i, int j, const float* K, const S* xi, const S* xj, S* out) const {
    using C = CcConstants;
    const S x2 = xi[1];
    const S x2sq = x2 * x2;
    const S th = static_cast<S>(p.theta_h[static_cast<std::size_t>(i)]);
    const S pref = cst<S>(p.k0, C::k0, i) * th * cst<S>(p.a, C::a, i) / (th + x2sq * x2sq);
    out[0] = pref * (kij<S, HasK>(p, K, i, j) * std::atan(xj[0] - xi[0]));
    out[1] = S(0);
    out[2] = S(0);
    out[3] = S(0);
  }
};

// eval_core, systems.cpp:30-64: ascending j including j = i, every slot.
template <int D, class FS, class SS, class GS, bool HasK, class Kernel>
void eval_core(const Kernel& kern, const ModelParams& p, const Vec& x, Vec& out) {
  const int n = p.n;
  std::vector<FS> xf(x.size());
  std::vector<GS> xg(x.size());
  for (std::size_t k = 0; k < x.size(); ++k) {
    xf[k] = static_cast<FS>(x[k]);
    xg[k] = static_cast<GS>(x[k]);
  }
  SS mw[D];
  for (int s = 0; s < D; ++s) mw[s] = static_cast<SS>(p.m[static_cast<std::size_t>(s)]);
  const float* K = p.K ? p.K->data() : nullptr;
  using WS = wider_t<FS, SS>;
#pragma omp parallel for schedule(static) num_threads(g_threads) if (g_threads > 1 && n >= 64)
  for (int i = 0; i < n; ++i) {
    const FS* xi_f = xf.data() + static_cast<std::ptrdiff_t>(i) * D;
    const GS* xi_g = xg.data() + static_cast<std::ptrdiff_t>(i) * D;
    FS fval[D];
    kern.template f<FS>(i, xi_f, fval);
    SS acc[D];
    for (int s = 0; s < D; ++s) acc[s] = SS(0);
    for (int j = 0; j < n; ++j) {
      GS gval[D];
      kern.template g<GS, HasK>(i, j, K, xi_g, xg.data() + static_cast<std::ptrdiff_t>(j) * D,
                                gval);
      for (int s = 0; s < D; ++s) acc[s] = acc[s] + mw[s] * static_cast<SS>(gval[s]);
    }
    for (int s = 0; s < D; ++s)
      out[static_cast<std::size_t>(i) * D + s] =
          static_cast<double>(static_cast<WS>(fval[s]) + static_cast<WS>(acc[s]));
  }
}

// Split Kuramoto: s_j = sin_GS(RN_GS(x_j)),
// c_j = cos_GS(RN_GS(x_j)); A_i = sum_j RN_SS(RN_GS(K_ij) *_GS s_j),
// B_i likewise with c_j, ascending j; coupling = mw *_SS (c_i A_i - s_i B_i);
// out = (double)(RN_WS(omega_i) + RN_WS(coupling)).
template <class FS, class SS, class GS, bool HasK>
void eval_kuramoto_split(const ModelParams& p, const Vec& x, Vec& out) {
  const int n = p.n;
  std::vector<GS> s(static_cast<std::size_t>(n)), c(static_cast<std::size_t>(n));
  for (int j = 0; j < n; ++j) {
    const GS xg = static_cast<GS>(x[static_cast<std::size_t>(j)]);
    s[static_cast<std::size_t>(j)] = std::sin(xg);
    c[static_cast<std::size_t>(j)] = std::cos(xg);
  }
  // tensor-core ensemble semantics (ms_batch_*, csrc/ms_gemm_tc.cuh): each
  // binary32 sin/cos enters the GEMM as hi + lo in K's 16-bit format
  // (hi = RN16(v), lo = RN16(v - hi)); the two partial sums are accumulated
  // separately in binary32 and added once: A = RN32(A_hi + A_lo).
  const bool tc = p.op_round && sizeof(SS) == 4 && sizeof(GS) == 4;
  std::vector<GS> sh = s, sl(s.size(), GS(0)), ch = c, cl(c.size(), GS(0));
  if (tc) {
    auto r16 = [&](float v) -> float {
      return p.op_round == 2 ? static_cast<float>(static_cast<_Float16>(v)) : static_cast<float>(static_cast<__bf16>(v));
    };
    for (std::size_t j = 0; j < s.size(); ++j) {
      const float sv = static_cast<float>(s[j]), cv = static_cast<float>(c[j]);
      sh[j] = static_cast<GS>(r16(sv));
      sl[j] = static_cast<GS>(r16(sv - static_cast<float>(sh[j])));
      ch[j] = static_cast<GS>(r16(cv));
      cl[j] = static_cast<GS>(r16(cv - static_cast<float>(ch[j])));
    }
  }
  const SS mw = static_cast<SS>(p.m[0]);
  const float* K = p.K ? p.K->data() : nullptr;
  using WS = wider_t<FS, SS>;
#pragma omp parallel for schedule(static) num_threads(g_threads) if (g_threads > 1 && n >= 64)
  for (int i = 0; i < n; ++i) {
    const FS fval = static_cast<FS>(p.omega[static_cast<std::size_t>(i)]);
    SS A = SS(0), B = SS(0);
    if (tc) {
      SS Al = SS(0), Bl = SS(0);
      for (int j = 0; j < n; ++j) {
        const GS k = kij<GS, HasK>(p, K, i, j);
        const std::size_t u = static_cast<std::size_t>(j);
        A = A + static_cast<SS>(k * sh[u]);
        Al = Al + static_cast<SS>(k * sl[u]);
        B = B + static_cast<SS>(k * ch[u]);
        Bl = Bl + static_cast<SS>(k * cl[u]);
      }
      A = A + Al;
      B = B + Bl;
    } else {
      for (int j = 0; j < n; ++j) {
        const GS k = kij<GS, HasK>(p, K, i, j);
        A = A + static_cast<SS>(k * s[static_cast<std::size_t>(j)]);
        B = B + static_cast<SS>(k * c[static_cast<std::size_t>(j)]);
      }
    }
    const SS coup = mw * ((static_cast<SS>(c[static_cast<std::size_t>(i)]) * A) -
                          (static_cast<SS>(s[static_cast<std::size_t>(i)]) * B));
    out[static_cast<std::size_t>(i)] =
        static_cast<double>(static_cast<WS>(fval) + static_cast<WS>(coup));
  }
}

template <class FS, class SS, class GS>
void dispatch_model(const ModelParams& p, const Vec& x, Vec& out) {
  const bool hk = static_cast<bool>(p.K);
  switch (p.kind) {
    case ModelKind::LCO: {
      LcoKernel k{p};
      if (hk) eval_core<2, FS, SS, GS, true>(k, p, x, out);
      else eval_core<2, FS, SS, GS, false>(k, p, x, out);
      return;
    }
    case ModelKind::Kuramoto: {
      if (p.split) {
        if (hk) eval_kuramoto_split<FS, SS, GS, true>(p, x, out);
        else eval_kuramoto_split<FS, SS, GS, false>(p, x, out);
        return;
      }
      KuramotoKernel k{p};
      if (hk) eval_core<1, FS, SS, GS, true>(k, p, x, out);
      else eval_core<1, FS, SS, GS, false>(k, p, x, out);
      return;
    }
    case ModelKind::CC: {
      CcKernel k{p};
      if (hk) eval_core<4, FS, SS, GS, true>(k, p, x, out);
      else eval_core<4, FS, SS, GS, false>(k, p, x, out);
      return;
    }
    default: break;
  }
}

// eval_dispatch, systems.cpp:66-89
void eval_dispatch(const ModelParams& p, const Vec& x, const StagePrecision& sp, Vec& out) {
  const bool f32 = sp.f_prec == FloatFormat::Binary32;
  const bool s32 = sp.sum_prec == FloatFormat::Binary32;
  const bool g32 = sp.g_prec == FloatFormat::Binary32;
  if (f32) {
    if (s32) {
      if (g32) dispatch_model<float, float, float>(p, x, out);
      else dispatch_model<float, float, double>(p, x, out);
    } else {
      if (g32) dispatch_model<float, double, float>(p, x, out);
      else dispatch_model<float, double, double>(p, x, out);
    }
  } else {
    if (s32) {
      if (g32) dispatch_model<double, float, float>(p, x, out);
      else dispatch_model<double, float, double>(p, x, out);
    } else {
      if (g32) dispatch_model<double, double, float>(p, x, out);
      else dispatch_model<double, double, double>(p, x, out);
    }
  }
}

FlopProfile profile_for(const ModelParams& p) {
  switch (p.kind) {
    case ModelKind::LCO: return {1, 1, 4, 2};        // systems.cpp:217
    case ModelKind::Kuramoto: return {1, 3, 2, 1};   // systems.cpp:238
    case ModelKind::CC: return {28, 10, 8, 4};       // systems.cpp:266
    default: return {1, 1, 2, 1};                    // test_support.hpp:23
  }
}

}  // namespace

CoupledSystem::CoupledSystem(ModelParams p) : p_(std::move(p)), flops_(profile_for(p_)) {
  if (p_.n < 1) throw std::invalid_argument("CoupledSystem: N must be >= 1");
  if (static_cast<int>(p_.m.size()) != p_.d) throw std::invalid_argument("CoupledSystem: |m| != d");
  if (p_.K && p_.K->size() != static_cast<std::size_t>(p_.n) * static_cast<std::size_t>(p_.n))
    throw std::invalid_argument("CoupledSystem: K must be N x N");
}

void CoupledSystem::eval_rhs(double, const Vec& x, const StagePrecision& sp, Vec& out) const {
  out.resize(x.size());
  switch (p_.kind) {
    case ModelKind::ScalarExp:  // test_support.hpp:25-29
      for (std::size_t k = 0; k < x.size(); ++k) out[k] = round_to(x[k], sp.f_prec);
      return;
    case ModelKind::ScalarZero:  // test_support.hpp:37-40
      for (auto& v : out) v = 0.0;
      return;
    case ModelKind::ScalarNan:  // test_support.hpp:48-52
      for (auto& v : out) v = kNaN;
      return;
    default: break;
  }
  eval_dispatch(p_, x, sp, out);
}

std::unique_ptr<CoupledSystem> make_lco(int n_agents, std::uint64_t) {  // systems.cpp:209-218
  if (n_agents < 1) throw std::invalid_argument("make_lco: N must be >= 1");
  ModelParams p;
  p.kind = ModelKind::LCO;
  p.n = n_agents;
  p.d = 2;
  p.m = {1.0 / n_agents, 0.0};
  p.coupling_k = 1.0;
  return std::make_unique<CoupledSystem>(std::move(p));
}

std::unique_ptr<CoupledSystem> make_kuramoto(int n_agents, double sigma, double coupling_k,
                                             std::uint64_t seed) {  // systems.cpp:220-239
  if (n_agents < 1) throw std::invalid_argument("make_kuramoto: N must be >= 1");
  if (sigma < 0.0) throw std::invalid_argument("make_kuramoto: sigma must be >= 0");
  ModelParams p;
  p.kind = ModelKind::Kuramoto;
  p.n = n_agents;
  p.d = 1;
  p.coupling_k = coupling_k;
  p.omega.resize(static_cast<std::size_t>(n_agents));
  SplitMix64 rng(seed, 0);
  for (int i = 0; i < n_agents; ++i) p.omega[static_cast<std::size_t>(i)] = sigma * rng.normal();
  p.m = {1.0 / n_agents};
  return std::make_unique<CoupledSystem>(std::move(p));
}

std::unique_ptr<CoupledSystem> make_cc(int n_agents, double coupling_k, double stimulus_i0,
                                       std::uint64_t seed) {  // systems.cpp:241-268
  if (n_agents < 1) throw std::invalid_argument("make_cc: N must be >= 1");
  ModelParams p;
  p.kind = ModelKind::CC;
  p.n = n_agents;
  p.d = 4;
  p.coupling_k = coupling_k;
  p.stimulus_i0 = stimulus_i0;
  p.k1.resize(static_cast<std::size_t>(n_agents));
  p.theta_h.resize(static_cast<std::size_t>(n_agents));
  SplitMix64 rng(seed, 0);
  for (int i = 0; i < n_agents; ++i) {
    double k1;
    do {
      k1 = CcConstants::k1_mean + CcConstants::k1_sdev * rng.normal();
    } while (!(k1 > 0.05 && k1 < 1.95));
    p.k1[static_cast<std::size_t>(i)] = k1;
    p.theta_h[static_cast<std::size_t>(i)] = k1 / (CcConstants::k0 - k1);
  }
  p.m = {1.0 / n_agents, 0.0, 0.0, 0.0};
  return std::make_unique<CoupledSystem>(std::move(p));
}

Vec lco_analytic(const Vec& x0, double t) {  // systems.cpp:270-306
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
  const double xm = xm0 * ct + vm0 * st;
  const double vm = -xm0 * st + vm0 * ct;
  const double w = std::sqrt(3.0) / 2.0;
  const double decay = std::exp(-0.5 * t);
  const double cw = std::cos(w * t);
  const double sw = std::sin(w * t) / w;
  const double p00 = decay * (cw - 0.5 * sw);
  const double p01 = decay * sw;
  const double p10 = decay * -sw;
  const double p11 = decay * (cw + 0.5 * sw);
  Vec out(x0.size());
  for (std::size_t i = 0; i < n; ++i) {
    const double du = x0[2 * i] - xm0;
    const double dv = x0[2 * i + 1] - vm0;
    out[2 * i] = xm + p00 * du + p01 * dv;
    out[2 * i + 1] = vm + p10 * du + p11 * dv;
  }
  return out;
}

// ---- solver.cpp ---------------------------------------------------------------
namespace {

ButcherTableau make_bs32() {  // solver.cpp:15-33
  ButcherTableau t;
  t.c = {0.0, 0.5, 0.75, 1.0};
  t.a.assign(4, Vec(4, 0.0));
  t.a[1][0] = 0.5;
  t.a[2][1] = 0.75;
  t.a[3][0] = 2.0 / 9.0;
  t.a[3][1] = 1.0 / 3.0;
  t.a[3][2] = 4.0 / 9.0;
  t.b = {2.0 / 9.0, 1.0 / 3.0, 4.0 / 9.0, 0.0};
  t.b_tilde = {7.0 / 24.0, 0.25, 1.0 / 3.0, 0.125};
  t.order_high = 3;
  t.order_low = 2;
  t.fsal = true;
  return t;
}

ButcherTableau make_dp54() {  // solver.cpp:35-68
  ButcherTableau t;
  t.c = {0.0, 0.2, 0.3, 0.8, 8.0 / 9.0, 1.0, 1.0};
  t.a.assign(7, Vec(7, 0.0));
  t.a[1][0] = 0.2;
  t.a[2][0] = 3.0 / 40.0;
  t.a[2][1] = 9.0 / 40.0;
  t.a[3][0] = 44.0 / 45.0;
  t.a[3][1] = -56.0 / 15.0;
  t.a[3][2] = 32.0 / 9.0;
  t.a[4][0] = 19372.0 / 6561.0;
  t.a[4][1] = -25360.0 / 2187.0;
  t.a[4][2] = 64448.0 / 6561.0;
  t.a[4][3] = -212.0 / 729.0;
  t.a[5][0] = 9017.0 / 3168.0;
  t.a[5][1] = -355.0 / 33.0;
  t.a[5][2] = 46732.0 / 5247.0;
  t.a[5][3] = 49.0 / 176.0;
  t.a[5][4] = -5103.0 / 18656.0;
  t.a[6][0] = 35.0 / 384.0;
  t.a[6][2] = 500.0 / 1113.0;
  t.a[6][3] = 125.0 / 192.0;
  t.a[6][4] = -2187.0 / 6784.0;
  t.a[6][5] = 11.0 / 84.0;
  t.b = t.a[6];
  t.b_tilde = {5179.0 / 57600.0, 0.0, 7571.0 / 16695.0, 393.0 / 640.0, -92097.0 / 339200.0,
               187.0 / 2100.0, 1.0 / 40.0};
  t.order_high = 5;
  t.order_low = 4;
  t.fsal = true;
  return t;
}

bool all_finite(const Vec& v) {
  for (double e : v)
    if (!std::isfinite(e)) return false;
  return true;
}

void tally_eval(FlopTally* tally, const CoupledSystem& sys, const StagePrecision& sp) {
  // solver.cpp:70-82
  if (!tally) return;
  const FlopProfile fp = sys.flop_profile();
  const auto n = static_cast<std::int64_t>(sys.agents());
  auto& f_bucket = sp.f_prec == FloatFormat::Binary32 ? tally->low : tally->high;
  auto& g_bucket = sp.g_prec == FloatFormat::Binary32 ? tally->low : tally->high;
  auto& w_bucket = sp.sum_prec == FloatFormat::Binary32 ? tally->low : tally->high;
  f_bucket += fp.theta_f * n;
  g_bucket += fp.theta_g * n * n;
  w_bucket += fp.theta_w * n * n;
  ++tally->rhs_evals;
}

// solver.cpp:86-104
Vec combine_binary32(const ButcherTableau& tab, int row, const Vec& x_n, double h,
                     const std::vector<Vec>& k) {
  const auto hf = static_cast<float>(h);
  const int s = tab.stages();
  Vec out(x_n.size());
  std::vector<float> coef(static_cast<std::size_t>(s), 0.0f);
  for (int m = 0; m < s; ++m)
    coef[static_cast<std::size_t>(m)] =
        hf * static_cast<float>(tab.a[static_cast<std::size_t>(row)][static_cast<std::size_t>(m)]);
  for (std::size_t i = 0; i < x_n.size(); ++i) {
    auto acc = static_cast<float>(x_n[i]);
    for (int m = 0; m < row; ++m) {
      if (tab.a[static_cast<std::size_t>(row)][static_cast<std::size_t>(m)] == 0.0) continue;
      acc += coef[static_cast<std::size_t>(m)] * static_cast<float>(k[static_cast<std::size_t>(m)][i]);
    }
    out[i] = static_cast<double>(acc);
  }
  return out;
}

// combo = sum_{m : coef[m] != 0} coef[m] * k[m] (first nonzero assigns), then
// out = x + h * combo — the Eigen expressions of solver.cpp:130-142, 188-199.
void lin_combo(const Vec& x, double h, const Vec& coefs, int count, const std::vector<Vec>& k,
               Vec& combo, Vec& out) {
  const std::size_t nv = x.size();
  bool first = true;
  for (int m = 0; m < count; ++m) {
    const double a = coefs[static_cast<std::size_t>(m)];
    if (a == 0.0) continue;
    const Vec& km = k[static_cast<std::size_t>(m)];
    if (first) {
      for (std::size_t i = 0; i < nv; ++i) combo[i] = a * km[i];
      first = false;
    } else {
      for (std::size_t i = 0; i < nv; ++i) combo[i] += a * km[i];
    }
  }
  out.resize(nv);
  for (std::size_t i = 0; i < nv; ++i) out[i] = x[i] + h * combo[i];
}

// rk_step, solver.cpp:110-215
StepOutcome rk_step(const CoupledSystem& sys, const ButcherTableau& tab,
                    const std::vector<StagePrecision>& rows, double t, const Vec& x_n, double h,
                    const Vec& k1, FloatFormat storage, const SolverConfig& cfg, FlopTally* tally) {
  const int s = tab.stages();
  const std::size_t nv = x_n.size();
  const bool store32 = storage == FloatFormat::Binary32;
  StepOutcome out;
  out.h_used = h;
  out.err = kNaN;
  out.accepted = false;
  std::vector<Vec> k(static_cast<std::size_t>(s));
  k[0] = k1;
  Vec combo(nv), arg(nv);
  bool finite = true;
  for (int l = 1; l < s && finite; ++l) {
    lin_combo(x_n, h, tab.a[static_cast<std::size_t>(l)], l, k, combo, arg);
    if (tab.fsal && l == s - 1) {
      out.x_next = arg;
      if (store32) {
        out.x_store = combine_binary32(tab, l, x_n, h, k);
        arg = out.x_store;
      }
    }
    k[static_cast<std::size_t>(l)].resize(nv);
    sys.eval_rhs(t + tab.c[static_cast<std::size_t>(l)] * h, arg,
                 rows[static_cast<std::size_t>(l - 1)], k[static_cast<std::size_t>(l)]);
    tally_eval(tally, sys, rows[static_cast<std::size_t>(l - 1)]);
    finite = all_finite(k[static_cast<std::size_t>(l)]);
  }
  if (tally) tally->high += static_cast<std::int64_t>(scheme_flops_per_component(tab)) *
                            static_cast<std::int64_t>(nv);
  if (!finite) {
    out.h_next = h * cfg.fac_min * 0.5;
    return out;
  }
  out.k4 = k[static_cast<std::size_t>(s - 1)];
  if (!tab.fsal) {
    lin_combo(x_n, h, tab.b, s, k, combo, out.x_next);
  }
  if (!store32) {
    out.x_store = out.x_next;
  } else if (out.x_store.empty()) {
    out.x_store = out.x_next;
    for (double& v : out.x_store) v = round_to(v, FloatFormat::Binary32);
  }
  lin_combo(x_n, h, tab.b_tilde, s, k, combo, out.x_tilde);
  if (!all_finite(out.x_next) || !all_finite(out.x_tilde) || !all_finite(out.x_store)) {
    out.h_next = h * cfg.fac_min * 0.5;
    return out;
  }
  out.err = estimate_error(x_n, out.x_next, out.x_tilde, cfg.abs_tol, cfg.rel_tol);
  if (!std::isfinite(out.err)) {
    out.h_next = h * cfg.fac_min * 0.5;
    return out;
  }
  out.accepted = out.err <= cfg.rel_tol;
  out.h_next = adjust_step(h, out.err, cfg.rel_tol, cfg);
  return out;
}

void validate(const SolverConfig& cfg, double t0, double t_final) {  // solver.cpp:217-224
  if (!(cfg.abs_tol > 0.0 && cfg.abs_tol <= cfg.rel_tol && cfg.rel_tol < 1.0))
    throw std::invalid_argument("solver: need 0 < abs_tol <= rel_tol < 1");
  if (!(cfg.fac_min < 1.0 && cfg.fac_max > 1.0))
    throw std::invalid_argument("solver: need fac_min < 1 < fac_max");
  if (!(t_final > t0)) throw std::invalid_argument("solver: need t_final > t0");
}

// Dense output (D6 extension): cubic Hermite of an accepted step from (x_n, k1)
// to (x_{n+1}, k_last), in the device kernel's operation order (k_dense).
double hermite(double th, double h, double xn, double k1, double xn1, double k4) {
  const double om = 1.0 - th;
  const double om2 = om * om;
  const double th2 = th * th;
  const double h00 = (1.0 + 2.0 * th) * om2;
  const double h10 = th * om2;
  const double h01 = th2 * (3.0 - 2.0 * th);
  const double h11 = th2 * (th - 1.0);
  double v = h00 * xn;
  v = v + h10 * (h * k1);
  v = v + h01 * xn1;
  return v + h11 * (h * k4);
}

// solve_core, solver.cpp:226-347
SolveResult solve_core(const CoupledSystem& sys, const ButcherTableau& tab,
                       const std::vector<StagePrecision>& rows, const StagePrecision& k1_row,
                       FloatFormat lowest, FloatFormat storage, const Vec& x0, double t0,
                       double t_final, const SolverConfig& cfg) {
  validate(cfg, t0, t_final);
  const bool round_state = storage == FloatFormat::Binary32;
  auto store = [&](Vec& v) {
    if (!round_state) return;
    for (double& e : v) e = round_to(e, FloatFormat::Binary32);
  };
  SolveResult res;
  res.final_state = x0;
  res.t_reached = t0;
  const double h_min = cfg.h_min_factor * machine_epsilon(lowest);
  const auto t_start = std::chrono::steady_clock::now();
  auto elapsed = [&] {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
  };
  double h = initial_step(sys, t0, t_final, x0, cfg, tab.order_high, &res.flops);
  if (!std::isfinite(h)) {
    res.status = SolveStatus::NonFinite;
    return res;
  }
  double t = t0;
  Vec x = x0;
  store(x);
  std::size_t next_eval = 0;
  while (next_eval < cfg.t_eval.size() && cfg.t_eval[next_eval] <= t0) {
    res.y_eval.push_back(x);
    ++next_eval;
  }
  Vec k1 = sys.eval_rhs(t0, x, k1_row);
  tally_eval(&res.flops, sys, k1_row);
  if (!all_finite(k1)) {
    res.status = SolveStatus::NonFinite;
    return res;
  }
  bool need_k1 = false;
  for (;;) {
    if (res.total_steps() >= cfg.max_iterations) {
      res.status = SolveStatus::MaxIterations;
      break;
    }
    if (res.n_failed >= cfg.max_failed_steps) {
      res.status = SolveStatus::MaxFailedSteps;
      break;
    }
    if (cfg.time_limits_enabled) {
      const double el = elapsed();
      if (el > cfg.wall_clock_limit) {
        res.status = SolveStatus::WallClock;
        break;
      }
      if (el > cfg.slow_solver_elapsed && (t - t0) < cfg.slow_solver_progress * (t_final - t0)) {
        res.status = SolveStatus::SlowSolver;
        break;
      }
    }
    if (h <= h_min) {
      res.status = SolveStatus::StepTooSmall;
      break;
    }
    if (need_k1) {
      k1 = sys.eval_rhs(t, x, k1_row);
      tally_eval(&res.flops, sys, k1_row);
      need_k1 = false;
      if (!all_finite(k1)) {
        res.status = SolveStatus::NonFinite;
        break;
      }
    }
    bool last = false;
    double h_att = h;
    if (t + 1.01 * h >= t_final) {
      h_att = t_final - t;
      last = true;
    }
    StepOutcome o = rk_step(sys, tab, rows, t, x, h_att, k1, storage, cfg, &res.flops);
    if (cfg.record_step_log) res.step_log.push_back({t, h_att, o.err, o.accepted});
    if (o.accepted) {
      ++res.n_accepted;
      Vec x_prev;
      if (cfg.record_snapshots || !cfg.t_eval.empty()) x_prev = x;
      x = std::move(o.x_store);
      const double t_prev = t;
      t = last ? t_final : (round_state ? round_to(t + h_att, FloatFormat::Binary32) : t + h_att);
      while (next_eval < cfg.t_eval.size() && cfg.t_eval[next_eval] <= t) {
        const double th = (cfg.t_eval[next_eval] - t_prev) / h_att;
        Vec y(x.size());
        for (std::size_t e = 0; e < x.size(); ++e) y[e] = hermite(th, h_att, x_prev[e], k1[e], x[e], o.k4[e]);
        res.y_eval.push_back(std::move(y));
        ++next_eval;
      }
      if (cfg.record_snapshots) res.snapshots.push_back({std::move(x_prev), x, h_att});
      k1 = std::move(o.k4);
      h = o.h_next;
      if (t >= t_final) {
        res.status = SolveStatus::Completed;
        break;
      }
    } else {
      ++res.n_failed;
      h = o.h_next;
      need_k1 = true;
    }
  }
  res.final_state = std::move(x);
  res.t_reached = t;
  return res;
}

}  // namespace

const ButcherTableau& ButcherTableau::bs32() {
  static const ButcherTableau t = make_bs32();
  return t;
}
const ButcherTableau& ButcherTableau::dp54() {
  static const ButcherTableau t = make_dp54();
  return t;
}

int scheme_flops_per_component(const ButcherTableau& tab) {  // solver.cpp:361-384
  int flops = 0;
  const int s = tab.stages();
  for (int l = 1; l < s; ++l) {
    int nz = 0;
    for (int m = 0; m < l; ++m)
      if (tab.a[static_cast<std::size_t>(l)][static_cast<std::size_t>(m)] != 0.0) ++nz;
    flops += 2 * nz + 1;
  }
  if (!tab.fsal) {
    int nz = 0;
    for (int l = 0; l < s; ++l)
      if (tab.b[static_cast<std::size_t>(l)] != 0.0) ++nz;
    flops += 2 * nz + 1;
  }
  int nz = 0;
  for (int l = 0; l < s; ++l)
    if (tab.b_tilde[static_cast<std::size_t>(l)] != 0.0) ++nz;
  flops += 2 * nz + 1;
  flops += 8;
  return flops;
}

double estimate_error(const Vec& x_n, const Vec& x_next, const Vec& x_tilde, double ab,
                      double rel) {  // solver.cpp:399-411
  if (x_n.size() != x_next.size() || x_n.size() != x_tilde.size())
    throw std::invalid_argument("estimate_error: length mismatch");
  const double floor_w = ab / rel;
  double err = 0.0;
  for (std::size_t i = 0; i < x_n.size(); ++i) {
    const double w = std::max(std::max(std::abs(x_n[i]), std::abs(x_next[i])), floor_w);
    err = std::max(err, std::abs(x_next[i] - x_tilde[i]) / w);
  }
  return err;
}

double adjust_step(double h, double err, double rel_tol, const SolverConfig& cfg) {
  // solver.cpp:413-418
  if (err <= 0.0) return h * cfg.fac_max;
  const double fac = cfg.safety * std::pow(rel_tol / err, cfg.controller_exponent);
  return h * std::clamp(fac, cfg.fac_min, cfg.fac_max);
}

double initial_step(const CoupledSystem& sys, double t0, double t_final, const Vec& x0,
                    const SolverConfig& cfg, int order, FlopTally* tally) {
  // solver.cpp:420-451; the three Eigen .sum() reductions are ascending.
  const double cap = (t_final - t0) / 10.0;
  const Vec f0 = sys.eval_rhs(t0, x0, kAllBinary64);
  if (tally) tally_eval(tally, sys, kAllBinary64);
  if (!all_finite(f0)) return kNaN;
  const std::size_t n = x0.size();
  Vec sk(n);
  for (std::size_t i = 0; i < n; ++i) sk[i] = cfg.abs_tol + cfg.rel_tol * std::abs(x0[i]);
  const double inv_n = 1.0 / static_cast<double>(n);
  double s0 = 0.0, s1 = 0.0;
  for (std::size_t i = 0; i < n; ++i) {
    const double q0 = x0[i] / sk[i];
    s0 += q0 * q0;
  }
  for (std::size_t i = 0; i < n; ++i) {
    const double q1 = f0[i] / sk[i];
    s1 += q1 * q1;
  }
  const double d0 = std::sqrt(s0 * inv_n);
  const double d1 = std::sqrt(s1 * inv_n);
  if (d1 < 1e-12) return cap;
  const double h1 = (d0 >= 1e-8) ? 0.01 * d0 / d1 : 1e-6;
  Vec x1(n);
  for (std::size_t i = 0; i < n; ++i) x1[i] = x0[i] + h1 * f0[i];
  const Vec f1 = sys.eval_rhs(t0 + h1, x1, kAllBinary64);
  if (tally) tally_eval(tally, sys, kAllBinary64);
  double h2;
  if (!all_finite(f1)) {
    h2 = h1 * 1e-3;
  } else {
    double s2 = 0.0;
    for (std::size_t i = 0; i < n; ++i) {
      const double q2 = (f1[i] - f0[i]) / sk[i];
      s2 += q2 * q2;
    }
    const double d2 = std::sqrt(s2 * inv_n) / h1;
    const double der = std::max(d1, d2);
    h2 = der < 1e-12 ? cap : std::pow(0.01 / der, 1.0 / static_cast<double>(order + 1));
  }
  return std::min({100.0 * h1, h2, cap});
}

StepOutcome bs32_step(const CoupledSystem& sys, double t, const Vec& x_n, double h, const Vec& k1,
                      const PrecisionPolicy& policy, const SolverConfig& cfg, FlopTally* tally) {
  // solver.cpp:453-460
  const std::vector<StagePrecision> rows = {policy.stage(2), policy.stage(3), policy.stage(4)};
  return rk_step(sys, ButcherTableau::bs32(), rows, t, x_n, h, k1, policy.storage, cfg, tally);
}

SolveResult solve(const CoupledSystem& sys, const Vec& x0, double t0, double t_final,
                  const PrecisionPolicy& policy, const SolverConfig& cfg) {  // solver.cpp:462-470
  const std::vector<StagePrecision> rows = {policy.stage(2), policy.stage(3), policy.stage(4)};
  return solve_core(sys, ButcherTableau::bs32(), rows, policy.first_step_k1, policy.lowest_format(),
                    policy.storage, x0, t0, t_final, cfg);
}

SolveResult dp54_reference(const CoupledSystem& sys, const Vec& x0, double t0, double t_final,
                           const SolverConfig& cfg) {  // solver.cpp:472-483
  SolverConfig ref_cfg = cfg;
  ref_cfg.rel_tol = 1e-9;
  ref_cfg.abs_tol = 1e-9;
  ref_cfg.controller_exponent = 1.0 / 5.0;
  ref_cfg.record_snapshots = false;
  const std::vector<StagePrecision> rows(6, kAllBinary64);
  return solve_core(sys, ButcherTableau::dp54(), rows, kAllBinary64, FloatFormat::Binary64,
                    FloatFormat::Binary64, x0, t0, t_final, ref_cfg);
}

}  // namespace orc
