// ms_batch.cu — batched ensembles sharing one K: step kernels, orchestration
// (a CUDA graph whose WHILE node runs lock-step attempts until every
// trajectory is done) and the ms_batch_* C-ABI.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "ms_batch.cuh"
#include "ms_gemm_tc.cuh"
#include "ms_internal.h"

using namespace msb;

namespace msb {
MS_DEFINE_LAUNCH_READER(launches_tu_batch)
}  // namespace msb

namespace {

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct InvalidArg : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};

#define BCK(call)                                                                                   \
  do {                                                                                              \
    cudaError_t e_ = (call);                                                                        \
    if (e_ != cudaSuccess)                                                                          \
      throw CudaError(std::string(#call) + ": " + cudaGetErrorString(e_) + " (ms_batch.cu:" +       \
                      std::to_string(__LINE__) + ")");                                              \
  } while (0)

template <class F>
int bguard(F&& f) {
  try {
    f();
    return MS_OK;
  } catch (const std::invalid_argument& e) {
    set_last_error(e.what());
    return MS_EINVAL;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return MS_ECUDA;
  }
}

const ms_stage_prec kDDDb{MS_BINARY64, MS_BINARY64, MS_BINARY64, 0};
bool is_sss(const ms_stage_prec& s) { return is32(s.f_prec) && is32(s.sum_prec) && is32(s.g_prec); }
bool same_row(const ms_stage_prec& a, const ms_stage_prec& b) {
  return a.f_prec == b.f_prec && a.sum_prec == b.sum_prec && a.g_prec == b.g_prec;
}

// ---- per-trajectory step kernels -------------------------------------------------

struct BFinArgs {
  BatchDev d;
  int S, nbt, k1_elided;
  double bt[kMaxStages];
  int bslot_[kMaxStages];
  int use_p;  // the last prep wrote P = b~1 k1 + b~2 k2 + b~3 k3 into scr1
  int ctl_smem;  // controller on a shared-memory copy of Ctl[b] (MS_CTL_SMEM)
  int err_epi;   // the last contraction's epilogue formed the error (d.errb / d.nfe): read and clear it
  int quot;      // the error norm's max without a division per element (QuotMax; MS_BFIN_QUOT=off: per element)
};

// x_tilde, weighted max-norm and the controller of one trajectory per CTA;
// the last CTA to finish (ticket) also evaluates the loop condition, so an
// attempt ends without a separate condition kernel
#ifndef MS_BFIN_THREADS
#define MS_BFIN_THREADS 128  // 8 x 128 threads per SM: 64 registers, unrolled loads, one wave
#endif
constexpr int kBFinThreads = MS_BFIN_THREADS;
#ifndef MS_BFIN_UNROLL
#define MS_BFIN_UNROLL 8  // element-loop unroll (0: the compiler's choice)
#endif
constexpr int kBFinUnroll = MS_BFIN_UNROLL;
// resident blocks per SM: 8 so all B = 1024 trajectory blocks run in one wave
// (61 registers x 256 threads gave 4 blocks per SM, 1.7 waves); 128-thread
// blocks leave 64 registers for an unrolled element loop, where 256 x 32
// registers spilled and kept one element's loads in flight per thread
// (292.0 -> 287.0 ms per C5 solve, tools/gpu_bfin2.sh)
#ifndef MS_BFIN_MINB
#define MS_BFIN_MINB 8
#endif
__global__ void __launch_bounds__(kBFinThreads, MS_BFIN_MINB) kb_finalize(BFinArgs f, int has_handle, cudaGraphConditionalHandle h) {
  msb::count_launch();
  pdl_enter();
  const int b = blockIdx.x;
  const BatchDev& d = f.d;
  Ctl* cg = d.ctl + b;
  // the trajectory's control block: a shared-memory copy (one round trip in,
  // one out) unless MS_CTL_SMEM=off; no other block touches Ctl[b] here
  __shared__ __align__(16) Ctl cs;
  if (f.ctl_smem) {
    ctl_copy(&cs, cg);
    __syncthreads();
  }
  Ctl* c = f.ctl_smem ? &cs : cg;
  const bool dead = c->done != 0;
  const bool stage_nf = c->nf_mask != 0;
  double m = 0.0;
  bool nf = false;
  if (f.err_epi) {
    if (threadIdx.x == 0) {
      if (!dead && !stage_nf) {
        m = __longlong_as_double((long long)d.errb[b]);
        nf = d.nfe[b] != 0;
      }
      d.errb[b] = 0ull;
      d.nfe[b] = 0;
    }
  } else if (!dead && !stage_nf) {
    const int ix = c->ix;
    const int64_t o = (int64_t)b * d.n;
    const double* __restrict__ x = d.xb[ix] + o;
    const double* __restrict__ xst = d.xb[ix ^ 1] + o;
    const double* __restrict__ xnx = c->store32 ? d.xn + o : xst;
    // the four BS3(2) error weights b~ (all nonzero, bplan checks nbt == 4)
    const double* __restrict__ k0 = bslot(d, f.S, f.bslot_[0], c) + o;
    const double* __restrict__ k1 = bslot(d, f.S, f.bslot_[1], c) + o;
    const double* __restrict__ k2 = bslot(d, f.S, f.bslot_[2], c) + o;
    const double* __restrict__ k3 = bslot(d, f.S, f.bslot_[3], c) + o;
    const double b0 = f.bt[0], b1 = f.bt[1], b2 = f.bt[2], b3 = f.bt[3];
    const double h = c->h_att;
    const double floor_w = __ddiv_rn(c->abs_tol, c->rel_tol);
    const double* __restrict__ pp = d.scr1 + o;
    QuotMax qm;
#if MS_BFIN_UNROLL > 0
#pragma unroll kBFinUnroll
#endif
    for (int i = threadIdx.x; i < d.n; i += kBFinThreads) {
      double comb;
      if (f.use_p) {
        comb = pp[i];
      } else {
        comb = __dmul_rn(b0, k0[i]);
        comb = __dadd_rn(comb, __dmul_rn(b1, k1[i]));
        comb = __dadd_rn(comb, __dmul_rn(b2, k2[i]));
      }
      comb = __dadd_rn(comb, __dmul_rn(b3, k3[i]));
      const double xi = x[i];
      const double xt = __dadd_rn(xi, __dmul_rn(h, comb));
      const double xn = xnx[i];
      nf |= !isfinite(xn) || !isfinite(xt) || !isfinite(xst[i]);
      const double w = fmax(fmax(fabs(xi), fabs(xn)), floor_w);
      if (f.quot) qm.add(fabs(__dsub_rn(xn, xt)), w);
      else m = fmax(m, __ddiv_rn(fabs(__dsub_rn(xn, xt)), w));
    }
    if (f.quot) m = qm.value();
  }
  __shared__ double red[kBFinThreads / 32];
  __shared__ int rnf[kBFinThreads / 32];
  __shared__ int last;
  for (int s = 16; s >= 1; s >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, s));
  nf = __any_sync(0xffffffffu, nf);
  if ((threadIdx.x & 31) == 0) {
    red[threadIdx.x >> 5] = m;
    rnf[threadIdx.x >> 5] = nf;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double e = 0.0;
    int anynf = 0;
    for (int w = 0; w < kBFinThreads / 32; ++w) {
      e = fmax(e, red[w]);
      anynf |= rnf[w];
    }
    attempt_controller(c, f.S, FIN_SOLVE, f.k1_elided, 0, dead, stage_nf, anynf != 0, e, nullptr);
  }
  if (f.ctl_smem) {
    __syncthreads();
    ctl_copy(cg, &cs);
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(d.ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  // loop condition: does any trajectory still run?
  __threadfence();
  int any = 0;
  for (int q = threadIdx.x; q < d.B; q += kBFinThreads) any |= reinterpret_cast<volatile const Ctl*>(d.ctl + q)->done == 0;
  any = __syncthreads_or(any);
  if (threadIdx.x == 0) {
    *d.flag = any;
    *d.ticket = 0u;
    if (has_handle) cudaGraphSetConditional(h, any ? 1 : 0);
  }
}

__global__ void kb_stamp(Ctl* ctl, int B) {
  msb::count_launch();
  const uint64_t t = globaltimer_ns();
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < B; b += gridDim.x * blockDim.x) ctl[b].t_start_ns = t;
}

__global__ void kb_loop_head(Ctl* ctl, int B) {
  msb::count_launch();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  Ctl* c = ctl + b;
  if (c->done) return;
  if (c->nf_mask & 1) {
    c->status = MS_NON_FINITE;
    c->done = 1;
    c->nf_mask = 0;
    return;
  }
  c->nf_mask = 0;
  loop_check(c);
}

// initial_step (solver.cpp:420-451) per trajectory: terms in parallel, the
// sums by one thread in ascending order (the oracle's order)
__global__ void __launch_bounds__(256) kb_init_a(BatchDev d) {
  msb::count_launch();
  const int b = blockIdx.x;
  Ctl* c = d.ctl + b;
  if (c->done) return;
  const int64_t o = (int64_t)b * d.n;
  const double* x0 = d.xb[0] + o;
  const double* f0 = d.kb[1] + o;
  __shared__ int nf;
  if (threadIdx.x == 0) nf = 0;
  __syncthreads();
  bool my = false;
  for (int i = threadIdx.x; i < d.n; i += blockDim.x) {
    const double sk = __dadd_rn(c->abs_tol, __dmul_rn(c->rel_tol, fabs(x0[i])));
    const double q0 = __ddiv_rn(x0[i], sk), q1 = __ddiv_rn(f0[i], sk);
    d.scr0[o + i] = __dmul_rn(q0, q0);
    d.scr1[o + i] = __dmul_rn(q1, q1);
    my |= !isfinite(f0[i]);
  }
  if (my) atomicOr(&nf, 1);
  __syncthreads();
  __shared__ double s01[2];
  if (threadIdx.x == 0) s01[0] = seq_sum(d.scr0 + o, d.n);
  if (threadIdx.x == 32) s01[1] = seq_sum(d.scr1 + o, d.n);
  __syncthreads();
  if (threadIdx.x != 0) return;
  c->cap = __ddiv_rn(__dsub_rn(c->tf, c->t0), 10.0);
  if (nf) {
    c->h = nan64();
    c->init_skip2 = 1;
    return;
  }
  const double inv_n = __ddiv_rn(1.0, (double)d.n);
  const double d0 = __dsqrt_rn(__dmul_rn(s01[0], inv_n));
  const double d1 = __dsqrt_rn(__dmul_rn(s01[1], inv_n));
  c->d1 = d1;
  if (d1 < 1e-12) {
    c->h = c->cap;
    c->init_skip2 = 1;
    return;
  }
  c->h1 = (d0 >= 1e-8) ? __ddiv_rn(__dmul_rn(0.01, d0), d1) : 1e-6;
  c->init_skip2 = 0;
}

__global__ void __launch_bounds__(256) kb_init_b(BatchDev d, double exponent) {
  msb::count_launch();
  const int b = blockIdx.x;
  Ctl* c = d.ctl + b;
  if (c->done) return;
  const bool skip2 = c->init_skip2 != 0;
  const int64_t o = (int64_t)b * d.n;
  const double* x0 = d.xb[0] + o;
  const double* f0 = d.kb[1] + o;
  const double* f1 = d.kb[2] + o;
  __shared__ int nf;
  if (threadIdx.x == 0) nf = 0;
  __syncthreads();
  if (!skip2) {
    bool my = false;
    for (int i = threadIdx.x; i < d.n; i += blockDim.x) {
      const double sk = __dadd_rn(c->abs_tol, __dmul_rn(c->rel_tol, fabs(x0[i])));
      const double q2 = __ddiv_rn(__dsub_rn(f1[i], f0[i]), sk);
      d.scr0[o + i] = __dmul_rn(q2, q2);
      my |= !isfinite(f1[i]);
    }
    if (my) atomicOr(&nf, 1);
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  double h0;
  if (skip2) {
    h0 = c->h;
  } else {
    const double h1 = c->h1;
    double h2;
    if (nf) {
      h2 = __dmul_rn(h1, 1e-3);
    } else {
      const double inv_n = __ddiv_rn(1.0, (double)d.n);
      const double d2 = __ddiv_rn(__dsqrt_rn(__dmul_rn(seq_sum(d.scr0 + o, d.n), inv_n)), h1);
      const double der = c->d1 < d2 ? d2 : c->d1;
      h2 = der < 1e-12 ? c->cap : pow_cr(__ddiv_rn(0.01, der), exponent);
    }
    h0 = __dmul_rn(100.0, h1);
    if (h2 < h0) h0 = h2;
    if (c->cap < h0) h0 = c->cap;
  }
  c->h = h0;
  c->init_skip2 = 0;
  if (!isfinite(h0)) {
    c->status = MS_NON_FINITE;
    c->done = 1;
  }
}

}  // namespace

// =====================================================================================
struct ms_batch {
  SysView sv{};
  int B = 0;
  bool tc = false;      // tcgen05 GEMM for binary32 rows
  int op_ks = 0;        // operand format (K's 16-bit format) when tc
  BatchDev d{};
  void* mem = nullptr;
  double* omega = nullptr;
  Ctl* ctl_host = nullptr;
  int* flag_host = nullptr;
  cudaStream_t st = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  TcGemm gemm{};
  std::map<std::string, std::pair<cudaGraph_t, cudaGraphExec_t>> graphs;
  std::mutex mu;
};

namespace {

struct BTableau {
  int S = 4;
  double a[4][4] = {};
  double bt[4] = {7.0 / 24.0, 0.25, 1.0 / 3.0, 0.125};
  BTableau() {
    a[1][0] = 0.5;
    a[2][1] = 0.75;
    a[3][0] = 2.0 / 9.0;
    a[3][1] = 1.0 / 3.0;
    a[3][2] = 4.0 / 9.0;
  }
};
const BTableau kBT;

struct BEval {
  int l = 0, kind = PREP_X, gate = GATE_ALWAYS, count = CNT_NONE, out_slot = SLOT_K1, nterms = 0;
  double coef[kMaxStages] = {};
  int slot[kMaxStages] = {};
  int is_last = 0, round_x = 0;
};

// MS_BFIN_P=off: the finalize combines k1..k4 itself (read per launch; graphs capture it once)
bool bfin_p_enabled() {
  const char* v = std::getenv("MS_BFIN_P");
  return !(v && std::strcmp(v, "off") == 0);
}

// MS_BFIN_EPI=on: the last contraction's epilogue forms the error (read per
// launch; graphs capture it once). Off by default: measured +35 us in that
// contraction's epilogue (four more latency-bound loads per element on 8 warps
// per SM) against -8 us in the finalize (profiles/r2_c5_epi_ab.txt)
bool bfin_epi_enabled() {
  const char* v = std::getenv("MS_BFIN_EPI");
  return v && std::strcmp(v, "on") == 0;
}

template <class FS>
void launch_bprep(ms_batch* m, cudaStream_t st, const BPrepArgs& p, bool gs32) {
  dim3 grid((m->d.n + 255) / 256, m->B);
  if (gs32) BCK(launch_k(kb_prep<FS, float>, grid, 256, 0, st, p));
  else BCK(launch_k(kb_prep<FS, double>, grid, 256, 0, st, p));
}

// the specialised tensor-core stage prep (kb_prep_tc); false = not applicable
template <int OPKS>
bool launch_bprep_tc_ks(ms_batch* m, cudaStream_t st, const BPrepArgs& p) {
  dim3 grid((m->d.n + 256 * kPrepTcElems - 1) / (256 * kPrepTcElems), m->B);
  auto go = [&](auto kern) { BCK(launch_k(kern, grid, 256, 0, st, p)); return true; };
  if (p.is_last) {
    if (p.nterms == 1) return go(kb_prep_tc<OPKS, 1, true>);
    if (p.nterms == 2) return go(kb_prep_tc<OPKS, 2, true>);
    if (p.nterms == 3) return go(kb_prep_tc<OPKS, 3, true>);
  } else {
    if (p.nterms == 1) return go(kb_prep_tc<OPKS, 1, false>);
    if (p.nterms == 2) return go(kb_prep_tc<OPKS, 2, false>);
    if (p.nterms == 3) return go(kb_prep_tc<OPKS, 3, false>);
  }
  return false;
}

bool launch_bprep_tc(ms_batch* m, cudaStream_t st, const BPrepArgs& p) {
  const char* v = std::getenv("MS_PREP_TC");  // read per launch (graphs capture it once)
  const bool on = !(v && std::strcmp(v, "0") == 0);
  if (!on || !MS_TC_PACKED || p.kind != PREP_STAGE || p.count != CNT_STAGE || !p.fs32) return false;
  if (p.op_ks == MS_K_BF16) return launch_bprep_tc_ks<MS_K_BF16>(m, st, p);
  if (p.op_ks == MS_K_F16) return launch_bprep_tc_ks<MS_K_F16>(m, st, p);
  return false;
}

template <class SS, class GS>
void launch_brhs_cc(ms_batch* m, cudaStream_t st, const BRhsArgs& a) {
  dim3 grid((m->d.n + kBT_I - 1) / kBT_I, (m->B + kBT_B - 1) / kBT_B);
  switch (m->sv.ks) {
    case MS_K_F32: BCK(launch_k(kb_rhs_cc<SS, GS, MS_K_F32>, grid, 256, 0, st, a)); break;
    case MS_K_F16: BCK(launch_k(kb_rhs_cc<SS, GS, MS_K_F16>, grid, 256, 0, st, a)); break;
    default: BCK(launch_k(kb_rhs_cc<SS, GS, MS_K_BF16>, grid, 256, 0, st, a)); break;
  }
}

void beval(ms_batch* m, cudaStream_t st, const BEval& e, const ms_stage_prec& sp, cudaEvent_t mid0 = nullptr,
           cudaEvent_t mid1 = nullptr, bool fin = false) {
  const bool fs32 = is32(sp.f_prec), ss32 = is32(sp.sum_prec), gs32 = is32(sp.g_prec);
  const bool use_tc = m->tc && is_sss(sp);
  BPrepArgs p{};
  p.d = m->d;
  p.S = 4;
  p.l = e.l;
  p.kind = e.kind;
  p.gate = e.gate;
  p.count = e.count;
  p.out_slot = e.out_slot;
  p.nterms = e.nterms;
  for (int t = 0; t < kMaxStages; ++t) {
    p.coef[t] = e.coef[t];
    p.slot[t] = e.slot[t];
  }
  p.is_last = e.is_last;
  p.round_x = e.round_x;
  p.ws32 = fs32 && ss32;
  p.fs32 = fs32;
  p.op_ks = use_tc ? m->op_ks : 0;
  // the BS3 last stage combines k1, k2, k3 (slots K1, 1, 2), the first three terms
  // of the finalize's x_tilde sum in its order
  if (e.kind == PREP_STAGE && e.is_last && e.nterms == 3 && e.slot[0] == SLOT_K1 && e.slot[1] == 1 &&
      e.slot[2] == 2 && bfin_p_enabled()) {
    p.write_p = 1;
    for (int t = 0; t < 3; ++t) p.pb[t] = kBT.bt[t];
  }
  if (!(use_tc && launch_bprep_tc(m, st, p))) {
    if (fs32) launch_bprep<float>(m, st, p, gs32);
    else launch_bprep<double>(m, st, p, gs32);
  }
  BCK(cudaGetLastError());
  BRhsArgs a{};
  a.d = m->d;
  a.S = 4;
  a.l = e.l;
  a.gate = e.gate;
  a.out_slot = e.out_slot;
  a.ws32 = p.ws32;
  a.fs32 = p.fs32;
  if (fin) {
    if (!(use_tc && p.write_p)) throw InvalidArg("batch: the folded error estimate needs the tensor-core path and P");
    a.fin = 1;
    a.bt_last = kBT.bt[3];
  }
  if (mid0) BCK(cudaEventRecord(mid0, st));
  if (use_tc) {
    launch_tc_gemm(m->gemm, a, st);
  } else if (ss32) {
    if (gs32) launch_brhs_cc<float, float>(m, st, a);
    else launch_brhs_cc<float, double>(m, st, a);
  } else {
    if (gs32) launch_brhs_cc<double, float>(m, st, a);
    else launch_brhs_cc<double, double>(m, st, a);
  }
  BCK(cudaGetLastError());
  if (mid1) BCK(cudaEventRecord(mid1, st));
}

BEval bstage(int l) {
  BEval e;
  e.l = l;
  e.kind = PREP_STAGE;
  e.count = CNT_STAGE;
  e.out_slot = (l == 3) ? SLOT_KLAST : l;
  e.is_last = l == 3;
  for (int mm = 0; mm < l; ++mm) {
    if (kBT.a[l][mm] == 0.0) continue;
    e.coef[e.nterms] = kBT.a[l][mm];
    e.slot[e.nterms] = mm == 0 ? SLOT_K1 : mm;
    ++e.nterms;
  }
  return e;
}

struct BPlan {
  ms_stage_prec rows[3], k1_row;
  int storage, lowest;
  bool k1_elided;
};

BPlan bplan(const ms_policy& pol) {
  BPlan P{};
  for (int l = 0; l < 3; ++l) P.rows[l] = pol.per_stage[l];
  P.k1_row = pol.first_step_k1;
  P.storage = pol.storage;
  int lowest = pol.storage == MS_BINARY32 ? MS_BINARY32 : MS_BINARY64;
  const ms_stage_prec all[4] = {pol.per_stage[0], pol.per_stage[1], pol.per_stage[2], pol.first_step_k1};
  for (const auto& s : all)
    if (is32(s.f_prec) || is32(s.sum_prec) || is32(s.g_prec)) lowest = MS_BINARY32;
  P.lowest = lowest;
  P.k1_elided = same_row(pol.first_step_k1, pol.per_stage[2]);
  return P;
}

void battempt(ms_batch* m, cudaStream_t st, const BPlan& P, bool has_handle, cudaGraphConditionalHandle h) {
  if (!P.k1_elided) {
    BEval e;
    e.l = 0;
    e.kind = PREP_X;
    e.gate = GATE_NEED_K1;
    e.count = CNT_K1;
    e.out_slot = SLOT_K1;
    beval(m, st, e, P.k1_row);
  }
  // the error estimate in the last contraction's epilogue (MS_BFIN_EPI=off: in the finalize)
  const bool epi = MS_TC_FIN && bfin_epi_enabled() && m->tc && is_sss(P.rows[2]) && bfin_p_enabled();
  for (int l = 1; l < 4; ++l) beval(m, st, bstage(l), P.rows[l - 1], nullptr, nullptr, epi && l == 3);
  BFinArgs f{};
  f.err_epi = epi ? 1 : 0;
  f.d = m->d;
  f.S = 4;
  f.k1_elided = P.k1_elided;
  for (int mm = 0; mm < 4; ++mm) {
    f.bt[f.nbt] = kBT.bt[mm];
    f.bslot_[f.nbt] = mm == 0 ? SLOT_K1 : (mm == 3 ? SLOT_KLAST : mm);
    ++f.nbt;
  }
  if (f.nbt != 4) throw InvalidArg("batch: finalize expects the four BS3(2) error weights");
  f.use_p = bfin_p_enabled() ? 1 : 0;
  f.ctl_smem = ctl_smem_enabled() ? 1 : 0;
  {
    const char* v = std::getenv("MS_BFIN_QUOT");  // read per launch (graphs capture it once)
    f.quot = (v && std::strcmp(v, "off") == 0) ? 0 : 1;
  }
  BCK(launch_k(kb_finalize, m->B, kBFinThreads, 0, st, f, has_handle ? 1 : 0, h));
}

void binit(ms_batch* m, cudaStream_t st, const BPlan& P) {
  kb_stamp<<<(m->B + 255) / 256, 256, 0, st>>>(m->d.ctl, m->B);
  BEval f0;
  f0.l = 7;
  f0.kind = PREP_X;
  f0.count = CNT_DDD;
  f0.out_slot = 1;
  beval(m, st, f0, kDDDb);
  kb_init_a<<<m->B, 256, 0, st>>>(m->d);
  BCK(cudaGetLastError());
  BEval f1 = f0;
  f1.kind = PREP_INIT_X1;
  f1.gate = GATE_INIT2;
  f1.out_slot = 2;
  beval(m, st, f1, kDDDb);
  kb_init_b<<<m->B, 256, 0, st>>>(m->d, 0.25);
  BCK(cudaGetLastError());
  BEval k1;
  k1.l = 0;
  k1.kind = PREP_X;
  k1.count = CNT_K1;
  k1.out_slot = SLOT_K1;
  k1.round_x = P.storage == MS_BINARY32 ? 1 : 0;
  beval(m, st, k1, P.k1_row);
  kb_loop_head<<<(m->B + 255) / 256, 256, 0, st>>>(m->d.ctl, m->B);
  BCK(cudaGetLastError());
}

cudaGraphExec_t bgraph(ms_batch* m, const BPlan& P) {
  char key[96];
  std::snprintf(key, sizeof(key), "%d%d%d:%d%d%d:%d%d%d:%d%d%d:%d", P.rows[0].f_prec, P.rows[0].sum_prec,
                P.rows[0].g_prec, P.rows[1].f_prec, P.rows[1].sum_prec, P.rows[1].g_prec, P.rows[2].f_prec,
                P.rows[2].sum_prec, P.rows[2].g_prec, P.k1_row.f_prec, P.k1_row.sum_prec, P.k1_row.g_prec,
                (int)P.k1_elided);
  auto it = m->graphs.find(key);
  if (it != m->graphs.end()) return it->second.second;
  cudaGraph_t g;
  BCK(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle h;
  BCK(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams cp{};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  BCK(cudaGraphAddNode(&node, g, nullptr, 0, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  BCK(cudaStreamBeginCaptureToGraph(m->st, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  try {
    battempt(m, m->st, P, true, h);
  } catch (...) {
    cudaGraph_t dummy;
    cudaStreamEndCapture(m->st, &dummy);
    throw;
  }
  BCK(cudaStreamEndCapture(m->st, &body));
  cudaGraphExec_t exec;
  BCK(cudaGraphInstantiate(&exec, g, 0));
  m->graphs[key] = {g, exec};
  return exec;
}

void check_prec_b(const ms_stage_prec& sp) {
  if (sp.f_prec > 1 || sp.sum_prec > 1 || sp.g_prec > 1) throw InvalidArg("stage precision: format must be 0 or 1");
}

}  // namespace

extern "C" {

int ms_batch_create(ms_system_t sys, int32_t batch, const double* omega, int32_t tensor_cores, ms_batch_t* out) {
  return bguard([&] {
    if (!sys || !omega || !out || batch < 1) throw InvalidArg("batch_create: bad arguments");
    auto m = std::make_unique<ms_batch>();
    m->sv = sys_view(sys);
    const SysView& v = m->sv;
    if (v.mkind != MD_KUR) throw InvalidArg("batch_create: batched ensembles are Kuramoto systems");
    if (v.ks == MS_K_SCALAR) throw InvalidArg("batch_create: the ensemble shares a dense K");
    if (v.row0 != 0 || v.row1 != v.n) throw InvalidArg("batch_create: needs a handle owning all rows");
    if (tensor_cores && v.ks != MS_K_BF16 && v.ks != MS_K_F16)
      throw InvalidArg("batch_create: tensor cores need K stored in bf16 or f16");
    BCK(cudaSetDevice(v.dev));
    m->B = batch;
    m->tc = tensor_cores != 0;
    m->op_ks = m->tc ? v.ks : 0;
    const int n = v.n, ld = v.ld;
    const size_t bn = (size_t)batch * n;
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    const size_t vec = al(sizeof(double) * bn);
    size_t total = vec /*omega*/ + 2 * vec + (kMaxStages + 1) * vec + 3 * vec /*xn, scr0, scr1*/ +
                   2 * vec /*sc*/ + al(sizeof(uint16_t) * 4 * (size_t)batch * ld) /*op*/ + vec /*fvc*/ + 2 * vec /*rec*/ +
                   al(sizeof(Ctl) * batch) + al(sizeof(int)) + al(sizeof(unsigned long long) * batch) +
                   al(sizeof(int) * batch);
    char* base = nullptr;
    BCK(cudaMalloc(&base, total));
    BCK(cudaMemset(base, 0, total));
    m->mem = base;
    char* p = base;
    auto take = [&](size_t b) {
      char* r = p;
      p += al(b);
      return r;
    };
    BatchDev& d = m->d;
    d.B = batch;
    d.n = n;
    d.ld = ld;
    d.K = v.K;
    d.ks = v.ks;
    m->omega = reinterpret_cast<double*>(take(sizeof(double) * bn));
    d.omega = m->omega;
    for (int i = 0; i < 2; ++i) d.xb[i] = reinterpret_cast<double*>(take(sizeof(double) * bn));
    for (int i = 0; i < kMaxStages + 1; ++i) d.kb[i] = reinterpret_cast<double*>(take(sizeof(double) * bn));
    d.xn = reinterpret_cast<double*>(take(sizeof(double) * bn));
    d.scr0 = reinterpret_cast<double*>(take(sizeof(double) * bn));
    d.scr1 = reinterpret_cast<double*>(take(sizeof(double) * bn));
    d.sc = take(sizeof(double) * 2 * bn);
    d.op = take(sizeof(uint16_t) * 4 * (size_t)batch * ld);
    d.fvc = reinterpret_cast<double*>(take(sizeof(double) * bn));
    d.rec = take(2 * sizeof(double) * bn);
    d.ctl = reinterpret_cast<Ctl*>(take(sizeof(Ctl) * batch));
    d.flag = reinterpret_cast<int*>(take(2 * sizeof(int)));
    d.ticket = reinterpret_cast<unsigned*>(d.flag + 1);
    d.errb = reinterpret_cast<unsigned long long*>(take(sizeof(unsigned long long) * batch));
    d.nfe = reinterpret_cast<int*>(take(sizeof(int) * batch));
    d.mw = 1.0 / n;
    BCK(cudaMemcpy(m->omega, omega, sizeof(double) * bn, cudaMemcpyHostToDevice));
    {  // the records' F: RN32(omega), F of a binary32 row (systems.cpp:136-139; the
       // host cast rounds to nearest); the tensor-core path runs binary32 rows only
#if MS_TC_PACKED == 3
      std::vector<float> r(bn);
      for (size_t e = 0; e < bn; ++e) r[e] = (float)omega[e];
      BCK(cudaMemcpy(d.rec, r.data(), sizeof(float) * bn, cudaMemcpyHostToDevice));
#else
      std::vector<TcRec> r(bn);
      for (size_t e = 0; e < bn; ++e) r[e] = TcRec{0.f, 0.f, (double)(float)omega[e]};
      BCK(cudaMemcpy(d.rec, r.data(), sizeof(TcRec) * bn, cudaMemcpyHostToDevice));
#endif
    }
    BCK(cudaStreamCreateWithFlags(&m->st, cudaStreamNonBlocking));
    BCK(cudaEventCreate(&m->ev0));
    BCK(cudaEventCreate(&m->ev1));
    BCK(cudaMallocHost(&m->ctl_host, sizeof(Ctl) * batch));
    BCK(cudaMallocHost(&m->flag_host, sizeof(int)));
    if (m->tc) tc_gemm_setup(m->gemm, d, v.sms);
    // the zeroing and omega upload ran on the legacy stream; m->st is
    // non-blocking, so finish them before any kernel of the batch can start
    BCK(cudaDeviceSynchronize());
    *out = m.release();
  });
}

int ms_batch_destroy(ms_batch_t m) {
  if (!m) return MS_OK;
  return bguard([&] {
    cudaSetDevice(m->sv.dev);
    for (auto& kv : m->graphs) {
      cudaGraphExecDestroy(kv.second.second);
      cudaGraphDestroy(kv.second.first);
    }
    tc_gemm_teardown(m->gemm);
    if (m->mem) cudaFree(m->mem);
    if (m->ctl_host) cudaFreeHost(m->ctl_host);
    if (m->flag_host) cudaFreeHost(m->flag_host);
    if (m->ev0) cudaEventDestroy(m->ev0);
    if (m->ev1) cudaEventDestroy(m->ev1);
    if (m->st) cudaStreamDestroy(m->st);
    delete m;
  });
}

int ms_batch_eval_rhs(ms_batch_t m, const double* x, ms_stage_prec sp, double* out) {
  return bguard([&] {
    if (!m || !x || !out) throw InvalidArg("batch_eval_rhs: null argument");
    check_prec_b(sp);
    std::lock_guard<std::mutex> lk(m->mu);
    BCK(cudaSetDevice(m->sv.dev));
    const size_t bn = (size_t)m->B * m->d.n;
    std::memset(m->ctl_host, 0, sizeof(Ctl) * m->B);
    BCK(cudaMemcpyAsync(m->d.ctl, m->ctl_host, sizeof(Ctl) * m->B, cudaMemcpyHostToDevice, m->st));
    BCK(cudaMemcpyAsync(m->d.xb[0], x, sizeof(double) * bn, cudaMemcpyHostToDevice, m->st));
    BEval e;
    e.l = 0;
    e.kind = PREP_X;
    e.out_slot = 0;
    beval(m, m->st, e, sp);
    BCK(cudaMemcpyAsync(out, m->d.kb[0], sizeof(double) * bn, cudaMemcpyDeviceToHost, m->st));
    BCK(cudaStreamSynchronize(m->st));
  });
}

int ms_batch_profile_rhs(ms_batch_t m, const double* x, ms_stage_prec sp, int iters, double* rhs_ms,
                         double* prep_ms) {
  return bguard([&] {
    if (!m || !x || iters < 1) throw InvalidArg("batch_profile_rhs: bad arguments");
    check_prec_b(sp);
    std::lock_guard<std::mutex> lk(m->mu);
    BCK(cudaSetDevice(m->sv.dev));
    const size_t bn = (size_t)m->B * m->d.n;
    std::memset(m->ctl_host, 0, sizeof(Ctl) * m->B);
    BCK(cudaMemcpyAsync(m->d.ctl, m->ctl_host, sizeof(Ctl) * m->B, cudaMemcpyHostToDevice, m->st));
    BCK(cudaMemcpyAsync(m->d.xb[0], x, sizeof(double) * bn, cudaMemcpyHostToDevice, m->st));
    BEval e;
    e.l = 0;
    e.kind = PREP_X;
    e.out_slot = 0;
    beval(m, m->st, e, sp);
    std::vector<cudaEvent_t> ev(3 * (size_t)iters);
    for (auto& v : ev) BCK(cudaEventCreate(&v));
    for (int i = 0; i < iters; ++i) {
      BCK(cudaEventRecord(ev[3 * i], m->st));
      beval(m, m->st, e, sp, ev[3 * i + 1], ev[3 * i + 2]);
    }
    BCK(cudaStreamSynchronize(m->st));
    double tr = 0, tp = 0;
    for (int i = 0; i < iters; ++i) {
      float a = 0, b = 0;
      BCK(cudaEventElapsedTime(&a, ev[3 * i], ev[3 * i + 1]));
      BCK(cudaEventElapsedTime(&b, ev[3 * i + 1], ev[3 * i + 2]));
      tp += a;
      tr += b;
    }
    for (auto& v : ev) cudaEventDestroy(v);
    if (rhs_ms) *rhs_ms = tr / iters;
    if (prep_ms) *prep_ms = tp / iters;
  });
}

int ms_batch_solve(ms_batch_t m, const double* x0, double t0, double tf, const ms_policy* pol,
                   const ms_solver_config* cfg, ms_batch_result* res) {
  return bguard([&] {
    if (!m || !x0 || !pol || !cfg || !res) throw InvalidArg("batch_solve: null argument");
    for (int l = 0; l < 3; ++l) check_prec_b(pol->per_stage[l]);
    check_prec_b(pol->first_step_k1);
    if (!(cfg->abs_tol > 0.0 && cfg->abs_tol <= cfg->rel_tol && cfg->rel_tol < 1.0))
      throw InvalidArg("solver: need 0 < abs_tol <= rel_tol < 1");
    if (!(cfg->fac_min < 1.0 && cfg->fac_max > 1.0)) throw InvalidArg("solver: need fac_min < 1 < fac_max");
    if (!(tf > t0)) throw InvalidArg("solver: need t_final > t0");
    if (cfg->record_snapshots) throw InvalidArg("batch_solve: snapshots are recorded by ms_solve only");
    std::lock_guard<std::mutex> lk(m->mu);
    BCK(cudaSetDevice(m->sv.dev));
    const BPlan P = bplan(*pol);
    const int B = m->B;
    const size_t bn = (size_t)B * m->d.n;
    for (int b = 0; b < B; ++b) {
      Ctl& c = m->ctl_host[b];
      std::memset(&c, 0, sizeof(Ctl));
      c.t = t0;
      c.t0 = t0;
      c.tf = tf;
      c.h_min = cfg->h_min_factor * (P.lowest == MS_BINARY32 ? 0x1p-23 : 0x1p-52);
      c.rel_tol = cfg->rel_tol;
      c.abs_tol = cfg->abs_tol;
      c.safety = cfg->safety;
      c.fac_min = cfg->fac_min;
      c.fac_max = cfg->fac_max;
      c.ctrl_exp = cfg->controller_exponent;
      c.wall_clock_limit = cfg->wall_clock_limit;
      c.slow_elapsed = cfg->slow_solver_elapsed;
      c.slow_progress = cfg->slow_solver_progress;
      c.max_iterations = cfg->max_iterations;
      c.max_failed = cfg->max_failed_steps;
      c.store32 = P.storage == MS_BINARY32 ? 1 : 0;
      c.time_limits = cfg->time_limits_enabled ? 1 : 0;
      c.record_log = 0;
      c.status = MS_COMPLETED;
    }
    cudaStream_t st = m->st;
    BCK(cudaMemcpyAsync(m->d.ctl, m->ctl_host, sizeof(Ctl) * B, cudaMemcpyHostToDevice, st));
    BCK(cudaMemcpyAsync(m->d.xb[0], x0, sizeof(double) * bn, cudaMemcpyHostToDevice, st));
    const bool host_loop = getenv("MS_LOOP") && std::string(getenv("MS_LOOP")) == "host";
    cudaGraphExec_t exec = host_loop ? nullptr : bgraph(m, P);
    BCK(cudaEventRecord(m->ev0, st));
    binit(m, st, P);
    int64_t attempts = 0;
    if (host_loop) {
      for (;;) {
        battempt(m, st, P, false, 0);
        ++attempts;
        BCK(cudaMemcpyAsync(m->flag_host, m->d.flag, sizeof(int), cudaMemcpyDeviceToHost, st));
        BCK(cudaStreamSynchronize(st));
        if (!*m->flag_host) break;
      }
    } else {
      BCK(cudaGraphLaunch(exec, st));
    }
    BCK(cudaEventRecord(m->ev1, st));
    BCK(cudaMemcpyAsync(m->ctl_host, m->d.ctl, sizeof(Ctl) * B, cudaMemcpyDeviceToHost, st));
    BCK(cudaStreamSynchronize(st));
    float ms = 0.f;
    BCK(cudaEventElapsedTime(&ms, m->ev0, m->ev1));
    if (res->final_state) {
      // each trajectory's x lives in xb[ix_b]
      std::vector<double> tmp;
      const int n = m->d.n;
      for (int w = 0; w < 2; ++w) {
        bool any = false;
        for (int b = 0; b < B; ++b) any |= m->ctl_host[b].ix == w;
        if (!any) continue;
        tmp.resize(bn);
        BCK(cudaMemcpyAsync(tmp.data(), m->d.xb[w], sizeof(double) * bn, cudaMemcpyDeviceToHost, st));
        BCK(cudaStreamSynchronize(st));
        for (int b = 0; b < B; ++b)
          if (m->ctl_host[b].ix == w)
            std::memcpy(res->final_state + (size_t)b * n, tmp.data() + (size_t)b * n, sizeof(double) * n);
      }
    }
    int64_t max_att = 0;
    for (int b = 0; b < B; ++b) {
      const Ctl& c = m->ctl_host[b];
      if (res->status) res->status[b] = c.status;
      if (res->t_reached) res->t_reached[b] = c.t;
      if (res->n_accepted) res->n_accepted[b] = c.n_acc;
      if (res->n_failed) res->n_failed[b] = c.n_fail;
      if (res->rhs_evals) {
        int64_t ev = c.evals_ddd + c.evals_k1;
        for (int l = 1; l < 4; ++l) ev += c.evals_stage[l];
        res->rhs_evals[b] = ev;
      }
      max_att = std::max<int64_t>(max_att, c.attempts);
    }
    res->attempts = host_loop ? attempts : max_att;
    res->device_ms = ms;
  });
}

}  // extern "C"
