// ms_api.cu — system handles, the device-resident adaptive loop and the C-ABI
// of include/mixedstep_b200.h.
//
// The solve (solver.cpp:226-347) runs as: stamp -> initial_step (2 binary64
// evaluations + norms) -> cold k1 -> loop head -> one CUDA graph whose single
// WHILE conditional node holds one attempt [k1 recompute] -> (prep, rhs) per
// stage -> finalize. finalize's last block runs the controller and sets the
// conditional, so the step loop never returns to the host; the host sees the
// result only after the graph completes.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#define MS_DEFINE_STEP_KERNELS 1
#include "ms_dispatch.h"
#include "ms_multi.cuh"
#include "ms_internal.h"

using namespace msb;

namespace {

thread_local std::string g_err;

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct InvalidArg : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};

#define CK(call)                                                                                  \
  do {                                                                                            \
    cudaError_t e_ = (call);                                                                      \
    if (e_ != cudaSuccess)                                                                        \
      throw CudaError(std::string(#call) + ": " + cudaGetErrorString(e_) + " (" __FILE__ ":" + \
                      std::to_string(__LINE__) + ")");                                            \
  } while (0)

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

// ---- tableaus (solver.cpp:15-68), literal doubles as written there ----------
struct Tableau {
  int S;
  double a[kMaxStages][kMaxStages];
  double b_tilde[kMaxStages];
  int order_high;
  int scheme_flops;  // scheme_flops_per_component (solver.cpp:361-384)
};

Tableau make_bs32() {
  Tableau t{};
  t.S = 4;
  t.a[1][0] = 0.5;
  t.a[2][1] = 0.75;
  t.a[3][0] = 2.0 / 9.0;
  t.a[3][1] = 1.0 / 3.0;
  t.a[3][2] = 4.0 / 9.0;
  const double bt[4] = {7.0 / 24.0, 0.25, 1.0 / 3.0, 0.125};
  for (int i = 0; i < 4; ++i) t.b_tilde[i] = bt[i];
  t.order_high = 3;
  return t;
}

Tableau make_dp54() {
  Tableau t{};
  t.S = 7;
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
  const double bt[7] = {5179.0 / 57600.0, 0.0, 7571.0 / 16695.0, 393.0 / 640.0, -92097.0 / 339200.0,
                        187.0 / 2100.0, 1.0 / 40.0};
  for (int i = 0; i < 7; ++i) t.b_tilde[i] = bt[i];
  t.order_high = 5;
  return t;
}

int scheme_flops(const Tableau& t) {
  int flops = 0;
  for (int l = 1; l < t.S; ++l) {
    int nz = 0;
    for (int m = 0; m < l; ++m) nz += t.a[l][m] != 0.0;
    flops += 2 * nz + 1;
  }
  int nz = 0;
  for (int l = 0; l < t.S; ++l) nz += t.b_tilde[l] != 0.0;
  return flops + 2 * nz + 1 + 8;
}

const Tableau& bs32() {
  static const Tableau t = [] {
    Tableau x = make_bs32();
    x.scheme_flops = scheme_flops(x);
    return x;
  }();
  return t;
}
const Tableau& dp54() {
  static const Tableau t = [] {
    Tableau x = make_dp54();
    x.scheme_flops = scheme_flops(x);
    return x;
  }();
  return t;
}

bool sp_eq(const ms_stage_prec& a, const ms_stage_prec& b) {
  return a.f_prec == b.f_prec && a.sum_prec == b.sum_prec && a.g_prec == b.g_prec;
}
const ms_stage_prec kDDD{MS_BINARY64, MS_BINARY64, MS_BINARY64, 0};

// ---- seeded inputs: SplitMix64 (rng.hpp:13-52) ---------------------------------
struct SplitMix64 {
  uint64_t state;
  double cached = 0.0;
  bool has_cached = false;
  SplitMix64(uint64_t seed, uint64_t stream) : state(seed + stream * 0xD1342543DE82EF95ull) {}
  uint64_t next() {
    uint64_t z = (state += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  double uniform01() { return static_cast<double>(next() >> 11) * 0x1p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform01(); }
  double normal() {
    if (has_cached) {
      has_cached = false;
      return cached;
    }
    double u1 = uniform01();
    if (u1 <= 0.0) u1 = 0x1p-53;
    const double u2 = uniform01();
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double a = 6.283185307179586476925286766559 * u2;
    cached = r * std::sin(a);
    has_cached = true;
    return r * std::cos(a);
  }
};

// ---- device helper kernels ----------------------------------------------------
__device__ __forceinline__ uint64_t splitmix_at(uint64_t state0, uint64_t q) {
  // the q-th output (0-based) of SplitMix64: the Weyl state advances first
  uint64_t z = state0 + (q + 1) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

template <int KS> __device__ __forceinline__ typename KElem<KS>::T to_k(double v);
template <> __device__ __forceinline__ float to_k<MS_K_F32>(double v) { return __double2float_rn(v); }
template <> __device__ __forceinline__ __half to_k<MS_K_F16>(double v) { return __double2half(v); }
template <> __device__ __forceinline__ __nv_bfloat16 to_k<MS_K_BF16>(double v) { return __double2bfloat16(v); }

template <int KS>
__global__ void k_fill_uniform(typename KElem<KS>::T* K, int n, int row0, int rows, int64_t ld, uint64_t state0,
                               double lo, double hi) {
  msb::count_launch();
  const int64_t total = (int64_t)rows * n;
  const double span = __dsub_rn(hi, lo);
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = q / n, j = q % n;
    const uint64_t draw = (uint64_t)(row0 + r) * (uint64_t)n + (uint64_t)j;
    const double u = (double)(splitmix_at(state0, draw) >> 11) * 0x1p-53;
    K[r * ld + j] = to_k<KS>(__dadd_rn(lo, __dmul_rn(span, u)));
  }
}

template <int KS, class SRC>
__global__ void k_convert_rows(typename KElem<KS>::T* K, const SRC* src, int n, int rows, int64_t ld) {
  msb::count_launch();
  const int64_t total = (int64_t)rows * n;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = q / n, j = q % n;
    K[r * ld + j] = to_k<KS>((double)src[q]);
  }
}

// any nonzero |K| below kPkMinK (a product could then be subnormal, where the
// packed FTZ multiply of the split sweeps would flush it)
template <int KS>
__global__ void k_scan_tiny(const typename KElem<KS>::T* K, int n, int rows, int64_t ld, int* flag) {
  msb::count_launch();
  const int64_t total = (int64_t)rows * n;
  bool tiny = false;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
    const float v = fabsf(k2f(K[(q / n) * ld + q % n]));
    tiny |= v != 0.f && v < kPkMinK;
  }
  if (__any_sync(0xffffffffu, tiny) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

template <int KS>
__global__ void k_get_rows(const typename KElem<KS>::T* K, double* dst, int n, int rows, int64_t ld) {
  msb::count_launch();
  const int64_t total = (int64_t)rows * n;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = q / n, j = q % n;
    dst[q] = (double)k2f(K[r * ld + j]);
  }
}

__global__ void k_estimate_error(int64_t n, const double* a, const double* b, const double* c, double ab, double rel,
                                 double* out) {
  msb::count_launch();
  // estimate_error, solver.cpp:399-411 (max is order-independent)
  __shared__ double red[32];
  // the max without a division per element (QuotMax, bitwise the per-element
  // fmax of the rounded quotients: also the unit-level test of the device
  // finalizes' reduction, tests/test_gpu_solver.py)
  const double floor_w = __ddiv_rn(ab, rel);
  QuotMax qm;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double w = fmax(fmax(fabs(a[i]), fabs(b[i])), floor_w);
    qm.add(fabs(__dsub_rn(b[i], c[i])), w);
  }
  double m = qm.value();
  for (int o = 16; o >= 1; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double r = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) r = fmax(r, red[w]);
    *out = r;
  }
}

__global__ void k_adjust_step(double h, double err, double rel, double safety, double fmin, double fmax_,
                              double ex, double* out) {
  msb::count_launch();
  *out = d_adjust_step(h, err, rel, safety, fmin, fmax_, ex);
}

// prep instantiations
template <int MODEL>
void launch_prep_model(bool fs32, bool gs32, int grid, cudaStream_t st, const PrepArgs& p) {
  if (fs32) {
    if (gs32) CK(launch_k(k_prep<MODEL, float, float>, grid, 256, 0, st, p));
    else CK(launch_k(k_prep<MODEL, float, double>, grid, 256, 0, st, p));
  } else {
    if (gs32) CK(launch_k(k_prep<MODEL, double, float>, grid, 256, 0, st, p));
    else CK(launch_k(k_prep<MODEL, double, double>, grid, 256, 0, st, p));
  }
}

}  // namespace

struct SolvePlanStore;
// =====================================================================================
struct ms_system {
  int model = 0;      // MS_MODEL_*
  int mkind = 0;      // MD_* (or the fixture id)
  bool fixture = false;
  int n = 0, d = 0, cs = 0, ld = 0;
  int row0 = 0, row1 = 0;
  int ks = MS_K_SCALAR, rhs_mode = MS_RHS_FAST;
  int k_tiny = 0;     // some nonzero |K| < 2^-80: the packed FTZ sweep path is off (ms_common.cuh mac2)
  int dev = 0, sms = kNumSMsDefault;
  cudaStream_t stream = nullptr;
  void* K = nullptr;
  std::vector<void*> dev_arrays;
  ModelDev md{};
  int64_t flop_theta[3] = {0, 0, 0};
  // workspace
  bool ws_ready = false;
  void* ws_mem = nullptr;
  Bufs B{};
  int fin_blocks = 1, fin_threads = kFinThreads;
  int64_t log_cap = 0;
  Ctl* ctl_host = nullptr;  // pinned mirror
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  struct GraphEntry {
    cudaGraph_t g = nullptr;
    cudaGraphExec_t exec = nullptr;
  };
  std::map<std::string, GraphEntry> graphs;
  std::mutex mu;
  // StepSnapshot buffer: (snap_cap + 1) rows of dN, then snap_cap step sizes
  double* snap = nullptr;
  double* snap_h = nullptr;
  int64_t snap_cap = -1;
  // dense output: device copy of the output times, then n_eval x dN rows
  double* dense = nullptr;
  double* dense_t = nullptr;
  int64_t dense_cap = -1;
  // f16-K tensor-core sweep resources (ms_gemv_tc.cuh GvRes) or null
  void* gv = nullptr;
  // push exchange of the row-sharded loop (ms_loop_push_*): peers' workspaces
  // and mailbox slots; mem = this handle's mailbox [8] + epoch [1]
  struct PushState {
    int world = 1, rank = 0, np = 0;
    char* peer_ws[kMaxPeers] = {};
    unsigned long long* peer_slot[kMaxPeers] = {};
    int peer_rank[kMaxPeers] = {};
    unsigned long long* mem = nullptr;
    const void* ws_at_setup = nullptr;  // the workspace the peers were told about
  } push;
  // host-driven (sharded) loop
  bool loop_active = false;
  SolvePlanStore* loop_plan = nullptr;

  int64_t dn() const { return (int64_t)n * d; }
};

// the Kuramoto sin/cos split: the column data are (s_j, c_j) pairs
bool split_of(const ms_system* s) {
  return s->mkind == MD_KUR && (s->rhs_mode == MS_RHS_FAST || s->rhs_mode == MS_RHS_ORDERED);
}


namespace {

void set_device(ms_system* s) { CK(cudaSetDevice(s->dev)); }

double* upload_array(ms_system* s, const double* host, int n) {
  if (!host) return nullptr;
  double* d = nullptr;
  CK(cudaMalloc(&d, sizeof(double) * n));
  s->dev_arrays.push_back(d);
  CK(cudaMemcpy(d, host, sizeof(double) * n, cudaMemcpyHostToDevice));
  return d;
}

size_t kelem_bytes(int ks) { return ks == MS_K_F32 ? 4 : 2; }

size_t al256(size_t b) { return (b + 255) & ~size_t(255); }

// bytes of one solve workspace (Bufs) with a step log of log_cap records
size_t bufs_bytes(const ms_system* s, int64_t log_cap) {
  const int64_t dn = s->dn();
  const int fin_blocks = (int)std::max<int64_t>(1, std::min<int64_t>((dn + kFinThreads - 1) / kFinThreads, 2 * s->sms));
  const size_t vec = al256(sizeof(double) * dn);
  size_t total = 0;
  total += 2 * vec;                                      // xb
  total += (kMaxStages + 1) * vec;                       // kb
  total += 3 * vec;                                      // xn, xt, scratch
  total += 2 * al256(sizeof(double) * 2 * s->ld);        // gin, gin2
  total += 2 * al256((size_t)(s->ld / 64 + 1) * 512);     // op16, op16b
  total += al256(sizeof(double) * s->ld);                // rowc
  total += al256(sizeof(double) * s->n);                 // fvc
  total += al256(sizeof(double) * fin_blocks);           // part
  total += al256(sizeof(StepLogRec) * std::max<int64_t>(log_cap, 1));
  total += al256(sizeof(Ctl));
  return total;
}

void carve_bufs(const ms_system* s, char* base, int64_t log_cap, Bufs& B) {
  const int64_t dn = s->dn();
  const int fin_blocks = (int)std::max<int64_t>(1, std::min<int64_t>((dn + kFinThreads - 1) / kFinThreads, 2 * s->sms));
  char* p = base;
  auto take = [&](size_t b) {
    char* r = p;
    p += al256(b);
    return r;
  };
  for (int i = 0; i < 2; ++i) B.xb[i] = reinterpret_cast<double*>(take(sizeof(double) * dn));
  for (int i = 0; i < kMaxStages + 1; ++i) B.kb[i] = reinterpret_cast<double*>(take(sizeof(double) * dn));
  B.xn = reinterpret_cast<double*>(take(sizeof(double) * dn));
  B.xt = reinterpret_cast<double*>(take(sizeof(double) * dn));
  B.scratch = reinterpret_cast<double*>(take(sizeof(double) * dn));
  B.gin = take(sizeof(double) * 2 * s->ld);
  B.gin2 = take(sizeof(double) * 2 * s->ld);
  B.op16 = take((size_t)(s->ld / 64 + 1) * 512);
  B.op16b = take((size_t)(s->ld / 64 + 1) * 512);
  if (!s->gv) B.op16 = B.op16b = nullptr;  // written by the preps only for the tensor-core sweep
  B.rowc = take(sizeof(double) * s->ld);
  B.fvc = reinterpret_cast<double*>(take(sizeof(double) * s->n));
  B.part = reinterpret_cast<double*>(take(sizeof(double) * fin_blocks));
  B.log = reinterpret_cast<StepLogRec*>(take(sizeof(StepLogRec) * std::max<int64_t>(log_cap, 1)));
  B.ctl = reinterpret_cast<Ctl*>(take(sizeof(Ctl)));
}

void ensure_workspace(ms_system* s, int64_t log_cap) {
  if (s->ws_ready && log_cap <= s->log_cap) return;
  if (s->ws_ready) {
    // grow only the log: reallocate the whole workspace (rare)
    for (auto& kv : s->graphs) {
      if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
      if (kv.second.g) cudaGraphDestroy(kv.second.g);
    }
    s->graphs.clear();
    CK(cudaStreamSynchronize(s->stream));
    CK(cudaFree(s->ws_mem));
    s->ws_ready = false;
  }
  s->fin_blocks = (int)std::min<int64_t>((s->dn() + kFinThreads - 1) / kFinThreads, 2 * s->sms);
  if (s->fin_blocks < 1) s->fin_blocks = 1;
  s->fin_threads = kFinThreads;
  if (s->dn() <= kFinSmallMax) {
    s->fin_blocks = 1;
    s->fin_threads = kFinSmallThreads;
  }
  const size_t total = bufs_bytes(s, log_cap);
  char* base = nullptr;
  CK(cudaMalloc(&base, total));
  // zero on the system's own (non-blocking) stream: a legacy-stream memset
  // is not ordered before kernels on s->stream and can land after them
  CK(cudaMemsetAsync(base, 0, total, s->stream));
  s->ws_mem = base;
  carve_bufs(s, base, log_cap, s->B);
  s->log_cap = std::max<int64_t>(log_cap, 1);
  if (!s->ctl_host) CK(cudaMallocHost(&s->ctl_host, sizeof(Ctl)));
  s->ws_ready = true;
}

// ---- one RHS evaluation: prep + coupling sweep ---------------------------------
struct EvalSpec {
  int l = 0;
  int kind = PREP_X;
  int gate = GATE_ALWAYS;
  int count = CNT_NONE;
  int out_slot = SLOT_K1;
  int nterms = 0;
  double coef[kMaxStages] = {};
  int slot[kMaxStages] = {};
  int is_last = 0;
  int round_x = 0;
  int S = 4;
  const double* xsrc = nullptr;
};

// prep of one evaluation into workspace B; false when the model has no
// coupling sweep (the reference's scalar test fixtures)
PrepArgs prep_args(ms_system* s, const Bufs& B, const EvalSpec& e, const ms_stage_prec& sp) {
  const bool fs32 = is32(sp.f_prec), ss32 = is32(sp.sum_prec);
  PrepArgs p{};
  p.md = s->md;
  p.B = B;
  p.S = e.S;
  p.l = e.l;
  p.kind = e.kind;
  p.gate = e.gate;
  p.count = e.count;
  p.out_slot = e.out_slot;
  p.nterms = e.nterms;
  for (int i = 0; i < kMaxStages; ++i) {
    p.coef[i] = e.coef[i];
    p.slot[i] = e.slot[i];
  }
  p.is_last = e.is_last;
  p.round_x = e.round_x;
  p.split = split_of(s) ? 1 : 0;
  p.ws32 = (fs32 && ss32) ? 1 : 0;
  p.fs32 = fs32 ? 1 : 0;
  p.ld = s->ld;
  p.xsrc = e.xsrc;
  return p;
}

bool launch_prep(ms_system* s, cudaStream_t st, const PrepArgs& p, const ms_stage_prec& sp) {
  const bool fs32 = is32(sp.f_prec), gs32 = is32(sp.g_prec);
  const int pgrid = (int)std::max<int64_t>(1, std::min<int64_t>((s->n + 255) / 256, 4 * s->sms));
  if (s->fixture) {
    launch_prep_model<-1>(fs32, gs32, pgrid, st, p);
    CK(cudaGetLastError());
    return false;
  }
  switch (s->mkind) {
    case MD_LCO: launch_prep_model<MD_LCO>(fs32, gs32, pgrid, st, p); break;
    case MD_KUR: launch_prep_model<MD_KUR>(fs32, gs32, pgrid, st, p); break;
    default: launch_prep_model<MD_CC>(fs32, gs32, pgrid, st, p); break;
  }
  CK(cudaGetLastError());
  return true;
}

bool launch_prep(ms_system* s, const Bufs& B, cudaStream_t st, const EvalSpec& e, const ms_stage_prec& sp) {
  return launch_prep(s, st, prep_args(s, B, e, sp), sp);
}

bool env_is(const char* name, const char* value) {
  const char* v = std::getenv(name);
  return v && std::strcmp(v, value) == 0;
}

// K beyond ~3/4 of the 126 MB L2 cannot stay resident between evaluations:
// the sweeps stream it with an evict-first policy
int k_stream_of(const ms_system* s) {
  const int64_t kbytes = (int64_t)(s->row1 - s->row0) * s->ld * (s->ks == MS_K_F32 ? 4 : 2);
  return (s->ks != MS_K_SCALAR && kbytes > ((int64_t)96 << 20)) ? 1 : 0;
}

RhsArgs rhs_args(ms_system* s, const Bufs& B, const EvalSpec& e, const ms_stage_prec& sp) {
  RhsArgs a{};
  a.ctl = B.ctl;
  a.nf_mask = &B.ctl->nf_mask;
  a.l = e.l;
  a.gate = e.gate;
  a.S = e.S;
  a.out_slot = e.out_slot;
  a.K = s->K;
  a.ld = s->ld;
  a.n = s->n;
  a.row0 = s->row0;
  a.row1 = s->row1;
  a.gin = B.gin;
  a.rowc = B.rowc;
  a.fvc = B.fvc;
  for (int i = 0; i < kMaxStages + 1; ++i) a.kb[i] = B.kb[i];
  a.d = s->d;
  a.cs = s->cs;
  a.mw = s->md.m[s->cs];
  a.coupling_k = s->md.coupling_k;
  a.ws32 = (is32(sp.f_prec) && is32(sp.sum_prec)) ? 1 : 0;
  a.k_stream = k_stream_of(s);
  a.pk = env_is("MS_SWEEP_PK", "off") ? 0 : 1;
  a.tc16 = s->gv;
  a.op16 = B.op16;
  if (s->push.np && s->loop_active) {
    a.push.ws = static_cast<const char*>(s->ws_mem);
    a.push.np = s->push.np;
    for (int q = 0; q < s->push.np; ++q) a.push.peer[q] = s->push.peer_ws[q];
  }
  return a;
}

void launch_sweep(ms_system* s, cudaStream_t st, const RhsArgs& a, const ms_stage_prec& sp) {
  const bool split = split_of(s);
  RhsLaunch L{s->mkind, split, is32(sp.sum_prec), is32(sp.g_prec), s->ks, s->sms, st};
  if (s->rhs_mode == MS_RHS_FAST) launch_rhs_fast(L, a);
  else launch_rhs_faithful(L, a);
  CK(cudaGetLastError());
}

// PrepArgs of one evaluation (what launch_prep hands to k_prep)
PrepArgs prep_args(ms_system* s, const Bufs& B, const EvalSpec& e, const ms_stage_prec& sp);

void launch_eval(ms_system* s, const Bufs& B, cudaStream_t st, const EvalSpec& e, const ms_stage_prec& sp,
                 cudaEvent_t mid0 = nullptr, cudaEvent_t mid1 = nullptr) {
  // small systems: prep fused into the sweep (whole, unsharded handles only:
  // the fused kernel preps just the rows it sweeps)
  if (!mid0 && !s->fixture && s->rhs_mode == MS_RHS_FAST && s->row0 == 0 && s->row1 == s->n) {
    const bool split = s->mkind == MD_KUR;
    RhsLaunch L{s->mkind, split, is32(sp.sum_prec), is32(sp.g_prec), s->ks, s->sms, st};
    if (launch_eval_fused(L, prep_args(s, B, e, sp), rhs_args(s, B, e, sp), is32(sp.f_prec))) return;
  }
  if (!launch_prep(s, B, st, e, sp)) return;
  const RhsArgs a = rhs_args(s, B, e, sp);
  if (mid0) CK(cudaEventRecord(mid0, st));
  const bool split = s->mkind == MD_KUR && s->rhs_mode == MS_RHS_FAST;  // fast-mode sweeps only
  RhsLaunch L{s->mkind, split, is32(sp.sum_prec), is32(sp.g_prec), s->ks, s->sms, st};
  if (!(split && launch_sweep_small(L, prep_args(s, B, e, sp), a))) launch_sweep(s, st, a, sp);
  if (mid1) CK(cudaEventRecord(mid1, st));
}

void launch_eval(ms_system* s, cudaStream_t st, const EvalSpec& e, const ms_stage_prec& sp,
                 cudaEvent_t mid0 = nullptr, cudaEvent_t mid1 = nullptr) {
  launch_eval(s, s->B, st, e, sp, mid0, mid1);
}

// one evaluation of the row-sharded loop: the finiteness scan of the previous
// stage's gathered vector (scan, all rows; NULL = none) runs inside the prep,
// and the sweep, not the prep, counts the evaluation, so an evaluation the scan
// cancels is not counted (the separate-scan order of the one-GPU loop)
void launch_scan(ms_system* s, cudaStream_t st, const double* buf, int l);

void launch_eval_loop(ms_system* s, cudaStream_t st, const EvalSpec& e, const ms_stage_prec& sp, const double* scan,
                      int scan_bit) {
  PrepArgs p = prep_args(s, s->B, e, sp);
  // MS_LOOP_SCAN=separate: the unfolded order (a scan launch before the
  // evaluation, the prep counting) -- the A/B check of the folded one
  const char* ls = std::getenv("MS_LOOP_SCAN");
  if (s->fixture || (ls && std::strcmp(ls, "separate") == 0)) {  // fixtures: no sweep to count in
    if (scan) launch_scan(s, st, scan, scan_bit);
    if (launch_prep(s, st, p, sp)) launch_sweep(s, st, rhs_args(s, s->B, e, sp), sp);
    return;
  }
  p.scan = scan;
  p.scan_n = scan ? s->dn() : 0;
  p.scan_bit = scan_bit;
  p.count = CNT_NONE;
  if (!launch_prep(s, st, p, sp)) return;
  RhsArgs a = rhs_args(s, s->B, e, sp);
  a.count_ctl = s->B.ctl;
  a.count = e.count;
  launch_sweep(s, st, a, sp);
}

// stage l of an attempt (rk_step, solver.cpp:130-154)
EvalSpec stage_spec(const Tableau& T, int l) {
  EvalSpec e;
  e.S = T.S;
  e.l = l;
  e.kind = PREP_STAGE;
  e.count = CNT_STAGE;
  e.out_slot = (l == T.S - 1) ? SLOT_KLAST : l;
  e.is_last = (l == T.S - 1) ? 1 : 0;
  for (int m = 0; m < l; ++m) {
    if (T.a[l][m] == 0.0) continue;
    e.coef[e.nterms] = T.a[l][m];
    e.slot[e.nterms] = (m == 0) ? SLOT_K1 : m;
    ++e.nterms;
  }
  return e;
}

}  // namespace
// MS_CTL_SMEM=off: the controller works on Ctl in global memory (read per launch)
bool msb::ctl_smem_enabled() {
  const char* v = std::getenv("MS_CTL_SMEM");
  return !(v && std::strcmp(v, "off") == 0);
}
namespace {
FinArgs fin_args(ms_system* s, const Bufs& B, const Tableau& T, int mode, int k1_elided) {
  FinArgs f{};
  f.B = B;
  f.S = T.S;
  for (int m = 0; m < T.S; ++m) {
    if (T.b_tilde[m] == 0.0) continue;
    f.bt[f.nbt] = T.b_tilde[m];
    f.bslot[f.nbt] = (m == 0) ? SLOT_K1 : (m == T.S - 1 ? SLOT_KLAST : m);
    ++f.nbt;
  }
  f.dn = s->dn();
  f.mode = mode;
  f.k1_elided = k1_elided;
  f.write_xt = mode == FIN_STEP ? 1 : 0;
  f.ctl_smem = ctl_smem_enabled() ? 1 : 0;
  return f;
}

struct SolvePlan {
  const Tableau* T;
  ms_stage_prec rows[kMaxStages];  // rows[l-1] for stage l
  ms_stage_prec k1_row;
  int storage;
  int lowest;
  bool k1_elided;
  bool snaps;  // record StepSnapshots (k_snapshot after each finalize)
  bool dense;  // dense output (k_dense after each finalize)
};

int snap_grid(const ms_system* s) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((s->dn() + 255) / 256, 2 * s->sms));
}

// snapshot rows for `cap` accepted steps; the loop graphs capture the buffer
// address, so growing it drops them
void ensure_snapshots(ms_system* s, int64_t cap) {
  if (cap <= s->snap_cap) return;
  CK(cudaStreamSynchronize(s->stream));
  for (auto& kv : s->graphs) {
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
    if (kv.second.g) cudaGraphDestroy(kv.second.g);
  }
  s->graphs.clear();
  if (s->snap) CK(cudaFree(s->snap));
  s->snap = nullptr;
  s->snap_cap = -1;
  const size_t bytes = sizeof(double) * ((size_t)(cap + 1) * (size_t)s->dn() + (size_t)cap);
  CK(cudaMalloc(&s->snap, bytes));
  s->snap_h = s->snap + (size_t)(cap + 1) * (size_t)s->dn();
  s->snap_cap = cap;
}

// dense-output rows for n output times (graphs capture the address: growing drops them)
void ensure_dense(ms_system* s, int64_t n) {
  if (n <= s->dense_cap) return;
  CK(cudaStreamSynchronize(s->stream));
  for (auto& kv : s->graphs) {
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
    if (kv.second.g) cudaGraphDestroy(kv.second.g);
  }
  s->graphs.clear();
  if (s->dense) CK(cudaFree(s->dense));
  s->dense = nullptr;
  s->dense_cap = -1;
  CK(cudaMalloc(&s->dense, sizeof(double) * ((size_t)n * (size_t)s->dn() + (size_t)n)));
  s->dense_t = s->dense + (size_t)n * (size_t)s->dn();
  s->dense_cap = n;
}

// one attempt: [k1 recompute] -> stages -> finalize
// Stage l of an attempt (BS3/DP5 stage spec e on row sp). prepped: its prep
// already ran at the end of the previous sweep, into gin_now. With a next
// stage (en, spn) whose prep can be folded into this sweep (fuse_next_ok),
// the sweep runs it into the other column buffer; returns whether it did
// (gin_now then names that buffer). The counters stay those of k_prep + sweep:
// a folded prep does not count, the sweep of its stage does.
bool launch_stage(ms_system* s, cudaStream_t st, const EvalSpec& e, const ms_stage_prec& sp, bool prepped,
                  void*& gin_now, const EvalSpec* en, const ms_stage_prec* spn) {
  Bufs B = s->B;
  B.gin = gin_now;
  B.op16 = gin_now == s->B.gin ? s->B.op16 : s->B.op16b;  // the operand image travels with its column buffer
  const bool split = s->mkind == MD_KUR && s->rhs_mode == MS_RHS_FAST;
  RhsLaunch L{s->mkind, split, is32(sp.sum_prec), is32(sp.g_prec), s->ks, s->sms, st};
  L.tc16 = split && is32(sp.sum_prec) && is32(sp.g_prec) && tc16_selected(rhs_args(s, B, e, sp), s->ks);
  const bool whole = s->row0 == 0 && s->row1 == s->n;
  const bool can = en && whole && !s->fixture && split && fuse_next_ok(L, is32(spn->f_prec), is32(spn->g_prec));
  if (!prepped && !can) {
    launch_eval(s, B, st, e, sp);
    return false;
  }
  if (!prepped && !launch_prep(s, B, st, e, sp)) return false;
  RhsArgs a = rhs_args(s, B, e, sp);
  if (prepped) {
    a.count_ctl = B.ctl;
    a.count = e.count;
  }
  PrepArgs pn{};
  bool fused = false;
  void* other = gin_now == s->B.gin ? s->B.gin2 : s->B.gin;
  if (can) {
    Bufs B2 = s->B;
    B2.gin = other;
    B2.op16 = other == s->B.gin ? s->B.op16 : s->B.op16b;
    pn = prep_args(s, B2, *en, *spn);
    L.next = &pn;
    L.next_fs32 = is32(spn->f_prec);
    L.next_gs32 = is32(spn->g_prec);
    L.fused = &fused;
  }
  launch_rhs_fast(L, a);
  CK(cudaGetLastError());
  if (fused) gin_now = other;
  return fused;
}

void launch_attempt(ms_system* s, cudaStream_t st, const SolvePlan& P, bool has_handle,
                    cudaGraphConditionalHandle h) {
  const Tableau& T = *P.T;
  if (!P.k1_elided) {
    EvalSpec e;
    e.S = T.S;
    e.l = 0;
    e.kind = PREP_X;
    e.gate = GATE_NEED_K1;
    e.count = CNT_K1;
    e.out_slot = SLOT_K1;
    launch_eval(s, st, e, P.k1_row);
  }
  void* gin_now = s->B.gin;
  bool prepped = false;
  for (int l = 1; l < T.S; ++l) {
    const EvalSpec e = stage_spec(T, l);
    if (l + 1 < T.S) {
      const EvalSpec en = stage_spec(T, l + 1);
      prepped = launch_stage(s, st, e, P.rows[l - 1], prepped, gin_now, &en, &P.rows[l]);
    } else {
      launch_stage(s, st, e, P.rows[l - 1], prepped, gin_now, nullptr, nullptr);
    }
  }
  FinArgs f = fin_args(s, s->B, T, FIN_SOLVE, P.k1_elided ? 1 : 0);
  f.has_handle = has_handle ? 1 : 0;
  f.handle = h;
  CK(launch_k(k_finalize, s->fin_blocks, s->fin_threads, 0, st, f));
  CK(cudaGetLastError());
  if (P.snaps) {
    CK(launch_k(k_snapshot, snap_grid(s), 256, 0, st, s->B, s->snap, s->snap_h, s->snap_cap, s->dn(), 0));
    CK(cudaGetLastError());
  }
  if (P.dense) {
    CK(launch_k(k_dense, snap_grid(s), 256, 0, st, s->B, T.S, s->dense, s->dn(), 0, 0));
    CK(cudaGetLastError());
  }
}

// initial_step + cold k1 + loop head (solver.cpp:247-269)
void launch_init(ms_system* s, cudaStream_t st, const SolvePlan& P, bool with_k1) {
  const Tableau& T = *P.T;
  CK(launch_k(k_stamp_start, 1, 1, 0, st, s->B.ctl));
  EvalSpec f0;
  f0.S = T.S;
  f0.l = 7;
  f0.kind = PREP_X;
  f0.count = CNT_DDD;
  f0.out_slot = 1;
  launch_eval(s, st, f0, kDDD);
  InitArgs ia{};
  ia.B = s->B;
  ia.x0 = s->B.xb[0];
  ia.dn = s->dn();
  ia.exponent = 1.0 / static_cast<double>(T.order_high + 1);
  CK(launch_k(k_init_a, 1, 1024, 0, st, ia));
  CK(cudaGetLastError());
  EvalSpec f1 = f0;
  f1.kind = PREP_INIT_X1;
  f1.gate = GATE_INIT2;
  f1.out_slot = 2;
  launch_eval(s, st, f1, kDDD);
  CK(launch_k(k_init_b, 1, 1024, 0, st, ia));
  CK(cudaGetLastError());
  if (!with_k1) return;
  EvalSpec k1;
  k1.S = T.S;
  k1.l = 0;
  k1.kind = PREP_X;
  k1.count = CNT_K1;
  k1.out_slot = SLOT_K1;
  k1.round_x = P.storage == MS_BINARY32 ? 1 : 0;
  launch_eval(s, st, k1, P.k1_row);
  CK(launch_k(k_loop_head, 1, 1, 0, st, s->B.ctl));
  CK(cudaGetLastError());
}

void validate_cfg(const ms_solver_config& c, double t0, double tf) {  // solver.cpp:217-224
  if (!(c.abs_tol > 0.0 && c.abs_tol <= c.rel_tol && c.rel_tol < 1.0))
    throw InvalidArg("solver: need 0 < abs_tol <= rel_tol < 1");
  if (!(c.fac_min < 1.0 && c.fac_max > 1.0)) throw InvalidArg("solver: need fac_min < 1 < fac_max");
  if (!(tf > t0)) throw InvalidArg("solver: need t_final > t0");
}

void init_ctl(ms_system* s, Ctl& c, const ms_solver_config& cfg, double t0, double tf, const SolvePlan& P,
              int64_t log_cap) {
  std::memset(&c, 0, sizeof(Ctl));
  c.t = t0;
  c.t0 = t0;
  c.tf = tf;
  c.h_min = cfg.h_min_factor * (P.lowest == MS_BINARY32 ? 0x1p-23 : 0x1p-52);
  c.rel_tol = cfg.rel_tol;
  c.abs_tol = cfg.abs_tol;
  c.safety = cfg.safety;
  c.fac_min = cfg.fac_min;
  c.fac_max = cfg.fac_max;
  c.ctrl_exp = cfg.controller_exponent;
  c.wall_clock_limit = cfg.wall_clock_limit;
  c.slow_elapsed = cfg.slow_solver_elapsed;
  c.slow_progress = cfg.slow_solver_progress;
  c.max_iterations = cfg.max_iterations;
  c.max_failed = cfg.max_failed_steps;
  c.log_capacity = log_cap;
  c.store32 = P.storage == MS_BINARY32 ? 1 : 0;
  c.pk_off = s->k_tiny;
  c.time_limits = cfg.time_limits_enabled ? 1 : 0;
  c.record_log = cfg.record_step_log ? 1 : 0;
  c.snap_on = P.snaps ? 1 : 0;
  c.status = MS_COMPLETED;
  (void)s;
}

std::string plan_key(const SolvePlan& P) {
  char buf[160];
  int o = std::snprintf(buf, sizeof(buf), "S%d:st%d:el%d:sn%d:dn%d:k1%d%d%d", P.T->S, P.storage, (int)P.k1_elided,
                        (int)P.snaps, (int)P.dense,
                        P.k1_row.f_prec, P.k1_row.sum_prec, P.k1_row.g_prec);
  for (int l = 0; l < P.T->S - 1; ++l)
    o += std::snprintf(buf + o, sizeof(buf) - o, ":%d%d%d", P.rows[l].f_prec, P.rows[l].sum_prec, P.rows[l].g_prec);
  return std::string(buf);
}

bool use_host_loop() {
  const char* v = std::getenv("MS_LOOP");
  return v && std::strcmp(v, "host") == 0;
}

cudaGraphExec_t get_loop_graph(ms_system* s, const SolvePlan& P) {
  const std::string key = plan_key(P);
  auto it = s->graphs.find(key);
  if (it != s->graphs.end()) return it->second.exec;
  ms_system::GraphEntry ge;
  CK(cudaGraphCreate(&ge.g, 0));
  cudaGraphConditionalHandle handle;
  CK(cudaGraphConditionalHandleCreate(&handle, ge.g, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams cp{};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = handle;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  CK(cudaGraphAddNode(&node, ge.g, nullptr, 0, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  CK(cudaStreamBeginCaptureToGraph(s->stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  try {
    launch_attempt(s, s->stream, P, true, handle);
  } catch (...) {
    cudaGraph_t dummy;
    cudaStreamEndCapture(s->stream, &dummy);
    throw;
  }
  CK(cudaStreamEndCapture(s->stream, &body));
  CK(cudaGraphInstantiate(&ge.exec, ge.g, 0));
  s->graphs[key] = ge;
  return ge.exec;
}

void tally(ms_system* s, const Ctl& c, const SolvePlan& P, int64_t out[3]) {
  // FlopTally (solver.cpp:70-82) from the per-row evaluation counts
  const int64_t n = s->n;
  int64_t low = 0, high = 0, evals = 0;
  auto add = [&](const ms_stage_prec& sp, int64_t cnt) {
    if (cnt <= 0) return;
    (is32(sp.f_prec) ? low : high) += s->flop_theta[0] * n * cnt;
    (is32(sp.g_prec) ? low : high) += s->flop_theta[1] * n * n * cnt;
    (is32(sp.sum_prec) ? low : high) += s->flop_theta[2] * n * n * cnt;
    evals += cnt;
  };
  add(kDDD, c.evals_ddd);
  add(P.k1_row, c.evals_k1);
  for (int l = 1; l < P.T->S; ++l) add(P.rows[l - 1], c.evals_stage[l]);
  high += (int64_t)P.T->scheme_flops * s->dn() * (c.n_acc + c.n_fail);
  out[0] = evals;
  out[1] = low;
  out[2] = high;
}

void run_solve(ms_system* s, const double* x0, bool x0_dev, double t0, double tf, const SolvePlan& P0,
               const ms_solver_config& cfg, ms_solve_result* res, cudaStream_t user_stream, bool out_dev) {
  validate_cfg(cfg, t0, tf);
  std::lock_guard<std::mutex> lk(s->mu);
  set_device(s);
  const int64_t cap = (cfg.record_step_log && res->step_log) ? std::max<int64_t>(res->step_log_capacity, 1) : 1;
  ensure_workspace(s, cap);
  SolvePlan P = P0;
  P.snaps = cfg.record_snapshots && res->snapshots && res->snapshot_h && res->snapshot_capacity >= 0;
  if (P.snaps) ensure_snapshots(s, std::max<int64_t>(res->snapshot_capacity, 1));
  P.dense = res->t_eval && res->y_eval && res->n_eval > 0;
  int64_t dense0 = 0;  // output times at or before t0
  if (P.dense) {
    for (int64_t q = 0; q < res->n_eval; ++q) {
      const double tq = res->t_eval[q];
      if (!(tq >= t0 && tq <= tf) || (q > 0 && tq < res->t_eval[q - 1]))
        throw InvalidArg("solve: t_eval must be sorted within [t0, t_final]");
      if (tq <= t0) dense0 = q + 1;
    }
    ensure_dense(s, res->n_eval);
  }
  cudaStream_t st = s->stream;
  if (user_stream && user_stream != st) {
    // order the solve after the caller's prior work on its stream
    cudaEvent_t e;
    CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    CK(cudaEventRecord(e, user_stream));
    CK(cudaStreamWaitEvent(st, e, 0));
    CK(cudaEventDestroy(e));
  }
  Ctl& c = *s->ctl_host;
  init_ctl(s, c, cfg, t0, tf, P, cap);
  const int64_t dn = s->dn();
  if (P.dense) {
    CK(cudaMemcpyAsync(s->dense_t, res->t_eval, sizeof(double) * res->n_eval, cudaMemcpyHostToDevice, st));
    c.t_eval = s->dense_t;
    c.n_eval = res->n_eval;
    c.eval_next = dense0;
  }
  CK(cudaMemcpyAsync(s->B.ctl, &c, sizeof(Ctl), cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(s->B.xb[0], x0, sizeof(double) * dn, x0_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                     st));
  const bool host_loop = use_host_loop();
  cudaGraphExec_t exec = host_loop ? nullptr : get_loop_graph(s, P);
  CK(cudaEventRecord(s->ev0, st));
  launch_init(s, st, P, true);
  if (P.snaps) {
    CK(launch_k(k_snapshot, snap_grid(s), 256, 0, st, s->B, s->snap, s->snap_h, s->snap_cap, dn, 1));
    CK(cudaGetLastError());
  }
  if (P.dense && dense0 > 0) {
    CK(launch_k(k_dense, snap_grid(s), 256, 0, st, s->B, P.T->S, s->dense, dn, 1, dense0));
    CK(cudaGetLastError());
  }
  if (host_loop) {
    for (;;) {
      launch_attempt(s, st, P, false, 0);
      CK(cudaMemcpyAsync(&c.done, &s->B.ctl->done, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      if (c.done) break;
    }
  } else {
    CK(cudaGraphLaunch(exec, st));
  }
  CK(cudaEventRecord(s->ev1, st));
  CK(cudaMemcpyAsync(&c, s->B.ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, s->ev0, s->ev1));
  if (res->final_state) {
    CK(cudaMemcpyAsync(res->final_state, s->B.xb[c.ix], sizeof(double) * dn,
                       out_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
  }
  res->step_log_count = c.record_log ? c.log_count : 0;
  if (res->step_log && c.record_log) {
    const int64_t m = std::min<int64_t>(res->step_log_capacity, c.log_count);
    if (m > 0) {
      std::vector<StepLogRec> tmp((size_t)m);
      CK(cudaMemcpyAsync(tmp.data(), s->B.log, sizeof(StepLogRec) * m, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      for (int64_t i = 0; i < m; ++i) {
        res->step_log[i].t = tmp[(size_t)i].t;
        res->step_log[i].h = tmp[(size_t)i].h;
        res->step_log[i].err = tmp[(size_t)i].err;
        res->step_log[i].accepted = tmp[(size_t)i].accepted;
      }
    }
  }
  res->n_eval_done = P.dense ? c.eval_next : 0;
  if (P.dense && c.eval_next > 0)
    CK(cudaMemcpyAsync(res->y_eval, s->dense, sizeof(double) * (size_t)c.eval_next * (size_t)dn,
                       out_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
  res->snapshot_count = P.snaps ? c.n_acc : 0;
  if (P.snaps) {
    const int64_t m = std::min<int64_t>(res->snapshot_capacity, c.n_acc);
    CK(cudaMemcpyAsync(res->snapshots, s->snap, sizeof(double) * (size_t)(m + 1) * (size_t)dn,
                       out_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
    if (m > 0)
      CK(cudaMemcpyAsync(res->snapshot_h, s->snap_h, sizeof(double) * (size_t)m,
                         out_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
  }
  CK(cudaStreamSynchronize(st));
  if (user_stream && user_stream != st) {
    cudaEvent_t e;
    CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    CK(cudaEventRecord(e, st));
    CK(cudaStreamWaitEvent(user_stream, e, 0));
    CK(cudaEventDestroy(e));
  }
  res->status = c.status;
  res->t_reached = c.t;
  res->n_accepted = c.n_acc;
  res->n_failed = c.n_fail;
  int64_t tl[3];
  tally(s, c, P, tl);
  res->rhs_evals = tl[0];
  res->flops_low = tl[1];
  res->flops_high = tl[2];
  res->device_ms = ms;
}

SolvePlan plan_bs32(const ms_policy& pol) {
  SolvePlan P{};
  P.T = &bs32();
  for (int l = 0; l < 3; ++l) P.rows[l] = pol.per_stage[l];
  P.k1_row = pol.first_step_k1;
  P.storage = pol.storage;
  // PrecisionPolicy::lowest_format (precision.cpp:9-20)
  int lowest = MS_BINARY64;
  if (pol.storage == MS_BINARY32) lowest = MS_BINARY32;
  const ms_stage_prec all[4] = {pol.per_stage[0], pol.per_stage[1], pol.per_stage[2], pol.first_step_k1};
  for (const auto& sp : all)
    if (is32(sp.f_prec) || is32(sp.sum_prec) || is32(sp.g_prec)) lowest = MS_BINARY32;
  P.lowest = lowest;
  // The k1 recomputed after a rejection (solver.cpp:298-306) evaluates the
  // same autonomous field at the same x as the stored k1; when the k1 row equals
  // the last stage's row the stored value is bit-identical, so the launch is
  // elided (and still counted).
  P.k1_elided = sp_eq(pol.first_step_k1, pol.per_stage[2]);
  return P;
}

SolvePlan plan_dp54() {
  SolvePlan P{};
  P.T = &dp54();
  for (int l = 0; l < 6; ++l) P.rows[l] = kDDD;
  P.k1_row = kDDD;
  P.storage = MS_BINARY64;
  P.lowest = MS_BINARY64;
  P.k1_elided = true;
  return P;
}

}  // namespace

struct SolvePlanStore {
  SolvePlan P;
  ms_solver_config cfg;
  int64_t log_cap;
};

namespace {

cudaStream_t pick_stream(ms_system* s, void* stream) {
  return stream ? static_cast<cudaStream_t>(stream) : s->stream;
}

PushSig push_sig(const ms_system* s) {
  PushSig g{};
  g.mbox = s->push.mem;
  g.epoch = s->push.mem + 8;
  g.np = s->push.np;
  for (int q = 0; q < s->push.np; ++q) {
    g.peer_slot[q] = s->push.peer_slot[q];
    g.peer_rank[q] = s->push.peer_rank[q];
  }
  return g;
}

void set_exch(ms_system* s, ms_exchange* ex, double* buf) {
  if (!ex) return;
  ex->needed = 1;
  ex->buf = buf;
  ex->offset = (int64_t)s->row0 * s->d;
  ex->count = (int64_t)(s->row1 - s->row0) * s->d;
  ex->total = s->dn();
}

void launch_scan(ms_system* s, cudaStream_t st, const double* buf, int l) {
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((s->dn() + 255) / 256, 2 * s->sms));
  k_nf_scan<<<grid, 256, 0, st>>>(s->B.ctl, buf, s->dn(), l);
  CK(cudaGetLastError());
}

// segment lists of the host-driven loop (ms_loop_* in the header)
int loop_segments(const SolvePlan& P, int list) {
  if (list == 0) return 4;
  return (P.k1_elided ? 0 : 1) + (P.T->S - 1) + 1;
}

void loop_run(ms_system* s, const SolvePlan& P, int list, int index, cudaStream_t st, ms_exchange* ex) {
  const Tableau& T = *P.T;
  if (ex) std::memset(ex, 0, sizeof(*ex));
  const int S = T.S;
  if (list == 0) {
    InitArgs ia{};
    ia.B = s->B;
    ia.x0 = s->B.xb[0];
    ia.dn = s->dn();
    ia.exponent = 1.0 / static_cast<double>(T.order_high + 1);
    EvalSpec f;
    f.S = S;
    f.l = 7;
    f.kind = PREP_X;
    f.count = CNT_DDD;
    switch (index) {
      case 0:
        CK(launch_k(k_stamp_start, 1, 1, 0, st, s->B.ctl));
        f.out_slot = 1;
        launch_eval(s, st, f, kDDD);
        set_exch(s, ex, s->B.kb[1]);
        return;
      case 1:
        launch_scan(s, st, s->B.kb[1], 7);
        CK(launch_k(k_init_a, 1, 1024, 0, st, ia));
        CK(cudaGetLastError());
        f.kind = PREP_INIT_X1;
        f.gate = GATE_INIT2;
        f.out_slot = 2;
        launch_eval(s, st, f, kDDD);
        set_exch(s, ex, s->B.kb[2]);
        return;
      case 2: {
        CK(launch_k(k_init_b, 1, 1024, 0, st, ia));
        CK(cudaGetLastError());
        EvalSpec k1;
        k1.S = S;
        k1.l = 0;
        k1.kind = PREP_X;
        k1.count = CNT_K1;
        k1.out_slot = 0;
        k1.round_x = P.storage == MS_BINARY32 ? 1 : 0;
        launch_eval(s, st, k1, P.k1_row);
        set_exch(s, ex, s->B.kb[0]);
        return;
      }
      case 3:
        launch_scan(s, st, s->B.kb[0], 0);
        CK(launch_k(k_loop_head, 1, 1, 0, st, s->B.ctl));
        CK(cudaGetLastError());
        return;
      default: throw InvalidArg("loop: bad init segment");
    }
  }
  int idx = index;
  if (!P.k1_elided) {
    if (idx == 0) {
      EvalSpec e;
      e.S = S;
      e.l = 0;
      e.kind = PREP_X;
      e.gate = GATE_NEED_K1;
      e.count = CNT_K1;
      e.out_slot = 0;
      launch_eval(s, st, e, P.k1_row);
      set_exch(s, ex, s->B.kb[0]);
      return;
    }
    --idx;
  }
  // k1 stays in slot 0 (k1i == 0 throughout), the last stage writes slot S
  auto out_of = [&](int l) { return l == S - 1 ? s->B.kb[S] : s->B.kb[l]; };
  const int l = idx + 1;
  if (l < S) {
    if (l > 1) launch_eval_loop(s, st, stage_spec(T, l), P.rows[l - 1], out_of(l - 1), l - 1);
    else launch_eval_loop(s, st, stage_spec(T, l), P.rows[l - 1], P.k1_elided ? nullptr : s->B.kb[0], 0);
    set_exch(s, ex, out_of(l));
    return;
  }
  if (l != S) throw InvalidArg("loop: bad attempt segment");
  // no scan of the gathered last stage: a non-finite element of it makes
  // x_tilde non-finite (b~_S != 0), and the finalize's any_nf takes the same
  // reject branch as stage_nf would
  const char* ls = std::getenv("MS_LOOP_SCAN");
  if (T.b_tilde[S - 1] == 0.0 || s->fixture || (ls && std::strcmp(ls, "separate") == 0))
    launch_scan(s, st, out_of(S - 1), S - 1);
  FinArgs f = fin_args(s, s->B, T, FIN_SOLVE, P.k1_elided ? 1 : 0);
  f.fixed_k1 = 1;
  CK(launch_k(k_finalize, s->fin_blocks, s->fin_threads, 0, st, f));
  CK(cudaGetLastError());
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((s->dn() + 255) / 256, 2 * s->sms));
  k_fsal_copy<<<grid, 256, 0, st>>>(s->B.ctl, s->B.kb[0], s->B.kb[S], s->dn());
  CK(cudaGetLastError());
}


void check_prec(const ms_stage_prec& sp) {
  if (sp.f_prec > 1 || sp.sum_prec > 1 || sp.g_prec > 1) throw InvalidArg("stage precision: format must be 0 or 1");
}
void check_policy(const ms_policy& p) {
  for (int l = 0; l < 3; ++l) check_prec(p.per_stage[l]);
  check_prec(p.first_step_k1);
  if (p.storage > 1) throw InvalidArg("policy: bad storage format");
}

}  // namespace


// =====================================================================================
// Concurrent policy variants: up to four solves of one system
// (the harness's Single/Mixed1/Mixed2/Double, harness.cpp:113-121) advanced in
// lock-step attempts, each lane with its own workspace and controller. Every
// stage is the lanes' preps followed by ONE K sweep (k_rhs_multi) when the
// model is the split Kuramoto over a stored K; otherwise by the lanes' own
// sweeps back to back. A lane that finishes stops launching work of its own.

namespace {

bool use_multi_sweep(const ms_system* s) {
  const char* v = std::getenv("MS_MULTI");
  if (v && std::strcmp(v, "off") == 0) return false;
  return !s->fixture && s->mkind == MD_KUR && s->rhs_mode == MS_RHS_FAST && s->ks != MS_K_SCALAR;
}

struct LaneCtls {
  Ctl* c[kMaxLanes];
};

// loop condition over the lanes (the WHILE node of the variants graph)
__global__ void k_lanes_cond(LaneCtls L, int nl, int* flag, int has_handle, cudaGraphConditionalHandle h) {
  msb::count_launch();
  int any = 0;
  for (int v = 0; v < nl; ++v) any |= L.c[v]->done == 0;
  *flag = any;
  if (has_handle) cudaGraphSetConditional(h, any ? 1 : 0);
}

}  // namespace

struct ms_variants {
  ms_system* s = nullptr;
  int nl = 0;
  char* mem = nullptr;
  int64_t log_cap = 0;
  Bufs B[kMaxLanes];
  Ctl* ctl_host = nullptr;  // pinned [kMaxLanes]
  int* flag = nullptr;      // device: any lane still running
  int* flag_host = nullptr;
  std::map<std::string, ms_system::GraphEntry> graphs;
  std::mutex mu;
};

namespace {

void drop_graphs(ms_variants* v) {
  for (auto& kv : v->graphs) {
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
    if (kv.second.g) cudaGraphDestroy(kv.second.g);
  }
  v->graphs.clear();
}

void variants_workspace(ms_variants* v, int64_t log_cap) {
  ms_system* s = v->s;
  if (v->mem && log_cap <= v->log_cap) return;
  CK(cudaStreamSynchronize(s->stream));
  drop_graphs(v);
  if (v->mem) CK(cudaFree(v->mem));
  v->mem = nullptr;
  const size_t one = bufs_bytes(s, log_cap);
  CK(cudaMalloc(&v->mem, one * v->nl + 256));
  CK(cudaMemsetAsync(v->mem, 0, one * v->nl + 256, s->stream));
  for (int l = 0; l < v->nl; ++l) carve_bufs(s, v->mem + one * l, log_cap, v->B[l]);
  v->flag = reinterpret_cast<int*>(v->mem + one * v->nl);
  v->log_cap = log_cap;
}

// one evaluation of every participating lane: preps, then the shared sweep
void mlaunch_eval(ms_variants* v, cudaStream_t st, const EvalSpec* e, const ms_stage_prec* sp, const bool* on) {
  ms_system* s = v->s;
  bool sweep = false;
  for (int l = 0; l < v->nl; ++l)
    if (on[l]) sweep |= launch_prep(s, v->B[l], st, e[l], sp[l]);
  if (!sweep) return;
  // participating lanes sorted by (SS, GS): (f32,f32) | (f64,f32) | (f64,f64)
  int order[kMaxLanes], cnt[3] = {0, 0, 0}, np = 0;
  bool fusable = use_multi_sweep(s);
  for (int pass = 0; pass < 3; ++pass)
    for (int l = 0; l < v->nl; ++l) {
      if (!on[l]) continue;
      const bool ss64 = !is32(sp[l].sum_prec), gs64 = !is32(sp[l].g_prec);
      const int ty = !ss64 ? (gs64 ? -1 : 0) : (gs64 ? 2 : 1);
      if (ty < 0) fusable = false;  // (f32 sum, f64 G): no fused kernel
      if (ty == pass) {
        order[np++] = l;
        ++cnt[pass];
      }
    }
  if (fusable && np >= 2) {
    MultiArgs m{};
    m.nl = np;
    m.l = e[order[0]].l;
    m.gate = e[order[0]].gate;
    m.S = e[order[0]].S;
    m.out_slot = e[order[0]].out_slot;
    m.ld = s->ld;
    m.n = s->n;
    m.row0 = s->row0;
    m.row1 = s->row1;
    m.mw = s->md.m[s->cs];
    m.k_stream = k_stream_of(s);
    for (int i = 0; i < np; ++i) {
      const int l = order[i];
      LaneArgs& L = m.lane[i];
      L.ctl = v->B[l].ctl;
      L.nf_mask = &v->B[l].ctl->nf_mask;
      L.gin = v->B[l].gin;
      L.fvc = v->B[l].fvc;
      for (int j = 0; j < kMaxStages + 1; ++j) L.kb[j] = v->B[l].kb[j];
      L.ws32 = (is32(sp[l].f_prec) && is32(sp[l].sum_prec)) ? 1 : 0;
    }
    launch_rhs_multi(m, cnt[0], cnt[1], cnt[2], s->ks, s->K, s->sms, st);
    CK(cudaGetLastError());
  } else {
    for (int l = 0; l < v->nl; ++l)
      if (on[l]) launch_sweep(s, st, rhs_args(s, v->B[l], e[l], sp[l]), sp[l]);
  }
}

// initial_step + cold k1 of every lane (launch_init, lane-parallel)
void mlaunch_init(ms_variants* v, cudaStream_t st, const SolvePlan* P) {
  ms_system* s = v->s;
  const Tableau& T = *P[0].T;
  const int nl = v->nl;
  bool on[kMaxLanes] = {};
  EvalSpec e[kMaxLanes];
  ms_stage_prec sp[kMaxLanes];
  for (int l = 0; l < nl; ++l) {
    on[l] = true;
    CK(launch_k(k_stamp_start, 1, 1, 0, st, v->B[l].ctl));
    e[l].S = T.S;
    e[l].l = 7;
    e[l].kind = PREP_X;
    e[l].count = CNT_DDD;
    e[l].out_slot = 1;
    sp[l] = kDDD;
  }
  mlaunch_eval(v, st, e, sp, on);
  InitArgs ia[kMaxLanes];
  for (int l = 0; l < nl; ++l) {
    ia[l] = InitArgs{};
    ia[l].B = v->B[l];
    ia[l].x0 = v->B[l].xb[0];
    ia[l].dn = s->dn();
    ia[l].exponent = 1.0 / static_cast<double>(T.order_high + 1);
    CK(launch_k(k_init_a, 1, 1024, 0, st, ia[l]));
    CK(cudaGetLastError());
    e[l].kind = PREP_INIT_X1;
    e[l].gate = GATE_INIT2;
    e[l].out_slot = 2;
  }
  mlaunch_eval(v, st, e, sp, on);
  for (int l = 0; l < nl; ++l) {
    CK(launch_k(k_init_b, 1, 1024, 0, st, ia[l]));
    CK(cudaGetLastError());
    e[l] = EvalSpec{};
    e[l].S = T.S;
    e[l].l = 0;
    e[l].kind = PREP_X;
    e[l].count = CNT_K1;
    e[l].out_slot = SLOT_K1;
    e[l].round_x = P[l].storage == MS_BINARY32 ? 1 : 0;
    sp[l] = P[l].k1_row;
  }
  mlaunch_eval(v, st, e, sp, on);
  for (int l = 0; l < nl; ++l) CK(launch_k(k_loop_head, 1, 1, 0, st, v->B[l].ctl));
  CK(cudaGetLastError());
}

// one lock-step attempt of every lane (launch_attempt, lane-parallel)
void mlaunch_attempt(ms_variants* v, cudaStream_t st, const SolvePlan* P, bool has_handle,
                     cudaGraphConditionalHandle h) {
  ms_system* s = v->s;
  const Tableau& T = *P[0].T;
  const int nl = v->nl;
  bool on[kMaxLanes] = {};
  EvalSpec e[kMaxLanes];
  ms_stage_prec sp[kMaxLanes];
  bool any_k1 = false;
  for (int l = 0; l < nl; ++l) {
    on[l] = !P[l].k1_elided;
    any_k1 |= on[l];
    e[l].S = T.S;
    e[l].l = 0;
    e[l].kind = PREP_X;
    e[l].gate = GATE_NEED_K1;
    e[l].count = CNT_K1;
    e[l].out_slot = SLOT_K1;
    sp[l] = P[l].k1_row;
  }
  if (any_k1) mlaunch_eval(v, st, e, sp, on);
  for (int st_l = 1; st_l < T.S; ++st_l) {
    for (int l = 0; l < nl; ++l) {
      on[l] = true;
      e[l] = stage_spec(T, st_l);
      sp[l] = P[l].rows[st_l - 1];
    }
    mlaunch_eval(v, st, e, sp, on);
  }
  LaneCtls lc{};
  for (int l = 0; l < nl; ++l) {
    FinArgs f = fin_args(s, v->B[l], T, FIN_SOLVE, P[l].k1_elided ? 1 : 0);
    f.has_handle = 0;
    CK(launch_k(k_finalize, s->fin_blocks, s->fin_threads, 0, st, f));
    CK(cudaGetLastError());
    lc.c[l] = v->B[l].ctl;
  }
  k_lanes_cond<<<1, 1, 0, st>>>(lc, nl, v->flag, has_handle ? 1 : 0, h);
  CK(cudaGetLastError());
}

cudaGraphExec_t variants_graph(ms_variants* v, const SolvePlan* P) {
  std::string key;
  for (int l = 0; l < v->nl; ++l) key += plan_key(P[l]) + "|";
  auto it = v->graphs.find(key);
  if (it != v->graphs.end()) return it->second.exec;
  ms_system* s = v->s;
  ms_system::GraphEntry ge;
  CK(cudaGraphCreate(&ge.g, 0));
  cudaGraphConditionalHandle handle;
  CK(cudaGraphConditionalHandleCreate(&handle, ge.g, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams cp{};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = handle;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  CK(cudaGraphAddNode(&node, ge.g, nullptr, 0, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  CK(cudaStreamBeginCaptureToGraph(s->stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  try {
    mlaunch_attempt(v, s->stream, P, true, handle);
  } catch (...) {
    cudaGraph_t dummy;
    cudaStreamEndCapture(s->stream, &dummy);
    throw;
  }
  CK(cudaStreamEndCapture(s->stream, &body));
  CK(cudaGraphInstantiate(&ge.exec, ge.g, 0));
  v->graphs[key] = ge;
  return ge.exec;
}

void run_variants(ms_variants* v, const double* x0, double t0, double tf, const ms_policy* pols,
                  const ms_solver_config& cfg, ms_solve_result* res) {
  validate_cfg(cfg, t0, tf);
  if (cfg.record_snapshots) throw InvalidArg("variants: snapshots are recorded by ms_solve only");
  ms_system* s = v->s;
  std::lock_guard<std::mutex> lk(s->mu);
  std::lock_guard<std::mutex> lk2(v->mu);
  set_device(s);
  ensure_workspace(s, 1);  // sets fin_blocks; the lanes carry their own buffers
  SolvePlan P[kMaxLanes];
  int64_t cap = 1;
  for (int l = 0; l < v->nl; ++l) {
    check_policy(pols[l]);
    if (res[l].t_eval && res[l].n_eval > 0) throw InvalidArg("variants: dense output is produced by ms_solve only");
    P[l] = plan_bs32(pols[l]);
    if (cfg.record_step_log && res[l].step_log) cap = std::max<int64_t>(cap, res[l].step_log_capacity);
  }
  variants_workspace(v, cap);
  cudaStream_t st = s->stream;
  const int64_t dn = s->dn();
  for (int l = 0; l < v->nl; ++l) {
    init_ctl(s, v->ctl_host[l], cfg, t0, tf, P[l], v->log_cap);
    CK(cudaMemcpyAsync(v->B[l].ctl, &v->ctl_host[l], sizeof(Ctl), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(v->B[l].xb[0], x0, sizeof(double) * dn, cudaMemcpyHostToDevice, st));
  }
  const bool host_loop = use_host_loop();
  cudaGraphExec_t exec = host_loop ? nullptr : variants_graph(v, P);
  CK(cudaEventRecord(s->ev0, st));
  mlaunch_init(v, st, P);
  if (host_loop) {
    for (;;) {
      mlaunch_attempt(v, st, P, false, 0);
      CK(cudaMemcpyAsync(v->flag_host, v->flag, sizeof(int), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      if (!*v->flag_host) break;
    }
  } else {
    CK(cudaGraphLaunch(exec, st));
  }
  CK(cudaEventRecord(s->ev1, st));
  for (int l = 0; l < v->nl; ++l)
    CK(cudaMemcpyAsync(&v->ctl_host[l], v->B[l].ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, s->ev0, s->ev1));
  for (int l = 0; l < v->nl; ++l) {
    const Ctl& c = v->ctl_host[l];
    ms_solve_result* r = &res[l];
    if (r->final_state)
      CK(cudaMemcpyAsync(r->final_state, v->B[l].xb[c.ix], sizeof(double) * dn, cudaMemcpyDeviceToHost, st));
    r->step_log_count = c.record_log ? c.log_count : 0;
    if (r->step_log && c.record_log) {
      const int64_t m = std::min<int64_t>(std::min<int64_t>(r->step_log_capacity, c.log_count), v->log_cap);
      if (m > 0) {
        std::vector<StepLogRec> tmp((size_t)m);
        CK(cudaMemcpyAsync(tmp.data(), v->B[l].log, sizeof(StepLogRec) * m, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        for (int64_t i = 0; i < m; ++i) {
          r->step_log[i].t = tmp[(size_t)i].t;
          r->step_log[i].h = tmp[(size_t)i].h;
          r->step_log[i].err = tmp[(size_t)i].err;
          r->step_log[i].accepted = tmp[(size_t)i].accepted;
        }
      }
    }
    r->snapshot_count = 0;
    r->status = c.status;
    r->t_reached = c.t;
    r->n_accepted = c.n_acc;
    r->n_failed = c.n_fail;
    int64_t tl[3];
    tally(s, c, P[l], tl);
    r->rhs_evals = tl[0];
    r->flops_low = tl[1];
    r->flops_high = tl[2];
    r->device_ms = ms;
  }
  CK(cudaStreamSynchronize(st));
}

}  // namespace

void msb::set_last_error(const char* msg) { g_err = msg; }

msb::SysView msb::sys_view(ms_system_t s) {
  SysView v{};
  v.mkind = s->mkind;
  v.n = s->n;
  v.d = s->d;
  v.ld = s->ld;
  v.row0 = s->row0;
  v.row1 = s->row1;
  v.ks = s->ks;
  v.dev = s->dev;
  v.sms = s->sms;
  v.K = s->K;
  v.coupling_k = s->md.coupling_k;
  v.stream = s->stream;
  return v;
}

namespace {
void scan_k_tiny(ms_system* s) {
  int* flag = nullptr;
  CK(cudaMalloc(&flag, sizeof(int)));
  CK(cudaMemsetAsync(flag, 0, sizeof(int), s->stream));
  const int rows = s->row1 - s->row0, grid = 4 * s->sms;
  if (s->ks == MS_K_F32) k_scan_tiny<MS_K_F32><<<grid, 256, 0, s->stream>>>((const float*)s->K, s->n, rows, s->ld, flag);
  else if (s->ks == MS_K_F16) k_scan_tiny<MS_K_F16><<<grid, 256, 0, s->stream>>>((const __half*)s->K, s->n, rows, s->ld, flag);
  else k_scan_tiny<MS_K_BF16><<<grid, 256, 0, s->stream>>>((const __nv_bfloat16*)s->K, s->n, rows, s->ld, flag);
  CK(cudaGetLastError());
  int h = 0;
  CK(cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, s->stream));
  CK(cudaStreamSynchronize(s->stream));
  CK(cudaFree(flag));
  s->k_tiny = h;
}
}  // namespace

// =====================================================================================
extern "C" {

int ms_abi_version(void) { return MS_ABI_VERSION; }
const char* ms_last_error(void) { return g_err.c_str(); }

int ms_abi_sizes(int64_t out[8]) {
  out[0] = sizeof(ms_stage_prec);
  out[1] = sizeof(ms_policy);
  out[2] = sizeof(ms_solver_config);
  out[3] = sizeof(ms_step_record);
  out[4] = sizeof(ms_system_desc);
  out[5] = sizeof(ms_solve_result);
  out[6] = sizeof(ms_step_outcome);
  out[7] = sizeof(ms_exchange);
  return MS_OK;
}

int64_t ms_launch_count(void) {
  if (cudaDeviceSynchronize() != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  unsigned long long v = 0;
  if (cudaMemcpyFromSymbol(&v, msb::g_ms_launches, sizeof(v)) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  v += launches_tu_fast() + launches_tu_faithful() + launches_tu_multi() + launches_tu_batch();
  return static_cast<int64_t>(v);
}

int ms_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

void ms_default_config(ms_solver_config* c) {  // solver.hpp:39-61
  std::memset(c, 0, sizeof(*c));
  c->rel_tol = 1e-6;
  c->abs_tol = 1e-8;
  c->h_min_factor = 100.0;
  c->max_iterations = 100000;
  c->max_failed_steps = 85000;
  c->time_limits_enabled = 1;
  c->record_step_log = 1;
  c->wall_clock_limit = 5400.0;
  c->slow_solver_elapsed = 2700.0;
  c->slow_solver_progress = 0.10;
  c->safety = 0.9;
  c->fac_min = 0.2;
  c->fac_max = 5.0;
  c->controller_exponent = 1.0 / 3.0;
  c->record_snapshots = 0;
}

int ms_policy_for(int variant, ms_policy* out) {  // precision.cpp:22-42
  return guard([&] {
    if (variant < MS_SINGLE || variant > MS_DOUBLE) throw InvalidArg("policy_for: unknown variant");
    const ms_stage_prec sss{MS_BINARY32, MS_BINARY32, MS_BINARY32, 0};
    const ms_stage_prec dds{MS_BINARY64, MS_BINARY64, MS_BINARY32, 0};
    const ms_stage_prec ddd = kDDD;
    std::memset(out, 0, sizeof(*out));
    out->variant = (uint8_t)variant;
    switch (variant) {
      case MS_SINGLE: out->per_stage[0] = out->per_stage[1] = out->per_stage[2] = sss; break;
      case MS_MIXED1: out->per_stage[0] = out->per_stage[1] = sss; out->per_stage[2] = dds; break;
      case MS_MIXED2: out->per_stage[0] = out->per_stage[1] = out->per_stage[2] = dds; break;
      default: out->per_stage[0] = out->per_stage[1] = out->per_stage[2] = ddd; break;
    }
    out->first_step_k1 = out->per_stage[2];
    out->storage = variant == MS_SINGLE ? MS_BINARY32 : MS_BINARY64;
  });
}

int ms_policy_lowest_format(const ms_policy* p) { return plan_bs32(*p).lowest; }

int ms_rng_uniform(uint64_t seed, uint64_t stream, int64_t n, double lo, double hi, double* out) {
  SplitMix64 r(seed, stream);
  for (int64_t i = 0; i < n; ++i) out[i] = r.uniform(lo, hi);
  return MS_OK;
}
int ms_rng_normal(uint64_t seed, uint64_t stream, int64_t n, double* out) {
  SplitMix64 r(seed, stream);
  for (int64_t i = 0; i < n; ++i) out[i] = r.normal();
  return MS_OK;
}

int ms_system_create(const ms_system_desc* d, ms_system_t* out) {
  return guard([&] {
    if (!d || !out) throw InvalidArg("system_create: null argument");
    auto s = std::make_unique<ms_system>();
    const int n = d->n_agents;
    if (n < 1) throw InvalidArg("system: N must be >= 1");  // systems.cpp:210,223,244
    s->model = d->model;
    switch (d->model) {
      case MS_MODEL_LCO: s->mkind = MD_LCO; s->d = 2; break;
      case MS_MODEL_KURAMOTO: s->mkind = MD_KUR; s->d = 1; break;
      case MS_MODEL_CC: s->mkind = MD_CC; s->d = 4; break;
      case MS_MODEL_SCALAR_EXP:
      case MS_MODEL_SCALAR_ZERO:
      case MS_MODEL_SCALAR_NAN:
        s->mkind = d->model;
        s->fixture = true;
        s->d = 1;
        break;
      default: throw InvalidArg("system: unknown model");
    }
    s->n = n;
    s->cs = d->model == MS_MODEL_LCO ? d->coupled_slot : 0;
    if (s->cs < 0 || s->cs >= s->d) throw InvalidArg("system: bad coupled slot");
    s->ks = d->k_storage;
    if (s->ks < MS_K_SCALAR || s->ks > MS_K_BF16) throw InvalidArg("system: bad K storage");
    s->rhs_mode = d->rhs_mode;
    if (s->rhs_mode != MS_RHS_FAST && s->rhs_mode != MS_RHS_FAITHFUL && s->rhs_mode != MS_RHS_ORDERED)
      throw InvalidArg("system: bad rhs mode");
    s->ld = (n + 7) & ~7;
    s->row0 = d->row_begin;
    s->row1 = d->row_end;
    if (s->row0 == 0 && s->row1 == 0) s->row1 = n;
    if (s->row0 < 0 || s->row1 > n || s->row0 >= s->row1) throw InvalidArg("system: bad row range");
    if (s->mkind == MD_KUR && !d->omega) throw InvalidArg("kuramoto: omega required");
    if (s->mkind == MD_CC && (!d->cc_k1 || !d->cc_theta_h)) throw InvalidArg("cc: k1 and theta_h required");
    if (s->ks != MS_K_SCALAR && s->fixture) throw InvalidArg("fixture systems have no K");
    s->dev = d->device;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
      cudaGetLastError();
      throw CudaError("ms_system_create: no CUDA device (the B200 path has no CPU fallback)");
    }
    set_device(s.get());
    CK(cudaDeviceGetAttribute(&s->sms, cudaDevAttrMultiProcessorCount, s->dev));
    CK(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking));
    CK(cudaEventCreate(&s->ev0));
    CK(cudaEventCreate(&s->ev1));
    ModelDev& md = s->md;
    md.kind = s->mkind;
    md.n = n;
    md.d = s->d;
    md.cs = s->cs;
    for (int q = 0; q < 4; ++q) md.m[q] = 0.0;
    if (d->m) {
      for (int q = 0; q < s->d; ++q) md.m[q] = d->m[q];
    } else if (!s->fixture) {
      md.m[s->cs] = 1.0 / n;
    }
    md.coupling_k = d->coupling_k;
    md.i0 = d->stimulus_i0;
    md.omega = upload_array(s.get(), d->omega, n);
    md.w2 = upload_array(s.get(), d->w2, n);
    md.k1 = upload_array(s.get(), d->cc_k1, n);
    md.th = upload_array(s.get(), d->cc_theta_h, n);
    md.k0 = upload_array(s.get(), d->cc_k0, n);
    md.k2 = upload_array(s.get(), d->cc_k2, n);
    md.ca = upload_array(s.get(), d->cc_a, n);
    md.cb = upload_array(s.get(), d->cc_b, n);
    md.cc = upload_array(s.get(), d->cc_c, n);
    md.eps = upload_array(s.get(), d->cc_eps, n);
    switch (s->mkind) {  // FlopProfile (systems.cpp:217, 238, 266; test_support.hpp:23)
      case MD_LCO: s->flop_theta[0] = 1; s->flop_theta[1] = 1; s->flop_theta[2] = 4; break;
      case MD_KUR: s->flop_theta[0] = 1; s->flop_theta[1] = 3; s->flop_theta[2] = 2; break;
      case MD_CC: s->flop_theta[0] = 28; s->flop_theta[1] = 10; s->flop_theta[2] = 8; break;
      default: s->flop_theta[0] = 1; s->flop_theta[1] = 1; s->flop_theta[2] = 2; break;
    }
    if (s->ks != MS_K_SCALAR) {
      const int rows = s->row1 - s->row0;
      const size_t bytes = (size_t)rows * s->ld * kelem_bytes(s->ks);
      CK(cudaMalloc(&s->K, bytes));
      CK(cudaMemset(s->K, 0, bytes));
      if (d->K) {
        // upload in row blocks of <= 64 MiB, convert to the storage format once
        const size_t hb = d->k_host_dtype == MS_HOST_F32 ? 4 : 8;
        const int rb = (int)std::max<size_t>(1, (size_t(64) << 20) / ((size_t)n * hb));
        void* stage = nullptr;
        CK(cudaMalloc(&stage, (size_t)rb * n * hb));
        for (int r = 0; r < rows; r += rb) {
          const int nr = std::min(rb, rows - r);
          const char* src = static_cast<const char*>(d->K) + ((size_t)(s->row0 + r) * n) * hb;
          CK(cudaMemcpy(stage, src, (size_t)nr * n * hb, cudaMemcpyHostToDevice));
          const int64_t off = (int64_t)r * s->ld;
          const int grid = 1024;
          if (hb == 4) {
            const float* sp = static_cast<const float*>(stage);
            if (s->ks == MS_K_F32) k_convert_rows<MS_K_F32, float><<<grid, 256>>>((float*)s->K + off, sp, n, nr, s->ld);
            else if (s->ks == MS_K_F16) k_convert_rows<MS_K_F16, float><<<grid, 256>>>((__half*)s->K + off, sp, n, nr, s->ld);
            else k_convert_rows<MS_K_BF16, float><<<grid, 256>>>((__nv_bfloat16*)s->K + off, sp, n, nr, s->ld);
          } else {
            const double* sp = static_cast<const double*>(stage);
            if (s->ks == MS_K_F32) k_convert_rows<MS_K_F32, double><<<grid, 256>>>((float*)s->K + off, sp, n, nr, s->ld);
            else if (s->ks == MS_K_F16) k_convert_rows<MS_K_F16, double><<<grid, 256>>>((__half*)s->K + off, sp, n, nr, s->ld);
            else k_convert_rows<MS_K_BF16, double><<<grid, 256>>>((__nv_bfloat16*)s->K + off, sp, n, nr, s->ld);
          }
          CK(cudaGetLastError());
          CK(cudaDeviceSynchronize());
        }
        CK(cudaFree(stage));
      }
      CK(cudaDeviceSynchronize());
      scan_k_tiny(s.get());
      if (s->mkind == MD_KUR) s->gv = tc16_create(s->K, s->ld, s->row1 - s->row0, s->ks);
    }
    CK(cudaDeviceSynchronize());
    *out = s.release();
  });
}


int ms_system_destroy(ms_system_t s) {
  if (!s) return MS_OK;
  return guard([&] {
    cudaSetDevice(s->dev);
    for (auto& kv : s->graphs) {
      if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
      if (kv.second.g) cudaGraphDestroy(kv.second.g);
    }
    for (void* p : s->dev_arrays) cudaFree(p);
    if (s->K) cudaFree(s->K);
    tc16_destroy(s->gv);
    if (s->push.mem) cudaFree(s->push.mem);
    if (s->ws_mem) cudaFree(s->ws_mem);
    if (s->snap) cudaFree(s->snap);
    if (s->dense) cudaFree(s->dense);
    if (s->ctl_host) cudaFreeHost(s->ctl_host);
    delete s->loop_plan;
    if (s->ev0) cudaEventDestroy(s->ev0);
    if (s->ev1) cudaEventDestroy(s->ev1);
    if (s->stream) cudaStreamDestroy(s->stream);
    delete s;
  });
}

int ms_system_fill_k_uniform(ms_system_t s, uint64_t seed, uint64_t stream, double lo, double hi) {
  return guard([&] {
    if (!s || s->ks == MS_K_SCALAR) throw InvalidArg("fill_k: system has scalar coupling");
    set_device(s);
    const uint64_t state0 = seed + stream * 0xD1342543DE82EF95ull;
    const int rows = s->row1 - s->row0;
    const int grid = 8 * s->sms;
    if (s->ks == MS_K_F32) k_fill_uniform<MS_K_F32><<<grid, 256, 0, s->stream>>>((float*)s->K, s->n, s->row0, rows, s->ld, state0, lo, hi);
    else if (s->ks == MS_K_F16) k_fill_uniform<MS_K_F16><<<grid, 256, 0, s->stream>>>((__half*)s->K, s->n, s->row0, rows, s->ld, state0, lo, hi);
    else k_fill_uniform<MS_K_BF16><<<grid, 256, 0, s->stream>>>((__nv_bfloat16*)s->K, s->n, s->row0, rows, s->ld, state0, lo, hi);
    CK(cudaGetLastError());
    tc16_refresh(s->gv, s->K, s->ld, rows, s->stream);
    scan_k_tiny(s);
  });
}

int ms_system_get_k(ms_system_t s, double* out) {
  return guard([&] {
    if (!s || s->ks == MS_K_SCALAR) throw InvalidArg("get_k: system has scalar coupling");
    set_device(s);
    const int rows = s->row1 - s->row0;
    double* tmp = nullptr;
    CK(cudaMalloc(&tmp, sizeof(double) * (size_t)rows * s->n));
    if (s->ks == MS_K_F32) k_get_rows<MS_K_F32><<<1024, 256, 0, s->stream>>>((const float*)s->K, tmp, s->n, rows, s->ld);
    else if (s->ks == MS_K_F16) k_get_rows<MS_K_F16><<<1024, 256, 0, s->stream>>>((const __half*)s->K, tmp, s->n, rows, s->ld);
    else k_get_rows<MS_K_BF16><<<1024, 256, 0, s->stream>>>((const __nv_bfloat16*)s->K, tmp, s->n, rows, s->ld);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out, tmp, sizeof(double) * (size_t)rows * s->n, cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    CK(cudaFree(tmp));
  });
}

int ms_system_dim(ms_system_t s) { return s ? s->d : -1; }
int ms_system_agents(ms_system_t s) { return s ? s->n : -1; }
int ms_system_flop_profile(ms_system_t s, int64_t out[4]) {
  if (!s) return MS_EINVAL;
  out[0] = s->flop_theta[0];
  out[1] = s->flop_theta[1];
  out[2] = s->flop_theta[2];
  out[3] = s->d;
  return MS_OK;
}

int ms_eval_rhs(ms_system_t s, double t, const double* x, ms_stage_prec sp, double* out) {
  return guard([&] {
    (void)t;  // every model is autonomous (systems.cpp:118,137,159,177)
    if (!s || !x || !out) throw InvalidArg("eval_rhs: null argument");
    check_prec(sp);
    std::lock_guard<std::mutex> lk(s->mu);
    set_device(s);
    ensure_workspace(s, 1);
    Ctl& c = *s->ctl_host;
    std::memset(&c, 0, sizeof(Ctl));
    c.pk_off = s->k_tiny;
    const int64_t dn = s->dn();
    CK(cudaMemcpyAsync(s->B.ctl, &c, sizeof(Ctl), cudaMemcpyHostToDevice, s->stream));
    CK(cudaMemcpyAsync(s->B.xb[0], x, sizeof(double) * dn, cudaMemcpyHostToDevice, s->stream));
    EvalSpec e;
    e.l = 0;
    e.kind = PREP_X;
    e.out_slot = 0;
    launch_eval(s, s->stream, e, sp);
    CK(cudaMemcpyAsync(out, s->B.kb[0], sizeof(double) * dn, cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
  });
}

int ms_profile_rhs(ms_system_t s, const double* x, ms_stage_prec sp, int iters, double* rhs_ms, double* prep_ms) {
  return guard([&] {
    if (!s || !x || iters < 1) throw InvalidArg("profile_rhs: bad arguments");
    check_prec(sp);
    std::lock_guard<std::mutex> lk(s->mu);
    set_device(s);
    ensure_workspace(s, 1);
    Ctl& c = *s->ctl_host;
    std::memset(&c, 0, sizeof(Ctl));
    c.pk_off = s->k_tiny;
    cudaStream_t st = s->stream;
    CK(cudaMemcpyAsync(s->B.ctl, &c, sizeof(Ctl), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(s->B.xb[0], x, sizeof(double) * s->dn(), cudaMemcpyHostToDevice, st));
    EvalSpec e;
    e.l = 0;
    e.kind = PREP_X;
    e.out_slot = 0;
    std::vector<cudaEvent_t> ev(3 * (size_t)iters);
    for (auto& v : ev) CK(cudaEventCreate(&v));
    launch_eval(s, st, e, sp);  // warm-up
    for (int i = 0; i < iters; ++i) {
      CK(cudaEventRecord(ev[3 * i], st));
      launch_eval(s, st, e, sp, ev[3 * i + 1], ev[3 * i + 2]);
    }
    CK(cudaStreamSynchronize(st));
    double tr = 0, tp = 0;
    for (int i = 0; i < iters; ++i) {
      float a = 0, b = 0;
      CK(cudaEventElapsedTime(&a, ev[3 * i], ev[3 * i + 1]));
      CK(cudaEventElapsedTime(&b, ev[3 * i + 1], ev[3 * i + 2]));
      tp += a;
      tr += b;
    }
    for (auto& v : ev) cudaEventDestroy(v);
    if (rhs_ms) *rhs_ms = tr / iters;
    if (prep_ms) *prep_ms = tp / iters;
  });
}

int ms_estimate_error(int64_t n, const double* x_n, const double* x_next, const double* x_tilde, double ab,
                      double rel, double* err) {
  return guard([&] {
    if (n < 0 || !err) throw InvalidArg("estimate_error: bad arguments");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
      cudaGetLastError();
      throw CudaError("ms_estimate_error: no CUDA device");
    }
    double* buf = nullptr;
    const size_t b = sizeof(double) * (size_t)std::max<int64_t>(n, 1);
    CK(cudaMalloc(&buf, 3 * b + sizeof(double)));
    if (n > 0) {
      CK(cudaMemcpy(buf, x_n, sizeof(double) * n, cudaMemcpyHostToDevice));
      CK(cudaMemcpy((char*)buf + b, x_next, sizeof(double) * n, cudaMemcpyHostToDevice));
      CK(cudaMemcpy((char*)buf + 2 * b, x_tilde, sizeof(double) * n, cudaMemcpyHostToDevice));
    }
    double* o = reinterpret_cast<double*>((char*)buf + 3 * b);
    k_estimate_error<<<1, 1024>>>(n, buf, (double*)((char*)buf + b), (double*)((char*)buf + 2 * b), ab, rel, o);
    CK(cudaGetLastError());
    CK(cudaMemcpy(err, o, sizeof(double), cudaMemcpyDeviceToHost));
    CK(cudaFree(buf));
  });
}

int ms_adjust_step(double h, double err, double rel_tol, const ms_solver_config* cfg, double* h_next) {
  return guard([&] {
    if (!cfg || !h_next) throw InvalidArg("adjust_step: null argument");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
      cudaGetLastError();
      throw CudaError("ms_adjust_step: no CUDA device");
    }
    double* o = nullptr;
    CK(cudaMalloc(&o, sizeof(double)));
    k_adjust_step<<<1, 1>>>(h, err, rel_tol, cfg->safety, cfg->fac_min, cfg->fac_max, cfg->controller_exponent, o);
    CK(cudaGetLastError());
    CK(cudaMemcpy(h_next, o, sizeof(double), cudaMemcpyDeviceToHost));
    CK(cudaFree(o));
  });
}

int ms_initial_step(ms_system_t s, double t0, double t_final, const double* x0, const ms_solver_config* cfg,
                    int order, double* h0, int64_t* rhs_evals) {
  return guard([&] {
    if (!s || !x0 || !cfg || !h0) throw InvalidArg("initial_step: null argument");
    std::lock_guard<std::mutex> lk(s->mu);
    set_device(s);
    ensure_workspace(s, 1);
    Tableau T = bs32();
    T.order_high = order;
    SolvePlan P{};
    P.T = &T;
    P.k1_row = kDDD;
    P.storage = MS_BINARY64;
    P.lowest = MS_BINARY64;
    Ctl& c = *s->ctl_host;
    init_ctl(s, c, *cfg, t0, t_final, P, 1);
    CK(cudaMemcpyAsync(s->B.ctl, &c, sizeof(Ctl), cudaMemcpyHostToDevice, s->stream));
    CK(cudaMemcpyAsync(s->B.xb[0], x0, sizeof(double) * s->dn(), cudaMemcpyHostToDevice, s->stream));
    launch_init(s, s->stream, P, false);
    CK(cudaMemcpyAsync(&c, s->B.ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    *h0 = c.h;
    if (rhs_evals) *rhs_evals = c.evals_ddd;
  });
}

int ms_bs32_step(ms_system_t s, double t, const double* x_n, double h, const double* k1, const ms_policy* pol,
                 const ms_solver_config* cfg, ms_step_outcome* out) {
  return guard([&] {
    if (!s || !x_n || !k1 || !pol || !cfg || !out) throw InvalidArg("bs32_step: null argument");
    check_policy(*pol);
    std::lock_guard<std::mutex> lk(s->mu);
    set_device(s);
    ensure_workspace(s, 1);
    const SolvePlan P = plan_bs32(*pol);
    const Tableau& T = *P.T;
    Ctl& c = *s->ctl_host;
    init_ctl(s, c, *cfg, t, t + 1.0, P, 1);
    c.h_att = h;
    c.h = h;
    const int64_t dn = s->dn();
    cudaStream_t st = s->stream;
    CK(cudaMemcpyAsync(s->B.ctl, &c, sizeof(Ctl), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(s->B.xb[0], x_n, sizeof(double) * dn, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(s->B.kb[0], k1, sizeof(double) * dn, cudaMemcpyHostToDevice, st));
    for (int l = 1; l < T.S; ++l) launch_eval(s, st, stage_spec(T, l), P.rows[l - 1]);
    FinArgs f = fin_args(s, s->B, T, FIN_STEP, 0);
    CK(launch_k(k_finalize, s->fin_blocks, s->fin_threads, 0, st, f));
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(&c, s->B.ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const bool store32 = P.storage == MS_BINARY32;
    // first non-finite stage decides which outputs exist (solver.cpp:143-162)
    int nf_stage = 0;
    for (int l = 1; l < T.S; ++l)
      if (c.nf_mask & (1 << l)) {
        nf_stage = l;
        break;
      }
    const bool have_xnext = nf_stage == 0 || nf_stage == T.S - 1;
    const bool have_xstore = nf_stage == 0 || (nf_stage == T.S - 1 && store32);
    const bool have_rest = nf_stage == 0;
    auto get = [&](double* dst, const double* src, bool have) {
      if (!dst) return;
      if (have) {
        CK(cudaMemcpyAsync(dst, src, sizeof(double) * dn, cudaMemcpyDeviceToHost, st));
      } else {
        for (int64_t i = 0; i < dn; ++i) dst[i] = std::numeric_limits<double>::quiet_NaN();
      }
    };
    get(out->x_next, store32 ? s->B.xn : s->B.xb[1], have_xnext);
    get(out->x_store, s->B.xb[1], have_xstore);
    get(out->k4, s->B.kb[T.S], have_rest);
    get(out->x_tilde, s->B.xt, have_rest);
    CK(cudaStreamSynchronize(st));
    out->err = c.err;
    out->accepted = c.accepted;
    out->h_used = h;
    out->h_next = c.h_next;
    int64_t evals = 0, low = 0, high = 0;
    const int64_t n = s->n;
    for (int l = 1; l < T.S; ++l) {
      const int64_t cnt = c.evals_stage[l];
      const ms_stage_prec& sp = P.rows[l - 1];
      (is32(sp.f_prec) ? low : high) += s->flop_theta[0] * n * cnt;
      (is32(sp.g_prec) ? low : high) += s->flop_theta[1] * n * n * cnt;
      (is32(sp.sum_prec) ? low : high) += s->flop_theta[2] * n * n * cnt;
      evals += cnt;
    }
    high += (int64_t)T.scheme_flops * dn;
    out->rhs_evals = evals;
    out->flops_low = low;
    out->flops_high = high;
  });
}

int ms_solve(ms_system_t s, const double* x0, double t0, double t_final, const ms_policy* pol,
             const ms_solver_config* cfg, ms_solve_result* res) {
  return guard([&] {
    if (!s || !x0 || !pol || !cfg || !res) throw InvalidArg("solve: null argument");
    check_policy(*pol);
    run_solve(s, x0, false, t0, t_final, plan_bs32(*pol), *cfg, res, nullptr, false);
  });
}

int ms_solve_device(ms_system_t s, const double* x0_dev, double t0, double t_final, const ms_policy* pol,
                    const ms_solver_config* cfg, ms_solve_result* res, void* stream) {
  return guard([&] {
    if (!s || !x0_dev || !pol || !cfg || !res) throw InvalidArg("solve_device: null argument");
    check_policy(*pol);
    run_solve(s, x0_dev, true, t0, t_final, plan_bs32(*pol), *cfg, res, static_cast<cudaStream_t>(stream), true);
  });
}

int ms_loop_begin(ms_system_t s, const double* x0, int x0_on_device, double t0, double t_final,
                  const ms_policy* pol, const ms_solver_config* cfg, int64_t log_cap, void* stream) {
  return guard([&] {
    if (!s || !x0 || !pol || !cfg) throw InvalidArg("loop_begin: null argument");
    check_policy(*pol);
    validate_cfg(*cfg, t0, t_final);
    std::lock_guard<std::mutex> lk(s->mu);
    set_device(s);
    const int64_t cap = (cfg->record_step_log && log_cap > 0) ? log_cap : 1;
    ensure_workspace(s, cap);
    if (!s->loop_plan) s->loop_plan = new SolvePlanStore();
    s->loop_plan->P = plan_bs32(*pol);
    s->loop_plan->cfg = *cfg;
    s->loop_plan->log_cap = cap;
    cudaStream_t st = pick_stream(s, stream);
    Ctl& c = *s->ctl_host;
    init_ctl(s, c, *cfg, t0, t_final, s->loop_plan->P, cap);
    CK(cudaMemcpyAsync(s->B.ctl, &c, sizeof(Ctl), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(s->B.xb[0], x0, sizeof(double) * s->dn(),
                       x0_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
    CK(cudaEventRecord(s->ev0, st));
    s->loop_active = true;
  });
}

int ms_loop_segment_count(ms_system_t s, int list, int* count) {
  return guard([&] {
    if (!s || !count || !s->loop_active) throw InvalidArg("loop_segment_count: no active loop");
    if (list != 0 && list != 1) throw InvalidArg("loop_segment_count: list is 0 or 1");
    *count = loop_segments(s->loop_plan->P, list);
  });
}

int ms_loop_run_segment(ms_system_t s, int list, int index, void* stream, ms_exchange* ex) {
  return guard([&] {
    if (!s || !s->loop_active) throw InvalidArg("loop_run_segment: no active loop");
    if (list != 0 && list != 1) throw InvalidArg("loop_run_segment: list is 0 or 1");
    if (index < 0 || index >= loop_segments(s->loop_plan->P, list)) throw InvalidArg("loop_run_segment: bad index");
    set_device(s);
    if (s->push.np && s->push.ws_at_setup != s->ws_mem)
      throw InvalidArg("loop_run_segment: the workspace moved since ms_loop_push_setup (set it up again)");
    loop_run(s, s->loop_plan->P, list, index, pick_stream(s, stream), ex);
    if (s->push.np) {
      // the segment's sweeps already stored their rows into every peer: no
      // gather; signal the segment's end (the caller runs ms_loop_push_wait)
      if (ex) ex->needed = 0;
      CK(launch_k(k_push_signal, 1, 32, 0, pick_stream(s, stream), push_sig(s)));
      CK(cudaGetLastError());
    }
  });
}

int ms_loop_push_info(ms_system_t s, void** ws_base, size_t* ws_bytes, void** mailbox) {
  return guard([&] {
    if (!s || !ws_base || !mailbox) throw InvalidArg("loop_push_info: null argument");
    if (!s->ws_ready) throw InvalidArg("loop_push_info: no workspace yet (call ms_loop_begin first)");
    set_device(s);
    if (!s->push.mem) {
      CK(cudaMalloc(&s->push.mem, sizeof(unsigned long long) * 16));
      CK(cudaMemset(s->push.mem, 0, sizeof(unsigned long long) * 16));
    }
    *ws_base = s->ws_mem;
    if (ws_bytes) *ws_bytes = bufs_bytes(s, s->log_cap);
    *mailbox = s->push.mem;
  });
}

int ms_loop_push_setup(ms_system_t s, int world, int rank, void* const* peer_ws, void* const* peer_mailbox) {
  return guard([&] {
    if (!s) throw InvalidArg("loop_push_setup: null handle");
    set_device(s);
    s->push.np = 0;
    s->push.world = world;
    s->push.rank = rank;
    if (world <= 1) return;
    if (world - 1 > kMaxPeers || rank < 0 || rank >= world || !peer_ws || !peer_mailbox)
      throw InvalidArg("loop_push_setup: need 2 <= world <= 8, 0 <= rank < world and peer arrays");
    if (!s->push.mem) throw InvalidArg("loop_push_setup: call ms_loop_push_info first");
    int np = 0;
    for (int q = 0; q < world; ++q) {
      if (q == rank) continue;
      if (!peer_ws[q] || !peer_mailbox[q]) throw InvalidArg("loop_push_setup: null peer pointer");
      s->push.peer_ws[np] = static_cast<char*>(peer_ws[q]);
      s->push.peer_slot[np] = static_cast<unsigned long long*>(peer_mailbox[q]) + rank;
      s->push.peer_rank[np] = q;
      ++np;
    }
    // a fresh epoch sequence: the caller synchronizes the ranks after every
    // rank's setup, before any segment runs
    CK(cudaMemset(s->push.mem, 0, sizeof(unsigned long long) * 16));
    CK(cudaDeviceSynchronize());
    s->push.np = np;
    s->push.ws_at_setup = s->ws_mem;
  });
}

int ms_loop_push_wait(ms_system_t s, void* stream) {
  return guard([&] {
    if (!s || !s->loop_active) throw InvalidArg("loop_push_wait: no active loop");
    if (!s->push.np) return;
    set_device(s);
    CK(launch_k(k_push_wait, 1, 32, 0, pick_stream(s, stream), push_sig(s)));
    CK(cudaGetLastError());
  });
}

int ms_ipc_export(void* dev_ptr, unsigned char* handle64) {
  return guard([&] {
    if (!dev_ptr || !handle64) throw InvalidArg("ipc_export: null argument");
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, dev_ptr));
    static_assert(sizeof(h) == 64, "CUDA IPC handle size");
    std::memcpy(handle64, &h, 64);
  });
}

int ms_ipc_import(const unsigned char* handle64, void** dev_ptr) {
  return guard([&] {
    if (!handle64 || !dev_ptr) throw InvalidArg("ipc_import: null argument");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle64, 64);
    CK(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  });
}

int ms_ipc_close(void* dev_ptr) {
  return guard([&] {
    if (!dev_ptr) throw InvalidArg("ipc_close: null argument");
    CK(cudaIpcCloseMemHandle(dev_ptr));
  });
}

int ms_loop_done(ms_system_t s, void* stream, int* done) {
  return guard([&] {
    if (!s || !done || !s->loop_active) throw InvalidArg("loop_done: no active loop");
    set_device(s);
    cudaStream_t st = pick_stream(s, stream);
    CK(cudaMemcpyAsync(&s->ctl_host->done, &s->B.ctl->done, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    *done = s->ctl_host->done;
  });
}

int ms_loop_end(ms_system_t s, ms_solve_result* res, int final_on_device, void* stream) {
  return guard([&] {
    if (!s || !res || !s->loop_active) throw InvalidArg("loop_end: no active loop");
    set_device(s);
    cudaStream_t st = pick_stream(s, stream);
    CK(cudaEventRecord(s->ev1, st));
    Ctl& c = *s->ctl_host;
    CK(cudaMemcpyAsync(&c, s->B.ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, s->ev0, s->ev1));
    const int64_t dn = s->dn();
    if (res->final_state)
      CK(cudaMemcpyAsync(res->final_state, s->B.xb[c.ix], sizeof(double) * dn,
                         final_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
    res->step_log_count = c.record_log ? c.log_count : 0;
    if (res->step_log && c.record_log) {
      const int64_t m = std::min<int64_t>(std::min<int64_t>(res->step_log_capacity, c.log_count), s->log_cap);
      if (m > 0) {
        std::vector<StepLogRec> tmp((size_t)m);
        CK(cudaMemcpyAsync(tmp.data(), s->B.log, sizeof(StepLogRec) * m, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        for (int64_t i = 0; i < m; ++i) {
          res->step_log[i].t = tmp[(size_t)i].t;
          res->step_log[i].h = tmp[(size_t)i].h;
          res->step_log[i].err = tmp[(size_t)i].err;
          res->step_log[i].accepted = tmp[(size_t)i].accepted;
        }
      }
    }
    CK(cudaStreamSynchronize(st));
    res->status = c.status;
    res->t_reached = c.t;
    res->n_accepted = c.n_acc;
    res->n_failed = c.n_fail;
    int64_t tl[3];
    tally(s, c, s->loop_plan->P, tl);
    res->rhs_evals = tl[0];
    res->flops_low = tl[1];
    res->flops_high = tl[2];
    res->device_ms = ms;
    s->loop_active = false;
  });
}


int ms_dp54_reference(ms_system_t s, const double* x0, double t0, double t_final, const ms_solver_config* cfg,
                      ms_solve_result* res) {
  return guard([&] {
    if (!s || !x0 || !cfg || !res) throw InvalidArg("dp54_reference: null argument");
    ms_solver_config rc = *cfg;  // solver.cpp:474-478
    rc.rel_tol = 1e-9;
    rc.abs_tol = 1e-9;
    rc.controller_exponent = 1.0 / 5.0;
    rc.record_snapshots = 0;
    run_solve(s, x0, false, t0, t_final, plan_dp54(), rc, res, nullptr, false);
  });
}

int ms_variants_create(ms_system_t s, int count, ms_variants_t* out) {
  return guard([&] {
    if (!s || !out) throw InvalidArg("variants_create: null argument");
    if (count < 1 || count > kMaxLanes) throw InvalidArg("variants_create: count must be 1..4");
    set_device(s);
    auto v = std::make_unique<ms_variants>();
    v->s = s;
    v->nl = count;
    CK(cudaMallocHost(&v->ctl_host, sizeof(Ctl) * kMaxLanes));
    CK(cudaMallocHost(&v->flag_host, sizeof(int)));
    *out = v.release();
  });
}

int ms_variants_destroy(ms_variants_t v) {
  if (!v) return MS_OK;
  return guard([&] {
    cudaSetDevice(v->s->dev);
    cudaStreamSynchronize(v->s->stream);
    drop_graphs(v);
    if (v->mem) cudaFree(v->mem);
    if (v->ctl_host) cudaFreeHost(v->ctl_host);
    if (v->flag_host) cudaFreeHost(v->flag_host);
    delete v;
  });
}

int ms_variants_solve(ms_variants_t v, const double* x0, double t0, double t_final, const ms_policy* policies,
                      const ms_solver_config* cfg, ms_solve_result* results) {
  return guard([&] {
    if (!v || !x0 || !policies || !cfg || !results) throw InvalidArg("variants_solve: null argument");
    run_variants(v, x0, t0, t_final, policies, *cfg, results);
  });
}

}  // extern "C"
