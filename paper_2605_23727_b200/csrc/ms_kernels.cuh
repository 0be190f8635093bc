// ms_kernels.cuh — sm_100a kernels of the mixed-precision BS3(2) hot path.
//
//   prep        stage combination of rk_step (solver.cpp:130-149, 86-104) fused
//               with the per-agent part of eval_core: F_i in FS, the GS cast of
//               the coupled slot (or sin/cos of it for the Kuramoto split), the
//               CC prefactor, and the uncoupled output slots (systems.cpp:35-62)
//   rhs_fast    the all-pairs coupling sweep (systems.cpp:50-57) as a K-row
//               stream: 128-bit loads of K, column data staged in shared memory
//               by cp.async.bulk (TMA) through an mbarrier ring, warp-shuffle
//               row reductions. HBM-bound at large N.
//   rhs_faithful  the same sum in the reference's exact order: one thread per
//               row, ascending j including j = i, per-pair G (parity mode)
//   finalize    x_tilde, weighted max-norm error, accept/reject, adjust_step and
//               the loop bookkeeping of solve_core (solver.cpp:188-214,
//               272-342, 399-418), last-block-done over a grid reduction
//   init_a/b    initial_step norms (solver.cpp:420-451)
#pragma once
#include <type_traits>

#include "ms_common.cuh"
#include "ms_ddpow.cuh"

namespace msb {

// ------------------------------------------------------------------------------
// model parameters on the device
struct ModelDev {
  int kind;     // MD_* or a fixture MS_MODEL_SCALAR_*
  int n, d, cs; // agents, dim, coupled slot
  double m[4];  // per-slot weights (systems.hpp:71)
  double coupling_k, i0;
  const double* omega;
  const double* w2;
  const double* k1;
  const double* th;
  const double* k0;
  const double* k2;
  const double* ca;
  const double* cb;
  const double* cc;
  const double* eps;
};

// reference CcConstants (systems.hpp:32-43)
constexpr double kCcK0 = 2.0, kCcK2 = 0.144832, kCcA = 2.0, kCcB = 0.7, kCcC = 0.8,
                 kCcEps = 0.228249;

enum : int { PREP_X = 0, PREP_STAGE = 1, PREP_INIT_X1 = 2 };
enum : int { GATE_ALWAYS = 0, GATE_NEED_K1 = 1, GATE_INIT2 = 2 };
enum : int { CNT_DDD = 0, CNT_K1 = 1, CNT_STAGE = 2, CNT_NONE = 3 };
// k-buffer references resolved at run time through ctl->k1i
enum : int { SLOT_K1 = -1, SLOT_KLAST = -2 };

struct PrepArgs {
  ModelDev md;
  Bufs B;
  int S;          // tableau stages
  int l;          // stage index in rk_step (0 = k1 / plain evaluation)
  int kind;       // PREP_*
  int gate;       // GATE_*
  int count;      // CNT_*
  int out_slot;   // k-buffer receiving the evaluation (SLOT_* or index)
  int nterms;
  double coef[kMaxStages];
  int slot[kMaxStages];
  int is_last;    // FSAL last stage: x_next (and binary32 x_store) is the argument
  int round_x;    // binary32 storage cold start: x <- RN32(x) in place
  int split;      // Kuramoto split column data (sin, cos)
  int ws32;       // WS = wider(FS, SS) is binary32
  int fs32;       // F precision is binary32 (fixtures: round_to(x, f_prec))
  int ld;         // padded column count
  const double* xsrc;  // PREP_X source (NULL = xb[ix])
  // row-sharded loop: the finiteness scan of the previous stage's gathered
  // vector (all rows) folded into this prep; bit scan_bit of nf_mask
  const double* scan;
  int64_t scan_n;
  int scan_bit;
};

struct RhsArgs {
  const Ctl* ctl;
  int* nf_mask;
  int l, gate, S, out_slot;
  const void* K;
  int64_t ld;
  int n, row0, row1;
  const void* gin;
  const void* rowc;
  const double* fvc;
  double* kb[kMaxStages + 1];
  int d, cs;
  double mw;
  double coupling_k;
  int ws32;
  // row-sharded loop: the sweep (not the prep) counts the evaluation, so an
  // evaluation skipped after the prep's folded scan is not counted
  Ctl* count_ctl;
  int count;
  // K larger than L2 can hold across evaluations: stream it evict-first
  int k_stream;
  // packed FMUL2.FTZ products allowed (MS_SWEEP_PK != off; the device flag
  // Ctl::pk_off can still veto them)
  int pk;
  // host-side: the handle's tensor-core sweep resources (GvRes, ms_gemv_tc.cuh) or null
  const void* tc16;
  // the column data's f16 operand image (Bufs::op16), written by the prep
  const void* op16;
  // push exchange of the row-sharded loop (np = 0: none)
  PushDev push;
};

// store one output element of a sweep: here and, in the push exchange, at the
// same workspace offset in every peer (then visible system-wide at the
// sweep's push_fence)
__device__ __forceinline__ void push_row(const PushDev& p, double* dst, double v) {
  *dst = v;
  for (int q = 0; q < p.np; ++q)
    *reinterpret_cast<double*>(p.peer[q] + (reinterpret_cast<const char*>(dst) - p.ws)) = v;
}
__device__ __forceinline__ void push_fence(const PushDev& p) {
  if (p.np) __threadfence_system();
}

__device__ __forceinline__ void sweep_count(const RhsArgs& a) {
  if (a.count_ctl && blockIdx.x == 0 && threadIdx.x == 0) {
    if (a.count == CNT_DDD) a.count_ctl->evals_ddd += 1;
    else if (a.count == CNT_K1) a.count_ctl->evals_k1 += 1;
    else if (a.count == CNT_STAGE) a.count_ctl->evals_stage[a.l] += 1;
  }
}

__device__ __forceinline__ double* resolve_slot(const Bufs& B, int S, int slot, int k1i) {
  if (slot == SLOT_K1) return B.kb[k1i];
  if (slot == SLOT_KLAST) return B.kb[S - k1i];
  return B.kb[slot];
}

// Shared skip rule of every kernel of stage l (prep and rhs decide alike).
__device__ __forceinline__ bool stage_skip(const Ctl* c, int l, int gate) {
  if (c->done) return true;
  if (gate == GATE_NEED_K1 && !c->need_k1) return true;
  if (gate == GATE_INIT2 && c->init_skip2) return true;
  if (l > 0 && (c->nf_mask & ((1 << l) - 1))) return true;
  return false;
}

// ------------------------------------------------------------------------------
// F_i in FS (systems.cpp:117-120, 136-139, 159-174 + D2/D4 extensions)
template <class S>
__device__ __forceinline__ void model_f(const ModelDev& md, int i, const double* a, S* f) {
  if (md.kind == MD_LCO) {
    const S x0 = cvt<S>(a[0]), x1 = cvt<S>(a[1]);
    f[0] = x1;
    f[1] = md.w2 ? -mul<S>(cvt<S>(md.w2[i]), x0) : -x0;
  } else if (md.kind == MD_KUR) {
    f[0] = cvt<S>(md.omega[i]);
  } else {
    const S x1 = cvt<S>(a[0]), x2 = cvt<S>(a[1]), x3 = cvt<S>(a[2]), x4 = cvt<S>(a[3]);
    const S th = cvt<S>(md.th[i]);
    const S k0 = cvt<S>(md.k0 ? md.k0[i] : kCcK0);
    const S ca = cvt<S>(md.ca ? md.ca[i] : kCcA);
    const S x2sq = mul<S>(x2, x2);
    const S x2h = mul<S>(x2sq, x2sq);
    // ((k0*th)/(th+x2h)) * ((a*x1)*x1 + 1) - k1*x1
    f[0] = sub<S>(mul<S>(dvd<S>(mul<S>(k0, th), add<S>(th, x2h)),
                         add<S>(mul<S>(mul<S>(ca, x1), x1), S(1))),
                  mul<S>(cvt<S>(md.k1[i]), x1));
    f[1] = mul<S>(cvt<S>(md.k2 ? md.k2[i] : kCcK2), sub<S>(x1, x2));
    const S x1sq = mul<S>(x1, x1);
    // (x3*(1 - (x3*x3)/3) - x4) + I0*(1 - 4/(4 + x1sq)); k3^2 = 4 fixed
    f[2] = add<S>(sub<S>(mul<S>(x3, sub<S>(S(1), dvd<S>(mul<S>(x3, x3), S(3)))), x4),
                  mul<S>(cvt<S>(md.i0), sub<S>(S(1), dvd<S>(S(4), add<S>(S(4), x1sq)))));
    // eps*((x3 + b) - c*x4)
    f[3] = mul<S>(cvt<S>(md.eps ? md.eps[i] : kCcEps),
                  sub<S>(add<S>(x3, cvt<S>(md.cb ? md.cb[i] : kCcB)),
                         mul<S>(cvt<S>(md.cc ? md.cc[i] : kCcC), x4)));
  }
}

// CC row constant pref = ((k0*th)*a)/(th + x2sq*x2sq) in GS (systems.cpp:176-186):
// row-invariant, so hoisting it out of the j loop is bitwise safe.
template <class S>
__device__ __forceinline__ S cc_pref(const ModelDev& md, int i, double x2d) {
  const S x2 = cvt<S>(x2d);
  const S x2sq = mul<S>(x2, x2);
  const S th = cvt<S>(md.th[i]);
  const S k0 = cvt<S>(md.k0 ? md.k0[i] : kCcK0);
  const S ca = cvt<S>(md.ca ? md.ca[i] : kCcA);
  return dvd<S>(mul<S>(mul<S>(k0, th), ca), add<S>(th, mul<S>(x2sq, x2sq)));
}

__device__ __forceinline__ double ws_add(double fval, double coupling, int ws32) {
  // out = (double)((WS)f + (WS)acc), systems.cpp:59-62
  if (ws32) return (double)__fadd_rn((float)fval, (float)coupling);
  return __dadd_rn(fval, coupling);
}

// ------------------------------------------------------------------------------
// prep: one thread per agent.
struct PrepCtx {
  Ctl* ctl;
  int k1i, ix;
  double* x;          // xb[ix]
  const double* xs;   // the argument's source (x, or an explicit vector)
  double* out;        // the k slot this evaluation fills
  double h;
  bool store32;
};

__device__ __forceinline__ PrepCtx prep_ctx(const PrepArgs& p) {
  PrepCtx c;
  c.ctl = p.B.ctl;
  c.k1i = c.ctl->k1i;
  c.ix = c.ctl->ix;
  c.x = p.B.xb[c.ix];
  c.xs = p.xsrc ? p.xsrc : c.x;
  c.out = resolve_slot(p.B, p.S, p.out_slot, c.k1i);
  c.h = p.kind == PREP_INIT_X1 ? c.ctl->h1 : c.ctl->h_att;
  c.store32 = c.ctl->store32 != 0;
  return c;
}

__device__ __forceinline__ void prep_count(const PrepArgs& p, Ctl* ctl) {
  if (p.count == CNT_DDD) ctl->evals_ddd += 1;
  else if (p.count == CNT_K1) ctl->evals_k1 += 1;
  else if (p.count == CNT_STAGE) ctl->evals_stage[p.l] += 1;
}

// The stage argument of state element e (rk_step, solver.cpp:130-149). With
// own = false nothing is written (a fused sweep recomputing other agents'
// column values); the in-place binary32 rounding of x is idempotent, so
// readers racing with the owner see the same value either way.
#ifndef MS_PREP_ROLL
#define MS_PREP_ROLL 1
#endif
constexpr int kPrepUnroll = MS_PREP_ROLL ? 1 : 4;
__device__ __forceinline__ double prep_arg(const PrepArgs& p, const PrepCtx& c, int64_t e, bool own) {
  double v;
  if (p.kind == PREP_X) {
    v = c.xs[e];
    if (p.round_x) {
      v = rn32(v);
      if (own) c.x[e] = v;
    }
  } else if (p.kind == PREP_INIT_X1) {
    v = __dadd_rn(c.xs[e], __dmul_rn(c.h, p.B.kb[1][e]));  // x0 + h1 * f0 (solver.cpp:435)
  } else {
    // combo = a_l0*k_0 (+ a_lm*k_m ...), arg = x + h*combo (solver.cpp:130-142)
    // the short runtime loops below stay rolled (MS_PREP_ROLL): unrolled copies of
    // every stage shape made the preps 3-4 x larger than the path an attempt executes
    double cm = __dmul_rn(p.coef[0], resolve_slot(p.B, p.S, p.slot[0], c.k1i)[e]);
#pragma unroll kPrepUnroll
    for (int t = 1; t < p.nterms; ++t)
      cm = __dadd_rn(cm, __dmul_rn(p.coef[t], resolve_slot(p.B, p.S, p.slot[t], c.k1i)[e]));
    v = __dadd_rn(c.xs[e], __dmul_rn(c.h, cm));
    if (p.is_last) {
      if (c.store32) {
        // combine_binary32 (solver.cpp:86-104)
        const float hf = __double2float_rn(c.h);
        float acc = __double2float_rn(c.xs[e]);
#pragma unroll kPrepUnroll
        for (int t = 0; t < p.nterms; ++t) {
          const float cf = __fmul_rn(hf, __double2float_rn(p.coef[t]));
          acc = __fadd_rn(acc, __fmul_rn(cf, __double2float_rn(resolve_slot(p.B, p.S, p.slot[t], c.k1i)[e])));
        }
        if (own) p.B.xn[e] = v;  // x_next
        v = (double)acc;
      }
      if (own) p.B.xb[c.ix ^ 1][e] = v;  // x_store (= x_next under binary64 storage)
    }
  }
  return v;
}

// The tensor-core sweep's operand image of column j (ms_gemv_tc.cuh): per
// 64-column k-block 512 bytes = four 128-byte rows s_hi, s_lo, c_hi, c_lo of
// f16 (hi = RN16(v), lo = RN16(v - hi)), 16-byte chunks in the SWIZZLE_128B
// order (chunk index XOR row), i.e. rows 0-3 of the MMA's B tile as they sit
// in shared memory.
__device__ __forceinline__ void op16_put(void* img, int j, float s, float c) {
  unsigned char* base = static_cast<unsigned char*>(img) + (size_t)(j >> 6) * 512;
  const int col = j & 63;
  const __half sh = __float2half_rn(s), ch = __float2half_rn(c);
  const __half v[4] = {sh, __float2half_rn(__fsub_rn(s, __half2float(sh))), ch,
                       __float2half_rn(__fsub_rn(c, __half2float(ch)))};
#pragma unroll
  for (int r = 0; r < 4; ++r)
    *reinterpret_cast<__half*>(base + r * 128 + ((((col >> 3) ^ r) & 7) << 4) + (col & 7) * 2) = v[r];
}

// Every per-agent output of one evaluation for agent i: F in FS, the uncoupled
// slots, the coupled slot's F (fvc), the column value(s) (gin) and the CC row
// constant (systems.cpp:35-62). Returns whether an output is non-finite.
template <int MODEL, class FS, class GS>
__device__ __forceinline__ bool prep_agent(const PrepArgs& p, const PrepCtx& c, int i) {
  const int d = p.md.d;
  bool nonfinite = false;
  double a[4];
#pragma unroll kPrepUnroll
  for (int s = 0; s < d; ++s) a[s] = prep_arg(p, c, (int64_t)i * d + s, true);
  if (MODEL < 0) {
    // reference test fixtures (test_support.hpp:21-53): the whole RHS is F
    const int kind = p.md.kind;
    for (int s = 0; s < d; ++s) {
      double o;
      if (kind == MS_MODEL_SCALAR_EXP) o = p.fs32 ? rn32(a[s]) : a[s];  // round_to(x, f_prec)
      else if (kind == MS_MODEL_SCALAR_ZERO) o = 0.0;
      else o = __longlong_as_double(0x7ff8000000000000ll);
      c.out[(int64_t)i * d + s] = o;
      nonfinite |= !isfinite(o);
    }
    return nonfinite;
  }
  FS f[4];
  model_f<FS>(p.md, i, a, f);
  const int cs = p.md.cs;
  for (int s = 0; s < d; ++s) {
    if (s == cs) continue;
    const double o = ws_add((double)f[s], 0.0, p.ws32);  // acc of an uncoupled slot is +0
    c.out[(int64_t)i * d + s] = o;
    nonfinite |= !isfinite(o);
  }
  p.B.fvc[i] = (double)f[cs];
  GS* gin = reinterpret_cast<GS*>(p.B.gin);
  // G reads slot 0 of both agents (x_j0 - x_i0, theta_j - theta_i), whatever
  // slot it is added to (systems.cpp:123-126, 141-143, 183-184)
  const GS xg = cvt<GS>(a[0]);
  if (p.split) {
    GS sv, cv;
    dsincos(xg, &sv, &cv);
    MS_CHECK(i >= 0 && 2 * i + 1 < 2 * p.ld, "prep: column data index");
    gin[2 * i] = sv;  // split column data: interleaved (s_j, c_j) pairs
    gin[2 * i + 1] = cv;
    if constexpr (sizeof(GS) == 4 && MODEL == MD_KUR)
      if (p.B.op16) op16_put(p.B.op16, i, sv, cv);
    if constexpr (sizeof(GS) == 4)
      if (sc_tiny(sv, cv)) c.ctl->pk_off = 1;
  } else {
    gin[i] = xg;
  }
  if (MODEL == MD_CC) reinterpret_cast<GS*>(p.B.rowc)[i] = cc_pref<GS>(p.md, i, a[1]);
  return nonfinite;
}

template <int MODEL, class FS, class GS>
__global__ void __launch_bounds__(256) k_prep(PrepArgs p) {
  msb::count_launch();
  pdl_enter();
  Ctl* ctl = p.B.ctl;
  if (stage_skip(ctl, p.l, p.gate)) return;
  const PrepCtx c = prep_ctx(p);
  if (blockIdx.x == 0 && threadIdx.x == 0) prep_count(p, ctl);
  bool nonfinite = false;
  if (p.scan) {
    bool bad = false;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < p.scan_n; e += (int64_t)gridDim.x * blockDim.x)
      bad |= !isfinite(p.scan[e]);
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(&ctl->nf_mask, 1 << p.scan_bit);
  }
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < p.md.n; i += gridDim.x * blockDim.x)
    nonfinite |= prep_agent<MODEL, FS, GS>(p, c, i);
  // zero the padding columns [n, ld) of the column data in THIS evaluation's
  // type: the buffer is shared by binary32 and binary64 rows, and the scalar
  // coupling (no zero-padded K) sums over every column of the chunk
  if (MODEL >= 0) {
    GS* gin = reinterpret_cast<GS*>(p.B.gin);
    for (int j = p.md.n + blockIdx.x * blockDim.x + threadIdx.x; j < p.ld; j += gridDim.x * blockDim.x) {
      if (p.split) {
        gin[2 * j] = GS(0);
        gin[2 * j + 1] = GS(0);
      } else {
        gin[j] = GS(0);
      }
    }
  }
  if (__any_sync(0xffffffffu, nonfinite) && (threadIdx.x & 31) == 0) atomicOr(&ctl->nf_mask, 1 << p.l);
}

// ------------------------------------------------------------------------------
// mbarrier / bulk-copy helpers (sm_90+ PTX, used on sm_100a)
__device__ __forceinline__ uint32_t smem_u32(const void* ptr) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(ptr));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// Wait for an mbarrier phase. try_wait itself suspends for a while; after
// ~2^16 unsuccessful tries the wait starts checking the clock and traps after
// 10 s, so a pipeline bug ends the kernel with an error instead of hanging the GPU.
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ uint64_t mbar_clock_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
static __device__ __noinline__ void mbar_wait_slow(uint64_t* bar, uint32_t parity) {
  const uint64_t t0 = mbar_clock_ns();
  for (;;) {
    for (int k = 0; k < 1024; ++k)
      if (mbar_try(bar, parity)) return;
    if (mbar_clock_ns() - t0 > 10000000000ull) __trap();
  }
}
#ifndef MS_MBAR_ROLL
#define MS_MBAR_ROLL 0  // 1: the try loop stays rolled (smaller code; C2 -0.5 %, but C4 f32 solves measured 0.5 % slower under the power cap)
#endif
constexpr int kMbarUnroll = MS_MBAR_ROLL ? 1 : 64;
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
#pragma unroll kMbarUnroll
  for (int k = 0; k < 65536; ++k)
    if (mbar_try(bar, parity)) return;
  mbar_wait_slow(bar, parity);
}
// dst inside this CTA's dynamic shared memory, 16-byte granularity (checked builds)
__device__ __forceinline__ void check_bulk(const void* dst, const void* src, uint32_t bytes) {
#if MS_CHECKS
  extern __shared__ unsigned char ms_dyn_smem[];
  const uint32_t base = smem_u32(ms_dyn_smem), d = smem_u32(dst);
  MS_CHECK(d >= base && d + bytes <= base + dyn_smem_bytes(), "bulk copy outside dynamic shared memory");
  MS_CHECK((d & 15u) == 0 && (reinterpret_cast<uintptr_t>(src) & 15u) == 0 && (bytes & 15u) == 0,
           "bulk copy alignment");
#else
  (void)dst; (void)src; (void)bytes;
#endif
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  check_bulk(dst, src, bytes);
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// the same copy with an L2 eviction-priority policy (createpolicy)
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                              uint64_t pol) {
  check_bulk(dst, src, bytes);
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ uint64_t l2_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint4 ldg_stream(const void* ptr) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(ptr));
  return r;
}
// evict-first K loads in the register sweep: measured -1.5 % on C4 f16 whole
// solves (profiles/r1_sustained_sweep.txt), so off; the TMA sweep keeps them
#ifndef MS_LDG_KHINT
#define MS_LDG_KHINT 0
#endif
__device__ __forceinline__ uint4 ldg_stream(const void* ptr, uint64_t pol) {
  if (!MS_LDG_KHINT) return ldg_stream(ptr);
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(ptr), "l"(pol));
  return r;
}

template <class T> __device__ __forceinline__ T shfl_xor(T v, int m) { return __shfl_xor_sync(0xffffffffu, v, m); }

// K element j of a 16-byte vector as f32 (exact for every storage format)
template <int KS> struct KVec;
template <> struct KVec<MS_K_F32> {
  static constexpr int N = 4;
  __device__ __forceinline__ static void unpack(const uint4& v, float* o) {
    o[0] = __uint_as_float(v.x); o[1] = __uint_as_float(v.y);
    o[2] = __uint_as_float(v.z); o[3] = __uint_as_float(v.w);
  }
};
template <> struct KVec<MS_K_F16> {
  static constexpr int N = 8;
  __device__ __forceinline__ static void unpack(const uint4& v, float* o) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w[q]));
      o[2 * q] = f.x; o[2 * q + 1] = f.y;
    }
  }
};
template <> struct KVec<MS_K_BF16> {
  static constexpr int N = 8;
  __device__ __forceinline__ static void unpack(const uint4& v, float* o) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      o[2 * q] = __uint_as_float(w[q] << 16);
      o[2 * q + 1] = __uint_as_float(w[q] & 0xffff0000u);
    }
  }
};
template <> struct KVec<MS_K_SCALAR> {
  static constexpr int N = 4;
  __device__ __forceinline__ static void unpack(const uint4&, float* o) {  // never reached (no matrix)
    o[0] = o[1] = o[2] = o[3] = 0.f;
  }
};

// Sweep geometry (overridable at build time for tuning sweeps)
#ifndef MS_FAST_THREADS
#define MS_FAST_THREADS 512  // 16 warps
#endif
#ifndef MS_FAST_MINB
#define MS_FAST_MINB 1       // resident CTAs per SM (grid = SMs x MINB)
#endif
#ifndef MS_FAST_R
#define MS_FAST_R 8          // rows per warp per sweep (fp32 accumulation)
#endif
#ifndef MS_CHUNK
#define MS_CHUNK 2048        // columns per staged chunk
#endif
#ifndef MS_NS
#define MS_NS 4              // mbarrier ring depth
#endif
#ifndef MS_FAST_FADD2
#define MS_FAST_FADD2 0      // packed FADD2 accumulation in the register sweep: measured slower (f16 K)
#endif
constexpr bool kFastFadd2 = MS_FAST_FADD2;
// packed (FMUL2.FTZ + FADD2, ms_common.cuh mac2) products in the binary32
// split sweeps; 0 = two scalar FMUL per K element
#ifndef MS_SWEEP_PK
#define MS_SWEEP_PK 1
#endif
#ifndef MS_PK_PREFETCH
#define MS_PK_PREFETCH 0   // software-pipelined K loads in the packed register sweep
#endif
constexpr int kFastThreads = MS_FAST_THREADS;
constexpr int kFastMinBlocks = MS_FAST_MINB;
constexpr int kFastWarps = kFastThreads / 32;
constexpr int kChunkCols = MS_CHUNK;
constexpr int kStagesNS = MS_NS;

template <class GS, bool SPLIT>
constexpr size_t fast_smem_bytes() {
  return (size_t)kStagesNS * (SPLIT ? 2 : 1) * kChunkCols * sizeof(GS) + 2 * kStagesNS * sizeof(uint64_t);
}

// Rows per warp per sweep.
template <class SS, class GS> struct FastRows {
  static constexpr int R = (sizeof(GS) == 8 || sizeof(SS) == 8) ? (MS_FAST_R > 4 ? 4 : MS_FAST_R) : MS_FAST_R;
};

// one 128-bit K vector per row against VEC staged columns (split: A += K s, B += K c;
// per-pair: A += G(x_i, x_j, K))
template <int MODEL, bool SPLIT, class SS, class GS, int KS, int R, int VEC>
__device__ __forceinline__ void sweep_step(const uint4 (&kv)[R], int nr, const GS (&s_loc)[VEC],
                                           const GS (&c_loc)[VEC], const GS (&xi)[R], const GS (&pref)[R],
                                           SS (&A)[R], SS (&B)[R]) {
#pragma unroll
  for (int k = 0; k < R; ++k) {
    if (k < nr) {
      float kf[VEC];
      KVec<KS>::unpack(kv[k], kf);
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        const GS kg = (GS)kf[v];
        if (SPLIT) {
          add2<SS, kFastFadd2>(A[k], B[k], (SS)mul<GS>(kg, s_loc[v]), (SS)mul<GS>(kg, c_loc[v]));
        } else {
          GS g;
          if (MODEL == MD_LCO) g = mul<GS>(kg, sub<GS>(s_loc[v], xi[k]));
          else g = mul<GS>(pref[k], mul<GS>(kg, fatan<GS>(sub<GS>(s_loc[v], xi[k]))));
          A[k] = add<SS>(A[k], (SS)g);
        }
      }
    }
  }
}

// ------------------------------------------------------------------------------
// rhs_fast: one persistent CTA per SM; the CTA owns a contiguous balanced row
// range; its 16 warps take rows round-robin and sweep all columns together,
// R rows per warp per sweep, so each staged chunk of column data is shared by
// 16*R rows. Per lane: one 128-bit K load per row per step. Row totals come
// from a warp-shuffle tree; the order of every row's sum depends only on N
// (not on the row partition), so sharded runs are bitwise identical.
template <int MODEL, bool SPLIT, class SS, class GS, int KS>
__global__ void __launch_bounds__(kFastThreads, kFastMinBlocks) k_rhs_fast(RhsArgs a) {
  msb::count_launch();
  pdl_enter();
  if (stage_skip(a.ctl, a.l, a.gate)) return;
  sweep_count(a);
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr int NCOL = SPLIT ? 2 : 1;
  constexpr int VEC = KVec<KS>::N;
  constexpr int COLS_IT = 32 * VEC;
  constexpr int R = FastRows<SS, GS>::R;
  GS* stage_buf = reinterpret_cast<GS*>(smem);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)kStagesNS * NCOL * kChunkCols * sizeof(GS));
  uint64_t* empty = full + kStagesNS;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t total = a.row1 - a.row0;
  const int rb = a.row0 + (int)(total * blockIdx.x / gridDim.x);
  const int re = a.row0 + (int)(total * (blockIdx.x + 1) / gridDim.x);
  const int nrows = re - rb;
  const int per_warp = (nrows + kFastWarps - 1) / kFastWarps;
  const int nsweeps = (per_warp + R - 1) / R;
  const int ld = (int)a.ld;
  const int nchunks = (ld + kChunkCols - 1) / kChunkCols;
  const int Q = nsweeps * nchunks;
  const GS* gin = reinterpret_cast<const GS*>(a.gin);

  auto chunk_cols = [&](int c) { return min(kChunkCols, ld - c * kChunkCols); };
  auto issue = [&](int q) {
    const int c = q % nchunks, st = q % kStagesNS;
    const int cc = chunk_cols(c);
    const uint32_t bytes = (uint32_t)(cc * sizeof(GS));
    mbar_expect_tx(&full[st], bytes * NCOL);
    // split: the (s_j, c_j) pairs of the chunk are one contiguous run
    bulk_g2s(stage_buf + (size_t)st * NCOL * kChunkCols, gin + (size_t)NCOL * c * kChunkCols, bytes * NCOL,
             &full[st]);
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStagesNS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kFastWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int q = 0; q < min(kStagesNS, Q); ++q) issue(q);

  constexpr bool kPk = SPLIT && sizeof(SS) == 4 && sizeof(GS) == 4 && KS != MS_K_SCALAR && MS_SWEEP_PK;
  const bool use_pk = kPk && a.pk && a.ctl->pk_off == 0;
  const SS mw = cvt<SS>(a.mw);
  const GS kscal = cvt<GS>(a.coupling_k);
  using KT = typename KElem<KS == MS_K_SCALAR ? MS_K_F32 : KS>::T;
  const KT* Kbase = reinterpret_cast<const KT*>(a.K);
  double* out = a.kb[a.out_slot == SLOT_K1 ? a.ctl->k1i : (a.out_slot == SLOT_KLAST ? a.S - a.ctl->k1i : a.out_slot)];
  bool nonfinite = false;
  const uint64_t kpol = a.k_stream ? l2_evict_first() : l2_evict_normal();

  int q = 0;
  for (int sw = 0; sw < nsweeps; ++sw) {
    int rows[R];
    GS xi[R], pref[R];
    int nr = 0;
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const int r = rb + warp + kFastWarps * (sw * R + k);
      rows[k] = r < re ? r : -1;
      if (r < re) nr = k + 1;
      xi[k] = GS(0);
      pref[k] = GS(0);
      if (!SPLIT && r < re) {
        xi[k] = gin[r];
        if (MODEL == MD_CC) pref[k] = reinterpret_cast<const GS*>(a.rowc)[r];
      }
    }
    SS A[R], B[R];
#pragma unroll
    for (int k = 0; k < R; ++k) { A[k] = SS(0); B[k] = SS(0); }
    uint64_t AB[R];
#pragma unroll
    for (int k = 0; k < R; ++k) AB[k] = 0ull;

    for (int c = 0; c < nchunks; ++c, ++q) {
      const int st = q % kStagesNS;
      const int cc = chunk_cols(c);
      mbar_wait(&full[st], (q / kStagesNS) & 1);
      const GS* sv = stage_buf + (size_t)(st * NCOL) * kChunkCols;  // split: (s, c) pairs
#ifndef MS_PREFETCH
#define MS_PREFETCH 0
#endif
      // fp64 accumulation (R = 4) gains from software pipelining, fp32 (R = 8)
      // from more rows in flight (tools/tune_rhs.py, profiles/r1_tune_rhs.txt)
      constexpr bool kPrefetch = MS_PREFETCH || (sizeof(SS) == 8 || sizeof(GS) == 8);
      if constexpr (kPk) {
        // binary32 split rows, packed products: the lane's (s, c) pairs are
        // read straight from the interleaved chunk, one FMUL2 + FADD2 per element
        if (nr > 0) {
          // row offsets of this chunk in 16-byte units (lane offset included);
          // a row past the CTA's range re-reads row rows[0] (valid memory) and
          // its sums are never written
          const uint4* kb4 = reinterpret_cast<const uint4*>(Kbase);
          uint32_t ko[R];  // < 2^32 x 16 B: K of up to 64 GB per handle
#pragma unroll
          for (int k = 0; k < R; ++k)
            ko[k] = (uint32_t)(((size_t)((k < nr ? rows[k] : rows[0]) - a.row0) * ld + (size_t)c * kChunkCols) / VEC +
                               lane);
          const uint4* sp = reinterpret_cast<const uint4*>(sv) + lane * (VEC / 2);
          const int nit = cc == kChunkCols ? kChunkCols / COLS_IT : (cc - lane * VEC + COLS_IT - 1) / COLS_IT;
#if MS_CHECKS
          for (int k = 0; k < R; ++k)
            MS_CHECK(nit <= 0 || ((size_t)ko[k] + (size_t)(nit - 1) * 32 + 1) * VEC <= (size_t)(a.row1 - a.row0) * ld,
                     "register sweep: K load past the handle's rows");
          MS_CHECK(nit <= 0 || (lane * (VEC / 2) + (nit - 1) * 16 * VEC + VEC / 2) * 16 <=
                                   (int)(NCOL * kChunkCols * sizeof(GS)), "register sweep: column pair past the chunk");
#endif
          auto sweep_chunk = [&](auto ftz) {
#if MS_PK_PREFETCH
          // software-pipelined: the next step's K vectors are in flight while
          // the current ones are consumed (twice the bytes in flight per thread)
          uint4 kn[R];
          if (nit > 0) {
#pragma unroll
            for (int k = 0; k < R; ++k) kn[k] = ldg_stream(kb4 + ko[k], kpol);
          }
#endif
#pragma unroll 1
          for (int it = 0; it < nit; ++it) {
            uint4 kv[R];
#if MS_PK_PREFETCH
#pragma unroll
            for (int k = 0; k < R; ++k) kv[k] = kn[k];
            if (it + 1 < nit) {
#pragma unroll
              for (int k = 0; k < R; ++k) kn[k] = ldg_stream(kb4 + ko[k] + (it + 1) * 32, kpol);
            }
#else
#pragma unroll
            for (int k = 0; k < R; ++k) kv[k] = ldg_stream(kb4 + ko[k] + it * 32, kpol);
#endif
            uint64_t pr[VEC];
#pragma unroll
            for (int v = 0; v < VEC / 2; ++v) {
              const uint4 qv = sp[it * 16 * VEC + v];
              pr[2 * v] = pk2u(qv.x, qv.y);
              pr[2 * v + 1] = pk2u(qv.z, qv.w);
            }
#pragma unroll
            for (int k = 0; k < R; ++k) {
              float kf[VEC];
              KVec<KS>::unpack(kv[k], kf);
#pragma unroll
              for (int v = 0; v < VEC; ++v) mac2<decltype(ftz)::value>(AB[k], pr[v], kf[v]);
            }
          }
          };
          if (use_pk) sweep_chunk(std::true_type{});
          else sweep_chunk(std::false_type{});  // unflushed products (Ctl::pk_off, MS_SWEEP_PK=off)
        }
      } else if (nr > 0 && kPrefetch && KS != MS_K_SCALAR) {
        // software-pipelined: the next step's K vectors are in flight while
        // the current ones are consumed
        const int c0 = c * kChunkCols;
        int col = lane * VEC;
        uint4 kv[R];
#pragma unroll
        for (int k = 0; k < R; ++k)
          if (k < nr && col < cc) kv[k] = ldg_stream(Kbase + (size_t)(rows[k] - a.row0) * ld + c0 + col, kpol);
        for (; col < cc; col += COLS_IT) {
          uint4 kn[R];
          const int nc = col + COLS_IT;
#pragma unroll
          for (int k = 0; k < R; ++k)
            if (k < nr && nc < cc) kn[k] = ldg_stream(Kbase + (size_t)(rows[k] - a.row0) * ld + c0 + nc, kpol);
          GS s_loc[VEC], c_loc[VEC];
#pragma unroll
          for (int v = 0; v < VEC; ++v) {
            s_loc[v] = sv[NCOL * (col + v)];
            if (SPLIT) c_loc[v] = sv[NCOL * (col + v) + 1];
          }
          sweep_step<MODEL, SPLIT, SS, GS, KS, R, VEC>(kv, nr, s_loc, c_loc, xi, pref, A, B);
#pragma unroll
          for (int k = 0; k < R; ++k) kv[k] = kn[k];
        }
      } else if (nr > 0) {
        const int c0 = c * kChunkCols;
        for (int col = lane * VEC; col < cc; col += COLS_IT) {
          GS s_loc[VEC], c_loc[VEC];
#pragma unroll
          for (int v = 0; v < VEC; ++v) {
            s_loc[v] = sv[NCOL * (col + v)];
            if (SPLIT) c_loc[v] = sv[NCOL * (col + v) + 1];
          }
          if constexpr (KS == MS_K_SCALAR) {
#pragma unroll
            for (int k = 0; k < R; ++k) {
              if (k >= nr) break;
#pragma unroll
              for (int v = 0; v < VEC; ++v) {
                if (SPLIT) {
                  add2<SS, kFastFadd2>(A[k], B[k], (SS)mul<GS>(kscal, s_loc[v]), (SS)mul<GS>(kscal, c_loc[v]));
                } else if (c0 + col + v < a.n) {
                  GS g;
                  if (MODEL == MD_LCO) g = mul<GS>(kscal, sub<GS>(s_loc[v], xi[k]));
                  else g = mul<GS>(pref[k], mul<GS>(kscal, fatan<GS>(sub<GS>(s_loc[v], xi[k]))));
                  A[k] = add<SS>(A[k], (SS)g);
                }
              }
            }
          } else {
            uint4 kv[R];
#pragma unroll
            for (int k = 0; k < R; ++k)
              if (k < nr) kv[k] = ldg_stream(Kbase + (size_t)(rows[k] - a.row0) * ld + c0 + col, kpol);
            sweep_step<MODEL, SPLIT, SS, GS, KS, R, VEC>(kv, nr, s_loc, c_loc, xi, pref, A, B);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
      if (warp == 0) {
        if (lane == 0 && q + kStagesNS < Q) {
          mbar_wait(&empty[st], (q / kStagesNS) & 1);
          issue(q + kStagesNS);
        }
        __syncwarp();
      }
    }
    if constexpr (kPk) {
#pragma unroll
      for (int k = 0; k < R; ++k) {
        float a0, b0;
        unpk2(AB[k], a0, b0);
        A[k] = a0;
        B[k] = b0;
      }
    }
    // warp-shuffle reduction of every row, then lane k writes row k
#pragma unroll
    for (int k = 0; k < R; ++k) {
#pragma unroll
      for (int m = 16; m >= 1; m >>= 1) {
        A[k] = add<SS>(A[k], shfl_xor(A[k], m));
        if (SPLIT) B[k] = add<SS>(B[k], shfl_xor(B[k], m));
      }
    }
#pragma unroll
    for (int k = 0; k < R; ++k) {
      if (lane == k && k < nr) {
        const int r = rows[k];
        SS coup;
        if (SPLIT) {
          const SS si = (SS)gin[2 * r], ci = (SS)gin[2 * r + 1];
          coup = mul<SS>(mw, sub<SS>(mul<SS>(ci, A[k]), mul<SS>(si, B[k])));
        } else {
          coup = mul<SS>(mw, A[k]);
        }
        MS_CHECK(r >= a.row0 && r < a.row1, "register sweep: output row outside the handle");
        const double o = ws_add(a.fvc[r], (double)coup, a.ws32);
        push_row(a.push, out + (int64_t)r * a.d + a.cs, o);
        nonfinite |= !isfinite(o);
      }
    }
  }
  push_fence(a.push);
  if (__any_sync(0xffffffffu, nonfinite) && lane == 0) atomicOr(a.nf_mask, 1 << a.l);
}

// ------------------------------------------------------------------------------
// eval_fused: prep + sweep of one evaluation in ONE launch, for systems whose
// column data fits in shared memory (the BASELINE C1-C3 sizes). Every CTA
// recomputes the column value(s) of all N agents from the stage combination
// (slot 0 only: O(N) work, no transcendental but the split's sin/cos) into
// shared memory and runs the full per-agent prep for its own rows only; then
// it sweeps its rows exactly like k_rhs_fast (same lane/column order, same
// shuffle tree: the result is bit-identical to prep + k_rhs_fast). Small
// evaluations are latency-bound, and this removes one launch and one
// dependent global round trip per stage.
constexpr size_t kFusedMaxSmem = 96 * 1024;
#ifndef MS_FUSED_R
#define MS_FUSED_R 1
#endif
#ifndef MS_FUSED_UNROLL
#define MS_FUSED_UNROLL 8
#endif
#define MS_PRAGMA(x) _Pragma(#x)
#define MS_UNROLL(n) MS_PRAGMA(unroll n)

// PREPPED: the column values were written by k_prep (gin) and are only staged
// into shared memory — the split Kuramoto's sin/cos are too costly to recompute
// in every CTA, but its small sweeps gain from the same one-row-per-warp,
// unrolled loop.
template <int MODEL, bool SPLIT, class FS, class SS, class GS, int KS, bool PREPPED = false>
__global__ void __launch_bounds__(kFastThreads, kFastMinBlocks) k_eval_fused(PrepArgs p, RhsArgs a) {
  msb::count_launch();
  pdl_enter();
  if (stage_skip(a.ctl, a.l, a.gate)) return;
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr int VEC = KVec<KS>::N;
  constexpr int COLS_IT = 32 * VEC;
  // few rows per CTA at these sizes: 1 row per warp and the column loop
  // unrolled, so a lane's K loads of several steps are in flight together
  constexpr int R = MS_FUSED_R;
  GS* colv = reinterpret_cast<GS*>(smem);  // [NCOL][ld]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t total = a.row1 - a.row0;
  const int rb = a.row0 + (int)(total * blockIdx.x / gridDim.x);
  const int re = a.row0 + (int)(total * (blockIdx.x + 1) / gridDim.x);
  const int ld = (int)a.ld, n = p.md.n, d = p.md.d;

  // ---- phase 1: column values of all agents; full prep of this CTA's rows
  const PrepCtx c = prep_ctx(p);
  if (!PREPPED && blockIdx.x == 0 && threadIdx.x == 0) prep_count(p, c.ctl);
  bool nonfinite = false;
  for (int j = threadIdx.x; j < ld; j += blockDim.x) {
    if (PREPPED) {
      const GS* g = reinterpret_cast<const GS*>(a.gin);
      if (SPLIT) {
        colv[j] = j < n ? g[2 * j] : GS(0);
        colv[ld + j] = j < n ? g[2 * j + 1] : GS(0);
      } else {
        colv[j] = j < n ? g[j] : GS(0);
      }
    } else if (j < n) {
      const GS xg = cvt<GS>(prep_arg(p, c, (int64_t)j * d, false));
      if (SPLIT) {
        GS sv, cv;
        dsincos(xg, &sv, &cv);
        colv[j] = sv;
        colv[ld + j] = cv;
      } else {
        colv[j] = xg;
      }
    } else {
      colv[j] = GS(0);
      if (SPLIT) colv[ld + j] = GS(0);
    }
  }
  if (!PREPPED)
    for (int i = rb + (int)threadIdx.x; i < re; i += blockDim.x) nonfinite |= prep_agent<MODEL, FS, GS>(p, c, i);
  __syncthreads();  // own rows' gin/fvc/rowc (global) and the column values (shared)

  // ---- phase 2: the sweep of k_rhs_fast over one whole-width chunk
  const int nrows = re - rb;
  const int per_warp = (nrows + kFastWarps - 1) / kFastWarps;
  const int nsweeps = (per_warp + R - 1) / R;
  const GS* gin = reinterpret_cast<const GS*>(a.gin);
  const SS mw = cvt<SS>(a.mw);
  const GS kscal = cvt<GS>(a.coupling_k);
  using KT = typename KElem<KS == MS_K_SCALAR ? MS_K_F32 : KS>::T;
  const KT* Kbase = reinterpret_cast<const KT*>(a.K);
  double* out = c.out;
  const GS* sv = colv;
  const GS* cv = colv + ld;
  for (int sw = 0; sw < nsweeps; ++sw) {
    int rows[R];
    GS xi[R], pref[R];
    int nr = 0;
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const int r = rb + warp + kFastWarps * (sw * R + k);
      rows[k] = r < re ? r : -1;
      if (r < re) nr = k + 1;
      xi[k] = GS(0);
      pref[k] = GS(0);
      if (!SPLIT && r < re) {
        xi[k] = gin[r];
        if (MODEL == MD_CC) pref[k] = reinterpret_cast<const GS*>(a.rowc)[r];
      }
    }
    SS A[R], B[R];
#pragma unroll
    for (int k = 0; k < R; ++k) { A[k] = SS(0); B[k] = SS(0); }
    if (nr > 0) {
      MS_UNROLL(MS_FUSED_UNROLL)
      for (int col = lane * VEC; col < ld; col += COLS_IT) {
        GS s_loc[VEC], c_loc[VEC];
#pragma unroll
        for (int v = 0; v < VEC; ++v) {
          s_loc[v] = sv[col + v];
          if (SPLIT) c_loc[v] = cv[col + v];
        }
        if constexpr (KS == MS_K_SCALAR) {
#pragma unroll
          for (int k = 0; k < R; ++k) {
            if (k >= nr) break;
#pragma unroll
            for (int v = 0; v < VEC; ++v) {
              if (SPLIT) {
                add2<SS, kFastFadd2>(A[k], B[k], (SS)mul<GS>(kscal, s_loc[v]), (SS)mul<GS>(kscal, c_loc[v]));
              } else if (col + v < a.n) {
                GS g;
                if (MODEL == MD_LCO) g = mul<GS>(kscal, sub<GS>(s_loc[v], xi[k]));
                else g = mul<GS>(pref[k], mul<GS>(kscal, fatan<GS>(sub<GS>(s_loc[v], xi[k]))));
                A[k] = add<SS>(A[k], (SS)g);
              }
            }
          }
        } else {
          uint4 kv[R];
#pragma unroll
          for (int k = 0; k < R; ++k)
            if (k < nr) kv[k] = ldg_stream(Kbase + (size_t)(rows[k] - a.row0) * ld + col);
          sweep_step<MODEL, SPLIT, SS, GS, KS, R, VEC>(kv, nr, s_loc, c_loc, xi, pref, A, B);
        }
      }
    }
#pragma unroll
    for (int k = 0; k < R; ++k) {
#pragma unroll
      for (int m = 16; m >= 1; m >>= 1) {
        A[k] = add<SS>(A[k], shfl_xor(A[k], m));
        if (SPLIT) B[k] = add<SS>(B[k], shfl_xor(B[k], m));
      }
    }
#pragma unroll
    for (int k = 0; k < R; ++k) {
      if (lane == k && k < nr) {
        const int r = rows[k];
        SS coup;
        if (SPLIT) {
          const SS si = (SS)gin[2 * r], ci = (SS)gin[2 * r + 1];
          coup = mul<SS>(mw, sub<SS>(mul<SS>(ci, A[k]), mul<SS>(si, B[k])));
        } else {
          coup = mul<SS>(mw, A[k]);
        }
        const double o = ws_add(a.fvc[r], (double)coup, a.ws32);
        push_row(a.push, out + (int64_t)r * a.d + a.cs, o);
        nonfinite |= !isfinite(o);
      }
    }
  }
  push_fence(a.push);
  if (__any_sync(0xffffffffu, nonfinite) && lane == 0) atomicOr(a.nf_mask, 1 << a.l);
}

// ------------------------------------------------------------------------------
// rhs_tma: the split-Kuramoto K sweep with K itself streamed by cp.async.bulk.
// The register-fed sweep above keeps ~64 KB of K in flight per SM, the
// register file's limit, and tops out near 6.5 TB/s; a plain read probe needs
// ~4x that in flight to reach ~7.3 TB/s (tools/bw_probe.cu). Here the bytes
// in flight live in shared memory: one producer warp streams, per stage, the
// row segments [TC columns] of a row group plus the matching s/c columns
// into a 3-deep ring (~216 KB); the consumer warps (TmaGeom::CONS) own RPW rows
// each of the group and sum them from shared memory. Lane l handles columns 4l + 128m
// (8l + 256m for 16-bit K) in ascending order, exactly like k_rhs_fast, so
// both sweeps produce bit-identical rows.
#ifndef MS_TMA_LANES
#define MS_TMA_LANES 1     // 1: the whole producer warp issues the row copies
#endif
// per (GS, K storage): rows per consumer warp and K bytes per stage, chosen by
// tools/tune_rhs.py (profiles/r1_tune_tma.txt); macros override for tuning
#ifndef MS_TMA_RPW_F32
#define MS_TMA_RPW_F32 1
#endif
#ifndef MS_TMA_KB_F32
#define MS_TMA_KB_F32 65536
#endif
#ifndef MS_TMA_RPW_F64
#define MS_TMA_RPW_F64 2
#endif
#ifndef MS_TMA_KB_F64
#define MS_TMA_KB_F64 65536
#endif
#ifndef MS_TMA_KB_K16
#define MS_TMA_KB_K16 65536
#endif
#ifndef MS_TMA_RPW_K16
#define MS_TMA_RPW_K16 4
#endif
#ifndef MS_TMA_CONS
#define MS_TMA_CONS 16
#endif
#ifndef MS_TMA_CONS_K16
#define MS_TMA_CONS_K16 8
#endif
#ifndef MS_TMA_STAGES
#define MS_TMA_STAGES 4
#endif
// the all-binary32 row (SSS, f32 K) runs 8 consumer warps x 2 rows: half the
// s/c shared-memory reads per K element, +3 % sustained under the board's power
// cap (profiles/r1_sustained_sweep.txt); rows with binary64 sums or columns keep
// 16 warps to hide their f64/XU latency
#ifndef MS_TMA_KHINT
#define MS_TMA_KHINT 1
#endif
#ifndef MS_TMA_CONS_SSS
#define MS_TMA_CONS_SSS 8
#endif
#ifndef MS_TMA_RPW_SSS
#define MS_TMA_RPW_SSS 2
#endif
constexpr int kTmaConsMax = MS_TMA_CONS > MS_TMA_CONS_SSS ? MS_TMA_CONS : MS_TMA_CONS_SSS;
constexpr int kTmaThreadsMax = ((kTmaConsMax > MS_TMA_CONS_K16 ? kTmaConsMax : MS_TMA_CONS_K16) + 1) * 32;
constexpr int kTmaStages = MS_TMA_STAGES;
#ifndef MS_TMA_UNROLL
#define MS_TMA_UNROLL 4    // column steps unrolled in the full-tile consumer loop
#endif
#ifndef MS_TMA_MINB
#define MS_TMA_MINB 1      // resident CTAs per SM (grid = SMs x MINB; the ring must fit MINB times)
#endif
constexpr int kTmaUnroll = MS_TMA_UNROLL;

template <class SS, class GS, int KS>
struct TmaGeom {
  using KT = typename KElem<KS>::T;
  static constexpr bool SSS = sizeof(SS) == 4 && sizeof(GS) == 4 && sizeof(KT) == 4;
  static constexpr int CONS = SSS ? MS_TMA_CONS_SSS : (sizeof(KT) == 2 ? MS_TMA_CONS_K16 : MS_TMA_CONS);  // consumer warps
  static constexpr int THREADS = (CONS + 1) * 32;
  static constexpr int RPW = SSS ? MS_TMA_RPW_SSS
                                 : (sizeof(KT) == 2 ? MS_TMA_RPW_K16 : (sizeof(GS) == 8 ? MS_TMA_RPW_F64 : MS_TMA_RPW_F32));
  static constexpr int RG = CONS * RPW;  // rows per group
  static constexpr int KBYTES = sizeof(KT) == 2 ? MS_TMA_KB_K16 : (sizeof(GS) == 8 ? MS_TMA_KB_F64 : MS_TMA_KB_F32);
  static constexpr int TC = KBYTES / (RG * (int)sizeof(KT));   // columns per tile
  static constexpr int SC_BYTES = 2 * TC * (int)sizeof(GS);
  static constexpr int STAGE_BYTES = KBYTES + SC_BYTES;
  static constexpr int NS = (232448 / MS_TMA_MINB - 1536) / STAGE_BYTES < kTmaStages ? (232448 / MS_TMA_MINB - 1536) / STAGE_BYTES : kTmaStages;
  static constexpr size_t SMEM = (size_t)NS * STAGE_BYTES + 2 * kTmaStages * sizeof(uint64_t) + 128;
  static_assert(TC % (32 * KVec<KS>::N) == 0, "tile width must be a whole number of warp steps");
};

// One warp step of the TMA sweep: lane columns [col, col + VEC) of the
// staged tile against each of the warp's rows (A += K s, B += K c; ascending
// columns per lane, as in k_rhs_fast).
template <class SS, class GS, int KS, int RPW, int TC, bool CHECK>
__device__ __forceinline__ void tma_col_step(const unsigned char* sk, const GS* sc, int col,
                                             const int (&rows)[RPW], int nr, SS (&A)[RPW], SS (&B)[RPW]) {
  using KT = typename KElem<KS>::T;
  constexpr int VEC = KVec<KS>::N;
  GS s_loc[VEC], c_loc[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) {
    s_loc[v] = sc[2 * (col + v)];
    c_loc[v] = sc[2 * (col + v) + 1];
  }
#pragma unroll
  for (int k = 0; k < RPW; ++k) {
    if (!CHECK || k < nr) {
      const uint4 kv = *reinterpret_cast<const uint4*>(sk + ((size_t)rows[k] * TC + col) * sizeof(KT));
      float kf[VEC];
      KVec<KS>::unpack(kv, kf);
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        const GS kg = (GS)kf[v];
        add2<SS>(A[k], B[k], (SS)mul<GS>(kg, s_loc[v]), (SS)mul<GS>(kg, c_loc[v]));
      }
    }
  }
}

// The same warp step for binary32 sums and columns with packed accumulators
// AB[k] = {A_k, B_k}: the lane's (s, c) pairs come straight from the
// interleaved staged columns (LDS.128 = two pairs), one FMUL2 + one FADD2 per
// K element (mac2). Bit-identical to tma_col_step (same products, same sums,
// same order).
template <int KS, int RPW, int TC, bool CHECK>
__device__ __forceinline__ void tma_col_step_pk(const unsigned char* sk, const float* sc, int col,
                                                const int (&rows)[RPW], int nr, uint64_t (&AB)[RPW]) {
  using KT = typename KElem<KS>::T;
  constexpr int VEC = KVec<KS>::N;
  uint64_t pr[VEC];
  const uint4* sp = reinterpret_cast<const uint4*>(sc + 2 * col);
#pragma unroll
  for (int v = 0; v < VEC / 2; ++v) {
    const uint4 q = sp[v];
    pr[2 * v] = pk2u(q.x, q.y);
    pr[2 * v + 1] = pk2u(q.z, q.w);
  }
#pragma unroll
  for (int k = 0; k < RPW; ++k) {
    if (!CHECK || k < nr) {
      const uint4 kv = *reinterpret_cast<const uint4*>(sk + ((size_t)rows[k] * TC + col) * sizeof(KT));
      float kf[VEC];
      KVec<KS>::unpack(kv, kf);
#pragma unroll
      for (int v = 0; v < VEC; ++v) mac2<true>(AB[k], pr[v], kf[v]);
    }
  }
}

// NEXT: the prep of the attempt's next stage (pn) runs at the end of this
// sweep, for this CTA's own rows: every per-agent input of that prep (x, the
// k slots including the k_l this CTA just wrote) is row-local, so only the
// column data needs another buffer (pn.B.gin: the other CTAs still read this
// stage's). The arithmetic is prep_agent's, so the results are bit-identical to
// k_prep + sweep; host side: launch_attempt (fuse_next_ok in ms_rhs_fast.cu).
#ifndef MS_TMA_KEEP
#define MS_TMA_KEEP 0
#endif
template <class SS, class GS, int KS, bool NEXT = false>
__global__ void __launch_bounds__(kTmaThreadsMax, MS_TMA_MINB) k_rhs_tma(RhsArgs a, PrepArgs pn) {
  msb::count_launch();
  pdl_enter();
  if (stage_skip(a.ctl, a.l, a.gate)) return;
  sweep_count(a);
  using G = TmaGeom<SS, GS, KS>;
  using KT = typename G::KT;
  constexpr int VEC = KVec<KS>::N;
  constexpr int COLS_IT = 32 * VEC;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)G::NS * G::STAGE_BYTES);
  uint64_t* empty = full + G::NS;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t total = a.row1 - a.row0;
  const int rb = a.row0 + (int)(total * blockIdx.x / gridDim.x);
  const int re = a.row0 + (int)(total * (blockIdx.x + 1) / gridDim.x);
  const int ngroups = (re - rb + G::RG - 1) / G::RG;
  const int ld = (int)a.ld;
  const int ntiles = (ld + G::TC - 1) / G::TC;
  const int Q = ngroups * ntiles;
  const GS* gin = reinterpret_cast<const GS*>(a.gin);
  const KT* Kbase = reinterpret_cast<const KT*>(a.K);

  if (threadIdx.x == 0) {
    for (int s = 0; s < G::NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], G::CONS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();

  if (warp == G::CONS) {  // producer warp
#if MS_TMA_KHINT
    // K is streamed once per evaluation: evict it first; the s/c columns are
    // re-read by every CTA
    const uint64_t pol_k = a.k_stream ? l2_evict_first() : l2_evict_normal(), pol_sc = l2_evict_last();
#endif
    for (int q = 0; q < Q; ++q) {
      const int st = q % G::NS;
      if (q >= G::NS) {
        if (lane == 0) mbar_wait(&empty[st], ((q / G::NS) & 1) ^ 1);
        __syncwarp();
      }
      const int g = q / ntiles, t = q % ntiles;
      const int r0 = rb + g * G::RG;
      const int nr = min(G::RG, re - r0);
      const int c0 = t * G::TC;
      const int cc = min(G::TC, ld - c0);
      const uint32_t kbytes = (uint32_t)(cc * sizeof(KT));
      const uint32_t sbytes = (uint32_t)(cc * sizeof(GS));
      MS_CHECK(r0 >= a.row0 && r0 + nr <= a.row1 && c0 + cc <= ld && nr <= G::RG && cc <= G::TC,
               "TMA sweep: tile outside the handle");
      unsigned char* sk = smem + (size_t)st * G::STAGE_BYTES;
      GS* ss = reinterpret_cast<GS*>(sk + G::KBYTES);
      if (lane == 0) {
        mbar_expect_tx(&full[st], kbytes * nr + 2 * sbytes);
        // the tile's (s_j, c_j) pairs: one contiguous run of the interleaved column data
#if MS_TMA_KHINT
        bulk_g2s_hint(ss, gin + 2 * (size_t)c0, 2 * sbytes, &full[st], pol_sc);
#else
        bulk_g2s(ss, gin + 2 * (size_t)c0, 2 * sbytes, &full[st]);
#endif
      }
      if (MS_TMA_LANES) {
        for (int r = lane; r < nr; r += 32)
#if MS_TMA_KHINT
          // the first MS_TMA_KEEP rows of every CTA's range stay in L2 across
          // evaluations (evict-last); the rest of a streamed K is evict-first
          bulk_g2s_hint(sk + (size_t)r * G::TC * sizeof(KT), Kbase + (size_t)(r0 + r - a.row0) * ld + c0, kbytes,
                        &full[st], (a.k_stream && r0 + r < rb + MS_TMA_KEEP) ? pol_sc : pol_k);
#else
          bulk_g2s(sk + (size_t)r * G::TC * sizeof(KT), Kbase + (size_t)(r0 + r - a.row0) * ld + c0, kbytes,
                   &full[st]);
#endif
      } else if (lane == 0) {
        for (int r = 0; r < nr; ++r)
          bulk_g2s(sk + (size_t)r * G::TC * sizeof(KT), Kbase + (size_t)(r0 + r - a.row0) * ld + c0, kbytes,
                   &full[st]);
      }
      __syncwarp();
    }
    return;
  }

  // consumers: warp w owns rows w, w + CONS, ... of every group
  constexpr bool kPk = sizeof(SS) == 4 && sizeof(GS) == 4 && MS_SWEEP_PK;
  const bool use_pk = kPk && a.pk && a.ctl->pk_off == 0;
  const SS mw = cvt<SS>(a.mw);
  double* out = a.kb[a.out_slot == SLOT_K1 ? a.ctl->k1i : (a.out_slot == SLOT_KLAST ? a.S - a.ctl->k1i : a.out_slot)];
  bool nonfinite = false;
  int q = 0;
  for (int g = 0; g < ngroups; ++g) {
    const int r0 = rb + g * G::RG;
    int rows[G::RPW];
    int nr = 0;
#pragma unroll
    for (int k = 0; k < G::RPW; ++k) {
      const int rl = warp + G::CONS * k;  // local row in the group
      rows[k] = (r0 + rl < re) ? rl : -1;
      if (r0 + rl < re) nr = k + 1;
    }
    SS A[G::RPW], B[G::RPW];
#pragma unroll
    for (int k = 0; k < G::RPW; ++k) { A[k] = SS(0); B[k] = SS(0); }
    uint64_t AB[G::RPW];
#pragma unroll
    for (int k = 0; k < G::RPW; ++k) AB[k] = 0ull;
    for (int t = 0; t < ntiles; ++t, ++q) {
      const int st = q % G::NS;
      const int cc = min(G::TC, ld - t * G::TC);
      mbar_wait(&full[st], (q / G::NS) & 1);
      const unsigned char* sk = smem + (size_t)st * G::STAGE_BYTES;
      const GS* sc = reinterpret_cast<const GS*>(sk + G::KBYTES);  // (s, c) pairs
      if (kPk && use_pk) {
        const float* scf = reinterpret_cast<const float*>(sc);
        if (nr == G::RPW && cc == G::TC) {
#pragma unroll kTmaUnroll
          for (int it = 0; it < G::TC / COLS_IT; ++it)
            tma_col_step_pk<KS, G::RPW, G::TC, false>(sk, scf, lane * VEC + it * COLS_IT, rows, nr, AB);
        } else if (nr > 0) {
          for (int col = lane * VEC; col < cc; col += COLS_IT)
            tma_col_step_pk<KS, G::RPW, G::TC, true>(sk, scf, col, rows, nr, AB);
        }
      } else if (nr == G::RPW && cc == G::TC) {
        // full tile, every row valid: a fixed trip count the compiler unrolls,
        // so the shared-memory loads of later column steps are issued ahead
#pragma unroll kTmaUnroll
        for (int it = 0; it < G::TC / COLS_IT; ++it)
          tma_col_step<SS, GS, KS, G::RPW, G::TC, false>(sk, sc, lane * VEC + it * COLS_IT, rows, nr, A, B);
      } else if (nr > 0) {
        for (int col = lane * VEC; col < cc; col += COLS_IT)
          tma_col_step<SS, GS, KS, G::RPW, G::TC, true>(sk, sc, col, rows, nr, A, B);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
    if (kPk && use_pk) {
#pragma unroll
      for (int k = 0; k < G::RPW; ++k) {
        float a0, b0;
        unpk2(AB[k], a0, b0);
        A[k] = a0;
        B[k] = b0;
      }
    }
#pragma unroll
    for (int k = 0; k < G::RPW; ++k) {
#pragma unroll
      for (int m = 16; m >= 1; m >>= 1) {
        A[k] = add<SS>(A[k], shfl_xor(A[k], m));
        B[k] = add<SS>(B[k], shfl_xor(B[k], m));
      }
    }
#pragma unroll
    for (int k = 0; k < G::RPW; ++k) {
      if (lane == k && k < nr) {
        const int r = r0 + rows[k];
        MS_CHECK(r >= a.row0 && r < a.row1, "TMA sweep: output row outside the handle");
        const SS si = (SS)gin[2 * r], ci = (SS)gin[2 * r + 1];
        const SS coup = mul<SS>(mw, sub<SS>(mul<SS>(ci, A[k]), mul<SS>(si, B[k])));
        const double o = ws_add(a.fvc[r], (double)coup, a.ws32);
        push_row(a.push, out + (int64_t)r * a.d + a.cs, o);
        nonfinite |= !isfinite(o);
      }
    }
  }
  push_fence(a.push);
  if (__any_sync(0xffffffffu, nonfinite) && lane == 0) atomicOr(a.nf_mask, 1 << a.l);
  if constexpr (NEXT) {
    // the k_l rows of this CTA are written by the consumer warps (the producer
    // warp has returned): a named barrier over the consumers only
    asm volatile("bar.sync 1, %0;" ::"r"(G::CONS * 32) : "memory");
    const PrepCtx c = prep_ctx(pn);
    bool nfp = false;
    for (int i = rb + (int)threadIdx.x; i < re; i += G::CONS * 32) nfp |= prep_agent<MD_KUR, SS, GS>(pn, c, i);
    if (__any_sync(0xffffffffu, nfp) && lane == 0) atomicOr(a.nf_mask, 1 << pn.l);
    if (blockIdx.x == 0) {  // the padding columns of the target buffer (k_prep does the same)
      GS* g = reinterpret_cast<GS*>(pn.B.gin);
      for (int j = pn.md.n + (int)threadIdx.x; j < pn.ld; j += G::CONS * 32) {
        g[2 * j] = GS(0);
        g[2 * j + 1] = GS(0);
      }
    }
  }
}

// ------------------------------------------------------------------------------
// rhs_seq: every row's coupling sum in eval_core's exact order
// (systems.cpp:50-57): ascending j including j = i, acc = acc (+) term_j in SS,
// with term_j = mw * (SS)G_ij (faithful: per-pair G in GS with RN_GS(K_ij))
// or, for the Kuramoto split in sequential order (MS_RHS_ORDERED), the pair
// (RN_SS(K s_j), RN_SS(K c_j)) and the coupling mw (c_i A - s_i B) at the end —
// the oracle's split form bit for bit (up to the libm ulp of sin/cos).
// Only the additions are sequential: a CTA owns kSeqRows rows; per tile of
// kSeqCols columns its warps 1..7 compute the terms of all (row, column) pairs
// in parallel (K read row-major, coalesced along j) into a double-buffered
// shared tile, while warp 0 (lane = row) adds the previous tile's terms in
// ascending j. Terms of a tile are summed only after the tile is complete.
constexpr int kSeqRows = 32, kSeqThreads = 256;
template <class SS, bool SPLIT> struct SeqGeom {
  static constexpr int COLS = sizeof(SS) == 8 && SPLIT ? 64 : 128;   // columns per tile
  static constexpr int PITCH = COLS + 1;                              // conflict-free row reads
  static constexpr int NACC = SPLIT ? 2 : 1;
  static constexpr size_t SMEM = (size_t)2 * NACC * kSeqRows * PITCH * sizeof(SS);
};

template <int MODEL, bool SPLIT, class SS, class GS, int KS>
__global__ void __launch_bounds__(kSeqThreads) k_rhs_seq(RhsArgs a) {
  msb::count_launch();
  pdl_enter();
  if (stage_skip(a.ctl, a.l, a.gate)) return;
  sweep_count(a);
  using Gm = SeqGeom<SS, SPLIT>;
  constexpr int TC = Gm::COLS, P = Gm::PITCH, NA = Gm::NACC;
  extern __shared__ __align__(16) unsigned char seq_smem[];
  SS* tile = reinterpret_cast<SS*>(seq_smem);  // [2][NA][kSeqRows][P]
  const int r0 = a.row0 + blockIdx.x * kSeqRows;
  const int nrows = min(kSeqRows, a.row1 - r0);
  const int n = a.n;
  const int ntiles = (n + TC - 1) / TC;
  const GS* gin = reinterpret_cast<const GS*>(a.gin);
  const SS mw = cvt<SS>(a.mw);
  const GS kscal = cvt<GS>(a.coupling_k);
  using KT = typename KElem<KS == MS_K_SCALAR ? MS_K_F32 : KS>::T;
  const KT* K = reinterpret_cast<const KT*>(a.K);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  auto compute = [&](int t, int buf) {  // warps 1..7: the terms of tile t
    const int j0 = t * TC;
    for (int q = threadIdx.x - 32; q < kSeqRows * TC; q += kSeqThreads - 32) {
      const int rr = q / TC, jj = q % TC, j = j0 + jj;
      if (rr >= nrows || j >= n) continue;
      const int r = r0 + rr;
      GS kg;
      MS_CHECK(r >= a.row0 && r < a.row1 && j < a.n && j <= a.ld, "seq sweep: K index");
      if constexpr (KS == MS_K_SCALAR) kg = kscal;
      else kg = (GS)k2f(K[(size_t)(r - a.row0) * a.ld + j]);
      SS* dst = tile + ((size_t)buf * NA * kSeqRows + rr) * P + jj;
      MS_CHECK((size_t)((dst - tile) + (NA - 1) * kSeqRows * P + 1) * sizeof(SS) <= Gm::SMEM, "seq sweep: tile index");
      if constexpr (SPLIT) {
        dst[0] = (SS)mul<GS>(kg, gin[2 * j]);
        dst[kSeqRows * P] = (SS)mul<GS>(kg, gin[2 * j + 1]);
      } else {
        const GS xi = gin[r];
        const GS diff = sub<GS>(gin[j], xi);
        GS g;
        if (MODEL == MD_LCO) g = mul<GS>(kg, diff);
        else if (MODEL == MD_KUR) g = mul<GS>(kg, dsin<GS>(diff));
        else g = mul<GS>(reinterpret_cast<const GS*>(a.rowc)[r], mul<GS>(kg, datan<GS>(diff)));
        dst[0] = mul<SS>(mw, (SS)g);
      }
    }
  };
  SS A = SS(0), Bc = SS(0);
  if (warp != 0) compute(0, 0);
  __syncthreads();
  for (int t = 0; t < ntiles; ++t) {
    const int buf = t & 1;
    if (warp == 0) {
      if (lane < nrows) {
        const SS* row = tile + ((size_t)buf * NA * kSeqRows + lane) * P;
        const int cols = min(TC, n - t * TC);
        for (int jj = 0; jj < cols; ++jj) {
          A = add<SS>(A, row[jj]);
          if constexpr (SPLIT) Bc = add<SS>(Bc, row[kSeqRows * P + jj]);
        }
      }
    } else if (t + 1 < ntiles) {
      compute(t + 1, buf ^ 1);
    }
    __syncthreads();
  }
  bool nonfinite = false;
  if (warp == 0 && lane < nrows) {
    const int r = r0 + lane;
    SS coup;
    if constexpr (SPLIT) {
      const SS si = (SS)gin[2 * r], ci = (SS)gin[2 * r + 1];
      coup = mul<SS>(mw, sub<SS>(mul<SS>(ci, A), mul<SS>(si, Bc)));
    } else {
      coup = A;
    }
    double* out = a.kb[a.out_slot == SLOT_K1 ? a.ctl->k1i : (a.out_slot == SLOT_KLAST ? a.S - a.ctl->k1i : a.out_slot)];
    const double o = ws_add(a.fvc[r], (double)coup, a.ws32);
    push_row(a.push, out + (int64_t)r * a.d + a.cs, o);
    nonfinite = !isfinite(o);
  }
  push_fence(a.push);
  if (warp == 0 && __any_sync(0xffffffffu, nonfinite) && lane == 0) atomicOr(a.nf_mask, 1 << a.l);
}

// ------------------------------------------------------------------------------
// controller helpers (solver.cpp:413-418, 272-314)
__device__ __forceinline__ double d_clamp(double v, double lo, double hi) {
  return v < lo ? lo : (hi < v ? hi : v);  // std::clamp
}
__device__ __forceinline__ double d_adjust_step(double h, double err, double rel, double safety,
                                                double fac_min, double fac_max, double ctrl_exp) {
  if (err <= 0.0) return __dmul_rn(h, fac_max);
  const double fac = __dmul_rn(safety, pow_cr(__ddiv_rn(rel, err), ctrl_exp));
  return __dmul_rn(h, d_clamp(fac, fac_min, fac_max));
}
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// top of the solve_core loop (solver.cpp:273-296) and the final-step clip (:309-314)
__device__ inline void loop_check(Ctl* c) {
  if (c->n_acc + c->n_fail >= c->max_iterations) {
    c->status = MS_MAX_ITERATIONS; c->done = 1; return;
  }
  if (c->n_fail >= c->max_failed) {
    c->status = MS_MAX_FAILED_STEPS; c->done = 1; return;
  }
  if (c->time_limits) {
    const double el = (double)(globaltimer_ns() - c->t_start_ns) * 1e-9;
    if (el > c->wall_clock_limit) {
      c->status = MS_WALL_CLOCK; c->done = 1; return;
    }
    if (el > c->slow_elapsed &&
        __dsub_rn(c->t, c->t0) < __dmul_rn(c->slow_progress, __dsub_rn(c->tf, c->t0))) {
      c->status = MS_SLOW_SOLVER; c->done = 1; return;
    }
  }
  if (c->h <= c->h_min) {
    c->status = MS_STEP_TOO_SMALL; c->done = 1; return;
  }
  c->last = 0;
  c->h_att = c->h;
  if (__dadd_rn(c->t, __dmul_rn(1.01, c->h)) >= c->tf) {
    c->h_att = __dsub_rn(c->tf, c->t);
    c->last = 1;
  }
}

enum : int { FIN_SOLVE = 0, FIN_STEP = 1 };

struct FinArgs {
  Bufs B;
  int S;
  int nbt;
  double bt[kMaxStages];
  int bslot[kMaxStages];
  int64_t dn;
  int mode;
  int k1_elided;
  int write_xt;
  int has_handle;
  int fixed_k1;  // host-driven sharded loop: k1 stays in slot 0 (k_fsal_copy), no ping-pong
  int ctl_smem;  // run the controller on a shared-memory copy of Ctl (MS_CTL_SMEM, default on)
  cudaGraphConditionalHandle handle;
};

// The controller's ~40 dependent field reads and writes of the control block
// are global round trips when it runs on Ctl in place; on a shared-memory copy
// (copied in and out by the whole block: one round trip each) they are not.
static_assert(sizeof(Ctl) % 8 == 0, "Ctl is copied as 64-bit words");
constexpr int kCtlWords = (int)(sizeof(Ctl) / 8);
__device__ __forceinline__ void ctl_copy(void* dst, const void* src) {
  for (int w = threadIdx.x; w < kCtlWords; w += blockDim.x)
    static_cast<uint64_t*>(dst)[w] = static_cast<const uint64_t*>(src)[w];
}

constexpr int kFinThreads = 256;
// small state vectors: one 1024-thread block does the whole reduction and the
// controller, without the grid ticket (one dependent round trip fewer)
constexpr int kFinSmallThreads = 1024;
#ifndef MS_FIN_SMALL_MAX
#define MS_FIN_SMALL_MAX 2048
#endif
constexpr int64_t kFinSmallMax = MS_FIN_SMALL_MAX;  // measured: C1 (2048) -3 %, C3 (8192) +20 % per attempt

__device__ __forceinline__ double nan64() { return __longlong_as_double(0x7ff8000000000000ll); }

// Running max of RN(a_i / w_i) (the weighted error norm, solver.cpp:403-408)
// without a division per element: rounding is monotone, so the max of the
// rounded quotients is RN of the largest exact quotient. Candidates are
// compared exactly, a1 w2 vs a2 w1 as (RN product, FMA remainder) pairs, and
// one division per thread remains (value()). Elements whose quotient is not a
// regular one (w == 0, a not finite, factors outside [1e-140, 1e140]) take
// the division directly, combined with fmax as before (NaN
// ignored) — the result is bitwise the per-element fmax(m, RN(a / w)).
struct QuotMax {
  double ab = 0.0, wb = 1.0;  // best regular candidate (quotient 0 to start)
  double ms = 0.0;            // fmax over the irregular elements
  __device__ __forceinline__ void add(double a, double w) {
    // both factors in [1e-140, 1e140]: every product is a normal double whose
    // FMA remainder is exact
    if (a >= 1e-140 && a <= 1e140 && w >= 1e-140 && w <= 1e140) {
      const double p = __dmul_rn(a, wb), q = __dmul_rn(ab, w);
      bool gt = p > q;
      if (p == q) gt = __fma_rn(a, wb, -p) > __fma_rn(ab, w, -q);
      if (gt) {
        ab = a;
        wb = w;
      }
    } else if (!(a == 0.0 && w > 0.0)) {  // a zero quotient changes nothing
      ms = fmax(ms, __ddiv_rn(a, w));
    }
  }
  __device__ __forceinline__ double value() const { return fmax(ms, __ddiv_rn(ab, wb)); }
};

// The controller of one attempt (rk_step tail, solver.cpp:158-162, 201-214, and
// the solve_core bookkeeping, :298-342), run by one thread once the weighted
// max-norm err_max of the attempt is known. Returns whether the loop goes on.
__device__ inline bool attempt_controller(Ctl* c, int S, int mode, int k1_elided, int fixed_k1, bool dead, bool stage_nf,
                                   bool any_nf, double err_max, StepLogRec* log) {
  if (mode == FIN_SOLVE && dead) return false;
  // the need_k1 recompute of this attempt (solver.cpp:298-306)
  if (mode == FIN_SOLVE && c->need_k1) {
    if (k1_elided) c->evals_k1 += 1;
    else if (c->nf_mask & 1) {
      c->status = MS_NON_FINITE;
      c->done = 1;
      c->nf_mask = 0;
      return false;
    }
  }
  double err = nan64(), h_next;
  bool accepted = false;
  const double h = c->h_att;
  if (stage_nf || any_nf) {
    h_next = __dmul_rn(__dmul_rn(h, c->fac_min), 0.5);  // solver.cpp:158-162, 201-211
  } else {
    err = err_max;
    if (!isfinite(err)) {
      h_next = __dmul_rn(__dmul_rn(h, c->fac_min), 0.5);
    } else {
      accepted = err <= c->rel_tol;  // solver.cpp:212
      h_next = d_adjust_step(h, err, c->rel_tol, c->safety, c->fac_min, c->fac_max, c->ctrl_exp);
    }
  }
  c->err = err;
  c->accepted = accepted;
  c->h_next = h_next;
  if (mode == FIN_STEP) return false;  // bs32_step: nf_mask is read back by the host
  c->attempts += 1;
  if (c->record_log) {
    if (log && c->log_count < c->log_capacity) {
      StepLogRec& r = log[c->log_count];
      r.t = c->t; r.h = h; r.err = err; r.accepted = accepted;
    }
    c->log_count += 1;
  }
  c->need_k1 = 0;
  c->nf_mask = 0;
  c->snap_pending = (accepted && c->snap_on) ? 1 : 0;
  if (accepted) c->snap_hv = h;
  c->dense_lo = c->dense_hi = c->eval_next;
  if (accepted) c->t_prev = c->t;
  if (accepted) {  // solver.cpp:321-336
    c->n_acc += 1;
    c->ix ^= 1;
    const double tn = __dadd_rn(c->t, h);
    c->t = c->last ? c->tf : (c->store32 ? rn32(tn) : tn);
    if (!fixed_k1) c->k1i = S - c->k1i;  // FSAL: k1 <- k_last
    c->h = h_next;
    if (c->t >= c->tf) {
      c->status = MS_COMPLETED;
      c->done = 1;
    }
    // output times inside the accepted step (t_prev, t]
    int64_t e = c->eval_next;
    while (e < c->n_eval && c->t_eval[e] <= c->t) ++e;
    c->dense_hi = e;
    c->eval_next = e;
  } else {  // solver.cpp:337-341
    c->n_fail += 1;
    c->h = h_next;
    c->need_k1 = 1;
  }
  if (!c->done) loop_check(c);
  return !c->done;
}

struct InitArgs {
  Bufs B;
  const double* x0;
  int64_t dn;
  double exponent;  // 1/(order+1)
};

__device__ inline double seq_sum(const double* v, int64_t n) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s = __dadd_rn(s, v[i]);
  return s;
}

#ifdef MS_DEFINE_STEP_KERNELS
#ifndef MS_FIN_UNROLL
#define MS_FIN_UNROLL 1
#endif
constexpr int kFinUnroll = MS_FIN_UNROLL;
__global__ void __launch_bounds__(kFinSmallThreads) k_finalize(FinArgs f) {
  msb::count_launch();
  pdl_enter();
  Ctl* c = f.B.ctl;
  const bool dead = c->done != 0;
  const bool stage_nf = c->nf_mask != 0;
  __shared__ double red[kFinSmallThreads / 32];
  __shared__ int red_nf[kFinSmallThreads / 32];
  double m = 0.0;
  bool nf = false;
  if (!dead && !stage_nf) {
    const int ix = c->ix, k1i = c->k1i;
    const double* x = f.B.xb[ix];
    const double* xst = f.B.xb[ix ^ 1];
    const double* xnx = c->store32 ? f.B.xn : xst;
    const double h = c->h_att;
    const double floor_w = __ddiv_rn(c->abs_tol, c->rel_tol);
    // not unrolled: a thread has at most a few elements at every BASELINE size (the grid
    // covers dn), and the kernel's time is its instruction footprint (MS_FIN_UNROLL)
#pragma unroll kFinUnroll
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < f.dn; e += (int64_t)gridDim.x * blockDim.x) {
      // x_tilde = x + h * (sum b~_l k_l), solver.cpp:188-199
      double comb = __dmul_rn(f.bt[0], resolve_slot(f.B, f.S, f.bslot[0], k1i)[e]);
      for (int t = 1; t < f.nbt; ++t)
        comb = __dadd_rn(comb, __dmul_rn(f.bt[t], resolve_slot(f.B, f.S, f.bslot[t], k1i)[e]));
      const double xt = __dadd_rn(x[e], __dmul_rn(h, comb));
      if (f.write_xt) f.B.xt[e] = xt;
      const double xn = xnx[e];
      nf |= !isfinite(xn) || !isfinite(xt) || !isfinite(xst[e]);
      // estimate_error, solver.cpp:399-411
      const double w = fmax(fmax(fabs(x[e]), fabs(xn)), floor_w);
      m = fmax(m, __ddiv_rn(fabs(__dsub_rn(xn, xt)), w));
    }
  }
  for (int o = 16; o >= 1; o >>= 1) {
    m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    nf = __any_sync(0xffffffffu, nf);
  }
  const int warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  if ((threadIdx.x & 31) == 0) { red[warp] = m; red_nf[warp] = nf; }
  __syncthreads();
  double e = 0.0;
  bool any_nf = false;  // e and any_nf: thread 0 of the controlling block
  if (gridDim.x == 1) {
    if (threadIdx.x == 0) {
      int bnf = 0;
      for (int w = 0; w < nwarps; ++w) { e = fmax(e, red[w]); bnf |= red_nf[w]; }
      any_nf = bnf != 0;
      if (dead || stage_nf || any_nf) e = 0.0;
    }
  } else {
    __shared__ bool is_last;
    if (threadIdx.x == 0) {
      double bm = 0.0;
      int bnf = 0;
      for (int w = 0; w < nwarps; ++w) { bm = fmax(bm, red[w]); bnf |= red_nf[w]; }
      f.B.part[blockIdx.x] = bm;
      if (bnf) atomicOr(&c->any_nonfinite, 1);
      __threadfence();
      const unsigned t = atomicAdd(&c->ticket, 1u);
      is_last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (!is_last) return;
    if (threadIdx.x == 0) {
      __threadfence();
      c->ticket = 0;
      any_nf = atomicAdd(&c->any_nonfinite, 0) != 0;
      c->any_nonfinite = 0;
      if (!(dead || stage_nf || any_nf))
        for (int b = 0; b < (int)gridDim.x; ++b) e = fmax(e, f.B.part[b]);
    }
  }
  if (!f.ctl_smem) {
    if (threadIdx.x != 0) return;
    const bool more = attempt_controller(c, f.S, f.mode, f.k1_elided, f.fixed_k1, dead, stage_nf, any_nf, e, f.B.log);
    if (f.has_handle && f.mode == FIN_SOLVE) cudaGraphSetConditional(f.handle, more ? 1 : 0);
    return;
  }
  // no other block touches Ctl from here on; thread 0's resets above are
  // visible to the block after the barrier
  __shared__ __align__(16) Ctl cs;
  __syncthreads();
  ctl_copy(&cs, c);
  __syncthreads();
  if (threadIdx.x == 0) {
    const bool more = attempt_controller(&cs, f.S, f.mode, f.k1_elided, f.fixed_k1, dead, stage_nf, any_nf, e, f.B.log);
    if (f.has_handle && f.mode == FIN_SOLVE) cudaGraphSetConditional(f.handle, more ? 1 : 0);
  }
  __syncthreads();
  ctl_copy(c, &cs);
}

// StepSnapshot capture (solver.cpp:324-327): after an accepted attempt copy the
// new loop state into row n_acc of the snapshot buffer (row 0 = the starting
// state, written once after initialisation with row0 = 1).
__global__ void __launch_bounds__(256) k_snapshot(Bufs B, double* snap, double* snap_h, int64_t cap, int64_t dn,
                                                  int row0) {
  msb::count_launch();
  pdl_enter();
  const Ctl* c = B.ctl;
  if (!row0 && !c->snap_pending) return;
  const int64_t row = row0 ? 0 : c->n_acc;
  if (row > cap) return;
  const double* x = B.xb[c->ix];
  double* dst = snap + row * dn;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < dn; e += (int64_t)gridDim.x * blockDim.x)
    dst[e] = x[e];
  if (!row0 && blockIdx.x == 0 && threadIdx.x == 0) snap_h[row - 1] = c->snap_hv;
}

// Dense output (D6 extension): the cubic Hermite interpolant of
// an accepted step from (x_n, k1 = f(x_n)) to (x_{n+1}, k_last = f(x_{n+1})),
//   th = (tau - t_n) / h,  x(tau) = h00 x_n + h10 h k1 + h01 x_{n+1} + h11 h k_last
// with h00 = (1 + 2 th)(1 - th)^2, h10 = th (1 - th)^2, h01 = th^2 (3 - 2 th),
// h11 = th^2 (th - 1), evaluated in binary64 in exactly this order (the oracle's
// dense_eval restates it). After the swap on accept, x_{n+1} = xb[ix] and
// k_last = kb[k1i]; with row0 = 1 it writes the starting state to the output
// times <= t0 (before any step).
__device__ __forceinline__ double hermite(double th, double h, double xn, double k1, double xn1, double k4) {
  const double om = __dsub_rn(1.0, th);
  const double om2 = __dmul_rn(om, om);
  const double th2 = __dmul_rn(th, th);
  const double h00 = __dmul_rn(__dadd_rn(1.0, __dmul_rn(2.0, th)), om2);
  const double h10 = __dmul_rn(th, om2);
  const double h01 = __dmul_rn(th2, __dsub_rn(3.0, __dmul_rn(2.0, th)));
  const double h11 = __dmul_rn(th2, __dsub_rn(th, 1.0));
  double v = __dmul_rn(h00, xn);
  v = __dadd_rn(v, __dmul_rn(h10, __dmul_rn(h, k1)));
  v = __dadd_rn(v, __dmul_rn(h01, xn1));
  return __dadd_rn(v, __dmul_rn(h11, __dmul_rn(h, k4)));
}

__global__ void __launch_bounds__(256) k_dense(Bufs B, int S, double* y, int64_t dn, int row0, int64_t row0_count) {
  msb::count_launch();
  pdl_enter();
  const Ctl* c = B.ctl;
  int64_t lo, hi;
  if (row0) {
    lo = 0;
    hi = row0_count;
  } else {
    if (!c->accepted) return;
    lo = c->dense_lo;
    hi = c->dense_hi;
  }
  if (lo >= hi) return;
  const double* xn1 = B.xb[c->ix];
  const double* xn = B.xb[c->ix ^ 1];
  const double* k4 = B.kb[c->k1i];
  const double* k1 = B.kb[S - c->k1i];
  const double h = c->snap_hv, t0 = c->t_prev;
  for (int64_t q = lo; q < hi; ++q) {
    double* dst = y + q * dn;
    const double th = row0 ? 0.0 : __ddiv_rn(__dsub_rn(c->t_eval[q], t0), h);
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < dn; e += (int64_t)gridDim.x * blockDim.x)
      dst[e] = row0 ? xn1[e] : hermite(th, h, xn[e], k1[e], xn1[e], k4[e]);
  }
}

// ------------------------------------------------------------------------------
// initial_step (solver.cpp:420-451). The per-element terms are formed in
// parallel; each of the three sums is then added by one thread in ascending
// order (the oracle's fixed order).
__global__ void __launch_bounds__(1024) k_init_a(InitArgs a) {
  msb::count_launch();
  pdl_enter();
  Ctl* c = a.B.ctl;
  if (c->done) return;
  __shared__ int nf;
  if (threadIdx.x == 0) nf = 0;
  __syncthreads();
  const double* f0 = a.B.kb[1];
  double* t0 = a.B.scratch;
  double* t1 = a.B.xn;
  bool mynf = false;
  for (int64_t e = threadIdx.x; e < a.dn; e += blockDim.x) {
    const double sk = __dadd_rn(c->abs_tol, __dmul_rn(c->rel_tol, fabs(a.x0[e])));
    const double q0 = __ddiv_rn(a.x0[e], sk);
    const double q1 = __ddiv_rn(f0[e], sk);
    t0[e] = __dmul_rn(q0, q0);
    t1[e] = __dmul_rn(q1, q1);
    mynf |= !isfinite(f0[e]);
  }
  if (mynf) atomicOr(&nf, 1);
  __syncthreads();
  __shared__ double s01[2];
  if (threadIdx.x == 0) s01[0] = seq_sum(t0, a.dn);
  if (threadIdx.x == 32) s01[1] = seq_sum(t1, a.dn);
  __syncthreads();
  if (threadIdx.x != 0) return;
  c->cap = __ddiv_rn(__dsub_rn(c->tf, c->t0), 10.0);
  if (nf) {  // solver.cpp:426
    c->h = nan64();
    c->init_skip2 = 1;
    return;
  }
  const double inv_n = __ddiv_rn(1.0, (double)a.dn);
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

__global__ void __launch_bounds__(1024) k_init_b(InitArgs a) {
  msb::count_launch();
  pdl_enter();
  Ctl* c = a.B.ctl;
  if (c->done) return;
  const bool skip2 = c->init_skip2 != 0;
  __shared__ int nf;
  if (threadIdx.x == 0) nf = 0;
  __syncthreads();
  const double* f0 = a.B.kb[1];
  const double* f1 = a.B.kb[2];
  double* t2 = a.B.scratch;
  if (!skip2) {
    bool mynf = false;
    for (int64_t e = threadIdx.x; e < a.dn; e += blockDim.x) {
      const double sk = __dadd_rn(c->abs_tol, __dmul_rn(c->rel_tol, fabs(a.x0[e])));
      const double q2 = __ddiv_rn(__dsub_rn(f1[e], f0[e]), sk);
      t2[e] = __dmul_rn(q2, q2);
      mynf |= !isfinite(f1[e]);
    }
    if (mynf) atomicOr(&nf, 1);
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
      const double inv_n = __ddiv_rn(1.0, (double)a.dn);
      const double d2 = __ddiv_rn(__dsqrt_rn(__dmul_rn(seq_sum(t2, a.dn), inv_n)), h1);
      const double der = c->d1 < d2 ? d2 : c->d1;  // std::max
      h2 = der < 1e-12 ? c->cap : pow_cr(__ddiv_rn(0.01, der), a.exponent);
    }
    // std::min({100*h1, h2, cap})
    h0 = __dmul_rn(100.0, h1);
    if (h2 < h0) h0 = h2;
    if (c->cap < h0) h0 = c->cap;
  }
  c->h = h0;
  c->init_skip2 = 0;
  if (!isfinite(h0)) {  // solver.cpp:256-259
    c->status = MS_NON_FINITE;
    c->done = 1;
  }
}

// after the cold k1 (solver.cpp:263-269) and before the first attempt
__global__ void k_loop_head(Ctl* c) {
  msb::count_launch();
  pdl_enter();
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

__global__ void k_stamp_start(Ctl* c) {
  msb::count_launch();
  pdl_enter();
  c->t_start_ns = globaltimer_ns();
}

// sharded loop: finiteness of a gathered stage vector, identical on every rank
__global__ void k_nf_scan(Ctl* c, const double* v, int64_t n, int l) {
  msb::count_launch();
  bool nf = false;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    nf |= !isfinite(v[e]);
  if (__any_sync(0xffffffffu, nf) && (threadIdx.x & 31) == 0) atomicOr(&c->nf_mask, 1 << l);
}

// sharded loop: FSAL k1 <- k_last on an accepted attempt (slot 0 stays k1)
// Push exchange barrier (ms_loop_push_*): after every loop segment each rank
// bumps its epoch and stores it into its slot of every peer's mailbox (system
// scope, after the segment's pushes); before the next segment it waits until
// every peer's slot in its own mailbox has reached its epoch. All ranks run the
// same segment sequence, so the epochs agree.
struct PushSig {
  unsigned long long* epoch;                // this rank's counter
  unsigned long long* mbox;                 // this rank's mailbox [world]
  unsigned long long* peer_slot[kMaxPeers]; // &mailbox_q[rank] of every peer q
  int peer_rank[kMaxPeers];                 // q of peer_slot[i]
  int np;
};
__global__ void k_push_signal(PushSig s) {
  msb::count_launch();
  pdl_enter();
  if (threadIdx.x != 0) return;
  const unsigned long long e = *s.epoch + 1;
  *s.epoch = e;
  __threadfence_system();  // the segment's pushes (earlier kernels, stream order) before the flag
  for (int q = 0; q < s.np; ++q)
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(s.peer_slot[q]), "l"(e) : "memory");
}
__global__ void k_push_wait(PushSig s) {
  msb::count_launch();
  pdl_enter();
  if (threadIdx.x != 0) return;
  const unsigned long long e = *s.epoch;
  uint64_t t0 = 0;
  for (int q = 0; q < s.np; ++q) {
    for (uint32_t it = 0;; ++it) {
      unsigned long long v;
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(s.mbox + s.peer_rank[q]) : "memory");
      if (v >= e) break;
      if ((it & 1023) == 0) {  // a peer that never arrives ends the kernel instead of hanging the GPU
        const uint64_t now = globaltimer_ns();
        if (t0 == 0) t0 = now;
        else if (now - t0 > 20000000000ull) __trap();
      }
    }
  }
}

__global__ void k_fsal_copy(const Ctl* c, double* k1, const double* klast, int64_t n) {
  msb::count_launch();
  if (!c->accepted) return;  // set by this attempt's k_finalize (stale only once done)
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    k1[e] = klast[e];
}

#endif  // MS_DEFINE_STEP_KERNELS

}  // namespace msb
