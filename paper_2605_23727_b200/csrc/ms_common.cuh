// ms_common.cuh — shared device/host definitions of the B200 integrator.
//
// Arithmetic contract: every floating operation below
// is a single IEEE operation rounded once in its stated format, with no FMA
// contraction (the translation units are compiled with -fmad=false, and the
// hot loops spell their roundings with __fmul_rn/__fadd_rn/__dmul_rn/__dadd_rn).
#pragma once

#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <cstdio>

#include "../../include/mixedstep_b200.h"

namespace msb {

constexpr int kMaxStages = 7;  // DP5(4) has 7 (solver.cpp:35-68)
constexpr int kNumSMsDefault = 148;

// ---- formats -------------------------------------------------------------
__host__ __device__ inline bool is32(uint8_t f) { return f == MS_BINARY32; }

// RN into f32 of a double (precision.hpp:21-24: (double)(float)x)
__device__ __forceinline__ double rn32(double x) { return (double)__double2float_rn(x); }

// Correctly-rounded-by-construction f32 transcendentals: evaluate in binary64
// and round once. glibc's sinf/atanf (the reference's libm, systems.cpp:142,
// 184) are correctly rounded in nearly all cases, so this is the closest
// device counterpart; CUDA's own sinf/atanf carry up to 2 ulp.
__device__ __forceinline__ float cr_sinf(float x) { return __double2float_rn(sin((double)x)); }
__device__ __forceinline__ float cr_cosf(float x) { return __double2float_rn(cos((double)x)); }
__device__ __forceinline__ float cr_atanf(float x) { return __double2float_rn(atan((double)x)); }

template <class S> __device__ __forceinline__ S dsin(S x);
template <> __device__ __forceinline__ float dsin<float>(float x) { return cr_sinf(x); }
template <> __device__ __forceinline__ double dsin<double>(double x) { return sin(x); }
template <class S> __device__ __forceinline__ S dcos(S x);
template <> __device__ __forceinline__ float dcos<float>(float x) { return cr_cosf(x); }
template <> __device__ __forceinline__ double dcos<double>(double x) { return cos(x); }
// sin and cos of one argument with a shared argument reduction (CUDA's
// sincos evaluates the same kernels as sin and cos)
__device__ __forceinline__ void dsincos(float x, float* s, float* c) {
  double sd, cd;
  sincos((double)x, &sd, &cd);
  *s = __double2float_rn(sd);
  *c = __double2float_rn(cd);
}
__device__ __forceinline__ void dsincos(double x, double* s, double* c) { sincos(x, s, c); }
// fast-path arctangent: CUDA's own atanf (<= 2 ulp) in binary32 — the fast
// sweep is held to tolerance parity, only the faithful sweep needs cr_atanf
template <class S> __device__ __forceinline__ S fatan(S x);
template <> __device__ __forceinline__ float fatan<float>(float x) { return atanf(x); }
template <> __device__ __forceinline__ double fatan<double>(double x) { return atan(x); }
template <class S> __device__ __forceinline__ S datan(S x);
template <> __device__ __forceinline__ float datan<float>(float x) { return cr_atanf(x); }
template <> __device__ __forceinline__ double datan<double>(double x) { return atan(x); }

// single-rounding arithmetic in format S
template <class S> __device__ __forceinline__ S add(S a, S b);
template <class S> __device__ __forceinline__ S sub(S a, S b);
template <class S> __device__ __forceinline__ S mul(S a, S b);
template <class S> __device__ __forceinline__ S dvd(S a, S b);
template <> __device__ __forceinline__ float add<float>(float a, float b) { return __fadd_rn(a, b); }
template <> __device__ __forceinline__ float sub<float>(float a, float b) { return __fsub_rn(a, b); }
template <> __device__ __forceinline__ float mul<float>(float a, float b) { return __fmul_rn(a, b); }
template <> __device__ __forceinline__ float dvd<float>(float a, float b) { return __fdiv_rn(a, b); }
template <> __device__ __forceinline__ double add<double>(double a, double b) { return __dadd_rn(a, b); }
template <> __device__ __forceinline__ double sub<double>(double a, double b) { return __dsub_rn(a, b); }
template <> __device__ __forceinline__ double mul<double>(double a, double b) { return __dmul_rn(a, b); }
template <> __device__ __forceinline__ double dvd<double>(double a, double b) { return __ddiv_rn(a, b); }

// (a, b) = (a + x, b + y): two independent single-rounding adds. For binary32
// one packed FADD2 (sm_100): the same two IEEE adds in one issue slot. The
// products fed in must come from scalar mul.rn (FMUL): ptxas contracts
// mul.rn.f32x2 + add.rn.f32x2 into FFMA2 even under -fmad=false, but never a
// scalar mul.rn into a packed add (checked in the SASS, tests/test_abi.py).
template <class S, bool PACK = true> __device__ __forceinline__ void add2(S& a, S& b, S x, S y) {
#ifndef MS_NO_FADD2
  if constexpr (PACK && sizeof(S) == 4) {
    unsigned long long acc, p;
    asm("mov.b64 %0, {%1, %2};" : "=l"(acc) : "f"(a), "f"(b));
    asm("mov.b64 %0, {%1, %2};" : "=l"(p) : "f"(x), "f"(y));
    asm("add.rn.f32x2 %0, %0, %1;" : "+l"(acc) : "l"(p));
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(acc));
    return;
  }
#endif
  a = add<S>(a, x);
  b = add<S>(b, y);
}

// ---- packed products for the split Kuramoto sweeps ---------------------------
// {A, B} += {RN32(s k), RN32(c k)} for a packed accumulator AB = {A, B} and a
// packed column pair sc = {s_j, c_j}: one FMUL2 (K broadcast) and one FADD2
// instead of two FMUL and two FADD. The multiply carries .ftz: ptxas contracts
// mul.rn.f32x2 + add.rn.f32x2 into FFMA2 even under -fmad=false (one rounding
// less), but not a flush-to-zero multiply into a non-flushing add. The .ftz
// changes nothing while no operand or product is subnormal: |K| >= 2^-80 for
// every nonzero K (checked when K is created, ms_system::k_tiny) and
// |s|, |c| >= 2^-46 for every nonzero s, c (checked by every prep, sticky in
// Ctl::pk_off) bound every nonzero product by 2^-126 from below. Otherwise the
// sweeps take the unflushed path (two FMUL, one FADD2), the same arithmetic.
constexpr float kPkMinK = 0x1p-80f;
constexpr float kPkMinSC = 0x1p-46f;
__device__ __forceinline__ uint64_t pk2(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ uint64_t pk2u(uint32_t a, uint32_t b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "r"(a), "r"(b));
  return r;
}
__device__ __forceinline__ void unpk2(uint64_t v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
template <bool FTZ>
__device__ __forceinline__ void mac2(uint64_t& ab, uint64_t sc, float k) {
  uint64_t p;
  if constexpr (FTZ) {
    asm("mul.rn.ftz.f32x2 %0, %1, %2;" : "=l"(p) : "l"(sc), "l"(pk2(k, k)));
  } else {
    float s, c;
    unpk2(sc, s, c);
    p = pk2(__fmul_rn(s, k), __fmul_rn(c, k));
  }
  asm("add.rn.f32x2 %0, %0, %1;" : "+l"(ab) : "l"(p));
}
// sticky Ctl::pk_off when a column value is nonzero and below 2^-46
__device__ __forceinline__ bool sc_tiny(float s, float c) {
  return (s != 0.f && fabsf(s) < kPkMinSC) || (c != 0.f && fabsf(c) < kPkMinSC);
}

// RN into S of a double
template <class S> __device__ __forceinline__ S cvt(double x);
template <> __device__ __forceinline__ float cvt<float>(double x) { return __double2float_rn(x); }
template <> __device__ __forceinline__ double cvt<double>(double x) { return x; }

// ---- programmatic dependent launch ---------------------------------------------
// Every kernel of the attempt chain waits for its predecessor grid here (a no-op
// when launched without the PDL attribute) and at once lets its successor be
// scheduled, so a kernel's launch and prologue overlap the previous one's tail.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ---- checked builds ------------------------------------------------------------
// -DMS_CHECKS=1 (tools/build_checked.py) compiles bounds and alignment checks into
// the kernels' memory movement: a failed check prints its site and traps, so a
// bad access ends the kernel with an error instead of corrupting memory. The
// pool runs no compute-sanitizer (profiles/r2_sanitizer_closed.txt); the checked
// build run over the GPU tests stands in for memcheck.
#ifndef MS_CHECKS
#define MS_CHECKS 0
#endif
#if MS_CHECKS
#define MS_CHECK(cond, what)                                                                               \
  do {                                                                                                     \
    if (!(cond)) {                                                                                         \
      printf("MS_CHECK failed: %s (%s:%d) block (%d,%d) thread %d\n", what, __FILE__, __LINE__, blockIdx.x, \
             blockIdx.y, threadIdx.x);                                                                     \
      __trap();                                                                                            \
    }                                                                                                      \
  } while (0)
#else
#define MS_CHECK(cond, what) \
  do {                       \
  } while (0)
#endif
__device__ __forceinline__ uint32_t dyn_smem_bytes() {
  uint32_t v;
  asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(v));
  return v;
}

// ---- launch accounting ---------------------------------------------------------
// Every kernel of the library starts with count_launch(): the first thread of
// block (0,0,0) adds one to a per-translation-unit device counter, so
// ms_launch_count() reports how many of this library's kernels actually ran
// (CUDA-graph replays and early-exiting kernels included) — a count, not a
// formula. One counter per TU (no relocatable device code); each .cu defines a
// host reader with MS_DEFINE_LAUNCH_READER.
static __device__ unsigned long long g_ms_launches;
__device__ __forceinline__ void count_launch() {
  if ((blockIdx.x | blockIdx.y | blockIdx.z | threadIdx.x | threadIdx.y | threadIdx.z) == 0)
    atomicAdd(&g_ms_launches, 1ull);
}
#define MS_DEFINE_LAUNCH_READER(fn)                                                        \
  unsigned long long fn() {                                                                \
    unsigned long long v = 0;                                                              \
    if (cudaMemcpyFromSymbol(&v, msb::g_ms_launches, sizeof(v)) != cudaSuccess) return 0;  \
    return v;                                                                              \
  }

// ---- coupling storage --------------------------------------------------------
struct KScalar {};  // no matrix: G uses RN_S(coupling_k)
template <int KS> struct KElem;
template <> struct KElem<MS_K_F32> { using T = float; };
template <> struct KElem<MS_K_F16> { using T = __half; };
template <> struct KElem<MS_K_BF16> { using T = __nv_bfloat16; };

__device__ __forceinline__ float k2f(float v) { return v; }
__device__ __forceinline__ float k2f(__half v) { return __half2float(v); }
__device__ __forceinline__ float k2f(__nv_bfloat16 v) { return __bfloat162float(v); }

// ---- model ids for templates ------------------------------------------------
enum : int { MD_LCO = 0, MD_KUR = 1, MD_CC = 2 };

// ---- device control block (one per solve workspace) -------------------------
// Replicated controller state of solve_core (solver.cpp:226-347); every kernel
// reads it, only the single-thread controller sections write it.
struct Ctl {
  // clock and step
  double t, h, h_att, t0, tf, h_min;
  double h1, cap, d1;  // initial_step scratch (solver.cpp:420-451)
  double err, h_next;
  // config (solver.hpp:39-61)
  double rel_tol, abs_tol, safety, fac_min, fac_max, ctrl_exp;
  double wall_clock_limit, slow_elapsed, slow_progress;
  int64_t max_iterations, max_failed;
  // counters
  int64_t n_acc, n_fail, attempts;
  int64_t evals_ddd, evals_k1, evals_stage[kMaxStages];
  int64_t log_count, log_capacity;
  uint64_t t_start_ns;
  // flags
  int32_t status, done, need_k1, last, accepted;
  int32_t nf_mask;        // bit l: stage l produced a non-finite value this attempt
  int32_t ix;             // current x buffer (x = xb[ix], x_store -> xb[ix^1])
  int32_t k1i;            // k1 slot: 0 or S (FSAL ping-pong with the last stage)
  int32_t store32, time_limits, record_log, init_skip2;
  int32_t any_nonfinite;  // finalize scratch
  uint32_t ticket;        // last-block-done counter (finalize / init)
  int32_t snap_on;        // record StepSnapshots (solver.cpp:324-327)
  int32_t snap_pending;   // this attempt was accepted: k_snapshot copies x
  int32_t pk_off;         // packed FMUL2.FTZ sweep disabled: K has tiny entries, or a prep saw a tiny s/c
  double snap_hv;         // h of the accepted attempt (h_att before loop_check moves on)
  // dense output (D6 extension): sorted output times, the next unfilled one,
  // and the range [dense_lo, dense_hi) the accepted attempt covers
  const double* t_eval;
  int64_t n_eval, eval_next, dense_lo, dense_hi;
  double t_prev;          // t at the start of the accepted attempt
};

struct StepLogRec {
  double t, h, err;
  int32_t accepted, _pad;
};

// Pointers of one solve workspace (device addresses).
// Row-sharded loop, push exchange (ms_loop_push_setup): a sweep stores each of
// its output rows into its own workspace AND at the same offset into every
// peer's workspace (peer memory over NVLink, P2P/IPC-mapped), so the exchange
// rides on the sweep's own stores instead of a following all-gather.
constexpr int kMaxPeers = 7;  // world <= 8
struct PushDev {
  const char* ws;              // this handle's workspace base
  char* peer[kMaxPeers];       // the peers' workspace bases (same layout)
  int np;                      // number of peers (0: no push)
};

struct Bufs {
  double* xb[2];                 // x / x_store ping-pong
  double* kb[kMaxStages + 1];    // stage derivatives; slot 0 <-> slot S for FSAL
  double* xn;                    // x_next under binary32 storage
  double* xt;                    // x_tilde (only when requested)
  double* scratch;               // dN terms for initial_step sums
  void* gin;                     // GS-typed column data (2 * ld doubles)
  void* gin2;                    // the other column buffer: a sweep that runs the next stage's prep writes it
  void* op16;                    // f16 operand image of the column data for the tensor-core sweep, or null
  void* op16b;                   // gin2's operand image (a tensor-core sweep that runs the next stage's prep writes it)
  void* rowc;                    // GS-typed per-row G constant (CC prefactor)
  double* fvc;                   // F of the coupled slot, per agent
  double* part;                  // per-block partials of finalize
  StepLogRec* log;
  Ctl* ctl;
};

}  // namespace msb
