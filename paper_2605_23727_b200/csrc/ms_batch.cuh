// ms_batch.cuh — batched Kuramoto ensembles that share one coupling matrix K
// (BASELINE.json configs[4]: B trajectories, each with its own omega_b and
// theta0_b, each integrated by its own adaptive BS3(2) controller).
//
// The reference runs B independent solves (harness.cpp:113-121 pattern); here
// all trajectories advance in lock-step attempts — each attempt is one BS3(2)
// attempt of every unfinished trajectory with its own h, t, FSAL k1, status —
// so one stage evaluation of the whole ensemble is the dense contraction
//   A[i][b] = sum_j K_ij sin(theta_bj),  B[i][b] = sum_j K_ij cos(theta_bj)
// (the Kuramoto sin/cos split) over all b at once.
#pragma once

#include "ms_kernels.cuh"

namespace msb {

// Device view of one ensemble (all [B][N] arrays trajectory-major, N = n).
struct BatchDev {
  int B, n, ld;
  const void* K;  // the system's K (rows 0..n), storage ks
  int ks;
  const double* omega;            // [B][n]
  double* xb[2];                  // x / x_store ping-pong, selected per trajectory by ctl[b].ix
  double* kb[kMaxStages + 1];     // stage derivatives, k1 <-> k_last via ctl[b].k1i
  double* xn;                     // x_next under binary32 storage
  double* scr0;                   // initial_step terms
  double* scr1;
  void* sc;                       // GS-typed s (first B*n) and c (next B*n)
  void* op;                       // GEMM operand [B][4][ld] in K's 16-bit format: s_hi, s_lo, c_hi, c_lo
  double* fvc;                    // F (omega in FS) [B][n]
  void* rec;                      // tensor-core epilogue F: TcRec [B][n] records, or RN32(omega) floats (MS_TC_PACKED 3); written at creation
  Ctl* ctl;                       // [B]
  int* flag;                      // [1] any trajectory still running (host loop / conditional)
  // error estimate folded into the last stage's contraction epilogue (MS_BFIN_EPI):
  // per trajectory the bit pattern of the weighted max-norm so far (non-negative
  // doubles order like their bits) and a non-finite flag; kb_finalize reads and
  // clears them
  unsigned long long* errb;       // [B]
  int* nfe;                       // [B]
  unsigned* ticket;               // [1] finalize last-block counter (reset by the last block)
  double mw;                      // 1/N
};

__device__ __forceinline__ double* bslot(const BatchDev& d, int S, int slot, const Ctl* c) {
  if (slot == SLOT_K1) return d.kb[c->k1i];
  if (slot == SLOT_KLAST) return d.kb[S - c->k1i];
  return d.kb[slot];
}

template <int KS> struct K16;
template <> struct K16<MS_K_F16> {
  using T = __half;
  __device__ static T from(float v) { return __float2half_rn(v); }
};
template <> struct K16<MS_K_BF16> {
  using T = __nv_bfloat16;
  __device__ static T from(float v) { return __float2bfloat16_rn(v); }
};

// F of the Kuramoto agent in FS (systems.cpp:136-139): RN_FS(omega), exact in binary64
__device__ __forceinline__ double b_fval(const BatchDev& d, int64_t e, int fs32) {
  const double w = d.omega[e];
  return fs32 ? (double)__double2float_rn(w) : w;
}

// Per-element inputs of the tensor-core coupling epilogue: (s, c) of theta_bi
// in binary32 (the row side, exact GS values), written by the prep kernel as
// float2 pairs into the `sc` buffer on that path, and F = RN_FS(omega_bi),
// which the epilogue reads from omega itself (it never changes).
#ifndef MS_TC_PACKED
// 2: {s, c, F} records in their own buffer with F = RN32(omega) written once at
//    creation: the prep stores only the (s, c) half and never reads omega, the
//    epilogue still takes one 16-byte load. (Splitting the record into (s, c)
//    pairs + a separate F array instead measured 21 vs 26 us per prep but a
//    64 vs 41 us contraction.)
// 1: the prep writes whole {s, c, F} records every stage; 0: (s, c) pairs + omega
// 3: (s, c) pairs in `sc` (written by the prep) and F = RN32(omega) as a binary32
//    array in `rec` (written once at creation): 12 B per element, both arrays
//    copied into shared memory by the contraction's bulk copies (MS_T2_SREC).
//    Measured: prep 20.9 vs 23.0 us, contraction 47.3 vs 38.9 us
//    (profiles/r2_c5_srec.txt), so the default stays 2
#define MS_TC_PACKED 2
#endif
// The contraction's windowed accumulation (MS_T2_DRAIN = default k-blocks per
// window, 0 = one accumulator over all of K; ms_gemm_tc.cuh) folds hi and lo into
// one accumulator and needs each plane's (s, c) rows of a tile of trajectories
// contiguous: planes [hi, lo][B][s, c][ld]. Otherwise [B][4][ld].
#ifndef MS_T2_DRAIN
#define MS_T2_DRAIN 2
#endif
// element i of operand row `which` (0 s_hi, 1 s_lo, 2 c_hi, 3 c_lo) of trajectory b
__device__ __forceinline__ int64_t op_index(const BatchDev& d, int b, int which, int i) {
#if MS_T2_DRAIN
  return ((int64_t)((which & 1) * d.B + b) * 2 + (which >> 1)) * d.ld + i;
#else
  return ((int64_t)b * 4 + which) * d.ld + i;
#endif
}

struct __align__(16) TcRec {
  float s, c;
  double f;
};

struct BPrepArgs {
  BatchDev d;
  int S, l, kind, gate, count, out_slot, nterms;
  double coef[kMaxStages];
  int slot[kMaxStages];
  int is_last, round_x, ws32, fs32;
  int op_ks;  // 0: no GEMM operand; MS_K_F16 / MS_K_BF16: write the rounded operand
  // last stage: also write P = b~1 k1 + b~2 k2 + b~3 k3 (the first three terms of
  // x_tilde's combination, in its order) into scr1, so the finalize reads P and
  // k4 instead of k1..k4 (bit-identical: the same operations in the same order)
  int write_p;
  double pb[3];
};

// stage combination + F + sin/cos (+ rounded GEMM operand) of element i of
// trajectory b (the caller has checked stage_skip and counted the evaluation)
template <class FS, class GS>
__device__ __forceinline__ void bprep_elem(const BPrepArgs& p, int b, int i, Ctl* c) {
  const BatchDev& d = p.d;
  const int64_t e = (int64_t)b * d.n + i;
  const int ix = c->ix;
  double* x = d.xb[ix];
  double v;
  const double h = p.kind == PREP_INIT_X1 ? c->h1 : c->h_att;
  if (p.kind == PREP_X) {
    v = x[e];
    if (p.round_x) {
      v = rn32(v);
      x[e] = v;
    }
  } else if (p.kind == PREP_INIT_X1) {
    v = __dadd_rn(x[e], __dmul_rn(h, d.kb[1][e]));
  } else {
    double cm = __dmul_rn(p.coef[0], bslot(d, p.S, p.slot[0], c)[e]);
    for (int t = 1; t < p.nterms; ++t) cm = __dadd_rn(cm, __dmul_rn(p.coef[t], bslot(d, p.S, p.slot[t], c)[e]));
    v = __dadd_rn(x[e], __dmul_rn(h, cm));
    if (p.is_last) {
      if (c->store32) {
        const float hf = __double2float_rn(h);
        float acc = __double2float_rn(x[e]);
        for (int t = 0; t < p.nterms; ++t) {
          const float cf = __fmul_rn(hf, __double2float_rn(p.coef[t]));
          acc = __fadd_rn(acc, __fmul_rn(cf, __double2float_rn(bslot(d, p.S, p.slot[t], c)[e])));
        }
        d.xn[e] = v;
        v = (double)acc;
      }
      d.xb[ix ^ 1][e] = v;
      if (p.write_p) {
        double pp = __dmul_rn(p.pb[0], bslot(d, p.S, p.slot[0], c)[e]);
        pp = __dadd_rn(pp, __dmul_rn(p.pb[1], bslot(d, p.S, p.slot[1], c)[e]));
        d.scr1[e] = __dadd_rn(pp, __dmul_rn(p.pb[2], bslot(d, p.S, p.slot[2], c)[e]));
      }
    }
  }
  const GS xg = cvt<GS>(v);
  GS sv, cv;
  dsincos(xg, &sv, &cv);
  if (p.op_ks) {  // tensor-core path: the epilogue's record
#if MS_TC_PACKED == 1
    TcRec r;
    r.s = (float)sv;
    r.c = (float)cv;
    r.f = b_fval(d, e, p.fs32);
    reinterpret_cast<TcRec*>(d.sc)[e] = r;
#elif MS_TC_PACKED == 2
    *reinterpret_cast<float2*>(reinterpret_cast<TcRec*>(d.rec) + e) = make_float2((float)sv, (float)cv);
#else
    reinterpret_cast<float2*>(d.sc)[e] = make_float2((float)sv, (float)cv);
#endif
  } else {
    GS* sc = reinterpret_cast<GS*>(d.sc);
    sc[e] = sv;
    sc[(int64_t)d.B * d.n + e] = cv;
  }
  // two-term operands: v = hi + lo with hi = RN16(v), lo = RN16(v - hi) (the
  // difference is exact in binary32), so K*hi + K*lo carries ~16-22 bits of v
  if (p.op_ks == MS_K_BF16) {
    __nv_bfloat16* op = reinterpret_cast<__nv_bfloat16*>(d.op);
    const float s32 = (float)sv, c32 = (float)cv;
    const __nv_bfloat16 sh = __float2bfloat16_rn(s32), ch = __float2bfloat16_rn(c32);
    op[op_index(d, b, 0, i)] = sh;
    op[op_index(d, b, 1, i)] = __float2bfloat16_rn(__fsub_rn(s32, __bfloat162float(sh)));
    op[op_index(d, b, 2, i)] = ch;
    op[op_index(d, b, 3, i)] = __float2bfloat16_rn(__fsub_rn(c32, __bfloat162float(ch)));
  } else if (p.op_ks == MS_K_F16) {
    __half* op = reinterpret_cast<__half*>(d.op);
    const float s32 = (float)sv, c32 = (float)cv;
    const __half sh = __float2half_rn(s32), ch = __float2half_rn(c32);
    op[op_index(d, b, 0, i)] = sh;
    op[op_index(d, b, 1, i)] = __float2half_rn(__fsub_rn(s32, __half2float(sh)));
    op[op_index(d, b, 2, i)] = ch;
    op[op_index(d, b, 3, i)] = __float2half_rn(__fsub_rn(c32, __half2float(ch)));
  }
}

// every trajectory: grid (ceil(n/256), B)
template <class FS, class GS>
__global__ void __launch_bounds__(256) kb_prep(BPrepArgs p) {
  msb::count_launch();
  pdl_enter();
  const int b = blockIdx.y;
  const BatchDev& d = p.d;
  Ctl* c = d.ctl + b;
  if (stage_skip(c, p.l, p.gate)) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (p.count == CNT_DDD) c->evals_ddd += 1;
    else if (p.count == CNT_K1) c->evals_k1 += 1;
    else if (p.count == CNT_STAGE) c->evals_stage[p.l] += 1;
  }
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= d.n) return;
  bprep_elem<FS, GS>(p, b, i, c);
}

// The tensor-core path's stage prep (binary32 row, BS3 stage with NT terms,
// LAST = the x_next stage), specialised: the trajectory's pointers and h are
// resolved once per block into shared memory, and each thread first loads the
// inputs of its kPrepTcElems elements (read-only path), then prepares them —
// the generic prep is latency-bound on one element's dependent loads. Same
// arithmetic as bprep_elem<float, float> (bitwise; MS_PREP_TC=0 keeps the
// generic kernel).
#ifndef MS_PREP_TC_ELEMS
#define MS_PREP_TC_ELEMS 4
#endif
constexpr int kPrepTcElems = MS_PREP_TC_ELEMS;
template <int OPKS, int NT, bool LAST>
__global__ void __launch_bounds__(256) kb_prep_tc(BPrepArgs p) {
  msb::count_launch();
  pdl_enter();
  const int b = blockIdx.y;
  const BatchDev& d = p.d;
  Ctl* c = d.ctl + b;
  struct Row {
    const double* x;
    const double* k[NT];
    double* xst;
    double* xn;
    double* pp;
    double h;
    int store32;
  };
  __shared__ Row row;
  __shared__ int skip;
  if (threadIdx.x == 0) {
    skip = stage_skip(c, p.l, p.gate) ? 1 : 0;
    if (!skip) {
      if (blockIdx.x == 0) c->evals_stage[p.l] += 1;  // CNT_STAGE
      const int64_t o = (int64_t)b * d.n;
      const int ix = c->ix;
      row.x = d.xb[ix] + o;
#pragma unroll
      for (int t = 0; t < NT; ++t) row.k[t] = bslot(d, p.S, p.slot[t], c) + o;
      row.xst = d.xb[ix ^ 1] + o;
      row.xn = d.xn + o;
      row.pp = d.scr1 + o;
      row.h = c->h_att;
      row.store32 = c->store32;
    }
  }
  __syncthreads();
  if (skip) return;
  using T = typename K16<OPKS>::T;
  T* op = reinterpret_cast<T*>(d.op);
  const int64_t o_sh = op_index(d, b, 0, 0), o_sl = op_index(d, b, 1, 0), o_ch = op_index(d, b, 2, 0),
                o_cl = op_index(d, b, 3, 0);
#if MS_TC_PACKED == 1
  TcRec* rec = reinterpret_cast<TcRec*>(d.sc) + (int64_t)b * d.n;
  const double* om = d.omega + (int64_t)b * d.n;
#elif MS_TC_PACKED == 3
  float2* rec = reinterpret_cast<float2*>(d.sc) + (int64_t)b * d.n;
#else
  TcRec* rec = reinterpret_cast<TcRec*>(d.rec) + (int64_t)b * d.n;
#endif
  const double h = row.h;
  const int i0 = blockIdx.x * kPrepTcElems * blockDim.x + threadIdx.x;
  MS_CHECK(b < d.B, "batch prep: trajectory index");
  double xv[kPrepTcElems], kv[kPrepTcElems][NT];
#if MS_TC_PACKED == 1
  double wv[kPrepTcElems];
#endif
#pragma unroll
  for (int u = 0; u < kPrepTcElems; ++u) {
    const int i = i0 + u * blockDim.x;
    if (i < d.n) {
      xv[u] = __ldg(row.x + i);
#pragma unroll
      for (int t = 0; t < NT; ++t) kv[u][t] = __ldg(row.k[t] + i);
#if MS_TC_PACKED == 1
      wv[u] = __ldg(om + i);
#endif
    }
  }
#pragma unroll
  for (int u = 0; u < kPrepTcElems; ++u) {
    const int i = i0 + u * blockDim.x;
    if (i >= d.n) break;
    double cm = __dmul_rn(p.coef[0], kv[u][0]);
#pragma unroll
    for (int t = 1; t < NT; ++t) cm = __dadd_rn(cm, __dmul_rn(p.coef[t], kv[u][t]));
    double v = __dadd_rn(xv[u], __dmul_rn(h, cm));
    if (LAST) {
      if (row.store32) {
        const float hf = __double2float_rn(h);
        float acc = __double2float_rn(xv[u]);
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          const float cf = __fmul_rn(hf, __double2float_rn(p.coef[t]));
          acc = __fadd_rn(acc, __fmul_rn(cf, __double2float_rn(kv[u][t])));
        }
        row.xn[i] = v;
        v = (double)acc;
      }
      row.xst[i] = v;
      if (NT == 3 && p.write_p) {
        double pp = __dmul_rn(p.pb[0], kv[u][0]);
        pp = __dadd_rn(pp, __dmul_rn(p.pb[1], kv[u][1]));
        row.pp[i] = __dadd_rn(pp, __dmul_rn(p.pb[2], kv[u][2]));
      }
    }
    float sv, cv;
    dsincos(__double2float_rn(v), &sv, &cv);
#if MS_TC_PACKED == 1
    TcRec r;
    r.s = sv;
    r.c = cv;
    r.f = (double)__double2float_rn(wv[u]);  // b_fval, fs32
    rec[i] = r;
#elif MS_TC_PACKED == 3
    rec[i] = make_float2(sv, cv);  // F was written at creation
#else
    *reinterpret_cast<float2*>(rec + i) = make_float2(sv, cv);  // F was written at creation
#endif
    const T sh = K16<OPKS>::from(sv), ch = K16<OPKS>::from(cv);
    op[o_sh + i] = sh;
    op[o_sl + i] = K16<OPKS>::from(__fsub_rn(sv, (float)sh));
    op[o_ch + i] = ch;
    op[o_cl + i] = K16<OPKS>::from(__fsub_rn(cv, (float)ch));
  }
}

struct BRhsArgs {
  BatchDev d;
  int S, l, gate, out_slot, ws32, fs32;
  // last stage with MS_BFIN_EPI: the epilogue also forms x_tilde = x + h (P + b~4 k4)
  // (P = b~1 k1 + b~2 k2 + b~3 k3 from the last prep) and the weighted error of
  // solver.cpp:399-411 per element, reduced into d.errb / d.nfe
  int fin;
  double bt_last;
};

// coupling epilogue of one (row i, trajectory b): k = (double)(RN_WS(omega) +
// RN_WS(mw (c_i A - s_i B))), SS arithmetic
template <class SS, class GS>
__device__ __forceinline__ void b_epilogue(const BRhsArgs& a, int i, int b, SS A, SS Bv) {
  const BatchDev& d = a.d;
  Ctl* c = d.ctl + b;
  if (stage_skip(c, a.l, a.gate)) return;
  const int64_t e = (int64_t)b * d.n + i;
  const GS* sc = reinterpret_cast<const GS*>(d.sc);
  const SS si = (SS)sc[e], ci = (SS)sc[(int64_t)d.B * d.n + e];
  const SS coup = mul<SS>(cvt<SS>(d.mw), sub<SS>(mul<SS>(ci, A), mul<SS>(si, Bv)));
  const double o = ws_add(b_fval(d, e, a.fs32), (double)coup, a.ws32);
  bslot(d, a.S, a.out_slot, c)[i + (int64_t)b * d.n] = o;
  if (!isfinite(o)) atomicOr(&c->nf_mask, 1 << a.l);
}

// CUDA-core batched sweep: 64 rows x 32 trajectories per CTA, j in chunks of
// 32 through shared memory; each (i, b) sums j in ascending order — the
// oracle's split order, so with binary64 or binary32 sin/cos it matches it
// up to the libm ulp of sin/cos.
constexpr int kBT_I = 64, kBT_B = 32, kBT_J = 32;
template <class SS, class GS, int KS>
__global__ void __launch_bounds__(256) kb_rhs_cc(BRhsArgs a) {
  msb::count_launch();
  pdl_enter();
  const BatchDev& d = a.d;
  __shared__ GS Ks[kBT_I][kBT_J + 1];
  __shared__ GS Ss[kBT_B][kBT_J + 1];
  __shared__ GS Cs[kBT_B][kBT_J + 1];
  const int i0 = blockIdx.x * kBT_I, b0 = blockIdx.y * kBT_B;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;  // 16 x 16
  using KT = typename KElem<KS>::T;
  const KT* K = reinterpret_cast<const KT*>(d.K);
  const GS* S = reinterpret_cast<const GS*>(d.sc);
  const GS* Cc = S + (int64_t)d.B * d.n;
  SS A[4][2], Bv[4][2];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int q = 0; q < 2; ++q) { A[r][q] = SS(0); Bv[r][q] = SS(0); }
  for (int j0 = 0; j0 < d.n; j0 += kBT_J) {
    for (int t = threadIdx.x; t < kBT_I * kBT_J; t += 256) {
      const int r = t / kBT_J, jj = t % kBT_J;
      const int i = i0 + r, j = j0 + jj;
      Ks[r][jj] = (i < d.n && j < d.n) ? (GS)k2f(K[(int64_t)i * d.ld + j]) : GS(0);
    }
    for (int t = threadIdx.x; t < kBT_B * kBT_J; t += 256) {
      const int q = t / kBT_J, jj = t % kBT_J;
      const int b = b0 + q, j = j0 + jj;
      const bool ok = b < d.B && j < d.n;
      Ss[q][jj] = ok ? S[(int64_t)b * d.n + j] : GS(0);
      Cs[q][jj] = ok ? Cc[(int64_t)b * d.n + j] : GS(0);
    }
    __syncthreads();
    const int jn = min(kBT_J, d.n - j0);
    for (int jj = 0; jj < jn; ++jj) {
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const GS kv = Ks[ty * 4 + r][jj];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          A[r][q] = add<SS>(A[r][q], (SS)mul<GS>(kv, Ss[tx * 2 + q][jj]));
          Bv[r][q] = add<SS>(Bv[r][q], (SS)mul<GS>(kv, Cs[tx * 2 + q][jj]));
        }
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int i = i0 + ty * 4 + r, b = b0 + tx * 2 + q;
      if (i < d.n && b < d.B) b_epilogue<SS, GS>(a, i, b, A[r][q], Bv[r][q]);
    }
}

}  // namespace msb
