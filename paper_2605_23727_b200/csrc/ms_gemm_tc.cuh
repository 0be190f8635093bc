// ms_gemm_tc.cuh — the ensemble's stage contraction on the 5th-generation
// tensor cores (tcgen05), with the Kuramoto coupling as its fused epilogue.
//
//   A_bi = D[i][4b] + D[i][4b+1] = sum_j K_ij (s_hi + s_lo)(theta_bj)
//   B_bi = D[i][4b+2] + D[i][4b+3] = sum_j K_ij (c_hi + c_lo)(theta_bj)
//   k_b[i] = (double)(omega_bi + (1/N)(c_bi A_bi - s_bi B_bi))
//
// A = K (N x N, bf16/f16, K-major, row stride ld), B = the operand rows the
// prep kernel writes ([B][4][ld]: the two-term split of sin and of cos per
// trajectory, K-major), M = N, N_gemm = 4B, K_gemm = N. One CTA computes a
// 128 x 256 tile (64 trajectories):
//   warp 0        TMA producer: cp.async.bulk.tensor (SWIZZLE_128B) of the A
//                 and B k-blocks (64 columns) into a 4-stage mbarrier ring
//   warp 1        TMEM allocator + MMA issuer: one elected thread issues
//                 tcgen05.mma.cta_group::1.kind::f16 (M128 N256 K16) x 4 per
//                 k-block, fp32 accumulation in TMEM (256 columns), and
//                 tcgen05.commit releases each smem stage / signals the epilogue
//   warps 2..5    epilogue: tcgen05.ld 32x32b.x32 (one TMEM lane = one row),
//                 the coupling formula above in binary32, binary64 stores
// Each binary32 sin/cos value enters as hi + lo, both in K's 16-bit format
// (hi = RN16(v), lo = RN16(v - hi)); K is exact in its storage format, so every
// product is exact in fp32 and the operand keeps ~16 (bf16) / 22 (f16) bits.
// Accumulation order/precision is the tensor core's: parity with the oracle
// (same split) is by the reordering tolerance.
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <stdexcept>
#include <string>

#include "ms_batch.cuh"
#include "ms_dispatch.h"
#include "ms_tcgen05.cuh"

namespace msb {

// the error estimate folded into the last contraction's epilogue (MS_BFIN_EPI):
// compiled out unless MS_TC_FIN=1 (measured slower, ms_batch.cu bfin_epi_enabled)
#ifndef MS_TC_FIN
#define MS_TC_FIN 0
#endif
#ifndef MS_TC_REC128
#define MS_TC_REC128 0   // 128-bit loads of the epilogue records: measured 57 vs 39 us per contraction
#endif
#ifndef MS_TC_STCG
#define MS_TC_STCG 0     // st.global.cg for the k stores (else a generic store)
#endif
#ifndef MS_TC_STAGES
#define MS_TC_STAGES 2   // 2 x 48 KB: two CTAs per SM, one's epilogue overlaps the other's MMA
#endif
#ifndef MS_TC_EPI_WARPS
#define MS_TC_EPI_WARPS 8  // 4 or 8 (two warps per TMEM lane quarter, half the columns each)
#endif
#ifndef MS_TC_MINB
#define MS_TC_MINB 2
#endif
constexpr int kTcBM = 128, kTcBN = 256, kTcBK = 64, kTcStages = MS_TC_STAGES;
constexpr int kTcEpiWarps = MS_TC_EPI_WARPS;
constexpr int kTcABytes = kTcBM * kTcBK * 2;  // 16 KB
constexpr int kTcBBytes = kTcBN * kTcBK * 2;  // 32 KB
constexpr int kTcStageBytes = kTcABytes + kTcBBytes;
constexpr int kTcThreads = 64 + 32 * kTcEpiWarps;
constexpr size_t kTcSmem = 1024 /*align slack*/ + (size_t)kTcStages * kTcStageBytes + 256;

struct TcGemm {
  CUtensorMap tmA;
  CUtensorMap tmB;   // 256-row operand boxes (single-CTA kernel)
  CUtensorMap tmB2;  // 128-row operand boxes (CTA-pair kernel)
  int grid_m = 0, grid_n = 0;
  bool pair = true;  // CTA-pair kernel (MS_TC=1cta selects the single-CTA one)
  bool ready = false;
};

struct TcArgs {
  BRhsArgs a;
  int n, ncol;  // rows of K, GEMM columns (4B: s_hi, s_lo, c_hi, c_lo per trajectory)
  uint32_t idesc;
  // MS_TC_PDL=early: release the dependent launch (the next stage's prep / the
  // finalize) once this CTA's mainloop is done, so its blocks are scheduled while
  // the epilogue runs (they still wait for this grid in griddepcontrol.wait).
  // Measured slower (whole C5 solve 292 vs 282 ms: the waiting blocks crowd the
  // epilogue), so the default releases at exit
  int pdl_early;
  // MS_T2_DRAIN builds: k-blocks per accumulation window (MS_TC_WINDOW, default MS_T2_DRAIN)
  int window;
};

__device__ __forceinline__ void tc_ld32(uint32_t addr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(addr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void tc_ld32_nw(uint32_t addr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(addr));
}
__device__ __forceinline__ void tc_st32(uint32_t addr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(addr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void tc_ld8(uint32_t addr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(addr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tc_ld8_nw(uint32_t addr, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(addr));
}
__device__ __forceinline__ void tc_st8(uint32_t addr, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(addr), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
__device__ __forceinline__ void tc_ld16(uint32_t addr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(addr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Coupling epilogue of one warp: TMEM lane = row i, columns [c_beg, c_end) of
// the tile (4 per trajectory: s_hi, s_lo, c_hi, c_lo sums). The (s, c, omega) loads
// of the next 8 trajectories are issued before the current 8 are finished.
// The first 8 trajectories' records are loaded while the MMAs still run (the
// epilogue warps are idle until tmem_full), then the accumulators are awaited.
// per-trajectory inputs of the folded error estimate (TcArgs::a.fin)
struct TcFin {
  const double* x;   // x_n
  const double* xs;  // x_store (finite check)
  const double* xn;  // x_next (x_store unless binary32 storage)
  const double* p;   // P = b~1 k1 + b~2 k2 + b~3 k3
  double h, fw;      // h of the attempt, weight floor ab / rel
};

__device__ __forceinline__ void tc_fin_setup(const TcArgs& t, int b, TcFin& f) {
  const BatchDev& d = t.a.d;
  const Ctl* c = d.ctl + b;
  const int64_t o = (int64_t)b * d.n;
  const int ix = c->ix;
  f.x = d.xb[ix] + o;
  f.xs = d.xb[ix ^ 1] + o;
  f.xn = c->store32 ? d.xn + o : f.xs;
  f.p = d.scr1 + o;
  f.h = c->h_att;
  f.fw = __ddiv_rn(c->abs_tol, c->rel_tol);
}

__device__ __forceinline__ void tc_epilogue(const TcArgs& t, uint32_t lane_addr, int i, int tb0, int c_beg, int c_end,
                                            const int* skip, double* const* outp, uint64_t* tmem_full,
                                            const TcFin* fin = nullptr) {
  const BatchDev& d = t.a.d;
  const float mw = (float)d.mw;
  [[maybe_unused]] const float2* sc2 = reinterpret_cast<const float2*>(d.sc);  // (s, c)-pair record layouts
  const bool row_ok = i < t.n;
  TcRec cur[8];
  auto load = [&](int c0, TcRec (&v)[8]) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int tq = (c0 >> 2) + q;
      if (row_ok && !skip[tq]) {
        const int64_t e = (int64_t)(tb0 + tq) * d.n + i;
#if MS_TC_PACKED == 1
        v[q] = reinterpret_cast<const TcRec*>(d.sc)[e];
#elif MS_TC_PACKED == 2
#if MS_TC_REC128
        // one 128-bit load per record (the struct copy compiles to two LDG.64)
        const double2 raw = __ldg(reinterpret_cast<const double2*>(d.rec) + e);
        const unsigned long long sc_bits = (unsigned long long)__double_as_longlong(raw.x);
        v[q].s = __uint_as_float((unsigned)(sc_bits & 0xffffffffull));
        v[q].c = __uint_as_float((unsigned)(sc_bits >> 32));
        v[q].f = raw.y;
#else
        v[q] = reinterpret_cast<const TcRec*>(d.rec)[e];
#endif
#elif MS_TC_PACKED == 3
        const float2 p = sc2[e];
        v[q].s = p.x;
        v[q].c = p.y;
        v[q].f = (double)reinterpret_cast<const float*>(d.rec)[e];
#else
        const float2 p = sc2[e];
        v[q].s = p.x;
        v[q].c = p.y;
        v[q].f = b_fval(d, e, t.a.fs32);
#endif
      }
    }
  };
  load(c_beg, cur);
  tc_wait(tmem_full, 0);
  tc_fence_after();
  if (t.pdl_early) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#pragma unroll 1
  for (int c0 = c_beg; c0 < c_end; c0 += 32) {
    uint32_t r[32];
    tc_ld32(lane_addr + (uint32_t)c0, r);
#if MS_TC_FIN
    double rk[8];
#endif
    TcRec nxt[8];
    if (c0 + 32 < c_end) load(c0 + 32, nxt);
    if (row_ok) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int tq = (c0 >> 2) + q;
        if (skip[tq]) continue;
        const float A = __fadd_rn(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]));
        const float Bv = __fadd_rn(__uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3]));
        const float coup = __fmul_rn(mw, __fsub_rn(__fmul_rn(cur[q].c, A), __fmul_rn(cur[q].s, Bv)));
        MS_CHECK(i < d.n && tb0 + tq < d.B, "contraction epilogue: element outside the ensemble");
        const double o = ws_add(cur[q].f, (double)coup, t.a.ws32);
#if MS_TC_STCG
        __stcg(outp[tq] + i, o);  // a global store (the pointer comes through shared memory)
#else
        outp[tq][i] = o;
#endif
        if (!isfinite(o)) atomicOr(&d.ctl[tb0 + tq].nf_mask, 1 << t.a.l);
#if MS_TC_FIN
        if (fin) rk[q] = o;
#endif
      }
    }
#if MS_TC_FIN
    if (fin) {
      // the finalize's element loop for these 8 trajectories (kb_finalize order
      // and arithmetic; max and or are order-free, so the result is bitwise)
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int tq = (c0 >> 2) + q;
        if (skip[tq]) continue;  // uniform over the warp
        double m = 0.0;
        bool nf = false;
        if (row_ok) {
          const TcFin& fr = fin[tq];
          const double comb = __dadd_rn(fr.p[i], __dmul_rn(t.a.bt_last, rk[q]));
          const double xi = fr.x[i];
          const double xt = __dadd_rn(xi, __dmul_rn(fr.h, comb));
          const double xn = fr.xn[i];
          nf = !isfinite(xn) || !isfinite(xt) || !isfinite(fr.xs[i]);
          const double w = fmax(fmax(fabs(xi), fabs(xn)), fr.fw);
          m = fmax(0.0, __ddiv_rn(fabs(__dsub_rn(xn, xt)), w));
        }
#pragma unroll
        for (int sft = 16; sft >= 1; sft >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, sft));
        nf = __any_sync(0xffffffffu, nf);
        if ((threadIdx.x & 31) == 0) {
          atomicMax(d.errb + tb0 + tq, (unsigned long long)__double_as_longlong(m));
          if (nf) atomicOr(d.nfe + tb0 + tq, 1);
        }
      }
    }
#endif
#pragma unroll
    for (int q = 0; q < 8; ++q) cur[q] = nxt[q];
  }
}

__global__ void __launch_bounds__(kTcThreads, MS_TC_MINB)
    k_tc_gemm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, TcArgs t) {
  msb::count_launch();
  extern __shared__ __align__(1024) unsigned char tc_smem_raw[];
  // 1024-byte alignment for SWIZZLE_128B tiles
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(tc_smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)kTcStages * kTcStageBytes);
  uint64_t* empty = full + kTcStages;
  uint64_t* tmem_full = empty + kTcStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

  __shared__ int tc_skip[kTcBN / 4];
  __shared__ double* tc_out[kTcBN / 4];
#if MS_TC_FIN
  __shared__ TcFin tc_fin[kTcBN / 4];
#else
  constexpr TcFin* tc_fin = nullptr;
#endif
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * kTcBM, n0 = blockIdx.y * kTcBN;
  const int nkb = (t.n + kTcBK - 1) / kTcBK;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    for (int s = 0; s < kTcStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // TMA producer
      for (int kb = 0; kb < nkb; ++kb) {
        const int st = kb % kTcStages;
        if (kb >= kTcStages) tc_wait(&empty[st], ((kb / kTcStages) & 1) ^ 1);
        unsigned char* sa = smem + (size_t)st * kTcStageBytes;
        unsigned char* sb = sa + kTcABytes;
        mbar_expect_tx(&full[st], kTcStageBytes);
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
                smem_u32(sa)),
            "l"(reinterpret_cast<uint64_t>(&tmA)), "r"(smem_u32(&full[st])), "r"(kb * kTcBK), "r"(m0)
            : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
                smem_u32(sb)),
            "l"(reinterpret_cast<uint64_t>(&tmB)), "r"(smem_u32(&full[st])), "r"(kb * kTcBK), "r"(n0)
            : "memory");
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      for (int kb = 0; kb < nkb; ++kb) {
        const int st = kb % kTcStages;
        tc_wait(&full[st], (kb / kTcStages) & 1);
        tc_fence_after();
        const uint32_t sa = smem_u32(smem + (size_t)st * kTcStageBytes);
        const uint32_t sb = sa + kTcABytes;
#pragma unroll
        for (int k = 0; k < kTcBK / 16; ++k) {
          const uint64_t adesc = umma_smem_desc(sa + k * 32);
          const uint64_t bdesc = umma_smem_desc(sb + k * 32);
          const uint32_t acc = (kb > 0 || k > 0) ? 1u : 0u;
          asm volatile(
              "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
              " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
              "l"(adesc), "l"(bdesc), "r"(t.idesc), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_u32(&empty[st]))
                     : "memory");
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       smem_u32(tmem_full))
                   : "memory");
    }
  } else {  // epilogue warps 2..5: TMEM lanes 32*(warp%4) .. +32
    const int q4 = warp & 3;
    const int half = (warp - 2) >> 2;  // column half (8 epilogue warps) or 0
    const int et = threadIdx.x - 64;   // 0 .. 32*kTcEpiWarps-1
    const int tb0 = n0 >> 2;          // first trajectory of this tile
    const BatchDev& d = t.a.d;
    // per-trajectory decisions of this tile, read once (not per element)
    if (et < kTcBN / 4) {
      const int b = tb0 + et;
      int skip = 1;
      double* outp = nullptr;
      if (b < d.B) {
        const Ctl* c = d.ctl + b;
        skip = stage_skip(c, t.a.l, t.a.gate) ? 1 : 0;
        outp = bslot(d, t.a.S, t.a.out_slot, c) + (int64_t)b * d.n;
      }
      tc_skip[et] = skip;
      tc_out[et] = outp;
#if MS_TC_FIN
      if (t.a.fin && !skip) tc_fin_setup(t, b, tc_fin[et]);
#endif
    }
    asm volatile("bar.sync 1, %0;" ::"r"(32 * kTcEpiWarps) : "memory");
    const int i = m0 + q4 * 32 + lane;
    const uint32_t lane_addr = tmem + ((uint32_t)(q4 * 32) << 16);
    constexpr int kCols = kTcBN * 4 / kTcEpiWarps;  // columns per epilogue warp
    tc_epilogue(t, lane_addr, i, tb0, half * kCols, (half + 1) * kCols, tc_skip, tc_out, tmem_full,
                t.a.fin ? tc_fin : nullptr);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
  }
}

// ------------------------------------------------------------------------------
// CTA-pair variant (cta_group::2): a cluster of two CTAs on one TPC computes a
// 256 x 512 tile (128 trajectories). Each CTA stages its 128 rows of K and its
// two 128-column halves of the operand tile, so one k-block moves 96 KB for
// 16.8 MFLOP (5.7 B/kFLOP, against 11.4 for the single-CTA 128 x 256 tile):
// the stage contraction is bound by the L2->SM operand stream (~6.3 KB/cycle
// chip-wide), not by the tensor pipe, so halving the bytes per flop is the
// lever. The leader CTA (rank 0) issues tcgen05.mma.cta_group::2 M256 N256
// twice per k-step (columns 0-255 and 256-511 of the tile into TMEM columns
// 0-255 / 256-511 of both CTAs); both CTAs' TMA copies complete on the
// leader's full barrier, and the leader's commits arrive on both CTAs' empty
// barriers (multicast), so each producer refills only stages the pair's MMAs
// have drained. Each CTA's epilogue owns its 128 rows x 128 trajectories.
#ifndef MS_T2_BN
#define MS_T2_BN 512     // GEMM columns per pair tile: 512 (two N256 MMAs, all of TMEM) or 256
#endif
// MS_T2_SREC: the epilogue reads its {s, c, F} records from shared memory,
// staged by bulk copies (two 32 KB slots prefetched while the MMAs run, the
// rest into the drained operand ring), instead of per-thread global loads
#ifndef MS_T2_SREC
#define MS_T2_SREC 1
#endif
#ifndef MS_T2_STAGES
#if MS_T2_SREC
#define MS_T2_STAGES 3   // leaves room for the two prefetched record slots
#else
#define MS_T2_STAGES 4
#endif
#endif
#ifndef MS_T2_MINB
#define MS_T2_MINB 1
#endif
constexpr int kT2BM = 128;           // rows per CTA (256 per pair)
constexpr int kT2BN = MS_T2_BN;      // GEMM columns per pair tile
constexpr int kT2NMma = kT2BN / 256; // N256 MMAs per k-step
constexpr int kT2Half = 128;         // operand rows (columns of D) staged per CTA per MMA
constexpr int kT2Stages = MS_T2_STAGES;
#ifndef MS_T2_EPI
#define MS_T2_EPI 8      // epilogue warps: 4 TMEM lane quarters x (MS_T2_EPI / 4) column parts
#endif
constexpr int kT2EpiWarps = MS_T2_EPI;
constexpr int kT2ABytes = kT2BM * kTcBK * 2;               // 16 KB
constexpr int kT2BBytes = kT2NMma * kT2Half * kTcBK * 2;   // 16 KB per N256 MMA
constexpr int kT2StageBytes = kT2ABytes + kT2BBytes;
// MS_T2_DRAIN: 4 more warps join the window drains (12 warps = 3 per TMEM lane
// quarter, 88/88/80 columns each, so the running totals fit in registers)
#ifndef MS_T2_XWARPS
#define MS_T2_XWARPS 4
#endif
// MS_T2_REGEPI=1: the 12 drain warps run the coupling epilogue from their register
// totals instead of storing them back to TMEM for the 8-warp record-staged
// epilogue. Bitwise the same; measured 67.7 vs 47.5 us per contraction (three
// fully unrolled per-warp trajectory orders: a large instruction footprint), so off
#ifndef MS_T2_REGEPI
#define MS_T2_REGEPI 0
#endif
constexpr int kT2XWarps = MS_T2_DRAIN ? MS_T2_XWARPS : 0;
constexpr int kT2DrainWarpsPerQ = (kT2EpiWarps + kT2XWarps) / 4;   // drain warps per TMEM lane quarter
constexpr int kT2DrainCh = (32 + kT2DrainWarpsPerQ - 1) / kT2DrainWarpsPerQ;  // 8-column chunks per drain warp (max)
static_assert((kT2EpiWarps + kT2XWarps) % 4 == 0, "drain warps cover the lane quarters evenly");
constexpr int kT2Threads = 64 + 32 * (kT2EpiWarps + kT2XWarps);
// the windowed accumulation keeps up to 88 running totals per drain thread in
// registers: 14 warps per CTA put 4 on a sub-partition of 16 K registers, so
// 128 per thread is the ceiling
#if MS_T2_DRAIN
#define MS_T2_BOUNDS __maxnreg__(MS_T2_XWARPS == 4 ? 128 : (MS_T2_XWARPS == 8 ? 96 : 64))
#else
#define MS_T2_BOUNDS __launch_bounds__(kT2Threads, MS_T2_MINB)
#endif
// record staging (MS_T2_SREC): slot g holds the records of epilogue group g of
// both column parts (trajectories 8g..8g+7 and 64+8g..64+8g+7 of the pair tile)
// for this CTA's 128 rows: 16 x 128 x 16 B = 32 KB, laid out [part*8+q][row]
#if MS_TC_PACKED == 3
// (s, c) pairs and F in separate arrays: per trajectory a 128 x 8 B (s, c) block
// and a 128 x 4 B F block, each copied as the 16-byte-aligned run covering it
// (+16 B slack: ragged N leaves the source unaligned)
constexpr int kT2ScStride = kT2BM * 8 + 16, kT2FStride = kT2BM * 4 + 16;
constexpr int kT2SlotBytes = 16 * (kT2ScStride + kT2FStride);
constexpr int kT2SpareSlots = 3;
#else
constexpr int kT2ScStride = kT2BM * 16, kT2FStride = 0;  // whole 16-byte {s, c, F} records
constexpr int kT2SlotBytes = 16 * kT2BM * 16;
constexpr int kT2SpareSlots = 2;
#endif
constexpr int kT2NSlot = 8;
constexpr int kT2Spare = MS_T2_SREC ? kT2SpareSlots : 0;  // slots prefetched at kernel start
constexpr int kT2RingSlots = (kT2Stages * kT2StageBytes) / kT2SlotBytes;
constexpr int kT2RingUse = kT2RingSlots < kT2NSlot - kT2Spare ? kT2RingSlots : kT2NSlot - kT2Spare;
static_assert(!MS_T2_SREC || (kT2BN == 512 && kT2EpiWarps == 8 && !MS_TC_FIN), "record staging layout");
static_assert(!MS_T2_SREC || kT2Spare + kT2RingUse + kT2Spare >= kT2NSlot, "record slots: each spare reused once");
static_assert(!MS_T2_DRAIN || (MS_T2_SREC && kT2BN == 512 && kT2EpiWarps == 8), "windowed accumulation layout");
static_assert(!MS_T2_SREC || kT2NSlot - kT2Spare - kT2RingUse <= 2, "record slots: at most two spares refilled");
constexpr size_t kT2Smem = 1024 + (size_t)kT2Stages * kT2StageBytes + (size_t)kT2Spare * kT2SlotBytes + 256;

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t map_to_rank(uint32_t smem_addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// end-of-kernel pair barrier without release semantics: it only orders the two
// CTAs' TMEM use before the collective dealloc; a .release arrive compiles to
// MEMBAR.ALL.GPU, which makes every CTA wait for its k stores to drain first
// MS_T2_DRAIN_RELAXED: the drain warps' "window buffer read" arrive on the leader's barrier carries no
// memory release (see the arrive in the drain loop)
#ifndef MS_T2_DRAIN_RELAXED
#define MS_T2_DRAIN_RELAXED 1
#endif
#ifndef MS_T2_PRO_RELAXED
#define MS_T2_PRO_RELAXED 0  // measured no change (the prologue runs under the previous kernel's tail): the release barrier stays
#endif
#ifndef MS_T2_END_RELAXED
#define MS_T2_END_RELAXED 1
#endif
__device__ __forceinline__ void cluster_sync_end() {
#if MS_T2_END_RELAXED
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\nbarrier.cluster.wait.aligned;" ::: "memory");
#else
  cluster_sync_all();
#endif
}
__device__ __forceinline__ void tma2_load(uint32_t dst, const CUtensorMap* tm, uint32_t bar_cluster, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
      ::"r"(dst), "l"(reinterpret_cast<uint64_t>(tm)), "r"(bar_cluster), "r"(c0), "r"(c1)
      : "memory");
}

// Coupling epilogue with the records in shared memory (MS_T2_SREC): warp
// (q4, part) handles rows q4*32 + lane of this CTA and trajectories
// part*64 .. part*64+63 of the pair tile, eight per group g (TMEM columns
// part*256 + 32g ..), group g's records in slot g. The arithmetic is
// tc_epilogue's, element for element.
template <class SlotPtr>
__device__ __forceinline__ void tc_epilogue_srec(const TcArgs& t, uint32_t lane_addr, int i, int rr, int tb0, int part,
                                                 const int* skip, double* const* outp, uint64_t* tmem_full,
                                                 uint64_t* rec_full, uint64_t* rec_free, SlotPtr slot_ptr) {
  const BatchDev& d = t.a.d;
  const float mw = (float)d.mw;
  const bool row_ok = i < t.n;
#if MS_T2_DRAIN
  (void)tmem_full;  // the caller's window drains stored the totals in TMEM columns 0..255
#else
  tc_wait(tmem_full, 0);
  tc_fence_after();
#endif
#pragma unroll 1
  for (int g = 0; g < kT2NSlot; ++g) {
#ifndef MS_T2_EXP_EPI  // timing experiments only (results wrong): 1 no k stores, 2 no record reads, 3 no TMEM loads
#define MS_T2_EXP_EPI 0
#endif
#if MS_T2_DRAIN
    // totals (A, B) of trajectory part*64 + 8g + q in columns part*128 + 16g + 2q, +1
    uint32_t r[16];
    tc_ld16(lane_addr + (uint32_t)(part * 128 + g * 16), r);
#else
    uint32_t r[32];
#if MS_T2_EXP_EPI == 3
#pragma unroll
    for (int k = 0; k < 32; ++k) r[k] = (uint32_t)(k + g);
#else
    tc_ld32(lane_addr + (uint32_t)(part * 256 + g * 32), r);
#endif
#endif
#if MS_T2_EXP_EPI != 2
    tc_wait(&rec_full[g], 0);
#endif
    const unsigned char* sb = slot_ptr(g);
    if (row_ok) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int tq = part * 64 + g * 8 + q;
        if (skip[tq]) continue;
#if MS_T2_EXP_EPI == 2
        const TcRec rc{0.5f + (float)q, 0.25f, 1.0};
        (void)sb;
#else
        const int j = part * 8 + q;
#if MS_TC_PACKED == 3
        // block j starts at the 16-byte boundary below the trajectory's first row
        const int64_t e0 = (int64_t)(tb0 + tq) * d.n + (i - rr);
        const uint32_t sco = (uint32_t)(reinterpret_cast<uintptr_t>(reinterpret_cast<const float2*>(d.sc) + e0) & 15);
        const uint32_t fo = (uint32_t)(reinterpret_cast<uintptr_t>(reinterpret_cast<const float*>(d.rec) + e0) & 15);
        const float2 scv = *reinterpret_cast<const float2*>(sb + (size_t)j * kT2ScStride + sco + (size_t)rr * 8);
        const float fv = *reinterpret_cast<const float*>(sb + 16 * kT2ScStride + (size_t)j * kT2FStride + fo + (size_t)rr * 4);
        const TcRec rc{scv.x, scv.y, (double)fv};
#else
        const TcRec rc = *reinterpret_cast<const TcRec*>(sb + (size_t)j * kT2ScStride + (size_t)rr * 16);
#endif
#endif
#if MS_T2_DRAIN
        const float A = __uint_as_float(r[2 * q]), Bv = __uint_as_float(r[2 * q + 1]);
#else
        const float A = __fadd_rn(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]));
        const float Bv = __fadd_rn(__uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3]));
#endif
        const float coup = __fmul_rn(mw, __fsub_rn(__fmul_rn(rc.c, A), __fmul_rn(rc.s, Bv)));
        MS_CHECK(i < d.n && (tb0 + tq < d.B), "contraction epilogue: element outside the ensemble");
        const double o = ws_add(rc.f, (double)coup, t.a.ws32);
#if MS_T2_EXP_EPI == 1
        if (o == 12345.678) outp[tq][i] = o;
#else
        outp[tq][i] = o;
#endif
        if (!isfinite(o)) atomicOr(&d.ctl[tb0 + tq].nf_mask, 1 << t.a.l);
      }
    }
    if (g < kT2Spare && kT2Spare + kT2RingUse + g < kT2NSlot) {  // this spare is refilled with a later slot
      __syncwarp();
      if ((threadIdx.x & 31) == 0) mbar_arrive(&rec_free[g]);
    }
  }
}

__global__ void __cluster_dims__(2, 1, 1) MS_T2_BOUNDS
    k_tc_gemm2(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, TcArgs t) {
  msb::count_launch();
  extern __shared__ __align__(1024) unsigned char tc_smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(tc_smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* spare = smem + (size_t)kT2Stages * kT2StageBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(spare + (size_t)kT2Spare * kT2SlotBytes);
  uint64_t* empty = full + kT2Stages;
  uint64_t* tmem_full = empty + kT2Stages;
  uint64_t* rec_full = tmem_full + 1;       // [kT2NSlot] (MS_T2_SREC)
  uint64_t* rec_free = rec_full + kT2NSlot; // [2]: a spare slot's first records consumed
  uint64_t* drain_full = rec_free + 2;      // MS_T2_DRAIN [2]: a window's MMAs into TMEM buffer b are done (both CTAs)
  uint64_t* drain_empty = drain_full + 2;   // [2]: buffer b has been read (leader; 16 warps of the pair)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(drain_empty + 2);
  // where record slot g lives: spare 0/1, then the drained ring, then the spares again
  auto slot_ptr = [&](int g) -> unsigned char* {
    if (g < kT2Spare) return spare + (size_t)g * kT2SlotBytes;
    if (g < kT2Spare + kT2RingUse) return smem + (size_t)(g - kT2Spare) * kT2SlotBytes;
    return spare + (size_t)((g - kT2Spare - kT2RingUse) & 1) * kT2SlotBytes;
  };
  (void)slot_ptr;

  __shared__ int tc_skip[kT2BN / 4];
  __shared__ double* tc_out[kT2BN / 4];
#if MS_TC_FIN
  __shared__ TcFin tc_fin[kT2BN / 4];
#else
  constexpr TcFin* tc_fin = nullptr;
  (void)tc_fin;
#endif
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int m0 = (blockIdx.x >> 1) * (2 * kT2BM) + (int)rank * kT2BM;  // this CTA's rows
  const int n0 = blockIdx.y * kT2BN;                                    // the pair's columns
  const int nkb = (t.n + kTcBK - 1) / kTcBK;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    for (int s = 0; s < kT2Stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    for (int g = 0; g < kT2NSlot; ++g) mbar_init(&rec_full[g], 1);
    mbar_init(&rec_free[0], kT2EpiWarps);
    mbar_init(&rec_free[1], kT2EpiWarps);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&drain_full[b], 1);
      mbar_init(&drain_empty[b], 2 * (kT2EpiWarps + kT2XWarps));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {  // same warp in both CTAs (cta_group::2 allocation is collective over the pair)
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(kT2BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
#if MS_T2_PRO_RELAXED
  // the barrier inits were published cluster-wide by fence.mbarrier_init.release.cluster,
  // the TMEM slot is this CTA's own shared memory (__syncthreads): the pair barrier only
  // has to order execution, and a .release arrive is a MEMBAR.ALL.GPU in every thread
  __syncthreads();
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
#else
  cluster_sync_all();  // the peer's barriers exist before any remote arrive
#endif
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // the prologue above (barriers, TMEM, tensor-map prefetch) overlaps the
  // prep's tail; everything below reads what the prep wrote. The successor is
  // not released early (its blocks would sit on the SMs through the mainloop)
  asm volatile("griddepcontrol.wait;" ::: "memory");

  // bulk copies of record slot g: for each valid trajectory of the slot, this
  // CTA's rows [m0, m0 + rows) are one contiguous 16-byte-per-row run
  auto issue_slot = [&](int g) {
    const BatchDev& d = t.a.d;
    const int rows = min(kT2BM, d.n - m0);
    const int tb0 = n0 >> 2;
    unsigned char* dst = slot_ptr(g);
#if MS_TC_PACKED == 3
    // per valid trajectory: the 16-byte-aligned runs covering its (s, c) rows and
    // F rows (the epilogue recomputes each run's start offset from the address)
    auto run = [](const void* src, uint32_t bytes, uint32_t& lo_off) {
      const uintptr_t a = reinterpret_cast<uintptr_t>(src);
      const uintptr_t lo = a & ~uintptr_t(15), hi = (a + bytes + 15) & ~uintptr_t(15);
      lo_off = (uint32_t)(a - lo);
      return (uint32_t)(hi - lo);
    };
    uint32_t total = 0;
    if (rows > 0)
      for (int j = 0; j < 16; ++j) {
        const int b = tb0 + (j >> 3) * 64 + g * 8 + (j & 7);
        if (b >= d.B) continue;
        uint32_t o;
        total += run(reinterpret_cast<const float2*>(d.sc) + (int64_t)b * d.n + m0, rows * 8, o);
        total += run(reinterpret_cast<const float*>(d.rec) + (int64_t)b * d.n + m0, rows * 4, o);
      }
    mbar_expect_tx(&rec_full[g], total);
    if (rows <= 0) return;
    for (int j = 0; j < 16; ++j) {
      const int b = tb0 + (j >> 3) * 64 + g * 8 + (j & 7);
      if (b >= d.B) continue;
      uint32_t o1, o2;
      const float2* s1 = reinterpret_cast<const float2*>(d.sc) + (int64_t)b * d.n + m0;
      const float* s2 = reinterpret_cast<const float*>(d.rec) + (int64_t)b * d.n + m0;
      const uint32_t n1 = run(s1, rows * 8, o1), n2 = run(s2, rows * 4, o2);
      unsigned char* d1 = dst + (size_t)j * kT2ScStride;
      unsigned char* d2 = dst + 16 * kT2ScStride + (size_t)j * kT2FStride;
      bulk_g2s(d1, reinterpret_cast<const unsigned char*>(s1) - o1, n1, &rec_full[g]);
      bulk_g2s(d2, reinterpret_cast<const unsigned char*>(s2) - o2, n2, &rec_full[g]);
    }
#else
    uint32_t bytes = 0;
    if (rows > 0)
      for (int j = 0; j < 16; ++j) bytes += (tb0 + (j >> 3) * 64 + g * 8 + (j & 7) < d.B) ? rows * 16 : 0;
    mbar_expect_tx(&rec_full[g], bytes);
    if (rows <= 0) return;
    const TcRec* rec = reinterpret_cast<const TcRec*>(d.rec);
    for (int j = 0; j < 16; ++j) {
      const int b = tb0 + (j >> 3) * 64 + g * 8 + (j & 7);
      if (b < d.B) bulk_g2s(dst + (size_t)j * kT2ScStride, rec + (int64_t)b * d.n + m0, (uint32_t)rows * 16, &rec_full[g]);
    }
#endif
  };
  (void)issue_slot;

  if (warp == 0) {
    if (lane == 0) {  // TMA producer (both CTAs): own smem, completion on the leader's barrier
#if MS_T2_SREC && MS_T2_EXP_EPI != 2
      for (int g = 0; g < kT2Spare; ++g) issue_slot(g);  // overlap the mainloop
#endif
      for (int kb = 0; kb < nkb; ++kb) {
        const int st = kb % kT2Stages;
        if (kb >= kT2Stages) tc_wait(&empty[st], ((kb / kT2Stages) & 1) ^ 1);
        const uint32_t sa = smem_u32(smem + (size_t)st * kT2StageBytes);
        const uint32_t sb = sa + kT2ABytes;
#ifndef MS_T2_EXP_NB
#define MS_T2_EXP_NB kT2NMma  // timing experiments only: operand halves loaded per k-block (results wrong if fewer)
#endif
        if (rank == 0) mbar_expect_tx(&full[st], 2 * (kT2ABytes + MS_T2_EXP_NB * (kT2Half * kTcBK * 2)));
        const uint32_t bar = map_to_rank(smem_u32(&full[st]), 0);
        tma2_load(sa, &tmA, bar, kb * kTcBK, m0);
#pragma unroll
        for (int hf = 0; hf < MS_T2_EXP_NB; ++hf)
#if MS_T2_DRAIN
          // plane hf (hi, lo): the (s, c) rows of the pair's 128 trajectories, this CTA's half
          tma2_load(sb + hf * (kT2Half * kTcBK * 2), &tmB, bar, kb * kTcBK,
                    hf * 2 * t.a.d.B + 2 * (n0 >> 2) + (int)rank * kT2Half);
#else
          tma2_load(sb + hf * (kT2Half * kTcBK * 2), &tmB, bar, kb * kTcBK, n0 + hf * 2 * kT2Half + (int)rank * kT2Half);
#endif
      }
#if MS_T2_SREC && MS_T2_EXP_EPI != 2
      // the ring is free once the last use of every stage has been committed
      // (the leader's commits arrive on both CTAs' empty barriers)
      for (int st = 0; st < kT2Stages && st < nkb; ++st) {
        const int kb_last = st + ((nkb - 1 - st) / kT2Stages) * kT2Stages;
        tc_wait(&empty[st], (kb_last / kT2Stages) & 1);
      }
      for (int g = kT2Spare; g < kT2Spare + kT2RingUse; ++g) issue_slot(g);
      for (int g = kT2Spare + kT2RingUse; g < kT2NSlot; ++g) {
        tc_wait(&rec_free[(g - kT2Spare - kT2RingUse) & 1], 0);  // the spare's first slot is consumed
        issue_slot(g);
      }
#endif
    }
    if (t.pdl_early) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {  // MMA issuer: the leader only
      for (int kb = 0; kb < nkb; ++kb) {
        const int st = kb % kT2Stages;
#if MS_T2_DRAIN
        // window wv accumulates into TMEM buffer wv & 1 from zero; it may start once
        // both CTAs' epilogue warps have read that buffer's previous window (wv - 2)
        const int wv = kb / t.window;
        if (kb % t.window == 0 && wv >= 2) tc_wait(&drain_empty[wv & 1], ((wv >> 1) - 1) & 1);
#endif
        tc_wait(&full[st], (kb / kT2Stages) & 1);
        tc_fence_after();
        const uint32_t sa = smem_u32(smem + (size_t)st * kT2StageBytes);
        const uint32_t sb = sa + kT2ABytes;
#pragma unroll
        for (int k = 0; k < kTcBK / 16; ++k) {
          const uint64_t adesc = umma_smem_desc(sa + k * 32);
#if MS_T2_DRAIN
          const uint32_t acc0 = (kb % t.window > 0 || k > 0) ? 1u : 0u;  // the window's first MMA overwrites
#else
          const uint32_t acc = (kb > 0 || k > 0) ? 1u : 0u;
#endif
#ifndef MS_T2_EXP_NMMA
#define MS_T2_EXP_NMMA kT2NMma  // timing experiments only: MMAs issued per k-step
#endif
#pragma unroll
          for (int hf = 0; hf < MS_T2_EXP_NMMA; ++hf) {
            const uint64_t bdesc = umma_smem_desc(sb + hf * (kT2Half * kTcBK * 2) + k * 32);
#if MS_T2_DRAIN
            // hi and lo planes into the same accumulator (the window's buffer)
            const uint32_t acc = hf > 0 ? 1u : acc0;
            const uint32_t dcol = (uint32_t)((wv & 1) * 256);
#else
            const uint32_t dcol = (uint32_t)(hf * 256);
#endif
            asm volatile(
                "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                " tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem + dcol),
                "l"(adesc), "l"(bdesc), "r"(t.idesc), "r"(acc));
          }
        }
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                smem_u32(&empty[st])),
            "h"((uint16_t)3)
            : "memory");
#if MS_T2_DRAIN
        if (kb % t.window == t.window - 1 || kb == nkb - 1)
          asm volatile(
              "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                  smem_u32(&drain_full[wv & 1])),
              "h"((uint16_t)3)
              : "memory");
#endif
      }
      asm volatile(
          "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
              smem_u32(tmem_full)),
          "h"((uint16_t)3)
          : "memory");
    }
    if (t.pdl_early) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  } else {  // epilogue: TMEM lane quarter warp%4, column part (warp-2)/4
    const int q4 = warp & 3;
    const int part = (warp - 2) >> 2;
    const int et = threadIdx.x - 64;
    const int tb0 = n0 >> 2;  // first trajectory of the pair tile (both CTAs: same columns)
    const BatchDev& d = t.a.d;
    if (et < kT2BN / 4) {
      const int b = tb0 + et;
      int skip = 1;
      double* outp = nullptr;
      if (b < d.B) {
        const Ctl* c = d.ctl + b;
        skip = stage_skip(c, t.a.l, t.a.gate) ? 1 : 0;
        outp = bslot(d, t.a.S, t.a.out_slot, c) + (int64_t)b * d.n;
      }
      tc_skip[et] = skip;
      tc_out[et] = outp;
#if MS_TC_FIN
      if (t.a.fin && !skip) tc_fin_setup(t, b, tc_fin[et]);
#endif
    }
    asm volatile("bar.sync 1, %0;" ::"r"(32 * (kT2EpiWarps + kT2XWarps)) : "memory");
    const int i = m0 + q4 * 32 + lane;
    const uint32_t lane_addr = tmem + ((uint32_t)(q4 * 32) << 16);
    constexpr int kCols = kT2BN / (kT2EpiWarps / 4);  // columns per epilogue warp
#if MS_T2_DRAIN
    // window drains: each window's sums (TMEM buffer wv & 1: 128 trajectories x
    // (A, B) in columns 0..255) are added into binary32 running totals in
    // registers (RN) and the buffer is released for window wv + 2 while the MMAs
    // of window wv + 1 fill the other one. Each window starts from zero, so the
    // tensor core never adds into a large running sum: its truncation per add
    // stays at a window's scale instead of biasing the whole K sum. Warp j of a
    // lane quarter owns 8-column chunks [11 j, min(32, 11 j + 11)).
    {
      constexpr int kMaxCh = kT2DrainCh;
      const int jw = (warp - 2) >> 2;
      const int ch0 = jw * kMaxCh, nch = min(kMaxCh, 32 - ch0);
      float R[kMaxCh * 8];
      const int nwin = (nkb + t.window - 1) / t.window;
      const uint32_t remote_empty0 = map_to_rank(smem_u32(&drain_empty[0]), 0);
#pragma unroll 1
      for (int wv = 0; wv < nwin; ++wv) {
        const int buf = wv & 1;
        tc_wait(&drain_full[buf], (wv >> 1) & 1);
        tc_fence_after();
        // two 8-column loads in flight per wait; the buffer is released as soon
        // as its last load has landed
#pragma unroll
        for (int c = 0; c < kMaxCh; c += 2) {
          uint32_t dv[16];
          if (c < nch) tc_ld8_nw(lane_addr + (uint32_t)(buf * 256 + (ch0 + c) * 8), dv);
          if (c + 1 < kMaxCh && c + 1 < nch) tc_ld8_nw(lane_addr + (uint32_t)(buf * 256 + (ch0 + c + 1) * 8), dv + 8);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          if (c < nch && c + 2 >= nch) {  // this warp's last pair: exactly one arrive per window
            tc_fence_before();
            __syncwarp();
            if (lane == 0)
#if MS_T2_DRAIN_RELAXED
              // the buffer's reads are complete (tcgen05.wait::ld) and fenced for the issuer
              // (tcgen05.fence::before_thread_sync); no memory of this thread has to be
              // published. A .release.cluster arrive compiles to MEMBAR.ALL.GPU + ERRBAR in
              // every drain warp, once per window, in the path that frees the buffer
              asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote_empty0 + 8u * buf)
                           : "memory");
#else
              asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote_empty0 + 8u * buf)
                           : "memory");
#endif
          }
#ifndef MS_T2_EXP_DRAIN  // timing experiments only (results wrong): 1 = no adds into the totals
#define MS_T2_EXP_DRAIN 0
#endif
#pragma unroll
          for (int h = 0; h < 2; ++h)
            if (c + h < kMaxCh && c + h < nch) {
#pragma unroll
              for (int k = 0; k < 8; ++k)
#if MS_T2_EXP_DRAIN == 1
                R[(c + h) * 8 + k] = __uint_as_float(dv[h * 8 + k]);
#else
                R[(c + h) * 8 + k] = wv > 0 ? __fadd_rn(R[(c + h) * 8 + k], __uint_as_float(dv[h * 8 + k]))
                                            : __uint_as_float(dv[h * 8 + k]);
#endif
            }
        }
      }
#if MS_T2_REGEPI
      // the coupling epilogue straight from the registers: warp jw's 44 (jw = 2:
      // 40) trajectories in record-slot order -- slots 6 and 7 reuse the spare
      // buffers of slots 0 and 1, so every warp finishes those first
      {
        static_assert(kT2XWarps == 4 && kMaxCh == 11 && MS_TC_PACKED == 2 && MS_T2_SREC, "register epilogue layout");
        const BatchDev& d = t.a.d;
        const float mw = (float)d.mw;
        const int rr = q4 * 32 + lane;
        const bool row_ok = i < t.n;
        auto one = [&](const int c2) {
          const int tq = jw * 44 + c2;
          const int g = (tq & 63) >> 3, jj = (tq >> 6) * 8 + (tq & 7);
          tc_wait(&rec_full[g], 0);
          if (row_ok && !tc_skip[tq]) {
            const TcRec rc = *reinterpret_cast<const TcRec*>(slot_ptr(g) + (size_t)jj * kT2ScStride + (size_t)rr * 16);
            const float A = R[2 * c2], Bv = R[2 * c2 + 1];
            const float coup = __fmul_rn(mw, __fsub_rn(__fmul_rn(rc.c, A), __fmul_rn(rc.s, Bv)));
            MS_CHECK(i < d.n && tb0 + tq < d.B, "contraction epilogue: element outside the ensemble");
            const double o = ws_add(rc.f, (double)coup, t.a.ws32);
            tc_out[tq][i] = o;
            if (!isfinite(o)) atomicOr(&d.ctl[tb0 + tq].nf_mask, 1 << t.a.l);
          }
        };
        auto release = [&](int g) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&rec_free[g]);
        };
        if (jw == 0) {  // trajectories 0..43: slots 0..5
#pragma unroll
          for (int c2 = 0; c2 < 44; ++c2) {
            one(c2);
            if (c2 == 7) release(0);
            if (c2 == 15) release(1);
          }
        } else if (jw == 1) {  // 64..87 (slots 0..2) first, then 44..63 (slots 5..7)
#pragma unroll
          for (int c2 = 20; c2 < 44; ++c2) {
            one(c2);
            if (c2 == 27) release(0);
            if (c2 == 35) release(1);
          }
#pragma unroll
          for (int c2 = 0; c2 < 20; ++c2) one(c2);
        } else {  // 88..127: slots 3..7
#pragma unroll
          for (int c2 = 0; c2 < 40; ++c2) one(c2);
        }
      }
#else
      // all MMAs are done: the totals go back to buffer 0 (same columns) for the
      // record-staged epilogue, which reads them with the 8-warp column split
#pragma unroll
      for (int c = 0; c < kMaxCh; ++c)
        if (c < nch) tc_st8(lane_addr + (uint32_t)((ch0 + c) * 8), reinterpret_cast<const uint32_t*>(R) + c * 8);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      asm volatile("bar.sync 1, %0;" ::"r"(32 * (kT2EpiWarps + kT2XWarps)) : "memory");
      tc_fence_after();
#endif
    }
    if (MS_T2_REGEPI || warp - 2 >= kT2EpiWarps) {
      (void)kCols;
    } else
#endif
    {
#ifndef MS_T2_NOEPI
#if MS_T2_SREC
    (void)kCols;
    tc_epilogue_srec(t, lane_addr, i, q4 * 32 + lane, tb0, part, tc_skip, tc_out, tmem_full, rec_full, rec_free,
                     slot_ptr);
#else
    tc_epilogue(t, lane_addr, i, tb0, part * kCols, (part + 1) * kCols, tc_skip, tc_out, tmem_full,
                t.a.fin ? tc_fin : nullptr);
#endif
#else
    tc_wait(tmem_full, 0);
    tc_fence_after();
    (void)lane_addr; (void)i; (void)kCols;
#endif
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_end();  // both CTAs done with the pair's TMEM and barriers
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kT2BN));
  }
}

inline void tc_gemm_setup(TcGemm& g, const BatchDev& d, int sms) {
  (void)sms;
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
      throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const CUtensorMapDataType dt = d.ks == MS_K_F16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  {
    const cuuint64_t dims[2] = {(cuuint64_t)d.n, (cuuint64_t)d.n};
    const cuuint64_t strides[1] = {(cuuint64_t)d.ld * 2};
    const cuuint32_t box[2] = {kTcBK, kTcBM};
    const cuuint32_t es[2] = {1, 1};
    CUresult r = encode(&g.tmA, dt, 2, const_cast<void*>(d.K), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw std::runtime_error("tensor map (K) encode failed");
  }
  {
    const cuuint64_t dims[2] = {(cuuint64_t)d.n, (cuuint64_t)(4 * d.B)};
    const cuuint64_t strides[1] = {(cuuint64_t)d.ld * 2};
    const cuuint32_t box[2] = {kTcBK, kTcBN};
    const cuuint32_t es[2] = {1, 1};
    CUresult r = encode(&g.tmB, dt, 2, d.op, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw std::runtime_error("tensor map (operand) encode failed");
    const cuuint32_t box2[2] = {kTcBK, kT2Half};
    r = encode(&g.tmB2, dt, 2, d.op, dims, strides, box2, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw std::runtime_error("tensor map (operand, pair) encode failed");
  }
  const char* v = std::getenv("MS_TC");
  g.pair = !(v && std::string(v) == "1cta");
  if (!g.pair && MS_T2_DRAIN)
    throw std::runtime_error("MS_TC=1cta needs a build with MS_T2_DRAIN=0 (the pair kernel's operand planes)");
  if (g.pair) {
    g.grid_m = 2 * ((d.n + 2 * kT2BM - 1) / (2 * kT2BM));
    g.grid_n = (4 * d.B + kT2BN - 1) / kT2BN;
    if (const char* gn = std::getenv("MS_T2_GRIDN")) g.grid_n = std::max(1, std::min(g.grid_n, std::atoi(gn)));  // tuning only
    cudaError_t e = cudaFuncSetAttribute(k_tc_gemm2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kT2Smem);
    if (e != cudaSuccess) throw std::runtime_error(std::string("tc gemm2 smem attribute: ") + cudaGetErrorString(e));
  } else {
    g.grid_m = (d.n + kTcBM - 1) / kTcBM;
    g.grid_n = (4 * d.B + kTcBN - 1) / kTcBN;
    cudaError_t e = cudaFuncSetAttribute(k_tc_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTcSmem);
    if (e != cudaSuccess) throw std::runtime_error(std::string("tc gemm smem attribute: ") + cudaGetErrorString(e));
  }
  g.ready = true;
}

inline void tc_gemm_teardown(TcGemm& g) { g.ready = false; }

// instruction descriptor of tcgen05.mma kind::f16: D f32, A/B bf16 (1) or
// f16 (0), both K-major, N = 256, M = 128 (single CTA) or 256 (CTA pair)
inline uint32_t tc_idesc(int ks, int m) {
  const uint32_t ab = ks == MS_K_F16 ? 0u : 1u;
  return (1u << 4) | (ab << 7) | (ab << 10) | ((uint32_t)(256 >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

inline void launch_tc_gemm(const TcGemm& g, const BRhsArgs& a, cudaStream_t st) {
  if (!g.ready) throw std::runtime_error("tensor-core GEMM not set up");
  TcArgs t{};
  t.a = a;
  t.n = a.d.n;
  t.ncol = 4 * a.d.B;
  dim3 grid(g.grid_m, g.grid_n);
  {
    const char* v = std::getenv("MS_TC_PDL");  // read per launch (graphs capture it once)
    t.pdl_early = (v && std::string(v) == "early") ? 1 : 0;
  }
  t.window = MS_T2_DRAIN > 0 ? MS_T2_DRAIN : 1;
  if (const char* wv = std::getenv("MS_TC_WINDOW")) t.window = std::max(1, std::atoi(wv));  // read per launch
  if (g.pair) {
    t.idesc = tc_idesc(a.d.ks, 2 * kT2BM);
    cudaError_t e = launch_k(k_tc_gemm2, grid, kT2Threads, kT2Smem, st, g.tmA, g.tmB2, t);
    if (e != cudaSuccess) throw std::runtime_error(std::string("tc gemm2 launch: ") + cudaGetErrorString(e));
  } else {
    t.idesc = tc_idesc(a.d.ks, kTcBM);
    k_tc_gemm<<<grid, kTcThreads, kTcSmem, st>>>(g.tmA, g.tmB, t);
  }
}

}  // namespace msb
