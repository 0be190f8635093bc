// ms_multi.cuh — one K sweep for several concurrent solves.
//
// The reference's harness runs the Single/Mixed1/Mixed2/Double variants of a
// test case one after another on the same system (harness.cpp:113-121). Run
// in lock-step on the device, their stage evaluations can share the K stream:
// k_rhs_multi reads each K element once and accumulates it into every active
// lane's sums, each lane in its own stage precision — a GEMV turned into a
// narrow GEMM on the CUDA cores.
//
//   producer warp   per stage: one 2D tensor copy of a 32-row x (32*VEC)-column
//                   K tile + the lanes' sin/cos columns (bulk copies) into an
//                   8-deep mbarrier ring (~24 KB per stage for f32 K)
//   16 consumer     warp w owns rows w and w+16 of the 32-row group; lane l
//   warps           owns columns VEC*l .. VEC*l+VEC-1 of every tile, so each
//                   lane of each row sums columns VEC*l + 32*VEC*m in
//                   ascending m — the order of the single-solve sweeps — and
//                   the row total comes from the same shuffle tree: every
//                   lane's result is bit-identical to its own solve. Geometry
//                   from tools/tune_multi.py (profiles/r1_tune_multi.txt).
//
// Lane types are compile-time: NS lanes (SS, GS) = (f32, f32), NDS lanes
// (f64, f32), NDD lanes (f64, f64), in that order (the host sorts them).
// Binary64 sums over binary32 products need one f32->f64 conversion per
// product; those conversions (XU pipe, 16/clk/SM) bound the fp64-heavy mixes.
#pragma once

#include <cuda.h>

#include "ms_kernels.cuh"

namespace msb {

constexpr int kMaxLanes = 4;

struct LaneArgs {
  const Ctl* ctl;
  int* nf_mask;
  const void* gin;    // GS-typed s (ld) then c (ld)
  const double* fvc;  // F of the coupled slot (FS value)
  double* kb[kMaxStages + 1];
  int ws32;
  int _pad;
};

struct MultiArgs {
  LaneArgs lane[kMaxLanes];
  int nl;
  int l, gate, S, out_slot;
  int64_t ld;
  int n, row0, row1;
  double mw;
  Ctl* count_ctl;  // single-lane row-sharded loop: the sweep counts (RhsArgs::count)
  int count;
  int k_stream;    // K beyond L2: evict-first tile loads (RhsArgs::k_stream)
  PushDev push;    // single-lane row-sharded loop: push exchange (RhsArgs::push)
};

#ifndef MS_MULTI_WARPS
#define MS_MULTI_WARPS 16
#endif
#ifndef MS_MULTI_R
#define MS_MULTI_R 2
#endif
constexpr int kMultiWarps = MS_MULTI_WARPS;      // consumer warps
constexpr int kMultiR = MS_MULTI_R;              // rows per consumer warp
constexpr int kMultiTR = kMultiWarps * kMultiR;  // rows per group / K tile
constexpr int kMultiThreads = (kMultiWarps + 1) * 32;

#ifndef MS_MULTI_R1
#define MS_MULTI_R1 2    // rows per warp of the one-lane tile sweep (4 measured slower: C4 f16 5.84 vs 6.1 TB/s)
#endif
template <int KS, int NL = kMaxLanes>
struct MultiGeom {
  using KT = typename KElem<KS>::T;
  static constexpr int VEC = KVec<KS>::N;
  static constexpr int TC = 32 * VEC;                          // tile columns = one warp step
  // one lane: more rows per warp share each staged sin/cos value (the 16-bit
  // sweep is shared-memory bound at 2 rows)
  static constexpr int R = NL == 1 ? MS_MULTI_R1 : kMultiR;
  static constexpr int TR = kMultiWarps * R;                   // rows per group / K tile
  static constexpr int KTILE = TR * TC * (int)sizeof(KT);
  static constexpr int LANEB = 2 * TC * 8;                     // s + c at the widest GS
  static constexpr int STAGE = KTILE + NL * LANEB;
  // ring depth: as many stages as fit in ~200 KB, at most 8
  static constexpr int NS = (200 * 1024) / STAGE > 8 ? 8 : (200 * 1024) / STAGE;
  static constexpr size_t SMEM = (size_t)NS * STAGE + 2 * NS * sizeof(uint64_t) + 128;
};

#ifndef MS_MULTI_KHINT
#define MS_MULTI_KHINT 1
#endif
#ifndef MS_MULTI_INTCVT
#define MS_MULTI_INTCVT 0
#endif
// exact binary32 -> binary64 widening on the integer pipes (normal numbers and
// zeros; anything else takes the hardware conversion): moves part of the f2f
// work off the XU pipe, the bound of the binary64-sum lanes
__device__ __forceinline__ double widen(float f) {
#if MS_MULTI_INTCVT
  const uint32_t u = __float_as_uint(f);
  const uint32_t ex = u & 0x7f800000u;
  if (ex == 0u || ex == 0x7f800000u) {
    if ((u << 1) == 0u) return __hiloint2double((int)(u & 0x80000000u), 0);  // signed zero
    return (double)f;
  }
  const uint32_t hi = (u & 0x80000000u) | (((u & 0x7fffffffu) >> 3) + (896u << 20));
  return __hiloint2double((int)hi, (int)(u << 29));
#else
  return (double)f;
#endif
}

__device__ __forceinline__ void tma_tile2d_hint(void* dst, const CUtensorMap* tm, uint64_t* bar, int c0, int c1,
                                                uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma_tile2d(void* dst, const CUtensorMap* tm, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// one K tile of one warp: R rows x VEC columns of this lane, every lane type;
// CHECK = false is the common case (all rows valid, every lane active)
template <int KS, int NS, int NDS, int NDD, bool CHECK>
__device__ __forceinline__ void multi_tile(const unsigned char* sk, int warp, int col, int nr,
                                           const bool (&act)[NS + NDS + NDD],
                                           float (&AS)[NS > 0 ? NS : 1][MultiGeom<KS, NS + NDS + NDD>::R][2],
                                           double (&AD)[NDS + NDD > 0 ? NDS + NDD : 1][MultiGeom<KS, NS + NDS + NDD>::R][2]) {
  using G = MultiGeom<KS, NS + NDS + NDD>;
  constexpr int VEC = G::VEC, TC = G::TC, R = G::R;
  // this lane's K vectors of the warp's rows, then one lane type at a time
  float kf[R][VEC];
#pragma unroll
  for (int k = 0; k < R; ++k) {
    if (!CHECK || k < nr) {
      const uint4 kv = *reinterpret_cast<const uint4*>(
          sk + ((size_t)(warp + kMultiWarps * k) * TC + col) * sizeof(typename G::KT));
      KVec<KS>::unpack(kv, kf[k]);
    }
  }
#pragma unroll
  for (int v = 0; v < NS + NDS; ++v) {
    if (CHECK && !act[v]) continue;
    const float* p = reinterpret_cast<const float*>(sk + G::KTILE + (size_t)v * G::LANEB);
    float s0[VEC], c0[VEC];
#pragma unroll
    for (int e = 0; e < VEC; ++e) {
      s0[e] = p[2 * (col + e)];
      c0[e] = p[2 * (col + e) + 1];
    }
#pragma unroll
    for (int k = 0; k < R; ++k) {
      if (CHECK && k >= nr) continue;
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        const float ps = __fmul_rn(kf[k][e], s0[e]), pc = __fmul_rn(kf[k][e], c0[e]);
        if (v < NS) {
          add2<float>(AS[v][k][0], AS[v][k][1], ps, pc);
        } else {
          AD[v - NS][k][0] = __dadd_rn(AD[v - NS][k][0], (double)ps);
          AD[v - NS][k][1] = __dadd_rn(AD[v - NS][k][1], widen(pc));
        }
      }
    }
  }
#pragma unroll
  for (int v = 0; v < NDD; ++v) {
    if (CHECK && !act[NS + NDS + v]) continue;
    const double* p = reinterpret_cast<const double*>(sk + G::KTILE + (size_t)(NS + NDS + v) * G::LANEB);
    double s0[VEC], c0[VEC];
#pragma unroll
    for (int e = 0; e < VEC; ++e) {
      s0[e] = p[2 * (col + e)];
      c0[e] = p[2 * (col + e) + 1];
    }
#pragma unroll
    for (int k = 0; k < R; ++k) {
      if (CHECK && k >= nr) continue;
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        const double kd = (double)kf[k][e];
        AD[NDS + v][k][0] = __dadd_rn(AD[NDS + v][k][0], __dmul_rn(kd, s0[e]));
        AD[NDS + v][k][1] = __dadd_rn(AD[NDS + v][k][1], __dmul_rn(kd, c0[e]));
      }
    }
  }
}

template <int KS, int NS, int NDS, int NDD>
__global__ void __launch_bounds__(kMultiThreads, 1)
    k_rhs_multi(const __grid_constant__ CUtensorMap tmK, MultiArgs a) {
  msb::count_launch();
  constexpr int NL = NS + NDS + NDD;
  static_assert(NL >= 1 && NL <= kMaxLanes, "lane count");
  using G = MultiGeom<KS, NL>;
  constexpr int VEC = G::VEC, TC = G::TC, R = G::R, TRW = G::TR;
  bool act[NL];
  bool any = false;
#pragma unroll
  for (int v = 0; v < NL; ++v) {
    act[v] = !stage_skip(a.lane[v].ctl, a.l, a.gate);
    any |= act[v];
  }
  if (!any) return;
  if (NL == 1 && a.count_ctl && blockIdx.x == 0 && threadIdx.x == 0) {
    if (a.count == CNT_DDD) a.count_ctl->evals_ddd += 1;
    else if (a.count == CNT_K1) a.count_ctl->evals_k1 += 1;
    else if (a.count == CNT_STAGE) a.count_ctl->evals_stage[a.l] += 1;
  }
  bool all_act = true;
#pragma unroll
  for (int v = 0; v < NL; ++v) all_act &= act[v];
  extern __shared__ __align__(128) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)G::NS * G::STAGE);
  uint64_t* empty = full + G::NS;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ld = (int)a.ld;
  const int T = a.row1 - a.row0;
  const int ngroups = (T + TRW - 1) / TRW;
  const int my_groups = ngroups > (int)blockIdx.x ? (ngroups - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  const int ntiles = (ld + TC - 1) / TC;
  const int Q = my_groups * ntiles;

  if (threadIdx.x == 0) {
    for (int s = 0; s < G::NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kMultiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();

  if (warp == kMultiWarps) {  // producer
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmK)) : "memory");
      const uint64_t kpol = (MS_MULTI_KHINT && a.k_stream) ? l2_evict_first() : l2_evict_normal();
      int st = 0;
      uint32_t ph = 0;  // ring slot and its phase, advanced without divisions
      for (int q = 0; q < Q; ++q) {
        if (q >= G::NS) mbar_wait(&empty[st], ph ^ 1);
        const int g = (int)blockIdx.x + (q / ntiles) * (int)gridDim.x;
        const int t = q % ntiles;
        const int cc = min(TC, ld - t * TC);
        uint32_t bytes = (uint32_t)G::KTILE;
#pragma unroll
        for (int v = 0; v < NL; ++v)
          if (act[v]) bytes += 2u * (uint32_t)cc * (v >= NS + NDS ? 8u : 4u);
        unsigned char* sk = smem + (size_t)st * G::STAGE;
        mbar_expect_tx(&full[st], bytes);
        tma_tile2d_hint(sk, &tmK, &full[st], t * TC, g * TRW, kpol);
#pragma unroll
        for (int v = 0; v < NL; ++v) {
          if (!act[v]) continue;
          const uint32_t es = v >= NS + NDS ? 8u : 4u;
          const unsigned char* gp = reinterpret_cast<const unsigned char*>(a.lane[v].gin);
          unsigned char* dst = sk + G::KTILE + (size_t)v * G::LANEB;
          // the lane's (s_j, c_j) pairs of the tile: one run of the interleaved column data
          bulk_g2s(dst, gp + (size_t)2 * t * TC * es, 2u * (uint32_t)cc * es, &full[st]);
        }
        if (++st == G::NS) {
          st = 0;
          ph ^= 1;
        }
      }
    }
    return;
  }

  bool nonfinite[NL];
#pragma unroll
  for (int v = 0; v < NL; ++v) nonfinite[v] = false;
  int st = 0;
  uint32_t ph = 0;
  const int col = lane * VEC;
  for (int gi = 0; gi < my_groups; ++gi) {
    const int g = (int)blockIdx.x + gi * (int)gridDim.x;
    int rows[R];
    int nr = 0;
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const int rl = warp + kMultiWarps * k;
      const int r = g * TRW + rl;
      rows[k] = r < T ? rl : -1;
      if (r < T) nr = k + 1;
    }
    float AS[NS > 0 ? NS : 1][R][2];
    double AD[NDS + NDD > 0 ? NDS + NDD : 1][R][2];
    const bool fast = all_act && nr == R;
#pragma unroll
    for (int k = 0; k < R; ++k) {
#pragma unroll
      for (int v = 0; v < NS; ++v) AS[v][k][0] = AS[v][k][1] = 0.f;
#pragma unroll
      for (int v = 0; v < NDS + NDD; ++v) AD[v][k][0] = AD[v][k][1] = 0.0;
    }
    for (int t = 0; t < ntiles; ++t) {
      mbar_wait(&full[st], ph);
      const unsigned char* sk = smem + (size_t)st * G::STAGE;
      if (nr > 0 && t * TC + col < ld) {
        if (fast) multi_tile<KS, NS, NDS, NDD, false>(sk, warp, col, nr, act, AS, AD);
        else multi_tile<KS, NS, NDS, NDD, true>(sk, warp, col, nr, act, AS, AD);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
      if (++st == G::NS) {
        st = 0;
        ph ^= 1;
      }
    }
    // the single sweep's shuffle tree per lane, then lane k writes row k
#pragma unroll
    for (int k = 0; k < R; ++k) {
#pragma unroll
      for (int m = 16; m >= 1; m >>= 1) {
#pragma unroll
        for (int v = 0; v < NS; ++v) {
          AS[v][k][0] = __fadd_rn(AS[v][k][0], __shfl_xor_sync(0xffffffffu, AS[v][k][0], m));
          AS[v][k][1] = __fadd_rn(AS[v][k][1], __shfl_xor_sync(0xffffffffu, AS[v][k][1], m));
        }
#pragma unroll
        for (int v = 0; v < NDS + NDD; ++v) {
          AD[v][k][0] = __dadd_rn(AD[v][k][0], __shfl_xor_sync(0xffffffffu, AD[v][k][0], m));
          AD[v][k][1] = __dadd_rn(AD[v][k][1], __shfl_xor_sync(0xffffffffu, AD[v][k][1], m));
        }
      }
    }
#pragma unroll
    for (int k = 0; k < R; ++k) {
      if (lane != k || k >= nr) continue;
      const int r = a.row0 + g * TRW + rows[k];
#pragma unroll
      for (int v = 0; v < NL; ++v) {
        if (!act[v]) continue;
        const LaneArgs& L = a.lane[v];
        double coup;
        if (v < NS) {
          const float si = reinterpret_cast<const float*>(L.gin)[2 * r], ci = reinterpret_cast<const float*>(L.gin)[2 * r + 1];
          const float mwf = __double2float_rn(a.mw);
          coup = (double)__fmul_rn(mwf, __fsub_rn(__fmul_rn(ci, AS[v][k][0]), __fmul_rn(si, AS[v][k][1])));
        } else {
          double si, ci;
          if (v < NS + NDS) {
            si = (double)reinterpret_cast<const float*>(L.gin)[2 * r];
            ci = (double)reinterpret_cast<const float*>(L.gin)[2 * r + 1];
          } else {
            si = reinterpret_cast<const double*>(L.gin)[2 * r];
            ci = reinterpret_cast<const double*>(L.gin)[2 * r + 1];
          }
          const int w = NS > 0 ? (v - NS) : v;
          coup = __dmul_rn(a.mw, __dsub_rn(__dmul_rn(ci, AD[w][k][0]), __dmul_rn(si, AD[w][k][1])));
        }
        const double o = ws_add(L.fvc[r], coup, L.ws32);
        double* out = L.kb[a.out_slot == SLOT_K1 ? L.ctl->k1i : (a.out_slot == SLOT_KLAST ? a.S - L.ctl->k1i : a.out_slot)];
        push_row(a.push, out + r, o);
        nonfinite[v] |= !isfinite(o);
      }
    }
  }
  push_fence(a.push);
#pragma unroll
  for (int v = 0; v < NL; ++v)
    if (act[v] && __any_sync(0xffffffffu, nonfinite[v]) && lane == 0) atomicOr(a.lane[v].nf_mask, 1 << a.l);
}

// host: launch over lanes sorted (f32,f32) | (f64,f32) | (f64,f64); K of the
// system (row range [row0, row1), row stride ld), storage ks
void launch_rhs_multi(const MultiArgs& m, int ns, int nds, int ndd, int ks, const void* K, int sms, cudaStream_t st);

}  // namespace msb
