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

#include <stdexcept>
#include <string>

#include "ms_batch.cuh"

namespace msb {

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
  CUtensorMap tmB;
  int grid_m = 0, grid_n = 0;
  bool ready = false;
};

struct TcArgs {
  BRhsArgs a;
  int n, ncol;  // rows of K, GEMM columns (4B: s_hi, s_lo, c_hi, c_lo per trajectory)
  uint32_t idesc;
};

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// bounded mbarrier wait: a pipeline bug traps (kernel error, process exits)
// instead of hanging the GPU
__device__ __forceinline__ void tc_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  uint64_t t0 = 0;
  for (uint32_t it = 0;; ++it) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (done) return;
    if ((it & 1023) == 0) {
      const uint64_t now = globaltimer_ns();
      if (t0 == 0) t0 = now;
      else if (now - t0 > 2000000000ull) __trap();
    }
  }
}

__device__ __forceinline__ uint64_t umma_smem_desc(uint32_t smem_addr) {
  // K-major, SWIZZLE_128B canonical layout: 8-row x 128-byte atoms,
  // stride between 8-row groups (SBO) 1024 B, LBO unused (1), version 1.
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;                    // LBO (16 B, ignored for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;          // SBO
  d |= (uint64_t)1 << 46;                    // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;                    // layout: SWIZZLE_128B
  return d;
}

__global__ void __launch_bounds__(kTcThreads, MS_TC_MINB)
    k_tc_gemm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, TcArgs t) {
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
    }
    asm volatile("bar.sync 1, %0;" ::"r"(32 * kTcEpiWarps) : "memory");
    tc_wait(tmem_full, 0);
    tc_fence_after();
    const int i = m0 + q4 * 32 + lane;
    const uint32_t lane_addr = tmem + ((uint32_t)(q4 * 32) << 16);
    const float mw = (float)d.mw;
    const float* scf = reinterpret_cast<const float*>(d.sc);
    const int64_t bn = (int64_t)d.B * d.n;
    constexpr int kCols = kTcBN * 4 / kTcEpiWarps;  // columns per epilogue warp
#pragma unroll 1
    for (int c0 = half * kCols; c0 < (half + 1) * kCols; c0 += 32) {
      uint32_t r[32];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
          "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
            "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
            "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
            "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
          : "r"(lane_addr + (uint32_t)c0));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (i >= t.n) continue;
      // 8 trajectories per 32 columns: issue all their loads, then compute
      float sv[8], cv[8];
      double fv[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int tq = (c0 >> 2) + q;
        const int b = tb0 + tq;
        sv[q] = cv[q] = 0.f;
        fv[q] = 0.0;
        if (!tc_skip[tq]) {
          const int64_t e = (int64_t)b * d.n + i;
          sv[q] = scf[e];
          cv[q] = scf[bn + e];
          fv[q] = b_fval(d, e, t.a.fs32);
        }
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int tq = (c0 >> 2) + q;
        if (tc_skip[tq]) continue;
        const float A = __fadd_rn(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]));
        const float Bv = __fadd_rn(__uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3]));
        const float coup = __fmul_rn(mw, __fsub_rn(__fmul_rn(cv[q], A), __fmul_rn(sv[q], Bv)));
        const double o = ws_add(fv[q], (double)coup, t.a.ws32);
        tc_out[tq][i] = o;
        if (!isfinite(o)) atomicOr(&d.ctl[tb0 + tq].nf_mask, 1 << t.a.l);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
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
  }
  g.grid_m = (d.n + kTcBM - 1) / kTcBM;
  g.grid_n = (4 * d.B + kTcBN - 1) / kTcBN;
  cudaError_t e = cudaFuncSetAttribute(k_tc_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTcSmem);
  if (e != cudaSuccess) throw std::runtime_error(std::string("tc gemm smem attribute: ") + cudaGetErrorString(e));
  g.ready = true;
}

inline void tc_gemm_teardown(TcGemm& g) { g.ready = false; }

// instruction descriptor of tcgen05.mma kind::f16: D f32, A/B bf16 (1) or
// f16 (0), both K-major, N = 256, M = 128
inline uint32_t tc_idesc(int ks) {
  const uint32_t ab = ks == MS_K_F16 ? 0u : 1u;
  return (1u << 4) | (ab << 7) | (ab << 10) | ((uint32_t)(kTcBN >> 3) << 17) | ((uint32_t)(kTcBM >> 4) << 24);
}

inline void launch_tc_gemm(const TcGemm& g, const BRhsArgs& a, cudaStream_t st) {
  if (!g.ready) throw std::runtime_error("tensor-core GEMM not set up");
  TcArgs t{};
  t.a = a;
  t.n = a.d.n;
  t.ncol = 4 * a.d.B;
  t.idesc = tc_idesc(a.d.ks);
  dim3 grid(g.grid_m, g.grid_n);
  k_tc_gemm<<<grid, kTcThreads, kTcSmem, st>>>(g.tmA, g.tmB, t);
}

}  // namespace msb
