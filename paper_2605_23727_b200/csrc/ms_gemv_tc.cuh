// ms_gemv_tc.cuh — the split Kuramoto's K sweep for f16 K on the 5th-generation
// tensor cores (MS_SWEEP=tc16).
//
//   A_i = sum_j K_ij s_j,  B_i = sum_j K_ij c_j      (systems.cpp:141-143, split)
//   k_i = (double)(F_i + RN(mw (c_i A_i - s_i B_i)))  (systems.cpp:59-62)
//
// The CUDA-core sweeps spend three instructions per f16 K element (convert,
// packed multiply, packed add) and sustain ~5.5 TB/s in the board's power
// cap; here the products run on the tensor pipe and the SM only moves bytes.
// Operands: A = a 128-row x 64-column tile of K (a 16 KB SWIZZLE_128B image
// kept beside the row-major K, k_tile_k16; one bulk copy each), B = the
// tile's 64 column values as four f16 rows s_hi, s_lo, c_hi, c_lo (hi =
// RN16(v), lo = RN16(v - hi): ~22 bits of the binary32 value; products with
// f16 K are exact; the stage prep writes them as a swizzled image,
// ms_kernels.cuh op16_put) plus 12 zero rows (N = 16, the smallest M128 shape).
//
// Rounding: every MMA (16 columns) starts from a zero accumulator, so the
// tensor core only forms a 16-term dot product; the products' sums are then
// added in binary32 RN on the CUDA cores, in ascending column order:
//   a_hi += dot_hi (k-step by k-step), a_lo += dot_lo, per 2048-column chunk
//   A_chunk = a_hi + a_lo;  A = ((A_0 + A_1) + A_2) + ...
// The order depends only on N (never on the row partition or the grid), so
// sharded handles give the rows of the whole handle bit for bit. It is not the
// CUDA-core sweeps' order: parity with the oracle is by tolerance (counts and
// final state, tests/test_gpu_tc16.py).
//
// Work: units = (128-row tile, 2048-column chunk), split contiguously over one
// CTA per SM. Per CTA:
//   warp 0   producer: bulk copies of the K tile images (evict-first when K is
//            streamed) and of the operand rows
//   warp 1   TMEM allocator + MMA issuer (4 x M128 N16 K16 per k-block, into a
//            ring of 8 TMEM groups)
//   warps 2-5  accumulators: tcgen05.ld of each MMA's 4 useful columns, binary32
//            sums; at a unit's end the chunk sums go to a partial buffer and
//            the CTA that completes a tile's last chunk (ticket) forms the rows'
//            totals in chunk order and writes k.
#pragma once

#include <cuda.h>

#include "ms_kernels.cuh"
#include "ms_tcgen05.cuh"

namespace msb {

constexpr int kGvBM = 128;      // rows per tile (TMEM lanes)
constexpr int kGvBK = 64;       // columns per k-block: one 128-byte SW128 row of f16
constexpr int kGvChunk = 2048;  // columns per unit (fixed: the sums' order depends on N only)
// MS_GV_FINE: one k-block per ring stage (released as soon as its MMAs are
// done), issued four at a time, and 1 KB operand tiles (rows 0-7; the MMA reads
// rows 8-15 from one shared zero atom through the descriptor's stride), which
// fits 13 stages = 208 KB of K in flight instead of 192
#ifndef MS_GV_FINE
#define MS_GV_FINE 0  // measured slower: 5.73 vs 6.43 TB/s (profiles/r2_tc16.txt)
#endif
// K-blocks per pipeline stage: their copies are issued together
#ifndef MS_GV_KB
#define MS_GV_KB (MS_GV_FINE ? 1 : 4)
#endif
constexpr int kGvKB = MS_GV_KB;
#ifndef MS_GV_ISSUE
#define MS_GV_ISSUE 4
#endif
constexpr int kGvIssue = MS_GV_ISSUE;         // MS_GV_FINE: stages issued per producer step
constexpr int kGvABytes = kGvBM * kGvBK * 2;  // 16 KB of K per k-block
// MS_GV_ZATOM: rows 8-15 of every operand tile are one shared zero atom (descriptor stride)
#ifndef MS_GV_ZATOM
#define MS_GV_ZATOM MS_GV_FINE
#endif
// operand tile per k-block: rows 4.. stay zero (MS_GV_ZATOM: rows 8-15 are the zero atom)
constexpr int kGvBBytes = (MS_GV_ZATOM ? 8 : 16) * kGvBK * 2;
constexpr int kGvStageBytes = kGvKB * (kGvABytes + kGvBBytes);
#ifndef MS_GV_STAGES
#define MS_GV_STAGES (MS_GV_FINE ? 13 : 12 / MS_GV_KB)
#endif
constexpr int kGvStages = MS_GV_STAGES;
#ifndef MS_GV_PF
#define MS_GV_PF 0  // stages of K tile images prefetched into L2 ahead of the ring (measured slower: profiles/r2_tc16.txt)
#endif
static_assert(kGvChunk % (kGvKB * kGvBK) == 0, "stages tile the chunk");
#ifndef MS_GV_GROUPS
#define MS_GV_GROUPS 8
#endif
constexpr int kGvGroups = MS_GV_GROUPS;       // TMEM groups (k-blocks between issuer and accumulators)
#ifndef MS_GV_BATCH
#define MS_GV_BATCH 1
#endif
constexpr int kGvBatch = MS_GV_BATCH;         // k-blocks the accumulators read per TMEM round trip
static_assert(kGvBatch <= kGvGroups, "accumulator batch");
// MS_GV_UISSUE: warp-uniform MMA issuer (descriptors and barrier addresses in uniform registers)
#ifndef MS_GV_UISSUE
#define MS_GV_UISSUE 1
#endif
// MS_GV_PRE: the prologue runs before griddepcontrol.wait; MS_GV_COMB: batched loads in the chunk combine
#ifndef MS_GV_PRE
#define MS_GV_PRE 1
#endif
#ifndef MS_GV_COMB
#define MS_GV_COMB 1
#endif
// MS_GV_KBFULL: one full barrier per k-block of a stage (the MMAs of a k-block start when its 16 KB have
// landed, while the rest of the stage is still arriving); the stage is still released as a whole
#ifndef MS_GV_KBFULL
#define MS_GV_KBFULL 0
#endif
// MS_GV_OWN: tiles whose chunks all belong to one CTA skip the partial buffer, the fences and the ticket
#ifndef MS_GV_OWN
#define MS_GV_OWN 0  // measured slower: 6.60 vs 6.91 TB/s per launch (profiles/r2_tc16.txt)
#endif
constexpr int kGvMaxOwn = 32;  // chunks per tile the owner keeps (N <= 65536)
// MS_GV_ATOMREL: the unit-end ticket is one acq_rel atomic after a barrier instead of a fence in every thread
#ifndef MS_GV_ATOMREL
#define MS_GV_ATOMREL 1
#endif
#ifndef MS_GV_EXP
#define MS_GV_EXP 0  // timing experiments only (results wrong): 1 = accumulators skip the TMEM loads
#endif
constexpr int kGvNFull = (MS_GV_KBFULL && !MS_GV_FINE) ? kGvStages * kGvKB : kGvStages;
constexpr int kGvThreads = 6 * 32;
constexpr size_t kGvZeroBytes = MS_GV_ZATOM ? 1024 : 0;  // the shared zero atom (rows 8-15 of every B tile)
constexpr size_t kGvSmem = 1024 + (size_t)kGvStages * kGvStageBytes + kGvZeroBytes + 256;
static_assert(!MS_GV_FINE || (kGvKB == 1 && kGvChunk % (kGvIssue * kGvBK) == 0), "fine ring layout");
constexpr uint32_t kGvTmemCols = kGvGroups * 64;  // kGvGroups x 4 MMAs x 16 columns (power of two)
static_assert(kGvTmemCols == 256 || kGvTmemCols == 512, "TMEM allocation");
static_assert(!MS_GV_KBFULL || MS_GV_UISSUE, "per-k-block full barriers: uniform issuer only");
static_assert((kGvNFull + kGvStages + 2 * kGvGroups) * 8 + 4 <= 256, "barrier block");

// per-handle resources (created with the system, ms_api.cu)
struct GvRes {
  unsigned char* kt;  // K as MMA tile images: [tile][k-block][16 KB, SWIZZLE_128B] (kept beside row-major K)
  float2* part;       // [tiles][chunks][128] chunk sums (A, B)
  int* cnt;           // [tiles] chunk tickets (zero between launches)
  int tiles, chunks, kblocks;
};

struct GvArgs {
  const unsigned char* kt;
  float2* part;
  int* cnt;
  int tiles, chunks, kblocks;
  uint32_t idesc;
};

// Tile images of the handle's f16 K rows: 16-byte piece c of row r of
// (tile, k-block) at r*128 + ((c ^ (r % 8)) * 16) -- the SWIZZLE_128B K-major
// layout the MMA reads, so one contiguous 16 KB bulk copy stages a tile (the
// row-major K's 128-byte row pieces cost DRAM page locality). Rows past the
// handle are zero.
__global__ void __launch_bounds__(256) k_tile_k16(const __half* K, unsigned char* kt, int64_t ld, int rows,
                                                  int tiles, int kblocks) {
  msb::count_launch();
  const int64_t pieces = (int64_t)tiles * kblocks * kGvBM * 8;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < pieces; q += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(q & 7), r = (int)((q >> 3) % kGvBM);
    const int64_t tk = q / (8 * kGvBM);  // tile * kblocks + kblock
    const int tile = (int)(tk / kblocks), kb = (int)(tk % kblocks);
    const int row = tile * kGvBM + r;
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    if (row < rows) v = *reinterpret_cast<const uint4*>(K + (int64_t)row * ld + (int64_t)kb * kGvBK + c * 8);
    *reinterpret_cast<uint4*>(kt + tk * kGvABytes + r * 128 + ((c ^ (r & 7)) << 4)) = v;
  }
}

__device__ __forceinline__ void gv_ld4(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}

__device__ __forceinline__ uint32_t gv_pack(__half lo_col, __half hi_col) {
  return (uint32_t)__half_as_ushort(lo_col) | ((uint32_t)__half_as_ushort(hi_col) << 16);
}

// MS_GV_REV: every CTA walks its units in the opposite order on alternate
// launches (a per-CTA toggle), so a sweep starts with the unit the CTA's previous
// sweep read last -- still in L2 under the evict-first stream. Each unit's sums go
// to their own partial slot, combined in chunk order, so the order is free.
#ifndef MS_GV_REV
#define MS_GV_REV 1
#endif
static __device__ unsigned int g_gv_rev[4096];
// MS_GV_KEEPKB: the last MS_GV_KEEPKB k-blocks of a CTA's stream are read with
// policy MS_GV_KEEPPOL (1 evict-normal, 2 evict-last) instead of evict-first, so
// more of what the next (reversed) sweep reads first survives in L2
#ifndef MS_GV_KEEPKB
#define MS_GV_KEEPKB 0
#endif
#ifndef MS_GV_KEEPPOL
#define MS_GV_KEEPPOL 1
#endif

// unit u -> (tile, chunk); its k-block count
__device__ __forceinline__ int gv_nkb(const RhsArgs& a, int ch) {
  const int cols = min(kGvChunk, (int)a.ld - ch * kGvChunk);
  return (cols + kGvBK - 1) / kGvBK;
}

// NEXT: the CTA that completes a tile also runs the next stage's prep (pn) for
// the tile's rows -- every per-agent input of that prep is row-local (x, the k
// slots including the one just written by the same thread), and its column data
// and operand image go to the other buffers (pn.B.gin / pn.B.op16: this stage's
// are still being read). prep_agent's arithmetic, so bit-identical to k_prep +
// sweep; host side: launch_stage (fuse_next_ok in ms_rhs_fast.cu).
template <int KS, bool NEXT = false>
__global__ void __launch_bounds__(kGvThreads, 1)
    k_rhs_tc16(RhsArgs a, GvArgs g, PrepArgs pn) {
  static_assert(KS == MS_K_F16, "tc16 sweep: f16 K");
  msb::count_launch();
#if !MS_GV_PRE
  pdl_enter();
  if (stage_skip(a.ctl, a.l, a.gate)) return;
  sweep_count(a);
#endif
  extern __shared__ __align__(1024) unsigned char gv_raw[];
  unsigned char* smem =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(gv_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* zero_atom = smem + (size_t)kGvStages * kGvStageBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(zero_atom + kGvZeroBytes);
  uint64_t* empty = full + kGvNFull;
  uint64_t* tfull = empty + kGvStages;
  uint64_t* tempty = tfull + kGvGroups;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + kGvGroups);
  __shared__ int s_last;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int U = g.tiles * g.chunks;
  const int u0 = (int)((int64_t)U * blockIdx.x / gridDim.x);
  const int u1 = (int)((int64_t)U * (blockIdx.x + 1) / gridDim.x);

  __shared__ int s_rev;
  if (threadIdx.x == 0) {
    // one L2 atomic: coherent whatever this SM's L1 holds (the order is free, so a
    // stale toggle could only cost the L2 reuse, never a result)
    s_rev = MS_GV_REV ? (int)(atomicXor(&g_gv_rev[blockIdx.x & 4095], 1u) & 1u) : 0;
    for (int s = 0; s < kGvNFull; ++s) mbar_init(&full[s], 1);
    for (int s = 0; s < kGvStages; ++s) mbar_init(&empty[s], 1);
    for (int q = 0; q < kGvGroups; ++q) {
      mbar_init(&tfull[q], 1);
      mbar_init(&tempty[q], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // rows 4.. of every operand tile (and the zero atom) are zero for the whole kernel
  constexpr int kZeroRowBytes = kGvBBytes - 4 * 128;
  for (int idx = threadIdx.x; idx < kGvStages * kGvKB * (kZeroRowBytes / 16); idx += blockDim.x) {
    const int t = idx / (kZeroRowBytes / 16), o = idx % (kZeroRowBytes / 16);
    *reinterpret_cast<uint4*>(smem + (size_t)(t / kGvKB) * kGvStageBytes + kGvKB * kGvABytes +
                              (t % kGvKB) * kGvBBytes + 4 * 128 + o * 16) = make_uint4(0u, 0u, 0u, 0u);
  }
  for (int o = threadIdx.x; o < (int)(kGvZeroBytes / 16); o += blockDim.x)
    reinterpret_cast<uint4*>(zero_atom)[o] = make_uint4(0u, 0u, 0u, 0u);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                 "n"(kGvTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
#if MS_GV_PRE
  // the prologue above (barriers, zero rows, TMEM) touches nothing the previous
  // kernel writes, so under programmatic dependent launch it overlaps that
  // kernel's tail; everything below reads its results
  pdl_enter();
  if (stage_skip(a.ctl, a.l, a.gate)) {
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kGvTmemCols));
    return;
  }
  sweep_count(a);
#endif
  bool nonfinite = false, nfp = false;
  const int rev = s_rev;
  // the CTA's k-th unit this launch
  auto unit = [&](int uu) { return rev ? u1 - 1 - (uu - u0) : uu; };

  if (warp == 0) {
    // producer: bulk copies of the K tile images and of the operand rows 0-3
    const uint64_t pol = a.k_stream ? l2_evict_first() : l2_evict_normal();
    const unsigned char* op = static_cast<const unsigned char*>(a.op16);
    int sg = 0;  // stage counter
    // L2 prefetch MS_GV_PF stages ahead: the DRAM reads of the tile images are in
    // flight beyond the shared-memory ring, whose refills then come from L2
    int pu = u0, pkb = 0;
    auto prefetch_next = [&]() {
      if (pu >= u1) return;
      const int ptile = pu / g.chunks, pch = pu % g.chunks;
      const unsigned char* src = g.kt + ((int64_t)ptile * g.kblocks + pch * (kGvChunk / kGvBK) + pkb) * kGvABytes;
      asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(src),
                   "r"((uint32_t)(kGvKB * kGvABytes)), "l"(pol)
                   : "memory");
      pkb += kGvKB;
      if (pkb >= gv_nkb(a, pch)) { pkb = 0; ++pu; }
    };
    if (lane == 0)
      for (int p = 0; p < MS_GV_PF; ++p) prefetch_next();
#if MS_GV_FINE
    // lane j fills stage sg + j (its own empty wait), kGvIssue stages per step
    for (int uu = u0; uu < u1; ++uu) {
      const int u = unit(uu);
      const int tile = u / g.chunks, ch = u % g.chunks;
      const int nkb = gv_nkb(a, ch);
      for (int kb = 0; kb < nkb; kb += kGvIssue) {
        const int nb = min(kGvIssue, nkb - kb);
        if (lane < nb) {
          const int s_ = sg + lane, st = s_ % kGvStages;
          if (s_ >= kGvStages) tc_wait(&empty[st], ((s_ / kGvStages) & 1) ^ 1);
          unsigned char* sa = smem + (size_t)st * kGvStageBytes;
          const int kbi = ch * (kGvChunk / kGvBK) + kb + lane;  // k-block of the row
          MS_CHECK(tile < g.tiles && kbi < g.kblocks, "tc16 sweep: tile image outside the handle's K");
          mbar_expect_tx(&full[st], kGvABytes + 512);
          bulk_g2s_hint(sa, g.kt + ((int64_t)tile * g.kblocks + kbi) * kGvABytes, kGvABytes, &full[st], pol);
          bulk_g2s(sa + kGvABytes, op + (size_t)kbi * 512, 512, &full[st]);
        }
        __syncwarp();
        sg += nb;
      }
    }
#else
    for (int uu = u0; uu < u1; ++uu) {
      const int u = unit(uu);
      const int tile = u / g.chunks, ch = u % g.chunks;
      const int nkb = gv_nkb(a, ch);
      for (int kb = 0; kb < nkb; kb += kGvKB, ++sg) {
        const int st = sg % kGvStages;
        if (lane == 0 && MS_GV_PF > 0) prefetch_next();
        if (sg >= kGvStages) {
          if (lane == 0) tc_wait(&empty[st], ((sg / kGvStages) & 1) ^ 1);
          __syncwarp();
        }
        unsigned char* sa = smem + (size_t)st * kGvStageBytes;
        unsigned char* sb = sa + kGvKB * kGvABytes;
        const int c0 = ch * kGvChunk + kb * kGvBK;
#if MS_GV_KBFULL
        if (lane < kGvKB) mbar_expect_tx(&full[st * kGvKB + lane], kGvABytes + 512);
#else
        if (lane == 0) mbar_expect_tx(&full[st], kGvKB * (kGvABytes + 512));
#endif
        __syncwarp();
        MS_CHECK(tile < g.tiles && (c0 / kGvBK) + kGvKB <= g.kblocks && (c0 % kGvBK) == 0,
                 "tc16 sweep: tile image outside the handle's K");
        uint64_t upol = pol;
        if (MS_GV_KEEPKB > 0 && a.k_stream && uu == u1 - 1 && kb + kGvKB > nkb - MS_GV_KEEPKB)
          upol = MS_GV_KEEPPOL == 2 ? l2_evict_last() : l2_evict_normal();
        uint64_t* fb = MS_GV_KBFULL ? &full[st * kGvKB + (lane % kGvKB)] : &full[st];
        if (lane < kGvKB)  // one contiguous 16 KB tile image per k-block
          bulk_g2s_hint(sa + lane * kGvABytes,
                        g.kt + ((int64_t)tile * g.kblocks + (c0 / kGvBK) + lane) * kGvABytes, kGvABytes, fb, upol);
        else if (lane < 2 * kGvKB)  // and the operand rows 0-3 of its B tile (the prep's image)
          bulk_g2s(sb + (lane - kGvKB) * kGvBBytes, op + (size_t)((c0 / kGvBK) + lane - kGvKB) * 512, 512, fb);
      }
    }
#endif
  } else if (warp == 1) {
#if MS_GV_UISSUE
    // MMA issuer, warp-uniform: the whole warp walks the loops and waits (every
    // address, descriptor and counter stays in uniform registers); one elected
    // lane issues the tcgen05 instructions. Descriptors are a per-stage base
    // plus a 16-byte-unit offset (no carry: the ring lies below 256 KB).
    {
      const uint32_t tmem_u = __shfl_sync(0xffffffffu, tmem, 0);
      const uint32_t idesc = g.idesc;
      int kbg = 0, sg = 0;
      for (int uu = u0; uu < u1; ++uu) {
        const int u = unit(uu);
        const int nkb = gv_nkb(a, u % g.chunks);
        for (int kb = 0; kb < nkb; kb += kGvKB, ++sg) {
          const int st = sg % kGvStages;
          if (!(MS_GV_KBFULL && !MS_GV_FINE)) tc_wait(&full[st], (sg / kGvStages) & 1);
          const uint32_t sa = smem_u32(smem + (size_t)st * kGvStageBytes);
          const uint32_t sb = sa + kGvKB * kGvABytes;
          const uint64_t adesc0 = umma_smem_desc(sa);
#if MS_GV_ZATOM
          const uint32_t zat = smem_u32(zero_atom);
#else
          const uint64_t bdesc0 = umma_smem_desc(sb);
#endif
#pragma unroll
          for (int j = 0; j < kGvKB; ++j, ++kbg) {
            const int grp = kbg % kGvGroups;
            if (MS_GV_KBFULL && !MS_GV_FINE) tc_wait(&full[st * kGvKB + j], (sg / kGvStages) & 1);
            if (kbg >= kGvGroups) tc_wait(&tempty[grp], ((kbg / kGvGroups) & 1) ^ 1);
            tc_fence_after();
            if (elect_one()) {
#pragma unroll
              for (int k = 0; k < kGvBK / 16; ++k) {
                const uint64_t adesc = adesc0 + (uint64_t)((j * kGvABytes + k * 32) >> 4);
#if MS_GV_ZATOM
                const uint64_t bdesc =
                    umma_smem_desc_sbo(sb + j * kGvBBytes + k * 32, zat - (sb + j * kGvBBytes));
#else
                const uint64_t bdesc = bdesc0 + (uint64_t)((j * kGvBBytes + k * 32) >> 4);
#endif
                asm volatile(
                    "{\n .reg .pred p;\n setp.ne.b32 p, 0, 0;\n"
                    " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(
                        tmem_u + (uint32_t)(grp * 64 + k * 16)),
                    "l"(adesc), "l"(bdesc), "r"(idesc));
              }
              asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                               smem_u32(&tfull[grp]))
                           : "memory");
              if (j == kGvKB - 1)
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                 smem_u32(&empty[st]))
                             : "memory");
            }
            __syncwarp();
          }
        }
      }
    }
#else
    if (lane == 0) {  // MMA issuer
      int kbg = 0, sg = 0;
      for (int uu = u0; uu < u1; ++uu) {
      const int u = unit(uu);
        const int nkb = gv_nkb(a, u % g.chunks);
        for (int kb = 0; kb < nkb; kb += kGvKB, ++sg) {
          const int st = sg % kGvStages;
          tc_wait(&full[st], (sg / kGvStages) & 1);
          const uint32_t sa = smem_u32(smem + (size_t)st * kGvStageBytes);
          const uint32_t sb = sa + kGvKB * kGvABytes;
#pragma unroll 1
          for (int j = 0; j < kGvKB; ++j, ++kbg) {
            const int grp = kbg % kGvGroups;
            if (kbg >= kGvGroups) tc_wait(&tempty[grp], ((kbg / kGvGroups) & 1) ^ 1);
            tc_fence_after();
#pragma unroll
            for (int k = 0; k < kGvBK / 16; ++k) {
              const uint64_t adesc = umma_smem_desc(sa + j * kGvABytes + k * 32);
#if MS_GV_ZATOM
              // rows 8-15 of the B tile: the zero atom (descriptor stride = its distance)
              const uint64_t bdesc = umma_smem_desc_sbo(sb + j * kGvBBytes + k * 32,
                                                        smem_u32(zero_atom) - (sb + j * kGvBBytes));
#else
              const uint64_t bdesc = umma_smem_desc(sb + j * kGvBBytes + k * 32);
#endif
              asm volatile(
                  "{\n .reg .pred p;\n setp.ne.b32 p, 0, 0;\n"
                  " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(
                      tmem + (uint32_t)(grp * 64 + k * 16)),
                  "l"(adesc), "l"(bdesc), "r"(g.idesc));
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                             smem_u32(&tfull[grp]))
                         : "memory");
          }
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                           smem_u32(&empty[st]))
                       : "memory");
        }
      }
    }
#endif
  } else {
    // accumulators: warp%4 = TMEM lane quarter; row rr of the tile
    const int q4 = warp & 3;
    const int rr = q4 * 32 + lane;
    const uint32_t lane_base = tmem + ((uint32_t)(q4 * 32) << 16);
    const float* gin = reinterpret_cast<const float*>(a.gin);
    const float mw = (float)a.mw;
    double* out = a.kb[a.out_slot == SLOT_K1 ? a.ctl->k1i : (a.out_slot == SLOT_KLAST ? a.S - a.ctl->k1i : a.out_slot)];
    int kbg = 0, own_done = 0;
    float2 cs[kGvMaxOwn];  // chunk sums of a tile this CTA owns entirely (MS_GV_OWN)
    PrepCtx pc{};
    if constexpr (NEXT) pc = prep_ctx(pn);
    for (int uu = u0; uu < u1; ++uu) {
      const int u = unit(uu);
      const int tile = u / g.chunks, ch = u % g.chunks;
      const int nkb = gv_nkb(a, ch);
      float ah = 0.f, al = 0.f, bh = 0.f, bl = 0.f;
      // batches of up to kGvBatch k-blocks: one TMEM round trip per batch
      for (int kb = 0; kb < nkb; kb += kGvBatch) {
        const int nb = min(kGvBatch, nkb - kb);
#pragma unroll
        for (int j = 0; j < kGvBatch; ++j)
          if (j < nb) tc_wait(&tfull[(kbg + j) % kGvGroups], ((kbg + j) / kGvGroups) & 1);
        tc_fence_after();
        uint32_t r[kGvBatch][4][4];
#if MS_GV_EXP != 1
#pragma unroll
        for (int j = 0; j < kGvBatch; ++j)
          if (j < nb) {
#pragma unroll
            for (int k = 0; k < 4; ++k) gv_ld4(lane_base + (uint32_t)(((kbg + j) % kGvGroups) * 64 + k * 16), r[j][k]);
          }
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#else
#pragma unroll
        for (int j = 0; j < kGvBatch; ++j)
#pragma unroll
          for (int k = 0; k < 4; ++k) r[j][k][0] = r[j][k][1] = r[j][k][2] = r[j][k][3] = 0u;
#endif
        tc_fence_before();
        __syncwarp();
        if (lane == 0)
          for (int j = 0; j < nb; ++j) mbar_arrive(&tempty[(kbg + j) % kGvGroups]);
#pragma unroll
        for (int j = 0; j < kGvBatch; ++j)
          if (j < nb) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              ah = __fadd_rn(ah, __uint_as_float(r[j][k][0]));
              al = __fadd_rn(al, __uint_as_float(r[j][k][1]));
              bh = __fadd_rn(bh, __uint_as_float(r[j][k][2]));
              bl = __fadd_rn(bl, __uint_as_float(r[j][k][3]));
            }
          }
        kbg += nb;
      }
      MS_CHECK(tile < g.tiles && ch < g.chunks, "tc16 sweep: partial outside the workspace");
      float2* pt = g.part + ((int64_t)tile * g.chunks) * kGvBM;
      const float2 usum = make_float2(__fadd_rn(ah, al), __fadd_rn(bh, bl));
      // A tile whose chunks all lie in this CTA's unit range needs no partial buffer,
      // fence or ticket: its chunk sums wait in the thread's own (local-memory) array and
      // are combined in the same ascending chunk order when its last unit is done (the
      // walk is contiguous, so the tile's units follow one another). Same bits either way.
      const bool owned = MS_GV_OWN && g.chunks <= kGvMaxOwn && tile * g.chunks >= u0 && (tile + 1) * g.chunks <= u1;
      bool finish;
      if (owned) {
        cs[ch] = usum;
        finish = ++own_done == g.chunks;
        if (finish) own_done = 0;
      } else {
        pt[(int64_t)ch * kGvBM + rr] = usum;
#if MS_GV_ATOMREL
        // the barrier orders the 128 partial stores before thread (warp 2, lane 0), whose
        // acq_rel ticket publishes them (release) and, for the CTA that takes the last
        // ticket, orders the other CTAs' partials before its reads (acquire; the readers
        // follow through the second barrier and read at L2): one fenced atomic per unit
        // instead of a MEMBAR.ALL.GPU + CCTL.IVALL in every accumulator thread
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (warp == 2 && lane == 0) {
          int tk;
          asm volatile("atom.add.acq_rel.gpu.global.s32 %0, [%1], 1;" : "=r"(tk) : "l"(g.cnt + tile) : "memory");
          s_last = tk == g.chunks - 1 ? 1 : 0;
        }
#else
        __threadfence();
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (warp == 2 && lane == 0) s_last = (atomicAdd(g.cnt + tile, 1) == g.chunks - 1) ? 1 : 0;
#endif
        asm volatile("bar.sync 1, 128;" ::: "memory");
        finish = s_last != 0;
        if (finish) __threadfence();
      }
      if (finish) {
        const int row = a.row0 + tile * kGvBM + rr;
        if (row < a.row1) {
          float A, B;
          if (owned) {
            A = cs[0].x;
            B = cs[0].y;
            for (int c = 1; c < g.chunks; ++c) {
              A = __fadd_rn(A, cs[c].x);
              B = __fadd_rn(B, cs[c].y);
            }
          } else {
            float2 p = __ldcg(pt + rr);
            A = p.x;
            B = p.y;
#if MS_GV_COMB
            // the chunk sums in batches of 8 independent loads, added in chunk order
            for (int c0 = 1; c0 < g.chunks; c0 += 8) {
              float2 q[8];
#pragma unroll
              for (int e = 0; e < 8; ++e)
                q[e] = c0 + e < g.chunks ? __ldcg(pt + (int64_t)(c0 + e) * kGvBM + rr) : make_float2(0.f, 0.f);
#pragma unroll
              for (int e = 0; e < 8; ++e)
                if (c0 + e < g.chunks) {
                  A = __fadd_rn(A, q[e].x);
                  B = __fadd_rn(B, q[e].y);
                }
            }
#else
            for (int c = 1; c < g.chunks; ++c) {
              p = __ldcg(pt + (int64_t)c * kGvBM + rr);
              A = __fadd_rn(A, p.x);
              B = __fadd_rn(B, p.y);
            }
#endif
          }
          const float si = gin[2 * row], ci = gin[2 * row + 1];
          const float coup = __fmul_rn(mw, __fsub_rn(__fmul_rn(ci, A), __fmul_rn(si, B)));
          MS_CHECK(row >= a.row0 && row < a.row1, "tc16 sweep: output row outside the handle");
          const double o = ws_add(a.fvc[row], (double)coup, a.ws32);
          push_row(a.push, out + (int64_t)row * a.d + a.cs, o);
          nonfinite |= !isfinite(o);
          if constexpr (NEXT) nfp |= prep_agent<MD_KUR, float, float>(pn, pc, row);
        }
        if (!owned && warp == 2 && lane == 0) g.cnt[tile] = 0;  // ready for the next launch
      }
      if (!owned) asm volatile("bar.sync 1, 128;" ::: "memory");
    }
  }
  if (warp >= 2) push_fence(a.push);
  if (warp >= 2 && __any_sync(0xffffffffu, nonfinite) && lane == 0) atomicOr(a.nf_mask, 1 << a.l);
  if constexpr (NEXT) {
    if (warp >= 2 && __any_sync(0xffffffffu, nfp) && lane == 0) atomicOr(a.nf_mask, 1 << pn.l);
    if (blockIdx.x == 0 && warp >= 2) {  // the padding columns of the target buffer (k_prep does the same)
      float* gp = reinterpret_cast<float*>(pn.B.gin);
      for (int j = pn.md.n + (int)threadIdx.x - 64; j < pn.ld; j += 128) {
        gp[2 * j] = 0.f;
        gp[2 * j + 1] = 0.f;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kGvTmemCols));
  }
}

// instruction descriptor: D f32, A/B f16, both K-major, N = 16, M = 128
constexpr uint32_t kGvIdesc = (1u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(16 >> 3) << 17) |
                              ((uint32_t)(128 >> 4) << 24);

}  // namespace msb
