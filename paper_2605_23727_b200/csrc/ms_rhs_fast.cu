// ms_rhs_fast.cu — instantiation and launch of k_rhs_fast for every
// (model, SS, GS, K storage) combination a policy row can ask for.
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>

#include <cudaTypedefs.h>

#include "ms_dispatch.h"
#include "ms_gemv_tc.cuh"
#include "ms_multi.cuh"

namespace msb {

namespace {

// K sweep selection for the split Kuramoto: MS_SWEEP=ldg keeps the
// register-fed sweep, MS_SWEEP=tile the 2D-tensor-tiled one-lane k_rhs_multi;
// by default f32 K takes the row-copy TMA sweep and 16-bit K the tile sweep
bool use_tma_sweep_env() {
  const char* v = std::getenv("MS_SWEEP");
  return !(v && std::strcmp(v, "ldg") == 0);
}
// 16-bit K through the row-copy TMA sweep (MS_SWEEP=tma16; tuning)
bool use_tma16_env() {
  const char* v = std::getenv("MS_SWEEP");
  return v && std::strcmp(v, "tma16") == 0;
}
// 16-bit K at moderate N defaults to the 2D-tile sweep (C2, N = 4096: 53 vs
// 59-64 us per attempt); at C4 (N = 32768) the register sweep stays ahead
// (bench: 726 vs 698 steps/s). f32 K keeps the row-copy TMA sweep.
bool use_tile_sweep(int ks, int64_t ld) {
  const char* v = std::getenv("MS_SWEEP");
  if (v && std::strcmp(v, "tile") == 0) return true;
  if (v && (std::strcmp(v, "ldg") == 0 || std::strcmp(v, "small") == 0)) return false;
  return (ks == MS_K_F16 || ks == MS_K_BF16) && ld <= 8192;
}

// f16 K through the tensor-core sweep (ms_gemv_tc.cuh): the default for
// binary32 rows once K outgrows L2 (N >= 16384; C4: 806 vs 726 accepted
// steps/s, profiles/r2_tc16.txt), MS_SWEEP=tc16 forces it at any N, any other
// MS_SWEEP value selects a CUDA-core sweep
bool use_tc16(const RhsArgs& a, int ks) {
  if (!(ks == MS_K_F16 && a.tc16 != nullptr && a.op16 != nullptr && a.ld % (kGvKB * kGvBK) == 0)) return false;
  const char* v = std::getenv("MS_SWEEP");
  if (v && *v) return std::strcmp(v, "tc16") == 0;
  return a.ld >= 16384;
}

template <bool NEXT>
void go_tc16(const RhsLaunch& L, const RhsArgs& a, const PrepArgs& pn = PrepArgs{}) {
  const GvRes* r = static_cast<const GvRes*>(a.tc16);
  auto kern = k_rhs_tc16<MS_K_F16, NEXT>;
  static bool attr_done = false;
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kGvSmem);
    if (e != cudaSuccess) throw std::runtime_error(std::string("rhs_tc16 attribute: ") + cudaGetErrorString(e));
    attr_done = true;
  }
  GvArgs g{r->kt, r->part, r->cnt, r->tiles, r->chunks, r->kblocks, kGvIdesc};
  const int units = r->tiles * r->chunks;
  static const int cap = [] {  // MS_GV_GRID: CTAs (tuning; default one per SM)
    const char* v = std::getenv("MS_GV_GRID");
    return v ? std::atoi(v) : 0;
  }();
  const int slots = cap > 0 && cap < L.num_sms ? cap : L.num_sms;
  const int grid = units < slots ? units : slots;
  cudaError_t e = launch_k(kern, grid, kGvThreads, kGvSmem, L.stream, a, g, pn);
  if (e != cudaSuccess) throw std::runtime_error(std::string("rhs_tc16 launch: ") + cudaGetErrorString(e));
}

template <class SS, class GS, int KS>
void go_tile(const RhsLaunch& L, const RhsArgs& a) {
  MultiArgs m{};
  m.nl = 1;
  m.l = a.l;
  m.gate = a.gate;
  m.S = a.S;
  m.out_slot = a.out_slot;
  m.ld = a.ld;
  m.n = a.n;
  m.row0 = a.row0;
  m.row1 = a.row1;
  m.mw = a.mw;
  m.count_ctl = a.count_ctl;
  m.count = a.count;
  m.k_stream = a.k_stream;
  m.push = a.push;
  LaneArgs& ln = m.lane[0];
  ln.ctl = a.ctl;
  ln.nf_mask = a.nf_mask;
  ln.gin = a.gin;
  ln.fvc = a.fvc;
  for (int i = 0; i < kMaxStages + 1; ++i) ln.kb[i] = a.kb[i];
  ln.ws32 = a.ws32;
  const bool ss64 = sizeof(SS) == 8, gs64 = sizeof(GS) == 8;
  launch_rhs_multi(m, !ss64 ? 1 : 0, ss64 && !gs64 ? 1 : 0, ss64 && gs64 ? 1 : 0, KS, a.K, L.num_sms, L.stream);
}

template <class SS, class GS, int KS, bool NEXT = false>
void go_tma(const RhsLaunch& L, const RhsArgs& a, const PrepArgs& pn = PrepArgs{}) {
  auto kern = k_rhs_tma<SS, GS, KS, NEXT>;
  using G = TmaGeom<SS, GS, KS>;
  constexpr size_t smem = G::SMEM;
  static bool attr_done = false;
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) throw std::runtime_error(std::string("rhs_tma attribute: ") + cudaGetErrorString(e));
    attr_done = true;
  }
  const int rows = a.row1 - a.row0;
  static const int cap = [] {  // MS_TMA_GRID: CTAs (tuning; default one per SM)
    const char* v = std::getenv("MS_TMA_GRID");
    return v ? std::atoi(v) : 0;
  }();
  const int slots = cap > 0 && cap < L.num_sms * MS_TMA_MINB ? cap : L.num_sms * MS_TMA_MINB;
  const int grid = rows < slots ? rows : slots;
  cudaError_t e = launch_k(kern, grid, G::THREADS, smem, L.stream, a, pn);
  if (e != cudaSuccess) throw std::runtime_error(std::string("rhs_tma launch: ") + cudaGetErrorString(e));
}

template <int MODEL, bool SPLIT, class SS, class GS, int KS>
void go(const RhsLaunch& L, const RhsArgs& a) {
  // the TMA-fed sweep wins for f32 K (7.2 vs 6.5 TB/s); with 16-bit K its
  // row copies get small and the s/c traffic per K byte doubles, and the
  // register-fed sweep stays ahead (profiles/r1_tune_tma.txt)
  if constexpr (MODEL == MD_KUR && SPLIT && KS == MS_K_F16 && sizeof(SS) == 4 && sizeof(GS) == 4) {
    if (use_tc16(a, KS)) {
      if (L.next && L.tc16 && fuse_next_ok(L, L.next_fs32, L.next_gs32)) {
        go_tc16<true>(L, a, *L.next);
        if (L.fused) *L.fused = true;
        return;
      }
      go_tc16<false>(L, a);
      return;
    }
  }
  if constexpr (MODEL == MD_KUR && SPLIT && KS != MS_K_SCALAR && !(sizeof(SS) == 4 && sizeof(GS) == 8)) {
    if (use_tile_sweep(KS, a.ld)) {
      go_tile<SS, GS, KS>(L, a);
      return;
    }
  }
  if constexpr (MODEL == MD_KUR && SPLIT && KS == MS_K_F32) {
    if (use_tma_sweep_env()) {
      if (L.next && fuse_next_ok(L, L.next_fs32, L.next_gs32)) {
        go_tma<SS, GS, KS, true>(L, a, *L.next);
        if (L.fused) *L.fused = true;
        return;
      }
      go_tma<SS, GS, KS>(L, a);
      return;
    }
  }
  if constexpr (MODEL == MD_KUR && SPLIT && (KS == MS_K_F16 || KS == MS_K_BF16)) {
    if (use_tma16_env()) {
      go_tma<SS, GS, KS>(L, a);
      return;
    }
  }
  auto kern = k_rhs_fast<MODEL, SPLIT, SS, GS, KS>;
  constexpr size_t smem = fast_smem_bytes<GS, SPLIT>();
  static bool attr_done = false;
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) throw std::runtime_error(std::string("rhs_fast attribute: ") + cudaGetErrorString(e));
    attr_done = true;
  }
  const int rows = a.row1 - a.row0;
  const int slots = L.num_sms * kFastMinBlocks;
  const int grid = rows < slots ? rows : slots;
  cudaError_t e = launch_k(kern, grid, kFastThreads, smem, L.stream, a);
  if (e != cudaSuccess) throw std::runtime_error(std::string("rhs_fast launch: ") + cudaGetErrorString(e));
}

template <int MODEL, bool SPLIT, class SS, class GS>
void by_k(const RhsLaunch& L, const RhsArgs& a) {
  switch (L.ks) {
    case MS_K_SCALAR: go<MODEL, SPLIT, SS, GS, MS_K_SCALAR>(L, a); break;
    case MS_K_F32: go<MODEL, SPLIT, SS, GS, MS_K_F32>(L, a); break;
    case MS_K_F16: go<MODEL, SPLIT, SS, GS, MS_K_F16>(L, a); break;
    case MS_K_BF16: go<MODEL, SPLIT, SS, GS, MS_K_BF16>(L, a); break;
    default: throw std::invalid_argument("rhs_fast: bad K storage");
  }
}

template <int MODEL, bool SPLIT>
void by_prec(const RhsLaunch& L, const RhsArgs& a) {
  if (L.ss32) {
    if (L.gs32) by_k<MODEL, SPLIT, float, float>(L, a);
    else by_k<MODEL, SPLIT, float, double>(L, a);
  } else {
    if (L.gs32) by_k<MODEL, SPLIT, double, float>(L, a);
    else by_k<MODEL, SPLIT, double, double>(L, a);
  }
}

}  // namespace

namespace {

template <int MODEL, bool SPLIT, class FS, class SS, class GS, int KS, bool PREPPED = false>
void go_fused(const RhsLaunch& L, const PrepArgs& p, const RhsArgs& a, size_t smem) {
  auto kern = k_eval_fused<MODEL, SPLIT, FS, SS, GS, KS, PREPPED>;
  static bool attr_done = false;
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFusedMaxSmem);
    if (e != cudaSuccess) throw std::runtime_error(std::string("eval_fused attribute: ") + cudaGetErrorString(e));
    attr_done = true;
  }
  const int rows = a.row1 - a.row0;
  const int slots = L.num_sms * kFastMinBlocks;
  const int grid = rows < slots ? rows : slots;
  cudaError_t e = launch_k(kern, grid, kFastThreads, smem, L.stream, p, a);
  if (e != cudaSuccess) throw std::runtime_error(std::string("eval_fused launch: ") + cudaGetErrorString(e));
}

template <int MODEL, bool SPLIT, class FS, class SS, class GS>
void fused_by_k(const RhsLaunch& L, const PrepArgs& p, const RhsArgs& a, size_t smem) {
  switch (L.ks) {
    case MS_K_SCALAR: go_fused<MODEL, SPLIT, FS, SS, GS, MS_K_SCALAR>(L, p, a, smem); break;
    case MS_K_F32: go_fused<MODEL, SPLIT, FS, SS, GS, MS_K_F32>(L, p, a, smem); break;
    case MS_K_F16: go_fused<MODEL, SPLIT, FS, SS, GS, MS_K_F16>(L, p, a, smem); break;
    default: go_fused<MODEL, SPLIT, FS, SS, GS, MS_K_BF16>(L, p, a, smem); break;
  }
}

template <int MODEL, bool SPLIT>
bool fused_by_prec(const RhsLaunch& L, const PrepArgs& p, const RhsArgs& a, bool fs32) {
  const size_t ncol = SPLIT ? 2 : 1;
  if (fs32 && L.ss32 && L.gs32) {
    const size_t smem = ncol * (size_t)a.ld * 4;
    if (smem > kFusedMaxSmem) return false;
    fused_by_k<MODEL, SPLIT, float, float, float>(L, p, a, smem);
  } else if (!fs32 && !L.ss32 && L.gs32) {
    const size_t smem = ncol * (size_t)a.ld * 4;
    if (smem > kFusedMaxSmem) return false;
    fused_by_k<MODEL, SPLIT, double, double, float>(L, p, a, smem);
  } else if (!fs32 && !L.ss32 && !L.gs32) {
    const size_t smem = ncol * (size_t)a.ld * 8;
    if (smem > kFusedMaxSmem) return false;
    fused_by_k<MODEL, SPLIT, double, double, double>(L, p, a, smem);
  } else {
    return false;
  }
  return true;
}

// the split Kuramoto's small sweep over prepped column values (any FS: the
// prep already ran)
template <class SS, class GS>
bool small_split(const RhsLaunch& L, const PrepArgs& p, const RhsArgs& a) {
  const size_t smem = 2 * (size_t)a.ld * sizeof(GS);
  if (smem > kFusedMaxSmem) return false;
  switch (L.ks) {
    case MS_K_F32: go_fused<MD_KUR, true, SS, SS, GS, MS_K_F32, true>(L, p, a, smem); return true;
    case MS_K_F16: go_fused<MD_KUR, true, SS, SS, GS, MS_K_F16, true>(L, p, a, smem); return true;
    case MS_K_BF16: go_fused<MD_KUR, true, SS, SS, GS, MS_K_BF16, true>(L, p, a, smem); return true;
    default: return false;
  }
}

}  // namespace

bool launch_sweep_small(const RhsLaunch& L, const PrepArgs& p, const RhsArgs& a) {
  // measured slower than prep + k_rhs_tma / k_rhs_fast at C2 (73.7 vs 54 us per
  // attempt: the split's rows want the pipelined sweeps), so opt-in only
  const char* v = std::getenv("MS_SWEEP");
  if (!(v && std::strcmp(v, "small") == 0) || L.model != MD_KUR || !L.split) return false;
  if (L.ss32) return L.gs32 ? small_split<float, float>(L, p, a) : small_split<float, double>(L, p, a);
  return L.gs32 ? small_split<double, float>(L, p, a) : small_split<double, double>(L, p, a);
}

bool launch_eval_fused(const RhsLaunch& L, const PrepArgs& p, const RhsArgs& a, bool fs32) {
  const char* env = std::getenv("MS_FUSE");
  if (env && std::strcmp(env, "off") == 0) return false;
  switch (L.model) {
    case MD_LCO: return fused_by_prec<MD_LCO, false>(L, p, a, fs32);
    // the split Kuramoto would recompute N sin/cos pairs in every CTA: measured
    // 2x slower than prep + TMA sweep at C2 (N = 4096), so it keeps two launches
    case MD_KUR: return false;
    case MD_CC: return fused_by_prec<MD_CC, false>(L, p, a, fs32);
    default: return false;
  }
}

bool tc16_selected(const RhsArgs& a, int ks) { return use_tc16(a, ks); }

bool fuse_next_ok(const RhsLaunch& L, bool next_fs32, bool next_gs32) {
  const char* f = std::getenv("MS_FUSE_NEXT");  // read per launch (graphs capture it once)
  const bool on = !(f && std::strcmp(f, "off") == 0);
  const char* v = std::getenv("MS_SWEEP");
  const bool tma = !(v && (std::strcmp(v, "ldg") == 0 || std::strcmp(v, "tile") == 0 || std::strcmp(v, "small") == 0));
  // the kernel runs prep_agent<KUR, FS = SS, GS>: the next row's F must be this row's sum format
  const bool f32_tma = tma && L.ks == MS_K_F32;
  const bool f16_tc = L.tc16 && L.ks == MS_K_F16 && L.ss32 && L.gs32;  // the tensor-core sweep (binary32 rows)
  return on && L.model == MD_KUR && L.split && (f32_tma || f16_tc) && next_fs32 == L.ss32 && next_gs32 == L.gs32;
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("MS_PDL");
    return !(v && std::strcmp(v, "off") == 0);
  }();
  return on;
}

void launch_rhs_fast(const RhsLaunch& L, const RhsArgs& a) {
  switch (L.model) {
    case MD_LCO: by_prec<MD_LCO, false>(L, a); break;
    case MD_KUR:
      if (!L.split) throw std::invalid_argument("rhs_fast: Kuramoto runs split");
      by_prec<MD_KUR, true>(L, a);
      break;
    case MD_CC: by_prec<MD_CC, false>(L, a); break;
    default: throw std::invalid_argument("rhs_fast: bad model");
  }
}

void* tc16_create(const void* K, int64_t ld, int rows, int ks) {
  if (ks != MS_K_F16 || ld % (kGvKB * kGvBK) != 0 || rows < 1) return nullptr;
  GvRes* r = new GvRes{};
  r->tiles = (rows + kGvBM - 1) / kGvBM;
  r->chunks = (int)((ld + kGvChunk - 1) / kGvChunk);
  r->kblocks = (int)(ld / kGvBK);
  const size_t ktbytes = (size_t)r->tiles * r->kblocks * kGvABytes;
  const size_t pbytes = sizeof(float2) * (size_t)r->tiles * r->chunks * kGvBM;
  if (cudaMalloc(&r->kt, ktbytes) != cudaSuccess || cudaMalloc(&r->part, pbytes) != cudaSuccess ||
      cudaMalloc(&r->cnt, sizeof(int) * r->tiles) != cudaSuccess ||
      cudaMemset(r->cnt, 0, sizeof(int) * r->tiles) != cudaSuccess) {
    cudaGetLastError();
    tc16_destroy(r);
    return nullptr;  // no room for the tile images: the CUDA-core sweeps serve f16 K
  }
  tc16_refresh(r, K, ld, rows, nullptr);
  return r;
}

void tc16_refresh(void* p, const void* K, int64_t ld, int rows, cudaStream_t st) {
  GvRes* r = static_cast<GvRes*>(p);
  if (!r) return;
  k_tile_k16<<<1024, 256, 0, st>>>(static_cast<const __half*>(K), r->kt, ld, rows, r->tiles, r->kblocks);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string("tc16 tile images: ") + cudaGetErrorString(e));
}

void tc16_destroy(void* p) {
  GvRes* r = static_cast<GvRes*>(p);
  if (!r) return;
  if (r->kt) cudaFree(r->kt);
  if (r->part) cudaFree(r->part);
  if (r->cnt) cudaFree(r->cnt);
  delete r;
}

MS_DEFINE_LAUNCH_READER(launches_tu_fast)

}  // namespace msb
