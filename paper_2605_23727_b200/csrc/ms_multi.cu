// ms_multi.cu — instantiations and launch of k_rhs_multi (ms_multi.cuh): one
// kernel per (K storage, lane-type counts) with 1..4 lanes (one lane: the
// 2D-TMA-tiled single-system split sweep, MS_SWEEP=tile).
#include <cudaTypedefs.h>

#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <tuple>

#include "ms_multi.cuh"

namespace msb {

namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess || !p)
      throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// K tile maps: [rows][ld] row-major, 64-row x (32*VEC)-column boxes, cached per
// (K pointer, shape, storage)
const CUtensorMap& k_map(const void* K, int64_t ld, int rows, int ks, int tr) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int64_t, int, int, int>, CUtensorMap> cache;
  std::lock_guard<std::mutex> lk(mu);
  const auto key = std::make_tuple(K, ld, rows, ks, tr);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  CUtensorMap m;
  const bool k16 = ks != MS_K_F32;
  const CUtensorMapDataType dt = ks == MS_K_F32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                 : ks == MS_K_F16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                                  : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  const cuuint64_t dims[2] = {(cuuint64_t)ld, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * (k16 ? 2 : 4)};
  const cuuint32_t box[2] = {(cuuint32_t)(k16 ? MultiGeom<MS_K_F16>::TC : MultiGeom<MS_K_F32>::TC),
                             (cuuint32_t)tr};
  const cuuint32_t es[2] = {1, 1};
  CUresult r = encode_fn()(&m, dt, 2, const_cast<void*>(K), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw std::runtime_error("tensor map (K tiles) encode failed");
  return cache.emplace(key, m).first->second;
}

template <int KS, int NS, int NDS, int NDD>
void go(const CUtensorMap& tm, const MultiArgs& m, int grid, cudaStream_t st) {
  auto kern = k_rhs_multi<KS, NS, NDS, NDD>;
  static bool attr_done = false;
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)MultiGeom<KS, NS + NDS + NDD>::SMEM);
    if (e != cudaSuccess) throw std::runtime_error(std::string("rhs_multi attribute: ") + cudaGetErrorString(e));
    attr_done = true;
  }
  kern<<<grid, kMultiThreads, MultiGeom<KS, NS + NDS + NDD>::SMEM, st>>>(tm, m);
}

template <int KS, int NS, int NDS>
void by_dd(int ndd, const CUtensorMap& tm, const MultiArgs& m, int grid, cudaStream_t st) {
  constexpr int left = kMaxLanes - NS - NDS;
  switch (ndd) {
    case 0: if constexpr (NS + NDS >= 1) { go<KS, NS, NDS, 0>(tm, m, grid, st); return; } break;
    case 1: if constexpr (left >= 1) { go<KS, NS, NDS, 1>(tm, m, grid, st); return; } break;
    case 2: if constexpr (left >= 2) { go<KS, NS, NDS, 2>(tm, m, grid, st); return; } break;
    case 3: if constexpr (left >= 3) { go<KS, NS, NDS, 3>(tm, m, grid, st); return; } break;
    case 4: if constexpr (left >= 4) { go<KS, NS, NDS, 4>(tm, m, grid, st); return; } break;
    default: break;
  }
  throw std::invalid_argument("rhs_multi: unsupported lane mix");
}

template <int KS, int NS>
void by_ds(int nds, int ndd, const CUtensorMap& tm, const MultiArgs& m, int grid, cudaStream_t st) {
  switch (nds) {
    case 0: by_dd<KS, NS, 0>(ndd, tm, m, grid, st); return;
    case 1: if constexpr (NS <= 3) { by_dd<KS, NS, 1>(ndd, tm, m, grid, st); return; } break;
    case 2: if constexpr (NS <= 2) { by_dd<KS, NS, 2>(ndd, tm, m, grid, st); return; } break;
    case 3: if constexpr (NS <= 1) { by_dd<KS, NS, 3>(ndd, tm, m, grid, st); return; } break;
    case 4: if constexpr (NS == 0) { by_dd<KS, NS, 4>(ndd, tm, m, grid, st); return; } break;
    default: break;
  }
  throw std::invalid_argument("rhs_multi: unsupported lane mix");
}

template <int KS>
void by_s(int ns, int nds, int ndd, const CUtensorMap& tm, const MultiArgs& m, int grid, cudaStream_t st) {
  switch (ns) {
    case 0: by_ds<KS, 0>(nds, ndd, tm, m, grid, st); return;
    case 1: by_ds<KS, 1>(nds, ndd, tm, m, grid, st); return;
    case 2: by_ds<KS, 2>(nds, ndd, tm, m, grid, st); return;
    case 3: by_ds<KS, 3>(nds, ndd, tm, m, grid, st); return;
    case 4: by_ds<KS, 4>(nds, ndd, tm, m, grid, st); return;
    default: throw std::invalid_argument("rhs_multi: unsupported lane mix");
  }
}

}  // namespace

void launch_rhs_multi(const MultiArgs& m, int ns, int nds, int ndd, int ks, const void* K, int sms, cudaStream_t st) {
  if (ns + nds + ndd != m.nl || m.nl < 1 || m.nl > kMaxLanes) throw std::invalid_argument("rhs_multi: lane count");
  const int rows = m.row1 - m.row0;
  const int tr = m.nl == 1 ? MultiGeom<MS_K_F32, 1>::TR : MultiGeom<MS_K_F32>::TR;
  const CUtensorMap& tm = k_map(K, m.ld, rows, ks, tr);
  const int groups = (rows + tr - 1) / tr;
  const int grid = groups < sms ? groups : sms;
  switch (ks) {
    case MS_K_F32: by_s<MS_K_F32>(ns, nds, ndd, tm, m, grid, st); break;
    case MS_K_F16: by_s<MS_K_F16>(ns, nds, ndd, tm, m, grid, st); break;
    case MS_K_BF16: by_s<MS_K_BF16>(ns, nds, ndd, tm, m, grid, st); break;
    default: throw std::invalid_argument("rhs_multi: K storage");
  }
}

MS_DEFINE_LAUNCH_READER(launches_tu_multi)

}  // namespace msb
