// ms_rhs_faithful.cu — instantiation and launch of k_rhs_seq (the
// reference-order coupling sum, systems.cpp:50-57; rhs modes faithful and,
// for the Kuramoto split in sequential order, ordered).
#include <stdexcept>
#include <string>

#include "ms_dispatch.h"

namespace msb {

namespace {

template <int MODEL, bool SPLIT, class SS, class GS, int KS>
void go_split(const RhsLaunch& L, const RhsArgs& a) {
  auto kern = k_rhs_seq<MODEL, SPLIT, SS, GS, KS>;
  constexpr size_t smem = SeqGeom<SS, SPLIT>::SMEM;
  static bool attr_done = false;
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) throw std::runtime_error(std::string("rhs_seq attribute: ") + cudaGetErrorString(e));
    attr_done = true;
  }
  const int rows = a.row1 - a.row0;
  const int grid = (rows + kSeqRows - 1) / kSeqRows;
  cudaError_t e = launch_k(kern, grid, kSeqThreads, smem, L.stream, a);
  if (e != cudaSuccess) throw std::runtime_error(std::string("rhs_seq launch: ") + cudaGetErrorString(e));
}

template <int MODEL, class SS, class GS, int KS>
void go(const RhsLaunch& L, const RhsArgs& a) {
  if (MODEL == MD_KUR && L.split) go_split<MODEL, true, SS, GS, KS>(L, a);
  else go_split<MODEL, false, SS, GS, KS>(L, a);
}

template <int MODEL, class SS, class GS>
void by_k(const RhsLaunch& L, const RhsArgs& a) {
  switch (L.ks) {
    case MS_K_SCALAR: go<MODEL, SS, GS, MS_K_SCALAR>(L, a); break;
    case MS_K_F32: go<MODEL, SS, GS, MS_K_F32>(L, a); break;
    case MS_K_F16: go<MODEL, SS, GS, MS_K_F16>(L, a); break;
    case MS_K_BF16: go<MODEL, SS, GS, MS_K_BF16>(L, a); break;
    default: throw std::invalid_argument("rhs_faithful: bad K storage");
  }
}

template <int MODEL>
void by_prec(const RhsLaunch& L, const RhsArgs& a) {
  if (L.ss32) {
    if (L.gs32) by_k<MODEL, float, float>(L, a);
    else by_k<MODEL, float, double>(L, a);
  } else {
    if (L.gs32) by_k<MODEL, double, float>(L, a);
    else by_k<MODEL, double, double>(L, a);
  }
}

}  // namespace

void launch_rhs_faithful(const RhsLaunch& L, const RhsArgs& a) {
  switch (L.model) {
    case MD_LCO: by_prec<MD_LCO>(L, a); break;
    case MD_KUR: by_prec<MD_KUR>(L, a); break;
    case MD_CC: by_prec<MD_CC>(L, a); break;
    default: throw std::invalid_argument("rhs_faithful: bad model");
  }
}

MS_DEFINE_LAUNCH_READER(launches_tu_faithful)

}  // namespace msb
