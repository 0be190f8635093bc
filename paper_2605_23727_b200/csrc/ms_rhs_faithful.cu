// ms_rhs_faithful.cu — instantiation and launch of k_rhs_faithful (the
// reference-order coupling sum, systems.cpp:50-57).
#include <stdexcept>

#include "ms_dispatch.h"

namespace msb {

namespace {

constexpr int kFaithThreads = 128;

template <int MODEL, class SS, class GS, int KS>
void go(const RhsLaunch& L, const RhsArgs& a) {
  const int rows = a.row1 - a.row0;
  const int grid = (rows + kFaithThreads - 1) / kFaithThreads;
  k_rhs_faithful<MODEL, SS, GS, KS><<<grid, kFaithThreads, 0, L.stream>>>(a);
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
