// ms_dispatch.h — host launchers of the templated coupling kernels.
#pragma once
#include "ms_kernels.cuh"

namespace msb {

struct RhsLaunch {
  int model;   // MD_*
  bool split;  // Kuramoto sin/cos split (fast mode only)
  bool ss32, gs32;
  int ks;      // MS_K_*
  int num_sms;
  cudaStream_t stream;
};

// rhs_fast over rows [a.row0, a.row1): one persistent CTA per SM
void launch_rhs_fast(const RhsLaunch& L, const RhsArgs& a);
// rhs_faithful: one thread per row
void launch_rhs_faithful(const RhsLaunch& L, const RhsArgs& a);

}  // namespace msb
