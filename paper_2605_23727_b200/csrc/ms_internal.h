// ms_internal.h — what other translation units may know of a system handle.
#pragma once
#include <cuda_runtime.h>
#include "../../include/mixedstep_b200.h"

namespace msb {
struct SysView {
  int mkind;        // MD_* (or a fixture id)
  int n, d, ld;
  int row0, row1;
  int ks;           // MS_K_*
  int dev, sms;
  const void* K;
  double coupling_k;
  cudaStream_t stream;
};
SysView sys_view(ms_system_t s);
// the thread-local message behind ms_last_error()
void set_last_error(const char* msg);
// MS_CTL_SMEM: controllers run on a shared-memory copy of Ctl (default on)
bool ctl_smem_enabled();
// per-translation-unit kernel launch counters (ms_common.cuh count_launch)
unsigned long long launches_tu_fast();
unsigned long long launches_tu_faithful();
unsigned long long launches_tu_multi();
unsigned long long launches_tu_batch();
}  // namespace msb
