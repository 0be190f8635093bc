// ms_dispatch.h — host launchers of the templated coupling kernels.
#pragma once
#include <utility>

#include "ms_kernels.cuh"

namespace msb {

struct RhsLaunch {
  int model;   // MD_*
  bool split;  // Kuramoto sin/cos split (fast mode only)
  bool ss32, gs32;
  int ks;      // MS_K_*
  int num_sms;
  cudaStream_t stream;
  // optional: the prep of the attempt's next stage, run at the end of this
  // sweep when fuse_next_ok() holds (*fused is set when it did)
  const PrepArgs* next = nullptr;
  bool next_fs32 = false, next_gs32 = false;
  bool* fused = nullptr;
  bool tc16 = false;  // this sweep runs on the tensor cores (tc16_selected)
};

// whether launch_rhs_fast sends this binary32 split-Kuramoto sweep to the
// tensor-core kernel (f16 K with tile images, operand image present, size / MS_SWEEP)
bool tc16_selected(const RhsArgs& a, int ks);

// whether launch_rhs_fast folds the next stage's prep (row F/G precisions
// next_fs32/next_gs32) into this sweep: the split Kuramoto's row-copy TMA sweep
// of f32 K, next row with F in this row's sum format and the same G format,
// whole (unsharded) handles; MS_FUSE_NEXT=off disables it
bool fuse_next_ok(const RhsLaunch& L, bool next_fs32, bool next_gs32);

// rhs_fast over rows [a.row0, a.row1): one persistent CTA per SM
void launch_rhs_fast(const RhsLaunch& L, const RhsArgs& a);
// rhs_faithful: one thread per row
void launch_rhs_faithful(const RhsLaunch& L, const RhsArgs& a);
// prep + sweep in one launch (k_eval_fused) when the column data fits in shared
// memory and the row (F, Sigma, G) is SSS / DDS / DDD; false = not applicable
// (the caller then launches k_prep + the sweep). MS_FUSE=off disables it.
bool launch_eval_fused(const RhsLaunch& L, const PrepArgs& p, const RhsArgs& a, bool fs32);
// the split Kuramoto's sweep for small N after k_prep (column values staged in
// shared memory, one row per warp), MS_SWEEP=small only; false = not used
bool launch_sweep_small(const RhsLaunch& L, const PrepArgs& p, const RhsArgs& a);

// the f16-K tensor-core sweep's per-handle resources (K tensor map, chunk
// partials, tickets): created with a Kuramoto system whose K is f16, null if
// not applicable
void* tc16_create(const void* K, int64_t ld, int rows, int ks);
// rebuild the tile images after K changed (ms_system_fill_k_uniform)
void tc16_refresh(void* r, const void* K, int64_t ld, int rows, cudaStream_t st);
void tc16_destroy(void* r);

// Programmatic dependent launch for the kernels of the attempt chain (each
// starts with pdl_enter()); MS_PDL=off launches them plainly.
bool pdl_enabled();
template <class... KArgs, class... Args>
inline cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                            Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

}  // namespace msb
