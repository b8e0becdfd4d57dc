// nvtx.h -- NVTX ranges around the C ABI's phases (host-side ranges at
// enqueue time), so `ncu --nvtx --nvtx-include "pn_newton_step/"` or any
// NVTX-aware profiler can select a phase's kernels.  NVTX v3 is header-only;
// without an attached tool a push/pop is a predictable branch.
#pragma once
#include <nvtx3/nvToolsExt.h>

namespace pn {
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange &) = delete;
  NvtxRange &operator=(const NvtxRange &) = delete;
};
}  // namespace pn
