// NVTX ranges around the C-ABI entry points (SURVEY §5 tracing): an Nsight
// timeline shows upload / factor / download / PCG as named spans. nvtx3 is
// header-only; with no tool attached a push/pop is a few nanoseconds.
#pragma once

#include <nvtx3/nvToolsExt.h>

namespace parac_gpu {
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
}  // namespace parac_gpu
