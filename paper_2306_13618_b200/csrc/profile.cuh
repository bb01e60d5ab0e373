// RAII event bracket for live kernel timing (see profile.cu).
#pragma once
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

namespace uotk {

// NVTX range over a host-side phase (visible in Nsight Systems / ncu --nvtx; header-only
// NVTX3: a no-op unless a tool is attached).  Every API call and every ProfScope-tagged
// pass is one range ("uotk_uot_sinkhorn", "setup", "pointsets", "iterations", "spread", ...).
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

enum ProfTag { kProfSpread = 0, kProfGather = 1, kProfFused = 2, kProfFft = 3, kProfDirect = 4, kProfSetup = 5 };
constexpr int kProfTags = 6;

bool profiling_enabled();

class ProfScope {
   public:
    ProfScope(int tag, cudaStream_t s);
    ~ProfScope();
    ProfScope(const ProfScope&) = delete;
    ProfScope& operator=(const ProfScope&) = delete;

   private:
    int tag_;
    cudaStream_t s_;
    bool active_ = false;
    cudaEvent_t a_ = nullptr, b_ = nullptr;
};

}  // namespace uotk
