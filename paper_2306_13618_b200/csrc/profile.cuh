// RAII event bracket for live kernel timing (see profile.cu).
#pragma once
#include <cuda_runtime.h>

namespace uotk {

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
