// Optional live kernel timing (bench.py's roofline): when enabled, every instrumented
// launch is bracketed by CUDA events recorded on the launching stream; the per-tag
// sums of the event intervals are read back with uotk_profile_read.
#include <cstring>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "profile.cuh"

namespace uotk {

namespace {
struct Rec {
    int tag;
    cudaEvent_t a, b;
};
struct Prof {
    std::mutex mu;
    bool on = false;
    std::vector<cudaEvent_t> pool;
    size_t used = 0;
    std::vector<Rec> recs;
};
Prof& prof() {
    static Prof* p = new Prof();
    return *p;
}
cudaEvent_t take_event(Prof& p) {
    if (p.used == p.pool.size()) {
        cudaEvent_t e;
        UOTK_CUDA(cudaEventCreate(&e));
        p.pool.push_back(e);
    }
    return p.pool[p.used++];
}
const char* kTagNames[kProfTags] = {"spread", "gather", "fused", "fft", "direct", "setup"};
}  // namespace

bool profiling_enabled() {
    Prof& p = prof();
    std::lock_guard<std::mutex> lk(p.mu);
    return p.on;
}

ProfScope::ProfScope(int tag, cudaStream_t s) : tag_(tag), s_(s) {
    nvtxRangePushA(kTagNames[tag]);
    Prof& p = prof();
    if (!p.on) return;
    std::lock_guard<std::mutex> lk(p.mu);
    a_ = take_event(p);
    b_ = take_event(p);
    UOTK_CUDA(cudaEventRecord(a_, s));
    active_ = true;
}

ProfScope::~ProfScope() {
    nvtxRangePop();
    if (!active_) return;
    Prof& p = prof();
    std::lock_guard<std::mutex> lk(p.mu);
    cudaEventRecord(b_, s_);
    p.recs.push_back({tag_, a_, b_});
}

}  // namespace uotk

using namespace uotk;

extern "C" {

void uotk_profile_enable(int on) {
    Prof& p = prof();
    std::lock_guard<std::mutex> lk(p.mu);
    p.on = on != 0;
}

void uotk_profile_reset(void) {
    Prof& p = prof();
    std::lock_guard<std::mutex> lk(p.mu);
    p.recs.clear();
    p.used = 0;
}

int uotk_profile_read(const char* tag, double* ms, int64_t* count) {
    Prof& p = prof();
    std::lock_guard<std::mutex> lk(p.mu);
    int t = -1;
    for (int i = 0; i < kProfTags; ++i)
        if (tag && strcmp(tag, kTagNames[i]) == 0) t = i;
    if (t < 0 || !ms || !count) return UOTK_EINVAL;
    double sum = 0;
    int64_t c = 0;
    for (const Rec& r : p.recs) {
        if (r.tag != t) continue;
        if (cudaEventSynchronize(r.b) != cudaSuccess) return UOTK_ECUDA;
        float e = 0;
        if (cudaEventElapsedTime(&e, r.a, r.b) != cudaSuccess) return UOTK_ECUDA;
        sum += e;
        ++c;
    }
    *ms = sum;
    *count = c;
    return UOTK_OK;
}

}  // extern "C"
