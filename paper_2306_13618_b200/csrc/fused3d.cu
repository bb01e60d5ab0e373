// Tuned d = 3 NFFT half-step (placeholder until the cell-group kernel lands).
#include "common.cuh"
#include "epilogue.cuh"

namespace uotk {

bool fused3d_available(const FastParams& fp) {
    (void)fp;
    return false;
}

void fused3d_gather_spread(const PointSet&, const double*, double*, const FastParams&, const EpiSinkhorn&,
                           unsigned long long*, cudaStream_t) {
    fail(UOTK_EUNSUPPORTED, "fused3d kernel not built");
}

}  // namespace uotk
