// Site-ring step kernel instantiations (complex layout; see step_ring.cuh).
#include "step_ring.cuh"

namespace cfd {
bool launch_ring_c(Context& ctx, const StepArgs& s, cudaStream_t st, int units, int pitch) {
    return dispatch_ring(ctx, s, st, units, pitch);
}
}  // namespace cfd
