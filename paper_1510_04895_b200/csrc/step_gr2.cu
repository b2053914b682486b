// Row-group step kernel instantiations for one scalar layout (see step_group.cuh).
#include "step_group.cuh"

namespace cfd {
bool launch_group_r2(Context& ctx, const StepArgs& s, cudaStream_t st, int units, int pitch) {
    return dispatch_group<false, double2>(ctx, s, st, units, pitch);
}
}  // namespace cfd
