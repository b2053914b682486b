// Row-group step kernel instantiations for one scalar layout (see step_group.cuh).
#include "step_group.cuh"

namespace cfd {
bool launch_group_c(Context& ctx, const StepArgs& s, cudaStream_t st, int units, int pitch) {
    return dispatch_group<true, double2>(ctx, s, st, units, pitch);
}
}  // namespace cfd
