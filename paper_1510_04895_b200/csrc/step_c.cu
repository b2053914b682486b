// Step-kernel instantiations for one scalar layout (split from kernels.cu so the
// three layouts compile in parallel).
#include "step_kernels.cuh"

namespace cfd {
void launch_step_c(Context& ctx, const StepArgs& s, cudaStream_t st, int units, int pitch) {
    dispatch_kind<true, double2>(ctx, s, st, units, pitch);
}
}  // namespace cfd
