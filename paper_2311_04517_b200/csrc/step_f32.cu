// fp32 instantiations of the worker-step kernel (padded row widths NP).
#include "step_launch.cuh"

namespace hpcg {

cudaError_t launch_step_f32(const StepParams& p, cudaStream_t st, StepGeometry* g, std::string* why, int np) {
    switch (np) {
        case 2: return launch_step_t<float, 2>(p, st, g, why);
        case 4: return launch_step_t<float, 4>(p, st, g, why);
        case 8: return launch_step_t<float, 8>(p, st, g, why);
        case 12: return launch_step_t<float, 12>(p, st, g, why);
        case 16: return launch_step_t<float, 16>(p, st, g, why);
        case 24: return launch_step_t<float, 24>(p, st, g, why);
        case 32: return launch_step_t<float, 32>(p, st, g, why);
    }
    return cudaErrorInvalidValue;
}

cudaError_t geometry_f32(int np, int64_t s, int k, int ncand, int W, StepGeometry* g, std::string* why) {
    switch (np) {
        case 2: return step_geometry_t<float, 2>(s, k, ncand, W, g, why);
        case 4: return step_geometry_t<float, 4>(s, k, ncand, W, g, why);
        case 8: return step_geometry_t<float, 8>(s, k, ncand, W, g, why);
        case 12: return step_geometry_t<float, 12>(s, k, ncand, W, g, why);
        case 16: return step_geometry_t<float, 16>(s, k, ncand, W, g, why);
        case 24: return step_geometry_t<float, 24>(s, k, ncand, W, g, why);
        case 32: return step_geometry_t<float, 32>(s, k, ncand, W, g, why);
    }
    return cudaErrorInvalidValue;
}

}  // namespace hpcg
