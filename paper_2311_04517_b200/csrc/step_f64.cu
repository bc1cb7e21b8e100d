// fp64 instantiations of the worker-step kernel (padded row widths NP).
#include "step_launch.cuh"

namespace hpcg {

cudaError_t launch_step_f64(const StepParams& p, cudaStream_t st, StepGeometry* g, std::string* why, int np) {
    switch (np) {
        case 1: return launch_step_t<double, 1>(p, st, g, why);
        case 2: return launch_step_t<double, 2>(p, st, g, why);
        case 3: return launch_step_t<double, 3>(p, st, g, why);
        case 4: return launch_step_t<double, 4>(p, st, g, why);
        case 6: return launch_step_t<double, 6>(p, st, g, why);
        case 8: return launch_step_t<double, 8>(p, st, g, why);
        case 12: return launch_step_t<double, 12>(p, st, g, why);
        case 16: return launch_step_t<double, 16>(p, st, g, why);
        case 24: return launch_step_t<double, 24>(p, st, g, why);
        case 32: return launch_step_t<double, 32>(p, st, g, why);
    }
    return cudaErrorInvalidValue;
}

cudaError_t geometry_f64(int np, int64_t s, int k, int ncand, int W, StepGeometry* g, std::string* why) {
    switch (np) {
        case 1: return step_geometry_t<double, 1>(s, k, ncand, W, g, why);
        case 2: return step_geometry_t<double, 2>(s, k, ncand, W, g, why);
        case 3: return step_geometry_t<double, 3>(s, k, ncand, W, g, why);
        case 4: return step_geometry_t<double, 4>(s, k, ncand, W, g, why);
        case 6: return step_geometry_t<double, 6>(s, k, ncand, W, g, why);
        case 8: return step_geometry_t<double, 8>(s, k, ncand, W, g, why);
        case 12: return step_geometry_t<double, 12>(s, k, ncand, W, g, why);
        case 16: return step_geometry_t<double, 16>(s, k, ncand, W, g, why);
        case 24: return step_geometry_t<double, 24>(s, k, ncand, W, g, why);
        case 32: return step_geometry_t<double, 32>(s, k, ncand, W, g, why);
    }
    return cudaErrorInvalidValue;
}

}  // namespace hpcg
