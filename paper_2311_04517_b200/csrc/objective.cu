// Instantiations and dispatch for the full-data objective kernel, plus the NP tables
// shared by every launcher.
#include "launch.h"

namespace hpcg {

cudaError_t launch_step_f32(const StepParams& p, cudaStream_t st, StepGeometry* g, std::string* why, int np);
cudaError_t launch_step_f64(const StepParams& p, cudaStream_t st, StepGeometry* g, std::string* why, int np);
cudaError_t geometry_f32(int np, int64_t s, int k, int ncand, int W, StepGeometry* g, std::string* why);
cudaError_t geometry_f64(int np, int64_t s, int k, int ncand, int W, StepGeometry* g, std::string* why);

int pick_np(int dtype, int n) {
    static const int f32[] = {2, 4, 8, 12, 16, 24, 32};
    static const int f64[] = {1, 2, 3, 4, 6, 8, 12, 16, 24, 32};
    if (dtype == 0) {
        for (int v : f32)
            if (v >= n) return v;
    } else {
        for (int v : f64)
            if (v >= n) return v;
    }
    return 0;
}

cudaError_t launch_step(int dtype, const StepParams& p, cudaStream_t st, StepGeometry* g, std::string* why) {
    const int np = pick_np(dtype, p.n);
    if (np == 0) return cudaErrorInvalidValue;
    return dtype == 0 ? launch_step_f32(p, st, g, why, np) : launch_step_f64(p, st, g, why, np);
}

cudaError_t step_geometry(int dtype, int n, int64_t s, int k, int ncand, int W, StepGeometry* g, std::string* why) {
    const int np = pick_np(dtype, n);
    if (np == 0) return cudaErrorInvalidValue;
    return dtype == 0 ? geometry_f32(np, s, k, ncand, W, g, why) : geometry_f64(np, s, k, ncand, W, g, why);
}

int objective_blocks() {  // upper bound on the grid of any objective launch
    static int nb = 0;
    if (nb == 0) {
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        nb = sms * 8;
    }
    return nb;
}

// grid = SMs x resident blocks per SM (a pure function of device, kernel and kv, so the
// block partials -- and hence f(C,X) -- are reproducible)
template <typename T, int NP>
static cudaError_t launch_obj_t(const ObjParams& p, int* nblocks, cudaStream_t st) {
    const int smem = objective_smem<T, NP>(p.kv);
    auto kern = objective_kernel<T, NP>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0, dev = 0, sms = 148;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kObjThreads, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int nb = sms * per_sm;
    if (nblocks[0] < nb) {  // caller's partial buffer too small: report the size needed
        nblocks[0] = nb;
        return cudaErrorNotReady;
    }
    nblocks[0] = nb;
    kern<<<nb, kObjThreads, smem, st>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_objective(int dtype, const ObjParams& p, int* nblocks, cudaStream_t st) {
    const int np = pick_np(dtype, p.n);
    if (dtype == 0) {
        switch (np) {
            case 2: return launch_obj_t<float, 2>(p, nblocks, st);
            case 4: return launch_obj_t<float, 4>(p, nblocks, st);
            case 8: return launch_obj_t<float, 8>(p, nblocks, st);
            case 12: return launch_obj_t<float, 12>(p, nblocks, st);
            case 16: return launch_obj_t<float, 16>(p, nblocks, st);
            case 24: return launch_obj_t<float, 24>(p, nblocks, st);
            case 32: return launch_obj_t<float, 32>(p, nblocks, st);
        }
    } else {
        switch (np) {
            case 1: return launch_obj_t<double, 1>(p, nblocks, st);
            case 2: return launch_obj_t<double, 2>(p, nblocks, st);
            case 3: return launch_obj_t<double, 3>(p, nblocks, st);
            case 4: return launch_obj_t<double, 4>(p, nblocks, st);
            case 6: return launch_obj_t<double, 6>(p, nblocks, st);
            case 8: return launch_obj_t<double, 8>(p, nblocks, st);
            case 12: return launch_obj_t<double, 12>(p, nblocks, st);
            case 16: return launch_obj_t<double, 16>(p, nblocks, st);
            case 24: return launch_obj_t<double, 24>(p, nblocks, st);
            case 32: return launch_obj_t<double, 32>(p, nblocks, st);
        }
    }
    return cudaErrorInvalidValue;
}

}  // namespace hpcg
