// Launch plumbing for worker_step_kernel<T, NP>: cluster-size choice and
// cudaLaunchKernelEx with a runtime cluster dimension. Included once per dtype TU.
#pragma once
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>

#include "launch.h"

namespace hpcg {

constexpr int kMaxDynSmem = 232448 - (int)sizeof(StepShared) - 256;  // 227 KB opt-in minus static smem

template <typename T, int NP>
cudaError_t step_geometry_uncached(int64_t s, int k, int ncand, int W, StepGeometry* g, std::string* why) {
    auto kern = worker_step_kernel<T, NP>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    int cmin = 0;
    for (int c = 1; c <= 16; ++c) {
        if (c > s) break;
        const int rows = (int)((s + c - 1) / c);
        if (step_layout<T, NP>(rows, k, ncand, c).total <= kMaxDynSmem) {
            cmin = c;
            break;
        }
    }
    if (cmin == 0) {
        if (why) *why = "sample does not fit a 16-CTA cluster's shared memory";
        return cudaErrorInvalidValue;
    }
    // widen the cluster while it raises the number of SMs busy (few workers) or the
    // packing of clusters into GPCs; stop at 16 and at >= 128 rows per CTA.
    int best_c = cmin, best_used = -1, best_active = 0;
    const char* force = getenv("HPCG_CLUSTER");  // diagnostics: pin the cluster size
    const int fc = force ? atoi(force) : 0;
    for (int c = cmin; c <= 16 && c <= s; ++c) {
        if (fc && c != fc) continue;
        const int rows = (int)((s + c - 1) / c);
        if (c > cmin && rows < 128) break;
        const int smem = step_layout<T, NP>(rows, k, ncand, c).total;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)(c * (W > 0 ? W : 1)));
        cfg.blockDim = dim3(kStepThreads);
        cfg.dynamicSmemBytes = (size_t)smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = (unsigned)c;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int active = 0;
        e = cudaOccupancyMaxActiveClusters(&active, kern, &cfg);
        if (e != cudaSuccess) {
            cudaGetLastError();
            continue;
        }
        if (active <= 0) continue;
        const int conc = active < W ? active : W;
        const int used = conc * c;  // CTAs resident at once (2 per SM when the smem allows)
        if (used > best_used) {
            best_used = used;
            best_c = c;
            best_active = active;
        }
    }
    if (best_used < 0) {
        if (why) *why = "no schedulable cluster configuration";
        return cudaErrorInvalidConfiguration;
    }
    g->cluster = best_c;
    g->rows_cap = (int)((s + best_c - 1) / best_c);
    g->smem = step_layout<T, NP>(g->rows_cap, k, ncand, best_c).total;
    g->active_clusters = best_active;
    return cudaSuccess;
}

// Geometry is a pure function of (device, shape): cache it (the occupancy queries cost
// tens of microseconds each and the engine launches one step per round).
template <typename T, int NP>
cudaError_t step_geometry_t(int64_t s, int k, int ncand, int W, StepGeometry* g, std::string* why) {
    static std::mutex mu;
    static std::map<std::tuple<int, int64_t, int, int, int>, StepGeometry> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    const auto key = std::make_tuple(dev, s, k, ncand, W);
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = cache.find(key);
        if (it != cache.end()) {
            *g = it->second;
            return cudaSuccess;
        }
    }
    cudaError_t e = step_geometry_uncached<T, NP>(s, k, ncand, W, g, why);
    if (e == cudaSuccess) {
        std::lock_guard<std::mutex> lk(mu);
        cache[key] = *g;
    }
    return e;
}

template <typename T, int NP>
cudaError_t launch_step_t(const StepParams& p_in, cudaStream_t st, StepGeometry* geo_out, std::string* why) {
    StepGeometry g;
    cudaError_t e = step_geometry_t<T, NP>(p_in.s, p_in.k, p_in.candidates, p_in.geo_W > 0 ? p_in.geo_W : p_in.W, &g,
                                           why);
    if (e != cudaSuccess) return e;
    StepParams p = p_in;
    p.rows_cap = g.rows_cap;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(g.cluster * p.W));
    cfg.blockDim = dim3(kStepThreads);
    cfg.dynamicSmemBytes = (size_t)g.smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)g.cluster;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (p.trace) {  // the diagnostic timeline build (same geometry: the attributes are set for both)
        auto kt = worker_step_kernel<T, NP, true>;
        cudaFuncSetAttribute(kt, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem);
        cudaFuncSetAttribute(kt, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        e = cudaLaunchKernelEx(&cfg, kt, p);
    } else {
        e = cudaLaunchKernelEx(&cfg, worker_step_kernel<T, NP>, p);
    }
    if (geo_out) *geo_out = g;
    static const bool dbg = getenv("HPCG_DEBUG") != nullptr;
    if (dbg)
        fprintf(stderr, "[hpcg] step NP=%d s=%lld k=%d W=%d: cluster %d rows_cap %d smem %d active_clusters %d\n", NP,
                (long long)p.s, p.k, p.W, g.cluster, g.rows_cap, g.smem, g.active_clusters);
    return e;
}

}  // namespace hpcg
