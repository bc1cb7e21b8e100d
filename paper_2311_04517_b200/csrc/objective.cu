// Instantiations and dispatch for the full-data objective kernel, plus the NP tables
// shared by every launcher.
#include <cstdlib>
#include <cstring>
#include <cudaTypedefs.h>

#define HPCG_OBJECTIVE_TU  // this TU owns the objective kernels and their constant bank
#include "launch.h"
#include "objective_rows.cuh"
#include "objective_tcw.cuh"

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
    // the cluster-resident kernel when the shape fits it (n <= 32, k <= 32, sample in a
    // cluster's shared memory), the grid-wide HBM path otherwise
    const int np = pick_np(dtype, p.n);
    static const bool force_wide = getenv("HPCG_WIDE") != nullptr;
    // one worker with a large sample (the inner strategy, engine.hpp:243-246, 446): the grid-wide
    // path spreads its rows over every SM (G CTAs per pass) instead of one <= 16-CTA cluster
    const bool one_big = (p.geo_W > 0 ? p.geo_W : p.W) == 1 && p.s >= kInnerWideRows;
    if (np != 0 && p.k <= kMaxK && p.candidates <= kMaxCandidates && !force_wide && !one_big) {
        StepGeometry tmp;
        std::string w2;
        if (step_geometry(dtype, p.n, p.s, p.k, p.candidates, p.geo_W > 0 ? p.geo_W : p.W, &tmp, &w2) == cudaSuccess)
            return dtype == 0 ? launch_step_f32(p, st, g, why, np) : launch_step_f64(p, st, g, why, np);
    }
    if (g) *g = StepGeometry{};
    if (p.go) {  // per-worker go flags are read by the cluster-resident kernel only
        if (why) *why = "the free-running schedule needs a cluster-resident shape";
        return cudaErrorNotSupported;
    }
    return launch_step_wide(dtype, p, st, why);
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
// TMA applicability: unpadded rows of 16/32/48/64/128 bytes (the swizzle spans that equal
// Geo::swz), 16-B aligned base.
template <typename T, int NP>
static bool tma_ok(const ObjParams& p) {
    using G = Geo<T, NP>;
    if (p.n != NP || (reinterpret_cast<uintptr_t>(p.X) & 15) != 0) return false;
    const int rb = G::RS;
    return rb == 16 || rb == 32 || rb == 48 || rb == 64 || rb == 128;
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    }
    return fn;
}

template <typename T>
static bool make_tmap(const ObjParams& p, int box_rows, CUtensorMap* map) {
    auto fn = encode_fn();
    if (!fn) return false;
    const cuuint64_t dims[2] = {(cuuint64_t)p.n, (cuuint64_t)p.m};
    const cuuint64_t strides[1] = {(cuuint64_t)p.n * sizeof(T)};
    const cuuint32_t box[2] = {(cuuint32_t)p.n, (cuuint32_t)box_rows};
    const cuuint32_t estr[2] = {1, 1};
    const int rb = p.n * (int)sizeof(T);
    const CUtensorMapSwizzle sw = rb == 32    ? CU_TENSOR_MAP_SWIZZLE_32B
                                  : rb == 64  ? CU_TENSOR_MAP_SWIZZLE_64B
                                  : rb == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                              : CU_TENSOR_MAP_SWIZZLE_NONE;
    const CUresult r = fn(map, sizeof(T) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2,
                          const_cast<void*>(p.X), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

template <typename K>
static cudaError_t launch_grid(K kern, int smem, const ObjParams& p, const CUtensorMap& tmap, int* nblocks,
                               cudaStream_t st) {
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
    kern<<<nb, kObjThreads, smem, st>>>(p, tmap);
    if (p.launched) *p.launched += 1;
    return cudaGetLastError();
}

// tensor-core screen kernel (objective_tc.cuh): persistent, one CTA per SM
template <int NP, int N, int KPS>
static cudaError_t launch_tc(const ObjParams& p, const CUtensorMap& tmap, int* nblocks, cudaStream_t st) {
    using TG = TcGeo<NP, N>;
    // the cost-only pass (no labels / counts) compiles without the output path: fewer live registers
    auto kern = (p.labels || p.counts) ? objective_tc_kernel<NP, N, KPS, true> : objective_tc_kernel<NP, N, KPS, false>;
    const int smem = objective_tc_smem<NP, N>(p.kv);
    // per device and instantiation: the opt-in shared-memory size (the largest asked so far) and the SM
    // count are set / read once -- this launch sits on the critical path of a ~0.13 ms pass
    static int smem_set[2][16] = {};
    static int sm_count[16] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    const int di = dev & 15, oi = (p.labels || p.counts) ? 1 : 0;
    cudaError_t e = cudaSuccess;
    if (smem_set[oi][di] < smem) {
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        smem_set[oi][di] = smem;
    }
    if (sm_count[di] == 0) {
        int v = 148;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        sm_count[di] = v;
    }
    const int sms = sm_count[di];
    if (nblocks[0] < sms) {
        nblocks[0] = sms;
        return cudaErrorNotReady;
    }
    nblocks[0] = sms;
    kern<<<sms, TG::THREADS, smem, st>>>(p, tmap);
    if (p.launched) *p.launched += 1;
    if (p.finalized) *p.finalized = p.cost_out ? 1 : 0;  // the last CTA wrote the fixed-order total
    return cudaGetLastError();
}

template <typename T, int NP>
static cudaError_t launch_obj_t(const ObjParams& p_in, int* nblocks, cudaStream_t st) {
    ObjParams p = p_in;
    CUtensorMap tmap;
    memset(&tmap, 0, sizeof tmap);
    static const bool old = getenv("HPCG_OBJ_OLD") != nullptr || getenv("HPCG_NO_TMA") != nullptr;
    static const bool no_tc = getenv("HPCG_OBJ_NO_TC") != nullptr;
    if constexpr (sizeof(T) == 4 && (NP == 8 || NP == 16 || NP == 32)) {  // tensor-core screen
        if (!old && !no_tc && p.kv >= 1 && p.kv <= 32 && tma_ok<T, NP>(p) && make_tmap<T>(p, TcGeo<NP, 16>::BOX, &tmap)) {
            p.use_tma = 1;
            switch ((p.kv + 1) / 2) {  // screened centre pairs
                case 1: return launch_tc<NP, 16, 1>(p, tmap, nblocks, st);
                case 2: return launch_tc<NP, 16, 2>(p, tmap, nblocks, st);
                case 3: return launch_tc<NP, 16, 3>(p, tmap, nblocks, st);
                case 4: return launch_tc<NP, 16, 4>(p, tmap, nblocks, st);
                case 5: return launch_tc<NP, 16, 5>(p, tmap, nblocks, st);
                case 6: return launch_tc<NP, 16, 6>(p, tmap, nblocks, st);
                case 7: return launch_tc<NP, 16, 7>(p, tmap, nblocks, st);
                case 8: return launch_tc<NP, 16, 8>(p, tmap, nblocks, st);
                default: return launch_tc<NP, 32, 16>(p, tmap, nblocks, st);
            }
        }
    }
    if constexpr (sizeof(T) == 4 && NP % 4 == 0 && NP != 24) {  // centre-pair kernel (fp32, TMA widths)
        if (!old && tma_ok<T, NP>(p) && make_tmap<T>(p, PairGeo<NP>::GR, &tmap)) {
            p.use_tma = 1;
            static const bool no_crec = getenv("HPCG_NO_CREC") != nullptr;
            if (!no_crec && p.rec_slot >= 0 && p.rec_slot < kRecSlots && p.rec_scratch &&
                p.kv <= 2 * kRecMaxPairs) {
                build_pair_records_kernel<NP><<<1, 64, 0, st>>>(p);
                cudaError_t e = cudaGetLastError();
                if (e != cudaSuccess) return e;
                if (p.launched) *p.launched += 1;
                const size_t bytes = (size_t)((p.kv + 1) / 2) * PairGeo<NP>::RST * sizeof(float2);
                e = cudaMemcpyToSymbolAsync(c_pair_rec4, p.rec_scratch, bytes,
                                            (size_t)p.rec_slot * kRecSlotF4 * sizeof(float4), cudaMemcpyDeviceToDevice,
                                            st);
                if (e != cudaSuccess) return e;
                return launch_grid(objective_pairs_kernel<NP, true>, objective_pairs_smem<NP>(p.kv), p, tmap,
                                   nblocks, st);
            }
            return launch_grid(objective_pairs_kernel<NP, false>, objective_pairs_smem<NP>(p.kv), p, tmap, nblocks,
                               st);
        }
    }
    // narrow rows (fp64 n <= 3, fp32 n = 2): bulk-copy ring + centre-pair screen
    static const bool no_rows = getenv("HPCG_OBJ_NO_ROWS") != nullptr;
    if constexpr ((sizeof(T) == 8 && NP <= 3) || (sizeof(T) == 4 && NP == 2)) {
        if (!old && !no_rows && p.n == NP && (reinterpret_cast<uintptr_t>(p.X) & 15) == 0) {
            static const bool no_grid = getenv("HPCG_OBJ_NO_GRID") != nullptr;
            if (p.grid && p.kv <= 32 && !no_grid) {  // cell filter: the masks, then the pass
                auto kern = objective_rows_kernel<T, NP, true>;
                const int smem = objective_rows_smem<T, NP, true>(p.kv);
                cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
                if (e != cudaSuccess) return e;
                int per_sm = 0, dev = 0, sms = 148;
                e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kObjThreads, smem);
                if (e != cudaSuccess) return e;
                cudaGetDevice(&dev);
                cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
                if (per_sm >= 1 && nblocks[0] >= sms * per_sm) {
                    grid_mask_kernel<NP><<<kGridCells / 256, 256, 0, st>>>(p);
                    e = cudaGetLastError();
                    if (e != cudaSuccess) return e;
                    if (p.launched) *p.launched += 1;
                }
                return launch_grid(kern, smem, p, tmap, nblocks, st);
            }
            return launch_grid(objective_rows_kernel<T, NP>, objective_rows_smem<T, NP>(p.kv), p, tmap, nblocks, st);
        }
    }
    p.use_tma = (!getenv("HPCG_NO_TMA") && tma_ok<T, NP>(p) && make_tmap<T>(p, ObjGeo<T, NP>::GR, &tmap)) ? 1 : 0;
    return launch_grid(objective_kernel<T, NP>, objective_smem<T, NP>(p.kv), p, tmap, nblocks, st);
}

// true when launch_objective takes a resident kernel for this shape, i.e. one that honours
// ObjParams::kv_dev (the grid-wide kernel needs the exact count on the host)
bool objective_device_kv(int dtype, int n, int kv) {
    static const bool force_wide = getenv("HPCG_WIDE") != nullptr;
    return pick_np(dtype, n) != 0 && kv <= kObjMaxK && !force_wide;
}

// wide fp32 rows (n = 64, 128) on the tensor cores (objective_tcw.cuh): TMA boxes of one
// 128-B swizzle atom ({32 floats, 128 rows}, SWIZZLE_128B)
template <int NA, int KPS>
static cudaError_t launch_tcw(const ObjParams& p, int* nblocks, cudaStream_t st) {
    using TG = TcwGeo<NA>;
    auto fn = encode_fn();
    if (!fn) return cudaErrorNotSupported;
    CUtensorMap tmap;
    memset(&tmap, 0, sizeof tmap);
    const cuuint64_t dims[2] = {(cuuint64_t)p.n, (cuuint64_t)p.m};
    const cuuint64_t strides[1] = {(cuuint64_t)p.n * 4};
    const cuuint32_t box[2] = {32, (cuuint32_t)TG::M};
    const cuuint32_t estr[2] = {1, 1};
    if (fn(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(p.X), dims, strides, box, estr,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return cudaErrorNotSupported;
    auto kern = objective_tcw_kernel<NA, KPS>;
    const int smem = objective_tcw_smem<NA>();
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (nblocks[0] < sms) {
        nblocks[0] = sms;
        return cudaErrorNotReady;
    }
    nblocks[0] = sms;
    kern<<<sms, TG::THREADS, smem, st>>>(p, tmap);
    if (p.launched) *p.launched += 1;
    return cudaGetLastError();
}

cudaError_t launch_objective(int dtype, const ObjParams& p, int* nblocks, cudaStream_t st) {
    if (p.finalized) *p.finalized = 0;  // set by the launchers whose kernel sums its own blocks
    const int np = pick_np(dtype, p.n);
    static const bool force_wide = getenv("HPCG_WIDE") != nullptr;
    static const bool no_tc = getenv("HPCG_OBJ_NO_TC") != nullptr;
    if (dtype == 0 && (p.n == 64 || p.n == 128) && p.kv >= 1 && p.kv <= 32 && !force_wide && !no_tc &&
        (reinterpret_cast<uintptr_t>(p.X) & 15) == 0) {
        if (p.n == 128) return p.kv <= 16 ? launch_tcw<4, 8>(p, nblocks, st) : launch_tcw<4, 16>(p, nblocks, st);
        return p.kv <= 16 ? launch_tcw<2, 8>(p, nblocks, st) : launch_tcw<2, 16>(p, nblocks, st);
    }
    if (np == 0 || p.kv > kObjMaxK || force_wide) {
        const cudaError_t e = launch_objective_wide(dtype, p, nblocks, st);
        if (p.launched) *p.launched += 1;
        return e;
    }
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
