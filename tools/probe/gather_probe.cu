// Micro-probe: gather R random 64-B rows (fp32 x 16) per CTA into shared memory, one
// 512-thread CTA per SM on every SM, the worker-step gather's shape. Variants:
//   A  cp.async 16 B per lane, chunk-major (the current step kernel)
//   B  cp.async.bulk 64 B per row (1-D bulk copy, one thread per row, mbarrier)
//   C  cp.async.bulk.tensor 2-D tile::gather4 (4 rows per instruction, 64B swizzle)
//   D  ld.global.nc.v4 register staging + st.shared (8 rows in flight per thread)
// Prints per-CTA cycles (median) and the kernel time.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda.h>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

constexpr int NT = 512, NP = 16;
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ int swz(int row) { return (row >> 1) & 3; }

__device__ __forceinline__ void mbar_init(uint64_t* b, int c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
    asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" ::"r"(su32(b)), "r"(ph) : "memory");
}

__global__ void __launch_bounds__(NT, 1) kA(const float* X, const int* idx, int R, long long* cyc, float* sink) {
    extern __shared__ __align__(1024) float sm[];
    const long long t0 = clock64();
    const int* id = idx + (size_t)blockIdx.x * R;
    for (int e = threadIdx.x; e < R * 4; e += NT) {
        const int li = e >> 2, q = e & 3;
        const uint32_t d = su32(sm + li * NP + ((q ^ swz(li)) * 4));
        const float* s = X + (size_t)id[li] * NP + q * 4;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(s) : "memory");
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) { cyc[blockIdx.x] = clock64() - t0; sink[blockIdx.x] = sm[threadIdx.x * 7 % (R * NP)]; }
}

__global__ void __launch_bounds__(NT, 1) kB(const float* X, const int* idx, int R, long long* cyc, float* sink) {
    extern __shared__ __align__(1024) float sm[];
    __shared__ uint64_t bar;
    const long long t0 = clock64();
    if (threadIdx.x == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    __syncthreads();
    if (threadIdx.x == 0) mbar_expect(&bar, (uint32_t)(R * 64));
    const int* id = idx + (size_t)blockIdx.x * R;
    for (int li = threadIdx.x; li < R; li += NT) {
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 64, [%2];" ::"r"(su32(sm + li * NP)),
                     "l"(X + (size_t)id[li] * NP), "r"(su32(&bar)) : "memory");
    }
    mbar_wait(&bar, 0);
    if (threadIdx.x == 0) { cyc[blockIdx.x] = clock64() - t0; sink[blockIdx.x] = sm[threadIdx.x * 7 % (R * NP)]; }
}

__global__ void __launch_bounds__(NT, 1) kC(const __grid_constant__ CUtensorMap map, const int* idx, int R, long long* cyc, float* sink) {
    extern __shared__ __align__(1024) float sm[];
    __shared__ uint64_t bar;
    const long long t0 = clock64();
    if (threadIdx.x == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    __syncthreads();
    if (threadIdx.x == 0) mbar_expect(&bar, (uint32_t)(R * 64));
    const int* id = idx + (size_t)blockIdx.x * R;
    for (int g = threadIdx.x; g * 4 < R; g += NT) {
        const int r0 = id[4 * g], r1 = id[4 * g + 1], r2 = id[4 * g + 2], r3 = id[4 * g + 3];
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(su32(sm + g * 4 * NP)),
                     "l"(&map), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(su32(&bar)) : "memory");
    }
    mbar_wait(&bar, 0);
    if (threadIdx.x == 0) { cyc[blockIdx.x] = clock64() - t0; sink[blockIdx.x] = sm[threadIdx.x * 7 % (R * NP)]; }
}

// E: rows [0, R/2) by cp.async (LSU path), rows [R/2, R) by cp.async.bulk (TMA path)
__global__ void __launch_bounds__(NT, 1) kE(const float* X, const int* idx, int R, long long* cyc, float* sink) {
    extern __shared__ __align__(1024) float sm[];
    __shared__ uint64_t bar;
    const long long t0 = clock64();
    const int h = (R / 2) & ~3;
    if (threadIdx.x == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    __syncthreads();
    if (threadIdx.x == 0) mbar_expect(&bar, (uint32_t)((R - h) * 64));
    const int* id = idx + (size_t)blockIdx.x * R;
    for (int li = h + threadIdx.x; li < R; li += NT)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 64, [%2];" ::"r"(su32(sm + li * NP)),
                     "l"(X + (size_t)id[li] * NP), "r"(su32(&bar)) : "memory");
    for (int e = threadIdx.x; e < h * 4; e += NT) {
        const int li = e >> 2, q = e & 3;
        const uint32_t d = su32(sm + li * NP + ((q ^ swz(li)) * 4));
        const float* s = X + (size_t)id[li] * NP + q * 4;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(s) : "memory");
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    mbar_wait(&bar, 0);
    __syncthreads();
    if (threadIdx.x == 0) { cyc[blockIdx.x] = clock64() - t0; sink[blockIdx.x] = sm[threadIdx.x * 7 % (R * NP)]; }
}

__global__ void flush_l2(float* buf, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) buf[i] += 1.0f;
}

__global__ void __launch_bounds__(NT, 1) kD(const float* X, const int* idx, int R, long long* cyc, float* sink) {
    extern __shared__ __align__(1024) float sm[];
    const long long t0 = clock64();
    const int* id = idx + (size_t)blockIdx.x * R;
    constexpr int U = 8;
    for (int e0 = threadIdx.x; e0 < R * 4; e0 += NT * U) {
        float4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int e = e0 + u * NT;
            if (e < R * 4) {
                const int li = e >> 2, q = e & 3;
                v[u] = __ldg(reinterpret_cast<const float4*>(X + (size_t)id[li] * NP + q * 4));
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int e = e0 + u * NT;
            if (e < R * 4) {
                const int li = e >> 2, q = e & 3;
                *reinterpret_cast<float4*>(sm + li * NP + ((q ^ swz(li)) * 4)) = v[u];
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) { cyc[blockIdx.x] = clock64() - t0; sink[blockIdx.x] = sm[threadIdx.x * 7 % (R * NP)]; }
}

int main(int argc, char** argv) {
    const long long M = 10000000;
    const int R = argc > 1 ? atoi(argv[1]) : 2224;  // multiple of 4
    int sms = 0; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const int grid = sms;
    float* X; int* idx; long long* cyc; float* sink;
    CK(cudaMalloc(&X, M * NP * 4)); CK(cudaMemset(X, 0, M * NP * 4));
    std::vector<int> h((size_t)grid * R); std::mt19937_64 g(1);
    for (auto& v : h) v = (int)(g() % M);
    CK(cudaMalloc(&idx, h.size() * 4)); CK(cudaMemcpy(idx, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMalloc(&cyc, grid * 8)); CK(cudaMalloc(&sink, grid * 4));
    const int smem = R * 64;
    CK(cudaFuncSetAttribute(kA, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    CK(cudaFuncSetAttribute(kB, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    CK(cudaFuncSetAttribute(kC, cudaFuncAttributeMaxDynamicSharedMemorySize, smem + 1024));
    CK(cudaFuncSetAttribute(kD, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    CK(cudaFuncSetAttribute(kE, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const size_t FL = (size_t)256 << 20;  // 1 GB of floats: larger than L2
    float* fbuf; CK(cudaMalloc(&fbuf, FL * 4)); CK(cudaMemset(fbuf, 0, FL * 4));
    bool cold = false;
    CUtensorMap map; memset(&map, 0, sizeof map);
    bool have_map = false;
    {
        void* f = nullptr; cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess && f) {
            auto fn = reinterpret_cast<CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                                                    const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill)>(f);
            const cuuint64_t dims[2] = {NP, (cuuint64_t)M};
            const cuuint64_t str[1] = {NP * 4};
            const cuuint32_t box[2] = {NP, 1};
            const cuuint32_t es[2] = {1, 1};
            CUresult r = fn(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, X, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            have_map = r == CUDA_SUCCESS;
            printf("tensor map encode: %d\n", (int)r);
        }
    }
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    std::vector<long long> hc(grid);
    auto run = [&](const char* nm, auto launch) {
        for (int w = 0; w < 3; ++w) launch();
        CK(cudaDeviceSynchronize());
        float best = 1e9f;
        for (int rep = 0; rep < 10; ++rep) {
            if (cold) flush_l2<<<1184, 512>>>(fbuf, FL);
            cudaEventRecord(e0); launch(); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
            float ms; cudaEventElapsedTime(&ms, e0, e1); best = std::min(best, ms);
        }
        CK(cudaMemcpy(hc.data(), cyc, grid * 8, cudaMemcpyDeviceToHost));
        std::sort(hc.begin(), hc.end());
        const double bytes = (double)grid * R * 64;
        printf("%-28s kernel %7.2f us  CTA cycles median %7lld max %7lld  %6.0f GB/s %s\n", nm, best * 1e3, hc[grid / 2], hc[grid - 1],
               bytes / (best * 1e-3) / 1e9, cold ? "cold" : "warm");
    };
  for (int c = 0; c < 2; ++c) {
    cold = c == 1;
    run("A cp.async 16B", [&] { kA<<<grid, NT, smem>>>(X, idx, R, cyc, sink); });
    run("E half cp.async half bulk", [&] { kE<<<grid, NT, smem>>>(X, idx, R, cyc, sink); });
    run("B cp.async.bulk 64B/row", [&] { kB<<<grid, NT, smem>>>(X, idx, R, cyc, sink); });
    run("D ldg.v4 x8 + sts", [&] { kD<<<grid, NT, smem>>>(X, idx, R, cyc, sink); });
    if (have_map && (argc < 3 || atoi(argv[2]) != 0)) run("C tensor gather4 (64B swz)", [&] { kC<<<grid, NT, smem + 1024>>>(map, idx, R, cyc, sink); });
  }
    CK(cudaGetLastError());
    return 0;
}
