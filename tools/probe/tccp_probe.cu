// Probe: tcgen05.cp.128x256b (shared -> TMEM) from a K-major swizzled tile (the TMA / UMMA layout
// of the f(C,X) stages), read back with tcgen05.ld 32x32b: is row r, floats [8h, 8h+8) landed in
// TMEM lane r, columns [8h, 8h+8) when the descriptor start advances by 32 B per h?
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

template <int NP> struct L {
    static constexpr int RS = NP * 4, CPR = RS / 16;
    __host__ __device__ static int swz(int r) { return CPR == 8 ? (r & 7) : CPR == 4 ? ((r >> 1) & 3) : CPR == 2 ? ((r >> 2) & 1) : 0; }
    __host__ __device__ static int off(int r, int d) { return r * NP + (((d / 4) ^ swz(r)) * 4) + (d % 4); }
    static constexpr uint32_t layout = CPR == 8 ? 2u : CPR == 4 ? 4u : CPR == 2 ? 6u : 0u;
};
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t sbo_bytes, uint32_t layout) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)layout << 61;
    return d;
}

template <int NP>
__global__ void cp_kernel(const float* A, float* D, long long* cyc) {
    using G = L<NP>;
    __shared__ __align__(1024) float sa[128 * NP];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int e = tid; e < 128 * NP; e += blockDim.x) sa[G::off(e / NP, e % NP)] = A[e];
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tbase)), "r"(64));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = tbase;
    if (tid == 0) {
        long long t0 = clock64();
        for (int h = 0; h < NP / 8; ++h) {
            const uint64_t d = sdesc(su32(sa) + h * 32, 8 * G::RS, G::layout);
            asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(tm + 8 * h), "l"(d) : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
        cyc[0] = clock64() - t0;
    }
    asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W_%=;\n}\n" ::"r"(su32(&bar)) : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp < 4) {
        for (int c0 = 0; c0 < NP; c0 += 8) {
            uint32_t v[8];
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                         : "r"(tm + ((uint32_t)(32 * warp) << 16) + (uint32_t)c0));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            for (int j = 0; j < 8; ++j) D[(32 * warp + lane) * NP + c0 + j] = __uint_as_float(v[j]);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(64));
}

template <int NP>
int run() {
    std::vector<float> A(128 * NP), D(128 * NP);
    for (int i = 0; i < 128 * NP; ++i) A[i] = (float)i + 0.25f;
    float *dA, *dD;
    long long* dc;
    CK(cudaMalloc(&dA, A.size() * 4)); CK(cudaMalloc(&dD, D.size() * 4)); CK(cudaMalloc(&dc, 8));
    CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemset(dD, 0, D.size() * 4));
    cp_kernel<NP><<<1, 256>>>(dA, dD, dc);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
    long long cy; CK(cudaMemcpy(&cy, dc, 8, cudaMemcpyDeviceToHost));
    int bad = 0;
    for (int i = 0; i < 128 * NP; ++i)
        if (D[i] != A[i]) { if (bad < 6) printf("  NP=%d mismatch at row %d col %d: got %g want %g\n", NP, i / NP, i % NP, D[i], A[i]); ++bad; }
    printf("NP=%d: %s (bad %d), issue %lld cyc\n", NP, bad ? "FAIL" : "ok", bad, cy);
    return bad != 0;
}

int main() { return run<8>() | run<16>() | run<32>(); }
