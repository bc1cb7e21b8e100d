// Probe: tcgen05 kind::tf32 MMA over the worker-step sample layout (K-major rows of
// NP fp32 with the 16-B-chunk XOR swizzle = SWIZZLE_{32,64,128}B), D in TMEM read back with
// tcgen05.ld 32x32b. Checks the descriptors/lane mapping against host dot products.
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cmath>
#include <vector>
#include <random>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

template <int NP> struct L {
    static constexpr int RS = NP * 4, CPR = RS / 16;
    __host__ __device__ static int swz(int r) { return CPR == 8 ? (r & 7) : CPR == 4 ? ((r >> 1) & 3) : CPR == 2 ? ((r >> 2) & 1) : 0; }
    __host__ __device__ static int off(int r, int d) { return r * NP + (((d / 4) ^ swz(r)) * 4) + (d % 4); }
    static constexpr uint32_t layout = CPR == 8 ? 2u : CPR == 4 ? 4u : CPR == 2 ? 6u : 0u;  // SW128 / SW64 / SW32
};

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t sbo_bytes, uint32_t layout) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;                          // LBO (ignored for swizzled K-major)
    d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;                          // version 1 (sm100)
    d |= (uint64_t)layout << 61;
    return d;
}

template <int NP, int N>
__global__ void tc_kernel(const float* A, const float* B, int R, float* D, long long* cyc, int REPS) {
    using G = L<NP>;
    extern __shared__ __align__(1024) unsigned char smraw[];
    unsigned char* sm = smraw + ((1024 - (su32(smraw) & 1023)) & 1023);
    float* sa = reinterpret_cast<float*>(sm);
    float* sb = reinterpret_cast<float*>(sm + R * G::RS);
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int e = tid; e < R * NP; e += blockDim.x) sa[G::off(e / NP, e % NP)] = A[e];
    for (int e = tid; e < N * NP; e += blockDim.x) sb[G::off(e / NP, e % NP)] = B[e];
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tbase)), "r"(512));
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
    const int tiles = R / 128;
    constexpr uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    long long t0 = clock64();
    if (tid == 0) {
        for (int rep = 0; rep < REPS; ++rep)
        for (int t = 0; t < tiles; ++t)
            for (int ks = 0; ks < NP / 8; ++ks) {
                const uint64_t ad = sdesc(su32(sa) + t * 128 * G::RS + ks * 32, 8 * G::RS, G::layout);
                const uint64_t bd = sdesc(su32(sb) + ks * 32, 8 * G::RS, G::layout);
                asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                             " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, {%5, %5, %5, %5}, p;\n}\n" ::"r"(tm + t * N),
                             "l"(ad), "l"(bd), "r"(idesc), "r"(ks), "r"(0u));
            }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
        const long long t1 = clock64();
        if (cyc) cyc[0] = t1 - t0;
    }
    asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W_%=;\n}\n" ::"r"(su32(&bar)) : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (tid == 0 && cyc) cyc[1] = clock64() - t0;
    for (int u = warp; u < tiles * 4; u += blockDim.x / 32) {
        if ((u & 3) != (warp & 3)) continue;  // a warp reads only its TMEM lane quarter
        const int t = u >> 2, q = u & 3;
        uint32_t v[16];
        for (int c0 = 0; c0 < N; c0 += 16) {
            const uint32_t addr = tm + ((uint32_t)(32 * q) << 16) + (uint32_t)(t * N + c0);
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                         : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                           "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                         : "r"(addr));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            const int row = t * 128 + 32 * q + lane;
            for (int j = 0; j < 16; ++j) D[row * N + c0 + j] = __uint_as_float(v[j]);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(512));
}

template <int NP, int N>
int run(bool integers) {
    const int R = 2304;
    std::vector<float> A(R * NP), B(N * NP), D(R * N);
    std::mt19937 g(NP * 7 + N);
    std::uniform_real_distribution<float> u(-10.f, 10.f);
    for (auto& v : A) v = integers ? (float)(int)(g() % 17) - 8.f : u(g);
    for (auto& v : B) v = integers ? (float)(int)(g() % 9) - 4.f : u(g);
    float *dA, *dB, *dD;
    CK(cudaMalloc(&dA, A.size() * 4)); CK(cudaMalloc(&dB, B.size() * 4)); CK(cudaMalloc(&dD, D.size() * 4));
    CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemset(dD, 0xff, D.size() * 4));
    const int smem = R * NP * 4 + N * NP * 4 + 1024;
    CK(cudaFuncSetAttribute(tc_kernel<NP, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    long long* dc; CK(cudaMalloc(&dc, 16));
    tc_kernel<NP, N><<<1, 512, smem>>>(dA, dB, R, dD, dc, 1);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
    double maxrel = 0; int bad = 0;
    for (int r = 0; r < R; ++r)
        for (int j = 0; j < N; ++j) {
            double ref = 0, mag = 0;
            for (int d = 0; d < NP; ++d) { ref += (double)A[r * NP + d] * B[j * NP + d]; mag += fabs((double)A[r * NP + d] * B[j * NP + d]); }
            const double err = fabs(D[r * N + j] - ref);
            if (integers ? err != 0 : err > 4e-3 * mag) { if (bad < 5) printf("  mismatch r=%d j=%d got %g want %g\n", r, j, D[r * N + j], ref); ++bad; }
            if (mag > 0) maxrel = fmax(maxrel, err / mag);
        }
    printf("NP=%d N=%d %s: %s (bad %d, max err/sum|ab| %.3g)\n", NP, N, integers ? "ints" : "reals", bad ? "FAIL" : "ok", bad, maxrel);
    for (int reps : {1, 4, 16}) {
        tc_kernel<NP, N><<<1, 512, smem>>>(dA, dB, R, dD, dc, reps);
        CK(cudaDeviceSynchronize());
        long long hc[2]; CK(cudaMemcpy(hc, dc, 16, cudaMemcpyDeviceToHost));
        const int nm = reps * (R / 128) * (NP / 8);
        printf("   reps %2d: %4d MMAs issue %6lld cyc (%.1f/MMA), complete %6lld cyc (%.1f/MMA)\n", reps, nm, hc[0], (double)hc[0] / nm, hc[1], (double)hc[1] / nm);
    }
    return bad != 0;
}

int main() {
    int f = 0;
    f |= run<16, 16>(true); f |= run<16, 16>(false);
    f |= run<16, 32>(true); f |= run<16, 32>(false);
    f |= run<32, 16>(true); f |= run<32, 16>(false);
    f |= run<8, 16>(true);  f |= run<8, 16>(false);
    return f;
}
