// Shared device helpers for the HPClust B200 kernels (sm_100a only).
#pragma once
#include <cstdint>
#include <cmath>
#include <cuda_runtime.h>
#include <cooperative_groups.h>

namespace hpcg {
namespace cg = cooperative_groups;

#define HPCG_DEV __device__ __forceinline__

// ---------------------------------------------------------------- Philox4x32-10
// Counter-based RNG (Salmon et al., SC'11). Used for product-mode sample indices
// (via the Feistel PRP below) and K-means++ draws; the reference's mt19937_64
// stream is replayed on the host instead when bit-parity with the reference run
// is requested (see runtime.cpp, RngMode::reference).
struct u32x4 {
    uint32_t x, y, z, w;
};

#define HPCG_HD __host__ __device__ __forceinline__
HPCG_HD uint32_t hd_umulhi(uint32_t a, uint32_t b) {
#ifdef __CUDA_ARCH__
    return __umulhi(a, b);
#else
    return (uint32_t)(((uint64_t)a * b) >> 32);
#endif
}
HPCG_HD uint64_t hd_umul64hi(uint64_t a, uint64_t b) {
#ifdef __CUDA_ARCH__
    return __umul64hi(a, b);
#else
    return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}

// Host and device: the host replays a PHILOX round's draws for parity tests (hpcg_philox_seed_draws).
HPCG_HD u32x4 philox4x32(u32x4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = hd_umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = hd_umulhi(0xCD9E8D57u, c.z);
        c = u32x4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return c;
}

// 53-bit unit double in [0,1) from a counter, like rng.hpp:38-40 but Philox-keyed.
HPCG_HD double philox_unit(uint64_t key, uint32_t a, uint32_t b, uint32_t c) {
    u32x4 r = philox4x32(u32x4{a, b, c, 0x68706367u}, (uint32_t)key, (uint32_t)(key >> 32));
    const uint64_t v = ((uint64_t)r.x << 32) | r.y;
    return (double)(v >> 11) * 0x1.0p-53;
}

// Uniform integer in [0, n) (n <= 2^40 in practice): 64x64 high product.
HPCG_HD uint64_t philox_index(uint64_t key, uint32_t a, uint32_t b, uint32_t c, uint64_t n) {
    u32x4 r = philox4x32(u32x4{a, b, c, 0x69647831u}, (uint32_t)key, (uint32_t)(key >> 32));
    const uint64_t v = ((uint64_t)r.x << 32) | r.y;
    return hd_umul64hi(v, n);
}

// ------------------------------------------------------ sample-index permutation
// s distinct rows of [0, m) in "draw order": a keyed pseudo-random permutation of [0, a*b)
// with a = ceil(sqrt(m)), b = ceil(m / a) — a 4-round Feistel network over Z_a x Z_b with
// modular addition (the halves alternate between the two moduli, so every round is a
// bijection) — and cycle walking back into [0, m), which a*b - m < a makes rare (< 1/b).
// Distinctness is by construction (bijection), replacing the reference's O(m) partial
// Fisher-Yates (engine.hpp:165-177) with O(1) work per draw and no divergent walks.
struct SamplePRP {
    uint64_t m;
    uint32_t a, b;
    float inv_b;
    uint32_t rk[4];

    // host side: the moduli depend on m only (StepParams carries them)
    static inline void moduli(uint64_t m, uint32_t& a, uint32_t& b, float& inv_b) {
        m = m > 0 ? m : 1;
        uint64_t r = (uint64_t)sqrt((double)m);
        while (r * r < m) ++r;
        while (r > 1 && (r - 1) * (r - 1) >= m) --r;
        a = (uint32_t)r;
        b = (uint32_t)((m + r - 1) / r);
        inv_b = 1.0f / (float)b;
    }
    HPCG_DEV static SamplePRP make(uint64_t key, uint32_t round, uint32_t worker, uint64_t m, uint32_t a, uint32_t b,
                                   float inv_b) {
        SamplePRP p;
        p.m = m > 0 ? m : 1;
        p.a = a;
        p.b = b;
        p.inv_b = inv_b;
        u32x4 r = philox4x32(u32x4{round, worker, 0x50525031u, 0x50525032u}, (uint32_t)key, (uint32_t)(key >> 32));
        p.rk[0] = r.x;
        p.rk[1] = r.y;
        p.rk[2] = r.z;
        p.rk[3] = r.w;
        return p;
    }
    HPCG_DEV uint64_t permute_once(uint64_t x) const {
        // x = L*b + R, L in Z_a, R in Z_b (fp32 quotient estimate, exact after one correction
        // each way: a*b <= 2^42 keeps the estimate within +-1 of floor(x/b))
        uint64_t Lq = (uint64_t)((float)x * inv_b);
        if (Lq * b > x) --Lq;
        if (x - Lq * b >= b) ++Lq;
        uint32_t L = (uint32_t)Lq, R = (uint32_t)(x - Lq * b);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const uint32_t mod = (i & 1) ? b : a;  // L lives in Z_mod
            uint32_t f = R * 0x9E3779B1u ^ rk[i];
            f ^= f >> 15;
            f *= 0x85EBCA77u;
            f ^= f >> 13;
            uint32_t t = L + __umulhi(f, mod);  // F(R) in [0, mod)
            if (t >= mod) t -= mod;
            L = R;
            R = t;
        }
        return (uint64_t)L * b + R;  // L in Z_a, R in Z_b again after an even round count
    }
    HPCG_DEV uint64_t operator()(uint64_t i) const {
        uint64_t v = permute_once(i);
        while (v >= m) v = permute_once(v);  // cycle walking: P(step) < 1/b
        return v;
    }
};

// ------------------------------------------------------------------ reductions
HPCG_DEV double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
HPCG_DEV float warp_sum_f(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// parallel.hpp:106-112 chunk_range, the partition every reference reduction uses.
__host__ __device__ inline void chunk_range(int64_t rows, int64_t n_chunks, int64_t chunk, int64_t& b, int64_t& e) {
    const int64_t base = rows / n_chunks, extra = rows % n_chunks;
    b = chunk * base + (chunk < extra ? chunk : extra);
    e = b + base + (chunk < extra ? 1 : 0);
}

// Exact reference distance (core.hpp:147-152): ascending d, separately rounded
// sub, mul and add — the __d*_rn intrinsics forbid contraction into DFMA.
template <typename T>
HPCG_DEV double ref_sqdist(const T* x, const double* c, int n) {
    double acc = 0.0;
    for (int d = 0; d < n; ++d) {
        const double diff = __dsub_rn((double)x[d], c[d]);
        acc = __dadd_rn(acc, __dmul_rn(diff, diff));
    }
    return acc;
}

}  // namespace hpcg
