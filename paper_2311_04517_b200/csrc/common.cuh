// Shared device helpers for the HPClust B200 kernels (sm_100a only).
#pragma once
#include <cstdint>
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

HPCG_DEV u32x4 philox4x32(u32x4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = u32x4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return c;
}

// 53-bit unit double in [0,1) from a counter, like rng.hpp:38-40 but Philox-keyed.
HPCG_DEV double philox_unit(uint64_t key, uint32_t a, uint32_t b, uint32_t c) {
    u32x4 r = philox4x32(u32x4{a, b, c, 0x68706367u}, (uint32_t)key, (uint32_t)(key >> 32));
    const uint64_t v = ((uint64_t)r.x << 32) | r.y;
    return (double)(v >> 11) * 0x1.0p-53;
}

// Uniform integer in [0, n) (n <= 2^40 in practice): 64x64 high product.
HPCG_DEV uint64_t philox_index(uint64_t key, uint32_t a, uint32_t b, uint32_t c, uint64_t n) {
    u32x4 r = philox4x32(u32x4{a, b, c, 0x69647831u}, (uint32_t)key, (uint32_t)(key >> 32));
    const uint64_t v = ((uint64_t)r.x << 32) | r.y;
    return __umul64hi(v, n);
}

// ------------------------------------------------------ sample-index permutation
// s distinct rows of [0, m) in "draw order": a keyed pseudo-random permutation of
// [0, 2^bits) (4-round Feistel over Philox-derived round keys) with cycle walking
// back into [0, m). Distinctness is by construction (bijection), replacing the
// reference's O(m) partial Fisher-Yates (engine.hpp:165-177) with O(1) per draw.
struct FeistelPRP {
    uint64_t m;
    uint32_t half_bits, half_mask;
    uint32_t rk[4];

    HPCG_DEV static FeistelPRP make(uint64_t key, uint32_t round, uint32_t worker, uint64_t m) {
        FeistelPRP p;
        p.m = m;
        int bits = 64 - __clzll((long long)(m > 1 ? m - 1 : 1));
        bits = bits < 2 ? 2 : bits;
        bits += bits & 1;
        p.half_bits = (uint32_t)bits / 2;
        p.half_mask = (1u << p.half_bits) - 1u;
        u32x4 r = philox4x32(u32x4{round, worker, 0x50525031u, 0x50525032u}, (uint32_t)key, (uint32_t)(key >> 32));
        p.rk[0] = r.x;
        p.rk[1] = r.y;
        p.rk[2] = r.z;
        p.rk[3] = r.w;
        return p;
    }
    HPCG_DEV uint64_t permute_once(uint64_t v) const {
        uint32_t L = (uint32_t)(v >> half_bits) & half_mask, R = (uint32_t)v & half_mask;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            uint32_t f = R * 0x9E3779B1u ^ rk[i];
            f ^= f >> 15;
            f *= 0x85EBCA77u;
            f ^= f >> 13;
            const uint32_t nl = R;
            R = (L ^ f) & half_mask;
            L = nl;
        }
        return ((uint64_t)L << half_bits) | R;
    }
    HPCG_DEV uint64_t operator()(uint64_t i) const {
        uint64_t v = permute_once(i);
        while (v >= m) v = permute_once(v);  // cycle walking: expected < 4 steps
        return v;
    }
};

// ------------------------------------------------------------------ reductions
HPCG_DEV double warp_sum(double v) {
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
