// Full-data objective f(C, X) (engine.hpp:197-229, core.hpp:224-233) for WIDE fp32 rows (n = 64 or
// 128: BASELINE config 4) with the nearest-centre screen on the tensor cores -- the s x n x k
// contraction the north star assigns to tcgen05.
//
// Same pipeline as objective_tc_kernel (csrc/objective_tc.cuh), adapted to rows wider than one
// 128-B swizzle atom: a row is NA = n/32 K-atoms, so a 128-row tile lands by NA TMA box loads
// ({32 floats, 128 rows}, SWIZZLE_128B) into NA sub-tiles [128 rows x 128 B], and the MMA warp
// walks K in 8-float steps across the atoms (start address + 16 KB per atom + 32 B per step);
// -2c (tf32) is the B operand in the same layout, N = 32 centre columns, D in TMEM. The epilogue
// (8 warps, 2 groups alternating tiles, one row per thread) cannot hold a 128-float row in
// registers: it streams the row's chunks from the stage once, accumulating |x|^2 and the fp64
// cost to the screened nearest centre together; a row inside the tf32 bound is re-screened in
// fp32 (FFMA2) and, if still inside that bound, given the exact fp64 argmin (warp-parallel over
// centres), and its cost is recomputed if the label moved. The stage is released after its rows
// have been read. fp64 centres and fp32 records are read from global memory (L1-resident).
#pragma once
#include "objective_tc.cuh"

namespace hpcg {

template <int NA>
struct TcwGeo {
    static constexpr int N = 32;                          // centre columns (kv <= 32)
    static constexpr int M = 128;                         // rows per tile
    static constexpr int NPW = 32 * NA;                   // row width (floats)
    static constexpr int SUB = M * 128;                   // bytes per K-atom sub-tile
    static constexpr int TILE = NA * SUB;                 // bytes per stage
    static constexpr int BSUB = N * 128;                  // bytes per K-atom of the B tile
    static constexpr int CEN = N * NPW * 4;               // bytes of the fp32 low-part centre table
    // ring stages in what is left of 224 KB after the B tile and the low-part table
    static constexpr int STAGES = (229376 - NA * BSUB - CEN) / TILE < 6 ? (229376 - NA * BSUB - CEN) / TILE : 6;
    static constexpr int TCOLS = 512;
    static constexpr int NB = TCOLS / N;                  // TMEM tile buffers
    static constexpr int EPI_WARPS = 8;
    static constexpr int THREADS = (EPI_WARPS + 2) * 32;
    static constexpr uint32_t IDESC =
        (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    static_assert(STAGES >= 2, "stages");
};

template <int NA>
__host__ __device__ inline int objective_tcw_smem() {
    using TG = TcwGeo<NA>;
    return 1024 + TG::STAGES * TG::TILE + NA * TG::BSUB + TG::CEN;  // + fp32 low parts (fp32-mode cost)
}

// fp32 low-part table of the row cost: chunk-major [NPW/4][N][4], so 32 lanes reading chunk c of 32
// different centres touch 32 distinct 16-B slots of one 512-B span (no bank conflicts)
template <int N>
HPCG_DEV int cen_off(int j, int d) { return (((d >> 2) * N + j) << 2) + (d & 3); }

// byte offset of float d of row r inside a tile of NA [rows x 128 B] SWIZZLE_128B atoms
HPCG_DEV uint32_t sw128_off(int rows, int r, int d) {
    const int a = d >> 5, q = (d >> 2) & 7;
    return (uint32_t)(a * rows * 128 + r * 128 + ((q ^ (r & 7)) << 4) + ((d & 3) << 2));
}

template <int NA, int KPS>
__global__ void __launch_bounds__(TcwGeo<NA>::THREADS, 1)
    objective_tcw_kernel(const ObjParams p, const __grid_constant__ CUtensorMap tmap) {
    using TG = TcwGeo<NA>;
    constexpr int N = TG::N, NPW = TG::NPW, STAGES = TG::STAGES, NB = TG::NB, TILE = TG::TILE, EW = TG::EPI_WARPS;
    extern __shared__ __align__(16) unsigned char osm[];
    unsigned char* ring = osm + ((1024 - (smem_u32(osm) & 1023)) & 1023);
    unsigned char* Bt = ring + STAGES * TILE;
    __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES], tfull[NB], tempty[NB];
    __shared__ uint32_t s_tmem;
    __shared__ __align__(8) float s_cc[N];
    __shared__ double s_wcost[EW];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int kv = obj_kv(p);
    const double* __restrict__ Cg = p.C;  // [kv x NPW] fp64 centres (L1-resident)
    const int64_t m = p.m;
    const int64_t ntiles = (m + TG::M - 1) / TG::M;
    const int my = (int64_t)blockIdx.x < ntiles ? (int)((ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x) : 0;
    // the producer thread initialises the barriers and puts the first ring of tiles in flight before the
    // centre tables are built: the prologue overlaps the first HBM round trip (as in objective_tc.cuh)
    const int pre = my < STAGES ? my : STAGES;
    if (warp == EW && lane == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 4);  // the 4 warps of the group that read the tile's rows
        }
        for (int b = 0; b < NB; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], 4);
        }
        mbar_init_fence();
        fence_proxy_async();
        for (int i = 0; i < pre; ++i) {
            mbar_expect_tx(&full[i], (uint32_t)TILE);
            const int row0 = (int)(((int64_t)blockIdx.x + (int64_t)i * gridDim.x) * TG::M);
#pragma unroll
            for (int a = 0; a < NA; ++a) tma_load_2d(ring + i * TILE + a * TG::SUB, &tmap, 32 * a, row0, &full[i]);
        }
    }

    // -c for the fp32-mode row cost as hi + lo: hi = B / 2 (exact: the tf32 -2c of the MMA operand,
    // read from the B tile), lo = fl32(-c - hi) (|lo| <= 2^-11 |c|, so hi + lo is -c to 2^-35 |c|)
    float* neglo = reinterpret_cast<float*>(Bt + NA * TG::BSUB);
    for (int e = tid; e < N * NPW; e += TG::THREADS) {
        const int j = e / NPW, d = e - j * NPW;
        const double c = j < kv ? Cg[(int64_t)j * NPW + d] : 0.0;
        const float b = tf32_rna((float)(-2.0 * c));
        *reinterpret_cast<float*>(Bt + sw128_off(N, j, d)) = b;
        neglo[cen_off<N>(j, d)] = (float)(-c - 0.5 * (double)b);
    }
    if (tid < N) {
        float cc = 1e38f;
        if (tid < kv) {
            double s = 0.0;
            for (int d = 0; d < NPW; ++d) {
                const double c = Cg[(int64_t)tid * NPW + d];
                s += c * c;
            }
            cc = (float)s;
        }
        s_cc[tid] = cc;
    }
    if (warp == EW + 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                     "r"(TG::TCOLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tm = s_tmem;
    double cost = 0.0;

    if (warp == EW) {  // ---- TMA producer: NA box loads per tile
        if (lane == 0) {
            int s = pre == STAGES ? 0 : pre;
            uint32_t pl = pre == STAGES ? 1u : 0u;
            for (int i = pre; i < my; ++i) {
                if (i >= STAGES) mbar_wait_cta(&empty[s], pl ^ 1u);
                mbar_expect_tx(&full[s], (uint32_t)TILE);
                const int row0 = (int)(((int64_t)blockIdx.x + (int64_t)i * gridDim.x) * TG::M);
#pragma unroll
                for (int a = 0; a < NA; ++a) tma_load_2d(ring + s * TILE + a * TG::SUB, &tmap, 32 * a, row0, &full[s]);
                if (++s == STAGES) {
                    s = 0;
                    pl ^= 1u;
                }
            }
        }
    } else if (warp == EW + 1) {  // ---- MMA issuer: K = NPW in 8-float steps across the atoms
        if (lane == 0) {
            const uint64_t a0 = umma_desc(smem_u32(ring), 1024, 2u);  // SWIZZLE_128B, SBO = 8 rows x 128 B
            const uint64_t b0 = umma_desc(smem_u32(Bt), 1024, 2u);
            int s = 0, b = 0;
            uint32_t pl = 0, pb = 0;
            for (int i = 0; i < my; ++i) {
                mbar_wait_cta(&full[s], pl);
                if (i >= NB) mbar_wait_cta(&tempty[b], pb ^ 1u);
                tc_fence_after();
#pragma unroll
                for (int ks = 0; ks < NPW / 8; ++ks) {
                    const uint64_t ad = a0 + (uint64_t)((s * TILE + (ks >> 2) * TG::SUB + (ks & 3) * 32) >> 4);
                    const uint64_t bd = b0 + (uint64_t)(((ks >> 2) * TG::BSUB + (ks & 3) * 32) >> 4);
                    asm volatile(
                        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                        " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tm + (uint32_t)(b * N)),
                        "l"(ad), "l"(bd), "r"(TG::IDESC), "r"(ks));
                }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                 smem_u32(&tfull[b]))
                             : "memory");
                if (++s == STAGES) {
                    s = 0;
                    pl ^= 1u;
                }
                if (++b == NB) {
                    b = 0;
                    pb ^= 1u;
                }
            }
        }
    } else {  // ---- epilogue: group g takes local tiles g, g + 2, ...
        const int g = warp >> 2, wq = warp & 3, r = wq * 32 + lane;
        float cmax = 0.f;
        for (int j = 0; j < kv; ++j) cmax = fmaxf(cmax, sqrtf(s_cc[j]) * 1.0001f);
        const float cmax2 = cmax * cmax;
        constexpr int TB = 5, TMASK = (1 << TB) - 1;
        const float kap2 = 2.0f * (0.0078125f + __int_as_float((127 + TB - 22) << 23)) * 1.0001f;
        constexpr float kap32 = 2.0f * 2.0f * (float)(NPW / 2 + 12) * 5.9604645e-8f * 1.0001f;
        int32_t* const labels_out = p.labels;
        unsigned long long* const counts_out = p.counts;
        const int32_t* const remap = p.remap;
        const float2* ccp = reinterpret_cast<const float2*>(s_cc);
        int s = g, b = g;
        uint32_t pb = 0;
        for (int i = g; i < my; i += 2) {
            mbar_wait_sleep(&tfull[b], pb);
            tc_fence_after();
            uint32_t v[N];
            const uint32_t taddr = tm + ((uint32_t)(wq * 32) << 16) + (uint32_t)(b * N);
            tmem_ld16(taddr, v);
            tmem_ld16(taddr + 16, v + 16);
            tmem_wait_ld();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[b]);
            const unsigned char* tile = ring + s * TILE;
            const int64_t row = ((int64_t)blockIdx.x + (int64_t)i * gridDim.x) * TG::M + r;
            const bool valid = row < m;
            // top-2 of the screened values (column index in the low mantissa bits)
            float p1[KPS], p2[KPS];
#pragma unroll
            for (int q = 0; q < KPS; ++q) {
                const float2 d2 = __fadd2_rn(make_float2(__uint_as_float(v[2 * q]), __uint_as_float(v[2 * q + 1])), ccp[q]);
                const float da = __int_as_float((__float_as_int(d2.x) & ~TMASK) | (2 * q));
                const float db = __int_as_float((__float_as_int(d2.y) & ~TMASK) | (2 * q + 1));
                p1[q] = fminf(da, db);
                p2[q] = fmaxf(da, db);
            }
#pragma unroll
            for (int w = 1; w < KPS; w *= 2)
#pragma unroll
                for (int q = 0; q + w < KPS; q += 2 * w) {
                    p2[q] = fmin3f(p2[q], p2[q + w], fmaxf(p1[q], p1[q + w]));
                    p1[q] = fminf(p1[q], p1[q + w]);
                }
            int lab = __float_as_int(p1[0]) & TMASK;
            // the fp64 cost to the screened centre, one pass over the row's chunks of the stage
            // (row base and swizzle phase hoisted: chunk c of the row is atom c / 8, slot (c % 8) ^ (r % 8))
            const unsigned char* rowp = tile + r * 128;
            const int rsw = r & 7;
            auto xchunk = [&](int c) -> float4 {
                return *reinterpret_cast<const float4*>(rowp + (c >> 3) * (TG::M * 128) + (((c & 7) ^ rsw) << 4));
            };
            auto row_cost = [&](int j) -> double {
                if (p.fast_cost) {  // fp32 mode: ((x + hi) + lo)^2 in fp32 FFMA2 chains, widened once per row
                    const unsigned char* bj = Bt + j * 128;  // centre j's row of the B tile
                    const int jsw = j & 7;
                    auto bchunk = [&](int c) -> float4 {
                        return *reinterpret_cast<const float4*>(bj + (c >> 3) * TG::BSUB + (((c & 7) ^ jsw) << 4));
                    };
                    const float4* lc = reinterpret_cast<const float4*>(neglo) + j;
                    const float2 h = make_float2(0.5f, 0.5f);
                    float2 a0 = make_float2(0.f, 0.f), a1 = a0, a2 = a0, a3 = a0;
#pragma unroll 4
                    for (int c = 0; c < NPW / 4; c += 2) {
                        const float4 x4 = xchunk(c), y4 = xchunk(c + 1);
                        const float4 c4 = bchunk(c), d4 = bchunk(c + 1);
                        const float4 l4 = lc[c * N], m4 = lc[(c + 1) * N];
                        const float2 e0 = __fadd2_rn(__ffma2_rn(make_float2(c4.x, c4.y), h, make_float2(x4.x, x4.y)),
                                                     make_float2(l4.x, l4.y));
                        const float2 e1 = __fadd2_rn(__ffma2_rn(make_float2(c4.z, c4.w), h, make_float2(x4.z, x4.w)),
                                                     make_float2(l4.z, l4.w));
                        const float2 e2 = __fadd2_rn(__ffma2_rn(make_float2(d4.x, d4.y), h, make_float2(y4.x, y4.y)),
                                                     make_float2(m4.x, m4.y));
                        const float2 e3 = __fadd2_rn(__ffma2_rn(make_float2(d4.z, d4.w), h, make_float2(y4.z, y4.w)),
                                                     make_float2(m4.z, m4.w));
                        a0 = __ffma2_rn(e0, e0, a0);
                        a1 = __ffma2_rn(e1, e1, a1);
                        a2 = __ffma2_rn(e2, e2, a2);
                        a3 = __ffma2_rn(e3, e3, a3);
                    }
                    return (double)(((a0.x + a0.y) + (a1.x + a1.y)) + ((a2.x + a2.y) + (a3.x + a3.y)));
                }
                const double* cj = Cg + (int64_t)j * NPW;
                double a[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll 4
                for (int c = 0; c < NPW / 4; ++c) {
                    const float4 x4 = xchunk(c);
                    const double2 c01 = __ldg(reinterpret_cast<const double2*>(cj + 4 * c));
                    const double2 c23 = __ldg(reinterpret_cast<const double2*>(cj + 4 * c + 2));
                    const double e0 = (double)x4.x - c01.x, e1 = (double)x4.y - c01.y;
                    const double e2 = (double)x4.z - c23.x, e3 = (double)x4.w - c23.y;
                    a[0] = fma(e0, e0, a[0]);
                    a[1] = fma(e1, e1, a[1]);
                    a[2] = fma(e2, e2, a[2]);
                    a[3] = fma(e3, e3, a[3]);
                }
                return (a[0] + a[1]) + (a[2] + a[3]);
            };
            double rc = row_cost(valid ? lab : 0);
            const int lab0 = lab;
            // |x|^2 bound of the screens' error terms from the cost just computed: |x| <= |x - c| + |c|
            // (1.0001 covers the fp32-mode cost and the rounded |c|^2)
            const float sxc = (sqrtf(fmaxf((float)rc, 0.f)) + sqrtf(s_cc[valid ? lab : 0])) * 1.0001f;
            const float nn = valid ? sxc * sxc : 0.f;
            const float btc = kap2 * (nn + cmax2);
            unsigned tie = __ballot_sync(0xffffffffu, valid && !(p2[0] - p1[0] > btc));
            if (tie) {
                // second tier: fp32 FFMA2 re-screen of the flagged rows over the centres whose tf32
                // value is within the bound of the minimum (the others are provably farther)
                bool still = false;
                if (tie & (1u << lane)) {
                    const float thr = p1[0] + btc;
                    uint32_t cand = 0;
#pragma unroll
                    for (int q = 0; q < KPS; ++q) {
                        const float2 c2 = ccp[q];
                        if (__uint_as_float(v[2 * q]) + c2.x <= thr) cand |= 1u << (2 * q);
                        if (__uint_as_float(v[2 * q + 1]) + c2.y <= thr) cand |= 1u << (2 * q + 1);
                    }
                    cand &= kv >= 32 ? 0xffffffffu : ((1u << kv) - 1u);
                    float n1 = __int_as_float(0x7f800000), n2 = n1;
                    int l1 = 0;
                    for (; cand; cand &= cand - 1) {  // ascending j
                        const int j = __ffs(cand) - 1;
                        const double* cj = Cg + (int64_t)j * NPW;
                        float2 acc = make_float2(s_cc[j], 0.f), acc2 = make_float2(0.f, 0.f);
                        for (int c = 0; c < NPW / 4; ++c) {
                            const float4 x4 = *reinterpret_cast<const float4*>(tile + sw128_off(TG::M, r, 4 * c));
                            const double2 c01 = __ldg(reinterpret_cast<const double2*>(cj + 4 * c));
                            const double2 c23 = __ldg(reinterpret_cast<const double2*>(cj + 4 * c + 2));
                            acc = __ffma2_rn(make_float2(x4.x, x4.y),
                                             make_float2((float)(-2.0 * c01.x), (float)(-2.0 * c01.y)), acc);
                            acc2 = __ffma2_rn(make_float2(x4.z, x4.w),
                                              make_float2((float)(-2.0 * c23.x), (float)(-2.0 * c23.y)), acc2);
                        }
                        const float dj = (acc.x + acc.y) + (acc2.x + acc2.y);
                        if (dj < n1) {
                            n2 = n1;
                            n1 = dj;
                            l1 = j;
                        } else {
                            n2 = fminf(n2, dj);
                        }
                    }
                    lab = l1;
                    still = !(n2 - n1 > kap32 * (nn + cmax2));
                }
                tie = __ballot_sync(0xffffffffu, still);
                // near ties of both screens: the exact reference argmin (core.hpp:146-157), lanes over
                // centres reading the flagged row from the stage
                while (tie) {
                    const int src = __ffs(tie) - 1;
                    tie &= tie - 1;
                    const int rs = (r & ~31) + src;
                    double dv = __longlong_as_double(0x7ff0000000000000LL);
                    int dj = 0x7fffffff;
                    for (int j = lane; j < kv; j += 32) {
                        const double* cj = Cg + (int64_t)j * NPW;
                        double acc = 0.0;
                        for (int d = 0; d < NPW; ++d) {
                            const double diff =
                                __dsub_rn((double)*reinterpret_cast<const float*>(tile + sw128_off(TG::M, rs, d)), cj[d]);
                            acc = __dadd_rn(acc, __dmul_rn(diff, diff));
                        }
                        if (acc < dv) {
                            dv = acc;
                            dj = j;
                        }
                    }
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) {
                        const double ov = __shfl_xor_sync(0xffffffffu, dv, o);
                        const int oj = __shfl_xor_sync(0xffffffffu, dj, o);
                        if (ov < dv || (ov == dv && oj < dj)) {
                            dv = ov;
                            dj = oj;
                        }
                    }
                    if (lane == src) lab = dj;
                }
                if (valid && lab != lab0) rc = row_cost(lab);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);  // this warp's rows are read
            if (valid) {
                cost += rc;
                if (labels_out) labels_out[row] = remap[lab];
                if (counts_out) atomicAdd(counts_out + remap[lab], 1ULL);
            }
            if (s += 2, s >= STAGES) s -= STAGES;
            if (b += 2, b >= NB) {
                b -= NB;
                pb ^= 1u;
            }
        }
        cost = warp_sum(cost);
        if (lane == 0) s_wcost[warp] = cost;
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == EW + 1)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(TG::TCOLS));
    if (tid == 0) {
        double t = 0.0;
        for (int w = 0; w < EW; ++w) t += s_wcost[w];
        p.block_cost[blockIdx.x] = t;
    }
}

}  // namespace hpcg
