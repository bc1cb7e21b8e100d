// Full-data objective f(C, X) (engine.hpp:197-229 final_assignment / assign_valid_subset,
// core.hpp:224-233 mssc_objective) with the nearest-centre screen on the tensor cores.
//
// fp32 rows of 32/64/128 bytes (n = 8, 16, 32), up to 32 valid centres. Warp-specialised and
// persistent (one CTA per SM, 128-row tiles strided over the grid):
//   * producer warp: TMA (cp.async.bulk.tensor, hardware swizzle) streams tiles of X into a ring
//     of shared-memory stages -- the only HBM traffic, m*n*4 bytes per pass;
//   * MMA warp: one elected thread issues tcgen05.mma.kind::tf32 (M = 128 rows, N = 16/32
//     centre columns, K = n) reading the stage in place as the K-major A operand and -2c as B;
//     the 128 x N screen block lands in TMEM (4 buffers) and tcgen05.commit signals it;
//   * 8 epilogue warps (two groups of 4, alternate tiles): tcgen05.ld one row's N screened
//     values per thread, add |c_j|^2, top-2 with the centre index in the low mantissa bits, an
//     exact fp64 argmin (warp-parallel over centres) for rows whose top-2 gap is inside the
//     screen's error bound, then the row cost as the fp64 distance to the chosen centre.
// The CUDA cores thus only do the per-row epilogue, so the pass runs at the HBM rate.
//
// Screen error. d~_j = fl(|c_j|^2) + MMA(x, -2c_j) with B rounded to tf32 (2^-11) and A
// truncated by the tensor core (< 2^-10, measured 1.2e-3 of sum|x.c| by tools/probe/tc_probe.cu):
// |d~_j - (|c_j|^2 - 2 x.c_j)| <= 2^-9 * 2|x||c_j| + 2^-23 (|x| + |c_j|)^2 (accumulation,
// |c|^2 and the add rounding), and the index bits move a value by < 2^(tb-23) |d~_j|. With
// 2|x||c| <= (|x| + |c|)^2 / 2 the gap test uses kappa (|x| + cmax)^2, kappa = 2^-7 + 2^(tb-22)
// (a 2x margin over the worst case; evaluated as 2 kappa (|x|^2 + cmax^2) >= kappa (|x| + cmax)^2
// to avoid a square root per row), so a row outside it has the reference's label
// (core.hpp:144-157: strict <, ties to the lowest index) and a row inside it gets the exact one.
#pragma once
#include "objective_kernel.cuh"



#ifndef HPCG_TC_EPI
#define HPCG_TC_EPI 16  // epilogue warps of the tensor-core f(C,X) kernel
#endif

namespace hpcg {

template <int NP, int N>
struct TcGeo {
    static constexpr int M = 128;                     // rows per MMA (= TMEM lanes)
    static constexpr int TR = NP <= 16 ? 2 : 1;       // MMA row blocks per tile (one commit per tile)
    static constexpr int RPT = (NP == 8 && N == 16) ? 2 : 1;  // row blocks an epilogue thread takes per tile (n = 8:
                                                      // both; n = 16 would spill at the 96-register cap)
    static constexpr int BOX = TR * M < 256 ? TR * M : 256;   // TMA box rows (<= 256): TM / BOX loads per tile
    static constexpr int TM = M * TR;                 // rows per tile (= TMA box rows)
    static constexpr int RS = NP * 4;                 // row bytes (= swizzle span)
    static constexpr int TILE = TM * RS;              // bytes per stage
    static constexpr int STAGES = 196608 / TILE;     // 192 KB ring: tiles in flight from HBM
    static constexpr int TCOLS = 512;                 // all of TMEM (one CTA per SM)
    static constexpr int NB = TCOLS / (TR * N);       // TMEM tile buffers (even: 2 epilogue groups)
    static constexpr int EPI_WARPS = HPCG_TC_EPI;     // groups of 4 warps, one per tile phase
    static constexpr int GSTEP = EPI_WARPS / 4 / (TR / RPT);  // tile phases: a group = (phase, RPT row blocks)
                                                              // takes every GSTEP-th tile
    static constexpr int THREADS = (EPI_WARPS + 2) * 32;
    static constexpr int CDS = NP + 1;                // fp64 centre stride (doubles): odd, so the 8-B
                                                      // loads of up to 16 distinct centres in a half-warp
                                                      // phase hit distinct bank pairs
    static constexpr uint32_t LAYOUT = RS == 128 ? 2u : RS == 64 ? 4u : 6u;  // UMMA SW128 / SW64 / SW32
    // kind::tf32, D f32, A/B tf32 K-major, N >> 3, M >> 4
    static constexpr uint32_t IDESC =
        (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    static_assert(NB % GSTEP == 0 && STAGES >= GSTEP, "pipeline depth");
};

template <int NP, int N>
__host__ __device__ inline int objective_tc_smem(int kv) {
    using TG = TcGeo<NP, N>;
    return 1024 + TG::STAGES * TG::TILE + ((N * TG::RS + 1023) & ~1023) + kv * TG::CDS * 8;
}

HPCG_DEV void tma_prefetch_2d(const CUtensorMap* map, int c0, int c1) {
    asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(map), "r"(c0), "r"(c1)
                 : "memory");
}

// UMMA shared-memory descriptor: K-major, swizzled, SBO = 8 rows (tools/probe/tc_probe.cu)
HPCG_DEV uint64_t umma_desc(uint32_t saddr, uint32_t sbo_bytes, uint32_t layout) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;  // LBO (unused for swizzled K-major)
    d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
    d |= (uint64_t)layout << 61;
    return d;
}
HPCG_DEV void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
HPCG_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
HPCG_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
HPCG_DEV void tmem_ld16(uint32_t addr, uint32_t* v) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(addr));
}
HPCG_DEV void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
HPCG_DEV float tf32_rna(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

// try_wait with a short sleep between polls: waiting epilogue warps leave the issue slots to
// the warps that have rows to finish
HPCG_DEV bool mbar_try(uint64_t* bar, uint32_t phase) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
    return ok != 0;
}
HPCG_DEV void mbar_wait_sleep(uint64_t* bar, uint32_t phase) {
    while (!mbar_try(bar, phase)) __nanosleep(40);
}
// the same on a shared-memory address already converted (hot loops keep the u32 base)
HPCG_DEV void mbar_wait_sleep_u32(uint32_t addr, uint32_t phase) {
    for (;;) {
        uint32_t ok;
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(ok)
            : "r"(addr), "r"(phase)
            : "memory");
        if (ok) return;
        __nanosleep(40);
    }
}
HPCG_DEV void mbar_arrive_u32(uint32_t addr) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(addr) : "memory");
}

// KPS: centre pairs screened (ceil(kv / 2) of the N / 2 columns pairs; a compile-time count keeps
// the top-2 branch free)
template <int NP, int N, int KPS, bool OUT = true>  // OUT: labels / counts requested (else cost only)
__global__ void __launch_bounds__(TcGeo<NP, N>::THREADS, 1)
    objective_tc_kernel(const ObjParams p, const __grid_constant__ CUtensorMap tmap) {
    using TG = TcGeo<NP, N>;
    using G = Geo<float, NP>;
    constexpr int STAGES = TG::STAGES, NB = TG::NB, TILE = TG::TILE, CDS = TG::CDS, EW = TG::EPI_WARPS;
    extern __shared__ __align__(16) unsigned char osm[];
    unsigned char* ring = osm + ((1024 - (smem_u32(osm) & 1023)) & 1023);  // swizzle atoms: 1 KB aligned
    float* Bt = reinterpret_cast<float*>(ring + STAGES * TILE);
    double* Cd = reinterpret_cast<double*>(ring + STAGES * TILE + ((N * TG::RS + 1023) & ~1023));
    __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES], tfull[NB], tempty[NB];
    __shared__ uint32_t s_tmem;
    __shared__ __align__(8) float s_cc[N];
    __shared__ __align__(16) float s_rec[N][NP + 4];  // fp32 re-screen records: -2c, then |c|^2 at NP
    __shared__ __align__(16) float s_clo[N][NP + 4];  // fp32-mode cost: -(c - fl32(c)) (low parts)
    __shared__ double s_wcost[EW];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int kv = obj_kv(p);  // device-side valid count (p.kv: the launch bound, <= 2 KPS)

    // centres: fp64 copy (exact recheck, row cost) and the B operand -2c (tf32, K-major, swizzled
    // like the X stages); columns past the valid count screen to 1e38 and never win
    for (int e = tid; e < kv * CDS; e += TG::THREADS) {
        const int j = e / CDS, d = e - j * CDS;
        Cd[e] = d < NP ? p.C[(int64_t)j * NP + d] : 0.0;
    }
    for (int e = tid; e < N * NP; e += TG::THREADS) {
        const int j = e / NP, d = e - j * NP;
        const float c2 = j < kv ? (float)(-2.0 * p.C[(int64_t)j * NP + d]) : 0.f;
        Bt[G::elem_off(j, d)] = tf32_rna(c2);
        s_rec[j][d] = c2;
        if (p.fast_cost && j < kv) {  // the centre's low part: -(c - fl32(c))
            const double c = p.C[(int64_t)j * NP + d];
            s_clo[j][d] = (float)-(c - (double)(float)c);
        } else {
            s_clo[j][d] = 0.f;
        }
    }
    if (tid < N) {
        float cc = 1e38f;
        if (tid < kv) {
            double s = 0.0;
            for (int d = 0; d < NP; ++d) {
                const double c = p.C[(int64_t)tid * NP + d];
                s += c * c;
            }
            cc = (float)s;
        }
        s_cc[tid] = cc;
        s_rec[tid][NP] = cc;
    }
    if (warp == EW + 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                     "r"(TG::TCOLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    const int64_t m = p.m;
    const int64_t ntiles = (m + TG::TM - 1) / TG::TM;
    const int my = (int64_t)blockIdx.x < ntiles ? (int)((ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x) : 0;
    // The producer thread initialises the barriers itself and puts the first ring of tiles in flight
    // BEFORE the CTA-wide barrier below, so the centre tables, the TMEM allocation and the barrier
    // overlap the first HBM round trip instead of preceding it.
    const int pre = my < STAGES ? my : STAGES;
    if (warp == EW && lane == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 4 * (TG::TR / TG::RPT));  // the warps of the tile's groups
        }
        for (int b = 0; b < NB; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], 4 * (TG::TR / TG::RPT));
        }
        mbar_init_fence();
        fence_proxy_async();
        for (int i = 0; i < pre; ++i) {
            mbar_expect_tx(&full[i], (uint32_t)TILE);
#pragma unroll
            for (int h = 0; h < TG::TM / TG::BOX; ++h)
                tma_load_2d(ring + i * TILE + h * TG::BOX * TG::RS, &tmap, 0,
                            (int)(((int64_t)blockIdx.x + (int64_t)i * gridDim.x) * TG::TM + h * TG::BOX), &full[i]);
        }
    }
    fence_proxy_async();  // B tile (generic stores) -> tensor-core reads (async proxy)
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tm = s_tmem;
    double cost = 0.0;

    if (warp == EW) {  // ---- TMA producer: stage s, lap parity pl
        if (lane == 0) {
            int s = pre == STAGES ? 0 : pre;
            uint32_t pl = pre == STAGES ? 1u : 0u;
            for (int i = pre; i < my; ++i) {
                if (i >= STAGES) mbar_wait_cta(&empty[s], pl ^ 1u);
                mbar_expect_tx(&full[s], (uint32_t)TILE);
#pragma unroll
                for (int h = 0; h < TG::TM / TG::BOX; ++h)
                    tma_load_2d(ring + s * TILE + h * TG::BOX * TG::RS, &tmap, 0,
                                (int)(((int64_t)blockIdx.x + (int64_t)i * gridDim.x) * TG::TM + h * TG::BOX), &full[s]);
                if (++s == STAGES) {
                    s = 0;
                    pl ^= 1u;
                }
            }
        }
    } else if (warp == EW + 1) {  // ---- MMA issuer: TR x K/8 MMAs and one commit per tile
        if (lane == 0) {
            const uint64_t a0 = umma_desc(smem_u32(ring), 8 * TG::RS, TG::LAYOUT);
            const uint64_t b0 = umma_desc(smem_u32(Bt), 8 * TG::RS, TG::LAYOUT);
            int s = 0, b = 0;
            uint32_t pl = 0, pb = 0;
            for (int i = 0; i < my; ++i) {
                mbar_wait_cta(&full[s], pl);
                if (i >= NB) mbar_wait_cta(&tempty[b], pb ^ 1u);
                tc_fence_after();
#pragma unroll
                for (int rb = 0; rb < TG::TR; ++rb) {
#pragma unroll
                    for (int ks = 0; ks < NP / 8; ++ks) {
                        // descriptor start address (16-B units) advanced to stage s, row block rb, K chunk ks
                        const uint64_t ad = a0 + (uint64_t)((s * TILE + rb * TG::M * TG::RS + ks * 32) >> 4);
                        const uint64_t bd = b0 + (uint64_t)((ks * 32) >> 4);
                        asm volatile(
                            "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                            " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(
                                tm + (uint32_t)((b * TG::TR + rb) * N)),
                            "l"(ad), "l"(bd), "r"(TG::IDESC), "r"(ks));
                    }
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
    } else {  // ---- epilogue: group g = (tile phase tp, row blocks rbase..rbase+RPT-1): local tiles tp,
              // tp + GSTEP, ..., rows rb*128 + r of those blocks; warp quarter wq = its TMEM lanes
        constexpr int KP = KPS;
        static_assert(KPS >= 1 && KPS <= N / 2, "screened pairs");
        constexpr int STEP = TG::GSTEP;
        constexpr int RPT = TG::RPT;
        const int g = warp >> 2, wq = warp & 3, tp = g / (TG::TR / RPT), rbase = (g % (TG::TR / RPT)) * RPT;
        const int r = wq * 32 + lane;  // row within the 128-row block (= TMEM lane)
        const float2* cc = reinterpret_cast<const float2*>(s_cc);  // broadcast loads (registers are scarce)
        float cmax = 0.f;
        for (int j = 0; j < kv; ++j) cmax = fmaxf(cmax, sqrtf(s_cc[j]) * 1.0001f);
        constexpr int TB = N == 16 ? 4 : 5, TMASK = (1 << TB) - 1;  // column index bits
        // gap bound kappa (|x| + cmax)^2 <= 2 kappa (|x|^2 + cmax^2): no square root per row
        const float kap2 = 2.0f * (0.0078125f + __int_as_float((127 + TB - 22) << 23)) * 1.0001f;
        const float cmax2 = cmax * cmax;
        int32_t* const labels_out = p.labels;
        unsigned long long* const counts_out = p.counts;
        const int32_t* const remap = p.remap;
        int s = tp, b = tp;
        uint32_t pb = 0;
        int64_t row0 = ((int64_t)blockIdx.x + (int64_t)tp * gridDim.x) * TG::TM + rbase * TG::M + r;
        const int64_t row_step = STEP * (int64_t)gridDim.x * TG::TM;
        // loop invariants: barrier addresses, this lane's TMEM column base, its rows' chunk offsets in a stage
        const uint32_t tfull_u = smem_u32(&tfull[0]), tempty_u = smem_u32(&tempty[0]), empty_u = smem_u32(&empty[0]);
        const uint32_t tbase = tm + ((uint32_t)(wq * 32) << 16) + (uint32_t)(rbase * N);
        const uint32_t ring_u = smem_u32(ring);
        uint32_t xoff[RPT][NP / 4];
#pragma unroll
        for (int rb = 0; rb < RPT; ++rb)
#pragma unroll
            for (int q = 0; q < NP / 4; ++q) xoff[rb][q] = (uint32_t)G::elem_off((rbase + rb) * TG::M + r, q * 4) * 4u;
        for (int i = tp; i < my; i += STEP, row0 += row_step) {
            mbar_wait_sleep_u32(tfull_u + 8u * (uint32_t)b, pb);
            tc_fence_after();
            // the first row block's screened values: tcgen05.ld in flight while the rows are read
            uint32_t v[N];
            {
                const uint32_t taddr = tbase + (uint32_t)(b * TG::TR * N);
                tmem_ld16(taddr, v);
                if constexpr (N == 32) tmem_ld16(taddr + 16, v + 16);
                if constexpr (RPT == 1) {  // one row block: its values read, the TMEM buffer share is free
                    tmem_wait_ld();
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive_u32(tempty_u + 8u * (uint32_t)b);
                }
            }
            // the rows of this group's row blocks: their stage has landed (the MMAs that read it completed)
            const uint32_t tile_u = ring_u + (uint32_t)(s * TILE);
            float xr[RPT][NP];
#pragma unroll
            for (int rb = 0; rb < RPT; ++rb)
#pragma unroll
                for (int q = 0; q < NP / 4; ++q) {
                    float4 t4;
                    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                                 : "=f"(t4.x), "=f"(t4.y), "=f"(t4.z), "=f"(t4.w)
                                 : "r"(tile_u + xoff[rb][q]));
                    xr[rb][4 * q] = t4.x;
                    xr[rb][4 * q + 1] = t4.y;
                    xr[rb][4 * q + 2] = t4.z;
                    xr[rb][4 * q + 3] = t4.w;
                }
            __syncwarp();
            if (lane == 0) mbar_arrive_u32(empty_u + 8u * (uint32_t)s);
            const int bcur = b;
            if (s += STEP, s >= STAGES) s -= STAGES;
            if (b += STEP, b >= NB) {
                b -= NB;
                pb ^= 1u;
            }
#pragma unroll
            for (int rb = 0; rb < RPT; ++rb) {
            const int64_t row = row0 + rb * TG::M;
            const float* x = xr[rb];
            if (rb > 0) {
                const uint32_t taddr = tbase + (uint32_t)((bcur * TG::TR + rb) * N);
                tmem_ld16(taddr, v);
                if constexpr (N == 32) tmem_ld16(taddr + 16, v + 16);
            }
            if constexpr (RPT > 1) tmem_wait_ld();
            if (RPT > 1 && rb == RPT - 1) {  // this group's values read: its share of the TMEM buffer is free
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_u32(tempty_u + 8u * (uint32_t)bcur);
            }
            {
                // top-2 of d~_j = |c_j|^2 - 2 x.c_j over all N columns (unused ones screen to 1e38);
                // the column index rides in the low TB mantissa bits, so a min carries its argmin.
                // Sorted pairs, then a tree of (min, second-min) merges: short dependency chains.
                float p1[KP], p2[KP];
#pragma unroll
                for (int q = 0; q < KP; ++q) {
                    const float2 d2 = __fadd2_rn(make_float2(__uint_as_float(v[2 * q]), __uint_as_float(v[2 * q + 1])),
                                                 cc[q]);
                    const float da = __int_as_float((__float_as_int(d2.x) & ~TMASK) | (2 * q));
                    const float db = __int_as_float((__float_as_int(d2.y) & ~TMASK) | (2 * q + 1));
                    p1[q] = fminf(da, db);
                    p2[q] = fmaxf(da, db);
                }
#pragma unroll
                for (int w = 1; w < KP; w *= 2)
#pragma unroll
                    for (int q = 0; q + w < KP; q += 2 * w) {
                        p2[q] = fmin3f(p2[q], p2[q + w], fmaxf(p1[q], p1[q + w]));
                        p1[q] = fminf(p1[q], p1[q + w]);
                    }
                const float m1 = p1[0], m2 = p2[0];
                int lab = __float_as_int(m1) & TMASK;
                const bool valid = row < m;
                float2 nn2 = make_float2(0.f, 0.f), nn3 = nn2;
#pragma unroll
                for (int d = 0; d < NP; d += 4) {
                    nn2 = __ffma2_rn(make_float2(x[d], x[d + 1]), make_float2(x[d], x[d + 1]), nn2);
                    nn3 = __ffma2_rn(make_float2(x[d + 2], x[d + 3]), make_float2(x[d + 2], x[d + 3]), nn3);
                }
                const float nn = (nn2.x + nn2.y) + (nn3.x + nn3.y);
                const float btc = kap2 * (nn + cmax2);
                unsigned tie = __ballot_sync(0xffffffffu, valid && !(m2 - m1 > btc));
                if (tie) {
                    // second tier: rows the tf32 screen cannot settle get the fp32 FFMA2 screen
                    // (error <= 2 (NP/2 + 12) 2^-24 (|x| + |c|)^2 per value, the bound of the centre-pair
                    // kernel) over the centres whose tf32 value is within the bound of the minimum (any
                    // other centre is provably farther than the nearest), with broadcast record loads
                    bool still = false;
                    if (tie & (1u << lane)) {
                        const float thr = m1 + btc;
                        uint32_t cand = 0;
#pragma unroll
                        for (int q = 0; q < KP; ++q) {
                            const float2 c2 = cc[q];
                            if (__uint_as_float(v[2 * q]) + c2.x <= thr) cand |= 1u << (2 * q);
                            if (__uint_as_float(v[2 * q + 1]) + c2.y <= thr) cand |= 1u << (2 * q + 1);
                        }
                        cand &= kv >= 32 ? 0xffffffffu : ((1u << kv) - 1u);
                        float n1 = __int_as_float(0x7f800000), n2 = n1;
                        int l1 = 0;
                        for (; cand; cand &= cand - 1) {  // ascending j
                            const int j = __ffs(cand) - 1;
                            const float* rc = s_rec[j];
                            float2 a0 = make_float2(rc[NP], 0.f), a1 = make_float2(0.f, 0.f);
#pragma unroll
                            for (int d = 0; d < NP; d += 4) {
                                const float4 c4 = *reinterpret_cast<const float4*>(rc + d);
                                a0 = __ffma2_rn(make_float2(x[d], x[d + 1]), make_float2(c4.x, c4.y), a0);
                                a1 = __ffma2_rn(make_float2(x[d + 2], x[d + 3]), make_float2(c4.z, c4.w), a1);
                            }
                            const float dj = (a0.x + a0.y) + (a1.x + a1.y);
                            if (dj < n1) {
                                n2 = n1;
                                n1 = dj;
                                l1 = j;
                            } else {
                                n2 = fminf(n2, dj);
                            }
                        }
                        lab = l1;
                        constexpr float kap32 = 2.0f * 2.0f * (float)(NP / 2 + 12) * 5.9604645e-8f * 1.0001f;
                        still = !(n2 - n1 > kap32 * (nn + cmax2));
                    }
                    tie = __ballot_sync(0xffffffffu, still);
                }
                // near ties of both screens: the exact reference argmin, warp-parallel over centres
                // (core.hpp:146-157)
                while (tie) {
                    const int src = __ffs(tie) - 1;
                    tie &= tie - 1;
                    float xr[NP];
#pragma unroll
                    for (int d = 0; d < NP; ++d) xr[d] = __shfl_sync(0xffffffffu, x[d], src);
                    double dv = __longlong_as_double(0x7ff0000000000000LL);
                    int dj = 0x7fffffff;
                    for (int j = lane; j < kv; j += 32) {
                        const double dd = exact_dist_regs<float, NP>(xr, Cd + j * CDS);
                        if (dd < dv) {
                            dv = dd;
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
                if (valid) {
                    if (p.fast_cost) {
                        // fp32 mode: (x - c~)^2 in fp32 (c~ = -0.5 * the record's -2c: exact), two FFMA2
                        // chains per row, the row sum widened once into the fp64 accumulator
                        // difference (x - c_hi) - c_lo: both steps rounded to ~2^-24 |x - c|
                        const float* rc = s_rec[lab];
                        const float* rl = s_clo[lab];
                        float2 a0 = make_float2(0.f, 0.f), a1 = a0;
#pragma unroll
                        for (int d = 0; d < NP; d += 4) {
                            const float4 c4 = *reinterpret_cast<const float4*>(rc + d);
                            const float4 l4 = *reinterpret_cast<const float4*>(rl + d);
                            const float2 e0 = __fadd2_rn(__ffma2_rn(make_float2(c4.x, c4.y), make_float2(0.5f, 0.5f),
                                                                    make_float2(x[d], x[d + 1])),
                                                         make_float2(l4.x, l4.y));
                            const float2 e1 = __fadd2_rn(__ffma2_rn(make_float2(c4.z, c4.w), make_float2(0.5f, 0.5f),
                                                                    make_float2(x[d + 2], x[d + 3])),
                                                         make_float2(l4.z, l4.w));
                            a0 = __ffma2_rn(e0, e0, a0);
                            a1 = __ffma2_rn(e1, e1, a1);
                        }
                        cost += (double)((a0.x + a0.y) + (a1.x + a1.y));
                    } else {
                        // row cost: fp64 distance to the chosen centre (interleaved DFMA chains; within
                        // 1e-15 relative of the reference's per-row value)
                        const double* cj = Cd + lab * CDS;
                        double a[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
                        for (int d = 0; d < NP; ++d) {
                            const double e = (double)x[d] - cj[d];
                            a[d & 3] = fma(e, e, a[d & 3]);
                        }
                        cost += (a[0] + a[1]) + (a[2] + a[3]);
                    }
                    if constexpr (OUT) {
                        if (labels_out) labels_out[row] = remap[lab];
                        if (counts_out) atomicAdd(counts_out + remap[lab], 1ULL);
                    }
                }
            }
            }  // row blocks
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
    if (p.cost_out) finalize_block_sums(p, s_wcost);  // s_wcost reused as the 8 warp partials
}

}  // namespace hpcg
