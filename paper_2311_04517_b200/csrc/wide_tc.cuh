// Grid-wide Lloyd pass, nearest-centre screen on the tensor cores for wide fp32 samples (n = 64 or
// 128, k <= 32: BASELINE config 4's s x n x k contraction). Included by wide.cu.
//
// One persistent kernel per pass screens every row of every active worker's HBM-resident sample
// S[w] (s x n): a contiguous range of 128-row tiles per CTA, TMA boxes of one 128-B swizzle atom
// ({32 floats, 128 rows}, SWIZZLE_128B), tcgen05.mma.kind::tf32 (M = 128, N = 32, K = n in 8-float
// steps across the atoms) against the tile's worker's -2c (tf32, rebuilt in a double-buffered B
// tile when the worker changes), D in TMEM. The epilogue takes the top-2 (column index in the low
// mantissa bits), re-screens rows inside the tf32 bound with fp32 FFMA2 (objective_tcw.cuh), and
// writes one code per row into the pass's label buffer: the label, with bit 31 set when the row
// is still inside the fp32 bound. wide_assign_kernel then takes the label from the code and gives
// only the flagged rows the exact reference argmin (core.hpp:144-157).
#pragma once

namespace hpcg {
namespace {

constexpr int kTcwN = 32;  // centre columns

// |c_j|^2 (fp32, 1e38 past k) and max |c_j| (rounded up) of every worker's current centres
__global__ void wide_cc_kernel(const StepParams p, WideBufs b, float* ccw) {
    const int w = blockIdx.x, j = threadIdx.x;  // 32 threads
    const int k = p.k, n = p.n;
    float cc = 1e38f;
    if (j < k) {
        const double* c = b.Cm + ((int64_t)w * k + j) * n;
        double s = 0.0;
        for (int d = 0; d < n; ++d) s += c[d] * c[d];
        cc = (float)s;
    }
    ccw[w * (kTcwN + 1) + j] = cc;
    const unsigned cm = __reduce_max_sync(0xffffffffu, __float_as_uint(j < k ? sqrtf(cc) * 1.0001f : 0.f));
    if (j == 0) ccw[w * (kTcwN + 1) + kTcwN] = __uint_as_float(cm);
}

template <int NA>
struct WtcGeo {
    static constexpr int N = kTcwN, M = 128, NPW = 32 * NA;
    static constexpr int SUB = M * 128, TILE = NA * SUB;
    static constexpr int STAGES = 196608 / TILE < 6 ? 196608 / TILE : 6;  // 192 KB ring (3 stages at n = 128)
    static constexpr int BSUB = N * 128, BT = NA * BSUB;                  // one B buffer
    static constexpr int TCOLS = 512, NB = TCOLS / N;
    static constexpr int EPI_WARPS = 8, THREADS = (EPI_WARPS + 2) * 32;
    static constexpr uint32_t IDESC =
        (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    static_assert(STAGES >= 2, "stages");
};

template <int NA>
inline int wide_tc_smem() {
    using TG = WtcGeo<NA>;
    return 1024 + TG::STAGES * TG::TILE + 2 * TG::BT;
}

template <int NA, int KPS>
__global__ void __launch_bounds__(WtcGeo<NA>::THREADS, 1)
    wide_screen_tc_kernel(const StepParams p, WideBufs b, const float* __restrict__ ccw, int T, int tpw,
                          const __grid_constant__ CUtensorMap tmap) {
    using TG = WtcGeo<NA>;
    constexpr int N = TG::N, NPW = TG::NPW, STAGES = TG::STAGES, NB = TG::NB, TILE = TG::TILE, EW = TG::EPI_WARPS;
    extern __shared__ double wsm[];  // (the dynamic smem symbol wide.cu's kernels declare)
    unsigned char* wraw = reinterpret_cast<unsigned char*>(wsm);
    unsigned char* ring = wraw + ((1024 - (smem_u32(wraw) & 1023)) & 1023);
    unsigned char* Bt = ring + STAGES * TILE;  // [2][BT]
    __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES], tfull[NB], tempty[NB], bsafe;
    __shared__ uint32_t s_tmem;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int k = p.k;
    const int64_t s = p.s;
    int64_t t0, t1;
    chunk_range(T, gridDim.x, blockIdx.x, t0, t1);
    if (warp == EW + 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                     "r"(TG::TCOLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        for (int i = 0; i < STAGES; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 4);
        }
        for (int i = 0; i < NB; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 4);
        }
        mbar_init(&bsafe, 1);
        mbar_init_fence();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tm = s_tmem;
    auto active = [&](int64_t t) { return b.st[t / tpw].done == 0; };  // done flags are fixed for the pass

    if (warp == EW) {  // ---- TMA producer
        if (lane == 0) {
            int st = 0;
            uint32_t pl = 0;
            int i = 0;
            for (int64_t t = t0; t < t1; ++t) {
                if (!active(t)) continue;
                if (i >= STAGES) mbar_wait_cta(&empty[st], pl ^ 1u);
                mbar_expect_tx(&full[st], (uint32_t)TILE);
                const int row0 = (int)((t / tpw) * s + (t % tpw) * TG::M);
#pragma unroll
                for (int a = 0; a < NA; ++a) tma_load_2d(ring + st * TILE + a * TG::SUB, &tmap, 32 * a, row0, &full[st]);
                ++i;
                if (++st == STAGES) {
                    st = 0;
                    pl ^= 1u;
                }
            }
        }
    } else if (warp == EW + 1) {  // ---- MMA warp: B tile of the current worker (all lanes), MMAs (lane 0)
        const uint64_t a0 = umma_desc(smem_u32(ring), 1024, 2u);
        int st = 0, bb = 0, buf = -1, nsw = 0;
        uint32_t pl = 0, pb = 0, psafe = 0;
        int64_t cur_w = -1;
        int i = 0;
        for (int64_t t = t0; t < t1; ++t) {
            if (!active(t)) continue;
            const int64_t w = t / tpw;
            if (w != cur_w) {
                const int nb = buf < 0 ? 0 : buf ^ 1;
                if (nsw >= 2) {  // nb was used by earlier tiles: let every MMA issued so far complete
                    if (lane == 0)
                        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                         smem_u32(&bsafe))
                                     : "memory");
                    mbar_wait_cta(&bsafe, psafe);
                    psafe ^= 1u;
                }
                const double* C = b.Cm + w * (int64_t)k * NPW;
                unsigned char* B = Bt + nb * TG::BT;
                for (int e = lane; e < N * NPW; e += 32) {
                    const int j = e / NPW, d = e - j * NPW;
                    const float c2 = j < k ? (float)(-2.0 * C[(int64_t)j * NPW + d]) : 0.f;
                    *reinterpret_cast<float*>(B + sw128_off(N, j, d)) = tf32_rna(c2);
                }
                fence_proxy_async();
                __syncwarp();
                buf = nb;
                cur_w = w;
                ++nsw;
            }
            if (lane == 0) {
                mbar_wait_cta(&full[st], pl);
                if (i >= NB) mbar_wait_cta(&tempty[bb], pb ^ 1u);
                tc_fence_after();
                const uint64_t b0 = umma_desc(smem_u32(Bt + buf * TG::BT), 1024, 2u);
#pragma unroll
                for (int ks = 0; ks < NPW / 8; ++ks) {
                    const uint64_t ad = a0 + (uint64_t)((st * TILE + (ks >> 2) * TG::SUB + (ks & 3) * 32) >> 4);
                    const uint64_t bd = b0 + (uint64_t)(((ks >> 2) * TG::BSUB + (ks & 3) * 32) >> 4);
                    asm volatile(
                        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                        " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tm + (uint32_t)(bb * N)),
                        "l"(ad), "l"(bd), "r"(TG::IDESC), "r"(ks));
                }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                 smem_u32(&tfull[bb]))
                             : "memory");
            }
            __syncwarp();
            ++i;
            if (++st == STAGES) {
                st = 0;
                pl ^= 1u;
            }
            if (++bb == NB) {
                bb = 0;
                pb ^= 1u;
            }
        }
    } else {  // ---- epilogue: group g takes the g-th, (g+2)-th, ... active tile of the range
        const int g = warp >> 2, wq = warp & 3, r = wq * 32 + lane;
        constexpr int TB = 5, TMASK = (1 << TB) - 1;
        const float kap2 = 2.0f * (0.0078125f + __int_as_float((127 + TB - 22) << 23)) * 1.0001f;
        constexpr float kap32 = 2.0f * 2.0f * (float)(NPW / 2 + 12) * 5.9604645e-8f * 1.0001f;
        int st = 0, bb = 0, i = 0;
        uint32_t pb = 0;
        int64_t cur_w = -1;
        float2 cc[KPS];
        float cmax2 = 0.f;
        for (int64_t t = t0; t < t1; ++t) {
            if (!active(t)) continue;
            const bool mine = (i & 1) == g;
            const int myst = st, mybb = bb;
            const uint32_t mypb = pb;
            ++i;
            if (++st == STAGES) st = 0;
            if (++bb == NB) {
                bb = 0;
                pb ^= 1u;
            }
            if (!mine) continue;
            const int64_t w = t / tpw, tl = t % tpw;
            if (w != cur_w) {
                const float* cw = ccw + w * (kTcwN + 1);
#pragma unroll
                for (int q = 0; q < KPS; ++q) cc[q] = make_float2(__ldg(cw + 2 * q), __ldg(cw + 2 * q + 1));
                const float cm = __ldg(cw + kTcwN);
                cmax2 = cm * cm;
                cur_w = w;
            }
            mbar_wait_sleep(&tfull[mybb], mypb);
            tc_fence_after();
            uint32_t v[N];
            const uint32_t taddr = tm + ((uint32_t)(wq * 32) << 16) + (uint32_t)(mybb * N);
            tmem_ld16(taddr, v);
            tmem_ld16(taddr + 16, v + 16);
            tmem_wait_ld();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[mybb]);
            const unsigned char* tile = ring + myst * TILE;
            const int64_t lrow = tl * TG::M + r;
            const bool valid = lrow < s;
            float p1[KPS], p2[KPS];
#pragma unroll
            for (int q = 0; q < KPS; ++q) {
                const float2 d2 = __fadd2_rn(make_float2(__uint_as_float(v[2 * q]), __uint_as_float(v[2 * q + 1])), cc[q]);
                const float da = __int_as_float((__float_as_int(d2.x) & ~TMASK) | (2 * q));
                const float db = __int_as_float((__float_as_int(d2.y) & ~TMASK) | (2 * q + 1));
                p1[q] = fminf(da, db);
                p2[q] = fmaxf(da, db);
            }
#pragma unroll
            for (int ww = 1; ww < KPS; ww *= 2)
#pragma unroll
                for (int q = 0; q + ww < KPS; q += 2 * ww) {
                    p2[q] = fmin3f(p2[q], p2[q + ww], fmaxf(p1[q], p1[q + ww]));
                    p1[q] = fminf(p1[q], p1[q + ww]);
                }
            int lab = __float_as_int(p1[0]) & TMASK;
            float2 nn2 = make_float2(0.f, 0.f);
#pragma unroll 8
            for (int c = 0; c < NPW / 4; ++c) {
                const float4 x4 = *reinterpret_cast<const float4*>(tile + sw128_off(TG::M, r, 4 * c));
                nn2 = __ffma2_rn(make_float2(x4.x, x4.y), make_float2(x4.x, x4.y), nn2);
                nn2 = __ffma2_rn(make_float2(x4.z, x4.w), make_float2(x4.z, x4.w), nn2);
            }
            const float nn = nn2.x + nn2.y;
            bool flag = false;
            const float btc = kap2 * (nn + cmax2);
            if (valid && !(p2[0] - p1[0] > btc)) {
                // second tier: fp32 FFMA2 re-screen over the centres whose tf32 value is within the
                // bound of the minimum (any other centre is provably farther than the nearest one)
                const double* C = b.Cm + w * (int64_t)k * NPW;
                const float thr = p1[0] + btc;
                uint32_t cand = 0;  // centres within the bound (register-resident values, unrolled)
#pragma unroll
                for (int q = 0; q < KPS; ++q) {
                    if (__uint_as_float(v[2 * q]) + cc[q].x <= thr) cand |= 1u << (2 * q);
                    if (__uint_as_float(v[2 * q + 1]) + cc[q].y <= thr) cand |= 1u << (2 * q + 1);
                }
                cand &= k >= 32 ? 0xffffffffu : ((1u << k) - 1u);
                float n1 = __int_as_float(0x7f800000), n2 = n1;
                int l1 = 0;
                for (; cand; cand &= cand - 1) {  // ascending j, as the reference scans
                    const int j = __ffs(cand) - 1;
                    const double* cj = C + (int64_t)j * NPW;
                    float2 acc = make_float2(__ldg(ccw + w * (kTcwN + 1) + j), 0.f), acc2 = make_float2(0.f, 0.f);
                    for (int c = 0; c < NPW / 4; ++c) {
                        const float4 x4 = *reinterpret_cast<const float4*>(tile + sw128_off(TG::M, r, 4 * c));
                        const double2 c01 = __ldg(reinterpret_cast<const double2*>(cj + 4 * c));
                        const double2 c23 = __ldg(reinterpret_cast<const double2*>(cj + 4 * c + 2));
                        acc = __ffma2_rn(make_float2(x4.x, x4.y), make_float2((float)(-2.0 * c01.x), (float)(-2.0 * c01.y)),
                                         acc);
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
                flag = !(n2 - n1 > kap32 * (nn + cmax2));
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[myst]);
            if (valid) b.labels[w * s + lrow] = lab | (flag ? (int32_t)0x80000000 : 0);
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == EW + 1)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(TG::TCOLS));
}

}  // namespace
}  // namespace hpcg
