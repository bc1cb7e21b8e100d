// Full-data objective f(C, X) (engine.hpp:197-229, core.hpp:224-233) for NARROW rows: fp64 rows of
// 1-3 values (BASELINE config 1: n = 2, config 3: n = 3) and fp32 rows of 2 values -- widths a
// tensor map cannot express (24-B rows) or too narrow for the tensor-core screen to pay.
//
// Each warp streams groups of 128 consecutive rows (contiguous bytes) through a ring of
// shared-memory stages filled by 1-D bulk copies (cp.async.bulk + mbarrier complete_tx). The
// nearest-centre screen is the centre-pair form: one FFMA2 evaluates one dimension for TWO
// centres, the row value a broadcast operand, records (-2c_a,d, -2c_b,d; |c_a|^2, |c_b|^2) read as
// broadcast 16-B shared loads shared by the R = 4 rows of a lane; top-2 with the centre index in
// the low mantissa bits. Rows whose top-2 gap is inside the screen bound get the exact reference
// argmin (core.hpp:144-157); the row cost is the fp64 distance to the chosen centre.
//
// Screen error: x rounded to fp32, a sequential fused chain of NP terms on rounded records:
// |d~ - d| <= (NP + 2) u (|x| + |c|)^2 plus the conversions (inside the +12 slack), doubled for a
// difference; the index bits add 2^(tb-22) (|x| + cmax)^2 (as in objective_pairs_kernel).
#pragma once
#include "objective_tc.cuh"

namespace hpcg {

// Cell filter for rows of n <= 3 (GRID variant): the centres' bounding box, padded, is cut into
// kGridCells cells (G per dimension); per cell a mask of the centres that can be the nearest to some
// point of the cell (grid_mask_kernel). A row inside the grid computes the exact reference distance
// to its cell's candidates only; rows outside it (or kv > 32) take every centre.
template <int NP>
struct GridGeo {
    static constexpr int G = NP == 1 ? 4096 : NP == 2 ? 64 : 16;  // cells per dimension (kGridCells cells)
};

template <typename T, int NP, bool GRID = false>
struct RowsGeo {
    static constexpr int R = 4;                              // rows per lane
    static constexpr int GR = 32 * R;                        // rows per stage
    static constexpr int RB = NP * (int)sizeof(T);           // row bytes
    static constexpr int STAGE = GR * RB;                    // bytes per stage (multiple of 16)
    static constexpr int WARPS = 8;
    static constexpr int RING = GRID ? 49152 : 98304;        // ring bytes (GRID: + 16 KB of cell masks, 3 CTAs/SM)
    static constexpr int STAGES = RING / (WARPS * STAGE) < 8 ? RING / (WARPS * STAGE) : 8;
    static constexpr int RST = ((NP + 2) / 2) * 2;           // record stride (float2, even: 16-B loads)
    static constexpr int CDS = NP | 1;                       // fp64 centre stride: odd (8-B loads)
    static constexpr float kappa = 2.0f * (float)(NP + 12) * 5.9604645e-8f;
    static_assert(STAGE % 16 == 0 && STAGES >= 2, "stage geometry");
};

template <typename T, int NP, bool GRID = false>
__host__ __device__ inline int objective_rows_smem(int kv) {
    using RG = RowsGeo<T, NP, GRID>;
    const int kp = (kv + 1) / 2;
    return ((kp * RG::RST * 8 + kv * RG::CDS * 8 + 127) & ~127) + RG::WARPS * RG::STAGES * RG::STAGE + 128 +
           (GRID ? kGridCells * 4 : 0);
}

// The cell masks (one thread per cell). Cell box = [lo + i w, lo + (i + 1) w] per dimension, widened
// by 1e-6 w (the fp64 cell index of a row is exact to far less). z* = the centre nearest the cell's
// midpoint; centre j is dropped iff max over the box of 2 x.(c_j - z*) < |c_j|^2 - |z*|^2 - delta,
// i.e. every point of the box is nearer z* than c_j by more than delta = 1e-9 (|x|max + |c|max)^2 in
// exact arithmetic -- far above the rounding of the reference distance (~1e-15 of the same scale),
// so the fp64 distances keep that order and a dropped centre can neither be the nearest nor tie it.
template <int NP>
__global__ void __launch_bounds__(256) grid_mask_kernel(const ObjParams p) {
    constexpr int G = GridGeo<NP>::G;
    __shared__ double sc[32][3], s_n2[32], s_lo[3], s_w[3], s_rc;
    const int kv = obj_kv(p);
    for (int e = threadIdx.x; e < 32 * 3; e += blockDim.x) {
        const int j = e / 3, d = e - j * 3;
        sc[j][d] = (j < kv && d < NP) ? p.C[(int64_t)j * NP + d] : 0.0;
    }
    __syncthreads();
    if (threadIdx.x < 32) {
        const int j = threadIdx.x;
        s_n2[j] = sc[j][0] * sc[j][0] + sc[j][1] * sc[j][1] + sc[j][2] * sc[j][2];
    }
    if (threadIdx.x == 0) {
        double rc = 0.0;
        for (int j = 0; j < kv; ++j) rc = fmax(rc, sqrt(sc[j][0] * sc[j][0] + sc[j][1] * sc[j][1] + sc[j][2] * sc[j][2]));
        s_rc = rc;
        for (int d = 0; d < 3; ++d) {
            double mn = kv > 0 ? sc[0][d] : 0.0, mx = mn;
            for (int j = 1; j < kv; ++j) {
                mn = fmin(mn, sc[j][d]);
                mx = fmax(mx, sc[j][d]);
            }
            const double span = mx - mn;
            const double pad = 0.15 * span + 1e-3 * (fabs(mn) + fabs(mx)) + 1e-3;
            s_lo[d] = mn - pad;
            s_w[d] = (span + 2.0 * pad) / G;
        }
        if (blockIdx.x == 0) {
            GridHdr* h = reinterpret_cast<GridHdr*>(p.grid + kGridCells);
            for (int d = 0; d < 3; ++d) {
                h->lo[d] = s_lo[d];
                h->inv_w[d] = 1.0 / s_w[d];
            }
        }
    }
    __syncthreads();
    for (int cell = blockIdx.x * blockDim.x + threadIdx.x; cell < kGridCells; cell += gridDim.x * blockDim.x) {
        double blo[3] = {0.0, 0.0, 0.0}, bhi[3] = {0.0, 0.0, 0.0}, mid[3] = {0.0, 0.0, 0.0};
        int rest = cell;
        double rb2 = 0.0;
        for (int d = NP - 1; d >= 0; --d) {
            const int i = rest % G;
            rest /= G;
            blo[d] = s_lo[d] + ((double)i - 1e-6) * s_w[d];
            bhi[d] = s_lo[d] + ((double)i + 1.0 + 1e-6) * s_w[d];
            mid[d] = 0.5 * (blo[d] + bhi[d]);
            rb2 += fmax(blo[d] * blo[d], bhi[d] * bhi[d]);
        }
        int zs = 0;
        double bd = __longlong_as_double(0x7ff0000000000000LL);
        for (int j = 0; j < kv; ++j) {
            double dd = 0.0;
            for (int d = 0; d < NP; ++d) dd += (mid[d] - sc[j][d]) * (mid[d] - sc[j][d]);
            if (dd < bd) {
                bd = dd;
                zs = j;
            }
        }
        const double sr = sqrt(rb2) + s_rc;
        const double delta = 1e-9 * sr * sr;
        uint32_t mask = 0;
        for (int j = 0; j < kv; ++j) {
            bool keep = j == zs;
            if (!keep) {
                double mx = 0.0;
                for (int d = 0; d < NP; ++d) {
                    const double w = sc[j][d] - sc[zs][d];
                    mx += fmax(blo[d] * w, bhi[d] * w);
                }
                keep = !(2.0 * mx < (s_n2[j] - s_n2[zs]) - delta);
            }
            if (keep) mask |= 1u << j;
        }
        p.grid[cell] = mask;
    }
}

HPCG_DEV void bulk_load(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(sdst)),
        "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

template <typename T, int NP, bool GRID = false>
__global__ void __launch_bounds__(256, GRID ? 3 : 2) objective_rows_kernel(const ObjParams p, const __grid_constant__ CUtensorMap) {
    using RG = RowsGeo<T, NP, GRID>;
    constexpr int R = RG::R, GR = RG::GR, RST = RG::RST, CDS = RG::CDS, WARPS = RG::WARPS, STAGES = RG::STAGES;
    extern __shared__ __align__(16) unsigned char osm[];
    const int kvl = p.kv, kpl = (kvl + 1) / 2;  // launch bound: smem layout, uniform trip count
    const int kv = obj_kv(p);
    float2* rp = reinterpret_cast<float2*>(osm);
    double* Cd = reinterpret_cast<double*>(osm + kpl * RST * 8);
    unsigned char* rings = osm + ((kpl * RST * 8 + kvl * CDS * 8 + 127) & ~127);
    uint32_t* s_mask = reinterpret_cast<uint32_t*>(rings + WARPS * STAGES * RG::STAGE + 128);  // GRID only
    __shared__ __align__(8) uint64_t s_bar[WARPS][STAGES];
    __shared__ float s_cmax;
    __shared__ double s_wcost[WARPS];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    for (int e = tid; e < kv * CDS; e += 256) {
        const int j = e / CDS, d = e - j * CDS;
        Cd[e] = d < NP ? p.C[(int64_t)j * NP + d] : 0.0;
    }
    // records: pair q = centres 2q, 2q+1; a missing centre screens to 1e38 and never wins
    for (int j = tid; j < 2 * kpl; j += 256) {
        float* rec = reinterpret_cast<float*>(rp + (j >> 1) * RST) + (j & 1);
        double cc = 0.0;
        for (int d = 0; d < NP; ++d) {
            const double c = j < kv ? p.C[(int64_t)j * NP + d] : 0.0;
            cc += c * c;
            rec[2 * d] = (float)(-2.0 * c);
        }
        rec[2 * NP] = j < kv ? (float)cc : 1e38f;
        for (int d = NP + 1; d < RST; ++d) rec[2 * d] = 0.f;
    }
    if constexpr (GRID)
        for (int e = tid; e < kGridCells; e += 256) s_mask[e] = p.grid[e];
    if (lane == 0) {
        for (int st = 0; st < STAGES; ++st) mbar_init(&s_bar[warp][st], 1);
        mbar_init_fence();
    }
    fence_proxy_async();
    __syncthreads();
    if (tid == 0) {
        float cm = 0.f;
        for (int j = 0; j < kv; ++j) {
            double cc = 0.0;
            for (int d = 0; d < NP; ++d) cc += Cd[j * CDS + d] * Cd[j * CDS + d];
            cm = fmaxf(cm, (float)sqrt(cc) * 1.0001f);
        }
        s_cmax = cm;
    }
    __syncthreads();
    const float cmax = s_cmax;
    const int tbits = 32 - __clz(2 * kpl - 1 > 0 ? 2 * kpl - 1 : 1);
    const int tmask = (1 << tbits) - 1;
    const float kap = RG::kappa + __int_as_float((127 + tbits - 22) << 23);  // + 2^(tb-22)

    // cell filter: the grid's origin and inverse cell widths in registers (GRID only)
    double glo[NP], giw[NP];
#pragma unroll
    for (int d = 0; d < NP; ++d) {
        glo[d] = GRID ? reinterpret_cast<const GridHdr*>(p.grid + kGridCells)->lo[d] : 0.0;
        giw[d] = GRID ? reinterpret_cast<const GridHdr*>(p.grid + kGridCells)->inv_w[d] : 0.0;
    }
    const T* X = static_cast<const T*>(p.X);
    const int64_t m = p.m;
    const int64_t ngroups = (m + GR - 1) / GR, nfull = m / GR;
    const int64_t wg = (int64_t)blockIdx.x * WARPS + warp, wstride = (int64_t)gridDim.x * WARPS;
    const int64_t my = wg < ngroups ? (ngroups - wg + wstride - 1) / wstride : 0;
    unsigned char* ring = rings + warp * STAGES * RG::STAGE;
    auto issue = [&](int64_t i) {
        if (i < my && lane == 0) {
            const int64_t g = wg + i * wstride;
            uint64_t* bar = &s_bar[warp][i % STAGES];
            if (g < nfull) {
                fence_proxy_async();  // this warp's generic reads of the stage precede the async write
                mbar_expect_tx(bar, (uint32_t)RG::STAGE);
                bulk_load(ring + (i % STAGES) * RG::STAGE, X + g * GR * NP, (uint32_t)RG::STAGE, bar);
            } else {
                mbar_arrive(bar);  // the partial tail group is read from global memory directly
            }
        }
    };
#pragma unroll 1
    for (int st = 0; st < STAGES; ++st) issue(st);

    double cost = 0.0;
#pragma unroll 1
    for (int64_t i = 0; i < my; ++i) {
        mbar_wait_cta(&s_bar[warp][i % STAGES], (uint32_t)((i / STAGES) & 1));
        const int64_t g = wg + i * wstride, row0 = g * GR;
        const bool full = g < nfull;
        const T* slot = reinterpret_cast<const T*>(ring + (i % STAGES) * RG::STAGE);
        T x[R][NP];
        if (full) {
#pragma unroll
            for (int r = 0; r < R; ++r)
#pragma unroll
                for (int d = 0; d < NP; ++d) x[r][d] = slot[(r * 32 + lane) * NP + d];
        } else {
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int64_t row = row0 + r * 32 + lane;
#pragma unroll
                for (int d = 0; d < NP; ++d) x[r][d] = row < m ? X[row * NP + d] : T(0);
            }
        }
        __syncwarp();
        issue(i + STAGES);
        if constexpr (GRID) {
            // the cell's candidates, exact reference distances (core.hpp:146-157: ascending j, strict <)
            constexpr int G = GridGeo<NP>::G;
            const uint32_t all = kv >= 32 ? 0xffffffffu : ((1u << kv) - 1u);
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int64_t row = row0 + r * 32 + lane;
                const bool valid = full || row < m;
                bool in = true;
                int cell = 0;
#pragma unroll
                for (int d = 0; d < NP; ++d) {
                    const double t = ((double)x[r][d] - glo[d]) * giw[d];
                    in &= (t >= 0.0) & (t < (double)G);
                    cell = cell * G + (in ? __double2int_rz(t) : 0);
                }
                uint32_t msk = in ? s_mask[cell] : all;
                int lab = msk ? __ffs(msk) - 1 : 0;
                double dv = __longlong_as_double(0x7ff0000000000000LL);
                for (; msk; msk &= msk - 1) {
                    const int j = __ffs(msk) - 1;
                    const double dd = exact_dist_regs<T, NP>(x[r], Cd + j * CDS);
                    if (dd < dv) {
                        dv = dd;
                        lab = j;
                    }
                }
                if (valid) {
                    cost += dv;
                    if (p.labels) p.labels[row] = p.remap[lab];
                    if (p.counts) atomicAdd(p.counts + p.remap[lab], 1ULL);
                }
            }
            continue;
        }
        float xf[R][NP];
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
            for (int d = 0; d < NP; ++d) xf[r][d] = (float)x[r][d];
        float m1[R], m2[R];
#pragma unroll
        for (int r = 0; r < R; ++r) m1[r] = m2[r] = __int_as_float(0x7f800000);
        // screened values of centre pair q for row r, index embedded (sorted: lo <= hi)
        auto pair_lohi = [&](int q, const float2 (&rec)[RST], int r, float& lo, float& hi) {
            float2 acc = rec[NP];
#pragma unroll
            for (int d = 0; d < NP; ++d) acc = __ffma2_rn(make_float2(xf[r][d], xf[r][d]), rec[d], acc);
            const float da = __int_as_float((__float_as_int(acc.x) & ~tmask) | (2 * q));
            const float db = __int_as_float((__float_as_int(acc.y) & ~tmask) | (2 * q + 1));
            lo = fminf(da, db);
            hi = fmaxf(da, db);
        };
        auto load_rec = [&](int q, float2 (&rec)[RST]) {
#pragma unroll
            for (int h = 0; h < RST / 2; ++h) {
                const float4 v = reinterpret_cast<const float4*>(rp + q * RST)[h];
                rec[2 * h] = make_float2(v.x, v.y);
                rec[2 * h + 1] = make_float2(v.z, v.w);
            }
        };
        // four centres at a time: their (min, second) in 7 min/max ops, merged into the running
        // top-2 with 3 more (2.5 per centre instead of 3.5 pair by pair)
#pragma unroll 1
        for (int q = 0; q + 1 < kpl; q += 2) {
            float2 ra[RST], rb[RST];
            load_rec(q, ra);
            load_rec(q + 1, rb);
#pragma unroll
            for (int r = 0; r < R; ++r) {
                float la, ha, lb, hb;
                pair_lohi(q, ra, r, la, ha);
                pair_lohi(q + 1, rb, r, lb, hb);
                const float l = fminf(la, lb), sgd = fmin3f(fmaxf(la, lb), ha, hb);
                m2[r] = fmin3f(m2[r], sgd, fmaxf(m1[r], l));
                m1[r] = fminf(m1[r], l);
            }
        }
        if (kpl & 1) {
            float2 ra[RST];
            load_rec(kpl - 1, ra);
#pragma unroll
            for (int r = 0; r < R; ++r) {
                float lo, hi;
                pair_lohi(kpl - 1, ra, r, lo, hi);
                m2[r] = fmin3f(m2[r], hi, fmaxf(m1[r], lo));
                m1[r] = fminf(m1[r], lo);
            }
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int64_t row = row0 + r * 32 + lane;
            const bool valid = full || row < m;
            int lab = __float_as_int(m1[r]) & tmask;
            float nn = 0.f;
#pragma unroll
            for (int d = 0; d < NP; ++d) nn = fmaf(xf[r][d], xf[r][d], nn);
            float sx;
            asm("sqrt.approx.f32 %0, %1;" : "=f"(sx) : "f"(nn));
            const float sc = fmaf(sx, 1.0001f, cmax);
            // near ties: the exact reference argmin, warp-parallel over centres (core.hpp:146-157)
            unsigned tie = __ballot_sync(0xffffffffu, valid && !(m2[r] - m1[r] > kap * sc * sc));
            while (tie) {
                const int src = __ffs(tie) - 1;
                tie &= tie - 1;
                T xr[NP];
#pragma unroll
                for (int d = 0; d < NP; ++d) xr[d] = __shfl_sync(0xffffffffu, x[r][d], src);
                double dv = __longlong_as_double(0x7ff0000000000000LL);
                int dj = 0x7fffffff;
                for (int j = lane; j < kv; j += 32) {
                    const double dd = exact_dist_regs<T, NP>(xr, Cd + j * CDS);
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
                const double* cj = Cd + lab * CDS;
                double a0 = 0.0, a1 = 0.0;
#pragma unroll
                for (int d = 0; d < NP; ++d) {
                    const double e = (double)x[r][d] - cj[d];
                    if (d & 1)
                        a1 = fma(e, e, a1);
                    else
                        a0 = fma(e, e, a0);
                }
                cost += a0 + a1;
                if (p.labels) p.labels[row] = p.remap[lab];
                if (p.counts) atomicAdd(p.counts + p.remap[lab], 1ULL);
            }
        }
    }
    cost = warp_sum(cost);
    if (lane == 0) s_wcost[warp] = cost;
    __syncthreads();
    if (tid == 0) {
        double v = 0.0;
        for (int w = 0; w < WARPS; ++w) v += s_wcost[w];
        p.block_cost[blockIdx.x] = v;
    }
}

}  // namespace hpcg
