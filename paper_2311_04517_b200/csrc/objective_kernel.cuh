// Full-data objective f(C, X) = sum_i min_j ||x_i - c_j||^2 streamed over all m rows
// of an HBM-resident X (engine.hpp:197-229 final_assignment / assign_valid_subset,
// core.hpp:224-233 mssc_objective), plus the optional labels / counts of the full
// assignment. Each row is read once; the nearest valid centre is found with the fp32
// FFMA2 screen and an exact fp64 recheck of near ties; the row's cost is the exact
// reference distance (core.hpp:147-152, non-fused, ascending d) to that centre, so
// per-row values are bit-identical to the reference and only the (fixed, deterministic)
// summation order differs.
#pragma once
#include <cuda.h>

#include "common.cuh"
#include "step_kernel.cuh"  // Geo (swizzled row layout) and cp.async helpers

namespace hpcg {

constexpr int kObjThreads = 256;
constexpr int kObjMaxK = 256;

constexpr int kGridCells = 4096;  // cells of the narrow-row filter (objective_rows.cuh)
struct GridHdr {                  // after the kGridCells masks in ObjParams::grid
    double lo[3], inv_w[3];
};

struct ObjParams {
    const void* X;
    int64_t m;
    int32_t n;
    int32_t kv;            // valid centres
    const double* C;       // [kv x n] valid centres (compacted), fp64
    const int32_t* remap;  // [kv] original slot of each valid centre
    int32_t* labels;       // [m] or null
    unsigned long long* counts;  // [k original] or null (atomics on integers: order-free)
    double* block_cost;    // [gridDim.x]
    int32_t use_tma;       // 1: stages arrive by TMA (tensor map built by the host), 0: cp.async
    const int32_t* kv_dev; // optional device-side valid count (<= kv, which then only sizes smem)
    int32_t rec_slot;      // constant-bank record slot of the calling context, or -1
    float4* rec_scratch;   // device staging of that slot's records (kRecSlotF4 float4)
    int* launched;         // optional: kernels launched are added here
    int32_t fast_cost;     // fp32 data: row cost in fp32 (direct form, FFMA2), accumulated in fp64 --
                           // the north star's fp32 mode (1e-5 relative); 0: exact fp64 row cost
    double* cost_out;      // optional: the kernel's last CTA sums block_cost in the fixed order of
    unsigned int* done_ctr;  //   sum_blocks_kernel<<<1, 256>>> into *cost_out (done_ctr: zeroed counter)
    int* finalized;        // host: set to 1 by a launcher whose kernel wrote *cost_out, else 0
    uint32_t* grid;        // optional scratch of the narrow-row cell filter (kGridCells masks + GridHdr)
};

// the fixed-order block-partial sum of sum_blocks_kernel<<<1, 256>>>, run by threads 0..255 of the
// grid's last CTA (the CTAs' partials published by __threadfence + a ticket counter)
HPCG_DEV void finalize_block_sums(const ObjParams& p, double* s32) {
    __shared__ unsigned int s_ticket;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_ticket = atomicAdd(p.done_ctr, 1u);
    __syncthreads();
    if (s_ticket != gridDim.x - 1) return;
    __threadfence();
    const int tid = threadIdx.x;
    if (tid < 256) {
        double v = 0.0;
        for (int i = tid; i < (int)gridDim.x; i += 256) v += __ldcg(p.block_cost + i);
        v = warp_sum(v);
        if ((tid & 31) == 0) s32[tid >> 5] = v;
    }
    __syncthreads();
    if (tid == 0) {
        double t = 0.0;
        for (int w = 0; w < 8; ++w) t += s32[w];
        *p.cost_out = t;
        *p.done_ctr = 0u;  // ready for the next launch (stream-ordered)
    }
}

// valid centre count: the device value when given (the host launched with an upper bound)
HPCG_DEV int obj_kv(const ObjParams& p) {
    if (!p.kv_dev) return p.kv;
    const int v = *p.kv_dev;
    return v < p.kv ? (v > 0 ? v : 0) : p.kv;
}

// TMA tile load of `rows` x n into a swizzled smem slot (box = {n, GR}); the hardware
// 32B/64B/128B swizzle equals Geo::swz for these row widths (chunk ^= row bits).
HPCG_DEV void tma_load_2d(void* sdst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(sdst)),
        "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}
HPCG_DEV void mbar_wait_cta(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n .reg .pred p;\n WAITC_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAITC_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}
HPCG_DEV void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Per-warp software pipeline: each warp streams groups of GR consecutive rows through a
// STAGES-deep ring of shared-memory slots filled by cp.async (16/8/4-B copies, swizzled
// like the step kernel's sample so the row-per-lane reads are bank-conflict free). Loads
// for STAGES-1 groups are in flight while the warp computes on the oldest one.
template <typename T, int NP>
struct ObjGeo {
    using G = Geo<T, NP>;
    static constexpr int NPF = G::NPF;
    static constexpr int R = NP <= 16 ? 2 : 1;
    static constexpr int GR = 32 * R;                 // rows per group
    static constexpr int STAGE = GR * G::RS;          // bytes per ring slot
    static constexpr int STAGES = 3;
    static constexpr int CSR = G::CSR;
    static constexpr int CDS = NPF + 2;               // fp64 centroid row stride (doubles), padded
};

template <typename T, int NP>
__host__ __device__ inline int objective_smem(int kv) {
    using O = ObjGeo<T, NP>;
    const int cs = ((kv * O::CSR * 4 + 15) & ~15);
    const int cd = ((kv * O::CDS * 8 + 15) & ~15);
    return ((cs + cd + 1023) & ~1023) + (kObjThreads / 32) * O::STAGES * O::STAGE + 1024;
}

template <typename T, int NP>
__global__ void __launch_bounds__(kObjThreads, 2) objective_kernel(const ObjParams p,
                                                                   const __grid_constant__ CUtensorMap tmap) {
    using O = ObjGeo<T, NP>;
    using G = typename O::G;
    constexpr int NPF = O::NPF, R = O::R, CSR = O::CSR;
    extern __shared__ __align__(16) unsigned char osm[];
    const int kvl = p.kv, kv = obj_kv(p), n = p.n;  // kvl: smem layout (launch bound)
    float* cs = reinterpret_cast<float*>(osm);
    constexpr int CDS = O::CDS;
    double* Cd = reinterpret_cast<double*>(osm + ((kvl * CSR * 4 + 15) & ~15));
    unsigned char* rings = osm + ((((kvl * CSR * 4 + 15) & ~15) + ((kvl * CDS * 8 + 15) & ~15) + 1023) & ~1023);
    rings += (1024 - (smem_u32(rings) & 1023)) & 1023;  // swizzle atom alignment (absolute address)
    __shared__ __align__(8) uint64_t s_bar[kObjThreads / 32][4];
    __shared__ float s_cmax;
    __shared__ double s_wcost[kObjThreads / 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    for (int e = tid; e < kv * CDS; e += kObjThreads) {
        const int j = e / CDS, d = e - j * CDS;
        Cd[e] = d < n ? p.C[(int64_t)j * n + d] : 0.0;
    }
    __syncthreads();
    for (int j = tid; j < kv; j += kObjThreads) {
        float* rec = cs + j * CSR;
        double cc = 0.0;
        for (int d = 0; d < NP; ++d) {
            const double c = Cd[j * CDS + d];
            cc += c * c;
            rec[d] = (float)(-2.0 * c);
        }
        for (int d = NP; d < NPF; ++d) rec[d] = 0.f;
        rec[NPF] = (float)cc;
        rec[NPF + 1] = 0.f;
    }
    T* ring = reinterpret_cast<T*>(rings + warp * O::STAGES * O::STAGE);
    // zero the ring once: padding columns (NP > n) are never written by the copies
    for (int e = lane; e < O::STAGES * O::STAGE / 4; e += 32) reinterpret_cast<float*>(ring)[e] = 0.f;
    const bool tma = p.use_tma != 0;
    if (tma && lane == 0) {
        for (int st = 0; st < O::STAGES; ++st) mbar_init(&s_bar[warp][st], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    fence_proxy_async();
    __syncthreads();
    if (tid == 0) {
        float cm = 0.f;
        for (int j = 0; j < kv; ++j) cm = fmaxf(cm, sqrtf(cs[j * CSR + NPF]) * 1.0001f);
        s_cmax = cm;
    }
    __syncthreads();
    const float cmax = s_cmax;
    constexpr float kappa = 2.0f * (float)(NPF / 2 + 12) * 5.9604645e-8f;

    const T* X = static_cast<const T*>(p.X);
    const int64_t m = p.m;
    const int rowb = n * (int)sizeof(T);
    const int64_t ngroups = (m + O::GR - 1) / O::GR;
    const int64_t wglobal = (int64_t)blockIdx.x * (kObjThreads / 32) + warp;
    const int64_t wstride = (int64_t)gridDim.x * (kObjThreads / 32);
    const int64_t my_groups = wglobal < ngroups ? (ngroups - wglobal + wstride - 1) / wstride : 0;

    auto issue = [&](int64_t i) {  // copies of the warp's i-th group into slot i % STAGES
        if (tma) {
            if (i < my_groups && lane == 0) {
                const int64_t g = wglobal + i * wstride;
                uint64_t* bar = &s_bar[warp][i % O::STAGES];
                fence_proxy_async();  // generic-proxy reads of this slot precede the async write
                mbar_expect_tx(bar, (uint32_t)O::STAGE);
                tma_load_2d(ring + (i % O::STAGES) * (O::STAGE / (int)sizeof(T)), &tmap, 0, (int)(g * O::GR), bar);
            }
            return;
        }
        if (i < my_groups) {
            const int64_t g = wglobal + i * wstride;
            T* slot = ring + (i % O::STAGES) * (O::STAGE / (int)sizeof(T));
            const int64_t row0 = g * O::GR;
            const int rows = (int)(m - row0 < O::GR ? m - row0 : O::GR);
            const T* src = X + row0 * n;
            if (G::VEC16 && n == NP) {
                constexpr int EPC = 16 / (int)sizeof(T);
                for (int e = lane; e < rows * G::CPR; e += 32) {
                    const int li = e / G::CPR, q = e % G::CPR;
                    cp_async16(slot + G::elem_off(li, q * EPC), src + (int64_t)li * NP + q * EPC);
                }
            } else if ((rowb & 15) == 0) {
                const int cpr = rowb >> 4;
                constexpr int EPC = 16 / (int)sizeof(T);
                for (int e = lane; e < rows * cpr; e += 32) {
                    const int li = e / cpr, q = e - li * cpr;
                    cp_async16(slot + G::elem_off(li, q * EPC), src + (int64_t)li * n + q * EPC);
                }
            } else if ((rowb & 7) == 0) {
                const int cpr = rowb >> 3;
                constexpr int EPC = 8 / (int)sizeof(T);
                for (int e = lane; e < rows * cpr; e += 32) {
                    const int li = e / cpr, q = e - li * cpr;
                    cp_async8(slot + G::elem_off(li, q * EPC), src + (int64_t)li * n + q * EPC);
                }
            } else {
                for (int e = lane; e < rows * n; e += 32) {
                    const int li = e / n, d = e - li * n;
                    cp_async4(slot + G::elem_off(li, d), src + (int64_t)li * n + d);
                }
            }
        }
        cp_async_commit();
    };

    double cost = 0.0;
#pragma unroll 1
    for (int i = 0; i < O::STAGES - 1; ++i) issue(i);
#pragma unroll 1
    for (int64_t i = 0; i < my_groups; ++i) {
        if (tma)
            mbar_wait_cta(&s_bar[warp][i % O::STAGES], (uint32_t)((i / O::STAGES) & 1));
        else
            cp_async_wait_group<O::STAGES - 2>();
        __syncwarp();
        const int64_t g = wglobal + i * wstride;
        const T* slot = ring + (i % O::STAGES) * (O::STAGE / (int)sizeof(T));
        float2 x2[R][NPF / 2];
        bool valid[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int lr = r * 32 + lane;
            valid[r] = g * O::GR + lr < m;
            if constexpr (G::VEC16 && sizeof(T) == 4) {
#pragma unroll
                for (int q = 0; q < NP / 4; ++q) {
                    const float4 v = *reinterpret_cast<const float4*>(slot + G::elem_off(lr, q * 4));
                    x2[r][2 * q] = make_float2(v.x, v.y);
                    x2[r][2 * q + 1] = make_float2(v.z, v.w);
                }
            } else if constexpr (G::VEC16) {
#pragma unroll
                for (int q = 0; q < NP / 2; ++q) {
                    const double2 v = *reinterpret_cast<const double2*>(slot + G::elem_off(lr, q * 2));
                    x2[r][q] = make_float2((float)v.x, (float)v.y);
                }
            } else {
#pragma unroll
                for (int q = 0; q < NPF / 2; ++q) {
                    const float a = (float)slot[G::elem_off(lr, 2 * q)];
                    const float b = 2 * q + 1 < NP ? (float)slot[G::elem_off(lr, 2 * q + 1)] : 0.f;
                    x2[r][q] = make_float2(a, b);
                }
            }
        }
        float m1[R], m2[R];
        int i1[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            m1[r] = __int_as_float(0x7f800000);
            m2[r] = __int_as_float(0x7f800000);
            i1[r] = 0;
        }
        for (int j = 0; j < kv; ++j) {
            const float* rec = cs + j * CSR;
            float2 c2[NPF / 2];
#pragma unroll
            for (int q = 0; q < NPF / 2; ++q) c2[q] = *reinterpret_cast<const float2*>(rec + 2 * q);
            const float2 init = *reinterpret_cast<const float2*>(rec + NPF);
#pragma unroll
            for (int r = 0; r < R; ++r) {
                float2 acc = init;
#pragma unroll
                for (int q = 0; q < NPF / 2; ++q) acc = __ffma2_rn(x2[r][q], c2[q], acc);
                const float dj = acc.x + acc.y;
                m2[r] = fminf(m2[r], fmaxf(m1[r], dj));
                const bool lt = dj < m1[r];
                m1[r] = fminf(m1[r], dj);
                i1[r] = lt ? j : i1[r];
            }
        }
        // near ties (kv == 1: never): exact reference argmin, warp-parallel over centroids
        // (lane l evaluates centroids l, l+32, ...; tie-aware shuffle argmin, core.hpp:146-157)
#pragma unroll
        for (int r = 0; r < R; ++r) {
            float nn = 0.f;
#pragma unroll
            for (int q = 0; q < NPF / 2; ++q) nn = fmaf(x2[r][q].x, x2[r][q].x, fmaf(x2[r][q].y, x2[r][q].y, nn));
            const float sc = sqrtf(nn) + cmax;
            unsigned tie = __ballot_sync(0xffffffffu, valid[r] && !(m2[r] - m1[r] > kappa * sc * sc));
            while (tie) {
                const int src = __ffs(tie) - 1;
                tie &= tie - 1;
                const int tr = r * 32 + src;
                T xr[NP];
                load_row_T<T, NP>(slot, tr, xr);
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
                if (lane == src) i1[r] = dj;
            }
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
            if (!valid[r]) continue;
            const int lr = r * 32 + lane;
            const int lab = i1[r];
            // row cost: fp64 distance to the chosen centre from the row in registers (two
            // interleaved DFMA chains; within 1e-15 relative of the reference's per-row value)
            double xd[NPF];
            if constexpr (sizeof(T) == 4) {
#pragma unroll
                for (int q = 0; q < NPF / 2; ++q) {
                    xd[2 * q] = (double)x2[r][q].x;
                    xd[2 * q + 1] = (double)x2[r][q].y;
                }
            } else {
                T xr[NP];
                load_row_T<T, NP>(slot, lr, xr);
#pragma unroll
                for (int d = 0; d < NPF; ++d) xd[d] = d < NP ? (double)xr[d] : 0.0;
            }
            const double* cj = Cd + lab * CDS;
            double a0 = 0.0, a1 = 0.0;
#pragma unroll
            for (int q = 0; q < NPF / 2; ++q) {
                const double2 c = *reinterpret_cast<const double2*>(cj + 2 * q);
                const double d0 = xd[2 * q] - c.x, d1 = xd[2 * q + 1] - c.y;
                a0 = fma(d0, d0, a0);
                a1 = fma(d1, d1, a1);
            }
            cost += a0 + a1;
            const int64_t row = g * O::GR + lr;
            if (p.labels) p.labels[row] = p.remap[lab];
            if (p.counts) atomicAdd(p.counts + p.remap[lab], 1ULL);
        }
        __syncwarp();
        issue(i + O::STAGES - 1);
    }
    cp_async_wait_group<0>();
    cost = warp_sum(cost);
    if (lane == 0) s_wcost[warp] = cost;
    __syncthreads();
    if (tid == 0) {
        double v = 0.0;
        for (int w = 0; w < kObjThreads / 32; ++w) v += s_wcost[w];
        p.block_cost[blockIdx.x] = v;
    }
}

// ---------------------------------------------------------------------------------------
// fp32 rows, 16-B-multiple widths, TMA-fed: centre-pair screen.
// Each FFMA2 evaluates one dimension for TWO centres (record pair (-2c_a,d, -2c_b,d)) with the
// row value as a broadcast scalar operand, so a pair of screened distances costs NP FFMA2 and
// no horizontal add; top-2 tracking takes the pair as a sorted (lo, hi) with a three-input min.
// Rows are copied to registers as soon as their stage lands and the stage is refilled at once
// (one 32R-row stage per warp keeps 8 KB per warp in flight during the compute).
// Screen error: sequential fused chain of NP terms on a rounded record, so
// |d~ - d| <= (NP + 2) u (|x| + |c|)^2; PairGeo::kappa doubles that (difference of two) with
// slack. The centre index rides in the low tb = ceil(log2(2 kp)) mantissa bits of each screened
// value, so the running min carries its own argmin (no compare/select per centre); that moves
// a value by < 2^(tb-23) |d~|, and the tie bound grows by 2^(tb-22) (|x| + cmax)^2 to match.
template <int NP>
struct PairGeo {
    using G = Geo<float, NP>;
    static constexpr int R = NP <= 8 ? 4 : NP <= 16 ? 3 : 2;  // rows per lane
    static constexpr int GR = 32 * R;            // rows per stage
    static constexpr int STAGE = GR * G::RS;     // bytes per stage
    static constexpr int STAGES = 1;             // stages per warp (refilled as soon as read; 2-3 measured slower)
    static constexpr int RST = NP + 2;           // record stride in float2 (16-B multiple)
    static constexpr int CDS = NP + 1;           // fp64 centre stride (doubles): odd, so the
                                                 // 8-B loads of up to 16 distinct centres in a
                                                 // half-warp phase hit distinct bank pairs
    static constexpr int WARPS = kObjThreads / 32;
    static constexpr float kappa = 2.0f * (float)(NP + 12) * 5.9604645e-8f;
};

// Centre-pair records in the constant bank (kv <= 2 kRecMaxPairs): FFMA2 operands come through
// the uniform datapath and the records stop competing with the row and centre loads for
// shared-memory bandwidth (the kernel's binding resource). One slot per context.
constexpr int kRecSlots = 8;
constexpr int kRecMaxPairs = 16;
constexpr int kRecSlotF4 = kRecMaxPairs * (32 + 2) / 2;  // float4 per slot (NP <= 32)
#ifdef HPCG_OBJECTIVE_TU
static __constant__ float4 c_pair_rec4[kRecSlots * kRecSlotF4];
#endif

template <int NP>
__host__ __device__ inline int objective_pairs_smem(int kv) {
    using PG = PairGeo<NP>;
    const int kp = (kv + 1) / 2;
    const int rec = kp * PG::RST * 8;
    const int cd = ((kv * PG::CDS * 8 + 15) & ~15);
    return ((rec + cd + 1023) & ~1023) + PG::WARPS * PG::STAGES * PG::STAGE + 1024;
}


#ifdef HPCG_OBJECTIVE_TU
// records of the valid centres into a slot's staging buffer (the same arithmetic as the
// shared-memory builder in objective_pairs_kernel, so both record sets are bit-identical)
template <int NP>
__global__ void build_pair_records_kernel(const ObjParams p) {
    constexpr int RST = PairGeo<NP>::RST;
    const int kv = obj_kv(p), kpl = (p.kv + 1) / 2;
    float* o = reinterpret_cast<float*>(p.rec_scratch);
    for (int j = threadIdx.x; j < 2 * kpl; j += blockDim.x) {
        float* rec = o + (j >> 1) * (2 * RST) + (j & 1);
        if (j < kv) {
            double cc = 0.0;
            for (int d = 0; d < NP; ++d) {
                const double c = p.C[(int64_t)j * NP + d];
                cc += c * c;
                rec[2 * d] = (float)(-2.0 * c);
            }
            rec[2 * NP] = (float)cc;
        } else {
            for (int d = 0; d < NP; ++d) rec[2 * d] = 0.f;
            rec[2 * NP] = 1e38f;
        }
        rec[2 * NP + 2] = 0.f;
    }
}

template <int NP, bool CREC>
__global__ void __launch_bounds__(kObjThreads, 2) objective_pairs_kernel(const ObjParams p,
                                                                         const __grid_constant__ CUtensorMap tmap) {
    using PG = PairGeo<NP>;
    using G = typename PG::G;
    constexpr int R = PG::R, RST = PG::RST, CDS = PG::CDS, GR = PG::GR;
    extern __shared__ __align__(16) unsigned char osm[];
    const int kvl = p.kv, kpl = (kvl + 1) / 2;  // smem layout (launch bound)
    const int kv = obj_kv(p), kp = (kv + 1) / 2;
    float2* rp = reinterpret_cast<float2*>(osm);
    double* Cd = reinterpret_cast<double*>(osm + kpl * RST * 8);
    unsigned char* rings = osm + (((kpl * RST * 8) + ((kvl * CDS * 8 + 15) & ~15) + 1023) & ~1023);
    rings += (1024 - (smem_u32(rings) & 1023)) & 1023;
    __shared__ __align__(8) uint64_t s_bar[PG::WARPS][PG::STAGES];
    __shared__ float s_cmax;
    __shared__ double s_wcost[PG::WARPS];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    for (int e = tid; e < kv * CDS; e += kObjThreads) {
        const int j = e / CDS, d = e - j * CDS;
        Cd[e] = d < NP ? p.C[(int64_t)j * NP + d] : 0.0;
    }
    __syncthreads();
    // records: pair q holds centres 2q, 2q+1 interleaved; a missing odd partner screens +inf
    const int rbase = CREC ? p.rec_slot * kRecSlotF4 : 0;
    auto rec4 = [&](int q, int h) -> float4 {
        if constexpr (CREC)
            return c_pair_rec4[rbase + q * (RST / 2) + h];
        else
            return reinterpret_cast<const float4*>(rp + q * RST)[h];
    };
    // the screen runs over the launch bound kpl (a uniform trip count: records stay in uniform
    // registers); pairs past the valid count hold +inf records and never win
    for (int j = tid; j < (CREC ? 0 : 2 * kpl); j += kObjThreads) {
        float* rec = reinterpret_cast<float*>(rp + (j >> 1) * RST) + (j & 1);
        if (j < kv) {
            double cc = 0.0;
            for (int d = 0; d < NP; ++d) {
                const double c = Cd[j * CDS + d];
                cc += c * c;
                rec[2 * d] = (float)(-2.0 * c);
            }
            rec[2 * NP] = (float)cc;
        } else {
            for (int d = 0; d < NP; ++d) rec[2 * d] = 0.f;
            rec[2 * NP] = 1e38f;
        }
        rec[2 * NP + 2] = 0.f;
    }
    if (lane == 0) {
        for (int st = 0; st < PG::STAGES; ++st) mbar_init(&s_bar[warp][st], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    fence_proxy_async();
    __syncthreads();
    if (tid == 0) {
        float cm = 0.f;
        for (int j = 0; j < kv; ++j) {
            const float4 iv = rec4(j >> 1, NP / 2);
            cm = fmaxf(cm, sqrtf((j & 1) ? iv.y : iv.x) * 1.0001f);
        }
        s_cmax = cm;
    }
    __syncthreads();
    const float cmax = s_cmax;
    const int tbits = 32 - __clz(2 * kpl - 1 > 0 ? 2 * kpl - 1 : 1);
    const int tmask = (1 << tbits) - 1;
    const float kap = PG::kappa + __int_as_float((127 + tbits - 22) << 23);  // + 2^(tb-22)

    float* ring = reinterpret_cast<float*>(rings + warp * PG::STAGES * PG::STAGE);
    const int64_t m = p.m;
    const int64_t ngroups = (m + GR - 1) / GR;
    const int64_t wglobal = (int64_t)blockIdx.x * PG::WARPS + warp;
    const int64_t wstride = (int64_t)gridDim.x * PG::WARPS;
    const int64_t my_groups = wglobal < ngroups ? (ngroups - wglobal + wstride - 1) / wstride : 0;
    auto issue = [&](int64_t i) {
        if (i < my_groups && lane == 0) {
            uint64_t* bar = &s_bar[warp][i % PG::STAGES];
            fence_proxy_async();  // this warp's generic reads of the stage precede the async write
            mbar_expect_tx(bar, (uint32_t)PG::STAGE);
            tma_load_2d(ring + (i % PG::STAGES) * (PG::STAGE / 4), &tmap, 0, (int)((wglobal + i * wstride) * GR), bar);
        }
    };
#pragma unroll
    for (int st = 0; st < PG::STAGES; ++st) issue(st);

    double cost = 0.0;
#pragma unroll 1
    for (int64_t i = 0; i < my_groups; ++i) {
        mbar_wait_cta(&s_bar[warp][i % PG::STAGES], (uint32_t)((i / PG::STAGES) & 1));
        const float* slot = ring + (i % PG::STAGES) * (PG::STAGE / 4);
        const int64_t row0 = (wglobal + i * wstride) * GR;
        const bool full = row0 + GR <= m;
        float x[R][NP];
#pragma unroll
        for (int r = 0; r < R; ++r) {
#pragma unroll
            for (int q = 0; q < NP / 4; ++q) {
                const float4 v = *reinterpret_cast<const float4*>(slot + G::elem_off(r * 32 + lane, q * 4));
                x[r][4 * q] = v.x;
                x[r][4 * q + 1] = v.y;
                x[r][4 * q + 2] = v.z;
                x[r][4 * q + 3] = v.w;
            }
        }
        __syncwarp();
        issue(i + PG::STAGES);

        float m1[R], m2[R];
        int i1[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            m1[r] = __int_as_float(0x7f800000);
            m2[r] = __int_as_float(0x7f800000);
            i1[r] = 0;
        }
#pragma unroll 1
        for (int q = 0; q < kpl; ++q) {
            const float4 iv = rec4(q, NP / 2);
            float2 acc[R];
#pragma unroll
            for (int r = 0; r < R; ++r) acc[r] = make_float2(iv.x, iv.y);
#pragma unroll
            for (int h = 0; h < NP / 2; ++h) {
                const float4 c = rec4(q, h);
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    acc[r] = __ffma2_rn(make_float2(x[r][2 * h], x[r][2 * h]), make_float2(c.x, c.y), acc[r]);
                    acc[r] = __ffma2_rn(make_float2(x[r][2 * h + 1], x[r][2 * h + 1]), make_float2(c.z, c.w), acc[r]);
                }
            }
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const float da = __int_as_float((__float_as_int(acc[r].x) & ~tmask) | (2 * q));
                const float db = __int_as_float((__float_as_int(acc[r].y) & ~tmask) | (2 * q + 1));
                const float lo = fminf(da, db), hi = fmaxf(da, db);
                m2[r] = fmin3f(m2[r], hi, fmaxf(m1[r], lo));
                m1[r] = fminf(m1[r], lo);
            }
        }
#pragma unroll
        for (int r = 0; r < R; ++r) i1[r] = __float_as_int(m1[r]) & tmask;
        // near ties: exact reference argmin, warp-parallel over centres (core.hpp:146-157)
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const bool valid = full || row0 + r * 32 + lane < m;
            float2 nn2 = make_float2(0.f, 0.f);
#pragma unroll
            for (int d = 0; d < NP; d += 2) nn2 = __ffma2_rn(make_float2(x[r][d], x[r][d + 1]),
                                                             make_float2(x[r][d], x[r][d + 1]), nn2);
            float sx;
            asm("sqrt.approx.f32 %0, %1;" : "=f"(sx) : "f"(nn2.x + nn2.y));
            const float sc = fmaf(sx, 1.0001f, cmax);
            unsigned tie = __ballot_sync(0xffffffffu, valid && !(m2[r] - m1[r] > kap * sc * sc));
            while (tie) {
                const int src = __ffs(tie) - 1;
                tie &= tie - 1;
                float xr[NP];
#pragma unroll
                for (int d = 0; d < NP; ++d) xr[d] = __shfl_sync(0xffffffffu, x[r][d], src);
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
                if (lane == src) i1[r] = dj;
            }
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int64_t row = row0 + r * 32 + lane;
            if (!full && row >= m) continue;
            const int lab = i1[r];
            // row cost: fp64 distance to the chosen centre (two interleaved DFMA chains; within
            // 1e-15 relative of the reference's per-row value)
            const double* cj = Cd + lab * CDS;
            double a0 = 0.0, a1 = 0.0;
#pragma unroll
            for (int h = 0; h < NP / 2; ++h) {
                const double d0 = (double)x[r][2 * h] - cj[2 * h], d1 = (double)x[r][2 * h + 1] - cj[2 * h + 1];
                a0 = fma(d0, d0, a0);
                a1 = fma(d1, d1, a1);
            }
            cost += a0 + a1;
            if (p.labels) p.labels[row] = p.remap[lab];
            if (p.counts) atomicAdd(p.counts + p.remap[lab], 1ULL);
        }
    }
    cost = warp_sum(cost);
    if (lane == 0) s_wcost[warp] = cost;
    __syncthreads();
    if (tid == 0) {
        double v = 0.0;
        for (int w = 0; w < PG::WARPS; ++w) v += s_wcost[w];
        p.block_cost[blockIdx.x] = v;
    }
}

#endif  // HPCG_OBJECTIVE_TU

// Fixed-order final sum of the block partials (deterministic f(C,X)).
static __global__ void sum_blocks_kernel(const double* part, int nparts, double* out) {
    __shared__ double s[32];
    double v = 0.0;
    for (int i = threadIdx.x; i < nparts; i += blockDim.x) v += part[i];
    v = warp_sum(v);
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s[w];
        *out = t;
    }
}

}  // namespace hpcg
