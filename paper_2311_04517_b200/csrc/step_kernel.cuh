// The HPClust worker step on sm_100a: sample gather -> greedy K-means++ reseeding of
// degenerate slots -> Lloyd to convergence -> keep-the-best acceptance, for many
// workers at once. One thread-block CLUSTER per worker; the worker's sample is split
// row-wise over the cluster's CTAs and stays resident in their shared memory for the
// whole step (it is read from HBM exactly once). Cross-CTA reductions (Lloyd partial
// sums, K-means++ CDF totals / draws / candidate costs) go through distributed shared
// memory in fixed rank order, so every result is bit-reproducible run to run.
//
// Reference semantics followed (paths under /root/reference/proj/include/hpclust/):
//   gather          engine.hpp:165-177 (draw order kept; indices supplied or Philox PRP)
//   seeding         seeding.hpp:20-42, 47-105, 125-133; rng.hpp:83-93
//   assign pass     core.hpp:138-207 (strict <, ties -> lowest index)
//   Lloyd loop      lloyd.hpp:75-89, 100-164 (reciprocal-multiply means, fixed point,
//                   rel-tol, max-iters, closing pass, monotone guard)
//   acceptance      engine.hpp:251-266 (strict <)
//   n_d accounting  core.hpp:205, seeding.hpp:38
#pragma once
#include "common.cuh"

namespace hpcg {

#ifndef HPCG_STEP_THREADS
#define HPCG_STEP_THREADS 512
#endif
constexpr int kStepThreads = HPCG_STEP_THREADS;  // 512: one CTA per SM, 16 warps; 256: two CTAs per SM
constexpr int kStepWarps = kStepThreads / 32;
constexpr int kStepMinBlocks = kStepThreads >= 512 ? 1 : 512 / kStepThreads;  // 256: two CTAs per SM at 128 registers
constexpr int kMaxK = 32;          // label fits u8 and the per-warp partial table fits smem
constexpr int kMaxCandidates = 4;  // K-means++ candidates per slot (reference default 3) in one sweep

constexpr int kMaxShards = 8;      // row shards of a dataset (one per GPU of a node)

enum StepErr : int32_t { kErrNone = 0, kErrDegenerateInit = 1, kErrMonotone = 2 };

struct StepParams {
    // sample source
    const void* X;
    int64_t m;
    int32_t n;
    int64_t s;
    int32_t W;            // workers in this launch (one cluster each)
    int32_t geo_W;        // worker count the launch geometry is chosen for (0: W). A multi-rank engine
                          // passes the all-rank total, so every rank partitions a sample exactly as
                          // one engine with every worker would (bit-identical sums)
    int32_t sample_mode;  // 0 explicit idx[W*s], 1 Philox PRP over [0,m), 2 contiguous (X is [W*s x n])
    const int64_t* idx;
    uint64_t key;        // Philox key (sample PRP and K-means++ draws)
    uint32_t prp_a, prp_b;  // sample PRP moduli (SamplePRP::moduli of m)
    float prp_inv_b;
    uint32_t round;      // Philox counter component
    int32_t worker_base;  // global id of local worker 0 (Philox stream id)
    // initial centroids
    const double* init_c;
    int64_t init_stride;  // doubles between consecutive workers' inits; 0 = one shared init
    const uint8_t* init_f;
    int64_t initf_stride;
    const int64_t* shared_version;  // if set and *shared_version == 0: init is all-degenerate
    // K-means++
    int32_t candidates;
    int32_t seed_mode;  // 0 explicit draws, 1 Philox
    const int64_t* first_row;
    const double* units;
    int32_t units_stride;
    // Lloyd
    int32_t k;
    int32_t max_iters;
    double rel_tol;
    int32_t do_lloyd;
    // row-sharded X (multi-GPU global sampling: remote shards peer-mapped): nshards > 1 selects
    // the shard of global row g by the cumulative row ends; nshards <= 1: X holds every row
    int32_t nshards;
    const void* shard_ptr[kMaxShards];
    int64_t shard_end[kMaxShards];
    // geometry chosen by the host
    int32_t rows_cap;  // max rows per CTA (smem layout)
    // outputs (indexed by local worker)
    double* out_c;
    uint8_t* out_f;
    double* out_obj;
    int32_t* out_iters;
    int32_t* out_stop;
    int64_t* out_nd;
    int32_t* out_filled;
    int32_t* out_err;
    int32_t* out_labels;  // [W*s] or null
    int64_t* out_counts;  // [W*k] or null
    double* out_hist;     // [W*hist_cap] or null
    int32_t hist_cap;
    int32_t* out_hist_len;
    // keep-the-best acceptance (engine); null -> no acceptance
    double* inc_c;
    uint8_t* inc_f;
    double* inc_obj;
    uint8_t* accepted;
    // free-running schedule: go[wl] == 0 -> this worker's cluster does nothing (its deadline or
    // sample cap was reached when the schedule prepared the step); null -> every worker runs
    const int32_t* go;
    // optional phase timeline (ns, %globaltimer) per CTA: [W*C][kTraceSlots]
    int64_t* trace;
    int32_t trace_mode;  // 0: first Lloyd pass in detail, 1: first K-means++ slot in detail
};

constexpr int kTraceSlots = 32;

// address of global row g (n elements of T) through the shard table
template <typename T>
HPCG_DEV const T* row_ptr(const StepParams& p, int64_t g) {
    if (p.nshards <= 1) return static_cast<const T*>(p.X) + g * p.n;
    int sh = 0;
    while (sh + 1 < p.nshards && g >= p.shard_end[sh]) ++sh;
    const int64_t base = sh ? p.shard_end[sh - 1] : 0;
    return static_cast<const T*>(p.shard_ptr[sh]) + (g - base) * p.n;
}
template <int V>
struct IntC {
    static constexpr int value = V;
};

HPCG_DEV int64_t gtimer() {
    int64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// ------------------------------------------------------------- smem geometry
template <typename T, int NP>
struct Geo {
    static constexpr int RS = NP * (int)sizeof(T);            // sample row bytes in smem
    static constexpr bool VEC16 = (RS % 16) == 0;              // 16-B chunks (swizzled)
    static constexpr int CPR = VEC16 ? RS / 16 : 1;            // chunks per row
    static constexpr int NPF = (NP + 1) & ~1;                  // fp32 screen dims (pairs)
    static constexpr int CSR = ((NPF + 2) + 3) & ~3;           // screen record floats (16-B mult)
    static constexpr int RST = NPF + 2;                        // centre-pair record stride (float2)
    static constexpr int R = (NP <= 16 && kStepThreads <= 512) ? 4 : 2;  // rows per thread in the assign pass
    static constexpr int GROUP = 32 * R;                       // rows per warp group
    static constexpr int LPR = NP <= 1 ? 1 : NP <= 2 ? 2 : NP <= 4 ? 4 : NP <= 8 ? 8 : NP <= 16 ? 16 : 32;
    static constexpr int RPS = 32 / LPR;                       // rows per warp step in the update

    // 2-adic swizzle of 16-B chunks so 8 consecutive rows' chunk q hit 8 distinct
    // bank groups.
    HPCG_DEV static int swz(int row) {
        if constexpr (!VEC16) {
            return 0;
        } else if constexpr ((CPR & 7) == 0) {
            return row & 7;
        } else if constexpr ((CPR & 3) == 0) {
            return (row >> 1) & 3;
        } else if constexpr ((CPR & 1) == 0) {
            return (row >> 2) & 1;
        } else {
            return 0;
        }
    }
    HPCG_DEV static int elem_off(int row, int d) {  // element offset (in T) of (row, d)
        if constexpr (VEC16) {
            constexpr int EPC = 16 / (int)sizeof(T);
            return row * NP + (((d / EPC) ^ swz(row)) * EPC) + (d % EPC);
        } else {
            return row * NP + d;
        }
    }
};

struct SmemLayout {  // byte offsets into dynamic smem
    int samp, cm, cs, part, scratch, total;
    int labels, pos, perm, wpart, d2, gidx, xnorm, wlist, nflag;
};

// per-warp exact-work list: the entries one step appends (ncand per row) plus a carried
// partial batch of < 32 (the D^2 update appends two chunks per step, hence the floor of 2)
__host__ __device__ constexpr int list_cap(int ncand) { return 32 * ((ncand > 2 ? ncand : 2) + 1); }

// cluster exchange buffers (doubles): all-to-all slots for the seeding scalars, and the
// reduce-scatter / all-gather slices of the Lloyd partial (k*NP sums + k counts + cost)
constexpr int kXchSmall = 2 * kMaxCandidates;
__host__ __device__ inline int xch_slice(int k, int NP, int C) { return (k * NP + k + 1 + C - 1) / C; }
__host__ __device__ inline int xch_doubles(int k, int NP, int C) {
    return 2 * C * kXchSmall + 2 * C * xch_slice(k, NP, C) + 2 * C * xch_slice(k, NP, C);
}

template <typename T, int NP>
__host__ __device__ inline SmemLayout step_layout(int rows_cap, int k, int ncand, int C) {
    using G = Geo<T, NP>;
    SmemLayout L;
    auto up = [](int v) { return (v + 15) & ~15; };
    const int part_d = k * NP + k + 1;
    L.samp = 0;
    L.cm = up(L.samp + rows_cap * G::RS);
    L.cs = up(L.cm + k * NP * 8);
    L.part = up(L.cs + ((k + 1) / 2) * G::RST * 8);
    L.scratch = up(L.part + xch_doubles(k, NP, C) * 8);  // exchange receive buffers
    L.labels = L.scratch;
    L.pos = up(L.labels + rows_cap);
    L.perm = up(L.pos + rows_cap * 2);
    L.wpart = up(L.perm + rows_cap * 2);
    const int lloyd_end = L.wpart + kStepWarps * part_d * 8;
    L.d2 = L.scratch;    // seeding only
    L.gidx = L.scratch;  // gather only
    L.xnorm = up(L.d2 + rows_cap * 8);
    L.wlist = up(L.xnorm + rows_cap * 4);
    L.nflag = up(L.wlist + kStepWarps * list_cap(ncand) * 4);
    const int seed_end = L.nflag + rows_cap;
    L.total = up(lloyd_end > seed_end ? lloyd_end : seed_end);
    return L;
}

struct StepShared {  // static smem: per-step scalars and exchange slots
    uint64_t xbar[2];                        // exchange mbarriers (parity buffered)
    uint64_t rbar1[2], rbar2[2];             // reduce-scatter / all-gather mbarriers
    uint64_t cbar;                           // K-means++ candidate push mbarrier
    uint8_t flags[kMaxK];
    int32_t pending[kMaxK];
    int32_t n_pending, n_valid;
    double cta_total;                        // CTA CDF total of the current slot
    double cand[kMaxCandidates][32];         // candidate coordinates (fp64, n <= 32)
    float candf[kMaxCandidates][32];         // -2 * candidate (fp32) for the screen
    float candn[kMaxCandidates];             // |candidate|^2 (fp32)
    double wsum[kStepWarps][kMaxCandidates];
    double werr[kStepWarps][kMaxCandidates];
    double wtot[kStepWarps];
    uint32_t whit[kStepWarps][kMaxCandidates];
    double units[kMaxK][kMaxCandidates];     // K-means++ draws of every slot (unit interval)
    float cnorm[kMaxK];  // |c_j| (fp32, rounded up) of the current screen records
    uint16_t wcnt[kStepWarps][kMaxK];  // per-warp label counts (counting sort; rows per CTA < 2^16)
    uint16_t woff[kStepWarps][kMaxK];  // sorted-order offset of (warp, label)
    int32_t cstart[kMaxK + 1];        // sorted-order start of each cluster
    int32_t decision;  // K-means++ slot: 1 = the approximate costs decided the winner
    int32_t best_c;    // K-means++ slot: winning candidate
    double cdf_P, cdf_T;  // K-means++ slot: this rank's CDF offset and the cluster total
    int32_t exact_passes;  // K-means++ slots that needed the exact cost pass (diagnostic)
    int32_t exact_rows;    // rows given an exact distance in the D^2 updates (diagnostic)
    int32_t exact_rows1;   // ... in the first K-means++ slot's update (diagnostic)
    int32_t err;
};

// ------------------------------------------------- cluster exchange primitives
// Push model (no cluster barrier): every CTA st.async's its values into a slot of each peer's
// receive buffer with mbarrier complete_tx; each CTA then waits only on its own mbarrier.
HPCG_DEV uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
HPCG_DEV uint32_t mapa_u32(uint32_t addr, int rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
HPCG_DEV void st_async_f64(uint32_t raddr, double v, uint32_t rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(raddr),
                 "l"(__double_as_longlong(v)), "r"(rbar)
                 : "memory");
}
HPCG_DEV void mbar_init(uint64_t* bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
HPCG_DEV void mbar_init_fence() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
HPCG_DEV void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
HPCG_DEV void mbar_wait_cluster(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n"
        " mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}

HPCG_DEV void cp_async16(void* sdst, const void* gsrc) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gsrc) : "memory");
}
HPCG_DEV void cp_async8(void* sdst, const void* gsrc) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gsrc) : "memory");
}
HPCG_DEV void cp_async4(void* sdst, const void* gsrc) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(gsrc) : "memory");
}
// Gather variants for random sample rows: without a prefetch size the L2 fills a whole 128-B line per
// missed sector pair (measured: 609 MB of DRAM reads for 328 MB of random 64-B rows, unchanged by
// cudaLimitMaxL2FetchGranularity = 32/64/128); `.L2::64B` caps the fill at the 64 B that hold the row
// (315 MB for the same gather). Streaming readers keep the default.
HPCG_DEV void cp_async16_row(void* sdst, const void* gsrc) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
#ifdef HPCG_NO_ROW_HINT  // A/B switch (tools/ab.sh)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gsrc) : "memory");
#else
    asm volatile("cp.async.cg.shared.global.L2::64B [%0], [%1], 16;\n" ::"r"(sa), "l"(gsrc) : "memory");
#endif
}
HPCG_DEV void cp_async8_row(void* sdst, const void* gsrc) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
    asm volatile("cp.async.ca.shared.global.L2::64B [%0], [%1], 8;\n" ::"r"(sa), "l"(gsrc) : "memory");
}
HPCG_DEV void cp_async4_row(void* sdst, const void* gsrc) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
    asm volatile("cp.async.ca.shared.global.L2::64B [%0], [%1], 4;\n" ::"r"(sa), "l"(gsrc) : "memory");
}
// register-staged row chunk (16 / 8 / 4 bytes) with the same fill cap
template <typename VT>
HPCG_DEV VT ld_row_chunk(const void* gsrc) {
    if constexpr (sizeof(VT) == 16) {
        uint4 t;
        asm volatile("ld.global.nc.L2::64B.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(t.x), "=r"(t.y), "=r"(t.z), "=r"(t.w) : "l"(gsrc));
        return t;
    } else if constexpr (sizeof(VT) == 8) {
        uint2 t;
        asm volatile("ld.global.nc.L2::64B.v2.u32 {%0,%1}, [%2];" : "=r"(t.x), "=r"(t.y) : "l"(gsrc));
        return t;
    } else {
        uint32_t t;
        asm volatile("ld.global.nc.L2::64B.u32 %0, [%1];" : "=r"(t) : "l"(gsrc));
        return t;
    }
}
HPCG_DEV void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }
HPCG_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
HPCG_DEV void cp_async_wait_group() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// ---------------------------------------------------------- row helpers
// Row `row` of the smem sample as fp32 pairs (operand of the fp32 screens).
template <typename T, int NP>
HPCG_DEV void load_row_f32(const T* samp, int row, float2 (&x2)[Geo<T, NP>::NPF / 2]) {
    using G = Geo<T, NP>;
    if constexpr (G::VEC16 && sizeof(T) == 4) {
#pragma unroll
        for (int q = 0; q < NP / 4; ++q) {
            const float4 v = *reinterpret_cast<const float4*>(samp + G::elem_off(row, q * 4));
            x2[2 * q] = make_float2(v.x, v.y);
            x2[2 * q + 1] = make_float2(v.z, v.w);
        }
    } else if constexpr (G::VEC16) {
#pragma unroll
        for (int q = 0; q < NP / 2; ++q) {
            const double2 v = *reinterpret_cast<const double2*>(samp + G::elem_off(row, q * 2));
            x2[q] = make_float2((float)v.x, (float)v.y);
        }
    } else {
#pragma unroll
        for (int q = 0; q < G::NPF / 2; ++q) {
            const float a = (float)samp[G::elem_off(row, 2 * q)];
            const float b = 2 * q + 1 < NP ? (float)samp[G::elem_off(row, 2 * q + 1)] : 0.f;
            x2[q] = make_float2(a, b);
        }
    }
}

HPCG_DEV float fmin3f(float a, float b, float c) {  // three-input min (sm_100 FMNMX3)
    float r;
    asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}

// |x|^2 of a row in fp32 (one FFMA2 chain)
template <int NPF>
HPCG_DEV float row_sq(const float2 (&x)[NPF / 2]) {
    float2 nn = make_float2(0.f, 0.f);
#pragma unroll
    for (int q = 0; q < NPF / 2; ++q) nn = __ffma2_rn(x[q], x[q], nn);
    return nn.x + nn.y;
}

// K-means++ screens, expanded form: dist ~ s + x.(-2c), s = |x|^2 + |c|^2, with the seed
// (s, or s minus the bound) folded into the first chain; two rows per call, four independent
// FFMA2 chains. |screen - exact| <= kScreenK (|x| + |c|)^2 <= 2 kScreenK s (the fp32 rounding
// of x.c, of s and of c, and the chain sums are inside kScreenK's slack).
template <int NPF>
HPCG_DEV void screen_exp2(const float2 (&xa)[NPF / 2], const float2 (&xb)[NPF / 2], const float2* m2c, float sa,
                          float sb, float& da, float& db) {
    float2 a0 = make_float2(sa, 0.f), a1 = make_float2(0.f, 0.f), b0 = make_float2(sb, 0.f), b1 = a1;
#pragma unroll
    for (int q = 0; q < NPF / 2; ++q) {
        const float2 c = m2c[q];
        if (q & 1) {
            a1 = __ffma2_rn(xa[q], c, a1);
            b1 = __ffma2_rn(xb[q], c, b1);
        } else {
            a0 = __ffma2_rn(xa[q], c, a0);
            b0 = __ffma2_rn(xb[q], c, b0);
        }
    }
    da = (a0.x + a1.x) + (a0.y + a1.y);
    db = (b0.x + b1.x) + (b0.y + b1.y);
}
template <int NPF>
HPCG_DEV float screen_exp1(const float2 (&x)[NPF / 2], const float2* m2c, float sx) {
    float2 a0 = make_float2(sx, 0.f), a1 = make_float2(0.f, 0.f);
#pragma unroll
    for (int q = 0; q < NPF / 2; ++q) {
        if (q & 1)
            a1 = __ffma2_rn(x[q], m2c[q], a1);
        else
            a0 = __ffma2_rn(x[q], m2c[q], a0);
    }
    return (a0.x + a1.x) + (a0.y + a1.y);
}

// Row `row` of the smem sample in its storage type (vector loads through the swizzle).
template <typename T, int NP>
HPCG_DEV void load_row_T(const T* samp, int row, T (&x)[NP]) {
    using G = Geo<T, NP>;
    if constexpr (G::VEC16) {
        constexpr int EPC = 16 / (int)sizeof(T);
#pragma unroll
        for (int q = 0; q < NP / EPC; ++q) {
            const uint4 v = *reinterpret_cast<const uint4*>(samp + G::elem_off(row, q * EPC));
            const T* tv = reinterpret_cast<const T*>(&v);
#pragma unroll
            for (int e = 0; e < EPC; ++e) x[q * EPC + e] = tv[e];
        }
    } else {
#pragma unroll
        for (int d = 0; d < NP; ++d) x[d] = samp[row * NP + d];
    }
}

// The reference distance (core.hpp:100-108) of a row held in registers: ascending d,
// separately rounded sub/mul/add; padding columns (d >= n) are zero in both operands.
template <typename T, int NP>
HPCG_DEV double exact_dist_regs(const T (&x)[NP], const double* c) {
    double acc = 0.0;
#pragma unroll
    for (int d = 0; d < NP; ++d) {
        const double diff = __dsub_rn((double)x[d], c[d]);
        acc = __dadd_rn(acc, __dmul_rn(diff, diff));
    }
    return acc;
}

// The reference distance (core.hpp:100-108): ascending d, separately rounded sub/mul/add.
template <typename T, int NP>
HPCG_DEV double exact_dist(const T* samp, int row, const double* c, int n) {
    using G = Geo<T, NP>;
    double acc = 0.0;
#pragma unroll
    for (int d = 0; d < NP; ++d) {
        if (d < n) {
            const double diff = __dsub_rn((double)samp[G::elem_off(row, d)], c[d]);
            acc = __dadd_rn(acc, __dmul_rn(diff, diff));
        }
    }
    return acc;
}

// ------------------------------------------------------------------ the kernel
template <typename T, int NP, bool TRACE = false>  // TRACE: the phase timeline (diagnostics) compiled in
__global__ void __launch_bounds__(kStepThreads, kStepMinBlocks) worker_step_kernel(const StepParams p) {
    if (p.go) {  // free-running schedule: the whole cluster reads one flag -- uniform exit before any barrier.
        // First statement, on %clusterid (= the local worker): placed after the index setup it cost the
        // kernel its register allocation (4 -> 196 bytes of spills, +3 % per step)
        unsigned cid;
        asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(cid));
        if (p.go[cid] == 0) return;
    }
    using G = Geo<T, NP>;
    cg::cluster_group cluster = cg::this_cluster();
    const int C = (int)cluster.num_blocks();
    const int cr = (int)cluster.block_rank();
    const int wl = blockIdx.x / C;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n = p.n, k = p.k;
    const int64_t s = p.s;
    int64_t r0, r1;
    chunk_range(s, C, cr, r0, r1);
    const int nr = (int)(r1 - r0);

    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ StepShared sh;
    int64_t* trace = (TRACE && p.trace) ? p.trace + (int64_t)blockIdx.x * kTraceSlots : nullptr;
    int tslot = 0;
    auto mark = [&]() {
        if (trace && tid == 0 && tslot < kTraceSlots) trace[tslot] = gtimer();
        ++tslot;
    };
    // fixed-slot diagnostic stamp (slots 16..25), warp 0's view
    auto stamp = [&](int slot) {  // SM clock (cycles): finer than %globaltimer's 256 ns
        if (trace && tid == 0) trace[slot] = clock64();
    };
    mark();  // 0: start
    if (trace && tid == 0) trace[kTraceSlots - 6] = clock64();  // SM clock rate check
    const SmemLayout L = step_layout<T, NP>(p.rows_cap, k, p.candidates, C);
    T* samp = reinterpret_cast<T*>(smem + L.samp);
    double* Cm = reinterpret_cast<double*>(smem + L.cm);
    float* cs = reinterpret_cast<float*>(smem + L.cs);
    double* part = reinterpret_cast<double*>(smem + L.part);
    uint8_t* labels = smem + L.labels;
    uint16_t* pos = reinterpret_cast<uint16_t*>(smem + L.pos);
    uint16_t* perm = reinterpret_cast<uint16_t*>(smem + L.perm);
    double* wpart = reinterpret_cast<double*>(smem + L.wpart);
    double* d2 = reinterpret_cast<double*>(smem + L.d2);
    const int part_d = k * NP + k + 1;
    // Cluster exchanges. Push model (no cluster barrier): values are st.async'd into peers'
    // receive slots with mbarrier complete_tx; each CTA waits only on its own mbarrier. Callers
    // separate the reads of one exchange from the pushes of the next with a __syncthreads.
    const int xs = kXchSmall;
    double* rxs = part;                                // [2][C][kXchSmall]
    const int sl = xch_slice(k, NP, C);
    double* rx1 = part + 2 * C * kXchSmall;            // [2][C][sl]   reduce-scatter inputs
    double* rx2 = rx1 + 2 * C * sl;                    // [2][C*sl]    all-gathered totals
    uint32_t xcount = 0;  // exchanges so far: buffer = count & 1, its mbarrier phase = (count >> 1) & 1
    // all-to-all of nv <= kXchSmall scalars: returns [C][xs] slots in rank order. w0_only: only
    // warp 0 waits for (and may read) the slots; it publishes what the others need through shared
    // memory before a __syncthreads
    auto exchange = [&](int nv, auto&& value_of, bool w0_only = false) -> const double* {
        const uint32_t ph = (xcount >> 1) & 1u;
        const int par = (int)(xcount++ & 1);
        double* rx = rxs + par * C * xs;
        uint64_t* bar = &sh.xbar[par];
        if (tid == 0) mbar_expect_tx(bar, (uint32_t)(C * nv * 8));
        const uint32_t rbar_local = smem_u32(bar), slot_local = smem_u32(rx + cr * xs);
        for (int e = tid; e < nv; e += kStepThreads) {
            const double v = value_of(e);
            for (int r = 0; r < C; ++r) st_async_f64(mapa_u32(slot_local + e * 8, r), v, mapa_u32(rbar_local, r));
        }
        if (!w0_only || warp == 0) mbar_wait_cluster(bar, ph);
        return rx;
    };
    // cluster-wide sum of nv values per CTA, reduced in rank order by the element's owner rank
    // (reduce-scatter) and broadcast (all-gather): returns the nv totals, identical in every CTA
    uint32_t rcount = 0;  // reductions so far (buffers / mbarrier phases as for the exchanges)
    auto reduce_all = [&](int nv, auto&& value_of) -> const double* {
        const uint32_t ph = (rcount >> 1) & 1u;
        const int par = (int)(rcount++ & 1);
        double* in = rx1 + par * C * sl;
        double* tot = rx2 + par * C * sl;
        uint64_t* b1 = &sh.rbar1[par];
        uint64_t* b2 = &sh.rbar2[par];
        const int mylo = cr * sl, mylen = max(0, min(sl, nv - mylo));
        if (tid == 0) {
            mbar_expect_tx(b1, (uint32_t)(C * mylen * 8));
            mbar_expect_tx(b2, (uint32_t)(nv * 8));
        }
        const uint32_t in_l = smem_u32(in + cr * sl), b1_l = smem_u32(b1);
        for (int e = tid; e < nv; e += kStepThreads) {
            const double v = value_of(e);
            const int o = e / sl;
            st_async_f64(mapa_u32(in_l + (e - o * sl) * 8, o), v, mapa_u32(b1_l, o));
        }
        mbar_wait_cluster(b1, ph);
        const uint32_t tot_l = smem_u32(tot), b2_l = smem_u32(b2);
        for (int e = tid; e < mylen; e += kStepThreads) {
            double t = in[e];
            for (int r = 1; r < C; ++r) t += in[r * sl + e];
            for (int r = 0; r < C; ++r) st_async_f64(mapa_u32(tot_l + (mylo + e) * 8, r), t, mapa_u32(b2_l, r));
        }
        mbar_wait_cluster(b2, ph);
        return tot;
    };

    // ---------------------------------------------------------------- gather
    {
        const T* X = static_cast<const T*>(p.X);
        // initial centroids and flags: loads issued first so their latency hides under the gather
        const int64_t v = p.shared_version ? *p.shared_version : 1;
        const double* ic = p.init_c + (int64_t)wl * p.init_stride;
        const uint8_t* ifl = p.init_f + (int64_t)wl * p.initf_stride;
        constexpr int kIC = (kMaxK * 32 + kStepThreads - 1) / kStepThreads;
        double icv[kIC];
#pragma unroll
        for (int u = 0; u < kIC; ++u) {
            const int e = tid + u * kStepThreads, j = e / NP, d = e - j * NP;
            icv[u] = (e < k * NP && d < n) ? ic[(int64_t)j * n + d] : 0.0;
        }
        const uint8_t fl0 = tid < k ? ifl[tid] : (uint8_t)1;
        SamplePRP prp;
        if (p.sample_mode == 1)
            prp = SamplePRP::make(p.key, p.round, (uint32_t)(p.worker_base + wl), (uint64_t)p.m, p.prp_a, p.prp_b,
                                  p.prp_inv_b);
        auto gidx_of = [&](int64_t i) -> int64_t {
            if (p.sample_mode == 0) return p.idx[(int64_t)wl * s + i];
            if (p.sample_mode == 1) return (int64_t)prp((uint64_t)i);
            return (int64_t)wl * s + i;
        };
        if ((TRACE && p.trace_mode == 0)) stamp(16);
        const int rowb = n * (int)sizeof(T);
        if constexpr (G::VEC16 && 32 % G::CPR == 0) {
            if (n == NP) {  // whole rows of 16-B chunks. Per warp step: every lane computes one
                // row's index, then the warp copies those 32 rows chunk-major (CPR consecutive
                // lanes per row) with the indices shuffled across: no index buffer, no barrier,
                // and the next indices are computed while these copies are in flight
                constexpr int EPC = 16 / (int)sizeof(T), RPI = 32 / G::CPR;
                const int q = lane % G::CPR;
                for (int g = warp; g * 32 < nr; g += kStepWarps) {
                    const int li = g * 32 + lane;
                    const int64_t gi = li < nr ? gidx_of(r0 + li) : 0;
#pragma unroll
                    for (int j = 0; j < G::CPR; ++j) {
                        const int rl = j * RPI + lane / G::CPR, row = g * 32 + rl;
                        const int64_t src = __shfl_sync(0xffffffffu, gi, rl);
                        if (row < nr) cp_async16_row(samp + G::elem_off(row, q * EPC), row_ptr<T>(p, src) + q * EPC);
                    }
                }
            }
        }
        if (!(G::VEC16 && 32 % G::CPR == 0 && n == NP)) {
            // general rows: one sample index per row into smem, then the copies
            int64_t* gx = reinterpret_cast<int64_t*>(smem + L.gidx);
            for (int li = tid; li < nr; li += kStepThreads) gx[li] = gidx_of(r0 + li);
            __syncthreads();
            if ((rowb & 15) == 0) {  // 16-B chunks
                const int cpr = rowb >> 4;
                constexpr int EPC = 16 / (int)sizeof(T);
                for (int e = tid; e < nr * cpr; e += kStepThreads) {
                    const int li = e / cpr, q = e - li * cpr;
                    cp_async16_row(samp + G::elem_off(li, q * EPC), row_ptr<T>(p, gx[li]) + q * EPC);
                }
            } else if ((rowb & 7) == 0) {  // 8-B chunks
                const int cpr = rowb >> 3;
                constexpr int EPC = 8 / (int)sizeof(T);
                for (int e = tid; e < nr * cpr; e += kStepThreads) {
                    const int li = e / cpr, q = e - li * cpr;
                    cp_async8_row(samp + G::elem_off(li, q * EPC), row_ptr<T>(p, gx[li]) + q * EPC);
                }
            } else {  // 4-B elements (fp32, odd n)
                for (int e = tid; e < nr * n; e += kStepThreads) {
                    const int li = e / n, d = e - li * n;
                    cp_async4_row(samp + G::elem_off(li, d), row_ptr<T>(p, gx[li]) + d);
                }
            }
        }
        if ((TRACE && p.trace_mode == 0)) stamp(17);
        if (NP > n)
            for (int e = tid; e < nr * (NP - n); e += kStepThreads) {
                const int li = e / (NP - n), d = n + (e - li * (NP - n));
                samp[G::elem_off(li, d)] = T(0);
            }
        // initial centroids (fp64 master, zero padded) and flags; a zero shared version means
        // no incumbent yet: every slot pending
#pragma unroll
        for (int u = 0; u < kIC; ++u) {
            const int e = tid + u * kStepThreads;
            if (e < k * NP) Cm[e] = v != 0 ? icv[u] : 0.0;
        }
        if (tid < k) sh.flags[tid] = v != 0 ? fl0 : (uint8_t)1;
        if (tid == 0) {
            sh.err = kErrNone;
            sh.exact_passes = 0;
            sh.exact_rows = 0;
            sh.exact_rows1 = 0;
        }
    }
    if (tid == 0) {
        mbar_init(&sh.xbar[0], 1);
        mbar_init(&sh.xbar[1], 1);
        for (int q = 0; q < 2; ++q) {
            mbar_init(&sh.rbar1[q], 1);
            mbar_init(&sh.rbar2[q], 1);
        }
        mbar_init(&sh.cbar, 1);
        mbar_init_fence();
    }
    if ((TRACE && p.trace_mode == 0)) stamp(18);
    mark();  // 1: copies issued
    cp_async_wait_all();
    __syncthreads();  // gx (aliases d2) fully consumed before seeding reuses the region
    if (tid == 0) {   // pending slots in slot order
        int np_ = 0, nv = 0;
        for (int j = 0; j < k; ++j) {
            if (sh.flags[j])
                sh.pending[np_++] = j;
            else
                ++nv;
        }
        sh.n_pending = np_;
        sh.n_valid = nv;
    }
    mark();  // 2: sample landed
    cluster.sync();  // sample rows of every CTA now visible cluster-wide (DSMEM)
    mark();  // 3: cluster synced

    int64_t nd = 0;  // distance evaluations (reference accounting)
    int filled = 0;

    // --------------------------------------------------------------- seeding
    // seeding.hpp:47-105. d2 and every candidate cost use the exact reference
    // distance; the CDF is a fixed-order (segment, block, rank) prefix sum.
    if (sh.n_pending > 0) {
        const int np_ = sh.n_pending;
        const int ncand = p.candidates;
        uint32_t* wlist = reinterpret_cast<uint32_t*>(smem + L.wlist) + warp * list_cap(ncand);
        float* xsq = reinterpret_cast<float*>(smem + L.xnorm);  // |x|^2 (fp32) per local row
        uint8_t* nflag = smem + L.nflag;  // bit c: the cost screen could not settle (row, candidate c)
        // screen bound B = kScreenK2 * s (see screen_exp2); s itself is rounded, hence the 1.001
        constexpr float kScreenK2 = 2.002f * 2.0f * (float)(G::NPF / 2 + 12) * 5.9604645e-8f;
        constexpr float kScreenTiny = 1e-42f;  // absolute slack: fp32 denormal rounding
        constexpr float kD2Round = 2.5e-7f;     // |ru(d2) - d2| <= 2^-23 d2, plus one fp32 subtraction
        constexpr float kOneK2 = 1.0f - kScreenK2;  // screen - bound = (1 - K2) s + x.(-2c) - tiny
        for (int li = tid; li < nr; li += kStepThreads) {
            d2[li] = __longlong_as_double(0x7ff0000000000000LL);
            float2 x2[G::NPF / 2];
            load_row_f32<T, NP>(samp, li, x2);
            xsq[li] = row_sq<G::NPF>(x2);
        }
        // fp32 screen record of slot c of sh.cand (-2c and |c|^2); one warp, caller syncs
        auto make_candf = [&](int c) {
            const float cf = lane < n ? (float)sh.cand[c][lane] : 0.f;
            if (lane < G::NPF) sh.candf[c][lane] = -2.f * cf;
            const float cc = warp_sum_f(cf * cf);
            if (lane == 0) sh.candn[c] = cc;
        };
        // d2 = min(d2, dist(., cand c)) for every local row (seeding.hpp:20-42); the exact
        // reference distance is evaluated only where the fp32 screen cannot prove
        // dist >= d2, and those rows are compacted so the fp64 work runs on full warps.
        auto d2_update = [&](int c) {
            int cnt = 0;
            float2 nc2[G::NPF / 2];  // candidate screen record held in registers
#pragma unroll
            for (int q = 0; q < G::NPF / 2; ++q) nc2[q] = *reinterpret_cast<const float2*>(&sh.candf[c][2 * q]);
            const double* cd = sh.cand[c];
            const float cnp = fmaf(sh.candn[c], kOneK2, -kScreenTiny);
            // exact distances for the listed rows, 32 at a time (the warp owns its rows' d2)
            auto flush = [&](bool all) {
                while (cnt >= 32 || (all && cnt > 0)) {
                    const int take = cnt < 32 ? cnt : 32;
                    if (trace && lane == 0) atomicAdd(&sh.exact_rows, take);
                    if (lane < take) {
                        const int r = (int)wlist[lane];
                        T xr[NP];
                        load_row_T<T, NP>(samp, r, xr);
                        d2[r] = fmin(d2[r], exact_dist_regs<T, NP>(xr, cd));
                    }
                    __syncwarp();
                    for (int t = lane; t + take < cnt; t += 32) wlist[t] = wlist[t + take];
                    __syncwarp();
                    cnt -= take;
                }
            };
            const int nchunks = (nr + 31) / 32;
            const unsigned lt = (1u << lane) - 1u;
            for (int ch = warp; ch < nchunks; ch += 2 * kStepWarps) {  // two rows per lane per step
                const int ra = ch * 32 + lane, rb = ra + kStepWarps * 32;
                const bool va = ra < nr, vb = rb < nr;
                float2 xa[G::NPF / 2], xb[G::NPF / 2];
                load_row_f32<T, NP>(samp, va ? ra : 0, xa);
                load_row_f32<T, NP>(samp, vb ? rb : 0, xb);
                float dfa, dfb;  // screen - bound
                screen_exp2<G::NPF>(xa, xb, nc2, fmaf(va ? xsq[ra] : 0.f, kOneK2, cnp),
                                    fmaf(vb ? xsq[rb] : 0.f, kOneK2, cnp), dfa, dfb);
                const bool na = va && !(dfa > __double2float_ru(d2[ra]));
                const bool nb = vb && !(dfb > __double2float_ru(d2[rb]));
                const unsigned ma = __ballot_sync(0xffffffffu, na);
                if (na) wlist[cnt + __popc(ma & lt)] = (uint32_t)ra;
                cnt += __popc(ma);
                const unsigned mb = __ballot_sync(0xffffffffu, nb);
                if (nb) wlist[cnt + __popc(mb & lt)] = (uint32_t)rb;
                cnt += __popc(mb);
                __syncwarp();
                flush(false);
            }
            flush(true);
        };
        // the first D^2 update of a step (every d2 still +inf): every row takes the exact distance
        // (seeding.hpp:20-42 with d2 = inf), so no screen and no work list -- two rows per thread
        // with interleaved fp64 chains
        auto d2_first = [&](int c) {
            const double* cd = sh.cand[c];
            int li = tid;
            constexpr bool kTwo = NP * sizeof(T) <= 64;  // two rows in registers (wider rows: one)
            for (; kTwo && li + kStepThreads < nr; li += 2 * kStepThreads) {
                T xa[NP], xb[NP];
                load_row_T<T, NP>(samp, li, xa);
                load_row_T<T, NP>(samp, li + kStepThreads, xb);
                double a = 0.0, b = 0.0;
#pragma unroll
                for (int d = 0; d < NP; ++d) {
                    const double cv = cd[d];
                    const double ea = __dsub_rn((double)xa[d], cv), eb = __dsub_rn((double)xb[d], cv);
                    a = __dadd_rn(a, __dmul_rn(ea, ea));
                    b = __dadd_rn(b, __dmul_rn(eb, eb));
                }
                d2[li] = a;
                d2[li + kStepThreads] = b;
            }
            for (; li < nr; li += kStepThreads) {
                T xr[NP];
                load_row_T<T, NP>(samp, li, xr);
                d2[li] = exact_dist_regs<T, NP>(xr, cd);
            }
        };
        bool d2_fresh = true;
        // the same update for the winning candidate of a K-means++ slot: the cost pass already
        // screened every row against it, so only its flagged rows get an exact distance
        auto d2_update_flagged = [&](int c, bool tr) {
            int cnt = 0;
            const double* cd = sh.cand[c];
            // exact distances of the listed rows, up to two per lane with interleaved fp64 chains
            // (narrow rows; wider rows one per lane); flushed once 64 are listed (list_cap >= 96)
            constexpr int kPer = NP * sizeof(T) <= 64 ? 2 : 1;
            auto flush = [&](bool all) {
                while (cnt >= 32 * kPer || (all && cnt > 0)) {
                    const int take = cnt < 32 * kPer ? cnt : 32 * kPer;
                    if (tr && lane == 0) atomicAdd(&sh.exact_rows1, take);
                    if constexpr (kPer == 2) {
                        if (lane + 32 < take) {
                            const int ra = (int)wlist[lane], rb = (int)wlist[lane + 32];
                            T xa[NP], xb[NP];
                            load_row_T<T, NP>(samp, ra, xa);
                            load_row_T<T, NP>(samp, rb, xb);
                            double a = 0.0, b = 0.0;
#pragma unroll
                            for (int d = 0; d < NP; ++d) {
                                const double cv = cd[d];
                                const double ea = __dsub_rn((double)xa[d], cv), eb = __dsub_rn((double)xb[d], cv);
                                a = __dadd_rn(a, __dmul_rn(ea, ea));
                                b = __dadd_rn(b, __dmul_rn(eb, eb));
                            }
                            d2[ra] = fmin(d2[ra], a);
                            d2[rb] = fmin(d2[rb], b);
                        } else if (lane < take) {
                            const int r = (int)wlist[lane];
                            T xr[NP];
                            load_row_T<T, NP>(samp, r, xr);
                            d2[r] = fmin(d2[r], exact_dist_regs<T, NP>(xr, cd));
                        }
                    } else if (lane < take) {
                        const int r = (int)wlist[lane];
                        T xr[NP];
                        load_row_T<T, NP>(samp, r, xr);
                        d2[r] = fmin(d2[r], exact_dist_regs<T, NP>(xr, cd));
                    }
                    __syncwarp();
                    for (int t = lane; t + take < cnt; t += 32) wlist[t] = wlist[t + take];
                    __syncwarp();
                    cnt -= take;
                }
            };
            const int nchunks = (nr + 31) / 32;
            const unsigned lt = (1u << lane) - 1u;
            for (int ch = warp; ch < nchunks; ch += kStepWarps) {
                const int r = ch * 32 + lane;
                const bool nd_ = r < nr && ((nflag[r] >> c) & 1u);
                const unsigned m = __ballot_sync(0xffffffffu, nd_);
                if (nd_) wlist[cnt + __popc(m & lt)] = (uint32_t)r;
                cnt += __popc(m);
                __syncwarp();
                flush(false);
            }
            if (tr) stamp(22);
            flush(true);
            if (tr) stamp(23);
        };
        __syncthreads();
        // valid centres in slot order (seeding.hpp:60-68)
        for (int j = 0; j < k; ++j) {
            if (sh.flags[j]) continue;
            if (warp == 0) {
                for (int d = lane; d < 32; d += 32) sh.cand[0][d] = d < n ? Cm[j * NP + d] : 0.0;
                __syncwarp();
                make_candf(0);
            }
            __syncthreads();
            if (d2_fresh)
                d2_first(0);
            else
                d2_update(0);
            d2_fresh = false;
            __syncthreads();
            nd += s;
        }
        // fetch a sample row (global sample position) from its owner CTA into dst[n]
        auto fetch_row = [&](int64_t row, double* dst) {
            // owner rank: invert chunk_range (the whole sample is cluster-resident: 32-bit)
            const int si = (int)s, r32 = (int)row;
            const int base = si / C, extra = si - base * C;
            int owner, lr;
            if (r32 < extra * (base + 1)) {
                owner = r32 / (base + 1);
                lr = r32 - owner * (base + 1);
            } else {
                const int q = r32 - extra * (base + 1);
                owner = extra + q / base;  // base > 0 here: rows past the extras exist only then
                lr = q - (owner - extra) * base;
            }
            const T* rs = cluster.map_shared_rank(samp, owner);
            for (int d = lane; d < 32; d += 32) dst[d] = d < n ? (double)rs[G::elem_off(lr, d)] : 0.0;
        };
        int next = 0;
        __syncthreads();
        if (sh.n_valid == 0) {  // seeding.hpp:72-79: uniform first centre
            int64_t row;
            if (p.seed_mode == 0)
                row = p.first_row[wl];
            else
                row = (int64_t)philox_index(p.key, p.round, (uint32_t)(p.worker_base + wl), 0xF1F1u, (uint64_t)s);
            const int j = sh.pending[next++];
            if (warp == 0) {
                fetch_row(row, sh.cand[0]);
                __syncwarp();
                make_candf(0);
                for (int d = lane; d < NP; d += 32) Cm[j * NP + d] = d < n ? sh.cand[0][d] : 0.0;
                if (lane == 0) sh.flags[j] = 0;
            }
            __syncthreads();
            if (d2_fresh)
                d2_first(0);
            else
                d2_update(0);
            d2_fresh = false;
            nd += s;
            ++filled;
            __syncthreads();
        }
        // per-thread contiguous segment of local rows for the CDF
        const int seg = (nr + kStepThreads - 1) / kStepThreads;
        const int sb = tid * seg < nr ? tid * seg : nr;
        const int se = sb + seg < nr ? sb + seg : nr;
        // every slot's K-means++ draws up front, one per thread (read after the CDF's barriers)
        for (int e = tid; e < (np_ - next) * ncand; e += kStepThreads) {
            const int it_ = e / ncand, c = e - it_ * ncand;
            sh.units[it_][c] = p.seed_mode == 0 ? p.units[(int64_t)wl * p.units_stride + (int64_t)it_ * ncand + c]
                                                : philox_unit(p.key, p.round, (uint32_t)(p.worker_base + wl),
                                                              (uint32_t)(0x10000 + (next + it_) * kMaxCandidates + c));
        }
        int it = 0;
        uint32_t cph = 0u;  // sh.cbar phase
        for (; next < np_; ++next, ++it) {
            // (1) segment sums, block exclusive scan (fixed tree), CTA total
            double tsum = 0.0;
            for (int li = sb; li < se; ++li) tsum += d2[li];
            double incl = tsum;  // warp inclusive scan (fixed shuffle tree)
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const double y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            double lexcl = __shfl_up_sync(0xffffffffu, incl, 1);
            if (lane == 0) lexcl = 0.0;
            if (lane == 31) sh.wtot[warp] = incl;
            __syncthreads();
            double wexcl;
            {  // exclusive prefix of the warp totals, shuffle scan (fixed order, same for all lanes)
                double v = lane < kStepWarps ? sh.wtot[lane] : 0.0;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const double y = __shfl_up_sync(0xffffffffu, v, o);
                    if (lane >= o) v += y;
                }
                wexcl = __shfl_sync(0xffffffffu, v, warp > 0 ? warp - 1 : 0);
                if (warp == 0) wexcl = 0.0;
            }
            const double texcl = wexcl + lexcl;  // exclusive prefix of this thread's segment
            // CTA total := local cum at the CTA's last row, computed exactly as the search does
            if (se == nr && sb < se) {
                double run = 0.0;
                for (int li = sb; li < se; ++li) run += d2[li];
                sh.cta_total = texcl + run;
            }
            __syncthreads();
            if (it == 0 && (TRACE && p.trace_mode == 1)) mark();  // 5: CDF local done
            const double* rxt = exchange(1, [&](int) { return sh.cta_total; }, true);
            if (it == 0 && (TRACE && p.trace_mode == 1)) mark();  // 6: CDF exchange complete
            // P = sum of lower ranks' totals (rank order); total = P_{C-1} + T_{C-1}: one thread,
            // published to the CTA
            if (tid == 0) {
                double acc = 0.0, P0 = 0.0;
                for (int rr = 0; rr < C - 1; ++rr) {
                    if (rr == cr) P0 = acc;
                    acc += rxt[rr * xs];
                }
                if (cr == C - 1) P0 = acc;
                sh.cdf_P = P0;
                sh.cdf_T = acc + rxt[(C - 1) * xs];
            }
            __syncthreads();
            const double P = sh.cdf_P, total = sh.cdf_T;
            if (!(total > 0.0)) break;  // distinct rows exhausted (seeding.hpp:87)
            // (2) candidate draws u_c = unit * total; first global row with cum > u_c
            double u[kMaxCandidates];
            uint32_t hit[kMaxCandidates];  // local row of the first crossing (0xffffffff: none)
#pragma unroll
            for (int c = 0; c < kMaxCandidates; ++c) {
                hit[c] = 0xffffffffu;
                u[c] = c < ncand ? sh.units[it][c] * total : 0.0;
            }
            bool any = false;
            if (sb < se) {  // cum is non-decreasing along a segment: scan only where a draw crosses it
                const double seg_hi = P + (texcl + tsum), seg_lo = P + (texcl + d2[sb]);
#pragma unroll
                for (int c = 0; c < kMaxCandidates; ++c) {
                    if (c >= ncand) break;
                    if (seg_lo > u[c])
                        hit[c] = (uint32_t)sb;
                    else
                        any |= seg_hi > u[c];
                }
            }
            if (any) {
                double run = 0.0;
                for (int li = sb; li < se; ++li) {
                    run += d2[li];
                    const double cum = P + (texcl + run);
#pragma unroll
                    for (int c = 0; c < kMaxCandidates; ++c)
                        if (c < ncand && hit[c] == 0xffffffffu && cum > u[c]) hit[c] = (uint32_t)li;
                }
            }
#pragma unroll
            for (int c = 0; c < kMaxCandidates; ++c) {
                if (c >= ncand) break;
                const uint32_t h = __reduce_min_sync(0xffffffffu, hit[c]);
                if (lane == 0) sh.whit[warp][c] = h;
            }
            __syncthreads();
            if (it == 0 && (TRACE && p.trace_mode == 1)) mark();  // 7: search done
            // cum is monotone across the cluster and P equals the previous rank's last cum
            // exactly, so exactly one CTA holds the first global row with cum > u_c: the CTA with a
            // local crossing and P <= u_c (rank 0: P = 0); if no row crosses, rank C-1 takes the
            // fallback row s - 1 (rng.hpp:87-92). That CTA pushes the row's coordinates straight
            // into every CTA's candidate slot c (st.async + mbarrier): draw and fetch in one step.
            if (tid == 0) mbar_expect_tx(&sh.cbar, (uint32_t)(ncand * NP * 8));
            for (int c = warp; c < ncand; c += kStepWarps) {
                const uint32_t h = __reduce_min_sync(0xffffffffu, lane < kStepWarps ? sh.whit[lane][c] : 0xffffffffu);
                const double uc = sh.units[it][c] * total;
                int own = -1;
                if (h != 0xffffffffu && (cr == 0 || !(P > uc)))
                    own = (int)h;
                else if (cr == C - 1 && !(total > uc))
                    own = nr - 1;
                if (own >= 0) {
                    const uint32_t dst = smem_u32(&sh.cand[c][0]), bar = smem_u32(&sh.cbar);
                    for (int d = lane; d < NP; d += 32) {
                        const double v = d < n ? (double)samp[G::elem_off(own, d)] : 0.0;
                        for (int rr = 0; rr < C; ++rr) st_async_f64(mapa_u32(dst + d * 8, rr), v, mapa_u32(bar, rr));
                    }
                }
            }
            mbar_wait_cluster(&sh.cbar, cph);
            cph ^= 1u;
            if (it == 0 && (TRACE && p.trace_mode == 1)) mark();  // 8: candidates received
            for (int c = warp; c < ncand; c += kStepWarps) make_candf(c);
            __syncthreads();
            if (it == 0 && (TRACE && p.trace_mode == 1)) mark();  // 9: candidates fetched
            if (it == 0 && (TRACE && p.trace_mode == 1)) stamp(16);
            // (3) candidate costs sum_i min(d2_i, dist(S_i, cand_c)) (seeding.hpp:93). First from
            // the fp32 screen with a rigorous per-row error budget; only if two candidates are
            // within their budgets (or tie) are the costs recomputed with exact distances.
            // (a) approximate pass, templated on the candidate count so the candidates' screen
            //     chains interleave. Per row and candidate: dfB = screen - B (one FFMA2 chain
            //     seeded with (1 - K2) s - tiny), the cost reduction d' = max(ru(d2) - dfB, 0),
            //     and for the rows the screen cannot settle (dfB <= ru(d2)) the error terms. The
            //     local cost is T - sum d' + [0, E], E = sum (2B + kD2Round ru(d2)); T, the CTA's
            //     CDF total, is common to all candidates, so only sum d' and E are exchanged.
            auto approx_costs = [&](auto ncc) {
                constexpr int NC = decltype(ncc)::value;
                float red[NC], efx[NC], eff[NC], cnp[NC];
                int efn[NC];
#pragma unroll
                for (int c = 0; c < NC; ++c) {
                    red[c] = efx[c] = eff[c] = 0.f;
                    efn[c] = 0;
                    cnp[c] = fmaf(sh.candn[c], kOneK2, -kScreenTiny);
                }
                auto rows = [&](auto rr, int rbase) {  // rows rbase + i * kStepThreads, i < R
                    constexpr int R = decltype(rr)::value;
                    float2 x[R][G::NPF / 2];
                    float f[R], xq[R];
#pragma unroll
                    for (int i = 0; i < R; ++i) {
                        const int r = rbase + i * kStepThreads;
                        const bool v = r < nr;
                        load_row_f32<T, NP>(samp, v ? r : 0, x[i]);
                        f[i] = v ? __double2float_ru(d2[r]) : 0.f;
                        xq[i] = v ? xsq[r] : __int_as_float(0x7f800000);  // invalid rows: dfB = inf
                    }
                    uint32_t fl[R];
#pragma unroll
                    for (int i = 0; i < R; ++i) fl[i] = 0u;
#pragma unroll
                    for (int c = 0; c < NC; ++c) {
                        const float2* m2c = reinterpret_cast<const float2*>(sh.candf[c]);
#pragma unroll
                        for (int i = 0; i < R; ++i) {
                            float2 acc = make_float2(fmaf(xq[i], kOneK2, cnp[c]), 0.f);
#pragma unroll
                            for (int q = 0; q < G::NPF / 2; ++q) acc = __ffma2_rn(x[i][q], m2c[q], acc);
                            const float dfB = acc.x + acc.y;
                            red[c] += fmaxf(f[i] - dfB, 0.f);
                            if (!(dfB > f[i])) {  // unsettled (NaN included: its error is NaN)
                                efx[c] += xq[i];
                                eff[c] += f[i];
                                ++efn[c];
                                fl[i] |= 1u << c;
                            }
                        }
                    }
                    // the flags are the D^2 update's work list for whichever candidate wins
#pragma unroll
                    for (int i = 0; i < R; ++i)
                        if (rbase + i * kStepThreads < nr) nflag[rbase + i * kStepThreads] = (uint8_t)fl[i];
                };
                // two rows per thread per step while any lane of the warp has a second row (wider
                // CTAs run at a lower register cap: one row per step)
                int r = tid;
                if constexpr (kStepThreads <= 512)
                    for (; r - lane + kStepThreads < nr; r += 2 * kStepThreads) rows(IntC<2>{}, r);
                if (it == 0 && (TRACE && p.trace_mode == 1)) stamp(17);
                for (; r - lane < nr; r += kStepThreads) rows(IntC<1>{}, r);
                if (it == 0 && (TRACE && p.trace_mode == 1)) stamp(18);
                // midpoint and half-width per candidate; the slack covers the fp32 lane and warp sums.
                // The 2 NC butterfly sums run interleaved (same per-value order as warp_sum_f).
                float vs[NC], es[NC];
#pragma unroll
                for (int c = 0; c < NC; ++c) {
                    const float E = fmaf(2.f * kScreenK2, fmaf((float)efn[c], sh.candn[c], efx[c]),
                                         fmaf(kD2Round, eff[c], 4e-42f * (float)efn[c]));
                    vs[c] = 0.5f * E - red[c];
                    es[c] = 0.5005f * E + 1e-5f * red[c];
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1)
#pragma unroll
                    for (int c = 0; c < NC; ++c) {
                        vs[c] += __shfl_xor_sync(0xffffffffu, vs[c], o);
                        es[c] += __shfl_xor_sync(0xffffffffu, es[c], o);
                    }
                if (lane == 0)
#pragma unroll
                    for (int c = 0; c < NC; ++c) {
                        sh.wsum[warp][c] = (double)vs[c];
                        sh.werr[warp][c] = (double)es[c];
                    }
                if (it == 0 && (TRACE && p.trace_mode == 1)) stamp(19);
            };
            // (b) exact pass (only when (a) cannot separate the winner): exact distances for every
            //     row the screen cannot settle, compacted into the warp's work list
            auto exact_costs = [&]() {
                double cost[kMaxCandidates];
#pragma unroll
                for (int c = 0; c < kMaxCandidates; ++c) cost[c] = 0.0;
                int cnt = 0;
                auto flush = [&](bool all) {
                    while (cnt >= 32 || (all && cnt > 0)) {
                        const int take = cnt < 32 ? cnt : 32;
                        if (lane < take) {
                            const uint32_t e = wlist[lane];
                            const int r = (int)(e & 0xffffu), c = (int)(e >> 16);
                            T xr[NP];
                            load_row_T<T, NP>(samp, r, xr);
                            const double v = fmin(d2[r], exact_dist_regs<T, NP>(xr, sh.cand[c]));
#pragma unroll
                            for (int cc = 0; cc < kMaxCandidates; ++cc)
                                if (cc == c) cost[cc] += v;
                        }
                        __syncwarp();
                        for (int t = lane; t + take < cnt; t += 32) wlist[t] = wlist[t + take];
                        __syncwarp();
                        cnt -= take;
                    }
                };
                const int nchunks = (nr + 31) / 32;
                const unsigned lt = (1u << lane) - 1u;
                for (int ch = warp; ch < nchunks; ch += kStepWarps) {
                    const int row = ch * 32 + lane;
                    const bool valid = row < nr;
                    float2 x2[G::NPF / 2];
                    load_row_f32<T, NP>(samp, valid ? row : 0, x2);
                    const double d2i = valid ? d2[row] : 0.0;
                    const float xq = valid ? xsq[row] : 0.f;
#pragma unroll
                    for (int c = 0; c < kMaxCandidates; ++c) {
                        if (c >= ncand) break;
                        const float sc = xq + sh.candn[c];
                        const float df = screen_exp1<G::NPF>(x2, reinterpret_cast<const float2*>(sh.candf[c]), sc);
                        const bool need = valid && !(df - fmaf(kScreenK2, sc, kScreenTiny) > __double2float_ru(d2i));
                        if (valid && !need) cost[c] += d2i;
                        const unsigned msk = __ballot_sync(0xffffffffu, need);
                        if (need) wlist[cnt + __popc(msk & lt)] = (uint32_t)row | ((uint32_t)c << 16);
                        cnt += __popc(msk);
                    }
                    __syncwarp();
                    flush(false);
                }
                flush(true);
#pragma unroll
                for (int c = 0; c < kMaxCandidates; ++c) {
                    if (c >= ncand) break;
                    const double v = warp_sum(cost[c]);
                    if (lane == 0) {
                        sh.wsum[warp][c] = v;
                        sh.werr[warp][c] = 0.0;
                    }
                }
            };
            // cluster totals in rank order; strict <, first candidate wins ties (seeding.hpp:94-98).
            // Every CTA evaluates the same totals, so the decision is cluster-uniform.
            int best = 0;
            auto exchange_decide = [&](bool exact) -> bool {
                __syncthreads();
                const double* rxc = exchange(
                    2 * ncand,
                    [&](int e) {
                        const int c = e < ncand ? e : e - ncand;
                        double v = 0.0;
                        for (int w2 = 0; w2 < kStepWarps; ++w2) v += e < ncand ? sh.wsum[w2][c] : sh.werr[w2][c];
                        return v;
                    },
                    true);
                if (it == 0 && (TRACE && p.trace_mode == 1) && !exact) mark();  // 11: cost exchange complete
                if (it == 0 && (TRACE && p.trace_mode == 1) && !exact) stamp(20);
                // warp 0 decides (lane e < 2*ncand sums column e over ranks in rank order) and
                // publishes the decision to the CTA
                if (warp == 0) {
                    double col = 0.0;
                    if (lane < 2 * ncand)
                        for (int rr = 0; rr < C; ++rr) col += rxc[rr * xs + lane];
                    double tc[kMaxCandidates], te[kMaxCandidates];
                    double bc = __longlong_as_double(0x7ff0000000000000LL), be = 0.0;
                    int b0 = 0;
#pragma unroll
                    for (int c = 0; c < kMaxCandidates; ++c) {
                        tc[c] = (exact ? 0.0 : total) + __shfl_sync(0xffffffffu, col, c);
                        te[c] = __shfl_sync(0xffffffffu, col, (ncand + c) & 31);
                        if (c >= ncand) continue;
                        te[c] += 1e-9 * fabs(tc[c]);  // summation-order slack
                        if (tc[c] < bc) {
                            bc = tc[c];
                            be = te[c];
                            b0 = c;
                        }
                    }
                    bool dec = true;
                    if (!exact)
#pragma unroll
                        for (int c = 0; c < kMaxCandidates; ++c)
                            if (c < ncand && c != b0 && !(tc[c] - te[c] > bc + be)) dec = false;
                    if (lane == 0) {
                        sh.best_c = b0;
                        sh.decision = dec ? 1 : 0;
                    }
                }
                __syncthreads();
                best = sh.best_c;
                return sh.decision != 0;
            };
            switch (ncand) {
                case 1: approx_costs(IntC<1>{}); break;
                case 2: approx_costs(IntC<2>{}); break;
                case 3: approx_costs(IntC<3>{}); break;
                default: approx_costs(IntC<kMaxCandidates>{}); break;
            }
            if (it == 0 && (TRACE && p.trace_mode == 1)) mark();  // 10: costs local done
            if (!exchange_decide(false)) {
                __syncthreads();  // all reads of this exchange precede the exact pass's pushes
                if (tid == 0) ++sh.exact_passes;
                exact_costs();
                exchange_decide(true);
            }
            nd += (int64_t)ncand * s;
            const int j = sh.pending[next];
            for (int d = tid; d < NP; d += kStepThreads) Cm[j * NP + d] = d < n ? sh.cand[best][d] : 0.0;
            if (tid == 0) sh.flags[j] = 0;
            if (it == 0 && (TRACE && p.trace_mode == 1)) stamp(21);
            d2_update_flagged(best, it == 0 && (TRACE && p.trace_mode == 1));
            ++filled;
            __syncthreads();
            if (it == 0 && (TRACE && p.trace_mode == 1)) mark();  // 12: d2 updated (slot done)
            if (it == 0 && (TRACE && p.trace_mode == 1)) stamp(24);
        }
        __syncthreads();
    }

    mark();  // 4: seeding done
    // ---------------------------------------------------------------- Lloyd
    int iters = 0, stop = 1 /*max_iters*/, hist_len = 0;
    double f_final = 0.0, f_prev = __longlong_as_double(0x7ff0000000000000LL), last = 0.0;
    bool degenerate_init = false;
    for (int j = 0; j < k; ++j) degenerate_init |= sh.flags[j] != 0;
    const bool run_lloyd = p.do_lloyd && !degenerate_init;
    if (p.do_lloyd && degenerate_init && tid == 0) sh.err = kErrDegenerateInit;

    if (run_lloyd) {
        // error bound of the fp32 expanded-form screen vs the exact fp64 distance:
        // |screen - exact| <= kappa (|x| + max|c|)^2 per centroid; two centroids compared
        // (centre-pair screen: one fused chain of NPF terms per distance)
        constexpr float kappa = 2.0f * (float)(G::NPF + 12) * 5.9604645e-8f;
        bool closing = false;
        int pass = 0;
        // screen record of centroid j from its fp64 master value c (lane = dimension):
        // c' = -2c (fp32), |c|^2 (fp32 sum of rounded squares), |c| rounded up into sh.cnorm
        // Records are centre PAIRS: pair q interleaves centres 2q, 2q+1 per dimension, so one
        // FFMA2 with the row value as broadcast scalar advances both distances.
        auto make_rec = [&](int j, double c) {
            float* rec = cs + (j >> 1) * (2 * G::RST) + (j & 1);
            if (lane < G::NPF) rec[2 * lane] = lane < NP ? (float)(-2.0 * c) : 0.f;
            const float cc = warp_sum_f(lane < NP ? (float)(c * c) : 0.f);
            if (lane == 0) {
                rec[2 * G::NPF] = cc;
                rec[2 * G::NPF + 2] = 0.f;
                sh.cnorm[j] = sqrtf(cc) * 1.0001f;
            }
        };
        for (int j = warp; j < k; j += kStepWarps) make_rec(j, lane < NP ? Cm[j * NP + lane] : 0.0);
        if ((k & 1) && warp == kStepWarps - 1) {  // odd k: the missing partner never wins
            float* rec = cs + (k >> 1) * (2 * G::RST) + 1;
            if (lane < G::NPF) rec[2 * lane] = 0.f;
            if (lane == 0) {
                rec[2 * G::NPF] = 1e38f;
                rec[2 * G::NPF + 2] = 0.f;
            }
        }
        __syncthreads();
        for (;; ++pass) {
            // max |c_j| over the centroids (records made by the previous means phase)
            const float cmax =
                __uint_as_float(__reduce_max_sync(0xffffffffu, lane < k ? __float_as_uint(sh.cnorm[lane]) : 0u));
            if (pass == 0 && (TRACE && p.trace_mode == 0)) mark();  // 5: prep done
            // ---- assign: fp32 FFMA2 screen, exact fp64 recheck of near ties. Rows are dealt
            // to warps as 32-row chunks (chunk c -> warp c % NW) and each warp screens 4, 2 or 1
            // of its chunks at a time, so warps differ by at most one chunk of work.
            if (lane < kMaxK) sh.wcnt[warp][lane] = 0;
            __syncwarp();
            const int nchunks = (nr + 31) / 32;
            const int nchw = warp < nchunks ? (nchunks - warp + kStepWarps - 1) / kStepWarps : 0;
            auto screen_chunks = [&](auto RRc, int t0) {
                constexpr int RR = decltype(RRc)::value;
                float2 x2[RR][G::NPF / 2];
                float xn[RR];
                bool valid[RR];
                int rowr[RR];
#pragma unroll
                for (int r = 0; r < RR; ++r) {
                    const int row = (warp + kStepWarps * (t0 + r)) * 32 + lane;
                    rowr[r] = row;
                    valid[r] = row < nr;
                    load_row_f32<T, NP>(samp, valid[r] ? row : 0, x2[r]);
                    float nn = 0.f;
#pragma unroll
                    for (int q = 0; q < G::NPF / 2; ++q) nn = fmaf(x2[r][q].x, x2[r][q].x, fmaf(x2[r][q].y, x2[r][q].y, nn));
                    xn[r] = sqrtf(nn);
                }
                float m1[RR], m2[RR];
                int i1[RR];
#pragma unroll
                for (int r = 0; r < RR; ++r) {
                    m1[r] = __int_as_float(0x7f800000);
                    m2[r] = __int_as_float(0x7f800000);
                    i1[r] = 0;
                }
                const int kp = (k + 1) >> 1;
#pragma unroll 1
                for (int jp = 0; jp < kp; ++jp) {
                    const float4* rq = reinterpret_cast<const float4*>(cs + jp * (2 * G::RST));
                    const float4 iv = rq[G::NPF / 2];
                    float2 acc[RR];
#pragma unroll
                    for (int r = 0; r < RR; ++r) acc[r] = make_float2(iv.x, iv.y);
#pragma unroll
                    for (int h = 0; h < G::NPF / 2; ++h) {
                        const float4 c = rq[h];
#pragma unroll
                        for (int r = 0; r < RR; ++r) {
                            acc[r] = __ffma2_rn(make_float2(x2[r][h].x, x2[r][h].x), make_float2(c.x, c.y), acc[r]);
                            acc[r] = __ffma2_rn(make_float2(x2[r][h].y, x2[r][h].y), make_float2(c.z, c.w), acc[r]);
                        }
                    }
#pragma unroll
                    for (int r = 0; r < RR; ++r) {  // sorted pair into the top-2
                        const float da = acc[r].x, db = acc[r].y;
                        const float lo = fminf(da, db), hi = fmaxf(da, db);
                        const int li = 2 * jp + (db < da ? 1 : 0);
                        m2[r] = fmin3f(m2[r], hi, fmaxf(m1[r], lo));
                        i1[r] = lo < m1[r] ? li : i1[r];
                        m1[r] = fminf(m1[r], lo);
                    }
                }
                // near ties (k == 1 gives m2 = inf: never): exact reference argmin, warp-parallel --
                // lane j evaluates centroid j, then a tie-aware shuffle argmin (core.hpp:146-157)
                unsigned ties[RR];
#pragma unroll
                for (int r = 0; r < RR; ++r) {
                    const float sc = xn[r] + cmax;
                    ties[r] = __ballot_sync(0xffffffffu, valid[r] && !(m2[r] - m1[r] > kappa * sc * sc));
                }
#pragma unroll
                for (int r = 0; r < RR; ++r) {
                    unsigned tie = ties[r];
                    while (tie) {
                        const int src = __ffs(tie) - 1;
                        tie &= tie - 1;
                        const int trow = rowr[r] - lane + src;
                        double dv = __longlong_as_double(0x7ff0000000000000LL);
                        int dj = lane;
                        if (lane < k) {
                            T xr[NP];
                            load_row_T<T, NP>(samp, trow, xr);
                            dv = exact_dist_regs<T, NP>(xr, Cm + lane * NP);
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
                // labels + stable counting-sort rank among this warp's rows of the same label
#pragma unroll
                for (int r = 0; r < RR; ++r) {
                    const int lab = i1[r];
                    const unsigned peers = __match_any_sync(0xffffffffu, valid[r] ? lab : 0xff);
                    const int rank = __popc(peers & ((1u << lane) - 1u));
                    const int base = valid[r] ? sh.wcnt[warp][lab] : 0;
                    __syncwarp();
                    if (valid[r]) {
                        labels[rowr[r]] = (uint8_t)lab;
                        if (rank == 0) sh.wcnt[warp][lab] = base + __popc(peers);
                        pos[rowr[r]] = (uint16_t)(base + rank);
                    }
                    __syncwarp();
                }
            };
            {
                int t = 0;
                for (; t + G::R <= nchw; t += G::R) screen_chunks(IntC<G::R>{}, t);
                if constexpr (G::R > 2) {
                    if (t + 2 <= nchw) {
                        screen_chunks(IntC<2>{}, t);
                        t += 2;
                    }
                }
                if (t < nchw) screen_chunks(IntC<1>{}, t);
            }
            if (pass == 0 && (TRACE && p.trace_mode == 0)) mark();  // 6: assign done
            __syncthreads();
            // CTA-wide stable counting sort by label: cluster ranges + (warp, label) offsets
            if (warp == 0) {
                int col = 0;
                for (int w2 = 0; w2 < kStepWarps; ++w2) col += lane < k ? sh.wcnt[w2][lane] : 0;
                int incl = col;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += y;
                }
                const int start = incl - col;
                if (lane < k) {
                    sh.cstart[lane] = start;
                    int run = start;
                    for (int w2 = 0; w2 < kStepWarps; ++w2) {
                        sh.woff[w2][lane] = run;
                        run += sh.wcnt[w2][lane];
                    }
                }
                if (lane == k - 1) sh.cstart[k] = incl;
            }
            __syncthreads();
            for (int t = 0; t < nchw; ++t) {
                const int row = (warp + kStepWarps * t) * 32 + lane;
                // VEC16 rows: the 16-B unit index of the row's chunk 0 with its swizzle folded in,
                // (row * CPR + swz(row)); chunk q of the row is unit (entry ^ q)
                if (row < nr)
                    perm[sh.woff[warp][labels[row]] + pos[row]] =
                        (uint16_t)(G::VEC16 ? row * G::CPR + G::swz(row) : row);
            }
            __syncthreads();
            if (pass == 0 && (TRACE && p.trace_mode == 0)) mark();  // 7: sort done
            // ---- update: sums / cost of the warp's own rows, cluster by cluster along its
            // label-sorted segment; per cluster the lanes cover ROWS_PER_STEP rows x
            // LANES_PER_ROW units (16-B chunks or single elements) so every smem read is a
            // vector load and no label test sits in the inner loop. Fixed order throughout.
            {
                constexpr int U = G::VEC16 ? 16 / (int)sizeof(T) : 1;       // elements per lane unit
                constexpr int UPR = G::VEC16 ? G::CPR : NP;                  // units per row
                constexpr int LR = UPR <= 1 ? 1 : UPR <= 2 ? 2 : UPR <= 4 ? 4 : UPR <= 8 ? 8 : UPR <= 16 ? 16 : 32;
                constexpr int RPS = 32 / LR;                                 // rows per step
                double* wp = wpart + warp * part_d;
                const int gi = lane / LR, q = lane % LR;
                const bool active_unit = q < UPR;
                const uint16_t* wperm = perm;
                double cost_w = 0.0;
                // this warp's contiguous range of the label-sorted order (1-3 clusters)
                const int Lw = (nr + kStepWarps - 1) / kStepWarps;
                const int lo = warp * Lw < nr ? warp * Lw : nr;
                const int hi = lo + Lw < nr ? lo + Lw : nr;
                for (int e = lane; e < part_d; e += 32) wp[e] = 0.0;
                __syncwarp();
                for (int j = 0; j < k; ++j) {
                    const int a = max(sh.cstart[j], lo), b = min(sh.cstart[j + 1], hi);
                    if (a >= b) continue;  // warp-uniform
                    double acc[U], cj[U], accc[U], acc2[U], accc2[U];
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        acc[u] = 0.0;
                        accc[u] = 0.0;
                        acc2[u] = 0.0;
                        accc2[u] = 0.0;
                        const int d = q * U + u;
                        cj[u] = (active_unit && d < NP) ? Cm[j * NP + d] : 0.0;
                    }
                    const unsigned char* sbytes = reinterpret_cast<const unsigned char*>(samp);
                    // row: perm entry (see the scatter above); two accumulator sets (even / odd steps)
                    // halve the fp64 dependency chains; the order stays fixed
                    auto add_row = [&](int row, double(&sa)[U], double(&sc)[U]) {
                        if constexpr (G::VEC16 && sizeof(T) == 4) {
                            const float4 v = *reinterpret_cast<const float4*>(sbytes + ((row ^ q) << 4));
                            const double xv[4] = {(double)v.x, (double)v.y, (double)v.z, (double)v.w};
#pragma unroll
                            for (int u = 0; u < 4; ++u) {
                                sa[u] += xv[u];
                                const double diff = xv[u] - cj[u];
                                sc[u] = fma(diff, diff, sc[u]);
                            }
                        } else if constexpr (G::VEC16) {
                            const double2 v = *reinterpret_cast<const double2*>(sbytes + ((row ^ q) << 4));
                            sa[0] += v.x;
                            sa[1] += v.y;
                            const double d0 = v.x - cj[0], d1 = v.y - cj[1];
                            sc[0] = fma(d0, d0, sc[0]);
                            sc[1] = fma(d1, d1, sc[1]);
                        } else {
                            const double xv = (double)samp[G::elem_off(row, q)];
                            sa[0] += xv;
                            const double diff = xv - cj[0];
                            sc[0] = fma(diff, diff, sc[0]);
                        }
                    };
                    if (active_unit) {
                        int p0 = a + gi;
#pragma unroll 2
                        for (; p0 + RPS < b; p0 += 2 * RPS) {
                            add_row(wperm[p0], acc, accc);
                            add_row(wperm[p0 + RPS], acc2, accc2);
                        }
                        if (p0 < b) add_row(wperm[p0], acc, accc);
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            acc[u] += acc2[u];
                            accc[u] += accc2[u];
                        }
                    }
                    // fold the row groups (fixed tree): lanes gi == 0 hold the sums
#pragma unroll
                    for (int o = 16; o >= LR; o >>= 1)
#pragma unroll
                        for (int u = 0; u < U; ++u) acc[u] += __shfl_down_sync(0xffffffffu, acc[u], o);
                    if (gi == 0 && active_unit)
#pragma unroll
                        for (int u = 0; u < U; ++u)
                            if (q * U + u < NP) wp[j * NP + q * U + u] = acc[u];
                    if (lane == 0) wp[k * NP + j] = (double)(b > a ? b - a : 0);
#pragma unroll
                    for (int u = 0; u < U; ++u) cost_w += accc[u];  // per lane; reduced once below
                }
                cost_w = warp_sum(cost_w);
                if (lane == 0) wp[k * NP + k] = cost_w;
            }
            __syncthreads();
            if (pass == 0 && (TRACE && p.trace_mode == 0)) mark();  // 8: update done
            // ---- CTA partial (warps in order) pushed to every CTA; totals in rank order
            const double* totx = reduce_all(part_d, [&](int e) {
                double v = 0.0;
                for (int w2 = 0; w2 < kStepWarps; ++w2) v += wpart[w2 * part_d + e];
                return v;
            });
            if (pass == 0 && (TRACE && p.trace_mode == 0)) mark();  // 9: partials pushed
            if (pass == 0 && (TRACE && p.trace_mode == 0)) mark();  // 10: exchange complete
            __syncthreads();  // every warp partial consumed before tot overwrites wpart
            double* tot = wpart;
            for (int e = tid; e < part_d; e += kStepThreads) tot[e] = totx[e];
            __syncthreads();
            if (pass == 0 && (TRACE && p.trace_mode == 0)) mark();  // 11: cluster reduce done
            const double f = tot[k * NP + k];
            if (hist_len > 0 && f > last * (1.0 + 1e-12)) {  // lloyd.hpp:114-121
                if (tid == 0) sh.err = kErrMonotone;
                stop = -1;
                break;
            }
            if (tid == 0 && cr == 0 && p.out_hist && hist_len < p.hist_cap) p.out_hist[(int64_t)wl * p.hist_cap + hist_len] = f;
            last = f;
            ++hist_len;
            nd += s * (int64_t)k;
            if (closing) {  // lloyd.hpp:155-163
                f_final = f;
                break;
            }
            ++iters;
            // means_from_sums (lloyd.hpp:75-89) + fixed-point test (lloyd.hpp:131), one warp per
            // centroid (lane = dimension; only that warp touches the centroid here), and the
            // next pass's screen record from the new means
            bool same = true;
            for (int j = warp; j < k; j += kStepWarps) {
                const double cnt = tot[k * NP + j];
                const double old = lane < NP ? Cm[j * NP + lane] : 0.0;
                double v = old;
                if (lane < NP && cnt > 0.0) {
                    const double inv = 1.0 / cnt;
                    v = tot[j * NP + lane] * inv;
                }
                same &= (v == old);
                if (lane < NP) Cm[j * NP + lane] = v;
                make_rec(j, v);
            }
            const bool all_same = __syncthreads_and(same);
            if (all_same) {
                stop = 2;  // fixed_point
                f_final = f;
                __syncthreads();
                break;
            }
            bool go_close = false;
            if (isfinite(f_prev)) {
                const double improvement = f_prev > 0.0 ? (f_prev - f) / f_prev : 0.0;
                if (improvement < p.rel_tol) {
                    stop = 0;  // tolerance
                    go_close = true;
                }
            }
            f_prev = f;
            if (!go_close && iters == p.max_iters) {
                stop = 1;
                go_close = true;
            }
            closing = go_close;
            __syncthreads();
            if (pass == 0 && (TRACE && p.trace_mode == 0)) mark();  // 12: means done
        }
        // outputs of the last pass: labels (sample order), flags = empty clusters
        if (stop >= 0) {
            if (p.out_labels)
                for (int li = tid; li < nr; li += kStepThreads)
                    p.out_labels[(int64_t)wl * s + r0 + li] = (int32_t)labels[li];
            const double* tot = wpart;
            if (tid < k) sh.flags[tid] = tot[k * NP + tid] == 0.0 ? 1 : 0;
            if (p.out_counts && cr == 0 && tid < k) p.out_counts[(int64_t)wl * k + tid] = (int64_t)tot[k * NP + tid];
        }
    }
    __syncthreads();

    // ------------------------------------------------------------- outputs
    if (cr == 0) {
        const int64_t kn = (int64_t)k * n;
        if (p.out_c)
            for (int e = tid; e < kn; e += kStepThreads) {
                const int j = e / n, d = e - j * n;
                p.out_c[(int64_t)wl * kn + e] = Cm[j * NP + d];
            }
        if (p.out_f && tid < k) p.out_f[(int64_t)wl * k + tid] = sh.flags[tid];
        if (tid == 0) {
            const int err = sh.err;
            if (p.out_obj) p.out_obj[wl] = f_final;
            if (p.out_iters) p.out_iters[wl] = iters;
            if (p.out_stop) p.out_stop[wl] = stop;
            if (p.out_nd) p.out_nd[wl] = nd;
            if (p.out_filled) p.out_filled[wl] = filled;
            if (p.out_err) p.out_err[wl] = err;
            if (p.out_hist_len) p.out_hist_len[wl] = hist_len;
        }
        // keep-the-best (engine.hpp:254, strict <)
        if (p.inc_obj) {
            const bool acc = run_lloyd && sh.err == kErrNone && f_final < p.inc_obj[wl];
            __syncthreads();
            if (acc) {
                for (int e = tid; e < kn; e += kStepThreads) {
                    const int j = e / n, d = e - j * n;
                    p.inc_c[(int64_t)wl * kn + e] = Cm[j * NP + d];
                }
                if (tid < k) p.inc_f[(int64_t)wl * k + tid] = sh.flags[tid];
            }
            __syncthreads();
            if (tid == 0) {
                if (acc) p.inc_obj[wl] = f_final;
                p.accepted[wl] = acc ? 1 : 0;
            }
        }
    }
    if (trace && tid == 0) {
        if ((TRACE && p.trace_mode == 1)) {
            trace[kTraceSlots - 3] = sh.exact_passes;
            trace[kTraceSlots - 4] = sh.exact_rows;
            trace[kTraceSlots - 7] = sh.exact_rows1;
        }
        trace[kTraceSlots - 5] = clock64();
        trace[kTraceSlots - 2] = gtimer();
    }
    cluster.sync();  // no CTA may exit while peers can still read its smem
    if (trace && tid == 0) trace[kTraceSlots - 1] = gtimer();
}

}  // namespace hpcg
