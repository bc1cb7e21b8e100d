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

constexpr int kStepThreads = 256;  // 2 CTAs per SM: one cluster gathers while another computes
constexpr int kStepWarps = kStepThreads / 32;
constexpr int kMaxK = 32;          // label fits u8 and the per-warp partial table fits smem
constexpr int kMaxCandidates = 8;  // K-means++ candidates per slot evaluated in one sweep

enum StepErr : int32_t { kErrNone = 0, kErrDegenerateInit = 1, kErrMonotone = 2 };

struct StepParams {
    // sample source
    const void* X;
    int64_t m;
    int32_t n;
    int64_t s;
    int32_t W;            // workers in this launch (one cluster each)
    int32_t sample_mode;  // 0 explicit idx[W*s], 1 Philox PRP over [0,m), 2 contiguous (X is [W*s x n])
    const int64_t* idx;
    uint64_t key;        // Philox key (sample PRP and K-means++ draws)
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
};

// ------------------------------------------------------------- smem geometry
template <typename T, int NP>
struct Geo {
    static constexpr int RS = NP * (int)sizeof(T);            // sample row bytes in smem
    static constexpr bool VEC16 = (RS % 16) == 0;              // 16-B chunks (swizzled)
    static constexpr int CPR = VEC16 ? RS / 16 : 1;            // chunks per row
    static constexpr int NPF = (NP + 1) & ~1;                  // fp32 screen dims (pairs)
    static constexpr int CSR = ((NPF + 2) + 3) & ~3;           // screen record floats (16-B mult)
    static constexpr int R = NP <= 16 ? 4 : 2;                 // rows per thread in the assign pass
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
    int labels, pos, perm, wpart, d2, gidx;
};

template <typename T, int NP>
__host__ __device__ inline SmemLayout step_layout(int rows_cap, int k) {
    using G = Geo<T, NP>;
    SmemLayout L;
    auto up = [](int v) { return (v + 15) & ~15; };
    const int part_d = k * NP + k + 1;
    L.samp = 0;
    L.cm = up(L.samp + rows_cap * G::RS);
    L.cs = up(L.cm + k * NP * 8);
    L.part = up(L.cs + k * G::CSR * 4);
    L.scratch = up(L.part + 2 * part_d * 8);
    L.labels = L.scratch;
    L.pos = up(L.labels + rows_cap);
    L.perm = up(L.pos + rows_cap * 2);
    L.wpart = up(L.perm + rows_cap * 2);
    const int lloyd_end = L.wpart + kStepWarps * part_d * 8;
    L.d2 = L.scratch;    // seeding only
    L.gidx = L.scratch;  // gather only
    const int seed_end = L.d2 + rows_cap * 8;
    L.total = up(lloyd_end > seed_end ? lloyd_end : seed_end);
    return L;
}

struct StepShared {  // static smem: per-step scalars and exchange slots
    uint8_t flags[kMaxK];
    int32_t pending[kMaxK];
    int32_t n_pending, n_valid;
    double xch_total[2];                     // CTA CDF totals (parity buffered)
    long long xch_hit[2][kMaxCandidates];    // first CDF hit per candidate
    double xch_cost[2][kMaxCandidates];      // candidate cost partials
    double cand[kMaxCandidates][32];         // candidate coordinates (fp64, n <= 32)
    double wsum[kStepWarps][kMaxCandidates];
    double rank_val[16];
    double rank_cost[kMaxCandidates][16];
    double wtot[kStepWarps];
    long long whit[kStepWarps][kMaxCandidates];
    float cmax;
    int32_t wcnt[kStepWarps][kMaxK];  // per-warp label counts (counting sort)
    int32_t woff[kStepWarps][kMaxK];  // sorted-order offset of (warp, label)
    int32_t cstart[kMaxK + 1];        // sorted-order start of each cluster
    int32_t decision;  // 0 continue, 1 done
    int32_t err;
};

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
HPCG_DEV void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }
HPCG_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
HPCG_DEV void cp_async_wait_group() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// ------------------------------------------------------------------ the kernel
template <typename T, int NP>
__global__ void __launch_bounds__(kStepThreads, 2) worker_step_kernel(const StepParams p) {
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
    const SmemLayout L = step_layout<T, NP>(p.rows_cap, k);
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

    // ---------------------------------------------------------------- gather
    {
        const T* X = static_cast<const T*>(p.X);
        FeistelPRP prp;
        if (p.sample_mode == 1) prp = FeistelPRP::make(p.key, p.round, (uint32_t)(p.worker_base + wl), (uint64_t)p.m);
        auto gidx_of = [&](int64_t i) -> int64_t {
            if (p.sample_mode == 0) return p.idx[(int64_t)wl * s + i];
            if (p.sample_mode == 1) return (int64_t)prp((uint64_t)i);
            return (int64_t)wl * s + i;
        };
        // (a) one sample index per row into smem; (b) every copy is issued before any is
        // awaited (cp.async, no register staging) so the CTA's whole chunk is in flight at once
        int64_t* gx = reinterpret_cast<int64_t*>(smem + L.gidx);
        for (int li = tid; li < nr; li += kStepThreads) gx[li] = gidx_of(r0 + li);
        __syncthreads();
        const int rowb = n * (int)sizeof(T);
        if ((rowb & 15) == 0) {  // 16-B chunks
            const int cpr = rowb >> 4;
            constexpr int EPC = 16 / (int)sizeof(T);
            for (int e = tid; e < nr * cpr; e += kStepThreads) {
                const int li = e / cpr, q = e - li * cpr;
                cp_async16(samp + G::elem_off(li, q * EPC), X + gx[li] * n + q * EPC);
            }
        } else if ((rowb & 7) == 0) {  // 8-B chunks
            const int cpr = rowb >> 3;
            constexpr int EPC = 8 / (int)sizeof(T);
            for (int e = tid; e < nr * cpr; e += kStepThreads) {
                const int li = e / cpr, q = e - li * cpr;
                cp_async8(samp + G::elem_off(li, q * EPC), X + gx[li] * n + q * EPC);
            }
        } else {  // 4-B elements (fp32, odd n)
            for (int e = tid; e < nr * n; e += kStepThreads) {
                const int li = e / n, d = e - li * n;
                cp_async4(samp + G::elem_off(li, d), X + gx[li] * n + d);
            }
        }
        if (NP > n)
            for (int e = tid; e < nr * (NP - n); e += kStepThreads) {
                const int li = e / (NP - n), d = n + (e - li * (NP - n));
                samp[G::elem_off(li, d)] = T(0);
            }
        // initial centroids (fp64 master, zero padded) and flags
        const int64_t v = p.shared_version ? *p.shared_version : 1;
        const double* ic = p.init_c + (int64_t)wl * p.init_stride;
        const uint8_t* ifl = p.init_f + (int64_t)wl * p.initf_stride;
        for (int e = tid; e < k * NP; e += kStepThreads) {
            const int j = e / NP, d = e - j * NP;
            Cm[e] = (d < n && v != 0) ? ic[(int64_t)j * n + d] : 0.0;
        }
        if (tid < k) sh.flags[tid] = v != 0 ? ifl[tid] : (uint8_t)1;
        if (tid == 0) {
            sh.err = kErrNone;
            int np_ = 0, nv = 0;
            for (int j = 0; j < k; ++j) {
                const uint8_t f = v != 0 ? ifl[j] : (uint8_t)1;
                if (f)
                    sh.pending[np_++] = j;
                else
                    ++nv;
            }
            sh.n_pending = np_;
            sh.n_valid = nv;
        }
    }
    cp_async_wait_all();
    __syncthreads();  // gx (aliases d2) fully consumed before seeding reuses the region
    cluster.sync();  // sample rows of every CTA now visible cluster-wide (DSMEM)

    int64_t nd = 0;  // distance evaluations (reference accounting)
    int filled = 0;

    // --------------------------------------------------------------- seeding
    // seeding.hpp:47-105. d2 and every candidate cost use the exact reference
    // distance; the CDF is a fixed-order (segment, block, rank) prefix sum.
    if (sh.n_pending > 0) {
        const int np_ = sh.n_pending;
        const int ncand = p.candidates;
        for (int li = tid; li < nr; li += kStepThreads) d2[li] = __longlong_as_double(0x7ff0000000000000LL);
        __syncthreads();
        // valid centres in slot order (seeding.hpp:60-68)
        for (int j = 0; j < k; ++j) {
            if (sh.flags[j]) continue;
            for (int li = tid; li < nr; li += kStepThreads) {
                double dd = 0.0;
                for (int d = 0; d < n; ++d) {
                    const double diff = __dsub_rn((double)samp[G::elem_off(li, d)], Cm[j * NP + d]);
                    dd = __dadd_rn(dd, __dmul_rn(diff, diff));
                }
                d2[li] = fmin(d2[li], dd);
            }
            nd += s;
        }
        // fetch a sample row (global sample position) from its owner CTA into dst[n]
        auto fetch_row = [&](int64_t row, double* dst) {
            // owner rank: invert chunk_range
            const int64_t base = s / C, extra = s % C;
            int owner;
            if (row < extra * (base + 1))
                owner = (int)(row / (base + 1));
            else
                owner = (int)(extra + (row - extra * (base + 1)) / (base > 0 ? base : 1));
            int64_t ob, oe;
            chunk_range(s, C, owner, ob, oe);
            const T* rs = cluster.map_shared_rank(samp, owner);
            const int lr = (int)(row - ob);
            for (int d = lane; d < n; d += 32) dst[d] = (double)rs[G::elem_off(lr, d)];
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
                for (int d = lane; d < NP; d += 32) Cm[j * NP + d] = d < n ? sh.cand[0][d] : 0.0;
                if (lane == 0) sh.flags[j] = 0;
            }
            __syncthreads();
            for (int li = tid; li < nr; li += kStepThreads) {
                double dd = 0.0;
                for (int d = 0; d < n; ++d) {
                    const double diff = __dsub_rn((double)samp[G::elem_off(li, d)], Cm[j * NP + d]);
                    dd = __dadd_rn(dd, __dmul_rn(diff, diff));
                }
                d2[li] = fmin(d2[li], dd);
            }
            nd += s;
            ++filled;
            __syncthreads();  // d2 written row-strided above, read per contiguous segment below
        }
        // per-thread contiguous segment of local rows for the CDF
        const int seg = (nr + kStepThreads - 1) / kStepThreads;
        const int sb = tid * seg < nr ? tid * seg : nr;
        const int se = sb + seg < nr ? sb + seg : nr;
        int it = 0;
        for (; next < np_; ++next, ++it) {
            const int par = it & 1;
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
            double wexcl = 0.0;
            for (int w2 = 0; w2 < warp; ++w2) wexcl += sh.wtot[w2];
            const double texcl = wexcl + lexcl;  // exclusive prefix of this thread's segment
            // CTA total := local cum at the CTA's last row, computed exactly as the search does
            if (se == nr && sb < se) {
                double run = 0.0;
                for (int li = sb; li < se; ++li) run += d2[li];
                sh.xch_total[par] = texcl + run;
            }
            cluster.sync();
            // P = sum of lower ranks' totals (rank order); total = P_{C-1} + T_{C-1}
            if (warp == 0 && lane < C) sh.rank_val[lane] = *cluster.map_shared_rank(&sh.xch_total[par], lane);
            __syncthreads();
            double P = 0.0, total = 0.0;
            {
                double acc = 0.0;
                for (int rr = 0; rr < C; ++rr) {
                    const double tr = sh.rank_val[rr];
                    if (rr == cr) P = acc;
                    if (rr == C - 1)
                        total = acc + tr;
                    else
                        acc += tr;
                }
            }
            if (!(total > 0.0)) break;  // distinct rows exhausted (seeding.hpp:87)
            // (2) candidate draws u_c = unit * total; first global row with cum > u_c
            double u[kMaxCandidates];
            for (int c = 0; c < ncand; ++c) {
                const double unit = p.seed_mode == 0
                                        ? p.units[(int64_t)wl * p.units_stride + (int64_t)it * ncand + c]
                                        : philox_unit(p.key, p.round, (uint32_t)(p.worker_base + wl),
                                                      (uint32_t)(0x10000 + next * kMaxCandidates + c));
                u[c] = unit * total;
            }
            long long hit[kMaxCandidates];
            for (int c = 0; c < ncand; ++c) hit[c] = LLONG_MAX;
            {
                double run = 0.0;
                for (int li = sb; li < se; ++li) {
                    run += d2[li];
                    const double cum = P + (texcl + run);
                    for (int c = 0; c < ncand; ++c)
                        if (hit[c] == LLONG_MAX && cum > u[c]) hit[c] = r0 + li;
                }
            }
            for (int c = 0; c < ncand; ++c) {
                long long h = hit[c];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) h = min(h, __shfl_xor_sync(0xffffffffu, h, o));
                if (lane == 0) sh.whit[warp][c] = h;
            }
            __syncthreads();
            if (tid < ncand) {
                long long h = LLONG_MAX;
                for (int w2 = 0; w2 < kStepWarps; ++w2) h = min(h, sh.whit[w2][tid]);
                sh.xch_hit[par][tid] = h;
            }
            cluster.sync();
            // every CTA: global first hit per candidate (rank order == row order)
            for (int c = warp; c < ncand; c += kStepWarps) {
                long long h = lane < C ? *cluster.map_shared_rank(&sh.xch_hit[par][c], lane) : LLONG_MAX;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) h = min(h, __shfl_xor_sync(0xffffffffu, h, o));
                const int64_t row = h == LLONG_MAX ? s - 1 : (int64_t)h;  // rng.hpp:87-92 fallback
                fetch_row(row, sh.cand[c]);
            }
            __syncthreads();
            // (3) candidate costs sum_i min(d2_i, dist(S_i, cand_c)), fixed order
            double cost[kMaxCandidates];
            for (int c = 0; c < ncand; ++c) cost[c] = 0.0;
            for (int li = sb; li < se; ++li) {
                for (int c = 0; c < ncand; ++c) {
                    double dd = 0.0;
                    for (int d = 0; d < n; ++d) {
                        const double diff = __dsub_rn((double)samp[G::elem_off(li, d)], sh.cand[c][d]);
                        dd = __dadd_rn(dd, __dmul_rn(diff, diff));
                    }
                    cost[c] += fmin(d2[li], dd);
                }
            }
            for (int c = 0; c < ncand; ++c) {
                const double v = warp_sum(cost[c]);
                if (lane == 0) sh.wsum[warp][c] = v;
            }
            __syncthreads();
            if (tid < ncand) {
                double v = 0.0;
                for (int w2 = 0; w2 < kStepWarps; ++w2) v += sh.wsum[w2][tid];
                sh.xch_cost[par][tid] = v;
            }
            cluster.sync();
            for (int e = tid; e < ncand * C; e += kStepThreads) {
                const int c = e / C, rr = e - c * C;
                sh.rank_cost[c][rr] = *cluster.map_shared_rank(&sh.xch_cost[par][c], rr);
            }
            __syncthreads();
            int best = 0;
            {
                double bc = __longlong_as_double(0x7ff0000000000000LL);
                for (int c = 0; c < ncand; ++c) {
                    double tc = 0.0;
                    for (int rr = 0; rr < C; ++rr) tc += sh.rank_cost[c][rr];
                    if (tc < bc) {  // strict <, first candidate wins ties (seeding.hpp:94-98)
                        bc = tc;
                        best = c;
                    }
                }
            }
            nd += (int64_t)ncand * s;
            const int j = sh.pending[next];
            __syncthreads();
            for (int d = tid; d < NP; d += kStepThreads) Cm[j * NP + d] = d < n ? sh.cand[best][d] : 0.0;
            if (tid == 0) sh.flags[j] = 0;
            for (int li = tid; li < nr; li += kStepThreads) {
                double dd = 0.0;
                for (int d = 0; d < n; ++d) {
                    const double diff = __dsub_rn((double)samp[G::elem_off(li, d)], sh.cand[best][d]);
                    dd = __dadd_rn(dd, __dmul_rn(diff, diff));
                }
                d2[li] = fmin(d2[li], dd);
            }
            ++filled;
            __syncthreads();
        }
        __syncthreads();
    }

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
        constexpr float kappa = 2.0f * (float)(G::NPF / 2 + 12) * 5.9604645e-8f;
        bool closing = false;
        int pass = 0;
        const int ngroups = (nr + G::GROUP - 1) / G::GROUP;
        for (;; ++pass) {
            // ---- screen prep: c' = -2c (fp32), cc = |c|^2, cmax
            if (tid < k) {
                const int j = tid;
                float* rec = cs + j * G::CSR;
                double cc = 0.0;
                for (int d = 0; d < NP; ++d) {
                    const double c = Cm[j * NP + d];
                    cc += c * c;
                    rec[d] = (float)(-2.0 * c);
                }
                for (int d = NP; d < G::NPF; ++d) rec[d] = 0.f;
                rec[G::NPF] = (float)cc;
                rec[G::NPF + 1] = 0.f;
            }
            __syncthreads();
            if (tid == 0) {  // max |c_j| (k <= 32): scales the screen's error bound
                float cm = 0.f;
                for (int j = 0; j < k; ++j) cm = fmaxf(cm, sqrtf(cs[j * G::CSR + G::NPF]) * 1.0001f);
                sh.cmax = cm;
            }
            __syncthreads();
            const float cmax = sh.cmax;

            // ---- assign: fp32 FFMA2 screen, exact fp64 recheck of near ties
            if (lane < kMaxK) sh.wcnt[warp][lane] = 0;
            __syncwarp();
            for (int g = warp; g < ngroups; g += kStepWarps) {
                float2 x2[G::R][G::NPF / 2];
                float xn[G::R];
                bool valid[G::R];
#pragma unroll
                for (int r = 0; r < G::R; ++r) {
                    const int row = g * G::GROUP + r * 32 + lane;
                    valid[r] = row < nr;
                    const int rowc = valid[r] ? row : 0;
                    if constexpr (G::VEC16 && sizeof(T) == 4) {
#pragma unroll
                        for (int q = 0; q < NP / 4; ++q) {
                            const float4 v = *reinterpret_cast<const float4*>(samp + G::elem_off(rowc, q * 4));
                            x2[r][2 * q] = make_float2(v.x, v.y);
                            x2[r][2 * q + 1] = make_float2(v.z, v.w);
                        }
                    } else if constexpr (G::VEC16) {  // fp64, 16-B chunks of 2 doubles
#pragma unroll
                        for (int q = 0; q < NP / 2; ++q) {
                            const double2 v = *reinterpret_cast<const double2*>(samp + G::elem_off(rowc, q * 2));
                            x2[r][q] = make_float2((float)v.x, (float)v.y);
                        }
                    } else {
#pragma unroll
                        for (int q = 0; q < G::NPF / 2; ++q) {
                            const float a = (float)samp[G::elem_off(rowc, 2 * q)];
                            const float b = 2 * q + 1 < NP ? (float)samp[G::elem_off(rowc, 2 * q + 1)] : 0.f;
                            x2[r][q] = make_float2(a, b);
                        }
                    }
                    float nn = 0.f;
#pragma unroll
                    for (int q = 0; q < G::NPF / 2; ++q) nn = fmaf(x2[r][q].x, x2[r][q].x, fmaf(x2[r][q].y, x2[r][q].y, nn));
                    xn[r] = sqrtf(nn);
                }
                float m1[G::R], m2[G::R];
                int i1[G::R];
#pragma unroll
                for (int r = 0; r < G::R; ++r) {
                    m1[r] = __int_as_float(0x7f800000);
                    m2[r] = __int_as_float(0x7f800000);
                    i1[r] = 0;
                }
                for (int j = 0; j < k; ++j) {
                    const float* rec = cs + j * G::CSR;
                    float2 c2[G::NPF / 2];
#pragma unroll
                    for (int q = 0; q < G::NPF / 2; ++q) c2[q] = *reinterpret_cast<const float2*>(rec + 2 * q);
                    const float2 init = *reinterpret_cast<const float2*>(rec + G::NPF);
#pragma unroll
                    for (int r = 0; r < G::R; ++r) {
                        float2 acc = init;
#pragma unroll
                        for (int q = 0; q < G::NPF / 2; ++q) acc = __ffma2_rn(x2[r][q], c2[q], acc);
                        const float dj = acc.x + acc.y;
                        m2[r] = fminf(m2[r], fmaxf(m1[r], dj));
                        const bool lt = dj < m1[r];
                        m1[r] = fminf(m1[r], dj);
                        i1[r] = lt ? j : i1[r];
                    }
                }
#pragma unroll
                for (int r = 0; r < G::R; ++r) {
                    const int row = g * G::GROUP + r * 32 + lane;
                    int lab = i1[r];
                    if (valid[r]) {
                    const float sc = xn[r] + cmax;
                    if (!(m2[r] - m1[r] > kappa * sc * sc)) {  // near tie (or k == 1 -> m2 = inf skips)
                        double best = __longlong_as_double(0x7ff0000000000000LL);
                        lab = 0;
                        for (int j = 0; j < k; ++j) {
                            double dd = 0.0;
                            for (int d = 0; d < n; ++d) {
                                const double diff = __dsub_rn((double)samp[G::elem_off(row, d)], Cm[j * NP + d]);
                                dd = __dadd_rn(dd, __dmul_rn(diff, diff));
                            }
                            if (dd < best) {
                                best = dd;
                                lab = j;
                            }
                        }
                    }
                    labels[row] = (uint8_t)lab;
                    }
                    // stable counting-sort rank of this row among the warp's rows with its label
                    const unsigned peers = __match_any_sync(0xffffffffu, valid[r] ? lab : 0xff);
                    const int rank = __popc(peers & ((1u << lane) - 1u));
                    const int base = valid[r] ? sh.wcnt[warp][lab] : 0;
                    __syncwarp();
                    if (valid[r]) {
                        if (rank == 0) sh.wcnt[warp][lab] = base + __popc(peers);
                        pos[row] = (uint16_t)(base + rank);
                    }
                    __syncwarp();
                }
            }
            __syncthreads();
            // cluster ranges of the sorted order and (warp, label) offsets
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
            for (int li = tid; li < nr; li += kStepThreads) {
                const int w2 = (li / G::GROUP) % kStepWarps;
                perm[sh.woff[w2][labels[li]] + pos[li]] = (uint16_t)li;
            }
            __syncthreads();

            // ---- update: sums / cost along the label-sorted order. Warp w owns sorted
            // positions [w*L, (w+1)*L); per cluster its lanes cover ROWS_PER_STEP rows x
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
                const int Lw = (nr + kStepWarps - 1) / kStepWarps;
                const int lo = warp * Lw < nr ? warp * Lw : nr;
                const int hi = lo + Lw < nr ? lo + Lw : nr;
                double cost_w = 0.0;
                for (int j = 0; j < k; ++j) {
                    const int a = max(sh.cstart[j], lo), b = min(sh.cstart[j + 1], hi);
                    double acc[U], cj[U];
                    double accc = 0.0;
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        acc[u] = 0.0;
                        const int d = q * U + u;
                        cj[u] = (active_unit && d < NP) ? Cm[j * NP + d] : 0.0;
                    }
                    for (int p0 = a; p0 < b; p0 += RPS) {
                        const int pp = p0 + gi;
                        if (pp < b && active_unit) {
                            const int row = perm[pp];
                            if constexpr (G::VEC16 && sizeof(T) == 4) {
                                const float4 v = *reinterpret_cast<const float4*>(samp + G::elem_off(row, q * 4));
                                const double xv[4] = {(double)v.x, (double)v.y, (double)v.z, (double)v.w};
#pragma unroll
                                for (int u = 0; u < 4; ++u) {
                                    acc[u] += xv[u];
                                    const double diff = xv[u] - cj[u];
                                    accc = fma(diff, diff, accc);
                                }
                            } else if constexpr (G::VEC16) {
                                const double2 v = *reinterpret_cast<const double2*>(samp + G::elem_off(row, q * 2));
                                acc[0] += v.x;
                                acc[1] += v.y;
                                const double d0 = v.x - cj[0], d1 = v.y - cj[1];
                                accc = fma(d0, d0, accc);
                                accc = fma(d1, d1, accc);
                            } else {
                                const double xv = (double)samp[G::elem_off(row, q)];
                                acc[0] += xv;
                                const double diff = xv - cj[0];
                                accc = fma(diff, diff, accc);
                            }
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
                    cost_w += warp_sum(accc);
                }
                if (lane == 0) wp[k * NP + k] = cost_w;
            }
            __syncthreads();
            // ---- CTA partial (warps in order) -> cluster exchange
            double* pb = part + (pass & 1) * part_d;
            for (int e = tid; e < part_d; e += kStepThreads) {
                double v = 0.0;
                for (int w2 = 0; w2 < kStepWarps; ++w2) v += wpart[w2 * part_d + e];
                pb[e] = v;
            }
            cluster.sync();
            // totals in rank order (identical in every CTA), new means
            double* tot = wpart;  // reuse (warp partials consumed)
            for (int e = tid; e < part_d; e += kStepThreads) {
                double t = 0.0;  // batches of remote loads issued before the (rank-ordered) sum
                for (int r8 = 0; r8 < C; r8 += 8) {
                    double v[8];
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        if (r8 + q < C) v[q] = cluster.map_shared_rank(pb, r8 + q)[e];
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        if (r8 + q < C) t = (r8 + q == 0) ? v[q] : t + v[q];
                }
                tot[e] = t;
            }
            __syncthreads();
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
            // means_from_sums (lloyd.hpp:75-89) + fixed-point test (lloyd.hpp:131)
            bool same = true;
            double nv[(kMaxK * 32 + kStepThreads - 1) / kStepThreads];
            {
                int q = 0;
                for (int e = tid; e < k * NP; e += kStepThreads, ++q) {
                    const int j = e / NP;
                    const double cnt = tot[k * NP + j];
                    double v = Cm[e];
                    if (cnt > 0.0) {
                        const double inv = 1.0 / cnt;
                        v = tot[e] * inv;
                    }
                    nv[q] = v;
                    same &= (v == Cm[e]);
                }
            }
            const bool all_same = __syncthreads_and(same);
            {
                int q = 0;
                for (int e = tid; e < k * NP; e += kStepThreads, ++q) Cm[e] = nv[q];
            }
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
    cluster.sync();  // no CTA may exit while peers can still read its smem
}

}  // namespace hpcg
