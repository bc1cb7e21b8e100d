#include <cstdlib>
#include <cstring>
// The HPClust worker step for shapes the cluster-resident kernel cannot hold: n > 32 features
// (config 4: n = 128), k > 32 centres, or samples larger than a 16-CTA cluster's shared
// memory. Same contract as worker_step_kernel (StepParams in, the same per-worker outputs,
// acceptance and n_d accounting out), built from grid-wide kernels over samples materialised
// in HBM:
//
//   gather     sample rows -> S[w][i][:]                     engine.hpp:165-177 (PRP indices)
//   seeding    D^2 init, per pending slot: block CDF totals, draw, candidate costs, decision,
//              D^2 update                                    seeding.hpp:47-105
//   Lloyd      per pass: assign + per-CTA partial sums/counts/cost, fixed-order reduce, means,
//              stop rules                                    lloyd.hpp:75-89, 100-164
//   outputs    centroids, flags, objective, iterations, stop, n_d, keep-the-best (engine.hpp:254)
//
// Distances are the reference's own (core.hpp:100-108: fp64, ascending d, separately rounded
// sub/mul/add), so labels and argmins are exact by construction. Every reduction is in a fixed
// order (row blocks in order, CTAs in order), so results are deterministic.
#include <algorithm>
#include <type_traits>
#include <map>
#include <mutex>
#include "launch.h"

#include <cudaTypedefs.h>
#include "objective_tcw.cuh"

namespace hpcg {
namespace {

constexpr int kWT = 256;           // threads per CTA
constexpr int kSeedRows = 256;     // rows per seeding block (CDF and cost partials)
constexpr int kJT = 8;             // centroids per distance tile (registers)

// ---------------------------------------------------------------- per-worker state
struct WState {
    int32_t n_pending, n_valid, next, it, filled, seed_stop;  // seeding progress
    int32_t best;                                             // winner of the current slot
    int32_t ambig;  // the slot's interval costs did not separate the winner: exact cost pass pending
    int32_t iters, stop, hist_len, closing, done, err, run_lloyd;
    int64_t nd;
    double f_prev, last, f_final;
};

struct WideBufs {  // device scratch for one worker batch
    void* S = nullptr;
    double* bcost_hi = nullptr;  // upper ends of the candidate-cost partials (interval pass)
    double *Cm = nullptr, *d2 = nullptr, *cand = nullptr, *btot = nullptr, *bcost = nullptr,
           *part = nullptr, *lastcnt = nullptr;
    uint8_t* flags = nullptr;
    uint8_t* rflag = nullptr;  // [Wb][s] per-row candidate flags of the current K-means++ slot
    int32_t *pend = nullptr, *labels = nullptr, *active = nullptr;
    WState* st = nullptr;
};

// the reference distance (core.hpp:100-108) of one row to JT centroids (row-major, stride n),
// in registers; centroids past jn are skipped
template <typename T>
__device__ __forceinline__ void dist_tile(const T* __restrict__ x, int n, const double* __restrict__ C, int jn,
                                          double (&acc)[kJT]) {
#pragma unroll
    for (int j = 0; j < kJT; ++j) acc[j] = 0.0;
    for (int d = 0; d < n; ++d) {
        const double xv = (double)x[d];
#pragma unroll
        for (int j = 0; j < kJT; ++j)
            if (j < jn) {
                const double diff = __dsub_rn(xv, __ldg(C + (int64_t)j * n + d));
                acc[j] = __dadd_rn(acc[j], __dmul_rn(diff, diff));
            }
    }
}

// the reference distance of one row to one centroid, row read in 16-B pieces (float4 /
// double2) when aligned: same ascending-d, separately rounded arithmetic as dist_tile
template <typename T>
__device__ __forceinline__ double dist1(const T* __restrict__ x, int n, const double* __restrict__ c, bool vec) {
    double acc = 0.0;
    int d = 0;
    if (vec) {
        constexpr int E = 16 / (int)sizeof(T);
        for (; d + E <= n; d += E) {
            double xv[E];
            if constexpr (sizeof(T) == 4) {
                const float4 f = __ldg(reinterpret_cast<const float4*>(x + d));
                xv[0] = f.x;
                xv[1] = f.y;
                xv[2] = f.z;
                xv[3] = f.w;
            } else {
                const double2 f = __ldg(reinterpret_cast<const double2*>(x + d));
                xv[0] = f.x;
                xv[1] = f.y;
            }
#pragma unroll
            for (int u = 0; u < E; ++u) {
                const double diff = __dsub_rn(xv[u], __ldg(c + d + u));
                acc = __dadd_rn(acc, __dmul_rn(diff, diff));
            }
        }
    }
    for (; d < n; ++d) {
        const double diff = __dsub_rn((double)x[d], __ldg(c + d));
        acc = __dadd_rn(acc, __dmul_rn(diff, diff));
    }
    return acc;
}

// fixed-order tree sum over a CTA of AT threads; result in every thread
template <int AT>
__device__ double cta_sum_t(double v, double* red) {
    const int tid = threadIdx.x;
    red[tid] = v;
    __syncthreads();
#pragma unroll
    for (int o = AT / 2; o > 0; o >>= 1) {
        if (tid < o) red[tid] = red[tid] + red[tid + o];
        __syncthreads();
    }
    const double r = red[0];
    __syncthreads();
    return r;
}

// fixed-order tree sum over the CTA (kWT threads); result valid in thread 0
__device__ double cta_sum(double v, double* red) {
    const int tid = threadIdx.x;
    red[tid] = v;
    __syncthreads();
#pragma unroll
    for (int o = kWT / 2; o > 0; o >>= 1) {
        if (tid < o) red[tid] = red[tid] + red[tid + o];
        __syncthreads();
    }
    const double r = red[0];
    __syncthreads();
    return r;
}

// ---------------------------------------------------------------- fp32 screen
// d~_j = |c_j|^2 + x.(-2c_j) in fp32 (FFMA2 pairs, two chains of n/2 terms like the resident
// kernel's screen), top-2 tracked; |d~_j - exact| <= kappa (|x| + cmax)^2 with
// kappa = 2 (ceil(n/2) + 12) 2^-24 (covers fp64 inputs rounded to fp32). Rows whose best and
// second-best are within the bound get the exact reference argmin. Records: rec[j][0..n) = -2c_j
// (fp32, rows padded to kKT multiples with zeros), ccs[j] = |c_j|^2 (+inf on padding rows).
constexpr int kKT = 16;  // centroids per screen tile

template <typename T>
__device__ __forceinline__ float4 load4(const T* __restrict__ x, int d, int n, bool vec) {
    if constexpr (sizeof(T) == 4) {
        if (vec) return __ldg(reinterpret_cast<const float4*>(x + d));
    }
    float4 v;
    v.x = d < n ? (float)x[d] : 0.f;
    v.y = d + 1 < n ? (float)x[d + 1] : 0.f;
    v.z = d + 2 < n ? (float)x[d + 2] : 0.f;
    v.w = d + 3 < n ? (float)x[d + 3] : 0.f;
    return v;
}

// the same four elements in full precision (the sums: fp32 data widened, fp64 data as is)
template <typename T>
__device__ __forceinline__ void load4d(const T* __restrict__ x, int d, int n, bool vec, double (&v)[4]) {
    if constexpr (sizeof(T) == 4) {
        const float4 f = load4<T>(x, d, n, vec);
        v[0] = f.x;
        v[1] = f.y;
        v[2] = f.z;
        v[3] = f.w;
    } else {
        if (vec) {
            const double2 a = __ldg(reinterpret_cast<const double2*>(x + d));
            const double2 b = __ldg(reinterpret_cast<const double2*>(x + d + 2));
            v[0] = a.x;
            v[1] = a.y;
            v[2] = b.x;
            v[3] = b.y;
        } else {
#pragma unroll
            for (int u = 0; u < 4; ++u) v[u] = d + u < n ? (double)x[d + u] : 0.0;
        }
    }
}

// records of the worker's k centroids into shared memory (rec: kpad x n4 floats, ccs: kpad)
__device__ void build_records(const double* __restrict__ Cm, int k, int kpad, int n, int n4, float* rec, float* ccs,
                              const uint8_t* skip = nullptr) {
    for (int e = threadIdx.x; e < kpad * n4; e += blockDim.x) {
        const int j = e / n4, d = e - j * n4;
        rec[e] = (j < k && d < n) ? (float)(-2.0 * Cm[(int64_t)j * n + d]) : 0.f;
    }
    for (int j = threadIdx.x; j < kpad; j += blockDim.x) {
        float cc = __int_as_float(0x7f800000);
        if (j < k && !(skip && skip[j])) {
            double a = 0.0;
            for (int d = 0; d < n; ++d) {
                const double c = Cm[(int64_t)j * n + d];
                a += c * c;
            }
            cc = (float)a;
        }
        ccs[j] = cc;
    }
}

__device__ float records_cmax(const float* ccs, int kpad, float* red_f) {  // max |c| (rounded up), CTA-wide
    __syncthreads();
    if (threadIdx.x == 0) {
        float cm = 0.f;
        for (int j = 0; j < kpad; ++j)
            if (ccs[j] < __int_as_float(0x7f800000)) cm = fmaxf(cm, sqrtf(ccs[j]) * 1.0001f);
        red_f[0] = cm;
    }
    __syncthreads();
    return red_f[0];
}

// screen of one row against all centroids: best index, best/second screen values, |x|^2
template <typename T>
__device__ __forceinline__ void screen_row(const T* __restrict__ x, int n, int n4, int kpad, const float* rec,
                                           const float* ccs, bool vec, int& i1, float& m1, float& m2, float& xx) {
    m1 = __int_as_float(0x7f800000);
    m2 = m1;
    i1 = 0;
    float2 nn = make_float2(0.f, 0.f);
    for (int j0 = 0; j0 < kpad; j0 += kKT) {
        float2 a[kKT];
#pragma unroll
        for (int j = 0; j < kKT; ++j) a[j] = make_float2(ccs[j0 + j], 0.f);
        for (int d = 0; d < n4; d += 4) {
            const float4 xv = load4<T>(x, d, n, vec);
            const float2 xa = make_float2(xv.x, xv.y), xb = make_float2(xv.z, xv.w);
            if (j0 == 0) {
                nn = __ffma2_rn(xa, xa, nn);
                nn = __ffma2_rn(xb, xb, nn);
            }
#pragma unroll
            for (int j = 0; j < kKT; ++j) {
                const float4 c = *reinterpret_cast<const float4*>(rec + (j0 + j) * n4 + d);
                a[j] = __ffma2_rn(xa, make_float2(c.x, c.y), a[j]);
                a[j] = __ffma2_rn(xb, make_float2(c.z, c.w), a[j]);
            }
        }
#pragma unroll
        for (int j = 0; j < kKT; ++j) {
            const float dj = a[j].x + a[j].y;
            m2 = fminf(m2, fmaxf(m1, dj));
            const bool lt = dj < m1;
            m1 = fminf(m1, dj);
            i1 = lt ? j0 + j : i1;
        }
    }
    xx = nn.x + nn.y;
}

// exact reference argmin (core.hpp:146-157: strict <, ties -> lowest j) of row x for the lanes
// in `tie`, warp-parallel over centroids; the winner lands in i1 of the owning lane
template <typename T>
__device__ void exact_ties_masked(unsigned tie, const T* __restrict__ S, int64_t row0, int n, int k,
                                  const double* __restrict__ Cm, const uint8_t* skip, int& i1) {
    const int lane = threadIdx.x & 31;
    while (tie) {
        const int src = __ffs(tie) - 1;
        tie &= tie - 1;
        const T* x = S + (row0 + src) * n;
        double dv = __longlong_as_double(0x7ff0000000000000LL);
        int dj = 0x7fffffff;
        const bool vecd = sizeof(T) == 4 ? (n & 3) == 0 : (n & 1) == 0;
        for (int j = lane; j < k; j += 32) {
            if (skip && skip[j]) continue;
            const double a = dist1<T>(x, n, Cm + (int64_t)j * n, vecd);
            if (a < dv) {
                dv = a;
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
        if (lane == src) i1 = dj;
    }
}

template <typename T>
__device__ __forceinline__ void exact_ties(unsigned tie, const T* __restrict__ S, int64_t row0, int n, int k,
                                           const double* __restrict__ Cm, int& i1) {
    exact_ties_masked<T>(tie, S, row0, n, k, Cm, nullptr, i1);
}

// ---------------------------------------------------------------- gather + init
// Sample rows into S[w][i][:] (engine.hpp:165-177 with the launch's indices): per warp 32 rows, one
// index per lane (PRP / explicit / contiguous), then the rows' V-byte chunks chunk-major across the
// warp with the row addresses shuffled -- every lane's loads issued before its stores, so a narrow
// row (config 5: 32 B) costs one vector load per lane instead of a warp per row.
template <int V>
__global__ void __launch_bounds__(256) wide_gather_kernel(const StepParams p, int w0, int64_t rowb,
                                                          unsigned char* __restrict__ S) {
    using VT = typename std::conditional<V == 16, uint4, typename std::conditional<V == 8, uint2, uint32_t>::type>::type;
    const int w = blockIdx.y, wl = w0 + w, lane = threadIdx.x & 31;
    const int64_t s = p.s;
    const int64_t i0 = ((int64_t)blockIdx.x * 8 + (threadIdx.x >> 5)) * 32;
    if (i0 >= s) return;
    SamplePRP prp;
    if (p.sample_mode == 1)
        prp = SamplePRP::make(p.key, p.round, (uint32_t)(p.worker_base + wl), (uint64_t)p.m, p.prp_a, p.prp_b,
                              p.prp_inv_b);
    const int64_t i = i0 + lane;
    int64_t g = 0;
    if (i < s) {
        if (p.sample_mode == 0)
            g = p.idx[(int64_t)wl * s + i];
        else if (p.sample_mode == 1)
            g = (int64_t)prp((uint64_t)i);
        else
            g = (int64_t)wl * s + i;
    }
    const unsigned char* src;
    if (p.nshards > 1) {
        int sh = 0;
        while (sh + 1 < p.nshards && g >= p.shard_end[sh]) ++sh;
        src = static_cast<const unsigned char*>(p.shard_ptr[sh]) + (g - (sh ? p.shard_end[sh - 1] : 0)) * rowb;
    } else {
        src = static_cast<const unsigned char*>(p.X) + g * rowb;
    }
    unsigned char* dst = S + ((int64_t)w * s + i0) * rowb;
    const int cpr = (int)(rowb / V), total = 32 * cpr;
    constexpr int U = 8;
    for (int e0 = 0; e0 < total; e0 += 32 * U) {
        VT v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int e = e0 + u * 32 + lane, r = e / cpr, q = e - r * cpr;
            const unsigned char* sp = reinterpret_cast<const unsigned char*>(
                __shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(src), r & 31));
            if (e < total && i0 + r < s) v[u] = ld_row_chunk<VT>(sp + (int64_t)q * V);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int e = e0 + u * 32 + lane, r = e / cpr;
            if (e < total && i0 + r < s) reinterpret_cast<VT*>(dst)[e] = v[u];
        }
    }
}

template <typename T>
__global__ void wide_init_kernel(const StepParams p, int w0, WideBufs b) {
    const int w = blockIdx.x, wl = w0 + w, tid = threadIdx.x;
    const int k = p.k, n = p.n;
    const int64_t kn = (int64_t)k * n, s = p.s;
    const int64_t v = p.shared_version ? *p.shared_version : 1;
    const double* ic = p.init_c + (int64_t)wl * p.init_stride;
    const uint8_t* ifl = p.init_f + (int64_t)wl * p.initf_stride;
    double* Cm = b.Cm + (int64_t)w * kn;
    uint8_t* fl = b.flags + (int64_t)w * k;
    for (int64_t e = tid; e < kn; e += kWT) Cm[e] = v != 0 ? ic[e] : 0.0;
    for (int j = tid; j < k; j += kWT) fl[j] = v != 0 ? ifl[j] : (uint8_t)1;
    __syncthreads();
    __shared__ int64_t first_row;
    if (tid == 0) {
        WState st = {};
        int32_t* pend = b.pend + (int64_t)w * k;
        for (int j = 0; j < k; ++j) {
            if (fl[j])
                pend[st.n_pending++] = j;
            else
                ++st.n_valid;
        }
        st.stop = 1;
        st.f_prev = __longlong_as_double(0x7ff0000000000000LL);
        first_row = -1;
        if (st.n_pending > 0) {
            st.nd += s * st.n_valid;  // one D^2 pass per valid centre (seeding.hpp:60-68)
            if (st.n_valid == 0) {    // seeding.hpp:72-79: uniform first centre
                first_row = p.seed_mode == 0 ? p.first_row[wl]
                                             : (int64_t)philox_index(p.key, p.round, (uint32_t)(p.worker_base + wl),
                                                                     0xF1F1u, (uint64_t)s);
                st.next = 1;
                st.filled = 1;
                st.nd += s;
            }
        }
        b.st[w] = st;
    }
    __syncthreads();
    if (first_row >= 0) {
        const int j = b.pend[(int64_t)w * k];
        const T* S = static_cast<const T*>(b.S) + ((int64_t)w * s + first_row) * n;
        for (int d = tid; d < n; d += kWT) Cm[(int64_t)j * n + d] = (double)S[d];
        if (tid == 0) fl[j] = 0;
    }
}

// D^2 from every valid centre (including a first centre just drawn): the screen's argmin over
// the valid centres (near ties exact) and the reference distance to it
constexpr int kD2Blocks = 8;  // blocks of kWT rows per CTA of the D^2 initialisation
template <typename T, int NP = 0>
__global__ void __launch_bounds__(kWT) wide_d2init_kernel(const StepParams p, WideBufs b) {
    extern __shared__ __align__(16) float wrec[];
    __shared__ float red_f[1];
    const int w = blockIdx.y, k = p.k, n = NP ? NP : p.n;
    const int64_t s = p.s;
    if (b.st[w].n_pending == 0) return;
    const int kpad = (k + kKT - 1) / kKT * kKT, n4 = (n + 3) & ~3;
    float* rec = wrec;
    float* ccs = rec + (int64_t)kpad * n4;
    const double* Cm = b.Cm + (int64_t)w * k * n;
    const uint8_t* fl = b.flags + (int64_t)w * k;
    __shared__ int s_nv, s_j;
    if (threadIdx.x == 0) {
        int nv = 0, j1 = 0;
        for (int j = 0; j < k; ++j)
            if (!fl[j]) {
                if (nv++ == 0) j1 = j;
            }
        s_nv = nv;
        s_j = j1;
    }
    __syncthreads();
    // a CTA covers kD2Blocks blocks of kWT rows: the per-CTA prologue (valid-centre scan, records) was
    // the cost of this pass when every CTA did one row per thread (200 K CTAs at config 5)
    const bool vecd = sizeof(T) == 4 ? (n & 3) == 0 : (n & 1) == 0;
    const T* S = static_cast<const T*>(b.S) + (int64_t)w * s * n;
    if (s_nv == 1) {  // one valid centre (round 0: the first centre just drawn): D^2 is its distance
        const double* c1 = Cm + (int64_t)s_j * n;
#pragma unroll 2
        for (int t = 0; t < kD2Blocks; ++t) {
            const int64_t i = ((int64_t)blockIdx.x * kD2Blocks + t) * kWT + threadIdx.x;
            if (i < s) b.d2[(int64_t)w * s + i] = dist1<T>(S + i * n, n, c1, vecd);
        }
        return;
    }
    build_records(Cm, k, kpad, n, n4, rec, ccs, fl);
    const float cmax = records_cmax(ccs, kpad, red_f);
    const float kappa = 2.0f * (float)((n + 1) / 2 + 12) * 5.9604645e-8f;
    const bool vec = sizeof(T) == 4 && (n & 3) == 0;
    for (int t = 0; t < kD2Blocks; ++t) {
        const int64_t i = ((int64_t)blockIdx.x * kD2Blocks + t) * kWT + threadIdx.x;
        if (i - (threadIdx.x & 31) >= s) break;  // warp-uniform: the whole warp is past the sample
        const bool valid = i < s;
        int lab = 0;
        float m1 = 0.f, m2 = 0.f, xx = 0.f;
        if (valid) screen_row<T>(S + i * n, n, n4, kpad, rec, ccs, vec, lab, m1, m2, xx);
        const float sc = sqrtf(xx) * 1.0001f + cmax;
        const unsigned tie = __ballot_sync(0xffffffffu, valid && !(m2 - m1 > kappa * sc * sc));
        if (tie) exact_ties_masked<T>(tie, S, i - (threadIdx.x & 31), n, k, Cm, fl, lab);
        if (valid) b.d2[(int64_t)w * s + i] = dist1<T>(S + i * n, n, Cm + (int64_t)lab * n, vecd);
    }
}

// ---------------------------------------------------------------- K-means++ slot
__device__ __forceinline__ bool slot_live(const WState& st) {
    return st.seed_stop == 0 && st.next < st.n_pending;
}

// ---- K-means++ CDF on HBM-resident samples (seeding.hpp:81-92), warp-parallel and deterministic.
// A 256-row block is one warp: lane L owns rows r0 + 8L .. r0 + 8L + 7 (summed sequentially), the
// lanes combine by an exclusive shuffle scan, and the in-block cumulative value of row i is
// fl(excl_L + run_{L,i}). The block total T_q is DEFINED as that value at the block's last row, so the
// draw, which recomputes the same values, always finds its crossing inside the block it selected.
// Block prefixes P_{q+1} = fl(P_q + T_q) run sequentially over the blocks (one warp per worker, from
// shared memory), so cum is monotone across blocks and exactly one row is the first with cum > u
// (rng.hpp:83-93; CDF rounding differs from the reference's row-sequential sum only in the last bits:
// the documented CDF-boundary tie class).
constexpr int kLaneRows = kSeedRows / 32;

struct BlockScan {  // one lane's view of a 256-row block
    double run[kLaneRows];  // sequential running sums of the lane's rows
    double excl;            // exclusive prefix of the lanes below (shuffle scan)
    int nrows;              // rows of this lane (0 past the end of the sample)
};

__device__ __forceinline__ BlockScan block_scan(const double* __restrict__ d2, int64_t r0, int64_t r1, int lane) {
    BlockScan b;
    const int64_t a = r0 + (int64_t)lane * kLaneRows;
    const int64_t left = r1 - a;
    b.nrows = left <= 0 ? 0 : (left >= kLaneRows ? kLaneRows : (int)left);
    double v[kLaneRows];
#pragma unroll
    for (int j = 0; j < kLaneRows; ++j) v[j] = j < b.nrows ? d2[a + j] : 0.0;
    double run = 0.0;
#pragma unroll
    for (int j = 0; j < kLaneRows; ++j) {
        run += v[j];
        b.run[j] = run;
    }
    double incl = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    b.excl = __shfl_up_sync(0xffffffffu, incl, 1);
    if (lane == 0) b.excl = 0.0;
    return b;
}

// block totals: one warp per (block, worker). From the second slot on, the lanes first apply the
// previous slot's D^2 update to their rows (seeding.hpp:100-103): only rows that slot's cost pass
// flagged for its winner can change, and they take min(d2, the reference distance) -- the value the
// cost pass added. (After the last slot D^2 is not read again, so no separate update pass runs.)
template <typename T, int NP = 0>
__global__ void wide_cdf_kernel(const StepParams p, WideBufs b, int nblk, int it) {
    const int w = blockIdx.y;
    const WState& st = b.st[w];
    if (!slot_live(st)) return;
    const int lane = threadIdx.x & 31;
    const int blk = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (blk >= nblk) return;
    const int64_t s = p.s, r0 = (int64_t)blk * kSeedRows, r1 = min(s, r0 + kSeedRows);
    if (it > 0 && st.it == it) {
        // the block's flagged rows, compacted across the warp (an exclusive shuffle scan of the lanes'
        // counts), then up to kCdfIL of them per lane with their exact chains interleaved: each chain is
        // still the reference's sequential distance, only the latency of several overlaps
        constexpr int kCdfIL = 4;
        __shared__ uint16_t flist[256 / 32][kSeedRows];
        const int n = NP ? NP : p.n, best = st.best;
        const double* cd = b.cand + ((int64_t)w * kMaxCandidates + best) * n;
        const int64_t a = r0 + (int64_t)lane * kLaneRows;
        uint32_t fm = 0;
#pragma unroll
        for (int j = 0; j < kLaneRows; ++j)
            if (a + j < r1 && ((b.rflag[(int64_t)w * s + a + j] >> best) & 1u)) fm |= 1u << j;
        const int cnt = __popc(fm);
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        const int total = __shfl_sync(0xffffffffu, incl, 31);
        uint16_t* fl_w = flist[threadIdx.x >> 5];
        for (int e = incl - cnt; fm; fm &= fm - 1, ++e) fl_w[e] = (uint16_t)(lane * kLaneRows + __ffs(fm) - 1);
        __syncwarp();
        for (int e0 = 0; e0 < total; e0 += 32 * kCdfIL) {
            const T* xr[kCdfIL];
            double acc[kCdfIL];
            bool on[kCdfIL];
#pragma unroll
            for (int q = 0; q < kCdfIL; ++q) {
                const int e = e0 + q * 32 + lane;
                on[q] = e < total;
                xr[q] = static_cast<const T*>(b.S) + ((int64_t)w * s + r0 + (on[q] ? fl_w[e] : 0)) * n;
                acc[q] = 0.0;
            }
            int d = 0;
            if constexpr (sizeof(T) == 4) {
                if ((n & 3) == 0)
                    for (; d < n; d += 4) {  // 16-B row loads; the four steps of each chain in order
                        const double2 c01 = __ldg(reinterpret_cast<const double2*>(cd + d));
                        const double2 c23 = __ldg(reinterpret_cast<const double2*>(cd + d + 2));
                        float4 xv[kCdfIL];
#pragma unroll
                        for (int q = 0; q < kCdfIL; ++q) xv[q] = __ldg(reinterpret_cast<const float4*>(xr[q] + d));
#pragma unroll
                        for (int q = 0; q < kCdfIL; ++q) {
                            double diff = __dsub_rn((double)xv[q].x, c01.x);
                            acc[q] = __dadd_rn(acc[q], __dmul_rn(diff, diff));
                            diff = __dsub_rn((double)xv[q].y, c01.y);
                            acc[q] = __dadd_rn(acc[q], __dmul_rn(diff, diff));
                            diff = __dsub_rn((double)xv[q].z, c23.x);
                            acc[q] = __dadd_rn(acc[q], __dmul_rn(diff, diff));
                            diff = __dsub_rn((double)xv[q].w, c23.y);
                            acc[q] = __dadd_rn(acc[q], __dmul_rn(diff, diff));
                        }
                    }
            }
            for (; d < n; ++d) {
                const double cv = __ldg(cd + d);
#pragma unroll
                for (int q = 0; q < kCdfIL; ++q) {
                    const double diff = __dsub_rn((double)__ldg(xr[q] + d), cv);
                    acc[q] = __dadd_rn(acc[q], __dmul_rn(diff, diff));
                }
            }
#pragma unroll
            for (int q = 0; q < kCdfIL; ++q)
                if (on[q]) {
                    double* d2 = b.d2 + (int64_t)w * s + r0 + fl_w[e0 + q * 32 + lane];
                    *d2 = fmin(*d2, acc[q]);
                }
        }
        __syncwarp();  // every updated D^2 of the block visible to the lanes that scan it
    }
    const BlockScan bs = block_scan(b.d2 + (int64_t)w * s, r0, r1, lane);
    // T_q := the cumulative value at the block's last row, exactly as the draw computes it
    const int last_lane = (int)((r1 - 1 - r0) / kLaneRows);
    if (lane == last_lane) {
        const int j = bs.nrows - 1;
        double t = 0.0;
#pragma unroll
        for (int q = 0; q < kLaneRows; ++q)
            if (q == j) t = bs.excl + bs.run[q];
        b.btot[(int64_t)w * (nblk + 1) + blk] = t;
    }
}

// block prefixes in place: btot[q] <- P_q (exclusive, sequential over blocks), btot[nblk] <- total.
// One warp per worker: the totals are staged in shared memory by the warp, lane 0 runs the chain.
__global__ void wide_cdfscan_kernel(WideBufs b, int nblk, int staged) {
    extern __shared__ double sbuf[];
    const int w = blockIdx.x;
    if (!slot_live(b.st[w])) return;
    double* bt = b.btot + (int64_t)w * (nblk + 1);
    double* sb = staged ? sbuf : bt;  // very long samples: the chain runs on the global copy
    if (staged)
        for (int q = threadIdx.x; q < nblk; q += blockDim.x) sb[q] = bt[q];
    __syncwarp();
    if (threadIdx.x == 0) {
        double P = 0.0;
#pragma unroll 8
        for (int q = 0; q < nblk; ++q) {
            const double t = sb[q];
            sb[q] = P;
            P += t;
        }
        sb[nblk] = P;
    }
    __syncwarp();
    if (staged)
        for (int q = threadIdx.x; q <= nblk; q += blockDim.x) bt[q] = sb[q];
}

// inverse-CDF draw of candidate c (seeding.hpp:85-92; rng.hpp:83-93): first row with cum > u; no
// crossing -> row s-1. One warp per (candidate, worker): binary search of the block prefixes, then
// the block's cumulative values recomputed exactly as wide_cdf_kernel did.
template <typename T>
__global__ void wide_draw_kernel(const StepParams p, int w0, WideBufs b, int nblk) {
    const int c = blockIdx.x, w = blockIdx.y, wl = w0 + w, lane = threadIdx.x;
    WState* stp = b.st + w;
    if (!slot_live(*stp)) return;
    const int64_t s = p.s;
    const int n = p.n;
    const double* P = b.btot + (int64_t)w * (nblk + 1);
    const double total = P[nblk];
    if (!(total > 0.0)) {  // distinct rows exhausted (seeding.hpp:87)
        if (c == 0 && lane == 0) stp->seed_stop = 1;
        return;
    }
    const int it = stp->it, next = stp->next, ncand = p.candidates;
    const double unit = p.seed_mode == 0 ? p.units[(int64_t)wl * p.units_stride + (int64_t)it * ncand + c]
                                         : philox_unit(p.key, p.round, (uint32_t)(p.worker_base + wl),
                                                       (uint32_t)(0x10000 + next * kMaxCandidates + c));
    const double u = unit * total;
    // first block q with P_{q+1} > u (P is non-decreasing); none -> the fallback row
    int lo = 0, hi = nblk;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (P[mid + 1] > u)
            hi = mid;
        else
            lo = mid + 1;
    }
    int64_t row = s - 1;
    if (lo < nblk) {
        const int64_t r0 = (int64_t)lo * kSeedRows, r1 = min(s, r0 + kSeedRows);
        const BlockScan bs = block_scan(b.d2 + (int64_t)w * s, r0, r1, lane);
        const double Pq = P[lo];
        int hit = kLaneRows;
#pragma unroll
        for (int j = kLaneRows - 1; j >= 0; --j)
            if (j < bs.nrows && Pq + (bs.excl + bs.run[j]) > u) hit = j;
        const unsigned m = __ballot_sync(0xffffffffu, hit < kLaneRows);
        if (m) {
            const int src = __ffs(m) - 1;
            const int h = __shfl_sync(0xffffffffu, hit, src);
            row = r0 + (int64_t)src * kLaneRows + h;
        }
    }
    const T* x = static_cast<const T*>(b.S) + ((int64_t)w * s + row) * n;
    double* cd = b.cand + ((int64_t)w * kMaxCandidates + c) * n;
    for (int d = lane; d < n; d += 32) cd[d] = (double)x[d];
}

// candidate costs sum_i min(d2_i, dist(S_i, cand_c)) (seeding.hpp:93): an fp32 screen decides the
// rows a candidate provably cannot improve (value d2_i, exact); the others get the reference
// distance. Per row one flag byte (bit c: candidate c may improve the row) is the work list of the
// winner's D^2 update, which recomputes only those rows -- no per-candidate value array. Each CTA
// covers kCostBPC consecutive 256-row blocks; a thread sums its rows in order, then a warp tree and
// the warps in order give one partial per (CTA, candidate): costs are exact sums in a fixed order.
constexpr int kCostBPC = 8;  // 256-row blocks per CTA of the candidate-cost pass

template <typename T, bool IV>  // exact either way (hi = lo); !IV: only the workers the interval decision left open
__global__ void __launch_bounds__(kWT) wide_cost_kernel(const StepParams p, WideBufs b, int nblk) {
    __shared__ double wred[kMaxCandidates][kWT / 32];
    extern __shared__ __align__(16) float crec_raw[];  // [ncand][n4] -2 * candidate (fp32)
    __shared__ float ccn[kMaxCandidates];
    const int w = blockIdx.y, n = p.n, ncand = p.candidates;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (!slot_live(b.st[w]) || (!IV && !b.st[w].ambig)) return;
    const int n4 = (n + 3) & ~3;
    auto crec = [&](int c) { return crec_raw + (int64_t)c * n4; };
    const double* cand = b.cand + (int64_t)w * kMaxCandidates * n;
    for (int e = threadIdx.x; e < ncand * n4; e += kWT) {
        const int c = e / n4, d = e - c * n4;
        crec(c)[d] = d < n ? (float)(-2.0 * cand[(int64_t)c * n + d]) : 0.f;
    }
    if (threadIdx.x < ncand) {
        double a = 0.0;
        for (int d = 0; d < n; ++d) a += cand[(int64_t)threadIdx.x * n + d] * cand[(int64_t)threadIdx.x * n + d];
        ccn[threadIdx.x] = (float)a;
    }
    __syncthreads();
    const float kappa = 2.0f * (float)((n + 1) / 2 + 12) * 5.9604645e-8f;
    const bool vec = sizeof(T) == 4 && (n & 3) == 0;
    const bool vecd = sizeof(T) == 4 ? (n & 3) == 0 : (n & 1) == 0;
    const int64_t s = p.s;
    const int blk0 = blockIdx.x * kCostBPC, blk1 = min(nblk, blk0 + kCostBPC);
    const T* Sw = static_cast<const T*>(b.S) + (int64_t)w * s * n;
    const double* d2w = b.d2 + (int64_t)w * s;
    uint8_t* flw = b.rflag + (int64_t)w * s;
    double acc[kMaxCandidates];
#pragma unroll
    for (int c = 0; c < kMaxCandidates; ++c) acc[c] = 0.0;
    for (int blk = blk0; blk < blk1; ++blk) {
        const int64_t i = (int64_t)blk * kSeedRows + threadIdx.x;
        if (i >= s) break;
        const T* x = Sw + i * n;
        const double d2i = d2w[i];
        // screen: s~_c = |c|^2 + x.(-2c); dist~_c = |x|^2 + s~_c
        float2 a[kMaxCandidates], nn = make_float2(0.f, 0.f);
#pragma unroll
        for (int c = 0; c < kMaxCandidates; ++c) a[c] = make_float2(c < ncand ? ccn[c] : 0.f, 0.f);
        for (int d = 0; d < n4; d += 4) {
            const float4 xv = load4<T>(x, d, n, vec);
            const float2 xa = make_float2(xv.x, xv.y), xb = make_float2(xv.z, xv.w);
            nn = __ffma2_rn(xa, xa, nn);
            nn = __ffma2_rn(xb, xb, nn);
#pragma unroll
            for (int c = 0; c < kMaxCandidates; ++c)
                if (c < ncand) {
                    const float4 cv = *reinterpret_cast<const float4*>(crec(c) + d);
                    a[c] = __ffma2_rn(xa, make_float2(cv.x, cv.y), a[c]);
                    a[c] = __ffma2_rn(xb, make_float2(cv.z, cv.w), a[c]);
                }
        }
        const float xx = nn.x + nn.y, xn = sqrtf(xx) * 1.0001f;
        const float f2 = __double2float_ru(d2i);
        uint32_t fl = 0;
#pragma unroll
        for (int c = 0; c < kMaxCandidates; ++c) {
            if (c >= ncand) break;
            double v = d2i;
            const float sc = xn + sqrtf(ccn[c]) * 1.0001f;
            const float dt = xx + (a[c].x + a[c].y);
            if (!(dt - kappa * sc * sc > f2)) {  // may improve: the reference distance
                v = fmin(d2i, dist1<T>(x, n, cand + (int64_t)c * n, vecd));
                fl |= 1u << c;
            }
            acc[c] += v;
        }
        flw[i] = (uint8_t)fl;
    }
#pragma unroll
    for (int c = 0; c < kMaxCandidates; ++c) {
        if (c >= ncand) break;
        const double v = warp_sum(acc[c]);  // warp trees, then the warps in order (fixed order)
        if (lane == 0) wred[c][warp] = v;
    }
    __syncthreads();
    if (threadIdx.x < ncand) {
        double tot = 0.0;
        for (int q = 0; q < kWT / 32; ++q) tot += wred[threadIdx.x][q];
        b.bcost[((int64_t)w * kMaxCandidates + threadIdx.x) * nblk + blockIdx.x] = tot;
        b.bcost_hi[((int64_t)w * kMaxCandidates + threadIdx.x) * nblk + blockIdx.x] = tot;
    }
}

// The same pass for a compile-time row width NP (n = 8 / 16 / 32: config 5 and the like): rows in
// registers, candidates' fp32 records and fp64 coordinates in shared memory (broadcast loads), the
// screen bounds' |c| terms hoisted; identical arithmetic and summation order to wide_cost_kernel, so
// the partials are bit-identical to it.
template <typename T, int NP, bool IV>  // exact (hi = lo: the first decision is final); IV false: gated re-run
__global__ void __launch_bounds__(kWT) wide_cost_np_kernel(const StepParams p, WideBufs b, int nblk) {
    __shared__ double wred[kMaxCandidates][kWT / 32];
    __shared__ __align__(16) float crec[kMaxCandidates][NP];
    __shared__ __align__(16) double cdv[kMaxCandidates][NP];
    __shared__ float ccn[kMaxCandidates], ccr[kMaxCandidates];
    const int w = blockIdx.y, ncand = p.candidates;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (!slot_live(b.st[w]) || (!IV && !b.st[w].ambig)) return;
    const double* cand = b.cand + (int64_t)w * kMaxCandidates * NP;
    for (int e = threadIdx.x; e < kMaxCandidates * NP; e += kWT) {
        const int c = e / NP, d = e - c * NP;
        const double v = c < ncand ? cand[(int64_t)c * NP + d] : 0.0;
        cdv[c][d] = v;
        crec[c][d] = (float)(-2.0 * v);
    }
    if (threadIdx.x < kMaxCandidates) {
        const int c = threadIdx.x;
        double a = 0.0;
        if (c < ncand)
            for (int d = 0; d < NP; ++d) a += cand[(int64_t)c * NP + d] * cand[(int64_t)c * NP + d];
        ccn[c] = (float)a;
        ccr[c] = sqrtf((float)a) * 1.0001f;
    }
    __syncthreads();
    constexpr float kappa = 2.0f * (float)((NP + 1) / 2 + 12) * 5.9604645e-8f;
    const int64_t s = p.s;
    const int blk0 = blockIdx.x * kCostBPC, blk1 = min(nblk, blk0 + kCostBPC);
    const T* Sw = static_cast<const T*>(b.S) + (int64_t)w * s * NP;
    const double* d2w = b.d2 + (int64_t)w * s;
    uint8_t* flw = b.rflag + (int64_t)w * s;
    double acc[kMaxCandidates];
#pragma unroll
    for (int c = 0; c < kMaxCandidates; ++c) acc[c] = 0.0;
    for (int blk = blk0; blk < blk1; ++blk) {
        const int64_t i = (int64_t)blk * kSeedRows + threadIdx.x;
        if (i >= s) break;
        T x[NP];
        if constexpr (sizeof(T) == 4) {
#pragma unroll
            for (int q = 0; q < NP / 4; ++q) {
                const float4 v = __ldg(reinterpret_cast<const float4*>(Sw + i * NP) + q);
                x[4 * q] = v.x;
                x[4 * q + 1] = v.y;
                x[4 * q + 2] = v.z;
                x[4 * q + 3] = v.w;
            }
        } else {
#pragma unroll
            for (int q = 0; q < NP / 2; ++q) {
                const double2 v = __ldg(reinterpret_cast<const double2*>(Sw + i * NP) + q);
                x[2 * q] = v.x;
                x[2 * q + 1] = v.y;
            }
        }
        const double d2i = d2w[i];
        float2 a[kMaxCandidates], nn = make_float2(0.f, 0.f);
#pragma unroll
        for (int c = 0; c < kMaxCandidates; ++c) a[c] = make_float2(ccn[c], 0.f);
#pragma unroll
        for (int d = 0; d < NP; d += 4) {
            const float2 xa = make_float2((float)x[d], (float)x[d + 1]), xb = make_float2((float)x[d + 2], (float)x[d + 3]);
            nn = __ffma2_rn(xa, xa, nn);
            nn = __ffma2_rn(xb, xb, nn);
#pragma unroll
            for (int c = 0; c < kMaxCandidates; ++c)
                if (c < ncand) {
                    const float4 cv = *reinterpret_cast<const float4*>(&crec[c][d]);
                    a[c] = __ffma2_rn(xa, make_float2(cv.x, cv.y), a[c]);
                    a[c] = __ffma2_rn(xb, make_float2(cv.z, cv.w), a[c]);
                }
        }
        const float xx = nn.x + nn.y, xn = sqrtf(xx) * 1.0001f;
        const float f2 = __double2float_ru(d2i);
        uint32_t fl = 0;
#pragma unroll
        for (int c = 0; c < kMaxCandidates; ++c) {
            if (c >= ncand) break;
            double v = d2i;
            const float sc = xn + ccr[c];
            const float dt = xx + (a[c].x + a[c].y);
            const float B = kappa * sc * sc;
            if (!(dt - B > f2)) {  // may improve: the reference distance (narrow rows: about what interval
                                   // bookkeeping would cost, so this pass is exact and the decision final)
                fl |= 1u << c;
                double e = 0.0;
#pragma unroll
                for (int d = 0; d < NP; ++d) {
                    const double diff = __dsub_rn((double)x[d], cdv[c][d]);
                    e = __dadd_rn(e, __dmul_rn(diff, diff));
                }
                v = fmin(d2i, e);
            }
            acc[c] += v;
        }
        if (IV) flw[i] = (uint8_t)fl;
    }
#pragma unroll
    for (int c = 0; c < kMaxCandidates; ++c) {
        if (c >= ncand) break;
        const double v = warp_sum(acc[c]);  // warp trees, then the warps in order (fixed order)
        if (lane == 0) wred[c][warp] = v;
    }
    __syncthreads();
    if (threadIdx.x < ncand) {
        double tot = 0.0;
        for (int q = 0; q < kWT / 32; ++q) tot += wred[threadIdx.x][q];
        b.bcost[((int64_t)w * kMaxCandidates + threadIdx.x) * nblk + blockIdx.x] = tot;
        b.bcost_hi[((int64_t)w * kMaxCandidates + threadIdx.x) * nblk + blockIdx.x] = tot;
    }
}

// The same pass for wide fp32 rows (n = 64 / 128: config 4), warp-cooperative so the row loads are
// coalesced: a warp takes 8 rows at a time, lane L holding dims 4L.. of each (n = 128; n = 64: lanes
// 0-15 of two row halves... simply the dims 4L < n). Each lane forms its partial |x|^2 and x.(-2c)
// for the 8 rows, a transposing butterfly (31 shuffles) leaves lane L = 4r + q with the total of row
// r's quantity q (q = 0: |x|^2, q = 1..3: candidate q-1), which tests its (row, candidate) pair
// exactly like wide_cost_kernel and, when the candidate may improve, evaluates the reference
// distance (ascending d, non-fused, one lane per pair). Sums: per candidate over rows in a fixed
// order (the lanes' running sums, then a fixed tree and the warps in order).
template <int NP, bool IV>  // IV: interval pass; else the exact pass for the workers it left undecided
__global__ void __launch_bounds__(kWT) wide_cost_rows_kernel(const StepParams p, WideBufs b, int nblk) {
    static_assert(NP % 4 == 0 && NP <= 128, "row width");
    __shared__ double wred[kMaxCandidates][kWT / 32];
    __shared__ double wred_hi[kMaxCandidates][kWT / 32];
    __shared__ __align__(16) float crec[3][NP];
    __shared__ float ccn[3], ccr[3];
    const int w = blockIdx.y, ncand = p.candidates;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (!slot_live(b.st[w]) || (!IV && !b.st[w].ambig)) return;
    const double* cand = b.cand + (int64_t)w * kMaxCandidates * NP;
    for (int e = threadIdx.x; e < 3 * NP; e += kWT) {
        const int c = e / NP, d = e - c * NP;
        crec[c][d] = c < ncand ? (float)(-2.0 * cand[(int64_t)c * NP + d]) : 0.f;
    }
    if (threadIdx.x < 3) {
        const int c = threadIdx.x;
        double a = 0.0;
        if (c < ncand)
            for (int d = 0; d < NP; ++d) a += cand[(int64_t)c * NP + d] * cand[(int64_t)c * NP + d];
        ccn[c] = (float)a;
        ccr[c] = sqrtf((float)a) * 1.0001f;
    }
    __syncthreads();
    constexpr float kappa = 2.0f * (float)((NP + 1) / 2 + 12) * 5.9604645e-8f;
    const int64_t s = p.s;
    const int64_t row_lo = (int64_t)blockIdx.x * kCostBPC * kSeedRows;
    const int64_t row_hi = min(s, row_lo + (int64_t)kCostBPC * kSeedRows);
    const float* Sw = static_cast<const float*>(b.S) + (int64_t)w * s * NP;
    const double* d2w = b.d2 + (int64_t)w * s;
    uint8_t* flw = b.rflag + (int64_t)w * s;
    const int d0 = 4 * lane;              // this lane's dims in the screen
    const bool has = d0 < NP;
    const int r = lane >> 2, q = lane & 3;  // the (row, quantity) this lane ends up owning
    const int c = q - 1;
    float4 cv[3];
#pragma unroll
    for (int cc = 0; cc < 3; ++cc) cv[cc] = has ? *reinterpret_cast<const float4*>(&crec[cc][d0]) : make_float4(0, 0, 0, 0);
    double acc = 0.0, acch = 0.0;  // lane's running cost interval of candidate c (q >= 1)
    const int64_t gstep = (int64_t)(kWT / 32) * 8;
    float4 xn8[8];  // the next group's rows, loaded while the current group is screened
    auto load_group = [&](int64_t g0) {
#pragma unroll
        for (int rr = 0; rr < 8; ++rr) {
            const int64_t i = g0 + rr;
            xn8[rr] = (has && i < row_hi) ? __ldg(reinterpret_cast<const float4*>(Sw + i * NP + d0))
                                          : make_float4(0, 0, 0, 0);
        }
    };
    load_group(row_lo + (int64_t)warp * 8);
    for (int64_t i0 = row_lo + (int64_t)warp * 8; i0 < row_hi; i0 += gstep) {
        float4 xc[8];
#pragma unroll
        for (int rr = 0; rr < 8; ++rr) xc[rr] = xn8[rr];
        if (i0 + gstep < row_hi) load_group(i0 + gstep);
        float v[32];
#pragma unroll
        for (int rr = 0; rr < 8; ++rr) {
            const float4 x = xc[rr];
            const float2 xa = make_float2(x.x, x.y), xb = make_float2(x.z, x.w);
            float2 nn = __ffma2_rn(xa, xa, make_float2(0.f, 0.f));
            nn = __ffma2_rn(xb, xb, nn);
            v[rr * 4] = nn.x + nn.y;
#pragma unroll
            for (int cc = 0; cc < 3; ++cc) {
                float2 a = __ffma2_rn(xa, make_float2(cv[cc].x, cv[cc].y), make_float2(0.f, 0.f));
                a = __ffma2_rn(xb, make_float2(cv[cc].z, cv[cc].w), a);
                v[rr * 4 + 1 + cc] = a.x + a.y;
            }
        }
        // transposing butterfly: after the stage with offset o, the lane keeps the half of its values
        // selected by its bit o; finally lane L holds the warp total of value L
#pragma unroll
        for (int o = 16, m = 32; o > 0; o >>= 1, m >>= 1) {
            const bool up = (lane & o) != 0;
#pragma unroll
            for (int t = 0; t < m / 2; ++t) {
                const float send = up ? v[t] : v[t + m / 2];
                const float keep = up ? v[t + m / 2] : v[t];
                v[t] = keep + __shfl_xor_sync(0xffffffffu, send, o);
            }
        }
        const float tot = v[0];  // row r's quantity q
        const float xx = __shfl_sync(0xffffffffu, tot, lane & ~3);
        const int64_t i = i0 + r;
        const bool valid = i < row_hi;
        const double d2i = valid ? d2w[i] : 0.0;
        bool may = false;
        if (q >= 1 && c < ncand && valid) {
            const float xn = sqrtf(xx) * 1.0001f, f2 = __double2float_ru(d2i);
            const float sc = xn + ccr[c];
            const float dt = xx + (ccn[c] + tot);
            const float B = kappa * sc * sc;
            may = !(dt - B > f2);
            double vv = d2i, vh = d2i;
            if (IV && may) {  // the true min(d2, dist) lies in [min(d2, dt - B), min(d2, dt + B)]
                vv = fmin(d2i, (double)fmaxf(dt - B, 0.f));
                vh = fmin(d2i, (double)(dt + B));
            } else if (may) {  // the reference distance (core.hpp:100-108), this lane alone
                const float* xr = Sw + i * NP;
                const double* cd = cand + (int64_t)c * NP;
                double e = 0.0;
#pragma unroll 8
                for (int d = 0; d < NP; d += 4) {
                    const float4 x4 = __ldg(reinterpret_cast<const float4*>(xr + d));
                    const double2 c01 = __ldg(reinterpret_cast<const double2*>(cd + d));
                    const double2 c23 = __ldg(reinterpret_cast<const double2*>(cd + d + 2));
                    double df = __dsub_rn((double)x4.x, c01.x);
                    e = __dadd_rn(e, __dmul_rn(df, df));
                    df = __dsub_rn((double)x4.y, c01.y);
                    e = __dadd_rn(e, __dmul_rn(df, df));
                    df = __dsub_rn((double)x4.z, c23.x);
                    e = __dadd_rn(e, __dmul_rn(df, df));
                    df = __dsub_rn((double)x4.w, c23.y);
                    e = __dadd_rn(e, __dmul_rn(df, df));
                }
                vv = vh = fmin(d2i, e);
            }
            acc += vv;
            acch += vh;
        }
        // the row's flag byte: bit c from lane 4r + 1 + c
        const unsigned bal = __ballot_sync(0xffffffffu, may);
        if (IV && q == 0 && valid) flw[i] = (uint8_t)((bal >> (lane + 1)) & 7u);
    }
    // candidate c: lanes 4r + 1 + c (r = 0..7), a fixed tree, then the warps in order
    double t = acc, th = acch;
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
        t += __shfl_xor_sync(0xffffffffu, t, o);
        th += __shfl_xor_sync(0xffffffffu, th, o);
    }
    if (lane >= 1 && lane <= 3) {
        wred[lane - 1][warp] = t;
        wred_hi[lane - 1][warp] = th;
    }
    __syncthreads();
    if (threadIdx.x < ncand) {
        double tot2 = 0.0, toth2 = 0.0;
        for (int q2 = 0; q2 < kWT / 32; ++q2) {
            tot2 += wred[threadIdx.x][q2];
            toth2 += wred_hi[threadIdx.x][q2];
        }
        b.bcost[((int64_t)w * kMaxCandidates + threadIdx.x) * nblk + blockIdx.x] = tot2;
        b.bcost_hi[((int64_t)w * kMaxCandidates + threadIdx.x) * nblk + blockIdx.x] = toth2;
    }
}

// winner of the slot (strict <, first candidate wins ties: seeding.hpp:94-98) into its slot. Warp c
// sums candidate c's block partials (lanes strided, then a shuffle tree: a fixed order).
// EXACT = false: after the interval pass. The cost of candidate c lies in [lo_c, hi_c] (sums of the
// per-row interval ends, a 1e-9 relative slack for the summation order); if one candidate's hi is
// below every other's lo it is the strict winner of the exact costs and the slot is decided, else
// the worker is marked for the exact pass. EXACT = true: after the exact pass, for marked workers.
template <bool EXACT>
__global__ void wide_decide_kernel(const StepParams p, WideBufs b, int nblk) {
    const int w = blockIdx.x, n = p.n, k = p.k, ncand = p.candidates;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    WState* stp = b.st + w;
    if (!slot_live(*stp) || (EXACT && !stp->ambig)) return;
    __shared__ double tot_s[kMaxCandidates], toth_s[kMaxCandidates];
    __shared__ int best_s;
    if (warp < ncand) {  // one partial per cost CTA
        const double* bc_c = b.bcost + ((int64_t)w * kMaxCandidates + warp) * nblk;
        const double* bh_c = b.bcost_hi + ((int64_t)w * kMaxCandidates + warp) * nblk;
        const int ncta = (nblk + kCostBPC - 1) / kCostBPC;
        double t = 0.0, th = 0.0;
        for (int q = lane; q < ncta; q += 32) {
            t += bc_c[q];
            th += bh_c[q];
        }
        t = warp_sum(t);
        th = warp_sum(th);
        if (lane == 0) {
            tot_s[warp] = t;
            toth_s[warp] = th;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double bc = __longlong_as_double(0x7ff0000000000000LL);
        int best = 0;
        bool exact = true;
        for (int c = 0; c < ncand; ++c) exact &= tot_s[c] == toth_s[c];
        if (EXACT || exact) {  // strict <, the first candidate wins ties (seeding.hpp:94-98)
            for (int c = 0; c < ncand; ++c)
                if (tot_s[c] < bc) {
                    bc = tot_s[c];
                    best = c;
                }
        } else {
            for (int c = 0; c < ncand; ++c)
                if (toth_s[c] < bc) {
                    bc = toth_s[c];
                    best = c;
                }
            const double hb = toth_s[best] * (1.0 + 1e-9);
            for (int c = 0; c < ncand; ++c)
                if (c != best && !(hb < tot_s[c] * (1.0 - 1e-9))) best = -1;
        }
        best_s = best;
        stp->ambig = best < 0 ? 1 : 0;
    }
    __syncthreads();
    const int best = best_s;
    if (best < 0) return;  // the exact pass decides
    const int j = b.pend[(int64_t)w * k + stp->next];
    const double* cd = b.cand + ((int64_t)w * kMaxCandidates + best) * n;
    for (int d = threadIdx.x; d < n; d += blockDim.x) b.Cm[((int64_t)w * k + j) * n + d] = cd[d];
    __syncthreads();
    if (threadIdx.x == 0) {
        b.flags[(int64_t)w * k + j] = 0;
        stp->best = best;
        stp->nd += (int64_t)ncand * p.s;
        stp->filled += 1;
        stp->next += 1;
        stp->it += 1;
    }
}

// ---------------------------------------------------------------- Lloyd
__global__ void wide_lloyd_begin_kernel(const StepParams p, WideBufs b) {
    const int w = blockIdx.x, k = p.k;
    if (threadIdx.x != 0) return;
    WState& st = b.st[w];
    bool degenerate = false;
    for (int j = 0; j < k; ++j) degenerate |= b.flags[(int64_t)w * k + j] != 0;
    st.run_lloyd = p.do_lloyd && !degenerate;
    if (p.do_lloyd && degenerate) st.err = kErrDegenerateInit;
    st.done = st.run_lloyd ? 0 : 1;
}

// one pass for CTA g of worker w: rows chunk_range(s, G, g) in rounds of kWT; labels by exact
// strict-< argmin (core.hpp:146-157); per-cluster sums of each round's rows (label-sorted, row
// order) and its cost tree-sum are added to the CTA accumulators in round order
#ifndef WIDE_ASSIGN_MINB
#define WIDE_ASSIGN_MINB 3  // CTAs per SM the register cap is set for (80 registers at 256 threads)
#endif
template <typename T, int AT, int NP = 0, int AR = 1>  // NP: the row width at compile time (0: p.n); AR rows per thread per round
__global__ void __launch_bounds__(AT, WIDE_ASSIGN_MINB) wide_assign_kernel(const StepParams p, WideBufs b, int G, int tc_codes) {
    constexpr int AW = AT / 32;  // warps
    extern __shared__ double wsm[];
    const int w = blockIdx.y, g = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (b.st[w].done) return;
    const int k = p.k, n = NP ? NP : p.n;
    const int64_t s = p.s, kn = (int64_t)k * n;
    const int kpad = (k + kKT - 1) / kKT * kKT, n4 = (n + 3) & ~3;
    double* acc = wsm;                  // [k*n] sums
    double* cnt = acc + kn;             // [k] counts
    double* red = cnt + k;              // [AT] tree
    float* rec = reinterpret_cast<float*>(red + AT + ((kn + k + AT) & 1));  // [kpad][n4], 16-B aligned
    float* ccs = rec + (int64_t)kpad * n4;             // [kpad]
    int* wcnt = reinterpret_cast<int*>(ccs + kpad);    // [AR][AW][k] per-(slot, warp) label counts
    int* cstart = wcnt + AR * AW * k;   // [k+1]
    int* sorted = cstart + k + 1;       // [AT * AR] label-sorted round rows
    __shared__ float cmax_s;
    for (int64_t e = tid; e < kn + k; e += AT) acc[e] = 0.0;
    double cost = 0.0;
    int64_t r0, r1;
    chunk_range(s, G, g, r0, r1);
    const T* S = static_cast<const T*>(b.S) + (int64_t)w * s * n;
    const double* Cm = b.Cm + (int64_t)w * kn;
    int32_t* labels = b.labels + (int64_t)w * s;
    build_records(Cm, k, kpad, n, n4, rec, ccs);
    __syncthreads();
    if (tid == 0) {
        float cm = 0.f;
        for (int j = 0; j < k; ++j) cm = fmaxf(cm, sqrtf(ccs[j]) * 1.0001f);
        cmax_s = cm;
    }
    __syncthreads();
    const float cmax = cmax_s;
    const float kappa = 2.0f * (float)((n + 1) / 2 + 12) * 5.9604645e-8f;
    const bool vec = sizeof(T) == 4 && (n & 3) == 0;                           // float4 screen loads
    const bool vecd = sizeof(T) == 4 ? (n & 3) == 0 : (n & 1) == 0;           // 16-B sum loads
    for (int64_t base = r0; base < r1; base += (int64_t)AT * AR) {
        // R rows per thread per round (rows base + tid + AT r): the round's sort and fold barriers
        // are shared by AT * AR rows; thread t still visits rows r0 + t + AT i in order
        int labr[AR];
        bool validr[AR];
#pragma unroll
        for (int r = 0; r < AR; ++r) {
            const int64_t i = base + tid + (int64_t)AT * r;
            const bool valid = i < r1;
            validr[r] = valid;
            int lab = 0;
            float m1 = 0.f, m2 = 0.f, xx = 0.f;
            unsigned tie;
            if (tc_codes) {  // the tensor-core screen's code: label, bit 31 = still a near tie
                const int32_t code = valid ? labels[i] : 0;
                lab = code & 0x7fffffff;
                tie = __ballot_sync(0xffffffffu, valid && code < 0);
            } else {
                if (valid) screen_row<T>(S + i * n, n, n4, kpad, rec, ccs, vec, lab, m1, m2, xx);
                const float sc = sqrtf(xx) * 1.0001f + cmax;
                tie = __ballot_sync(0xffffffffu, valid && !(m2 - m1 > kappa * sc * sc));
            }
            if (tie) exact_ties<T>(tie, S, base + (int64_t)AT * r + warp * 32, n, k, Cm, lab);
            if (valid) labels[i] = lab;
            labr[r] = lab;
        }
        // stable counting sort of the round's rows by label: (row slot r, warp) major, lane minor
        for (int e = tid; e < AR * AW * k; e += AT) wcnt[e] = 0;
        __syncthreads();
        unsigned peersr[AR];
#pragma unroll
        for (int r = 0; r < AR; ++r) {
            peersr[r] = __match_any_sync(0xffffffffu, validr[r] ? labr[r] : -1);
            if (validr[r] && (peersr[r] & ((1u << lane) - 1u)) == 0)
                wcnt[(r * AW + warp) * k + labr[r]] = __popc(peersr[r]);
        }
        __syncthreads();
        if (warp == 0) {  // cluster-major, (slot, warp)-minor offsets: a shuffle scan over 32 clusters at a time
            int base2 = 0;
            for (int j0 = 0; j0 < k; j0 += 32) {
                const int j = j0 + lane;
                int col = 0;
                if (j < k)
                    for (int q = 0; q < AR * AW; ++q) col += wcnt[q * k + j];
                int incl = col;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += y;
                }
                if (j < k) {
                    int run = base2 + incl - col;
                    cstart[j] = run;
                    for (int q = 0; q < AR * AW; ++q) {
                        const int c = wcnt[q * k + j];
                        wcnt[q * k + j] = run;
                        run += c;
                    }
                }
                base2 += __shfl_sync(0xffffffffu, incl, 31);
            }
            if (lane == 0) cstart[k] = base2;
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < AR; ++r) {
            if (validr[r])
                sorted[wcnt[(r * AW + warp) * k + labr[r]] + __popc(peersr[r] & ((1u << lane) - 1u))] = tid + AT * r;
        }
        __syncthreads();              // sorted[] complete before the sums read it
        // per-cluster sums of this round: warp w takes clusters w, w+8, ..., walks the cluster's
        // rows in order with lanes over dims (coalesced row loads), then adds to the CTA
        // accumulator (each (j, d) owned by one lane: fixed order, no atomics)
        // n <= 128: LR lanes cover a row's dims (4 per lane), 32/LR rows in flight per step, each
        // lane summing rows gi, gi + RPS, ... in order, then a fixed shuffle tree over gi
        const int LR = n <= 4 ? 1 : n <= 8 ? 2 : n <= 16 ? 4 : n <= 32 ? 8 : n <= 64 ? 16 : 32;
        const int RPS = 32 / LR, gi = lane / LR, dq = (lane % LR) * 4;
        for (int j = warp; j < k && n <= 128; j += AW) {
            const int q0 = cstart[j], q1 = cstart[j + 1];
            if (q0 == q1) continue;
            double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
            if (dq < n) {
                // the rows' objective terms ride along: this lane's four coordinates of centre j stay in
                // registers and its squared differences go to its own running cost (fixed order: cluster,
                // then row; reduced over the CTA at the end) -- no second walk over the rows
                const double* cp = Cm + (int64_t)j * n + dq;
                const double c0 = cp[0], c1 = dq + 1 < n ? cp[1] : 0.0, c2 = dq + 2 < n ? cp[2] : 0.0,
                             c3 = dq + 3 < n ? cp[3] : 0.0;
                double ca = 0.0, cb = 0.0;
#pragma unroll 4
                for (int q = q0 + gi; q < q1; q += RPS) {
                    double v[4];
                    load4d<T>(S + (base + sorted[q]) * n, dq, n, vecd, v);
                    a0 += v[0];
                    a1 += v[1];
                    a2 += v[2];
                    a3 += v[3];
                    const double e0 = v[0] - c0, e1 = v[1] - c1, e2 = v[2] - c2, e3 = v[3] - c3;
                    ca = fma(e0, e0, ca);
                    cb = fma(e1, e1, cb);
                    ca = fma(e2, e2, ca);
                    cb = fma(e3, e3, cb);
                }
                cost += ca + cb;
            }
            for (int o = LR; o < 32; o <<= 1) {
                a0 += __shfl_xor_sync(0xffffffffu, a0, o);
                a1 += __shfl_xor_sync(0xffffffffu, a1, o);
                a2 += __shfl_xor_sync(0xffffffffu, a2, o);
                a3 += __shfl_xor_sync(0xffffffffu, a3, o);
            }
            if (gi == 0 && dq < n) {
                double* aj = acc + (int64_t)j * n + dq;
                aj[0] += a0;
                if (dq + 1 < n) aj[1] += a1;
                if (dq + 2 < n) aj[2] += a2;
                if (dq + 3 < n) aj[3] += a3;
            }
        }
        for (int j = warp; j < k && n > 128; j += AW) {
            const int q0 = cstart[j], q1 = cstart[j + 1];
            if (q0 == q1) continue;
            for (int d0 = lane * 4; d0 < n; d0 += 128) {
                double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
                const double* cp = Cm + (int64_t)j * n + d0;
                const double c0 = cp[0], c1 = d0 + 1 < n ? cp[1] : 0.0, c2 = d0 + 2 < n ? cp[2] : 0.0,
                             c3 = d0 + 3 < n ? cp[3] : 0.0;
                double ca = 0.0, cb = 0.0;
#pragma unroll 4
                for (int q = q0; q < q1; ++q) {
                    double v[4];
                    load4d<T>(S + (base + sorted[q]) * n, d0, n, vecd, v);
                    a0 += v[0];
                    a1 += v[1];
                    a2 += v[2];
                    a3 += v[3];
                    const double e0 = v[0] - c0, e1 = v[1] - c1, e2 = v[2] - c2, e3 = v[3] - c3;
                    ca = fma(e0, e0, ca);
                    cb = fma(e1, e1, cb);
                    ca = fma(e2, e2, ca);
                    cb = fma(e3, e3, cb);
                }
                cost += ca + cb;
                double* aj = acc + (int64_t)j * n + d0;
                aj[0] += a0;
                if (d0 + 1 < n) aj[1] += a1;
                if (d0 + 2 < n) aj[2] += a2;
                if (d0 + 3 < n) aj[3] += a3;
            }
        }
        for (int j = tid; j < k; j += AT) cnt[j] += (double)(cstart[j + 1] - cstart[j]);
        __syncthreads();
    }
    const int64_t pd = kn + k + 1;
    double* out = b.part + ((int64_t)w * G + g) * pd;
    for (int64_t e = tid; e < kn + k; e += AT) out[e] = acc[e];
    cost = cta_sum_t<AT>(cost, red);  // fixed tree over the threads' running sums
    if (tid == 0) out[kn + k] = cost;
}

// partials in CTA order -> objective, monotone check, history, means, stop rules
// (lloyd.hpp:100-164 with means_from_sums lloyd.hpp:75-89)
__global__ void wide_lloyd_reduce_kernel(const StepParams p, WideBufs b, int G, int w0) {
    const int w = blockIdx.x, wl = w0 + w, tid = threadIdx.x;
    WState* stp = b.st + w;
    if (stp->done) return;
    const int k = p.k, n = p.n;
    const int64_t kn = (int64_t)k * n, pd = kn + k + 1, s = p.s;
    const double* part = b.part + (int64_t)w * G * pd;
    double* Cm = b.Cm + (int64_t)w * kn;
    __shared__ double f_s;
    __shared__ int flag_s;  // 0 continue, 1 done after this pass
    if (tid == 0) {
        double f = 0.0;
        for (int g = 0; g < G; ++g) f += part[(int64_t)g * pd + kn + k];
        f_s = f;
        WState st = *stp;
        flag_s = 0;
        if (st.hist_len > 0 && f > st.last * (1.0 + 1e-12)) {  // lloyd.hpp:114-121
            st.err = kErrMonotone;
            st.stop = -1;
            st.done = 1;
            flag_s = 2;
        } else {
            if (p.out_hist && st.hist_len < p.hist_cap) p.out_hist[(int64_t)wl * p.hist_cap + st.hist_len] = f;
            st.last = f;
            st.hist_len += 1;
            st.nd += s * (int64_t)k;
            if (st.closing) {  // lloyd.hpp:155-163
                st.f_final = f;
                st.done = 1;
                flag_s = 1;
            } else {
                st.iters += 1;
            }
        }
        *stp = st;
    }
    __syncthreads();
    if (flag_s == 2) return;
    // counts of this pass (flags / output counts if it is the last)
    for (int j = tid; j < k; j += blockDim.x) {
        double c = 0.0;
        for (int g = 0; g < G; ++g) c += part[(int64_t)g * pd + kn + j];
        b.lastcnt[(int64_t)w * k + j] = c;
    }
    if (flag_s == 1) return;
    bool same = true;
    for (int64_t e = tid; e < kn; e += blockDim.x) {
        const int j = (int)(e / n);
        double c = 0.0, sum = 0.0;
        for (int g = 0; g < G; ++g) {
            c += part[(int64_t)g * pd + kn + j];
            sum += part[(int64_t)g * pd + e];
        }
        double v = Cm[e];
        if (c > 0.0) {
            const double inv = 1.0 / c;
            v = sum * inv;
        }
        same &= (v == Cm[e]);
        Cm[e] = v;
    }
    const bool all_same = __syncthreads_and(same);
    if (tid == 0) {
        WState st = *stp;
        const double f = f_s;
        if (all_same) {
            st.stop = 2;  // fixed_point
            st.f_final = f;
            st.done = 1;
        } else {
            bool go_close = false;
            if (isfinite(st.f_prev)) {
                const double improvement = st.f_prev > 0.0 ? (st.f_prev - f) / st.f_prev : 0.0;
                if (improvement < p.rel_tol) {
                    st.stop = 0;  // tolerance
                    go_close = true;
                }
            }
            st.f_prev = f;
            if (!go_close && st.iters == p.max_iters) {
                st.stop = 1;
                go_close = true;
            }
            st.closing = go_close ? 1 : 0;
        }
        *stp = st;
    }
}

__global__ void wide_max_pending_kernel(WideBufs b, int Wb) {  // K-means++ slots still to run
    __shared__ int c;
    if (threadIdx.x == 0) c = 0;
    __syncthreads();
    for (int w = threadIdx.x; w < Wb; w += blockDim.x) atomicMax(&c, b.st[w].n_pending - b.st[w].next);
    __syncthreads();
    if (threadIdx.x == 0) *b.active = c;
}

__global__ void wide_count_active_kernel(WideBufs b, int Wb) {
    __shared__ int c;
    if (threadIdx.x == 0) c = 0;
    __syncthreads();
    for (int w = threadIdx.x; w < Wb; w += blockDim.x)
        if (!b.st[w].done) atomicAdd(&c, 1);
    __syncthreads();
    if (threadIdx.x == 0) *b.active = c;
}

// ---------------------------------------------------------------- outputs
__global__ void wide_output_kernel(const StepParams p, WideBufs b, int w0) {
    const int w = blockIdx.x, wl = w0 + w, tid = threadIdx.x, k = p.k, n = p.n;
    const int64_t kn = (int64_t)k * n, s = p.s;
    WState* stp = b.st + w;
    uint8_t* fl = b.flags + (int64_t)w * k;
    const double* Cm = b.Cm + (int64_t)w * kn;
    if (stp->run_lloyd && stp->stop >= 0) {  // flags = empty clusters of the last pass
        for (int j = tid; j < k; j += blockDim.x) fl[j] = b.lastcnt[(int64_t)w * k + j] == 0.0 ? 1 : 0;
        if (p.out_counts)
            for (int j = tid; j < k; j += blockDim.x)
                p.out_counts[(int64_t)wl * k + j] = (int64_t)b.lastcnt[(int64_t)w * k + j];
        if (p.out_labels)
            for (int64_t i = tid; i < s; i += blockDim.x) p.out_labels[(int64_t)wl * s + i] = b.labels[(int64_t)w * s + i];
    }
    __syncthreads();
    if (p.out_c)
        for (int64_t e = tid; e < kn; e += blockDim.x) p.out_c[(int64_t)wl * kn + e] = Cm[e];
    if (p.out_f)
        for (int j = tid; j < k; j += blockDim.x) p.out_f[(int64_t)wl * k + j] = fl[j];
    const WState st = *stp;
    if (tid == 0) {
        if (p.out_obj) p.out_obj[wl] = st.f_final;
        if (p.out_iters) p.out_iters[wl] = st.iters;
        if (p.out_stop) p.out_stop[wl] = st.stop;
        if (p.out_nd) p.out_nd[wl] = st.nd;
        if (p.out_filled) p.out_filled[wl] = st.filled;
        if (p.out_err) p.out_err[wl] = st.err;
        if (p.out_hist_len) p.out_hist_len[wl] = st.hist_len;
    }
    if (p.inc_obj) {  // keep-the-best (engine.hpp:254, strict <)
        const bool acc = st.run_lloyd && st.err == kErrNone && st.f_final < p.inc_obj[wl];
        __syncthreads();
        if (acc) {
            for (int64_t e = tid; e < kn; e += blockDim.x) p.inc_c[(int64_t)wl * kn + e] = Cm[e];
            for (int j = tid; j < k; j += blockDim.x) p.inc_f[(int64_t)wl * k + j] = fl[j];
        }
        __syncthreads();
        if (tid == 0) {
            if (acc) p.inc_obj[wl] = st.f_final;
            p.accepted[wl] = acc ? 1 : 0;
        }
    }
}

// ---------------------------------------------------------------- f(C, X)
// full-data assignment/objective for n > 32 (mssc_objective core.hpp:224-233, final_assignment
// engine.hpp:197-229): block b takes rows b*kWT + t (+ grid strides); exact distances, strict
// argmin over the valid centres, per-block cost by thread-sequential sums and a fixed tree
template <typename T>
__global__ void __launch_bounds__(kWT) wide_objective_kernel(const ObjParams p) {
    extern __shared__ __align__(16) float orec[];
    __shared__ double red[kWT];
    __shared__ float red_f[1];
    const T* X = static_cast<const T*>(p.X);
    const int n = p.n, kv = p.kv;
    const int kpad = (kv + kKT - 1) / kKT * kKT, n4 = (n + 3) & ~3;
    float* rec = orec;
    float* ccs = rec + (int64_t)kpad * n4;
    build_records(p.C, kv, kpad, n, n4, rec, ccs);
    const float cmax = records_cmax(ccs, kpad, red_f);
    const float kappa = 2.0f * (float)((n + 1) / 2 + 12) * 5.9604645e-8f;
    const bool vec = sizeof(T) == 4 && (n & 3) == 0;
    const bool vecd = sizeof(T) == 4 ? (n & 3) == 0 : (n & 1) == 0;
    double cost = 0.0;
    const int64_t stride = (int64_t)gridDim.x * kWT;
    const int64_t iters = (p.m + stride - 1) / stride;  // uniform trip count: warp-collective ties
    for (int64_t it = 0; it < iters; ++it) {
        const int64_t i = it * stride + (int64_t)blockIdx.x * kWT + threadIdx.x;
        const bool valid = i < p.m;
        int lab = 0;
        float m1 = 0.f, m2 = 0.f, xx = 0.f;
        if (valid) screen_row<T>(X + i * n, n, n4, kpad, rec, ccs, vec, lab, m1, m2, xx);
        const float sc = sqrtf(xx) * 1.0001f + cmax;
        const unsigned tie = __ballot_sync(0xffffffffu, valid && !(m2 - m1 > kappa * sc * sc));
        if (tie) exact_ties<T>(tie, X, i - (threadIdx.x & 31), n, kv, p.C, lab);
        if (!valid) continue;
        cost += dist1<T>(X + i * n, n, p.C + (int64_t)lab * n, vecd);
        const int orig = p.remap ? p.remap[lab] : lab;
        if (p.labels) p.labels[i] = orig;
        if (p.counts) atomicAdd(p.counts + orig, 1ull);
    }
    const double tot = cta_sum(cost, red);
    if (threadIdx.x == 0) p.block_cost[blockIdx.x] = tot;
}

// ---------------------------------------------------------------- host side
struct Arena {  // grow-only device scratch per device
    void* p = nullptr;
    size_t cap = 0;
};
std::mutex g_mu;
std::map<int, Arena> g_arena;

cudaError_t arena_get(size_t bytes, void** out) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_mu);
    Arena& a = g_arena[dev];
    if (a.cap < bytes) {
        if (a.p) {
            cudaDeviceSynchronize();
            cudaFree(a.p);
        }
        a.p = nullptr;
        a.cap = 0;
        cudaError_t e = cudaMalloc(&a.p, bytes);
        if (e != cudaSuccess) return e;
        a.cap = bytes;
    }
    *out = a.p;
    return cudaSuccess;
}

}  // namespace
}  // namespace hpcg
#include "wide_tc.cuh"
namespace hpcg {
namespace {

// the tensor-core screen's launch: tensor map over the batch's samples, one CTA per SM
template <int NA, int KPS>
cudaError_t launch_wide_tc(const StepParams& p, const WideBufs& b, const float* ccw, int Wb, int sms,
                           const CUtensorMap& tmap, cudaStream_t st) {
    const int tpw = (int)((p.s + 127) / 128);
    const int smem = wide_tc_smem<NA>();
    cudaError_t e = cudaFuncSetAttribute(wide_screen_tc_kernel<NA, KPS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         smem);
    if (e != cudaSuccess) return e;
    wide_screen_tc_kernel<NA, KPS><<<sms, WtcGeo<NA>::THREADS, smem, st>>>(p, b, ccw, Wb * tpw, tpw, tmap);
    return cudaGetLastError();
}

bool wide_tmap(const void* S, int n, int64_t rows, CUtensorMap* map) {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return false;
        fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    }
    memset(map, 0, sizeof *map);
    const cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)n * 4};
    const cuuint32_t box[2] = {32, 128};
    const cuuint32_t estr[2] = {1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(S), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

size_t up256(size_t v) { return (v + 255) & ~(size_t)255; }

template <typename T>
cudaError_t run_batch(const StepParams& p, int w0, int Wb, cudaStream_t st, std::string* why) {
    const int k = p.k, n = p.n, ncand = p.candidates;
    const int64_t s = p.s, kn = (int64_t)k * n;
    const int nblk = (int)((s + kSeedRows - 1) / kSeedRows);
    int sms = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // CTAs per worker for the Lloyd pass: enough CTAs for the whole GPU, each at least a few rounds
    // (enough CTAs to fill the GPU twice, and at most ~RPC 256-row rounds per CTA: each round is a
    // sequence of barriers, so long per-CTA row ranges serialise)
    static const int rpc = getenv("HPCG_WIDE_RPC") ? atoi(getenv("HPCG_WIDE_RPC")) : 24;  // diagnostics
    // the geometry of a batch of the engine's size (p.geo_W), so CTA partitions -- and the sums --
    // do not depend on how many workers this rank holds
    const size_t per_worker_b = (size_t)s * ((size_t)n * sizeof(T) + 8 + 1 + 4) + 1024;
    const int Wgeo = p.geo_W > 0 ? (int)std::max<size_t>(1, std::min<size_t>((size_t)p.geo_W, ((size_t)4 << 30) /
                                                                                        std::max<size_t>(per_worker_b, 1)))
                                 : Wb;
    int G = std::max<int>(std::min<int>((int)((int64_t)2 * sms / Wgeo), (int)((s + 4 * kWT - 1) / (4 * kWT))),
                          (int)((s + (int64_t)rpc * kWT - 1) / ((int64_t)rpc * kWT)));
    G = std::max(G, 1);
    const int64_t pd = kn + k + 1;
    // scratch layout
    size_t off = 0;
    auto take = [&](size_t bytes) {
        const size_t o = off;
        off = up256(off + bytes);
        return o;
    };
    const size_t oS = take((size_t)Wb * s * n * sizeof(T)), oC = take((size_t)Wb * kn * 8),
                 od2 = take((size_t)Wb * s * 8), orf = take((size_t)Wb * s),
                 ocand = take((size_t)Wb * kMaxCandidates * n * 8), obt = take((size_t)Wb * (nblk + 1) * 8),
                 obc = take((size_t)Wb * kMaxCandidates * nblk * 8), obch = take((size_t)Wb * kMaxCandidates * nblk * 8),
                 opart = take((size_t)Wb * G * pd * 8),
                 olc = take((size_t)Wb * k * 8), ofl = take((size_t)Wb * k), opend = take((size_t)Wb * k * 4),
                 olab = take((size_t)Wb * s * 4), oact = take(4), ost = take((size_t)Wb * sizeof(WState)),
                 occw = take((size_t)Wb * (kTcwN + 1) * 4);
    void* base = nullptr;
    cudaError_t e = arena_get(off, &base);
    if (e != cudaSuccess) {
        if (why) *why = "wide step: scratch allocation";
        return e;
    }
    char* c8 = static_cast<char*>(base);
    WideBufs b;
    b.S = c8 + oS;
    b.Cm = reinterpret_cast<double*>(c8 + oC);
    b.d2 = reinterpret_cast<double*>(c8 + od2);
    b.rflag = reinterpret_cast<uint8_t*>(c8 + orf);
    b.cand = reinterpret_cast<double*>(c8 + ocand);
    b.btot = reinterpret_cast<double*>(c8 + obt);
    b.bcost = reinterpret_cast<double*>(c8 + obc);
    b.bcost_hi = reinterpret_cast<double*>(c8 + obch);
    b.part = reinterpret_cast<double*>(c8 + opart);
    b.lastcnt = reinterpret_cast<double*>(c8 + olc);
    b.flags = reinterpret_cast<uint8_t*>(c8 + ofl);
    b.pend = reinterpret_cast<int32_t*>(c8 + opend);
    b.labels = reinterpret_cast<int32_t*>(c8 + olab);
    b.active = reinterpret_cast<int32_t*>(c8 + oact);
    b.st = reinterpret_cast<WState*>(c8 + ost);

    const dim3 rows_grid((unsigned)((s + kWT - 1) / kWT), (unsigned)Wb);
    {
        const int64_t rowb = (int64_t)n * sizeof(T);
        const dim3 gg((unsigned)((s + 255) / 256), (unsigned)Wb);
        unsigned char* Sb = static_cast<unsigned char*>(b.S);
        const bool aligned = p.nshards > 1 || (reinterpret_cast<uintptr_t>(p.X) & 15) == 0;
        if (rowb % 16 == 0 && aligned)
            wide_gather_kernel<16><<<gg, 256, 0, st>>>(p, w0, rowb, Sb);
        else if (rowb % 8 == 0)
            wide_gather_kernel<8><<<gg, 256, 0, st>>>(p, w0, rowb, Sb);
        else
            wide_gather_kernel<4><<<gg, 256, 0, st>>>(p, w0, rowb, Sb);
    }
    wide_init_kernel<T><<<Wb, kWT, 0, st>>>(p, w0, b);
    {
        const int kpad = (k + kKT - 1) / kKT * kKT, n4 = (n + 3) & ~3;
        const size_t rs = (size_t)kpad * n4 * 4 + (size_t)kpad * 4;
        auto go = [&](auto kern) -> cudaError_t {
            cudaError_t e2 = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rs);
            if (e2 != cudaSuccess) return e2;
            const dim3 d2_grid((unsigned)((s + (int64_t)kWT * kD2Blocks - 1) / ((int64_t)kWT * kD2Blocks)), (unsigned)Wb);
            kern<<<d2_grid, kWT, rs, st>>>(p, b);
            return cudaSuccess;
        };
        e = n == 8 ? go(wide_d2init_kernel<T, 8>) : n == 16 ? go(wide_d2init_kernel<T, 16>)
            : n == 32 ? go(wide_d2init_kernel<T, 32>) : n == 128 ? go(wide_d2init_kernel<T, 128>)
                      : go(wide_d2init_kernel<T, 0>);
        if (e != cudaSuccess) return e;
    }
    // K-means++ slots: as many host iterations as the worker with the most pending slots
    int32_t slots = 0;
    wide_max_pending_kernel<<<1, 256, 0, st>>>(b, Wb);
    e = cudaMemcpyAsync(&slots, b.active, 4, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return e;
    const size_t cost_smem = (size_t)ncand * ((n + 3) & ~3) * 4;
    if (slots > 0) {
        e = cudaFuncSetAttribute(wide_cost_kernel<T, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cost_smem);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(wide_cost_kernel<T, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cost_smem);
        if (e != cudaSuccess) return e;
    }
    const int staged = (size_t)(nblk + 1) * 8 <= 200 * 1024 ? 1 : 0;
    const size_t scan_smem = staged ? (size_t)(nblk + 1) * 8 : 0;
    if (slots > 0 && scan_smem > 48 * 1024) {
        e = cudaFuncSetAttribute(wide_cdfscan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)scan_smem);
        if (e != cudaSuccess) return e;
    }
    for (int it = 0; it < slots; ++it) {
        const dim3 fgrid((unsigned)((nblk + 7) / 8), (unsigned)Wb);
        if (n == 8)
            wide_cdf_kernel<T, 8><<<fgrid, 256, 0, st>>>(p, b, nblk, it);
        else if (n == 16)
            wide_cdf_kernel<T, 16><<<fgrid, 256, 0, st>>>(p, b, nblk, it);
        else if (n == 128)
            wide_cdf_kernel<T, 128><<<fgrid, 256, 0, st>>>(p, b, nblk, it);
        else
            wide_cdf_kernel<T, 0><<<fgrid, 256, 0, st>>>(p, b, nblk, it);
        wide_cdfscan_kernel<<<(unsigned)Wb, 32, scan_smem, st>>>(b, nblk, staged);
        wide_draw_kernel<T><<<dim3((unsigned)ncand, (unsigned)Wb), 32, 0, st>>>(p, w0, b, nblk);
        const dim3 cgrid((unsigned)((nblk + kCostBPC - 1) / kCostBPC), (unsigned)Wb);
        // the interval pass and its decision, then the exact pass + decision for undecided workers
        const bool interval = sizeof(T) == 4 && (n == 128 || n == 64) && ncand <= 3;
        auto cost_pass = [&](auto ivc) {
            constexpr bool IV = decltype(ivc)::value != 0;
            if (n == 8)
                wide_cost_np_kernel<T, 8, IV><<<cgrid, kWT, 0, st>>>(p, b, nblk);
            else if (n == 16)
                wide_cost_np_kernel<T, 16, IV><<<cgrid, kWT, 0, st>>>(p, b, nblk);
            else if (n == 32)
                wide_cost_np_kernel<T, 32, IV><<<cgrid, kWT, 0, st>>>(p, b, nblk);
            else if (sizeof(T) == 4 && n == 128 && ncand <= 3)
                wide_cost_rows_kernel<128, IV><<<cgrid, kWT, 0, st>>>(p, b, nblk);
            else if (sizeof(T) == 4 && n == 64 && ncand <= 3)
                wide_cost_rows_kernel<64, IV><<<cgrid, kWT, 0, st>>>(p, b, nblk);
            else
                wide_cost_kernel<T, IV><<<cgrid, kWT, cost_smem, st>>>(p, b, nblk);
        };
        cost_pass(IntC<1>{});
        wide_decide_kernel<false><<<Wb, 32 * kMaxCandidates, 0, st>>>(p, b, nblk);
        if (interval) {  // only the wide-row pass leaves workers undecided
            cost_pass(IntC<0>{});
            wide_decide_kernel<true><<<Wb, 32 * kMaxCandidates, 0, st>>>(p, b, nblk);
        }
    }
    // Lloyd: passes until every worker of the batch stopped
    wide_lloyd_begin_kernel<<<Wb, 32, 0, st>>>(p, b);
    const int kpad = (k + kKT - 1) / kKT * kKT, n4 = (n + 3) & ~3;
    // the assign pass in rounds of kAT rows (fewer round barriers per row than kWT)
    constexpr int kAT = 256, kAR = 8;  // 2048 rows per round
    const size_t smem = (size_t)(kn + k + kAT + 1) * 8 + (size_t)kpad * n4 * 4 + (size_t)kpad * 4 +
                        (size_t)(kAR * (kAT / 32) * k + k + 1 + kAT * kAR) * 4;
    // the assign pass specialised for common row widths (index and loop arithmetic at compile time)
    auto assign_kern = n == 8     ? wide_assign_kernel<T, kAT, 8, kAR>
                       : n == 16  ? wide_assign_kernel<T, kAT, 16, kAR>
                       : n == 32  ? wide_assign_kernel<T, kAT, 32, kAR>
                       : n == 64  ? wide_assign_kernel<T, kAT, 64, kAR>
                       : n == 128 ? wide_assign_kernel<T, kAT, 128, kAR>
                                  : wide_assign_kernel<T, kAT, 0, kAR>;
    e = cudaFuncSetAttribute(assign_kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) {
        if (why) *why = "wide step: k*n too large for the pass accumulator";
        return e;
    }
    // tensor-core screen for wide fp32 samples (config 4): n = 64 / 128, k <= 32
    static const bool no_tc = getenv("HPCG_WIDE_NO_TC") != nullptr;
    float* ccw = reinterpret_cast<float*>(static_cast<char*>(base) + occw);
    CUtensorMap stmap;
    const bool tc = sizeof(T) == 4 && (n == 64 || n == 128) && k <= 32 && !no_tc &&
                    wide_tmap(b.S, n, (int64_t)Wb * s, &stmap);
    if (p.do_lloyd) {
        int32_t active = 0;
        for (int pass = 0; pass <= p.max_iters + 1; ++pass) {
            if (tc) {
                wide_cc_kernel<<<Wb, 32, 0, st>>>(p, b, ccw);
                e = n == 128 ? (k <= 16 ? launch_wide_tc<4, 8>(p, b, ccw, Wb, sms, stmap, st)
                                        : launch_wide_tc<4, 16>(p, b, ccw, Wb, sms, stmap, st))
                             : (k <= 16 ? launch_wide_tc<2, 8>(p, b, ccw, Wb, sms, stmap, st)
                                        : launch_wide_tc<2, 16>(p, b, ccw, Wb, sms, stmap, st));
                if (e != cudaSuccess) return e;
            }
            assign_kern<<<dim3((unsigned)G, (unsigned)Wb), kAT, smem, st>>>(p, b, G, tc ? 1 : 0);
            wide_lloyd_reduce_kernel<<<Wb, kWT, 0, st>>>(p, b, G, w0);
            if ((pass & 3) == 3 || pass == p.max_iters + 1) {  // stop check every few passes
                wide_count_active_kernel<<<1, 256, 0, st>>>(b, Wb);
                e = cudaMemcpyAsync(&active, b.active, 4, cudaMemcpyDeviceToHost, st);
                if (e == cudaSuccess) e = cudaStreamSynchronize(st);
                if (e != cudaSuccess) return e;
                if (active == 0) break;
            }
        }
    }
    wide_output_kernel<<<Wb, kWT, 0, st>>>(p, b, w0);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_objective_wide(int dtype, const ObjParams& p, int* nblocks, cudaStream_t st) {
    int sms = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int nb = std::max(1, std::min(nblocks[0], sms * 4));  // fixed per device: reproducible
    nblocks[0] = nb;
    const int kpad = (p.kv + kKT - 1) / kKT * kKT, n4 = (p.n + 3) & ~3;
    const size_t rs = (size_t)kpad * n4 * 4 + (size_t)kpad * 4;
    cudaError_t e = dtype == 0 ? cudaFuncSetAttribute(wide_objective_kernel<float>,
                                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rs)
                               : cudaFuncSetAttribute(wide_objective_kernel<double>,
                                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rs);
    if (e != cudaSuccess) return e;
    if (dtype == 0)
        wide_objective_kernel<float><<<nb, kWT, rs, st>>>(p);
    else
        wide_objective_kernel<double><<<nb, kWT, rs, st>>>(p);
    return cudaGetLastError();
}

// Wide-shape worker step: same contract as launch_step, any n and k (k*n bounded by the
// pass accumulator in shared memory), any s; workers in batches bounded by the scratch size.
cudaError_t launch_step_wide(int dtype, const StepParams& p, cudaStream_t st, std::string* why) {
    const size_t row_bytes = (size_t)p.n * (dtype == 0 ? 4 : 8);
    const size_t per_worker = (size_t)p.s * (row_bytes + 8 + 1 + 4) + 1024;
    const size_t budget = (size_t)4 << 30;
    const int Wb = (int)std::max<size_t>(1, std::min<size_t>((size_t)p.W, budget / std::max<size_t>(per_worker, 1)));
    for (int w0 = 0; w0 < p.W; w0 += Wb) {
        const int nb = std::min(Wb, p.W - w0);
        StepParams q = p;
        cudaError_t e = dtype == 0 ? run_batch<float>(q, w0, nb, st, why) : run_batch<double>(q, w0, nb, st, why);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace hpcg
