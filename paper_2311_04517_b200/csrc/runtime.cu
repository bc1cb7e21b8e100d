// Host runtime of libhpcg.so: the C-ABI declared in include/hpcg.h.
//
// Owns device memory and streams, validates arguments with the reference's own error
// texts, drives the lockstep HPClust engine round by round (engine.hpp:380-436) with the
// worker-step kernel, and replays the reference's mt19937_64 worker streams on the host
// when RNG parity with the reference is requested. No CPU compute fallback exists: every
// numeric result comes from the sm_100a kernels.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda.h>
#include <dlfcn.h>
#include <nccl.h>
#include <limits>
#include <mutex>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>
#include <type_traits>

#include "../../include/hpcg.h"
#include "launch.h"

using namespace hpcg;

// ============================================================== errors
namespace {
thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define CU(call)                                                                              \
    do {                                                                                      \
        cudaError_t e_ = (call);                                                              \
        if (e_ != cudaSuccess) return fail(HPCG_ECUDA, std::string("CUDA error: ") +         \
                                                           cudaGetErrorString(e_) + " at " + \
                                                           #call);                            \
    } while (0)

constexpr double kInf = std::numeric_limits<double>::infinity();

// Every entry point binds its device and clears this host thread's last CUDA error first: a failed
// runtime call elsewhere in the process (non-sticky) must not surface as this call's launch error.
inline void bind_device(int device) {
    cudaSetDevice(device);
    cudaGetLastError();
}

// ------------------------------------------------------------ device buffers
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    cudaError_t reserve(size_t b) {
        if (b <= bytes) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
        cudaError_t e = cudaMalloc(&p, b ? b : 16);
        if (e == cudaSuccess) bytes = b;
        return e;
    }
    // grow to b bytes keeping the first `keep` bytes (stream-ordered copy; the old block is freed
    // after the copy completes because cudaFree synchronises the device)
    cudaError_t grow(size_t b, size_t keep, cudaStream_t st) {
        if (b <= bytes) return cudaSuccess;
        void* q = nullptr;
        cudaError_t e = cudaMalloc(&q, b);
        if (e != cudaSuccess) return e;
        if (p && keep) e = cudaMemcpyAsync(q, p, std::min(keep, bytes), cudaMemcpyDeviceToDevice, st);
        if (e != cudaSuccess) {
            cudaFree(q);
            return e;
        }
        if (p) cudaFree(p);
        p = q;
        bytes = b;
        return cudaSuccess;
    }
    template <typename T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

// ------------------------------------------------ std::mt19937_64 (host replay)
// The 64-bit Mersenne Twister with the parameters fixed by [rand.predef]; plus the
// reference's hand-rolled distributions (rng.hpp:38-53) and seed derivation (rng.hpp:12-33).
uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

struct Mt64 {
    uint64_t mt[312];
    int pos = 312;
    void seed(uint64_t s) {
        mt[0] = s;
        for (int i = 1; i < 312; ++i) mt[i] = 6364136223846793005ULL * (mt[i - 1] ^ (mt[i - 1] >> 62)) + (uint64_t)i;
        pos = 312;
    }
    void twist() {
        for (int i = 0; i < 312; ++i) {
            const uint64_t y = (mt[i] & 0xFFFFFFFF80000000ULL) | (mt[(i + 1) % 312] & 0x7FFFFFFFULL);
            uint64_t v = mt[(i + 156) % 312] ^ (y >> 1);
            if (y & 1) v ^= 0xB5026F5AA96619E9ULL;
            mt[i] = v;
        }
        pos = 0;
    }
    uint64_t next() {
        if (pos >= 312) twist();
        uint64_t z = mt[pos++];
        z ^= (z >> 29) & 0x5555555555555555ULL;
        z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
        z ^= (z << 37) & 0xFFF7EEE000000000ULL;
        return z ^ (z >> 43);
    }
    double unit() { return (double)(next() >> 11) * 0x1.0p-53; }
    uint64_t uniform_index(uint64_t n) {
        const uint64_t limit = UINT64_MAX - UINT64_MAX % n;
        uint64_t x;
        do {
            x = next();
        } while (x >= limit);
        return x % n;
    }
    static Mt64 derive(uint64_t master, uint64_t domain, uint64_t index) {
        Mt64 r;
        r.seed(splitmix64(master ^ splitmix64(domain ^ splitmix64(index))));
        return r;
    }
};

// engine.hpp:165-177 partial Fisher-Yates over iota(m) in O(s): only displaced slots are
// stored, so the draws (and the stream advance) are exactly the reference's.
void sparse_fisher_yates(Mt64& rng, int64_t m, int64_t s, int64_t* out) {
    std::unordered_map<int64_t, int64_t> moved;
    moved.reserve((size_t)(2 * s));
    auto at = [&](int64_t i) {
        auto it = moved.find(i);
        return it == moved.end() ? i : it->second;
    };
    for (int64_t i = 0; i < s; ++i) {
        const int64_t j = i + (int64_t)rng.uniform_index((uint64_t)(m - i));
        const int64_t vi = at(i), vj = at(j);
        moved[i] = vj;
        moved[j] = vi;
        out[i] = vj;
    }
}
}  // namespace

// ------------------------------------------------------------ NCCL (loaded at run time)
// The library links no NCCL: the communicator entry points are resolved from libnccl.so.2 when a
// multi-rank exchange is first set up, so a process that already loaded torch's NCCL shares it.
struct NcclApi {
    bool ok = false;
    std::string why;
    decltype(&ncclGetUniqueId) get_unique_id = nullptr;
    decltype(&ncclCommInitRank) comm_init_rank = nullptr;
    decltype(&ncclCommDestroy) comm_destroy = nullptr;
    decltype(&ncclAllGather) all_gather = nullptr;
    decltype(&ncclGetErrorString) error_string = nullptr;
};
const NcclApi& nccl_api() {
    static const NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            a.why = std::string("libnccl.so.2 not loadable: ") + dlerror();
            return a;
        }
        a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
        a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
        a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
        a.all_gather = reinterpret_cast<decltype(a.all_gather)>(dlsym(h, "ncclAllGather"));
        a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(h, "ncclGetErrorString"));
        a.ok = a.get_unique_id && a.comm_init_rank && a.comm_destroy && a.all_gather && a.error_string;
        if (!a.ok) a.why = "libnccl.so.2 lacks a required entry point";
        return a;
    }();
    return api;
}

// ============================================================== handles
struct hpcg_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    std::mutex mu;
    std::atomic<int64_t> launches{0};
    std::atomic<int64_t> upload_bytes{0};  // host -> device bytes of dataset uploads (hpcg_dataset_upload)
    int fp32_exact_cost = 0;               // f(C,X) over fp32 data: 1 = exact fp64 row cost, 0 = fp32 mode
    DevBuf s_a, s_b, s_c, s_d, s_e, s_f;  // scratch for one-shot calls
    DevBuf grid;                          // cell masks of the narrow-row f(C,X) filter
    DevBuf done_ctr;                      // CTA ticket counter of the self-finalising f(C,X) kernel
    int rec_slot = -1;                     // constant-bank slot of the objective records
    DevBuf rec_scratch;
    // per-kernel-class event timing (class 0 worker step, 1 objective)
    bool timing = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pending[2];
    int64_t t_count[2] = {0, 0};
    double t_ms[2] = {0.0, 0.0};
    // allocations kept across one-call runs (hpcg_run: upload, engine, finish, teardown per call):
    // the device buffer of the last destroyed uploaded dataset and the pinned finish staging
    std::mutex cache_mu;
    void* spare_x = nullptr;
    size_t spare_x_bytes = 0;
    void* pin = nullptr;
    size_t pin_bytes = 0;
    // NCCL communicator of the multi-rank exchange (hpcg_ctx_attach_comm); one rank per GPU
    ncclComm_t comm = nullptr;
    int nranks = 1, rank = 0;
};

namespace {
// constant-bank record slots (objective_kernel.cuh kRecSlots), one per live context
std::mutex g_slot_mu;
uint32_t g_slot_used = 0;
int acquire_rec_slot() {
    std::lock_guard<std::mutex> lk(g_slot_mu);
    for (int i = 0; i < kRecSlots; ++i)
        if (!(g_slot_used & (1u << i))) {
            g_slot_used |= 1u << i;
            return i;
        }
    return -1;  // more live contexts than slots: records from shared memory
}
void release_rec_slot(int i) {
    if (i < 0) return;
    std::lock_guard<std::mutex> lk(g_slot_mu);
    g_slot_used &= ~(1u << i);
}

// Brackets one launch with events on the launching stream when timing is enabled.
struct KTimer {
    hpcg_ctx* c;
    int cls;
    cudaEvent_t a = nullptr, b = nullptr;
    KTimer(hpcg_ctx* c_, int cls_) : c(c_), cls(cls_) {
        if (c->timing) {
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            cudaEventRecord(a, c->stream);
        }
    }
    void done() {
        if (a) {
            cudaEventRecord(b, c->stream);
            c->pending[cls].emplace_back(a, b);
            a = b = nullptr;
        }
    }
    ~KTimer() {
        if (a) {
            cudaEventDestroy(a);
            cudaEventDestroy(b);
        }
    }
};

__global__ void fma_probe_kernel(float* out, float a, float b, int iters) {
    float2 x[8];
    const float2 A = make_float2(a, a), B = make_float2(b, b);
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = make_float2((float)threadIdx.x + i, (float)i);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = __ffma2_rn(x[i], A, B);
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i].x + x[i].y;
    if (s == 1234.5f) out[0] = s;
}
}  // namespace

struct hpcg_dataset {
    hpcg_ctx* ctx = nullptr;
    const void* X = nullptr;  // shard 0 (the whole X when unsharded)
    int nshards = 1;          // row shards (hpcg_dataset_wrap_sharded); shard s holds rows
    const void* shard_ptr[kMaxShards] = {};   // [shard_end[s-1], shard_end[s])
    int64_t shard_end[kMaxShards] = {};
    bool owned = false;
    size_t bytes = 0;  // owned allocation size
    int dtype = 0;
    int64_t m = 0, n = 0;
    ~hpcg_dataset() {
        if (!(owned && X)) return;
        // keep the largest freed upload buffer for the next upload on this context
        std::lock_guard<std::mutex> lk(ctx->cache_mu);
        if (bytes > ctx->spare_x_bytes) {
            if (ctx->spare_x) cudaFree(ctx->spare_x);
            ctx->spare_x = const_cast<void*>(X);
            ctx->spare_x_bytes = bytes;
        } else {
            cudaFree(const_cast<void*>(X));
        }
    }
};

namespace {
size_t dsize(int dtype) { return dtype == HPCG_F32 ? 4 : 8; }

void set_shards(StepParams& p, const hpcg_dataset* ds) {
    p.nshards = ds->nshards;
    for (int i = 0; i < ds->nshards && i < kMaxShards; ++i) {
        p.shard_ptr[i] = ds->shard_ptr[i];
        p.shard_end[i] = ds->shard_end[i];
    }
}

int check_shape(int dtype, int64_t n, int64_t k) {
    if (dtype != HPCG_F32 && dtype != HPCG_F64) return fail(HPCG_EINVAL, "unknown dtype");
    if (n < 1) return fail(HPCG_EINVAL, "dataset needs at least one feature");
    // n <= 32 and k <= 32 run cluster-resident; larger shapes take the grid-wide path (wide.cu)
    if (n > kWideMaxN || k > kWideMaxK || n * k > kWideMaxKN)
        return fail(HPCG_EUNSUPPORTED, "k * n beyond the grid-wide path's pass accumulator (16384)");
    return HPCG_OK;
}

// ------------------------------------------------------------ small kernels
struct ShardTable {
    int n = 1;
    const unsigned char* ptr[kMaxShards] = {};
    int64_t end[kMaxShards] = {};
};

__global__ void gather_kernel(const ShardTable t, int64_t rowb, const int64_t* idx, int64_t s, unsigned char* out) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= s * rowb) return;
    const int64_t i = e / rowb, b = e - i * rowb;
    int64_t g = idx[i];
    int sh = 0;
    while (sh + 1 < t.n && g >= t.end[sh]) ++sh;
    if (sh) g -= t.end[sh - 1];
    out[e] = t.ptr[sh][g * rowb + b];
}

// Dense sample gather S[w][i][:] = X[prp_w(i)][:] for W workers (the worker step's gather phase on
// its own, for measuring the gather at HBM rate): per warp 32 rows, one PRP index per lane, then
// the rows' V-byte chunks chunk-major across the warp with the indices shuffled across; all of a
// lane's loads are issued before its stores.
template <int V>
__global__ void __launch_bounds__(256) sample_gather_kernel(const ShardTable t, int64_t m, int64_t rowb, int64_t s,
                                                            uint64_t key, uint32_t round, int32_t worker_base,
                                                            uint32_t pa, uint32_t pb, float pinv,
                                                            unsigned char* __restrict__ S) {
    using VT = typename std::conditional<V == 16, uint4, typename std::conditional<V == 8, uint2, uint32_t>::type>::type;
    const int w = blockIdx.y, lane = threadIdx.x & 31;
    const SamplePRP prp = SamplePRP::make(key, round, (uint32_t)(worker_base + w), (uint64_t)m, pa, pb, pinv);
    const int cpr = (int)(rowb / V);
    const int64_t i0 = ((int64_t)blockIdx.x * 8 + (threadIdx.x >> 5)) * 32;
    if (i0 >= s) return;
    const int64_t i = i0 + lane;
    const int64_t g = i < s ? (int64_t)prp((uint64_t)i) : 0;
    int sh = 0;
    while (sh + 1 < t.n && g >= t.end[sh]) ++sh;
    const unsigned char* src = t.ptr[sh] + (g - (sh ? t.end[sh - 1] : 0)) * rowb;
    unsigned char* dst = S + ((int64_t)w * s + i0) * rowb;
    const int total = 32 * cpr;
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

struct RoundEndParams {
    int W, k, n;
    int64_t round;  // 0-based round just finished
    int publish;    // round was cooperative (publish accepted) ...
    int carry;      // ... or hybrid carry-over round (publish finite incumbents)
    int log;        // record the round (accept/objective logs, n_d, errors); 0 = publication only
    int worker_base;
    double ts;      // publication timestamp: round + 1 (lockstep) or seconds (wall clock)
    const uint8_t* accepted;
    const double* inc_obj;
    const double* inc_c;
    const uint8_t* inc_f;
    const int64_t* nd;
    const int32_t* err;
    uint8_t* log_acc;  // [R x W]
    double* log_obj;   // [R x W]
    int32_t* err_first;
    unsigned long long* nd_total;
    int64_t* sh_version;
    double* sh_obj;
    int32_t* sh_worker;
    double* sh_c;
    uint8_t* sh_f;
    double* pub_log;  // [cap x 4]
    int64_t* pub_count;
    int64_t pub_cap;
};

// engine.hpp:391-402 on_round_end: publications in worker-id order, strict < (engine.hpp:131)
// The worker records are staged in shared memory by all threads first, so the sequential
// publication scan (thread 0, worker-id order) reads shared memory instead of global memory.
__global__ void round_end_kernel(const RoundEndParams p) {
    __shared__ int s_winner;
    __shared__ unsigned long long s_nd[256];
    extern __shared__ double rs_obj[];  // [W] incumbent objectives, then [W] accepted flags
    uint8_t* rs_acc = reinterpret_cast<uint8_t*>(rs_obj + p.W);
    unsigned long long nd = 0;
    for (int w = threadIdx.x; w < p.W; w += blockDim.x) {
        const uint8_t a = p.log ? p.accepted[w] : (uint8_t)0;
        const double f = p.inc_obj[w];
        rs_acc[w] = a;
        rs_obj[w] = f;
        if (p.log) {
            p.log_acc[p.round * p.W + w] = a;
            p.log_obj[p.round * p.W + w] = f;
            nd += (unsigned long long)p.nd[w];
            if (p.err[w] != 0 && p.err_first[w] == 0) p.err_first[w] = p.err[w];
        }
    }
    s_nd[threadIdx.x] = nd;
    __syncthreads();
    if (threadIdx.x < 32) {
        // n_d: lane sums of 8 slots, then a warp tree (integers: order-free)
        const int lane = threadIdx.x;
        unsigned long long t = 0;
        for (int i = lane; i < (int)blockDim.x; i += 32) t += s_nd[i];
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (lane == 0 && p.log) *p.nd_total += t;
        // publication in worker-id order with strict < (engine.hpp:391-402): worker w publishes iff
        // its candidate objective is below min(shared best, every earlier candidate) -- an
        // exclusive prefix-min, 32 workers per step
        int winner = -1;
        if (p.publish || p.carry) {
            double best = *p.sh_obj;
            int64_t ver = *p.sh_version;
            int64_t cnt = *p.pub_count;
            const double inf = __longlong_as_double(0x7ff0000000000000LL);
            for (int w0 = 0; w0 < p.W; w0 += 32) {
                const int w = w0 + lane;
                const double f = w < p.W ? rs_obj[w] : inf;
                const bool cand = w < p.W && ((p.publish && rs_acc[w]) || (p.carry && isfinite(f)));
                const double c = cand ? f : inf;
                double incl = c;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const double y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl = fmin(incl, y);
                }
                double excl = __shfl_up_sync(0xffffffffu, incl, 1);
                if (lane == 0) excl = inf;
                const bool pub = cand && c < fmin(best, excl);
                const unsigned mask = __ballot_sync(0xffffffffu, pub);
                const int rank = __popc(mask & ((1u << lane) - 1u));
                if (pub && cnt + rank < p.pub_cap) {
                    const int64_t at = cnt + rank;
                    p.pub_log[at * 4 + 0] = (double)(ver + rank + 1);
                    p.pub_log[at * 4 + 1] = (double)(p.worker_base + w);
                    p.pub_log[at * 4 + 2] = f;
                    p.pub_log[at * 4 + 3] = p.ts;
                }
                if (mask) {
                    const int last = 31 - __clz(mask);
                    winner = w0 + last;
                    best = __shfl_sync(0xffffffffu, c, last);
                    ver += __popc(mask);
                    cnt += __popc(mask);
                }
            }
            if (lane == 0) {
                *p.pub_count = cnt;
                if (winner >= 0) {
                    *p.sh_obj = best;
                    *p.sh_version = ver;
                    *p.sh_worker = p.worker_base + winner;
                }
            }
        }
        if (lane == 0) s_winner = winner;
    }
    __syncthreads();
    const int wn = s_winner;
    if (wn >= 0) {
        const int64_t kn = (int64_t)p.k * p.n;
        for (int64_t e = threadIdx.x; e < kn; e += blockDim.x) p.sh_c[e] = p.inc_c[wn * kn + e];
        for (int j = threadIdx.x; j < p.k; j += blockDim.x) p.sh_f[j] = p.inc_f[(int64_t)wn * p.k + j];
    }
}

// ---------------------------------------------------------------- multi-rank exchange
// A round of a multi-rank engine (one rank per GPU, workers [base_r, base_r + W_r) on rank r,
// bases contiguous in rank order) publishes exactly as ONE engine with all ranks' workers would:
// every rank packs its round candidates (the objective of each local worker that would publish --
// accepted in a cooperative round, or a finite incumbent at the hybrid carry-over -- else +inf) and
// the centroids of its local minimum; the records are all-gathered (NCCL over NVLink, or a caller
// collective); every rank then replays the reference's publication scan over the global worker
// order (engine.hpp:391-402: worker-id order, strict < against the shared best) on the device. The
// scan's last publisher is necessarily its rank's first local minimum, whose centroids travelled
// in the record, so every rank installs the identical shared best and logs identical publications.
//   round record (doubles): [W_r, base_r, clock, local argmin | cand[Wmax] | C[k*n] | flags[k]]
__host__ __device__ inline int64_t xch_round_len(int64_t Wmax, int64_t kn, int64_t k) { return 4 + Wmax + kn + k; }

struct XPackParams {
    int W, Wmax, k, n, base;
    int publish, carry;
    double now;
    const uint8_t* accepted;
    const double* inc_obj;
    const double* inc_c;
    const uint8_t* inc_f;
    double* rec;
};

__global__ void xch_pack_round_kernel(const XPackParams p) {
    __shared__ double so[32];
    __shared__ int si[32];
    __shared__ int s_best;
    const double inf = __longlong_as_double(0x7ff0000000000000LL);
    double bo = inf;
    int bi = -1;
    for (int w = threadIdx.x; w < p.Wmax; w += blockDim.x) {
        double c = inf;
        if (w < p.W) {
            const double f = p.inc_obj[w];
            const bool cand = (p.publish && p.accepted[w]) || (p.carry && isfinite(f));
            c = cand ? f : inf;
        }
        p.rec[4 + w] = c;
        if (c < bo) {  // per-thread strided scan: ids increase, strict < keeps the first
            bo = c;
            bi = w;
        }
    }
    auto better = [](double o, int i, double bo_, int bi_) {
        return i >= 0 && (bi_ < 0 || o < bo_ || (o == bo_ && i < bi_));
    };
    for (int off = 16; off > 0; off >>= 1) {
        const double oo = __shfl_down_sync(0xffffffffu, bo, off);
        const int oi = __shfl_down_sync(0xffffffffu, bi, off);
        if (better(oo, oi, bo, bi)) {
            bo = oo;
            bi = oi;
        }
    }
    if ((threadIdx.x & 31) == 0) {
        so[threadIdx.x >> 5] = bo;
        si[threadIdx.x >> 5] = bi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double b = inf;
        int bw = -1;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w)
            if (better(so[w], si[w], b, bw)) {
                b = so[w];
                bw = si[w];
            }
        s_best = bw;
        p.rec[0] = (double)p.W;
        p.rec[1] = (double)p.base;
        p.rec[2] = p.now;
        p.rec[3] = (double)bw;
    }
    __syncthreads();
    const int bw = s_best;
    const int64_t kn = (int64_t)p.k * p.n;
    double* rc = p.rec + 4 + p.Wmax;
    for (int64_t e = threadIdx.x; e < kn; e += blockDim.x) rc[e] = bw >= 0 ? p.inc_c[(int64_t)bw * kn + e] : 0.0;
    for (int j = threadIdx.x; j < p.k; j += blockDim.x) rc[kn + j] = bw >= 0 ? (double)p.inc_f[(int64_t)bw * p.k + j] : 1.0;
}

struct XMergeParams {
    int G, Wmax, k, n;
    int ts_from_clock;  // wall clock: the publication timestamp is the latest clock among the ranks
    double ts;
    const double* recv;  // [G][round record]
    int64_t* sh_version;
    double* sh_obj;
    int32_t* sh_worker;
    double* sh_c;
    uint8_t* sh_f;
    double* pub_log;
    int64_t* pub_count;
    int64_t pub_cap;
    int32_t* err;  // set when the scan's winner is not its rank's packed minimum (cannot happen)
};

__global__ void xch_merge_round_kernel(const XMergeParams p) {
    __shared__ int s_wr, s_ww;
    const int lane = threadIdx.x & 31;
    const double inf = __longlong_as_double(0x7ff0000000000000LL);
    const int64_t L = xch_round_len(p.Wmax, (int64_t)p.k * p.n, p.k);
    if (threadIdx.x < 32) {
        double ts = p.ts;
        if (p.ts_from_clock) {
            ts = 0.0;
            for (int r = 0; r < p.G; ++r) ts = fmax(ts, p.recv[r * L + 2]);
        }
        double best = *p.sh_obj;
        int64_t ver = *p.sh_version, cnt = *p.pub_count;
        int wr = -1, ww = -1;
        for (int r = 0; r < p.G; ++r) {
            const double* rec = p.recv + r * L;
            const int Wr = (int)rec[0];
            const int64_t base = (int64_t)rec[1];
            for (int w0 = 0; w0 < Wr; w0 += 32) {  // the round_end_kernel scan, in global worker order
                const int w = w0 + lane;
                const double c = w < Wr ? rec[4 + w] : inf;
                double incl = c;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const double y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl = fmin(incl, y);
                }
                double excl = __shfl_up_sync(0xffffffffu, incl, 1);
                if (lane == 0) excl = inf;
                const bool pub = c < fmin(best, excl);
                const unsigned mask = __ballot_sync(0xffffffffu, pub);
                const int rank = __popc(mask & ((1u << lane) - 1u));
                if (pub && cnt + rank < p.pub_cap) {
                    const int64_t at = cnt + rank;
                    p.pub_log[at * 4 + 0] = (double)(ver + rank + 1);
                    p.pub_log[at * 4 + 1] = (double)(base + w);
                    p.pub_log[at * 4 + 2] = c;
                    p.pub_log[at * 4 + 3] = ts;
                }
                if (mask) {
                    const int last = 31 - __clz(mask);
                    wr = r;
                    ww = w0 + last;
                    best = __shfl_sync(0xffffffffu, c, last);
                    ver += __popc(mask);
                    cnt += __popc(mask);
                }
            }
        }
        if (lane == 0) {
            *p.pub_count = cnt;
            if (wr >= 0) {
                const double* rec = p.recv + (int64_t)wr * L;
                *p.sh_obj = best;
                *p.sh_version = ver;
                *p.sh_worker = (int32_t)((int64_t)rec[1] + ww);
                if ((int)rec[3] != ww && p.err) *p.err = 1;
            }
            s_wr = wr;
            s_ww = ww;
        }
    }
    __syncthreads();
    if (s_wr >= 0) {
        const double* rc = p.recv + (int64_t)s_wr * L + 4 + p.Wmax;
        const int64_t kn = (int64_t)p.k * p.n;
        for (int64_t e = threadIdx.x; e < kn; e += blockDim.x) p.sh_c[e] = rc[e];
        for (int j = threadIdx.x; j < p.k; j += blockDim.x) p.sh_f[j] = (uint8_t)rc[kn + j];
    }
}

// select_best across ranks (engine.hpp:180-194: lowest objective, ties to the lowest global worker
// id; an all-infinite field is NoSolutionError): each rank packs its local select_best
// [objective, global id, C, flags]; every rank picks the same global winner and compacts its valid
// centres (engine.hpp:211-229). out: sel = {winner found ? 1 : -1, k_valid}; gobj / ggid.
__global__ void xch_pack_select_kernel(const int32_t* sel, const double* inc_obj, const double* best_c,
                                       const uint8_t* best_f, int k, int n, int base, double* rec) {
    const int b = sel[0];
    const int64_t kn = (int64_t)k * n;
    if (threadIdx.x == 0) {
        rec[0] = b >= 0 ? inc_obj[b] : __longlong_as_double(0x7ff0000000000000LL);
        rec[1] = b >= 0 ? (double)(base + b) : -1.0;
    }
    for (int64_t e = threadIdx.x; e < kn; e += blockDim.x) rec[2 + e] = b >= 0 ? best_c[e] : 0.0;
    for (int j = threadIdx.x; j < k; j += blockDim.x) rec[2 + kn + j] = b >= 0 ? (double)best_f[j] : 1.0;
}

__global__ void xch_merge_select_kernel(const double* recv, int G, int k, int n, int32_t* sel, double* best_c,
                                        uint8_t* best_f, double* cv, int32_t* remap, double* gobj, int64_t* ggid) {
    __shared__ int s_r, s_kv;
    const int64_t kn = (int64_t)k * n, L = 2 + kn + k;
    if (threadIdx.x == 0) {
        int br = -1;
        double bo = 0.0, bg = 0.0;
        for (int r = 0; r < G; ++r) {
            const double o = recv[r * L], g = recv[r * L + 1];
            if (g < 0.0 || !(o < __longlong_as_double(0x7ff0000000000000LL))) continue;
            if (br < 0 || o < bo || (o == bo && g < bg)) {
                br = r;
                bo = o;
                bg = g;
            }
        }
        int kv = 0;
        if (br >= 0)
            for (int j = 0; j < k; ++j)
                if (recv[br * L + 2 + kn + j] == 0.0) remap[kv++] = j;
        s_r = br;
        s_kv = kv;
        sel[0] = br >= 0 ? 1 : -1;
        sel[1] = kv;
        *gobj = bo;
        *ggid = (int64_t)bg;
    }
    __syncthreads();
    const int br = s_r, kv = s_kv;
    if (br < 0) return;
    const double* rc = recv + br * L + 2;
    for (int64_t e = threadIdx.x; e < kn; e += blockDim.x) best_c[e] = rc[e];
    for (int j = threadIdx.x; j < k; j += blockDim.x) best_f[j] = (uint8_t)rc[kn + j];
    for (int64_t e = threadIdx.x; e < (int64_t)kv * n; e += blockDim.x) {
        const int64_t r = e / n;
        cv[e] = rc[(int64_t)remap[r] * n + (e - r * n)];
    }
}

// Engine state of sample 0 in ONE launch (was ten memsets and two fills: ~25 us of host API time
// between a run's finish and the next run's first worker step, with the GPU idle): all-degenerate
// incumbents at +inf (engine.hpp:456), an empty shared best, cleared error / evaluation / publication
// counters and accept log.
struct EngineResetParams {
    double *inc_c, *inc_obj, *sh_obj, *sh_c;
    uint8_t *inc_f, *sh_f, *log_acc;
    int32_t *err_first, *sh_worker;
    int64_t *sh_ver, *pub_count;
    unsigned long long* nd_total;
    int64_t W, k, kn, log_bytes;
};
__global__ void engine_reset_kernel(const EngineResetParams q) {
    const int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, step = (int64_t)gridDim.x * blockDim.x;
    const double inf = __longlong_as_double(0x7ff0000000000000LL);
    for (int64_t i = i0; i < q.W * q.kn; i += step) q.inc_c[i] = 0.0;
    for (int64_t i = i0; i < q.W * q.k; i += step) q.inc_f[i] = 1;
    for (int64_t i = i0; i < q.W; i += step) {
        q.inc_obj[i] = inf;
        q.err_first[i] = 0;
    }
    for (int64_t i = i0; i < q.kn; i += step) q.sh_c[i] = 0.0;
    for (int64_t i = i0; i < q.k; i += step) q.sh_f[i] = 1;
    for (int64_t i = i0; i < q.log_bytes; i += step) q.log_acc[i] = 0;
    if (i0 == 0) {
        *q.sh_obj = inf;
        *q.sh_ver = 0;
        *q.sh_worker = -1;
        *q.nd_total = 0;
        *q.pub_count = 0;
    }
}


// The result pieces of a finish (incumbent objectives, logs, counters, the winner's centroids, f(C,X))
// packed into one device staging block, so ONE device-to-host copy carries them: eleven small copies
// cost ~5 us each on the stream after the f(C,X) pass.
struct PackSeg {
    const unsigned char* src;
    int64_t off, bytes;
};
struct PackParams {
    PackSeg seg[12];
    int n;
    unsigned char* dst;
};
__global__ void pack_segments_kernel(const PackParams q) {
    const int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, step = (int64_t)gridDim.x * blockDim.x;
    for (int sg = 0; sg < q.n; ++sg) {
        const PackSeg g = q.seg[sg];
        if (((reinterpret_cast<uintptr_t>(g.src) | (uintptr_t)g.off | (uintptr_t)g.bytes) & 7) == 0) {
            const uint64_t* s8 = reinterpret_cast<const uint64_t*>(g.src);
            uint64_t* d8 = reinterpret_cast<uint64_t*>(q.dst + g.off);
            for (int64_t i = i0; i < g.bytes / 8; i += step) d8[i] = s8[i];
        } else {
            for (int64_t i = i0; i < g.bytes; i += step) q.dst[g.off + i] = g.src[i];
        }
    }
}

// select_best (engine.hpp:180-194: strict <, worker-id order, infinite never wins) and the
// valid-subset compaction of the winner (engine.hpp:211-229) on the device, so the final
// objective launches without a host round trip. sel = {best worker or -1, valid count}.
__global__ void finish_select_kernel(const double* inc_obj, const double* inc_c, const uint8_t* inc_f, int W, int k,
                                     int n, int32_t* sel, double* best_c, uint8_t* best_f, double* cv, int32_t* remap) {
    __shared__ double so[32];
    __shared__ int si[32];
    __shared__ int s_best, s_kv;
    double bo = __longlong_as_double(0x7ff0000000000000LL);
    int bi = -1;
    for (int w = threadIdx.x; w < W; w += blockDim.x) {
        const double o = inc_obj[w];
        if (o < bo) {
            bo = o;
            bi = w;
        }
    }
    auto better = [](double o, int i, double bo_, int bi_) {
        return i >= 0 && (bi_ < 0 || o < bo_ || (o == bo_ && i < bi_));
    };
    for (int off = 16; off > 0; off >>= 1) {
        const double oo = __shfl_down_sync(0xffffffffu, bo, off);
        const int oi = __shfl_down_sync(0xffffffffu, bi, off);
        if (better(oo, oi, bo, bi)) {
            bo = oo;
            bi = oi;
        }
    }
    if ((threadIdx.x & 31) == 0) {
        so[threadIdx.x >> 5] = bo;
        si[threadIdx.x >> 5] = bi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double b = __longlong_as_double(0x7ff0000000000000LL);
        int bw = -1;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w)
            if (better(so[w], si[w], b, bw)) {
                b = so[w];
                bw = si[w];
            }
        int kv = 0;
        if (bw >= 0)
            for (int j = 0; j < k; ++j)
                if (!inc_f[(int64_t)bw * k + j]) remap[kv++] = j;
        s_best = bw;
        s_kv = kv;
        sel[0] = bw;
        sel[1] = kv;
    }
    __syncthreads();
    const int bw = s_best, kv = s_kv;
    if (bw < 0) return;
    const int64_t kn = (int64_t)k * n;
    for (int64_t e = threadIdx.x; e < kn; e += blockDim.x) best_c[e] = inc_c[bw * kn + e];
    for (int j = threadIdx.x; j < k; j += blockDim.x) best_f[j] = inc_f[(int64_t)bw * k + j];
    for (int64_t e = threadIdx.x; e < (int64_t)kv * n; e += blockDim.x) {
        const int64_t r = e / n;
        cv[e] = inc_c[bw * kn + (int64_t)remap[r] * n + (e - r * n)];
    }
}

template <typename T>
cudaError_t h2d(T* dst, const T* src, size_t count, cudaStream_t st) {
    return cudaMemcpyAsync(dst, src, count * sizeof(T), cudaMemcpyHostToDevice, st);
}
template <typename T>
cudaError_t d2h(T* dst, const T* src, size_t count, cudaStream_t st) {
    return cudaMemcpyAsync(dst, src, count * sizeof(T), cudaMemcpyDeviceToHost, st);
}

// Full-data assignment on device: valid centres C_valid_dev [kv x n], remap [kv];
// labels_dev may be null; counts_dev (u64 x k) may be null; cost to cost_dev.
int run_assign(hpcg_ctx* ctx, const hpcg_dataset* ds, const double* C_valid_dev, const int32_t* remap_dev, int kv,
               int32_t* labels_dev, unsigned long long* counts_dev, double* cost_dev, DevBuf& blocks,
               const int32_t* kv_dev = nullptr) {
    const int nb = objective_blocks();
    CU(blocks.reserve((size_t)nb * sizeof(double)));
    ObjParams op = {};
    op.kv_dev = kv_dev;
    int launched = 0;
    op.launched = &launched;
    op.fast_cost = (ds->dtype == HPCG_F32 && !ctx->fp32_exact_cost) ? 1 : 0;
    if (ds->n <= 3 && kv <= 32) {  // narrow rows: the cell filter's masks (objective_rows.cuh)
        CU(ctx->grid.reserve((size_t)kGridCells * 4 + sizeof(GridHdr)));
        op.grid = ctx->grid.as<uint32_t>();
    }
    op.rec_slot = -1;
    if (ctx->rec_slot >= 0 && ctx->rec_scratch.reserve((size_t)kRecSlotF4 * sizeof(float4)) == cudaSuccess) {
        op.rec_slot = ctx->rec_slot;
        op.rec_scratch = ctx->rec_scratch.as<float4>();
    }
    op.n = (int)ds->n;
    op.kv = kv;
    op.C = C_valid_dev;
    op.remap = remap_dev;
    op.counts = counts_dev;
    op.block_cost = blocks.as<double>();
    if (ds->nshards <= 1) {
        op.X = ds->X;
        op.m = ds->m;
        op.labels = labels_dev;
        // the tensor-core kernel's last CTA writes the total (no separate sum launch)
        if (!ctx->done_ctr.p) {
            CU(ctx->done_ctr.reserve(16));
            CU(cudaMemsetAsync(ctx->done_ctr.p, 0, 16, ctx->stream));
        }
        op.cost_out = cost_dev;
        op.done_ctr = ctx->done_ctr.as<unsigned int>();
        int fin = 0;
        op.finalized = &fin;
        int used = nb;
        KTimer kt(ctx, 1);
        CU(launch_objective(ds->dtype, op, &used, ctx->stream));
        kt.done();
        if (!fin) {
            sum_blocks_kernel<<<1, 256, 0, ctx->stream>>>(blocks.as<double>(), used, cost_dev);
            CU(cudaGetLastError());
            ctx->launches += 1;
        }
        ctx->launches += launched;
        return HPCG_OK;
    }
    // row-sharded X: one pass per shard (labels at the shard's global offset), the shard sums in
    // shard order (fixed), then their sum
    CU(blocks.reserve((size_t)(nb + kMaxShards) * sizeof(double)));
    double* shard_cost = blocks.as<double>() + nb;
    op.block_cost = blocks.as<double>();
    for (int sh = 0; sh < ds->nshards; ++sh) {
        const int64_t b0 = sh ? ds->shard_end[sh - 1] : 0;
        op.X = ds->shard_ptr[sh];
        op.m = ds->shard_end[sh] - b0;
        op.labels = labels_dev ? labels_dev + b0 : nullptr;
        int used = nb;
        CU(launch_objective(ds->dtype, op, &used, ctx->stream));
        sum_blocks_kernel<<<1, 256, 0, ctx->stream>>>(blocks.as<double>(), used, shard_cost + sh);
        CU(cudaGetLastError());
        ctx->launches += 1;
    }
    sum_blocks_kernel<<<1, 32, 0, ctx->stream>>>(shard_cost, ds->nshards, cost_dev);
    CU(cudaGetLastError());
    ctx->launches += launched + 1;
    return HPCG_OK;
}
}  // namespace

// ============================================================== C-ABI
extern "C" {

const char* hpcg_last_error(void) { return g_err.c_str(); }
int hpcg_abi_version(void) { return HPCG_ABI_VERSION; }

int hpcg_ctx_create(int device, hpcg_ctx** out) {
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0)
        return fail(HPCG_ECUDA, std::string("no CUDA device available (libhpcg has no CPU fallback): ") +
                                    cudaGetErrorString(e));
    if (device < 0 || device >= count) return fail(HPCG_EINVAL, "device index out of range");
    cudaDeviceProp prop;
    CU(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
        return fail(HPCG_ECUDA, "libhpcg is built for sm_100a (B200); device has compute capability " +
                                    std::to_string(prop.major) + "." + std::to_string(prop.minor));
    CU(cudaSetDevice(device));
    auto* c = new hpcg_ctx;
    c->device = device;
    e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        delete c;
        return fail(HPCG_ECUDA, cudaGetErrorString(e));
    }
    c->own_stream = true;
    c->rec_slot = acquire_rec_slot();
    *out = c;
    return HPCG_OK;
}

int hpcg_ctx_destroy(hpcg_ctx* ctx) {
    if (!ctx) return HPCG_OK;
    bind_device(ctx->device);
    if (ctx->rec_slot >= 0) {
        cudaDeviceSynchronize();  // no launch of this context may still read its record slot
        release_rec_slot(ctx->rec_slot);
    }
    if (ctx->comm && nccl_api().ok) nccl_api().comm_destroy(ctx->comm);
    if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
    if (ctx->spare_x) cudaFree(ctx->spare_x);
    if (ctx->pin) cudaFreeHost(ctx->pin);
    delete ctx;
    return HPCG_OK;
}

int hpcg_ctx_set_stream(hpcg_ctx* ctx, void* st) {
    std::lock_guard<std::mutex> lk(ctx->mu);
    bind_device(ctx->device);
    if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
    ctx->stream = static_cast<cudaStream_t>(st);  // NULL: legacy default stream
    ctx->own_stream = false;
    return HPCG_OK;
}

int hpcg_ctx_synchronize(hpcg_ctx* ctx) {
    bind_device(ctx->device);
    CU(cudaStreamSynchronize(ctx->stream));
    return HPCG_OK;
}

int64_t hpcg_ctx_launch_count(const hpcg_ctx* ctx) { return ctx->launches.load(); }
int64_t hpcg_ctx_upload_bytes(const hpcg_ctx* ctx) { return ctx->upload_bytes.load(); }

int hpcg_ctx_set_fp32_cost(hpcg_ctx* ctx, int exact) {
    std::lock_guard<std::mutex> lk(ctx->mu);
    ctx->fp32_exact_cost = exact ? 1 : 0;
    return HPCG_OK;
}

int hpcg_ctx_enable_timing(hpcg_ctx* ctx, int enable) {
    std::lock_guard<std::mutex> lk(ctx->mu);
    ctx->timing = enable != 0;
    return HPCG_OK;
}

int hpcg_ctx_kernel_times(hpcg_ctx* ctx, int64_t* counts, double* total_ms) {
    std::lock_guard<std::mutex> lk(ctx->mu);
    bind_device(ctx->device);
    for (int c = 0; c < 2; ++c) {
        for (auto& ev : ctx->pending[c]) {
            float ms = 0.f;
            CU(cudaEventSynchronize(ev.second));
            CU(cudaEventElapsedTime(&ms, ev.first, ev.second));
            ctx->t_ms[c] += ms;
            ctx->t_count[c] += 1;
            cudaEventDestroy(ev.first);
            cudaEventDestroy(ev.second);
        }
        ctx->pending[c].clear();
        if (counts) counts[c] = ctx->t_count[c];
        if (total_ms) total_ms[c] = ctx->t_ms[c];
    }
    return HPCG_OK;
}

int hpcg_probe_fma_peak(hpcg_ctx* ctx, double* tfma) {
    std::lock_guard<std::mutex> lk(ctx->mu);
    bind_device(ctx->device);
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
    DevBuf out;
    CU(out.reserve(64));
    const int blocks = sms * 8, threads = 256, iters = 8192;
    cudaEvent_t a, b;
    CU(cudaEventCreate(&a));
    CU(cudaEventCreate(&b));
    fma_probe_kernel<<<blocks, threads, 0, ctx->stream>>>(out.as<float>(), 1.0001f, 0.5f, iters);  // warm-up
    CU(cudaEventRecord(a, ctx->stream));
    for (int r = 0; r < 5; ++r) fma_probe_kernel<<<blocks, threads, 0, ctx->stream>>>(out.as<float>(), 1.0001f, 0.5f, iters);
    CU(cudaEventRecord(b, ctx->stream));
    CU(cudaEventSynchronize(b));
    float ms = 0.f;
    CU(cudaEventElapsedTime(&ms, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    ctx->launches += 6;
    const double fmas = 5.0 * blocks * threads * (double)iters * 8 * 2;
    *tfma = fmas / (ms * 1e-3) / 1e12;
    return HPCG_OK;
}

// ------------------------------------------------------------------ datasets
int hpcg_host_register(void* host, int64_t bytes) {
    if (!host || bytes < 1) return fail(HPCG_EINVAL, "host_register: empty range");
    cudaError_t e = cudaHostRegister(host, (size_t)bytes, cudaHostRegisterPortable);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(HPCG_ECUDA, cudaGetErrorString(e));
    }
    return HPCG_OK;
}

int hpcg_host_unregister(void* host) {
    if (!host) return fail(HPCG_EINVAL, "host_unregister: null pointer");
    cudaError_t e = cudaHostUnregister(host);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(HPCG_ECUDA, cudaGetErrorString(e));
    }
    return HPCG_OK;
}

static int dataset_upload(hpcg_ctx* ctx, const void* X_host, hpcg_dtype dtype, int64_t m, int64_t n, hpcg_dataset** out,
                          bool wait);
int hpcg_dataset_upload(hpcg_ctx* ctx, const void* X_host, hpcg_dtype dtype, int64_t m, int64_t n,
                        hpcg_dataset** out) {
    return dataset_upload(ctx, X_host, dtype, m, n, out, true);
}
// wait = false (hpcg_run): the copy stays in flight on the context's stream and everything the run
// enqueues is ordered behind it, so the engine's allocations and the first launches' host work
// overlap the transfer; the caller synchronises before X_host may change (the run's finish does)
static int dataset_upload(hpcg_ctx* ctx, const void* X_host, hpcg_dtype dtype, int64_t m, int64_t n, hpcg_dataset** out,
                          bool wait) {
    if (m < 1 || n < 1) return fail(HPCG_EINVAL, "Dataset: needs at least one row and one column");
    if (dtype != HPCG_F32 && dtype != HPCG_F64) return fail(HPCG_EINVAL, "unknown dtype");
    bind_device(ctx->device);
    void* d = nullptr;
    const size_t bytes = (size_t)m * (size_t)n * dsize(dtype);
    size_t have = 0;
    {
        std::lock_guard<std::mutex> lk(ctx->cache_mu);
        if (ctx->spare_x && ctx->spare_x_bytes >= bytes) {  // reuse the last freed upload buffer
            d = ctx->spare_x;
            have = ctx->spare_x_bytes;
            ctx->spare_x = nullptr;
            ctx->spare_x_bytes = 0;
        }
    }
    if (!d) {
        CU(cudaMalloc(&d, bytes));
        have = bytes;
    }
    cudaError_t e = cudaMemcpyAsync(d, X_host, bytes, cudaMemcpyHostToDevice, ctx->stream);
    ctx->upload_bytes += (int64_t)bytes;
    if (e == cudaSuccess && wait) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) {
        cudaFree(d);
        return fail(HPCG_ECUDA, cudaGetErrorString(e));
    }
    auto* ds = new hpcg_dataset;
    ds->ctx = ctx;
    ds->X = d;
    ds->shard_ptr[0] = d;
    ds->shard_end[0] = m;
    ds->owned = true;
    ds->bytes = have;
    ds->dtype = dtype;
    ds->m = m;
    ds->n = n;
    *out = ds;
    return HPCG_OK;
}

int hpcg_dataset_wrap(hpcg_ctx* ctx, const void* X_dev, hpcg_dtype dtype, int64_t m, int64_t n, hpcg_dataset** out) {
    if (m < 1 || n < 1) return fail(HPCG_EINVAL, "Dataset: needs at least one row and one column");
    if (dtype != HPCG_F32 && dtype != HPCG_F64) return fail(HPCG_EINVAL, "unknown dtype");
    auto* ds = new hpcg_dataset;
    ds->ctx = ctx;
    ds->X = X_dev;
    ds->shard_ptr[0] = X_dev;
    ds->shard_end[0] = m;
    ds->owned = false;
    ds->dtype = dtype;
    ds->m = m;
    ds->n = n;
    *out = ds;
    return HPCG_OK;
}

int hpcg_dataset_wrap_sharded(hpcg_ctx* ctx, const void* const* shard_dev, const int64_t* shard_rows, int32_t nshards,
                              hpcg_dtype dtype, int64_t n, hpcg_dataset** out) {
    if (nshards < 1 || nshards > kMaxShards) return fail(HPCG_EINVAL, "Dataset: 1 to 8 row shards");
    if (n < 1) return fail(HPCG_EINVAL, "Dataset: needs at least one row and one column");
    if (dtype != HPCG_F32 && dtype != HPCG_F64) return fail(HPCG_EINVAL, "unknown dtype");
    int64_t m = 0;
    for (int i = 0; i < nshards; ++i) {
        if (shard_rows[i] < 1 || !shard_dev[i]) return fail(HPCG_EINVAL, "Dataset: empty shard");
        m += shard_rows[i];
    }
    // shards resident on other devices of this process: the gathers read them over NVLink (peer
    // access; IPC-opened shards of other processes are already mapped)
    bind_device(ctx->device);
    for (int i = 0; i < nshards; ++i) {
        cudaPointerAttributes at{};
        if (cudaPointerGetAttributes(&at, shard_dev[i]) != cudaSuccess) {
            cudaGetLastError();
            continue;
        }
        if (at.type == cudaMemoryTypeDevice && at.device != ctx->device) {
            const cudaError_t pe = cudaDeviceEnablePeerAccess(at.device, 0);
            if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled)
                return fail(HPCG_ECUDA, std::string("peer access to a shard's device: ") + cudaGetErrorString(pe));
            cudaGetLastError();
        }
    }
    auto* ds = new hpcg_dataset;
    ds->ctx = ctx;
    ds->X = shard_dev[0];
    ds->nshards = nshards;
    int64_t end = 0;
    for (int i = 0; i < nshards; ++i) {
        end += shard_rows[i];
        ds->shard_ptr[i] = shard_dev[i];
        ds->shard_end[i] = end;
    }
    ds->owned = false;
    ds->dtype = dtype;
    ds->m = m;
    ds->n = n;
    *out = ds;
    return HPCG_OK;
}

// the IPC handle names the whole allocation: the pointer's offset inside it travels along
// (allocators such as torch's sub-allocate), found with the driver's cuMemGetAddressRange
int hpcg_ipc_export(const void* dev_ptr, void* handle_out) {
    using RangeFn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
    static RangeFn range = nullptr;
    if (!range) {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return fail(HPCG_ECUDA, "ipc: cuMemGetAddressRange unavailable");
        range = reinterpret_cast<RangeFn>(f);
    }
    CUdeviceptr base = 0;
    size_t size = 0;
    if (range(&base, &size, reinterpret_cast<CUdeviceptr>(dev_ptr)) != CUDA_SUCCESS)
        return fail(HPCG_EINVAL, "ipc: not a device allocation");
    cudaIpcMemHandle_t h;
    CU(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
    const uint64_t off = (uint64_t)(reinterpret_cast<CUdeviceptr>(dev_ptr) - base);
    std::memcpy(handle_out, &h, sizeof h);
    std::memcpy(static_cast<char*>(handle_out) + sizeof h, &off, 8);
    return HPCG_OK;
}

int hpcg_ipc_open(hpcg_ctx* ctx, const void* handle, void** dev_ptr_out) {
    bind_device(ctx->device);
    cudaIpcMemHandle_t h;
    uint64_t off = 0;
    std::memcpy(&h, handle, sizeof h);
    std::memcpy(&off, static_cast<const char*>(handle) + sizeof h, 8);
    void* base = nullptr;
    CU(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
    *dev_ptr_out = static_cast<char*>(base) + off;
    return HPCG_OK;
}

int hpcg_ipc_close(hpcg_ctx* ctx, void* dev_ptr, const void* handle) {
    bind_device(ctx->device);
    uint64_t off = 0;
    std::memcpy(&off, static_cast<const char*>(handle) + sizeof(cudaIpcMemHandle_t), 8);
    CU(cudaIpcCloseMemHandle(static_cast<char*>(dev_ptr) - off));
    return HPCG_OK;
}

int hpcg_dataset_destroy(hpcg_dataset* ds) {
    if (ds) {
        cudaSetDevice(ds->ctx->device);
        delete ds;
    }
    return HPCG_OK;
}

const void* hpcg_dataset_device_ptr(const hpcg_dataset* ds) { return ds->X; }

// ---------------------------------------------------------- full assignment
int hpcg_assign(hpcg_ctx* ctx, const hpcg_dataset* ds, const double* C_host, const uint8_t* deg, int64_t k,
                int require_valid, int32_t* labels_host, int64_t* counts_host, double* cost, int64_t* n_d) {
    std::lock_guard<std::mutex> lk(ctx->mu);
    bind_device(ctx->device);
    if (k < 1) return fail(HPCG_EINVAL, "assign: need at least one centroid");
    const int64_t n = ds->n;
    std::vector<double> cv;
    std::vector<int32_t> remap;
    for (int64_t j = 0; j < k; ++j) {
        if (deg && deg[j]) {
            if (require_valid) return fail(HPCG_EINVAL, "assign: degenerate centroid present");
            continue;
        }
        remap.push_back((int32_t)j);
        cv.insert(cv.end(), C_host + j * n, C_host + (j + 1) * n);
    }
    if (remap.empty()) return fail(HPCG_EINVAL, "assignment: every centroid is degenerate");
    const int kv = (int)remap.size();
    if (int rc = check_shape(ds->dtype, n, kv)) return rc;
    CU(ctx->s_a.reserve(cv.size() * 8));
    CU(ctx->s_b.reserve(remap.size() * 4 + 16));
    CU(ctx->s_c.reserve(8));
    CU(h2d(ctx->s_a.as<double>(), cv.data(), cv.size(), ctx->stream));
    CU(h2d(ctx->s_b.as<int32_t>(), remap.data(), remap.size(), ctx->stream));
    int32_t* lab_dev = nullptr;
    unsigned long long* cnt_dev = nullptr;
    if (labels_host) {
        CU(ctx->s_d.reserve((size_t)ds->m * 4));
        lab_dev = ctx->s_d.as<int32_t>();
    }
    if (counts_host) {
        CU(ctx->s_e.reserve((size_t)k * 8));
        cnt_dev = ctx->s_e.as<unsigned long long>();
        CU(cudaMemsetAsync(cnt_dev, 0, (size_t)k * 8, ctx->stream));
    }
    int rc = run_assign(ctx, ds, ctx->s_a.as<double>(), ctx->s_b.as<int32_t>(), kv, lab_dev, cnt_dev,
                        ctx->s_c.as<double>(), ctx->s_f);
    if (rc) return rc;
    double c = 0;
    CU(d2h(&c, ctx->s_c.as<double>(), 1, ctx->stream));
    if (labels_host) CU(d2h(labels_host, lab_dev, (size_t)ds->m, ctx->stream));
    std::vector<unsigned long long> cnt(counts_host ? (size_t)k : 0);
    if (counts_host) CU(d2h(cnt.data(), cnt_dev, (size_t)k, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    if (counts_host)
        for (int64_t j = 0; j < k; ++j) counts_host[j] = (int64_t)cnt[j];
    if (cost) *cost = c;
    if (n_d) *n_d = ds->m * kv;
    return HPCG_OK;
}

int hpcg_assign_dev(hpcg_ctx* ctx, const hpcg_dataset* ds, const double* C_dev, int64_t k_valid,
                    int32_t* labels_dev, double* cost_dev) {
    std::lock_guard<std::mutex> lk(ctx->mu);
    bind_device(ctx->device);
    if (k_valid < 1) return fail(HPCG_EINVAL, "assign: need at least one centroid");
    if (int rc = check_shape(ds->dtype, ds->n, k_valid)) return rc;
    if (ctx->s_b.bytes < (size_t)k_valid * 4) {
        std::vector<int32_t> remap((size_t)k_valid);
        for (int64_t j = 0; j < k_valid; ++j) remap[(size_t)j] = (int32_t)j;
        CU(ctx->s_b.reserve(remap.size() * 4));
        CU(h2d(ctx->s_b.as<int32_t>(), remap.data(), remap.size(), ctx->stream));
    } else {
        // identity remap kept in s_b by construction of this path
        std::vector<int32_t> remap((size_t)k_valid);
        for (int64_t j = 0; j < k_valid; ++j) remap[(size_t)j] = (int32_t)j;
        CU(h2d(ctx->s_b.as<int32_t>(), remap.data(), remap.size(), ctx->stream));
    }
    return run_assign(ctx, ds, C_dev, ctx->s_b.as<int32_t>(), (int)k_valid, labels_dev, nullptr, cost_dev,
                      ctx->s_f);
}

// ---------------------------------------------------------------- gather
int hpcg_gather(hpcg_ctx* ctx, const hpcg_dataset* ds, const int64_t* idx_host, int64_t s, void* S_host) {
    std::lock_guard<std::mutex> lk(ctx->mu);
    bind_device(ctx->device);
    if (s < 1 || s > ds->m) return fail(HPCG_EINVAL, "draw_sample: sample size must be in [1, m]");
    for (int64_t i = 0; i < s; ++i)
        if (idx_host[i] < 0 || idx_host[i] >= ds->m) return fail(HPCG_EINVAL, "gather: row index out of range");
    const int64_t rowb = ds->n * (int64_t)dsize(ds->dtype);
    CU(ctx->s_a.reserve((size_t)s * 8));
    CU(ctx->s_b.reserve((size_t)(s * rowb)));
    CU(h2d(ctx->s_a.as<int64_t>(), idx_host, (size_t)s, ctx->stream));
    const int64_t tot = s * rowb;
    ShardTable tab;
    tab.n = ds->nshards;
    for (int i = 0; i < ds->nshards; ++i) {
        tab.ptr[i] = static_cast<const unsigned char*>(ds->shard_ptr[i]);
        tab.end[i] = ds->shard_end[i];
    }
    gather_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, ctx->stream>>>(tab, rowb, ctx->s_a.as<int64_t>(), s,
                                                                        ctx->s_b.as<unsigned char>());
    CU(cudaGetLastError());
    ctx->launches += 1;
    CU(cudaMemcpyAsync(S_host, ctx->s_b.p, (size_t)tot, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    return HPCG_OK;
}

// the device sample definition of RngMode::philox (SamplePRP), for tests and reproduction
__global__ void sample_prp_kernel(uint64_t m, uint32_t a, uint32_t b, float inv_b, uint64_t key, uint32_t round,
                                  uint32_t worker, int64_t s, int64_t* out) {
    const SamplePRP prp = SamplePRP::make(key, round, worker, m, a, b, inv_b);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < s; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (int64_t)prp((uint64_t)i);
}

int hpcg_sample_indices(hpcg_ctx* ctx, int64_t m, int64_t s, uint64_t key, uint32_t round, uint32_t worker,
                        int64_t* idx_out) {
    if (!ctx || !idx_out) return fail(HPCG_EINVAL, "sample_indices: null argument");
    if (s < 1 || s > m) return fail(HPCG_EINVAL, "draw_sample: sample size must be in [1, m]");
    std::lock_guard<std::mutex> lk(ctx->mu);
    bind_device(ctx->device);
    uint32_t a, b;
    float inv_b;
    SamplePRP::moduli((uint64_t)m, a, b, inv_b);
    CU(ctx->s_a.reserve((size_t)s * 8));
    const unsigned grid = (unsigned)std::min<int64_t>((s + 255) / 256, 4096);
    sample_prp_kernel<<<grid, 256, 0, ctx->stream>>>((uint64_t)m, a, b, inv_b, key, round, worker, s,
                                                     ctx->s_a.as<int64_t>());
    CU(cudaGetLastError());
    ctx->launches += 1;
    CU(cudaMemcpyAsync(idx_out, ctx->s_a.p, (size_t)s * 8, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    return HPCG_OK;
}

int hpcg_sample_gather_dev(hpcg_ctx* ctx, const hpcg_dataset* ds, int64_t W, int64_t s, uint64_t key,
                           uint32_t round, int32_t worker_base, void* S_dev) {
    if (!ctx || !ds || !S_dev) return fail(HPCG_EINVAL, "sample_gather: null argument");
    if (s < 1 || s > ds->m) return fail(HPCG_EINVAL, "draw_sample: sample size must be in [1, m]");
    if (W < 1 || W > 65535) return fail(HPCG_EINVAL, "sample_gather: worker count must be in [1, 65535]");
    std::lock_guard<std::mutex> lk(ctx->mu);
    bind_device(ctx->device);
    ShardTable t;
    t.n = ds->nshards;
    for (int i = 0; i < ds->nshards; ++i) {
        t.ptr[i] = static_cast<const unsigned char*>(ds->shard_ptr[i]);
        t.end[i] = ds->shard_end[i];
    }
    uint32_t a, b;
    float inv_b;
    SamplePRP::moduli((uint64_t)ds->m, a, b, inv_b);
    const int64_t rowb = ds->n * (int64_t)dsize(ds->dtype);
    const dim3 grid((unsigned)((s + 255) / 256), (unsigned)W);
    unsigned char* S = static_cast<unsigned char*>(S_dev);
    if (rowb % 16 == 0)
        sample_gather_kernel<16><<<grid, 256, 0, ctx->stream>>>(t, ds->m, rowb, s, key, round, worker_base, a, b, inv_b, S);
    else if (rowb % 8 == 0)
        sample_gather_kernel<8><<<grid, 256, 0, ctx->stream>>>(t, ds->m, rowb, s, key, round, worker_base, a, b, inv_b, S);
    else
        sample_gather_kernel<4><<<grid, 256, 0, ctx->stream>>>(t, ds->m, rowb, s, key, round, worker_base, a, b, inv_b, S);
    CU(cudaGetLastError());
    ctx->launches += 1;
    return HPCG_OK;
}

int hpcg_philox_seed_draws(uint64_t key, uint32_t round, uint32_t worker, int64_t s, int32_t no_valid,
                           int64_t loops, int64_t candidates, int64_t* first_row, double* units) {
    if (candidates < 1 || candidates > kMaxCandidates) return fail(HPCG_EINVAL, "seeding: candidates out of range");
    if (first_row) *first_row = no_valid ? (int64_t)philox_index(key, round, worker, 0xF1F1u, (uint64_t)s) : 0;
    if (units)
        for (int64_t t = 0; t < loops; ++t)
            for (int64_t c = 0; c < candidates; ++c)  // pending-slot index p = t + no_valid (step_kernel.cuh)
                units[t * candidates + c] = philox_unit(
                    key, round, worker, (uint32_t)(0x10000 + (t + (no_valid ? 1 : 0)) * kMaxCandidates + c));
    return HPCG_OK;
}

int hpcg_reference_draw_indices(uint64_t* mt_state, int32_t* mt_pos, int64_t m, int64_t s, int64_t* idx_out) {
    if (s < 1 || s > m) return fail(HPCG_EINVAL, "draw_sample: sample size must be in [1, m]");
    Mt64 r;
    std::memcpy(r.mt, mt_state, sizeof r.mt);
    r.pos = *mt_pos;
    sparse_fisher_yates(r, m, s, idx_out);
    std::memcpy(mt_state, r.mt, sizeof r.mt);
    *mt_pos = r.pos;
    return HPCG_OK;
}

// ------------------------------------------------------- reference streams
int hpcg_rng_seed(uint64_t seed, uint64_t* st, int32_t* pos) {
    Mt64 r;
    r.seed(seed);
    std::memcpy(st, r.mt, sizeof r.mt);
    *pos = r.pos;
    return HPCG_OK;
}

int hpcg_rng_derive(uint64_t master, uint64_t domain, uint64_t index, uint64_t* st, int32_t* pos) {
    Mt64 r = Mt64::derive(master, domain, index);
    std::memcpy(st, r.mt, sizeof r.mt);
    *pos = r.pos;
    return HPCG_OK;
}

int hpcg_rng_draw(uint64_t* st, int32_t* pos, int32_t kind, uint64_t bound, int64_t count, void* out) {
    if (kind == 2 && bound == 0) return fail(HPCG_EINVAL, "uniform_index: n must be positive");
    Mt64 r;
    std::memcpy(r.mt, st, sizeof r.mt);
    r.pos = *pos;
    for (int64_t i = 0; i < count; ++i) {
        if (kind == 0)
            static_cast<uint64_t*>(out)[i] = r.next();
        else if (kind == 1)
            static_cast<double*>(out)[i] = r.unit();
        else
            static_cast<uint64_t*>(out)[i] = r.uniform_index(bound);
    }
    std::memcpy(st, r.mt, sizeof r.mt);
    *pos = r.pos;
    return HPCG_OK;
}

// ------------------------------------------------- batched worker step
int hpcg_worker_step_batched(hpcg_ctx* ctx, const hpcg_dataset* ds, const int64_t* idx_host, int64_t W, int64_t s,
                             const double* C_init, const uint8_t* flags_init, int64_t k, const hpcg_lloyd_cfg* cfg,
                             const int64_t* first_row_host, const double* units_host, int64_t units_stride,
                             int do_lloyd, double* C_out, uint8_t* flags_out, double* objective, int32_t* iterations,
                             int32_t* stop, int64_t* n_d, int32_t* filled, int32_t* labels, int64_t* counts,
                             double* history, int32_t hist_cap, int32_t* hist_len) {
    std::lock_guard<std::mutex> lk(ctx->mu);
    bind_device(ctx->device);
    const int64_t n = ds->n;
    if (W < 1) return fail(HPCG_EINVAL, "worker_step: need at least one worker");
    if (s < 1) return fail(HPCG_EINVAL, "seeding: empty sample");
    if (k < 1) return fail(HPCG_EINVAL, "kmeanspp_seed: k must be positive");
    if (cfg->candidates < 1) return fail(HPCG_EINVAL, "seeding: need at least one candidate");
    if (do_lloyd) {
        if (cfg->max_iters < 1) return fail(HPCG_EINVAL, "kmeans: max_iters must be positive");
        if (!(cfg->rel_tol > 0.0)) return fail(HPCG_EINVAL, "kmeans: rel_tol must be positive");
    }
    if (int rc = check_shape(ds->dtype, n, k)) return rc;
    if (cfg->candidates > kMaxCandidates) return fail(HPCG_EUNSUPPORTED, "more than 4 K-means++ candidates per centre");
    if (idx_host) {
        for (int64_t i = 0; i < W * s; ++i)
            if (idx_host[i] < 0 || idx_host[i] >= ds->m) return fail(HPCG_EINVAL, "sample index out of range");
    } else if (ds->m != W * s) {
        return fail(HPCG_EINVAL, "batched samples: dataset must hold W*s rows");
    }
    const bool explicit_draws = first_row_host != nullptr && units_host != nullptr;
    if (explicit_draws)
        for (int64_t w = 0; w < W; ++w)
            if (first_row_host[w] < 0 || first_row_host[w] >= s) return fail(HPCG_EINVAL, "first_row out of range");

    // device buffers (one allocation per call; this path serves tests and the drop-in API)
    DevBuf d_idx, d_ci, d_fi, d_fr, d_un, d_c, d_f, d_obj, d_it, d_st, d_nd, d_fl, d_err, d_lab, d_cnt, d_hist,
        d_hl;
    const int64_t kn = k * n;
    if (idx_host) CU(d_idx.reserve((size_t)(W * s) * 8));
    CU(d_ci.reserve((size_t)(W * kn) * 8));
    CU(d_fi.reserve((size_t)(W * k)));
    CU(d_c.reserve((size_t)(W * kn) * 8));
    CU(d_f.reserve((size_t)(W * k)));
    CU(d_obj.reserve((size_t)W * 8));
    CU(d_it.reserve((size_t)W * 4));
    CU(d_st.reserve((size_t)W * 4));
    CU(d_nd.reserve((size_t)W * 8));
    CU(d_fl.reserve((size_t)W * 4));
    CU(d_err.reserve((size_t)W * 4));
    if (idx_host) CU(h2d(d_idx.as<int64_t>(), idx_host, (size_t)(W * s), ctx->stream));
    CU(h2d(d_ci.as<double>(), C_init, (size_t)(W * kn), ctx->stream));
    if (flags_init)
        CU(h2d(d_fi.as<uint8_t>(), flags_init, (size_t)(W * k), ctx->stream));
    else
        CU(cudaMemsetAsync(d_fi.p, 0, (size_t)(W * k), ctx->stream));
    if (explicit_draws) {
        CU(d_fr.reserve((size_t)W * 8));
        CU(d_un.reserve((size_t)(W * std::max<int64_t>(units_stride, 1)) * 8));
        CU(h2d(d_fr.as<int64_t>(), first_row_host, (size_t)W, ctx->stream));
        if (units_stride > 0) CU(h2d(d_un.as<double>(), units_host, (size_t)(W * units_stride), ctx->stream));
    }
    if (labels) CU(d_lab.reserve((size_t)(W * s) * 4));
    if (counts) CU(d_cnt.reserve((size_t)(W * k) * 8));
    if (history && hist_cap > 0) CU(d_hist.reserve((size_t)(W * hist_cap) * 8));
    CU(d_hl.reserve((size_t)W * 4));

    StepParams p = {};
    p.X = ds->X;
    set_shards(p, ds);
    p.m = ds->m;
    SamplePRP::moduli((uint64_t)p.m, p.prp_a, p.prp_b, p.prp_inv_b);
    p.n = (int)n;
    p.s = s;
    p.W = (int)W;
    p.sample_mode = idx_host ? 0 : 2;
    p.idx = d_idx.as<int64_t>();
    p.key = 0x6870636c75737431ULL;
    p.round = 0;
    p.worker_base = 0;
    p.init_c = d_ci.as<double>();
    p.init_stride = kn;
    p.init_f = d_fi.as<uint8_t>();
    p.initf_stride = k;
    p.shared_version = nullptr;
    p.candidates = (int)cfg->candidates;
    p.seed_mode = explicit_draws ? 0 : 1;
    p.first_row = d_fr.as<int64_t>();
    p.units = d_un.as<double>();
    p.units_stride = (int)units_stride;
    p.k = (int)k;
    p.max_iters = (int)std::min<int64_t>(cfg->max_iters, INT32_MAX);
    p.rel_tol = cfg->rel_tol;
    p.do_lloyd = do_lloyd;
    p.out_c = d_c.as<double>();
    p.out_f = d_f.as<uint8_t>();
    p.out_obj = d_obj.as<double>();
    p.out_iters = d_it.as<int32_t>();
    p.out_stop = d_st.as<int32_t>();
    p.out_nd = d_nd.as<int64_t>();
    p.out_filled = d_fl.as<int32_t>();
    p.out_err = d_err.as<int32_t>();
    p.out_labels = labels ? d_lab.as<int32_t>() : nullptr;
    p.out_counts = counts ? d_cnt.as<int64_t>() : nullptr;
    p.out_hist = (history && hist_cap > 0) ? d_hist.as<double>() : nullptr;
    p.hist_cap = hist_cap;
    p.out_hist_len = d_hl.as<int32_t>();
    std::string why;
    KTimer kt(ctx, 0);
    cudaError_t e = launch_step(ds->dtype, p, ctx->stream, nullptr, &why);
    kt.done();
    if (e != cudaSuccess) return fail(HPCG_ECUDA, std::string("worker step launch: ") + cudaGetErrorString(e) + " " + why);
    ctx->launches += 1;
    std::vector<int32_t> err((size_t)W);
    CU(d2h(err.data(), d_err.as<int32_t>(), (size_t)W, ctx->stream));
    if (C_out) CU(d2h(C_out, d_c.as<double>(), (size_t)(W * kn), ctx->stream));
    if (flags_out) CU(d2h(flags_out, d_f.as<uint8_t>(), (size_t)(W * k), ctx->stream));
    if (objective) CU(d2h(objective, d_obj.as<double>(), (size_t)W, ctx->stream));
    if (iterations) CU(d2h(iterations, d_it.as<int32_t>(), (size_t)W, ctx->stream));
    if (stop) CU(d2h(stop, d_st.as<int32_t>(), (size_t)W, ctx->stream));
    if (n_d) CU(d2h(n_d, d_nd.as<int64_t>(), (size_t)W, ctx->stream));
    if (filled) CU(d2h(filled, d_fl.as<int32_t>(), (size_t)W, ctx->stream));
    if (labels) CU(d2h(labels, d_lab.as<int32_t>(), (size_t)(W * s), ctx->stream));
    if (counts) CU(d2h(counts, d_cnt.as<int64_t>(), (size_t)(W * k), ctx->stream));
    if (history && hist_cap > 0) CU(d2h(history, d_hist.as<double>(), (size_t)(W * hist_cap), ctx->stream));
    if (hist_len) CU(d2h(hist_len, d_hl.as<int32_t>(), (size_t)W, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    for (int64_t w = 0; w < W; ++w) {
        if (err[(size_t)w] == kErrDegenerateInit) return fail(HPCG_EINVAL, "kmeans: degenerate centroid in init");
        if (err[(size_t)w] == kErrMonotone) return fail(HPCG_ELOGIC, "kmeans: objective increased between iterations");
    }
    return HPCG_OK;
}

}  // extern "C"

// ============================================================== engine
struct hpcg_engine {
    hpcg_ctx* ctx = nullptr;
    const hpcg_dataset* ds = nullptr;
    int device = 0;  // the context's device (destroy must not read a context freed before it)
    hpcg_engine_cfg cfg{};
    int64_t W = 0, k = 0, n = 0, s = 0, R = 0;
    int64_t round = 0;
    uint64_t key = 0;
    std::chrono::steady_clock::time_point t0;
    bool wall = false;           // wall-clock schedule (cfg.time_limit > 0)
    std::vector<double> t_end;   // wall clock: seconds since t0 at the end of each round
    double elapsed() const { return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(); }
    DevBuf inc_c, inc_f, inc_obj, acc, nd, err, err_first, iters, stopb, filled, objb;
    DevBuf sh_ver, sh_obj, sh_worker, sh_c, sh_f;
    DevBuf log_acc, log_obj, nd_total, pub_log, pub_count;
    DevBuf d_idx, d_fr, d_un, scratch_a, scratch_b, scratch_c, blocks, fin, fin_stage;
    int64_t pub_cap = 0;   // publication-log entries allocated (grown on demand)
    int64_t pub_ub = 0;    // upper bound of the entries written so far (<= W per publishing launch)
    int64_t log_rounds = 0;  // rounds the per-round accept/objective logs can hold (grown on demand)
    bool entered_coop = false;  // wall clock, hybrid: the phase-1 incumbents were carried over
    // multi-rank exchange (hpcg_engine_set_exchange): nranks, this rank, the collective, the
    // workers of every rank (global ids contiguous in rank order) and the exchange buffers
    int xr = 1, xrank = 0;
    hpcg_allgather_fn xfn = nullptr;
    void* xuser = nullptr;
    int64_t xWmax = 0, xWtot = 0;
    DevBuf xsend, xrecv, xerr;
    std::vector<unsigned char> xhost;  // host staging of a caller collective
    double common_now = 0.0;           // wall clock, multi-rank: the latest clock of the last exchange
    // reference-RNG replay state
    std::vector<Mt64> streams;
    std::vector<int64_t> h_idx, h_fr;
    std::vector<double> h_un;
    int64_t ucap = 0;
    int64_t* trace_buf = nullptr;  // optional phase timeline (hpcg_engine_set_trace)
    int32_t trace_mode = 0;
    // free-running schedule (cfg.free_running): per-worker progress, init snapshots and traces
    bool free_mode = false;
    int64_t fr_cap = 0;  // trace entries kept per worker
    DevBuf fr_t0, fr_go, fr_coop, fr_entered, fr_samples, fr_tw, fr_init_c, fr_init_f, fr_tcnt, fr_trace, fr_lock;
};

namespace {
bool phase_cooperative(int strategy, double t1, double progress) {  // engine.hpp:288-296
    if (strategy == HPCG_COOPERATIVE) return true;
    if (strategy == HPCG_HYBRID) return progress >= t1;
    return false;
}

// Room for one more round in the logs and for `extra` more publications (doubling growth; the
// device copies are stream-ordered, so nothing is read back).
int engine_reserve(hpcg_engine* e, int64_t extra_pubs) {
    hpcg_ctx* ctx = e->ctx;
    const int64_t W = e->W;
    if (e->round >= e->log_rounds) {
        const int64_t nr = std::max<int64_t>(2 * e->log_rounds, e->round + 1);
        CU(e->log_acc.grow((size_t)(nr * W), (size_t)(e->log_rounds * W), ctx->stream));
        CU(e->log_obj.grow((size_t)(nr * W * 8), (size_t)(e->log_rounds * W * 8), ctx->stream));
        e->log_rounds = nr;
    }
    if (e->pub_ub + extra_pubs > e->pub_cap) {
        const int64_t nc = std::max<int64_t>(2 * e->pub_cap, e->pub_ub + extra_pubs);
        CU(e->pub_log.grow((size_t)(nc * 4 * 8), (size_t)(e->pub_cap * 4 * 8), ctx->stream));
        e->pub_cap = nc;
    }
    return HPCG_OK;
}

RoundEndParams round_end_params(hpcg_engine* e) {
    RoundEndParams q = {};
    q.W = (int)e->W;
    q.k = (int)e->k;
    q.n = (int)e->n;
    q.round = e->round;
    q.log = 1;
    q.worker_base = e->cfg.worker_base;
    q.accepted = e->acc.as<uint8_t>();
    q.inc_obj = e->inc_obj.as<double>();
    q.inc_c = e->inc_c.as<double>();
    q.inc_f = e->inc_f.as<uint8_t>();
    q.nd = e->nd.as<int64_t>();
    q.err = e->err.as<int32_t>();
    q.log_acc = e->log_acc.as<uint8_t>();
    q.log_obj = e->log_obj.as<double>();
    q.err_first = e->err_first.as<int32_t>();
    q.nd_total = e->nd_total.as<unsigned long long>();
    q.sh_version = e->sh_ver.as<int64_t>();
    q.sh_obj = e->sh_obj.as<double>();
    q.sh_worker = e->sh_worker.as<int32_t>();
    q.sh_c = e->sh_c.as<double>();
    q.sh_f = e->sh_f.as<uint8_t>();
    q.pub_log = e->pub_log.as<double>();
    q.pub_count = e->pub_count.as<int64_t>();
    q.pub_cap = e->pub_cap;
    return q;
}

int launch_round_end(hpcg_engine* e, const RoundEndParams& q) {
    const size_t rs_bytes = (size_t)e->W * 9;
    if (rs_bytes > 48 * 1024) {
        const cudaError_t ae = cudaFuncSetAttribute(round_end_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                    (int)rs_bytes);
        if (ae != cudaSuccess) return fail(HPCG_EUNSUPPORTED, "round end: too many workers for one engine");
    }
    round_end_kernel<<<1, 256, rs_bytes, e->ctx->stream>>>(q);
    CU(cudaGetLastError());
    e->ctx->launches += 1;
    return HPCG_OK;
}

// all-gather of `bytes` per rank from e->xsend into e->xrecv (rank order): NCCL on the context's
// stream, or the caller's host collective (staged through host memory)
int engine_allgather(hpcg_engine* e, size_t bytes) {
    hpcg_ctx* ctx = e->ctx;
    if (e->xfn) {
        e->xhost.resize(bytes * (size_t)(e->xr + 1));
        unsigned char* hs = e->xhost.data();
        unsigned char* hr = hs + bytes;
        CU(cudaMemcpyAsync(hs, e->xsend.p, bytes, cudaMemcpyDeviceToHost, ctx->stream));
        CU(cudaStreamSynchronize(ctx->stream));
        if (e->xfn(hs, hr, bytes, e->xuser) != 0) return fail(HPCG_ENCCL, "exchange: the caller's all-gather failed");
        CU(cudaMemcpyAsync(e->xrecv.p, hr, bytes * (size_t)e->xr, cudaMemcpyHostToDevice, ctx->stream));
        return HPCG_OK;
    }
    const NcclApi& a = nccl_api();
    if (!a.ok || !ctx->comm) return fail(HPCG_ENCCL, "exchange: no NCCL communicator attached to the context");
    const ncclResult_t r = a.all_gather(e->xsend.p, e->xrecv.p, bytes, ncclChar, ctx->comm, ctx->stream);
    if (r != ncclSuccess) return fail(HPCG_ENCCL, std::string("ncclAllGather: ") + a.error_string(r));
    return HPCG_OK;
}

// Multi-rank publication of one round (or of the hybrid carry-over): pack -> all-gather -> the
// global publication scan on every rank (xch_*_round_kernel). ts < 0: the latest rank clock.
int engine_publish_global(hpcg_engine* e, int publish, int carry, double clock, double ts) {
    hpcg_ctx* ctx = e->ctx;
    const int64_t kn = e->k * e->n, L = xch_round_len(e->xWmax, kn, e->k);
    XPackParams pk;
    pk.W = (int)e->W;
    pk.Wmax = (int)e->xWmax;
    pk.k = (int)e->k;
    pk.n = (int)e->n;
    pk.base = e->cfg.worker_base;
    pk.publish = publish;
    pk.carry = carry;
    pk.now = clock;
    pk.accepted = e->acc.as<uint8_t>();
    pk.inc_obj = e->inc_obj.as<double>();
    pk.inc_c = e->inc_c.as<double>();
    pk.inc_f = e->inc_f.as<uint8_t>();
    pk.rec = e->xsend.as<double>();
    xch_pack_round_kernel<<<1, 256, 0, ctx->stream>>>(pk);
    CU(cudaGetLastError());
    if (int rc = engine_allgather(e, (size_t)L * 8)) return rc;
    XMergeParams mp;
    mp.G = e->xr;
    mp.Wmax = (int)e->xWmax;
    mp.k = (int)e->k;
    mp.n = (int)e->n;
    mp.ts_from_clock = ts < 0.0 ? 1 : 0;
    mp.ts = ts;
    mp.recv = e->xrecv.as<double>();
    mp.sh_version = e->sh_ver.as<int64_t>();
    mp.sh_obj = e->sh_obj.as<double>();
    mp.sh_worker = e->sh_worker.as<int32_t>();
    mp.sh_c = e->sh_c.as<double>();
    mp.sh_f = e->sh_f.as<uint8_t>();
    mp.pub_log = e->pub_log.as<double>();
    mp.pub_count = e->pub_count.as<int64_t>();
    mp.pub_cap = e->pub_cap;
    mp.err = e->xerr.as<int32_t>();
    xch_merge_round_kernel<<<1, 256, 0, ctx->stream>>>(mp);
    CU(cudaGetLastError());
    ctx->launches += 2;
    e->pub_ub += e->xWtot;
    return HPCG_OK;
}

// One round of the schedule. `now`: seconds since the run start read ONCE by the caller (wall
// clock: the stop test, the phase test and the hybrid carry-over all use this one reading, as a
// reference worker does at the top of its loop, engine.hpp:353-364); ignored in lockstep.
int engine_round(hpcg_engine* e, double now) {
    hpcg_ctx* ctx = e->ctx;
    const int64_t r = e->round, W = e->W, k = e->k, n = e->n, s = e->s, kn = k * n;
    // phase test on the schedule's clock: samples processed (lockstep) or seconds (wall clock)
    const bool coop = phase_cooperative(e->cfg.strategy, e->cfg.phase_t1, e->wall ? now : (double)r);
    const bool hybrid = e->cfg.strategy == HPCG_HYBRID;
    const bool multi = e->xr > 1;
    if (int rc = engine_reserve(e, 2 * std::max(W, e->xWtot))) return rc;
    if (e->wall && hybrid && coop && !e->entered_coop) {
        // engine.hpp:359-364: entering the cooperative phase publishes each worker's finite
        // incumbent (worker-id order, strict <) before the step draws its init from the snapshot
        e->entered_coop = true;
        if (multi) {
            if (int rc = engine_publish_global(e, 0, 1, now, now)) return rc;
        } else {
            RoundEndParams q = round_end_params(e);
            q.log = 0;
            q.publish = 0;
            q.carry = 1;
            q.ts = now;
            if (int rc = launch_round_end(e, q)) return rc;
            e->pub_ub += W;
        }
    }
    const bool reference = e->cfg.rng_mode == HPCG_RNG_REFERENCE;
    const int64_t ncand = e->cfg.candidates;
    std::vector<int64_t> pending_loop, no_valid;
    std::vector<Mt64> snap;
    if (reference) {
        // which slots each worker will reseed (seeding.hpp:60-79) decides the draws it consumes
        std::vector<uint8_t> flags((size_t)(W * k), 1);
        int64_t ver = 1;
        if (coop) {
            CU(d2h(&ver, e->sh_ver.as<int64_t>(), 1, ctx->stream));
            std::vector<uint8_t> f1((size_t)k);
            CU(d2h(f1.data(), e->sh_f.as<uint8_t>(), (size_t)k, ctx->stream));
            CU(cudaStreamSynchronize(ctx->stream));
            for (int64_t w = 0; w < W; ++w)
                for (int64_t j = 0; j < k; ++j) flags[(size_t)(w * k + j)] = ver ? f1[(size_t)j] : 1;
        } else {
            CU(d2h(flags.data(), e->inc_f.as<uint8_t>(), (size_t)(W * k), ctx->stream));
            CU(cudaStreamSynchronize(ctx->stream));
        }
        pending_loop.assign((size_t)W, 0);
        no_valid.assign((size_t)W, 0);
        snap.resize((size_t)W);
        for (int64_t w = 0; w < W; ++w) {
            Mt64& rng = e->streams[(size_t)w];
            sparse_fisher_yates(rng, e->ds->m, s, e->h_idx.data() + w * s);  // engine.hpp:241
            int64_t np_ = 0, nv = 0;
            for (int64_t j = 0; j < k; ++j) (flags[(size_t)(w * k + j)] ? np_ : nv) += 1;
            e->h_fr[(size_t)w] = 0;
            if (np_ > 0 && nv == 0) {
                e->h_fr[(size_t)w] = (int64_t)rng.uniform_index((uint64_t)s);
                no_valid[(size_t)w] = 1;
            }
            snap[(size_t)w] = rng;
            const int64_t loops = np_ - no_valid[(size_t)w];
            pending_loop[(size_t)w] = loops;
            for (int64_t t = 0; t < loops * ncand; ++t) e->h_un[(size_t)(w * e->ucap + t)] = rng.unit();
        }
        CU(h2d(e->d_idx.as<int64_t>(), e->h_idx.data(), (size_t)(W * s), ctx->stream));
        CU(h2d(e->d_fr.as<int64_t>(), e->h_fr.data(), (size_t)W, ctx->stream));
        CU(h2d(e->d_un.as<double>(), e->h_un.data(), (size_t)(W * e->ucap), ctx->stream));
    }
    StepParams p = {};
    p.X = e->ds->X;
    set_shards(p, e->ds);
    p.m = e->ds->m;
    SamplePRP::moduli((uint64_t)p.m, p.prp_a, p.prp_b, p.prp_inv_b);
    p.n = (int)n;
    p.s = s;
    p.W = (int)W;
    p.geo_W = (int)std::max<int64_t>(W, e->xWtot);
    p.sample_mode = reference ? 0 : 1;
    p.idx = e->d_idx.as<int64_t>();
    p.key = e->key;
    p.round = (uint32_t)r;
    p.worker_base = e->cfg.worker_base;
    if (coop) {
        p.init_c = e->sh_c.as<double>();
        p.init_stride = 0;
        p.init_f = e->sh_f.as<uint8_t>();
        p.initf_stride = 0;
        p.shared_version = e->sh_ver.as<int64_t>();
    } else {
        p.init_c = e->inc_c.as<double>();
        p.init_stride = kn;
        p.init_f = e->inc_f.as<uint8_t>();
        p.initf_stride = k;
        p.shared_version = nullptr;
    }
    p.candidates = (int)ncand;
    p.seed_mode = reference ? 0 : 1;
    p.first_row = e->d_fr.as<int64_t>();
    p.units = e->d_un.as<double>();
    p.units_stride = (int)e->ucap;
    p.k = (int)k;
    p.max_iters = (int)std::min<int64_t>(e->cfg.max_iters, INT32_MAX);
    p.rel_tol = e->cfg.rel_tol;
    p.do_lloyd = 1;
    p.out_obj = e->objb.as<double>();
    p.out_iters = e->iters.as<int32_t>();
    p.out_stop = e->stopb.as<int32_t>();
    p.out_nd = e->nd.as<int64_t>();
    p.out_filled = e->filled.as<int32_t>();
    p.out_err = e->err.as<int32_t>();
    p.inc_c = e->inc_c.as<double>();
    p.inc_f = e->inc_f.as<uint8_t>();
    p.inc_obj = e->inc_obj.as<double>();
    p.accepted = e->acc.as<uint8_t>();
    p.trace = e->trace_buf;
    p.trace_mode = e->trace_mode;
    std::string why;
    KTimer kt(ctx, 0);
    cudaError_t ce = launch_step(e->ds->dtype, p, ctx->stream, nullptr, &why);
    kt.done();
    if (ce != cudaSuccess) return fail(HPCG_ECUDA, std::string("worker step launch: ") + cudaGetErrorString(ce) + " " + why);
    ctx->launches += 1;

    RoundEndParams q = round_end_params(e);
    q.publish = coop ? 1 : 0;  // round_was_coop (engine.hpp:393)
    double t_end = 0.0;
    if (e->wall) {  // the round's samples are done at t_end (trace / publication timestamp)
        CU(cudaStreamSynchronize(ctx->stream));
        t_end = e->elapsed();
        q.ts = t_end;
        q.carry = 0;  // wall clock: carried over at the start of the first cooperative round
    } else {
        q.ts = (double)(r + 1);
        q.carry = (hybrid && (r + 1) == (int64_t)(size_t)e->cfg.phase_t1) ? 1 : 0;  // engine.hpp:386,396
    }
    if (multi) {  // log the round locally, publish over every rank's workers
        const int pub = q.publish, car = q.carry;
        q.publish = 0;
        q.carry = 0;
        if (int rc = launch_round_end(e, q)) return rc;
        if (int rc = engine_publish_global(e, pub, car, t_end, e->wall ? -1.0 : q.ts)) return rc;
        if (e->wall) {  // the common clock of the ranks: the latest end of this round
            const int64_t L = xch_round_len(e->xWmax, kn, k);
            std::vector<double> clk((size_t)e->xr);
            for (int g = 0; g < e->xr; ++g) CU(d2h(&clk[(size_t)g], e->xrecv.as<double>() + g * L + 2, 1, ctx->stream));
            CU(cudaStreamSynchronize(ctx->stream));
            t_end = *std::max_element(clk.begin(), clk.end());
            e->common_now = t_end;
        }
    } else {
        if (q.publish || q.carry) e->pub_ub += W;
        if (int rc = launch_round_end(e, q)) return rc;
    }
    if (e->wall) e->t_end.push_back(t_end);

    if (reference) {  // rewind streams of workers whose seeding stopped early (seeding.hpp:87)
        std::vector<int32_t> fl((size_t)W);
        CU(d2h(fl.data(), e->filled.as<int32_t>(), (size_t)W, ctx->stream));
        CU(cudaStreamSynchronize(ctx->stream));
        for (int64_t w = 0; w < W; ++w) {
            const int64_t used = fl[(size_t)w] - no_valid[(size_t)w];
            if (used < pending_loop[(size_t)w]) {
                Mt64 rng = snap[(size_t)w];
                for (int64_t t = 0; t < used * ncand; ++t) rng.unit();
                e->streams[(size_t)w] = rng;
            }
        }
    }
    ++e->round;
    return HPCG_OK;
}

// ------------------------------------------------------------------------------------------
// Free-running wall-clock schedule with immediate publication (run_wall_clock, engine.hpp:348-374).
// The workers are cut into groups; each group advances on its own stream as a chain
//   between(prep) -> step -> between(post + prep) -> step -> ... -> between(post)
// and the groups run concurrently. `between` is one warp that does, per worker of the group and in
// worker-id order, what the reference's worker thread does around worker_step:
//   post: ++samples_processed, t_w = clock, trace entry of an accepted step (timestamp nudged with
//         nextafter, engine.hpp:258-262), SharedBest::try_publish of an accepted cooperative step
//         (engine.hpp:368-370) -- at once, not at a round end;
//   prep: the loop head (engine.hpp:353-365): one clock reading decides stop (time limit, sample
//         cap), phase, and the hybrid entry publication; then step_init (engine.hpp:337-343): the
//         snapshot of the shared best -- or the worker's own incumbent -- copied to the worker's
//         init slot, which the step kernel reads.
// The shared best is the device-side versioned incumbent: {version, objective, worker, centroids,
// flags} guarded by a spin lock taken by one lane (the mutex of engine.hpp:114-157), so snapshots
// are never torn and publications are strict-< in lock order. The clock is %globaltimer.
struct FreeParams {
    int W, k, n, worker_base, strategy;
    double t1, limit;
    int64_t max_samples;
    const unsigned long long* t0;
    const uint8_t* accepted;
    const double* inc_obj;
    const double* inc_c;
    const uint8_t* inc_f;
    const int64_t* nd;
    const int32_t* err;
    int32_t* err_first;
    int32_t* go;
    uint8_t* coop;
    uint8_t* entered;
    int64_t* samples;
    double* tw;
    double* init_c;
    uint8_t* init_f;
    int64_t* trace_cnt;
    double* trace;  // [W x trace_cap x 2]
    int64_t trace_cap;
    unsigned long long* nd_total;
    int* lock;
    int64_t* sh_version;
    double* sh_obj;
    int32_t* sh_worker;
    double* sh_c;
    uint8_t* sh_f;
    double* pub_log;
    int64_t* pub_count;
    int64_t pub_cap;
};

__device__ __forceinline__ unsigned long long free_gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// t0 such that (globaltimer - t0) continues the host's elapsed() (seconds since the engine's t0)
__global__ void free_t0_kernel(unsigned long long* t0, unsigned long long elapsed_ns) { *t0 = free_gtimer() - elapsed_ns; }

__device__ __forceinline__ void free_lock(int* lock, int lane) {
    if (lane == 0)
        while (atomicCAS(lock, 0, 1) != 0) __nanosleep(100);
    __syncwarp();
    __threadfence();
}
__device__ __forceinline__ void free_unlock(int* lock, int lane) {
    __threadfence();
    __syncwarp();
    if (lane == 0) atomicExch(lock, 0);
}

// SharedBest::try_publish (engine.hpp:126-136); the caller's warp holds the writers' lock. Readers do
// not take it: the record is a seqlock (lock[1] is odd while a writer is inside), so the snapshots of
// concurrent workers do not serialise behind one another -- publications are rare, snapshots are
// one per sample.
__device__ void free_try_publish(const FreeParams& q, int w, double obj, double ts, int lane) {
    if (!(obj < *(volatile double*)q.sh_obj)) return;
    const int kn = q.k * q.n;
    volatile int* seq = q.lock + 1;
    if (lane == 0) *seq = *seq + 1;  // odd: record in flux
    __syncwarp();
    __threadfence();
    for (int e = lane; e < kn; e += 32) ((volatile double*)q.sh_c)[e] = q.inc_c[(int64_t)w * kn + e];
    for (int e = lane; e < q.k; e += 32) ((volatile uint8_t*)q.sh_f)[e] = q.inc_f[(int64_t)w * q.k + e];
    if (lane == 0) {
        const int64_t ver = *(volatile int64_t*)q.sh_version + 1;
        *(volatile int64_t*)q.sh_version = ver;
        *(volatile double*)q.sh_obj = obj;
        *(volatile int32_t*)q.sh_worker = q.worker_base + w;
        const int64_t at = *(volatile int64_t*)q.pub_count;
        if (at < q.pub_cap) {
            double* rec = q.pub_log + at * 4;
            rec[0] = (double)ver;
            rec[1] = (double)(q.worker_base + w);
            rec[2] = obj;
            rec[3] = ts;
        }
        *(volatile int64_t*)q.pub_count = at + 1;
    }
    __threadfence();
    __syncwarp();
    if (lane == 0) *seq = *seq + 1;  // even: record stable
}

constexpr int kFreeWarps = 16;  // warps of the between kernel (one worker each in the parallel phases)

__global__ void __launch_bounds__(32 * kFreeWarps) free_between_kernel(const FreeParams q, int w0, int g, int do_post,
                                                                      int do_prep) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int kn = q.k * q.n;
    __shared__ double s_ts[64];
    __shared__ int s_pub[64];
    // ---- post: bookkeeping of the finished steps, one worker per warp; the publications after it in
    // worker-id order by warp 0 (so one group of all workers publishes exactly as a lockstep round end)
    for (int i0 = 0; do_post && i0 < g; i0 += 64) {
        for (int i = i0 + warp; i < min(g, i0 + 64); i += kFreeWarps) {
            const int w = w0 + i;
            if (lane == 0) {
                int pub = 0;
                double ts = 0.0;
                if (q.go[w]) {  // the step this worker was prepared for has run
                    const bool acc = q.accepted[w] != 0;
                    ts = (double)(free_gtimer() - *q.t0) * 1e-9;  // the clock is read once, after the sample
                    q.samples[w] += 1;
                    q.tw[w] = ts;
                    atomicAdd(q.nd_total, (unsigned long long)q.nd[w]);
                    if (q.err[w] != 0 && q.err_first[w] == 0) q.err_first[w] = q.err[w];
                    if (acc) {
                        const int64_t cnt = q.trace_cnt[w];
                        double* tr = q.trace + (int64_t)w * q.trace_cap * 2;
                        if (cnt > 0) {
                            const double last = tr[(min(cnt, q.trace_cap) - 1) * 2];
                            if (!(ts > last)) ts = nextafter(last, (double)INFINITY);
                        }
                        const int64_t at = min(cnt, q.trace_cap - 1);  // a full trace keeps its latest entry last
                        tr[at * 2] = ts;
                        tr[at * 2 + 1] = q.inc_obj[w];
                        q.trace_cnt[w] = cnt + 1;
                    }
                    pub = (acc && q.coop[w]) ? 1 : 0;
                }
                s_ts[i - i0] = ts;
                s_pub[i - i0] = pub;
            }
        }
        __syncthreads();
        if (warp == 0)
            for (int i = i0; i < min(g, i0 + 64); ++i)
                if (s_pub[i - i0]) {
                    free_lock(q.lock, lane);
                    free_try_publish(q, w0 + i, q.inc_obj[w0 + i], s_ts[i - i0], lane);
                    free_unlock(q.lock, lane);
                }
        __syncthreads();
    }
    if (!do_prep) return;
    // ---- prep: the loop head of every worker of the group, one worker per warp
    for (int i = warp; i < g; i += kFreeWarps) {
        const int w = w0 + i;
        int flags = 0;
        double now = 0.0;
        if (lane == 0) {
            now = (double)(free_gtimer() - *q.t0) * 1e-9;
            const bool go = now < q.limit && (q.max_samples < 1 || q.samples[w] < q.max_samples) && q.err_first[w] == 0;
            const bool coop = q.strategy == HPCG_COOPERATIVE || (q.strategy == HPCG_HYBRID && now >= q.t1);
            const bool enter = go && coop && q.strategy == HPCG_HYBRID && !q.entered[w];
            q.go[w] = go ? 1 : 0;
            q.coop[w] = coop ? 1 : 0;
            if (enter) q.entered[w] = 1;
            flags = (go ? 1 : 0) | (coop ? 2 : 0) | (enter ? 4 : 0);
        }
        flags = __shfl_sync(0xffffffffu, flags, 0);
        now = __shfl_sync(0xffffffffu, now, 0);
        if (!(flags & 1)) continue;
        double* ic = q.init_c + (int64_t)w * kn;
        uint8_t* ifl = q.init_f + (int64_t)w * q.k;
        if (flags & 2) {
            if (flags & 4) {  // engine.hpp:359-364: the phase-1 incumbent enters the shared best
                const double obj = q.inc_obj[w];
                if (isfinite(obj)) {
                    free_lock(q.lock, lane);
                    free_try_publish(q, w, obj, now, lane);
                    free_unlock(q.lock, lane);
                }
            }
            // snapshot() (engine.hpp:119-124) without the writers' lock: retry while a writer is inside or
            // the sequence moved under the copy; nullopt while version == 0
            volatile int* seq = q.lock + 1;
            for (;;) {
                int s1 = 0;
                if (lane == 0) s1 = *seq;
                s1 = __shfl_sync(0xffffffffu, s1, 0);
                if (s1 & 1) {
                    __nanosleep(200);
                    continue;
                }
                __threadfence();
                const int64_t ver = *(volatile int64_t*)q.sh_version;
                for (int e = lane; e < kn; e += 32) ic[e] = ver ? ((volatile double*)q.sh_c)[e] : 0.0;
                for (int e = lane; e < q.k; e += 32) ifl[e] = ver ? ((volatile uint8_t*)q.sh_f)[e] : (uint8_t)1;
                __threadfence();
                int s2 = 0;
                if (lane == 0) s2 = *seq;
                s2 = __shfl_sync(0xffffffffu, s2, 0);
                if (s1 == s2) break;
            }
        } else {
            for (int e = lane; e < kn; e += 32) ic[e] = q.inc_c[(int64_t)w * kn + e];
            for (int e = lane; e < q.k; e += 32) ifl[e] = q.inc_f[(int64_t)w * q.k + e];
        }
    }
}

int engine_run_free(hpcg_engine* e) {
    hpcg_ctx* ctx = e->ctx;
    const int64_t W = e->W, k = e->k, n = e->n, kn = k * n;
    cudaStream_t st0 = ctx->stream;
    if (e->round > 0 || e->free_mode) return fail(HPCG_EINVAL, "free-running schedule: the engine has already run");
    const int gsz = (int)(e->cfg.free_group > 0 ? std::min<int64_t>(e->cfg.free_group, W) : std::max<int64_t>(1, (W + 15) / 16));
    const int G = (int)((W + gsz - 1) / gsz);
    static const int max_streams = getenv("HPCG_FREE_STREAMS") ? std::max(1, atoi(getenv("HPCG_FREE_STREAMS"))) : 16;
    const int S = std::min(G, max_streams);
    e->fr_cap = 512;
    CU(e->fr_t0.reserve(8));
    CU(e->fr_go.reserve((size_t)W * 4));
    CU(e->fr_coop.reserve((size_t)W));
    CU(e->fr_entered.reserve((size_t)W));
    CU(e->fr_samples.reserve((size_t)W * 8));
    CU(e->fr_tw.reserve((size_t)W * 8));
    CU(e->fr_init_c.reserve((size_t)(W * kn) * 8));
    CU(e->fr_init_f.reserve((size_t)(W * k)));
    CU(e->fr_tcnt.reserve((size_t)W * 8));
    CU(e->fr_trace.reserve((size_t)(W * e->fr_cap) * 16));
    CU(e->fr_lock.reserve(8));  // [0] writers' lock, [1] seqlock sequence
    CU(cudaMemsetAsync(e->fr_go.p, 0, (size_t)W * 4, st0));
    CU(cudaMemsetAsync(e->fr_coop.p, 0, (size_t)W, st0));
    CU(cudaMemsetAsync(e->fr_entered.p, 0, (size_t)W, st0));
    CU(cudaMemsetAsync(e->fr_samples.p, 0, (size_t)W * 8, st0));
    CU(cudaMemsetAsync(e->fr_tw.p, 0, (size_t)W * 8, st0));
    CU(cudaMemsetAsync(e->fr_tcnt.p, 0, (size_t)W * 8, st0));
    CU(cudaMemsetAsync(e->fr_lock.p, 0, 8, st0));
    const int64_t want_pubs = std::max<int64_t>(e->pub_cap, 16384);
    CU(e->pub_log.grow((size_t)want_pubs * 32, (size_t)e->pub_cap * 32, st0));
    e->pub_cap = want_pubs;
    e->free_mode = true;

    FreeParams q = {};
    q.W = (int)W;
    q.k = (int)k;
    q.n = (int)n;
    q.worker_base = e->cfg.worker_base;
    q.strategy = e->cfg.strategy;
    q.t1 = e->cfg.phase_t1;
    q.limit = e->cfg.time_limit;
    q.max_samples = e->cfg.max_samples;
    q.t0 = e->fr_t0.as<unsigned long long>();
    q.accepted = e->acc.as<uint8_t>();
    q.inc_obj = e->inc_obj.as<double>();
    q.inc_c = e->inc_c.as<double>();
    q.inc_f = e->inc_f.as<uint8_t>();
    q.nd = e->nd.as<int64_t>();
    q.err = e->err.as<int32_t>();
    q.err_first = e->err_first.as<int32_t>();
    q.go = e->fr_go.as<int32_t>();
    q.coop = e->fr_coop.as<uint8_t>();
    q.entered = e->fr_entered.as<uint8_t>();
    q.samples = e->fr_samples.as<int64_t>();
    q.tw = e->fr_tw.as<double>();
    q.init_c = e->fr_init_c.as<double>();
    q.init_f = e->fr_init_f.as<uint8_t>();
    q.trace_cnt = e->fr_tcnt.as<int64_t>();
    q.trace = e->fr_trace.as<double>();
    q.trace_cap = e->fr_cap;
    q.nd_total = e->nd_total.as<unsigned long long>();
    q.lock = e->fr_lock.as<int>();
    q.sh_version = e->sh_ver.as<int64_t>();
    q.sh_obj = e->sh_obj.as<double>();
    q.sh_worker = e->sh_worker.as<int32_t>();
    q.sh_c = e->sh_c.as<double>();
    q.sh_f = e->sh_f.as<uint8_t>();
    q.pub_log = e->pub_log.as<double>();
    q.pub_count = e->pub_count.as<int64_t>();
    q.pub_cap = e->pub_cap;

    StepParams p = {};
    p.X = e->ds->X;
    set_shards(p, e->ds);
    p.m = e->ds->m;
    SamplePRP::moduli((uint64_t)p.m, p.prp_a, p.prp_b, p.prp_inv_b);
    p.n = (int)n;
    p.s = e->s;
    p.geo_W = (int)W;  // the cluster geometry of the whole engine, whatever the group size
    p.sample_mode = 1;
    p.key = e->key;
    p.init_stride = kn;
    p.initf_stride = k;
    p.shared_version = nullptr;
    p.candidates = (int)e->cfg.candidates;
    p.seed_mode = 1;
    p.units_stride = (int)e->ucap;
    p.k = (int)k;
    p.max_iters = (int)std::min<int64_t>(e->cfg.max_iters, INT32_MAX);
    p.rel_tol = e->cfg.rel_tol;
    p.do_lloyd = 1;

    std::vector<cudaStream_t> streams((size_t)S, nullptr);
    std::vector<cudaEvent_t> ev((size_t)(2 * S), nullptr);
    auto cleanup = [&]() {
        for (auto s_ : streams)
            if (s_) {
                cudaStreamSynchronize(s_);
                cudaStreamDestroy(s_);
            }
        for (auto v : ev)
            if (v) cudaEventDestroy(v);
    };
    for (auto& s_ : streams)
        if (cudaStreamCreateWithFlags(&s_, cudaStreamNonBlocking) != cudaSuccess) {
            cleanup();
            return fail(HPCG_ECUDA, "free-running schedule: stream creation failed");
        }
    for (auto& v : ev)
        if (cudaEventCreateWithFlags(&v, cudaEventDisableTiming) != cudaSuccess) {
            cleanup();
            return fail(HPCG_ECUDA, "free-running schedule: event creation failed");
        }
    // the device clock continues the engine's host clock (seconds since t0)
    free_t0_kernel<<<1, 1, 0, st0>>>(e->fr_t0.as<unsigned long long>(), (unsigned long long)(e->elapsed() * 1e9));
    cudaError_t ce = cudaStreamSynchronize(st0);
    ctx->launches += 1;
    int64_t laps = 0;
    std::string why;
    for (; ce == cudaSuccess; ++laps) {
        if (e->elapsed() >= e->cfg.time_limit) break;
        if (e->cfg.max_samples > 0 && laps >= e->cfg.max_samples) break;
        // at most two laps in flight per stream: the host does not run ahead of the device clock
        if (laps >= 2)
            for (int si = 0; si < S && ce == cudaSuccess; ++si) ce = cudaEventSynchronize(ev[(size_t)((laps & 1) * S + si)]);
        for (int grp = 0; grp < G && ce == cudaSuccess; ++grp) {
            cudaStream_t st = streams[(size_t)(grp % S)];
            const int w0 = grp * gsz, g = (int)std::min<int64_t>(gsz, W - w0);
            free_between_kernel<<<1, 32 * kFreeWarps, 0, st>>>(q, w0, g, laps > 0 ? 1 : 0, 1);
            p.W = g;
            p.round = (uint32_t)laps;
            p.worker_base = e->cfg.worker_base + w0;
            p.init_c = e->fr_init_c.as<double>() + (int64_t)w0 * kn;
            p.init_f = e->fr_init_f.as<uint8_t>() + (int64_t)w0 * k;
            p.first_row = e->d_fr.as<int64_t>() + w0;
            p.units = e->d_un.as<double>() + (int64_t)w0 * e->ucap;
            p.out_obj = e->objb.as<double>() + w0;
            p.out_iters = e->iters.as<int32_t>() + w0;
            p.out_stop = e->stopb.as<int32_t>() + w0;
            p.out_nd = e->nd.as<int64_t>() + w0;
            p.out_filled = e->filled.as<int32_t>() + w0;
            p.out_err = e->err.as<int32_t>() + w0;
            p.inc_c = e->inc_c.as<double>() + (int64_t)w0 * kn;
            p.inc_f = e->inc_f.as<uint8_t>() + (int64_t)w0 * k;
            p.inc_obj = e->inc_obj.as<double>() + w0;
            p.accepted = e->acc.as<uint8_t>() + w0;
            p.go = e->fr_go.as<int32_t>() + w0;
            ce = launch_step(e->ds->dtype, p, st, nullptr, &why);
            ctx->launches += 2;
        }
        for (int si = 0; si < S && ce == cudaSuccess; ++si) ce = cudaEventRecord(ev[(size_t)((laps & 1) * S + si)], streams[(size_t)si]);
    }
    if (ce == cudaSuccess && laps > 0)
        for (int grp = 0; grp < G; ++grp) {  // account for the last prepared steps
            const int w0 = grp * gsz, g = (int)std::min<int64_t>(gsz, W - w0);
            free_between_kernel<<<1, 32 * kFreeWarps, 0, streams[(size_t)(grp % S)]>>>(q, w0, g, 1, 0);
            ctx->launches += 1;
        }
    for (auto s_ : streams) {
        cudaError_t e2 = cudaStreamSynchronize(s_);
        if (ce == cudaSuccess) ce = e2;
    }
    if (ce == cudaSuccess) ce = cudaGetLastError();
    cleanup();
    if (ce != cudaSuccess) return fail(HPCG_ECUDA, std::string("free-running schedule: ") + cudaGetErrorString(ce) + " " + why);
    e->round = laps;  // laps enqueued: an upper bound of every worker's sample count
    return HPCG_OK;
}
}  // namespace

extern "C" {

int hpcg_comm_unique_id(void* id_out) {
    const NcclApi& a = nccl_api();
    if (!a.ok) return fail(HPCG_ENCCL, a.why);
    ncclUniqueId id;
    const ncclResult_t r = a.get_unique_id(&id);
    if (r != ncclSuccess) return fail(HPCG_ENCCL, std::string("ncclGetUniqueId: ") + a.error_string(r));
    std::memcpy(id_out, &id, sizeof(id));
    return HPCG_OK;
}

int hpcg_ctx_attach_comm(hpcg_ctx* ctx, int32_t nranks, int32_t rank, const void* id) {
    if (!ctx || !id || nranks < 1 || rank < 0 || rank >= nranks) return fail(HPCG_EINVAL, "attach_comm: bad rank layout");
    const NcclApi& a = nccl_api();
    if (!a.ok) return fail(HPCG_ENCCL, a.why);
    std::lock_guard<std::mutex> lk(ctx->mu);
    bind_device(ctx->device);
    if (ctx->comm) {
        a.comm_destroy(ctx->comm);
        ctx->comm = nullptr;
    }
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    const ncclResult_t r = a.comm_init_rank(&ctx->comm, nranks, uid, rank);
    if (r != ncclSuccess) {
        ctx->comm = nullptr;
        return fail(HPCG_ENCCL, std::string("ncclCommInitRank: ") + a.error_string(r));
    }
    ctx->nranks = nranks;
    ctx->rank = rank;
    return HPCG_OK;
}

int hpcg_ctx_comm_info(const hpcg_ctx* ctx, int32_t* nranks, int32_t* rank) {
    if (nranks) *nranks = ctx->comm ? ctx->nranks : 1;
    if (rank) *rank = ctx->comm ? ctx->rank : 0;
    return HPCG_OK;
}

static cudaError_t engine_reset_state(hpcg_engine* e, cudaStream_t st) {
    EngineResetParams q = {};
    q.inc_c = e->inc_c.as<double>();
    q.inc_obj = e->inc_obj.as<double>();
    q.sh_obj = e->sh_obj.as<double>();
    q.sh_c = e->sh_c.as<double>();
    q.inc_f = e->inc_f.as<uint8_t>();
    q.sh_f = e->sh_f.as<uint8_t>();
    q.log_acc = e->log_acc.as<uint8_t>();
    q.err_first = e->err_first.as<int32_t>();
    q.sh_worker = e->sh_worker.as<int32_t>();
    q.sh_ver = e->sh_ver.as<int64_t>();
    q.pub_count = e->pub_count.as<int64_t>();
    q.nd_total = e->nd_total.as<unsigned long long>();
    q.W = e->W;
    q.k = e->k;
    q.kn = e->k * e->n;
    q.log_bytes = e->log_rounds * e->W;
    const int64_t work = std::max<int64_t>(q.W * q.kn, q.log_bytes);
    const unsigned blocks = (unsigned)std::min<int64_t>(296, std::max<int64_t>(1, (work + 255) / 256));
    engine_reset_kernel<<<blocks, 256, 0, st>>>(q);
    e->ctx->launches += 1;
    return cudaGetLastError();
}

int hpcg_engine_create(hpcg_ctx* ctx, const hpcg_dataset* ds, const hpcg_engine_cfg* c, hpcg_engine** out) {
    std::lock_guard<std::mutex> lk(ctx->mu);
    bind_device(ctx->device);
    hpcg_engine_cfg cfg = *c;
    if (cfg.strategy == HPCG_INNER) cfg.n_workers = 1;  // engine.hpp:446
    // EngineConfig::validate (engine.hpp:70-86)
    if (cfg.k < 1) return fail(HPCG_EINVAL, "EngineConfig: k must be positive");
    if (cfg.sample_size < 1 || cfg.sample_size > ds->m)
        return fail(HPCG_EINVAL, "EngineConfig: sample_size must be in [1, m]");
    if (cfg.n_workers < 1) return fail(HPCG_EINVAL, "EngineConfig: need at least one worker");
    if (std::isnan(cfg.time_limit) || cfg.time_limit < 0.0)
        return fail(HPCG_EINVAL, "EngineConfig: time limit must be positive");
    const bool wall = cfg.time_limit > 0.0 && std::isfinite(cfg.time_limit);  // deterministic_mode() false
    if (!wall && cfg.max_samples < 1) return fail(HPCG_EINVAL, "EngineConfig: need a time limit or a max_samples bound");
    if (wall && cfg.max_samples < 0) return fail(HPCG_EINVAL, "EngineConfig: max_samples must be positive");
    if (cfg.strategy == HPCG_HYBRID) {
        if (!(cfg.phase_t1 >= 0.0 && cfg.phase_t2 >= 0.0))
            return fail(HPCG_EINVAL, "EngineConfig: hybrid phase durations must be nonnegative");
        const double b = wall ? cfg.time_limit : (double)cfg.max_samples;  // EngineConfig::budget()
        if (!(std::fabs(cfg.phase_t1 + cfg.phase_t2 - b) <= 1e-9 * std::max(1.0, std::fabs(b))))
            return fail(HPCG_EINVAL, "EngineConfig: hybrid phases must sum to the total budget");
    }
    if (cfg.max_iters < 1) return fail(HPCG_EINVAL, "kmeans: max_iters must be positive");
    if (!(cfg.rel_tol > 0.0)) return fail(HPCG_EINVAL, "kmeans: rel_tol must be positive");
    if (cfg.candidates < 1) return fail(HPCG_EINVAL, "seeding: need at least one candidate");
    if (cfg.candidates > kMaxCandidates) return fail(HPCG_EUNSUPPORTED, "more than 4 K-means++ candidates per centre");
    if (int rc = check_shape(ds->dtype, ds->n, cfg.k)) return rc;
    // shapes without a cluster-resident geometry run on the grid-wide path (launch_step decides)
    if (cfg.free_running) {
        if (!wall) return fail(HPCG_EINVAL, "EngineConfig: the free-running schedule needs a time limit");
        if (cfg.free_group < 0) return fail(HPCG_EINVAL, "EngineConfig: free_group must be nonnegative");
        if (cfg.rng_mode != HPCG_RNG_PHILOX)
            return fail(HPCG_EUNSUPPORTED, "the free-running schedule draws on the device: rng_mode must be philox");
        StepGeometry g_;
        std::string why_;
        if (cfg.k > kMaxK || cfg.n_workers > INT32_MAX ||
            step_geometry(ds->dtype, (int)ds->n, cfg.sample_size, (int)cfg.k, (int)cfg.candidates, (int)cfg.n_workers, &g_,
                          &why_) != cudaSuccess) {
            cudaGetLastError();
            return fail(HPCG_EUNSUPPORTED, "the free-running schedule needs a cluster-resident shape (n <= 32, k <= 32, "
                                           "sample within a cluster's shared memory)");
        }
    }

    auto* e = new hpcg_engine;
    e->ctx = ctx;
    e->device = ctx->device;
    e->ds = ds;
    e->cfg = cfg;
    e->W = cfg.n_workers;
    e->k = cfg.k;
    e->n = ds->n;
    e->s = cfg.sample_size;
    e->wall = wall;
    // rounds: max_samples, or in wall-clock mode that cap (none: until the time limit); the
    // per-round logs and the publication log grow on demand (engine_reserve)
    e->R = wall && cfg.max_samples < 1 ? INT64_MAX : cfg.max_samples;
    e->key = splitmix64(cfg.master_seed ^ 0x48504331ULL);
    e->t0 = std::chrono::steady_clock::now();
    const int64_t W = e->W, k = e->k, kn = k * e->n;
    auto bad = [&](cudaError_t err) {
        delete e;
        return fail(HPCG_ECUDA, std::string("engine allocation: ") + cudaGetErrorString(err));
    };
#define ALLOC(buf, bytes)                                  \
    do {                                                   \
        cudaError_t err_ = e->buf.reserve((size_t)(bytes)); \
        if (err_ != cudaSuccess) return bad(err_);          \
    } while (0)
    ALLOC(inc_c, W * kn * 8);
    ALLOC(inc_f, W * k);
    ALLOC(inc_obj, W * 8);
    ALLOC(acc, W);
    ALLOC(nd, W * 8);
    ALLOC(err, W * 4);
    ALLOC(err_first, W * 4);
    ALLOC(iters, W * 4);
    ALLOC(stopb, W * 4);
    ALLOC(filled, W * 4);
    ALLOC(objb, W * 8);
    ALLOC(sh_ver, 8);
    ALLOC(sh_obj, 8);
    ALLOC(sh_worker, 4);
    ALLOC(sh_c, kn * 8);
    ALLOC(sh_f, k);
    e->log_rounds = std::min<int64_t>(e->R, 64);
    ALLOC(log_acc, e->log_rounds * W);
    ALLOC(log_obj, e->log_rounds * W * 8);
    ALLOC(nd_total, 8);
    e->pub_cap = std::max<int64_t>(256, 4 * W);
    ALLOC(pub_log, e->pub_cap * 4 * 8);
    ALLOC(pub_count, 8);
    const bool reference = cfg.rng_mode == HPCG_RNG_REFERENCE;
    e->ucap = std::max<int64_t>(1, k * cfg.candidates);
    ALLOC(d_fr, W * 8);
    ALLOC(d_un, W * e->ucap * 8);
    if (reference) {
        ALLOC(d_idx, W * e->s * 8);
        e->h_idx.assign((size_t)(W * e->s), 0);
        e->h_fr.assign((size_t)W, 0);
        e->h_un.assign((size_t)(W * e->ucap), 0.0);
        for (int64_t w = 0; w < W; ++w)  // engine.hpp:457
            e->streams.push_back(Mt64::derive(cfg.master_seed, 1, (uint64_t)(cfg.worker_base + w)));
    }
#undef ALLOC
    cudaStream_t st = ctx->stream;
    cudaError_t ce = cudaSuccess;
    auto chk = [&](cudaError_t x) {
        if (ce == cudaSuccess) ce = x;
    };
    chk(engine_reset_state(e, st));  // all-degenerate incumbents (engine.hpp:456), empty shared best
    (void)kn;
    if (ce != cudaSuccess) return bad(ce);
    *out = e;
    return HPCG_OK;
}

int hpcg_engine_set_exchange(hpcg_engine* e, int32_t nranks, int32_t rank, hpcg_allgather_fn fn, void* user) {
    std::lock_guard<std::mutex> lk(e->ctx->mu);
    hpcg_ctx* ctx = e->ctx;
    bind_device(ctx->device);
    if (nranks < 1 || rank < 0 || rank >= nranks) return fail(HPCG_EINVAL, "set_exchange: bad rank layout");
    if (e->round > 0) return fail(HPCG_EINVAL, "set_exchange: rounds already run");
    if (!fn && nranks > 1 && (!ctx->comm || ctx->nranks != nranks || ctx->rank != rank))
        return fail(HPCG_ENCCL, "set_exchange: no matching NCCL communicator attached to the context");
    if (e->cfg.strategy == HPCG_INNER && nranks > 1)
        return fail(HPCG_EUNSUPPORTED, "the inner strategy runs one worker: no multi-rank exchange");
    if (e->cfg.free_running && nranks > 1)
        return fail(HPCG_EUNSUPPORTED, "the free-running schedule runs on one rank");
    e->xr = nranks;
    e->xrank = rank;
    e->xfn = fn;
    e->xuser = user;
    e->xWmax = e->xWtot = e->W;
    if (nranks == 1) return HPCG_OK;
    // every rank's worker count and base; global ids must be contiguous in rank order
    CU(e->xsend.reserve(16));
    CU(e->xrecv.reserve((size_t)nranks * 16));
    const double wb[2] = {(double)e->W, (double)e->cfg.worker_base};
    CU(cudaMemcpyAsync(e->xsend.p, wb, 16, cudaMemcpyHostToDevice, ctx->stream));
    if (int rc = engine_allgather(e, 16)) return rc;
    std::vector<double> all((size_t)(2 * nranks));
    CU(d2h(all.data(), e->xrecv.as<double>(), all.size(), ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    int64_t expect = 0, wmax = 0;
    for (int g = 0; g < nranks; ++g) {
        const int64_t wg = (int64_t)all[(size_t)(2 * g)], bg = (int64_t)all[(size_t)(2 * g + 1)];
        if (bg != expect) return fail(HPCG_EINVAL, "set_exchange: worker ids must be contiguous in rank order");
        expect += wg;
        wmax = std::max(wmax, wg);
    }
    e->xWmax = wmax;
    e->xWtot = expect;
    const int64_t kn = e->k * e->n;
    const int64_t L = std::max<int64_t>(xch_round_len(wmax, kn, e->k), 4 + kn + e->k) + 8;
    CU(e->xsend.reserve((size_t)L * 8));
    CU(e->xrecv.reserve((size_t)(L * nranks) * 8));
    CU(e->xerr.reserve(16));
    CU(cudaMemsetAsync(e->xerr.p, 0, 16, ctx->stream));
    return HPCG_OK;
}

int hpcg_engine_reset(hpcg_engine* e, uint64_t master_seed) {
    std::lock_guard<std::mutex> lk(e->ctx->mu);
    hpcg_ctx* ctx = e->ctx;
    bind_device(ctx->device);
    cudaStream_t st = ctx->stream;
    const int64_t W = e->W;
    e->cfg.master_seed = master_seed;
    e->key = splitmix64(master_seed ^ 0x48504331ULL);
    e->round = 0;
    e->t0 = std::chrono::steady_clock::now();
    e->t_end.clear();
    if (e->cfg.rng_mode == HPCG_RNG_REFERENCE)
        for (int64_t w = 0; w < W; ++w)
            e->streams[(size_t)w] = Mt64::derive(master_seed, 1, (uint64_t)(e->cfg.worker_base + w));
    CU(engine_reset_state(e, st));
    e->pub_ub = 0;
    e->entered_coop = false;
    e->common_now = 0.0;
    e->free_mode = false;
    return HPCG_OK;
}

int hpcg_engine_import_best(hpcg_engine* e, double obj, int64_t worker, const double* C, const uint8_t* f) {
    std::lock_guard<std::mutex> lk(e->ctx->mu);
    hpcg_ctx* ctx = e->ctx;
    bind_device(ctx->device);
    cudaStream_t st = ctx->stream;
    int64_t ver = 0;
    CU(d2h(&ver, e->sh_ver.as<int64_t>(), 1, st));
    CU(cudaStreamSynchronize(st));
    ++ver;
    const int32_t wk = (int32_t)worker;
    CU(h2d(e->sh_ver.as<int64_t>(), &ver, 1, st));
    CU(h2d(e->sh_obj.as<double>(), &obj, 1, st));
    CU(h2d(e->sh_worker.as<int32_t>(), &wk, 1, st));
    CU(h2d(e->sh_c.as<double>(), C, (size_t)(e->k * e->n), st));
    CU(h2d(e->sh_f.as<uint8_t>(), f, (size_t)e->k, st));
    CU(cudaStreamSynchronize(st));
    return HPCG_OK;
}

int hpcg_engine_rounds(hpcg_engine* e, int64_t n_rounds) {
    std::lock_guard<std::mutex> lk(e->ctx->mu);
    bind_device(e->ctx->device);
    if (e->cfg.free_running) return fail(HPCG_EINVAL, "engine: the free-running schedule has no rounds (hpcg_engine_run)");
    for (int64_t i = 0; i < n_rounds; ++i) {
        if (e->round >= e->R) return fail(HPCG_EINVAL, "engine: max_samples rounds already run");
        const double now = !e->wall ? 0.0 : e->xr > 1 ? (e->round ? e->common_now : 0.0) : e->elapsed();
        if (int rc = engine_round(e, now)) return rc;
    }
    return HPCG_OK;
}

int hpcg_engine_run(hpcg_engine* e) {
    std::lock_guard<std::mutex> lk(e->ctx->mu);
    bind_device(e->ctx->device);
    if (e->cfg.free_running) return engine_run_free(e);
    while (e->round < e->R) {
        // run_wall_clock (engine.hpp:353-357): one clock reading per round decides the stop,
        // the phase and the carry-over
        // multi-rank: the ranks' common clock (latest round end) so every rank decides alike
        const double now = !e->wall ? 0.0 : e->xr > 1 ? (e->round ? e->common_now : 0.0) : e->elapsed();
        if (e->wall && now >= e->cfg.time_limit) break;
        if (int rc = engine_round(e, now)) return rc;
    }
    return HPCG_OK;
}

int64_t hpcg_engine_round_index(const hpcg_engine* e) { return e->round; }
uint64_t hpcg_engine_philox_key(const hpcg_engine* e) { return e->key; }

int hpcg_engine_worker_progress(hpcg_engine* e, int64_t* samples, double* t_w) {
    std::lock_guard<std::mutex> lk(e->ctx->mu);
    bind_device(e->ctx->device);
    const size_t W = (size_t)e->W;
    if (e->free_mode) {
        if (samples) CU(d2h(samples, e->fr_samples.as<int64_t>(), W, e->ctx->stream));
        if (t_w) CU(d2h(t_w, e->fr_tw.as<double>(), W, e->ctx->stream));
        CU(cudaStreamSynchronize(e->ctx->stream));
        return HPCG_OK;
    }
    // round-granular schedules: every worker has processed `round` samples; t_w is the round count
    // (lockstep, engine.hpp:413) or the last round end in seconds
    const double tw = e->round == 0 ? 0.0 : e->wall && !e->t_end.empty() ? e->t_end.back() : (double)e->round;
    for (size_t w = 0; w < W; ++w) {
        if (samples) samples[w] = e->round;
        if (t_w) t_w[w] = tw;
    }
    return HPCG_OK;
}

int hpcg_engine_set_trace(hpcg_engine* e, int64_t* trace_dev, int32_t mode) {
    e->trace_buf = trace_dev;
    e->trace_mode = mode;
    return HPCG_OK;
}

int hpcg_engine_distance_evals(hpcg_engine* e, int64_t* n_d) {
    std::lock_guard<std::mutex> lk(e->ctx->mu);
    bind_device(e->ctx->device);
    unsigned long long v = 0;
    CU(d2h(&v, e->nd_total.as<unsigned long long>(), 1, e->ctx->stream));
    CU(cudaStreamSynchronize(e->ctx->stream));
    *n_d = (int64_t)v;
    return HPCG_OK;
}

int hpcg_engine_export_best(hpcg_engine* e, double* obj_out, int64_t* worker_out, double* C_out, uint8_t* f_out) {
    std::lock_guard<std::mutex> lk(e->ctx->mu);
    bind_device(e->ctx->device);
    hpcg_ctx* ctx = e->ctx;
    int32_t wk = -1;
    if (obj_out) CU(d2h(obj_out, e->sh_obj.as<double>(), 1, ctx->stream));
    CU(d2h(&wk, e->sh_worker.as<int32_t>(), 1, ctx->stream));
    if (C_out) CU(d2h(C_out, e->sh_c.as<double>(), (size_t)(e->k * e->n), ctx->stream));
    if (f_out) CU(d2h(f_out, e->sh_f.as<uint8_t>(), (size_t)e->k, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    if (worker_out) *worker_out = wk;
    return HPCG_OK;
}

// finish of a multi-rank engine (all ranks call it): local select_best -> all-gather of the
// rank winners (+ the rank's first worker error) -> the global winner on every rank -> f(C, X) over
// this rank's rows -> all-gather of the shard partials, n_d and clocks, summed in rank order.
static int engine_finish_multi(hpcg_engine* e, hpcg_run_out* out, double* centroids, uint8_t* flags, int32_t* labels,
                               double* worker_obj, double* traces, int64_t trace_cap, int64_t* trace_len) {
    hpcg_ctx* ctx = e->ctx;
    cudaStream_t st = ctx->stream;
    const int64_t W = e->W, k = e->k, n = e->n, kn = k * n, R = e->round, G = e->xr;
    const bool want_obj = e->cfg.compute_full_objective || e->cfg.compute_assignment;
    const bool want_labels = e->cfg.compute_assignment && labels;
    CU(e->scratch_a.reserve((size_t)kn * 8));
    CU(e->scratch_b.reserve((size_t)k * 4));
    CU(e->scratch_c.reserve(8));
    CU(e->fin.reserve(16 + (size_t)kn * 8 + (size_t)k + 8 + 16));
    int32_t* sel_d = e->fin.as<int32_t>();
    double* bc_d = reinterpret_cast<double*>(e->fin.as<unsigned char>() + 16);
    uint8_t* bf_d = e->fin.as<uint8_t>() + 16 + kn * 8;
    double* gobj_d = reinterpret_cast<double*>(e->fin.as<unsigned char>() + ((16 + kn * 8 + k + 7) & ~7LL));
    int64_t* ggid_d = reinterpret_cast<int64_t*>(gobj_d + 1);
    finish_select_kernel<<<1, 256, 0, st>>>(e->inc_obj.as<double>(), e->inc_c.as<double>(), e->inc_f.as<uint8_t>(),
                                            (int)W, (int)k, (int)n, sel_d, bc_d, bf_d, e->scratch_a.as<double>(),
                                            e->scratch_b.as<int32_t>());
    // the rank's first worker error travels with its winner (worker errors are rethrown before
    // select_best, lowest worker first: engine.hpp:330-331)
    std::vector<int32_t> errf((size_t)W);
    CU(d2h(errf.data(), e->err_first.as<int32_t>(), (size_t)W, st));
    CU(cudaStreamSynchronize(st));
    double err_code = 0.0, err_gid = -1.0;
    for (int64_t w = 0; w < W; ++w)
        if (errf[(size_t)w]) {
            err_code = errf[(size_t)w];
            err_gid = (double)(e->cfg.worker_base + w);
            break;
        }
    const int64_t L1 = 4 + kn + k;  // [obj, gid, err, err gid | C | f]
    double* snd = e->xsend.as<double>();
    xch_pack_select_kernel<<<1, 256, 0, st>>>(sel_d, e->inc_obj.as<double>(), bc_d, bf_d, (int)k, (int)n,
                                               e->cfg.worker_base, snd + 2);  // [obj, gid, C, f] at +2
    // shift: the select record is [err, err gid, obj, gid, C, f]
    const double eh[2] = {err_code, err_gid};
    CU(cudaMemcpyAsync(snd, eh, 16, cudaMemcpyHostToDevice, st));
    CU(cudaGetLastError());
    if (int rc = engine_allgather(e, (size_t)L1 * 8)) return rc;
    std::vector<double> errs((size_t)(2 * G));
    for (int64_t g = 0; g < G; ++g) CU(d2h(&errs[(size_t)(2 * g)], e->xrecv.as<double>() + g * L1, 2, st));
    CU(cudaStreamSynchronize(st));
    for (int64_t g = 0; g < G; ++g) {  // rank order = global worker order
        const int code = (int)errs[(size_t)(2 * g)];
        if (code == kErrDegenerateInit) return fail(HPCG_EINVAL, "kmeans: degenerate centroid in init");
        if (code == kErrMonotone) return fail(HPCG_ELOGIC, "kmeans: objective increased between iterations");
    }
    // the gathered records without their 2-double error header: repack contiguously for the merge
    CU(e->xerr.reserve(std::max<size_t>((size_t)(G * (L1 - 2)) * 8, 16)));
    for (int64_t g = 0; g < G; ++g)
        CU(cudaMemcpyAsync(e->xerr.as<double>() + g * (L1 - 2), e->xrecv.as<double>() + g * L1 + 2,
                           (size_t)(L1 - 2) * 8, cudaMemcpyDeviceToDevice, st));
    xch_merge_select_kernel<<<1, 256, 0, st>>>(e->xerr.as<double>(), (int)G, (int)k, (int)n, sel_d, bc_d, bf_d,
                                                e->scratch_a.as<double>(), e->scratch_b.as<int32_t>(), gobj_d, ggid_d);
    CU(cudaGetLastError());
    ctx->launches += 3;
    int32_t hsel[2];
    double gobj = 0.0;
    int64_t ggid = -1;
    CU(d2h(hsel, sel_d, 2, st));
    CU(d2h(&gobj, gobj_d, 1, st));
    CU(d2h(&ggid, ggid_d, 1, st));
    CU(cudaStreamSynchronize(st));
    if (hsel[0] < 0) return fail(HPCG_ENOSOL, "no solution produced: every worker incumbent is infinite");
    const int kv = hsel[1];
    // this rank's rows: shard `rank` of a dataset sharded over the ranks (global sampling), else all of it
    hpcg_dataset local;
    const hpcg_dataset* dsl = e->ds;
    if (e->ds->nshards == e->xr) {
        local.ctx = ctx;
        local.X = e->ds->shard_ptr[e->xrank];
        local.shard_ptr[0] = local.X;
        local.m = e->ds->shard_end[e->xrank] - (e->xrank ? e->ds->shard_end[e->xrank - 1] : 0);
        local.shard_end[0] = local.m;
        local.n = e->ds->n;
        local.dtype = e->ds->dtype;
        dsl = &local;
    }
    DevBuf lab;
    double part = 0.0;
    if (want_obj) {
        if (kv == 0) return fail(HPCG_EINVAL, "assignment: every centroid is degenerate");
        if (want_labels) CU(lab.reserve((size_t)dsl->m * 4));
        if (int rc = run_assign(ctx, dsl, e->scratch_a.as<double>(), e->scratch_b.as<int32_t>(), kv,
                                want_labels ? lab.as<int32_t>() : nullptr, nullptr, e->scratch_c.as<double>(), e->blocks))
            return rc;
        CU(d2h(&part, e->scratch_c.as<double>(), 1, st));
    }
    // local per-worker outputs (traces, objectives) and this rank's share of the totals
    const int64_t Rw = std::max<int64_t>(R, 1) * W;
    std::vector<uint8_t> lacc((size_t)Rw);
    std::vector<double> lobj((size_t)Rw), hobj((size_t)W);
    unsigned long long ndt = 0;
    int64_t npub = 0;
    if (R > 0) {
        CU(d2h(lacc.data(), e->log_acc.as<uint8_t>(), (size_t)(R * W), st));
        CU(d2h(lobj.data(), e->log_obj.as<double>(), (size_t)(R * W), st));
    }
    CU(d2h(hobj.data(), e->inc_obj.as<double>(), (size_t)W, st));
    CU(d2h(&ndt, e->nd_total.as<unsigned long long>(), 1, st));
    CU(d2h(&npub, e->pub_count.as<int64_t>(), 1, st));
    if (centroids) CU(d2h(centroids, bc_d, (size_t)kn, st));
    if (flags) CU(d2h(flags, bf_d, (size_t)k, st));
    CU(cudaStreamSynchronize(st));
    auto ts_of = [&](int64_t r) { return e->wall && r < (int64_t)e->t_end.size() ? e->t_end[(size_t)r] : (double)(r + 1); };
    double min_last = kInf, last0 = -1.0;
    for (int64_t w = 0; w < W; ++w) {
        int64_t cnt = 0;
        double last = -1.0;
        for (int64_t r = 0; r < R; ++r) {
            if (!lacc[(size_t)(r * W + w)]) continue;
            if (traces && cnt < trace_cap) {
                traces[(w * trace_cap + cnt) * 2 + 0] = ts_of(r);
                traces[(w * trace_cap + cnt) * 2 + 1] = lobj[(size_t)(r * W + w)];
            }
            last = ts_of(r);
            ++cnt;
        }
        if (trace_len) trace_len[w] = cnt;
        if (cnt > 0) min_last = std::min(min_last, last);
        if (w == 0) last0 = last;
    }
    const double nd_local = (double)ndt + (want_obj ? (double)dsl->m * kv : 0.0);
    const double tail[6] = {part, nd_local, min_last, last0, (double)(W * R), 0.0};
    CU(cudaMemcpyAsync(e->xsend.p, tail, sizeof(tail), cudaMemcpyHostToDevice, st));
    if (int rc = engine_allgather(e, sizeof(tail))) return rc;
    std::vector<double> tails((size_t)(6 * G));
    CU(d2h(tails.data(), e->xrecv.as<double>(), (size_t)(6 * G), st));
    if (want_labels) CU(d2h(labels, lab.as<int32_t>(), (size_t)dsl->m, st));
    CU(cudaStreamSynchronize(st));
    hpcg_run_out o = {};
    double f = 0.0, nd = 0.0, ml = kInf, tot = 0.0;
    for (int64_t g = 0; g < G; ++g) {  // rank order: the sum is reproducible
        f += tails[(size_t)(6 * g)];
        nd += tails[(size_t)(6 * g + 1)];
        ml = std::min(ml, tails[(size_t)(6 * g + 2)]);
        tot += tails[(size_t)(6 * g + 4)];
    }
    o.best_worker = (int32_t)ggid;
    o.best_sample_objective = gobj;
    o.clustering_time = ml;  // engine.hpp:472-475 over every rank's workers
    // lockstep: every t_w equals R, so the first finisher is global worker 0 (rank 0's worker 0)
    o.clustering_time_first_finisher = tails[3] >= 0 ? tails[3] : 0.0;
    if (want_obj) {
        o.full_objective = f;
        o.has_full_objective = 1;
    }
    o.last_timestamp = R > 0 ? ts_of(R - 1) : 0.0;
    o.total_samples = (uint64_t)tot;
    o.distance_evals = (int64_t)nd;
    o.n_publications = npub;
    if (worker_obj) std::memcpy(worker_obj, hobj.data(), (size_t)W * 8);
    o.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - e->t0).count();
    if (out) *out = o;
    return HPCG_OK;
}

int hpcg_engine_finish(hpcg_engine* e, hpcg_run_out* out, double* centroids, uint8_t* flags, int32_t* labels,
                       double* publications, int64_t pub_cap, double* worker_obj, double* traces, int64_t trace_cap,
                       int64_t* trace_len) {
    std::lock_guard<std::mutex> lk(e->ctx->mu);
    hpcg_ctx* ctx = e->ctx;
    bind_device(ctx->device);
    if (e->xr > 1) {
        (void)publications;
        (void)pub_cap;  // multi-rank: read the (replicated) log with hpcg_engine_publications
        return engine_finish_multi(e, out, centroids, flags, labels, worker_obj, traces, trace_cap, trace_len);
    }
    cudaStream_t st = ctx->stream;
    // free-running schedule: no per-round logs (R = 0 below); the per-worker traces are read further down
    const int64_t W = e->W, k = e->k, n = e->n, kn = k * n, R = e->free_mode ? 0 : e->round;
    const int64_t Rw = std::max<int64_t>(R, 1) * W;
    const bool want_obj = e->cfg.compute_full_objective || e->cfg.compute_assignment;
    const bool want_labels = e->cfg.compute_assignment && labels;
    // resident objective kernels take the valid count from the device: select_best, the
    // valid-subset compaction and f(C,X) are queued back to back and read back once
    const bool dev_obj = want_obj && objective_device_kv(e->ds->dtype, (int)n, (int)k);
    CU(e->scratch_a.reserve((size_t)kn * 8));
    CU(e->scratch_b.reserve((size_t)k * 4));
    CU(e->scratch_c.reserve(8));
    CU(e->fin.reserve(16 + (size_t)kn * 8 + (size_t)k));
    int32_t* sel_d = e->fin.as<int32_t>();
    double* bc_d = reinterpret_cast<double*>(e->fin.as<unsigned char>() + 16);
    uint8_t* bf_d = e->fin.as<uint8_t>() + 16 + kn * 8;
    finish_select_kernel<<<1, 256, 0, st>>>(e->inc_obj.as<double>(), e->inc_c.as<double>(), e->inc_f.as<uint8_t>(),
                                            (int)W, (int)k, (int)n, sel_d, bc_d, bf_d, e->scratch_a.as<double>(),
                                            e->scratch_b.as<int32_t>());
    CU(cudaGetLastError());
    ctx->launches += 1;
    DevBuf lab;
    if (dev_obj) {
        if (want_labels) CU(lab.reserve((size_t)e->ds->m * 4));
        int rc = run_assign(ctx, e->ds, e->scratch_a.as<double>(), e->scratch_b.as<int32_t>(), (int)k,
                            want_labels ? lab.as<int32_t>() : nullptr, nullptr, e->scratch_c.as<double>(), e->blocks,
                            sel_d + 1);
        if (rc) return rc;
    }
    // pinned staging: [inc_obj W][lobj Rw][bc kn][f][ndt][npub][sel 2x i32][errf W][lacc Rw][bf k]
    size_t need = (size_t)(W + Rw + kn + 3) * 8 + 8 + (size_t)W * 4 + (size_t)Rw + (size_t)k;
    // the publication log rides in the same staging (and the same synchronisation) when the host-known
    // bound of its length is small; otherwise it is read after the count is known
    const int64_t pub_stage = (publications && !e->free_mode) ? std::min(e->pub_ub, std::min(pub_cap, e->pub_cap)) : 0;
    const bool pubs_staged = pub_stage > 0 && pub_stage * 32 <= (1 << 20);
    const size_t pub_off = (need + 7) & ~(size_t)7;
    if (pubs_staged) need = pub_off + (size_t)pub_stage * 32;
    if (need > ctx->pin_bytes) {  // context-level: one allocation across engines / calls
        if (ctx->pin) cudaFreeHost(ctx->pin);
        ctx->pin = nullptr;
        ctx->pin_bytes = 0;
        CU(cudaHostAlloc(&ctx->pin, need, cudaHostAllocDefault));
        ctx->pin_bytes = need;
    }
    double* h_obj = static_cast<double*>(ctx->pin);
    double* h_lobj = h_obj + W;
    double* h_bc = h_lobj + Rw;
    double* h_f = h_bc + kn;
    unsigned long long* h_ndt = reinterpret_cast<unsigned long long*>(h_f + 1);
    int64_t* h_npub = reinterpret_cast<int64_t*>(h_f + 2);
    int32_t* h_sel = reinterpret_cast<int32_t*>(h_f + 3);
    int32_t* h_errf = h_sel + 2;
    uint8_t* h_lacc = reinterpret_cast<uint8_t*>(h_errf + W);
    uint8_t* h_bf = h_lacc + Rw;
    double* h_pubs = reinterpret_cast<double*>(static_cast<unsigned char*>(ctx->pin) + pub_off);
    {
        CU(e->fin_stage.reserve(need));
        PackParams pk = {};
        pk.dst = e->fin_stage.as<unsigned char>();
        unsigned char* hb = static_cast<unsigned char*>(ctx->pin);
        auto add = [&](const void* src, const void* host_at, size_t bytes) {
            if (bytes == 0) return;
            pk.seg[pk.n++] = PackSeg{static_cast<const unsigned char*>(src),
                                     (int64_t)(static_cast<const unsigned char*>(host_at) - hb), (int64_t)bytes};
        };
        add(e->inc_obj.p, h_obj, (size_t)W * 8);
        add(e->err_first.p, h_errf, (size_t)W * 4);
        if (R > 0) {
            add(e->log_acc.p, h_lacc, (size_t)(R * W));
            add(e->log_obj.p, h_lobj, (size_t)(R * W) * 8);
        }
        add(e->nd_total.p, h_ndt, 8);
        add(e->pub_count.p, h_npub, 8);
        add(sel_d, h_sel, 8);
        add(bc_d, h_bc, (size_t)kn * 8);
        add(bf_d, h_bf, (size_t)k);
        if (dev_obj) add(e->scratch_c.p, h_f, 8);
        if (pubs_staged) add(e->pub_log.p, h_pubs, (size_t)pub_stage * 32);
        pack_segments_kernel<<<8, 256, 0, st>>>(pk);
        CU(cudaGetLastError());
        ctx->launches += 1;
        CU(cudaMemcpyAsync(ctx->pin, e->fin_stage.p, need, cudaMemcpyDeviceToHost, st));
    }
    CU(cudaStreamSynchronize(st));
    const unsigned long long ndt = *h_ndt;
    const int64_t npub = *h_npub;
    // worker errors are rethrown after the join, lowest worker first (engine.hpp:330-331)
    for (int64_t w = 0; w < W; ++w) {
        if (h_errf[w] == kErrDegenerateInit) return fail(HPCG_EINVAL, "kmeans: degenerate centroid in init");
        if (h_errf[w] == kErrMonotone) return fail(HPCG_ELOGIC, "kmeans: objective increased between iterations");
    }
    // select_best (engine.hpp:180-194), evaluated on the device above
    const int best = h_sel[0];
    if (best < 0) return fail(HPCG_ENOSOL, "no solution produced: every worker incumbent is infinite");
    const double best_f = h_obj[best];
    hpcg_run_out o = {};
    o.best_worker = e->cfg.worker_base + best;
    o.best_sample_objective = best_f;
    // traces: lockstep timestamps are samples_processed + 1 = round + 1 (engine.hpp:413); wall
    // clock: seconds at the end of the round (strictly increasing per worker, engine.hpp:258-262)
    auto ts_of = [&](int64_t r) { return e->wall && r < (int64_t)e->t_end.size() ? e->t_end[(size_t)r] : (double)(r + 1); };
    double min_last = kInf;
    std::vector<double> last_ts((size_t)W, -1.0);
    for (int64_t w = 0; w < W; ++w) {
        int64_t cnt = 0;
        for (int64_t r = 0; r < R; ++r) {
            if (!h_lacc[r * W + w]) continue;
            if (traces && cnt < trace_cap) {
                traces[(w * trace_cap + cnt) * 2 + 0] = ts_of(r);
                traces[(w * trace_cap + cnt) * 2 + 1] = h_lobj[r * W + w];
            }
            last_ts[(size_t)w] = ts_of(r);
            ++cnt;
        }
        if (trace_len) trace_len[w] = cnt;
        if (cnt > 0) min_last = std::min(min_last, last_ts[(size_t)w]);
    }
    o.clustering_time = min_last;  // engine.hpp:472-475
    // every worker has t_w = R in lockstep, so the first finisher is worker 0 (engine.hpp:477-481)
    o.clustering_time_first_finisher = last_ts[0] >= 0 ? last_ts[0] : 0.0;
    int64_t free_samples = 0;
    double free_last = 0.0;
    if (e->free_mode) {  // each worker's own trace, sample count and clock
        std::vector<int64_t> cnt((size_t)W), smp((size_t)W);
        std::vector<double> tw((size_t)W), tr((size_t)(W * e->fr_cap * 2));
        CU(d2h(cnt.data(), e->fr_tcnt.as<int64_t>(), (size_t)W, st));
        CU(d2h(smp.data(), e->fr_samples.as<int64_t>(), (size_t)W, st));
        CU(d2h(tw.data(), e->fr_tw.as<double>(), (size_t)W, st));
        CU(d2h(tr.data(), e->fr_trace.as<double>(), tr.size(), st));
        CU(cudaStreamSynchronize(st));
        min_last = kInf;
        int64_t first = 0;
        for (int64_t w = 0; w < W; ++w) {
            const int64_t kept = std::min(cnt[(size_t)w], e->fr_cap);
            const double* t = tr.data() + w * e->fr_cap * 2;
            if (traces)
                for (int64_t i = 0; i < std::min(kept, trace_cap); ++i) {
                    // a trace longer than the caller's buffer keeps its latest entries
                    const int64_t src = kept > trace_cap ? kept - trace_cap + i : i;
                    traces[(w * trace_cap + i) * 2 + 0] = t[src * 2];
                    traces[(w * trace_cap + i) * 2 + 1] = t[src * 2 + 1];
                }
            if (trace_len) trace_len[w] = std::min(kept, trace_cap);
            last_ts[(size_t)w] = kept > 0 ? t[(kept - 1) * 2] : -1.0;
            if (kept > 0) min_last = std::min(min_last, last_ts[(size_t)w]);
            free_samples += smp[(size_t)w];
            free_last = std::max(free_last, tw[(size_t)w]);
            if (tw[(size_t)w] < tw[(size_t)first]) first = w;  // engine.hpp:477-479, strict <
        }
        o.clustering_time = min_last;
        o.clustering_time_first_finisher = last_ts[(size_t)first] >= 0 ? last_ts[(size_t)first] : 0.0;
    }
    std::vector<double> bc(h_bc, h_bc + kn);
    std::vector<uint8_t> bf(h_bf, h_bf + k);
    if (centroids) std::memcpy(centroids, bc.data(), (size_t)kn * 8);
    if (flags) std::memcpy(flags, bf.data(), (size_t)k);
    int64_t final_nd = 0;
    if (dev_obj) {  // engine.hpp:483-491
        const int kv = h_sel[1];
        if (kv == 0) return fail(HPCG_EINVAL, "assignment: every centroid is degenerate");
        if (want_labels) {
            CU(d2h(labels, lab.as<int32_t>(), (size_t)e->ds->m, st));
            CU(cudaStreamSynchronize(st));
        }
        o.full_objective = *h_f;
        o.has_full_objective = 1;
        final_nd = e->ds->m * (int64_t)kv;
    } else if (want_obj) {  // grid-wide objective: exact valid count needed on the host
        std::vector<double> cv;
        std::vector<int32_t> remap;
        for (int64_t j = 0; j < k; ++j)
            if (!bf[(size_t)j]) {
                remap.push_back((int32_t)j);
                cv.insert(cv.end(), bc.begin() + j * n, bc.begin() + (j + 1) * n);
            }
        if (remap.empty()) return fail(HPCG_EINVAL, "assignment: every centroid is degenerate");
        CU(h2d(e->scratch_a.as<double>(), cv.data(), cv.size(), st));
        CU(h2d(e->scratch_b.as<int32_t>(), remap.data(), remap.size(), st));
        if (want_labels) CU(lab.reserve((size_t)e->ds->m * 4));
        int rc = run_assign(ctx, e->ds, e->scratch_a.as<double>(), e->scratch_b.as<int32_t>(), (int)remap.size(),
                            want_labels ? lab.as<int32_t>() : nullptr, nullptr, e->scratch_c.as<double>(), e->blocks);
        if (rc) return rc;
        double f = 0;
        CU(d2h(&f, e->scratch_c.as<double>(), 1, st));
        if (want_labels) CU(d2h(labels, lab.as<int32_t>(), (size_t)e->ds->m, st));
        CU(cudaStreamSynchronize(st));
        o.full_objective = f;
        o.has_full_objective = 1;
        final_nd = e->ds->m * (int64_t)remap.size();
    }
    o.last_timestamp = e->free_mode ? free_last : R > 0 ? ts_of(R - 1) : 0.0;  // every worker's t_w (engine.hpp:250)
    o.total_samples = e->free_mode ? (uint64_t)free_samples : (uint64_t)(W * R);
    o.distance_evals = (int64_t)ndt + final_nd;
    o.n_publications = npub;
    if (publications && npub > 0) {
        const int64_t cnt = std::min(npub, std::min(pub_cap, e->pub_cap));
        if (pubs_staged && cnt <= pub_stage) {
            std::memcpy(publications, h_pubs, (size_t)cnt * 32);
        } else {
            CU(d2h(publications, e->pub_log.as<double>(), (size_t)(cnt * 4), st));
            CU(cudaStreamSynchronize(st));
        }
    }
    if (worker_obj) std::memcpy(worker_obj, h_obj, (size_t)W * 8);
    o.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - e->t0).count();
    if (out) *out = o;
    return HPCG_OK;
}

int hpcg_engine_round_outcome(hpcg_engine* e, double* objective, int32_t* iterations, int32_t* stop, int64_t* n_d,
                              uint8_t* accepted, int32_t* filled) {
    std::lock_guard<std::mutex> lk(e->ctx->mu);
    hpcg_ctx* ctx = e->ctx;
    bind_device(ctx->device);
    const size_t W = (size_t)e->W;
    if (objective) CU(d2h(objective, e->objb.as<double>(), W, ctx->stream));
    if (iterations) CU(d2h(iterations, e->iters.as<int32_t>(), W, ctx->stream));
    if (stop) CU(d2h(stop, e->stopb.as<int32_t>(), W, ctx->stream));
    if (n_d) CU(d2h(n_d, e->nd.as<int64_t>(), W, ctx->stream));
    if (accepted) CU(d2h(accepted, e->acc.as<uint8_t>(), W, ctx->stream));
    if (filled) CU(d2h(filled, e->filled.as<int32_t>(), W, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    return HPCG_OK;
}

int hpcg_engine_publications(hpcg_engine* e, double* publications, int64_t cap, int64_t* n_out) {
    std::lock_guard<std::mutex> lk(e->ctx->mu);
    hpcg_ctx* ctx = e->ctx;
    bind_device(ctx->device);
    int64_t npub = 0;
    CU(d2h(&npub, e->pub_count.as<int64_t>(), 1, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    const int64_t cnt = std::min(npub, std::min(cap, e->pub_cap));
    if (publications && cnt > 0) {
        CU(d2h(publications, e->pub_log.as<double>(), (size_t)(cnt * 4), ctx->stream));
        CU(cudaStreamSynchronize(ctx->stream));
    }
    if (n_out) *n_out = npub;
    return HPCG_OK;
}

int hpcg_engine_worker_incumbents(hpcg_engine* e, double* C_out, uint8_t* f_out, double* obj_out) {
    std::lock_guard<std::mutex> lk(e->ctx->mu);
    hpcg_ctx* ctx = e->ctx;
    bind_device(ctx->device);
    const int64_t W = e->W, k = e->k, kn = k * e->n;
    if (C_out) CU(d2h(C_out, e->inc_c.as<double>(), (size_t)(W * kn), ctx->stream));
    if (f_out) CU(d2h(f_out, e->inc_f.as<uint8_t>(), (size_t)(W * k), ctx->stream));
    if (obj_out) CU(d2h(obj_out, e->inc_obj.as<double>(), (size_t)W, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    return HPCG_OK;
}

int hpcg_engine_destroy(hpcg_engine* e) {
    if (e) {
        bind_device(e->device);
        delete e;
    }
    return HPCG_OK;
}

int hpcg_run(hpcg_ctx* ctx, const void* X_host, hpcg_dtype dtype, int64_t m, int64_t n, const hpcg_engine_cfg* cfg,
             hpcg_run_out* out, double* centroids, uint8_t* flags, int32_t* labels, double* publications,
             int64_t pub_cap, double* worker_obj, double* traces, int64_t trace_cap, int64_t* trace_len) {
    const auto t0 = std::chrono::steady_clock::now();
    hpcg_dataset* ds = nullptr;
    if (int rc = dataset_upload(ctx, X_host, dtype, m, n, &ds, false)) return rc;
    hpcg_engine* e = nullptr;
    int rc = hpcg_engine_create(ctx, ds, cfg, &e);
    if (!rc) {
        e->t0 = t0;
        rc = hpcg_engine_run(e);
    }
    if (!rc)
        rc = hpcg_engine_finish(e, out, centroids, flags, labels, publications, pub_cap, worker_obj, traces,
                                trace_cap, trace_len);
    if (rc) cudaStreamSynchronize(ctx->stream);  // the upload may still read X_host
    hpcg_engine_destroy(e);
    hpcg_dataset_destroy(ds);
    return rc;
}

// ------------------------------------------------------------ synthetic data
// Seeded Gaussian mixture keyed by global row index: row i picks its component by
// inverse CDF of the weights, then coordinates mean + sigma * N(0,1) (Box-Muller on
// splitmix64-hashed counters); a noise_frac share of rows is uniform in the noise box.
int hpcg_gen_mixture(void* X_out, hpcg_dtype dtype, int64_t m, int64_t n, int64_t n_comp, const double* means,
                     const double* sigmas, const double* weights, double noise_frac, double noise_lo,
                     double noise_hi, uint64_t seed, int n_threads) {
    if (m < 1 || n < 1 || n_comp < 1) return fail(HPCG_EINVAL, "gen_mixture: bad shape");
    std::vector<double> cum((size_t)n_comp);
    double t = 0;
    for (int64_t c = 0; c < n_comp; ++c) cum[(size_t)c] = (t += weights ? weights[c] : 1.0);
    for (auto& v : cum) v /= t;
    const uint64_t key = splitmix64(seed ^ 0x6d69787475726531ULL);
    auto u01 = [](uint64_t h) { return ((double)(h >> 11) + 0.5) * 0x1.0p-53; };
    auto work = [&](int64_t b, int64_t e_) {
        for (int64_t i = b; i < e_; ++i) {
            const uint64_t hr = splitmix64(key ^ splitmix64((uint64_t)i));
            const bool noise = u01(splitmix64(hr ^ 0x11)) < noise_frac;
            const double uc = u01(splitmix64(hr ^ 0x22));
            int64_t comp = 0;
            while (comp < n_comp - 1 && cum[(size_t)comp] <= uc) ++comp;
            for (int64_t d = 0; d < n; d += 2) {
                const uint64_t hd = splitmix64(hr + 0x9e3779b97f4a7c15ULL * (uint64_t)(d + 1));
                double v0, v1;
                if (noise) {
                    v0 = noise_lo + (noise_hi - noise_lo) * u01(hd);
                    v1 = noise_lo + (noise_hi - noise_lo) * u01(splitmix64(hd));
                } else {
                    const double a = u01(hd), bb = u01(splitmix64(hd));
                    const double r = std::sqrt(-2.0 * std::log(a));
                    v0 = means[comp * n + d] + sigmas[comp] * r * std::cos(6.283185307179586 * bb);
                    v1 = d + 1 < n ? means[comp * n + d + 1] + sigmas[comp] * r * std::sin(6.283185307179586 * bb) : 0;
                }
                if (dtype == HPCG_F32) {
                    float* X = static_cast<float*>(X_out) + i * n;
                    X[d] = (float)v0;
                    if (d + 1 < n) X[d + 1] = (float)v1;
                } else {
                    double* X = static_cast<double*>(X_out) + i * n;
                    X[d] = v0;
                    if (d + 1 < n) X[d + 1] = v1;
                }
            }
        }
    };
    int T = n_threads > 0 ? n_threads : (int)std::max(1u, std::thread::hardware_concurrency());
    if (m < 4096) T = 1;
    std::vector<std::thread> th;
    for (int ti = 0; ti < T; ++ti) {
        int64_t b, e_;
        chunk_range(m, T, ti, b, e_);
        th.emplace_back(work, b, e_);
    }
    for (auto& x : th) x.join();
    return HPCG_OK;
}

}  // extern "C"
