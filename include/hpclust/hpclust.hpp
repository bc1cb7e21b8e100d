// hpclust/hpclust.hpp — C++ drop-in for the reference's hot-path API (namespace hpclust,
// same public types and signatures as /root/reference/proj/include/hpclust), backed by the
// sm_100a kernels of libhpcg.so through the C-ABI in hpcg.h. Link with -lhpcg.
//
//   reference header      replaced symbols (reference file:line)
//   core.hpp              Dataset 34-50, CentroidSet 64-92, Assignment 95-98, DistCounter 23-31,
//                         squared_distance 100-108, ParallelPolicy 112-123,
//                         assign_nearest 212-221, mssc_objective 224-233
//   lloyd.hpp             LloydConfig 10-20, LloydStop 22-31, LloydOutcome 33-40,
//                         update_centroids 44-71, kmeans 100-164
//   seeding.hpp           SeedConfig 11-14, kmeanspp_seed 113-121, reinit_degenerate 125-133
//   rng.hpp               splitmix64 12-17, RngStream 26-99
//   engine.hpp            StrategyKind/Strategy 22-46, EngineConfig 48-87, TraceEntry/WorkerState
//                         89-102, PublicationRecord 104-109, SharedBest 114-157, NoSolutionError
//                         159-161, draw_sample 165-177, select_best 180-194, final_assignment
//                         197-205, assign_valid_subset 211-229, worker_step 238-267,
//                         ClusteringResult 269-284, run 444-499
//
// Semantics: identical results to the reference for the same inputs and streams (labels and
// counts bit-exact; centroids / objectives within 1e-12 relative, the fixed-order device
// reductions differing from the sequential host sums only in rounding). Error behaviour:
// the same exception types and message texts. Device parallelism replaces ParallelPolicy
// (accepted, ignored). run() supports both schedules: lockstep (max_samples, deterministic) and
// the wall-clock one (time_limit; rounds until the limit, see hpcg_engine_run in hpcg.h).
#pragma once

#include <algorithm>
#include <atomic>
#include <barrier>
#include <exception>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <memory>
#include <mutex>
#include <optional>
#include <random>
#include <span>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_map>
#include <type_traits>
#include <utility>
#include <vector>

#include "../hpcg.h"
#include "parallel.hpp"

namespace hpclust {

// ------------------------------------------------------------------ errors
inline void require(bool cond, const char* msg) {
    if (!cond) throw std::invalid_argument(msg);
}

struct NoSolutionError : std::runtime_error {
    NoSolutionError() : std::runtime_error("no solution produced: every worker incumbent is infinite") {}
};

namespace gpu {
// Map a C-ABI status onto the reference's exception types (messages are the reference's).
inline void check(int rc) {
    if (rc == HPCG_OK) return;
    const std::string msg = hpcg_last_error();
    switch (rc) {
        case HPCG_EINVAL: throw std::invalid_argument(msg);
        case HPCG_ELOGIC: throw std::logic_error(msg);
        case HPCG_ENOSOL: throw NoSolutionError();
        default: throw std::runtime_error("hpcg: " + msg);
    }
}

// Process-wide device context (device 0), created on first use; thread-safe (C++11 statics).
inline hpcg_ctx* context() {
    struct Holder {
        hpcg_ctx* c = nullptr;
        Holder() {
            // these headers mirror one struct layout of hpcg.h: refuse a library built from another
            if (hpcg_abi_version() != HPCG_ABI_VERSION)
                throw std::runtime_error("hpcg: libhpcg.so ABI version differs from include/hpcg.h (rebuild the library)");
            check(hpcg_ctx_create(0, &c));
        }
        ~Holder() { hpcg_ctx_destroy(c); }
    };
    static Holder h;
    return h.c;
}

// RAII handle over a device copy of a host matrix.
struct DeviceMatrix {
    hpcg_dataset* ds = nullptr;
    DeviceMatrix(const double* X, std::size_t m, std::size_t n) {
        check(hpcg_dataset_upload(context(), X, HPCG_F64, (int64_t)m, (int64_t)n, &ds));
    }
    ~DeviceMatrix() { hpcg_dataset_destroy(ds); }
    DeviceMatrix(const DeviceMatrix&) = delete;
    DeviceMatrix& operator=(const DeviceMatrix&) = delete;
};
}  // namespace gpu

// ----------------------------------------------------------------- counters
struct DistCounter {
    std::atomic<std::int64_t> count{0};
    void add(std::int64_t v) { count.fetch_add(v, std::memory_order_relaxed); }
    std::int64_t value() const { return count.load(std::memory_order_relaxed); }
};

inline void count_distances(DistCounter* c, std::int64_t v) {
    if (c) c->add(v);
}

// ------------------------------------------------------------------- data types
struct Dataset {  // row-major m x n, finite entries
    std::vector<double> values;
    std::size_t rows = 0;
    std::size_t cols = 0;

    Dataset() = default;
    Dataset(std::size_t m, std::size_t n) : values(m * n, 0.0), rows(m), cols(n) {}
    std::span<const double> row(std::size_t i) const { return {values.data() + i * cols, cols}; }
    std::span<double> row(std::size_t i) { return {values.data() + i * cols, cols}; }
    void validate() const {
        require(rows >= 1 && cols >= 1, "Dataset: needs at least one row and one column");
        require(std::all_of(values.begin(), values.end(), [](double v) { return std::isfinite(v); }),
                "Dataset: entries must be finite");
    }
};

inline Dataset dataset_from_rows(const std::vector<std::vector<double>>& in) {
    require(!in.empty(), "dataset_from_rows: empty input");
    Dataset d(in.size(), in.front().size());
    for (std::size_t i = 0; i < in.size(); ++i) {
        require(in[i].size() == d.cols, "dataset_from_rows: ragged rows");
        std::copy(in[i].begin(), in[i].end(), d.row(i).begin());
    }
    return d;
}

struct CentroidSet {  // k x n centres + degenerate flags
    std::vector<double> centers;
    std::vector<std::uint8_t> degenerate;
    std::size_t k = 0;
    std::size_t cols = 0;

    CentroidSet() = default;
    CentroidSet(std::size_t k_, std::size_t n) : centers(k_ * n, 0.0), degenerate(k_, 0), k(k_), cols(n) {}
    static CentroidSet all_degenerate(std::size_t k, std::size_t n) {
        CentroidSet c(k, n);
        std::fill(c.degenerate.begin(), c.degenerate.end(), std::uint8_t{1});
        return c;
    }
    std::span<const double> center(std::size_t j) const { return {centers.data() + j * cols, cols}; }
    std::span<double> center(std::size_t j) { return {centers.data() + j * cols, cols}; }
    bool any_degenerate() const {
        return std::any_of(degenerate.begin(), degenerate.end(), [](std::uint8_t f) { return f != 0; });
    }
    std::size_t degenerate_count() const {
        return (std::size_t)std::count(degenerate.begin(), degenerate.end(), std::uint8_t{1});
    }
    bool operator==(const CentroidSet& o) const {
        return k == o.k && cols == o.cols && centers == o.centers && degenerate == o.degenerate;
    }
};

struct Assignment {
    std::vector<std::int32_t> labels;
    std::vector<std::int64_t> counts;
};

inline double squared_distance(std::span<const double> a, std::span<const double> b) {
    require(a.size() == b.size(), "squared_distance: dimension mismatch");
    double s = 0.0;
    for (std::size_t d = 0; d < a.size(); ++d) {
        const double t = a[d] - b[d];
        s += t * t;
    }
    return s;
}

// Accepted for source compatibility; the device decides its own (fixed, deterministic) split.
struct ParallelPolicy {
    bool enabled = false;
    std::size_t n_chunks = 1;
    static ParallelPolicy sequential() { return {false, 1}; }
    static ParallelPolicy threads(std::size_t n) { return {n > 1, std::max<std::size_t>(n, 1)}; }
    std::size_t chunks_for(std::size_t rows) const { return (!enabled || rows == 0) ? 1 : std::min(n_chunks, rows); }
};

// ------------------------------------------------------------------- rng.hpp
inline std::uint64_t splitmix64(std::uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

// The reference stream: std::mt19937_64 plus hand-rolled distributions, so draws are the
// reference's bit for bit. Kernels consume draws produced here (parity mode).
class RngStream {
public:
    explicit RngStream(std::uint64_t seed) : g_(seed) {}
    static RngStream derive(std::uint64_t master, std::uint64_t domain, std::uint64_t index) {
        return RngStream(splitmix64(master ^ splitmix64(domain ^ splitmix64(index))));
    }
    std::uint64_t next_u64() { return g_(); }
    double next_unit() { return (double)(g_() >> 11) * 0x1.0p-53; }
    std::size_t uniform_index(std::size_t n) {
        if (n == 0) throw std::invalid_argument("uniform_index: n must be positive");
        const std::uint64_t top = std::numeric_limits<std::uint64_t>::max();
        const std::uint64_t cut = top - top % (std::uint64_t)n;
        std::uint64_t v = g_();
        while (v >= cut) v = g_();
        return (std::size_t)(v % n);
    }
    double uniform(double lo, double hi) { return lo + (hi - lo) * next_unit(); }
    double normal() {
        if (spare_ok_) {
            spare_ok_ = false;
            return spare_;
        }
        double a, b, r;
        do {
            a = 2.0 * next_unit() - 1.0;
            b = 2.0 * next_unit() - 1.0;
            r = a * a + b * b;
        } while (r >= 1.0 || r == 0.0);
        const double f = std::sqrt(-2.0 * std::log(r) / r);
        spare_ = b * f;
        spare_ok_ = true;
        return a * f;
    }
    double normal(double mean, double sd) { return mean + sd * normal(); }
    std::size_t weighted_index(std::span<const double> cum) {
        const double tot = cum.back();
        if (!(tot > 0.0)) throw std::invalid_argument("weighted_index: total weight must be positive");
        const double u = next_unit() * tot;
        const std::size_t i = (std::size_t)(std::upper_bound(cum.begin(), cum.end(), u) - cum.begin());
        return i < cum.size() ? i : cum.size() - 1;  // first cumulative weight above u
    }

private:
    std::mt19937_64 g_;
    double spare_ = 0.0;
    bool spare_ok_ = false;
};

// ----------------------------------------------------------- assignment / objective
// ------------------------------------------------------- device-resident datasets
enum class Precision { f64, f32 };

// X resident in HBM (ADDITIVE to the reference API): upload once -- in fp64, or
// rounded to fp32 (the north star's fp32 mode) -- or borrow device memory, then pass it to the
// overloads of draw_sample, worker_step, assign_nearest, mssc_objective, final_assignment,
// detail::assign_valid_subset and run below, which read it in place (no per-call upload of X; a
// 64 GB X need not live in a host std::vector<double>).
class DeviceDataset {
public:
    explicit DeviceDataset(const Dataset& X, Precision p = Precision::f64) : rows(X.rows), cols(X.cols), precision(p) {
        X.validate();
        if (p == Precision::f64) {
            gpu::check(hpcg_dataset_upload(gpu::context(), X.values.data(), HPCG_F64, (int64_t)rows, (int64_t)cols, &ds_));
        } else {
            std::vector<float> v(X.values.begin(), X.values.end());
            gpu::check(hpcg_dataset_upload(gpu::context(), v.data(), HPCG_F32, (int64_t)rows, (int64_t)cols, &ds_));
        }
    }
    // borrow row-major m x n device memory of the default context's device (must outlive this)
    static DeviceDataset borrow(const void* dev, std::size_t m, std::size_t n, Precision p) {
        DeviceDataset d;
        d.rows = m;
        d.cols = n;
        d.precision = p;
        gpu::check(hpcg_dataset_wrap(gpu::context(), dev, p == Precision::f64 ? HPCG_F64 : HPCG_F32, (int64_t)m,
                                     (int64_t)n, &d.ds_));
        return d;
    }
    DeviceDataset(DeviceDataset&& o) noexcept : rows(o.rows), cols(o.cols), precision(o.precision), ds_(o.ds_) {
        o.ds_ = nullptr;
    }
    DeviceDataset& operator=(DeviceDataset&& o) noexcept {
        std::swap(ds_, o.ds_);
        rows = o.rows;
        cols = o.cols;
        precision = o.precision;
        return *this;
    }
    DeviceDataset(const DeviceDataset&) = delete;
    DeviceDataset& operator=(const DeviceDataset&) = delete;
    ~DeviceDataset() {
        if (ds_) hpcg_dataset_destroy(ds_);
    }
    hpcg_dataset* handle() const { return ds_; }
    std::size_t rows = 0, cols = 0;
    Precision precision = Precision::f64;

private:
    DeviceDataset() = default;
    hpcg_dataset* ds_ = nullptr;
};

namespace gpu {
inline std::pair<Assignment, double> assign_ds(hpcg_dataset* ds, std::size_t rows, const CentroidSet& C, bool strict,
                                               bool want_labels, DistCounter* counter) {
    Assignment a;
    if (want_labels) a.labels.resize(rows);
    a.counts.assign(C.k, 0);
    double cost = 0.0;
    std::int64_t nd = 0;
    check(hpcg_assign(context(), ds, C.centers.data(), C.degenerate.data(), (int64_t)C.k, strict ? 1 : 0,
                      want_labels ? a.labels.data() : nullptr, a.counts.data(), &cost, &nd));
    count_distances(counter, nd);
    return {std::move(a), cost};
}
inline std::pair<Assignment, double> assign(const Dataset& X, const CentroidSet& C, bool strict, bool want_labels,
                                            DistCounter* counter) {
    DeviceMatrix dm(X.values.data(), X.rows, X.cols);
    return assign_ds(dm.ds, X.rows, C, strict, want_labels, counter);
}
inline std::pair<Assignment, double> assign(const DeviceDataset& X, const CentroidSet& C, bool strict, bool want_labels,
                                            DistCounter* counter) {
    return assign_ds(X.handle(), X.rows, C, strict, want_labels, counter);
}
}  // namespace gpu

// XS: Dataset (the reference signature; uploaded per call) or DeviceDataset (resident, additive)
template <typename XS>
concept AnyDataset = std::is_same_v<XS, Dataset> || std::is_same_v<XS, DeviceDataset>;

template <AnyDataset XS>
inline Assignment assign_nearest(const XS& X, const CentroidSet& C, const ParallelPolicy& = ParallelPolicy::sequential(),
                                 DistCounter* counter = nullptr) {
    require(C.k >= 1, "assign_nearest: need at least one centroid");
    require(C.cols == X.cols, "assign_nearest: dimension mismatch");
    require(!C.any_degenerate(), "assign_nearest: degenerate centroid present");
    return gpu::assign(X, C, true, true, counter).first;
}

template <AnyDataset XS>
inline double mssc_objective(const CentroidSet& C, const XS& X, const ParallelPolicy& = ParallelPolicy::sequential(),
                             DistCounter* counter = nullptr) {
    require(C.k >= 1, "mssc_objective: need at least one centroid");
    require(C.cols == X.cols, "mssc_objective: dimension mismatch");
    require(!C.any_degenerate(), "mssc_objective: degenerate centroid present");
    return gpu::assign(X, C, true, false, counter).second;
}

template <AnyDataset XS>
inline std::pair<Assignment, double> final_assignment(const XS& X, const CentroidSet& C,
                                                      const ParallelPolicy& = ParallelPolicy::sequential(),
                                                      DistCounter* counter = nullptr) {
    require(!C.any_degenerate(), "final_assignment: degenerate centroid present");
    require(C.cols == X.cols, "final_assignment: dimension mismatch");
    return gpu::assign(X, C, true, true, counter);
}

namespace detail {
template <AnyDataset XS>
inline std::pair<Assignment, double> assign_valid_subset(const XS& X, const CentroidSet& C, const ParallelPolicy&,
                                                         DistCounter* counter) {
    if (!C.any_degenerate()) return final_assignment(X, C, ParallelPolicy::sequential(), counter);
    require(C.degenerate_count() < C.k, "assignment: every centroid is degenerate");
    return gpu::assign(X, C, false, true, counter);
}
}  // namespace detail

// ----------------------------------------------------------------------- lloyd.hpp
struct LloydConfig {
    std::size_t max_iters = 300;
    double rel_tol = 1e-4;
    bool parallel_rows = false;
    std::size_t n_threads = 0;
    ParallelPolicy policy() const {  // lloyd.hpp:16-19
        if (!parallel_rows) return ParallelPolicy::sequential();
        return ParallelPolicy::threads(n_threads == 0 ? ThreadPool::default_threads() : n_threads);
    }
};

enum class LloydStop { tolerance, max_iters, fixed_point };

inline const char* to_string(LloydStop s) {
    return s == LloydStop::tolerance ? "tolerance" : s == LloydStop::max_iters ? "max_iters" : "fixed_point";
}

struct LloydOutcome {
    CentroidSet centroids;
    Assignment assignment;
    double objective = 0.0;
    std::size_t iterations = 0;
    LloydStop converged_by = LloydStop::max_iters;
    std::vector<double> objective_history;
};

// Host utility (not a hot-path kernel): means of labelled rows, empty -> fallback + flag.
inline CentroidSet update_centroids(const Dataset& S, const Assignment& A, std::size_t k,
                                    const CentroidSet* fallback = nullptr) {
    require(A.labels.size() == S.rows, "update_centroids: label/row mismatch");
    require(A.counts.size() == k, "update_centroids: counts size mismatch");
    CentroidSet out(k, S.cols);
    std::vector<double> acc(k * S.cols, 0.0);
    for (std::size_t i = 0; i < S.rows; ++i) {
        const auto j = (std::size_t)A.labels[i];
        require(j < k, "update_centroids: label out of range");
        for (std::size_t d = 0; d < S.cols; ++d) acc[j * S.cols + d] += S.values[i * S.cols + d];
    }
    for (std::size_t j = 0; j < k; ++j) {
        if (A.counts[j] > 0) {
            const double inv = 1.0 / (double)A.counts[j];
            for (std::size_t d = 0; d < S.cols; ++d) out.centers[j * S.cols + d] = acc[j * S.cols + d] * inv;
        } else {
            if (fallback) std::copy_n(fallback->centers.data() + j * S.cols, S.cols, out.centers.data() + j * S.cols);
            out.degenerate[j] = 1;
        }
    }
    return out;
}

namespace gpu {
struct StepOut {
    std::vector<double> C;
    std::vector<std::uint8_t> f;
    double obj = 0.0;
    std::int32_t iters = 0, stop = 0, filled = 0;
    std::int64_t nd = 0;
    std::vector<std::int32_t> labels;
    std::vector<std::int64_t> counts;
    std::vector<double> history;
};

// One (sample, init) problem on the device: reseed degenerate slots with the draws the
// reference would take from `rng`, then (optionally) Lloyd. rng is left exactly where the
// reference leaves it (draws not consumed because seeding stopped early are rewound).
inline StepOut step_ds(hpcg_dataset* ds, const std::int64_t* idx, std::size_t s, std::size_t n, const CentroidSet& init,
                       const LloydConfig& lc, std::size_t candidates, RngStream* rng, bool do_lloyd);
inline StepOut step(const Dataset& S, const CentroidSet& init, const LloydConfig& lc, std::size_t candidates,
                    RngStream* rng, bool do_lloyd) {
    DeviceMatrix dm(S.values.data(), S.rows, S.cols);
    return step_ds(dm.ds, nullptr, S.rows, S.cols, init, lc, candidates, rng, do_lloyd);
}
// The worker step on rows idx[0..s) of a device dataset (idx == nullptr: ds is the sample itself).
inline StepOut step_ds(hpcg_dataset* ds, const std::int64_t* idx, std::size_t s, std::size_t n, const CentroidSet& init,
                       const LloydConfig& lc, std::size_t candidates, RngStream* rng, bool do_lloyd) {
    const std::size_t k = init.k;
    std::size_t pend = 0;
    for (auto f : init.degenerate) pend += f ? 1 : 0;
    const bool no_valid = pend > 0 && pend == k;
    std::int64_t first = 0;
    std::vector<double> units(std::max<std::size_t>(1, k * candidates), 0.0);
    std::optional<RngStream> snap;
    std::size_t loops = 0;
    if (rng && pend > 0) {
        if (no_valid) first = (std::int64_t)rng->uniform_index(s);
        snap = *rng;
        loops = pend - (no_valid ? 1 : 0);
        for (std::size_t t = 0; t < loops * candidates; ++t) units[t] = rng->next_unit();
    }
    const hpcg_lloyd_cfg cfg{(int64_t)lc.max_iters, lc.rel_tol, (int64_t)candidates};
    StepOut o;
    o.C.resize(k * n);
    o.f.resize(k);
    o.labels.resize(s);
    o.counts.resize(k);
    const int32_t cap = (int32_t)std::min<std::size_t>(lc.max_iters + 1, 100001);
    o.history.resize((std::size_t)cap);
    int32_t hl = 0;
    const int rc = hpcg_worker_step_batched(
        context(), ds, idx, 1, (int64_t)s, init.centers.data(), init.degenerate.data(), (int64_t)k, &cfg,
        &first, units.data(), (int64_t)units.size(), do_lloyd ? 1 : 0, o.C.data(), o.f.data(), &o.obj, &o.iters,
        &o.stop, &o.nd, &o.filled, do_lloyd ? o.labels.data() : nullptr, do_lloyd ? o.counts.data() : nullptr,
        do_lloyd ? o.history.data() : nullptr, do_lloyd ? cap : 0, &hl);
    if (snap && (std::size_t)(o.filled - (no_valid ? 1 : 0)) < loops) {  // seeding.hpp:87 early stop
        RngStream r = *snap;
        for (int64_t t = 0; t < (int64_t)(o.filled - (no_valid ? 1 : 0)) * (int64_t)candidates; ++t) r.next_unit();
        *rng = r;
    }
    check(rc);
    o.history.resize((std::size_t)hl);
    return o;
}
}  // namespace gpu

inline LloydOutcome kmeans(const Dataset& S, const CentroidSet& C_init, const LloydConfig& cfg,
                           DistCounter* counter = nullptr) {
    require(cfg.max_iters >= 1, "kmeans: max_iters must be positive");
    require(cfg.rel_tol > 0.0, "kmeans: rel_tol must be positive");
    require(!C_init.any_degenerate(), "kmeans: degenerate centroid in init");
    require(C_init.cols == S.cols, "kmeans: dimension mismatch");
    auto o = gpu::step(S, C_init, cfg, 1, nullptr, true);
    count_distances(counter, o.nd);
    LloydOutcome out;
    out.centroids.k = C_init.k;
    out.centroids.cols = S.cols;
    out.centroids.centers = std::move(o.C);
    out.centroids.degenerate = std::move(o.f);
    out.assignment.labels = std::move(o.labels);
    out.assignment.counts = std::move(o.counts);
    out.objective = o.obj;
    out.iterations = (std::size_t)o.iters;
    out.converged_by = (LloydStop)o.stop;
    out.objective_history = std::move(o.history);
    return out;
}

// --------------------------------------------------------------------- seeding.hpp
struct SeedConfig {
    std::size_t candidates_per_center = 3;
};

inline CentroidSet reinit_degenerate(const CentroidSet& C, const Dataset& S, const SeedConfig& cfg, RngStream& rng,
                                     const ParallelPolicy& = ParallelPolicy::sequential(),
                                     DistCounter* counter = nullptr) {
    if (!C.any_degenerate()) return C;
    require(S.rows >= 1, "seeding: empty sample");
    require(C.cols == S.cols, "seeding: dimension mismatch");
    require(cfg.candidates_per_center >= 1, "seeding: need at least one candidate");
    auto o = gpu::step(S, C, LloydConfig{}, cfg.candidates_per_center, &rng, false);
    count_distances(counter, o.nd);
    CentroidSet out(C.k, C.cols);
    out.centers = std::move(o.C);
    out.degenerate = std::move(o.f);
    return out;
}

inline CentroidSet kmeanspp_seed(const Dataset& S, std::size_t k, const SeedConfig& cfg, RngStream& rng,
                                 const ParallelPolicy& par = ParallelPolicy::sequential(),
                                 DistCounter* counter = nullptr) {
    require(k >= 1, "kmeanspp_seed: k must be positive");
    return reinit_degenerate(CentroidSet::all_degenerate(k, S.cols), S, cfg, rng, par, counter);
}

// ---------------------------------------------------------------------- engine.hpp
enum class StrategyKind { inner, competitive, cooperative, hybrid };

inline const char* to_string(StrategyKind s) {
    switch (s) {
        case StrategyKind::inner: return "inner";
        case StrategyKind::competitive: return "competitive";
        case StrategyKind::cooperative: return "cooperative";
        case StrategyKind::hybrid: return "hybrid";
    }
    return "?";
}

struct Strategy {
    StrategyKind kind = StrategyKind::competitive;
    double phase_t1 = 0.0;
    double phase_t2 = 0.0;
    static Strategy inner() { return {StrategyKind::inner}; }
    static Strategy competitive() { return {StrategyKind::competitive}; }
    static Strategy cooperative() { return {StrategyKind::cooperative}; }
    static Strategy hybrid(double t1, double t2) { return {StrategyKind::hybrid, t1, t2}; }
};

enum class RngMode { reference, philox };  // extension: stream family of run()

struct EngineConfig {
    std::size_t k = 0;
    std::size_t sample_size = 0;
    std::size_t n_workers = 1;
    double time_limit = std::numeric_limits<double>::infinity();
    std::optional<std::size_t> max_samples;
    Strategy strategy;
    std::uint64_t master_seed = 0;
    SeedConfig seed;
    LloydConfig lloyd;
    std::size_t n_threads = 0;
    bool compute_full_objective = true;
    bool compute_assignment = false;
    RngMode rng_mode = RngMode::reference;  // extension (not in the reference)
    // extension, wall-clock schedule only: free-running workers with immediate publication
    // (run_wall_clock, engine.hpp:348-374) instead of round granularity; needs RngMode::philox
    bool free_running = false;
    std::size_t free_group = 0;  // workers per free-running group (0 = automatic, 1 = every worker alone)

    bool deterministic_mode() const { return !std::isfinite(time_limit) && max_samples.has_value(); }
    double budget() const { return deterministic_mode() ? (double)*max_samples : time_limit; }
    void validate(std::size_t m) const {
        require(k >= 1, "EngineConfig: k must be positive");
        require(sample_size >= 1 && sample_size <= m, "EngineConfig: sample_size must be in [1, m]");
        require(n_workers >= 1, "EngineConfig: need at least one worker");
        require(std::isfinite(time_limit) || max_samples.has_value(),
                "EngineConfig: need a time limit or a max_samples bound");
        if (std::isfinite(time_limit)) require(time_limit > 0.0, "EngineConfig: time limit must be positive");
        if (max_samples) require(*max_samples >= 1, "EngineConfig: max_samples must be positive");
        if (strategy.kind == StrategyKind::hybrid) {
            require(strategy.phase_t1 >= 0.0 && strategy.phase_t2 >= 0.0,
                    "EngineConfig: hybrid phase durations must be nonnegative");
            const double b = budget();
            require(std::abs(strategy.phase_t1 + strategy.phase_t2 - b) <= 1e-9 * std::max(1.0, std::abs(b)),
                    "EngineConfig: hybrid phases must sum to the total budget");
        }
    }
};

struct TraceEntry {
    double timestamp;
    double sample_objective;
};

struct WorkerState {
    int worker_id = 0;
    CentroidSet incumbent;
    double incumbent_objective = std::numeric_limits<double>::infinity();
    double t_w = 0.0;
    std::size_t samples_processed = 0;
    std::vector<TraceEntry> update_trace;
};

struct PublicationRecord {
    std::int64_t version;
    int worker_id;
    double objective;
    double timestamp;
};

// Conditional-publish best incumbent (strict <); snapshots are copies.
class SharedBest {
public:
    struct Snapshot {
        int worker_id;
        double objective;
        CentroidSet centroids;
        std::int64_t version;
    };
    std::optional<Snapshot> snapshot() const {
        std::lock_guard<std::mutex> g(mu_);
        if (!version_) return std::nullopt;
        return Snapshot{worker_, obj_, cs_, version_};
    }
    bool try_publish(int worker_id, double objective, const CentroidSet& c, double timestamp) {
        std::lock_guard<std::mutex> g(mu_);
        if (!(objective < obj_)) return false;
        ++version_;
        worker_ = worker_id;
        obj_ = objective;
        cs_ = c;
        log_.push_back({version_, worker_id, objective, timestamp});
        return true;
    }
    std::int64_t version() const {
        std::lock_guard<std::mutex> g(mu_);
        return version_;
    }
    std::vector<PublicationRecord> publication_log() const {
        std::lock_guard<std::mutex> g(mu_);
        return log_;
    }

private:
    mutable std::mutex mu_;
    std::int64_t version_ = 0;
    int worker_ = -1;
    double obj_ = std::numeric_limits<double>::infinity();
    CentroidSet cs_;
    std::vector<PublicationRecord> log_;
};

// s distinct rows in the reference's draw order: the partial Fisher-Yates replayed in O(s)
// (only displaced slots stored), rows gathered by the device.
namespace detail {
inline std::vector<std::int64_t> draw_indices(std::size_t m, std::size_t s, RngStream& rng) {
    require(s >= 1 && s <= m, "draw_sample: sample size must be in [1, m]");
    std::vector<std::int64_t> idx(s);
    std::unordered_map<std::size_t, std::size_t> moved;
    moved.reserve(2 * s);
    auto at = [&](std::size_t i) {
        auto it = moved.find(i);
        return it == moved.end() ? i : it->second;
    };
    for (std::size_t i = 0; i < s; ++i) {
        const std::size_t j = i + rng.uniform_index(m - i);
        const std::size_t a = at(i), b = at(j);
        moved[i] = b;
        moved[j] = a;
        idx[i] = (std::int64_t)b;
    }
    return idx;
}
}  // namespace detail

inline Dataset draw_sample(const Dataset& X, std::size_t s, RngStream& rng) {
    std::vector<std::int64_t> idx = detail::draw_indices(X.rows, s, rng);
    gpu::DeviceMatrix dm(X.values.data(), X.rows, X.cols);
    Dataset out(s, X.cols);
    gpu::check(hpcg_gather(gpu::context(), dm.ds, idx.data(), (int64_t)s, out.values.data()));
    return out;
}

// device-resident X: only the s sample rows cross PCIe (back to the host Dataset)
inline Dataset draw_sample(const DeviceDataset& X, std::size_t s, RngStream& rng) {
    std::vector<std::int64_t> idx = detail::draw_indices(X.rows, s, rng);
    Dataset out(s, X.cols);
    if (X.precision == Precision::f64) {
        gpu::check(hpcg_gather(gpu::context(), X.handle(), idx.data(), (int64_t)s, out.values.data()));
    } else {
        std::vector<float> f(s * X.cols);
        gpu::check(hpcg_gather(gpu::context(), X.handle(), idx.data(), (int64_t)s, f.data()));
        std::copy(f.begin(), f.end(), out.values.begin());
    }
    return out;
}

inline std::pair<int, const CentroidSet*> select_best(const std::vector<WorkerState>& ws) {
    require(!ws.empty(), "select_best: no workers");
    const WorkerState* best = nullptr;
    for (const auto& w : ws)
        if (w.incumbent_objective < (best ? best->incumbent_objective : std::numeric_limits<double>::infinity()))
            best = &w;
    if (!best) throw NoSolutionError{};
    return {best->worker_id, &best->incumbent};
}

template <typename Clock>
inline bool worker_step(WorkerState& w, RngStream& rng, const Dataset& X, const CentroidSet& init_source,
                        const EngineConfig& cfg, Clock&& clock, DistCounter* counter = nullptr) {
    Dataset S = draw_sample(X, cfg.sample_size, rng);
    CentroidSet init = reinit_degenerate(init_source, S, cfg.seed, rng, ParallelPolicy::sequential(), counter);
    LloydOutcome out = kmeans(S, init, cfg.lloyd, counter);
    ++w.samples_processed;
    double ts = clock();
    w.t_w = ts;
    if (!(out.objective < w.incumbent_objective)) return false;
    if (!w.update_trace.empty()) {
        if (!(out.objective < w.update_trace.back().sample_objective))
            throw std::logic_error("worker_step: non-decreasing incumbent accepted");
        if (!(ts > w.update_trace.back().timestamp))
            ts = std::nextafter(w.update_trace.back().timestamp, std::numeric_limits<double>::infinity());
    }
    w.incumbent = std::move(out.centroids);
    w.incumbent_objective = out.objective;
    w.update_trace.push_back({ts, out.objective});
    return true;
}

// device-resident X: gather, reseed and Lloyd in ONE device call on the resident rows (the same
// draws, in the same order, as draw_sample + reinit_degenerate + kmeans take from rng)
template <typename Clock>
inline bool worker_step(WorkerState& w, RngStream& rng, const DeviceDataset& X, const CentroidSet& init_source,
                        const EngineConfig& cfg, Clock&& clock, DistCounter* counter = nullptr) {
    std::vector<std::int64_t> idx = detail::draw_indices(X.rows, cfg.sample_size, rng);
    require(init_source.cols == X.cols, "seeding: dimension mismatch");
    require(cfg.seed.candidates_per_center >= 1, "seeding: need at least one candidate");
    require(cfg.lloyd.max_iters >= 1, "kmeans: max_iters must be positive");
    require(cfg.lloyd.rel_tol > 0.0, "kmeans: rel_tol must be positive");
    auto o = gpu::step_ds(X.handle(), idx.data(), cfg.sample_size, X.cols, init_source, cfg.lloyd,
                          cfg.seed.candidates_per_center, &rng, true);
    count_distances(counter, o.nd);
    ++w.samples_processed;
    double ts = clock();
    w.t_w = ts;
    if (!(o.obj < w.incumbent_objective)) return false;
    if (!w.update_trace.empty()) {
        if (!(o.obj < w.update_trace.back().sample_objective))
            throw std::logic_error("worker_step: non-decreasing incumbent accepted");
        if (!(ts > w.update_trace.back().timestamp))
            ts = std::nextafter(w.update_trace.back().timestamp, std::numeric_limits<double>::infinity());
    }
    w.incumbent = CentroidSet(init_source.k, X.cols);
    w.incumbent.centers = std::move(o.C);
    w.incumbent.degenerate = std::move(o.f);
    w.incumbent_objective = o.obj;
    w.update_trace.push_back({ts, o.obj});
    return true;
}

struct ClusteringResult {
    CentroidSet centroids;
    std::optional<double> full_objective;
    std::optional<Assignment> assignment;
    int best_worker = 0;
    double best_sample_objective = std::numeric_limits<double>::infinity();
    double clustering_time = 0.0;
    double clustering_time_first_finisher = 0.0;
    double wall_seconds = 0.0;
    std::size_t total_samples = 0;
    std::int64_t distance_evals = 0;
    std::vector<WorkerState> per_worker;
    std::vector<PublicationRecord> publications;
};

// The whole HPClust run on the device: lockstep rounds of gather -> reseed -> Lloyd ->
// keep-the-best -> publication for all workers, select_best, final full-data objective.
namespace detail {
inline ClusteringResult run_ds(hpcg_dataset* ds, std::size_t rows, std::size_t n, const EngineConfig& cfg_in);
}
inline ClusteringResult run(const Dataset& X, const EngineConfig& cfg_in) {
    gpu::DeviceMatrix dm(X.values.data(), X.rows, X.cols);
    return detail::run_ds(dm.ds, X.rows, X.cols, cfg_in);
}
// device-resident X (additive overload): no upload
inline ClusteringResult run(const DeviceDataset& X, const EngineConfig& cfg_in) {
    return detail::run_ds(X.handle(), X.rows, X.cols, cfg_in);
}
inline ClusteringResult detail::run_ds(hpcg_dataset* ds, std::size_t rows, std::size_t n, const EngineConfig& cfg_in) {
    EngineConfig cfg = cfg_in;
    if (cfg.strategy.kind == StrategyKind::inner) cfg.n_workers = 1;
    cfg.validate(rows);
    const std::size_t W = cfg.n_workers, k = cfg.k;
    hpcg_engine_cfg ec{};
    ec.k = (int64_t)k;
    ec.sample_size = (int64_t)cfg.sample_size;
    ec.n_workers = (int64_t)W;
    // lockstep (deterministic_mode) or the wall-clock schedule (engine.hpp:459-462)
    ec.max_samples = cfg.max_samples ? (int64_t)*cfg.max_samples : 0;
    ec.time_limit = cfg.deterministic_mode() ? 0.0 : cfg.time_limit;
    ec.strategy = (int32_t)cfg.strategy.kind;
    ec.phase_t1 = cfg.strategy.phase_t1;
    ec.phase_t2 = cfg.strategy.phase_t2;
    ec.master_seed = cfg.master_seed;
    ec.candidates = (int64_t)cfg.seed.candidates_per_center;
    ec.max_iters = (int64_t)cfg.lloyd.max_iters;
    ec.rel_tol = cfg.lloyd.rel_tol;
    ec.compute_full_objective = cfg.compute_full_objective ? 1 : 0;
    ec.compute_assignment = cfg.compute_assignment ? 1 : 0;
    ec.rng_mode = cfg.rng_mode == RngMode::reference ? HPCG_RNG_REFERENCE : HPCG_RNG_PHILOX;
    ec.free_running = cfg.free_running && !cfg.deterministic_mode() ? 1 : 0;
    ec.free_group = (int32_t)cfg.free_group;
    hpcg_engine* e = nullptr;
    gpu::check(hpcg_engine_create(gpu::context(), ds, &ec, &e));
    std::unique_ptr<hpcg_engine, int (*)(hpcg_engine*)> guard(e, hpcg_engine_destroy);
    gpu::check(hpcg_engine_run(e));
    const std::size_t R = (std::size_t)std::max<std::int64_t>(1, hpcg_engine_round_index(e));
    hpcg_run_out o{};
    ClusteringResult res;
    res.centroids = CentroidSet(k, n);
    std::vector<std::int32_t> labels(cfg.compute_assignment ? rows : 0);
    std::vector<double> wobj(W), traces(W * R * 2);
    std::vector<std::int64_t> tlen(W);
    gpu::check(hpcg_engine_finish(e, &o, res.centroids.centers.data(), res.centroids.degenerate.data(),
                                  cfg.compute_assignment ? labels.data() : nullptr, nullptr, 0, wobj.data(),
                                  traces.data(), (int64_t)R, tlen.data()));
    const std::int64_t pub_cap = o.n_publications;
    std::vector<double> pubs((std::size_t)std::max<std::int64_t>(pub_cap, 1) * 4);
    gpu::check(hpcg_engine_publications(e, pubs.data(), pub_cap, nullptr));
    std::vector<double> incC(W * k * n);
    std::vector<std::uint8_t> incF(W * k);
    gpu::check(hpcg_engine_worker_incumbents(e, incC.data(), incF.data(), nullptr));
    std::vector<std::int64_t> w_samples(W);
    std::vector<double> w_clock(W);
    gpu::check(hpcg_engine_worker_progress(e, w_samples.data(), w_clock.data()));
    if (o.has_full_objective) res.full_objective = o.full_objective;
    if (cfg.compute_assignment) {
        Assignment a;
        a.labels = std::move(labels);
        a.counts.assign(k, 0);
        for (auto l : a.labels) ++a.counts[(std::size_t)l];
        res.assignment = std::move(a);
    }
    res.best_worker = o.best_worker;
    res.best_sample_objective = o.best_sample_objective;
    res.clustering_time = o.clustering_time;
    res.clustering_time_first_finisher = o.clustering_time_first_finisher;
    res.wall_seconds = o.wall_seconds;
    res.total_samples = (std::size_t)o.total_samples;
    res.distance_evals = o.distance_evals;
    for (std::int64_t i = 0; i < std::min<std::int64_t>(o.n_publications, pub_cap); ++i)
        res.publications.push_back({(std::int64_t)pubs[4 * i], (int)pubs[4 * i + 1], pubs[4 * i + 2], pubs[4 * i + 3]});
    res.per_worker.resize(W);
    for (std::size_t w = 0; w < W; ++w) {
        WorkerState& ws = res.per_worker[w];
        ws.worker_id = (int)w;
        ws.incumbent = CentroidSet(k, n);
        std::copy_n(incC.data() + w * k * n, k * n, ws.incumbent.centers.data());
        std::copy_n(incF.data() + w * k, k, ws.incumbent.degenerate.data());
        ws.incumbent_objective = wobj[w];
        ws.samples_processed = (std::size_t)w_samples[w];
        ws.t_w = w_clock[w];  // the clock read after the worker's last step (engine.hpp:250)
        for (std::int64_t t = 0; t < tlen[w]; ++t)
            ws.update_trace.push_back({traces[(w * R + (std::size_t)t) * 2], traces[(w * R + (std::size_t)t) * 2 + 1]});
    }
    return res;
}

// The same run over several GPUs of this node (additive overload): X is row-sharded
// over `devices` (chunk_range, parallel.hpp:106-112), every rank samples over ALL rows through the
// peer-mapped shards (engine.hpp:165-177), the workers are split contiguously over the ranks, and each
// round publishes over every rank's workers through the library's NCCL exchange -- so the result
// equals run(X, cfg) on one GPU (centroids, n_d, best worker, publications; f(C,X) is a sum of shard
// partials). One host thread per device drives its rank.
inline ClusteringResult run(const Dataset& X, const EngineConfig& cfg_in, const std::vector<int>& devices) {
    EngineConfig cfg = cfg_in;
    if (cfg.strategy.kind == StrategyKind::inner) cfg.n_workers = 1;
    cfg.validate(X.rows);
    const std::size_t G = std::min<std::size_t>(devices.size(), cfg.n_workers);
    require(G >= 1, "run: need at least one device");
    if (G == 1 && devices.front() == 0) return run(X, cfg);
    const std::size_t W = cfg.n_workers, k = cfg.k, n = X.cols;
    unsigned char uid[128] = {};
    if (G > 1) gpu::check(hpcg_comm_unique_id(uid));
    std::vector<const void*> shard_ptr(G);
    std::vector<std::int64_t> shard_rows(G);
    std::vector<ClusteringResult> part(G);
    std::vector<std::size_t> w_lo(G), w_hi(G);
    std::vector<std::exception_ptr> errs(G);
    std::barrier sync((std::ptrdiff_t)G);
    auto rank_main = [&](std::size_t g) {
        hpcg_ctx* ctx = nullptr;
        hpcg_dataset *mine = nullptr, *all = nullptr;
        hpcg_engine* e = nullptr;
        bool arrived = false;
        try {
            gpu::check(hpcg_ctx_create(devices[g], &ctx));
            if (G > 1) gpu::check(hpcg_ctx_attach_comm(ctx, (int32_t)G, (int32_t)g, uid));
            const std::size_t base = X.rows / G, extra = X.rows % G;
            const std::size_t r0 = g * base + std::min(g, extra), r1 = r0 + base + (g < extra ? 1 : 0);
            gpu::check(hpcg_dataset_upload(ctx, X.values.data() + r0 * n, HPCG_F64, (int64_t)(r1 - r0), (int64_t)n, &mine));
            shard_ptr[g] = hpcg_dataset_device_ptr(mine);
            shard_rows[g] = (std::int64_t)(r1 - r0);
            sync.arrive_and_wait();  // every shard uploaded
            arrived = true;
            gpu::check(hpcg_dataset_wrap_sharded(ctx, shard_ptr.data(), shard_rows.data(), (int32_t)G, HPCG_F64,
                                                 (int64_t)n, &all));
            const std::size_t wb = W / G, wx = W % G;
            w_lo[g] = g * wb + std::min(g, wx);
            w_hi[g] = w_lo[g] + wb + (g < wx ? 1 : 0);
            hpcg_engine_cfg ec{};
            ec.k = (int64_t)k;
            ec.sample_size = (int64_t)cfg.sample_size;
            ec.n_workers = (int64_t)(w_hi[g] - w_lo[g]);
            ec.max_samples = cfg.max_samples ? (int64_t)*cfg.max_samples : 0;
            ec.time_limit = cfg.deterministic_mode() ? 0.0 : cfg.time_limit;
            ec.strategy = (int32_t)cfg.strategy.kind;
            ec.phase_t1 = cfg.strategy.phase_t1;
            ec.phase_t2 = cfg.strategy.phase_t2;
            ec.master_seed = cfg.master_seed;
            ec.candidates = (int64_t)cfg.seed.candidates_per_center;
            ec.max_iters = (int64_t)cfg.lloyd.max_iters;
            ec.rel_tol = cfg.lloyd.rel_tol;
            ec.compute_full_objective = cfg.compute_full_objective ? 1 : 0;
            ec.compute_assignment = cfg.compute_assignment ? 1 : 0;
            ec.rng_mode = cfg.rng_mode == RngMode::reference ? HPCG_RNG_REFERENCE : HPCG_RNG_PHILOX;
            ec.worker_base = (int32_t)w_lo[g];
            gpu::check(hpcg_engine_create(ctx, all, &ec, &e));
            if (G > 1) gpu::check(hpcg_engine_set_exchange(e, (int32_t)G, (int32_t)g, nullptr, nullptr));
            gpu::check(hpcg_engine_run(e));
            const std::size_t R = (std::size_t)std::max<std::int64_t>(1, hpcg_engine_round_index(e));
            const std::size_t Wg = w_hi[g] - w_lo[g];
            hpcg_run_out o{};
            ClusteringResult& res = part[g];
            res.centroids = CentroidSet(k, n);
            std::vector<std::int32_t> labels(cfg.compute_assignment ? (std::size_t)shard_rows[g] : 0);
            std::vector<double> wobj(Wg), traces(Wg * R * 2);
            std::vector<std::int64_t> tlen(Wg);
            gpu::check(hpcg_engine_finish(e, &o, res.centroids.centers.data(), res.centroids.degenerate.data(),
                                          cfg.compute_assignment ? labels.data() : nullptr, nullptr, 0, wobj.data(),
                                          traces.data(), (int64_t)R, tlen.data()));
            if (g == 0) {
                std::vector<double> pubs((std::size_t)std::max<std::int64_t>(o.n_publications, 1) * 4);
                gpu::check(hpcg_engine_publications(e, pubs.data(), o.n_publications, nullptr));
                for (std::int64_t i = 0; i < o.n_publications; ++i)
                    res.publications.push_back(
                        {(std::int64_t)pubs[4 * i], (int)pubs[4 * i + 1], pubs[4 * i + 2], pubs[4 * i + 3]});
            }
            std::vector<double> incC(Wg * k * n);
            std::vector<std::uint8_t> incF(Wg * k);
            gpu::check(hpcg_engine_worker_incumbents(e, incC.data(), incF.data(), nullptr));
            if (o.has_full_objective) res.full_objective = o.full_objective;
            if (cfg.compute_assignment) {
                Assignment a;
                a.labels = std::move(labels);
                res.assignment = std::move(a);
            }
            res.best_worker = o.best_worker;
            res.best_sample_objective = o.best_sample_objective;
            res.clustering_time = o.clustering_time;
            res.clustering_time_first_finisher = o.clustering_time_first_finisher;
            res.wall_seconds = o.wall_seconds;
            res.total_samples = (std::size_t)o.total_samples;
            res.distance_evals = o.distance_evals;
            res.per_worker.resize(Wg);
            for (std::size_t w = 0; w < Wg; ++w) {
                WorkerState& ws = res.per_worker[w];
                ws.worker_id = (int)(w_lo[g] + w);
                ws.incumbent = CentroidSet(k, n);
                std::copy_n(incC.data() + w * k * n, k * n, ws.incumbent.centers.data());
                std::copy_n(incF.data() + w * k, k, ws.incumbent.degenerate.data());
                ws.incumbent_objective = wobj[w];
                ws.samples_processed = R;
                ws.t_w = o.last_timestamp;
                for (std::int64_t t = 0; t < tlen[w]; ++t)
                    ws.update_trace.push_back(
                        {traces[(w * R + (std::size_t)t) * 2], traces[(w * R + (std::size_t)t) * 2 + 1]});
            }
        } catch (...) {
            errs[g] = std::current_exception();
        }
        if (e) hpcg_engine_destroy(e);
        if (ctx) hpcg_ctx_synchronize(ctx);
        if (arrived)
            sync.arrive_and_wait();  // no rank frees its shard while a peer may still read it
        else
            sync.arrive_and_drop();  // failed before its shard was published: leave both phases
        if (all) hpcg_dataset_destroy(all);
        if (mine) hpcg_dataset_destroy(mine);
        if (ctx) hpcg_ctx_destroy(ctx);
    };
    std::vector<std::thread> th;
    for (std::size_t g = 0; g < G; ++g) th.emplace_back(rank_main, g);
    for (auto& t : th) t.join();
    for (auto& e : errs)
        if (e) std::rethrow_exception(e);
    // every rank holds the global fields; the per-worker states and labels are per rank
    ClusteringResult res = std::move(part[0]);
    for (std::size_t g = 1; g < G; ++g) {
        for (auto& ws : part[g].per_worker) res.per_worker.push_back(std::move(ws));
        if (cfg.compute_assignment && res.assignment && part[g].assignment)
            res.assignment->labels.insert(res.assignment->labels.end(), part[g].assignment->labels.begin(),
                                          part[g].assignment->labels.end());
    }
    if (cfg.compute_assignment && res.assignment) {
        res.assignment->counts.assign(k, 0);
        for (auto l : res.assignment->labels) ++res.assignment->counts[(std::size_t)l];
    }
    return res;
}

}  // namespace hpclust
