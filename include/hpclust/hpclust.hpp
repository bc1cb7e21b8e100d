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
#include <unordered_map>
#include <utility>
#include <vector>

#include "../hpcg.h"

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
        Holder() { check(hpcg_ctx_create(0, &c)); }
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
namespace gpu {
inline std::pair<Assignment, double> assign(const Dataset& X, const CentroidSet& C, bool strict, bool want_labels,
                                            DistCounter* counter) {
    DeviceMatrix dm(X.values.data(), X.rows, X.cols);
    Assignment a;
    if (want_labels) a.labels.resize(X.rows);
    a.counts.assign(C.k, 0);
    double cost = 0.0;
    std::int64_t nd = 0;
    check(hpcg_assign(context(), dm.ds, C.centers.data(), C.degenerate.data(), (int64_t)C.k, strict ? 1 : 0,
                      want_labels ? a.labels.data() : nullptr, a.counts.data(), &cost, &nd));
    count_distances(counter, nd);
    return {std::move(a), cost};
}
}  // namespace gpu

inline Assignment assign_nearest(const Dataset& X, const CentroidSet& C,
                                 const ParallelPolicy& = ParallelPolicy::sequential(), DistCounter* counter = nullptr) {
    require(C.k >= 1, "assign_nearest: need at least one centroid");
    require(C.cols == X.cols, "assign_nearest: dimension mismatch");
    require(!C.any_degenerate(), "assign_nearest: degenerate centroid present");
    return gpu::assign(X, C, true, true, counter).first;
}

inline double mssc_objective(const CentroidSet& C, const Dataset& X,
                             const ParallelPolicy& = ParallelPolicy::sequential(), DistCounter* counter = nullptr) {
    require(C.k >= 1, "mssc_objective: need at least one centroid");
    require(C.cols == X.cols, "mssc_objective: dimension mismatch");
    require(!C.any_degenerate(), "mssc_objective: degenerate centroid present");
    return gpu::assign(X, C, true, false, counter).second;
}

inline std::pair<Assignment, double> final_assignment(const Dataset& X, const CentroidSet& C,
                                                      const ParallelPolicy& = ParallelPolicy::sequential(),
                                                      DistCounter* counter = nullptr) {
    require(!C.any_degenerate(), "final_assignment: degenerate centroid present");
    require(C.cols == X.cols, "final_assignment: dimension mismatch");
    return gpu::assign(X, C, true, true, counter);
}

namespace detail {
inline std::pair<Assignment, double> assign_valid_subset(const Dataset& X, const CentroidSet& C, const ParallelPolicy&,
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
    ParallelPolicy policy() const { return parallel_rows ? ParallelPolicy::threads(n_threads) : ParallelPolicy::sequential(); }
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
inline StepOut step(const Dataset& S, const CentroidSet& init, const LloydConfig& lc, std::size_t candidates,
                    RngStream* rng, bool do_lloyd) {
    const std::size_t s = S.rows, k = init.k;
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
    DeviceMatrix dm(S.values.data(), s, S.cols);
    const hpcg_lloyd_cfg cfg{(int64_t)lc.max_iters, lc.rel_tol, (int64_t)candidates};
    StepOut o;
    o.C.resize(k * S.cols);
    o.f.resize(k);
    o.labels.resize(s);
    o.counts.resize(k);
    const int32_t cap = (int32_t)std::min<std::size_t>(lc.max_iters + 1, 100001);
    o.history.resize((std::size_t)cap);
    int32_t hl = 0;
    const int rc = hpcg_worker_step_batched(
        context(), dm.ds, nullptr, 1, (int64_t)s, init.centers.data(), init.degenerate.data(), (int64_t)k, &cfg,
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
inline Dataset draw_sample(const Dataset& X, std::size_t s, RngStream& rng) {
    require(s >= 1 && s <= X.rows, "draw_sample: sample size must be in [1, m]");
    std::vector<std::int64_t> idx(s);
    std::unordered_map<std::size_t, std::size_t> moved;
    moved.reserve(2 * s);
    auto at = [&](std::size_t i) {
        auto it = moved.find(i);
        return it == moved.end() ? i : it->second;
    };
    for (std::size_t i = 0; i < s; ++i) {
        const std::size_t j = i + rng.uniform_index(X.rows - i);
        const std::size_t a = at(i), b = at(j);
        moved[i] = b;
        moved[j] = a;
        idx[i] = (std::int64_t)b;
    }
    gpu::DeviceMatrix dm(X.values.data(), X.rows, X.cols);
    Dataset out(s, X.cols);
    gpu::check(hpcg_gather(gpu::context(), dm.ds, idx.data(), (int64_t)s, out.values.data()));
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
inline ClusteringResult run(const Dataset& X, const EngineConfig& cfg_in) {
    EngineConfig cfg = cfg_in;
    if (cfg.strategy.kind == StrategyKind::inner) cfg.n_workers = 1;
    cfg.validate(X.rows);
    const std::size_t W = cfg.n_workers, k = cfg.k, n = X.cols;
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
    gpu::DeviceMatrix dm(X.values.data(), X.rows, n);
    hpcg_engine* e = nullptr;
    gpu::check(hpcg_engine_create(gpu::context(), dm.ds, &ec, &e));
    std::unique_ptr<hpcg_engine, int (*)(hpcg_engine*)> guard(e, hpcg_engine_destroy);
    gpu::check(hpcg_engine_run(e));
    const std::size_t R = (std::size_t)std::max<std::int64_t>(1, hpcg_engine_round_index(e));
    hpcg_run_out o{};
    ClusteringResult res;
    res.centroids = CentroidSet(k, n);
    std::vector<std::int32_t> labels(cfg.compute_assignment ? X.rows : 0);
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
        ws.samples_processed = R;
        ws.t_w = o.last_timestamp;  // the clock read after the worker's last step (engine.hpp:250)
        for (std::int64_t t = 0; t < tlen[w]; ++t)
            ws.update_trace.push_back({traces[(w * R + (std::size_t)t) * 2], traces[(w * R + (std::size_t)t) * 2 + 1]});
    }
    return res;
}

}  // namespace hpclust
