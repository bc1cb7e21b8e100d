// hpclust/bench.hpp: drop-in for the campaign half of the reference's bench.hpp on the B200
// library. Same names, fields, seeds, error texts and metric definitions:
//   relative_error / baseline_objective / baseline_convergence_time   bench.hpp:18-50
//   MetricSummary / summarize_values / MetricRecord / RunSeries / summarize   bench.hpp:52-135
//   BlobSpec / BlobData / gen_blobs   bench.hpp:140-205 (the config-1 generator; bit-reproducible
//                                     through the drop-in RngStream)
//   all_algorithms / is_hpclust_algorithm / strategy_from_name / CampaignConfig /
//   default_sample_size / run_campaign   bench.hpp:302-524
// What differs (additive): run_campaign uploads X to HBM ONCE (DeviceDataset) and every HPClust
// run of the k x algorithm x repetition cross product reads it in place -- the reference re-walks
// the host vector per run; `CampaignConfig::precision` picks the device copy's type (f64 keeps the
// reference's results; f32 is the north star's fp32 mode). The exact-enumeration oracle
// (brute_force_mssc, bench.hpp:207-298) is CPU test infrastructure and is not part of the drop-in.
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>
#include <map>
#include <optional>
#include <string>
#include <vector>

#include "baselines.hpp"
#include "hpclust.hpp"

namespace hpclust {

namespace detail {
// median of a value list (even length: mean of the two middle values); sorts its copy
inline double median_of(std::vector<double> v) {
    std::sort(v.begin(), v.end());
    const std::size_t h = v.size() / 2;
    return (v.size() & 1) ? v[h] : 0.5 * (v[h - 1] + v[h]);
}
}  // namespace detail

// epsilon = 100 (f - f*) / f* (bench.hpp:18-21); negative when the run beat the reference optimum
inline double relative_error(double f, double f_star) {
    require(f_star > 0.0, "relative_error: reference objective must be positive");
    return 100.0 * (f - f_star) / f_star;
}

// f_bar: the largest per-algorithm median of the best sample objectives (bench.hpp:25-38)
inline double baseline_objective(const std::map<std::string, std::vector<double>>& best_sample_objectives) {
    require(!best_sample_objectives.empty(), "baseline_objective: no algorithms");
    double bar = -std::numeric_limits<double>::infinity();
    for (const auto& kv : best_sample_objectives) {
        require(!kv.second.empty(), "baseline_objective: empty objective list");
        bar = std::max(bar, detail::median_of(kv.second));
    }
    return bar;
}

// earliest trace timestamp over all workers with an accepted objective <= f_bar (bench.hpp:42-54);
// a worker's trace objectives strictly decrease, so its first crossing is its earliest
inline std::optional<double> baseline_convergence_time(const std::vector<WorkerState>& workers, double f_bar) {
    std::optional<double> t;
    for (const auto& w : workers) {
        auto hit = std::find_if(w.update_trace.begin(), w.update_trace.end(),
                                [&](const auto& e) { return e.sample_objective <= f_bar; });
        if (hit != w.update_trace.end() && (!t || hit->timestamp < *t)) t = hit->timestamp;
    }
    return t;
}

struct MetricSummary {
    double median = 0.0;
    double min = 0.0;
    double max = 0.0;
    std::optional<double> stddev;  // sample (n - 1) deviation; absent for one value
};

inline MetricSummary summarize_values(std::vector<double> values) {
    require(!values.empty(), "summarize: empty value list");
    MetricSummary s;
    const auto [lo, hi] = std::minmax_element(values.begin(), values.end());
    s.min = *lo;
    s.max = *hi;
    const std::size_t n = values.size();
    if (n >= 2) {
        // the reference sums the SORTED values (bench.hpp:66-77): same order here, same bits
        std::sort(values.begin(), values.end());
        double mean = 0.0;
        for (double v : values) mean += v;
        mean /= static_cast<double>(n);
        double acc = 0.0;
        for (double v : values) acc += (v - mean) * (v - mean);
        s.stddev = std::sqrt(acc / static_cast<double>(n - 1));
    }
    s.median = detail::median_of(std::move(values));
    return s;
}

struct MetricRecord {
    std::string algorithm;
    std::size_t k = 0;
    int repetition = 0;
    double epsilon = 0.0;
    double t = 0.0;
    std::optional<double> t_bar;
    std::int64_t n_d = 0;
};

struct RunSeries {
    std::string dataset;
    std::string algorithm;
    std::size_t k = 0;
    std::vector<MetricRecord> records;
    MetricSummary epsilon;
    std::optional<MetricSummary> t_bar;
    MetricSummary t;
    double n_d_median = 0.0;
    double n_s_median = 0.0;
    double sample_size = 0.0;
    double time_limit = 0.0;  // budget in the active clock unit
    double t1 = 0.0;
    double t2 = 0.0;
    bool succ = false;
};

// summaries of one (algorithm, k) series (bench.hpp:112-135)
inline RunSeries summarize(std::vector<MetricRecord> records) {
    require(!records.empty(), "summarize: empty record list");
    RunSeries out;
    out.algorithm = records.front().algorithm;
    out.k = records.front().k;
    std::vector<double> eps, ts, bars, nds;
    for (const auto& r : records) {
        require(r.algorithm == out.algorithm && r.k == out.k, "summarize: records must share (algorithm, k)");
        eps.push_back(r.epsilon);
        ts.push_back(r.t);
        nds.push_back(static_cast<double>(r.n_d));
        if (r.t_bar) bars.push_back(*r.t_bar);
    }
    out.epsilon = summarize_values(std::move(eps));
    out.t = summarize_values(std::move(ts));
    if (!bars.empty()) out.t_bar = summarize_values(std::move(bars));
    out.n_d_median = detail::median_of(std::move(nds));
    out.records = std::move(records);
    return out;
}

// ------------------------------------------------------------- synthetic Gaussian blobs
struct BlobSpec {
    std::size_t num_points = 2187;  // blob rows; noise rows come on top
    std::size_t features = 10;
    std::size_t num_blobs = 10;
    double center_min = -40.0;
    double center_max = 40.0;
    double std_min = 0.0;
    double std_max = 10.0;
    std::size_t noise_points = 500;
    double noise_min = -50.0;
    double noise_max = 50.0;
    std::uint64_t seed = 0;

    void validate() const {
        require(num_points >= 1, "BlobSpec: num_points must be positive");
        require(features >= 1, "BlobSpec: features must be positive");
        require(num_blobs >= 1, "BlobSpec: num_blobs must be positive");
        require(center_min <= center_max, "BlobSpec: center box is inverted");
        require(std_min <= std_max && std_min >= 0.0, "BlobSpec: std range is invalid");
        require(noise_min <= noise_max, "BlobSpec: noise box is inverted");
    }
};

struct BlobData {
    Dataset points;                         // num_points + noise_points rows
    Dataset centers;                        // num_blobs x features
    std::vector<double> stds;               // per-blob standard deviation
    std::vector<std::int32_t> blob_of_row;  // generating blob; -1 for noise rows
};

// Stream order of the reference generator (bench.hpp:171-205): all centre coordinates, all
// spreads, then the blob rows blob by blob (the first num_points % num_blobs blobs hold one more
// row), then the uniform noise rows.
inline BlobData gen_blobs(const BlobSpec& spec) {
    spec.validate();
    RngStream rng(splitmix64(spec.seed));
    const std::size_t B = spec.num_blobs, n = spec.features, total = spec.num_points + spec.noise_points;
    BlobData out;
    out.centers = Dataset(B, n);
    for (double& c : out.centers.values) c = rng.uniform(spec.center_min, spec.center_max);
    out.stds.resize(B);
    for (double& s : out.stds) s = rng.uniform(spec.std_min, spec.std_max);
    out.points = Dataset(total, n);
    out.blob_of_row.assign(total, -1);
    double* p = out.points.values.data();
    std::size_t row = 0;
    for (std::size_t b = 0; b < B; ++b) {
        const std::size_t rows_b = spec.num_points / B + (b < spec.num_points % B ? 1 : 0);
        const double* c = out.centers.values.data() + b * n;
        for (std::size_t i = 0; i < rows_b; ++i, ++row) {
            for (std::size_t d = 0; d < n; ++d) *p++ = c[d] + out.stds[b] * rng.normal();
            out.blob_of_row[row] = static_cast<std::int32_t>(b);
        }
    }
    for (std::size_t i = spec.noise_points * n; i > 0; --i) *p++ = rng.uniform(spec.noise_min, spec.noise_max);
    return out;
}

// ------------------------------------------------------------------ campaign
inline const std::vector<std::string>& all_algorithms() {
    static const std::vector<std::string> names = {"inner", "competitive", "cooperative", "hybrid", "forgy", "pbk"};
    return names;
}

inline StrategyKind strategy_from_name(const std::string& name) {
    for (StrategyKind s : {StrategyKind::inner, StrategyKind::competitive, StrategyKind::cooperative, StrategyKind::hybrid})
        if (name == to_string(s)) return s;
    throw std::invalid_argument("unknown strategy: " + name);
}

inline bool is_hpclust_algorithm(const std::string& name) {
    return name == "inner" || name == "competitive" || name == "cooperative" || name == "hybrid";
}

struct CampaignConfig {
    std::string dataset_name = "dataset";
    std::vector<std::size_t> k_list;
    std::vector<std::string> algorithms;  // names from all_algorithms()
    int n_exec = 10;
    std::uint64_t master_seed = 0;
    std::size_t sample_size = 0;  // 0 = default_sample_size(m)
    std::size_t n_workers = 8;
    double time_limit = std::numeric_limits<double>::infinity();
    std::optional<std::size_t> max_samples;
    std::optional<double> t1, t2;             // hybrid split; default half / half
    std::optional<std::size_t> segment_size;  // pbk p; default = sample size
    std::optional<double> f_star;             // external reference optimum
    LloydConfig lloyd;
    SeedConfig seed_cfg;
    std::size_t n_threads = 0;
    // additive (not in the reference): type of the HBM copy the HPClust runs read, and their streams
    Precision precision = Precision::f64;
    RngMode rng_mode = RngMode::reference;

    void validate() const {
        require(!k_list.empty(), "CampaignConfig: k_list is empty");
        require(!algorithms.empty(), "CampaignConfig: algorithm list is empty");
        require(n_exec >= 1, "CampaignConfig: n_exec must be positive");
        const auto& known = all_algorithms();
        for (const auto& a : algorithms)
            require(std::find(known.begin(), known.end(), a) != known.end(),
                    ("CampaignConfig: unknown algorithm '" + a + "'").c_str());
        require(std::isfinite(time_limit) || max_samples.has_value(), "CampaignConfig: need a time limit or max_samples");
    }
};

inline std::size_t default_sample_size(std::size_t m) { return m <= 2000 ? m : std::min<std::size_t>(5000, m - 1000); }

namespace detail {
inline std::uint64_t fnv1a(const std::string& s) {
    std::uint64_t h = 0xcbf29ce484222325ULL;
    for (unsigned char c : s) h = (h ^ c) * 0x100000001b3ULL;
    return h;
}
// run seed: a function of (master seed, algorithm, k, repetition) only (bench.hpp:411-413), so a
// record does not depend on execution order or on which other algorithms were selected
inline std::uint64_t campaign_seed(std::uint64_t master, const std::string& algo, std::size_t k, int rep) {
    return splitmix64(master ^ splitmix64(fnv1a(algo) ^ (k * 0x9e37ULL) ^ static_cast<std::uint64_t>(rep)));
}
struct RawRun {
    double full_objective = 0.0;
    double best_sample_objective = std::numeric_limits<double>::infinity();
    double t = 0.0;
    std::size_t n_s = 0;
    std::int64_t n_d = 0;
    std::vector<WorkerState> workers;  // empty for the trace-less baselines
    explicit RawRun(ClusteringResult&& r, bool hpclust_run)
        : full_objective(*r.full_objective), t(r.clustering_time), n_s(r.total_samples), n_d(r.distance_evals) {
        if (hpclust_run) {
            best_sample_objective = r.best_sample_objective;
            workers = std::move(r.per_worker);
        }
    }
};
}  // namespace detail

// Cross-product campaign (bench.hpp:382-524): every (k, algorithm, repetition) runs once; epsilon
// against cfg.f_star or the best full objective of that k; t_bar against the max-of-medians bar over
// the HPClust strategies; succ = this algorithm's median full objective is below every other
// algorithm's MEAN full objective.
inline std::vector<RunSeries> run_campaign(const Dataset& X, const CampaignConfig& cfg_in) {
    CampaignConfig cfg = cfg_in;
    cfg.validate();
    X.validate();
    const std::size_t m = X.rows;
    if (cfg.sample_size == 0) cfg.sample_size = default_sample_size(m);
    require(cfg.sample_size >= 1 && cfg.sample_size <= m, "CampaignConfig: sample size out of range");
    const std::size_t p = cfg.segment_size.value_or(cfg.sample_size);
    const double budget = std::isfinite(cfg.time_limit) ? cfg.time_limit : static_cast<double>(cfg.max_samples.value());
    const double t1 = cfg.t1.value_or(budget / 2.0);
    const double t2 = cfg.t2.value_or(budget - t1);

    // one upload for every HPClust run of the campaign
    std::optional<DeviceDataset> resident;
    if (std::any_of(cfg.algorithms.begin(), cfg.algorithms.end(), is_hpclust_algorithm)) resident.emplace(X, cfg.precision);

    auto one_run = [&](const std::string& algo, std::size_t k, int rep) {
        const std::uint64_t seed = detail::campaign_seed(cfg.master_seed, algo, k, rep);
        if (is_hpclust_algorithm(algo)) {
            EngineConfig ec;
            ec.k = k;
            ec.sample_size = cfg.sample_size;
            ec.n_workers = cfg.n_workers;
            ec.time_limit = cfg.time_limit;
            ec.max_samples = cfg.max_samples;
            ec.master_seed = seed;
            ec.seed = cfg.seed_cfg;
            ec.lloyd = cfg.lloyd;
            ec.n_threads = cfg.n_threads;
            ec.rng_mode = cfg.rng_mode;
            const StrategyKind kind = strategy_from_name(algo);
            ec.strategy = kind == StrategyKind::hybrid ? Strategy::hybrid(t1, t2) : Strategy{kind};
            return detail::RawRun(run(*resident, ec), true);
        }
        RngStream rng(seed);
        if (algo == "forgy") return detail::RawRun(forgy_kmeans(X, k, cfg.lloyd, rng), false);
        PbkConfig pc;
        pc.segment_size = std::min(p, m);
        pc.inner_lloyd = cfg.lloyd;
        pc.n_threads = cfg.n_threads;
        return detail::RawRun(pbk_bdc(X, std::min(k, pc.segment_size), pc, rng), false);
    };

    std::vector<RunSeries> out;
    for (std::size_t k : cfg.k_list) {
        std::map<std::string, std::vector<detail::RawRun>> runs;
        for (const auto& algo : cfg.algorithms) {
            auto& list = runs[algo];
            for (int rep = 0; rep < cfg.n_exec; ++rep) list.push_back(one_run(algo, k, rep));
        }
        double f_star = cfg.f_star.value_or(std::numeric_limits<double>::infinity());
        if (!cfg.f_star)
            for (const auto& kv : runs)
                for (const auto& r : kv.second) f_star = std::min(f_star, r.full_objective);
        std::map<std::string, std::vector<double>> trace_bests;
        for (const auto& kv : runs)
            if (is_hpclust_algorithm(kv.first))
                for (const auto& r : kv.second) trace_bests[kv.first].push_back(r.best_sample_objective);
        std::optional<double> f_bar;
        if (!trace_bests.empty()) f_bar = baseline_objective(trace_bests);

        // medians and means of the full objectives per algorithm, for succ
        std::map<std::string, std::pair<double, double>> med_mean;
        for (const auto& kv : runs) {
            std::vector<double> f;
            double sum = 0.0;
            for (const auto& r : kv.second) {
                f.push_back(r.full_objective);
                sum += r.full_objective;
            }
            med_mean[kv.first] = {detail::median_of(std::move(f)), sum / static_cast<double>(kv.second.size())};
        }
        for (const auto& algo : cfg.algorithms) {
            const auto& list = runs[algo];
            std::vector<MetricRecord> records;
            std::vector<double> ns;
            for (std::size_t rep = 0; rep < list.size(); ++rep) {
                const auto& r = list[rep];
                MetricRecord rec;
                rec.algorithm = algo;
                rec.k = k;
                rec.repetition = static_cast<int>(rep);
                rec.epsilon = relative_error(r.full_objective, f_star);
                rec.t = r.t;
                rec.n_d = r.n_d;
                if (f_bar && !r.workers.empty()) rec.t_bar = baseline_convergence_time(r.workers, *f_bar);
                records.push_back(std::move(rec));
                ns.push_back(static_cast<double>(r.n_s));
            }
            RunSeries series = summarize(std::move(records));
            series.dataset = cfg.dataset_name;
            series.n_s_median = detail::median_of(std::move(ns));
            series.sample_size = static_cast<double>(is_hpclust_algorithm(algo) ? cfg.sample_size : algo == "pbk" ? p : m);
            series.time_limit = budget;
            if (algo == "hybrid") {
                series.t1 = t1;
                series.t2 = t2;
            }
            series.succ = std::all_of(cfg.algorithms.begin(), cfg.algorithms.end(), [&](const std::string& other) {
                return other == algo || med_mean[algo].first < med_mean[other].second;
            });
            out.push_back(std::move(series));
        }
    }
    return out;
}

}  // namespace hpclust
