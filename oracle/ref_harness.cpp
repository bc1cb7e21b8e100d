// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// C-ABI harness over the UNMODIFIED reference headers (/root/reference/proj/include,
// included at compile time, never copied). Built by oracle/Makefile into
// oracle/_ref/libhpclust_ref.so with the reference's Release flags plus
// -ffp-contract=off (contraction changes the reference's bits).
//
// Used by: tests/ (pinning the C restatement oracle/hpclust_oracle.c and generating
// tests/golden/ fixtures), bench.py --impl reference (the reference's own CPU path
// timed on the host), and bench.py's cpu_baseline leg.
//
// Every entry point returns 0 on success, 1 for std::invalid_argument,
// 2 for std::logic_error, 3 for NoSolutionError, 4 for any other exception; the
// message is kept in a thread-local buffer readable via hpref_last_error().

#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "hpclust/hpclust.hpp"

using namespace hpclust;

namespace {
thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const NoSolutionError& e) {
        g_err = e.what();
        return 3;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::logic_error& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 4;
    }
}

Dataset make_ds(const double* X, std::size_t m, std::size_t n) {
    Dataset d(m, n);
    std::memcpy(d.values.data(), X, m * n * sizeof(double));
    return d;
}

CentroidSet make_cs(const double* C, const std::uint8_t* flags, std::size_t k, std::size_t n) {
    CentroidSet c(k, n);
    if (C) std::memcpy(c.centers.data(), C, k * n * sizeof(double));
    if (flags) std::memcpy(c.degenerate.data(), flags, k);
    return c;
}

void put_cs(const CentroidSet& c, double* C, std::uint8_t* flags) {
    if (C) std::memcpy(C, c.centers.data(), c.centers.size() * sizeof(double));
    if (flags) std::memcpy(flags, c.degenerate.data(), c.degenerate.size());
}
}  // namespace

extern "C" {

const char* hpref_last_error() { return g_err.c_str(); }

// ---- rng.hpp -------------------------------------------------------------
void* hpref_rng_new(std::uint64_t seed) { return new RngStream(seed); }
void* hpref_rng_derive(std::uint64_t master, std::uint64_t domain, std::uint64_t index) {
    return new RngStream(RngStream::derive(master, domain, index));
}
void* hpref_rng_clone(void* h) { return new RngStream(*static_cast<RngStream*>(h)); }
void hpref_rng_free(void* h) { delete static_cast<RngStream*>(h); }
std::uint64_t hpref_rng_next_u64(void* h) { return static_cast<RngStream*>(h)->next_u64(); }
double hpref_rng_next_unit(void* h) { return static_cast<RngStream*>(h)->next_unit(); }
std::uint64_t hpref_rng_uniform_index(void* h, std::uint64_t n) {
    return static_cast<RngStream*>(h)->uniform_index(n);
}
std::uint64_t hpref_splitmix64(std::uint64_t x) { return splitmix64(x); }

// ---- core.hpp ------------------------------------------------------------
int hpref_assign(const double* X, std::size_t m, std::size_t n, const double* C, const std::uint8_t* flags,
                 std::size_t k, std::size_t n_chunks, std::int32_t* labels, std::int64_t* counts, double* cost,
                 std::int64_t* n_d) {
    return guard([&] {
        Dataset ds = make_ds(X, m, n);
        CentroidSet cs = make_cs(C, flags, k, n);
        DistCounter ctr;
        // final_assignment semantics over valid centres (engine.hpp:211-229)
        auto [a, f] = detail::assign_valid_subset(ds, cs, ParallelPolicy::threads(n_chunks), &ctr);
        if (labels) std::memcpy(labels, a.labels.data(), m * sizeof(std::int32_t));
        if (counts) std::memcpy(counts, a.counts.data(), k * sizeof(std::int64_t));
        if (cost) *cost = f;
        if (n_d) *n_d = ctr.value();
    });
}

int hpref_mssc_objective(const double* X, std::size_t m, std::size_t n, const double* C, std::size_t k,
                         std::size_t n_chunks, double* cost) {
    return guard([&] {
        Dataset ds = make_ds(X, m, n);
        CentroidSet cs = make_cs(C, nullptr, k, n);
        *cost = mssc_objective(cs, ds, ParallelPolicy::threads(n_chunks));
    });
}

// ---- lloyd.hpp -----------------------------------------------------------
int hpref_kmeans(const double* S, std::size_t s, std::size_t n, const double* C_init, const std::uint8_t* flags_init,
                 std::size_t k, std::size_t max_iters, double rel_tol, double* C_out, std::uint8_t* flags_out,
                 std::int32_t* labels, std::int64_t* counts, double* objective, std::int64_t* iterations,
                 std::int32_t* stop, std::int64_t* n_d, double* history, std::int64_t history_cap,
                 std::int64_t* history_len) {
    return guard([&] {
        Dataset ds = make_ds(S, s, n);
        CentroidSet c0 = make_cs(C_init, flags_init, k, n);
        LloydConfig cfg;
        cfg.max_iters = max_iters;
        cfg.rel_tol = rel_tol;
        DistCounter ctr;
        LloydOutcome out = kmeans(ds, c0, cfg, &ctr);
        put_cs(out.centroids, C_out, flags_out);
        if (labels) std::memcpy(labels, out.assignment.labels.data(), s * sizeof(std::int32_t));
        if (counts) std::memcpy(counts, out.assignment.counts.data(), k * sizeof(std::int64_t));
        if (objective) *objective = out.objective;
        if (iterations) *iterations = static_cast<std::int64_t>(out.iterations);
        if (stop) *stop = static_cast<std::int32_t>(out.converged_by);
        if (n_d) *n_d = ctr.value();
        if (history_len) *history_len = static_cast<std::int64_t>(out.objective_history.size());
        if (history)
            for (std::size_t i = 0; i < out.objective_history.size() && (std::int64_t)i < history_cap; ++i)
                history[i] = out.objective_history[i];
    });
}

// ---- seeding.hpp ---------------------------------------------------------
int hpref_reinit_degenerate(const double* S, std::size_t s, std::size_t n, const double* C_in,
                            const std::uint8_t* flags_in, std::size_t k, std::size_t candidates, void* rng,
                            double* C_out, std::uint8_t* flags_out, std::int64_t* n_d) {
    return guard([&] {
        Dataset ds = make_ds(S, s, n);
        CentroidSet c0 = make_cs(C_in, flags_in, k, n);
        SeedConfig cfg;
        cfg.candidates_per_center = candidates;
        DistCounter ctr;
        CentroidSet out = reinit_degenerate(c0, ds, cfg, *static_cast<RngStream*>(rng),
                                            ParallelPolicy::sequential(), &ctr);
        put_cs(out, C_out, flags_out);
        if (n_d) *n_d = ctr.value();
    });
}

// ---- engine.hpp ----------------------------------------------------------
// Index-dataset trick (SURVEY.md §8(c) iv): draw_sample on the m×1 row-id dataset
// yields the exact reference sample indices and leaves the stream where the real
// draw_sample would.
int hpref_draw_indices(std::size_t m, std::size_t s, void* rng, std::int64_t* idx_out) {
    return guard([&] {
        Dataset ids(m, 1);
        for (std::size_t i = 0; i < m; ++i) ids.values[i] = static_cast<double>(i);
        Dataset S = draw_sample(ids, s, *static_cast<RngStream*>(rng));
        for (std::size_t i = 0; i < s; ++i) idx_out[i] = static_cast<std::int64_t>(S.values[i]);
    });
}

int hpref_draw_sample(const double* X, std::size_t m, std::size_t n, std::size_t s, void* rng, double* S_out) {
    return guard([&] {
        Dataset ds = make_ds(X, m, n);
        Dataset S = draw_sample(ds, s, *static_cast<RngStream*>(rng));
        std::memcpy(S_out, S.values.data(), s * n * sizeof(double));
    });
}

struct hpref_run_cfg {
    std::uint64_t k, sample_size, n_workers, max_samples;  // max_samples 0 = none
    double time_limit;                                     // <=0 or inf = none
    std::int32_t strategy;                                 // 0 inner 1 competitive 2 cooperative 3 hybrid
    double phase_t1, phase_t2;
    std::uint64_t master_seed;
    std::uint64_t candidates, max_iters;
    double rel_tol;
    std::uint64_t n_threads;
    std::int32_t compute_full_objective, compute_assignment;
};

struct hpref_run_out {
    double full_objective;
    std::int32_t has_full_objective;
    std::int32_t best_worker;
    double best_sample_objective;
    double clustering_time, clustering_time_first_finisher, wall_seconds;
    std::uint64_t total_samples;
    std::int64_t distance_evals;
    std::int64_t n_publications;
};

// publications: [cap x 4] doubles (version, worker_id, objective, timestamp)
// traces: per worker up to trace_cap entries of (timestamp, objective), trace_len[W]
// worker_obj[W] = final incumbent objectives
int hpref_run(const double* X, std::size_t m, std::size_t n, const hpref_run_cfg* c, hpref_run_out* o,
              double* centroids, std::uint8_t* flags, std::int32_t* labels, double* publications,
              std::int64_t pub_cap, double* worker_obj, double* traces, std::int64_t trace_cap,
              std::int64_t* trace_len) {
    return guard([&] {
        Dataset ds = make_ds(X, m, n);
        EngineConfig cfg;
        cfg.k = c->k;
        cfg.sample_size = c->sample_size;
        cfg.n_workers = c->n_workers;
        if (c->max_samples) cfg.max_samples = c->max_samples;
        if (c->time_limit > 0) cfg.time_limit = c->time_limit;
        switch (c->strategy) {
            case 0: cfg.strategy = Strategy::inner(); break;
            case 1: cfg.strategy = Strategy::competitive(); break;
            case 2: cfg.strategy = Strategy::cooperative(); break;
            default: cfg.strategy = Strategy::hybrid(c->phase_t1, c->phase_t2); break;
        }
        cfg.master_seed = c->master_seed;
        cfg.seed.candidates_per_center = c->candidates;
        cfg.lloyd.max_iters = c->max_iters;
        cfg.lloyd.rel_tol = c->rel_tol;
        cfg.n_threads = c->n_threads;
        cfg.compute_full_objective = c->compute_full_objective != 0;
        cfg.compute_assignment = c->compute_assignment != 0;
        ClusteringResult r = run(ds, cfg);
        put_cs(r.centroids, centroids, flags);
        o->has_full_objective = r.full_objective.has_value();
        o->full_objective = r.full_objective.value_or(0.0);
        o->best_worker = r.best_worker;
        o->best_sample_objective = r.best_sample_objective;
        o->clustering_time = r.clustering_time;
        o->clustering_time_first_finisher = r.clustering_time_first_finisher;
        o->wall_seconds = r.wall_seconds;
        o->total_samples = r.total_samples;
        o->distance_evals = r.distance_evals;
        o->n_publications = static_cast<std::int64_t>(r.publications.size());
        if (labels && r.assignment) std::memcpy(labels, r.assignment->labels.data(), m * sizeof(std::int32_t));
        if (publications)
            for (std::size_t i = 0; i < r.publications.size() && (std::int64_t)i < pub_cap; ++i) {
                publications[4 * i + 0] = static_cast<double>(r.publications[i].version);
                publications[4 * i + 1] = r.publications[i].worker_id;
                publications[4 * i + 2] = r.publications[i].objective;
                publications[4 * i + 3] = r.publications[i].timestamp;
            }
        for (std::size_t w = 0; w < r.per_worker.size(); ++w) {
            const auto& ws = r.per_worker[w];
            if (worker_obj) worker_obj[w] = ws.incumbent_objective;
            if (trace_len) trace_len[w] = static_cast<std::int64_t>(ws.update_trace.size());
            if (traces)
                for (std::size_t t = 0; t < ws.update_trace.size() && (std::int64_t)t < trace_cap; ++t) {
                    traces[(w * trace_cap + t) * 2 + 0] = ws.update_trace[t].timestamp;
                    traces[(w * trace_cap + t) * 2 + 1] = ws.update_trace[t].sample_objective;
                }
        }
    });
}

// ---- bench.hpp -----------------------------------------------------------
int hpref_gen_blobs(std::size_t num_points, std::size_t features, std::size_t num_blobs, double center_min,
                    double center_max, double std_min, double std_max, std::size_t noise_points,
                    double noise_min, double noise_max, std::uint64_t seed, double* X_out) {
    return guard([&] {
        BlobSpec spec;
        spec.num_points = num_points;
        spec.features = features;
        spec.num_blobs = num_blobs;
        spec.center_min = center_min;
        spec.center_max = center_max;
        spec.std_min = std_min;
        spec.std_max = std_max;
        spec.noise_points = noise_points;
        spec.noise_min = noise_min;
        spec.noise_max = noise_max;
        spec.seed = seed;
        BlobData b = gen_blobs(spec);
        std::memcpy(X_out, b.points.values.data(), b.points.values.size() * sizeof(double));
    });
}

int hpref_brute_force(const double* X, std::size_t m, std::size_t n, std::size_t k, double* C_out,
                      std::uint8_t* flags_out, double* cost) {
    return guard([&] {
        Dataset ds = make_ds(X, m, n);
        auto [C, f] = brute_force_mssc(ds, k);
        put_cs(C, C_out, flags_out);
        *cost = f;
    });
}

// ---- CPU baseline leg ----------------------------------------------------
// The reference's own competitive threading model (engine.hpp:313-332): one
// std::thread per worker, each running the stock kmeans() on its own sample.
// samples: [W x s x n] fp64, inits: [W x k x n]. Returns summed Lloyd n_d.
int hpref_kmeans_threads(const double* samples, std::size_t W, std::size_t s, std::size_t n, const double* inits,
                         std::size_t k, std::size_t max_iters, double rel_tol, std::int64_t* n_d_total,
                         double* objectives) {
    return guard([&] {
        std::vector<std::thread> th;
        std::vector<std::int64_t> nd(W, 0);
        std::vector<std::string> errs(W);
        for (std::size_t w = 0; w < W; ++w)
            th.emplace_back([&, w] {
                try {
                    Dataset ds = make_ds(samples + w * s * n, s, n);
                    CentroidSet c0 = make_cs(inits + w * k * n, nullptr, k, n);
                    LloydConfig cfg;
                    cfg.max_iters = max_iters;
                    cfg.rel_tol = rel_tol;
                    DistCounter ctr;
                    LloydOutcome out = kmeans(ds, c0, cfg, &ctr);
                    nd[w] = ctr.value();
                    if (objectives) objectives[w] = out.objective;
                } catch (const std::exception& e) {
                    errs[w] = e.what();
                }
            });
        for (auto& t : th) t.join();
        for (auto& e : errs)
            if (!e.empty()) throw std::runtime_error(e);
        std::int64_t tot = 0;
        for (auto v : nd) tot += v;
        *n_d_total = tot;
    });
}

// baselines.hpp:29-47 forgy_kmeans / 58-147 pbk_bdc with RngStream(seed); p = 0 selects Forgy.
// Outputs: centroids[k*n], flags[k], labels[m], full objective, n_d, total_samples.
int hpref_baseline(const double* X, std::size_t m, std::size_t n, std::size_t k, std::size_t p,
                   std::uint64_t seed, std::size_t max_iters, double rel_tol, double* C_out,
                   std::uint8_t* flags_out, std::int32_t* labels_out, double* f_out, std::int64_t* nd_out,
                   std::int64_t* samples_out) {
    return guard([&] {
        Dataset ds = make_ds(X, m, n);
        RngStream rng(seed);
        LloydConfig lc;
        lc.max_iters = max_iters;
        lc.rel_tol = rel_tol;
        ClusteringResult r;
        if (p == 0) {
            r = forgy_kmeans(ds, k, lc, rng);
        } else {
            PbkConfig pc;
            pc.segment_size = p;
            pc.inner_lloyd = lc;
            pc.n_threads = 1;
            r = pbk_bdc(ds, k, pc, rng);
        }
        put_cs(r.centroids, C_out, flags_out);
        if (labels_out && r.assignment)
            for (std::size_t i = 0; i < m; ++i) labels_out[i] = r.assignment->labels[i];
        *f_out = r.full_objective.value_or(-1.0);
        *nd_out = r.distance_evals;
        *samples_out = (std::int64_t)r.total_samples;
    });
}

}  // extern "C"
