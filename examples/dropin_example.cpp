// A reference user's program, unchanged except for the include path and -lhpcg: it calls the
// hpclust:: API exactly as it would against /root/reference/proj/include. Reads X (fp64,
// row-major) from argv[1] with m, n in argv[2..3]; prints one JSON object of results.
#include <cstdio>
#include <fstream>
#include <vector>

#include "hpclust/hpclust.hpp"

int main(int argc, char** argv) {
    if (argc < 4) {
        std::fprintf(stderr, "usage: %s X.f64 m n\n", argv[0]);
        return 2;
    }
    const std::size_t m = std::stoul(argv[2]), n = std::stoul(argv[3]);
    hpclust::Dataset X(m, n);
    std::ifstream f(argv[1], std::ios::binary);
    f.read(reinterpret_cast<char*>(X.values.data()), (std::streamsize)(m * n * sizeof(double)));
    try {
        hpclust::RngStream rng(7);
        hpclust::Dataset S = hpclust::draw_sample(X, 500, rng);
        hpclust::DistCounter nd;
        hpclust::CentroidSet C0 = hpclust::kmeanspp_seed(S, 5, hpclust::SeedConfig{}, rng,
                                                         hpclust::ParallelPolicy::sequential(), &nd);
        hpclust::LloydOutcome lo = hpclust::kmeans(S, C0, hpclust::LloydConfig{}, &nd);
        const double f_full = hpclust::mssc_objective(lo.centroids.any_degenerate() ? C0 : lo.centroids, X);
        hpclust::EngineConfig cfg;
        cfg.k = 5;
        cfg.sample_size = 500;
        cfg.n_workers = 3;
        cfg.max_samples = 4;
        cfg.strategy = hpclust::Strategy::cooperative();
        cfg.master_seed = 11;
        hpclust::ClusteringResult r = hpclust::run(X, cfg);
        // the reference CLI's default schedule: a wall-clock budget (engine.hpp:348-374)
        hpclust::EngineConfig wcfg = cfg;
        wcfg.max_samples.reset();
        wcfg.time_limit = 0.2;
        hpclust::ClusteringResult rw = hpclust::run(X, wcfg);
        std::printf("{\"wall_seconds\": %.17g, \"wall_samples\": %zu, \"wall_full\": %.17g, ", rw.wall_seconds,
                    rw.total_samples, rw.full_objective.value_or(-1.0));
        // the same budget with free-running workers and immediate publication (engine.hpp:355-371;
        // EngineConfig::free_running, an extension): every worker on its own, device Philox streams
        hpclust::EngineConfig fcfg = wcfg;
        fcfg.rng_mode = hpclust::RngMode::philox;
        fcfg.free_running = true;
        fcfg.free_group = 1;
        hpclust::ClusteringResult rf = hpclust::run(X, fcfg);
        std::size_t fsum = 0, fmin = ~std::size_t{0};
        double tw_max = 0.0;
        for (const auto& w : rf.per_worker) {
            fsum += w.samples_processed;
            fmin = std::min(fmin, w.samples_processed);
            tw_max = std::max(tw_max, w.t_w);
        }
        std::printf("\"free_samples\": %zu, \"free_sum\": %zu, \"free_min\": %zu, \"free_tw_max\": %.17g, "
                    "\"free_full\": %.17g, \"free_pubs\": %zu, \"free_seconds\": %.17g, ",
                    rf.total_samples, fsum, fmin, tw_max, rf.full_objective.value_or(-1.0), rf.publications.size(),
                    rf.wall_seconds);
        std::printf("\"sample0\": %.17g, \"seed_c0\": %.17g, \"lloyd_obj\": %.17g, \"lloyd_iters\": %zu, "
                    "\"lloyd_stop\": \"%s\", \"nd\": %lld, \"f_full\": %.17g, \"run_full\": %.17g, "
                    "\"run_best\": %d, \"run_nd\": %lld, \"run_c0\": %.17g, \"pubs\": %zu}\n",
                    S.values[0], C0.centers[0], lo.objective, lo.iterations, hpclust::to_string(lo.converged_by),
                    (long long)nd.value(), f_full, r.full_objective.value_or(-1.0), r.best_worker,
                    (long long)r.distance_evals, r.centroids.centers[0], r.publications.size());
    } catch (const std::exception& e) {
        std::printf("{\"error\": \"%s\"}\n", e.what());
        return 1;
    }
    return 0;
}
