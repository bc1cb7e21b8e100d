// The device-resident drop-in overloads (hpclust::DeviceDataset, additive to the reference API):
// X is uploaded once, then draw_sample / worker_step / mssc_objective / run read it in place. Prints
// the H2D bytes of dataset uploads around 100 draw_sample calls and the results of the resident and
// the per-call paths (which must agree draw for draw). argv: X.f64 m n.
#include <cstdio>
#include <fstream>
#include <vector>

#include "hpclust/hpclust.hpp"
#include "hpclust/io.hpp"
#include "hpclust/parallel.hpp"

int main(int argc, char** argv) {
    if (argc < 4) return 2;
    const std::size_t m = std::stoul(argv[2]), n = std::stoul(argv[3]);
    hpclust::Dataset X(m, n);
    std::ifstream f(argv[1], std::ios::binary);
    f.read(reinterpret_cast<char*>(X.values.data()), (std::streamsize)(m * n * sizeof(double)));
    try {
        // reference code that uses parallel.hpp compiles unchanged
        hpclust::LloydConfig lc;
        lc.parallel_rows = true;
        const std::size_t chunks = lc.policy().n_chunks;
        const hpclust::RowRange rr = hpclust::chunk_range(m, 4, 3);
        std::vector<double> part(4, 0.0);
        hpclust::ThreadPool::global().run_chunks(4, [&](std::size_t c) {
            const auto r = hpclust::chunk_range(m, 4, c);
            for (std::size_t i = r.begin; i < r.end; ++i) part[c] += X.values[i * n];
        });
        hpclust::DeviceDataset dX(X);
        hpclust::gpu::context();
        const long long up0 = (long long)hpcg_ctx_upload_bytes(hpclust::gpu::context());
        hpclust::RngStream ra(5), rb(5);
        double chk = 0.0;
        std::vector<hpclust::Dataset> first;
        for (int i = 0; i < 100; ++i) {
            hpclust::Dataset S = hpclust::draw_sample(dX, 256, ra);
            chk += S.values[0];
            if (i < 3) first.push_back(std::move(S));
        }
        const long long up1 = (long long)hpcg_ctx_upload_bytes(hpclust::gpu::context());
        bool same = true;  // the reference-signature path (uploads X per call) draws the same rows
        for (int i = 0; i < 3; ++i) same = same && hpclust::draw_sample(X, 256, rb).values == first[(std::size_t)i].values;
        hpclust::EngineConfig cfg;
        cfg.k = 4;
        cfg.sample_size = 400;
        cfg.n_workers = 3;
        cfg.max_samples = 3;
        cfg.strategy = hpclust::Strategy::cooperative();
        cfg.master_seed = 3;
        hpclust::ClusteringResult r1 = hpclust::run(dX, cfg), r2 = hpclust::run(X, cfg);
        hpclust::WorkerState wa, wb;
        wa.incumbent = wb.incumbent = hpclust::CentroidSet::all_degenerate(4, n);
        hpclust::RngStream sa(9), sb(9);
        const bool acc_a = hpclust::worker_step(wa, sa, dX, wa.incumbent, cfg, [] { return 1.0; });
        const bool acc_b = hpclust::worker_step(wb, sb, X, wb.incumbent, cfg, [] { return 1.0; });
        // CSV ingest into page-locked memory (io.hpp load_dataset_pinned): same values as load_dataset,
        // the holder's rows upload and run like any Dataset
        hpclust::Dataset head(2000, n);
        std::copy_n(X.values.begin(), head.values.size(), head.values.begin());
        const std::string csv = std::string(argv[1]) + ".csv";
        hpclust::save_dataset(head, csv);
        hpclust::PinnedDataset pin = hpclust::load_dataset_pinned(csv);
        const bool pin_same = pin.X.values == hpclust::load_dataset(csv).values && pin.X.rows == 2000;
        hpclust::EngineConfig pcfg = cfg;
        pcfg.sample_size = 300;
        const bool pin_run = hpclust::run(pin.X, pcfg).centroids.centers == hpclust::run(head, pcfg).centroids.centers;
        std::printf("{\"pinned\": %d, \"pin_same\": %d, \"pin_run\": %d, ", pin.pinned ? 1 : 0, pin_same ? 1 : 0,
                    pin_run ? 1 : 0);
        std::printf("\"upload_bytes_100_draws\": %lld, \"draw_same\": %d, \"chk\": %.17g, \"run_same\": %d, "
                    "\"ws_same\": %d, \"ws_obj\": %.17g, \"f_dev\": %.17g, \"f_host\": %.17g, \"policy_chunks\": %zu, "
                    "\"rr\": [%zu, %zu], \"pool_sum\": %.17g}\n",
                    up1 - up0, same ? 1 : 0, chk,
                    (r1.centroids.centers == r2.centroids.centers && r1.distance_evals == r2.distance_evals) ? 1 : 0,
                    (acc_a == acc_b && wa.incumbent.centers == wb.incumbent.centers &&
                     wa.incumbent_objective == wb.incumbent_objective && sa.next_u64() == sb.next_u64()) ? 1 : 0,
                    wa.incumbent_objective, hpclust::mssc_objective(r1.centroids, dX),
                    hpclust::mssc_objective(r1.centroids, X), chunks, rr.begin, rr.end,
                    part[0] + part[1] + part[2] + part[3]);
    } catch (const std::exception& e) {
        std::printf("{\"error\": \"%s\"}\n", e.what());
        return 1;
    }
    return 0;
}
