// hpclust::run over every GPU of the node (additive overload run(X, cfg, devices)): X row-sharded,
// global sampling through peer-mapped shards, the library's NCCL exchange every round. Prints the
// multi-GPU and the single-GPU results (which must agree). argv: X.f64 m n.
#include <cstdio>
#include <fstream>
#include <vector>

#include <cuda_runtime_api.h>

#include "hpclust/hpclust.hpp"

int main(int argc, char** argv) {
    if (argc < 4) return 2;
    const std::size_t m = std::stoul(argv[2]), n = std::stoul(argv[3]);
    hpclust::Dataset X(m, n);
    std::ifstream f(argv[1], std::ios::binary);
    f.read(reinterpret_cast<char*>(X.values.data()), (std::streamsize)(m * n * sizeof(double)));
    int ndev = 0;
    cudaGetDeviceCount(&ndev);
    std::vector<int> devs;
    for (int d = 0; d < ndev; ++d) devs.push_back(d);
    try {
        hpclust::EngineConfig cfg;
        cfg.k = 6;
        cfg.sample_size = 2000;
        cfg.n_workers = 8;
        cfg.max_samples = 4;
        cfg.strategy = hpclust::Strategy::cooperative();
        cfg.master_seed = 12;
        hpclust::ClusteringResult rm = hpclust::run(X, cfg, devs), r1 = hpclust::run(X, cfg);
        std::printf("{\"devices\": %d, \"same_centroids\": %d, \"nd_multi\": %lld, \"nd_single\": %lld, "
                    "\"best_multi\": %d, \"best_single\": %d, \"f_multi\": %.17g, \"f_single\": %.17g, "
                    "\"pubs\": %zu, \"workers\": %zu}\n",
                    ndev, rm.centroids.centers == r1.centroids.centers ? 1 : 0, (long long)rm.distance_evals,
                    (long long)r1.distance_evals, rm.best_worker, r1.best_worker, rm.full_objective.value_or(-1),
                    r1.full_objective.value_or(-1), rm.publications.size(), rm.per_worker.size());
    } catch (const std::exception& e) {
        std::printf("{\"error\": \"%s\"}\n", e.what());
        return 1;
    }
    return 0;
}
