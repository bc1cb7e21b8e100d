// Drop-in use of the reference's baselines API (hpclust/baselines.hpp) on the B200 kernels:
// reads X (raw fp64, m x n), runs forgy_kmeans (p = 0) or pbk_bdc (segment size p) with
// RngStream(seed), prints a JSON line (objective, n_d, samples) and writes centroids, flags and
// labels next to X (X.path + ".C", ".F", ".L") for the test to compare with the reference.
#include <cstdio>
#include <cstdlib>
#include <fstream>

#include "hpclust/baselines.hpp"

int main(int argc, char** argv) {
    if (argc < 7) {
        std::fprintf(stderr, "usage: %s X.f64 m n k p seed\n", argv[0]);
        return 2;
    }
    const std::size_t m = std::strtoull(argv[2], nullptr, 10), n = std::strtoull(argv[3], nullptr, 10);
    const std::size_t k = std::strtoull(argv[4], nullptr, 10), p = std::strtoull(argv[5], nullptr, 10);
    const std::uint64_t seed = std::strtoull(argv[6], nullptr, 10);
    try {
        hpclust::Dataset X(m, n);
        std::ifstream(argv[1], std::ios::binary).read(reinterpret_cast<char*>(X.values.data()), (std::streamsize)(m * n * 8));
        hpclust::RngStream rng(seed);
        hpclust::ClusteringResult r;
        if (p == 0) {
            r = hpclust::forgy_kmeans(X, k, hpclust::LloydConfig{}, rng);
        } else {
            hpclust::PbkConfig pc;
            pc.segment_size = p;
            r = hpclust::pbk_bdc(X, k, pc, rng);
        }
        const std::string base = argv[1];
        std::ofstream(base + ".C", std::ios::binary)
            .write(reinterpret_cast<const char*>(r.centroids.centers.data()), (std::streamsize)(k * n * 8));
        std::ofstream(base + ".F", std::ios::binary)
            .write(reinterpret_cast<const char*>(r.centroids.degenerate.data()), (std::streamsize)k);
        std::ofstream(base + ".L", std::ios::binary)
            .write(reinterpret_cast<const char*>(r.assignment->labels.data()), (std::streamsize)(m * 4));
        std::printf("{\"f\": %.17g, \"nd\": %lld, \"samples\": %zu}\n", r.full_objective.value_or(-1.0),
                    (long long)r.distance_evals, r.total_samples);
    } catch (const std::exception& e) {
        std::printf("{\"error\": \"%s\"}\n", e.what());
        return 1;
    }
    return 0;
}
