// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// The reference's own worker step (engine.hpp:238-267: reinit_degenerate, seeding.hpp:125-133,
// then kmeans, lloyd.hpp:100-164) driven by INJECTED random draws, so a PHILOX-mode GPU round
// (sample indices and K-means++ draws generated on the device) can be replayed through the
// UNMODIFIED reference code with exactly the device's draws.
//
// How: the reference's RngStream owns a std::mt19937_64 (rng.hpp:95). This translation unit
// alone renames that engine type to `std::hpref_inject_engine` before including the reference
// headers; the injected engine returns queued 64-bit values while a queue is installed on the
// calling thread and otherwise behaves exactly like std::mt19937_64. Every draw the reference
// makes goes through RngStream's unmodified next_unit / uniform_index / weighted_index, so:
//   * the c-th unit of a D^2 slot = (v >> 11) * 2^-53 for the injected v (rng.hpp:38-40);
//   * the first-centre uniform_index(s) (seeding.hpp:74) returns x % s for an injected x < s.
// Built into its own shared object (oracle/_ref/libhpclust_ref_inject.so) so the one-definition
// rule holds: libhpclust_ref.so keeps the stock engine.
#include <cstdint>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>

namespace std {
struct hpref_inject_engine {
    using result_type = std::uint64_t;
    static constexpr result_type min() { return 0; }
    static constexpr result_type max() { return ~result_type(0); }
    explicit hpref_inject_engine(result_type seed = 5489u) : real(seed) {}
    result_type operator()();
    std::mt19937_64 real;
};
}  // namespace std

namespace {
thread_local const std::uint64_t* g_q = nullptr;
thread_local std::int64_t g_qn = 0, g_qpos = 0, g_overrun = 0;
thread_local std::string g_err;
}  // namespace

std::uint64_t std::hpref_inject_engine::operator()() {
    if (g_q) {
        if (g_qpos < g_qn) return g_q[g_qpos++];
        ++g_overrun;  // more draws than injected: flagged to the caller
        return 0;
    }
    return real();
}

#define mt19937_64 hpref_inject_engine
#include "hpclust/hpclust.hpp"
#undef mt19937_64

using namespace hpclust;

extern "C" {

const char* hpref_inject_last_error() { return g_err.c_str(); }

// One reference worker step on the sample S (s x n, fp64) from init (C_in, flags_in): reinit_degenerate
// with the injected draws, then kmeans. Outputs the reseeded init, the Lloyd outcome and n_d;
// *consumed = draws used (an overrun is an error: the caller injected too few).
int hpref_inject_step(const double* S, std::size_t s, std::size_t n, const double* C_in, const std::uint8_t* flags_in,
                      std::size_t k, std::size_t candidates, std::size_t max_iters, double rel_tol,
                      const std::uint64_t* draws, std::int64_t n_draws, double* C_seeded, double* C_out,
                      std::uint8_t* flags_out, double* objective, std::int64_t* iterations, std::int32_t* stop,
                      std::int64_t* n_d, std::int64_t* consumed, std::int32_t* labels) {
    try {
        Dataset ds(s, n);
        std::memcpy(ds.values.data(), S, s * n * sizeof(double));
        CentroidSet c0(k, n);
        std::memcpy(c0.centers.data(), C_in, k * n * sizeof(double));
        std::memcpy(c0.degenerate.data(), flags_in, k);
        SeedConfig sc;
        sc.candidates_per_center = candidates;
        DistCounter ctr;
        RngStream rng(0);
        g_q = draws;
        g_qn = n_draws;
        g_qpos = 0;
        g_overrun = 0;
        CentroidSet init = reinit_degenerate(c0, ds, sc, rng, ParallelPolicy::sequential(), &ctr);
        g_q = nullptr;
        if (consumed) *consumed = g_qpos;
        if (g_overrun) throw std::runtime_error("inject: the reference drew more values than were injected");
        if (C_seeded) std::memcpy(C_seeded, init.centers.data(), k * n * sizeof(double));
        LloydConfig lc;
        lc.max_iters = max_iters;
        lc.rel_tol = rel_tol;
        LloydOutcome out = kmeans(ds, init, lc, &ctr);
        std::memcpy(C_out, out.centroids.centers.data(), k * n * sizeof(double));
        std::memcpy(flags_out, out.centroids.degenerate.data(), k);
        *objective = out.objective;
        *iterations = static_cast<std::int64_t>(out.iterations);
        *stop = static_cast<std::int32_t>(out.converged_by);
        *n_d = ctr.value();
        if (labels) std::memcpy(labels, out.assignment.labels.data(), s * sizeof(std::int32_t));
        return 0;
    } catch (const std::invalid_argument& e) {
        g_q = nullptr;
        g_err = e.what();
        return 1;
    } catch (const std::logic_error& e) {
        g_q = nullptr;
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_q = nullptr;
        g_err = e.what();
        return 4;
    }
}

}  // extern "C"
