/* TEST INFRASTRUCTURE ONLY — the checker, never the product.
 *
 * Plain-C restatement of the reference HPClust hot path (/root/reference/proj/include/hpclust),
 * one function per reference routine, each citing the file:line it follows. Compiled by
 * oracle/Makefile with -ffp-contract=off so every fp64 operation rounds exactly as the
 * reference Release build does. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load it.
 *
 * Pinned against: the reference itself (oracle/_ref/libhpclust_ref.so, built from the
 * reference headers by oracle/Makefile) and the golden fixtures in tests/golden/
 * (SPEC.md examples + reference-generated traces).
 */
#ifndef HPCLUST_ORACLE_H
#define HPCLUST_ORACLE_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* rng.hpp:26-99 — std::mt19937_64 stream plus the hand-rolled distributions. */
typedef struct orc_rng {
    uint64_t mt[312];
    int idx;
    double spare;
    int has_spare;
} orc_rng;

uint64_t orc_splitmix64(uint64_t x);
void orc_rng_seed(orc_rng* r, uint64_t seed);
void orc_rng_derive(orc_rng* r, uint64_t master, uint64_t domain, uint64_t index);
uint64_t orc_rng_next_u64(orc_rng* r);
double orc_rng_next_unit(orc_rng* r);
uint64_t orc_rng_uniform_index(orc_rng* r, uint64_t n); /* n == 0 -> returns UINT64_MAX */
size_t orc_sizeof_rng(void);

/* status codes shared with the product C-ABI: 0 ok, 1 invalid_argument, 2 logic_error,
 * 3 no solution. orc_last_error() holds the reference's message text. */
const char* orc_last_error(void);

int orc_assign(const double* X, size_t m, size_t n, const double* C, const uint8_t* flags, size_t k,
               size_t n_chunks, int32_t* labels, int64_t* counts, double* cost, int64_t* n_d);

int orc_kmeans(const double* S, size_t s, size_t n, const double* C_init, const uint8_t* flags_init, size_t k,
               size_t max_iters, double rel_tol, size_t n_chunks, double* C_out, uint8_t* flags_out,
               int32_t* labels, int64_t* counts, double* objective, int64_t* iterations, int32_t* stop,
               int64_t* n_d, double* history, int64_t history_cap, int64_t* history_len);

int orc_reinit_degenerate(const double* S, size_t s, size_t n, const double* C_in, const uint8_t* flags_in,
                          size_t k, size_t candidates, size_t n_chunks, orc_rng* rng, double* C_out,
                          uint8_t* flags_out, int64_t* n_d);

/* Same as orc_reinit_degenerate but the random draws come from an explicit list, in the
 * order the reference consumes them: [first-row index (as double) if no valid centre],
 * then `candidates` next_unit() values per pending slot. Returns slots filled via *filled. */
int orc_seed_with_uniforms(const double* S, size_t s, size_t n, const double* C_in, const uint8_t* flags_in,
                           size_t k, size_t candidates, size_t first_row, const double* units,
                           double* C_out, uint8_t* flags_out, int64_t* n_d, int64_t* filled);

int orc_draw_indices(size_t m, size_t s, orc_rng* rng, int64_t* idx_out);

typedef struct orc_run_cfg {
    uint64_t k, sample_size, n_workers, max_samples;
    double time_limit; /* unused: the oracle restates the deterministic (lockstep) schedule only */
    int32_t strategy;  /* 0 inner 1 competitive 2 cooperative 3 hybrid */
    double phase_t1, phase_t2;
    uint64_t master_seed;
    uint64_t candidates, max_iters;
    double rel_tol;
    uint64_t n_threads; /* chunk count used by the inner strategy (0 -> 8) */
    int32_t compute_full_objective, compute_assignment;
} orc_run_cfg;

typedef struct orc_run_out {
    double full_objective;
    int32_t has_full_objective;
    int32_t best_worker;
    double best_sample_objective;
    double clustering_time, clustering_time_first_finisher, wall_seconds;
    uint64_t total_samples;
    int64_t distance_evals;
    int64_t n_publications;
} orc_run_out;

int orc_run(const double* X, size_t m, size_t n, const orc_run_cfg* c, orc_run_out* o, double* centroids,
            uint8_t* flags, int32_t* labels, double* publications, int64_t pub_cap, double* worker_obj,
            double* traces, int64_t trace_cap, int64_t* trace_len);

#ifdef __cplusplus
}
#endif
#endif
