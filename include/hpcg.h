/* hpcg.h — C-ABI of the B200-native HPClust hot path (libhpcg.so).
 *
 * The drop-in boundary: plain pointers, sizes and status codes; no C++ or torch types.
 * The C++ drop-in headers include/hpclust/ (*.hpp) (same namespace, types and signatures as
 * the reference's proj/include/hpclust) are implemented on top of these calls, and
 * INTEGRATION.md shows the ctypes binding the Python mirror uses.
 *
 * Each entry point cites the reference interface it replaces (paths relative to
 * /root/reference/proj/include/hpclust/).
 *
 * Conventions
 *   - return value: HPCG_OK or an HPCG_E* status; hpcg_last_error() returns the message
 *     (thread-local), which for EINVAL / ELOGIC / ENOSOL is the reference's own
 *     exception text (core.hpp:17-19 require(), lloyd.hpp:118, engine.hpp:159-161).
 *   - "host" pointers are caller-owned host memory; "dev" pointers are caller-owned
 *     device memory on the context's device. Nothing is retained after a call returns
 *     except inside opaque handles (hpcg_ctx, hpcg_dataset, hpcg_engine).
 *   - all fp64 centroid arrays are row-major k x n; degenerate flags are k bytes (1 = degenerate).
 *   - there is no CPU fallback: without a usable sm_100 device every call returns HPCG_ECUDA.
 */
#ifndef HPCG_H
#define HPCG_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HPCG_ABI_VERSION 2 /* 2: hpcg_engine_cfg gained free_running / free_group */
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

typedef enum hpcg_status {
    HPCG_OK = 0,
    HPCG_EINVAL = 1,      /* std::invalid_argument in the reference (core.hpp:17-19)       */
    HPCG_ELOGIC = 2,      /* std::logic_error (lloyd.hpp:118, engine.hpp:259, 193)         */
    HPCG_ENOSOL = 3,      /* NoSolutionError (engine.hpp:159-161)                          */
    HPCG_ECUDA = 4,       /* CUDA runtime / device failure                                */
    HPCG_ENCCL = 5,       /* collective failure (multi-GPU exchange)                      */
    HPCG_EUNSUPPORTED = 6 /* shape outside this build's kernels (e.g. n > 32 or k > 32)    */
} hpcg_status;

typedef enum hpcg_dtype { HPCG_F32 = 0, HPCG_F64 = 1 } hpcg_dtype;

/* lloyd.hpp:22 LloydStop */
typedef enum hpcg_stop { HPCG_STOP_TOLERANCE = 0, HPCG_STOP_MAX_ITERS = 1, HPCG_STOP_FIXED_POINT = 2 } hpcg_stop;

/* engine.hpp:22 StrategyKind ("collective" in BASELINE.json config 4 == cooperative) */
typedef enum hpcg_strategy {
    HPCG_INNER = 0,
    HPCG_COMPETITIVE = 1,
    HPCG_COOPERATIVE = 2,
    HPCG_HYBRID = 3
} hpcg_strategy;

/* Random streams of the engine: REFERENCE replays the reference's per-worker mt19937_64
 * streams (rng.hpp, engine.hpp:457) on the host so draw_sample / K-means++ pick exactly the
 * reference's rows; PHILOX generates sample indices (keyed Feistel permutation) and draws on
 * the device (no host work per round; the product/benchmark mode). */
typedef enum hpcg_rng_mode { HPCG_RNG_REFERENCE = 0, HPCG_RNG_PHILOX = 1 } hpcg_rng_mode;

typedef struct hpcg_ctx hpcg_ctx;
typedef struct hpcg_dataset hpcg_dataset;
typedef struct hpcg_engine hpcg_engine;

const char* hpcg_last_error(void);
int hpcg_abi_version(void);

/* ---- context ----------------------------------------------------------------------- */
int hpcg_ctx_create(int device, hpcg_ctx** out);
int hpcg_ctx_destroy(hpcg_ctx* ctx);
/* Run on a caller stream (e.g. torch.cuda.current_stream().cuda_stream; NULL = the legacy
 * default stream, which is what torch's default stream handle 0 denotes). A context starts on
 * its own non-blocking stream. */
int hpcg_ctx_set_stream(hpcg_ctx* ctx, void* cuda_stream);
int hpcg_ctx_synchronize(hpcg_ctx* ctx);
/* Number of kernels this library launched on the context since creation (bench evidence). */
int64_t hpcg_ctx_launch_count(const hpcg_ctx* ctx);
/* Host -> device bytes this context's dataset uploads moved (hpcg_dataset_upload / hpcg_run). */
int64_t hpcg_ctx_upload_bytes(const hpcg_ctx* ctx);
/* Row cost of f(C, X) over fp32 data (the labels are exact in both modes): exact != 0 -- the
 * reference's fp64 distance per row (1e-12 relative); 0 (default) -- the north star's fp32 mode: the
 * row's squared distance in fp32 (direct form, FFMA2), accumulated in fp64 (<= 1e-5 relative; in
 * practice ~1e-8), which keeps the pass at the HBM rate. fp64 data always takes the exact cost. */
int hpcg_ctx_set_fp32_cost(hpcg_ctx* ctx, int exact);
/* Per-kernel device timing: when enabled, every worker-step / objective launch is bracketed
 * by CUDA events on the launching stream; hpcg_ctx_kernel_times synchronises and returns
 * (launch count, summed milliseconds) per kernel class: 0 worker step, 1 objective. */
int hpcg_ctx_enable_timing(hpcg_ctx* ctx, int enable);
int hpcg_ctx_kernel_times(hpcg_ctx* ctx, int64_t* counts, double* total_ms);
/* Measured FP32 FMA throughput of this device (FFMA2 loop, all SMs) in TFMA/s: the roofline
 * denominator for the Lloyd screen, measured at the clocks the device is running. */
int hpcg_probe_fma_peak(hpcg_ctx* ctx, double* tfma_per_s);

/* ---- datasets: X (m x n, row-major) resident in HBM  (core.hpp:34-50 Dataset) ------------ */
int hpcg_dataset_upload(hpcg_ctx* ctx, const void* X_host, hpcg_dtype dtype, int64_t m, int64_t n,
                        hpcg_dataset** out);
/* Page-lock caller-owned host memory for the lifetime of an ingest buffer (io.hpp:68-102 load_dataset
 * fills a std::vector; registered, its upload runs at the full PCIe rate instead of through the
 * driver's staging copies). The memory stays the caller's; unregister before freeing it. */
int hpcg_host_register(void* host, int64_t bytes);
int hpcg_host_unregister(void* host);
int hpcg_dataset_wrap(hpcg_ctx* ctx, const void* X_dev, hpcg_dtype dtype, int64_t m, int64_t n,
                      hpcg_dataset** out); /* borrows X_dev (must outlive the handle) */
/* Row-sharded X (multi-GPU global sampling): shard i holds shard_rows[i] rows at
 * shard_dev[i] -- local or peer memory (hpcg_ipc_open) -- in global row order; m = the sum. Sample
 * indices are global (engine.hpp:165-177 over all m rows), the gathers read remote rows over
 * NVLink. Borrowed pointers (must outlive the handle); at most 8 shards. */
int hpcg_dataset_wrap_sharded(hpcg_ctx* ctx, const void* const* shard_dev, const int64_t* shard_rows, int32_t nshards,
                              hpcg_dtype dtype, int64_t n, hpcg_dataset** out);
/* CUDA IPC of device memory between the processes of one node: a 72-byte handle (the
 * allocation's cudaIpcMemHandle_t + the pointer's offset inside it). */
#define HPCG_IPC_HANDLE_BYTES 72
int hpcg_ipc_export(const void* dev_ptr, void* handle_out);
int hpcg_ipc_open(hpcg_ctx* ctx, const void* handle, void** dev_ptr_out);
int hpcg_ipc_close(hpcg_ctx* ctx, void* dev_ptr, const void* handle);
int hpcg_dataset_destroy(hpcg_dataset* ds);
const void* hpcg_dataset_device_ptr(const hpcg_dataset* ds);

/* ---- full-data assignment / objective ---------------------------------------------------
 * Replaces core.hpp:212-221 assign_nearest, core.hpp:224-233 mssc_objective,
 * engine.hpp:197-205 final_assignment and engine.hpp:211-229 assign_valid_subset:
 * nearest VALID centre per row (strict <, ties -> lowest index), labels in original slot
 * numbering, per-cluster counts, cost = sum of exact reference distances.
 * require_valid != 0 reproduces assign_nearest/mssc_objective's "degenerate centroid
 * present" precondition; 0 gives assign_valid_subset's tolerant behaviour.
 * labels_host (m) / counts_host (k) may be NULL. *n_d += m * k_valid (core.hpp:205). */
int hpcg_assign(hpcg_ctx* ctx, const hpcg_dataset* ds, const double* C_host, const uint8_t* degenerate_host,
                int64_t k, int require_valid, int32_t* labels_host, int64_t* counts_host, double* cost,
                int64_t* n_d);
/* Same, device-resident in/out (bench path; no host copies). */
int hpcg_assign_dev(hpcg_ctx* ctx, const hpcg_dataset* ds, const double* C_dev, int64_t k_valid,
                    int32_t* labels_dev, double* cost_dev);

/* ---- batched worker step on explicit samples ----------------------------------------------
 * W independent (sample, init) problems in one launch: reinit_degenerate (seeding.hpp:125-133)
 * with injected draws, then kmeans (lloyd.hpp:100-164). Samples are rows idx_host[w*s+i] of
 * ds (draw order), or, when idx_host == NULL, ds itself is [W*s x n] (sample w = rows w*s..).
 * Draws follow the reference's consumption order (seeding.hpp:72-99): first_row_host[w] is
 * the uniform_index(s) used when w has no valid centre; units_host[w*units_stride + t*c + j]
 * the j-th next_unit() of the t-th filled-by-D^2 slot. Outputs (host, may be NULL except C_out):
 * C_out[W*k*n], flags_out[W*k], objective[W], iterations[W], stop[W] (hpcg_stop), n_d[W],
 * filled[W] (slots reseeded), labels[W*s], counts[W*k], history[W*hist_cap] + hist_len[W].
 * do_lloyd == 0 stops after seeding (kmeanspp_seed / reinit_degenerate).
 * Status: EINVAL "kmeans: degenerate centroid in init" if a worker still has a degenerate
 * slot after seeding (lloyd.hpp:104); ELOGIC on the monotone guard (lloyd.hpp:117-118). */
typedef struct hpcg_lloyd_cfg {
    int64_t max_iters;  /* lloyd.hpp:11 */
    double rel_tol;     /* lloyd.hpp:12 */
    int64_t candidates; /* seeding.hpp:13 */
} hpcg_lloyd_cfg;

int hpcg_worker_step_batched(hpcg_ctx* ctx, const hpcg_dataset* ds, const int64_t* idx_host, int64_t W, int64_t s,
                             const double* C_init_host, const uint8_t* flags_init_host, int64_t k,
                             const hpcg_lloyd_cfg* cfg, const int64_t* first_row_host, const double* units_host,
                             int64_t units_stride, int do_lloyd, double* C_out, uint8_t* flags_out,
                             double* objective, int32_t* iterations, int32_t* stop, int64_t* n_d, int32_t* filled,
                             int32_t* labels, int64_t* counts, double* history, int32_t hist_cap, int32_t* hist_len);

/* ---- sample gather (engine.hpp:165-177 draw_sample with the indices it would draw) --------- */
int hpcg_gather(hpcg_ctx* ctx, const hpcg_dataset* ds, const int64_t* idx_host, int64_t s, void* S_host);
/* Device sample definition of HPCG_RNG_PHILOX rounds (replaces engine.hpp:165-177 there): the
 * first s images of [0, m) under the keyed permutation of worker `worker` in round `round`
 * (distinct by construction). The engine uses key = its Philox key (hpcg_engine_cfg seed). */
int hpcg_sample_indices(hpcg_ctx* ctx, int64_t m, int64_t s, uint64_t key, uint32_t round, uint32_t worker,
                        int64_t* idx_out);
/* The same samples materialised: S_dev[w][i][:] = row prp_w(i) of ds for w < W (W*s*n elements of
 * ds's dtype, caller-owned device memory); worker w uses the stream of global worker worker_base + w.
 * The gather phase of the worker step on its own (bench.py measures its GB/s against HBM). */
int hpcg_sample_gather_dev(hpcg_ctx* ctx, const hpcg_dataset* ds, int64_t W, int64_t s, uint64_t key,
                           uint32_t round, int32_t worker_base, void* S_dev);
/* The K-means++ draws an HPCG_RNG_PHILOX round gives worker `worker` (seeding.hpp:72-99 consumption
 * order): *first_row = the uniform first-centre row when no_valid != 0 (the sample had no valid
 * centre), units[t*candidates + c] = the c-th unit draw of the t-th D^2-sampled slot, t < loops.
 * Host-side; lets a parity test replay a PHILOX run through the reference with the same draws. */
int hpcg_philox_seed_draws(uint64_t key, uint32_t round, uint32_t worker, int64_t s, int32_t no_valid,
                           int64_t loops, int64_t candidates, int64_t* first_row, double* units);
/* Reference-exact draw_sample indices: partial Fisher-Yates of the stream seeded `seed_state`
 * in O(s) (sparse swaps); advances the 312-word mt19937_64 state in place (rng.hpp). */
int hpcg_reference_draw_indices(uint64_t* mt_state, int32_t* mt_pos, int64_t m, int64_t s, int64_t* idx_out);

/* ---- reference random streams (rng.hpp:26-99): std::mt19937_64 state = 312 words + position.
 * Used to feed the kernels the exact draws the reference would make (parity / replay). */
int hpcg_rng_seed(uint64_t seed, uint64_t* mt_state, int32_t* mt_pos);
int hpcg_rng_derive(uint64_t master, uint64_t domain, uint64_t index, uint64_t* mt_state, int32_t* mt_pos);
/* kind 0: next_u64 (out u64), 1: next_unit (out f64), 2: uniform_index(bound) (out u64) */
int hpcg_rng_draw(uint64_t* mt_state, int32_t* mt_pos, int32_t kind, uint64_t bound, int64_t count, void* out);

/* ---- the HPClust engine (engine.hpp:444-499 run; lockstep schedule engine.hpp:380-436) ---- */
typedef struct hpcg_engine_cfg {
    int64_t k, sample_size, n_workers, max_samples; /* max_samples: per worker (rounds)      */
    int32_t strategy;                               /* hpcg_strategy                          */
    double phase_t1, phase_t2;                      /* hybrid split in rounds (engine.hpp:37) */
    uint64_t master_seed;
    int64_t candidates, max_iters;
    double rel_tol;
    int32_t compute_full_objective, compute_assignment;
    int32_t rng_mode;     /* hpcg_rng_mode */
    int32_t worker_base;  /* global id of worker 0 on this rank (multi-GPU), else 0 */
    double time_limit;    /* seconds; > 0: wall-clock schedule (engine.hpp:348-374) with max_samples an
                             optional per-worker cap (0 = none); 0: lockstep over max_samples rounds */
    int32_t free_running; /* wall-clock schedule only. 0: round granularity (every worker of a round starts
                             from the round's snapshot). 1: free-running workers with immediate publication
                             (engine.hpp:355-371): groups of workers advance on their own streams, each step
                             draws its init from a device-side versioned incumbent under a lock and an
                             accepted cooperative result is published the moment its group's step ends;
                             the device clock decides stop and phase per worker. Philox streams, one rank,
                             cluster-resident shapes. */
    int32_t free_group;   /* workers per free-running group (0 = automatic: ceil(W / 16)); 1 = every
                             worker publishes on its own */
} hpcg_engine_cfg;

typedef struct hpcg_run_out {
    double full_objective;
    int32_t has_full_objective;
    int32_t best_worker;
    double best_sample_objective;
    double clustering_time, clustering_time_first_finisher, wall_seconds;
    uint64_t total_samples;
    int64_t distance_evals;
    int64_t n_publications;
    double last_timestamp; /* every worker's t_w: rounds run (lockstep) or seconds at the last round end */
} hpcg_run_out;

/* Stepwise engine: create (validates like engine.hpp:70-86, allocates device state),
 * run rounds, finish (select_best engine.hpp:180-194 + final pass engine.hpp:483-491). */
int hpcg_engine_create(hpcg_ctx* ctx, const hpcg_dataset* ds, const hpcg_engine_cfg* cfg, hpcg_engine** out);
/* Back to round 0 with a new master seed (no allocation; stream-ordered). */
int hpcg_engine_reset(hpcg_engine* e, uint64_t master_seed);
int hpcg_engine_rounds(hpcg_engine* e, int64_t n_rounds);
/* The configured schedule to its end (replaces engine.hpp:459-462): lockstep max_samples rounds,
 * or -- time_limit set -- rounds until the limit (run_wall_clock, engine.hpp:348-374, at round
 * granularity: every worker of a round starts from the round's snapshot, accepted cooperative
 * incumbents are published at the round end in worker-id order, the hybrid switch happens at the
 * first round end past phase_t1 seconds, trace timestamps are seconds). */
int hpcg_engine_run(hpcg_engine* e);
int64_t hpcg_engine_round_index(const hpcg_engine* e);
/* Per-worker progress (WorkerState::samples_processed and t_w, engine.hpp:100, 250): the rounds run and
 * the last round's clock for the round-granular schedules, each worker's own count and clock for
 * the free-running schedule. Either pointer may be NULL. */
int hpcg_engine_worker_progress(hpcg_engine* e, int64_t* samples, double* t_w);
/* Diagnostics: per-CTA phase timestamps (%globaltimer ns) of subsequent rounds written to
 * trace_dev[W * cluster * 32] (NULL disables); mode 0 details the first Lloyd pass, mode 1
 * the first K-means++ slot. */
int hpcg_engine_set_trace(hpcg_engine* e, int64_t* trace_dev, int32_t mode);
/* Sum of n_d over the rounds run so far (device-side exact count; synchronises). */
int hpcg_engine_distance_evals(hpcg_engine* e, int64_t* n_d);
/* Outputs as hpref/orc_run: centroids[k*n], flags[k], labels[m] (if compute_assignment),
 * publications[pub_cap*4] = (version, worker, objective, timestamp), worker_obj[W],
 * traces[W*trace_cap*2] = (timestamp, objective), trace_len[W]. Any array may be NULL. */
int hpcg_engine_finish(hpcg_engine* e, hpcg_run_out* out, double* centroids, uint8_t* flags, int32_t* labels,
                       double* publications, int64_t pub_cap, double* worker_obj, double* traces,
                       int64_t trace_cap, int64_t* trace_len);
/* Per-worker outcome of the last round run (worker_step, engine.hpp:238-267): the sample objective
 * and Lloyd iterations / stop reason of this round's kmeans, its n_d, whether keep-the-best
 * accepted it, and how many degenerate slots K-means++ refilled. Any array may be NULL. */
int hpcg_engine_round_outcome(hpcg_engine* e, double* objective, int32_t* iterations, int32_t* stop, int64_t* n_d,
                              uint8_t* accepted, int32_t* filled);
/* The publication log (SharedBest::publication_log, engine.hpp:149-152): up to cap records of
 * (version, worker, objective, timestamp); *n_out = the number published so far. */
int hpcg_engine_publications(hpcg_engine* e, double* publications, int64_t cap, int64_t* n_out);
/* Per-worker incumbents after finish/rounds: C_out[W*k*n], f_out[W*k], obj_out[W] (any may be NULL). */
int hpcg_engine_worker_incumbents(hpcg_engine* e, double* C_out, uint8_t* f_out, double* obj_out);
int hpcg_engine_destroy(hpcg_engine* e);

/* The engine's Philox key (HPCG_RNG_PHILOX streams derive from it; see hpcg_sample_indices). */
uint64_t hpcg_engine_philox_key(const hpcg_engine* e);

/* ---- multi-GPU: one rank per GPU ------------------------------------------
 * Ranks own row shards of X (hpcg_dataset_wrap_sharded with peer-mapped shards gives every rank
 * global sampling, engine.hpp:165-177) and the contiguous worker ids [worker_base, worker_base + W).
 * With an exchange set, every round of a cooperative / hybrid engine publishes over ALL ranks'
 * workers exactly as one engine with every worker would (engine.hpp:391-402: global worker-id order,
 * strict <; the hybrid carry-over at engine.hpp:386,396): each rank all-gathers its round candidates
 * and its local best's centroids (one record of 4 + W + k*n + k doubles), and a device kernel on
 * every rank replays the publication scan, so the shared best and the publication log are
 * replicated bit-identically. hpcg_engine_finish then runs select_best over every rank's workers
 * (engine.hpp:180-194), f(C, X) as this rank's shard partial, and sums partials, n_d and sample
 * counts in rank order (labels, if requested, are this rank's rows). The collective is NCCL
 * (ncclAllGather on the context's stream over NVLink; libnccl.so.2 is loaded at run time) or, for
 * callers with their own transport, a host all-gather callback. */
/* NCCL unique id (128 bytes) created on one rank and shared with the others by the caller. */
int hpcg_comm_unique_id(void* id_out);
/* Collective over the ranks: attach an NCCL communicator (nranks, rank) to the context. */
int hpcg_ctx_attach_comm(hpcg_ctx* ctx, int32_t nranks, int32_t rank, const void* id);
int hpcg_ctx_comm_info(const hpcg_ctx* ctx, int32_t* nranks, int32_t* rank);
/* Host all-gather: copy bytes_per_rank from send into recv[rank * bytes_per_rank] on every rank
 * (rank order); return 0 on success. */
typedef int (*hpcg_allgather_fn)(const void* send_host, void* recv_host, size_t bytes_per_rank, void* user);
/* Make e one rank of a multi-rank engine (before its first round; collective over the ranks).
 * fn == NULL: the context's NCCL communicator (must match nranks / rank). */
int hpcg_engine_set_exchange(hpcg_engine* e, int32_t nranks, int32_t rank, hpcg_allgather_fn fn, void* user);

/* Multi-rank exchange hooks (cooperative / hybrid across GPUs):
 * export this rank's round candidates, import the merged shared best. */
int hpcg_engine_export_best(hpcg_engine* e, double* obj_out, int64_t* worker_out, double* C_out, uint8_t* f_out);
/* Install a shared best merged across ranks (strict < against the local one; version bump). */
int hpcg_engine_import_best(hpcg_engine* e, double obj, int64_t worker, const double* C, const uint8_t* f);

/* One-call run on host data (upload + rounds + final pass): the e2e path. */
int hpcg_run(hpcg_ctx* ctx, const void* X_host, hpcg_dtype dtype, int64_t m, int64_t n, const hpcg_engine_cfg* cfg,
             hpcg_run_out* out, double* centroids, uint8_t* flags, int32_t* labels, double* publications,
             int64_t pub_cap, double* worker_obj, double* traces, int64_t trace_cap, int64_t* trace_len);

/* ---- synthetic data (BASELINE.json configs; seeded Gaussian mixtures, fp32 or fp64) ------- */
/* Generated on the host, keyed by global row index (independent of thread count). */
int hpcg_gen_mixture(void* X_out, hpcg_dtype dtype, int64_t m, int64_t n, int64_t n_comp, const double* means,
                     const double* sigmas, const double* weights, double noise_frac, double noise_lo,
                     double noise_hi, uint64_t seed, int n_threads);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif
