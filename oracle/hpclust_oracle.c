/* TEST INFRASTRUCTURE ONLY — the checker, never the product. See hpclust_oracle.h.
 *
 * Plain-C restatement of the reference's hot path. Reference paths are relative to
 * /root/reference/proj/include/hpclust/. Compile with -ffp-contract=off.
 */
#include "hpclust_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[256];
static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}
const char* orc_last_error(void) { return g_err; }

/* ------------------------------------------------------------------ rng.hpp */

/* rng.hpp:12-17 */
uint64_t orc_splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

/* std::mt19937_64 (parameters fixed by the C++ standard, [rand.predef]); rng.hpp:96 */
#define MT_N 312
#define MT_M 156
void orc_rng_seed(orc_rng* r, uint64_t seed) {
    r->mt[0] = seed;
    for (int i = 1; i < MT_N; ++i)
        r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->idx = MT_N;
    r->spare = 0.0;
    r->has_spare = 0;
}

/* rng.hpp:30-33 */
void orc_rng_derive(orc_rng* r, uint64_t master, uint64_t domain, uint64_t index) {
    orc_rng_seed(r, orc_splitmix64(master ^ orc_splitmix64(domain ^ orc_splitmix64(index))));
}

static void mt_twist(orc_rng* r) {
    const uint64_t upper = 0xFFFFFFFF80000000ULL, lower = 0x7FFFFFFFULL;
    for (int i = 0; i < MT_N; ++i) {
        uint64_t y = (r->mt[i] & upper) | (r->mt[(i + 1) % MT_N] & lower);
        uint64_t v = r->mt[(i + MT_M) % MT_N] ^ (y >> 1);
        if (y & 1ULL) v ^= 0xB5026F5AA96619E9ULL;
        r->mt[i] = v;
    }
    r->idx = 0;
}

uint64_t orc_rng_next_u64(orc_rng* r) {
    if (r->idx >= MT_N) mt_twist(r);
    uint64_t z = r->mt[r->idx++];
    z ^= (z >> 29) & 0x5555555555555555ULL;
    z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
    z ^= (z << 37) & 0xFFF7EEE000000000ULL;
    z ^= z >> 43;
    return z;
}

/* rng.hpp:38-40: 53-bit unit double */
double orc_rng_next_unit(orc_rng* r) { return (double)(orc_rng_next_u64(r) >> 11) * 0x1.0p-53; }

/* rng.hpp:43-53: rejection sampling below the largest multiple of n */
uint64_t orc_rng_uniform_index(orc_rng* r, uint64_t n) {
    if (n == 0) return UINT64_MAX;
    const uint64_t limit = UINT64_MAX - UINT64_MAX % n;
    uint64_t x;
    do {
        x = orc_rng_next_u64(r);
    } while (x >= limit);
    return x % n;
}

size_t orc_sizeof_rng(void) { return sizeof(orc_rng); }

/* rng.hpp:83-93: first index whose cumulative weight exceeds u = unit * total */
static size_t weighted_index_u(const double* cum, size_t len, double unit) {
    const double u = unit * cum[len - 1];
    size_t lo = 0, hi = len - 1;
    while (lo < hi) {
        size_t mid = lo + (hi - lo) / 2;
        if (cum[mid] <= u)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

/* ------------------------------------------------------------- parallel.hpp */

/* parallel.hpp:106-112 */
static void chunk_range(size_t rows, size_t n_chunks, size_t chunk, size_t* b, size_t* e) {
    size_t base = rows / n_chunks, extra = rows % n_chunks;
    *b = chunk * base + (chunk < extra ? chunk : extra);
    *e = *b + base + (chunk < extra ? 1 : 0);
}

/* core.hpp:119-122 (ParallelPolicy::chunks_for), n_chunks<=1 means sequential */
static size_t chunks_for(size_t n_chunks, size_t rows) {
    if (n_chunks <= 1 || rows == 0) return 1;
    return n_chunks < rows ? n_chunks : rows;
}

/* ----------------------------------------------------------------- core.hpp */

/* core.hpp:100-108 and the inlined copy at core.hpp:147-152: ascending d, no FMA */
static double sqdist(const double* a, const double* b, size_t n) {
    double acc = 0.0;
    for (size_t d = 0; d < n; ++d) {
        const double diff = a[d] - b[d];
        acc += diff * diff;
    }
    return acc;
}

/* core.hpp:138-207: assign rows chunk by chunk, merge partials in chunk order.
 * centre j is C + idx[j]*n (idx == NULL: identity). Produces labels in [0,kk),
 * counts[kk], sums[kk*n], cost. */
static void assign_and_reduce(const double* X, size_t m, size_t n, const double* C, const size_t* idx, size_t kk,
                              size_t n_chunks, int32_t* labels, int64_t* counts, double* sums, double* cost) {
    const size_t chunks = chunks_for(n_chunks, m);
    int64_t* pc = calloc(kk, sizeof(int64_t));
    double* ps = calloc(kk * n, sizeof(double));
    memset(counts, 0, kk * sizeof(int64_t));
    memset(sums, 0, kk * n * sizeof(double));
    double total = 0.0;
    for (size_t c = 0; c < chunks; ++c) {
        size_t b, e;
        chunk_range(m, chunks, c, &b, &e);
        memset(pc, 0, kk * sizeof(int64_t));
        memset(ps, 0, kk * n * sizeof(double));
        double pcost = 0.0;
        for (size_t i = b; i < e; ++i) {
            const double* x = X + i * n;
            double best = INFINITY;
            size_t bj = 0;
            for (size_t j = 0; j < kk; ++j) { /* strict <, ties -> lowest j (core.hpp:153) */
                const double dj = sqdist(x, C + (idx ? idx[j] : j) * n, n);
                if (dj < best) {
                    best = dj;
                    bj = j;
                }
            }
            labels[i] = (int32_t)bj;
            pc[bj] += 1;
            pcost += best;
            for (size_t d = 0; d < n; ++d) ps[bj * n + d] += x[d];
        }
        total += pcost; /* core.hpp:199-204 merge order */
        for (size_t j = 0; j < kk; ++j) counts[j] += pc[j];
        for (size_t q = 0; q < kk * n; ++q) sums[q] += ps[q];
    }
    *cost = total;
    free(pc);
    free(ps);
}

/* engine.hpp:197-229 (final_assignment / assign_valid_subset): valid centres only,
 * labels remapped to the original slots; n_d += m * k_valid (core.hpp:205). */
int orc_assign(const double* X, size_t m, size_t n, const double* C, const uint8_t* flags, size_t k,
               size_t n_chunks, int32_t* labels, int64_t* counts, double* cost, int64_t* n_d) {
    size_t* valid = malloc((k ? k : 1) * sizeof(size_t));
    size_t kv = 0;
    for (size_t j = 0; j < k; ++j)
        if (!flags || !flags[j]) valid[kv++] = j;
    if (kv == 0) {
        free(valid);
        return fail(1, "assignment: every centroid is degenerate");
    }
    int32_t* lab = malloc((m ? m : 1) * sizeof(int32_t));
    int64_t* cnt = malloc(kv * sizeof(int64_t));
    double* sums = malloc(kv * n * sizeof(double));
    double f;
    assign_and_reduce(X, m, n, C, valid, kv, n_chunks, lab, cnt, sums, &f);
    if (counts) memset(counts, 0, k * sizeof(int64_t));
    for (size_t i = 0; i < m; ++i) {
        const size_t j = valid[lab[i]];
        if (labels) labels[i] = (int32_t)j;
        if (counts) counts[j] += 1;
    }
    if (cost) *cost = f;
    if (n_d) *n_d = (int64_t)m * (int64_t)kv;
    free(valid);
    free(lab);
    free(cnt);
    free(sums);
    return 0;
}

/* ---------------------------------------------------------------- lloyd.hpp */

/* lloyd.hpp:75-89: reciprocal-then-multiply; empty cluster keeps the fallback centre */
static void means_from_sums(const double* sums, const int64_t* counts, size_t k, size_t n, const double* fallback,
                            double* out) {
    for (size_t j = 0; j < k; ++j) {
        if (counts[j] > 0) {
            const double inv = 1.0 / (double)counts[j];
            for (size_t d = 0; d < n; ++d) out[j * n + d] = sums[j * n + d] * inv;
        } else {
            memcpy(out + j * n, fallback + j * n, n * sizeof(double));
        }
    }
}

/* lloyd.hpp:100-164 (kmeans). stop: 0 tolerance, 1 max_iters, 2 fixed_point (lloyd.hpp:22). */
int orc_kmeans(const double* S, size_t s, size_t n, const double* C_init, const uint8_t* flags_init, size_t k,
               size_t max_iters, double rel_tol, size_t n_chunks, double* C_out, uint8_t* flags_out,
               int32_t* labels, int64_t* counts, double* objective, int64_t* iterations, int32_t* stop,
               int64_t* n_d, double* history, int64_t history_cap, int64_t* history_len) {
    if (max_iters < 1) return fail(1, "kmeans: max_iters must be positive");
    if (!(rel_tol > 0.0)) return fail(1, "kmeans: rel_tol must be positive");
    if (flags_init)
        for (size_t j = 0; j < k; ++j)
            if (flags_init[j]) return fail(1, "kmeans: degenerate centroid in init");

    double* C = malloc(k * n * sizeof(double));
    double* Cn = malloc(k * n * sizeof(double));
    double* sums = malloc(k * n * sizeof(double));
    int64_t* cnt = malloc(k * sizeof(int64_t));
    int32_t* lab = malloc((s ? s : 1) * sizeof(int32_t));
    memcpy(C, C_init, k * n * sizeof(double));
    int64_t iters = 0, hlen = 0, evals = 0;
    double f_prev = INFINITY, last = 0.0, f = 0.0;
    int32_t why = 1; /* max_iters (lloyd.hpp:38 default) */
    int rc = 0, done = 0;

#define PUSH_HISTORY(v)                                                                  \
    do {                                                                                 \
        if (hlen > 0 && (v) > last * (1.0 + 1e-12)) { /* lloyd.hpp:114-121 */           \
            rc = fail(2, "kmeans: objective increased between iterations");             \
            goto out;                                                                    \
        }                                                                                \
        if (history && hlen < history_cap) history[hlen] = (v);                          \
        last = (v);                                                                      \
        ++hlen;                                                                          \
    } while (0)

    while ((size_t)iters < max_iters) {
        ++iters;
        assign_and_reduce(S, s, n, C, NULL, k, n_chunks, lab, cnt, sums, &f);
        evals += (int64_t)s * (int64_t)k;
        PUSH_HISTORY(f);
        means_from_sums(sums, cnt, k, n, C, Cn);
        int same = 1;
        for (size_t q = 0; q < k * n; ++q)
            if (!(Cn[q] == C[q])) {
                same = 0;
                break;
            }
        if (same) { /* lloyd.hpp:131-138 */
            why = 2;
            memcpy(C, Cn, k * n * sizeof(double));
            done = 1;
            break;
        }
        memcpy(C, Cn, k * n * sizeof(double));
        if (isfinite(f_prev)) { /* lloyd.hpp:141-148 */
            const double improvement = f_prev > 0.0 ? (f_prev - f) / f_prev : 0.0;
            if (improvement < rel_tol) {
                why = 0;
                f_prev = f;
                break;
            }
        }
        f_prev = f;
        if ((size_t)iters == max_iters) why = 1;
    }
    if (!done) { /* closing pass, lloyd.hpp:155-163 */
        assign_and_reduce(S, s, n, C, NULL, k, n_chunks, lab, cnt, sums, &f);
        evals += (int64_t)s * (int64_t)k;
        PUSH_HISTORY(f);
    }
    if (C_out) memcpy(C_out, C, k * n * sizeof(double));
    if (flags_out)
        for (size_t j = 0; j < k; ++j) flags_out[j] = cnt[j] == 0 ? 1 : 0;
    if (labels) memcpy(labels, lab, s * sizeof(int32_t));
    if (counts) memcpy(counts, cnt, k * sizeof(int64_t));
    if (objective) *objective = f;
    if (iterations) *iterations = iters;
    if (stop) *stop = why;
    if (n_d) *n_d = evals;
    if (history_len) *history_len = hlen;
out:
#undef PUSH_HISTORY
    free(C);
    free(Cn);
    free(sums);
    free(cnt);
    free(lab);
    return rc;
}

/* -------------------------------------------------------------- seeding.hpp */

/* seeding.hpp:20-42: scratch = min(d2, dist(., c)), returns the chunk-ordered sum */
static double d2_min_update(const double* S, size_t s, size_t n, const double* c, const double* d2, double* scratch,
                            size_t n_chunks, int64_t* evals) {
    const size_t chunks = chunks_for(n_chunks, s);
    double total = 0.0;
    for (size_t ch = 0; ch < chunks; ++ch) {
        size_t b, e;
        chunk_range(s, chunks, ch, &b, &e);
        double acc = 0.0;
        for (size_t i = b; i < e; ++i) {
            const double d = sqdist(S + i * n, c, n);
            const double best = d2[i] < d ? d2[i] : d; /* std::min(d2[i], d) */
            scratch[i] = best;
            acc += best;
        }
        total += acc;
    }
    *evals += (int64_t)s;
    return total;
}

/* Source of the random draws seed_degenerate_slots consumes (seeding.hpp:72-99). */
typedef struct draw_src {
    orc_rng* rng;         /* live stream, or */
    size_t first_row;     /* pre-drawn uniform_index(s) */
    const double* units;  /* pre-drawn next_unit() values */
    size_t used;
} draw_src;

static size_t src_first(draw_src* q, size_t s) {
    return q->rng ? (size_t)orc_rng_uniform_index(q->rng, s) : q->first_row;
}
static double src_unit(draw_src* q) { return q->rng ? orc_rng_next_unit(q->rng) : q->units[q->used++]; }

/* seeding.hpp:47-105 */
static int seed_slots(const double* S, size_t s, size_t n, double* C, uint8_t* flags, size_t k, size_t candidates,
                      size_t n_chunks, draw_src* src, int64_t* evals, int64_t* filled) {
    if (s < 1) return fail(1, "seeding: empty sample");
    if (candidates < 1) return fail(1, "seeding: need at least one candidate");
    size_t* pending = malloc((k ? k : 1) * sizeof(size_t));
    size_t np = 0;
    double* d2 = malloc(s * sizeof(double));
    double* scratch = malloc(s * sizeof(double));
    double* best_scratch = malloc(s * sizeof(double));
    double* cum = malloc(s * sizeof(double));
    double* t;
    int have_center = 0;
    *filled = 0;
    for (size_t i = 0; i < s; ++i) d2[i] = INFINITY;
    for (size_t j = 0; j < k; ++j) { /* seeding.hpp:60-68: valid centres in slot order */
        if (flags[j]) {
            pending[np++] = j;
        } else {
            d2_min_update(S, s, n, C + j * n, d2, scratch, n_chunks, evals);
            t = d2, d2 = scratch, scratch = t;
            have_center = 1;
        }
    }
    size_t next = 0;
    if (np > 0 && !have_center) { /* seeding.hpp:72-79 */
        const size_t j = pending[next++];
        const size_t row = src_first(src, s);
        memcpy(C + j * n, S + row * n, n * sizeof(double));
        flags[j] = 0;
        ++*filled;
        d2_min_update(S, s, n, C + j * n, d2, scratch, n_chunks, evals);
        t = d2, d2 = scratch, scratch = t;
    }
    for (; next < np; ++next) { /* seeding.hpp:81-104 */
        double total = 0.0;
        for (size_t i = 0; i < s; ++i) {
            total += d2[i];
            cum[i] = total;
        }
        if (!(total > 0.0)) break;
        double best_cost = INFINITY;
        size_t best_row = s;
        for (size_t c = 0; c < candidates; ++c) {
            const size_t row = weighted_index_u(cum, s, src_unit(src));
            const double cost = d2_min_update(S, s, n, S + row * n, d2, scratch, n_chunks, evals);
            if (cost < best_cost) {
                best_cost = cost;
                best_row = row;
                t = best_scratch, best_scratch = scratch, scratch = t;
            }
        }
        const size_t j = pending[next];
        memcpy(C + j * n, S + best_row * n, n * sizeof(double));
        flags[j] = 0;
        ++*filled;
        t = d2, d2 = best_scratch, best_scratch = t;
    }
    free(pending);
    free(d2);
    free(scratch);
    free(best_scratch);
    free(cum);
    return 0;
}

/* seeding.hpp:125-133 */
int orc_reinit_degenerate(const double* S, size_t s, size_t n, const double* C_in, const uint8_t* flags_in,
                          size_t k, size_t candidates, size_t n_chunks, orc_rng* rng, double* C_out,
                          uint8_t* flags_out, int64_t* n_d) {
    memcpy(C_out, C_in, k * n * sizeof(double));
    memcpy(flags_out, flags_in, k);
    int64_t ev = 0, filled = 0;
    int any = 0;
    for (size_t j = 0; j < k; ++j) any |= flags_in[j] != 0;
    int rc = 0;
    if (any) {
        draw_src src = {rng, 0, NULL, 0};
        rc = seed_slots(S, s, n, C_out, flags_out, k, candidates, n_chunks, &src, &ev, &filled);
    }
    if (n_d) *n_d = ev;
    return rc;
}

int orc_seed_with_uniforms(const double* S, size_t s, size_t n, const double* C_in, const uint8_t* flags_in,
                           size_t k, size_t candidates, size_t first_row, const double* units, double* C_out,
                           uint8_t* flags_out, int64_t* n_d, int64_t* filled) {
    memcpy(C_out, C_in, k * n * sizeof(double));
    memcpy(flags_out, flags_in, k);
    int64_t ev = 0, fl = 0;
    int any = 0;
    for (size_t j = 0; j < k; ++j) any |= flags_in[j] != 0;
    int rc = 0;
    if (any) {
        draw_src src = {NULL, first_row, units, 0};
        rc = seed_slots(S, s, n, C_out, flags_out, k, candidates, 1, &src, &ev, &fl);
    }
    if (n_d) *n_d = ev;
    if (filled) *filled = fl;
    return rc;
}

/* --------------------------------------------------------------- engine.hpp */

/* engine.hpp:165-177: partial Fisher-Yates over iota(m), draw order kept */
int orc_draw_indices(size_t m, size_t s, orc_rng* rng, int64_t* idx_out) {
    if (s < 1 || s > m) return fail(1, "draw_sample: sample size must be in [1, m]");
    size_t* idx = malloc(m * sizeof(size_t));
    for (size_t i = 0; i < m; ++i) idx[i] = i;
    for (size_t i = 0; i < s; ++i) {
        const size_t j = i + (size_t)orc_rng_uniform_index(rng, m - i);
        size_t t = idx[i];
        idx[i] = idx[j];
        idx[j] = t;
        idx_out[i] = (int64_t)idx[i];
    }
    free(idx);
    return 0;
}

typedef struct worker {
    double* inc;      /* incumbent k x n */
    uint8_t* inc_deg; /* degenerate flags */
    double obj;
    double t_w;
    size_t samples;
    double* trace; /* (timestamp, objective) pairs */
    size_t trace_len, trace_cap;
} worker;

/* engine.hpp:288-296 */
static int phase_cooperative(int32_t kind, double t1, double progress) {
    if (kind == 2) return 1;
    if (kind == 3) return progress >= t1;
    return 0;
}

/* engine.hpp:239-267 (worker_step) with the lockstep clock (engine.hpp:413) */
static int worker_step(worker* w, orc_rng* rng, const double* X, size_t m, size_t n, const double* init,
                       const uint8_t* init_deg, const orc_run_cfg* c, size_t par_chunks, size_t n_threads,
                       int64_t* evals, int* accepted) {
    const size_t s = c->sample_size, k = c->k;
    int64_t* idx = malloc(s * sizeof(int64_t));
    double* S = malloc(s * n * sizeof(double));
    double* C0 = malloc(k * n * sizeof(double));
    uint8_t* f0 = malloc(k);
    double* Co = malloc(k * n * sizeof(double));
    uint8_t* fo = malloc(k);
    int rc = orc_draw_indices(m, s, rng, idx);
    if (rc) goto out;
    for (size_t i = 0; i < s; ++i) memcpy(S + i * n, X + (size_t)idx[i] * n, n * sizeof(double));
    int64_t ev = 0;
    rc = orc_reinit_degenerate(S, s, n, init, init_deg, k, c->candidates, par_chunks, rng, C0, f0, &ev);
    *evals += ev;
    if (rc) goto out;
    double obj;
    rc = orc_kmeans(S, s, n, C0, f0, k, c->max_iters, c->rel_tol, n_threads, Co, fo, NULL, NULL, &obj, NULL, NULL,
                    &ev, NULL, 0, NULL);
    if (rc) goto out;
    *evals += ev;
    w->samples += 1;
    double ts = (double)w->samples; /* sample-count clock: samples_processed + 1 */
    w->t_w = ts;
    *accepted = 0;
    if (!(obj < w->obj)) goto out;
    if (w->trace_len > 0) {
        if (!(obj < w->trace[2 * (w->trace_len - 1) + 1])) {
            rc = fail(2, "worker_step: non-decreasing incumbent accepted");
            goto out;
        }
        const double last_ts = w->trace[2 * (w->trace_len - 1)];
        if (!(ts > last_ts)) ts = nextafter(last_ts, INFINITY);
    }
    memcpy(w->inc, Co, k * n * sizeof(double));
    memcpy(w->inc_deg, fo, k);
    w->obj = obj;
    if (w->trace_len == w->trace_cap) {
        w->trace_cap = w->trace_cap ? 2 * w->trace_cap : 16;
        w->trace = realloc(w->trace, 2 * w->trace_cap * sizeof(double));
    }
    w->trace[2 * w->trace_len] = ts;
    w->trace[2 * w->trace_len + 1] = obj;
    ++w->trace_len;
    *accepted = 1;
out:
    free(idx);
    free(S);
    free(C0);
    free(f0);
    free(Co);
    free(fo);
    return rc;
}

/* engine.hpp:70-86 (validate) + engine.hpp:380-436 (run_lockstep) + engine.hpp:444-499 (run) */
int orc_run(const double* X, size_t m, size_t n, const orc_run_cfg* c_in, orc_run_out* o, double* centroids,
            uint8_t* flags, int32_t* labels, double* publications, int64_t pub_cap, double* worker_obj,
            double* traces, int64_t trace_cap, int64_t* trace_len) {
    orc_run_cfg cc = *c_in;
    const orc_run_cfg* c = &cc;
    if (cc.strategy == 0) cc.n_workers = 1; /* engine.hpp:446 */
    if (cc.k < 1) return fail(1, "EngineConfig: k must be positive");
    if (cc.sample_size < 1 || cc.sample_size > m) return fail(1, "EngineConfig: sample_size must be in [1, m]");
    if (cc.n_workers < 1) return fail(1, "EngineConfig: need at least one worker");
    if (cc.max_samples < 1) return fail(1, "EngineConfig: need a time limit or a max_samples bound");
    if (cc.strategy == 3) {
        if (!(cc.phase_t1 >= 0.0 && cc.phase_t2 >= 0.0))
            return fail(1, "EngineConfig: hybrid phase durations must be nonnegative");
        const double b = (double)cc.max_samples;
        if (!(fabs(cc.phase_t1 + cc.phase_t2 - b) <= 1e-9 * (b > 1.0 ? b : 1.0)))
            return fail(1, "EngineConfig: hybrid phases must sum to the total budget");
    }
    const size_t W = cc.n_workers, k = cc.k;
    const size_t inner_chunks = cc.n_threads ? cc.n_threads : 8;
    const size_t par_chunks = cc.strategy == 0 ? inner_chunks : 1;

    worker* ws = calloc(W, sizeof(worker));
    orc_rng* rngs = malloc(W * sizeof(orc_rng));
    for (size_t w = 0; w < W; ++w) {
        ws[w].inc = calloc(k * n, sizeof(double));
        ws[w].inc_deg = malloc(k);
        memset(ws[w].inc_deg, 1, k);
        ws[w].obj = INFINITY;
        orc_rng_derive(&rngs[w], cc.master_seed, 1, w); /* engine.hpp:457 */
    }
    /* SharedBest (engine.hpp:114-157) */
    int64_t version = 0;
    double sb_obj = INFINITY;
    double* sb_c = calloc(k * n, sizeof(double));
    uint8_t* sb_deg = malloc(k);
    memset(sb_deg, 1, k);
    int64_t npub = 0;
    double* pubs = NULL;
    size_t pubs_cap = 0;

    int* accepted = calloc(W, sizeof(int));
    int* errs = calloc(W, sizeof(int));
    char(*errmsg)[256] = calloc(W, 256);
    double* all_deg_c = calloc(k * n, sizeof(double));
    uint8_t* all_deg_f = malloc(k);
    memset(all_deg_f, 1, k);
    int64_t evals = 0;
    const int hybrid = cc.strategy == 3;
    const size_t phase1_rounds = hybrid ? (size_t)cc.phase_t1 : 0;
    int rc = 0;

    for (size_t r = 0; r < cc.max_samples; ++r) {
        for (size_t w = 0; w < W; ++w) {
            if (errs[w]) continue;
            const int coop = phase_cooperative(cc.strategy, cc.phase_t1, (double)ws[w].samples);
            const double* init = ws[w].inc;
            const uint8_t* init_deg = ws[w].inc_deg;
            if (coop) { /* engine.hpp:337-343 */
                init = version ? sb_c : all_deg_c;
                init_deg = version ? sb_deg : all_deg_f;
            }
            const size_t lloyd_chunks = cc.strategy == 0 ? inner_chunks : 1;
            int acc = 0;
            int e = worker_step(&ws[w], &rngs[w], X, m, n, init, init_deg, c, par_chunks, lloyd_chunks, &evals, &acc);
            if (e) {
                errs[w] = e;
                snprintf(errmsg[w], 256, "%s", g_err);
                acc = 0;
            }
            accepted[w] = acc;
        }
        /* on_round_end, engine.hpp:391-402 */
        const size_t round = r + 1;
        const int round_was_coop = phase_cooperative(cc.strategy, cc.phase_t1, (double)(round - 1));
        for (size_t w = 0; w < W; ++w) {
            const int carry = hybrid && round == phase1_rounds && isfinite(ws[w].obj);
            if ((accepted[w] && round_was_coop) || carry) {
                if (ws[w].obj < sb_obj) { /* try_publish: strict < (engine.hpp:131) */
                    ++version;
                    sb_obj = ws[w].obj;
                    memcpy(sb_c, ws[w].inc, k * n * sizeof(double));
                    memcpy(sb_deg, ws[w].inc_deg, k);
                    if ((size_t)npub == pubs_cap) {
                        pubs_cap = pubs_cap ? 2 * pubs_cap : 16;
                        pubs = realloc(pubs, 4 * pubs_cap * sizeof(double));
                    }
                    pubs[4 * npub + 0] = (double)version;
                    pubs[4 * npub + 1] = (double)w;
                    pubs[4 * npub + 2] = ws[w].obj;
                    pubs[4 * npub + 3] = (double)round;
                    ++npub;
                }
            }
            accepted[w] = 0;
        }
    }
    for (size_t w = 0; w < W; ++w)
        if (errs[w]) {
            snprintf(g_err, sizeof g_err, "%s", errmsg[w]);
            rc = errs[w];
            goto out;
        }
    /* select_best, engine.hpp:180-194 */
    int best = -1;
    double best_f = INFINITY;
    for (size_t w = 0; w < W; ++w)
        if (ws[w].obj < best_f) {
            best_f = ws[w].obj;
            best = (int)w;
        }
    if (best < 0) {
        rc = fail(3, "no solution produced: every worker incumbent is infinite");
        goto out;
    }
    memset(o, 0, sizeof *o);
    o->best_worker = best;
    o->best_sample_objective = ws[best].obj;
    double min_last = INFINITY; /* engine.hpp:472-475 */
    for (size_t w = 0; w < W; ++w)
        if (ws[w].trace_len) {
            const double t = ws[w].trace[2 * (ws[w].trace_len - 1)];
            if (t < min_last) min_last = t;
        }
    o->clustering_time = min_last;
    size_t ff = 0; /* engine.hpp:477-481 */
    for (size_t w = 0; w < W; ++w)
        if (ws[w].t_w < ws[ff].t_w) ff = w;
    o->clustering_time_first_finisher = ws[ff].trace_len ? ws[ff].trace[2 * (ws[ff].trace_len - 1)] : 0.0;
    if (centroids) memcpy(centroids, ws[best].inc, k * n * sizeof(double));
    if (flags) memcpy(flags, ws[best].inc_deg, k);
    if (cc.compute_full_objective || cc.compute_assignment) { /* engine.hpp:483-491 */
        int64_t ev = 0;
        double f;
        int32_t* lab = malloc(m * sizeof(int32_t));
        rc = orc_assign(X, m, n, ws[best].inc, ws[best].inc_deg, k, par_chunks, lab, NULL, &f, &ev);
        if (rc) {
            free(lab);
            goto out;
        }
        evals += ev;
        o->has_full_objective = 1;
        o->full_objective = f;
        if (labels && cc.compute_assignment) memcpy(labels, lab, m * sizeof(int32_t));
        free(lab);
    }
    for (size_t w = 0; w < W; ++w) o->total_samples += ws[w].samples;
    o->distance_evals = evals;
    o->n_publications = npub;
    if (publications)
        for (int64_t i = 0; i < npub && i < pub_cap; ++i) memcpy(publications + 4 * i, pubs + 4 * i, 4 * sizeof(double));
    for (size_t w = 0; w < W; ++w) {
        if (worker_obj) worker_obj[w] = ws[w].obj;
        if (trace_len) trace_len[w] = (int64_t)ws[w].trace_len;
        if (traces)
            for (size_t t = 0; t < ws[w].trace_len && (int64_t)t < trace_cap; ++t) {
                traces[(w * trace_cap + t) * 2 + 0] = ws[w].trace[2 * t];
                traces[(w * trace_cap + t) * 2 + 1] = ws[w].trace[2 * t + 1];
            }
    }
out:
    for (size_t w = 0; w < W; ++w) {
        free(ws[w].inc);
        free(ws[w].inc_deg);
        free(ws[w].trace);
    }
    free(ws);
    free(rngs);
    free(sb_c);
    free(sb_deg);
    free(pubs);
    free(accepted);
    free(errs);
    free(errmsg);
    free(all_deg_c);
    free(all_deg_f);
    return rc;
}
