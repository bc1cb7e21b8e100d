"""GPU parity: the sm_100a kernels (through libhpcg.so's C-ABI) against the CPU oracle
(oracle/hpclust_oracle.c) and, where present, the reference itself (oracle/_ref).

Bars (BASELINE.json north_star): labels and counts bit-exact; centroids and objectives within
1e-12 relative in fp64 mode (fp32 data is compared against the oracle run on the same values
widened to fp64; the Lloyd / K-means++ path keeps fp64 accumulation, so 1e-12 there too);
iterations and stop reason equal. The full-data f(C, X) over fp32 data runs in the north star's
fp32 mode by default (fp32 row cost, fp64 accumulation: FP32_RTOL = 1e-5) and in the exact fp64
row-cost mode on request (hpcg_ctx_set_fp32_cost; 1e-12, test_objective_fp32_exact_mode).
"""
import numpy as np
import pytest

import paper_2311_04517_b200 as hp
from oracle_py import orc, ref

pytestmark = pytest.mark.gpu

RTOL = 1e-12
FP32_RTOL = 1e-5  # f(C, X) over fp32 data in fp32 mode (north star)


def obj_rtol(X):
    """f(C, X) tolerance: fp32 mode for fp32 data, fp64 mode otherwise."""
    return FP32_RTOL if np.asarray(X).dtype == np.float32 else RTOL


def mixture(m, n, comps, seed, dtype=np.float64, spread=10.0, sigma=1.0):
    rs = np.random.default_rng(seed)
    means = rs.uniform(-spread, spread, (comps, n))
    lab = rs.integers(0, comps, m)
    X = means[lab] + sigma * rs.standard_normal((m, n))
    return X.astype(dtype)


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    scale = np.maximum(np.abs(b), 1e-300)
    return float(np.max(np.abs(a - b) / scale)) if a.size else 0.0


def centroid_close(a, b, rtol=RTOL):
    # norm-wise per centroid (coordinates near zero are judged against the centroid's norm)
    a, b = np.asarray(a), np.asarray(b)
    num = np.linalg.norm(a - b, axis=-1)
    den = np.maximum(np.linalg.norm(b, axis=-1), 1e-300)
    return float(np.max(num / den)) <= rtol


def test_spec_kmeans_example():
    # {0,1,2,10,11,12}, C_init {0,10} -> {1,11}, objective 4, fixed_point
    S = np.array([[0.0], [1], [2], [10], [11], [12]])
    out = hp.kmeans(S, np.array([[0.0], [10.0]]))
    assert out.centroids.ravel().tolist() == [1.0, 11.0]
    assert out.objective == 4.0
    assert out.converged_by == "fixed_point"
    assert out.labels.tolist() == [0, 0, 0, 1, 1, 1]


@pytest.mark.parametrize("dtype,n,k,s,W", [
    (np.float64, 2, 5, 5000, 4),    # config 1 shape
    (np.float32, 16, 10, 20000, 8),  # config 2 shape
    (np.float64, 3, 25, 50000, 2),   # config 3 shape
    (np.float32, 8, 15, 6000, 3),
    (np.float64, 7, 9, 1234, 3),     # odd widths / ragged chunks
    (np.float32, 5, 1, 777, 2),      # k = 1
])
def test_kmeans_batched_vs_oracle(dtype, n, k, s, W):
    m = max(4 * s, 20000)
    X = mixture(m, n, k + 2, seed=n * 100 + k, dtype=dtype)
    rs = np.random.default_rng(7)
    idx = np.stack([rs.choice(m, s, replace=False) for _ in range(W)])
    inits = np.stack([X[rs.choice(m, k, replace=False)].astype(np.float64) for _ in range(W)])
    r = hp.worker_step_batched(X, idx, inits, None, want_labels=True, want_counts=True, hist_cap=302)
    o = orc()
    Xw = X.astype(np.float64)
    for w in range(W):
        e = o.kmeans(Xw[idx[w]], inits[w])
        assert r["iterations"][w] == e["iterations"], w
        assert r["stop"][w] == e["stop"], w
        assert np.array_equal(r["labels"][w], e["labels"]), w
        assert np.array_equal(r["counts"][w], e["counts"]), w
        assert np.array_equal(r["degenerate"][w], e["degenerate"]), w
        assert centroid_close(r["centroids"][w], e["centroids"]), w
        assert rel(r["objective"][w], e["objective"]) <= RTOL, w
        assert r["n_d"][w] == e["n_d"], w
        hl = r["hist_len"][w]
        assert hl == len(e["history"])
        assert rel(r["history"][w, :hl], e["history"]) <= RTOL


def test_kmeans_max_iters_and_tolerance():
    X = mixture(30000, 4, 6, seed=3)
    rs = np.random.default_rng(1)
    idx = rs.choice(len(X), 3000, replace=False)[None]
    init = X[rs.choice(len(X), 6, replace=False)][None]
    for max_iters, tol in [(1, 1e-4), (2, 1e-4), (5, 0.5), (300, 1e-9)]:
        r = hp.worker_step_batched(X, idx, init, None, lloyd=hp.LloydConfig(max_iters, tol), want_labels=True)
        e = orc().kmeans(X[idx[0]], init[0], max_iters=max_iters, rel_tol=tol)
        assert r["stop"][0] == e["stop"] and r["iterations"][0] == e["iterations"]
        assert np.array_equal(r["labels"][0], e["labels"])
        assert rel(r["objective"][0], e["objective"]) <= RTOL


def test_empty_cluster_and_duplicates():
    # an init centre far away empties its cluster (kept during the run, flagged at the end)
    X = mixture(5000, 2, 3, seed=5)
    init = np.vstack([X[:3], [[1e6, 1e6]]])
    r = hp.worker_step_batched(X, np.arange(5000)[None], init[None], None, want_labels=True, want_counts=True)
    e = orc().kmeans(X, init)
    assert np.array_equal(r["degenerate"][0], e["degenerate"]) and e["degenerate"][3] == 1
    assert np.array_equal(r["labels"][0], e["labels"])
    assert centroid_close(r["centroids"][0], e["centroids"])


@pytest.mark.parametrize("n", [16, 128])
def test_exact_ties_fp32_rows_pair_kernel(n):
    # fp32 16-wide rows on an integer lattice, centres placed so many rows are exactly
    # equidistant from two or more centres (ties resolved to the lowest index, core.hpp:146-157)
    rs = np.random.default_rng(3)
    X = rs.integers(-4, 5, (100003, n)).astype(np.float32)
    C_ = np.zeros((9, n))
    for j in range(1, 9):
        C_[j, (j - 1) % n] = 2.0 if j % 2 else -2.0
    C_[5] = C_[1]  # duplicate centre: never chosen over slot 1
    lab, cnt, cost, _ = orc().assign(X.astype(np.float64), C_)
    a, f = hp.final_assignment(X, C_)
    assert np.array_equal(a.labels, lab) and np.array_equal(a.counts, cnt)
    assert f == cost  # small integers: exact


def test_exact_ties_go_to_lowest_index():
    # X={(5)}, C={(4),(6)} -> label 0; plus many exact ties on a lattice
    a = hp.assign_nearest(np.array([[5.0]]), np.array([[4.0], [6.0]]))
    assert a.labels.tolist() == [0]
    g = np.arange(-8, 9, dtype=np.float64)
    X = np.array([[x, y] for x in g for y in g])
    C_ = np.array([[-2.0, 0.0], [2.0, 0.0], [0.0, 2.0], [0.0, -2.0]])
    lab, cnt, cost, _ = orc().assign(X, C_)
    a = hp.assign_nearest(X, C_)
    assert np.array_equal(a.labels, lab) and np.array_equal(a.counts, cnt)
    assert hp.mssc_objective(C_, X) == cost  # small integers: exact


@pytest.mark.parametrize("dtype,n,k", [(np.float64, 2, 5), (np.float32, 16, 10), (np.float64, 3, 25),
                                       (np.float32, 8, 15), (np.float32, 1, 3),
                                       # centre-pair kernel widths (16/32/48/128-B rows), odd and
                                       # large centre counts
                                       (np.float32, 4, 7), (np.float32, 12, 33), (np.float32, 32, 64),
                                       (np.float32, 16, 1), (np.float32, 16, 255),
                                       # tensor-core screen kernel: N = 16 / 32 centre columns
                                       (np.float32, 32, 20), (np.float32, 16, 17), (np.float32, 8, 32),
                                       (np.float32, 32, 2),
                                       # narrow-row kernel (bulk-copy ring): fp64 n = 1..3, fp32 n = 2
                                       (np.float64, 1, 4), (np.float64, 2, 31), (np.float32, 2, 6),
                                       # wide rows on the tensor cores (K-atom tiles): config-4 shape
                                       (np.float32, 128, 25), (np.float32, 64, 10), (np.float32, 128, 32)])
def test_objective_vs_oracle(dtype, n, k):
    X = mixture(200003, n, k, seed=11 + n, dtype=dtype)
    C_ = mixture(k, n, k, seed=99, dtype=np.float64)
    lab, cnt, cost, nd = orc().assign(X.astype(np.float64), C_)
    a, f = hp.final_assignment(X, C_)
    assert np.array_equal(a.labels, lab)
    assert np.array_equal(a.counts, cnt)
    assert rel(f, cost) <= obj_rtol(X)
    if k == 1:
        return  # no valid subset left to test
    # valid-subset (engine.hpp:211-229)
    deg = np.zeros(k, np.uint8)
    deg[0] = 1
    lab2, cnt2, cost2, _ = orc().assign(X.astype(np.float64), C_, deg)
    a2, f2 = hp.assign_valid_subset(X, C_, deg)
    assert np.array_equal(a2.labels, lab2) and np.array_equal(a2.counts, cnt2)
    assert rel(f2, cost2) <= obj_rtol(X)


@pytest.mark.parametrize("m", [1, 100, 128, 640, 1000])
@pytest.mark.parametrize("dtype,n", [(np.float64, 3), (np.float64, 2), (np.float32, 16), (np.float32, 8),
                                     (np.float32, 128)])
def test_objective_small_m(m, dtype, n):
    # partial / single tail groups of the streaming kernels (rows read from global memory directly,
    # TMA boxes clipped at m)
    X = mixture(m, n, 4, seed=m + n, dtype=dtype)
    C_ = mixture(7, n, 4, seed=5)
    lab, cnt, cost, _ = orc().assign(X.astype(np.float64), C_)
    a, f = hp.final_assignment(X, C_)
    assert np.array_equal(a.labels, lab) and np.array_equal(a.counts, cnt)
    assert rel(f, cost) <= obj_rtol(X)


@pytest.mark.parametrize("n,k", [(16, 10), (8, 15), (32, 32), (128, 25), (64, 7)])
def test_objective_far_offset_near_ties(n, k):
    # rows far from the origin (|x| ~ 1e3) around centres 0.05 apart: the tensor-core screen's
    # error bound (kappa (|x| + cmax)^2) flags most rows, which then take the exact fp64 argmin
    rs = np.random.default_rng(n + k)
    base = 1000.0 + rs.standard_normal(n)
    C_ = base + 0.05 * rs.standard_normal((k, n))
    X = (C_[rs.integers(0, k, 50001)] + 0.05 * rs.standard_normal((50001, n))).astype(np.float32)
    lab, cnt, cost, _ = orc().assign(X.astype(np.float64), C_)
    a, f = hp.final_assignment(X, C_)
    assert np.array_equal(a.labels, lab) and np.array_equal(a.counts, cnt)
    # fp32 mode with |x - c| ~ 5e-5 |c|: the centre's low part keeps the row difference accurate
    assert rel(f, cost) <= FP32_RTOL


@pytest.mark.parametrize("n,k", [(16, 10), (8, 15), (32, 20), (128, 25), (64, 7)])
def test_objective_fp32_exact_mode(n, k):
    """hpcg_ctx_set_fp32_cost(exact): the fp64 row cost over fp32 data -- 1e-12 of the oracle; and the
    fp32 mode within its gate of the same value (labels identical in both)."""
    X = mixture(200003, n, k, seed=31 + n, dtype=np.float32)
    C_ = mixture(k, n, k, seed=7, dtype=np.float64)
    lab, cnt, cost, _ = orc().assign(X.astype(np.float64), C_)
    ctx = hp.default_context()
    try:
        ctx.set_fp32_cost(True)
        a, f = hp.final_assignment(X, C_)
    finally:
        ctx.set_fp32_cost(False)
    b, g = hp.final_assignment(X, C_)
    assert np.array_equal(a.labels, lab) and np.array_equal(b.labels, lab)
    assert rel(f, cost) <= RTOL
    assert rel(g, cost) <= FP32_RTOL


@pytest.mark.parametrize("dtype,n,k,s,npend", [(np.float64, 2, 5, 5000, 5), (np.float32, 16, 10, 20000, 10),
                                               (np.float64, 3, 25, 8000, 4), (np.float32, 8, 15, 3000, 15)])
def test_seeding_with_reference_draws(dtype, n, k, s, npend):
    X = mixture(s, n, k, seed=21 + k, dtype=dtype)
    rs = np.random.default_rng(5)
    init = X[rs.choice(s, k, replace=False)].astype(np.float64)
    deg = np.zeros(k, np.uint8)
    deg[rs.choice(k, npend, replace=False)] = 1
    init[deg == 1] = 0.0
    rng = hp.RngStream(1234 + k)
    twin = rng.copy()
    Cg, fg = hp.reinit_degenerate(init, deg, X, hp.SeedConfig(), rng)
    # oracle with the same stream (its own mt19937_64 restatement)
    o = orc()
    r2 = o.rng(seed=1234 + k)
    Co, fo, nd = o.reinit(X.astype(np.float64), init, deg, r2)
    assert np.array_equal(fg, fo)
    assert np.array_equal(Cg, Co)  # seeded centres are rows of S: bitwise
    # streams advanced identically
    assert rng.next_u64() == o.next_u64(r2)
    del twin


def test_seeding_exhausts_distinct_rows():
    # 4 rows, 2 distinct, k=3 -> one slot stays degenerate, kmeans throws
    S = np.array([[1.0, 1.0], [1.0, 1.0], [5.0, 5.0], [5.0, 5.0]])
    C_, f = hp.kmeanspp_seed(S, 3, hp.SeedConfig(), hp.RngStream(3))
    Co, fo, _ = orc().reinit(S, np.zeros((3, 2)), np.ones(3, np.uint8), orc().rng(seed=3))
    assert np.array_equal(f, fo) and f.sum() == 1
    assert np.array_equal(C_, Co)
    with pytest.raises(hp.InvalidArgument, match="kmeans: degenerate centroid in init"):
        hp.worker_step_batched(S, None, np.zeros((1, 3, 2)), np.ones((1, 3), np.uint8), rngs=[hp.RngStream(3)])


def test_draw_sample_matches_reference_stream():
    X = mixture(10000, 3, 4, seed=2)
    rng = hp.RngStream.derive(0, 1, 0)
    S = hp.draw_sample(X, 500, rng)
    o = orc()
    r2 = o.rng(derive=(0, 1, 0))
    idx = o.draw_indices(10000, 500, r2)
    assert np.array_equal(S, X[idx])
    assert rng.next_u64() == o.next_u64(r2)


@pytest.mark.parametrize("strategy,t1,t2", [("competitive", 0, 0), ("cooperative", 0, 0), ("hybrid", 2.5, 2.5),
                                            ("inner", 0, 0)])
def test_run_reference_rng_vs_oracle(strategy, t1, t2):
    X = mixture(6000, 2, 5, seed=17)
    kw = dict(k=5, sample_size=800, n_workers=3, max_samples=5, strategy=strategy, t1=t1, t2=t2, seed=42)
    e = orc().run(X, **kw)
    cfg = hp.EngineConfig(k=5, sample_size=800, n_workers=3, max_samples=5, strategy=strategy, phase_t1=t1,
                          phase_t2=t2, master_seed=42, rng="reference")
    g = hp.run(X, cfg)
    assert g.best_worker == e["best_worker"]
    assert g.distance_evals == e["distance_evals"]
    assert g.total_samples == e["total_samples"]
    assert centroid_close(g.centroids, e["centroids"])
    assert rel(g.full_objective, e["full_objective"]) <= RTOL
    assert rel(g.best_sample_objective, e["best_sample_objective"]) <= RTOL
    assert g.clustering_time == e["clustering_time"]
    assert g.publications.shape == e["publications"].shape
    if len(e["publications"]):
        assert np.array_equal(g.publications[:, [0, 1, 3]], e["publications"][:, [0, 1, 3]])
        assert rel(g.publications[:, 2], e["publications"][:, 2]) <= RTOL
    for w in range(len(e["traces"])):
        assert np.array_equal(g.traces[w][:, 0], e["traces"][w][:, 0])
        assert rel(g.traces[w][:, 1], e["traces"][w][:, 1]) <= RTOL


def test_run_matches_reference_itself_cfg1():
    R = ref()
    if R is None:
        pytest.skip("oracle/_ref not built")
    # BASELINE.json config 1 (reference gen_blobs, seed 0), shortened to 10 samples per worker
    X = R.gen_blobs(100000, 2, 5, center=(-10.0, 10.0), std=(1.0, 1.0), noise_points=0, seed=0)
    kw = dict(k=5, sample_size=5000, n_workers=4, max_samples=10, strategy="competitive", seed=0)
    e = R.run(X, **kw)
    g = hp.run(X, hp.EngineConfig(k=5, sample_size=5000, n_workers=4, max_samples=10, master_seed=0))
    assert g.best_worker == e["best_worker"]
    assert g.distance_evals == e["distance_evals"]
    assert centroid_close(g.centroids, e["centroids"])
    assert rel(g.full_objective, e["full_objective"]) <= RTOL


def test_philox_engine_runs_and_is_deterministic():
    X = mixture(200000, 16, 10, seed=8, dtype=np.float32)
    cfg = hp.EngineConfig(k=10, sample_size=20000, n_workers=16, max_samples=3, strategy="cooperative",
                          master_seed=5, rng="philox")
    a = hp.run(X, cfg)
    b = hp.run(X, cfg)
    assert np.array_equal(a.centroids, b.centroids)
    assert a.full_objective == b.full_objective and a.distance_evals == b.distance_evals
    # the reported full objective is f(C, X) of the returned centroids
    _, cost, _, _ = None, None, None, None
    lab, cnt, cost, nd = orc().assign(X.astype(np.float64), a.centroids, a.degenerate)
    assert rel(a.full_objective, cost) <= obj_rtol(X)


@pytest.mark.parametrize("m", [1, 2, 3, 5, 97, 1000, 4096, 65537, 100003])
def test_philox_sample_is_a_permutation(m):
    # s = m: the device sample of a philox round is a permutation of [0, m) (distinct by
    # construction: keyed Feistel bijection over Z_a x Z_b plus cycle walking)
    for worker in (0, 7):
        idx = hp.philox_sample_indices(m, m, key=0x1234567890ABCDEF, round_=3, worker=worker)
        assert np.array_equal(np.sort(idx), np.arange(m))


def test_philox_sample_distinct_in_range_and_keyed():
    m, s = 10_000_000, 20000
    a = hp.philox_sample_indices(m, s, key=5, round_=0, worker=0)
    assert a.min() >= 0 and a.max() < m and len(np.unique(a)) == s
    assert np.array_equal(a, hp.philox_sample_indices(m, s, key=5, round_=0, worker=0))
    b = hp.philox_sample_indices(m, s, key=5, round_=0, worker=1)
    c = hp.philox_sample_indices(m, s, key=5, round_=1, worker=0)
    assert len(np.intersect1d(a, b)) < 200 and len(np.intersect1d(a, c)) < 200  # ~ s^2/m = 40 expected
    # roughly uniform over [0, m): each decile holds ~s/10 rows
    h = np.bincount(a * 10 // m, minlength=10)
    assert h.min() > 0.8 * s / 10 and h.max() < 1.2 * s / 10


@pytest.mark.parametrize("strategy,dtype,n", [("competitive", np.float64, 3), ("cooperative", np.float64, 3),
                                              # the tensor-core f(C,X) kernels in the engine's finish:
                                              # device-side valid count (n = 16), host-side (n = 128)
                                              ("cooperative", np.float32, 16), ("competitive", np.float32, 128)])
def test_run_compute_assignment_vs_oracle(strategy, dtype, n):
    # the full assignment of a run (engine.hpp:60, 211-229, 490): labels of
    # the valid subset remapped to the original slots, from the device f(C, X) pass
    X = mixture(30000, n, 6, seed=23, dtype=dtype)
    e = orc().run(X.astype(np.float64), k=6, sample_size=1500, n_workers=4, max_samples=3, strategy=strategy, seed=9,
                  assignment=True)
    cfg = hp.EngineConfig(k=6, sample_size=1500, n_workers=4, max_samples=3, strategy=strategy, master_seed=9,
                          rng="reference", compute_assignment=True)
    g = hp.run(X, cfg)
    assert np.array_equal(g.assignment, e["labels"])
    assert rel(g.full_objective, e["full_objective"]) <= obj_rtol(X)
