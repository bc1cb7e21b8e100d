"""CPU: pin the C restatement oracle (oracle/hpclust_oracle.c) -- the checker every GPU parity
test relies on -- against (a) the SPEC.md known answers, (b) golden fixtures generated from the
reference itself (tests/golden/ref_cases.npz, tests/golden/make_golden.py), and (c) the live
reference build oracle/_ref when present. Bit-exact wherever the reference is deterministic.
"""
from pathlib import Path

import numpy as np
import pytest

from oracle_py import CheckerError, orc, ref

G = np.load(Path(__file__).resolve().parent / "golden" / "ref_cases.npz")


# ----------------------------------------------------------- SPEC.md known answers
def test_spec_squared_distance_and_assign():
    o = orc()
    # SPEC.md:50-53 (via the assignment kernel's per-row cost)
    _, _, c, _ = o.assign(np.array([[0.0, 0.0]]), np.array([[3.0, 4.0]]))
    assert c == 25.0
    _, _, c, _ = o.assign(np.array([[1.0, 2.0]]), np.array([[4.0, 6.0]]))
    assert c == 25.0
    # SPEC.md:59-62
    lab, cnt, _, _ = o.assign(np.array([[0.0], [10.0]]), np.array([[1.0], [9.0]]))
    assert lab.tolist() == [0, 1]
    lab, cnt, _, _ = o.assign(np.array([[5.0]]), np.array([[4.0], [6.0]]))
    assert lab.tolist() == [0]  # tie -> lowest index
    lab, cnt, _, _ = o.assign(np.array([[1.0], [2.0], [3.0]]), np.array([[0.0]]))
    assert cnt.tolist() == [3]


def test_spec_objective():
    o = orc()
    # SPEC.md:68-71
    assert o.assign(np.array([[0.0, 0.0], [2.0, 0.0]]), np.array([[1.0, 0.0]]))[2] == 2.0
    X = np.array([[0.0], [1], [2], [10], [11], [12]])
    assert o.assign(X, X)[2] == 0.0
    assert o.assign(X, np.array([[1.0], [11.0]]))[2] == 4.0


def test_spec_kmeans():
    o = orc()
    X = np.array([[0.0], [1], [2], [10], [11], [12]])
    e = o.kmeans(X, np.array([[0.0], [10.0]]))
    assert e["centroids"].ravel().tolist() == [1.0, 11.0] and e["objective"] == 4.0 and e["stop"] == 2
    e = o.kmeans(X, np.array([[1.0], [11.0]]))  # fixed point in one iteration
    assert e["iterations"] == 1 and e["stop"] == 2
    e = o.kmeans(np.ones((5, 2)), np.array([[1.0, 1.0], [7.0, 7.0]]))
    assert e["degenerate"].tolist() == [0, 1] and e["objective"] == 0.0


def test_spec_seeding():
    o = orc()
    # single row -> centre = row; all-identical -> one degenerate
    C, f, _ = o.reinit(np.array([[3.0, 4.0]]), np.zeros((1, 2)), np.ones(1, np.uint8), o.rng(seed=1))
    assert C.tolist() == [[3.0, 4.0]] and f.tolist() == [0]
    C, f, _ = o.reinit(np.full((4, 2), 2.0), np.zeros((2, 2)), np.ones(2, np.uint8), o.rng(seed=2))
    assert f.sum() == 1
    # SPEC.md:119 / 128: S={0,0,10}, first seed 0 -> second centre 10 with probability 1
    S = np.array([[0.0], [0.0], [10.0]])
    for seed in range(20):
        C, f, _ = o.reinit(S, np.array([[0.0], [0.0]]), np.array([0, 1], np.uint8), o.rng(seed=seed))
        assert C[1, 0] == 10.0


def test_spec_seeding_statistical():
    # S={0,1,100}, k=2, first seed at 0 -> second centre 100 in >= 97% of trials
    o = orc()
    S = np.array([[0.0], [1.0], [100.0]])
    hits = 0
    for seed in range(2000):
        C, _, _ = o.reinit(S, np.array([[0.0], [0.0]]), np.array([0, 1], np.uint8), o.rng(seed=seed))
        hits += C[1, 0] == 100.0
    assert hits / 2000 >= 0.97


def test_brute_force_lower_bound_ac1():
    # ACCEPTANCE 1 in miniature: brute force lower-bounds the engine; the engine
    # reaches it on easy instances.
    o = orc()
    rs = np.random.default_rng(1)
    reached = 0
    for t in range(20):
        X = rs.uniform(-5, 5, (int(rs.integers(6, 11)), 2))
        R = ref()
        if R is None:
            pytest.skip("oracle/_ref not built")
        _, _, fstar = R.brute_force(X, 2)
        e = o.run(X, k=2, sample_size=len(X), n_workers=4, max_samples=50, seed=t)
        assert e["full_objective"] >= fstar * (1 - 1e-12)
        # the oracle reproduces the reference run exactly (same local optima included)
        assert e["full_objective"] == R.run(X, k=2, sample_size=len(X), n_workers=4, max_samples=50,
                                            seed=t)["full_objective"]
        reached += abs(e["full_objective"] - fstar) <= 1e-9 * max(fstar, 1e-300)
    assert reached >= 15  # the reference itself reaches 16/20 on these uniform instances


# ---------------------------------------------------- golden fixtures from the reference
@pytest.mark.parametrize("t", range(6))
def test_golden_kmeans(t):
    mi, tol = G[f"km{t}_cfg"]
    e = orc().kmeans(G[f"km{t}_S"], G[f"km{t}_C0"], max_iters=int(mi), rel_tol=float(tol))
    for key in ("centroids", "degenerate", "labels", "counts", "history"):
        assert np.array_equal(e[key], G[f"km{t}_{key}"]), key
    obj, iters, stop, nd = G[f"km{t}_scalars"]
    assert e["objective"] == obj and e["iterations"] == iters and e["stop"] == stop and e["n_d"] == nd


@pytest.mark.parametrize("t", range(3))
def test_golden_seeding(t):
    o = orc()
    r = o.rng(seed=int(G[f"sd{t}_seed"][0]))
    C, f, nd = o.reinit(G[f"sd{t}_S"], G[f"sd{t}_C0"], G[f"sd{t}_f0"], r)
    assert np.array_equal(C, G[f"sd{t}_C"]) and np.array_equal(f, G[f"sd{t}_f"])
    assert nd == int(G[f"sd{t}_nd_next"][0])
    assert o.next_u64(r) == int(G[f"sd{t}_nd_next"][1])  # stream left exactly where the reference leaves it


@pytest.mark.parametrize("t", range(3))
def test_golden_draw_sample(t):
    o = orc()
    m, s, master, wi = (int(v) for v in G[f"dr{t}_cfg"])
    r = o.rng(derive=(master, 1, wi))
    assert np.array_equal(o.draw_indices(m, s, r), G[f"dr{t}_idx"])
    assert o.next_u64(r) == int(G[f"dr{t}_next"][0])


@pytest.mark.parametrize("t", range(5))
def test_golden_engine_run(t):
    strat_i, t1, t2, W = G[f"run{t}_cfg"]
    strat = ["competitive", "cooperative", "hybrid", "inner"][int(strat_i)]
    e = orc().run(G["run_X"], k=5, sample_size=500, n_workers=int(W), max_samples=5, strategy=strat, t1=float(t1),
                  t2=float(t2), seed=99, n_threads=4)
    assert np.array_equal(e["centroids"], G[f"run{t}_centroids"])
    sc = G[f"run{t}_scalars"]
    got = [e["full_objective"], e["best_worker"], e["best_sample_objective"], e["clustering_time"],
           e["clustering_time_first_finisher"], e["total_samples"], e["distance_evals"]]
    assert np.array_equal(np.array(got, dtype=np.float64), sc)
    assert np.array_equal(e["publications"], G[f"run{t}_pubs"])
    assert np.array_equal(e["worker_obj"], G[f"run{t}_wobj"])


def test_golden_strategy_degeneration_ac4():
    # hybrid(T1=budget, T2=0) == competitive (byte-identical centroids)
    assert np.array_equal(G["run3_centroids"], orc().run(G["run_X"], k=5, sample_size=500, n_workers=2,
                                                         max_samples=5, strategy="competitive", seed=99)["centroids"])
    X = G["run_X"]
    a = orc().run(X, k=5, sample_size=500, n_workers=1, max_samples=4, strategy="competitive", seed=5)
    b = orc().run(X, k=5, sample_size=500, n_workers=1, max_samples=4, strategy="cooperative", seed=5)
    c = orc().run(X, k=5, sample_size=500, n_workers=1, max_samples=4, strategy="hybrid", t1=2, t2=2, seed=5)
    assert np.array_equal(a["centroids"], b["centroids"]) and np.array_equal(a["centroids"], c["centroids"])


def test_lloyd_monotone_ac2():
    # ACCEPTANCE 2: objective history never increases (the oracle raises logic_error otherwise)
    o = orc()
    rs = np.random.default_rng(3)
    for _ in range(200):
        s, n, k = int(rs.integers(5, 60)), int(rs.integers(1, 4)), int(rs.integers(1, 5))
        S = rs.standard_normal((s, n))
        e = o.kmeans(S, S[rs.choice(s, min(k, s), replace=False)])
        assert np.all(np.diff(e["history"]) <= 1e-12 * np.abs(e["history"][:-1]))


def test_oracle_errors_match_reference_text():
    o = orc()
    with pytest.raises(CheckerError, match="kmeans: degenerate centroid in init"):
        o.kmeans(np.ones((3, 1)), np.zeros((2, 1)), flags=np.array([0, 1], np.uint8))
    with pytest.raises(CheckerError, match="kmeans: max_iters must be positive"):
        o.kmeans(np.ones((3, 1)), np.zeros((1, 1)), max_iters=0)
    with pytest.raises(CheckerError, match="EngineConfig: sample_size must be in"):
        o.run(np.ones((5, 1)), k=1, sample_size=9, n_workers=1, max_samples=1)
    with pytest.raises(CheckerError, match="EngineConfig: hybrid phases must sum to the total budget"):
        o.run(np.ones((5, 1)), k=1, sample_size=2, n_workers=1, max_samples=4, strategy="hybrid", t1=1, t2=1)


def test_golden_cfg1_generator_and_assign():
    R = ref()
    if R is None:
        pytest.skip("oracle/_ref not built")
    Xb = R.gen_blobs(100000, 2, 5, center=(-10.0, 10.0), std=(1.0, 1.0), noise_points=0, seed=0)
    assert np.array_equal(Xb[:16], G["cfg1_head"])
    lab, cnt, cost, nd = orc().assign(Xb, Xb[[0, 20000, 40000, 60000, 80000]])
    assert cost == G["cfg1_assign"][0] and nd == G["cfg1_assign"][1] and np.array_equal(cnt, G["cfg1_counts"])


# --------------------------------------------------- live reference (random cases)
def test_oracle_vs_live_reference_random():
    R = ref()
    if R is None:
        pytest.skip("oracle/_ref not built")
    o = orc()
    rs = np.random.default_rng(7)
    for _ in range(30):
        s, n, k = int(rs.integers(20, 300)), int(rs.integers(1, 6)), int(rs.integers(1, 7))
        S = rs.standard_normal((s, n)) * rs.uniform(0.1, 10)
        C0 = S[rs.choice(s, min(k, s), replace=False)]
        a, b = o.kmeans(S, C0), R.kmeans(S, C0)
        for key in ("centroids", "labels", "counts", "history"):
            assert np.array_equal(a[key], b[key]), key
        seed = int(rs.integers(1 << 30))
        fl = (rs.random(len(C0)) < 0.5).astype(np.uint8)
        ra, rb = o.rng(seed=seed), R.rng(seed=seed)
        Ca, fa, na = o.reinit(S, C0 * (1 - fl[:, None]), fl, ra)
        Cb, fb, nb = R.reinit(S, C0 * (1 - fl[:, None]), fl, rb)
        assert np.array_equal(Ca, Cb) and np.array_equal(fa, fb) and na == nb
        assert o.next_u64(ra) == rb.next_u64()


# ----------------------------------------- injected draws (PHILOX-round replay harness)
def test_injected_draws_replay_the_stock_reference():
    """oracle/ref_inject.cpp feeds queued 64-bit values to the reference's unmodified RngStream. Fed
    the very values a stock stream would produce, the reference's worker step (reinit_degenerate +
    kmeans) must come out bit-identical to the stock build's, consuming exactly the same count."""
    from oracle_py import ref_inject
    R, J = ref(), ref_inject()
    if R is None or J is None:
        pytest.skip("oracle/_ref not built")
    rs = np.random.default_rng(11)
    for case in range(12):
        s, n, k = int(rs.integers(50, 400)), int(rs.integers(1, 6)), int(rs.integers(2, 8))
        S = rs.standard_normal((s, n)) * 3 + rs.integers(0, 3, (s, 1))
        C0 = S[rs.choice(s, k, replace=False)]
        fl = np.ones(k, np.uint8) if case % 3 == 0 else (rs.random(k) < 0.5).astype(np.uint8)
        seed = int(rs.integers(1 << 30))
        probe = R.rng(seed=seed)
        draws = np.array([probe.next_u64() for _ in range(200)], dtype=np.uint64)
        stock = R.rng(seed=seed)
        Cb, fb, nb = R.reinit(S, C0 * (1 - fl[:, None]), fl, stock)
        b = R.kmeans(S, Cb)
        a = J.step(S, C0 * (1 - fl[:, None]), fl, draws)
        assert np.array_equal(a["seeded"], Cb)
        assert np.array_equal(a["centroids"], b["centroids"]) and a["objective"] == b["objective"]
        assert a["iterations"] == b["iterations"] and a["stop"] == b["stop"]
        # the stock stream after reinit sits exactly `consumed` draws in
        assert stock.next_u64() == int(draws[a["consumed"]])


def test_injected_philox_draw_encoding():
    """RefInject.philox_draws: the reference turns the injected values back into the given first
    row (uniform_index) and units (next_unit) exactly."""
    from oracle_py import ref_inject
    J = ref_inject()
    if J is None:
        pytest.skip("oracle/_ref not built")
    rs = np.random.default_rng(3)
    units = np.floor(rs.random(9) * 2.0 ** 53) / 2.0 ** 53
    d = J.philox_draws(17, units, True)
    assert int(d[0]) == 17
    back = (d[1:] >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    assert np.array_equal(back, units)
