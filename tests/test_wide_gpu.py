"""GPU parity of the grid-wide worker step (csrc/wide.cu): the shapes the cluster-resident
kernel cannot hold -- n > 32 (BASELINE config 4: n = 128), k > 32, samples larger than a
cluster's shared memory -- against the CPU oracle, with the same bars as test_parity_gpu.py."""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

import paper_2311_04517_b200 as hp
from oracle_py import orc
from test_parity_gpu import RTOL, centroid_close, mixture, obj_rtol, rel

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype,n,k,s,W", [
    (np.float32, 40, 6, 3000, 3),
    (np.float64, 64, 12, 2000, 2),
    (np.float32, 128, 25, 4000, 2),   # config 4 shape (smaller sample)
    (np.float64, 5, 40, 3000, 2),     # k > 32
    (np.float32, 16, 10, 300000, 1),  # sample beyond a cluster's shared memory
])
def test_wide_kmeans_vs_oracle(dtype, n, k, s, W):
    m = max(2 * s, 20000)
    X = mixture(m, n, k + 2, seed=n * 10 + k, dtype=dtype)
    rs = np.random.default_rng(3)
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


@pytest.mark.parametrize("dtype,n,k,s,npend", [(np.float64, 48, 10, 3000, 10), (np.float32, 128, 25, 2000, 7),
                                               (np.float64, 3, 40, 2500, 40),
                                               # k > 32 keeps these on the grid-wide path: the cost pass
                                               # specialised for n = 8 / 16 / 32
                                               (np.float32, 8, 40, 3000, 40), (np.float64, 16, 36, 2500, 30),
                                               (np.float32, 32, 34, 2000, 20)])
def test_wide_seeding_with_reference_draws(dtype, n, k, s, npend):
    X = mixture(s, n, k, seed=31 + k, dtype=dtype)
    rs = np.random.default_rng(5)
    init = X[rs.choice(s, k, replace=False)].astype(np.float64)
    deg = np.zeros(k, np.uint8)
    deg[rs.choice(k, npend, replace=False)] = 1
    init[deg == 1] = 0.0
    rng = hp.RngStream(777 + k)
    Cg, fg = hp.reinit_degenerate(init, deg, X, hp.SeedConfig(), rng)
    o = orc()
    r2 = o.rng(seed=777 + k)
    Co, fo, _ = o.reinit(X.astype(np.float64), init, deg, r2)
    assert np.array_equal(fg, fo)
    assert np.array_equal(Cg, Co)  # seeded centres are rows of S: bitwise
    assert rng.next_u64() == o.next_u64(r2)


@pytest.mark.parametrize("n", [64, 128])
def test_wide_seeding_duplicate_rows_exact_fallback(n):
    # a sample of 12 distinct rows repeated: K-means++ candidates coincide, their costs tie exactly, the
    # interval pass of the wide-row cost kernel cannot separate them and the exact pass decides (strict <,
    # the first candidate wins: seeding.hpp:94-98)
    rs = np.random.default_rng(n)
    base = rs.normal(0.0, 2.0, (12, n))
    X = (base[rs.integers(0, 12, 3000)] + 0.0).astype(np.float32)
    k = 20
    init = np.zeros((k, n))
    deg = np.ones(k, np.uint8)
    rng = hp.RngStream(4242 + n)
    Cg, fg = hp.reinit_degenerate(init, deg, X, hp.SeedConfig(), rng)
    o = orc()
    r2 = o.rng(seed=4242 + n)
    Co, fo, _ = o.reinit(X.astype(np.float64), init, deg, r2)
    assert np.array_equal(fg, fo)
    assert np.array_equal(Cg, Co)
    assert rng.next_u64() == o.next_u64(r2)


@pytest.mark.parametrize("dtype,n,k", [(np.float32, 128, 25), (np.float64, 33, 7), (np.float32, 8, 300)])
def test_wide_objective_vs_oracle(dtype, n, k):
    X = mixture(60001, n, min(k, 30), seed=7 + n, dtype=dtype)
    C_ = mixture(k, n, min(k, 30), seed=98, dtype=np.float64)
    lab, cnt, cost, _ = orc().assign(X.astype(np.float64), C_)
    a, f = hp.final_assignment(X, C_)
    assert np.array_equal(a.labels, lab)
    assert np.array_equal(a.counts, cnt)
    assert rel(f, cost) <= obj_rtol(X)


@pytest.mark.parametrize("strategy", ["competitive", "cooperative"])
def test_wide_run_reference_rng_vs_oracle(strategy):
    X = mixture(5000, 40, 6, seed=19)
    kw = dict(k=6, sample_size=700, n_workers=3, max_samples=4, strategy=strategy, seed=9)
    e = orc().run(X, **kw)
    g = hp.run(X, hp.EngineConfig(k=6, sample_size=700, n_workers=3, max_samples=4, strategy=strategy,
                                  master_seed=9, rng="reference"))
    assert g.best_worker == e["best_worker"]
    assert g.distance_evals == e["distance_evals"]
    assert centroid_close(g.centroids, e["centroids"])
    assert rel(g.full_objective, e["full_objective"]) <= RTOL
    assert rel(g.best_sample_objective, e["best_sample_objective"]) <= RTOL


def test_config4_shaped_philox_run():
    # BASELINE config 4 shape (n=128, k=25, equal-weight N(0,4I) means, sigma=1) at reduced m, s
    rs = np.random.default_rng(4)
    k, n = 25, 128
    X = hp.gen_mixture(100_000, n, rs.normal(0.0, 2.0, (k, n)), np.ones(k), np.ones(k) / k, seed=2)
    cfg = hp.EngineConfig(k=k, sample_size=10_000, n_workers=4, max_samples=2, strategy="cooperative",
                          master_seed=3, rng="philox")
    a = hp.run(X, cfg)
    b = hp.run(X, cfg)
    assert np.array_equal(a.centroids, b.centroids) and a.full_objective == b.full_objective
    lab, cnt, cost, _ = orc().assign(X.astype(np.float64), a.centroids, a.degenerate)
    assert rel(a.full_objective, cost) <= obj_rtol(X)


def test_forced_wide_path_matches_oracle_on_a_resident_shape(tmp_path):
    # HPCG_WIDE=1 sends a shape the resident kernel would take through wide.cu (read once per
    # process): Lloyd from given inits must still equal the oracle
    code = r'''
import sys, numpy as np
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + "/tests")
import paper_2311_04517_b200 as hp
from oracle_py import orc
from test_parity_gpu import mixture, centroid_close, rel
X = mixture(20000, 16, 10, seed=5, dtype=np.float32)
rs = np.random.default_rng(2)
idx = rs.choice(20000, 5000, replace=False)[None]
init = X[rs.choice(20000, 10, replace=False)].astype(np.float64)[None]
r = hp.worker_step_batched(X, idx, init, None, want_labels=True)
e = orc().kmeans(X.astype(np.float64)[idx[0]], init[0])
assert np.array_equal(r["labels"][0], e["labels"]) and r["iterations"][0] == e["iterations"]
assert centroid_close(r["centroids"][0], e["centroids"]) and rel(r["objective"][0], e["objective"]) <= 1e-12
print("ok")
'''
    env = dict(os.environ, HPCG_WIDE="1")
    root = str(Path(__file__).resolve().parents[1])
    out = subprocess.run([sys.executable, "-c", code, root], env=env, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and "ok" in out.stdout, out.stdout + out.stderr


@pytest.mark.parametrize("n,k", [(64, 12), (128, 30)])
def test_wide_tc_screen_near_ties_vs_oracle(n, k):
    # config-4 widths on the tensor-core Lloyd screen with rows far from the origin around nearby
    # centres: most rows fall inside the tf32 bound, take the fp32 re-screen and then the exact argmin
    rs = np.random.default_rng(n + k)
    base = 500.0 + rs.standard_normal(n)
    C0 = base + 0.2 * rs.standard_normal((k, n))
    m, s = 12000, 3000
    X = (C0[rs.integers(0, k, m)] + 0.2 * rs.standard_normal((m, n))).astype(np.float32)
    idx = np.stack([rs.choice(m, s, replace=False) for _ in range(2)])
    inits = np.stack([X[rs.choice(m, k, replace=False)].astype(np.float64) for _ in range(2)])
    r = hp.worker_step_batched(X, idx, inits, None, want_labels=True, want_counts=True)
    o = orc()
    Xw = X.astype(np.float64)
    for w in range(2):
        e = o.kmeans(Xw[idx[w]], inits[w])
        assert r["iterations"][w] == e["iterations"] and r["stop"][w] == e["stop"], w
        assert np.array_equal(r["labels"][w], e["labels"]), w
        assert np.array_equal(r["counts"][w], e["counts"]), w
        assert rel(r["objective"][w], e["objective"]) <= RTOL, w
