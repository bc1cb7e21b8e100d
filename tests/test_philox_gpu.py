"""The BENCHMARKED path replayed through the reference itself.

bench.py runs config 2 with rng="philox": every round's sample indices come from the device's
keyed permutation and every K-means++ draw from Philox. This test runs that exact engine (config-2
data and shape: m = 1e7 x 16 fp32, k = 10, s = 20,000, W = 256 workers, cooperative, 4 lockstep
rounds) round by round and replays EVERY worker of every round through the UNMODIFIED reference
worker step (oracle/_ref/libhpclust_ref_inject.so: reinit_degenerate + kmeans, engine.hpp:238-267)
fed the device's own sample indices and K-means++ draws. Bar (north star): Lloyd iterations, stop
reason, n_d, acceptance bit-exact; sample objectives and centroids within 1e-12 relative (fp32
data widened to fp64 in both; tighter than the 1e-5 fp32-mode gate); the shared best after each
round is the reference's publication rule applied to the replayed outcomes (engine.hpp:391-402).
"""
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import bench
import paper_2311_04517_b200 as hp
from oracle_py import ref_inject

pytestmark = pytest.mark.gpu
RTOL = 1e-12


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300))) if a.size else 0.0


@pytest.fixture(scope="module")
def cfg2():
    return bench.make_data(0)


def test_config2_philox_rounds_replay_through_reference(cfg2):
    J = ref_inject()
    if J is None:
        pytest.skip("oracle/_ref not built")
    X = cfg2
    m, n = X.shape
    k, s, W, R = bench.K, bench.S, bench.W_PER_GPU, bench.ROUNDS
    ds = hp.DeviceDataset(X)
    eng = hp.Engine(ds, hp.EngineConfig(k=k, sample_size=s, n_workers=W, max_samples=R, strategy="cooperative",
                                        rng="philox", master_seed=2024))
    key = eng.philox_key
    X64 = X  # rows widened per sample below
    shared_obj = np.inf
    for r in range(R):
        obj0, _, Csh, fsh = eng.export_best()
        _, _, inc_obj0 = eng.worker_incumbents()
        init_f = fsh.copy() if np.isfinite(obj0) else np.ones(k, np.uint8)
        init_c = Csh * (init_f == 0)[:, None]
        nv = int((init_f == 0).sum())
        no_valid = nv == 0
        loops = k - nv - (1 if no_valid else 0)
        eng.rounds(1)
        out = eng.round_outcome()
        Cw, fw, ow = eng.worker_incumbents()

        def replay(w):
            idx = hp.philox_sample_indices(m, s, key, r, w)
            assert len(np.unique(idx)) == s and idx.min() >= 0 and idx.max() < m
            S = X64[idx].astype(np.float64)
            fr, units = hp.philox_seed_draws(key, r, w, s, no_valid, loops, 3)
            return J.step(S, init_c, init_f, J.philox_draws(fr, units, no_valid))

        idxs = [hp.philox_sample_indices(m, s, key, r, w) for w in range(2)]  # warm the context once
        del idxs
        with ThreadPoolExecutor(max_workers=16) as ex:
            res = list(ex.map(replay, range(W)))
        acc_ref = np.array([res[w]["objective"] < inc_obj0[w] for w in range(W)])
        for w in range(W):
            e = res[w]
            assert out["iterations"][w] == e["iterations"], (r, w)
            assert out["stop"][w] == e["stop"], (r, w)
            assert out["n_d"][w] == e["n_d"], (r, w)
            assert rel(out["objective"][w], e["objective"]) <= RTOL, (r, w)
            if acc_ref[w]:
                assert rel(Cw[w], e["centroids"]) <= RTOL, (r, w)
                assert np.array_equal(fw[w], e["degenerate"]), (r, w)
        assert np.array_equal(out["accepted"], acc_ref), r
        # publication (engine.hpp:391-402): accepted incumbents in worker-id order, strict <
        best_w = -1
        for w in range(W):
            if acc_ref[w] and res[w]["objective"] < shared_obj:
                shared_obj, best_w = res[w]["objective"], w
        obj1, wk1, C1, f1 = eng.export_best()
        if best_w >= 0:
            assert wk1 == best_w and rel(obj1, shared_obj) <= RTOL and rel(C1, res[best_w]["centroids"]) <= RTOL
        shared_obj = obj1  # continue from the device's record (identical within the tolerance)
    eng.close()
    ds.close()
