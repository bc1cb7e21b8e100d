"""Generate tests/golden/*.npz from the REFERENCE ITSELF (oracle/_ref/libhpclust_ref.so, i.e.
the unmodified /root/reference/proj/include headers compiled by oracle/Makefile).

Run in the build container (where /root/reference exists):  python tests/golden/make_golden.py
The fixtures are small and committed; the GPU box never needs /root/reference.
"""
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
from oracle_py import ref  # noqa: E402

R = ref()
assert R is not None, "oracle/_ref not built (make -C oracle ref)"
out = {}


def mixture(rs, m, n, comps, spread=10.0):
    means = rs.uniform(-spread, spread, (comps, n))
    return means[rs.integers(0, comps, m)] + rs.standard_normal((m, n))


rs = np.random.default_rng(20231104)

# 1. kmeans (lloyd.hpp:100-164) on small samples with given inits
for t, (s, n, k, mi, tol) in enumerate([(200, 2, 3, 300, 1e-4), (500, 3, 5, 300, 1e-4), (300, 7, 4, 2, 1e-4),
                                        (400, 5, 6, 300, 0.3), (150, 1, 2, 300, 1e-4), (600, 16, 10, 300, 1e-4)]):
    S = mixture(rs, s, n, k + 1)
    C0 = S[rs.choice(s, k, replace=False)]
    e = R.kmeans(S, C0, max_iters=mi, rel_tol=tol)
    out[f"km{t}_S"], out[f"km{t}_C0"] = S, C0
    out[f"km{t}_cfg"] = np.array([mi, tol])
    for key in ("centroids", "degenerate", "labels", "counts", "history"):
        out[f"km{t}_{key}"] = e[key]
    out[f"km{t}_scalars"] = np.array([e["objective"], e["iterations"], e["stop"], e["n_d"]], dtype=np.float64)

# 2. seeding (seeding.hpp:113-133) with reference streams RngStream(seed)
for t, (s, n, k, npend, seed) in enumerate([(300, 2, 5, 5, 11), (500, 3, 8, 3, 12), (200, 4, 6, 6, 13)]):
    S = mixture(rs, s, n, k)
    C0 = S[rs.choice(s, k, replace=False)].copy()
    fl = np.zeros(k, np.uint8)
    fl[rs.choice(k, npend, replace=False)] = 1
    C0[fl == 1] = 0.0
    r = R.rng(seed=seed)
    Co, fo, nd = R.reinit(S, C0, fl, r)
    out[f"sd{t}_S"], out[f"sd{t}_C0"], out[f"sd{t}_f0"] = S, C0, fl
    out[f"sd{t}_seed"] = np.array([seed], np.uint64)
    out[f"sd{t}_C"], out[f"sd{t}_f"] = Co, fo
    out[f"sd{t}_nd_next"] = np.array([nd, r.next_u64()], dtype=np.uint64)

# 3. draw_sample indices (engine.hpp:165-177) for derived worker streams
for t, (m, s, master, wi) in enumerate([(1000, 50, 0, 0), (5000, 400, 7, 3), (64, 64, 1, 1)]):
    r = R.rng(derive=(master, 1, wi))
    out[f"dr{t}_cfg"] = np.array([m, s, master, wi], np.int64)
    out[f"dr{t}_idx"] = R.draw_indices(m, s, r)
    out[f"dr{t}_next"] = np.array([r.next_u64()], np.uint64)

# 4. engine run (engine.hpp:444-499), deterministic lockstep, every strategy
X = mixture(rs, 3000, 2, 5)
out["run_X"] = X
for t, (strat, t1, t2, W) in enumerate([("competitive", 0, 0, 3), ("cooperative", 0, 0, 3), ("hybrid", 2.5, 2.5, 3),
                                        ("hybrid", 5, 0, 2), ("inner", 0, 0, 1)]):
    e = R.run(X, k=5, sample_size=500, n_workers=W, max_samples=5, strategy=strat, t1=t1, t2=t2, seed=99, n_threads=4)
    out[f"run{t}_cfg"] = np.array([["competitive", "cooperative", "hybrid", "inner"].index(strat), t1, t2, W])
    out[f"run{t}_centroids"] = e["centroids"]
    out[f"run{t}_scalars"] = np.array([e["full_objective"], e["best_worker"], e["best_sample_objective"],
                                       e["clustering_time"], e["clustering_time_first_finisher"], e["total_samples"],
                                       e["distance_evals"]], dtype=np.float64)
    out[f"run{t}_pubs"] = e["publications"]
    out[f"run{t}_wobj"] = e["worker_obj"]

# 5. BASELINE config 1 data (bench.hpp gen_blobs) fingerprint + objective at the generator centres
Xb = R.gen_blobs(100000, 2, 5, center=(-10.0, 10.0), std=(1.0, 1.0), noise_points=0, seed=0)
out["cfg1_head"] = Xb[:16]
out["cfg1_sum"] = np.array([Xb.sum(), (Xb ** 2).sum()])
lab, cnt, cost, nd = R.assign(Xb, Xb[[0, 20000, 40000, 60000, 80000]])
out["cfg1_assign"] = np.array([cost, nd], np.float64)
out["cfg1_counts"] = cnt

# 6. brute force (bench.hpp:239-297) on tiny instances
for t in range(3):
    Xs = rs.uniform(-5, 5, (8 + t, 2))
    Cb, fb, cb = R.brute_force(Xs, 2)
    out[f"bf{t}_X"], out[f"bf{t}_cost"] = Xs, np.array([cb])

np.savez_compressed(HERE / "ref_cases.npz", **out)
print("wrote", HERE / "ref_cases.npz", len(out), "arrays")
