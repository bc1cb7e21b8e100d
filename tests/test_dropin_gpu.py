"""GPU: the C++ drop-in (include/hpclust/hpclust.hpp over libhpcg.so) used exactly as a
reference user would (examples/dropin_example.cpp) reproduces the reference semantics:
same draw_sample rows, same K-means++ centres, same Lloyd outcome, same engine run."""
import json
import subprocess
import tempfile
from pathlib import Path

import numpy as np
import pytest

from oracle_py import orc

ROOT = Path(__file__).resolve().parents[1]
EXE = ROOT / "examples" / "dropin_example"


def test_dropin_binary_builds():
    if not EXE.exists():
        subprocess.run(["make", "-C", str(ROOT / "examples")], check=True)
    assert EXE.exists()


@pytest.mark.gpu
def test_dropin_matches_reference_semantics():
    rs = np.random.default_rng(4)
    means = rs.uniform(-10, 10, (5, 2))
    X = means[rs.integers(0, 5, 8000)] + rs.standard_normal((8000, 2))
    with tempfile.NamedTemporaryFile(suffix=".f64", delete=False) as f:
        X.astype(np.float64).tofile(f.name)
        out = subprocess.run([str(EXE), f.name, "8000", "2"], capture_output=True, text=True, timeout=300)
    r = json.loads(out.stdout)
    assert "error" not in r, r
    o = orc()
    rng = o.rng(seed=7)
    idx = o.draw_indices(8000, 500, rng)
    S = X[idx]
    assert r["sample0"] == S[0, 0]
    C0, f0, nd_seed = o.reinit(S, np.zeros((5, 2)), np.ones(5, np.uint8), rng)
    assert r["seed_c0"] == C0[0, 0]
    e = o.kmeans(S, C0)
    assert abs(r["lloyd_obj"] - e["objective"]) <= 1e-12 * e["objective"]
    assert r["lloyd_iters"] == e["iterations"]
    assert r["lloyd_stop"] == ["tolerance", "max_iters", "fixed_point"][e["stop"]]
    assert r["nd"] == nd_seed + e["n_d"]
    _, _, fo, _ = o.assign(X, e["centroids"])
    assert abs(r["f_full"] - fo) <= 1e-12 * fo
    run = o.run(X, k=5, sample_size=500, n_workers=3, max_samples=4, strategy="cooperative", seed=11)
    assert abs(r["run_full"] - run["full_objective"]) <= 1e-12 * run["full_objective"]
    assert r["run_best"] == run["best_worker"] and r["run_nd"] == run["distance_evals"]
    assert abs(r["run_c0"] - run["centroids"][0, 0]) <= 1e-12 * abs(run["centroids"][0, 0])
    assert r["pubs"] == len(run["publications"])
    # wall-clock schedule through the drop-in: stops at the first round end past 0.2 s
    assert r["wall_seconds"] >= 0.2 and r["wall_samples"] > 0 and r["wall_samples"] % 3 == 0
    assert r["wall_full"] > 0
    # free-running workers through the drop-in: per-worker sample counts and clocks (WorkerState)
    assert r["free_samples"] == r["free_sum"] > 0 and r["free_min"] >= 1
    assert 0.1 < r["free_tw_max"] <= r["free_seconds"] and r["free_pubs"] >= 1 and r["free_full"] > 0


BEXE = ROOT / "examples" / "baselines_example"


@pytest.mark.gpu
@pytest.mark.parametrize("p", [0, 2000, 1700])  # Forgy; PBK-BDC with full segments; with a short tail
def test_dropin_baselines_match_reference(p):
    # hpclust/baselines.hpp on the device vs the reference's baselines.hpp (oracle/_ref): same RNG
    # consumption, same Lloyd outcomes per segment, same repository, same final assignment
    from oracle_py import ref
    r_ = ref()
    if r_ is None or not hasattr(r_.lib, "hpref_baseline"):
        pytest.skip("reference harness not built")
    if not BEXE.exists():
        subprocess.run(["make", "-C", str(ROOT / "examples")], check=True)
    rs = np.random.default_rng(8 + p)
    means = rs.uniform(-10, 10, (6, 3))
    X = means[rs.integers(0, 6, 10000)] + rs.standard_normal((10000, 3))
    with tempfile.TemporaryDirectory() as d:
        path = str(Path(d) / "X.f64")
        X.astype(np.float64).tofile(path)
        out = subprocess.run([str(BEXE), path, "10000", "3", "5", str(p), "77"], capture_output=True, text=True,
                             timeout=300)
        g = json.loads(out.stdout)
        assert "error" not in g, g
        C_ = np.fromfile(path + ".C").reshape(5, 3)
        F_ = np.fromfile(path + ".F", dtype=np.uint8)
        L_ = np.fromfile(path + ".L", dtype=np.int32)
    e = r_.baseline(X, 5, p, 77)
    assert g["samples"] == e["total_samples"]
    assert g["nd"] == e["n_d"]
    assert np.array_equal(F_, e["degenerate"])
    assert np.array_equal(L_, e["labels"])
    assert np.max(np.abs(C_ - e["centroids"])) <= 1e-12 * np.max(np.abs(e["centroids"]))
    assert abs(g["f"] - e["full_objective"]) <= 1e-12 * e["full_objective"]


@pytest.mark.gpu
def test_device_dataset_overloads_no_per_call_upload():
    """hpclust::DeviceDataset (additive overloads): 100 draw_sample calls on a resident
    X move no dataset bytes host -> device; the resident draw_sample / worker_step / run / mssc_objective
    equal the reference-signature (per-call upload) versions draw for draw; parallel.hpp's ThreadPool,
    RowRange and chunk_range and LloydConfig::policy() behave as the reference's (parallel.hpp:16-112,
    lloyd.hpp:16-19)."""
    import os
    exe = ROOT / "examples" / "device_dataset_example"
    if not exe.exists():
        subprocess.run(["make", "-C", str(ROOT / "examples")], check=True)
    rs = np.random.default_rng(8)
    m, n = 200_000, 4
    X = rs.uniform(-10, 10, (6, n))[rs.integers(0, 6, m)] + rs.standard_normal((m, n))
    with tempfile.NamedTemporaryFile(suffix=".f64", delete=False) as f:
        X.astype(np.float64).tofile(f.name)
        out = subprocess.run([str(exe), f.name, str(m), str(n)], capture_output=True, text=True, timeout=300)
    r = json.loads(out.stdout)
    assert "error" not in r, r
    assert r["upload_bytes_100_draws"] == 0
    assert r["pinned"] == 1 and r["pin_same"] == 1 and r["pin_run"] == 1  # io.hpp load_dataset_pinned
    assert r["draw_same"] == 1 and r["run_same"] == 1 and r["ws_same"] == 1
    assert r["f_dev"] == r["f_host"]
    assert r["policy_chunks"] == (os.cpu_count() or 1)
    base, extra = divmod(m, 4)
    assert r["rr"] == [3 * base + min(3, extra), 3 * base + min(3, extra) + base + (1 if 3 < extra else 0)]
    assert abs(r["pool_sum"] - X[:, 0].sum()) <= 1e-9 * np.abs(X[:, 0]).sum()


@pytest.mark.gpu
def test_multigpu_run_equals_single_gpu():
    """hpclust::run(X, cfg, devices): every GPU of the node as one rank (NCCL exchange) equals run(X, cfg)."""
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("one GPU in this pool: the multi-rank engine is covered by test_multirank_gpu.py")
    exe = ROOT / "examples" / "multigpu_example"
    rs = np.random.default_rng(9)
    m, n = 100_000, 5
    X = rs.uniform(-10, 10, (6, n))[rs.integers(0, 6, m)] + rs.standard_normal((m, n))
    with tempfile.NamedTemporaryFile(suffix=".f64", delete=False) as f:
        X.astype(np.float64).tofile(f.name)
        out = subprocess.run([str(exe), f.name, str(m), str(n)], capture_output=True, text=True, timeout=600)
    r = json.loads(out.stdout)
    assert "error" not in r, r
    assert r["same_centroids"] == 1 and r["nd_multi"] == r["nd_single"] and r["best_multi"] == r["best_single"]
    assert abs(r["f_multi"] - r["f_single"]) <= 1e-12 * r["f_single"]
