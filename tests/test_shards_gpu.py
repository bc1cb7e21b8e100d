"""Row-sharded datasets (multi-GPU global sampling): X split into shards at
different device addresses -- on a node, peer-mapped over NVLink by CUDA IPC -- and sampled over
all m rows. On one GPU the shards are separate allocations (and, for the IPC test, another
process's allocation); every result must equal the contiguous dataset's and the oracle's."""
import os
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np
import pytest

import paper_2311_04517_b200 as hp
from oracle_py import orc

pytestmark = pytest.mark.gpu
RTOL = 1e-12
ROOT = Path(__file__).resolve().parents[1]


def mixture(m, n, comps, seed, dtype):
    rs = np.random.default_rng(seed)
    means = rs.uniform(-10, 10, (comps, n))
    return (means[rs.integers(0, comps, m)] + rs.standard_normal((m, n))).astype(dtype)


def shards_of(X, cuts):
    import torch
    parts = np.split(X, cuts)
    return [torch.from_numpy(np.ascontiguousarray(p)).cuda() for p in parts]


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300))) if a.size else 0.0


@pytest.mark.parametrize("dtype,n,k,s", [(np.float32, 16, 10, 4000),   # 16-B chunk gather
                                         (np.float64, 3, 7, 3000),    # 8-B chunks
                                         (np.float32, 5, 4, 3000),    # 4-B elements
                                         (np.float32, 128, 25, 3000)])  # grid-wide gather
def test_sharded_worker_step_vs_oracle(dtype, n, k, s):
    m = 30000
    X = mixture(m, n, k + 1, seed=n + k, dtype=dtype)
    ts = shards_of(X, [9000, 21000])  # uneven shards
    ds = hp.DeviceDataset.from_shards(ts)
    assert ds.m == m
    rs = np.random.default_rng(1)
    idx = np.stack([rs.choice(m, s, replace=False) for _ in range(2)])
    inits = np.stack([X[rs.choice(m, k, replace=False)].astype(np.float64) for _ in range(2)])
    r = hp.worker_step_batched(ds, idx, inits, None, want_labels=True)
    Xw = X.astype(np.float64)
    for w in range(2):
        e = orc().kmeans(Xw[idx[w]], inits[w])
        assert r["iterations"][w] == e["iterations"] and r["stop"][w] == e["stop"]
        assert np.array_equal(r["labels"][w], e["labels"])
        assert rel(r["objective"][w], e["objective"]) <= RTOL


def test_sharded_engine_equals_contiguous():
    import torch
    X = mixture(40000, 16, 8, seed=3, dtype=np.float32)
    cfg = hp.EngineConfig(k=8, sample_size=3000, n_workers=6, max_samples=3, strategy="cooperative",
                          master_seed=5, rng="philox")
    Xd = torch.from_numpy(X).cuda()
    a = hp.Engine(hp.DeviceDataset.from_torch(Xd), cfg)
    a.run()
    ra = a.finish()
    ts = shards_of(X, [13000, 27000])
    b = hp.Engine(hp.DeviceDataset.from_shards(ts), cfg)
    b.run()
    rb = b.finish()
    assert rb.best_worker == ra.best_worker and rb.distance_evals == ra.distance_evals
    assert np.array_equal(rb.centroids, ra.centroids)
    assert rel(rb.full_objective, ra.full_objective) <= RTOL  # per-shard partial sums, then their sum


def test_sharded_gather_and_assignment():
    X = mixture(25000, 4, 5, seed=8, dtype=np.float64)
    ts = shards_of(X, [10000])
    ds = hp.DeviceDataset.from_shards(ts)
    rng = hp.RngStream(11)
    S = hp.draw_sample(ds, 2000, rng)
    idx = hp.reference_draw_indices(25000, 2000, hp.RngStream(11))
    assert np.array_equal(S, X[idx])
    C_ = X[:5].astype(np.float64)
    a, f = hp.final_assignment(ds, C_)
    lab, cnt, cost, _ = orc().assign(X, C_)
    assert np.array_equal(a.labels, lab) and np.array_equal(a.counts, cnt)
    assert rel(f, cost) <= RTOL


CHILD = r'''
import sys, time, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_2311_04517_b200 as hp
X = np.load(sys.argv[2])
pad = torch.empty(1000, device="cuda")  # the shard is not at its allocation's base
t = torch.from_numpy(X).cuda()
open(sys.argv[3] + ".tmp", "wb").write(hp.ipc_export(t.data_ptr()))
import os; os.replace(sys.argv[3] + ".tmp", sys.argv[3])
while not os.path.exists(sys.argv[3] + ".done"):
    time.sleep(0.05)
'''


def test_ipc_peer_shard_in_another_process():
    # the multi-GPU wiring on one device: another process owns shard 1 and exports it; this
    # process maps it (hpcg_ipc_open) and samples across both shards
    import torch
    X = mixture(20000, 16, 6, seed=13, dtype=np.float32)
    with tempfile.TemporaryDirectory() as d:
        np.save(Path(d) / "x1.npy", X[12000:])
        hfile = str(Path(d) / "h.bin")
        child = subprocess.Popen([sys.executable, "-c", CHILD, str(ROOT), str(Path(d) / "x1.npy"), hfile])
        try:
            t0 = time.time()
            while not os.path.exists(hfile):
                assert time.time() - t0 < 120 and child.poll() is None, "child did not export"
                time.sleep(0.05)
            handle = open(hfile, "rb").read()
            peer = hp.ipc_open(handle)
            local = torch.from_numpy(np.ascontiguousarray(X[:12000])).cuda()
            ds = hp.DeviceDataset.from_shards([(local.data_ptr(), 12000, 16, np.float32),
                                               (peer, 8000, 16, np.float32)], keepalive=local)
            rs = np.random.default_rng(2)
            idx = rs.choice(20000, 3000, replace=False)[None]
            init = X[rs.choice(20000, 6, replace=False)].astype(np.float64)[None]
            r = hp.worker_step_batched(ds, idx, init, None, want_labels=True)
            e = orc().kmeans(X[idx[0]].astype(np.float64), init[0])
            assert np.array_equal(r["labels"][0], e["labels"]) and r["iterations"][0] == e["iterations"]
            ds.close()
            hp.ipc_close(peer, handle)
        finally:
            open(hfile + ".done", "w").close()
            child.wait(timeout=60)
