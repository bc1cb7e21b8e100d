"""Multi-rank engine in the library (include/hpcg.h multi-GPU).

A G-rank run -- rank r owns rows chunk_range(m, G, r) of X and workers [r W, (r+1) W), samples are
global over all ranks' rows (row shards peer-mapped), every round's publication runs over all
ranks' workers through the library's exchange (pack -> all-gather -> device publication scan on
every rank), select_best and f(C, X) over all ranks -- must equal ONE engine with G W workers on
the whole X: centroids, n_d, best worker, per-worker incumbents and the publication log bit-exact
(the reference semantics: engine.hpp:165-177 global sampling, 391-402 id-ordered strict-< publication,
386/396 hybrid carry-over, 180-194 select_best, 483-491 final pass); f(C, X) within 1e-12 (a sum of
shard partials vs one pass).

This pool gives one GPU, so the ranks share it: (a) two ranks as two threads of one process, the
all-gather a host barrier; (b) two processes over torch.distributed gloo with the shard of the other
process mapped by CUDA IPC. On an 8-GPU box the same engine path runs over NCCL (bench.py).
"""
import os
import subprocess
import sys
import threading
from pathlib import Path

import numpy as np
import pytest

import paper_2311_04517_b200 as hp
from test_parity_gpu import mixture, rel

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


class ThreadAllGather:
    """Host all-gather between G threads of one process (rank order)."""

    def __init__(self, G):
        self.G, self.buf, self.bar = G, [None] * G, threading.Barrier(G)

    def fn(self, rank):
        def ag(b):
            self.buf[rank] = b
            self.bar.wait()
            out = b"".join(self.buf)
            self.bar.wait()
            return out
        return ag


def single_run(X, cfg_kw, W_total, seed):
    ds = hp.DeviceDataset(X)
    eng = hp.Engine(ds, hp.EngineConfig(n_workers=W_total, **cfg_kw))
    eng.reset(seed)
    eng.run()
    res = eng.finish()
    eng.close()
    ds.close()
    return res


def chunk(m, G, r):
    base, extra = divmod(m, G)
    b = r * base + min(r, extra)
    return b, b + base + (1 if r < extra else 0)


def threaded_run(X, cfg_kw, W, G, seed):
    import torch
    m, n = X.shape
    parts = [torch.from_numpy(np.ascontiguousarray(X[slice(*chunk(m, G, r))])).cuda() for r in range(G)]
    shards = [(p.data_ptr(), p.shape[0], n, X.dtype) for p in parts]
    ag = ThreadAllGather(G)
    out, errs = [None] * G, [None] * G

    def rank_main(r):
        try:
            ctx = hp.Context(0)
            ds = hp.DeviceDataset.from_shards(shards, ctx=ctx, keepalive=parts)
            eng = hp.Engine(ds, hp.EngineConfig(n_workers=W, worker_base=r * W, **cfg_kw))
            eng.set_exchange(G, r, ag.fn(r))
            eng.reset(seed)
            eng.run()
            out[r] = eng.finish()
            eng.close()
            ds.close()
        except Exception as ex:  # pragma: no cover - reported below
            errs[r] = ex
            ag.bar.abort()

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for e in errs:
        if e is not None:
            raise e
    return out


def assert_same(single, ranks, W):
    for r, res in enumerate(ranks):
        assert np.array_equal(res.centroids, single.centroids), r
        assert np.array_equal(res.degenerate, single.degenerate), r
        assert res.best_worker == single.best_worker, r
        assert res.best_sample_objective == single.best_sample_objective, r
        assert res.distance_evals == single.distance_evals, r
        assert res.total_samples == single.total_samples, r
        assert res.clustering_time == single.clustering_time, r
        assert np.array_equal(res.publications, single.publications), r
        assert np.array_equal(res.worker_objectives, single.worker_objectives[r * W:(r + 1) * W]), r
        for w in range(W):
            assert np.array_equal(res.traces[w], single.traces[r * W + w]), (r, w)
        assert rel(res.full_objective, single.full_objective) <= 1e-12, r


@pytest.mark.parametrize("strategy,t1,t2,rng", [("cooperative", 0.0, 0.0, "philox"),
                                                ("hybrid", 2.0, 3.0, "philox"),
                                                ("hybrid", 2.5, 2.5, "reference"),
                                                ("competitive", 0.0, 0.0, "philox")])
def test_two_rank_threads_equal_one_engine(strategy, t1, t2, rng):
    X = mixture(40001, 8, 7, seed=21, dtype=np.float32)
    W, G = 6, 2
    kw = dict(k=7, sample_size=3000, max_samples=5, strategy=strategy, phase_t1=t1, phase_t2=t2, rng=rng,
              compute_full_objective=True)
    single = single_run(X, kw, G * W, seed=99)
    ranks = threaded_run(X, kw, W, G, seed=99)
    assert_same(single, ranks, W)


def test_three_rank_threads_fp64_uneven_shards():
    X = mixture(30011, 3, 5, seed=8, dtype=np.float64)
    W, G = 4, 3
    kw = dict(k=5, sample_size=2000, max_samples=4, strategy="cooperative", rng="philox",
              compute_full_objective=True)
    single = single_run(X, kw, G * W, seed=5)
    ranks = threaded_run(X, kw, W, G, seed=5)
    assert_same(single, ranks, W)


def test_set_exchange_rejects_gaps_in_worker_ids():
    X = mixture(8000, 4, 3, seed=1, dtype=np.float32)
    G = 2
    ag = ThreadAllGather(G)
    errs = [None] * G

    def rank_main(r):
        ds = hp.DeviceDataset(X, ctx=hp.Context(0))
        eng = hp.Engine(ds, hp.EngineConfig(k=3, sample_size=500, n_workers=2, max_samples=1,
                                            strategy="cooperative", rng="philox", worker_base=r * 5))
        try:
            eng.set_exchange(G, r, ag.fn(r))
        except Exception as ex:
            errs[r] = ex

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(G)]
    [t.start() for t in th]
    [t.join() for t in th]
    assert all(isinstance(e, hp.InvalidArgument) and "contiguous" in str(e) for e in errs)


CHILD = r'''
import sys, os, numpy as np
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, os.path.join(sys.argv[1], "tests"))
import torch, torch.distributed as dist
import paper_2311_04517_b200 as hp
rank, world, port, xfile, out = int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], sys.argv[5], sys.argv[6]
dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
X = np.load(xfile); m, n = X.shape
base, extra = divmod(m, world)
lo = rank * base + min(rank, extra); hi = lo + base + (1 if rank < extra else 0)
mine = torch.from_numpy(np.ascontiguousarray(X[lo:hi])).cuda()
# exchange IPC handles of the shards over gloo, map the peers' shards (NVLink P2P on a multi-GPU box)
h = torch.tensor(list(hp.ipc_export(mine.data_ptr())), dtype=torch.uint8)
hs = [torch.empty_like(h) for _ in range(world)]
dist.all_gather(hs, h)
allrows = [None] * world
dist.all_gather_object(allrows, hi - lo)
shards, peers = [], []
for r in range(world):
    if r == rank:
        shards.append((mine.data_ptr(), hi - lo, n, X.dtype))
    else:
        hb = bytes(hs[r].tolist()); p = hp.ipc_open(hb); peers.append((p, hb))
        shards.append((p, allrows[r], n, X.dtype))
ds = hp.DeviceDataset.from_shards(shards, keepalive=mine)
W = 5
def ag(b):
    t = torch.frombuffer(bytearray(b), dtype=torch.uint8)
    outs = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(outs, t)
    return b"".join(bytes(o.numpy()) for o in outs)
eng = hp.Engine(ds, hp.EngineConfig(k=6, sample_size=2500, n_workers=W, max_samples=4, strategy="hybrid",
                                    phase_t1=1.5, phase_t2=2.5, rng="philox", worker_base=rank * W,
                                    compute_full_objective=True))
eng.set_exchange(world, rank, ag)
eng.reset(7)
eng.run()
r = eng.finish()
np.savez(out, centroids=r.centroids, pubs=r.publications, wobj=r.worker_objectives, nd=r.distance_evals,
         best=r.best_worker, f=r.full_objective)
eng.close(); ds.close()
dist.barrier()
for p, hb in peers: hp.ipc_close(p, hb)
dist.destroy_process_group()
'''


def test_two_processes_gloo_ipc_shards_equal_one_engine(tmp_path):
    X = mixture(30000, 6, 6, seed=44, dtype=np.float32)
    np.save(tmp_path / "x.npy", X)
    port = str(29500 + (os.getpid() % 1000))
    procs = [subprocess.Popen([sys.executable, "-c", CHILD, str(ROOT), str(r), "2", port, str(tmp_path / "x.npy"),
                               str(tmp_path / f"r{r}.npz")]) for r in range(2)]
    for p in procs:
        assert p.wait(timeout=300) == 0
    single = single_run(X, dict(k=6, sample_size=2500, max_samples=4, strategy="hybrid", phase_t1=1.5, phase_t2=2.5,
                                rng="philox", compute_full_objective=True), 10, seed=7)
    for r in range(2):
        d = np.load(tmp_path / f"r{r}.npz")
        assert np.array_equal(d["centroids"], single.centroids)
        assert np.array_equal(d["pubs"], single.publications)
        assert np.array_equal(d["wobj"], single.worker_objectives[r * 5:(r + 1) * 5])
        assert int(d["nd"]) == single.distance_evals and int(d["best"]) == single.best_worker
        assert rel(float(d["f"]), single.full_objective) <= 1e-12
