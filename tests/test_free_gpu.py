"""Free-running wall-clock schedule with immediate publication (run_wall_clock, engine.hpp:348-374;
SURVEY.md §8(f) rank 1): hpcg_engine_cfg.free_running. Groups of workers advance on their own
streams; each step draws its init from the device-side versioned incumbent under a lock and an
accepted cooperative result is published when its group's step ends, not at a round end.

Deterministic corners pin the machinery against the round-granular engine (hence the oracle):
  * competitive workers never interact, so with a sample cap the free-running run must equal the
    lockstep Philox run bit for bit whatever the grouping;
  * with ONE group holding every worker the chain prepare -> step -> publish is sequential and
    publishes in worker-id order, which is exactly the lockstep cooperative / hybrid schedule.
Free groups are non-deterministic by design (as the reference's threads): invariants are checked."""
import numpy as np
import pytest

import paper_2311_04517_b200 as hp
from oracle_py import orc

pytestmark = pytest.mark.gpu


def mixture(m, n, comps, seed):
    rs = np.random.default_rng(seed)
    means = rs.uniform(-10, 10, (comps, n))
    return means[rs.integers(0, comps, m)] + rs.standard_normal((m, n))


def run_engine(X, cfg):
    ds = hp.DeviceDataset(X)
    eng = hp.Engine(ds, cfg)
    try:
        eng.run()
        r = eng.finish()
        smp, tw = eng.worker_progress()
        Cw, fw, ow = eng.worker_incumbents()
        return r, smp, tw, Cw, fw, ow
    finally:
        eng.close()
        ds.close()


@pytest.mark.parametrize("group", [0, 1, 3])
def test_free_competitive_with_cap_equals_lockstep(group):
    X = mixture(30000, 4, 6, seed=21)
    base = dict(k=6, sample_size=3000, n_workers=7, strategy="competitive", master_seed=9, rng="philox")
    lock, _, _, Cl, fl, ol = run_engine(X, hp.EngineConfig(max_samples=5, **base))
    free, smp, tw, Cf, ff, of = run_engine(
        X, hp.EngineConfig(max_samples=5, time_limit=1e6, free_running=True, free_group=group, **base))
    assert np.array_equal(smp, np.full(7, 5)) and free.total_samples == lock.total_samples == 35
    assert free.distance_evals == lock.distance_evals
    assert np.array_equal(of, ol) and np.array_equal(Cf, Cl) and np.array_equal(ff, fl)
    assert free.best_worker == lock.best_worker and np.array_equal(free.centroids, lock.centroids)
    assert free.full_objective == lock.full_objective
    assert len(free.publications) == 0
    for w in range(7):  # same acceptances; the clock is seconds, strictly increasing per worker
        assert np.array_equal(free.traces[w][:, 1], lock.traces[w][:, 1])
        ts = free.traces[w][:, 0]
        assert np.all(np.diff(ts) > 0) and np.all(ts > 0) and ts[-1] <= tw[w] <= free.wall_seconds
    assert free.clustering_time == min(t[-1, 0] for t in free.traces)
    first = int(np.argmin(tw))
    assert free.clustering_time_first_finisher == free.traces[first][-1, 0]
    # and the lockstep Philox run is the oracle's run on the same draws elsewhere (tests/test_philox_gpu.py)
    _, _, cost, _ = orc().assign(X, free.centroids, free.degenerate)
    assert abs(free.full_objective - cost) <= 1e-12 * cost


@pytest.mark.parametrize("strategy", ["cooperative", "hybrid"])
def test_free_one_group_equals_lockstep_publication_order(strategy):
    X = mixture(30000, 4, 6, seed=22)
    W, R = 6, 6
    base = dict(k=6, sample_size=3000, n_workers=W, strategy=strategy, master_seed=5, rng="philox")
    # the wall-clock hybrid switches on seconds, not on sample counts: its cooperative corner (t1 = 0:
    # cooperative from the first step, infinite incumbents so nothing to carry over) is the comparable one
    free_kw = dict(phase_t1=0.0, phase_t2=1e6) if strategy == "hybrid" else {}
    lock, _, _, Cl, fl, ol = run_engine(X, hp.EngineConfig(max_samples=R, **{**base, "strategy": "cooperative"}))
    free, smp, tw, Cf, ff, of = run_engine(
        X, hp.EngineConfig(max_samples=R, time_limit=1e6, free_running=True, free_group=W, **base, **free_kw))
    assert np.array_equal(smp, np.full(W, R))
    assert free.distance_evals == lock.distance_evals
    assert np.array_equal(free.publications[:, :3], lock.publications[:, :3])  # version, worker, objective
    assert np.array_equal(of, ol) and np.array_equal(Cf, Cl) and np.array_equal(ff, fl)
    assert free.best_worker == lock.best_worker and free.full_objective == lock.full_objective
    for w in range(W):
        assert np.array_equal(free.traces[w][:, 1], lock.traces[w][:, 1])


def _check_invariants(r, smp, tw, ow, W):
    pubs = r.publications
    assert r.total_samples == int(smp.sum()) and np.all(smp > 0)
    assert np.array_equal(pubs[:, 0], np.arange(1, len(pubs) + 1))  # versions in lock order
    assert np.all(np.diff(pubs[:, 2]) < 0)  # strict improvement (engine.hpp:131)
    for ver, w, f, ts in pubs:  # every published incumbent is an accepted step of that worker
        tr = r.traces[int(w)]
        assert f in tr[:, 1]
        assert 0 < ts <= r.wall_seconds
    for w in range(W):
        tr = r.traces[w]
        assert len(tr) and np.all(np.diff(tr[:, 0]) > 0) and np.all(np.diff(tr[:, 1]) < 0)
        assert tr[-1, 1] == ow[w] and tr[-1, 0] <= tw[w]
    assert r.best_worker == int(np.argmin(ow)) and r.best_sample_objective == ow.min()


def test_free_cooperative_immediate_publication():
    X = mixture(60000, 8, 8, seed=23)
    W = 12
    cfg = hp.EngineConfig(k=8, sample_size=6000, n_workers=W, strategy="cooperative", master_seed=3, rng="philox",
                          time_limit=0.25, free_running=True, free_group=1)
    r, smp, tw, Cw, fw, ow = run_engine(X, cfg)
    assert r.wall_seconds >= 0.25
    _check_invariants(r, smp, tw, ow, W)
    pubs = r.publications
    assert len(pubs) >= 1
    # cooperative: the final shared best is the best accepted cooperative step, i.e. the global best
    assert pubs[-1, 2] == ow.min() and int(pubs[-1, 1]) == r.best_worker
    # immediate publication: workers started steps from incumbents published while other workers were
    # still on an earlier sample -- publication times are spread over the run, not bunched at lap ends,
    # and every worker's clock stopped near the limit (a step may end shortly after it)
    assert np.all(tw < 0.25 + 0.1) and np.all(tw > 0.1)
    _, _, cost, _ = orc().assign(X, r.centroids, r.degenerate)
    assert abs(r.full_objective - cost) <= 1e-12 * cost


def test_free_hybrid_enters_with_phase1_incumbents():
    X = mixture(60000, 8, 8, seed=24)
    W = 6
    cfg = hp.EngineConfig(k=8, sample_size=6000, n_workers=W, strategy="hybrid", phase_t1=0.12, phase_t2=0.18,
                          master_seed=4, rng="philox", time_limit=0.3, free_running=True, free_group=W)
    r, smp, tw, Cw, fw, ow = run_engine(X, cfg)
    _check_invariants(r, smp, tw, ow, W)
    pubs = r.publications
    assert len(pubs) >= 1 and np.all(pubs[:, 3] >= 0.12)  # nothing is published in the competitive phase
    # engine.hpp:359-364: a worker entering the cooperative phase first publishes its phase-1 incumbent.
    # Nothing can be published before the first entry, so the first record is an entry record: the
    # entering worker's last accepted objective before its entry clock (each worker reads its own clock,
    # so the workers of a group may enter in different prepare steps when t1 falls between two readings)
    a, t_c = int(pubs[0, 1]), pubs[0, 3]
    before = r.traces[a][r.traces[a][:, 0] < t_c]
    assert len(before) and pubs[0, 2] == before[-1, 1]
    # every worker had a finite phase-1 incumbent, and the best of them was published or beaten at once
    phase1 = [tr[tr[:, 0] < 0.12][-1, 1] for tr in r.traces]
    assert len(phase1) == W and pubs[:, 2].min() <= min(phase1)
    assert pubs[-1, 2] == ow.min()


def test_free_validation():
    X = mixture(4000, 2, 3, seed=1)
    kw = dict(k=3, sample_size=200, n_workers=2)
    with pytest.raises(hp.InvalidArgument, match="needs a time limit"):
        run_engine(X, hp.EngineConfig(max_samples=2, rng="philox", free_running=True, **kw))
    with pytest.raises(hp.Unsupported, match="rng_mode must be philox"):
        run_engine(X, hp.EngineConfig(time_limit=0.1, rng="reference", free_running=True, **kw))
    Xw = mixture(4000, 40, 3, seed=2)  # n = 40: the grid-wide path, no cluster-resident geometry
    with pytest.raises(hp.Unsupported, match="cluster-resident"):
        run_engine(Xw, hp.EngineConfig(time_limit=0.1, rng="philox", free_running=True, **kw))


def test_free_engine_reset_and_rerun():
    # hpcg_engine_reset returns a free-running engine to sample 0: the capped competitive schedule is
    # deterministic, so the second run reproduces the first; a new seed gives a different run
    X = mixture(30000, 4, 6, seed=25)
    cfg = hp.EngineConfig(k=6, sample_size=3000, n_workers=5, strategy="competitive", master_seed=9, rng="philox",
                          max_samples=4, time_limit=1e6, free_running=True, free_group=2)
    ds = hp.DeviceDataset(X)
    eng = hp.Engine(ds, cfg)
    try:
        eng.run()
        r1 = eng.finish()
        o1 = eng.worker_incumbents()[2].copy()
        with pytest.raises(hp.InvalidArgument, match="already run"):
            eng.run()
        eng.reset(9)
        eng.run()
        r2 = eng.finish()
        o2 = eng.worker_incumbents()[2].copy()
        eng.reset(10)
        eng.run()
        o3 = eng.worker_incumbents()[2].copy()
    finally:
        eng.close()
        ds.close()
    assert np.array_equal(o1, o2) and r1.distance_evals == r2.distance_evals and r1.total_samples == r2.total_samples == 20
    assert np.array_equal(r1.centroids, r2.centroids) and r1.full_objective == r2.full_objective
    assert not np.array_equal(o1, o3)


def test_free_config2_scale_many_groups():
    # the benchmark shape's worker count (256 workers, s = 20,000, k = 10, n = 16) on 16 streams: default
    # grouping, cooperative; every worker keeps stepping, publications keep improving, nothing stalls
    rs = np.random.default_rng(26)
    means = rs.uniform(-10, 10, (10, 16))
    X = (means[rs.integers(0, 10, 1_000_000)] + rs.standard_normal((1_000_000, 16))).astype(np.float32)
    W = 256
    cfg = hp.EngineConfig(k=10, sample_size=20000, n_workers=W, strategy="cooperative", master_seed=6, rng="philox",
                          time_limit=0.2, free_running=True)
    r, smp, tw, Cw, fw, ow = run_engine(X, cfg)
    _check_invariants(r, smp, tw, ow, W)
    assert smp.min() >= 20 and smp.max() - smp.min() <= 0.5 * smp.max()  # ~1 ms per lap of 256 workers
    assert len(r.publications) >= 1 and r.publications[-1, 2] == ow.min()
    assert 0.2 <= r.wall_seconds < 1.5
