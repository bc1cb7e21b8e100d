"""Wall-clock schedule (engine.hpp:348-374 run_wall_clock) through the
C-ABI hpcg_engine_run: rounds until cfg.time_limit seconds, every worker of a round starting from
the round's snapshot, accepted cooperative incumbents published at the round end in worker-id
order, the hybrid switch at the first round end past phase_t1 seconds, timestamps in seconds.

With a time limit that cannot bind and a max_samples cap the schedule runs exactly the lockstep
rounds, so everything but the clock-valued fields must equal the lockstep run (and hence the
oracle); with a binding limit the run must stop at the first round end past it.
"""
import numpy as np
import pytest

import paper_2311_04517_b200 as hp
from oracle_py import orc

pytestmark = pytest.mark.gpu

RTOL = 1e-12


def mixture(m, n, comps, seed):
    rs = np.random.default_rng(seed)
    means = rs.uniform(-10, 10, (comps, n))
    return means[rs.integers(0, comps, m)] + rs.standard_normal((m, n))


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300))) if a.size else 0.0


@pytest.mark.parametrize("strategy", ["competitive", "cooperative"])
def test_wall_schedule_with_cap_equals_lockstep(strategy):
    X = mixture(6000, 2, 5, seed=17)
    base = dict(k=5, sample_size=800, n_workers=3, strategy=strategy, master_seed=42, rng="reference")
    lock = hp.run(X, hp.EngineConfig(max_samples=5, **base))
    wall = hp.run(X, hp.EngineConfig(max_samples=5, time_limit=1e6, **base))
    e = orc().run(X, k=5, sample_size=800, n_workers=3, max_samples=5, strategy=strategy, t1=0.0, t2=0.0, seed=42)
    assert wall.total_samples == lock.total_samples == e["total_samples"]
    assert wall.distance_evals == lock.distance_evals == e["distance_evals"]
    assert wall.best_worker == lock.best_worker == e["best_worker"]
    assert np.array_equal(wall.centroids, lock.centroids)
    assert wall.full_objective == lock.full_objective
    assert rel(wall.full_objective, e["full_objective"]) <= RTOL
    assert np.array_equal(wall.publications[:, [0, 1, 2]], lock.publications[:, [0, 1, 2]])
    for w in range(3):  # same acceptances and objectives; timestamps are seconds, increasing
        assert np.array_equal(wall.traces[w][:, 1], lock.traces[w][:, 1])
        ts = wall.traces[w][:, 0]
        assert np.all(np.diff(ts) > 0) and np.all(ts > 0) and np.all(ts <= wall.wall_seconds)
    if len(wall.publications):
        assert np.all(np.diff(wall.publications[:, 3]) >= 0)


@pytest.mark.parametrize("strategy", ["competitive", "cooperative"])
def test_wall_schedule_stops_at_the_time_limit(strategy):
    X = mixture(20000, 4, 6, seed=3)
    cfg = hp.EngineConfig(k=6, sample_size=2000, n_workers=8, strategy=strategy, time_limit=0.25, rng="philox")
    r = hp.run(X, cfg)
    assert r.wall_seconds >= 0.25
    assert r.total_samples > 0 and r.total_samples % 8 == 0  # whole rounds of 8 workers
    rounds = r.total_samples // 8
    assert rounds >= 2
    last = max(t[-1, 0] for t in r.traces if len(t))
    assert last <= r.wall_seconds
    assert r.clustering_time == min(t[-1, 0] for t in r.traces if len(t))
    # f(C, X) of the winner against the oracle
    _, _, cost, _ = orc().assign(X, r.centroids, r.degenerate)
    assert rel(r.full_objective, cost) <= RTOL
    # select_best: the winner has the lowest incumbent objective, ties to the lowest id
    assert r.best_worker == int(np.argmin(r.worker_objectives))


def test_wall_hybrid_switches_after_t1_seconds():
    X = mixture(20000, 4, 6, seed=5)
    cfg = hp.EngineConfig(k=6, sample_size=2000, n_workers=6, strategy="hybrid", phase_t1=0.15, phase_t2=0.15,
                          time_limit=0.3, rng="philox")
    r = hp.run(X, cfg)
    pubs = r.publications
    assert len(pubs) >= 1
    # nothing is published during the competitive phase (before t1 seconds)
    assert np.all(pubs[:, 3] >= 0.15)
    assert np.all(np.diff(pubs[:, 0]) > 0) and np.all(np.diff(pubs[:, 2]) < 0)  # versions up, objective down


def test_wall_hybrid_carry_over_publishes_phase1_incumbents():
    """engine.hpp:353-364: one clock reading at the top of the first cooperative round both flips the
    phase and publishes every finite phase-1 incumbent (worker-id order, strict <) before the round
    draws its inits; so the carry-over records share that reading as timestamp and the last of them
    is the minimum over the workers' phase-1 incumbents."""
    X = mixture(20000, 4, 6, seed=7)
    cfg = hp.EngineConfig(k=6, sample_size=2000, n_workers=6, strategy="hybrid", phase_t1=0.12, phase_t2=0.18,
                          time_limit=0.3, rng="philox")
    r = hp.run(X, cfg)
    pubs = r.publications
    assert len(pubs) >= 1
    t_c = pubs[0, 3]
    carry = pubs[pubs[:, 3] == t_c]
    phase1 = [tr[tr[:, 0] < t_c][-1, 1] for tr in r.traces if len(tr) and np.any(tr[:, 0] < t_c)]
    assert len(phase1) == 6  # every worker finished a competitive round before the switch
    assert carry[-1, 2] == min(phase1)
    # the carried records are the strict prefix minima in worker-id order
    run_min, expect = np.inf, []
    for w, tr in enumerate(r.traces):
        f = tr[tr[:, 0] < t_c][-1, 1]
        if f < run_min:
            run_min = f
            expect.append((w, f))
    assert [(int(a), b) for a, b in carry[:, [1, 2]]] == expect
    # versions 1..len(carry) and later publications strictly improve on the carried best
    assert np.array_equal(carry[:, 0], np.arange(1, len(carry) + 1))
    assert np.all(pubs[len(carry):, 2] < carry[-1, 2])


def test_wall_schedule_validation():
    X = mixture(2000, 2, 3, seed=1)
    with pytest.raises(hp.InvalidArgument, match="time limit must be positive"):
        hp.run(X, hp.EngineConfig(k=3, sample_size=100, n_workers=2, max_samples=2, time_limit=-1.0))
    with pytest.raises(hp.InvalidArgument, match="need a time limit or a max_samples bound"):
        hp.run(X, hp.EngineConfig(k=3, sample_size=100, n_workers=2, max_samples=0))
    with pytest.raises(hp.InvalidArgument, match="hybrid phases must sum to the total budget"):
        hp.run(X, hp.EngineConfig(k=3, sample_size=100, n_workers=2, strategy="hybrid", phase_t1=0.1,
                                  phase_t2=0.1, time_limit=0.5))
