"""BASELINE.json configs 1, 3, 4 and 5 on ONE GPU through the engine (the bench line itself is
config 2, bench.py). Seeded synthetic data with each config's shapes and distributions (the
paper's datasets are not in the container); config 5 runs one GPU's shard of the 8-GPU job
(2.5e8 of the 2e9 rows, 256 of the 2,048 workers). Per config: whole-run time on the
device-resident X (rounds + select + full-data objective; config 3 adds the objective after every
round, as BASELINE.json asks), distance evaluations/s (reference n_d accounting), the steady
round time and the f(C,X) pass in GB/s. One JSON line per config.

usage: python tools/config_bench.py [1 3 4 5]
"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_2311_04517_b200 as hp


def gen(cfg):
    rs = np.random.default_rng(2311 + cfg)
    if cfg == 1:  # gen_blobs shape: 5 blobs, centres U[-10,10]^2, sigma 1, fp64, equal weights
        return hp.gen_mixture(100_000, 2, rs.uniform(-10, 10, (5, 2)), np.ones(5), np.ones(5) / 5, seed=0,
                              dtype=np.float64)
    if cfg == 3:  # 25 comps, U[0,255]^3, sigma 8, equal weights, 1% uniform noise in [0,255]^3, fp64
        return hp.gen_mixture(100_000_000, 3, rs.uniform(0, 255, (25, 3)), np.full(25, 8.0), np.ones(25) / 25,
                              noise_frac=0.01, noise_box=(0.0, 255.0), seed=3, dtype=np.float64)
    if cfg == 4:  # 25 comps, N(0, 4 I_128) means, sigma 1, equal weights, fp32
        return hp.gen_mixture(5_000_000, 128, rs.normal(0.0, 2.0, (25, 128)), np.ones(25), np.ones(25) / 25,
                              seed=4, dtype=np.float32)
    if cfg == 5:  # 15 comps, U[-20,20]^8, sigma U[0.5,3], Dirichlet(1) weights, fp32; one GPU's shard
        return hp.gen_mixture(250_000_000, 8, rs.uniform(-20, 20, (15, 8)), rs.uniform(0.5, 3.0, 15),
                              rs.dirichlet(np.ones(15)), seed=5, dtype=np.float32)
    raise ValueError(cfg)


SETUP = {  # k, s, workers, rounds (max_samples), strategy, t1, t2, objective each round
    1: (5, 5_000, 4, 50, "competitive", 0.0, 0.0, False),
    3: (25, 50_000, 64, 20, "hybrid", 10.0, 10.0, True),
    4: (25, 100_000, 16, 10, "collective", 0.0, 0.0, False),
    5: (15, 200_000, 256, 4, "cooperative", 0.0, 0.0, False),
}


def run(cfg):
    k, s, W, R, strat, t1, t2, obj_each = SETUP[cfg]
    t0 = time.perf_counter()
    X = gen(cfg)
    tgen = time.perf_counter() - t0
    m, n = X.shape
    st = torch.cuda.current_stream()
    ctx = hp.Context(0)
    ctx.set_stream(st.cuda_stream)
    Xd = torch.from_numpy(X).cuda()
    del X
    ds = hp.DeviceDataset.from_torch(Xd, ctx)
    ec = hp.EngineConfig(k=k, sample_size=s, n_workers=W, max_samples=R, strategy=strat, phase_t1=t1, phase_t2=t2,
                         rng="philox")
    eng = hp.Engine(ds, ec)
    cost = torch.zeros(1, dtype=torch.float64, device="cuda")

    def one_run(seed, times=None):
        eng.reset(seed)
        for r in range(R):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            eng.rounds(1)
            if obj_each:  # f(C, X) of the current shared best after every round (harness addition)
                b = eng.export_best()
                if np.isfinite(b[0]):
                    C_ = torch.from_numpy(b[2][b[3] == 0]).cuda()
                    hp._lib.check(hp._lib.lib.hpcg_assign_dev(ctx.h, ds.h, C_.data_ptr(), C_.shape[0], None,
                                                              cost.data_ptr()))
            e1.record(st)
            if times is not None:
                times.append((e0, e1))
        return eng.finish()

    one_run(1)  # warm-up (geometry caches, first-launch costs)
    torch.cuda.synchronize()
    ev = []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    res = one_run(2, ev)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    rounds_ms = [a.elapsed_time(b) for a, b in ev]
    # f(C, X) pass alone on the final centroids
    C_ = torch.from_numpy(res.centroids[res.degenerate == 0]).cuda()
    ts = []
    for i in range(8):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        hp._lib.check(hp._lib.lib.hpcg_assign_dev(ctx.h, ds.h, C_.data_ptr(), C_.shape[0], None, cost.data_ptr()))
        b.record(st)
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b))
    obj_ms = float(np.median(ts))
    nbytes = m * n * Xd.element_size()
    line = {"config": cfg, "m": m, "n": n, "k": k, "s": s, "workers": W, "rounds": R, "strategy": strat,
            "dtype": str(Xd.dtype).replace("torch.", ""), "run_ms": ms, "distance_evals": res.distance_evals,
            "evals_per_s": res.distance_evals / (ms * 1e-3), "round0_ms": rounds_ms[0],
            "steady_round_ms": float(np.median(rounds_ms[1:])) if R > 1 else None,
            "objective_ms": obj_ms, "objective_gbs": nbytes / (obj_ms * 1e-3) / 1e9,
            "full_objective": res.full_objective, "gen_s": tgen}
    print(json.dumps(line), flush=True)
    eng.close()
    ds.close()
    del Xd
    torch.cuda.empty_cache()


if __name__ == "__main__":
    for c in (sys.argv[1:] or ["1", "3", "4", "5"]):
        run(int(c))
