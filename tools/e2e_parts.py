"""Dev tool: where the one-call run's time goes on pinned host data (config 2): upload, engine create, rounds,
finish, destroy, against hpcg_run as a whole."""
import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
import bench
import paper_2311_04517_b200 as hp

X = torch.from_numpy(bench.make_data(0)).pin_memory().numpy()
ctx = hp.Context(0)
cfg = hp.EngineConfig(k=bench.K, sample_size=bench.S, n_workers=bench.W_PER_GPU, max_samples=bench.ROUNDS,
                      strategy="cooperative", rng="philox")
def parts():
    t = [time.perf_counter()]
    ds = hp.DeviceDataset(X, ctx=ctx); t.append(time.perf_counter())
    eng = hp.Engine(ds, cfg); ctx.synchronize(); t.append(time.perf_counter())
    eng.rounds(bench.ROUNDS); ctx.synchronize(); t.append(time.perf_counter())
    eng.finish(); t.append(time.perf_counter())
    eng.close(); t.append(time.perf_counter())
    ds.close(); t.append(time.perf_counter())
    return np.diff(t) * 1e3
for _ in range(3): parts()
p = np.median([parts() for _ in range(7)], axis=0)
print("upload %.3f  create %.3f  rounds %.3f  finish %.3f  engine destroy %.3f  dataset destroy %.3f  sum %.3f ms" % (*p, p.sum()))
def whole():
    t0 = time.perf_counter(); hp.run(X, cfg, ctx=ctx); return (time.perf_counter() - t0) * 1e3
for _ in range(3): whole()
print("hpcg_run %.3f ms" % np.median([whole() for _ in range(7)]))
