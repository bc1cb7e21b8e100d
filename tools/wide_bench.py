"""Dev tool: BASELINE config 4 shape (n=128, k=25, s=1e5) through the grid-wide path: per-round
timing of the engine on a device-resident X (philox streams)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import paper_2311_04517_b200 as hp
m = int(float(sys.argv[1])) if len(sys.argv) > 1 else 5_000_000
W = int(sys.argv[2]) if len(sys.argv) > 2 else 16
rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 3
k, n, s = 25, 128, 100_000
rs = np.random.default_rng(4)
t0 = time.perf_counter()
X = hp.gen_mixture(m, n, rs.normal(0.0, 2.0, (k, n)), np.ones(k), np.ones(k) / k, seed=2)
print(f"gen {time.perf_counter()-t0:.1f}s", flush=True)
ds = hp.DeviceDataset(X)
eng = hp.Engine(ds, hp.EngineConfig(k=k, sample_size=s, n_workers=W, max_samples=rounds, strategy="cooperative",
                                     rng="philox"))
ds.ctx.enable_timing(True)
for r in range(rounds):
    nd0 = eng.distance_evals()
    t0 = time.perf_counter()
    eng.rounds(1)
    ds.ctx.synchronize()
    dt = time.perf_counter() - t0
    nd = eng.distance_evals() - nd0
    print(f"round {r}: {dt*1e3:.1f} ms, n_d {nd:.3e} -> {nd/dt:.3e} evals/s", flush=True)
t0 = time.perf_counter()
res = eng.finish()
print(f"finish (f(C,X) over m={m}): {(time.perf_counter()-t0)*1e3:.1f} ms, f={res.full_objective:.6e}")
