"""Dev tool for ncu: config-2 cooperative engine, R rounds; prints geometry & timings."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import paper_2311_04517_b200 as hp

rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 3
W = int(sys.argv[2]) if len(sys.argv) > 2 else 256
m, n, k, s = 10_000_000, 16, 10, 20000
rs = np.random.default_rng(0)
X = hp.gen_mixture(m, n, rs.uniform(-10, 10, (10, n)), rs.uniform(0.5, 2, 10), 1.0 / np.arange(1, 11) ** 1.1,
                   seed=1, dtype=np.float32)
ds = hp.DeviceDataset(X)
eng = hp.Engine(ds, hp.EngineConfig(k=k, sample_size=s, n_workers=W, max_samples=rounds, strategy="cooperative",
                                     rng="philox"))
ds.ctx.enable_timing(True)
for r in range(rounds):
    nd0 = eng.distance_evals()
    t0 = time.perf_counter()
    eng.rounds(1)
    nd = eng.distance_evals() - nd0
    print(f"round {r}: {1e3*(time.perf_counter()-t0):.2f} ms wall, n_d {nd:.3e}", ds.ctx.kernel_times())
