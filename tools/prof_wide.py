"""Dev tool (ncu target): round 0 of the grid-wide path at config-4 / config-5 shapes.
usage: python tools/prof_wide.py 4|5 [rounds]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import paper_2311_04517_b200 as hp

c = int(sys.argv[1]) if len(sys.argv) > 1 else 5
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 1
rs = np.random.default_rng(2311 + c)
if c == 4:
    X = hp.gen_mixture(5_000_000, 128, rs.normal(0.0, 2.0, (25, 128)), np.ones(25), np.ones(25) / 25, seed=4)
    cfg = hp.EngineConfig(k=25, sample_size=100_000, n_workers=16, max_samples=rounds, strategy="cooperative",
                          rng="philox")
else:
    X = hp.gen_mixture(25_000_000, 8, rs.uniform(-20, 20, (15, 8)), rs.uniform(0.5, 3.0, 15),
                       rs.dirichlet(np.ones(15)), seed=5)
    cfg = hp.EngineConfig(k=15, sample_size=200_000, n_workers=256, max_samples=rounds, strategy="cooperative",
                          rng="philox")
ds = hp.DeviceDataset(X)
eng = hp.Engine(ds, cfg)
eng.rounds(rounds)
ds.ctx.synchronize()
print("ok", eng.distance_evals())
