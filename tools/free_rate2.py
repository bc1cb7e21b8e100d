"""Dev tool: free-running sample rates for small worker counts / strategies (chain latency per sample)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2311_04517_b200 as hp  # noqa: E402
X = bench.make_data(0)
Xd = torch.from_numpy(X).to("cuda")
ctx = hp.Context(0)
ds = hp.DeviceDataset.from_torch(Xd, ctx)
for W, strat, kw in [(15, "cooperative", {}), (15, "cooperative", dict(free_running=True, free_group=1)),
                     (15, "competitive", dict(free_running=True, free_group=1)),
                     (30, "cooperative", dict(free_running=True, free_group=1)),
                     (30, "cooperative", dict(free_running=True, free_group=2)),
                     (60, "cooperative", dict(free_running=True, free_group=4)),
                     (256, "competitive", {}), (256, "competitive", dict(free_running=True, free_group=16))]:
    cfg = hp.EngineConfig(k=bench.K, sample_size=bench.S, n_workers=W, strategy=strat, rng="philox", time_limit=0.4,
                          master_seed=3, **kw)
    eng = hp.Engine(ds, cfg)
    eng.run()
    r = eng.finish()
    smp, tw = eng.worker_progress()
    print(f"W {W:3d} {strat:12s} {str(kw):50s} samples/s {r.total_samples / max(tw.max(), 1e-9):9.0f} "
          f"us per sample per worker {1e6 * tw.max() / smp.max():7.1f}")
    eng.close()
