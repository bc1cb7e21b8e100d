"""Dev tool: samples/s of the wall-clock schedules on the config-2 shape (256 workers, cooperative, 0.5 s):
round granularity vs free-running groups of 16 / 4 / 1 workers."""
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
import os
groups = [int(g) for g in os.environ.get("GROUPS", "16,4,1").split(",")]
for name, kw in [("round-granular", {})] + [(f"free, groups of {g}", dict(free_running=True, free_group=g)) for g in groups]:
    cfg = hp.EngineConfig(k=bench.K, sample_size=bench.S, n_workers=bench.W_PER_GPU, strategy="cooperative",
                          rng="philox", time_limit=0.5, master_seed=3, **kw)
    eng = hp.Engine(ds, cfg)
    eng.run()
    r = eng.finish()
    smp, tw = eng.worker_progress()
    print(f"{name:22s} samples {r.total_samples:7d}  samples/s {r.total_samples / max(tw.max(), 1e-9):10.0f}  "
          f"per worker {smp.min()}..{smp.max()}  publications {len(r.publications):4d}  "
          f"best sample objective {r.best_sample_objective:.6e}  f(C,X) {r.full_objective:.6e}")
    eng.close()
