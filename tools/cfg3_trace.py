"""Dev tool: config-3 shape (1e8 x 3 fp64 would need 2.4 GB; m = 2e7 here) round timings and geometry."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_2311_04517_b200 as hp
m = int(float(sys.argv[1])) if len(sys.argv) > 1 else 20_000_000
rs = np.random.default_rng(2314)
X = hp.gen_mixture(m, 3, rs.uniform(0, 255, (25, 3)), np.full(25, 8.0), np.ones(25) / 25, noise_frac=0.01,
                   noise_box=(0.0, 255.0), seed=3, dtype=np.float64)
st = torch.cuda.current_stream(); ctx = hp.Context(0); ctx.set_stream(st.cuda_stream)
Xd = torch.from_numpy(X).cuda(); ds = hp.DeviceDataset.from_torch(Xd, ctx)
for strat, t1 in [("hybrid", 10.0), ("cooperative", 0.0), ("competitive", 0.0)]:
    eng = hp.Engine(ds, hp.EngineConfig(k=25, sample_size=50_000, n_workers=64, max_samples=20, strategy=strat,
                                        phase_t1=t1, phase_t2=20.0 - t1 if strat == "hybrid" else 0.0, rng="philox"))
    ts = []
    for r in range(20):
        nd0 = eng.distance_evals()
        torch.cuda.synchronize(); t0 = time.perf_counter()
        eng.rounds(1); torch.cuda.synchronize()
        ts.append(((time.perf_counter() - t0) * 1e3, (eng.distance_evals() - nd0) / (64 * 50_000 * 25)))
    print(strat, " ".join(f"{a:.2f}ms/{b:.1f}p" for a, b in ts))
    eng.close()
