"""Dev tool: BASELINE config-5 shard shape (2.5e8 x 8 fp32, k=15, s=2e5, 256 workers) through the
grid-wide path: round timings (argv[1] = rows, default 2.5e8; argv[2] = rounds)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_2311_04517_b200 as hp
m = int(float(sys.argv[1])) if len(sys.argv) > 1 else 250_000_000
R = int(sys.argv[2]) if len(sys.argv) > 2 else 2
rs = np.random.default_rng(2316)
X = hp.gen_mixture(m, 8, rs.uniform(-20, 20, (15, 8)), rs.uniform(0.5, 3.0, 15), rs.dirichlet(np.ones(15)), seed=5)
st = torch.cuda.current_stream(); ctx = hp.Context(0); ctx.set_stream(st.cuda_stream)
Xd = torch.from_numpy(X).cuda(); del X
ds = hp.DeviceDataset.from_torch(Xd, ctx)
eng = hp.Engine(ds, hp.EngineConfig(k=15, sample_size=200_000, n_workers=256, max_samples=R, strategy="cooperative", rng="philox"))
for r in range(R):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    eng.rounds(1); torch.cuda.synchronize()
    print(f"round {r}: {(time.perf_counter()-t0)*1e3:.1f} ms", flush=True)
