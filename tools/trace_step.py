"""Dev tool: per-CTA phase timeline of one config-2 round (ns)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_2311_04517_b200 as hp
rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 2
mode = int(sys.argv[2]) if len(sys.argv) > 2 else 0
m, n, k, s, W = 10_000_000, 16, 10, 20000, 256
rs = np.random.default_rng(0)
X = hp.gen_mixture(m, n, rs.uniform(-10, 10, (10, n)), rs.uniform(0.5, 2, 10), 1.0 / np.arange(1, 11) ** 1.1, seed=1)
ds = hp.DeviceDataset(X)
eng = hp.Engine(ds, hp.EngineConfig(k=k, sample_size=s, n_workers=W, max_samples=rounds, strategy="cooperative", rng="philox"))
C = 16
tr = torch.zeros(W * C * 16, dtype=torch.int64, device="cuda")
for r in range(rounds):
    tr.zero_()
    hp._lib.lib.hpcg_engine_set_trace(eng.h, tr.data_ptr(), mode)
    eng.rounds(1); ds.ctx.synchronize()
    t = tr.view(W * C, 16).cpu().numpy().astype(np.float64)
    t0 = t[:, 0][t[:, 0] > 0].min()
    names = (["start", "issued", "landed", "csync", "seeded", "prep", "assign", "sort", "update", "ctapart", "xsync",
              "xreduce", "means"] if mode == 0 else
             ["start", "issued", "landed", "csync", "seeded", "cdf", "cdfx", "search", "hitx", "fetch", "costs",
              "costx", "slot1"])
    print(f"round {r}: kernel span {(t[:,15].max()-t0)/1e3:.1f} us")
    rel = t - t[:, :1]
    for i, nm in enumerate(names):
        v = rel[:, i][t[:, i] > 0]
        if len(v): print(f"  {nm:7s} median {np.median(v)/1e3:8.2f} us  p90 {np.percentile(v,90)/1e3:8.2f}")
    v = (t[:, 15] - t[:, 0]); print(f"  life    median {np.median(v)/1e3:8.2f} us  p90 {np.percentile(v,90)/1e3:8.2f}")
    starts = np.sort(t[:, 0] - t0) / 1e3
    print("  CTA start times (us) percentiles 10/50/90/100:", np.percentile(starts, [10, 50, 90, 100]).round(1))
