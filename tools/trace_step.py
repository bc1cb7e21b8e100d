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
tr = torch.zeros(W * C * 32, dtype=torch.int64, device="cuda")
for r in range(rounds):
    tr.zero_()
    hp._lib.lib.hpcg_engine_set_trace(eng.h, tr.data_ptr(), mode)
    eng.rounds(1); ds.ctx.synchronize()
    t = tr.view(W * C, 32).cpu().numpy().astype(np.float64)
    t0 = t[:, 0][t[:, 0] > 0].min()
    names = (["start", "issued", "landed", "csync", "seeded", "prep", "assign", "sort", "update", "ctapart", "xsync",
              "xreduce", "means"] if mode == 0 else
             ["start", "issued", "landed", "csync", "cdf", "cdfx", "search", "hitx", "fetch", "costs",
              "costx", "slot1", "seeded"])
    print(f"round {r}: kernel span {(t[:,31].max()-t0)/1e3:.1f} us")
    rel = t - t[:, :1]
    for i, nm in enumerate(names):
        v = rel[:, i][t[:, i] > 0]
        if len(v): print(f"  {nm:7s} median {np.median(v)/1e3:8.2f} us  p90 {np.percentile(v,90)/1e3:8.2f}")
    if mode == 1:
        print(f"  exact cost passes per CTA: mean {t[:, 29].mean():.2f} max {t[:, 29].max():.0f}")
        print(f"  exact D2 rows per CTA: first centre + init {t[:, 28].mean():.0f}, first slot {t[:, 25].mean():.0f}")
    if mode == 1:  # SM-cycle stamps 16..24 (warp 0), first K-means++ slot
        nm = ["costs start", "cost pairs", "cost tail", "cost wsum", "cost xchg", "decision", "d2 screen",
              "d2 flush", "slot sync"]
        for i in range(17, 25):
            v = (t[:, i] - t[:, i - 1])[(t[:, i] > 0) & (t[:, i - 1] > 0)]
            if len(v): print(f"  {nm[i-16]:11s} median {np.median(v):8.0f} cyc")
    if mode == 0:  # SM-cycle stamps 16..21 (warp 0): gather phase
        nm = ["", "gidx+issue", "init+mbar"]
        for i in range(17, 19):
            v = (t[:, i] - t[:, i - 1])[(t[:, i] > 0) & (t[:, i - 1] > 0)]
            if len(v): print(f"  {nm[i-16]:14s} median {np.median(v):8.0f} cyc")
        v = (t[:, 16] - t[:, 26])[(t[:, 16] > 0)]
        print(f"  {'entry->gidx':14s} median {np.median(v):8.0f} cyc")
    mhz = (t[:, 27] - t[:, 26]) / np.maximum(t[:, 30] - t[:, 0], 1) * 1e3
    print(f"  SM clock over CTA life (MHz): median {np.median(mhz):.0f} min {mhz.min():.0f}")
    v = (t[:, 31] - t[:, 0]); print(f"  life    median {np.median(v)/1e3:8.2f} us  p90 {np.percentile(v,90)/1e3:8.2f}")
    starts = np.sort(t[:, 0] - t0) / 1e3
    print("  CTA start times (us) percentiles 10/50/90/100:", np.percentile(starts, [10, 50, 90, 100]).round(1))
