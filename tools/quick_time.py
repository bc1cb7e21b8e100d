"""Quick timing of one cooperative round at config-2 shape (dev tool, not the bench)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import paper_2311_04517_b200 as hp

m, n, k, s, W = 10_000_000, 16, 10, 20000, 256
rs = np.random.default_rng(0)
means = rs.uniform(-10, 10, (10, n)); sig = rs.uniform(0.5, 2, 10)
wts = 1.0 / np.arange(1, 11) ** 1.1
t = time.time(); X = hp.gen_mixture(m, n, means, sig, wts, seed=1, dtype=np.float32); print("gen", time.time() - t)
Xt = torch.from_numpy(X).cuda()
ctx = hp.default_context()
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
ds = hp.DeviceDataset.from_torch(Xt, ctx)
cfg = hp.EngineConfig(k=k, sample_size=s, n_workers=W, max_samples=20, strategy="cooperative", rng="philox")
eng = hp.Engine(ds, cfg)
for r in range(6):
    nd0 = eng.distance_evals()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    eng.rounds(1)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    nd = eng.distance_evals() - nd0
    print(f"round {r}: {dt*1e3:.2f} ms  n_d {nd:.3e}  {nd/dt:.3e} evals/s  ({nd*16/dt/1e12:.2f} TFMA/s)")
res = eng.finish()
print("full objective", res.full_objective, "best", res.best_worker)
C_ = torch.from_numpy(res.centroids).cuda()
cost = torch.zeros(1, dtype=torch.float64, device="cuda")
import ctypes
lib = hp._lib.lib
for i in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    hp._lib.check(lib.hpcg_assign_dev(ctx.h, ds.h, ctypes.c_void_p(C_.data_ptr()), k, None, ctypes.c_void_p(cost.data_ptr())))
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(f"objective pass {dt*1e3:.3f} ms  {m*n*4/dt/1e9:.1f} GB/s")
