import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch, ctypes
import os
import paper_2311_04517_b200 as hp
MU = np.random.default_rng(0).uniform(-10,10,(10,16))
X = hp.gen_mixture(10_000_000, 16, MU, np.ones(10), seed=1)
Xd = torch.from_numpy(X).cuda()
st = torch.cuda.current_stream()
ctx = hp.Context(0); ctx.set_stream(st.cuda_stream)
ds = hp.DeviceDataset.from_torch(Xd, ctx)
CH = MU if "--means" in sys.argv else X[:10].astype(np.float64)
C = torch.from_numpy(CH).cuda()
cost = torch.zeros(1, dtype=torch.float64, device="cuda")
ts = []
for i in range(20):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    e0.record(st)
    rc = hp._lib.lib.hpcg_assign_dev(ctx.h, ds.h, C.data_ptr(), 10, None, cost.data_ptr())
    e1.record(st)
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(rc, "events min", min(ts), "median", sorted(ts)[10], "cost", cost.item())
print("host path", hp.mssc_objective(CH, ds))
