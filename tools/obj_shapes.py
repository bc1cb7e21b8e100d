"""Dev tool: f(C,X) kernel time on several fp32 shapes (640 MB of X each), median of 10 launches.
Run twice (HPCG_OBJ_NO_TC=1 for the FFMA2 centre-pair kernel) to compare the kernels."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_2311_04517_b200 as hp
st = torch.cuda.current_stream()
ctx = hp.Context(0); ctx.set_stream(st.cuda_stream)
for n, k in [(16, 10), (16, 16), (16, 25), (8, 15), (8, 5), (32, 25), (32, 10)]:
    m = 160_000_000 // n
    rs = np.random.default_rng(n * 100 + k)
    MU = rs.uniform(-10, 10, (k, n))
    X = hp.gen_mixture(m, n, MU, np.ones(k), seed=1)
    Xd = torch.from_numpy(X).cuda()
    ds = hp.DeviceDataset.from_torch(Xd, ctx)
    C = torch.from_numpy(MU).cuda()
    cost = torch.zeros(1, dtype=torch.float64, device="cuda")
    ts = []
    for i in range(13):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        hp._lib.check(hp._lib.lib.hpcg_assign_dev(ctx.h, ds.h, C.data_ptr(), k, None, cost.data_ptr()))
        e1.record(st)
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(e0.elapsed_time(e1))
    ms = float(np.median(ts))
    print(f"n={n:3d} k={k:3d} m={m}: {ms*1e3:8.1f} us  {m*n*4/ms/1e6:7.0f} GB/s  cost={cost.item():.6e}", flush=True)
    del ds, Xd
