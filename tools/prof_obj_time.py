"""Dev tool: median time of the config-2 f(C,X) pass (1e7 x 16 fp32, k = 10, converged-like centres)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import bench
import paper_2311_04517_b200 as hp

X = torch.from_numpy(bench.make_data(0)).cuda()
ctx = hp.Context(0)
st = torch.cuda.current_stream()
ctx.set_stream(st.cuda_stream)
ds = hp.DeviceDataset.from_torch(X, ctx)
means, _, _ = bench.mixture_params()
C = torch.from_numpy(np.ascontiguousarray(means)).cuda()
cost = torch.zeros(1, dtype=torch.float64, device="cuda")
ts = []
for i in range(12):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    hp._lib.check(hp._lib.lib.hpcg_assign_dev(ctx.h, ds.h, C.data_ptr(), 10, None, cost.data_ptr()))
    b.record(st)
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
t = float(np.median(ts[3:]))
print(f"config 2: f(C,X) {t:.4f} ms {640e6 / t / 1e6:.0f} GB/s cost {float(cost.item()):.6e}")
