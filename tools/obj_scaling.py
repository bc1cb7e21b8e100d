"""Dev tool: f(C,X) pass time of the config-2 kernel against m (fixed cost a + per-row cost b)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import bench
import paper_2311_04517_b200 as hp

Xall = torch.from_numpy(bench.make_data(0, 20_000_000)).cuda()
ctx = hp.Context(0)
st = torch.cuda.current_stream()
ctx.set_stream(st.cuda_stream)
means, _, _ = bench.mixture_params()
C = torch.from_numpy(np.ascontiguousarray(means)).cuda()
cost = torch.zeros(1, dtype=torch.float64, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
res = []
for m in (1_250_000, 2_500_000, 5_000_000, 10_000_000, 20_000_000):
    X = Xall[:m]
    ds = hp.DeviceDataset.from_torch(X, ctx)
    ts = []
    for i in range(12):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        hp._lib.check(hp._lib.lib.hpcg_assign_dev(ctx.h, ds.h, C.data_ptr(), 10, None, cost.data_ptr()))
        b.record(st)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    t = float(np.median(ts[3:]))
    res.append((m, t))
    print(f"m {m:9d}: {t*1e3:8.1f} us  {m*64/t/1e6:6.0f} GB/s")
    ds.close()
(m0, t0), (m1, t1) = res[-2], res[-1]
b = (t1 - t0) / (m1 - m0)
print(f"per-row {b*1e6*1e3:.4f} ns -> {64/b/1e6:.0f} GB/s asymptotic; fixed cost {1e3*(t0 - b*m0):.1f} us")
