"""Dev tool (ncu target / timing): the f(C,X) pass of BASELINE config c (3, 4 or 5 shard) with the
mixture's own means as centres; prints the median pass time and GB/s. usage: prof_cfg_obj.py c [reps]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import bench
import paper_2311_04517_b200 as hp

c = int(sys.argv[1])
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 8
X = bench.cfg_data(hp, c)
m, n = X.shape
k = bench.CFG_SETUP[c][0]
Xd = torch.from_numpy(X).cuda()
del X
ctx = hp.Context(0)
st = torch.cuda.current_stream()
ctx.set_stream(st.cuda_stream)
ds = hp.DeviceDataset.from_torch(Xd, ctx)
# converged centres, as the bench's pass sees them: a short engine run of the config
_, s_, W_, _, strat, t1, t2, _ = bench.CFG_SETUP[c]
eng = hp.Engine(ds, hp.EngineConfig(k=k, sample_size=s_, n_workers=W_, max_samples=2, strategy="cooperative",
                                    rng="philox"))
eng.run()
res = eng.finish()
Cn = np.ascontiguousarray(res.centroids[res.degenerate == 0])
k = Cn.shape[0]
eng.close()
C = torch.from_numpy(Cn).cuda()
cost = torch.zeros(1, dtype=torch.float64, device="cuda")
ts = []
for i in range(reps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    hp._lib.check(hp._lib.lib.hpcg_assign_dev(ctx.h, ds.h, C.data_ptr(), k, None, cost.data_ptr()))
    b.record(st)
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
t = float(np.median(ts[2:] if reps > 3 else ts))
nb = m * n * Xd.element_size()
print(f"config {c}: m {m} n {n} k {k} {Xd.dtype}: f(C,X) {t:.4f} ms {nb / t / 1e6:.0f} GB/s cost {float(cost.item()):.6e}")
