"""Dev tool (ncu target): the config-2 f(C,X) pass (1e7 x 16 fp32, k = 10) a few times."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import bench
import paper_2311_04517_b200 as hp

X = torch.from_numpy(bench.make_data(0)).cuda()
ctx = hp.Context(0)
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
ds = hp.DeviceDataset.from_torch(X, ctx)
means, _, _ = bench.mixture_params()
C = torch.from_numpy(np.ascontiguousarray(means)).cuda()
cost = torch.zeros(1, dtype=torch.float64, device="cuda")
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 4):
    hp._lib.check(hp._lib.lib.hpcg_assign_dev(ctx.h, ds.h, C.data_ptr(), 10, None, cost.data_ptr()))
torch.cuda.synchronize()
print("ok", float(cost.item()))
