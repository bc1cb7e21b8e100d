import sys; sys.path.insert(0, '/root/repo')
import numpy as np, torch, paper_2311_04517_b200 as hp
rs = np.random.default_rng(2314)
MU = rs.uniform(0, 255, (25, 3))
X = hp.gen_mixture(100_000_000, 3, MU, np.full(25, 8.0), np.ones(25) / 25, noise_frac=0.01, noise_box=(0.0, 255.0), seed=3, dtype=np.float64)
st = torch.cuda.current_stream(); ctx = hp.Context(0); ctx.set_stream(st.cuda_stream)
Xd = torch.from_numpy(X).cuda(); ds = hp.DeviceDataset.from_torch(Xd, ctx)
C = torch.from_numpy(MU).cuda(); cost = torch.zeros(1, dtype=torch.float64, device="cuda")
for i in range(5):
    hp._lib.check(hp._lib.lib.hpcg_assign_dev(ctx.h, ds.h, C.data_ptr(), 25, None, cost.data_ptr()))
torch.cuda.synchronize(); print(cost.item())
