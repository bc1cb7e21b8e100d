"""Dev tool: DRAM bytes of the sample gather under different L2 fetch granularities
(cudaLimitMaxL2FetchGranularity = 32 / 64 / 128 B; set through torch's cudart on the primary context
libhpcg shares). Run under ncu:  ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum -k regex:sample_gather
python tools/gather_fetch.py <bytes|0>   (0 = leave the default)"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2311_04517_b200 as hp  # noqa: E402

gran = int(sys.argv[1]) if len(sys.argv) > 1 else 0
torch.cuda.init()
rt = ctypes.CDLL("libcudart.so.12")
cur = ctypes.c_size_t()
rt.cudaDeviceGetLimit(ctypes.byref(cur), 0x05)
print("default fetch granularity", cur.value)
if gran:
    rc = rt.cudaDeviceSetLimit(0x05, ctypes.c_size_t(gran))
    rt.cudaDeviceGetLimit(ctypes.byref(cur), 0x05)
    print("set", gran, "rc", rc, "now", cur.value)
M, N, W, S = 10_000_000, 16, 256, 20000
Xd = torch.randn(M, N, device="cuda")
ctx = hp.default_context()
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
ds = hp.DeviceDataset.from_torch(Xd, ctx)
Sd = torch.empty(W * S * N, dtype=torch.float32, device="cuda")
for i in range(4):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    hp._lib.check(hp._lib.lib.hpcg_sample_gather_dev(ctx.h, ds.h, W, S, 1234, 100 + i, 0, Sd.data_ptr()))
    e1.record()
    torch.cuda.synchronize()
    print("gather ms", e0.elapsed_time(e1))
