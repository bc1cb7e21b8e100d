"""Dev tool: where the e2e (host data) config-2 run spends its time: upload (alloc + H2D), engine
create, rounds, finish, teardown."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch, ctypes as C
import paper_2311_04517_b200 as hp
from paper_2311_04517_b200 import _lib
import bench
X = bench.make_data(0)
Xp = torch.from_numpy(X).pin_memory().numpy()
ctx = hp.default_context()
cfg = hp.EngineConfig(k=10, sample_size=20000, n_workers=256, max_samples=4, strategy="cooperative", rng="philox")
lib = _lib.lib
for rep in range(4):
    t = [time.perf_counter()]
    ds = C.c_void_p()
    _lib.check(lib.hpcg_dataset_upload(ctx.h, Xp.ctypes.data, 0, X.shape[0], X.shape[1], C.byref(ds)))
    t.append(time.perf_counter())
    e = C.c_void_p()
    c = cfg.to_c()
    _lib.check(lib.hpcg_engine_create(ctx.h, ds, C.byref(c), C.byref(e)))
    torch.cuda.synchronize(); t.append(time.perf_counter())
    _lib.check(lib.hpcg_engine_run(e))
    torch.cuda.synchronize(); t.append(time.perf_counter())
    out = _lib.RunOut()
    cent = np.empty((10, 16)); fl = np.empty(10, np.uint8)
    _lib.check(lib.hpcg_engine_finish(e, C.byref(out), cent.ctypes.data, fl.ctypes.data, None, None, 0, None, None, 0, None))
    t.append(time.perf_counter())
    lib.hpcg_engine_destroy(e); lib.hpcg_dataset_destroy(ds)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    d = np.diff(t) * 1e3
    print(f"upload {d[0]:.2f} ms ({X.nbytes/d[0]/1e6:.1f} GB/s)  create {d[1]:.2f}  rounds {d[2]:.2f}  finish {d[3]:.2f}  teardown {d[4]:.2f}  total {sum(d):.2f}")
