import sys, time, numpy as np, torch
sys.path.insert(0, ".")
import bench, paper_2311_04517_b200 as hp
X = bench.make_data(0)
dev = torch.device("cuda", 0)
Xd = torch.from_numpy(X).to(dev)
st = torch.cuda.current_stream(dev)
ctx = hp.Context(0); ctx.set_stream(st.cuda_stream)
ds = hp.DeviceDataset.from_torch(Xd, ctx)
cfg = hp.EngineConfig(k=bench.K, sample_size=bench.S, n_workers=bench.W_PER_GPU, max_samples=bench.ROUNDS, strategy="cooperative", rng="philox")
eng = hp.Engine(ds, cfg)
def t(fn, n=20):
    for i in range(3): fn(i)
    torch.cuda.synchronize(); e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); e0.record(st)
    for i in range(n): fn(100 + i)
    e1.record(st); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n, (time.perf_counter() - t0) * 1e3 / n
def full(i): eng.reset(i); eng.rounds(bench.ROUNDS); return eng.finish()
def full_nd(i): r = full(i); eng.distance_evals(); return r
def nofinish(i): eng.reset(i); eng.rounds(bench.ROUNDS)
print("reset+rounds+finish (ev ms, wall ms):", t(full))
print("  + distance_evals:", t(full_nd))
print("reset+rounds only:", t(nofinish))
ctx.enable_timing(True)
print("with kernel timing on, full_nd:", t(full_nd))
