#!/usr/bin/env python3
"""HPClust hot-path benchmark (BASELINE.json metric: point-centroid distance evaluations/s in
batched Lloyd; full-data f(C,X) GB/s).

Workload (N=1): BASELINE.json configs[1] ("config 2"): X = 10,000,000 x 16 fp32 from a
10-component Gaussian mixture (means U[-10,10]^16, sigma_c U[0.5,2], Zipf(1.1) weights;
seeded synthetic stand-in), k=10, s=20,000, 256 workers per GPU, cooperative strategy,
1,000 samples total -> max_samples=4 lockstep rounds (1,024 samples).

One STEP = one complete HPClust run of that workload on the device-resident X: 4 rounds of
{sample gather -> K-means++ reseed of degenerate slots -> Lloyd to convergence -> keep-best
-> incumbent publication} for all 256 workers, select_best, and the full-data objective
pass. value = distance evaluations of the step (the reference's n_d accounting:
core.hpp:205, seeding.hpp:38) / step time. e2e = the same run through the C-ABI's one-call
hpcg_run on HOST data (pinned), i.e. upload of X + rounds + final pass + result readback.

Multi-GPU (torchrun): weak scaling, every rank runs the same per-GPU workload (its own X
shard of 1e7 rows and 256 workers) and after every round the ranks all-gather their shared
best (objective, global worker id, centroids) over NCCL and install the global winner
(cooperative exchange).

--impl reference: the reference's own CPU implementation (oracle/_ref, built from the
reference headers) runs hpclust::run on the same rows (fp64 copy; the data generator is numpy
so this arm never loads libhpcg), n_workers = 256 (its thread-per-worker model), max_samples=4,
cooperative, on all host cores; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

M, N, K, S, W_PER_GPU, ROUNDS = 10_000_000, 16, 10, 20_000, 256, 4
METRIC = "point-centroid dist evals/s in batched Lloyd; full-data f(C,X) GB/s"
UNIT = "evals/s"
PEAKS = ROOT / "MEASURED_PEAKS.json"


def mixture_params(seed=2311):
    rs = np.random.default_rng(seed)
    means = rs.uniform(-10, 10, (10, N))
    sig = rs.uniform(0.5, 2.0, 10)
    w = 1.0 / np.arange(1, 11) ** 1.1
    return means, sig, w / w.sum()


def make_data(rank: int, m: int = M):
    """Config-2 rows of rank `rank` (numpy only, so the reference arm never loads libhpcg): component
    drawn from the Zipf(1.1) weights, then mean + sigma_c * N(0, I), fp32. Both arms call this."""
    means, sig, w = mixture_params()
    g = np.random.default_rng(1000 + rank)
    comp = g.choice(len(w), size=m, p=w)
    X = g.standard_normal((m, N), dtype=np.float32)
    X *= sig.astype(np.float32)[comp, None]
    X += means.astype(np.float32)[comp]
    return X


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region: NVML polled every 2 ms on a
    thread (the timed region can be ~20 ms, shorter than nvidia-smi's start-up), nvidia-smi -lms as
    the fallback when NVML is unavailable."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.thread = None
        self.samples = []  # (sm_mhz, max_mhz, set of reason names)
        self.source = "none"

    def _nvml_handle(self):
        import pynvml
        pynvml.nvmlInit()
        try:  # the CUDA device's PCI bus id (CUDA and NVML orderings can differ)
            import torch
            pr = torch.cuda.get_device_properties(self.device)
            bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
            return pynvml, pynvml.nvmlDeviceGetHandleByPciBusId_v2(bus)
        except Exception:
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.device)

    def _poll(self, nv, h):
        bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
        mx = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
        while not self.stop:
            try:
                sm = float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append((sm, mx, {k for k, b in bits.items() if rs & b}))
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        import threading
        self.stop = False
        try:
            nv, h = self._nvml_handle()
            self.thread = threading.Thread(target=self._poll, args=(nv, h), daemon=True)
            self.thread.start()
            self.source = "nvml (2 ms poll)"
            t0 = time.perf_counter()  # the first sample lands before the timed region starts
            while not self.samples and time.perf_counter() - t0 < 1.0:
                time.sleep(0.001)
            return self
        except Exception:
            self.thread = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.source = "nvidia-smi -lms 100"
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.stop = True
        if self.thread is not None:
            self.thread.join(timeout=1.0)
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            for ln in out.splitlines():
                f = [x.strip() for x in ln.split(",")]
                if len(f) < 9:
                    continue
                try:
                    sm, mx = float(f[1]), float(f[2])
                except ValueError:
                    continue
                self.samples.append((sm, mx, {nm for nm, v in zip(self.NAMES, f[5:9]) if v.lower().startswith("active")}))

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0,
                    "source": self.source}
        sm = [x[0] for x in self.samples]
        reasons = set().union(*[x[2] for x in self.samples])
        return {"sm_mhz": float(np.median(sm)), "sm_min_mhz": float(np.min(sm)),
                "sm_max_mhz": max(x[1] for x in self.samples), "reasons": sorted(reasons),
                "samples": len(sm), "source": self.source}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def map_global_shards(hp, ctx, Xd, world, rank, device):
    """Every rank's X shard mapped into this process (CUDA IPC; NVLink peer access on a multi-GPU
    box): the engine samples over all ranks' rows (engine.hpp:165-177), its f(C,X) covers this rank's
    shard. Returns (shards, peers) for DeviceDataset.from_shards and the later ipc_close."""
    import torch
    import torch.distributed as dist
    h = torch.tensor(list(hp.ipc_export(Xd.data_ptr())), dtype=torch.uint8, device=device)
    hs = [torch.empty_like(h) for _ in range(world)]
    dist.all_gather(hs, h)
    shards, peers = [], []
    for r in range(world):
        if r == rank:
            shards.append((Xd.data_ptr(), Xd.shape[0], N, np.float32))
        else:
            hb = bytes(hs[r].cpu().tolist())
            p = hp.ipc_open(hb, ctx)
            peers.append((p, hb))
            shards.append((p, Xd.shape[0], N, np.float32))
    return shards, peers


EXCHANGE = {"mode": "nccl", "allgather": None}  # how the engines exchange (set by attach_nccl)


def attach_nccl(hp, ctx, world, rank, device):
    """The library's own NCCL communicator (ncclCommInitRank; unique id broadcast by torch). If the
    library cannot set it up, the engines exchange through a gloo group instead (the library's host
    all-gather callback) and the bench line says so."""
    import torch
    import torch.distributed as dist
    uid = torch.tensor(list(hp.comm_unique_id()) if rank == 0 else [0] * 128, dtype=torch.uint8, device=device)
    dist.broadcast(uid, 0)
    err = None
    try:
        ctx.attach_comm(world, rank, bytes(uid.cpu().tolist()))
    except Exception as ex:  # noqa: BLE001 -- recorded in the bench line
        err = f"{type(ex).__name__}: {ex}"[:120]
    ok = torch.tensor([0 if err else 1], dtype=torch.int32, device=device)
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)  # every rank takes the same path
    if int(ok.item()) == 0:
        EXCHANGE["mode"] = f"gloo host all-gather (library NCCL unavailable: {err or 'on another rank'})"
        EXCHANGE["allgather"] = hp.gloo_allgather(dist.new_group(backend="gloo"))


def set_exchange(eng, world, rank):
    eng.set_exchange(world, rank, allgather=EXCHANGE["allgather"])


def gather_rate(hp, ctx, ds, stream, key, reps=8):
    """The sample gather alone: hpcg_sample_gather_dev (the worker step's PRP indices + 16-B row
    chunks) materialising W x s x n fp32 rows; GB/s of rows read (algorithmic) vs HBM."""
    import torch
    Sd = torch.empty(W_PER_GPU * S * N, dtype=torch.float32, device=stream.device)
    ms = []
    for i in range(3 + reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        hp._lib.check(hp._lib.lib.hpcg_sample_gather_dev(ctx.h, ds.h, W_PER_GPU, S, key, 100 + i, 0, Sd.data_ptr()))
        e1.record(stream)
        torch.cuda.synchronize()
        if i >= 3:
            ms.append(e0.elapsed_time(e1))
    t = float(np.median(ms))
    rd = W_PER_GPU * S * N * 4
    peaks = json.loads(PEAKS.read_text()) if PEAKS.exists() else {}
    hbm = peaks.get("hbm_gbs", 6650.0)
    del Sd
    return {"kernel": "sample_gather_kernel<16>", "ms": t, "bytes_read": rd, "gbs_read": rd / (t * 1e-3) / 1e9,
            "gbs_read_plus_write": 2 * rd / (t * 1e-3) / 1e9, "peak": hbm,
            "frac": 2 * rd / (t * 1e-3) / 1e9 / hbm,
            "note": "random 64-B rows (W=256 x s=20000 per round); frac counts read + write against the copy peak"}


def time_objective(hp, ctx, ds, C_ptr, k, cost_ptr, stream, reps, per_batch=4):
    """f(C,X) pass time: (average launch duration over back-to-back batches of `per_batch` launches,
    one launch bracketed on an idle stream). The first is the kernel's rate -- the host prepares launch
    i+1 while launch i runs, as in the engine's finish where the pass is queued behind the rounds; the
    second also holds the host's launch latency (the GPU idles between the event and the launch)."""
    import torch
    lib = hp._lib.lib
    batch, single = [], []
    for i in range(3 + reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(per_batch):
            hp._lib.check(lib.hpcg_assign_dev(ctx.h, ds.h, C_ptr, k, None, cost_ptr))
        e1.record(stream)
        torch.cuda.synchronize()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        hp._lib.check(lib.hpcg_assign_dev(ctx.h, ds.h, C_ptr, k, None, cost_ptr))
        a1.record(stream)
        torch.cuda.synchronize()
        if i >= 3:
            batch.append(e0.elapsed_time(e1) / per_batch)
            single.append(a0.elapsed_time(a1))
    return float(np.median(batch)), float(np.median(single))


def run_gpu(args, world, rank, local):
    import torch
    import paper_2311_04517_b200 as hp

    device = torch.device("cuda", local)
    torch.cuda.set_device(device)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=device)
    X = make_data(rank)
    Xd = torch.from_numpy(X).to(device)
    stream = torch.cuda.current_stream(device)
    ctx = hp.Context(local)
    ctx.set_stream(stream.cuda_stream)
    ds = hp.DeviceDataset.from_torch(Xd, ctx)
    cfg = hp.EngineConfig(k=K, sample_size=S, n_workers=W_PER_GPU, max_samples=ROUNDS, strategy="cooperative",
                          rng="philox", worker_base=rank * W_PER_GPU)
    sampling = "all rows"
    ds_eng, peers = ds, []
    if world > 1:
        attach_nccl(hp, ctx, world, rank, device)
        sampling = "local shard"
        if not args.local_sampling:
            try:  # global sampling over every rank's rows (the reference semantics), the default
                shards, peers = map_global_shards(hp, ctx, Xd, world, rank, device)
                ds_eng = hp.DeviceDataset.from_shards(shards, ctx=ctx, keepalive=Xd)
                sampling = f"global over {world} shards (NVLink P2P gathers)"
            except Exception as ex:  # keep the run: local-shard sampling, say why
                ds_eng = ds
                sampling = f"local shard (global sampling unavailable: {type(ex).__name__}: {ex})"[:160]
    eng = hp.Engine(ds_eng, cfg)
    if world > 1:  # every round publishes over all ranks' workers through the library (NCCL all-gather)
        set_exchange(eng, world, rank)
    fma_tfma = ctx.fma_peak()

    def step(seed):
        eng.reset(seed)
        eng.rounds(ROUNDS)
        return eng.finish()

    for i in range(args.warmup):
        step(10_000 + i)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    launches0 = ctx.launches
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    nd_total = 0
    objs = []
    with ClockSampler(local) as clk:  # the timed region: K complete runs, nothing but the public calls
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        ev0.record(stream)
        for i in range(args.steps):
            res = step(20_000 + i)
            nd_total += res.distance_evals  # all ranks' evaluations (the multi-rank finish sums them)
            objs.append(res.full_objective)
        ev1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
    launches = ctx.launches - launches0
    ms_total = ev0.elapsed_time(ev1)
    # the same K runs once more with the per-launch instrumentation (events around every worker-step /
    # f(C,X) launch, the worker steps' own evaluation count): the roofline's numerators and launch times.
    # Kept out of the timed region: the event pairs and the extra read-back cost ~2 % of a step.
    ctx.enable_timing(True)
    nd_rounds = 0  # the worker-step launches' own evaluations (the final pass's m x k_valid excluded)
    for i in range(args.steps):
        step(20_000 + i)
        nd_rounds += eng.distance_evals()  # this rank's worker-step evaluations (no final pass)
    torch.cuda.synchronize()
    kt = ctx.kernel_times()
    ctx.enable_timing(False)
    if world > 1:
        t = torch.tensor([ms_total], dtype=torch.float64, device=device)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms_total = float(t.item())
    nd_all = float(nd_total)
    ms_step = ms_total / args.steps
    value = nd_all / (ms_total * 1e-3)

    # ---- full-data objective pass alone (f(C,X) GB/s, HBM roofline); X (640 MB) > L2
    C_dev = torch.from_numpy(res.centroids).to(device)
    cost = torch.zeros(1, dtype=torch.float64, device=device)
    obj_t, obj_t1 = time_objective(hp, ctx, ds, C_dev.data_ptr(), K, cost.data_ptr(), stream, args.steps)
    obj_ms = [obj_t]
    obj_bytes = M * N * 4
    obj_gbs = obj_bytes / (obj_t * 1e-3) / 1e9

    peaks = json.loads(PEAKS.read_text()) if PEAKS.exists() else {}
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    hbm_src = "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback 6650 GB/s (B200_PROFILING.md)"
    # dominant kernel: the worker step. Algorithmic work = its own n_d (Lloyd + seeding evaluations,
    # core.hpp:205 / seeding.hpp:38; the final f(C,X) pass's m x k_valid is NOT charged to it) x n FMA.
    step_cnt, step_ms = kt["step"]
    step_flops_per_launch = nd_rounds / max(1, step_cnt) * N * 2
    mean_launch_ms = step_ms / max(1, step_cnt)
    achieved_tflops = step_flops_per_launch / (mean_launch_ms * 1e-3) / 1e12
    # the sample gather on its own (the worker step's gather phase as a dense kernel): GB/s vs HBM
    gat = gather_rate(hp, ctx, ds, stream, eng.philox_key)
    # what bounds a worker-step launch: its gather bytes at HBM peak plus its FMA work at the FMA peak
    gather_bytes_launch = W_PER_GPU * S * N * 4
    t_gather_ms = gather_bytes_launch / (hbm_peak * 1e9) * 1e3
    t_fma_ms = step_flops_per_launch / 2 / (fma_tfma * 1e12) * 1e3
    # DRAM bytes per launch from the committed ncu --set full captures of the current kernels
    trf = {}
    try:
        trf = json.load(open(ROOT / "profiles" / "traffic.json"))
    except (OSError, ValueError):
        pass
    step_traffic = None
    if "worker_step_round0_bytes" in trf and "worker_step_round1_bytes" in trf:  # 1 seeding + 3 steady rounds
        step_traffic = (trf["worker_step_round0_bytes"] + (ROUNDS - 1) * trf["worker_step_round1_bytes"]) / ROUNDS
    obj_traffic = trf.get("objective_bytes")
    peak_tflops = 2 * fma_tfma
    result = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32 screen + f64 accumulate/recheck", "data": "synthetic",
        "config": {"workload": "BASELINE config 2: X 1e7x16 fp32 Gaussian mixture (10 comps, Zipf(1.1)), k=10, "
                               "s=20000, 256 workers/GPU, cooperative, 4 lockstep rounds (1024 samples) + "
                               "full-data f(C,X)", "m_per_gpu": M, "n": N, "k": K, "s": S,
                   "workers_per_gpu": W_PER_GPU, "rounds": ROUNDS, "rng": "philox",
                   "l2": "X (640 MB/GPU) exceeds L2 (126 MB); samples gathered from HBM every round",
                   "parallelism": f"{world} GPU(s), one process per GPU; library NCCL all-gather of the round "
                                  f"candidates + device publication scan every round, select_best and f(C,X) "
                                  f"shard partials over all ranks",
                   "sampling": sampling, "exchange": EXCHANGE["mode"] if world > 1 else "none (1 rank)"},
        "distance_evals_per_step": nd_all / args.steps,
        "objective_pass": {"gbs": obj_gbs, "ms": float(np.median(obj_ms)), "bytes": obj_bytes,
                           "timing": "average launch duration over back-to-back batches of 4 launches (CUDA events "
                                     "on the launching stream); ms_isolated = one launch bracketed on an idle "
                                     "stream (adds the host's launch latency)",
                           "ms_isolated": obj_t1,
                           "roofline": {"bound": "hbm", "achieved": obj_gbs, "peak": hbm_peak, "unit": "GB/s",
                                        "frac": obj_gbs / hbm_peak, "traffic": obj_traffic,
                                        "traffic_unit": "bytes/launch (ncu, profiles/traffic.json)",
                                        "peak_source": hbm_src}},
        "roofline": {"bound": "fma", "kernel": "worker_step_kernel", "achieved": achieved_tflops,
                     "peak": peak_tflops, "unit": "TFLOP/s", "frac": achieved_tflops / peak_tflops,
                     "traffic": step_traffic,
                     "traffic_unit": "DRAM bytes/launch (ncu; mean of 1 seeding + 3 steady rounds)",
                     "algorithmic": "worker-step n_d (Lloyd + K-means++ evaluations of the rounds; the final "
                                    "f(C,X) pass excluded) x n FMA x 2 flop per launch / mean launch time",
                     "evals_per_launch": nd_rounds / max(1, step_cnt),
                     "peak_source": "FFMA2 loop measured in-run on this GPU (fp32 FMA; MEASURED_PEAKS.json has "
                                    "only hbm and bf16)",
                     "launches": step_cnt, "mean_launch_ms": mean_launch_ms,
                     "launch_bound_ms": {"gather_at_hbm": t_gather_ms, "fma_at_peak": t_fma_ms,
                                         "serial": t_gather_ms + t_fma_ms, "overlapped": max(t_gather_ms, t_fma_ms)},
                     "frac_of_combined_bound": (t_gather_ms + t_fma_ms) / mean_launch_ms},
        "gather": gat,
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "mean_full_objective": float(np.mean(objs)),
    }
    return result, X, eng, ctx


def e2e_run(X, args):
    """hpcg_run on pinned host data: upload + rounds + final pass + readback, per step."""
    import torch
    import paper_2311_04517_b200 as hp
    pinned = torch.from_numpy(X).pin_memory()
    Xp = pinned.numpy()
    cfg = hp.EngineConfig(k=K, sample_size=S, n_workers=W_PER_GPU, max_samples=ROUNDS, strategy="cooperative",
                          rng="philox")
    times, nds = [], []
    for i in range(1 + max(1, args.steps)):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        cfg.master_seed = 30_000 + i
        r = hp.run(Xp, cfg)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if i >= 1:
            times.append(dt)
            nds.append(r.distance_evals)
    h2d = X.nbytes
    d2h = K * N * 8 + K + 8 * 6
    return {"value": float(np.sum(nds) / np.sum(times)), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "ms_per_step": float(np.mean(times) * 1e3),
            "path": "hpcg_run (C-ABI one-call run, pinned host X) == hpclust::run"}


def e2e_run_multi(X, args, world, rank, ctx, device):
    """N > 1: the same run through the public API on every rank's pinned host shard -- upload
    (DeviceDataset), the shards mapped across ranks (CUDA IPC), an Engine with the library's NCCL
    exchange, run, finish (result read-back) -- timed on the host per step with a barrier on both
    sides, max over ranks."""
    import torch
    import torch.distributed as dist
    import paper_2311_04517_b200 as hp
    pinned = torch.from_numpy(X).pin_memory()
    Xp = pinned.numpy()
    cfg = hp.EngineConfig(k=K, sample_size=S, n_workers=W_PER_GPU, max_samples=ROUNDS, strategy="cooperative",
                          rng="philox", worker_base=rank * W_PER_GPU)
    times, nds = [], []
    for i in range(1 + max(1, args.steps)):
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        ds = hp.DeviceDataset(Xp, ctx=ctx)
        mine = torch.empty(0)  # the shard buffer is ds's own allocation
        peers = []
        ds_eng = ds
        if not args.local_sampling:
            base = hp._lib.lib.hpcg_dataset_device_ptr(ds.h)
            view = type("V", (), {"data_ptr": lambda self, b=base: b, "shape": (M, N)})()
            shards, peers = map_global_shards(hp, ctx, view, world, rank, device)
            ds_eng = hp.DeviceDataset.from_shards(shards, ctx=ctx, keepalive=ds)
        eng = hp.Engine(ds_eng, cfg)
        set_exchange(eng, world, rank)
        eng.reset(30_000 + i)
        eng.run()
        r = eng.finish()
        eng.close()
        dist.barrier()  # no rank may free its shard while a peer still maps it
        for p, hb in peers:
            hp.ipc_close(p, hb, ctx)
        if ds_eng is not ds:
            ds_eng.close()
        ds.close()
        del mine
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        t = torch.tensor([dt], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if i >= 1:
            times.append(float(t.item()))
            nds.append(float(r.distance_evals))  # already the all-rank total (engine finish)
    h2d = X.nbytes * world
    d2h = (K * N * 8 + K + 8 * 6) * world
    return {"value": float(np.sum(nds) / np.sum(times)), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "ms_per_step": float(np.mean(times) * 1e3),
            "path": "DeviceDataset upload + IPC-mapped shards + Engine with the library's NCCL exchange + finish, "
                    "per rank (max over ranks)"}


# ----------------------------------------------------------------------------- other configs
# BASELINE.json configs 3, 4 and a config-5 shard on this GPU (extra keys of the bench line; the
# headline is config 2). Seeded synthetic data with each config's shapes and distributions.
CFG_SETUP = {  # k, s, workers, rounds (max_samples), strategy, t1, t2, objective after every round
    3: (25, 50_000, 64, 20, "hybrid", 10.0, 10.0, True),
    4: (25, 100_000, 16, 10, "collective", 0.0, 0.0, False),
    5: (15, 200_000, 256, 4, "cooperative", 0.0, 0.0, False),
}
CFG_NOTE = {
    3: "1e8 x 3 fp64, 25 Gaussians U[0,255]^3 sigma 8 + 1% uniform noise; 64 workers, 20 rounds, hybrid "
       "t1=t2=10, f(C,X) of the shared best after every round (BASELINE.json) timed in the run",
    4: "5e6 x 128 fp32, 25 Gaussians N(0,4I) sigma 1; 16 workers, 10 rounds, collective (= cooperative); "
       "grid-wide path with the tcgen05 tf32 screen",
    5: "one GPU's shard of the 8-GPU job: 2.5e8 x 8 fp32 (of 2e9), 15 Gaussians U[-20,20]^8 sigma U[0.5,3], "
       "Dirichlet(1) weights; 256 of the 2,048 workers, 4 rounds, cooperative",
}


def cfg_data(hp, c):
    rs = np.random.default_rng(2311 + c)
    if c == 3:
        return hp.gen_mixture(100_000_000, 3, rs.uniform(0, 255, (25, 3)), np.full(25, 8.0), np.ones(25) / 25,
                              noise_frac=0.01, noise_box=(0.0, 255.0), seed=3, dtype=np.float64)
    if c == 4:
        return hp.gen_mixture(5_000_000, 128, rs.normal(0.0, 2.0, (25, 128)), np.ones(25), np.ones(25) / 25,
                              seed=4, dtype=np.float32)
    return hp.gen_mixture(250_000_000, 8, rs.uniform(-20, 20, (15, 8)), rs.uniform(0.5, 3.0, 15),
                          rs.dirichlet(np.ones(15)), seed=5, dtype=np.float32)


def config_extra(c, fma_tfma, device=0):
    """One BASELINE config on this GPU through the engine: whole run on the device-resident X
    (rounds + select + f(C,X)), per-round times (CUDA events), worker-step FMA fraction, f(C,X) GB/s
    against HBM, clocks sampled during the timed region."""
    import torch
    import paper_2311_04517_b200 as hp
    k, s, W, R, strat, t1, t2, obj_each = CFG_SETUP[c]
    X = cfg_data(hp, c)
    m, n = X.shape
    st = torch.cuda.current_stream(device)
    ctx = hp.Context(device)
    ctx.set_stream(st.cuda_stream)
    Xd = torch.from_numpy(X).to(f"cuda:{device}")
    del X
    ds = hp.DeviceDataset.from_torch(Xd, ctx)
    eng = hp.Engine(ds, hp.EngineConfig(k=k, sample_size=s, n_workers=W, max_samples=R, strategy=strat,
                                        phase_t1=t1, phase_t2=t2, rng="philox"))
    cost = torch.zeros(1, dtype=torch.float64, device=Xd.device)

    def one_run(seed, times=None):
        eng.reset(seed)
        for r in range(R):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            eng.rounds(1)
            if obj_each:
                b = eng.export_best()
                if np.isfinite(b[0]):
                    C_ = torch.from_numpy(b[2][b[3] == 0]).to(Xd.device)
                    hp._lib.check(hp._lib.lib.hpcg_assign_dev(ctx.h, ds.h, C_.data_ptr(), C_.shape[0], None,
                                                              cost.data_ptr()))
            e1.record(st)
            if times is not None:
                times.append((e0, e1))
        return eng.finish()

    one_run(1)
    one_run(2)
    torch.cuda.synchronize()
    ctx.enable_timing(True)
    runs = []  # whole runs repeated for >= 0.6 s so the clock sampler sees the load
    with ClockSampler(device) as clk:
        t_start = time.perf_counter()
        while len(runs) < 3 or (time.perf_counter() - t_start < 0.6 and len(runs) < 50):
            ev = []
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            res = one_run(3 + len(runs), ev)
            e1.record(st)
            torch.cuda.synchronize()
            runs.append((e0.elapsed_time(e1), [a.elapsed_time(b) for a, b in ev], res))
    kt = ctx.kernel_times()
    ctx.enable_timing(False)
    order = np.argsort([r[0] for r in runs])
    ms, rounds_ms, res = runs[order[len(runs) // 2]]  # the median run
    kt = {key: (cnt / len(runs), t / len(runs)) for key, (cnt, t) in kt.items()}
    kv = int((res.degenerate == 0).sum())
    nd_rounds = res.distance_evals - m * kv
    step_cnt, step_ms = kt["step"]
    step_tflops = nd_rounds * n * 2 / (step_ms * 1e-3) / 1e12 if step_ms > 0 else None
    C_ = torch.from_numpy(res.centroids[res.degenerate == 0]).to(Xd.device)
    obj_ms, obj_ms1 = time_objective(hp, ctx, ds, C_.data_ptr(), C_.shape[0], cost.data_ptr(), st, 5)
    nbytes = m * n * Xd.element_size()
    peaks = json.loads(PEAKS.read_text()) if PEAKS.exists() else {}
    hbm = peaks.get("hbm_gbs", 6650.0)
    out = {"config": c, "workload": CFG_NOTE[c], "m": m, "n": n, "k": k, "s": s, "workers": W, "rounds": R,
           "strategy": strat, "dtype": str(Xd.dtype).replace("torch.", ""), "run_ms": ms, "runs_timed": len(runs),
           "distance_evals": res.distance_evals, "evals_per_s": res.distance_evals / (ms * 1e-3),
           "round0_ms": rounds_ms[0], "steady_round_ms": float(np.median(rounds_ms[1:])) if R > 1 else None,
           "worker_step": {"launches": step_cnt, "ms": step_ms, "evals": nd_rounds, "achieved_tflops": step_tflops,
                           "peak_tflops": 2 * fma_tfma,
                           "frac": step_tflops / (2 * fma_tfma) if step_tflops else None,
                           "peak_source": "in-run FFMA2 (fp32 FMA) peak; the screen runs in fp32 for fp64 data too"},
           "objective_pass": {"ms": obj_ms, "ms_isolated": obj_ms1, "bytes": nbytes,
                              "gbs": nbytes / (obj_ms * 1e-3) / 1e9, "peak": hbm,
                              "frac": nbytes / (obj_ms * 1e-3) / 1e9 / hbm},
           "full_objective": res.full_objective, "clocks": clk.summary()}
    eng.close()
    ds.close()
    ctx.close()
    del Xd, C_, cost
    torch.cuda.empty_cache()
    return out


def cpu_baseline(X, budget_s=10.0):
    """The reference's own kmeans (oracle/_ref, stock code path) on config-2 samples, one
    std::thread per worker (its competitive threading model, engine.hpp:313-332), host cores."""
    sys.path.insert(0, str(ROOT / "tests"))
    from oracle_py import ref
    R = ref()
    if R is None:
        return None
    P = host_cores()
    rs = np.random.default_rng(0)
    nd_tot, t_tot, reps = 0, 0.0, 0
    while t_tot < budget_s and reps < 1000:
        idx = [rs.choice(M, S, replace=False) for _ in range(P)]
        samples = np.stack([X[i].astype(np.float64) for i in idx])
        inits = np.stack([smp[rs.choice(S, K, replace=False)] for smp in samples])
        t0 = time.perf_counter()
        nd, _ = R.kmeans_threads(samples, inits)
        t_tot += time.perf_counter() - t0
        nd_tot += nd
        reps += 1
    return {"value": nd_tot / t_tot, "unit": "Lloyd evals/s", "cores": P, "kind": "reference",
            "sample": f"{reps} batches x {P} workers: reference kmeans() (lloyd.hpp:100-164) on s=20000 x 16 "
                      f"config-2 samples from random-row inits, {t_tot:.1f} s CPU wall",
            "cpu_model": cpu_model()}


def run_reference(args, world, rank):
    """--impl reference: hpclust::run (reference, oracle/_ref) on the config-2 data in fp64."""
    if rank != 0:
        return None
    sys.path.insert(0, str(ROOT / "tests"))
    from oracle_py import ref
    R = ref()
    if R is None:
        return {"impl": "reference", "unavailable": "oracle/_ref/libhpclust_ref.so not built"}
    P = host_cores()
    X = make_data(0).astype(np.float64)  # the same rows as the GPU arm (numpy; libhpcg never loaded)
    Wr = W_PER_GPU  # the reference's own thread-per-worker model (engine.hpp:313-332) at the GPU arm's W
    times, nds = [], []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        r = R.run(X, k=K, sample_size=S, n_workers=Wr, max_samples=ROUNDS, strategy="cooperative", seed=40_000 + i,
                  n_threads=P, full=True)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
            nds.append(r["distance_evals"])
    value = float(np.sum(nds) / np.sum(times))
    return {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": float(np.mean(times) * 1e3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "BASELINE config 2: X 1e7x16 Gaussian mixture (10 comps, Zipf(1.1)), k=10, "
                                   "s=20000, 256 workers/GPU, cooperative, 4 lockstep rounds (1024 samples) + "
                                   "full-data f(C,X)", "m_per_gpu": M, "n": N, "k": K, "s": S,
                       "workers_per_gpu": Wr, "rounds": ROUNDS,
                       "reference_path": "hpclust::run (engine.hpp:444-499), oracle/_ref built from the unmodified "
                                         "headers; fp64 copy of the same rows; one std::thread per worker",
                       "same_config": True},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": P, "kind": "reference",
                             "sample": f"{args.steps} full reference runs of the workload ({Wr} workers x {ROUNDS} "
                                       f"rounds + final objective), each a timed step", "cpu_model": cpu_model()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the config 3/4/5 extra keys")
    ap.add_argument("--configs-only", default="", help="e.g. 3,4,5: print one JSON line per config and exit")
    ap.add_argument("--local-sampling", action="store_true",
                    help="N > 1: sample each rank's own shard instead of all ranks' rows (peer-mapped shards)")
    args = ap.parse_args()
    world, rank, local = dist_setup()
    if args.configs_only:
        import paper_2311_04517_b200 as hp
        fma = hp.Context(local).fma_peak()
        for c in args.configs_only.split(","):
            print(json.dumps(config_extra(int(c), fma, local)), flush=True)
        return
    if args.impl == "reference":
        out = run_reference(args, world, rank)
        if out is not None:
            print(json.dumps(out))
        return
    result, X, eng, ctx = run_gpu(args, world, rank, local)
    e2e_multi = None
    if world > 1 and not args.no_e2e:  # every rank takes part (collectives inside)
        import torch
        eng.close()
        try:
            e2e_multi = e2e_run_multi(X, args, world, rank, ctx, torch.device("cuda", local))
        except Exception as ex:  # keep the bench line; say why the e2e leg is missing
            e2e_multi = {"value": None, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
                         "error": f"{type(ex).__name__}: {ex}"[:200]}
    if rank == 0:
        if not args.no_e2e and world == 1:
            result["e2e"] = e2e_run(X, args)
        elif world > 1:
            result["e2e"] = e2e_multi or {"value": None, "unit": UNIT, "h2d_bytes_per_step": 0,
                                          "d2h_bytes_per_step": 0, "note": "--no-e2e"}
        if not args.no_cpu and world == 1:
            result["cpu_baseline"] = cpu_baseline(X)
        if not args.no_configs and world == 1:
            del eng, X
            fma = result["roofline"]["peak"] / 2
            extras = []
            for c in (3, 4, 5):
                try:
                    extras.append(config_extra(c, fma, local))
                except Exception as ex:  # keep the bench line; say which config failed and why
                    extras.append({"config": c, "error": f"{type(ex).__name__}: {ex}"[:200]})
            result["configs"] = extras
        print(json.dumps(result))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
