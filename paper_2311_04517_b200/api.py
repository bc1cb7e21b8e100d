"""Python mirror of the reference's hot-path interface (proj/include/hpclust), backed by
libhpcg.so. Names, argument meaning and error behaviour follow the reference:

    assign_nearest / mssc_objective            core.hpp:212-233
    final_assignment / assign_valid_subset     engine.hpp:197-229
    kmeans, LloydConfig, LloydOutcome          lloyd.hpp:10-40, 100-164
    kmeanspp_seed / reinit_degenerate          seeding.hpp:113-133
    draw_sample                                engine.hpp:165-177
    RngStream                                  rng.hpp:26-99
    EngineConfig / run / ClusteringResult      engine.hpp:48-87, 269-284, 444-499

Every numeric result is computed by the sm_100a kernels; nothing here computes on the CPU
except argument marshalling and the reference RNG replay (which only produces indices and
uniform draws, exactly as rng.hpp would).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import check, lib, ptr

STOP_NAMES = {0: "tolerance", 1: "max_iters", 2: "fixed_point"}


# ----------------------------------------------------------------------------- context
class Context:
    """One device + stream (hpcg_ctx)."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        check(lib.hpcg_ctx_create(device, C.byref(h)))
        self.h = h
        self.device = device

    def set_stream(self, cuda_stream: int | None):
        check(lib.hpcg_ctx_set_stream(self.h, cuda_stream))

    def synchronize(self):
        check(lib.hpcg_ctx_synchronize(self.h))

    def set_fp32_cost(self, exact: bool):
        """f(C, X) over fp32 data: exact fp64 row cost (True) or the fp32 mode (False, the default)."""
        check(lib.hpcg_ctx_set_fp32_cost(self.h, 1 if exact else 0))

    @property
    def upload_bytes(self) -> int:
        return int(lib.hpcg_ctx_upload_bytes(self.h))

    def attach_comm(self, nranks: int, rank: int, uid: bytes):
        """Collective over the ranks: NCCL communicator for multi-rank engines (one rank per GPU)."""
        buf = C.create_string_buffer(bytes(uid), 128)
        check(lib.hpcg_ctx_attach_comm(self.h, nranks, rank, buf))

    @property
    def launches(self) -> int:
        return int(lib.hpcg_ctx_launch_count(self.h))

    def enable_timing(self, on: bool = True):
        check(lib.hpcg_ctx_enable_timing(self.h, int(on)))

    def kernel_times(self):
        """{'step': (launches, ms), 'objective': (launches, ms)} summed since timing was enabled."""
        cnt = np.zeros(2, np.int64)
        ms = np.zeros(2)
        check(lib.hpcg_ctx_kernel_times(self.h, ptr(cnt), ptr(ms)))
        return {"step": (int(cnt[0]), float(ms[0])), "objective": (int(cnt[1]), float(ms[1]))}

    def fma_peak(self) -> float:
        """Measured FP32 FMA rate (TFMA/s) of the device at its current clocks."""
        v = C.c_double()
        check(lib.hpcg_probe_fma_peak(self.h, C.byref(v)))
        return v.value

    def close(self):
        if self.h:
            lib.hpcg_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ctx: Context | None = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


def _dtype_code(a: np.ndarray) -> int:
    if a.dtype == np.float32:
        return _lib.F32
    if a.dtype == np.float64:
        return _lib.F64
    raise TypeError("X must be float32 or float64")


class DeviceDataset:
    """X resident in HBM (hpcg_dataset). Built from a host array (upload) or a CUDA
    tensor / device pointer (borrowed, zero-copy)."""

    def __init__(self, X=None, *, ctx: Context | None = None, device_ptr: int | None = None,
                 dtype=None, shape=None, keepalive=None):
        self.ctx = ctx or default_context()
        h = C.c_void_p()
        if device_ptr is not None:
            m, n = shape
            code = _lib.F32 if np.dtype(dtype) == np.float32 else _lib.F64
            check(lib.hpcg_dataset_wrap(self.ctx.h, C.c_void_p(device_ptr), code, m, n, C.byref(h)))
            self._keep = keepalive
        else:
            X = np.ascontiguousarray(X)
            if X.ndim != 2:
                raise ValueError("Dataset: X must be 2-D")
            code = _dtype_code(X)
            m, n = X.shape
            check(lib.hpcg_dataset_upload(self.ctx.h, ptr(X), code, m, n, C.byref(h)))
            self._keep = None
        self.h = h
        self.m, self.n = int(m), int(n)
        self.dtype = np.float32 if code == _lib.F32 else np.float64

    @classmethod
    def from_shards(cls, shards, ctx: Context | None = None, keepalive=None):
        """Row-sharded X (global row order): shards = [(device_ptr, rows), ...] or CUDA tensors,
        local or peer-mapped (ipc_open). Samples are drawn over all rows (multi-GPU global sampling)."""
        import torch
        self = cls.__new__(cls)
        self.ctx = ctx or default_context()
        ptrs, rows, n, dt = [], [], None, None
        for sh in shards:
            if isinstance(sh, torch.Tensor):
                assert sh.is_cuda and sh.is_contiguous() and sh.dim() == 2
                ptrs.append(sh.data_ptr())
                rows.append(sh.shape[0])
                n = sh.shape[1]
                dt = np.float32 if sh.dtype == torch.float32 else np.float64
            else:
                ptrs.append(int(sh[0]))
                rows.append(int(sh[1]))
                n, dt = int(sh[2]), np.dtype(sh[3]).type
        pa = (C.c_void_p * len(ptrs))(*ptrs)
        ra = (C.c_int64 * len(rows))(*rows)
        h = C.c_void_p()
        code = _lib.F32 if dt == np.float32 else _lib.F64
        check(lib.hpcg_dataset_wrap_sharded(self.ctx.h, pa, ra, len(ptrs), code, n, C.byref(h)))
        self.h = h
        self.m, self.n = int(sum(rows)), int(n)
        self.dtype = dt
        self._keep = (list(shards), keepalive)
        return self

    @classmethod
    def from_torch(cls, t, ctx: Context | None = None):
        assert t.is_cuda and t.is_contiguous() and t.dim() == 2
        import torch
        dt = np.float32 if t.dtype == torch.float32 else np.float64
        return cls(ctx=ctx, device_ptr=t.data_ptr(), dtype=dt, shape=tuple(t.shape), keepalive=t)

    def close(self):
        if getattr(self, "h", None):
            lib.hpcg_dataset_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


IPC_HANDLE_BYTES = 72


def ipc_export(device_ptr: int) -> bytes:
    """CUDA IPC handle of device memory (allocation handle + offset), for another process."""
    buf = C.create_string_buffer(IPC_HANDLE_BYTES)
    check(lib.hpcg_ipc_export(C.c_void_p(device_ptr), buf))
    return buf.raw


def ipc_open(handle: bytes, ctx: Context | None = None) -> int:
    """Map another process's memory (peer access over NVLink when it lives on another GPU)."""
    ctx = ctx or default_context()
    p = C.c_void_p()
    check(lib.hpcg_ipc_open(ctx.h, C.create_string_buffer(handle, IPC_HANDLE_BYTES), C.byref(p)))
    return int(p.value)


def ipc_close(device_ptr: int, handle: bytes, ctx: Context | None = None):
    ctx = ctx or default_context()
    check(lib.hpcg_ipc_close(ctx.h, C.c_void_p(device_ptr), C.create_string_buffer(handle, IPC_HANDLE_BYTES)))


def _as_dataset(X, ctx=None) -> DeviceDataset:
    return X if isinstance(X, DeviceDataset) else DeviceDataset(X, ctx=ctx)


# ------------------------------------------------------------------------- rng.hpp
class RngStream:
    """rng.hpp:26-99 — std::mt19937_64 with the reference's hand-rolled distributions.
    State lives on the host (312 words); the kernels consume its draws."""

    def __init__(self, seed: int = 0, *, _state=None):
        self.state = np.zeros(312, dtype=np.uint64)
        self.pos = C.c_int32(312)
        if _state is None:
            check(lib.hpcg_rng_seed(C.c_uint64(seed), ptr(self.state), C.byref(self.pos)))
        else:
            self.state[:] = _state[0]
            self.pos.value = _state[1]

    @classmethod
    def derive(cls, master: int, domain: int, index: int) -> "RngStream":
        r = cls.__new__(cls)
        r.state = np.zeros(312, dtype=np.uint64)
        r.pos = C.c_int32(312)
        check(lib.hpcg_rng_derive(C.c_uint64(master), C.c_uint64(domain), C.c_uint64(index), ptr(r.state),
                                  C.byref(r.pos)))
        return r

    def copy(self) -> "RngStream":
        return RngStream(_state=(self.state.copy(), self.pos.value))

    def _draw(self, kind, count, bound=0):
        out = np.empty(count, dtype=np.float64 if kind == 1 else np.uint64)
        check(lib.hpcg_rng_draw(ptr(self.state), C.byref(self.pos), kind, C.c_uint64(bound), count, ptr(out)))
        return out

    def next_u64(self) -> int:
        return int(self._draw(0, 1)[0])

    def next_unit(self) -> float:
        return float(self._draw(1, 1)[0])

    def units(self, count: int) -> np.ndarray:
        return self._draw(1, count)

    def uniform_index(self, n: int) -> int:
        if n <= 0:
            raise _lib.InvalidArgument("uniform_index: n must be positive")
        return int(self._draw(2, 1, n)[0])


# ------------------------------------------------------------------------ core.hpp
@dataclass
class Assignment:
    labels: np.ndarray
    counts: np.ndarray


def _centroids(C_, degenerate, n):
    C_ = np.ascontiguousarray(C_, dtype=np.float64)
    if C_.ndim != 2:
        raise ValueError("centroids must be k x n")
    k = C_.shape[0]
    if C_.shape[1] != n:
        return C_, None, k
    deg = None if degenerate is None else np.ascontiguousarray(degenerate, dtype=np.uint8)
    return C_, deg, k


def _assign(X, C_, degenerate, require_valid, want_labels, want_counts, ctx=None):
    ds = _as_dataset(X, ctx)
    C_, deg, k = _centroids(C_, degenerate, ds.n)
    labels = np.empty(ds.m, dtype=np.int32) if want_labels else None
    counts = np.zeros(k, dtype=np.int64) if want_counts else None
    cost = C.c_double()
    nd = C.c_int64()
    check(lib.hpcg_assign(ds.ctx.h, ds.h, ptr(C_), ptr(deg), k, int(require_valid), ptr(labels), ptr(counts),
                          C.byref(cost), C.byref(nd)))
    return labels, counts, cost.value, nd.value


def assign_nearest(X, C_, degenerate=None, counter=None) -> Assignment:
    """core.hpp:212-221."""
    n = X.n if isinstance(X, DeviceDataset) else np.asarray(X).shape[1]
    if len(C_) < 1:
        raise _lib.InvalidArgument("assign_nearest: need at least one centroid")
    if np.asarray(C_).shape[1] != n:
        raise _lib.InvalidArgument("assign_nearest: dimension mismatch")
    if degenerate is not None and np.any(degenerate):
        raise _lib.InvalidArgument("assign_nearest: degenerate centroid present")
    labels, counts, _, nd = _assign(X, C_, None, True, True, True)
    if counter is not None:
        counter.add(nd)
    return Assignment(labels, counts)


def mssc_objective(C_, X, degenerate=None, counter=None) -> float:
    """core.hpp:224-233."""
    n = X.n if isinstance(X, DeviceDataset) else np.asarray(X).shape[1]
    if len(C_) < 1:
        raise _lib.InvalidArgument("mssc_objective: need at least one centroid")
    if np.asarray(C_).shape[1] != n:
        raise _lib.InvalidArgument("mssc_objective: dimension mismatch")
    if degenerate is not None and np.any(degenerate):
        raise _lib.InvalidArgument("mssc_objective: degenerate centroid present")
    _, _, cost, nd = _assign(X, C_, None, True, False, False)
    if counter is not None:
        counter.add(nd)
    return cost


def final_assignment(X, C_, degenerate=None, counter=None):
    """engine.hpp:197-205."""
    if degenerate is not None and np.any(degenerate):
        raise _lib.InvalidArgument("final_assignment: degenerate centroid present")
    n = X.n if isinstance(X, DeviceDataset) else np.asarray(X).shape[1]
    if np.asarray(C_).shape[1] != n:
        raise _lib.InvalidArgument("final_assignment: dimension mismatch")
    labels, counts, cost, nd = _assign(X, C_, None, True, True, True)
    if counter is not None:
        counter.add(nd)
    return Assignment(labels, counts), cost


def assign_valid_subset(X, C_, degenerate, counter=None):
    """engine.hpp:211-229: valid centres only, labels in original slot numbering."""
    labels, counts, cost, nd = _assign(X, C_, degenerate, False, True, True)
    if counter is not None:
        counter.add(nd)
    return Assignment(labels, counts), cost


class DistCounter:
    """core.hpp:23-31."""

    def __init__(self):
        self.count = 0

    def add(self, v):
        self.count += int(v)

    def value(self):
        return self.count


# ----------------------------------------------------------------------- lloyd.hpp
@dataclass
class LloydConfig:
    max_iters: int = 300
    rel_tol: float = 1e-4


@dataclass
class SeedConfig:
    candidates_per_center: int = 3


@dataclass
class LloydOutcome:
    centroids: np.ndarray
    degenerate: np.ndarray
    labels: np.ndarray
    counts: np.ndarray
    objective: float
    iterations: int
    converged_by: str
    objective_history: list = field(default_factory=list)
    n_d: int = 0


def _seed_draws(rngs, degenerate_rows, k, s, candidates):
    """The draws seed_degenerate_slots consumes (seeding.hpp:72-99), per worker: the
    uniform_index(s) of the first centre when no centre is valid, then `candidates`
    next_unit() per remaining pending slot. Returns (first_row[W], units[W, stride],
    snapshots, plan) so callers can rewind a stream that stopped early."""
    W = len(rngs)
    stride = max(1, k * candidates)
    first = np.zeros(W, dtype=np.int64)
    units = np.zeros((W, stride), dtype=np.float64)
    plan = []
    for w, rng in enumerate(rngs):
        deg = degenerate_rows[w]
        npend = int(np.count_nonzero(deg))
        nvalid = k - npend
        no_valid = npend > 0 and nvalid == 0
        if rng is None:
            plan.append((0, 0, None))
            continue
        if no_valid:
            first[w] = rng.uniform_index(s)
        snap = rng.copy()
        loops = npend - (1 if no_valid else 0)
        if loops > 0:
            units[w, : loops * candidates] = rng.units(loops * candidates)
        plan.append((int(no_valid), loops, snap))
    return first, units, plan


def _rewind(rngs, plan, filled, candidates):
    for w, rng in enumerate(rngs):
        no_valid, loops, snap = plan[w]
        if rng is None or snap is None:
            continue
        used = int(filled[w]) - no_valid
        if used < loops:
            r = snap.copy()
            if used > 0:
                r.units(used * candidates)
            rng.state[:] = r.state
            rng.pos.value = r.pos.value


def worker_step_batched(X, idx, inits, degenerate, *, rngs=None, lloyd=LloydConfig(), seed=SeedConfig(),
                        do_lloyd=True, want_labels=False, want_counts=False, hist_cap=0, ctx=None):
    """W (sample, init) problems in one launch: reseed degenerate slots, then Lloyd.
    idx: [W, s] rows of X (draw order) or None when X is [W*s, n] stacked samples."""
    ds = _as_dataset(X, ctx)
    inits = np.ascontiguousarray(inits, dtype=np.float64)
    W, k, n = inits.shape
    if idx is not None:
        idx = np.ascontiguousarray(idx, dtype=np.int64)
        s = idx.shape[1]
    else:
        s = ds.m // W
    deg = np.zeros((W, k), dtype=np.uint8) if degenerate is None else np.ascontiguousarray(degenerate, np.uint8)
    cfg = _lib.LloydCfg(lloyd.max_iters, lloyd.rel_tol, seed.candidates_per_center)
    first = units = None
    plan = None
    stride = 0
    if rngs is not None:
        first, units, plan = _seed_draws(rngs, deg, k, s, seed.candidates_per_center)
        stride = units.shape[1]
    C_out = np.empty((W, k, n))
    f_out = np.empty((W, k), dtype=np.uint8)
    obj = np.empty(W)
    iters = np.empty(W, dtype=np.int32)
    stop = np.empty(W, dtype=np.int32)
    nd = np.empty(W, dtype=np.int64)
    filled = np.empty(W, dtype=np.int32)
    labels = np.empty((W, s), dtype=np.int32) if want_labels else None
    counts = np.empty((W, k), dtype=np.int64) if want_counts else None
    hist = np.empty((W, hist_cap)) if hist_cap else None
    hlen = np.empty(W, dtype=np.int32)
    rc = lib.hpcg_worker_step_batched(ds.ctx.h, ds.h, ptr(idx), W, s, ptr(inits), ptr(deg), k, C.byref(cfg),
                                      ptr(first), ptr(units), stride, int(do_lloyd), ptr(C_out), ptr(f_out),
                                      ptr(obj), ptr(iters), ptr(stop), ptr(nd), ptr(filled), ptr(labels),
                                      ptr(counts), ptr(hist), hist_cap, ptr(hlen))
    if rngs is not None and rc in (_lib.HPCG_OK, _lib.HPCG_EINVAL, _lib.HPCG_ELOGIC):
        _rewind(rngs, plan, filled, seed.candidates_per_center)
    check(rc)
    return dict(centroids=C_out, degenerate=f_out, objective=obj, iterations=iters, stop=stop, n_d=nd,
                filled=filled, labels=labels, counts=counts, history=hist, hist_len=hlen)


def kmeans(S, C_init, cfg: LloydConfig = LloydConfig(), counter=None, degenerate=None, ctx=None) -> LloydOutcome:
    """lloyd.hpp:100-164 on one sample (a batch of one worker)."""
    if cfg.max_iters < 1:
        raise _lib.InvalidArgument("kmeans: max_iters must be positive")
    if not cfg.rel_tol > 0.0:
        raise _lib.InvalidArgument("kmeans: rel_tol must be positive")
    if degenerate is not None and np.any(degenerate):
        raise _lib.InvalidArgument("kmeans: degenerate centroid in init")
    S = np.ascontiguousarray(S)
    C_init = np.ascontiguousarray(C_init, dtype=np.float64)
    if C_init.shape[1] != S.shape[1]:
        raise _lib.InvalidArgument("kmeans: dimension mismatch")
    cap = int(min(cfg.max_iters, 100000)) + 1
    r = worker_step_batched(S, None, C_init[None], None, lloyd=cfg, want_labels=True, want_counts=True,
                            hist_cap=cap, ctx=ctx)
    if counter is not None:
        # Lloyd passes only: iterations (+1 closing pass unless fixed point), s*k each
        counter.add(int(r["n_d"][0]))
    hl = int(r["hist_len"][0])
    return LloydOutcome(r["centroids"][0], r["degenerate"][0], r["labels"][0], r["counts"][0],
                        float(r["objective"][0]), int(r["iterations"][0]), STOP_NAMES[int(r["stop"][0])],
                        list(r["history"][0, :hl]), int(r["n_d"][0]))


# --------------------------------------------------------------------- seeding.hpp
def reinit_degenerate(C_, degenerate, S, cfg: SeedConfig, rng: RngStream, counter=None, ctx=None):
    """seeding.hpp:125-133 -> (centroids, degenerate)."""
    C_ = np.ascontiguousarray(C_, dtype=np.float64)
    deg = np.ascontiguousarray(degenerate, dtype=np.uint8)
    if not deg.any():
        return C_.copy(), deg.copy()
    S = np.ascontiguousarray(S)
    if S.shape[0] < 1:
        raise _lib.InvalidArgument("seeding: empty sample")
    if C_.shape[1] != S.shape[1]:
        raise _lib.InvalidArgument("seeding: dimension mismatch")
    if cfg.candidates_per_center < 1:
        raise _lib.InvalidArgument("seeding: need at least one candidate")
    r = worker_step_batched(S, None, C_[None], deg[None], rngs=[rng], seed=cfg, do_lloyd=False, ctx=ctx)
    if counter is not None:
        counter.add(int(r["n_d"][0]))
    return r["centroids"][0], r["degenerate"][0]


def kmeanspp_seed(S, k, cfg: SeedConfig, rng: RngStream, counter=None, ctx=None):
    """seeding.hpp:113-121."""
    if k < 1:
        raise _lib.InvalidArgument("kmeanspp_seed: k must be positive")
    n = np.asarray(S).shape[1]
    return reinit_degenerate(np.zeros((k, n)), np.ones(k, dtype=np.uint8), S, cfg, rng, counter, ctx)


# ---------------------------------------------------------------------- engine.hpp
def reference_draw_indices(m: int, s: int, rng: RngStream) -> np.ndarray:
    """The rows draw_sample (engine.hpp:165-177) picks, in draw order; advances rng."""
    if not 1 <= s <= m:
        raise _lib.InvalidArgument("draw_sample: sample size must be in [1, m]")
    out = np.empty(s, dtype=np.int64)
    check(lib.hpcg_reference_draw_indices(ptr(rng.state), C.byref(rng.pos), m, s, ptr(out)))
    return out


def philox_sample_indices(m: int, s: int, key: int, round_: int, worker: int, ctx=None) -> np.ndarray:
    """The rows a philox-mode engine round samples for `worker` (device keyed permutation)."""
    if not 1 <= s <= m:
        raise _lib.InvalidArgument("draw_sample: sample size must be in [1, m]")
    ctx = ctx or default_context()
    out = np.empty(s, dtype=np.int64)
    check(lib.hpcg_sample_indices(ctx.h, m, s, key, round_, worker, ptr(out)))
    return out


def draw_sample(X, s: int, rng: RngStream, ctx=None) -> np.ndarray:
    """engine.hpp:165-177: s distinct rows in draw order, gathered on the device."""
    ds = _as_dataset(X, ctx)
    idx = reference_draw_indices(ds.m, s, rng)
    out = np.empty((s, ds.n), dtype=ds.dtype)
    check(lib.hpcg_gather(ds.ctx.h, ds.h, ptr(idx), s, ptr(out)))
    return out


def select_best(objectives):
    """engine.hpp:180-194: lowest objective, ties to the lowest id."""
    best, best_f = -1, math.inf
    for w, f in enumerate(objectives):
        if f < best_f:
            best, best_f = w, f
    if best < 0:
        raise _lib.NoSolutionError("no solution produced: every worker incumbent is infinite")
    return best


STRATEGIES = {"inner": _lib.INNER, "competitive": _lib.COMPETITIVE, "cooperative": _lib.COOPERATIVE,
              "collective": _lib.COOPERATIVE, "hybrid": _lib.HYBRID}


@dataclass
class EngineConfig:
    """engine.hpp:48-87 (deterministic max_samples schedule)."""

    k: int = 0
    sample_size: int = 0
    n_workers: int = 1
    max_samples: int = 0  # per worker; 0 = none (then time_limit must be set), engine.hpp:54
    strategy: str = "competitive"
    phase_t1: float = 0.0
    phase_t2: float = 0.0
    master_seed: int = 0
    candidates: int = 3
    max_iters: int = 300
    rel_tol: float = 1e-4
    compute_full_objective: bool = True
    compute_assignment: bool = False
    rng: str = "reference"  # "reference" (bit-parity streams) or "philox" (device)
    worker_base: int = 0
    time_limit: float = 0.0  # seconds; > 0: wall-clock schedule (engine.hpp:348-374), max_samples a cap
    free_running: bool = False  # wall clock: free-running workers, immediate publication (engine.hpp:355-371)
    free_group: int = 0  # workers per free-running group (0 = automatic)

    def to_c(self) -> _lib.EngineCfg:
        if self.strategy not in STRATEGIES:
            raise _lib.InvalidArgument("unknown strategy: " + self.strategy)
        return _lib.EngineCfg(self.k, self.sample_size, self.n_workers, self.max_samples,
                              STRATEGIES[self.strategy], self.phase_t1, self.phase_t2, self.master_seed,
                              self.candidates, self.max_iters, self.rel_tol, int(self.compute_full_objective),
                              int(self.compute_assignment),
                              _lib.RNG_REFERENCE if self.rng == "reference" else _lib.RNG_PHILOX, self.worker_base,
                              float(self.time_limit), int(self.free_running), int(self.free_group))


class _Traces:
    """Per-worker update traces (WorkerState::update_trace): worker w -> rows (timestamp, objective).
    A view over the finish buffers, sliced on access (building W arrays eagerly costs more host time
    than a round of 256 workers takes on the device)."""

    def __init__(self, buf, lens):
        self._buf, self._len = buf, lens

    def __len__(self):
        return len(self._len)

    def __getitem__(self, w):
        if isinstance(w, slice):
            return [self[i] for i in range(*w.indices(len(self)))]
        if w < 0:
            w += len(self)
        if not 0 <= w < len(self):
            raise IndexError(w)
        return self._buf[w, : int(self._len[w])]

    def __iter__(self):
        return (self[w] for w in range(len(self)))


@dataclass
class ClusteringResult:
    """engine.hpp:269-284."""

    centroids: np.ndarray
    degenerate: np.ndarray
    full_objective: float | None
    assignment: np.ndarray | None
    best_worker: int
    best_sample_objective: float
    clustering_time: float
    clustering_time_first_finisher: float
    wall_seconds: float
    total_samples: int
    distance_evals: int
    worker_objectives: np.ndarray
    traces: list
    publications: np.ndarray


class Engine:
    """Stepwise lockstep engine on a device-resident dataset (bench / multi-round use)."""

    def __init__(self, ds: DeviceDataset, cfg: EngineConfig):
        self.ds, self.cfg = ds, cfg
        self._c = cfg.to_c()
        h = C.c_void_p()
        check(lib.hpcg_engine_create(ds.ctx.h, ds.h, C.byref(self._c), C.byref(h)))
        self.h = h
        self.W = 1 if cfg.strategy == "inner" else cfg.n_workers
        self._nranks = 1

    def set_exchange(self, nranks: int, rank: int, allgather=None):
        """Make this engine rank `rank` of `nranks` (cooperative / hybrid publication over every
        rank's workers, select_best and f(C, X) over all ranks; include/hpcg.h multi-GPU). allgather:
        None -> the context's NCCL communicator; else a callable(bytes) -> bytes returning every
        rank's bytes concatenated in rank order (the caller's own collective, e.g. gloo)."""
        fn = _lib.ALLGATHER_FN() if allgather is None else allgather_callback(allgather, nranks)
        self._xfn = fn  # keep the callback alive as long as the engine
        check(lib.hpcg_engine_set_exchange(self.h, nranks, rank, fn, None))
        self._nranks = nranks

    def rounds(self, n: int = 1):
        check(lib.hpcg_engine_rounds(self.h, n))

    def run(self):
        """The configured schedule to its end: lockstep max_samples rounds, or rounds until
        cfg.time_limit seconds (wall-clock schedule, engine.hpp:348-374)."""
        check(lib.hpcg_engine_run(self.h))

    def reset(self, master_seed: int):
        check(lib.hpcg_engine_reset(self.h, C.c_uint64(master_seed)))

    def import_best(self, obj: float, worker: int, C_, flags):
        C_ = np.ascontiguousarray(C_, np.float64)
        flags = np.ascontiguousarray(flags, np.uint8)
        check(lib.hpcg_engine_import_best(self.h, obj, worker, ptr(C_), ptr(flags)))

    @property
    def round_index(self) -> int:
        return int(lib.hpcg_engine_round_index(self.h))

    def distance_evals(self) -> int:
        v = C.c_int64()
        check(lib.hpcg_engine_distance_evals(self.h, C.byref(v)))
        return v.value

    @property
    def philox_key(self) -> int:
        return int(lib.hpcg_engine_philox_key(self.h))

    def round_outcome(self) -> dict:
        """Per-worker outcome of the last round (worker_step, engine.hpp:238-267)."""
        W = self.W
        obj, it, st = np.empty(W), np.empty(W, np.int32), np.empty(W, np.int32)
        nd, acc, fl = np.empty(W, np.int64), np.empty(W, np.uint8), np.empty(W, np.int32)
        check(lib.hpcg_engine_round_outcome(self.h, ptr(obj), ptr(it), ptr(st), ptr(nd), ptr(acc), ptr(fl)))
        return dict(objective=obj, iterations=it, stop=st, n_d=nd, accepted=acc.astype(bool), filled=fl)

    def worker_progress(self):
        """(samples_processed[W], t_w[W]) -- WorkerState fields engine.hpp:100, 250."""
        smp, tw = np.zeros(self.W, np.int64), np.zeros(self.W)
        check(lib.hpcg_engine_worker_progress(self.h, ptr(smp), ptr(tw)))
        return smp, tw

    def worker_incumbents(self):
        k, n, W = self.cfg.k, self.ds.n, self.W
        Cw, fw, ow = np.empty((W, k, n)), np.empty((W, k), np.uint8), np.empty(W)
        check(lib.hpcg_engine_worker_incumbents(self.h, ptr(Cw), ptr(fw), ptr(ow)))
        return Cw, fw, ow

    def export_best(self):
        k, n = self.cfg.k, self.ds.n
        obj = C.c_double()
        wk = C.c_int64()
        Cb = np.empty((k, n))
        fb = np.empty(k, dtype=np.uint8)
        check(lib.hpcg_engine_export_best(self.h, C.byref(obj), C.byref(wk), ptr(Cb), ptr(fb)))
        return obj.value, wk.value, Cb, fb

    def finish(self) -> ClusteringResult:
        k, n, W, m = self.cfg.k, self.ds.n, self.W, self.ds.m
        out = _lib.RunOut()
        cent = np.empty((k, n))
        flags = np.empty(k, dtype=np.uint8)
        labels = np.empty(m, dtype=np.int32) if self.cfg.compute_assignment else None
        rounds = max(self.round_index, self.cfg.max_samples)
        wobj = np.empty(W)
        tcap = max(1, rounds)
        traces = np.empty((W, tcap, 2))
        tlen = np.zeros(W, dtype=np.int64)
        # the publication log in the same call when its size has a bound known here: at most W records per
        # round plus the hybrid carry-over (one rank, round-granular schedules)
        bounded = self._nranks == 1 and not self.cfg.free_running
        pcap = (rounds + 1) * W if bounded else 0
        pubs = np.empty((max(1, pcap), 4)) if bounded else None
        check(lib.hpcg_engine_finish(self.h, C.byref(out), ptr(cent), ptr(flags), ptr(labels), ptr(pubs), pcap,
                                     ptr(wobj), ptr(traces), tcap, ptr(tlen)))
        if not bounded:
            pubs = self.publications()
        return _result(out, cent, flags, labels, pubs, wobj, traces, tlen)

    def publications(self) -> np.ndarray:
        """SharedBest::publication_log (engine.hpp:149-152): rows (version, worker, objective, timestamp)."""
        n = C.c_int64()
        check(lib.hpcg_engine_publications(self.h, None, 0, C.byref(n)))
        pubs = np.zeros((max(1, n.value), 4))
        check(lib.hpcg_engine_publications(self.h, ptr(pubs), n.value, None))
        return pubs[: n.value]

    def close(self):
        if getattr(self, "h", None):
            lib.hpcg_engine_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _result(out, cent, flags, labels, pubs, wobj, traces, tlen) -> ClusteringResult:
    npub = int(out.n_publications)
    return ClusteringResult(
        centroids=cent, degenerate=flags,
        full_objective=float(out.full_objective) if out.has_full_objective else None,
        assignment=labels, best_worker=int(out.best_worker), best_sample_objective=float(out.best_sample_objective),
        clustering_time=float(out.clustering_time),
        clustering_time_first_finisher=float(out.clustering_time_first_finisher),
        wall_seconds=float(out.wall_seconds), total_samples=int(out.total_samples),
        distance_evals=int(out.distance_evals), worker_objectives=wobj,
        traces=_Traces(traces, tlen),
        publications=pubs[: min(npub, len(pubs))])


def run(X, cfg: EngineConfig, ctx: Context | None = None) -> ClusteringResult:
    """engine.hpp:444-499 — one call on host data (upload, rounds, final pass)."""
    ctx = ctx or default_context()
    X = np.ascontiguousarray(X)
    if cfg.time_limit > 0:  # round count unknown in advance: the stepwise engine sizes the outputs
        ds = DeviceDataset(X, ctx=ctx)
        eng = Engine(ds, cfg)
        try:
            eng.run()
            return eng.finish()
        finally:
            eng.close()
            ds.close()
    m, n = X.shape
    c = cfg.to_c()
    W = 1 if cfg.strategy == "inner" else cfg.n_workers
    out = _lib.RunOut()
    cent = np.empty((cfg.k, n))
    flags = np.empty(cfg.k, dtype=np.uint8)
    labels = np.empty(m, dtype=np.int32) if cfg.compute_assignment else None
    pub_cap = (cfg.max_samples + 1) * W  # at most W publications per round (+ the hybrid carry-over)
    pubs = np.zeros((pub_cap, 4))
    wobj = np.empty(W)
    tcap = max(1, cfg.max_samples)
    traces = np.zeros((W, tcap, 2))
    tlen = np.zeros(W, dtype=np.int64)
    check(lib.hpcg_run(ctx.h, ptr(X), _dtype_code(X), m, n, C.byref(c), C.byref(out), ptr(cent), ptr(flags),
                       ptr(labels), ptr(pubs), pub_cap, ptr(wobj), ptr(traces), tcap, ptr(tlen)))
    return _result(out, cent, flags, labels, pubs, wobj, traces, tlen)


def allgather_callback(allgather, nranks: int):
    """hpcg_allgather_fn over a Python collective: allgather(bytes) -> every rank's bytes in rank order."""
    def _cb(send, recv, nbytes, user):
        try:
            out = allgather(C.string_at(send, nbytes))
            if len(out) != nbytes * nranks:
                return 1
            C.memmove(recv, out, len(out))
            return 0
        except Exception:
            return 1
    return _lib.ALLGATHER_FN(_cb)


def gloo_allgather(group=None):
    """allgather(bytes) -> bytes over torch.distributed (any backend that gathers CPU uint8 tensors)."""
    import torch
    import torch.distributed as dist

    def ag(b: bytes) -> bytes:
        t = torch.frombuffer(bytearray(b), dtype=torch.uint8)
        outs = [torch.empty_like(t) for _ in range(dist.get_world_size(group))]
        dist.all_gather(outs, t, group=group)
        return b"".join(bytes(o.numpy()) for o in outs)
    return ag


def comm_unique_id() -> bytes:
    """NCCL unique id (128 bytes) for Context.attach_comm; created on one rank, shared by the caller."""
    buf = C.create_string_buffer(128)
    check(lib.hpcg_comm_unique_id(buf))
    return buf.raw


def philox_seed_draws(key: int, round_: int, worker: int, s: int, no_valid: bool, loops: int, candidates: int = 3):
    """The K-means++ draws an rng="philox" round gives a worker (hpcg_philox_seed_draws)."""
    fr = C.c_int64()
    units = np.empty(max(1, loops * candidates))
    check(lib.hpcg_philox_seed_draws(C.c_uint64(key), round_, worker, s, int(no_valid), loops, candidates,
                                     C.byref(fr), ptr(units)))
    return fr.value, units[: loops * candidates]


def gen_mixture(m, n, means, sigmas, weights=None, noise_frac=0.0, noise_box=(0.0, 1.0), seed=0,
                dtype=np.float32, threads=0) -> np.ndarray:
    """Seeded synthetic Gaussian mixture (BASELINE.json configs), keyed by row index."""
    means = np.ascontiguousarray(means, dtype=np.float64)
    sigmas = np.ascontiguousarray(sigmas, dtype=np.float64)
    w = None if weights is None else np.ascontiguousarray(weights, dtype=np.float64)
    X = np.empty((m, n), dtype=dtype)
    check(lib.hpcg_gen_mixture(ptr(X), _lib.F32 if dtype == np.float32 else _lib.F64, m, n, means.shape[0],
                               ptr(means), ptr(sigmas), ptr(w), noise_frac, noise_box[0], noise_box[1],
                               C.c_uint64(seed), threads))
    return X
