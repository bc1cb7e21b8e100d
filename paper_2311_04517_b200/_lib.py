"""ctypes binding of libhpcg.so (the C-ABI in include/hpcg.h).

The library is built in-tree (``paper_2311_04517_b200/libhpcg.so``, see
``__graft_entry__.build``). There is no fallback: if the library is missing this module
raises ImportError, and every compute call fails with CudaError without an sm_100 device.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(os.environ.get("HPCG_LIB_OVERRIDE") or (Path(__file__).resolve().parent / "libhpcg.so"))  # dev A/B

# Every symbol include/hpcg.h declares (checked by tests/test_abi.py).
ABI_VERSION = 2  # include/hpcg.h HPCG_ABI_VERSION

EXPORTS = (
    "hpcg_last_error", "hpcg_abi_version", "hpcg_ctx_create", "hpcg_ctx_destroy", "hpcg_ctx_set_stream",
    "hpcg_ctx_synchronize", "hpcg_ctx_launch_count", "hpcg_dataset_upload", "hpcg_dataset_wrap",
    "hpcg_dataset_wrap_sharded", "hpcg_ipc_export", "hpcg_ipc_open", "hpcg_ipc_close",
    "hpcg_dataset_destroy", "hpcg_dataset_device_ptr", "hpcg_assign", "hpcg_assign_dev",
    "hpcg_worker_step_batched", "hpcg_gather", "hpcg_sample_indices", "hpcg_reference_draw_indices", "hpcg_rng_seed",
    "hpcg_rng_derive", "hpcg_rng_draw", "hpcg_engine_create", "hpcg_engine_rounds", "hpcg_engine_run", "hpcg_engine_round_index",
    "hpcg_engine_distance_evals", "hpcg_engine_finish", "hpcg_engine_destroy", "hpcg_engine_export_best",
    "hpcg_run", "hpcg_gen_mixture", "hpcg_ctx_enable_timing", "hpcg_ctx_kernel_times", "hpcg_probe_fma_peak",
    "hpcg_engine_reset", "hpcg_engine_import_best", "hpcg_engine_set_trace", "hpcg_engine_worker_incumbents",
    "hpcg_engine_publications", "hpcg_sample_gather_dev", "hpcg_philox_seed_draws", "hpcg_engine_round_outcome",
    "hpcg_engine_philox_key", "hpcg_comm_unique_id", "hpcg_ctx_attach_comm", "hpcg_ctx_comm_info",
    "hpcg_engine_set_exchange", "hpcg_ctx_upload_bytes", "hpcg_ctx_set_fp32_cost", "hpcg_host_register",
    "hpcg_host_unregister", "hpcg_engine_worker_progress",
)

HPCG_OK, HPCG_EINVAL, HPCG_ELOGIC, HPCG_ENOSOL, HPCG_ECUDA, HPCG_ENCCL, HPCG_EUNSUPPORTED = range(7)
F32, F64 = 0, 1
INNER, COMPETITIVE, COOPERATIVE, HYBRID = range(4)
RNG_REFERENCE, RNG_PHILOX = 0, 1


class HpcgError(RuntimeError):
    """Base class; `.status` holds the hpcg_status code."""

    status = -1


class InvalidArgument(HpcgError, ValueError):
    """The reference's std::invalid_argument (core.hpp:17-19 require())."""

    status = HPCG_EINVAL


class LogicError(HpcgError):
    """The reference's std::logic_error (lloyd.hpp:118, engine.hpp:259)."""

    status = HPCG_ELOGIC


class NoSolutionError(HpcgError):
    """engine.hpp:159-161."""

    status = HPCG_ENOSOL


class CudaError(HpcgError):
    status = HPCG_ECUDA


class NcclError(HpcgError):
    status = HPCG_ENCCL


class Unsupported(HpcgError, NotImplementedError):
    status = HPCG_EUNSUPPORTED


_ERRORS = {HPCG_EINVAL: InvalidArgument, HPCG_ELOGIC: LogicError, HPCG_ENOSOL: NoSolutionError,
           HPCG_ECUDA: CudaError, HPCG_ENCCL: NcclError, HPCG_EUNSUPPORTED: Unsupported}


class LloydCfg(C.Structure):
    _fields_ = [("max_iters", C.c_int64), ("rel_tol", C.c_double), ("candidates", C.c_int64)]


class EngineCfg(C.Structure):
    _fields_ = [("k", C.c_int64), ("sample_size", C.c_int64), ("n_workers", C.c_int64),
                ("max_samples", C.c_int64), ("strategy", C.c_int32), ("phase_t1", C.c_double),
                ("phase_t2", C.c_double), ("master_seed", C.c_uint64), ("candidates", C.c_int64),
                ("max_iters", C.c_int64), ("rel_tol", C.c_double), ("compute_full_objective", C.c_int32),
                ("compute_assignment", C.c_int32), ("rng_mode", C.c_int32), ("worker_base", C.c_int32),
                ("time_limit", C.c_double), ("free_running", C.c_int32), ("free_group", C.c_int32)]


class RunOut(C.Structure):
    _fields_ = [("full_objective", C.c_double), ("has_full_objective", C.c_int32), ("best_worker", C.c_int32),
                ("best_sample_objective", C.c_double), ("clustering_time", C.c_double),
                ("clustering_time_first_finisher", C.c_double), ("wall_seconds", C.c_double),
                ("total_samples", C.c_uint64), ("distance_evals", C.c_int64), ("n_publications", C.c_int64),
                ("last_timestamp", C.c_double)]


# host all-gather callback of a multi-rank engine (include/hpcg.h hpcg_allgather_fn)
ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)


def _load():
    if not LIB_PATH.exists():
        raise ImportError(f"{LIB_PATH} is not built (run __graft_entry__.build()); there is no CPU fallback")
    lib = C.CDLL(str(LIB_PATH))
    lib.hpcg_abi_version.restype = C.c_int
    if lib.hpcg_abi_version() != ABI_VERSION:  # the structs below mirror one layout of include/hpcg.h
        raise ImportError(f"{LIB_PATH} has ABI version {lib.hpcg_abi_version()}, this binding expects {ABI_VERSION}: "
                          "rebuild with __graft_entry__.build()")
    P, I64, I32, U64, D = C.c_void_p, C.c_int64, C.c_int32, C.c_uint64, C.c_double
    sig = {
        "hpcg_last_error": (C.c_char_p, []),
        "hpcg_abi_version": (C.c_int, []),
        "hpcg_ctx_create": (C.c_int, [C.c_int, P]),
        "hpcg_ctx_destroy": (C.c_int, [P]),
        "hpcg_ctx_set_stream": (C.c_int, [P, P]),
        "hpcg_ctx_synchronize": (C.c_int, [P]),
        "hpcg_ctx_launch_count": (I64, [P]),
        "hpcg_ctx_upload_bytes": (I64, [P]),
        "hpcg_ctx_set_fp32_cost": (C.c_int, [P, C.c_int]),
        "hpcg_dataset_upload": (C.c_int, [P, P, C.c_int, I64, I64, P]),
        "hpcg_dataset_wrap_sharded": (C.c_int, [P, P, P, C.c_int32, C.c_int, I64, P]),
        "hpcg_ipc_export": (C.c_int, [P, P]),
        "hpcg_ipc_open": (C.c_int, [P, P, P]),
        "hpcg_ipc_close": (C.c_int, [P, P, P]),
        "hpcg_host_register": (C.c_int, [P, C.c_int64]),
        "hpcg_host_unregister": (C.c_int, [P]),
        "hpcg_engine_worker_progress": (C.c_int, [P, P, P]),
        "hpcg_dataset_wrap": (C.c_int, [P, P, C.c_int, I64, I64, P]),
        "hpcg_dataset_destroy": (C.c_int, [P]),
        "hpcg_dataset_device_ptr": (P, [P]),
        "hpcg_assign": (C.c_int, [P, P, P, P, I64, C.c_int, P, P, P, P]),
        "hpcg_assign_dev": (C.c_int, [P, P, P, I64, P, P]),
        "hpcg_worker_step_batched": (C.c_int, [P, P, P, I64, I64, P, P, I64, P, P, P, I64, C.c_int, P, P, P, P,
                                               P, P, P, P, P, P, I32, P]),
        "hpcg_gather": (C.c_int, [P, P, P, I64, P]),
        "hpcg_sample_indices": (C.c_int, [P, I64, I64, C.c_uint64, C.c_uint32, C.c_uint32, P]),
        "hpcg_reference_draw_indices": (C.c_int, [P, P, I64, I64, P]),
        "hpcg_rng_seed": (C.c_int, [U64, P, P]),
        "hpcg_rng_derive": (C.c_int, [U64, U64, U64, P, P]),
        "hpcg_rng_draw": (C.c_int, [P, P, I32, U64, I64, P]),
        "hpcg_engine_create": (C.c_int, [P, P, P, P]),
        "hpcg_engine_rounds": (C.c_int, [P, I64]),
        "hpcg_engine_run": (C.c_int, [P]),
        "hpcg_engine_round_index": (I64, [P]),
        "hpcg_engine_distance_evals": (C.c_int, [P, P]),
        "hpcg_engine_finish": (C.c_int, [P, P, P, P, P, P, I64, P, P, I64, P]),
        "hpcg_engine_destroy": (C.c_int, [P]),
        "hpcg_engine_export_best": (C.c_int, [P, P, P, P, P]),
        "hpcg_run": (C.c_int, [P, P, C.c_int, I64, I64, P, P, P, P, P, P, I64, P, P, I64, P]),
        "hpcg_gen_mixture": (C.c_int, [P, C.c_int, I64, I64, I64, P, P, P, D, D, D, U64, C.c_int]),
        "hpcg_ctx_enable_timing": (C.c_int, [P, C.c_int]),
        "hpcg_ctx_kernel_times": (C.c_int, [P, P, P]),
        "hpcg_probe_fma_peak": (C.c_int, [P, P]),
        "hpcg_engine_reset": (C.c_int, [P, U64]),
        "hpcg_engine_import_best": (C.c_int, [P, D, I64, P, P]),
        "hpcg_engine_set_trace": (C.c_int, [P, P, I32]),
        "hpcg_engine_worker_incumbents": (C.c_int, [P, P, P, P]),
        "hpcg_engine_publications": (C.c_int, [P, P, I64, P]),
        "hpcg_sample_gather_dev": (C.c_int, [P, P, I64, I64, U64, C.c_uint32, I32, P]),
        "hpcg_philox_seed_draws": (C.c_int, [U64, C.c_uint32, C.c_uint32, I64, I32, I64, I64, P, P]),
        "hpcg_engine_round_outcome": (C.c_int, [P, P, P, P, P, P, P]),
        "hpcg_engine_philox_key": (U64, [P]),
        "hpcg_comm_unique_id": (C.c_int, [P]),
        "hpcg_ctx_attach_comm": (C.c_int, [P, I32, I32, P]),
        "hpcg_ctx_comm_info": (C.c_int, [P, P, P]),
        "hpcg_engine_set_exchange": (C.c_int, [P, I32, I32, ALLGATHER_FN, P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


lib = _load()


def check(rc: int) -> None:
    if rc != HPCG_OK:
        msg = lib.hpcg_last_error().decode()
        raise _ERRORS.get(rc, HpcgError)(msg)


def ptr(a) -> int | None:
    """Data pointer of a numpy array (or None)."""
    if a is None:
        return None
    return a.ctypes.data_as(C.c_void_p).value


os.environ.setdefault("HPCG_LIB", str(LIB_PATH))
