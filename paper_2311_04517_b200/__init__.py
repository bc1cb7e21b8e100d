"""B200-native HPClust hot path (arXiv 2311.04517): sample gather, greedy K-means++
reseeding, batched Lloyd, incumbent selection and the full-data objective as sm_100a
kernels behind the C-ABI include/hpcg.h (libhpcg.so), with a Python mirror of the
reference's hpclust:: interface (api.py) and a C++ drop-in (include/hpclust/)."""
from ._lib import (CudaError, HpcgError, InvalidArgument, LogicError, NoSolutionError, Unsupported,  # noqa: F401
                   LIB_PATH)
from .api import (Assignment, ClusteringResult, Context, DeviceDataset, DistCounter, Engine,  # noqa: F401
                  EngineConfig, LloydConfig, LloydOutcome, RngStream, SeedConfig, assign_nearest,
                  assign_valid_subset, default_context, draw_sample, final_assignment, gen_mixture, kmeans,
                  ipc_close, ipc_export, ipc_open, kmeanspp_seed, mssc_objective, philox_sample_indices,
                  philox_seed_draws, comm_unique_id, allgather_callback, gloo_allgather,
                  reference_draw_indices, reinit_degenerate, run, select_best,
                  worker_step_batched)

__all__ = [n for n in dir() if not n.startswith("_")]
