// Internal launch interface between the host runtime (runtime.cu) and the kernel
// translation units (step_f32.cu, step_f64.cu, objective.cu).
#pragma once
#include <cstdint>
#include <string>
#include <cuda_runtime.h>

#include "step_kernel.cuh"
#include "objective_kernel.cuh"

namespace hpcg {

// Padded smem row widths with a compiled kernel. n -> smallest NP >= n.
int pick_np(int dtype, int n);  // dtype 0 f32, 1 f64; returns 0 if unsupported

struct StepGeometry {
    int cluster = 0;    // CTAs per worker
    int rows_cap = 0;   // max rows per CTA
    int smem = 0;       // dynamic smem bytes
    int active_clusters = 0;
};

// Chooses the cluster size (smallest that fits the sample in smem, widened while the
// occupancy API reports more SMs in use) and launches W clusters. Returns a CUDA error.
cudaError_t launch_step(int dtype, const StepParams& p, cudaStream_t st, StepGeometry* geo_out, std::string* why);
cudaError_t step_geometry(int dtype, int n, int64_t s, int k, int ncand, int W, StepGeometry* g, std::string* why);

// Grid-wide worker step over samples materialised in HBM (wide.cu): any n, k (k*n <= kWideMaxKN),
// any s. launch_step falls back to it when the cluster-resident kernel cannot hold the shape.
constexpr int64_t kWideMaxKN = 16384;
constexpr int64_t kInnerWideRows = 65536;  // W == 1 from this sample size on: the grid-wide path
constexpr int kWideMaxN = 4096, kWideMaxK = 4096;
cudaError_t launch_step_wide(int dtype, const StepParams& p, cudaStream_t st, std::string* why);
cudaError_t launch_objective_wide(int dtype, const ObjParams& p, int* nblocks, cudaStream_t st);

// *nblocks: in = capacity of p.block_cost, out = grid used (fixed per device/kernel/kv)
cudaError_t launch_objective(int dtype, const ObjParams& p, int* nblocks, cudaStream_t st);
bool objective_device_kv(int dtype, int n, int kv);  // resident kernel (honours kv_dev)?
int objective_blocks();  // fixed grid for deterministic block partials

}  // namespace hpcg
