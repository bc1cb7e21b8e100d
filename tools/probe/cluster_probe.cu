// Resident clusters of a 512-thread, 128-register, ~227 KB shared-memory CTA (the worker step's footprint)
// for cluster sizes 1..16: cudaOccupancyMaxActiveClusters on this device.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(512, 1) probe(float* out) {
    extern __shared__ float sm[];
    float acc[96];
#pragma unroll
    for (int i = 0; i < 96; ++i) acc[i] = sm[(threadIdx.x + i) & 1023] * (float)i;
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 96; ++i) s += acc[i] * acc[(i + 7) % 96];
    if (out) out[threadIdx.x] = s;
}
int main() {
    for (int smem : {188000, 209360, 232448 - 8192}) {
        cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        printf("smem %d:", smem);
        for (int c = 1; c <= 16; ++c) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(c * 64);
            cfg.blockDim = dim3(512);
            cfg.dynamicSmemBytes = smem;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = c;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            int n = -1;
            cudaError_t e = cudaOccupancyMaxActiveClusters(&n, probe, &cfg);
            if (e != cudaSuccess) { cudaGetLastError(); n = -1; }
            printf(" c%d=%d(%d SMs)", c, n, n * c);
        }
        printf("\n");
    }
    return 0;
}
