// Dependent-chain latency probe (cycles per op, single warp).
#include <cstdio>
#include <cuda_runtime.h>
constexpr int N = 4096;
__global__ void lat_dadd(double* o, double a, long long* c) {
    double x = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < N; ++i) x = x + a;
    long long t1 = clock64();
    if (threadIdx.x == 0) { c[0] = t1 - t0; o[0] = x; }
}
__global__ void lat_dfma(double* o, double a, long long* c) {
    double x = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < N; ++i) x = fma(x, a, 0.5);
    long long t1 = clock64();
    if (threadIdx.x == 0) { c[0] = t1 - t0; o[0] = x; }
}
__global__ void lat_ffma(float* o, float a, long long* c) {
    float x = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < N; ++i) x = fmaf(x, a, 0.5f);
    long long t1 = clock64();
    if (threadIdx.x == 0) { c[0] = t1 - t0; o[0] = x; }
}
__global__ void lat_ffma2(float* o, float a, long long* c) {
    float2 x = make_float2(threadIdx.x, 1.f), A = make_float2(a, a), B = make_float2(0.5f, 0.5f);
    long long t0 = clock64();
    for (int i = 0; i < N; ++i) x = __ffma2_rn(x, A, B);
    long long t1 = clock64();
    if (threadIdx.x == 0) { c[0] = t1 - t0; o[0] = x.x + x.y; }
}
__global__ void lat_f2f(double* o, float a, long long* c) {
    float x = threadIdx.x * a;
    long long t0 = clock64();
    for (int i = 0; i < N; ++i) { double d = (double)x; x = (float)(d * 1.0000001); }
    long long t1 = clock64();
    if (threadIdx.x == 0) { c[0] = t1 - t0; o[0] = x; }
}
__global__ void lat_lds(int* o, long long* c) {
    __shared__ int s[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = (i * 7 + 1) & 1023;
    __syncthreads();
    int p = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < N; ++i) p = s[p];
    long long t1 = clock64();
    if (threadIdx.x == 0) { c[0] = t1 - t0; o[0] = p; }
}
__global__ void lat_shfl(double* o, long long* c) {
    double v = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < N; ++i) v = __shfl_xor_sync(0xffffffffu, v, 1) + 1.0;
    long long t1 = clock64();
    if (threadIdx.x == 0) { c[0] = t1 - t0; o[0] = v; }
}
int main() {
    double* d; float* f; int* ip; long long* c; long long h;
    cudaMalloc(&d, 64); cudaMalloc(&f, 64); cudaMalloc(&ip, 64); cudaMalloc(&c, 64);
#define RUN(name, launch) launch; cudaDeviceSynchronize(); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("%-8s %.1f cycles/op\n", name, (double)h / N);
    RUN("DADD", (lat_dadd<<<1, 32>>>(d, 1.0000001, c)));
    RUN("DFMA", (lat_dfma<<<1, 32>>>(d, 1.0000001, c)));
    RUN("FFMA", (lat_ffma<<<1, 32>>>(f, 1.0000001f, c)));
    RUN("FFMA2", (lat_ffma2<<<1, 32>>>(f, 1.0000001f, c)));
    RUN("F2F+DMUL+F2F", (lat_f2f<<<1, 32>>>(d, 1.0f, c)));
    RUN("LDS", (lat_lds<<<1, 32>>>(ip, c)));
    RUN("SHFL+DADD", (lat_shfl<<<1, 32>>>(d, c)));
    return 0;
}
