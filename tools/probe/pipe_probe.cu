// Micro-probe of sm_100a issue/pipe rates that decide the Lloyd kernel design:
// FFMA vs FFMA2 (packed f32x2), F2F.F64.F32, DADD, IMNMX mix, and cluster barrier cost.
#include <cstdio>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

constexpr int ITERS = 4096;

__global__ void k_ffma(float* out, float a, float b) {
  float x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fmaf(x[i], a, b);
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 1234.5f) out[0] = s;
}
__global__ void k_ffma2(float* out, float a, float b) {
  float2 x[8]; float2 A = make_float2(a, a), B = make_float2(b, b);
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = make_float2(threadIdx.x + i, i);
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = __ffma2_rn(x[i], A, B);
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += x[i].x + x[i].y;
  if (s == 1234.5f) out[0] = s;
}
// FFMA2 + 1 integer min per 4 FFMA2 (argmin-like mix)
__global__ void k_ffma2_imnmx(float* out, float a, float b) {
  float2 x[8]; float2 A = make_float2(a, a), B = make_float2(b, b);
  unsigned m0 = 0xffffffffu, m1 = 0xffffffffu;
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = make_float2(threadIdx.x + i, i);
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = __ffma2_rn(x[i], A, B);
    m0 = min(m0, __float_as_uint(x[0].x) | 3u);
    m1 = min(m1, max(m0, __float_as_uint(x[4].y) | 5u));
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += x[i].x + x[i].y;
  if (s == 1234.5f || m1 == 7) out[0] = s + m0;
}
__global__ void k_f2f_dadd(double* out, float a) {
  double acc[8]; float v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { acc[i] = i; v[i] = threadIdx.x * a + i; }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) { acc[i] += (double)v[i]; v[i] = __int_as_float(__float_as_int(v[i]) ^ 1); }
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += acc[i];
  if (s == 1234.5) out[0] = s;
}
__global__ void k_dadd(double* out, double a) {
  double acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = i + threadIdx.x;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] += a;
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += acc[i];
  if (s == 1234.5) out[0] = s;
}
__global__ void k_dfma(double* out, double a, double b) {
  double acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = i + threadIdx.x;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += acc[i];
  if (s == 1234.5) out[0] = s;
}
// cluster barrier round trip cost (8-CTA cluster), ITERS/16 barriers
__global__ void __cluster_dims__(8, 1, 1) k_cluster_sync(unsigned long long* out) {
  cg::cluster_group cl = cg::this_cluster();
  unsigned long long t0 = clock64();
  for (int it = 0; it < ITERS / 16; ++it) cl.sync();
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
}

template <typename F>
float time_it(F f) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); cudaDeviceSynchronize();
  cudaEventRecord(a); for (int r = 0; r < 5; ++r) f(); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); return ms / 5;
}

int main() {
  int sms, clk; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs %d max clock %d kHz\n", sms, clk);
  float* fo; double* dout; unsigned long long* uo;
  CK(cudaMalloc(&fo, 64)); CK(cudaMalloc(&dout, 64)); CK(cudaMalloc(&uo, 64));
  const int blocks = sms * 4, threads = 256;
  double lanes_ops = (double)blocks * threads * ITERS * 8;
  float ms;
  ms = time_it([&] { k_ffma<<<blocks, threads>>>(fo, 1.0001f, 0.5f); });
  printf("FFMA    : %.3f ms  %.2f TFMA/s\n", ms, lanes_ops / ms / 1e9);
  ms = time_it([&] { k_ffma2<<<blocks, threads>>>(fo, 1.0001f, 0.5f); });
  printf("FFMA2   : %.3f ms  %.2f TFMA/s (2 per lane-op)\n", ms, 2 * lanes_ops / ms / 1e9);
  ms = time_it([&] { k_ffma2_imnmx<<<blocks, threads>>>(fo, 1.0001f, 0.5f); });
  printf("FFMA2+3ALU/8: %.3f ms  %.2f TFMA/s\n", ms, 2 * lanes_ops / ms / 1e9);
  ms = time_it([&] { k_f2f_dadd<<<blocks, threads>>>(dout, 1.0001f); });
  printf("F2F+DADD: %.3f ms  %.2f T(cvt+add)/s\n", ms, lanes_ops / ms / 1e9);
  ms = time_it([&] { k_dadd<<<blocks, threads>>>(dout, 1.0001); });
  printf("DADD    : %.3f ms  %.2f TDADD/s\n", ms, lanes_ops / ms / 1e9);
  ms = time_it([&] { k_dfma<<<blocks, threads>>>(dout, 1.0001, 0.5); });
  printf("DFMA    : %.3f ms  %.2f TDFMA/s\n", ms, lanes_ops / ms / 1e9);
  k_cluster_sync<<<8 * 18, 256>>>(uo); CK(cudaDeviceSynchronize());
  unsigned long long cyc; cudaMemcpy(&cyc, uo, 8, cudaMemcpyDeviceToHost);
  printf("cluster(8) sync: %.1f cycles each\n", (double)cyc / (ITERS / 16));
  CK(cudaGetLastError());
  return 0;
}
