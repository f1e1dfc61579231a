// Pipe-peak microbenchmarks for the roofline denominators of this repo:
// FFMA (fp32 SIMT), DFMA (fp64 SIMT), DMMA (mma.sync m8n8k4 f64) and
// mma.sync m16n8k8 tf32.  Prints one JSON line per pipe.
#include <cstdio>
#include <cuda_runtime.h>

#define ITERS 4096

__global__ void k_ffma(float* out, float a) {
  float x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x + i;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fmaf(x[i], a, 0.5f);
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i];
  if (s == 1.2345f) out[0] = s;
}
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  unsigned long long ua = *reinterpret_cast<unsigned long long*>(&a), ub = *reinterpret_cast<unsigned long long*>(&b),
                     uc = *reinterpret_cast<unsigned long long*>(&c), d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(ua), "l"(ub), "l"(uc));
  return *reinterpret_cast<float2*>(&d);
}
__global__ void k_ffma2(float* out, float a) {
  float2 x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = make_float2(threadIdx.x + i, i);
  const float2 aa = make_float2(a, a), h = make_float2(0.5f, 0.5f);
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = ffma2(x[i], aa, h);
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i].x + x[i].y;
  if (s == 1.2345f) out[0] = s;
}
__global__ void k_dfma(double* out, double a) {
  double x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x + i;
  for (int it = 0; it < ITERS / 4; ++it)
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fma(x[i], a, 0.5);
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i];
  if (s == 1.2345) out[0] = s;
}
__global__ void k_dmma(double* out) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = i * 0.1 + threadIdx.x; c[i][1] = i * 0.3 - threadIdx.x; }
  for (int it = 0; it < ITERS / 16; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 1.2345) out[0] = s;
}
__global__ void k_tf32(float* out) {
  unsigned a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = a0 * 3, b1 = a0 * 5;
  float c[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = i; c[i][1] = i + threadIdx.x; c[i][2] = -i; c[i][3] = i * 0.5f; }
  for (int it = 0; it < ITERS / 16; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(c[i][0]), "+f"(c[i][1]), "+f"(c[i][2]), "+f"(c[i][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 1.2345f) out[0] = s;
}

template <typename K>
float timeit(K launch) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  launch();
  cudaError_t err = cudaDeviceSynchronize();
  if (err != cudaSuccess || cudaGetLastError() != cudaSuccess) {
    printf("{\"error\": \"%s\"}\n", cudaGetErrorString(err));
    return -1.f;
  }
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* fo; double* dO;
  cudaMalloc(&fo, 64); cudaMalloc(&dO, 64);
  const int blocks = sms * 8, threads = 256;
  double nthr = (double)blocks * threads;
  float t;
  t = timeit([&] { k_ffma<<<blocks, threads>>>(fo, 0.999f); });
  printf("{\"pipe\": \"ffma_fp32\", \"tflops\": %.2f, \"ms\": %.3f}\n", nthr * ITERS * 16 * 2 / (t * 1e-3) / 1e12, t);
  t = timeit([&] { k_ffma2<<<blocks, threads>>>(fo, 0.999f); });
  printf("{\"pipe\": \"ffma2_fp32x2\", \"tflops\": %.2f, \"ms\": %.3f}\n", nthr * ITERS * 16 * 2 / (t * 1e-3) / 1e12, t);
  t = timeit([&] { k_dfma<<<blocks, threads>>>(dO, 0.999); });
  printf("{\"pipe\": \"dfma_fp64\", \"tflops\": %.2f, \"ms\": %.3f}\n", nthr * (ITERS / 4) * 16 * 2 / (t * 1e-3) / 1e12, t);
  t = timeit([&] { k_dmma<<<blocks, threads>>>(dO); });
  double warps = nthr / 32;
  printf("{\"pipe\": \"dmma_m8n8k4_fp64\", \"tflops\": %.2f, \"ms\": %.3f}\n", warps * (ITERS / 16) * 8 * 512 / (t * 1e-3) / 1e12, t);
  t = timeit([&] { k_tf32<<<blocks, threads>>>(fo); });
  printf("{\"pipe\": \"mma_sync_m16n8k8_tf32\", \"tflops\": %.2f, \"ms\": %.3f}\n", warps * (ITERS / 16) * 8 * 2048 / (t * 1e-3) / 1e12, t);
  printf("{\"sms\": %d, \"clock_khz\": %d}\n", sms, clk);
  return 0;
}
