// Pipe-peak microbenchmarks for the roofline denominators of this repo:
// FFMA (fp32 SIMT), DFMA (fp64 SIMT), DMMA (mma.sync m8n8k4 f64),
// mma.sync m16n8k8 tf32, and the 5th-generation tensor core through
// tcgen05.mma (kind::i8 and kind::tf32, M = 128, N = 256, operands resident in
// shared memory, accumulators in TMEM, one issuing thread per CTA, one CTA per
// SM).  Prints one JSON line per pipe.
#include <cstdio>
#include <cstdint>
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
template <bool BF>
__global__ void k_h16(float* out) {  // mma.sync m16n8k16, f16 / bf16 inputs, f32 accumulate
  unsigned a0 = threadIdx.x * 0x00010001u, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = a0 * 3, b1 = a0 * 5;
  float c[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = i; c[i][1] = i + threadIdx.x; c[i][2] = -i; c[i][3] = i * 0.5f; }
  for (int it = 0; it < ITERS / 16; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if constexpr (BF)
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+f"(c[i][0]), "+f"(c[i][1]), "+f"(c[i][2]), "+f"(c[i][3])
                     : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
      else
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+f"(c[i][0]), "+f"(c[i][1]), "+f"(c[i][2]), "+f"(c[i][3])
                     : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 1.2345f) out[0] = s;
}

// ---- tcgen05.mma throughput: operands stay in shared memory (128B-swizzled,
// K-major), so the tensor pipe is the only thing measured ----
constexpr int TC_M = 128, TC_N = 256, TC_KB = 128;  // 128-byte k-tile: 4 (i8) / 4 (tf32) MMAs per tile
constexpr int TC_SMEM = (TC_M + TC_N) * TC_KB + 1024;
__device__ __forceinline__ uint32_t s_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t kdesc128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3fff);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
template <int KIND>  // 0 = i8 (K = 32 per MMA), 1 = tf32 (K = 8 per MMA)
__global__ void __launch_bounds__(128, 1) k_tcgen05(int iters, int* out) {
  extern __shared__ __align__(1024) unsigned char smraw[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  unsigned char* sm = (unsigned char*)(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
  for (int i = threadIdx.x; i < (TC_M + TC_N) * TC_KB / 4; i += blockDim.x) reinterpret_cast<int*>(sm)[i] = 0x01010101 * (i & 3);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(s_u32(&tbase)), "r"(TC_N));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tbase;
  if (threadIdx.x == 0) {
    const uint32_t idesc = KIND == 0 ? ((2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(TC_N >> 3) << 17) | ((uint32_t)(TC_M >> 4) << 24))
                                     : ((1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(TC_N >> 3) << 17) | ((uint32_t)(TC_M >> 4) << 24));
    const uint64_t ad = kdesc128(s_u32(sm)), bd = kdesc128(s_u32(sm + TC_M * TC_KB));
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint64_t a = ad + (uint64_t)((k * 32) >> 4), b = bd + (uint64_t)((k * 32) >> 4);
        const uint32_t acc = (it | k) ? 1u : 0u;
        if (KIND == 0)
          asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                       ::"r"(tmem), "l"(a), "l"(b), "r"(idesc), "r"(acc));
        else
          asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
                       ::"r"(tmem), "l"(a), "l"(b), "r"(idesc), "r"(acc));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(s_u32(&bar)) : "memory");
    asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W_%=;\n}\n" ::"r"(s_u32(&bar)) : "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) {
    uint32_t v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(tmem));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (v == 0x12345678u) out[0] = (int)v;
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TC_N));
  }
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
  t = timeit([&] { k_h16<false><<<blocks, threads>>>(fo); });
  printf("{\"pipe\": \"mma_sync_m16n8k16_f16\", \"tflops\": %.2f, \"ms\": %.3f}\n", warps * (ITERS / 16) * 8 * 4096 / (t * 1e-3) / 1e12, t);
  t = timeit([&] { k_h16<true><<<blocks, threads>>>(fo); });
  printf("{\"pipe\": \"mma_sync_m16n8k16_bf16\", \"tflops\": %.2f, \"ms\": %.3f}\n", warps * (ITERS / 16) * 8 * 4096 / (t * 1e-3) / 1e12, t);
  {
    int* io; cudaMalloc(&io, 64);
    cudaFuncSetAttribute(k_tcgen05<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, TC_SMEM);
    cudaFuncSetAttribute(k_tcgen05<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, TC_SMEM);
    const int it = 4096;
    t = timeit([&] { k_tcgen05<0><<<sms, 128, TC_SMEM>>>(it, io); });
    printf("{\"pipe\": \"tcgen05_i8_m128n256\", \"tops\": %.1f, \"tflops\": %.1f, \"ms\": %.3f}\n",
           (double)sms * it * 4 * 2.0 * TC_M * TC_N * 32 / (t * 1e-3) / 1e12,
           (double)sms * it * 4 * 2.0 * TC_M * TC_N * 32 / (t * 1e-3) / 1e12, t);
    t = timeit([&] { k_tcgen05<1><<<sms, 128, TC_SMEM>>>(it, io); });
    printf("{\"pipe\": \"tcgen05_tf32_m128n256\", \"tflops\": %.1f, \"ms\": %.3f}\n",
           (double)sms * it * 4 * 2.0 * TC_M * TC_N * 8 / (t * 1e-3) / 1e12, t);
  }
  printf("{\"sms\": %d, \"clock_khz\": %d}\n", sms, clk);
  return 0;
}
