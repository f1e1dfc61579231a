// api.cu -- the C ABI of libexpmb.so (declared in include/expmb.h).
//
// Validation mirrors the reference's error behaviour (select.py:72-79
// check_tolerance, matrix.py:52-55 shape checks, engine.py:137 unknown
// scheme); dispatch picks the fused small-n kernel (n <= 64) or the large-n
// GEMM pipeline (n > 64).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../../include/expmb.h"
#include "fused_small.cuh"
#include "fused_w16.cuh"
#include "fused_dmma.cuh"
#include "large.cuh"
#include "fused_tile.cuh"
#include "lowrank.cuh"
#include "lowrank_large.cuh"
#include "timegrid.cuh"

namespace expmb {

static int sm_count() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return 148;
  if (!cached[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    cached[dev] = v > 0 ? v : 148;
  }
  return cached[dev];
}

template <typename T, int NPAD, int TM, int GROUPS, int SCHEME, int MINB = ((NPAD == 16 && sizeof(T) == 4) ? 2 : 1),
          int VARIANT = 0>
static int launch_fused(const T* W, T* X, int64_t batch, int n, double eps, PlanOut po, int* ctr, cudaStream_t st) {
  using F = Fused<T, NPAD, TM, GROUPS, SCHEME, (VARIANT == 2)>;
  auto kern = expm_fused_kernel<T, NPAD, TM, GROUPS, SCHEME, MINB, VARIANT>;
  constexpr size_t smem = F::kSmem + (MINB >= 3 ? GROUPS * F::kStageBytes : 0);
  static int occ = -1;  // per instantiation; identical on every B200
  if (occ < 0) {
    if (smem > 48 * 1024 &&
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return EXPMB_ERR_CUDA;
    int o = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, F::NT, smem) != cudaSuccess || o < 1)
      return EXPMB_ERR_CUDA;
    occ = o;
  }
  const int64_t ctas_needed = (batch + GROUPS - 1) / GROUPS;
  const int64_t persistent = (int64_t)sm_count() * occ;
  const int grid = (int)(ctas_needed < persistent ? ctas_needed : persistent);
  if (grid <= 0) return EXPMB_OK;
  // log2(eps) on the host: the same libm log2 as the reference's math.log2 (select.py:175)
  if (ctr != nullptr && cudaMemsetAsync(ctr, 0, sizeof(int), st) != cudaSuccess) return EXPMB_ERR_CUDA;
  kern<<<grid, F::NT, smem, st>>>(W, X, batch, n, log2(eps), eps, po, ctr);
  return cudaGetLastError() == cudaSuccess ? EXPMB_OK : EXPMB_ERR_CUDA;
}

// fp64 Sastre, 32 < n <= 64: the DMMA (FP64 tensor core) fused kernel.
static int launch_dmma(const double* W, double* X, int64_t batch, int n, double eps, PlanOut po, int* ctr,
                       cudaStream_t st) {
  static int occ = -1;
  if (occ < 0) {
    if (cudaFuncSetAttribute(expm_dmma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Dm::kSmem) !=
        cudaSuccess)
      return EXPMB_ERR_CUDA;
    int o = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, expm_dmma_kernel, Dm::NT, Dm::kSmem) != cudaSuccess || o < 1)
      return EXPMB_ERR_CUDA;
    occ = o;
  }
  const int64_t persistent = (int64_t)sm_count() * occ;
  const int grid = (int)(batch < persistent ? batch : persistent);
  if (ctr != nullptr && cudaMemsetAsync(ctr, 0, sizeof(int), st) != cudaSuccess) return EXPMB_ERR_CUDA;
  expm_dmma_kernel<<<grid, Dm::NT, Dm::kSmem, st>>>(W, X, batch, n, log2(eps), po, ctr);
  return cudaGetLastError() == cudaSuccess ? EXPMB_OK : EXPMB_ERR_CUDA;
}

// fp32 Sastre, n == 16: the warp-batched kernel (fused_w16.cuh).
template <int Q, int MINB>
static int launch_w16_q(const float* W, float* X, int64_t batch, double eps, PlanOut po, cudaStream_t st) {
  auto kern = w16::expm_w16_kernel<Q, MINB>;
  constexpr size_t smem = w16::smem_bytes<Q>();
  static int occ = -1;
  if (occ < 0) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return EXPMB_ERR_CUDA;
    int o = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, w16::NT, smem) != cudaSuccess || o < 1)
      return EXPMB_ERR_CUDA;
    occ = o;
  }
  const int64_t warps_needed = (batch + Q - 1) / Q;
  const int64_t ctas_needed = (warps_needed + w16::WARPS - 1) / w16::WARPS;
  const int64_t persistent = (int64_t)sm_count() * occ;
  const int grid = (int)(ctas_needed < persistent ? ctas_needed : persistent);
  if (grid <= 0) return EXPMB_OK;
  kern<<<grid, w16::NT, smem, st>>>(W, X, batch, log2(eps), po);
  return cudaGetLastError() == cudaSuccess ? EXPMB_OK : EXPMB_ERR_CUDA;
}

static int launch_w16(const float* W, float* X, int64_t batch, double eps, PlanOut po, int*, cudaStream_t st) {
  // EXPMB_W16_Q: matrices per warp batch (A/B); 6 x 8 warps x 2 CTAs = 212 KB of shared memory per SM
  static const int q = getenv("EXPMB_W16_Q") ? atoi(getenv("EXPMB_W16_Q")) : 4;
  static const int minb = getenv("EXPMB_W16_MINB") ? atoi(getenv("EXPMB_W16_MINB")) : 2;
  if (q == 8) return minb == 3 ? launch_w16_q<8, 3>(W, X, batch, eps, po, st) : launch_w16_q<8, 2>(W, X, batch, eps, po, st);
  if (q == 2) return minb == 3 ? launch_w16_q<2, 3>(W, X, batch, eps, po, st) : launch_w16_q<2, 2>(W, X, batch, eps, po, st);
  if (minb == 3) return launch_w16_q<4, 3>(W, X, batch, eps, po, st);
  return launch_w16_q<4, 2>(W, X, batch, eps, po, st);
}

template <typename T, int SCHEME>
static int dispatch_small(const T* W, T* X, int64_t batch, int n, double eps, PlanOut po, int* ctr, cudaStream_t st) {
  // Sastre runs as straight-line code per order (VARIANT 1: 10% faster than
  // the step machine on C2); EXPMB_VARIANT=0 selects the step machine.
  static const bool straight = !(getenv("EXPMB_VARIANT") && getenv("EXPMB_VARIANT")[0] == '0');  // 1 and 2 are straight-line
  // warp-per-matrix: ~100 matrices per SM balance statically; the claim
  // atomics only added latency there (7% of stall samples).  EXPMB_CLAIM=1
  // forces dynamic claiming (A/B experiments).
  static const bool claim16 = getenv("EXPMB_CLAIM") && getenv("EXPMB_CLAIM")[0] == '1';
  static const int minb = getenv("EXPMB_C2_MINB") ? atoi(getenv("EXPMB_C2_MINB")) : 2;
  if constexpr (sizeof(T) == 4 && SCHEME == 0) {
    static const bool w16 = !(getenv("EXPMB_W16") && getenv("EXPMB_W16")[0] == '0');
    if (n == 16 && w16) return launch_w16(W, X, batch, eps, po, ctr, st);
  }
  if (n <= 16) {
    int* c16 = claim16 ? ctr : nullptr;
    // fp32 Sastre default: variant 2 (3xTF32 mma.sync products); 1 = FFMA2 straight-line, 0 = step machine
    static const int variant = getenv("EXPMB_VARIANT") ? atoi(getenv("EXPMB_VARIANT")) : 2;
    if constexpr (sizeof(T) == 4) {
      if (minb == 3) {
        if constexpr (SCHEME == 0) {
          if (variant == 2) return launch_fused<T, 16, 2, 8, SCHEME, 3, 2>(W, X, batch, n, eps, po, c16, st);
        }
        if (SCHEME == 0 && straight) return launch_fused<T, 16, 2, 8, SCHEME, 3, 1>(W, X, batch, n, eps, po, c16, st);
        return launch_fused<T, 16, 2, 8, SCHEME, 3>(W, X, batch, n, eps, po, c16, st);
      }
      if (minb == 4) {
        if (SCHEME == 0 && straight) return launch_fused<T, 16, 2, 8, SCHEME, 4, 1>(W, X, batch, n, eps, po, c16, st);
        return launch_fused<T, 16, 2, 8, SCHEME, 4>(W, X, batch, n, eps, po, c16, st);
      }
    }
    if constexpr (sizeof(T) == 4 && SCHEME == 0) {
      if (variant == 2) return launch_fused<T, 16, 2, 8, SCHEME, 2, 2>(W, X, batch, n, eps, po, c16, st);
    }
    if (SCHEME == 0 && straight) return launch_fused<T, 16, 2, 8, SCHEME, (sizeof(T) == 4 ? 2 : 1), 1>(W, X, batch, n, eps, po, c16, st);
    return launch_fused<T, 16, 2, 8, SCHEME>(W, X, batch, n, eps, po, c16, st);
  }
  if (n <= 32) {
    if (SCHEME == 0 && straight) return launch_fused<T, 32, 4, 4, SCHEME, 1, 1>(W, X, batch, n, eps, po, ctr, st);
    return launch_fused<T, 32, 4, 4, SCHEME>(W, X, batch, n, eps, po, ctr, st);
  }
  if constexpr (sizeof(T) == 8 && SCHEME == 0) {
    static const bool dmma = !(getenv("EXPMB_NO_DMMA") && getenv("EXPMB_NO_DMMA")[0] == '1');
    if (dmma) return launch_dmma(W, X, batch, n, eps, po, ctr, st);
  }
  if (SCHEME == 0 && straight) return launch_fused<T, 64, 4, 1, SCHEME, 1, 1>(W, X, batch, n, eps, po, ctr, st);
  return launch_fused<T, 64, 4, 1, SCHEME>(W, X, batch, n, eps, po, ctr, st);
}

}  // namespace expmb

using namespace expmb;

// Low-rank path (engine.py:198-257): one CTA per matrix, grid-strided.
template <typename T, int TP, typename TI = T>
static int launch_lowrank(const TI* A1, const TI* A2, TI* X, int64_t batch, int n, int t, double eps, LrOut po,
                          cudaStream_t st) {
  using L = Lr<T, TP>;
  auto kern = expm_lowrank_kernel<T, TP, TI>;
  static int occ = -1;
  if (occ < 0) {
    if (L::kSmem > 48 * 1024 &&
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::kSmem) != cudaSuccess)
      return EXPMB_ERR_CUDA;
    int o = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, L::NT, L::kSmem) != cudaSuccess || o < 1)
      return EXPMB_ERR_CUDA;
    occ = o;
  }
  const int64_t persistent = (int64_t)sm_count() * occ;
  const int grid = (int)(batch < persistent ? batch : persistent);
  kern<<<grid, L::NT, L::kSmem, st>>>(A1, A2, X, batch, n, t, log2(eps), po);
  return cudaGetLastError() == cudaSuccess ? EXPMB_OK : EXPMB_ERR_CUDA;
}

template <typename T, bool FULL>
static int launch_lowrank_warp(const T* A1, const T* A2, T* X, int64_t batch, int n, int t, double eps, LrOut po,
                               cudaStream_t st) {
  using L = LrW<T>;
  auto kern = expm_lowrank_warp_kernel<T, FULL>;
  static int occ = -1;
  if (occ < 0) {
    if (L::kSmem > 48 * 1024 &&
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::kSmem) != cudaSuccess)
      return EXPMB_ERR_CUDA;
    int o = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, L::NT, L::kSmem) != cudaSuccess || o < 1)
      return EXPMB_ERR_CUDA;
    occ = o;
  }
  const int64_t ctas = (batch + L::WARPS - 1) / L::WARPS;
  const int64_t persistent = (int64_t)sm_count() * occ;
  const int grid = (int)(ctas < persistent ? ctas : persistent);
  kern<<<grid, L::NT, L::kSmem, st>>>(A1, A2, X, batch, n, t, log2(eps), po);
  return cudaGetLastError() == cudaSuccess ? EXPMB_OK : EXPMB_ERR_CUDA;
}

template <typename TI, bool FULL>
static int launch_lowrank_dmma(const TI* A1, const TI* A2, TI* X, int64_t batch, int n, int t,
                               double eps, LrOut po, cudaStream_t st) {
  using L = LrD;
  auto kern = expm_lowrank_dmma_kernel<TI, FULL>;
  static int occ = -1;
  if (occ < 0) {
    if (L::kSmem > 48 * 1024 &&
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::kSmem) != cudaSuccess)
      return EXPMB_ERR_CUDA;
    int o = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, L::NT, L::kSmem) != cudaSuccess || o < 1)
      return EXPMB_ERR_CUDA;
    occ = o;
  }
  const int64_t ctas = (batch + L::WARPS - 1) / L::WARPS;
  const int64_t persistent = (int64_t)sm_count() * occ;
  const int grid = (int)(ctas < persistent ? ctas : persistent);
  kern<<<grid, L::NT, L::kSmem, st>>>(A1, A2, X, batch, n, t, log2(eps), po);
  return cudaGetLastError() == cudaSuccess ? EXPMB_OK : EXPMB_ERR_CUDA;
}

template <typename T>
static int dispatch_lowrank(const T* A1, const T* A2, T* X, int64_t batch, int n, int t, double eps, LrOut po,
                            cudaStream_t st) {
  static const bool cta_only = getenv("EXPMB_LR_CTA") != nullptr;   // A/B switches
  static const bool no_dmma = getenv("EXPMB_LR_NO_DMMA") != nullptr;
  // the warp kernels use 16-byte vector accesses of the factors / result
  const bool a16 = (((uintptr_t)A1 | (uintptr_t)A2 | (uintptr_t)X) % 16) == 0;
  // fp64 on DMMA; fp32 stays on the FFMA warp kernel (measured faster:
  // 97 vs 177 us at n = 64, t = 8 through the binary64 DMMA kernel)
  if (!cta_only && !no_dmma && t <= 8 && n <= 64 && (sizeof(T) == 8 || getenv("EXPMB_LR_F32_DMMA"))) {
    if constexpr (sizeof(T) == 8)
      if (a16 && t == 8 && n == 64) return launch_lowrank_dmma<T, true>(A1, A2, X, batch, n, t, eps, po, st);
    return launch_lowrank_dmma<T, false>(A1, A2, X, batch, n, t, eps, po, st);
  }
  if (!cta_only && a16 && t <= 8 && n <= 64) {
    if (t == 8 && n == 64) return launch_lowrank_warp<T, true>(A1, A2, X, batch, n, t, eps, po, st);
    return launch_lowrank_warp<T, false>(A1, A2, X, batch, n, t, eps, po, st);
  }
  if (t <= 8) return launch_lowrank<T, 8>(A1, A2, X, batch, n, t, eps, po, st);
  // fp32 t > 8: binary64 compute on the DMMA path (faster than the fp32 FFMA
  // instantiation, which EXPMB_LR_F32_FMA keeps for A/B)
  static const bool f32_fma = getenv("EXPMB_LR_F32_FMA") != nullptr;
  if (sizeof(T) == 4 && !f32_fma) {
    if (t <= 16) return launch_lowrank<double, 16, T>(A1, A2, X, batch, n, t, eps, po, st);
    return launch_lowrank<double, 32, T>(A1, A2, X, batch, n, t, eps, po, st);
  }
  if (t <= 16) return launch_lowrank<T, 16>(A1, A2, X, batch, n, t, eps, po, st);
  return launch_lowrank<T, 32>(A1, A2, X, batch, n, t, eps, po, st);
}

// W_k = t_k A materialised (time-grid path for n <= 64, where the fused
// per-matrix kernels are cheaper than shared powers).
template <typename T>
__global__ void k_tg_materialize(const T* __restrict__ A, const T* __restrict__ t, T* __restrict__ W, int64_t K,
                                 size_t nn) {
  const int64_t k = blockIdx.y;
  const T tk = t[k];
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < nn; i += (size_t)gridDim.x * blockDim.x)
    W[k * nn + i] = tk * A[i];
}

static size_t tg_small_bytes(int64_t K, int n, int esize) {
  return align256((size_t)K * n * n * esize) + 256;
}

extern "C" {

int expmb_version(void) { return 100; }

const char* expmb_strerror(int code) {
  switch (code) {
    case EXPMB_OK: return "ok";
    case EXPMB_ERR_TOLERANCE: return "tolerance NaN or below the unit roundoff of the dtype";
    case EXPMB_ERR_SHAPE: return "matrix order must be at least 1 and batch non-negative";
    case EXPMB_ERR_SCHEME: return "unknown scheme; expected sastre (0), ps (1) or baseline (2)";
    case EXPMB_ERR_DTYPE: return "dtype must be fp32 (0) or fp64 (1)";
    case EXPMB_ERR_WORKSPACE: return "workspace missing or smaller than expmb_workspace_bytes()";
    case EXPMB_ERR_CUDA: return "CUDA launch or copy failed";
    case EXPMB_ERR_ALIGN: return "W and X must be 16-byte aligned";
    case EXPMB_ERR_UNSUPPORTED:
      return "combination not supported";
    default: return "unknown error";
  }
}

double expmb_unit_roundoff(int dtype) { return dtype == EXPMB_F32 ? 0x1p-24 : 0x1p-53; }

// fp64, 64 < n <= EXPMB_FUSED_TILE_MAX (default 128): one CTA per matrix
// (fused_tile.cuh; measured 1.14-1.26x the pipeline).  EXPMB_FUSED_TILE=0
// sends those orders to the pipeline, =1 also routes fp32 there (0.85x: A/B only).
static bool use_fused_tile(int n, int scheme, int dtype) {
  const char* e = getenv("EXPMB_FUSED_TILE");
  static const int mode = e ? (e[0] == '0' ? 0 : 2) : 1;
  static const int nmax = getenv("EXPMB_FUSED_TILE_MAX") ? atoi(getenv("EXPMB_FUSED_TILE_MAX")) : 128;
  if (mode == 0 || (mode == 1 && dtype != EXPMB_F64)) return false;
  return n > 64 && n <= nmax && (scheme == EXPMB_SASTRE || scheme == EXPMB_PS);
}

size_t expmb_workspace_bytes(int64_t batch, int32_t n, int dtype, int scheme) {
  if (batch <= 0) return 0;
  if (n <= 64) return 256;  // work counter of the persistent fused kernel
  const int es = dtype == EXPMB_F32 ? 4 : 8;
  if (use_fused_tile(n, scheme, dtype)) return ft_workspace_bytes(batch, n, es, scheme, ft_ctas(es));
  return large_workspace_bytes(batch, n, es, scheme);
}

int expmb_select_host(const double* norms, double eps, int scheme, int* m, int* s, double* e1, double* e2) {
  Plan p{};
  int have = 1;
  if (scheme == EXPMB_SASTRE && norms[0] != 0.0) {
    // the kernels' fast path first; it must agree with the exact walk below
    const double le = log2(eps);
    int nd = (norms[0] > rung0_threshold(le)) ? 2 : select_sastre_fast(norms[0], 0.0, 1, le, &p);
    if (nd == 2) {
      // both fast forms (select_sastre_fast2: fused kernels; select_sastre_bf:
      // the warp-batched n = 16 kernel); a decided plan from either must be
      // the exact walk's, which the loop below recomputes and checks
      Plan pb{};
      const int nb = select_sastre_bf(norms[0], norms[1], le, &pb);
      nd = select_sastre_fast2(norms[0], norms[1], le, &p), have = 2;
      if (nb == 0) {
        Plan px{};
        int hv = 1;
        for (int need; (need = select_walk(norms, hv, eps, scheme, &px)) != 0;) hv = need;
        if (px.m != pb.m || px.s != pb.s || pb.e1 != (nd == 0 ? p.e1 : pb.e1)) {
          if (m) *m = -1;  // surfaces as a plan mismatch in the tests
          return -1;
        }
      }
    }
    if (nd == 0) {
      if (m) *m = p.m;
      if (s) *s = p.s;
      if (e1) *e1 = p.e1;
      if (e2) *e2 = p.e2;
      return have;
    }
    have = 1;
  }
  for (;;) {
    int need = select_walk(norms, have, eps, scheme, &p);
    if (need == 0) break;
    have = need;
  }
  if (m) *m = p.m;
  if (s) *s = p.s;
  if (e1) *e1 = p.e1;
  if (e2) *e2 = p.e2;
  return have;
}

int expmb_expm(const void* W, void* X, int64_t batch, int32_t n, int dtype, double eps, int scheme, int8_t* m,
               int8_t* s, double* e1, double* e2, double* norms, int32_t* mults, uint8_t* nonfinite, void* workspace,
               size_t workspace_bytes, void* stream) {
  if (dtype != EXPMB_F32 && dtype != EXPMB_F64) return EXPMB_ERR_DTYPE;
  if (scheme != EXPMB_SASTRE && scheme != EXPMB_PS && scheme != EXPMB_BASELINE) return EXPMB_ERR_SCHEME;
  if (n < 1 || batch < 0) return EXPMB_ERR_SHAPE;
  if (isnan(eps) || eps < expmb_unit_roundoff(dtype)) return EXPMB_ERR_TOLERANCE;
  if (((uintptr_t)W | (uintptr_t)X) & 15u) return EXPMB_ERR_ALIGN;
  if (batch == 0) return EXPMB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  PlanOut po{m, s, e1, e2, norms, mults, nonfinite};
  if (n <= 64) {
    // optional: with a workspace the kernel claims matrices dynamically
    int* ctr = (workspace != nullptr && workspace_bytes >= sizeof(int)) ? (int*)workspace : nullptr;
    if (dtype == EXPMB_F32) {
      const float* w = (const float*)W;
      float* x = (float*)X;
      return scheme == EXPMB_SASTRE ? dispatch_small<float, 0>(w, x, batch, n, eps, po, ctr, st)
             : scheme == EXPMB_PS   ? dispatch_small<float, 1>(w, x, batch, n, eps, po, ctr, st)
                                    : dispatch_small<float, 2>(w, x, batch, n, eps, po, ctr, st);
    }
    const double* w = (const double*)W;
    double* x = (double*)X;
    return scheme == EXPMB_SASTRE ? dispatch_small<double, 0>(w, x, batch, n, eps, po, ctr, st)
           : scheme == EXPMB_PS   ? dispatch_small<double, 1>(w, x, batch, n, eps, po, ctr, st)
                                  : dispatch_small<double, 2>(w, x, batch, n, eps, po, ctr, st);
  }
  if (use_fused_tile(n, scheme, dtype)) {
    if (workspace == nullptr || workspace_bytes < expmb_workspace_bytes(batch, n, dtype, scheme))
      return EXPMB_ERR_WORKSPACE;
    unsigned char* ws = (unsigned char*)workspace;
    return dtype == EXPMB_F32 ? ft_run<float>((const float*)W, (float*)X, batch, n, eps, scheme, po, ws, st)
                              : ft_run<double>((const double*)W, (double*)X, batch, n, eps, scheme, po, ws, st);
  }
  const size_t need = large_workspace_bytes(batch, n, dtype == EXPMB_F32 ? 4 : 8, scheme);
  if (workspace == nullptr || workspace_bytes < need) return EXPMB_ERR_WORKSPACE;
  return large_expm(W, X, batch, n, dtype, eps, scheme, po, workspace, st);
}

int expmb_select(const void* W, int64_t batch, int32_t n, int dtype, double eps, int scheme, int8_t* m, int8_t* s,
                 double* e1, double* e2, double* norms, int32_t* mults, uint8_t* nonfinite, void* workspace,
                 size_t workspace_bytes, void* stream) {
  if (dtype != EXPMB_F32 && dtype != EXPMB_F64) return EXPMB_ERR_DTYPE;
  if (scheme != EXPMB_SASTRE && scheme != EXPMB_PS) return EXPMB_ERR_SCHEME;
  if (n < 1 || batch < 0) return EXPMB_ERR_SHAPE;
  if (isnan(eps) || eps < expmb_unit_roundoff(dtype)) return EXPMB_ERR_TOLERANCE;
  if (((uintptr_t)W) & 15u) return EXPMB_ERR_ALIGN;
  if (batch == 0) return EXPMB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  PlanOut po{m, s, e1, e2, norms, mults, nonfinite, 1};
  if (n <= 64) {
    // the generic fused kernels (step machine) stop after the ladder
    int* ctr = (workspace != nullptr && workspace_bytes >= sizeof(int)) ? (int*)workspace : nullptr;
    if (dtype == EXPMB_F32) {
      const float* w = (const float*)W;
      if (n == 16 && scheme == 0 && !(getenv("EXPMB_W16") && getenv("EXPMB_W16")[0] == '0'))
        return launch_w16(w, nullptr, batch, eps, po, ctr, st);  // the same kernel (and norms) as expmb_expm
      if (n <= 16) return scheme == 0 ? launch_fused<float, 16, 2, 8, 0>(w, nullptr, batch, n, eps, po, ctr, st)
                                      : launch_fused<float, 16, 2, 8, 1>(w, nullptr, batch, n, eps, po, ctr, st);
      if (n <= 32) return scheme == 0 ? launch_fused<float, 32, 4, 4, 0>(w, nullptr, batch, n, eps, po, ctr, st)
                                      : launch_fused<float, 32, 4, 4, 1>(w, nullptr, batch, n, eps, po, ctr, st);
      return scheme == 0 ? launch_fused<float, 64, 4, 1, 0>(w, nullptr, batch, n, eps, po, ctr, st)
                         : launch_fused<float, 64, 4, 1, 1>(w, nullptr, batch, n, eps, po, ctr, st);
    }
    const double* w = (const double*)W;
    if (n <= 16) return scheme == 0 ? launch_fused<double, 16, 2, 8, 0>(w, nullptr, batch, n, eps, po, ctr, st)
                                    : launch_fused<double, 16, 2, 8, 1>(w, nullptr, batch, n, eps, po, ctr, st);
    if (n <= 32) return scheme == 0 ? launch_fused<double, 32, 4, 4, 0>(w, nullptr, batch, n, eps, po, ctr, st)
                                    : launch_fused<double, 32, 4, 4, 1>(w, nullptr, batch, n, eps, po, ctr, st);
    return scheme == 0 ? launch_fused<double, 64, 4, 1, 0>(w, nullptr, batch, n, eps, po, ctr, st)
                       : launch_fused<double, 64, 4, 1, 1>(w, nullptr, batch, n, eps, po, ctr, st);
  }
  if (use_fused_tile(n, scheme, dtype)) {
    if (workspace == nullptr || workspace_bytes < expmb_workspace_bytes(batch, n, dtype, scheme))
      return EXPMB_ERR_WORKSPACE;
    unsigned char* ws = (unsigned char*)workspace;
    return dtype == EXPMB_F32 ? ft_run<float>((const float*)W, nullptr, batch, n, eps, scheme, po, ws, st)
                              : ft_run<double>((const double*)W, nullptr, batch, n, eps, scheme, po, ws, st);
  }
  const size_t need = large_workspace_bytes(batch, n, dtype == EXPMB_F32 ? 4 : 8, scheme);
  if (workspace == nullptr || workspace_bytes < need) return EXPMB_ERR_WORKSPACE;
  return large_expm(W, nullptr, batch, n, dtype, eps, scheme, po, workspace, st);
}

int expmb_expm_pipelined(const void* W_host, void* X_host, void* W_dev, void* X_dev, int64_t batch, int32_t n,
                         int dtype, double eps, int scheme, int8_t* m, int8_t* s, double* e1, double* e2,
                         double* norms, int32_t* mults, uint8_t* nonfinite, int chunks, void* workspace,
                         size_t workspace_bytes, void* s_in, void* s_comp, void* s_out) {
  if (dtype != EXPMB_F32 && dtype != EXPMB_F64) return EXPMB_ERR_DTYPE;
  if (n < 1 || batch < 0) return EXPMB_ERR_SHAPE;
  if (batch == 0) return EXPMB_OK;
  if (chunks < 1) chunks = 1;
  if (chunks > 256) chunks = 256;
  const size_t esz = dtype == EXPMB_F32 ? 4 : 8;
  const size_t mat = (size_t)n * n * esz;
  cudaStream_t si = (cudaStream_t)s_in, sc = (cudaStream_t)s_comp, so = (cudaStream_t)s_out;
  // chunk bounds on multiples of 4 matrices (16-byte aligned slices)
  int64_t bounds[257];
  int nb = 0;
  bounds[nb++] = 0;
  for (int c = 1; c < chunks; ++c) {
    const int64_t b = (batch * c / chunks) / 4 * 4;
    if (b > bounds[nb - 1] && b < batch) bounds[nb++] = b;
  }
  bounds[nb++] = batch;
  const int nch = nb - 1;
  cudaEvent_t ev_in[256], ev_c[256];
  for (int c = 0; c < nch; ++c) {
    if (cudaEventCreateWithFlags(&ev_in[c], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ev_c[c], cudaEventDisableTiming) != cudaSuccess)
      return EXPMB_ERR_CUDA;
  }
  int rc = EXPMB_OK;
  // every host->device copy first (the large-n path reads plans back per call)
  for (int c = 0; c < nch && rc == EXPMB_OK; ++c) {
    const size_t off = (size_t)bounds[c] * mat, bytes = (size_t)(bounds[c + 1] - bounds[c]) * mat;
    if (cudaMemcpyAsync((char*)W_dev + off, (const char*)W_host + off, bytes, cudaMemcpyHostToDevice, si) !=
            cudaSuccess ||
        cudaEventRecord(ev_in[c], si) != cudaSuccess)
      rc = EXPMB_ERR_CUDA;
  }
  for (int c = 0; c < nch && rc == EXPMB_OK; ++c) {
    const int64_t a = bounds[c], cnt = bounds[c + 1] - bounds[c];
    const size_t off = (size_t)a * mat, bytes = (size_t)cnt * mat;
    if (cudaStreamWaitEvent(sc, ev_in[c], 0) != cudaSuccess) { rc = EXPMB_ERR_CUDA; break; }
    rc = expmb_expm((const char*)W_dev + off, (char*)X_dev + off, cnt, n, dtype, eps, scheme, m ? m + a : nullptr,
                    s ? s + a : nullptr, e1 ? e1 + a : nullptr, e2 ? e2 + a : nullptr,
                    norms ? norms + 2 * a : nullptr, mults ? mults + a : nullptr,
                    nonfinite ? nonfinite + a : nullptr, workspace, workspace_bytes, s_comp);
    if (rc != EXPMB_OK) break;
    if (cudaEventRecord(ev_c[c], sc) != cudaSuccess || cudaStreamWaitEvent(so, ev_c[c], 0) != cudaSuccess ||
        cudaMemcpyAsync((char*)X_host + off, (const char*)X_dev + off, bytes, cudaMemcpyDeviceToHost, so) !=
            cudaSuccess)
      rc = EXPMB_ERR_CUDA;
  }
  for (int c = 0; c < nch; ++c) {  // released once their work completes
    cudaEventDestroy(ev_in[c]);
    cudaEventDestroy(ev_c[c]);
  }
  return rc;
}

int expmb_select_lowrank_host(const double* norms, int have_v2, double eps, int* m, double* e1, double* e2) {
  int mm = 0;
  double a = 0.0, b = 0.0;
  const int rc = select_lowrank(norms[0], have_v2 ? norms[1] : 0.0, have_v2, log2(eps), &mm, &a, &b);
  if (rc == 0) {
    if (m) *m = mm;
    if (e1) *e1 = a;
    if (e2) *e2 = b;
  }
  return rc;
}

size_t expmb_lowrank_workspace_bytes(int64_t batch, int32_t n, int32_t t, int dtype) {
  (void)dtype;
  if (batch <= 0 || n < 1 || t <= 32 || t > n) return 0;  // t <= 32: shared memory only
  return lrl_layout(batch, n, t).total;
}

int expmb_expm_lowrank(const void* A1, const void* A2, void* X, int64_t batch, int32_t n, int32_t t, int dtype,
                       double eps, int8_t* m, double* e1, double* e2, double* norms, int32_t* mults, uint8_t* flags,
                       void* workspace, size_t workspace_bytes, void* stream) {
  if (dtype != EXPMB_F32 && dtype != EXPMB_F64) return EXPMB_ERR_DTYPE;
  if (n < 1 || t < 1 || t > n || batch < 0) return EXPMB_ERR_SHAPE;
  if (isnan(eps) || eps < expmb_unit_roundoff(dtype)) return EXPMB_ERR_TOLERANCE;
  if (batch == 0) return EXPMB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  LrOut po{m, e1, e2, norms, mults, flags};
  if (t > 32) {  // t x t operands in the global workspace (lowrank_large.cuh)
    const LrlLayout L = lrl_layout(batch, n, t);
    if (workspace == nullptr || workspace_bytes < L.total) return EXPMB_ERR_WORKSPACE;
    unsigned char* ws = (unsigned char*)workspace;
    if (dtype == EXPMB_F32)
      return lrl_run<float>((const float*)A1, (const float*)A2, (float*)X, batch, n, t, eps, po, ws, L, st);
    return lrl_run<double>((const double*)A1, (const double*)A2, (double*)X, batch, n, t, eps, po, ws, L, st);
  }
  if (dtype == EXPMB_F32)
    return dispatch_lowrank<float>((const float*)A1, (const float*)A2, (float*)X, batch, n, t, eps, po, st);
  return dispatch_lowrank<double>((const double*)A1, (const double*)A2, (double*)X, batch, n, t, eps, po, st);
}

size_t expmb_timegrid_workspace_bytes(int64_t K, int32_t n, int dtype) {
  if (K <= 0 || n < 1) return 0;
  const int esize = dtype == EXPMB_F32 ? 4 : 8;
  if (n <= 64) return tg_small_bytes(K, n, esize);
  return tg_layout(K, n, esize).total;
}

int expmb_expm_timegrid(const void* A, const void* t, void* X, int64_t K, int32_t n, int dtype, double eps,
                        int scheme, int8_t* m, int8_t* s, double* e1, double* e2, double* norms, int32_t* mults,
                        uint8_t* nonfinite, void* workspace, size_t workspace_bytes, void* stream) {
  if (dtype != EXPMB_F32 && dtype != EXPMB_F64) return EXPMB_ERR_DTYPE;
  if (scheme != EXPMB_SASTRE && scheme != EXPMB_PS) return EXPMB_ERR_SCHEME;
  if (n < 1 || K < 0) return EXPMB_ERR_SHAPE;
  if (isnan(eps) || eps < expmb_unit_roundoff(dtype)) return EXPMB_ERR_TOLERANCE;
  if (((uintptr_t)A | (uintptr_t)X) & 15u) return EXPMB_ERR_ALIGN;
  if (K == 0) return EXPMB_OK;
  if (workspace == nullptr || workspace_bytes < expmb_timegrid_workspace_bytes(K, n, dtype)) return EXPMB_ERR_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  PlanOut po{m, s, e1, e2, norms, mults, nonfinite};
  const int esize = dtype == EXPMB_F32 ? 4 : 8;
  const size_t nn = (size_t)n * n;
  if (n <= 64) {
    unsigned char* ws = (unsigned char*)workspace;
    void* W = ws;
    int* ctr = (int*)(ws + align256((size_t)K * nn * esize));
    int bx = (int)std::min<size_t>((nn + 255) / 256, 64);
    for (int64_t k0 = 0; k0 < K; k0 += 65535) {
      const int64_t kc = std::min<int64_t>(65535, K - k0);
      if (dtype == EXPMB_F32)
        k_tg_materialize<float><<<dim3(bx, (unsigned)kc), 256, 0, st>>>(
            (const float*)A, (const float*)t + k0, (float*)W + k0 * nn, kc, nn);
      else
        k_tg_materialize<double><<<dim3(bx, (unsigned)kc), 256, 0, st>>>(
            (const double*)A, (const double*)t + k0, (double*)W + k0 * nn, kc, nn);
    }
    if (cudaGetLastError() != cudaSuccess) return EXPMB_ERR_CUDA;
    if (dtype == EXPMB_F32)
      return scheme == EXPMB_SASTRE ? dispatch_small<float, 0>((const float*)W, (float*)X, K, n, eps, po, ctr, st)
                                    : dispatch_small<float, 1>((const float*)W, (float*)X, K, n, eps, po, ctr, st);
    return scheme == EXPMB_SASTRE ? dispatch_small<double, 0>((const double*)W, (double*)X, K, n, eps, po, ctr, st)
                                  : dispatch_small<double, 1>((const double*)W, (double*)X, K, n, eps, po, ctr, st);
  }
  const TgLayout L = tg_layout(K, n, esize);
  if (dtype == EXPMB_F32)
    return tg_run<float>((const float*)A, (const float*)t, (float*)X, K, n, eps, scheme, po,
                         (unsigned char*)workspace, L, st);
  return tg_run<double>((const double*)A, (const double*)t, (double*)X, K, n, eps, scheme, po,
                        (unsigned char*)workspace, L, st);
}

}  // extern "C"
