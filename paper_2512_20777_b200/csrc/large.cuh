// large.cuh -- batched expm for n > 64: bucketed GEMM pipeline.
//
// Same algorithm as engine.py:119-152, re-scheduled for a batch:
//   K_colsum  ||W||_1 slab partials + K_select(have=1): the m=1 rung
//             (select.py:169-188); decides which matrices need W^2 (device
//             flag, no host sync).
//   G stage0  W^2 = W W for flagged matrices, epilogue writes per-tile column
//             abs-sum partials (select.py:192-193).  PS: W^3, W^4 likewise.
//   K_select  ||W^2||_1 (fixed-order reduction of the partials) and the
//             ladder (select.py:164-220) -> m, s, e1, e2, mults.
//   K_bucket  the device (m, s) bucket scheduler: stage lists and their sizes
//             in device memory (no host round trip; every later launch reads
//             its slot count on the device)
//   K_elem    T0/T1/T2 results, T4's inner factor, R1 = c1 A^2 + c2 A
//   G stage1..3  the products of poly.py:189-230, each epilogue emitting the
//             next linear combinations (y02/L2/R2, y12/L3/R3, X) so no
//             separate elementwise pass runs between products
//   G square  s squarings (engine.py:80-87), bucket = prefix of the batch
//             sorted by s descending; one launch per level up to MAX_SCALING,
//             levels beyond the batch's largest s find a zero count and exit.
// The 2^-s, 2^-2s scalings (engine.py:139-140) are folded into epilogue
// coefficients; they are powers of two so the folding is exact.
#pragma once

#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <stdio.h>
#include <stdlib.h>

#include <algorithm>

#include "fused_small.cuh"
#include "gemm_simt.cuh"
#include "gemm_tc.cuh"
#include "gemm_i8.cuh"
#include "select.cuh"

namespace expmb {

// ---------------------------------------------------------------------------
// workspace layout (per chunk of `chunk` matrices)
// ---------------------------------------------------------------------------
constexpr int kLargeBufsSastre = 7;  // W2 Y0 Y1 La Ra Lb Rb   (Tmp aliases Lb)
constexpr int kLargeBufsPS = 6;      // W2 W3 W4 Q0 Q1 Tmp
// Exact int8-slice (Ozaki) products on tcgen05 for fp32 (gemm_i8.cuh).
// Default: on for fp32 n >= 320 with n % 16 == 0, the measured crossover
// against the FFMA GEMM (tools/i8_crossover.py, round 2 with the persistent
// stage and the fast prep pass: 0.85x at 256, 1.17x at 320, 1.13x at 384,
// 1.40x at 448, 1.48x at 512, 1.93x at 768, 2.40x at 1024, 2.96x at 1536).
// EXPMB_I8=1 also enables it from n = 256, EXPMB_I8=0 disables it.  Each
// product is routed per matrix (k_i8_route): operands that are not "flat" go
// to the FFMA GEMM.
static inline bool use_i8_path(int n, int esize) {
  const char* e = getenv("EXPMB_I8");
  if (esize != 4 || n % 16 != 0) return false;
  if (e != nullptr && e[0] == '0') return false;
  if (e != nullptr && e[0] == '1') return n >= 256;
  return n >= 320;
}
static inline int i8_np(int n) { return (n + 15) / 16 * 16; }
constexpr size_t kLargeWsCap = (size_t)40 << 30;  // bound on the big buffers

struct LargeLayout {
  int64_t chunk;
  size_t mat_bytes;
  int nbufs;
  int tiles_m;
  size_t off_bufs, off_part, off_norm1, off_norm2, off_need, off_flags, off_m, off_s, off_e1, off_e2, off_list, off_cnt,
      total;
  size_t off_i8as, off_i8bs, off_i8er, off_i8ec, off_i8rc, off_i8cc, off_i8ok;  // int8-slice path
};

static inline size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

static inline LargeLayout large_layout(int64_t batch, int n, int esize, int scheme) {
  LargeLayout L{};
  L.mat_bytes = align256((size_t)n * n * esize);
  L.nbufs = scheme == 1 ? kLargeBufsPS : kLargeBufsSastre;
  const bool i8p = use_i8_path(n, esize);
  const size_t i8plane = (size_t)n * i8_np(n);
  const size_t per_bufs = L.mat_bytes * L.nbufs;
  // per-matrix bytes for sizing the chunk (the int8-slice regions sit after the lists)
  const size_t per = per_bufs + (i8p ? 2 * i8::NSL * i8plane + 2 * (size_t)n * sizeof(int) + 2 * (size_t)n * 8 + 4 : 0);
  int64_t chunk = (int64_t)(kLargeWsCap / per);
  if (chunk < 1) chunk = 1;
  if (chunk > 65535) chunk = 65535;  // gridDim.z
  if (chunk > batch) chunk = batch;
  L.chunk = chunk;
  L.tiles_m = (n + kGemmBM - 1) / kGemmBM;
  size_t off = 0;
  L.off_bufs = off; off += per_bufs * chunk;
  L.off_part = off; off += align256((size_t)chunk * L.tiles_m * n * sizeof(double));
  L.off_norm1 = off; off += align256((size_t)chunk * 4 * sizeof(double));
  L.off_norm2 = off; off += 0;  // norms for powers 1..4 live in the same [chunk][4] array
  L.off_need = off; off += align256((size_t)chunk * sizeof(int));
  L.off_flags = off; off += align256((size_t)chunk * sizeof(int));
  L.off_m = off; off += align256((size_t)chunk);
  L.off_s = off; off += align256((size_t)chunk);
  L.off_e1 = off; off += align256((size_t)chunk * sizeof(double));
  L.off_e2 = off; off += align256((size_t)chunk * sizeof(double));
  L.off_list = off; off += align256((size_t)chunk * 8 * sizeof(int));
  L.off_cnt = off; off += 256;
  L.off_i8as = off; off += i8p ? align256((size_t)chunk * i8::NSL * i8plane) : 0;
  L.off_i8bs = off; off += i8p ? align256((size_t)chunk * i8::NSL * i8plane) : 0;
  L.off_i8er = off; off += i8p ? align256((size_t)chunk * n * sizeof(int)) : 0;
  L.off_i8ec = off; off += i8p ? align256((size_t)chunk * n * sizeof(int)) : 0;
  L.off_i8rc = off; off += i8p ? align256((size_t)chunk * n * 8) : 0;
  L.off_i8cc = off; off += i8p ? align256((size_t)chunk * n * 8) : 0;
  L.off_i8ok = off; off += i8p ? align256((size_t)chunk * sizeof(int)) : 0;
  L.total = off;
  return L;
}

static inline size_t large_workspace_bytes(int64_t batch, int n, int esize, int scheme) {
  return large_layout(batch, n, esize, scheme).total;
}

// ---------------------------------------------------------------------------
// small kernels
// ---------------------------------------------------------------------------

// Reduce the per-tile column partials of W^p and walk the ladder again
// (select.py:164-220) for matrix z; the whole CTA takes part.
__device__ __forceinline__ void select_block(const double* __restrict__ part, int tiles_m, int n, int have,
                                             double eps, int scheme, double* __restrict__ nrm4, int* __restrict__ need,
                                             int8_t* __restrict__ pm, int8_t* __restrict__ ps,
                                             double* __restrict__ pe1, double* __restrict__ pe2, int z) {
  if (have > 1 && need[z] != have) return;  // this matrix did not form W^have
  __shared__ double red[256];
  const double* pz = part + (size_t)z * tiles_m * n;
  double mx = -INFINITY;
  for (int c = threadIdx.x; c < n; c += blockDim.x) {
    double a = 0.0;
    for (int t = 0; t < tiles_m; ++t) a += pz[(size_t)t * n + c];
    mx = nanmax(mx, a);
  }
  red[threadIdx.x] = mx;
  __syncthreads();
  for (int off = 128; off > 0; off >>= 1) {
    if (threadIdx.x < off) red[threadIdx.x] = nanmax(red[threadIdx.x], red[threadIdx.x + off]);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    nrm4[4 * z + have - 1] = red[0];
    if (have == 1) nrm4[4 * z + 1] = nrm4[4 * z + 2] = nrm4[4 * z + 3] = NAN;
    double nr[4];
    for (int q = 0; q < 4; ++q) nr[q] = nrm4[4 * z + q];
    Plan p{0, 0, 0.0, 0.0};
    double lw[4];
    for (int q = 0; q < have; ++q) lw[q] = log2_or_ninf(nr[q]);
    int nd = 0;
    if (nr[0] != 0.0) nd = select_walk_lw(lw, have, eps, scheme, &p);  // eps carries log2(eps)
    need[z] = nd;
    if (nd == 0) {
      pm[z] = (int8_t)p.m; ps[z] = (int8_t)p.s; pe1[z] = p.e1; pe2[z] = p.e2;
    }
  }
}
__global__ void __launch_bounds__(256) k_select(const double* __restrict__ part, int tiles_m, int n, int have,
                                                double eps, int scheme, double* __restrict__ nrm4,
                                                int* __restrict__ need, int8_t* __restrict__ pm,
                                                int8_t* __restrict__ ps, double* __restrict__ pe1,
                                                double* __restrict__ pe2) {
  select_block(part, tiles_m, n, have, eps, scheme, nrm4, need, pm, ps, pe1, pe2, blockIdx.x);
}

// Column abs-sum partials of W over 128-row slabs: grid (col blocks, slabs,
// matrices), one thread per column, coalesced row reads (select.py:169).
template <typename T>
__global__ void __launch_bounds__(256) k_colsum_partial(const T* __restrict__ W, int n, int64_t wstride,
                                                        double* __restrict__ part, int tiles_m) {
  const int z = blockIdx.z, c = blockIdx.x * 256 + threadIdx.x, r0 = blockIdx.y * kGemmBM;
  if (c >= n) return;
  const T* w = W + (int64_t)z * wstride;
  const int r1 = min(n, r0 + kGemmBM);
  double a = 0.0;
  for (int r = r0; r < r1; ++r) a += fabs((double)w[(size_t)r * n + c]);
  part[((size_t)z * tiles_m + blockIdx.y) * n + c] = a;
}

// Non-finite scan of the final values, spread over many CTAs per matrix.
template <typename T>
__global__ void __launch_bounds__(256) k_nonfinite(const T* __restrict__ X, int n, int64_t xstride,
                                                   int* __restrict__ flags) {
  const int z = blockIdx.y;
  const T* x = X + (int64_t)z * xstride;
  const size_t nn = (size_t)n * n;
  int bad = 0;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < nn; i += (size_t)gridDim.x * blockDim.x)
    bad |= !isfinite(x[i]);
  bad = __syncthreads_or(bad);
  if (bad && threadIdx.x == 0) atomicOr(flags + z, 1);
}

// Per-matrix outputs.  A non-finite input shows in ||W||_1 (NaN / Inf
// propagate through the abs-sums); non-finite outputs come from k_nonfinite.
__device__ __forceinline__ void finish_one(int z, int scheme, const double* __restrict__ nrm4,
                                           const int8_t* __restrict__ pm, const int8_t* __restrict__ ps,
                                           const double* __restrict__ pe1, const double* __restrict__ pe2, int bad,
                                           int64_t g, PlanOut po) {
  const int m = pm[z], s = ps[z];
  const double n1 = nrm4[4 * z], n2 = nrm4[4 * z + 1];
  if (po.m) po.m[g] = (int8_t)m;
  if (po.s) po.s[g] = (int8_t)s;
  if (po.e1) po.e1[g] = pe1[z];
  if (po.e2) po.e2[g] = pe2[z];
  if (po.norms) { po.norms[2 * g] = n1; po.norms[2 * g + 1] = n2; }
  if (po.mults) po.mults[g] = budget(m, scheme) + s;
  const double n3 = nrm4[4 * z + 2], n4 = nrm4[4 * z + 3];
  const bool pw_bad = scheme == 1 && ((n3 == n3 && !(n3 < INFINITY)) || (n4 == n4 && !(n4 < INFINITY)));
  if (po.nonfinite) po.nonfinite[g] = (uint8_t)(bad || pw_bad || !(n1 < INFINITY) || (n2 == n2 && !(n2 < INFINITY)));
}
__global__ void __launch_bounds__(256) k_finish(int cnt, int scheme, const double* __restrict__ nrm4,
                                                const int8_t* __restrict__ pm, const int8_t* __restrict__ ps,
                                                const double* __restrict__ pe1, const double* __restrict__ pe2,
                                                const int* __restrict__ flags, int64_t base, PlanOut po) {
  const int z = blockIdx.x * blockDim.x + threadIdx.x;
  if (z < cnt) finish_one(z, scheme, nrm4, pm, ps, pe1, pe2, flags[z], base + z, po);
}

// Device (m, s) bucket scheduler (the keys are the reference's plan,
// select.py:164-220; the reference batches by caller loops, bench.py:294-309).
// One CTA per chunk.  Writes `lists` = five slot lists of `ic` entries:
//   [0] every matrix (elementwise stage), [1..3] the matrices whose formula
//   uses evaluation product 1..3, [4] every matrix sorted by s descending
//   (counting sort), so squaring level q is the prefix of length #(s > q);
// and `cnt` = [ic, |E1|, |E2|, |E3|, #(s > 0), ..., #(s > kMaxSq - 1)].
// Order within a bucket is immaterial: every matrix's result depends only on
// its own data, so the output is bit-identical whatever CTA handles it.
constexpr int kMaxSq = 20;  // MAX_SCALING (select.py:56)
constexpr int kCntSq = 4;   // cnt index of squaring level 0
__global__ void __launch_bounds__(1024) k_bucket(const int8_t* __restrict__ pm, const int8_t* __restrict__ ps,
                                                 int ic, int scheme, int* __restrict__ lists, int* __restrict__ cnt) {
  __shared__ int hist[kMaxSq + 1], fill[kMaxSq + 1], base[kMaxSq + 1], ecnt[3];
  if (threadIdx.x <= kMaxSq) hist[threadIdx.x] = fill[threadIdx.x] = 0;
  if (threadIdx.x < 3) ecnt[threadIdx.x] = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < ic; i += blockDim.x) {
    const int s = min(max((int)ps[i], 0), kMaxSq);
    atomicAdd(&hist[s], 1);
    lists[i] = i;
    const int m = pm[i];
    int k = 0;  // evaluation products after the powers
    if (scheme == 0) k = (m >= 4) + (m >= 8) + (m >= 15);
    else if (m >= 1) k = min(ps_k_of(m) - 1, 3);
    for (int e = 0; e < k; ++e) lists[(size_t)(1 + e) * ic + atomicAdd(&ecnt[e], 1)] = i;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int q = kMaxSq; q >= 0; --q) {  // base[s] = #(s' > s)
      base[q] = acc;
      acc += hist[q];
    }
    cnt[0] = ic;
    for (int e = 0; e < 3; ++e) cnt[1 + e] = ecnt[e];
    for (int q = 0; q < kMaxSq; ++q) cnt[kCntSq + q] = base[q];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < ic; i += blockDim.x) {
    const int s = min(max((int)ps[i], 0), kMaxSq);
    lists[(size_t)4 * ic + base[s] + atomicAdd(&fill[s], 1)] = i;
  }
}

// ---------------------------------------------------------------------------
// host orchestration
// ---------------------------------------------------------------------------

// ||W||_1 for a chunk: slab partials over many CTAs, then the first rung.
template <typename T>
static void launch_norm1(const T* W, int n, int ic, const LargeLayout& L, double* part, double log_eps, int scheme,
                         double* nrm4, int* need, int8_t* dm, int8_t* ds, double* de1, double* de2, cudaStream_t st) {
  dim3 grid((n + 255) / 256, L.tiles_m, ic);
  k_colsum_partial<T><<<grid, 256, 0, st>>>(W, n, (int64_t)n * n, part, L.tiles_m);
  k_select<<<ic, 256, 0, st>>>(part, L.tiles_m, n, 1, log_eps, scheme, nrm4, need, dm, ds, de1, de2);
}

template <typename T>
static void launch_finish(const T* X, int n, int ic, int scheme, const LargeLayout& L, unsigned char* ws,
                          const double* nrm4, const int8_t* dm, const int8_t* ds, const double* de1,
                          const double* de2, int64_t base, PlanOut po, cudaStream_t st) {
  int* flags = reinterpret_cast<int*>(ws + L.off_flags);
  cudaMemsetAsync(flags, 0, (size_t)ic * sizeof(int), st);
  const size_t nn = (size_t)n * n;
  int bx = (int)((nn + 256 * 8 - 1) / (256 * 8));
  if (bx > 1024) bx = 1024;
  k_nonfinite<T><<<dim3(bx, ic), 256, 0, st>>>(X, n, (int64_t)nn, flags);
  k_finish<<<(ic + 255) / 256, 256, 0, st>>>(ic, scheme, nrm4, dm, ds, de1, de2, flags, base, po);
}

typedef CUresult (*TensorMapEncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                      const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                      CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static TensorMapEncodeFn tensor_map_encoder() {
  static TensorMapEncodeFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (TensorMapEncodeFn)p;
  }
  return fn;
}

// int8 slice planes [planes][rows = n][k = n, row stride np]; box 128 (k bytes) x box_rows, 128B swizzle.
// Columns k >= n are outside the tensor, so TMA fills them with zeros.
static bool encode_map_i8(CUtensorMap* m, const int8_t* base, int n, int np, int64_t planes, int box_rows) {
  TensorMapEncodeFn enc = tensor_map_encoder();
  if (!enc) return false;
  cuuint64_t dims[3] = {(cuuint64_t)n, (cuuint64_t)n, (cuuint64_t)planes};
  cuuint64_t strides[2] = {(cuuint64_t)np, (cuuint64_t)n * np};
  cuuint32_t box[3] = {(cuuint32_t)i8::BKB, (cuuint32_t)box_rows, 1};
  cuuint32_t es[3] = {1, 1, 1};
  const CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, (void*)base, dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE,
                         i8::kSw64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS && getenv("EXPMB_DEBUG_SYNC"))
    fprintf(stderr, "expmb i8: cuTensorMapEncodeTiled -> %d (base %p n %d np %d planes %lld box_rows %d)\n", (int)r,
            (const void*)base, n, np, (long long)planes, box_rows);
  return r == CUDA_SUCCESS;
}

// One product stage on the int8-slice path: exponents, slices, GEMM, over
// the first *dcount slots of `list` (dcount null: `count`).
static int i8_launch(const i8::Maps& maps, const GemmCtx<float>& g, int stage, const int* list, int count,
                     const i8::Bufs& b, cudaStream_t st, const int* dcount = nullptr) {
  if (count <= 0) return 0;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(i8::k_i8_stage, cudaFuncAttributeMaxDynamicSharedMemorySize, i8::SMEM_BYTES) !=
        cudaSuccess)
      return 1;
    attr = true;
  }
  const int n = g.n;
  static const bool dbg = getenv("EXPMB_DEBUG_SYNC") != nullptr;
  auto chk = [&](const char* what) {
    if (!dbg) return 0;
    const cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) fprintf(stderr, "expmb i8 stage %d: %s failed: %s\n", stage, what, cudaGetErrorString(e));
    return e != cudaSuccess ? 1 : 0;
  };
  static int occ_stage = 0, occ_prep = 0;
  {
    // one streaming pass per operand: scales, diagonal decision, routing statistics, slices
    const int64_t units = (int64_t)count * ((n + 7) / 8 + (n + 31) / 32);
    i8::k_i8_prep<<<persistent_grid(i8::k_i8_prep, 256, 0, units, &occ_prep), 256, 0, st>>>(g, stage, list, b,
                                                                                        dcount, count);
    if (chk("prep")) return 1;
    i8::k_i8_route<<<std::min(count, sm_count_dev() * 8), 256, 0, st>>>(g, stage, list, b, dcount, count);
    if (chk("route")) return 1;
  }
  // persistent stage with the split epilogue (default); EXPMB_I8_PERSIST=0: one unit per CTA
  const bool persist = !(getenv("EXPMB_I8_PERSIST") && getenv("EXPMB_I8_PERSIST")[0] == '0');  // read per call (tests A/B it)
  // 2-CTA clusters sharing the L panel by multicast (EXPMB_I8_MC=0: one CTA per tile)
  const bool mc = !(getenv("EXPMB_I8_MC") && getenv("EXPMB_I8_MC")[0] == '0');
  static bool attr_np = false;
  if (!persist) {
    if (!attr_np) {
      if (cudaFuncSetAttribute(i8::k_i8_stage_np<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               i8::SMEM_BYTES) != cudaSuccess ||
          cudaFuncSetAttribute(i8::k_i8_stage_np<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               i8::SMEM_BYTES) != cudaSuccess)
        return 1;
      attr_np = true;
    }
    const int tn = (n + i8::BN - 1) / i8::BN, tm = (n + i8::BM - 1) / i8::BM;
    if (mc) {
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3((unsigned)((tn + 1) & ~1), (unsigned)tm, (unsigned)count);  // whole pairs
      cfg.blockDim = dim3(i8::NTHREADS_NP);
      cfg.dynamicSmemBytes = i8::SMEM_BYTES;
      cfg.stream = st;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 2;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      if (cudaLaunchKernelEx(&cfg, i8::k_i8_stage_np<true>, maps, g, stage, list, b, dcount) != cudaSuccess) return 1;
    } else {
      i8::k_i8_stage_np<false><<<dim3(tn, tm, count), i8::NTHREADS_NP, i8::SMEM_BYTES, st>>>(maps, g, stage, list, b,
                                                                                        dcount);
    }
  }
  const int64_t units = (int64_t)count * ((n + i8::BN - 1) / i8::BN) * ((n + i8::BM - 1) / i8::BM);
  if (persist) i8::k_i8_stage<<<persistent_grid(i8::k_i8_stage, i8::NTHREADS_NP, i8::SMEM_BYTES, units, &occ_stage,
                                   i8::STAGE_BYTES * i8::STAGES <= 100 * 1024 ? 2 : 1), i8::NTHREADS_NP,
                   i8::SMEM_BYTES, st>>>(maps, g, stage, list, b, dcount, count);
  {
    const cudaError_t le = cudaGetLastError();
    if (le != cudaSuccess) {
      if (dbg) fprintf(stderr, "expmb i8 stage %d: launch failed: %s\n", stage, cudaGetErrorString(le));
      return 1;
    }
    if (chk("stage")) return 1;
  }
  // the products routed away run on the FFMA GEMM (its units for routed-here matrices exit at once)
  GemmCtx<float> gs = g;
  gs.route = b.ok;
  return gemm_launch<float>(gs, stage, list, count, st, dcount);
}

template <typename T>
static int large_run_chunk(const T* W, T* X, int64_t cnt, int n, double eps, int scheme, int64_t base, PlanOut po,
                           unsigned char* ws, const LargeLayout& L, cudaStream_t st) {
  const size_t nn = (size_t)n * n;
  auto buf = [&](int b) { return reinterpret_cast<T*>(ws + L.off_bufs + (size_t)b * L.mat_bytes * L.chunk); };
  // buffers are [buffer][matrix] with stride mat_bytes
  const int64_t mstride = (int64_t)(L.mat_bytes / sizeof(T));
  double* part = reinterpret_cast<double*>(ws + L.off_part);
  double* nrm4 = reinterpret_cast<double*>(ws + L.off_norm1);
  int* need = reinterpret_cast<int*>(ws + L.off_need);
  int8_t* dm = reinterpret_cast<int8_t*>(ws + L.off_m);
  int8_t* ds = reinterpret_cast<int8_t*>(ws + L.off_s);
  double* de1 = reinterpret_cast<double*>(ws + L.off_e1);
  double* de2 = reinterpret_cast<double*>(ws + L.off_e2);
  int* dlist = reinterpret_cast<int*>(ws + L.off_list);
  const int ic = (int)cnt;

  const double log_eps = log2(eps);  // host libm, as select.py:175
  launch_norm1<T>(W, n, ic, L, part, log_eps, scheme, nrm4, need, dm, ds, de1, de2, st);

  GemmCtx<T> g{};
  g.n = n;
  g.W = W;
  g.X = X;
  g.mstride = mstride;
  g.wstride = (int64_t)nn;
  g.m = dm;
  g.s = ds;
  g.need = need;
  g.part = part;
  g.tiles_m = L.tiles_m;
  g.scheme = scheme;
  if (scheme == 0) {
    g.W2 = buf(0); g.Y0 = buf(1); g.Y1 = buf(2); g.La = buf(3); g.Ra = buf(4); g.Lb = buf(5); g.Rb = buf(6);
    g.Tmp = g.Lb;
  } else {
    g.W2 = buf(0); g.W3 = buf(1); g.W4 = buf(2); g.La = buf(3); g.Ra = buf(4); g.Tmp = buf(5);
  }

  // product stages: FFMA / DMMA GEMM, or the exact int8-slice tensor-core GEMM (fp32, opt-in)
  i8::Maps i8maps{};
  i8::Bufs i8b{};
  bool i8p = false;
  if constexpr (sizeof(T) == 4) {
    if (use_i8_path(n, 4) && L.off_i8as != L.off_i8bs) {
      i8p = true;
      i8b.np = i8_np(n);
      i8b.as = reinterpret_cast<int8_t*>(ws + L.off_i8as);
      i8b.bs = reinterpret_cast<int8_t*>(ws + L.off_i8bs);
      i8b.er = reinterpret_cast<int*>(ws + L.off_i8er);
      i8b.ec = reinterpret_cast<int*>(ws + L.off_i8ec);
      i8b.rc = reinterpret_cast<unsigned long long*>(ws + L.off_i8rc);
      i8b.cc = reinterpret_cast<unsigned long long*>(ws + L.off_i8cc);
      i8b.ok = reinterpret_cast<int*>(ws + L.off_i8ok);
      if (!encode_map_i8(&i8maps.a, i8b.as, n, i8b.np, cnt * i8::NSL, i8::BM) ||
          !encode_map_i8(&i8maps.b, i8b.bs, n, i8b.np, cnt * i8::NSL, i8::BN)) {
        if (getenv("EXPMB_DEBUG_SYNC")) fprintf(stderr, "expmb i8: tensor map encoding failed (n=%d)\n", n);
        return EXPMB_ERR_CUDA;
      }
    }
  }
  auto stage_launch = [&](int stage, const int* list, int count, const int* dcount) -> int {
    if constexpr (sizeof(T) == 4) {
      if (i8p) return i8_launch(i8maps, g, stage, list, count, i8b, st, dcount);
    }
    return gemm_launch<T>(g, stage, list, count, st, dcount);
  };

  // powers + ladder, gated on device flags (no host round trip)
  const int maxp = scheme == 1 ? 4 : 2;
  for (int p = 2; p <= maxp; ++p) {
    if (stage_launch(p == 2 ? STAGE_W2 : (p == 3 ? STAGE_W3 : STAGE_W4), nullptr, ic, nullptr)) return EXPMB_ERR_CUDA;
    k_select<<<ic, 256, 0, st>>>(part, L.tiles_m, n, p, log_eps, scheme, nrm4, need, dm, ds, de1, de2);
  }

  if (po.plan_only) {  // select_sastre / select_ps (select.py:223-234): the plan only
    int* flags = reinterpret_cast<int*>(ws + L.off_flags);
    if (cudaMemsetAsync(flags, 0, (size_t)ic * sizeof(int), st) != cudaSuccess) return EXPMB_ERR_CUDA;
    k_finish<<<(ic + 255) / 256, 256, 0, st>>>(ic, scheme, nrm4, dm, ds, de1, de2, flags, base, po);
    return cudaGetLastError() == cudaSuccess ? EXPMB_OK : EXPMB_ERR_CUDA;
  }

  // device bucket scheduler: stage lists + their sizes stay on the device
  int* dcnt = reinterpret_cast<int*>(ws + L.off_cnt);
  k_bucket<<<1, 1024, 0, st>>>(dm, ds, ic, scheme, dlist, dcnt);
  if (elem_launch<T>(g, dlist, ic, st, dcnt)) return EXPMB_ERR_CUDA;
  for (int e = 0; e < 3; ++e)
    if (stage_launch(STAGE_E1 + e, dlist + (size_t)(1 + e) * ic, ic, dcnt + 1 + e)) return EXPMB_ERR_CUDA;
  for (int q = 0; q < kMaxSq; ++q) {
    g.sq_step = q;
    if (stage_launch(STAGE_SQ, dlist + (size_t)4 * ic, ic, dcnt + kCntSq + q)) return EXPMB_ERR_CUDA;
  }
  launch_finish<T>(X, n, ic, scheme, L, ws, nrm4, dm, ds, de1, de2, base, po, st);
  return cudaGetLastError() == cudaSuccess ? EXPMB_OK : EXPMB_ERR_CUDA;
}

// ---------------------------------------------------------------------------
// Alg. 1 for n > 64 (engine.py:90-116, the paper's comparator), sync-free:
// the term loop and the squaring loop are data dependent per matrix, so the
// host launches a bounded number of term stages over device-resident active
// lists, and one cooperative kernel runs every squaring level (grid-wide
// barrier between levels, as many levels as the largest s of the batch).
// ---------------------------------------------------------------------------
constexpr int kA1MaxTerms = 40;  // ||B||_1 < 1/2: ||B^k / k!||_1 < 2^-53 by k = 16 (the fused kernel caps at 398)
constexpr int kA1MaxS = 1100;    // ||W||_1 <= 2^1024 (the fused kernel's cap)

// ||W||_1 from the slab partials, s = min{s >= 0 : ||W||_1 2^-s < 1/2}
// (engine.py:102-104), the first termination test ||B||_1 > eps, and the
// initial active list of the term loop.
__global__ void __launch_bounds__(256) k_a1_init(const double* __restrict__ part, int tiles_m, int n, double eps,
                                                 double* __restrict__ nrm4, int* __restrict__ s32,
                                                 int* __restrict__ m32, double* __restrict__ pe1,
                                                 int* __restrict__ list0, int* __restrict__ cnt) {
  const int z = blockIdx.x;
  __shared__ double red[256];
  const double* pz = part + (size_t)z * tiles_m * n;
  double mx = -INFINITY;
  for (int c = threadIdx.x; c < n; c += blockDim.x) {
    double a = 0.0;
    for (int t = 0; t < tiles_m; ++t) a += pz[(size_t)t * n + c];
    mx = nanmax(mx, a);
  }
  red[threadIdx.x] = mx;
  __syncthreads();
  for (int off = 128; off > 0; off >>= 1) {
    if (threadIdx.x < off) red[threadIdx.x] = nanmax(red[threadIdx.x], red[threadIdx.x + off]);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double n1 = red[0];
    int s = 0;
    if (n1 >= 0.5) {  // while ldexp(n1, -s) >= 1/2: s += 1
      int e;
      frexp(n1, &e);  // n1 = f 2^e, f in [1/2, 1)
      s = (n1 <= 1e300) ? e + 1 : kA1MaxS;
    }
    if (!(n1 < INFINITY)) s = 0;  // NaN / Inf input: flagged (NonFiniteError), no work spent on it
    nrm4[4 * z] = n1;
    nrm4[4 * z + 1] = nrm4[4 * z + 2] = nrm4[4 * z + 3] = NAN;
    s32[z] = s;
    m32[z] = 0;
    const double nb = ldexp(n1, -s);  // ||B||_1 exactly (power-of-two scaling)
    pe1[z] = nb;
    if (nb > eps) list0[atomicAdd(&cnt[0], 1)] = z;
    atomicMax(&cnt[kA1MaxTerms + 1], s);
  }
}

// B = 2^-s W (W2 buffer), Y_0 = B, X_0 = I (the buffer the squarings end in X from).
template <typename T>
__global__ void __launch_bounds__(256) k_a1_setup(GemmCtx<T> g, int ic) {
  const size_t nn = (size_t)g.n * g.n;
  for (int z = blockIdx.y; z < ic; z += gridDim.y) {
    const int s = g.s32[z];
    const int64_t o = (int64_t)z * g.mstride;
    const T* Wz = g.W + (int64_t)z * g.wstride;
    T* Xz = sq_target(g, z, s, 0);
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < nn; i += (size_t)gridDim.x * blockDim.x) {
      const T b = (T)ldexp((double)Wz[i], -s);  // exact unless the result is subnormal (scale_pow2, matrix.py:159-167)
      g.W2[o + i] = b;
      g.Y0[o + i] = b;
      Xz[i] = (i / g.n == i % g.n) ? T(1) : T(0);
    }
  }
}

// After term j: ||Y_{j+1}||_1 from the GEMM's column partials; the matrices
// still above eps go on to term j + 1.
__global__ void __launch_bounds__(256) k_a1_check(const double* __restrict__ part, int tiles_m, int n, double eps,
                                                  int term, const int* __restrict__ list, const int* __restrict__ cnt,
                                                  int* __restrict__ next, int* __restrict__ next_cnt,
                                                  int* __restrict__ m32, double* __restrict__ pe1) {
  __shared__ double red[256];
  for (int slot = blockIdx.x; slot < *cnt; slot += gridDim.x) {
    const int z = list[slot];
    const double* pz = part + (size_t)z * tiles_m * n;
    double mx = -INFINITY;
    for (int c = threadIdx.x; c < n; c += blockDim.x) {
      double a = 0.0;
      for (int t = 0; t < tiles_m; ++t) a += pz[(size_t)t * n + c];
      mx = nanmax(mx, a);
    }
    red[threadIdx.x] = mx;
    __syncthreads();
    for (int off = 128; off > 0; off >>= 1) {
      if (threadIdx.x < off) red[threadIdx.x] = nanmax(red[threadIdx.x], red[threadIdx.x + off]);
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      const double ny = red[0];
      m32[z] = term + 1;  // products charged so far (one per term formed, engine.py:111)
      pe1[z] = ny;
      if (ny > eps) next[atomicAdd(next_cnt, 1)] = z;  // NaN stops, as the reference's comparison
    }
    __syncthreads();
  }
}

// Every squaring level of the batch in one cooperative launch (engine.py:113):
// level q squares the matrices with s > q; a grid-wide barrier separates the
// levels, whose count is the batch's largest s (read on the device).
template <typename T, bool TWO, bool MMA>
__global__ void __launch_bounds__(256, 1) k_a1_square(GemmCtx<T> g, int ic, const int* __restrict__ maxs_ptr) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cooperative_groups::grid_group grid = cooperative_groups::this_grid();
  const int maxs = *maxs_ptr;
  const int tn = (g.n + kGemmBN - 1) / kGemmBN, tiles = tn * g.tiles_m;
  const int total = ic * tiles;
  for (int q = 0; q < maxs; ++q) {
    GemmCtx<T> gq = g;
    gq.sq_step = q;
    for (int w = blockIdx.x; w < total; w += gridDim.x) {
      const int z = w / tiles, t = w - z * tiles;
      if (g.s32[z] <= q) continue;  // done squaring (uniform per CTA)
      __syncthreads();
      gemm_tile<T, TWO, MMA>(gq, STAGE_A1SQ, nullptr, z, t % tn, t / tn, smem_raw);
    }
    __threadfence();
    grid.sync();
  }
}

__global__ void __launch_bounds__(256) k_a1_finish(int ic, const double* __restrict__ nrm4, const int* __restrict__ s32,
                                                   const int* __restrict__ m32, const double* __restrict__ pe1,
                                                   const int* __restrict__ flags, int64_t base, PlanOut po) {
  const int z = blockIdx.x * blockDim.x + threadIdx.x;
  if (z < ic) {
    const int64_t gi = base + z;
    const int m = m32[z], s = s32[z];
    const double n1 = nrm4[4 * z];
    if (po.m) po.m[gi] = (int8_t)(m < 127 ? m : 127);  // int8 outputs saturate; mults is exact
    if (po.s) po.s[gi] = (int8_t)(s < 127 ? s : 127);
    if (po.e1) po.e1[gi] = pe1[z];
    if (po.e2) po.e2[gi] = 0.0;
    if (po.norms) { po.norms[2 * gi] = n1; po.norms[2 * gi + 1] = NAN; }
    if (po.mults) po.mults[gi] = m + s;
    if (po.nonfinite) po.nonfinite[gi] = (uint8_t)(flags[z] || !(n1 < INFINITY));
  }
}

template <typename T>
static int large_run_chunk_alg1(const T* W, T* X, int64_t cnt, int n, double eps, int64_t base, PlanOut po,
                                unsigned char* ws, const LargeLayout& L, cudaStream_t st) {
  const int ic = (int)cnt;
  const size_t nn = (size_t)n * n;
  auto buf = [&](int b) { return reinterpret_cast<T*>(ws + L.off_bufs + (size_t)b * L.mat_bytes * L.chunk); };
  double* part = reinterpret_cast<double*>(ws + L.off_part);
  double* nrm4 = reinterpret_cast<double*>(ws + L.off_norm1);
  double* de1 = reinterpret_cast<double*>(ws + L.off_e1);
  int* lists = reinterpret_cast<int*>(ws + L.off_list);  // [2][chunk] ping-pong, s32 [chunk], m32 [chunk]
  int* la = lists;
  int* lb = lists + L.chunk;
  int* s32 = lists + 2 * L.chunk;
  int* m32 = lists + 3 * L.chunk;
  int* dcnt = reinterpret_cast<int*>(ws + L.off_cnt);  // [0..kA1MaxTerms] list sizes, [kA1MaxTerms+1] max s
  if (cudaMemsetAsync(dcnt, 0, 256, st) != cudaSuccess) return EXPMB_ERR_CUDA;

  GemmCtx<T> g{};
  g.n = n;
  g.W = W;
  g.X = X;
  g.mstride = (int64_t)(L.mat_bytes / sizeof(T));
  g.wstride = (int64_t)nn;
  g.tiles_m = L.tiles_m;
  g.part = part;
  g.s32 = s32;
  g.W2 = buf(0); g.Y0 = buf(1); g.Y1 = buf(2); g.Tmp = buf(5);

  dim3 cgrid((n + 255) / 256, L.tiles_m, ic);
  k_colsum_partial<T><<<cgrid, 256, 0, st>>>(W, n, (int64_t)nn, part, L.tiles_m);
  k_a1_init<<<ic, 256, 0, st>>>(part, L.tiles_m, n, eps, nrm4, s32, m32, de1, la, dcnt);
  {
    int bx = (int)std::min<size_t>((nn + 255) / 256, 64);
    int by = std::min(ic, std::max(1, sm_count_dev() * 8 / bx));
    k_a1_setup<T><<<dim3(bx, by), 256, 0, st>>>(g, ic);
  }
  // term loop (engine.py:109-112): stage j runs on the matrices still active
  for (int j = 0; j < kA1MaxTerms; ++j) {
    int* cur = (j & 1) ? lb : la;
    int* nxt = (j & 1) ? la : lb;
    g.sq_step = j;
    if (gemm_launch<T>(g, STAGE_A1, cur, ic, st, dcnt + j)) return EXPMB_ERR_CUDA;
    k_a1_check<<<std::min(ic, sm_count_dev() * 4), 256, 0, st>>>(part, L.tiles_m, n, eps, j, cur, dcnt + j, nxt,
                                                                  dcnt + j + 1, m32, de1);
  }
  // squarings: one cooperative launch for every level
  {
    constexpr bool kMMA = sizeof(T) == 8;
    constexpr bool kTwo = sizeof(T) == 4;  // the 1-CTA/SM fp32 variant (two-level accumulation)
    auto kern = k_a1_square<T, kTwo, kMMA>;
    constexpr int smem = simt_smem_bytes<T>();
    static int occ = 0;
    if (occ == 0) {
      if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
        return EXPMB_ERR_CUDA;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, smem) != cudaSuccess || occ < 1) occ = 1;
    }
    const int tiles = ((n + kGemmBN - 1) / kGemmBN) * L.tiles_m;
    const int grid = (int)std::min<int64_t>((int64_t)sm_count_dev() * occ, (int64_t)ic * tiles);
    int icv = ic;
    const int* mp = dcnt + kA1MaxTerms + 1;
    void* args[] = {(void*)&g, (void*)&icv, (void*)&mp};
    if (cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(256), args, smem, st) != cudaSuccess)
      return EXPMB_ERR_CUDA;
  }
  // non-finite scan of X + per-matrix outputs (m = terms, s, e1 = ||last Y||_1, mults = m + s)
  int* flags = reinterpret_cast<int*>(ws + L.off_flags);
  if (cudaMemsetAsync(flags, 0, (size_t)ic * sizeof(int), st) != cudaSuccess) return EXPMB_ERR_CUDA;
  int bx = (int)((nn + 256 * 8 - 1) / (256 * 8));
  if (bx > 1024) bx = 1024;
  k_nonfinite<T><<<dim3(bx, ic), 256, 0, st>>>(X, n, (int64_t)nn, flags);
  k_a1_finish<<<(ic + 255) / 256, 256, 0, st>>>(ic, nrm4, s32, m32, de1, flags, base, po);
  return cudaGetLastError() == cudaSuccess ? EXPMB_OK : EXPMB_ERR_CUDA;
}

static inline int large_expm(const void* W, void* X, int64_t batch, int n, int dtype, double eps, int scheme,
                             PlanOut po, void* workspace, cudaStream_t st) {
  const int es = dtype == 0 ? 4 : 8;
  const LargeLayout L = large_layout(batch, n, es, scheme);
  unsigned char* ws = reinterpret_cast<unsigned char*>(workspace);
  for (int64_t b0 = 0; b0 < batch; b0 += L.chunk) {
    const int64_t cnt = std::min<int64_t>(L.chunk, batch - b0);
    const size_t off = (size_t)b0 * n * n;
    int rc;
    if (scheme == 2 && dtype == 0)
      rc = large_run_chunk_alg1<float>(reinterpret_cast<const float*>(W) + off, reinterpret_cast<float*>(X) + off, cnt,
                                       n, eps, b0, po, ws, L, st);
    else if (scheme == 2)
      rc = large_run_chunk_alg1<double>(reinterpret_cast<const double*>(W) + off, reinterpret_cast<double*>(X) + off,
                                        cnt, n, eps, b0, po, ws, L, st);
    else if (dtype == 0)
      rc = large_run_chunk<float>(reinterpret_cast<const float*>(W) + off, reinterpret_cast<float*>(X) + off, cnt, n,
                                  eps, scheme, b0, po, ws, L, st);
    else
      rc = large_run_chunk<double>(reinterpret_cast<const double*>(W) + off, reinterpret_cast<double*>(X) + off, cnt,
                                   n, eps, scheme, b0, po, ws, L, st);
    if (rc != EXPMB_OK) return rc;
  }
  return EXPMB_OK;
}

}  // namespace expmb
