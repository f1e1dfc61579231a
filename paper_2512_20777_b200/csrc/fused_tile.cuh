// fused_tile.cuh -- one CTA per matrix for 64 < n <= 128 (fp64; fp32 opt-in): the whole program
// of engine.py:119-152 in one persistent kernel.
//
// For these orders a matrix is exactly one 128 x 128 GEMM tile, so the CTA
// that owns it runs every step back to back with no launch boundary and no
// grid-wide dependency: ||W||_1 (the slab sums k_colsum_partial forms), the
// ladder (select.py:164-220, the block reduction k_select runs), W^2 (W^3,
// W^4 on the PS ladder) with its column norms in the GEMM epilogue, the
// first elementwise step, the evaluation products with the formula's linear
// combinations fused into their epilogues (poly.py:189-230), the s squarings
// (engine.py:80-87), the non-finite scan and the plan outputs.  The
// intermediates live in a per-CTA scratch region that the next matrix of the
// same CTA reuses, so the working set is SMs x CTAs/SM x a few n x n buffers
// and stays in L2: HBM sees one read of W and one write of e^W per matrix.
// Every step is the same device code the bucketed pipeline runs (gemm_tile,
// make_epi, select_block, elem_one, finish_one) in the same order, so the
// results are bit-identical to the pipeline's.
#pragma once

#include "large.cuh"

namespace expmb {

struct FtLayout {
  size_t mat_bytes, per_cta;
  int nbufs, tiles_m;
  size_t off_part, off_misc;
};

static inline FtLayout ft_layout(int n, int esize, int scheme) {
  FtLayout L{};
  L.mat_bytes = align256((size_t)n * n * esize);
  L.nbufs = scheme == 1 ? kLargeBufsPS : kLargeBufsSastre;
  L.tiles_m = (n + kGemmBM - 1) / kGemmBM;
  L.off_part = L.mat_bytes * L.nbufs;
  L.off_misc = L.off_part + align256((size_t)L.tiles_m * n * sizeof(double));
  L.per_cta = L.off_misc + 256;  // need, m, s, e1, e2, nrm4[4]
  return L;
}

// One product tile of the per-matrix program.
template <typename T, bool TWO, bool MMA>
__device__ __forceinline__ void ft_tile(const GemmCtx<T>& g, int stage, int bx, int by, unsigned char* smem_raw) {
  gemm_tile<T, TWO, MMA>(g, stage, nullptr, 0, bx, by, smem_raw);
}

// One CTA per SM (fp64 runs its products on DMMA at one CTA per SM in the
// pipeline too).  Measured on B200 against the pipeline (tools/fused_tile_bench.py,
// profiles/fused_tile_r02.json): fp64 1.26x at n = 96, 1.14x at n = 128; fp32
// 0.87x / 0.85x -- the fp32 stage kernel runs two CTAs per SM at 128 registers,
// which the per-matrix program cannot fit without spilling (1.7 KB inlined,
// 0.4 KB with an out-of-line tile), so fp32 stays on the pipeline by default.
template <typename T, bool TWO, bool MMA>
__global__ void __launch_bounds__(256, 1)
expm_tile_fused_kernel(GemmCtx<T> g0, int64_t batch, double log_eps, int scheme, PlanOut po, unsigned char* ws,
                       size_t per_cta, size_t mat_bytes, size_t off_part, size_t off_misc) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int n = g0.n;
  const size_t nn = (size_t)n * n;
  const int tiles_m = g0.tiles_m, tn = (n + kGemmBN - 1) / kGemmBN;
  unsigned char* mine = ws + (size_t)blockIdx.x * per_cta;
  auto buf = [&](int b) { return reinterpret_cast<T*>(mine + (size_t)b * mat_bytes); };
  double* part = reinterpret_cast<double*>(mine + off_part);
  unsigned char* misc = mine + off_misc;
  double* nrm4 = reinterpret_cast<double*>(misc);            // [4]
  double* pe1 = nrm4 + 4;
  double* pe2 = nrm4 + 5;
  int* need = reinterpret_cast<int*>(misc + 64);
  int8_t* pm = reinterpret_cast<int8_t*>(misc + 80);
  int8_t* ps = reinterpret_cast<int8_t*>(misc + 96);

  for (int64_t z = blockIdx.x; z < batch; z += gridDim.x) {
    // the pipeline's context, re-based so that "matrix 0" is this one and the
    // buffers are this CTA's scratch
    GemmCtx<T> g = g0;
    g.W = g0.W + (size_t)z * nn;
    g.X = g0.X + (size_t)z * nn;
    g.mstride = 0;
    g.m = pm;
    g.s = ps;
    g.need = need;
    g.part = part;
    if (scheme == 0) {
      g.W2 = buf(0); g.Y0 = buf(1); g.Y1 = buf(2); g.La = buf(3); g.Ra = buf(4); g.Lb = buf(5); g.Rb = buf(6);
      g.Tmp = g.Lb;
    } else {
      g.W2 = buf(0); g.W3 = buf(1); g.W4 = buf(2); g.La = buf(3); g.Ra = buf(4); g.Tmp = buf(5);
    }
    __syncthreads();  // the previous matrix's readers of the scratch and of `part` are done
    // ||W||_1 slab partials in k_colsum_partial's order
    for (int idx = threadIdx.x; idx < tiles_m * n; idx += blockDim.x) {
      const int slab = idx / n, c = idx - slab * n, r0 = slab * kGemmBM, r1 = min(n, r0 + kGemmBM);
      double a = 0.0;
      for (int r = r0; r < r1; ++r) a += fabs((double)g.W[(size_t)r * n + c]);
      part[(size_t)slab * n + c] = a;
    }
    __syncthreads();
    select_block(part, tiles_m, n, 1, log_eps, scheme, nrm4, need, pm, ps, pe1, pe2, 0);
    __syncthreads();
    // powers + ladder (W^2; PS: W^3, W^4)
    const int maxp = scheme == 1 ? 4 : 2;
    for (int p = 2; p <= maxp; ++p) {
      if (need[0] != p) break;
      const int stage = p == 2 ? STAGE_W2 : (p == 3 ? STAGE_W3 : STAGE_W4);
      for (int t = 0; t < tn * tiles_m; ++t) {
        __syncthreads();
        ft_tile<T, TWO, MMA>(g, stage, t % tn, t / tn, smem_raw);
      }
      __syncthreads();
      select_block(part, tiles_m, n, p, log_eps, scheme, nrm4, need, pm, ps, pe1, pe2, 0);
      __syncthreads();
    }
    if (po.plan_only) {  // select_sastre / select_ps: the plan is all the caller wants
      if (threadIdx.x == 0) finish_one(0, scheme, nrm4, pm, ps, pe1, pe2, 0, z, po);
      continue;
    }
    // first elementwise step, evaluation products, squarings
    elem_one(g, 0, threadIdx.x, blockDim.x);
    for (int stage = STAGE_E1; stage <= STAGE_E3; ++stage)
      for (int t = 0; t < tn * tiles_m; ++t) {
        __syncthreads();
        ft_tile<T, TWO, MMA>(g, stage, t % tn, t / tn, smem_raw);
      }
    const int s = ps[0];
    for (int q = 0; q < s; ++q) {
      g.sq_step = q;
      for (int t = 0; t < tn * tiles_m; ++t) {
        __syncthreads();
        ft_tile<T, TWO, MMA>(g, STAGE_SQ, t % tn, t / tn, smem_raw);
      }
    }
    __syncthreads();
    int bad = 0;
    for (size_t i = threadIdx.x; i < nn; i += blockDim.x) bad |= !isfinite(g.X[i]);
    bad = __syncthreads_or(bad);
    if (threadIdx.x == 0) finish_one(0, scheme, nrm4, pm, ps, pe1, pe2, bad, z, po);
  }
}

static inline size_t ft_workspace_bytes(int64_t batch, int n, int esize, int scheme, int ctas) {
  const FtLayout L = ft_layout(n, esize, scheme);
  const int64_t g = std::min<int64_t>(batch, ctas);
  return L.per_cta * (size_t)(g > 0 ? g : 1);
}

// resident CTAs of the fused tile kernel (its __launch_bounds__)
static inline int ft_ctas(int esize) {
  (void)esize;
  return sm_count_dev();
}

template <typename T>
static int ft_run(const T* W, T* X, int64_t batch, int n, double eps, int scheme, PlanOut po, unsigned char* ws,
                  cudaStream_t st) {
  const FtLayout L = ft_layout(n, sizeof(T), scheme);
  constexpr bool kMMA = sizeof(T) == 8;
  auto kern = expm_tile_fused_kernel<T, false, kMMA>;
  constexpr int smem = simt_smem_bytes<T>();
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
      return EXPMB_ERR_CUDA;
    attr = true;
  }
  GemmCtx<T> g{};
  g.n = n;
  g.scheme = scheme;
  g.tiles_m = L.tiles_m;
  g.wstride = (int64_t)n * n;
  g.W = W;
  g.X = X;
  const int grid = (int)std::min<int64_t>(batch, ft_ctas(sizeof(T)));
  kern<<<grid, 256, smem, st>>>(g, batch, log2(eps), scheme, po, ws, L.per_cta, L.mat_bytes, L.off_part,
                                L.off_misc);
  return cudaGetLastError() == cudaSuccess ? EXPMB_OK : EXPMB_ERR_CUDA;
}

}  // namespace expmb
