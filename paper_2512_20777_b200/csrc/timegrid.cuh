// timegrid.cuh -- exp(t_k A) for one A and many times t_k (SURVEY §8(f) rank 3:
// the time-grid / shared-power specialisation of the generative-flow use case,
// BASELINE config C3).
//
// The reference exponentiates every t_k A independently (engine.py:119-152):
// norms, ladder, (budget(m) + s) products each.  Here everything that does not
// depend on t_k is done once:
//   * the powers P_p = A^p, p = 1..16, in binary64 (tiled FMA GEMM, four
//     launches: A^2 | A^3, A^4 | A^5..A^8 | A^9..A^16, each level's products
//     independent);
//   * the power norms, so the plan of t_k A follows from
//     ||(t_k A)^p||_1 = |t_k|^p ||A^p||_1 (k_tg_select runs the same ladder as
//     every other path, select.py:164-220, on those norms);
// and per t_k only
//   * the scaled Taylor polynomial T_m(t_k A / 2^s) = sum_p gamma_{k,p} P_p as
//     one fused linear combination (k_tg_combine: each thread keeps 16 power
//     entries in registers and emits that entry of X_k for a chunk of k, so
//     the powers are read once per chunk, not once per k), gamma_{k,p} =
//     c_p (t_k 2^-s_k)^p with c_p = 1/p! (the Sastre order-8 and order-15+
//     formulas evaluate T_8 and T_15 + b16 A^16 exactly, poly.py:204-230,
//     PAPER eq. (11)-(13); PS evaluates T_m);
//   * the s_k squarings (engine.py:80-87) on the same bucketed GEMM stage as
//     the large-n path (gemm_simt.cuh STAGE_SQ).
// So a time point costs s_k products instead of budget(m_k) + s_k.  The
// evaluation order differs from the reference's formulas (a power sum
// instead of nested products), which the parity bar allows; the plans are
// the reference's up to the last-bit difference between |t| ||A||_1 and
// ||fl(t A)||_1 (the near-threshold exemption).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "gemm_simt.cuh"
#include "large.cuh"
#include "select.cuh"

namespace expmb {

constexpr int kTgPowers = 16;

struct TgLayout {
  int64_t chunk;
  size_t mat_bytes;  // one T matrix, 256-aligned
  size_t off_pow, off_tmp, off_part, off_nrmA, off_nrm4, off_flags, off_m, off_s, off_e1, off_e2, off_list, off_cnt,
      total;
};

static inline TgLayout tg_layout(int64_t K, int n, int esize) {
  TgLayout L{};
  L.mat_bytes = align256((size_t)n * n * esize);
  int64_t chunk = (int64_t)(kLargeWsCap / L.mat_bytes);
  if (chunk < 1) chunk = 1;
  if (chunk > 65535) chunk = 65535;
  if (chunk > K) chunk = K;
  L.chunk = chunk;
  size_t off = 0;
  L.off_pow = off; off += align256((size_t)kTgPowers * n * n * sizeof(double));
  L.off_tmp = off; off += L.mat_bytes * (size_t)chunk;
  L.off_part = off; off += align256((size_t)chunk * ((n + kGemmBM - 1) / kGemmBM) * n * sizeof(double));
  L.off_nrmA = off; off += align256(5 * sizeof(double));  // ||P_p||_1, p = 1..4, and sigma
  L.off_nrm4 = off; off += align256((size_t)chunk * 4 * sizeof(double));
  L.off_flags = off; off += align256((size_t)chunk * sizeof(int));
  L.off_m = off; off += align256((size_t)chunk);
  L.off_s = off; off += align256((size_t)chunk);
  L.off_e1 = off; off += align256((size_t)chunk * sizeof(double));
  L.off_e2 = off; off += align256((size_t)chunk * sizeof(double));
  L.off_list = off; off += align256((size_t)chunk * 5 * sizeof(int));  // k_bucket's five lists
  L.off_cnt = off; off += 256;
  L.total = off;
  return L;
}

template <typename T>
__global__ void k_tg_upcast(const T* __restrict__ A, double* __restrict__ P1, size_t nn) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < nn; i += (size_t)gridDim.x * blockDim.x)
    P1[i] = (double)A[i];
}

// P1 <- A / sigma with sigma = 2^e the power of two that brings ||A||_1 into
// [1/2, 1) (exact): the shared powers are then those of A / sigma, bounded by
// 1 in norm, so A^16 neither overflows for large ||A|| nor underflows for
// small; sigma^p goes into the per-time coefficients.  nrm[4] = sigma.
__global__ void k_tg_normalize(double* __restrict__ P1, size_t nn, double* __restrict__ nrm) {
  const double n0 = nrm[0];
  int e = 0;
  if (n0 > 0.0 && n0 < INFINITY) frexp(n0, &e);
  const double inv = ldexp(1.0, -e);
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < nn; i += (size_t)gridDim.x * blockDim.x)
    P1[i] *= inv;
  if (blockIdx.x == 0 && threadIdx.x == 0) nrm[4] = ldexp(1.0, e);
}

// Up to 8 independent products P[c] = P[a] P[b] per launch (blockIdx.z):
// the powers are built in 4 levels, A^2 | A^3 A^4 | A^5..A^8 | A^9..A^16.
struct TgProducts {
  int a[8], b[8], c[8];
};

// C = A B, binary64, 64 x 64 tiles, 256 threads with 4 x 4 outputs each.
__global__ void __launch_bounds__(256) k_tg_gemm(const double* __restrict__ P, TgProducts pr, int n) {
  __shared__ double sa[16][65];
  __shared__ double sb[16][65];
  const size_t nn = (size_t)n * n;
  const double* __restrict__ A = P + (size_t)pr.a[blockIdx.z] * nn;
  const double* __restrict__ B = P + (size_t)pr.b[blockIdx.z] * nn;
  double* __restrict__ C = const_cast<double*>(P) + (size_t)pr.c[blockIdx.z] * nn;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int r0 = blockIdx.y * 64, c0 = blockIdx.x * 64;
  double acc[4][4] = {};
  for (int k0 = 0; k0 < n; k0 += 16) {
    for (int i = threadIdx.x; i < 16 * 64; i += 256) {
      const int kk = i / 64, rr = i % 64;
      const int ar = r0 + rr, ak = k0 + kk;
      sa[kk][rr] = (ar < n && ak < n) ? A[(size_t)ar * n + ak] : 0.0;
      const int bk = k0 + kk, bc = c0 + rr;
      sb[kk][rr] = (bk < n && bc < n) ? B[(size_t)bk * n + bc] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = sa[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = sb[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = r0 + ty + 16 * i, c = c0 + tx + 16 * j;
      if (r < n && c < n) C[(size_t)r * n + c] = acc[i][j];
    }
}

// ||P_p||_1 for p = 1..4 (one CTA per power; fixed-order column sums).
__global__ void __launch_bounds__(256) k_tg_norms(const double* __restrict__ P, int n, double* __restrict__ nrm) {
  const int p = blockIdx.x;
  const double* M = P + (size_t)p * n * n;
  __shared__ double red[256];
  double mx = 0.0;
  for (int c = threadIdx.x; c < n; c += 256) {
    double a = 0.0;
    for (int r = 0; r < n; ++r) a += fabs(M[(size_t)r * n + c]);
    mx = nanmax(mx, a);
  }
  red[threadIdx.x] = mx;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] = nanmax(red[threadIdx.x], red[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) nrm[p] = red[0];
}

// Plan of t_k A from the shared power norms (select.py:164-220).
template <typename T>
__global__ void k_tg_select(const T* __restrict__ t, int64_t cnt, const double* __restrict__ nrmA, double eps,
                            int scheme, double* __restrict__ nrm4, int8_t* __restrict__ pm, int8_t* __restrict__ ps,
                            double* __restrict__ pe1, double* __restrict__ pe2) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= cnt) return;
  const double at = fabs((double)t[k]) * nrmA[4];  // |t_k| sigma: the powers are of A / sigma
  double nr[4];
  double tp = 1.0;
  for (int p = 0; p < 4; ++p) {
    tp *= at;
    nr[p] = tp * nrmA[p];
  }
  Plan pl{0, 0, 0.0, 0.0};
  if (nr[0] != 0.0 && isfinite(nr[0])) select_walk(nr, scheme == 1 ? 4 : 2, eps, scheme, &pl);
  pm[k] = (int8_t)pl.m;
  ps[k] = (int8_t)pl.s;
  pe1[k] = pl.e1;
  pe2[k] = pl.e2;
  nrm4[4 * k] = nr[0];
  nrm4[4 * k + 1] = pl.m >= 2 ? nr[1] : NAN;  // ||W^2||_1 only when the reference forms W^2
  nrm4[4 * k + 2] = NAN;
  nrm4[4 * k + 3] = NAN;
}

// X_k = sum_p gamma_{k,p} P_p (P_0 = I), written where the squarings expect it.
constexpr int kTgChunkK = 64;

template <typename T>
__global__ void __launch_bounds__(256) k_tg_combine(const double* __restrict__ P, const double* __restrict__ nrmA,
                                                    int n, const T* __restrict__ t,
                                                    int64_t cnt, const int8_t* __restrict__ pm,
                                                    const int8_t* __restrict__ ps, int scheme, T* X, T* Tmp,
                                                    int64_t mstride) {
  __shared__ double gam[kTgChunkK][kTgPowers + 1];
  const int64_t k0 = (int64_t)blockIdx.y * kTgChunkK;
  const int kc = (int)min((int64_t)kTgChunkK, cnt - k0);
  // coefficients of the chunk: gamma_p = c_p tau^p, tau = t 2^-s
  for (int i = threadIdx.x; i < kc; i += blockDim.x) {
    const int64_t k = k0 + i;
    const int m = pm[k], s = ps[k];
    const double tau = (double)t[k] * pow2_neg<double>(s) * nrmA[4];  // t 2^-s sigma (powers of A / sigma)
    const int deg = (scheme == 0 && m == 15) ? 16 : m;
    double tp = 1.0;
    gam[i][0] = 1.0;
    for (int p = 1; p <= kTgPowers; ++p) {
      tp *= tau;
      double c = 0.0;
      if (p <= deg) c = (p == 16 && scheme == 0) ? kT15[0] * kT15[0] * kT15[0] * kT15[0] : kInvFact[p];
      gam[i][p] = c * tp;
    }
  }
  __syncthreads();
  const size_t nn = (size_t)n * n;
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nn) return;
  double pw[kTgPowers];
#pragma unroll
  for (int p = 0; p < kTgPowers; ++p) pw[p] = P[(size_t)p * nn + e];
  const bool diag = (e / n) == (e % n);
  for (int i = 0; i < kc; ++i) {
    const int64_t k = k0 + i;
    double acc = diag ? gam[i][0] : 0.0;
#pragma unroll
    for (int p = 0; p < kTgPowers; ++p) acc = fma(gam[i][p + 1], pw[p], acc);
    const int s = ps[k];
    T* dst = (s % 2 == 0) ? X + k * (int64_t)nn : Tmp + k * mstride;
    dst[e] = (T)acc;
  }
}

// Host orchestration for one chunk of times.
template <typename T>
static int tg_run(const T* A, const T* t, T* X, int64_t K, int n, double eps, int scheme, PlanOut po,
                  unsigned char* ws, const TgLayout& L, cudaStream_t st) {
  const size_t nn = (size_t)n * n;
  double* P = reinterpret_cast<double*>(ws + L.off_pow);
  double* nrmA = reinterpret_cast<double*>(ws + L.off_nrmA);
  // shared powers A^1..A^16 in binary64 and their norms
  k_tg_upcast<T><<<256, 256, 0, st>>>(A, P, nn);
  k_tg_norms<<<1, 256, 0, st>>>(P, n, nrmA);          // ||A||_1
  k_tg_normalize<<<256, 256, 0, st>>>(P, nn, nrmA);   // P1 = A / sigma, nrmA[4] = sigma
  // level L forms A^(h+1) .. A^(2h) as A^h A^(i) (h = 1, 2, 4, 8); index = power - 1
  for (int h = 1; h < kTgPowers; h *= 2) {
    TgProducts pr{};
    int cnt = 0;
    for (int p = h + 1; p <= 2 * h && p <= kTgPowers; ++p, ++cnt) {
      pr.a[cnt] = h - 1;
      pr.b[cnt] = p - h - 1;
      pr.c[cnt] = p - 1;
    }
    k_tg_gemm<<<dim3((n + 63) / 64, (n + 63) / 64, cnt), 256, 0, st>>>(P, pr, n);
  }
  k_tg_norms<<<4, 256, 0, st>>>(P, n, nrmA);

  for (int64_t base = 0; base < K; base += L.chunk) {
    const int64_t cnt = std::min<int64_t>(L.chunk, K - base);
    const int ic = (int)cnt;
    double* nrm4 = reinterpret_cast<double*>(ws + L.off_nrm4);
    int8_t* dm = reinterpret_cast<int8_t*>(ws + L.off_m);
    int8_t* ds = reinterpret_cast<int8_t*>(ws + L.off_s);
    double* de1 = reinterpret_cast<double*>(ws + L.off_e1);
    double* de2 = reinterpret_cast<double*>(ws + L.off_e2);
    int* dlist = reinterpret_cast<int*>(ws + L.off_list);
    T* Xc = X + base * (int64_t)nn;
    T* Tmp = reinterpret_cast<T*>(ws + L.off_tmp);
    const int64_t mstride = (int64_t)(L.mat_bytes / sizeof(T));
    k_tg_select<T><<<(ic + 127) / 128, 128, 0, st>>>(t + base, cnt, nrmA, eps, scheme, nrm4, dm, ds, de1, de2);
    k_tg_combine<T><<<dim3((unsigned)((nn + 255) / 256), (unsigned)((cnt + kTgChunkK - 1) / kTgChunkK)), 256, 0, st>>>(
        P, nrmA, n, t + base, cnt, dm, ds, scheme, Xc, Tmp, mstride);
    // squarings: the device bucket scheduler sorts the chunk by s descending;
    // level q runs on the prefix #(s > q), a count that stays on the device
    int* dcnt = reinterpret_cast<int*>(ws + L.off_cnt);
    k_bucket<<<1, 1024, 0, st>>>(dm, ds, ic, scheme, dlist, dcnt);
    {
      GemmCtx<T> g{};
      g.n = n;
      g.scheme = scheme;
      g.tiles_m = (n + kGemmBM - 1) / kGemmBM;
      g.mstride = mstride;
      g.wstride = (int64_t)nn;
      g.W = Xc;
      g.X = Xc;
      g.Tmp = Tmp;
      g.m = dm;
      g.s = ds;
      g.part = reinterpret_cast<double*>(ws + L.off_part);
      for (int q = 0; q < kMaxSq; ++q) {
        g.sq_step = q;
        if (gemm_launch<T>(g, STAGE_SQ, dlist + (size_t)4 * ic, ic, st, dcnt + kCntSq + q)) return EXPMB_ERR_CUDA;
      }
    }
    // non-finite scan + per-time outputs (mults = the reference's ledger)
    LargeLayout LL{};
    LL.off_flags = L.off_flags;
    launch_finish<T>(Xc, n, ic, scheme, LL, ws, nrm4, dm, ds, de1, de2, base, po, st);
  }
  return cudaGetLastError() == cudaSuccess ? EXPMB_OK : EXPMB_ERR_CUDA;
}

}  // namespace expmb
