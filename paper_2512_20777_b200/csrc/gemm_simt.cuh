// gemm_simt.cuh -- bucketed batched GEMM with the evaluation formulas fused
// into the epilogue (large-n path, n > 64).
//
// One launch = one pipeline stage over a list of matrices (blockIdx.z ->
// list[z]).  Each CTA computes a 128x128 tile of L*R with a register-tiled
// FMA mainloop (8x8 outputs per thread, double-buffered shared memory) and
// then applies the stage's linear combination for ITS matrix's (m, s):
//   out0 = alpha*acc + sum_q c0q*in_q + d0*I
//   out1 = out0      + sum_q c1q*in_q + d1*I
//   out2 = out0      + sum_q c2q*in_q + d2*I
// which is exactly how poly.py:204-230 builds y02/L/R, y12/L/R and the final
// value; power-of-two scalings 2^-s, 2^-2s (engine.py:139-140) are folded
// into alpha and the c's.  Power stages (W^2, W^3, W^4) also emit per-tile
// binary64 column abs-sums for the 1-norm (select.py:193).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "fused_small.cuh"
#include "select.cuh"

namespace expmb {

constexpr int kGemmBM = 128;
constexpr int kGemmBN = 128;
constexpr int kGemmBK = 8;

enum Stage { STAGE_W2 = 0, STAGE_W3, STAGE_W4, STAGE_E1, STAGE_E2, STAGE_E3, STAGE_SQ };

template <typename T>
struct GemmCtx {
  int n;
  int scheme;
  int tiles_m;
  int sq_step;
  int64_t mstride;  // elements between consecutive matrices of a workspace buffer
  int64_t wstride;  // elements between consecutive matrices of W / X (n*n)
  const T* W;
  T* X;
  T *W2, *W3, *W4, *Y0, *Y1, *La, *Ra, *Lb, *Rb, *Tmp;
  const int8_t* m;
  const int8_t* s;
  const int* need;
  double* part;
};

template <typename T>
struct Epi {
  const T* L;
  const T* R;
  T alpha;
  int nin, nout;
  bool colnorm;
  const T* in[4];
  T c[3][4];
  T d[3];
  T* out[3];
};

// pre-squaring target for a matrix squared s times: the buffer that, after s
// ping-pong squarings, leaves the result in the user's X.
template <typename T>
__device__ __forceinline__ T* sq_target(const GemmCtx<T>& g, int z, int s, int k) {
  return ((s - k) % 2 == 0) ? g.X + (int64_t)z * g.wstride : g.Tmp + (int64_t)z * g.mstride;
}

template <typename T>
__device__ __forceinline__ bool make_epi(const GemmCtx<T>& g, int stage, int z, Epi<T>& e) {
  const int64_t o = (int64_t)z * g.mstride;
  const T* Wz = g.W + (int64_t)z * g.wstride;
  e.nin = 0; e.nout = 1; e.colnorm = false; e.alpha = T(1);
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    e.d[k] = T(0);
#pragma unroll
    for (int q = 0; q < 4; ++q) e.c[k][q] = T(0);
  }
  if (stage == STAGE_W2 || stage == STAGE_W3 || stage == STAGE_W4) {
    const int p = stage == STAGE_W2 ? 2 : stage == STAGE_W3 ? 3 : 4;
    if (g.need[z] != p) return false;
    e.L = p == 2 ? Wz : (p == 3 ? g.W2 + o : g.W3 + o);
    e.R = Wz;
    e.out[0] = p == 2 ? g.W2 + o : (p == 3 ? g.W3 + o : g.W4 + o);
    e.colnorm = true;
    return true;
  }
  const int m = g.m[z], s = g.s[z];
  const double sg = pow2_neg<double>(s), sg2 = pow2_neg<double>(2 * s);
  if (stage == STAGE_SQ) {
    if (s <= g.sq_step) return false;
    e.L = e.R = sq_target(g, z, s, g.sq_step);
    e.out[0] = sq_target(g, z, s, g.sq_step + 1);
    return true;
  }
  if (g.scheme == 1) {
    // Paterson-Stockmeyer Horner stage h (poly.py:179-181): q <- q A^j + block(rj, rj+j-1)
    const int h = stage - STAGE_E1;
    const int j = ps_j_of(m), k = ps_k_of(m);
    const int r = k - 2 - h;
    if (r < 0) return false;
    e.L = (h % 2 == 0) ? g.La + o : g.Ra + o;
    e.R = j == 2 ? g.W2 + o : (j == 3 ? g.W3 + o : g.W4 + o);
    e.alpha = (T)pow2_neg<double>(j * s);
    e.out[0] = (r == 0) ? sq_target(g, z, s, 0) : ((h % 2 == 0) ? g.Ra + o : g.La + o);
    e.in[0] = Wz; e.in[1] = g.W2 + o; e.in[2] = g.W3 + o; e.in[3] = g.W4 + o;
    const int lo = r * j, hi = r * j + j - 1;
    e.d[0] = (T)kInvFact[lo];
    e.nin = hi - lo;
    for (int t = 1; t <= hi - lo; ++t) e.c[0][t - 1] = (T)(kInvFact[lo + t] * pow2_neg<double>(t * s));
    return true;
  }
  // Sastre formulas
  const double* c = (m == 8) ? kT8 : kT15;
  e.in[0] = Wz; e.in[1] = g.W2 + o; e.in[2] = g.Y0 + o; e.in[3] = g.Y1 + o;
  if (stage == STAGE_E1) {
    if (m == 4) {  // poly.py:199: inner*A^2/2 + A + I   (s = 0)
      e.L = g.Lb + o; e.R = g.W2 + o;
      e.alpha = T(0.5);
      e.nin = 1; e.c[0][0] = T(1); e.d[0] = T(1);
      e.out[0] = sq_target(g, z, s, 0);
      return true;
    }
    if (m < 8) return false;
    // y02 = A2 (c1 A2 + c2 A); L2 = y02 + c3 A2 + c4 A; R2 = y02 + c5 A2
    e.L = g.W2 + o; e.R = g.Ra + o;
    e.alpha = (T)sg2;
    e.nin = 2; e.nout = 3;
    e.out[0] = g.Y0 + o; e.out[1] = g.Lb + o; e.out[2] = g.Rb + o;
    e.c[1][1] = (T)(c[2] * sg2); e.c[1][0] = (T)(c[3] * sg);
    e.c[2][1] = (T)(c[4] * sg2);
    return true;
  }
  if (stage == STAGE_E2) {
    if (m < 8) return false;
    e.L = g.Lb + o; e.R = g.Rb + o;
    if (m == 8) {  // poly.py:211 (s = 0)
      e.nin = 3;
      e.c[0][2] = (T)c[5]; e.c[0][1] = T(0.5); e.c[0][0] = T(1); e.d[0] = T(1);
      e.out[0] = sq_target(g, z, s, 0);
      return true;
    }
    // y12 = P + c6 y02 + c7 A2; L3 = y12 + c8 A2 + c9 A; R3 = y12 + c10 y02 + c11 A
    e.nin = 3; e.nout = 3;
    e.out[0] = g.Y1 + o; e.out[1] = g.La + o; e.out[2] = g.Ra + o;
    e.c[0][2] = (T)c[5]; e.c[0][1] = (T)(c[6] * sg2);
    e.c[1][1] = (T)(c[7] * sg2); e.c[1][0] = (T)(c[8] * sg);
    e.c[2][2] = (T)c[9]; e.c[2][0] = (T)(c[10] * sg);
    return true;
  }
  // STAGE_E3: y22 = P + c12 y12 + c13 y02 + c14 A2 + c15 A + c16 I
  if (m < 15) return false;
  e.L = g.La + o; e.R = g.Ra + o;
  e.nin = 4;
  e.c[0][3] = (T)c[11]; e.c[0][2] = (T)c[12]; e.c[0][1] = (T)(c[13] * sg2); e.c[0][0] = (T)(c[14] * sg);
  e.d[0] = (T)c[15];
  e.out[0] = sq_target(g, z, s, 0);
  return true;
}

template <typename T>
struct SimtTraits;
template <>
struct SimtTraits<float> {
  static constexpr int LDS = kGemmBM + 4;
};
template <>
struct SimtTraits<double> {
  static constexpr int LDS = kGemmBM + 2;
};

template <typename T>
__global__ void __launch_bounds__(256, 1)
gemm_stage_kernel(GemmCtx<T> g, int stage, const int* __restrict__ list) {
  constexpr int LDS = SimtTraits<T>::LDS;
  __shared__ __align__(16) T As[2][kGemmBK][LDS];
  __shared__ __align__(16) T Bs[2][kGemmBK][LDS];
  const int z = list ? list[blockIdx.z] : (int)blockIdx.z;
  Epi<T> e;
  if (!make_epi(g, stage, z, e)) return;
  const int n = g.n;
  const int m0 = blockIdx.y * kGemmBM, n0 = blockIdx.x * kGemmBN;
  const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
  const int arow = tid / 2, acol = (tid % 2) * 4;
  const int brow = tid / 32, bcol = (tid % 32) * 4;
  const bool vec = (n % 4) == 0;
  const T* __restrict__ Lp = e.L;
  const T* __restrict__ Rp = e.R;

  T ra[4], rb[4];
  auto gload = [&](int k0) {
    const int ar = m0 + arow, ac = k0 + acol;
    const int br = k0 + brow, bc = n0 + bcol;
    if (vec) {
      if (ar < n && ac < n) {
        const T* p = Lp + (size_t)ar * n + ac;
        if constexpr (sizeof(T) == 4) {
          float4 v = __ldg(reinterpret_cast<const float4*>(p));
          ra[0] = v.x; ra[1] = v.y; ra[2] = v.z; ra[3] = v.w;
        } else {
          double2 v0 = __ldg(reinterpret_cast<const double2*>(p)), v1 = __ldg(reinterpret_cast<const double2*>(p) + 1);
          ra[0] = v0.x; ra[1] = v0.y; ra[2] = v1.x; ra[3] = v1.y;
        }
      } else {
        ra[0] = ra[1] = ra[2] = ra[3] = T(0);
      }
      if (br < n && bc < n) {
        const T* p = Rp + (size_t)br * n + bc;
        if constexpr (sizeof(T) == 4) {
          float4 v = __ldg(reinterpret_cast<const float4*>(p));
          rb[0] = v.x; rb[1] = v.y; rb[2] = v.z; rb[3] = v.w;
        } else {
          double2 v0 = __ldg(reinterpret_cast<const double2*>(p)), v1 = __ldg(reinterpret_cast<const double2*>(p) + 1);
          rb[0] = v0.x; rb[1] = v0.y; rb[2] = v1.x; rb[3] = v1.y;
        }
      } else {
        rb[0] = rb[1] = rb[2] = rb[3] = T(0);
      }
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        ra[q] = (ar < n && ac + q < n) ? Lp[(size_t)ar * n + ac + q] : T(0);
        rb[q] = (br < n && bc + q < n) ? Rp[(size_t)br * n + bc + q] : T(0);
      }
    }
  };
  auto sstore = [&](int b) {
#pragma unroll
    for (int q = 0; q < 4; ++q) As[b][acol + q][arow] = ra[q];
#pragma unroll
    for (int q = 0; q < 4; ++q) Bs[b][brow][bcol + q] = rb[q];
  };

  T acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = T(0);

  // fp32: two-level accumulation (a fresh partial every kChunk k-tiles, then
  // added to the running sum) keeps the summation error near
  // (32 + n/32) u instead of n u -- needed for the 1e-5 bar at n = 2048.
  constexpr bool kTwoLevel = sizeof(T) == 4;
  constexpr int kChunk = 4;
  T pacc[kTwoLevel ? 8 : 1][kTwoLevel ? 8 : 1];
  const int nk = (n + kGemmBK - 1) / kGemmBK;
  gload(0);
  sstore(0);
  __syncthreads();
  for (int kt = 0; kt < nk; ++kt) {
    const int cur = kt & 1;
    if (kt + 1 < nk) gload((kt + 1) * kGemmBK);
    if constexpr (kTwoLevel) {
      if (kt % kChunk == 0) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 8; ++j) pacc[i][j] = T(0);
      }
    }
#pragma unroll
    for (int k = 0; k < kGemmBK; ++k) {
      T a[8], b[8];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const T* pa = &As[cur][k][h * 64 + ty * 4];
        const T* pb = &Bs[cur][k][h * 64 + tx * 4];
        if constexpr (sizeof(T) == 4) {
          float4 va = *reinterpret_cast<const float4*>(pa), vb = *reinterpret_cast<const float4*>(pb);
          a[4 * h] = va.x; a[4 * h + 1] = va.y; a[4 * h + 2] = va.z; a[4 * h + 3] = va.w;
          b[4 * h] = vb.x; b[4 * h + 1] = vb.y; b[4 * h + 2] = vb.z; b[4 * h + 3] = vb.w;
        } else {
          double2 a0 = reinterpret_cast<const double2*>(pa)[0], a1 = reinterpret_cast<const double2*>(pa)[1];
          double2 b0 = reinterpret_cast<const double2*>(pb)[0], b1 = reinterpret_cast<const double2*>(pb)[1];
          a[4 * h] = a0.x; a[4 * h + 1] = a0.y; a[4 * h + 2] = a1.x; a[4 * h + 3] = a1.y;
          b[4 * h] = b0.x; b[4 * h + 1] = b0.y; b[4 * h + 2] = b1.x; b[4 * h + 3] = b1.y;
        }
      }
      if constexpr (kTwoLevel) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 8; ++j) pacc[i][j] = fma(a[i], b[j], pacc[i][j]);
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
      }
    }
    if constexpr (kTwoLevel) {
      if (kt % kChunk == kChunk - 1 || kt + 1 == nk) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[i][j] += pacc[i][j];
      }
    }
    if (kt + 1 < nk) sstore(cur ^ 1);
    __syncthreads();
  }

  // ---- fused epilogue --------------------------------------------------
  double csum[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) csum[j] = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int row = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + i - 4);
    if (row >= n) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int col = n0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + j - 4);
      if (col >= n) continue;
      const size_t pos = (size_t)row * n + col;
      const T dg = (row == col) ? T(1) : T(0);
      T o0 = e.alpha * acc[i][j];
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (q < e.nin) o0 = fma(e.c[0][q], e.in[q][pos], o0);
      o0 = fma(e.d[0], dg, o0);
      e.out[0][pos] = o0;
      if (e.nout > 1) {
        T o1 = o0, o2 = o0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (q < e.nin) {
            const T v = e.in[q][pos];
            o1 = fma(e.c[1][q], v, o1);
            o2 = fma(e.c[2][q], v, o2);
          }
        }
        e.out[1][pos] = fma(e.d[1], dg, o1);
        e.out[2][pos] = fma(e.d[2], dg, o2);
      }
      if (e.colnorm) csum[j] += fabs((double)o0);
    }
  }
  if (e.colnorm) {
    // deterministic column reduction over the 16 thread rows of the tile
    double* red = reinterpret_cast<double*>(&As[0][0][0]);  // 16 x 128 doubles fit in As+Bs
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 8; ++j) red[ty * kGemmBN + (j < 4 ? tx * 4 + j : 64 + tx * 4 + j - 4)] = csum[j];
    __syncthreads();
    if (tid < kGemmBN && n0 + tid < n) {
      double a = 0.0;
      for (int r = 0; r < 16; ++r) a += red[r * kGemmBN + tid];
      g.part[((size_t)z * g.tiles_m + blockIdx.y) * n + n0 + tid] = a;
    }
  }
}

template <typename T>
static int gemm_launch(const GemmCtx<T>& g, int stage, const int* list, int count, cudaStream_t st) {
  if (count <= 0) return 0;
  const int tn = (g.n + kGemmBN - 1) / kGemmBN, tm = (g.n + kGemmBM - 1) / kGemmBM;
  dim3 grid(tn, tm, count);
  gemm_stage_kernel<T><<<grid, 256, 0, st>>>(g, stage, list);
  return cudaGetLastError() != cudaSuccess;
}

// ---------------------------------------------------------------------------
// elementwise stage (before the first evaluation product)
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(256) elem_kernel(GemmCtx<T> g, const int* __restrict__ list) {
  const int z = list[blockIdx.y];
  const int m = g.m[z], s = g.s[z];
  const int n = g.n;
  const size_t nn = (size_t)n * n;
  const int64_t o = (int64_t)z * g.mstride;
  const T* Wz = g.W + (int64_t)z * g.wstride;
  const T* A2 = g.W2 + o;
  const double sg = pow2_neg<double>(s), sg2 = pow2_neg<double>(2 * s);
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < nn; i += (size_t)gridDim.x * blockDim.x) {
    const int r = (int)(i / n), c = (int)(i % n);
    const T dg = (r == c) ? T(1) : T(0);
    if (g.scheme == 1) {
      if (m == 0) { sq_target(g, z, s, 0)[i] = dg; continue; }
      const int j = ps_j_of(m), k = ps_k_of(m);
      const int lo = (k - 1) * j;
      T acc = (T)kInvFact[lo] * dg;
      const T pw[4] = {Wz[i], m >= 2 ? A2[i] : T(0), j >= 3 ? g.W3[o + i] : T(0), j >= 4 ? g.W4[o + i] : T(0)};
      for (int t = 1; t <= m - lo; ++t) acc = fma((T)(kInvFact[lo + t] * pow2_neg<double>(t * s)), pw[t - 1], acc);
      if (k == 1) sq_target(g, z, s, 0)[i] = acc;
      else g.La[o + i] = acc;
      continue;
    }
    if (m == 0) {
      sq_target(g, z, s, 0)[i] = dg;
    } else if (m == 1) {  // poly.py:192
      sq_target(g, z, s, 0)[i] = Wz[i] + dg;
    } else if (m == 2) {  // poly.py:196 (s = 0)
      sq_target(g, z, s, 0)[i] = (A2[i] * T(0.5) + Wz[i]) + dg;
    } else if (m == 4) {  // poly.py:198 inner factor (s = 0)
      g.Lb[o + i] = (A2[i] * T(0.25) + Wz[i]) / T(3) + dg;
    } else {  // R1 = c1 A^2 + c2 A with A^p = 2^-ps W^p
      const double* cc = (m == 8) ? kT8 : kT15;
      g.Ra[o + i] = (T)(cc[0] * sg2) * A2[i] + (T)(cc[1] * sg) * Wz[i];
    }
  }
}

template <typename T>
static int elem_launch(const GemmCtx<T>& g, const int* list, int count, cudaStream_t st) {
  if (count <= 0) return 0;
  const size_t nn = (size_t)g.n * g.n;
  int bx = (int)((nn + 255) / 256);
  if (bx > 64) bx = 64;
  dim3 grid(bx, count);
  elem_kernel<T><<<grid, 256, 0, st>>>(g, list);
  return cudaGetLastError() != cudaSuccess;
}

}  // namespace expmb
