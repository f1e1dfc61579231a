// fused_small.cuh -- one fused kernel per matrix group for n <= 64.
//
// Everything /root/reference/pkg/src/expmkit/engine.py:119-152 does for one
// matrix -- ||W||_1, W^2 and ||W^2||_1 (select.py:169-194), the ladder
// (select.py:180-219), exact 2^-s rescaling (engine.py:139-140), the
// T1/T2/T4/T8/T15+ formulas (poly.py:189-230) or Paterson-Stockmeyer
// (poly.py:149-182), and s squarings (engine.py:80-87) -- runs inside one
// thread group with the matrix resident in registers and shared memory:
// one coalesced HBM read of W and one write of e^W per matrix.
//
// Layout.  A group of TPG = NPAD^2/(4*TM) threads owns one matrix; thread
// (tr, tc) holds rows {tr + i*NPAD/TM : i < TM} x cols {4tc .. 4tc+3} of every
// state matrix (B, A^2, y02, y12, ...) in registers.  Products stage their two
// operands row-major in shared memory (row stride NPAD + 16/sizeof(T) so
// the rows one warp reads fall in distinct bank groups) and every thread
// accumulates its TM x 4 tile with 128-bit shared loads: TM + 4*KV/KV... i.e.
// (TM + 4) vector loads per KV k-steps for 4*TM*KV FMAs.
//
// Groups never synchronise with each other, so matrices with different
// (m, s) in one CTA do not diverge: control flow is uniform per group.
// NPAD=16 uses one warp per matrix (8 matrices per 256-thread CTA);
// NPAD=32 two warps per matrix; NPAD=64 one 256-thread CTA per matrix.
// The CTAs are persistent and prefetch the next matrix into registers while
// the current one is being exponentiated.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "select.cuh"

namespace expmb {

// poly.py:75-101 -- published binary64 literals.
__constant__ double kT8[6] = {
    4.980119205559973e-3, 1.992047682223989e-2, 7.665265321119147e-2,
    8.765009801785554e-1, 1.225521150112075e-1, 2.974307204847627e0};
__constant__ double kT15[16] = {
    4.018761610201036e-4, 2.945531440279683e-3, -8.709066576837676e-3,
    4.017568440673568e-1, 3.230762888122312e-2, 5.768988513026145e0,
    2.338576034271299e-2, 2.381070373870987e-1, 2.224209172496374e0,
    -5.792361707073261e0, -4.130276365929783e-2, 1.040801735231354e1,
    -6.331712455883370e1, 3.484665863364574e-1, 1.0, 1.0};
// poly.py:56-59 taylor_coeffs_exp: 1/i! for i = 0..16, correctly rounded.
__constant__ double kInvFact[17] = {
    0x1.0000000000000p+0, 0x1.0000000000000p+0, 0x1.0000000000000p-1,
    0x1.5555555555555p-3, 0x1.5555555555555p-5, 0x1.1111111111111p-7,
    0x1.6c16c16c16c17p-10, 0x1.a01a01a01a01ap-13, 0x1.a01a01a01a01ap-16,
    0x1.71de3a556c734p-19, 0x1.27e4fb7789f5cp-22, 0x1.ae64567f544e4p-26,
    0x1.1eed8eff8d898p-29, 0x1.6124613a86d09p-33, 0x1.93974a8c07c9dp-37,
    0x1.ae7f3e733b81fp-41, 0x1.ae7f3e733b81fp-45};

struct PlanOut {
  int8_t* m;
  int8_t* s;
  double* e1;
  double* e2;
  double* norms;
  int32_t* mults;
  uint8_t* nonfinite;
};

template <typename T>
struct Vec;
template <>
struct Vec<float> {
  static constexpr int KV = 4;
};
template <>
struct Vec<double> {
  static constexpr int KV = 2;
};

__device__ __forceinline__ bool is_finite_t(float x) { return isfinite(x); }
__device__ __forceinline__ bool is_finite_t(double x) { return isfinite(x); }

// max that propagates NaN (a NaN norm must not be hidden by fmax).
__device__ __forceinline__ double nanmax(double a, double b) { return (a > b || a != a) ? a : b; }

template <typename T, int NPAD, int TM, int GROUPS, int SCHEME>
struct Fused {
  static constexpr int TC = NPAD / 4;            // column quads
  static constexpr int TR = NPAD / TM;           // row phases
  static constexpr int TPG = TC * TR;            // threads per group
  static constexpr int NT = TPG * GROUPS;        // threads per CTA
  static constexpr int KV = Vec<T>::KV;          // k-steps per 128-bit load
  static constexpr int LD = NPAD + KV;           // padded smem row stride (elements)
  static constexpr int WARPS_PG = (TPG + 31) / 32;
  static constexpr int BUF = NPAD * LD;          // one operand buffer (elements)
  // dynamic smem per CTA: two operand buffers per group + reduction scratch
  static constexpr size_t kSmemGroup = 2 * BUF * sizeof(T) + (WARPS_PG > 1 ? WARPS_PG * NPAD * sizeof(double) + 64 : 0);
  static constexpr size_t kSmem = GROUPS * kSmemGroup;

  using Tile = T[TM][4];

  int tr, tc, g, t;
  T* buf0;
  T* buf1;
  double* red;

  __device__ __forceinline__ void sync() const {
    if constexpr (TPG == 32) {
      __syncwarp();
    } else if constexpr (GROUPS == 1) {
      __syncthreads();
    } else {
      asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "r"(TPG) : "memory");
    }
  }

  __device__ __forceinline__ int row(int i) const { return tr + i * TR; }

  __device__ __forceinline__ void store(T* buf, const Tile& v) const {
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      T* p = buf + row(i) * LD + 4 * tc;
      if constexpr (sizeof(T) == 4) {
        *reinterpret_cast<float4*>(p) = make_float4(v[i][0], v[i][1], v[i][2], v[i][3]);
      } else {
        reinterpret_cast<double2*>(p)[0] = make_double2(v[i][0], v[i][1]);
        reinterpret_cast<double2*>(p)[1] = make_double2(v[i][2], v[i][3]);
      }
    }
  }

  // acc = L * R with L, R row-major NPAD x NPAD in shared memory.
  __device__ __forceinline__ void mm(const T* __restrict__ L, const T* __restrict__ R, Tile& acc) const {
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = T(0);
#pragma unroll(NPAD <= 16 ? NPAD / KV : 4)
    for (int kb = 0; kb < NPAD; kb += KV) {
      T a[TM][KV];
#pragma unroll
      for (int i = 0; i < TM; ++i) {
        const T* p = L + row(i) * LD + kb;
        if constexpr (sizeof(T) == 4) {
          float4 v = *reinterpret_cast<const float4*>(p);
          a[i][0] = v.x; a[i][1] = v.y; a[i][2] = v.z; a[i][3] = v.w;
        } else {
          double2 v = *reinterpret_cast<const double2*>(p);
          a[i][0] = v.x; a[i][1] = v.y;
        }
      }
#pragma unroll
      for (int kk = 0; kk < KV; ++kk) {
        T b[4];
        const T* q = R + (kb + kk) * LD + 4 * tc;
        if constexpr (sizeof(T) == 4) {
          float4 v = *reinterpret_cast<const float4*>(q);
          b[0] = v.x; b[1] = v.y; b[2] = v.z; b[3] = v.w;
        } else {
          double2 v0 = reinterpret_cast<const double2*>(q)[0];
          double2 v1 = reinterpret_cast<const double2*>(q)[1];
          b[0] = v0.x; b[1] = v0.y; b[2] = v1.x; b[3] = v1.y;
        }
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i][kk], b[j], acc[i][j]);
      }
    }
  }

  // out = L * R where L, R are register tiles (stages through smem).
  __device__ __forceinline__ void product(const Tile& Lt, const Tile& Rt, Tile& out) const {
    store(buf0, Lt);
    store(buf1, Rt);
    sync();
    mm(buf0, buf1, out);
    sync();
  }
  __device__ __forceinline__ void square(const Tile& Xt, Tile& out) const {
    store(buf0, Xt);
    sync();
    mm(buf0, buf0, out);
    sync();
  }

  // ||.||_1 of the group's matrix: column abs-sums in binary64, then max.
  __device__ __forceinline__ double norm1(const Tile& v) const {
    double cs[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      double a = 0.0;
#pragma unroll
      for (int i = 0; i < TM; ++i) a += fabs((double)v[i][j]);
      cs[j] = a;
    }
    // reduce over the thread rows that share this column quad inside the warp
#pragma unroll
    for (int off = TC; off < 32 && off < TPG; off *= 2)
#pragma unroll
      for (int j = 0; j < 4; ++j) cs[j] += __shfl_xor_sync(0xffffffffu, cs[j], off);
    if constexpr (WARPS_PG == 1) {
      double mx = nanmax(nanmax(cs[0], cs[1]), nanmax(cs[2], cs[3]));
#pragma unroll
      for (int off = 1; off < TC; off *= 2) mx = nanmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
      return mx;
    } else {
      const int w = t / 32, lane = t % 32;
      if (lane < TC) {
#pragma unroll
        for (int j = 0; j < 4; ++j) red[w * NPAD + 4 * lane + j] = cs[j];
      }
      sync();
      double* res = red + WARPS_PG * NPAD;
      if (t < 32) {
        double mx = -INFINITY;
        for (int col = t; col < NPAD; col += 32) {
          double a = 0.0;
          for (int ww = 0; ww < WARPS_PG; ++ww) a += red[ww * NPAD + col];
          mx = nanmax(mx, a);
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) mx = nanmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
        if (t == 0) res[0] = mx;
      }
      sync();
      double r = res[0];
      sync();
      return r;
    }
  }

  __device__ __forceinline__ bool any_group(bool f) const {
    if constexpr (WARPS_PG == 1) {
      return __any_sync(0xffffffffu, f);
    } else {
      int* flag = reinterpret_cast<int*>(red + WARPS_PG * NPAD) + 2;
      if (t == 0) *flag = 0;
      sync();
      if (__any_sync(0xffffffffu, f) && (t % 32) == 0) atomicOr(flag, 1);
      sync();
      int r = *flag;
      sync();
      return r != 0;
    }
  }

  __device__ __forceinline__ void load(const T* __restrict__ src, int n, bool vec, Tile& v) const {
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      const int r = row(i);
      if (vec) {
        const T* p = src + r * NPAD + 4 * tc;
        if constexpr (sizeof(T) == 4) {
          float4 q = __ldg(reinterpret_cast<const float4*>(p));
          v[i][0] = q.x; v[i][1] = q.y; v[i][2] = q.z; v[i][3] = q.w;
        } else {
          double2 q0 = __ldg(reinterpret_cast<const double2*>(p));
          double2 q1 = __ldg(reinterpret_cast<const double2*>(p) + 1);
          v[i][0] = q0.x; v[i][1] = q0.y; v[i][2] = q1.x; v[i][3] = q1.y;
        }
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int c = 4 * tc + j;
          v[i][j] = (r < n && c < n) ? __ldg(src + (size_t)r * n + c) : T(0);
        }
      }
    }
  }

  __device__ __forceinline__ void save(T* __restrict__ dst, int n, bool vec, const Tile& v) const {
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      const int r = row(i);
      if (vec) {
        T* p = dst + r * NPAD + 4 * tc;
        if constexpr (sizeof(T) == 4) {
          __stcs(reinterpret_cast<float4*>(p), make_float4(v[i][0], v[i][1], v[i][2], v[i][3]));
        } else {
          __stcs(reinterpret_cast<double2*>(p), make_double2(v[i][0], v[i][1]));
          __stcs(reinterpret_cast<double2*>(p) + 1, make_double2(v[i][2], v[i][3]));
        }
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int c = 4 * tc + j;
          if (r < n && c < n) dst[(size_t)r * n + c] = v[i][j];
        }
      }
    }
  }

  __device__ __forceinline__ bool is_diag(int i, int j) const { return row(i) == 4 * tc + j; }
};

template <typename T, int NPAD, int TM, int GROUPS, int SCHEME>
__global__ void __launch_bounds__(Fused<T, NPAD, TM, GROUPS, SCHEME>::NT, (NPAD == 16 && sizeof(T) == 4) ? 2 : 1)
expm_fused_kernel(const T* __restrict__ W, T* __restrict__ X, int64_t batch, int n, double eps, PlanOut po) {
  using F = Fused<T, NPAD, TM, GROUPS, SCHEME>;
  using Tile = typename F::Tile;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  F f;
  f.g = threadIdx.x / F::TPG;
  f.t = threadIdx.x % F::TPG;
  f.tr = f.t / F::TC;
  f.tc = f.t % F::TC;
  unsigned char* gbase = smem_raw + f.g * F::kSmemGroup;
  f.buf0 = reinterpret_cast<T*>(gbase);
  f.buf1 = f.buf0 + F::BUF;
  f.red = reinterpret_cast<double*>(f.buf1 + F::BUF);

  const bool vec = (n == NPAD);
  const size_t nn = (size_t)n * n;
  const int64_t stride = (int64_t)gridDim.x * GROUPS;
  int64_t idx = (int64_t)blockIdx.x * GROUPS + f.g;
  if (idx >= batch) return;  // whole group exits together

  Tile w;
  f.load(W + idx * nn, n, vec, w);
  for (; idx < batch; idx += stride) {
    // prefetch the next matrix of this group while this one is processed
    Tile nxt;
    const int64_t nidx = idx + stride;
    if (nidx < batch) f.load(W + nidx * nn, n, vec, nxt);

    bool bad = false;
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) bad |= !is_finite_t(w[i][j]);

    // ---- selection (select.py:164-220) --------------------------------
    double nrm[4];
    nrm[0] = f.norm1(w);
    nrm[1] = nrm[2] = nrm[3] = NAN;
    Plan p;
    int need = select_walk(nrm, 1, eps, SCHEME, &p);
    Tile a2, a3, a4;
    if (need >= 2) {  // W^2 = W W (select.py:192)
      f.square(w, a2);
      nrm[1] = f.norm1(a2);
      bad |= !(nrm[1] < INFINITY);  // W^2 overflowed or is NaN (matrix.py:97-98)
      need = select_walk(nrm, 2, eps, SCHEME, &p);
      if constexpr (SCHEME == 1) {
        if (need >= 3) {  // W^3 = W^2 W
          f.product(a2, w, a3);
          nrm[2] = f.norm1(a3);
          need = select_walk(nrm, 3, eps, SCHEME, &p);
          if (need >= 4) {  // W^4 = W^3 W
            f.product(a3, w, a4);
            nrm[3] = f.norm1(a4);
            need = select_walk(nrm, 4, eps, SCHEME, &p);
          }
        }
      }
    }
    const int m = p.m, s = p.s;

    // ---- exact 2^-s rescaling of W and cached powers (engine.py:139-140)
    const T sc = (T)ldexp(1.0, -s);
    const T sc2 = (T)ldexp(1.0, -2 * s);
    Tile B, A2;
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        B[i][j] = w[i][j] * sc;
        A2[i][j] = a2[i][j] * sc2;
      }

    Tile Xt;
    if (m == 0) {
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) Xt[i][j] = f.is_diag(i, j) ? T(1) : T(0);
    } else if constexpr (SCHEME == 0) {
      if (m == 1) {  // poly.py:192: A + I
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) Xt[i][j] = B[i][j] + (f.is_diag(i, j) ? T(1) : T(0));
      } else if (m == 2) {  // poly.py:196: A^2/2 + A + I
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j)
            Xt[i][j] = (A2[i][j] * T(0.5) + B[i][j]) + (f.is_diag(i, j) ? T(1) : T(0));
      } else if (m == 4) {  // poly.py:198-199
        Tile inner, P;
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j)
            inner[i][j] = (A2[i][j] * T(0.25) + B[i][j]) / T(3) + (f.is_diag(i, j) ? T(1) : T(0));
        f.product(inner, A2, P);
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j)
            Xt[i][j] = (P[i][j] * T(0.5) + B[i][j]) + (f.is_diag(i, j) ? T(1) : T(0));
      } else {
        // y02 = A2 (c1 A2 + c2 A)   (poly.py:209 / :221)
        const double* c = (m == 8) ? kT8 : kT15;
        Tile R, y02, L, P;
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) R[i][j] = (T)c[0] * A2[i][j] + (T)c[1] * B[i][j];
        f.product(A2, R, y02);
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            L[i][j] = (y02[i][j] + (T)c[2] * A2[i][j]) + (T)c[3] * B[i][j];
            R[i][j] = y02[i][j] + (T)c[4] * A2[i][j];
          }
        f.product(L, R, P);
        if (m == 8) {  // poly.py:211
#pragma unroll
          for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j)
              Xt[i][j] = (((P[i][j] + (T)c[5] * y02[i][j]) + A2[i][j] * T(0.5)) + B[i][j]) +
                         (f.is_diag(i, j) ? T(1) : T(0));
        } else {  // poly.py:222-229
          Tile y12;
#pragma unroll
          for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              y12[i][j] = (P[i][j] + (T)c[5] * y02[i][j]) + (T)c[6] * A2[i][j];
              L[i][j] = (y12[i][j] + (T)c[7] * A2[i][j]) + (T)c[8] * B[i][j];
              R[i][j] = (y12[i][j] + (T)c[9] * y02[i][j]) + (T)c[10] * B[i][j];
            }
          f.product(L, R, P);
#pragma unroll
          for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j)
              Xt[i][j] = ((((P[i][j] + (T)c[11] * y12[i][j]) + (T)c[12] * y02[i][j]) + (T)c[13] * A2[i][j]) +
                          (T)c[14] * B[i][j]) +
                         (f.is_diag(i, j) ? (T)c[15] : T(0));
        }
      }
    } else {
      // Paterson-Stockmeyer (poly.py:149-182) on B with cached A^2..A^4.
      const T sc3 = (T)ldexp(1.0, -3 * s);
      const T sc4 = (T)ldexp(1.0, -4 * s);
      Tile A3, A4;
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          A3[i][j] = a3[i][j] * sc3;
          A4[i][j] = a4[i][j] * sc4;
        }
      const int jj = ps_j_of(m), kk = ps_k_of(m);
      auto block = [&](int lo, int hi, Tile& acc) {
        const T c0 = (T)kInvFact[lo];
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = f.is_diag(i, j) ? c0 : T(0);
        const int cnt = hi - lo;
        if (cnt >= 1) {
          const T ct = (T)kInvFact[lo + 1];
#pragma unroll
          for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = acc[i][j] + ct * B[i][j];
        }
        if (cnt >= 2) {
          const T ct = (T)kInvFact[lo + 2];
#pragma unroll
          for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = acc[i][j] + ct * A2[i][j];
        }
        if (cnt >= 3) {
          const T ct = (T)kInvFact[lo + 3];
#pragma unroll
          for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = acc[i][j] + ct * A3[i][j];
        }
        if (cnt >= 4) {
          const T ct = (T)kInvFact[lo + 4];
#pragma unroll
          for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = acc[i][j] + ct * A4[i][j];
        }
      };
      block((kk - 1) * jj, m, Xt);
      if (kk >= 2) {
        // stage A^j once as the right operand of every Horner product
        if (jj == 2) f.store(f.buf1, A2);
        else if (jj == 3) f.store(f.buf1, A3);
        else f.store(f.buf1, A4);
        for (int r = kk - 2; r >= 0; --r) {
          Tile P, blk;
          f.store(f.buf0, Xt);
          f.sync();
          f.mm(f.buf0, f.buf1, P);
          f.sync();
          block(r * jj, r * jj + jj - 1, blk);
#pragma unroll
          for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) Xt[i][j] = P[i][j] + blk[i][j];
        }
      }
    }

    // ---- squaring phase (engine.py:80-87) ----------------------------
    for (int q = 0; q < s; ++q) {
      Tile Y;
      f.square(Xt, Y);
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) Xt[i][j] = Y[i][j];
    }

#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) bad |= !is_finite_t(Xt[i][j]);
    bad = f.any_group(bad);
    f.save(X + idx * nn, n, vec, Xt);
    if (f.t == 0) {
      if (po.m) po.m[idx] = (int8_t)m;
      if (po.s) po.s[idx] = (int8_t)s;
      if (po.e1) po.e1[idx] = p.e1;
      if (po.e2) po.e2[idx] = p.e2;
      if (po.norms) {
        po.norms[2 * idx] = nrm[0];
        po.norms[2 * idx + 1] = nrm[1];
      }
      if (po.mults) po.mults[idx] = budget(m, SCHEME) + s;
      if (po.nonfinite) po.nonfinite[idx] = (uint8_t)(bad || !(nrm[0] <= INFINITY));
    }
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) w[i][j] = nxt[i][j];
  }
}

}  // namespace expmb
