// lowrank.cuh -- batched low-rank exponential, SURVEY §8(f) rank 2.
//
// Reference: expm_lowrank (/root/reference/pkg/src/expmkit/engine.py:198-257)
// with LowRankPair (engine.py:159-191): for W = A1 A2 (A1 n x t, A2 t x n,
// t <= n) it returns e^W = I + A1 psi(V) A2 with V = A2 A1 (t x t) and
// psi(x) = sum_{i<=m} x^i/(i+1)! (poly.py:62-66) evaluated by
// Paterson-Stockmeyer (poly.py:149-182), unscaled, at the smallest order on
// LOWRANK_ORDERS (engine.py:195) whose two-term remainder bound meets eps.
//
// One CTA per matrix (grid-strided), everything of the t x t problem in
// shared memory:
//   phase 1  V = A2 A1, streaming k in 64-wide chunks (A2 rows and the
//            contiguous A1 row block are both coalesced reads), input
//            finiteness on the fly;
//   phase 2  ||V||_1, V^2 only if rung m=1 fails (engine.py:226-230), the
//            ladder (select_lowrank, host/device shared), PS powers and Horner
//            stages as t x t shared-memory products;
//   phase 3  out = I + A1 (psi A2), 64-column chunks of Y = psi A2 kept in
//            shared memory while 64-row tiles of A1 stream past: every output
//            element is written exactly once (n^2 per matrix is the HBM
//            floor of this op).
// t <= 32 (TP = 8/16/32 padded with zeros, which leaves V's powers and norms
// unchanged).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "select.cuh"
#include "lowrank_tables.h"

namespace expmb {

// flags[] bits (include/expmb.h)
constexpr uint8_t kLrBadInput = 1;   // non-finite factor entry (LowRankPair check, engine.py:179-180)
constexpr uint8_t kLrNonFinite = 2;  // V, a power, psi or the result not finite (matrix.py:95-102)
constexpr uint8_t kLrNoOrder = 4;    // LowRankOrderError (engine.py:236-240)

EXPMB_HD int lr_order(int i) {
  return i == 0 ? 1 : i == 1 ? 2 : i == 2 ? 4 : i == 3 ? 8 : i == 4 ? 15 : i == 5 ? 16 : i == 6 ? 20
         : i == 7 ? 25 : 30;
}

// engine.py:263-265: (q // 2) * lw2 + (q % 2) * lw1
EXPMB_HD double lr_power_bound_log(int q, double lw1, double lw2) {
  return rn_add(rn_mul((double)(q / 2), lw2), (q % 2) ? lw1 : 0.0);
}

// The ladder of engine.py:224-244 on ||V||_1 (and ||V^2||_1 once have_v2).
// Returns 0 with the plan written, 1 when ||V^2||_1 is needed first, -1 when
// no order qualifies (LowRankOrderError).
// (out of line on the device: one copy of the double-precision ladder)
#if defined(__CUDACC__)
__host__ __device__ __noinline__
#else
inline
#endif
int select_lowrank(double nv, double nv2, int have_v2, double log_eps, int* m, double* e1, double* e2) {
  if (nv == 0.0) {
    *m = 0;
    *e1 = 0.0;
    *e2 = 0.0;
    return 0;
  }
  const double lw1 = log2_or_ninf(nv);
  const double lw2 = have_v2 ? log2_or_ninf(nv2) : 0.0;
  for (int i = 0; i < 9; ++i) {
    const int mi = lr_order(i);
    double l1, l2;
    if (mi == 1) {
      l1 = rn_sub(rn_mul(2.0, lw1), lr_log2_fact(3));
      l2 = rn_sub(rn_mul(3.0, lw1), lr_log2_fact(4));
    } else {
      if (!have_v2) return 1;
      l1 = rn_sub(lr_power_bound_log(mi + 1, lw1, lw2), lr_log2_fact(mi + 2));
      l2 = rn_sub(lr_power_bound_log(mi + 2, lw1, lw2), lr_log2_fact(mi + 3));
    }
    // logaddexp2(l1, l2) lies in [max, max + 1]: only a rung whose bracket
    // straddles log_eps needs the transcendental (the decision is unchanged)
    const double mx = l1 > l2 ? l1 : l2;
    bool pass;
    if (mx > log_eps) pass = false;
    else if (rn_add(mx, 1.0 + 0x1p-30) < log_eps) pass = true;
    else pass = logaddexp2(l1, l2) <= log_eps;
    if (pass) {
      *m = mi;
      *e1 = exp2(l1);
      *e2 = exp2(l2);
      return 0;
    }
  }
  return -1;
}

// t x t products charged to the ledger: V^2 (selection), V^3..V^j, k-1 Horner stages.
EXPMB_HD int lr_mults(int m) {
  if (m < 2) return 0;
  const int j = ps_j_of(m);
  const int k = (m + j - 1) / j;
  return 1 + (j - 2) + (k - 1);
}

struct LrOut {
  int8_t* m;
  double* e1;
  double* e2;
  double* norms;
  int32_t* mults;
  uint8_t* flags;
};

template <typename T, int TP>
struct Lr {
  static constexpr int NT = 256;
  static constexpr int NC = 64;       // column / row / k chunk of the n-sized dimensions
  // fp64: strides = 8 banks mod 32 so the DMMA fragment walks of phase 3 are
  // conflict-free; fp32: odd strides for the FMA walks
  static constexpr int LDP = sizeof(T) == 8 ? TP + 4 : TP + 1;  // t x t tiles and the A1 row tile
  static constexpr int LDC = sizeof(T) == 8 ? NC + 4 : NC + 1;  // A2 / Y chunks
  static constexpr int kSlot = TP * LDP;
  // slot 0 = psi, 1..6 = V^p, 7 = scratch.  The factor chunks SA / SB and
  // the Y chunk SY alias slots 2.. : phase 1 is done with them before V^2 is
  // formed, and phase 3 needs only slot 0 (psi) -- halving the footprint
  // for t = 32 buys a second resident CTA per SM
  static constexpr int kSA = 2 * kSlot;
  static constexpr int kSB = kSA + TP * LDC;
  static constexpr int kSY = kSB + NC * LDP;
  static constexpr int kEnd = (kSY + TP * LDC) > 8 * kSlot ? (kSY + TP * LDC) : 8 * kSlot;
  static constexpr size_t kSmem = ((kEnd * sizeof(T) + 15) / 16) * 16 + 16 * sizeof(double);
};

__device__ __forceinline__ double lr_nanmax(double a, double b) { return (a != a || a > b) ? a : b; }

template <typename T>
__device__ __forceinline__ bool lr_finite(T v) {
  return isfinite(v);
}

// Norms + ladder on warp 0, plan broadcast through `scal` (one barrier).
// V2 == nullptr: first call (||V||_1 only).  Returns select_lowrank's code,
// or 2 when a norm is not finite (NonFiniteError in the reference).
template <typename T, int TP>
__device__ int lr_select_warp0(const T* V, const T* V2, double log_eps, double* scal, double* nv, double* nv2,
                               int* m, double* e1, double* e2) {
  using L = Lr<T, TP>;
  if (threadIdx.x < 32) {
    const T* S = V2 ? V2 : V;
    double c = 0.0;
    if (threadIdx.x < TP)
      for (int r = 0; r < TP; ++r) c += fabs((double)S[r * L::LDP + threadIdx.x]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c = lr_nanmax(c, __shfl_xor_sync(0xffffffffu, c, o));
    const double a = V2 ? scal[1] : c;
    const double b = V2 ? c : NAN;
    int mm = 0, rc;
    double x1 = NAN, x2 = NAN;
    if (!isfinite(c)) rc = 2;
    else rc = select_lowrank(a, V2 ? b : 0.0, V2 ? 1 : 0, log_eps, &mm, &x1, &x2);
    __syncwarp();
    if (threadIdx.x == 0) {
      scal[1] = a;
      scal[2] = b;
      scal[3] = x1;
      scal[4] = x2;
      scal[5] = (double)mm;
      scal[6] = (double)rc;
    }
  }
  __syncthreads();
  *nv = scal[1];
  *nv2 = scal[2];
  *e1 = scal[3];
  *e2 = scal[4];
  *m = (int)scal[5];
  const int rc = (int)scal[6];
  __syncthreads();
  return rc;
}

// fp64 DMMA (m8n8k4) accumulate: (d0, d1) += a b for one lane's fragments
__device__ __forceinline__ void lr_dmma_acc(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// C = A B for TP x TP shared tiles.
template <typename T, int TP>
__device__ void lr_mm(T* C, const T* A, const T* B) {
  using L = Lr<T, TP>;
  if constexpr (sizeof(T) == 8) {
    // fp64: 8x8 output tiles on DMMA (m8n8k4), warp w takes tiles w, w + 8, ...
    const int w = threadIdx.x >> 5, g = (threadIdx.x >> 2) & 7, q = threadIdx.x & 3;
    constexpr int NTL = TP / 8;
    for (int tile = w; tile < NTL * NTL; tile += L::NT / 32) {
      const int R = tile / NTL, Cc = tile % NTL;
      double d0 = 0.0, d1 = 0.0;
#pragma unroll
      for (int s4 = 0; s4 < TP / 4; ++s4)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(d0), "+d"(d1)
                     : "d"(A[(8 * R + g) * L::LDP + 4 * s4 + q]), "d"(B[(4 * s4 + q) * L::LDP + 8 * Cc + g]));
      C[(8 * R + g) * L::LDP + 8 * Cc + 2 * q] = d0;
      C[(8 * R + g) * L::LDP + 8 * Cc + 2 * q + 1] = d1;
    }
    return;
  }
  for (int e = threadIdx.x; e < TP * TP; e += L::NT) {
    const int r = e / TP, c = e % TP;
    T acc = 0;
#pragma unroll 8
    for (int k = 0; k < TP; ++k) acc = fma(A[r * L::LDP + k], B[k * L::LDP + c], acc);
    C[r * L::LDP + c] = acc;
  }
}

template <typename T, int TP>
__device__ void lr_fill_nan(T* x, size_t nn) {
  for (size_t i = threadIdx.x; i < nn; i += Lr<T, TP>::NT) x[i] = (T)NAN;
}

#ifndef LR_T16_MINB
#define LR_T16_MINB 4
#endif
#ifndef LR_T32_MINB
#define LR_T32_MINB 3
#endif

// TI: the factor / result type (T = double, TI = float: fp32 I/O computed
// in binary64 on the DMMA path, rounded once on the store)
template <typename T, int TP, typename TI = T>
__global__ void __launch_bounds__(256, (TP <= 16 ? LR_T16_MINB : LR_T32_MINB)) expm_lowrank_kernel(const TI* __restrict__ A1, const TI* __restrict__ A2,
                                                           TI* __restrict__ X, int64_t batch, int n, int t,
                                                           double log_eps, LrOut po) {
  using L = Lr<T, TP>;
  extern __shared__ __align__(16) unsigned char lr_smem[];
  T* P = reinterpret_cast<T*>(lr_smem);
  T* SA = P + L::kSA;
  T* SB = P + L::kSB;
  T* SY = P + L::kSY;
  double* scal = reinterpret_cast<double*>(lr_smem + L::kSmem - 16 * sizeof(double));
  const int tid = threadIdx.x;
  constexpr int NE = TP * TP;
  constexpr int G = NE >= 256 ? 1 : 256 / NE;  // k-groups per V element
  constexpr int R = NE >= 256 ? NE / 256 : 1;  // V elements per thread
  const size_t nn = (size_t)n * n;

  for (int64_t mat = blockIdx.x; mat < batch; mat += gridDim.x) {
    const TI* a1 = A1 + (size_t)mat * n * t;
    const TI* a2 = A2 + (size_t)mat * t * n;
    TI* x = X + (size_t)mat * nn;
    T* V = P + L::kSlot;

    // ---- phase 1: V = A2 A1 ----------------------------------------------
    T acc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = 0;
    const int g = NE >= 256 ? 0 : tid / NE;
    constexpr int NTL = TP / 8;
    const int dw = tid >> 5, dg = (tid >> 2) & 7, dq = tid & 3;
    double dv[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
    bool bad = false;
    for (int k0 = 0; k0 < n; k0 += L::NC) {
      const int kc = min(L::NC, n - k0);
      for (int idx = tid; idx < TP * L::NC; idx += L::NT) {
        const int a = idx / L::NC, kk = idx % L::NC;
        T v = 0;
        if (a < t && kk < kc) {
          v = (T)a2[(size_t)a * n + k0 + kk];
          bad |= !lr_finite(v);
        }
        SA[a * L::LDC + kk] = v;
      }
      for (int idx = tid; idx < L::NC * TP; idx += L::NT) {
        const int kk = idx / TP, b = idx % TP;
        T v = 0;
        if (b < t && kk < kc) {
          v = (T)a1[(size_t)(k0 + kk) * t + b];
          bad |= !lr_finite(v);
        }
        SB[kk * L::LDP + b] = v;
      }
      __syncthreads();
      if constexpr (sizeof(T) == 8) {
        // fp64: 8x8 tiles of V on DMMA, warp w owns tiles w and w + 8
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int tile = dw + 8 * i;
          if (tile < NTL * NTL) {
            const int TR = tile / NTL, TC = tile % NTL;
#pragma unroll 4
            for (int s4 = 0; s4 < L::NC / 4; ++s4)
              lr_dmma_acc(dv[i][0], dv[i][1], SA[(8 * TR + dg) * L::LDC + 4 * s4 + dq],
                          SB[(4 * s4 + dq) * L::LDP + 8 * TC + dg]);
          }
        }
      } else {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int e = NE >= 256 ? tid + 256 * r : tid % NE;
        const int a = e / TP, b = e % TP;
        T s = acc[r];
        for (int kk = g; kk < L::NC; kk += G) s = fma(SA[a * L::LDC + kk], SB[kk * L::LDP + b], s);
        acc[r] = s;
      }
      }
      __syncthreads();
    }
    if constexpr (sizeof(T) == 8) {
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int tile = dw + 8 * i;
        if (tile < NTL * NTL) {
          const int TR = tile / NTL, TC = tile % NTL;
          V[(8 * TR + dg) * L::LDP + 8 * TC + 2 * dq] = dv[i][0];
          V[(8 * TR + dg) * L::LDP + 8 * TC + 2 * dq + 1] = dv[i][1];
        }
      }
    } else if (G > 1) {
      SY[tid] = acc[0];
      __syncthreads();
      if (tid < NE) {
        T s = 0;
        for (int gg = 0; gg < G; ++gg) s += SY[gg * NE + tid];
        V[(tid / TP) * L::LDP + tid % TP] = s;
      }
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int e = tid + 256 * r;
        V[(e / TP) * L::LDP + e % TP] = acc[r];
      }
    }
    const int bad_in = __syncthreads_or(bad);

    int m = 0;
    double e1 = NAN, e2 = NAN, nv = NAN, nv2 = NAN;
    uint8_t flags = 0;
    if (bad_in) {
      flags = kLrBadInput;
    } else {
      // ---- phase 2: order selection and psi(V) ------------------------------
      // warp 0 runs the ladder (warp-uniform) and broadcasts the plan
      int rc = lr_select_warp0<T, TP>(V, nullptr, log_eps, scal, &nv, &nv2, &m, &e1, &e2);
      if (rc == 1) {
        lr_mm<T, TP>(P + 2 * L::kSlot, V, V);
        __syncthreads();
        rc = lr_select_warp0<T, TP>(V, P + 2 * L::kSlot, log_eps, scal, &nv, &nv2, &m, &e1, &e2);
      }
      if (rc == 2) {
        flags = kLrNonFinite;
      } else if (rc < 0) {
        flags = kLrNoOrder;
        e1 = e2 = NAN;
      }
    }
    if (flags) {
      lr_fill_nan<TI, TP>(x, nn);
    } else {
      T* Q = P;
      T* S7 = P + 7 * L::kSlot;
      if (m == 0) {
        for (int e = tid; e < NE; e += L::NT) Q[(e / TP) * L::LDP + e % TP] = (e / TP == e % TP) ? T(1) : T(0);
      } else {
        const int j = ps_j_of(m);
        const int k = (m + j - 1) / j;
        for (int p = 3; p <= j; ++p) {
          lr_mm<T, TP>(P + p * L::kSlot, P + (p - 1) * L::kSlot, V);
          __syncthreads();
        }
        // q = block((k-1)j, m); then q = q V^j + block(rj, rj+j-1), r = k-2..0
        // (poly.py:171-182; block(lo,hi) = c_lo I + sum_t c_{lo+t} V^t)
        for (int r = k - 1; r >= 0; --r) {
          const int lo = r * j, hi = (r == k - 1) ? m : r * j + j - 1;
          if (r < k - 1) {
            lr_mm<T, TP>(S7, Q, P + j * L::kSlot);
            __syncthreads();
          }
          // coefficients c_{lo+1..hi+1} hoisted (hi - lo <= j <= 6), the
          // element loop unrolled over a thread's NE / NT entries
          T cf[7];
#pragma unroll
          for (int tt = 0; tt < 7; ++tt) cf[tt] = tt <= hi - lo ? (T)lr_inv_fact(lo + tt + 1) : T(0);
          constexpr int EPT = (NE + L::NT - 1) / L::NT;
#pragma unroll
          for (int u = 0; u < EPT; ++u) {
            const int e = tid + u * L::NT;
            if (NE % L::NT == 0 || e < NE) {
              const int er = e / TP, ec = e % TP, off = er * L::LDP + ec;
              T q = er == ec ? cf[0] : T(0);
#pragma unroll
              for (int tt = 1; tt < 7; ++tt)
                if (tt <= hi - lo) q = fma(cf[tt], P[tt * L::kSlot + off], q);
              Q[off] = (r < k - 1) ? S7[off] + q : q;
            }
          }
          __syncthreads();
        }
      }
      __syncthreads();
      bool bq = false;
      for (int e = tid; e < NE; e += L::NT) bq |= !lr_finite(Q[(e / TP) * L::LDP + e % TP]);
      if (__syncthreads_or(bq)) {
        flags = kLrNonFinite;
        lr_fill_nan<TI, TP>(x, nn);
      } else {
        // ---- phase 3: out = I + A1 (psi A2) ---------------------------------
        const int tx = tid % 16, ty = tid / 16;
        bool bo = false;
        for (int c0 = 0; c0 < n; c0 += L::NC) {
          const int cc = min(L::NC, n - c0);
          for (int idx = tid; idx < TP * L::NC; idx += L::NT) {
            const int a = idx / L::NC, jj = idx % L::NC;
            SA[a * L::LDC + jj] = (a < t && jj < cc) ? (T)a2[(size_t)a * n + c0 + jj] : T(0);
          }
          __syncthreads();
          if constexpr (sizeof(T) == 8) {
            // fp64: Y = psi A2 chunk on DMMA, (TP/8) x 8 tiles over 8 warps
            for (int tile = dw; tile < NTL * 8; tile += 8) {
              const int TR = tile >> 3, TC = tile & 7;
              double y0 = 0.0, y1 = 0.0;
#pragma unroll
              for (int s4 = 0; s4 < TP / 4; ++s4)
                lr_dmma_acc(y0, y1, Q[(8 * TR + dg) * L::LDP + 4 * s4 + dq], SA[(4 * s4 + dq) * L::LDC + 8 * TC + dg]);
              SY[(8 * TR + dg) * L::LDC + 8 * TC + 2 * dq] = y0;
              SY[(8 * TR + dg) * L::LDC + 8 * TC + 2 * dq + 1] = y1;
            }
          } else {
          for (int e = tid; e < TP * L::NC; e += L::NT) {
            const int b = e / L::NC, jj = e % L::NC;
            T s = 0;
#pragma unroll 8
            for (int a = 0; a < TP; ++a) s = fma(Q[b * L::LDP + a], SA[a * L::LDC + jj], s);
            SY[b * L::LDC + jj] = s;
          }
          }
          __syncthreads();
          for (int r0 = 0; r0 < n; r0 += L::NC) {
            const int rcn = min(L::NC, n - r0);
            for (int idx = tid; idx < L::NC * TP; idx += L::NT) {
              const int rr = idx / TP, b = idx % TP;
              SB[rr * L::LDP + b] = (rr < rcn && b < t) ? (T)a1[(size_t)(r0 + rr) * t + b] : T(0);
            }
            __syncthreads();
            if constexpr (sizeof(T) == 8) {
              // fp64: the 64x64 tile on DMMA -- warp w owns rows 8w..8w+7,
              // all eight 8-column tiles; k = TP in steps of 4
              const int w = tid / 32, g = (tid % 32) / 4, q = tid % 4;
              double d[8][2];
#pragma unroll
              for (int C = 0; C < 8; ++C) d[C][0] = d[C][1] = 0.0;
#pragma unroll
              for (int s4 = 0; s4 < TP / 4; ++s4) {
                const double av = SB[(8 * w + g) * L::LDP + 4 * s4 + q];
#pragma unroll
                for (int C = 0; C < 8; ++C) {
                  const double bv = SY[(4 * s4 + q) * L::LDC + 8 * C + g];
                  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                               : "+d"(d[C][0]), "+d"(d[C][1])
                               : "d"(av), "d"(bv));
                }
              }
              const int row = r0 + 8 * w + g;
              if (row < n) {
#pragma unroll
                for (int C = 0; C < 8; ++C) {
                  const int col = c0 + 8 * C + 2 * q;
                  const double v0 = (row == col) ? d[C][0] + 1.0 : d[C][0];
                  const double v1 = (row == col + 1) ? d[C][1] + 1.0 : d[C][1];
                  TI* xp = x + (size_t)row * n + col;
                  const TI o0 = (TI)v0, o1 = (TI)v1;
                  if (sizeof(TI) == 8 && col + 1 < n && (n % 2) == 0 && (((uintptr_t)x) & 15) == 0) {
                    // 16-byte aligned pair
                    *reinterpret_cast<double2*>(xp) = make_double2(v0, v1);
                    bo |= !isfinite(v0) || !isfinite(v1);
                  } else if (col < n) {
                    xp[0] = o0;
                    bo |= !isfinite(o0);
                    if (col + 1 < n) {
                      xp[1] = o1;
                      bo |= !isfinite(o1);
                    }
                  }
                }
              }
            } else {
            T o[4][4];
#pragma unroll
            for (int ii = 0; ii < 4; ++ii)
#pragma unroll
              for (int jj = 0; jj < 4; ++jj) o[ii][jj] = 0;
#pragma unroll 4
            for (int b = 0; b < TP; ++b) {
              T ya[4], xa[4];
#pragma unroll
              for (int jj = 0; jj < 4; ++jj) ya[jj] = SY[b * L::LDC + tx + 16 * jj];
#pragma unroll
              for (int ii = 0; ii < 4; ++ii) xa[ii] = SB[(ty + 16 * ii) * L::LDP + b];
#pragma unroll
              for (int ii = 0; ii < 4; ++ii)
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) o[ii][jj] = fma(xa[ii], ya[jj], o[ii][jj]);
            }
#pragma unroll
            for (int ii = 0; ii < 4; ++ii) {
              const int row = r0 + ty + 16 * ii;
              if (row >= n) continue;
#pragma unroll
              for (int jj = 0; jj < 4; ++jj) {
                const int col = c0 + tx + 16 * jj;
                if (col < n) {
                  const T v = (row == col) ? o[ii][jj] + T(1) : o[ii][jj];
                  bo |= !lr_finite(v);
                  x[(size_t)row * n + col] = v;
                }
              }
            }
            }  // fp32 FMA tile
            __syncthreads();
          }
        }
        if (__syncthreads_or(bo)) {  // overflow in the assembly: a flagged X is NaN (include/expmb.h)
          flags = kLrNonFinite;
          lr_fill_nan<TI, TP>(x, nn);
        }
      }
    }
    if (tid == 0) {
      if (po.m) po.m[mat] = (int8_t)m;
      if (po.e1) po.e1[mat] = e1;
      if (po.e2) po.e2[mat] = e2;
      if (po.norms) {
        po.norms[2 * mat] = nv;
        po.norms[2 * mat + 1] = nv2;
      }
      if (po.mults) po.mults[mat] = flags ? 0 : lr_mults(m);
      if (po.flags) po.flags[mat] = flags;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Warp-per-matrix variant for the flow-layer shape t <= 8, n <= 64 (the
// reference generator's t = n/8 at n = 64).  No block barriers: each warp
// owns one matrix at a time in its private shared-memory slice (A1 rows,
// A2 rows, eight 8x8 tiles), zero-padded once per launch (padding is never
// written, so V's powers, norms and the assembly see exact zeros).
//   V = A2 A1      lane (a, b0..b0+1), k over n
//   psi(V)         t x t products, lane owns the same two entries
//   Y = psi A2     lane owns columns c0 = 2 lane, c0 + 1, kept in registers
//   out = I + A1 Y one row per iteration: four broadcast 16-byte loads of the
//                  A1 row, 16 FMAs, one coalesced 16-byte store per lane (the
//                  warp writes the whole 512-byte row)
// ---------------------------------------------------------------------------

#ifndef LRW_PAIRS
#define LRW_PAIRS 1  // FULL assembly: row pairs with the diagonal folded into the init
#endif

template <typename T>
struct LrW {
  static constexpr int WARPS = 4;
  static constexpr int NT = 32 * WARPS;
  static constexpr int LD1 = 8;   // A1 rows: 8 entries, 16-byte aligned pairs
  static constexpr int LD2 = 66;  // A2 rows: conflict-free column walks, 16-byte aligned
  static constexpr int LDP = 9;   // 8x8 tiles
  static constexpr int kSlot = 8 * LDP;
  static constexpr int kA2 = 64 * LD1;
  static constexpr int kP = kA2 + 8 * LD2;
  static constexpr int kStride = ((kP + 8 * kSlot) + 3) / 4 * 4;
  static constexpr size_t kSmem = (size_t)WARPS * kStride * sizeof(T);
};

template <typename T>
struct Pair2 {
  T x, y;
};
template <typename T>
__device__ __forceinline__ Pair2<T> ld_pair(const T* p) {
  if constexpr (sizeof(T) == 8) {
    const double2 v = *reinterpret_cast<const double2*>(p);
    return {v.x, v.y};
  } else {
    const float2 v = *reinterpret_cast<const float2*>(p);
    return {v.x, v.y};
  }
}
template <typename T>
__device__ __forceinline__ void st_pair(T* p, T a, T b) {
  if constexpr (sizeof(T) == 8) {
    *reinterpret_cast<double2*>(p) = make_double2(a, b);
  } else {
    *reinterpret_cast<float2*>(p) = make_float2(a, b);
  }
}

// ||tile||_1 over the warp (lanes 0..7 sum a column; NaN-propagating max).
template <typename T>
__device__ __forceinline__ double lrw_norm1(const T* S, int lane) {
  double c = 0.0;
  if (lane < 8)
    for (int r = 0; r < 8; ++r) c += fabs((double)S[r * LrW<T>::LDP + lane]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c = lr_nanmax(c, __shfl_xor_sync(0xffffffffu, c, o));
  return c;
}

// This lane's two entries (a, b0), (a, b0 + 1) of A B for 8x8 tiles.
template <typename T>
__device__ __forceinline__ void lrw_mm2(const T* A, const T* B, int a, int b0, T& o0, T& o1) {
  constexpr int LDP = LrW<T>::LDP;
  T s0 = 0, s1 = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const T av = A[a * LDP + k];
    s0 = fma(av, B[k * LDP + b0], s0);
    s1 = fma(av, B[k * LDP + b0 + 1], s1);
  }
  o0 = s0;
  o1 = s1;
}

// FULL: n == 64 and t == 8 exactly (vector loads/stores, no bounds checks).
template <typename T, bool FULL>
__global__ void __launch_bounds__(128) expm_lowrank_warp_kernel(const T* __restrict__ A1,
                                                                const T* __restrict__ A2, T* __restrict__ X,
                                                                int64_t batch, int n_, int t_, double log_eps,
                                                                LrOut po) {
  const int n = FULL ? 64 : n_;
  const int t = FULL ? 8 : t_;
  using L = LrW<T>;
  extern __shared__ __align__(16) unsigned char lrw_smem[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  T* base = reinterpret_cast<T*>(lrw_smem) + w * L::kStride;
  T* sA1 = base;
  T* sA2 = base + L::kA2;
  T* P = base + L::kP;  // slot 0 = psi, 1..6 = V^p, 7 = scratch
  for (int i = lane; i < L::kStride; i += 32) base[i] = T(0);
  __syncwarp();
  const int a_r = lane >> 2, b0 = (lane & 3) * 2;  // the t x t entries this lane owns
  const int c0 = 2 * lane;                         // the output columns this lane owns
  const bool vec_out = (n % 2) == 0;
  const int64_t nw = (int64_t)gridDim.x * L::WARPS;
  for (int64_t mat = (int64_t)blockIdx.x * L::WARPS + w; mat < batch; mat += nw) {
    const T* a1 = A1 + (size_t)mat * n * t;
    const T* a2 = A2 + (size_t)mat * t * n;
    T* x = X + (size_t)mat * n * n;
    // all loads of the factors issued back to back, then staged; z turns
    // NaN if any entry is NaN/Inf (x * 0 = NaN exactly for those)
    T z = 0;
    double amax1 = 0.0;  // FULL: max |A1| (overflow bound of the assembly)
    if constexpr (FULL) {
      Pair2<T> ra[8], rb[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) ra[q] = ld_pair(a1 + 2 * (lane + 32 * q));
#pragma unroll
      for (int q = 0; q < 8; ++q) rb[q] = ld_pair(a2 + q * 64 + 2 * lane);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int p = lane + 32 * q;
        st_pair(sA1 + (p >> 2) * L::LD1 + 2 * (p & 3), ra[q].x, ra[q].y);
        st_pair(sA2 + q * L::LD2 + 2 * lane, rb[q].x, rb[q].y);
        z = fma(ra[q].x, T(0), z);
        z = fma(ra[q].y, T(0), z);
        z = fma(rb[q].x, T(0), z);
        z = fma(rb[q].y, T(0), z);
        amax1 = fmax(amax1, fmax(fabs((double)ra[q].x), fabs((double)ra[q].y)));
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) amax1 = fmax(amax1, __shfl_xor_sync(0xffffffffu, amax1, o));
    } else {
      T ra[16], rb[16];
      const int b = lane & 7;
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int r = (lane >> 3) + 4 * q;
        ra[q] = (b < t && r < n) ? a1[(size_t)r * t + b] : T(0);
      }
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int a = q >> 1, c = lane + 32 * (q & 1);
        rb[q] = (a < t && c < n) ? a2[(size_t)a * n + c] : T(0);
      }
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        sA1[((lane >> 3) + 4 * q) * L::LD1 + b] = ra[q];
        sA2[(q >> 1) * L::LD2 + lane + 32 * (q & 1)] = rb[q];
        z = fma(ra[q], T(0), z);
        z = fma(rb[q], T(0), z);
      }
    }
    const bool bad = z != T(0);
    __syncwarp();
    int m = 0, rc = 0;
    bool wrote = false;
    double e1 = NAN, e2 = NAN, nv = NAN, nv2 = NAN;
    uint8_t flags = __any_sync(0xffffffffu, bad) ? kLrBadInput : 0;
    if (!flags) {
      // V = A2 A1
      T v0 = 0, v1 = 0;
#pragma unroll 4
      for (int k = 0; k < n; ++k) {
        const T s = sA2[a_r * L::LD2 + k];
        const Pair2<T> q = ld_pair(sA1 + k * L::LD1 + b0);
        v0 = fma(s, q.x, v0);
        v1 = fma(s, q.y, v1);
      }
      T* V = P + L::kSlot;
      V[a_r * L::LDP + b0] = v0;
      V[a_r * L::LDP + b0 + 1] = v1;
      __syncwarp();
      nv = lrw_norm1(V, lane);
      if (!isfinite(nv)) {
        rc = 2;
      } else {
        rc = select_lowrank(nv, 0.0, 0, log_eps, &m, &e1, &e2);
        if (rc == 1) {
          T o0, o1;
          lrw_mm2(V, V, a_r, b0, o0, o1);
          P[2 * L::kSlot + a_r * L::LDP + b0] = o0;
          P[2 * L::kSlot + a_r * L::LDP + b0 + 1] = o1;
          __syncwarp();
          nv2 = lrw_norm1(P + 2 * L::kSlot, lane);
          rc = isfinite(nv2) ? select_lowrank(nv, nv2, 1, log_eps, &m, &e1, &e2) : 2;
        }
      }
      if (rc == 2) flags = kLrNonFinite;
      if (rc < 0) {
        flags = kLrNoOrder;
        e1 = e2 = NAN;
      }
    }
    if (!flags) {
      // psi(V) by Paterson-Stockmeyer (poly.py:149-182), this lane's two entries
      T* Q = P;
      const int off = a_r * L::LDP + b0;
      T q0, q1;
      if (m == 0) {
        q0 = (a_r == b0) ? T(1) : T(0);
        q1 = (a_r == b0 + 1) ? T(1) : T(0);
      } else {
        const int j = ps_j_of(m);
        const int k = (m + j - 1) / j;
        for (int p = 3; p <= j; ++p) {
          T o0, o1;
          lrw_mm2(P + (p - 1) * L::kSlot, P + L::kSlot, a_r, b0, o0, o1);
          P[p * L::kSlot + off] = o0;
          P[p * L::kSlot + off + 1] = o1;
          __syncwarp();
        }
        q0 = q1 = 0;
        for (int r = k - 1; r >= 0; --r) {
          const int lo = r * j, hi = (r == k - 1) ? m : r * j + j - 1;
          T s0 = 0, s1 = 0;
          if (r < k - 1) lrw_mm2(Q, P + j * L::kSlot, a_r, b0, s0, s1);
          T c0v = (a_r == b0) ? (T)lr_inv_fact(lo + 1) : T(0);
          T c1v = (a_r == b0 + 1) ? (T)lr_inv_fact(lo + 1) : T(0);
          for (int tt = 1; tt <= hi - lo; ++tt) {
            const T c = (T)lr_inv_fact(lo + tt + 1);
            c0v = fma(c, P[tt * L::kSlot + off], c0v);
            c1v = fma(c, P[tt * L::kSlot + off + 1], c1v);
          }
          q0 = (r < k - 1) ? s0 + c0v : c0v;
          q1 = (r < k - 1) ? s1 + c1v : c1v;
          __syncwarp();
          Q[off] = q0;
          Q[off + 1] = q1;
          __syncwarp();
        }
      }
      Q[off] = q0;
      Q[off + 1] = q1;
      __syncwarp();
      if (__any_sync(0xffffffffu, !isfinite(q0) || !isfinite(q1))) {
        flags = kLrNonFinite;
      } else {
        // Y = psi A2, columns c0, c0 + 1 in registers
        T y0[8], y1[8];
        Pair2<T> ac[8];
#pragma unroll
        for (int a = 0; a < 8; ++a) ac[a] = ld_pair(sA2 + a * L::LD2 + c0);
#pragma unroll
        for (int b = 0; b < 8; ++b) {
          T s0 = 0, s1 = 0;
#pragma unroll
          for (int a = 0; a < 8; ++a) {
            const T qv = Q[b * L::LDP + a];
            s0 = fma(qv, ac[a].x, s0);
            s1 = fma(qv, ac[a].y, s1);
          }
          y0[b] = s0;
          y1[b] = s1;
        }
        // out = I + A1 Y
        bool bo = false;
        T zo = 0;  // NaN iff a checked output entry is NaN/Inf
        if constexpr (FULL && LRW_PAIRS) {
          // |out| <= 1 + max|A1| * max_c sum_b |Y[b][c]|: when that is far from
          // overflow (the usual case) no entry can be NaN/Inf and the
          // per-entry check is skipped; otherwise every entry is checked
          double ys0 = 0.0, ys1 = 0.0;
#pragma unroll
          for (int b = 0; b < 8; ++b) {
            ys0 += fabs((double)y0[b]);
            ys1 += fabs((double)y1[b]);
          }
          const double bound = 1.0 + amax1 * (ys0 > ys1 ? ys0 : ys1);
          const bool safe = __all_sync(0xffffffffu, bound < (sizeof(T) == 8 ? 1e300 : 1e37));
          T* xr = x + c0;
          // row pairs (2p, 2p + 1): lane's diagonal entries are (2p, c0) and
          // (2p + 1, c0 + 1) for p == lane, folded into the accumulator init
          // the next pair's A1 rows are loaded while this pair's FMAs run
          Pair2<T> xa[4], xb[4];
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            xa[b] = ld_pair(sA1 + 2 * b);
            xb[b] = ld_pair(sA1 + L::LD1 + 2 * b);
          }
#pragma unroll 1
          for (int p = 0; p < 32; ++p) {
            const T d = (p == lane) ? T(1) : T(0);
            const T* an = sA1 + 2 * ((p + 1) & 31) * L::LD1;
            Pair2<T> na[4], nb[4];
#pragma unroll
            for (int b = 0; b < 4; ++b) {
              na[b] = ld_pair(an + 2 * b);
              nb[b] = ld_pair(an + L::LD1 + 2 * b);
            }
            T o00 = d, o01 = 0, o10 = 0, o11 = d;
#pragma unroll
            for (int b = 0; b < 4; ++b) {
              o00 = fma(xa[b].x, y0[2 * b], o00);
              o01 = fma(xa[b].x, y1[2 * b], o01);
              o10 = fma(xb[b].x, y0[2 * b], o10);
              o11 = fma(xb[b].x, y1[2 * b], o11);
              o00 = fma(xa[b].y, y0[2 * b + 1], o00);
              o01 = fma(xa[b].y, y1[2 * b + 1], o01);
              o10 = fma(xb[b].y, y0[2 * b + 1], o10);
              o11 = fma(xb[b].y, y1[2 * b + 1], o11);
            }
            st_pair(xr, o00, o01);
            st_pair(xr + 64, o10, o11);
            xr += 128;
            if (!safe) {
              zo = fma(o00, T(0), zo);
              zo = fma(o01, T(0), zo);
              zo = fma(o10, T(0), zo);
              zo = fma(o11, T(0), zo);
            }
#pragma unroll
            for (int b = 0; b < 4; ++b) {
              xa[b] = na[b];
              xb[b] = nb[b];
            }
          }
        }
        const bool act0 = c0 < n, act1 = c0 + 1 < n;
#pragma unroll 2
        for (int r = 0; r < ((FULL && LRW_PAIRS) ? 0 : n); ++r) {
          const T* ar = sA1 + r * L::LD1;
          T o0 = 0, o1 = 0;
#pragma unroll
          for (int b = 0; b < 8; b += 2) {
            const Pair2<T> xa = ld_pair(ar + b);
            o0 = fma(xa.x, y0[b], o0);
            o1 = fma(xa.x, y1[b], o1);
            o0 = fma(xa.y, y0[b + 1], o0);
            o1 = fma(xa.y, y1[b + 1], o1);
          }
          if (r == c0) o0 += T(1);
          if (r == c0 + 1) o1 += T(1);
          T* xr = x + (size_t)r * n + c0;
          if (FULL) {
            st_pair(xr, o0, o1);
            zo = fma(o0, T(0), zo);
            zo = fma(o1, T(0), zo);
          } else if (vec_out && act1) {
            st_pair(xr, o0, o1);
            bo |= !isfinite(o0) || !isfinite(o1);
          } else {
            if (act0) {
              xr[0] = o0;
              bo |= !isfinite(o0);
            }
            if (act1) {
              xr[1] = o1;
              bo |= !isfinite(o1);
            }
          }
        }
        wrote = true;
        bo |= zo != T(0);
        if (__any_sync(0xffffffffu, bo)) flags = kLrNonFinite;
      }
    }
    if (flags) {  // also after an overflowing write: a flagged X is NaN (include/expmb.h)
      __syncwarp();
      for (size_t i = lane; i < (size_t)n * n; i += 32) x[i] = (T)NAN;
    }
    if (lane == 0) {
      if (po.m) po.m[mat] = (int8_t)m;
      if (po.e1) po.e1[mat] = e1;
      if (po.e2) po.e2[mat] = e2;
      if (po.norms) {
        po.norms[2 * mat] = nv;
        po.norms[2 * mat + 1] = nv2;
      }
      if (po.mults) po.mults[mat] = flags ? 0 : lr_mults(m);
      if (po.flags) po.flags[mat] = flags;
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// fp64 flow-layer shape n = 64, t = 8 on the FP64 tensor cores: every product
// of the path is DMMA (mma.sync.m8n8k4.f64): V = A2 A1 is 16 DMMA, each 8x8
// t x t product 2, Y = psi A2 16 and the assembly I + A1 Y 128 -- against
// ~1.3k DFMA warp-instructions per matrix on the FMA pipe, which left the
// warp kernel issue bound.  Lane (g = lane/4, q = lane%4) owns the
// accumulator entries (g, 2q), (g, 2q + 1) of every 8x8 tile, which is the
// same t x t ownership as the warp kernel above.  A1 and the t x t tiles
// use 8-wide rows with the column XOR-swizzled by bit 1 of the row so both
// the A-fragment (row g, column q) and B-fragment (row q, column g) walks
// are bank-conflict free.
// ---------------------------------------------------------------------------

struct LrD {
  static constexpr int WARPS = 4;
  static constexpr int NT = 32 * WARPS;
  static constexpr int LDY = 68;  // A2 / Y rows (8 x 64): conflict-free fragment walks
  static constexpr int kA2 = 512;
  static constexpr int kP = kA2 + 8 * LDY;
  static constexpr int kSlot = 64;
  static constexpr int kStride = kP + 7 * kSlot;  // slot 0 = psi, 1..6 = V^p
  static constexpr size_t kSmem = (size_t)WARPS * kStride * sizeof(double);
};

__device__ __forceinline__ int lr_sw8(int r, int c) { return r * 8 + (c ^ (((r >> 1) & 1) << 2)); }

__device__ __forceinline__ void lr_dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// (d0, d1) = entries (g, 2q), (g, 2q + 1) of A B for swizzled 8x8 tiles.
__device__ __forceinline__ void lr_mm8(const double* A, const double* B, int g, int q, double& d0, double& d1) {
  d0 = 0.0;
  d1 = 0.0;
  lr_dmma(d0, d1, A[lr_sw8(g, q)], B[lr_sw8(q, g)]);
  lr_dmma(d0, d1, A[lr_sw8(g, q + 4)], B[lr_sw8(q + 4, g)]);
}

__device__ __forceinline__ int hi_abs(double v) { return __double2hiint(v) & 0x7fffffff; }

// FULL: n = 64, t = 8 with 16-byte vector accesses.  Otherwise any n <= 64,
// t <= 8: the factors are zero-padded to 64 x 8 / 8 x 64 in shared memory
// (the padding stays exactly zero through V, psi(V) and Y, so every product
// is the padded one), only the ceil(n/8)^2 output tiles are computed, and
// loads / stores are scalar (no alignment requirement).
// TI = float: fp32 factors / result, computed in binary64 on the same DMMA
// path (the products are exact-er than the fp32 reference's; the result is
// rounded once on the store, and the overflow bound uses the fp32 range).
template <typename TI, bool FULL>
__global__ void __launch_bounds__(128, 3) expm_lowrank_dmma_kernel(const TI* __restrict__ A1,
                                                                const TI* __restrict__ A2,
                                                                TI* __restrict__ X, int64_t batch, int n,
                                                                int t, double log_eps, LrOut po) {
  static_assert(!FULL || sizeof(TI) == 8, "the vector-load variant is fp64 only");
  using L = LrD;
  extern __shared__ __align__(16) unsigned char lrd_smem[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int g = lane >> 2, q = lane & 3;
  double* base = reinterpret_cast<double*>(lrd_smem) + w * L::kStride;
  double* sA1 = base;
  double* sY = base + L::kA2;  // A2, then Y = psi A2
  double* P = base + L::kP;
  const int own = lr_sw8(g, 2 * q);  // this lane's entry pair in every t x t tile
  const int64_t nw = (int64_t)gridDim.x * L::WARPS;
  const int nt = FULL ? 512 : n * t, nn = FULL ? 4096 : n * n;
  const int nT = FULL ? 8 : (n + 7) >> 3;  // output tiles per dimension
  const float inv_t = 1.0f / (float)t, inv_n = 1.0f / (float)n;
  const bool vec = !FULL && (n & 7) == 0 && ((uintptr_t)X & (2 * sizeof(TI) - 1)) == 0;
  if (!FULL) {
    for (int i = lane; i < L::kP; i += 32) base[i] = 0.0;
    __syncwarp();
  }
  // the factors of matrix mat + nw are loaded into registers while matrix
  // mat is computed (16 loads in flight per lane)
  double2 ra[8], rb[8];
  auto fetch = [&](int64_t mm) {
    const TI* a1 = A1 + (size_t)mm * nt;
    const TI* a2 = A2 + (size_t)mm * nt;
    if constexpr (FULL) {
#pragma unroll
      for (int j = 0; j < 8; ++j) ra[j] = __ldcs(reinterpret_cast<const double2*>(a1 + 2 * (lane + 32 * j)));
#pragma unroll
      for (int j = 0; j < 8; ++j) rb[j] = __ldcs(reinterpret_cast<const double2*>(a2 + 64 * j + 2 * lane));
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int i0 = lane + 64 * j, i1 = i0 + 32;
        ra[j].x = i0 < nt ? (double)__ldcs(a1 + i0) : 0.0;
        ra[j].y = i1 < nt ? (double)__ldcs(a1 + i1) : 0.0;
        rb[j].x = i0 < nt ? (double)__ldcs(a2 + i0) : 0.0;
        rb[j].y = i1 < nt ? (double)__ldcs(a2 + i1) : 0.0;
      }
    }
  };
  int64_t mat = (int64_t)blockIdx.x * L::WARPS + w;
  if (mat < batch) fetch(mat);
  for (; mat < batch; mat += nw) {
    TI* x = X + (size_t)mat * nn;
    int hx1 = 0, hx2 = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if constexpr (FULL) {
        const int p = lane + 32 * j;
        *reinterpret_cast<double2*>(sA1 + lr_sw8(p >> 2, 2 * (p & 3))) = ra[j];
        *reinterpret_cast<double2*>(sY + j * L::LDY + 2 * lane) = rb[j];
      } else {
        // element i of the n x t / t x n factors -> (row, col); the float
        // quotient is exact enough (i < 512, fractional gap >= 1/128)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int i = lane + 64 * j + 32 * h;
          if (i < nt) {
            const int r1 = (int)(((float)i + 0.5f) * inv_t), r2 = (int)(((float)i + 0.5f) * inv_n);
            sA1[lr_sw8(r1, i - r1 * t)] = h ? ra[j].y : ra[j].x;
            sY[r2 * L::LDY + (i - r2 * n)] = h ? rb[j].y : rb[j].x;
          }
        }
      }
      hx1 = max(hx1, max(hi_abs(ra[j].x), hi_abs(ra[j].y)));
      hx2 = max(hx2, max(hi_abs(rb[j].x), hi_abs(rb[j].y)));
    }
    if (mat + nw < batch) fetch(mat + nw);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      hx1 = max(hx1, __shfl_xor_sync(0xffffffffu, hx1, o));
      hx2 = max(hx2, __shfl_xor_sync(0xffffffffu, hx2, o));
    }
    __syncwarp();
    int m = 0, rc = 0;
    bool wrote = false;
    double e1 = NAN, e2 = NAN, nv = NAN, nv2 = NAN;
    uint8_t flags = (max(hx1, hx2) >= 0x7ff00000) ? kLrBadInput : 0;  // NaN/Inf exponent field
    if (!flags) {
      // V = A2 A1: 16 k-steps of 4
      double v0 = 0.0, v1 = 0.0;
#pragma unroll
      for (int s = 0; s < 16; ++s)
        if (FULL || 4 * s < n) lr_dmma(v0, v1, sY[g * L::LDY + 4 * s + q], sA1[lr_sw8(4 * s + q, g)]);
      double* V = P + L::kSlot;
      *reinterpret_cast<double2*>(V + own) = make_double2(v0, v1);
      __syncwarp();
      double c = 0.0;
      if (lane < 8)
        for (int r = 0; r < 8; ++r) c += fabs(V[lr_sw8(r, lane)]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) c = lr_nanmax(c, __shfl_xor_sync(0xffffffffu, c, o));
      nv = c;
      if (!isfinite(nv)) {
        rc = 2;
      } else {
        rc = select_lowrank(nv, 0.0, 0, log_eps, &m, &e1, &e2);
        if (rc == 1) {
          double d0, d1;
          lr_mm8(V, V, g, q, d0, d1);
          *reinterpret_cast<double2*>(P + 2 * L::kSlot + own) = make_double2(d0, d1);
          __syncwarp();
          double c2 = 0.0;
          if (lane < 8)
            for (int r = 0; r < 8; ++r) c2 += fabs(P[2 * L::kSlot + lr_sw8(r, lane)]);
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) c2 = lr_nanmax(c2, __shfl_xor_sync(0xffffffffu, c2, o));
          nv2 = c2;
          rc = isfinite(nv2) ? select_lowrank(nv, nv2, 1, log_eps, &m, &e1, &e2) : 2;
        }
      }
      if (rc == 2) flags = kLrNonFinite;
      if (rc < 0) {
        flags = kLrNoOrder;
        e1 = e2 = NAN;
      }
    }
    if (!flags) {
      // ---- psi(V) by Paterson-Stockmeyer (poly.py:149-182) ----
      double q0, q1;
      const bool dg0 = g == 2 * q, dg1 = g == 2 * q + 1;  // own entries on the diagonal
      if (m == 0) {
        q0 = dg0 ? 1.0 : 0.0;
        q1 = dg1 ? 1.0 : 0.0;
      } else {
        const int j = ps_j_of(m);
        const int k = (m + j - 1) / j;
        for (int p = 3; p <= j; ++p) {
          double d0, d1;
          lr_mm8(P + (p - 1) * L::kSlot, P + L::kSlot, g, q, d0, d1);
          *reinterpret_cast<double2*>(P + p * L::kSlot + own) = make_double2(d0, d1);
          __syncwarp();
        }
        q0 = q1 = 0.0;
        for (int r = k - 1; r >= 0; --r) {
          const int lo = r * j, hi = (r == k - 1) ? m : r * j + j - 1;
          double s0 = 0.0, s1 = 0.0;
          if (r < k - 1) lr_mm8(P, P + j * L::kSlot, g, q, s0, s1);
          const double c0 = lr_inv_fact(lo + 1);
          double b0 = dg0 ? c0 : 0.0, b1 = dg1 ? c0 : 0.0;
          for (int tt = 1; tt <= hi - lo; ++tt) {
            const double cf = lr_inv_fact(lo + tt + 1);
            const double2 pv = *reinterpret_cast<const double2*>(P + tt * L::kSlot + own);
            b0 = fma(cf, pv.x, b0);
            b1 = fma(cf, pv.y, b1);
          }
          q0 = (r < k - 1) ? s0 + b0 : b0;
          q1 = (r < k - 1) ? s1 + b1 : b1;
          __syncwarp();
          *reinterpret_cast<double2*>(P + own) = make_double2(q0, q1);
          __syncwarp();
        }
      }
      *reinterpret_cast<double2*>(P + own) = make_double2(q0, q1);
      __syncwarp();
      if (__any_sync(0xffffffffu, !isfinite(q0) || !isfinite(q1))) {
        flags = kLrNonFinite;
      } else {
        // ---- Y = psi A2 (16 DMMA), written over A2 ----
        double ab0[8], ab1[8];
#pragma unroll
        for (int C = 0; C < 8; ++C) {
          ab0[C] = sY[q * L::LDY + 8 * C + g];
          ab1[C] = sY[(q + 4) * L::LDY + 8 * C + g];
        }
        const double pa0 = P[lr_sw8(g, q)], pa1 = P[lr_sw8(g, q + 4)];
        double y0[8], y1[8];
#pragma unroll
        for (int C = 0; C < 8; ++C) {
          y0[C] = 0.0;
          y1[C] = 0.0;
          lr_dmma(y0[C], y1[C], pa0, ab0[C]);
          lr_dmma(y0[C], y1[C], pa1, ab1[C]);
        }
        __syncwarp();
#pragma unroll
        for (int C = 0; C < 8; ++C)
          *reinterpret_cast<double2*>(sY + g * L::LDY + 8 * C + 2 * q) = make_double2(y0[C], y1[C]);
        __syncwarp();
        // overflow bound: |out| <= 1 + 8 max|A1| max|Y|; exponent words give
        // 2^(e+1) bounds, so the check is skipped unless the sum of exponents
        // comes near the top of the range
        int hy = 0;
#pragma unroll
        for (int C = 0; C < 8; ++C) hy = max(hy, max(hi_abs(y0[C]), hi_abs(y1[C])));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) hy = max(hy, __shfl_xor_sync(0xffffffffu, hy, o));
        const int eA = (hx1 >> 20) - 1023, eY = (hy >> 20) - 1023;
        const bool safe = eA + eY + 5 < (sizeof(TI) == 8 ? 1000 : 120);
        // ---- out = I + A1 Y (128 DMMA), Y as B fragments ----
        double yb0[8], yb1[8];
#pragma unroll
        for (int C = 0; C < 8; ++C) {
          yb0[C] = sY[q * L::LDY + 8 * C + g];
          yb1[C] = sY[(q + 4) * L::LDY + 8 * C + g];
        }
        bool bo = false;
        if (FULL && safe) {
#pragma unroll 2
          for (int R = 0; R < 8; ++R) {
            const double a0 = sA1[lr_sw8(8 * R + g, q)], a1v = sA1[lr_sw8(8 * R + g, q + 4)];
            double* xr = reinterpret_cast<double*>(x) + (8 * R + g) * 64 + 2 * q;
#pragma unroll
            for (int C = 0; C < 8; ++C) {
              double d0 = (R == C && dg0) ? 1.0 : 0.0;
              double d1 = (R == C && dg1) ? 1.0 : 0.0;
              lr_dmma(d0, d1, a0, yb0[C]);
              lr_dmma(d0, d1, a1v, yb1[C]);
              __stcs(reinterpret_cast<double2*>(xr + 8 * C), make_double2(d0, d1));
            }
          }
        } else {
#pragma unroll 1
          for (int R = 0; R < nT; ++R) {
            const int row = 8 * R + g;
            const double a0 = sA1[lr_sw8(row, q)], a1v = sA1[lr_sw8(row, q + 4)];
            TI* xr = x + row * (FULL ? 64 : n) + 2 * q;
#pragma unroll
            for (int C = 0; C < 8; ++C) {
              if (C < nT) {
                double d0 = (R == C && dg0) ? 1.0 : 0.0;
                double d1 = (R == C && dg1) ? 1.0 : 0.0;
                lr_dmma(d0, d1, a0, yb0[C]);
                lr_dmma(d0, d1, a1v, yb1[C]);
                const TI o0 = (TI)d0, o1 = (TI)d1;
                if constexpr (FULL) {
                  *reinterpret_cast<double2*>(xr + 8 * C) = make_double2(d0, d1);
                } else if (vec) {  // n % 8 == 0, aligned: every entry valid, pair stores
                  if constexpr (sizeof(TI) == 8)
                    __stcs(reinterpret_cast<double2*>(xr + 8 * C), make_double2(d0, d1));
                  else
                    __stcs(reinterpret_cast<float2*>(xr + 8 * C), make_float2(o0, o1));
                } else if (row < n) {
                  const int col = 8 * C + 2 * q;
                  if (col < n) __stcs(xr + 8 * C, o0);
                  if (col + 1 < n) __stcs(xr + 8 * C + 1, o1);
                }
                if (!safe) bo |= !isfinite(o0) || !isfinite(o1);
              }
            }
          }
        }
        wrote = true;
        if (__any_sync(0xffffffffu, bo)) flags = kLrNonFinite;
      }
    }
    if (flags) {  // also after an overflowing write: a flagged X is NaN (include/expmb.h)
      __syncwarp();
      for (int i = lane; i < nn; i += 32) x[i] = (TI)NAN;
    }
    if (lane == 0) {
      if (po.m) po.m[mat] = (int8_t)m;
      if (po.e1) po.e1[mat] = e1;
      if (po.e2) po.e2[mat] = e2;
      if (po.norms) {
        po.norms[2 * mat] = nv;
        po.norms[2 * mat + 1] = nv2;
      }
      if (po.mults) po.mults[mat] = flags ? 0 : lr_mults(m);
      if (po.flags) po.flags[mat] = flags;
    }
    __syncwarp();
  }
}

}  // namespace expmb
