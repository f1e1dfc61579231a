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
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>

#include "fused_small.cuh"
#include "select.cuh"

namespace expmb {

constexpr int kGemmBM = 128;
constexpr int kGemmBN = 128;
constexpr int kGemmBK = 8;

enum Stage { STAGE_W2 = 0, STAGE_W3, STAGE_W4, STAGE_E1, STAGE_E2, STAGE_E3, STAGE_SQ,
             STAGE_A1,      // Alg. 1 term (engine.py:109-112): X += Y; Y <- B Y / k, k = sq_step + 2
             STAGE_A1SQ };  // Alg. 1 squaring (engine.py:113): s from the int32 array s32

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
  const int* route;  // per list slot: 1 = another backend (the int8-slice GEMM) handles it; may be null
  const int* s32;    // Alg. 1: per-matrix scaling (may exceed int8)
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
  const T* acc_src;  // Alg. 1: acc_dst += acc_src elementwise (X += Y, engine.py:110)
  T* acc_dst;
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
  e.acc_src = nullptr; e.acc_dst = nullptr;
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
  if (stage == STAGE_A1) {
    // term j = sq_step (k = j + 2): the product B Y_j / k with B = 2^-s W
    // stored in W2, Y ping-ponging between Y0 / Y1; X += Y_j fused into the
    // same pass; column sums of Y_{j+1} for the termination test
    const int j = g.sq_step;
    e.L = g.W2 + o;
    e.R = ((j & 1) ? g.Y1 : g.Y0) + o;
    e.out[0] = ((j & 1) ? g.Y0 : g.Y1) + o;
    e.alpha = T(1) / T(j + 2);  // Y / k taken as Y * fl(1/k), as the fused kernel
    e.colnorm = true;
    e.acc_src = e.R;
    e.acc_dst = sq_target(g, z, g.s32[z], 0);
    return true;
  }
  if (stage == STAGE_A1SQ) {
    const int s = g.s32[z];
    if (s <= g.sq_step) return false;
    e.L = e.R = sq_target(g, z, s, g.sq_step);
    e.out[0] = sq_target(g, z, s, g.sq_step + 1);
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

// ---------------------------------------------------------------------------
// FMA GEMM mainloop: 128x128 CTA tile, 256 threads, 8x8 outputs per thread,
// multi-stage cp.async (LDGSTS) ring so global latency hides behind several
// k-tiles of FMAs.  Operand tiles stay row-major in shared memory: a thread
// reads its 8 L-rows with 16-byte loads along k and its 8 R-columns with
// 16-byte loads along n (fp64 columns are interleaved in 2-wide groups so the
// 16 lanes of a row read 256 contiguous bytes: no bank conflicts).
// ---------------------------------------------------------------------------
template <typename T>
struct SimtCfg;
template <>
struct SimtCfg<float> {
  static constexpr int BK = 16, STAGES = 4, KV = 4, VW = 4;
};
template <>
struct SimtCfg<double> {
  static constexpr int BK = 16, STAGES = 3, KV = 2, VW = 2;
};

__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool pred) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
  const int sz = pred ? 16 : 0;  // src-size 0 -> zero fill
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <typename T>
__device__ __forceinline__ int simt_col(int tx, int j) {
  if constexpr (sizeof(T) == 4) return (j < 4) ? tx * 4 + j : 64 + tx * 4 + (j - 4);
  else return (j >> 1) * 32 + tx * 2 + (j & 1);
}

// TWO: fp32 two-level accumulation (needed for long k: n > 512).  Without
// it the kernel fits 128 registers and two CTAs share an SM, so one CTA's
// prologue/epilogue overlaps the other's mainloop (short k at n <= 512).
// MMA (fp64 only): the mainloop issues DMMA (mma.sync.m8n8k4.f64, the FP64
// tensor cores) instead of DFMAs: warp (wr, wc) of the 2 x 4 warp grid owns a
// 64 x 32 sub-tile = 8 x 4 DMMA tiles, and thread "row slot" i / column pair
// j0 of the epilogue map onto the accumulator fragments.
// A1: the Alg. 1 term stage's extra X += Y epilogue (its own instantiation,
// so the other stages' epilogues carry no extra live registers: with it
// inline the fp32 kernel's spills grew from 48 to 84 bytes and C3 slowed 13%)
template <typename T, bool TWO, bool MMA, bool A1 = false>
__device__ __forceinline__ void gemm_tile(const GemmCtx<T>& g, int stage, const int* __restrict__ list, int slot,
                                          int bx, int by, unsigned char* smem_raw) {
  using C = SimtCfg<T>;
  constexpr int BK = C::BK, ST = C::STAGES, KV = C::KV, VW = C::VW;
  // padded rows: fp64 strides of 20 / 132 doubles (= 8 banks mod 32) make the
  // DMMA fragment loads conflict-free per half-warp (a 64-bit load is served
  // 16 lanes at a time); fp32 keeps 16-byte padding.
  constexpr int LDA = BK + (sizeof(T) == 4 ? KV : 4);
  // fp64 rows padded to 136 doubles (= 16 banks mod 32) so the DMMA B
  // fragments (4 k-rows x 8 columns per warp load) hit the 2-wavefront minimum
  constexpr int LDB = kGemmBN + 4;
  constexpr int A_ELEMS = kGemmBM * LDA, B_ELEMS = BK * LDB;
  T* As = reinterpret_cast<T*>(smem_raw);
  T* Bs = As + ST * A_ELEMS;

  const int z = list ? list[slot] : slot;
  if (g.route && g.route[slot]) return;
  Epi<T> e;
  if (!make_epi(g, stage, z, e)) return;
  const int n = g.n;
  const int m0 = by * kGemmBM, n0 = bx * kGemmBN;
  const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
  const int lane = tid % 32, warp = tid / 32, lg = lane >> 2, lt = lane & 3, wr = warp >> 2, wc = warp & 3;
  // epilogue coordinates of accumulator slot (i, j) within the CTA tile
  auto acc_row = [&](int i) { return MMA ? 64 * wr + 8 * i + lg : (i < 4 ? ty * 4 + i : 64 + ty * 4 + i - 4); };
  auto acc_col = [&](int j) { return MMA ? 32 * wc + 8 * (j >> 1) + 2 * lt + (j & 1) : simt_col<T>(tx, j); };
  auto red_slot = [&]() { return MMA ? wr * 8 + lg : ty; };
  const bool vec = (n % KV) == 0;  // 16-byte rows chunks are whole
  const T* __restrict__ Lp = e.L;
  const T* __restrict__ Rp = e.R;
  const int nk = (n + BK - 1) / BK;

  // ---- async tile loader ----
  constexpr int A_CHUNKS = kGemmBM * BK / KV, B_CHUNKS = BK * kGemmBN / KV;  // 16-byte chunks
  auto load_tile = [&](int kt, int st) {
    const int k0 = kt * BK;
    T* as = As + st * A_ELEMS;
    T* bs = Bs + st * B_ELEMS;
#pragma unroll
    for (int c = tid; c < A_CHUNKS; c += 256) {
      const int r = c / (BK / KV), kc = (c % (BK / KV)) * KV;
      const int gr = m0 + r, gk = k0 + kc;
      if (vec) {
        cp_async16(as + r * LDA + kc, Lp + (size_t)(gr < n ? gr : 0) * n + (gk < n ? gk : 0), gr < n && gk < n);
      } else {
#pragma unroll
        for (int q = 0; q < KV; ++q) as[r * LDA + kc + q] = (gr < n && gk + q < n) ? Lp[(size_t)gr * n + gk + q] : T(0);
      }
    }
#pragma unroll
    for (int c = tid; c < B_CHUNKS; c += 256) {
      const int r = c / (kGemmBN / KV), nc = (c % (kGemmBN / KV)) * KV;
      const int gk = k0 + r, gn = n0 + nc;
      if (vec) {
        cp_async16(bs + r * LDB + nc, Rp + (size_t)(gk < n ? gk : 0) * n + (gn < n ? gn : 0), gk < n && gn < n);
      } else {
#pragma unroll
        for (int q = 0; q < KV; ++q) bs[r * LDB + nc + q] = (gk < n && gn + q < n) ? Rp[(size_t)gk * n + gn + q] : T(0);
      }
    }
  };

  // fp32: two-level accumulation (a fresh partial every 32 k, added to the
  // running sum) keeps the summation error near (32 + n/32) u instead of n u.
  constexpr bool kTwoLevel = sizeof(T) == 4 && TWO;
  constexpr int kChunkTiles = 32 / BK;
  T acc[8][8];
  float2 pacc[kTwoLevel ? 8 : 1][kTwoLevel ? 4 : 1];  // fp32 partials as FFMA2 pairs
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = T(0);

#pragma unroll
  for (int s = 0; s < ST - 1; ++s) {
    if (s < nk) load_tile(s, s);
    cp_async_commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<ST - 2>();
    __syncthreads();
    {  // refill the stage consumed in iteration kt-1
      const int nt = kt + ST - 1;
      if (nt < nk) load_tile(nt, nt % ST);
      cp_async_commit();
    }
    const T* as = As + (kt % ST) * A_ELEMS;
    const T* bs = Bs + (kt % ST) * B_ELEMS;
    if constexpr (MMA && sizeof(T) == 8) {
      const double* la = reinterpret_cast<const double*>(as) + (64 * wr + lg) * LDA + lt;
      const double* rb = reinterpret_cast<const double*>(bs) + lt * LDB + 32 * wc + lg;
#pragma unroll
      for (int kk = 0; kk < BK; kk += 4) {
        double a[8], b[4];
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = la[8 * i * LDA + kk];
#pragma unroll
        for (int q = 0; q < 4; ++q) b[q] = rb[kk * LDB + 8 * q];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int q = 0; q < 4; ++q)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(acc[i][2 * q]), "+d"(acc[i][2 * q + 1])
                         : "d"(a[i]), "d"(b[q]));
      }
      continue;
    }
    if constexpr (kTwoLevel) {
      if (kt % kChunkTiles == 0) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) pacc[i][j] = make_float2(0.f, 0.f);
      }
    }
#pragma unroll
    for (int kb = 0; kb < BK; kb += KV) {
      T a[8][KV];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int r = (i < 4) ? ty * 4 + i : 64 + ty * 4 + (i - 4);
        const T* p = as + r * LDA + kb;
        if constexpr (sizeof(T) == 4) {
          const float4 v = *reinterpret_cast<const float4*>(p);
          a[i][0] = v.x; a[i][1] = v.y; a[i][2] = v.z; a[i][3] = v.w;
        } else {
          const double2 v = *reinterpret_cast<const double2*>(p);
          a[i][0] = v.x; a[i][1] = v.y;
        }
      }
#pragma unroll
      for (int kk = 0; kk < KV; ++kk) {
        T b[8];
        const T* q = bs + (kb + kk) * LDB;
        if constexpr (sizeof(T) == 4) {
          const float4 v0 = *reinterpret_cast<const float4*>(q + tx * 4);
          const float4 v1 = *reinterpret_cast<const float4*>(q + 64 + tx * 4);
          b[0] = v0.x; b[1] = v0.y; b[2] = v0.z; b[3] = v0.w;
          b[4] = v1.x; b[5] = v1.y; b[6] = v1.z; b[7] = v1.w;
        } else {
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            const double2 v = *reinterpret_cast<const double2*>(q + h * 32 + tx * 2);
            b[2 * h] = v.x; b[2 * h + 1] = v.y;
          }
        }
        if constexpr (kTwoLevel) {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float2 ai = make_float2((float)a[i][kk], (float)a[i][kk]);
#pragma unroll
            for (int j = 0; j < 4; ++j)
              pacc[i][j] = ffma2(make_float2((float)b[2 * j], (float)b[2 * j + 1]), ai, pacc[i][j]);
          }
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[i][j] = fma(a[i][kk], b[j], acc[i][j]);
        }
      }
    }
    if constexpr (kTwoLevel) {
      if (kt % kChunkTiles == kChunkTiles - 1 || kt + 1 == nk) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            acc[i][2 * j] += (T)pacc[i][j].x;
            acc[i][2 * j + 1] += (T)pacc[i][j].y;
          }
      }
    }
  }
  cp_async_wait<0>();

  // ---- fused epilogue (VW-wide vectors along a row) ----
  double csum[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) csum[j] = 0.0;
  const bool evec = (n % VW) == 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int row = m0 + acc_row(i);
    if (row >= n) continue;
#pragma unroll
    for (int j0 = 0; j0 < 8; j0 += VW) {
      const int col0 = n0 + acc_col(j0);
      if (col0 >= n) continue;
      const size_t pos = (size_t)row * n + col0;
      const bool full = evec && col0 + VW <= n;
      T o0[VW], in[4][VW];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (q < e.nin) {
          if (full) {
            if constexpr (sizeof(T) == 4) {
              const float4 v = *reinterpret_cast<const float4*>(e.in[q] + pos);
              in[q][0] = v.x; in[q][1] = v.y; in[q][2] = v.z; in[q][3] = v.w;
            } else {
              const double2 v = *reinterpret_cast<const double2*>(e.in[q] + pos);
              in[q][0] = v.x; in[q][1] = v.y;
            }
          } else {
#pragma unroll
            for (int v = 0; v < VW; ++v) in[q][v] = (col0 + v < n) ? e.in[q][pos + v] : T(0);
          }
        }
      }
#pragma unroll
      for (int v = 0; v < VW; ++v) {
        const T dg = (row == col0 + v) ? T(1) : T(0);
        T x = e.alpha * acc[i][j0 + v];
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (q < e.nin) x = fma(e.c[0][q], in[q][v], x);
        o0[v] = fma(e.d[0], dg, x);
      }
      auto put = [&](T* dst, const T (&val)[VW]) {
        if (full) {
          if constexpr (sizeof(T) == 4) *reinterpret_cast<float4*>(dst + pos) = make_float4(val[0], val[1], val[2], val[3]);
          else *reinterpret_cast<double2*>(dst + pos) = make_double2(val[0], val[1]);
        } else {
#pragma unroll
          for (int v = 0; v < VW; ++v)
            if (col0 + v < n) dst[pos + v] = val[v];
        }
      };
      put(e.out[0], o0);
      if (A1 && e.acc_dst != nullptr) {  // X += Y (Alg. 1): the same positions, one read-modify-write
        T xv[VW];
#pragma unroll
        for (int v = 0; v < VW; ++v) xv[v] = (col0 + v < n) ? e.acc_dst[pos + v] + e.acc_src[pos + v] : T(0);
        put(e.acc_dst, xv);
      }
      if (e.nout > 1) {
#pragma unroll
        for (int k = 1; k < 3; ++k) {
          T ok[VW];
#pragma unroll
          for (int v = 0; v < VW; ++v) {
            T x = o0[v];
#pragma unroll
            for (int q = 0; q < 4; ++q)
              if (q < e.nin) x = fma(e.c[k][q], in[q][v], x);
            ok[v] = fma(e.d[k], (row == col0 + v) ? T(1) : T(0), x);
          }
          put(e.out[k], ok);
        }
      }
      if (e.colnorm) {
#pragma unroll
        for (int v = 0; v < VW; ++v)
          if (col0 + v < n) csum[j0 + v] += fabs((double)o0[v]);
      }
    }
  }
  if (e.colnorm) {
    // deterministic column reduction over the 16 thread rows of the tile
    double* red = reinterpret_cast<double*>(smem_raw);  // 16 x 128 doubles
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 8; ++j) red[red_slot() * kGemmBN + acc_col(j)] = csum[j];
    __syncthreads();
    if (tid < kGemmBN && n0 + tid < n) {
      double a = 0.0;
      for (int r = 0; r < 16; ++r) a += red[r * kGemmBN + tid];
      g.part[((size_t)z * g.tiles_m + by) * n + n0 + tid] = a;
    }
  }
}

// One launch = one stage over the first *dcount slots of `list` (or `hcount`
// when dcount is null): a persistent grid walks the work units (slot, tile
// row, tile column) with the tile column fastest, so co-resident CTAs share
// operand panels in L2.  The slot count lives in device memory (written by
// the device bucket scheduler, k_bucket), so the host never waits for it.
template <typename T, bool TWO>
constexpr bool kZStride = sizeof(T) == 4 && !TWO;

template <typename T, bool TWO = (sizeof(T) == 4), bool MMA = false, bool A1 = false>
__global__ void __launch_bounds__(256, (sizeof(T) == 4 && !TWO) ? 2 : 1)
gemm_stage_kernel(GemmCtx<T> g, int stage, const int* __restrict__ list, const int* __restrict__ dcount, int hcount) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int cnt = dcount ? *dcount : hcount;
  if constexpr (kZStride<T, TWO>) {
    // 2 CTAs/SM at the 128-register cap: the tile stays (blockIdx.x, blockIdx.y)
    // and only the slot is walked (blockIdx.z stride), so the loop costs no
    // mainloop registers; n <= 512 keeps the tile count far below the resident
    // CTAs, so the z-stride grid is balanced
    for (int slot = blockIdx.z; slot < cnt; slot += gridDim.z) {
      __syncthreads();  // the previous unit's epilogue may still read shared memory
      gemm_tile<T, TWO, MMA, A1>(g, stage, list, slot, blockIdx.x, blockIdx.y, smem_raw);
    }
  } else {
    const int total = cnt * (((g.n + kGemmBN - 1) / kGemmBN) * g.tiles_m);
    for (int w = blockIdx.x; w < total; w += gridDim.x) {
      const int tn = (g.n + kGemmBN - 1) / kGemmBN, tiles = tn * g.tiles_m;
      const int slot = w / tiles, t = w - slot * tiles;
      __syncthreads();  // the previous unit's epilogue may still read shared memory
      gemm_tile<T, TWO, MMA, A1>(g, stage, list, slot, t % tn, t / tn, smem_raw);
    }
  }
}

template <typename T>
constexpr int simt_smem_bytes() {
  using C = SimtCfg<T>;
  return (int)(C::STAGES * (kGemmBM * (C::BK + (sizeof(T) == 4 ? C::KV : 4)) + C::BK * (kGemmBN + 4)) * sizeof(T));
}

static inline int sm_count_dev() {
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

// Persistent grid size for a kernel: resident CTAs per SM x SMs, capped by
// the work.  `resident` is the residency the kernel's __launch_bounds__
// guarantees (its minBlocksPerMultiprocessor, which register and shared
// memory use are built to meet); 0 asks the occupancy API instead.  (On this
// driver the API reported 1 CTA/SM for kernels the hardware runs two per SM
// -- the int8 and 2-CTA FFMA stages -- so the launch bounds are the source of
// truth where they exist.)
template <typename K>
static int persistent_grid(K kern, int threads, size_t smem, int64_t units, int* occ_cache, int resident = 0) {
  if (*occ_cache <= 0) {
    int o = resident;
    if (o <= 0 && (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, threads, smem) != cudaSuccess || o < 1))
      o = 1;
    *occ_cache = o;
    if (getenv("EXPMB_DEBUG_OCC"))
      fprintf(stderr, "expmb occupancy: %d CTAs/SM (%d threads, %zu B dynamic smem)\n", o, threads, smem);
  }
  const int64_t cap = (int64_t)sm_count_dev() * *occ_cache;
  return (int)(units < cap ? (units < 1 ? 1 : units) : cap);
}

// One product stage over `list` (null = slots 0..), the first *dcount slots
// (dcount null: `count`); `count` bounds the work on the host side.
template <typename T, bool A1>
static int gemm_launch_t(const GemmCtx<T>& g, int stage, const int* list, int count, cudaStream_t st,
                         const int* dcount) {
  if (count <= 0) return 0;
  static bool attr = false;
  constexpr int smem = simt_smem_bytes<T>();
  auto k_two = gemm_stage_kernel<T, true, false, A1>;
  auto k_one = gemm_stage_kernel<T, false, false, A1>;
  auto k_mma = gemm_stage_kernel<T, false, sizeof(T) == 8, A1>;
  if (!attr) {
    if (cudaFuncSetAttribute(k_two, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess ||
        cudaFuncSetAttribute(k_one, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess ||
        (sizeof(T) == 8 && cudaFuncSetAttribute(k_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess))
      return 1;
    attr = true;
  }
  static int occ[3] = {0, 0, 0};
  const int tn = (g.n + kGemmBN - 1) / kGemmBN, tm = (g.n + kGemmBM - 1) / kGemmBM;
  const int64_t units = (int64_t)count * tn * tm;
  static const bool dmma = !(getenv("EXPMB_NO_DMMA") && getenv("EXPMB_NO_DMMA")[0] == '1');
  if (sizeof(T) == 4 && g.n > 512)
    k_two<<<persistent_grid(k_two, 256, smem, units, &occ[0], 1), 256, smem, st>>>(g, stage, list, dcount, count);
  else if (sizeof(T) == 8 && dmma)
    k_mma<<<persistent_grid(k_mma, 256, smem, units, &occ[2], 1), 256, smem, st>>>(g, stage, list, dcount, count);
  else {
    // z-stride grid (kZStride): tiles x enough slots to fill every resident CTA once
    const int t2 = tn * tm;
    const int zc = std::max(1, persistent_grid(k_one, 256, smem, units, &occ[1], sizeof(T) == 4 ? 2 : 1) / t2);
    k_one<<<dim3(tn, tm, std::min(count, zc)), 256, smem, st>>>(g, stage, list, dcount, count);
  }
  return cudaGetLastError() != cudaSuccess;
}
template <typename T>
static int gemm_launch(const GemmCtx<T>& g, int stage, const int* list, int count, cudaStream_t st,
                       const int* dcount = nullptr) {
  return stage == STAGE_A1 ? gemm_launch_t<T, true>(g, stage, list, count, st, dcount)
                           : gemm_launch_t<T, false>(g, stage, list, count, st, dcount);
}

// ---------------------------------------------------------------------------
// elementwise stage (before the first evaluation product)
// ---------------------------------------------------------------------------
// The elementwise first step for matrix z, elements i0, i0 + stride, ...
template <typename T>
__device__ __forceinline__ void elem_one(const GemmCtx<T>& g, int z, size_t i0, size_t stride) {
  const int m = g.m[z], s = g.s[z];
  const int n = g.n;
  const size_t nn = (size_t)n * n;
  const int64_t o = (int64_t)z * g.mstride;
  const T* Wz = g.W + (int64_t)z * g.wstride;
  const T* A2 = g.W2 + o;
  const double sg = pow2_neg<double>(s), sg2 = pow2_neg<double>(2 * s);
  for (size_t i = i0; i < nn; i += stride) {
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
__global__ void __launch_bounds__(256) elem_kernel(GemmCtx<T> g, const int* __restrict__ list,
                                                   const int* __restrict__ dcount, int hcount) {
  const int cnt = dcount ? *dcount : hcount;
  for (int slot = blockIdx.y; slot < cnt; slot += gridDim.y)
    elem_one(g, list[slot], (size_t)blockIdx.x * blockDim.x + threadIdx.x, (size_t)gridDim.x * blockDim.x);
}

template <typename T>
static int elem_launch(const GemmCtx<T>& g, const int* list, int count, cudaStream_t st,
                       const int* dcount = nullptr) {
  if (count <= 0) return 0;
  const size_t nn = (size_t)g.n * g.n;
  int bx = (int)((nn + 255) / 256);
  if (bx > 64) bx = 64;
  // slots grid-strided: enough CTAs for ~8 per SM
  int by = (int)std::min<int64_t>(count, std::max<int64_t>(1, (int64_t)sm_count_dev() * 8 / bx));
  dim3 grid(bx, by);
  elem_kernel<T><<<grid, 256, 0, st>>>(g, list, dcount, count);
  return cudaGetLastError() != cudaSuccess;
}

}  // namespace expmb
