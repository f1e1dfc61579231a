// fused_dmma.cuh -- fp64 fused kernel for 32 < n <= 64 on the FP64 tensor
// cores (DMMA, mma.sync.m8n8k4.f64).
//
// Same per-matrix program as the straight-line Sastre path of
// fused_small.cuh (engine.py:119-152: norms + ladder, exact rescaling,
// poly.py:189-230 formulas, squarings), one 256-thread CTA per matrix, but
// every n x n product is 128 DMMA instructions per warp instead of 1024
// DFMAs: the FMA-pipe version was issue/latency bound at 31% of the FP64
// peak (profiles/ncu_C1_fused_r01.txt).
//
// Layout: warp w owns rows 16*(w/2) .. +15 and columns 32*(w%2) .. +31 of
// every state matrix (2 x 4 DMMA 8x8 tiles); lane (g = l/4, t = l%4) holds
// rows {r0, r0+8} x columns {32wc + 8q + 2t + h : q < 4, h < 2}, i.e. exactly
// the m8n8k4 accumulator fragments, so products land in place.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "fused_small.cuh"
#include "select.cuh"

namespace expmb {

struct Dm {
  static constexpr int NPAD = 64, LD = 68, NT = 256;
  static constexpr int BUF = NPAD * LD;  // doubles per operand buffer
  static constexpr size_t kSmem = 2 * BUF * sizeof(double) + 4 * NPAD * sizeof(double) + 64;
  using Tile = double[2][8];

  int warp, lane, g, t, wr, wc;
  double* buf0;
  double* buf1;
  double* red;

  __device__ __forceinline__ int row(int i) const { return 16 * wr + 8 * i + g; }
  __device__ __forceinline__ int col(int j) const { return 32 * wc + 8 * (j >> 1) + 2 * t + (j & 1); }
  __device__ __forceinline__ bool is_diag(int i, int j) const { return row(i) == col(j); }

  __device__ __forceinline__ void sync() const { __syncthreads(); }

  __device__ __forceinline__ void store(double* buf, const Tile& v) const {
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int q = 0; q < 4; ++q)
        *reinterpret_cast<double2*>(buf + row(i) * LD + col(2 * q)) = make_double2(v[i][2 * q], v[i][2 * q + 1]);
  }

  // acc = L * R (row-major NPAD x NPAD in shared memory) with DMMA
  __device__ __forceinline__ void mm(const double* __restrict__ L, const double* __restrict__ R, Tile& acc) const {
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[i][j] = 0.0;
    const double* la = L + (16 * wr + g) * LD + t;
    const double* rb = R + t * LD + 32 * wc + g;
#pragma unroll 4
    for (int kk = 0; kk < NPAD / 4; ++kk) {
      const double a0 = la[4 * kk], a1 = la[8 * LD + 4 * kk];
      double b[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) b[q] = rb[4 * kk * LD + 8 * q];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(acc[0][2 * q]), "+d"(acc[0][2 * q + 1])
                     : "d"(a0), "d"(b[q]));
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(acc[1][2 * q]), "+d"(acc[1][2 * q + 1])
                     : "d"(a1), "d"(b[q]));
      }
    }
  }

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

  // ||.||_1: column abs-sums (16 rows per warp, then the 4 warp-rows), max.
  __device__ __forceinline__ double norm1(const Tile& v) const {
    double cs[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) cs[j] = fabs(v[0][j]) + fabs(v[1][j]);
#pragma unroll
    for (int off = 4; off < 32; off *= 2)
#pragma unroll
      for (int j = 0; j < 8; ++j) cs[j] += __shfl_xor_sync(0xffffffffu, cs[j], off);
    if (g == 0) {
#pragma unroll
      for (int j = 0; j < 8; ++j) red[wr * NPAD + col(j)] = cs[j];
    }
    sync();
    double* res = red + 4 * NPAD;
    if (warp == 0) {
      double mx = -INFINITY;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = lane + 32 * h;
        const double a = ((red[c] + red[NPAD + c]) + red[2 * NPAD + c]) + red[3 * NPAD + c];
        mx = nanmax(mx, a);
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) mx = nanmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
      if (lane == 0) res[0] = mx;
    }
    sync();
    const double r = res[0];
    sync();
    return r;
  }

  __device__ __forceinline__ bool any(bool f) const { return __syncthreads_or(f) != 0; }

  __device__ __forceinline__ void load(const double* __restrict__ src, int n, bool vec, Tile& v) const {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int r = row(i);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int c = col(2 * q);
        if (vec) {
          const double2 x = __ldg(reinterpret_cast<const double2*>(src + r * NPAD + c));
          v[i][2 * q] = x.x; v[i][2 * q + 1] = x.y;
        } else {
          v[i][2 * q] = (r < n && c < n) ? __ldg(src + (size_t)r * n + c) : 0.0;
          v[i][2 * q + 1] = (r < n && c + 1 < n) ? __ldg(src + (size_t)r * n + c + 1) : 0.0;
        }
      }
    }
  }
  __device__ __forceinline__ void save(double* __restrict__ dst, int n, bool vec, const Tile& v) const {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int r = row(i);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int c = col(2 * q);
        if (vec) {
          __stcs(reinterpret_cast<double2*>(dst + r * NPAD + c), make_double2(v[i][2 * q], v[i][2 * q + 1]));
        } else {
          if (r < n && c < n) dst[(size_t)r * n + c] = v[i][2 * q];
          if (r < n && c + 1 < n) dst[(size_t)r * n + c + 1] = v[i][2 * q + 1];
        }
      }
    }
  }
};

__global__ void __launch_bounds__(Dm::NT, 1)
expm_dmma_kernel(const double* __restrict__ W, double* __restrict__ X, int64_t batch, int n, double log_eps,
                 PlanOut po, int* __restrict__ ctr) {
  using Tile = Dm::Tile;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int64_t next_sh;
  Dm f;
  f.warp = threadIdx.x / 32;
  f.lane = threadIdx.x % 32;
  f.g = f.lane >> 2;
  f.t = f.lane & 3;
  f.wr = f.warp >> 1;
  f.wc = f.warp & 1;
  f.buf0 = reinterpret_cast<double*>(smem_raw);
  f.buf1 = f.buf0 + Dm::BUF;
  f.red = f.buf1 + Dm::BUF;

  const bool vec = (n == Dm::NPAD);
  const size_t nn = (size_t)n * n;
  const int64_t stride = gridDim.x;
  int64_t idx = blockIdx.x;
#define EW(expr)                                 \
  _Pragma("unroll") for (int i = 0; i < 2; ++i) \
  _Pragma("unroll") for (int j = 0; j < 8; ++j) { expr; }
#define DG(i, j) (f.is_diag(i, j) ? 1.0 : 0.0)
  while (idx < batch) {
    // claim the next matrix early (dynamic: costs vary 0..11 products)
    if (threadIdx.x == 0) next_sh = ctr ? stride + atomicAdd(ctr, 1) : idx + stride;
    Tile B, A2, Y0, Y1, P;
    f.load(W + idx * nn, n, vec, B);
    double nrm[2] = {f.norm1(B), NAN};
    const int64_t nidx = next_sh;  // published before the norm's barriers
    Plan p{0, 0, 0.0, 0.0};
    bool bad = false;
    int need = 2;
    if (nrm[0] != 0.0 && !(nrm[0] > rung0_threshold(log_eps))) {
      need = select_sastre_fast(nrm[0], 0.0, 1, log_eps, &p);
      if (need < 0) {
        const double lw[4] = {log2_or_ninf(nrm[0]), 0, 0, 0};
        need = select_walk_lw(lw, 1, log_eps, 0, &p);
      }
    }
    if (nrm[0] == 0.0) {
      EW(P[i][j] = DG(i, j));
    } else if (need < 2) {
      EW(P[i][j] = B[i][j] + DG(i, j));
    } else {
      f.square(B, A2);
      nrm[1] = f.norm1(A2);
      bad |= !(nrm[1] < INFINITY);
      need = select_sastre_fast2(nrm[0], nrm[1], log_eps, &p);
      if (need < 0) {
        const double lw[4] = {log2_or_ninf(nrm[0]), log2_or_ninf(nrm[1]), 0, 0};
        select_walk_lw(lw, 2, log_eps, 0, &p);
      }
      const double sc = pow2_neg<double>(p.s), sc2 = pow2_neg<double>(2 * p.s);
      EW(B[i][j] *= sc; A2[i][j] *= sc2);
      if (p.m == 2) {
        EW(P[i][j] = (A2[i][j] * 0.5 + B[i][j]) + DG(i, j));
      } else if (p.m == 4) {
        Tile L;
        EW(L[i][j] = (A2[i][j] * 0.25 + B[i][j]) / 3.0 + DG(i, j));
        f.product(L, A2, P);
        EW(P[i][j] = (P[i][j] * 0.5 + B[i][j]) + DG(i, j));
      } else {
        const double* c = (p.m == 8) ? kT8 : kT15;
        Tile L, R;
        EW(R[i][j] = c[0] * A2[i][j] + c[1] * B[i][j]);
        f.product(A2, R, Y0);
        EW(L[i][j] = (Y0[i][j] + c[2] * A2[i][j]) + c[3] * B[i][j]; R[i][j] = Y0[i][j] + c[4] * A2[i][j]);
        f.product(L, R, P);
        if (p.m == 8) {
          EW(P[i][j] = (((P[i][j] + c[5] * Y0[i][j]) + A2[i][j] * 0.5) + B[i][j]) + DG(i, j));
        } else {
          EW(Y1[i][j] = (P[i][j] + c[5] * Y0[i][j]) + c[6] * A2[i][j];
             L[i][j] = (Y1[i][j] + c[7] * A2[i][j]) + c[8] * B[i][j];
             R[i][j] = (Y1[i][j] + c[9] * Y0[i][j]) + c[10] * B[i][j]);
          f.product(L, R, P);
          EW(P[i][j] = ((((P[i][j] + c[11] * Y1[i][j]) + c[12] * Y0[i][j]) + c[13] * A2[i][j]) + c[14] * B[i][j]) +
                       (f.is_diag(i, j) ? c[15] : 0.0));
          for (int q = 0; q < p.s; ++q) {
            f.square(P, Y1);
            EW(P[i][j] = Y1[i][j]);
          }
        }
      }
    }
    EW(bad |= !isfinite(P[i][j]));
    bad = f.any(bad);
    f.save(X + idx * nn, n, vec, P);
    if (threadIdx.x == 0) {
      if (po.m) po.m[idx] = (int8_t)p.m;
      if (po.s) po.s[idx] = (int8_t)p.s;
      if (po.e1) po.e1[idx] = p.e1;
      if (po.e2) po.e2[idx] = p.e2;
      if (po.norms) { po.norms[2 * idx] = nrm[0]; po.norms[2 * idx + 1] = nrm[1]; }
      if (po.mults) po.mults[idx] = budget(p.m, 0) + p.s;
      if (po.nonfinite) po.nonfinite[idx] = (uint8_t)(bad || !(nrm[0] < INFINITY));
    }
    idx = nidx;
  }
#undef EW
#undef DG
}

}  // namespace expmb
