// lowrank_large.cuh -- batched low-rank exponential for inner rank t > 32.
//
// Same algorithm as lowrank.cuh (engine.py:198-257: V = A2 A1, the LOWRANK_ORDERS
// ladder on ||V||_1 / ||V^2||_1, psi(V) = sum_{i<=m} V^i/(i+1)! by
// Paterson-Stockmeyer (poly.py:149-182), e^W = I + A1 (psi A2)), for t x t
// problems too large for one CTA's shared memory: every t x t operand lives in
// a global workspace (binary64, as the CTA kernel computes for t > 8), each
// step is one batched launch, and every per-matrix decision (order, powers,
// Horner stages, flags) is read on the device, so the host issues a fixed
// launch sequence with no synchronisation.
//
//   V = A2 A1 | ||V||_1, ladder | V^2 where needed | ||V^2||_1, ladder + plan |
//   V^3..V^6 where j(m) needs them | q = block((k-1)j, m) | k-1 Horner stages
//   q <- q V^j + block(rj, rj+j-1) | Y = psi A2 | X = I + A1 Y (+ flags).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "lowrank.cuh"

namespace expmb {

constexpr int kLrlSlots = 9;  // V^1..V^6, q (two), block scratch

struct LrlLayout {
  int64_t chunk;
  size_t t2, yb;  // bytes of one t x t slot, of one t x n Y
  size_t off_slots, off_y, off_state, total;
};

static inline LrlLayout lrl_layout(int64_t batch, int n, int t) {
  LrlLayout L{};
  L.t2 = (((size_t)t * t * 8) + 255) & ~(size_t)255;
  L.yb = (((size_t)t * n * 8) + 255) & ~(size_t)255;
  const size_t per = kLrlSlots * L.t2 + L.yb + 64;
  int64_t chunk = (int64_t)(((size_t)16 << 30) / per);
  if (chunk < 1) chunk = 1;
  if (chunk > 65535) chunk = 65535;
  if (chunk > batch) chunk = batch;
  L.chunk = chunk;
  size_t off = 0;
  L.off_slots = off; off += (size_t)kLrlSlots * L.t2 * chunk;
  L.off_y = off; off += L.yb * chunk;
  L.off_state = off; off += (((size_t)chunk * 64) + 255) & ~(size_t)255;
  L.total = off;
  return L;
}

// per-matrix state (64 bytes)
struct LrlState {
  double nv, nv2, e1, e2;
  int m, rc, j, k;
  int flags, pad0, pad1, pad2;
};

// Stage codes the GEMM launches gate on.
enum LrlGate : int {
  LG_ALL = 0,   // every matrix not yet flagged
  LG_V2,        // the ladder asked for ||V^2||_1
  LG_POW,       // V^p needed (p <= j(m)), p = arg
  LG_HORNER,    // Horner stage h = arg exists (k - 2 - h >= 0)
};

__device__ __forceinline__ bool lrl_gate(const LrlState& s, int gate, int arg) {
  if (s.flags) return false;
  switch (gate) {
    case LG_ALL: return true;
    case LG_V2: return s.rc == 1;
    case LG_POW: return s.m >= 2 && arg <= s.j;
    case LG_HORNER: return s.m >= 2 && s.k - 2 - arg >= 0;
  }
  return false;
}

// C = A B (+ Cadd) (+ d I), binary64 accumulation, 64 x 64 tiles, 256 threads
// with 4 x 4 outputs each; matrix b of the chunk runs only if its gate holds.
// TC = float / double output; finiteness of C is folded into the state flags.
// Operand selectors: the per-matrix slot of a t x t operand (slot groups are
// `t2e` doubles apart): SEL_FIXED as given, SEL_VJ = V^j (slot j - 1), SEL_PSI =
// the slot psi ends in after the k - 1 Horner stages (6 + (k - 1) % 2).
enum LrlSel : int { SEL_FIXED = 0, SEL_VJ, SEL_PSI };
__device__ __forceinline__ int64_t lrl_sel(const LrlState& s, int sel, int64_t t2e) {
  if (sel == SEL_VJ) return (int64_t)(s.j - 1) * t2e;
  if (sel == SEL_PSI) return (int64_t)(6 + (s.k - 1) % 2) * t2e;
  return 0;
}

template <typename TA, typename TB, typename TC>
__global__ void __launch_bounds__(256) k_lrl_gemm(const TA* __restrict__ A, int64_t sa, int lda,
                                                  const TB* __restrict__ B, int64_t sb, int ldb, TC* __restrict__ C,
                                                  int64_t sc, int ldc, const double* __restrict__ Cadd, int64_t sadd,
                                                  int M, int N, int K, double d, LrlState* __restrict__ st, int gate,
                                                  int arg, uint8_t flag_bit, int a_sel, int b_sel, int64_t t2e) {
  const int b = blockIdx.z;
  const LrlState s = st[b];
  if (!lrl_gate(s, gate, arg)) return;
  __shared__ double sa_[16][65];
  __shared__ double sb_[16][65];
  const TA* Ab = A + (size_t)b * sa + lrl_sel(s, a_sel, t2e);
  const TB* Bb = B + (size_t)b * sb + lrl_sel(s, b_sel, t2e);
  TC* Cb = C + (size_t)b * sc;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int r0 = blockIdx.y * 64, c0 = blockIdx.x * 64;
  double acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += 16) {
    for (int i = threadIdx.x; i < 16 * 64; i += 256) {
      const int kk = i / 64, rr = i % 64;
      // A tile read along k for a fixed row: k fastest within a row would be
      // coalesced, but rows are short (t) for the left factors: transpose via smem
      const int ar = r0 + rr, ak = k0 + kk;
      sa_[kk][rr] = (ar < M && ak < K) ? (double)Ab[(size_t)ar * lda + ak] : 0.0;
      const int bk = k0 + kk, bc = c0 + rr;
      sb_[kk][rr] = (bk < K && bc < N) ? (double)Bb[(size_t)bk * ldb + bc] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      double a[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = sa_[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = sb_[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
  bool bad = false;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = r0 + ty + 16 * i, c = c0 + tx + 16 * j;
      if (r < M && c < N) {
        double v = acc[i][j];
        if (Cadd) v += Cadd[(size_t)b * sadd + (size_t)r * ldc + c];
        if (r == c) v += d;
        const TC o = (TC)v;
        bad |= !isfinite(o);
        Cb[(size_t)r * ldc + c] = o;
      }
    }
  if (__syncthreads_or(bad) && threadIdx.x == 0 && flag_bit) atomicOr(&st[b].flags, (int)flag_bit);
}

// Factor finiteness (LowRankPair, engine.py:179-180) -> kLrBadInput.
template <typename TI>
__global__ void __launch_bounds__(256) k_lrl_scan(const TI* __restrict__ A1, const TI* __restrict__ A2, size_t per,
                                                  LrlState* __restrict__ st) {
  const int b = blockIdx.y;
  bool bad = false;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < per; i += (size_t)gridDim.x * blockDim.x)
    bad |= !isfinite(A1[(size_t)b * per + i]) || !isfinite(A2[(size_t)b * per + i]);
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&st[b].flags, (int)kLrBadInput);
}

// ||S||_1 (S = V or V^2) and the ladder (select_lowrank, engine.py:224-244).
// pass 1: ||V||_1; pass 2: ||V^2||_1 for the matrices that asked for it.
__global__ void __launch_bounds__(256) k_lrl_select(const double* __restrict__ S, size_t slot_stride, int t,
                                                    double log_eps, int pass, LrlState* __restrict__ st) {
  const int b = blockIdx.x;
  LrlState s = st[b];
  if (s.flags) return;
  if (pass == 2 && s.rc != 1) return;
  const double* Sb = S + (size_t)b * slot_stride;
  __shared__ double red[256];
  double mx = -INFINITY;
  for (int c = threadIdx.x; c < t; c += blockDim.x) {
    double a = 0.0;
    for (int r = 0; r < t; ++r) a += fabs(Sb[(size_t)r * t + c]);
    mx = lr_nanmax(mx, a);
  }
  red[threadIdx.x] = mx;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] = lr_nanmax(red[threadIdx.x], red[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double c = red[0];
    if (!isfinite(c)) {
      s.flags |= kLrNonFinite;
    } else {
      if (pass == 1) { s.nv = c; s.nv2 = NAN; } else { s.nv2 = c; }
      int m = 0;
      double x1 = NAN, x2 = NAN;
      const int rc = select_lowrank(s.nv, pass == 2 ? s.nv2 : 0.0, pass == 2 ? 1 : 0, log_eps, &m, &x1, &x2);
      s.rc = rc;
      if (rc == 0) {
        s.m = m; s.e1 = x1; s.e2 = x2;
        s.j = m >= 2 ? ps_j_of(m) : 1;
        s.k = m >= 2 ? (m + s.j - 1) / s.j : 1;
      } else if (rc < 0) {
        s.flags |= kLrNoOrder;
      }
    }
    st[b] = s;
  }
}

// block(lo, hi) = c_lo I + sum_{t=1}^{hi-lo} c_{lo+t} V^t with c_i = 1/(i+1)!
// (poly.py:62-66, :171-176) into `dst`; stage h = -1 is the top block
// ((k-1)j .. m), stage h >= 0 the Horner block of r = k-2-h.
__global__ void __launch_bounds__(256) k_lrl_block(const double* __restrict__ slots, size_t t2e, int t, int h,
                                                   int dst_slot, LrlState* __restrict__ st) {
  const int b = blockIdx.y;
  const LrlState s = st[b];
  if (s.flags) return;
  const int j = s.j, k = s.k, m = s.m;
  int lo, hi;
  if (h < 0) {
    lo = (k - 1) * j;
    hi = m;
  } else {
    const int r = k - 2 - h;
    if (m < 2 || r < 0) return;
    lo = r * j;
    hi = r * j + j - 1;
  }
  const double* base = slots + (size_t)b * kLrlSlots * t2e;
  double* dst = const_cast<double*>(base) + (size_t)dst_slot * t2e;
  double cf[7];
#pragma unroll
  for (int q = 0; q < 7; ++q) cf[q] = q <= hi - lo ? lr_inv_fact(lo + q + 1) : 0.0;
  const size_t tt = (size_t)t * t;
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < tt; e += (size_t)gridDim.x * blockDim.x) {
    double q = (e / t == e % t) ? cf[0] : 0.0;
#pragma unroll
    for (int p = 1; p < 7; ++p)
      if (p <= hi - lo) q = fma(cf[p], base[(size_t)(p - 1) * t2e + e], q);
    dst[e] = q;
  }
}

// Per-matrix outputs; a flagged matrix's X is NaN (include/expmb.h).
__global__ void __launch_bounds__(256) k_lrl_finish(const LrlState* __restrict__ st, int cnt, int64_t base, LrOut po) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= cnt) return;
  const LrlState s = st[b];
  const int64_t gi = base + b;
  const bool ok = !(s.flags & (kLrBadInput | kLrNoOrder)) && s.rc == 0;
  if (po.m) po.m[gi] = (int8_t)(ok ? s.m : 0);
  if (po.e1) po.e1[gi] = ok ? s.e1 : NAN;
  if (po.e2) po.e2[gi] = ok ? s.e2 : NAN;
  if (po.norms) { po.norms[2 * gi] = s.nv; po.norms[2 * gi + 1] = s.nv2; }
  if (po.mults) po.mults[gi] = ok ? lr_mults(s.m) : 0;
  if (po.flags) po.flags[gi] = (uint8_t)s.flags;
}

template <typename TI>
__global__ void __launch_bounds__(256) k_lrl_nanfill(TI* __restrict__ X, size_t nn, const LrlState* __restrict__ st) {
  const int b = blockIdx.y;
  if (!st[b].flags) return;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < nn; i += (size_t)gridDim.x * blockDim.x)
    X[(size_t)b * nn + i] = (TI)NAN;
}

template <typename TI>
static int lrl_run(const TI* A1, const TI* A2, TI* X, int64_t batch, int n, int t, double eps, LrOut po,
                   unsigned char* ws, const LrlLayout& L, cudaStream_t st) {
  const double log_eps = log2(eps);
  const size_t t2e = L.t2 / 8, ye = L.yb / 8, nn = (size_t)n * n;
  const int64_t sslot = (int64_t)kLrlSlots * t2e;  // doubles between matrices' slot groups
  for (int64_t b0 = 0; b0 < batch; b0 += L.chunk) {
    const int cnt = (int)std::min<int64_t>(L.chunk, batch - b0);
    const TI* a1 = A1 + (size_t)b0 * n * t;
    const TI* a2 = A2 + (size_t)b0 * t * n;
    TI* x = X + (size_t)b0 * nn;
    double* slots = reinterpret_cast<double*>(ws + L.off_slots);
    double* Y = reinterpret_cast<double*>(ws + L.off_y);
    LrlState* stt = reinterpret_cast<LrlState*>(ws + L.off_state);
    auto slot = [&](int k) { return slots + (size_t)k * t2e; };
    if (cudaMemsetAsync(stt, 0, (size_t)cnt * sizeof(LrlState), st) != cudaSuccess) return EXPMB_ERR_CUDA;
    {
      const size_t per = (size_t)n * t;
      const int bx = (int)std::min<size_t>((per + 255) / 256, 64);
      k_lrl_scan<TI><<<dim3(bx, cnt), 256, 0, st>>>(a1, a2, per, stt);
    }
    auto tiles = [](int M, int N, int c) { return dim3((N + 63) / 64, (M + 63) / 64, c); };
    // V = A2 A1 (rect 1)
    k_lrl_gemm<TI, TI, double><<<tiles(t, t, cnt), 256, 0, st>>>(a2, (int64_t)t * n, n, a1, (int64_t)n * t, t,
                                                                  slot(0), sslot, t, nullptr, 0, t, t, n, 0.0, stt,
                                                                  LG_ALL, 0, kLrNonFinite, SEL_FIXED, SEL_FIXED, t2e);
    k_lrl_select<<<cnt, 256, 0, st>>>(slot(0), sslot, t, log_eps, 1, stt);
    // V^2 where the ladder needs it (engine.py:226-230)
    k_lrl_gemm<double, double, double><<<tiles(t, t, cnt), 256, 0, st>>>(
        slot(0), sslot, t, slot(0), sslot, t, slot(1), sslot, t, nullptr, 0, t, t, t, 0.0, stt, LG_V2, 0, kLrNonFinite,
        SEL_FIXED, SEL_FIXED, t2e);
    k_lrl_select<<<cnt, 256, 0, st>>>(slot(1), sslot, t, log_eps, 2, stt);
    // V^3 .. V^6 as j(m) asks (poly.py:167-169)
    for (int p = 3; p <= 6; ++p)
      k_lrl_gemm<double, double, double><<<tiles(t, t, cnt), 256, 0, st>>>(
          slot(p - 2), sslot, t, slot(0), sslot, t, slot(p - 1), sslot, t, nullptr, 0, t, t, t, 0.0, stt, LG_POW, p,
          kLrNonFinite, SEL_FIXED, SEL_FIXED, t2e);
    // q = block((k-1)j, m) in slot 6 (m = 0: I; m = 1: I + V/2)
    const int bx2 = (int)std::min<size_t>(((size_t)t * t + 255) / 256, 32);
    k_lrl_block<<<dim3(bx2, cnt), 256, 0, st>>>(slots, t2e, t, -1, 6, stt);
    // Horner: q <- q V^j + block(rj, rj + j - 1), r = k-2 .. 0 (poly.py:179-181);
    // q ping-pongs between slots 6 and 7, the block goes to slot 8; k <= 5 (m <= 30)
    for (int h = 0; h < 4; ++h) {
      k_lrl_block<<<dim3(bx2, cnt), 256, 0, st>>>(slots, t2e, t, h, 8, stt);
      k_lrl_gemm<double, double, double><<<tiles(t, t, cnt), 256, 0, st>>>(
          slot(6 + h % 2), sslot, t, slot(0), sslot, t, slot(6 + (h + 1) % 2), sslot, t, slot(8), sslot, t, t, t, 0.0,
          stt, LG_HORNER, h, kLrNonFinite, SEL_FIXED, SEL_VJ, t2e);
    }
    // Y = psi A2 (rect 2), X = I + A1 Y (rect 3)
    k_lrl_gemm<double, TI, double><<<tiles(t, n, cnt), 256, 0, st>>>(slots, sslot, t, a2, (int64_t)t * n, n, Y,
                                                                      (int64_t)ye, n, nullptr, 0, t, n, t, 0.0, stt,
                                                                      LG_ALL, 0, kLrNonFinite, SEL_PSI, SEL_FIXED, t2e);
    k_lrl_gemm<TI, double, TI><<<tiles(n, n, cnt), 256, 0, st>>>(a1, (int64_t)n * t, t, Y, (int64_t)ye, n, x,
                                                                  (int64_t)nn, n, nullptr, 0, n, n, t, 1.0, stt, LG_ALL,
                                                                  0, kLrNonFinite, SEL_FIXED, SEL_FIXED, t2e);
    {
      const int bx = (int)std::min<size_t>((nn + 255) / 256, 128);
      k_lrl_nanfill<TI><<<dim3(bx, cnt), 256, 0, st>>>(x, nn, stt);
    }
    k_lrl_finish<<<(cnt + 255) / 256, 256, 0, st>>>(stt, cnt, b0, po);
    if (cudaGetLastError() != cudaSuccess) return EXPMB_ERR_CUDA;
  }
  return EXPMB_OK;
}

}  // namespace expmb
