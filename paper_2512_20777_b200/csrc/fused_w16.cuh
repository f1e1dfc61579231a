// fused_w16.cuh -- the n = 16 fp32 Sastre kernel (C2), warp-batched.
//
// Same per-matrix program as fused_small.cuh's HM variant (engine.py:119-152:
// ||W||_1, W^2, ||W^2||_1, the ladder of select.py:164-220, the 2^-s rescale of
// engine.py:139-140, T2/T4/T8/T15+ of poly.py:189-230 and the squarings of
// engine.py:80-87), with the same 3xTF32 mma.sync products, so e^W is
// bit-identical for an identical plan.  What changes is the schedule.  The
// fused_small kernel ran the scalar part of every matrix -- the ladder walk,
// the e1/e2 bounds and eight plan stores -- on all 32 lanes of its warp, and
// ncu put that at 34% of the instructions (profiles/ncu_C2_w16_r02.txt).  Here a
// warp takes Q = 4 consecutive matrices at a time in three phases:
//
//   1. for each matrix: W -> registers from shared memory, W^2 on the tensor
//      cores, both column-abs-sum norms in one transpose-reduction; W^2 is
//      parked in a lane-private shared-memory slot.  Lane j keeps the norms
//      of matrix j.
//   2. lanes 0..Q-1 walk the ladder for their own matrix at once and write its
//      plan record (m, s, e1, e2, norms, mults): one selector and one set of
//      plan stores per Q matrices.
//   3. for each matrix: broadcast (m, s), reload W and W^2, evaluate, square,
//      write e^W straight from the accumulator fragments.
//
// W arrives by cp.async (16-byte LDGSTS, L1 bypassed) into a per-warp slot
// with its 16-byte chunks XOR-swizzled so that both the accumulator-layout
// reads (LDS.64) and the B-fragment reads of the W^2 product (LDS.32) are
// bank-conflict free.  Slot j of the next batch is refilled as soon as phase 3
// has read W_j, so the copy overlaps the rest of the batch; nothing is
// prefetched into registers.  Each warp owns a contiguous range of matrices.
//
// Register layout of a 16x16 state matrix (the m16n8k8 accumulator layout,
// lane = 4 g + t): v[4 nt + q] = X[g + 8 (q >> 1)][8 nt + 2 t + (q & 1)].
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "fused_small.cuh"
#include "select.cuh"

namespace expmb {
namespace w16 {

// EXPMB_W16_DYN (opt-in, A/B): one 16-warp CTA per SM owns a contiguous
// range of the batch and its warps claim matrices from a shared-memory
// cursor, up to Q at a time and fewer near the end of the range (guided
// self-scheduling).  Measured slower than the static per-warp ranges (62.2
// vs 59.3 us on C2: the short batches at the end of a range lose the
// phase-1 pairing and pay a selector pass each), so the default is 0.
#ifndef EXPMB_W16_DYN
#define EXPMB_W16_DYN 0
#endif
#ifndef EXPMB_W16_WARPS
#define EXPMB_W16_WARPS (EXPMB_W16_DYN ? 16 : 8)
#endif
constexpr int WARPS = EXPMB_W16_WARPS;   // warps per CTA
constexpr int NT = 32 * WARPS;
constexpr int LDR = 20;    // product right-operand stride: B-fragment rows 2t, 2t+1 conflict-free

template <int Q>  // matrices per warp batch
struct WarpSmem {
  float w[Q][256];   // W of the batch (swizzled chunks, see widx)
  float a2[Q][256];  // W^2 of the batch, lane-private: lane l owns floats [8 l, 8 l + 8)
  float rb[16 * LDR];
};
template <int Q>
constexpr size_t smem_bytes() { return WARPS * sizeof(WarpSmem<Q>); }

// poly.py:75-101 coefficients rounded to binary32, as the fused kernels use them
__device__ constexpr float kT8f[6] = {(float)4.980119205559973e-3, (float)1.992047682223989e-2, (float)7.665265321119147e-2,
                           (float)8.765009801785554e-1, (float)1.225521150112075e-1, (float)2.974307204847627e0};
__device__ constexpr float kT15f[16] = {
    (float)4.018761610201036e-4,  (float)2.945531440279683e-3, (float)-8.709066576837676e-3,
    (float)4.017568440673568e-1,  (float)3.230762888122312e-2, (float)5.768988513026145e0,
    (float)2.338576034271299e-2,  (float)2.381070373870987e-1, (float)2.224209172496374e0,
    (float)-5.792361707073261e0,  (float)-4.130276365929783e-2, (float)1.040801735231354e1,
    (float)-6.331712455883370e1,  (float)3.484665863364574e-1, 1.0f, 1.0f};

// element offset of W[r][c] in a slot: chunk (c >> 2) of row r stored at
// chunk position (c >> 2) ^ f(r), f(r) = (r & 2) | ((r >> 2) & 1)
__device__ __forceinline__ int widx(int r, int c) {
  return r * 16 + ((((c >> 2) ^ ((r & 2) | ((r >> 2) & 1))) & 3) << 2) + (c & 3);
}

__device__ __forceinline__ void cp_async16(float* dst, const float* src) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// stage matrix idx (if idx < end) into a slot: lane copies chunks lane, lane + 32
__device__ __forceinline__ void stage(float* slot, const float* __restrict__ W, int64_t idx, int64_t end, int lane) {
  if (idx < end) {
    const float* src = W + idx * 256;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = lane + 32 * h, r = c >> 2, q = c & 3;
      cp_async16(slot + widx(r, 4 * q), src + 16 * r + 4 * q);
    }
  }
  cp_commit();  // one group per slot refill, empty or not: keeps wait_group counts static
}

// v <- W (accumulator layout) from a swizzled slot
__device__ __forceinline__ void load_w(const float* slot, int g, int t, float (&v)[8]) {
#pragma unroll
  for (int nt = 0; nt < 2; ++nt)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const float2 x = *reinterpret_cast<const float2*>(slot + widx(g + 8 * h, 8 * nt + 2 * t));
      v[4 * nt + 2 * h] = x.x;
      v[4 * nt + 2 * h + 1] = x.y;
    }
}

// EXPMB_W16_OPAQUE: the left operand's TF32 mask comes from constant memory.
// With the literal mask ptxas forwards the unmasked register to the HMMA (the
// tensor core ignores the low 13 bits) and then needs four moves per k-step
// to line the raw values up in fragment order; an opaque mask makes the LOP3
// results themselves the fragment (ncu: 62 moves per matrix before).
#ifndef EXPMB_W16_OPAQUE
#define EXPMB_W16_OPAQUE 1
#endif
__constant__ uint32_t kTf32Mask = 0xffffe000u;
__device__ __forceinline__ void split(float x, uint32_t& hi, uint32_t& lo) {
#if EXPMB_W16_OPAQUE
  const uint32_t u = __float_as_uint(x) & kTf32Mask;
#else
  const uint32_t u = __float_as_uint(x) & 0xffffe000u;
#endif
  hi = u;
  lo = __float_as_uint(x - __uint_as_float(u));
}
__device__ __forceinline__ void split2(float x0, float x1, uint32_t& h0, uint32_t& l0, uint32_t& h1, uint32_t& l1) {
  h0 = __float_as_uint(x0) & 0xffffe000u;
  h1 = __float_as_uint(x1) & 0xffffe000u;
  const float2 lo = fsub2(make_float2(x0, x1), make_float2(__uint_as_float(h0), __uint_as_float(h1)));
  l0 = __float_as_uint(lo.x);
  l1 = __float_as_uint(lo.y);
}
__device__ __forceinline__ void hmma(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// D = L R in 3xTF32 (small terms first).  L from registers: with the k index
// permuted (k = t -> column 2t, k = t + 4 -> column 2t + 1 of each 8-column
// half) a lane's accumulator entries are its A fragment; the B fragment then
// reads rows 2t, 2t + 1 of R.  rd(k, n) returns R[k][n] from shared memory.
// EXPMB_W16_ACC: accumulator chains of the 12 HMMAs.  0: one accumulator per
// 8-column tile (chains of 6 dependent HMMAs); 1: the small (lo) terms and the
// hi*hi term in separate accumulators (chains of 4 and 2, one FADD2 pass);
// 2: one accumulator per term (chains of 2, two FADD2 passes).
#ifndef EXPMB_W16_ACC
#define EXPMB_W16_ACC 0
#endif
// EXPMB_W16_P1X2: phase 1 forms W^2 for two matrices per loop iteration
#ifndef EXPMB_W16_P1X2
#define EXPMB_W16_P1X2 1
#endif

template <class RD>
__device__ __forceinline__ void product(const float (&L)[8], RD rd, int g, int t, float (&D)[8]) {
  constexpr int NA = EXPMB_W16_ACC == 0 ? 1 : EXPMB_W16_ACC == 1 ? 2 : 3;
  float acc[NA][2][4];
#pragma unroll
  for (int a = 0; a < NA; ++a)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[a][nt][q] = 0.f;
  constexpr int A_LB = 0, A_HL = NA == 3 ? 1 : 0, A_HH = NA - 1;  // accumulator of al*bh, ah*bl, ah*bh
#pragma unroll
  for (int ks = 0; ks < 2; ++ks) {
    uint32_t ah[4], al[4];
    split(L[4 * ks + 0], ah[0], al[0]);  // (g,     col 8ks + 2t)
    split(L[4 * ks + 2], ah[1], al[1]);  // (g + 8, col 8ks + 2t)
    split(L[4 * ks + 1], ah[2], al[2]);  // (g,     col 8ks + 2t + 1)
    split(L[4 * ks + 3], ah[3], al[3]);  // (g + 8, col 8ks + 2t + 1)
    uint32_t bh[2][2], bl[2][2];
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
      split2(rd(8 * ks + 2 * t, 8 * nt + g), rd(8 * ks + 2 * t + 1, 8 * nt + g), bh[nt][0], bl[nt][0], bh[nt][1],
             bl[nt][1]);
    hmma(acc[A_LB][0], al, bh[0][0], bh[0][1]);  // small terms first
    hmma(acc[A_LB][1], al, bh[1][0], bh[1][1]);
    hmma(acc[A_HL][0], ah, bl[0][0], bl[0][1]);
    hmma(acc[A_HL][1], ah, bl[1][0], bl[1][1]);
    hmma(acc[A_HH][0], ah, bh[0][0], bh[0][1]);
    hmma(acc[A_HH][1], ah, bh[1][0], bh[1][1]);
  }
#pragma unroll
  for (int nt = 0; nt < 2; ++nt)
#pragma unroll
    for (int q = 0; q < 4; q += 2) {
      float2 r = make_float2(acc[0][nt][q], acc[0][nt][q + 1]);
#pragma unroll
      for (int a = 1; a < NA; ++a) r = fadd2(r, make_float2(acc[a][nt][q], acc[a][nt][q + 1]));
      D[4 * nt + q] = r.x;
      D[4 * nt + q + 1] = r.y;
    }
}

// R (accumulator layout) -> the padded right-operand buffer
__device__ __forceinline__ void store_rb(float* rb, const float (&v)[8], int g, int t) {
#pragma unroll
  for (int nt = 0; nt < 2; ++nt)
#pragma unroll
    for (int h = 0; h < 2; ++h)
      *reinterpret_cast<float2*>(rb + (g + 8 * h) * LDR + 8 * nt + 2 * t) =
          make_float2(v[4 * nt + 2 * h], v[4 * nt + 2 * h + 1]);
}

// D = L R with R from registers (staged through the padded buffer)
__device__ __forceinline__ void product_rr(const float (&L)[8], const float (&R)[8], float* rb, int g, int t,
                                           float (&D)[8]) {
  store_rb(rb, R, g, t);
  __syncwarp();
  product(L, [rb](int k, int n) { return rb[k * LDR + n]; }, g, t, D);
  __syncwarp();  // the buffer is rewritten by the next product
}

// Both 1-norms (max column abs-sum) of two matrices in accumulator layout, in
// one transpose-reduction over the 8 lanes sharing t: each level halves the
// partial sums a lane carries, so the 8 partials (4 columns x 2 matrices)
// finish as one full column sum per lane, then a 16-lane max.  Column sums of
// non-negative floats compare as integers; NaN (0x7fffffff) orders above Inf,
// so a NaN anywhere propagates.  nx = ||X||_1, ny = ||Y||_1 on every lane.
#ifndef EXPMB_W16_REDUX
#define EXPMB_W16_REDUX 1
#endif
__device__ __forceinline__ void norms2(const float (&x)[8], const float (&y)[8], int lane, float& nx, float& ny) {
  float c[8];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int nt = k >> 1, q = k & 1;
    c[k] = fabsf(x[4 * nt + q]) + fabsf(x[4 * nt + q + 2]);      // column 8 nt + 2t + q, rows g and g + 8
    c[k + 4] = fabsf(y[4 * nt + q]) + fabsf(y[4 * nt + q + 2]);
  }
  // lane bit 4 (g bit 2): keep X (0) or Y (1)
  const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
  float d[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float keep = b4 ? c[k + 4] : c[k], send = b4 ? c[k] : c[k + 4];
    d[k] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
  // lane bit 3 (g bit 1): keep columns 2t, 2t+1 (0) or 8+2t, 9+2t (1)
  float e[2];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const float keep = b3 ? d[k + 2] : d[k], send = b3 ? d[k] : d[k + 2];
    e[k] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
  // lane bit 2 (g bit 0): keep column 2t (0) or 2t+1 (1)
  float f;
  {
    const float keep = b2 ? e[1] : e[0], send = b2 ? e[0] : e[1];
    f = keep + __shfl_xor_sync(0xffffffffu, send, 4);
  }
#if EXPMB_W16_REDUX
  // two warp-wide integer max reductions (REDUX) instead of a 4-level
  // shuffle butterfly per half; the result is warp-uniform
  const unsigned m = __float_as_uint(f);
  nx = __uint_as_float(__reduce_max_sync(0xffffffffu, b4 ? 0u : m));
  ny = __uint_as_float(__reduce_max_sync(0xffffffffu, b4 ? m : 0u));
#else
  int m = __float_as_int(f);
#pragma unroll
  for (int off = 1; off <= 8; off <<= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, off));
  const float nv = __int_as_float(m);
  const float other = __shfl_xor_sync(0xffffffffu, nv, 16);
  nx = b4 ? other : nv;
  ny = b4 ? nv : other;
#endif
}

// pairwise elementwise helpers on an 8-entry tile (column pairs (2p, 2p+1))
#define W16_EW(expr) _Pragma("unroll") for (int p = 0; p < 4; ++p) { expr; }
#define W16_G(v) (make_float2(v[2 * p], v[2 * p + 1]))
#define W16_S(v, e)            \
  {                            \
    const float2 _e = (e);     \
    v[2 * p] = _e.x;           \
    v[2 * p + 1] = _e.y;       \
  }

__device__ __forceinline__ float2 f2(float a) { return make_float2(a, a); }

// v += c I: the diagonal entries a lane holds are v[0|1] (pair 0) and v[6|7]
// (pair 3), selected by dg = (g == 2t, g == 2t + 1).  fma(c, 1, x) == x + c and
// fma(c, 0, x) == x, so this is bit-identical to adding c I to every pair.
__device__ __forceinline__ void add_ident(float (&v)[8], float c, float2 dg) {
  float2 a = ffma2(dg, f2(c), make_float2(v[0], v[1]));
  v[0] = a.x; v[1] = a.y;
  a = ffma2(dg, f2(c), make_float2(v[6], v[7]));
  v[6] = a.x; v[7] = a.y;
}

// T8 (poly.py:204-212) or T15+ (poly.py:215-230) on B = 2^-s W, A2 = 2^-2s W^2,
// then the s squarings (engine.py:80-87); constants fold into immediates.
template <bool M8>
__device__ __forceinline__ void eval_t8_t15(const float (&B)[8], const float (&A2)[8], int s, float* rb, int g,
                                            int t, float2 dg, float (&P)[8]) {
  constexpr const float* c = M8 ? kT8f : kT15f;
  float Y0[8];
  {
    float R[8];
    W16_EW(W16_S(R, ffma2(W16_G(A2), f2(c[0]), fmul2(W16_G(B), f2(c[1])))));
    product_rr(A2, R, rb, g, t, Y0);  // y02
  }
  {
    float L[8], R[8];
    W16_EW(W16_S(L, ffma2(W16_G(B), f2(c[3]), ffma2(W16_G(A2), f2(c[2]), W16_G(Y0))));
           W16_S(R, ffma2(W16_G(A2), f2(c[4]), W16_G(Y0))));
    product_rr(L, R, rb, g, t, P);
  }
  if constexpr (M8) {  // poly.py:211
    W16_EW(W16_S(P, fadd2(ffma2(W16_G(A2), f2(0.5f), ffma2(W16_G(Y0), f2(c[5]), W16_G(P))), W16_G(B))));
    add_ident(P, 1.f, dg);
  } else {  // poly.py:222-229
    float Y1[8];
    {
      float L[8], R[8];
      W16_EW(W16_S(Y1, ffma2(W16_G(A2), f2(c[6]), ffma2(W16_G(Y0), f2(c[5]), W16_G(P))));
             W16_S(L, ffma2(W16_G(B), f2(c[8]), ffma2(W16_G(A2), f2(c[7]), W16_G(Y1))));
             W16_S(R, ffma2(W16_G(B), f2(c[10]), ffma2(W16_G(Y0), f2(c[9]), W16_G(Y1)))));
      product_rr(L, R, rb, g, t, P);
    }
    W16_EW(W16_S(P, ffma2(W16_G(B), f2(c[14]),
                          ffma2(W16_G(A2), f2(c[13]),
                                ffma2(W16_G(Y0), f2(c[12]), ffma2(W16_G(Y1), f2(c[11]), W16_G(P)))))));
    add_ident(P, c[15], dg);
#pragma unroll 1
    for (int q = 0; q < s; ++q) {  // engine.py:80-87
      float Q2[8];
      product_rr(P, P, rb, g, t, Q2);
#pragma unroll
      for (int k = 0; k < 8; ++k) P[k] = Q2[k];
    }
  }
}

template <int Q, int MINB>
__global__ void __launch_bounds__(NT, (MINB * 8 / WARPS > 0 ? MINB * 8 / WARPS : 1))
expm_w16_kernel(const float* __restrict__ W, float* __restrict__ X, int64_t batch, double log_eps, PlanOut po) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  WarpSmem<Q>& S = reinterpret_cast<WarpSmem<Q>*>(smem_raw)[warp];
#if EXPMB_W16_DYN
  // the CTA owns [clo, chi); warp w starts on [clo + w Q, +Q) and claims the
  // rest from cta_next (an offset into the range)
  __shared__ int cta_next;
  const int64_t clo = batch * blockIdx.x / gridDim.x, chi = batch * (blockIdx.x + 1) / gridDim.x;
  const int cn = (int)(chi - clo);
  if (threadIdx.x == 0) cta_next = min(cn, WARPS * Q);
  __syncthreads();
  const int64_t lo = clo + (int64_t)warp * Q;
  const int64_t hi = min(chi, lo + Q);  // end of the batch being processed / staged
  if (lo >= hi) return;
#else
  // each warp owns a contiguous range of floor/ceil(batch / warps) matrices,
  // taken Q at a time (round-robin whole batches left a tail of up to one
  // batch per warp: 7 vs 6 batches at C2's 65536 / 2368 warps)
  const int64_t nwarps = (int64_t)gridDim.x * WARPS;
  const int64_t gw = (int64_t)blockIdx.x * WARPS + warp;
  const int64_t lo = batch * gw / nwarps, hi = batch * (gw + 1) / nwarps;
  if (lo >= hi) return;
#endif
  const double rung0_thr = rung0_threshold(log_eps);
  const float2 dg = make_float2(g == 2 * t ? 1.f : 0.f, g == 2 * t + 1 ? 1.f : 0.f);
  float* lane_a2 = &S.a2[0][0] + 8 * lane;
  int64_t base = lo;

#pragma unroll
  for (int j = 0; j < Q; ++j) stage(S.w[j], W, base + j, hi, lane);
#if EXPMB_W16_DYN
  int nq = (int)(hi - base);
#endif

  while (true) {
#if EXPMB_W16_DYN
    // claim the next batch now; its matrices are staged during phase 3
    int64_t nbase;
    int nnq;
    {
      int st = 0, sz = 0;
      if (lane == 0) {
        const int rem = cn - *(volatile int*)&cta_next;
        sz = min(Q, max(1, rem / WARPS));
        st = atomicAdd(&cta_next, sz);
        sz = max(0, min(sz, cn - st));
      }
      st = __shfl_sync(0xffffffffu, st, 0);
      nnq = __shfl_sync(0xffffffffu, sz, 0);
      nbase = clo + st;
    }
    const int64_t nhi = nbase + nnq;
#else
    const int64_t nbase = base + Q;
    const int nq = (int)min((int64_t)Q, hi - base);  // matrices in this batch (warp-uniform)
    const int64_t nhi = hi;
#endif
    // ---- phase 1: W^2 and both norms per matrix --------------------------------
    // (slot j's copy was issued while the previous batch's matrix j finished;
    // by now every one has landed, so one wait for all of them)
    cp_wait<0>();
    __syncwarp();
    float my_n1 = 0.f, my_n2 = 0.f;
    auto finish1 = [&](int j, const float (&w)[8], const float (&a)[8]) {
      float nx, ny;
      norms2(w, a, lane, nx, ny);
      if (lane == j) {
        my_n1 = nx;
        my_n2 = ny;
      }
      *reinterpret_cast<float4*>(lane_a2 + 256 * j) = make_float4(a[0], a[1], a[2], a[3]);
      *reinterpret_cast<float4*>(lane_a2 + 256 * j + 4) = make_float4(a[4], a[5], a[6], a[7]);
    };
#if EXPMB_W16_P1X2 == 4
    if (nq == 4) {  // four independent W^2 chains
      float w[4][8], a[4][8];
#pragma unroll
      for (int j = 0; j < 4; ++j) load_w(S.w[j], g, t, w[j]);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float* sj = S.w[j];
        product(w[j], [sj](int k, int n) { return sj[widx(k, n)]; }, g, t, a[j]);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) finish1(j, w[j], a[j]);
    }
#pragma unroll 1
    for (int j = (nq == 4 ? 4 : 0); j < nq; ++j) {
#elif EXPMB_W16_P1X2
    // two matrices per iteration: independent HMMA / shuffle chains interleave
#pragma unroll 1
    for (int j = 0; j + 1 < nq; j += 2) {
      const float* s0 = S.w[j];
      const float* s1 = S.w[j + 1];
      float w0[8], w1[8], a0[8], a1[8];
      load_w(s0, g, t, w0);
      load_w(s1, g, t, w1);
      product(w0, [s0](int k, int n) { return s0[widx(k, n)]; }, g, t, a0);  // W^2 (select.py:192)
      product(w1, [s1](int k, int n) { return s1[widx(k, n)]; }, g, t, a1);
      finish1(j, w0, a0);
      finish1(j + 1, w1, a1);
    }
    if (nq & 1) {
      const int j = nq - 1;
#else
#pragma unroll 1
    for (int j = 0; j < nq; ++j) {
#endif
      const float* slot = S.w[j];
      float w[8], a[8];
      load_w(slot, g, t, w);
      product(w, [slot](int k, int n) { return slot[widx(k, n)]; }, g, t, a);  // W^2 (select.py:192)
      finish1(j, w, a);
    }

    // ---- phase 2: lane j selects for matrix j (select.py:164-220) ---------------
    int packed = 0;  // m << 8 | s
    bool my_bad = false;
    if (lane < nq) {
      const int64_t idx = base + lane;
      const double n1 = (double)my_n1;
      double n2 = (double)my_n2;
      // the common case stays in registers (select_sastre_bf inlines); the
      // rung-0 check and the exact walk (rare) write a separate plan
      Plan pf{0, 0, 0.0, 0.0};
      int fast = 1;
      if (n1 == 0.0) {
        n2 = NAN;  // zero matrix: m = s = 0 (select.py:172-173)
      } else if (n1 > rung0_thr) {
        my_bad = !(n2 < INFINITY);  // W^2 overflowed or is NaN (matrix.py:97-98)
        fast = select_sastre_bf(n1, n2, log_eps, &pf) == 0;
      } else {
        fast = 0;
      }
      if (!fast) {
        Plan px{0, 0, 0.0, 0.0};
        double lw[4];
        int need = 2;
        if (!(n1 > rung0_thr)) {  // rung 0 (m = 1) can only pass for tiny norms
          need = select_sastre_fast(n1, 0.0, 1, log_eps, &px);
          if (need < 0) {
            lw[0] = log2_or_ninf(n1);
            need = select_walk_lw(lw, 1, log_eps, 0, &px);
          }
        }
        if (need < 2) {
          n2 = NAN;  // W^2 is not part of the plan (select.py:186-188)
        } else {
          my_bad = !(n2 < INFINITY);
          if (select_sastre_fast2(n1, n2, log_eps, &px) < 0) {
            lw[0] = log2_or_ninf(n1);
            lw[1] = log2_or_ninf(n2);
            select_walk_lw(lw, 2, log_eps, 0, &px);
          }
        }
        pf = px;
      }
      my_bad |= !(n1 < INFINITY);
      const int m = pf.m, sc = pf.s;
      packed = (m << 8) | sc;
      if (po.m) po.m[idx] = (int8_t)m;
      if (po.s) po.s[idx] = (int8_t)sc;
      if (po.e1) po.e1[idx] = pf.e1;
      if (po.e2) po.e2[idx] = pf.e2;
      if (po.norms) {
        po.norms[2 * idx] = n1;
        po.norms[2 * idx + 1] = n2;
      }
      // sastre_budget (poly.py:233-241) + s
      if (po.mults) po.mults[idx] = (m >= 2) + (m >= 4) + (m >= 8) + (m >= 15) + sc;
    }

    // ---- phase 3: evaluate and square ------------------------------------------
#pragma unroll 1
    for (int j = 0; j < Q; ++j) {
      const int64_t idx = base + j;
      const int pk = __shfl_sync(0xffffffffu, packed, j);
      float B[8];
      if (j < nq && !po.plan_only) load_w(S.w[j], g, t, B);
      __syncwarp();  // every lane has read slot j: refill it with the next batch's matrix j
      stage(S.w[j], W, nbase + j, nhi, lane);
      if (j >= nq || po.plan_only) continue;
      const int m = pk >> 8, s = pk & 0xff;
      float P[8];
      if (m <= 1) {  // zero matrix: I (engine.py:141-142); m = 1: W + I (poly.py:192)
        const float keep = m == 1 ? 1.f : 0.f;
        W16_EW(W16_S(P, fmul2(W16_G(B), f2(keep))));
        add_ident(P, 1.f, dg);
      } else {
        float A2[8];
        {
          const float4 x0 = *reinterpret_cast<const float4*>(lane_a2 + 256 * j);
          const float4 x1 = *reinterpret_cast<const float4*>(lane_a2 + 256 * j + 4);
          A2[0] = x0.x; A2[1] = x0.y; A2[2] = x0.z; A2[3] = x0.w;
          A2[4] = x1.x; A2[5] = x1.y; A2[6] = x1.z; A2[7] = x1.w;
        }
        if (s > 0) {  // exact 2^-s rescale (engine.py:139-140)
          const float sc = pow2_neg<float>(s), sc2 = pow2_neg<float>(2 * s);
          W16_EW(W16_S(B, fmul2(W16_G(B), f2(sc))); W16_S(A2, fmul2(W16_G(A2), f2(sc2))));
        }
        if (m == 2) {  // poly.py:196
          W16_EW(W16_S(P, ffma2(W16_G(A2), f2(0.5f), W16_G(B))));
          add_ident(P, 1.f, dg);
        } else if (m == 4) {  // poly.py:198-199
          float L[8];
          W16_EW(W16_S(L, fmul2(ffma2(W16_G(A2), f2(0.25f), W16_G(B)), f2(1.0f / 3.0f))));
          add_ident(L, 1.f, dg);
          product_rr(L, A2, S.rb, g, t, P);
          W16_EW(W16_S(P, ffma2(W16_G(P), f2(0.5f), W16_G(B))));
          add_ident(P, 1.f, dg);
        } else if (m == 8) {
          eval_t8_t15<true>(B, A2, s, S.rb, g, t, dg, P);
        } else {
          eval_t8_t15<false>(B, A2, s, S.rb, g, t, dg, P);
        }
      }
      {  // x * 0 is NaN exactly when x is Inf/NaN
        float2 z = make_float2(0.f, 0.f);
        W16_EW(z = ffma2(W16_G(P), f2(0.f), z));
        const bool bad = __any_sync(0xffffffffu, !(z.x == 0.f && z.y == 0.f));
        if (lane == j) my_bad |= bad;
      }
      float* dst = X + idx * 256;
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int h = 0; h < 2; ++h)
          __stcs(reinterpret_cast<float2*>(dst + (g + 8 * h) * 16 + 8 * nt + 2 * t),
                 make_float2(P[4 * nt + 2 * h], P[4 * nt + 2 * h + 1]));
    }
    if (po.nonfinite && lane < nq) po.nonfinite[base + lane] = (uint8_t)my_bad;
#if EXPMB_W16_DYN
    if (nnq == 0) break;
    nq = nnq;
#else
    if (nbase >= hi) break;
#endif
    base = nbase;
  }
  cp_wait<0>();
}

#undef W16_EW
#undef W16_G
#undef W16_S

}  // namespace w16
}  // namespace expmb
