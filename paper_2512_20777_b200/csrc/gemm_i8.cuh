// gemm_i8.cuh -- exact-accumulation fp32 products on the 5th-generation tensor
// cores: int8 mantissa slices with int32 accumulation (Ozaki scheme).
//
// Why: the tcgen05 tf32 path (gemm_tc.cuh) is 2.8x faster than the FFMA GEMM
// on C5, but the tensor core's fp32 accumulation truncates and the squaring
// phase amplifies that bias past the 1e-5 bar.  Integer accumulation is exact.
//
// Operands (per product P = L R of a stage, for every matrix of the bucket):
//   L[r][k] = 2^(er_r - 6) (s0 + s1/128 + s2/128^2 + s3/128^3),  |s_i| <= 64
//   R[k][c] = 2^(ec_c - 6) (t0 + t1/128 + t2/128^2 + t3/128^3)
// with er_r / ec_c the binary exponents of the row / column maxima (|x| < 2^e),
// every s_i, t_j an int8 obtained exactly (scaling by powers of two, rint,
// exact residuals); the truncation is 2^-29 of the row (column) maximum.
//   P[r][c] = 2^(er_r + ec_c - 12) sum_{L=0..3} 2^(-7L) acc_L[r][c],
//   acc_L = sum_{i+j=L} S_i T_j  (int32 on tcgen05.mma.kind::i8, exact)
// Ten slice-pair GEMMs (pairs with i + j > 3 contribute < 2^-28 of the row and
// column maxima and are dropped), the level sum as one exact 64-bit integer,
// one rounding to fp32 and the power-of-two scales.  A diagonal entry that
// exceeds its row's (column's) off-diagonal maximum is split off and applied
// in the epilogue (L R = Yl Yr + D_L Yr + Yl D_R + D_L D_R), so the squaring
// phase's dominant diagonal does not set the row scale.  Limitation: the
// scale is per row / column, so entries far below their row's maximum keep
// fewer bits than in fp32 -- on graded matrices (entries ~2^20 apart within a
// row) the error is 30x the FFMA path's (tools/i8_graded_probe.py).  Hence
// every product is routed per matrix (k_i8_route): only operands whose rows
// and columns are "flat" run here, the rest on the FFMA GEMM.  Default for
// fp32 n >= 320, n % 16 == 0 (large.cuh: use_i8_path).
//
// Kernels: k_i8_prep (scales, diagonal decision, routing statistics and the
// four int8 slices of each operand, K-major, in one streaming pass per
// operand), k_i8_route (the flatness test), k_i8_stage (persistent: a TMA
// 64B-swizzled 3-stage ring of 4 L + 4 R slices per 64-byte k-tile, one
// thread issuing the concatenated-slice MMAs into four int32 TMEM level
// accumulators, eight epilogue warps draining them and applying the stage's
// fused linear combination as gemm_simt.cuh's epilogue does, overlapped with
// the next unit's MMAs); k_i8_stage_np is the one-unit-per-CTA form
// (EXPMB_I8_PERSIST=0), optionally as 2-CTA clusters sharing the L panel by
// TMA multicast.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "gemm_simt.cuh"
#include "gemm_tc.cuh"

namespace expmb {
namespace i8 {

// k-tiles of 64 bytes with the 64B swizzle (TMA of the next k-tile overlaps
// this one's MMAs).
#ifndef EXPMB_I8_BK64
#define EXPMB_I8_BK64 1
#endif
// EXPMB_I8_BN: columns per tile.  64: a stage (4 L + 4 R slices) is 48 KB,
// two stages per CTA, two CTAs per SM (256 TMEM columns each; one CTA's
// epilogue overlaps the other's MMAs).  128 (default): one CTA per SM owning
// all 512 TMEM columns (four 128-column level accumulators), 64 KB stages in
// a three-stage ring, a third less operand traffic per MAC (L2 -> smem and
// smem -> tensor core), and eight epilogue warps because the epilogue now
// runs with the MMAs idle.  C5: 259 ms (BN 64) -> 238 ms per step, same bits.
#ifndef EXPMB_I8_BN
#define EXPMB_I8_BN 128
#endif
#ifndef EXPMB_I8_CW
#define EXPMB_I8_CW 16
#endif
#ifndef EXPMB_I8_STAGES
#define EXPMB_I8_STAGES (EXPMB_I8_BK64 ? (EXPMB_I8_BN == 128 ? 3 : 2) : 1)
#endif
// EXPMB_I8_CAT: slice i of L against the R slices 0..3-i stacked along N in
// one MMA (4 MMAs per 32-byte k-step); 0: the ten slice-pair MMAs
#ifndef EXPMB_I8_CAT
#define EXPMB_I8_CAT 1
#endif
constexpr int BM = 128, BN = EXPMB_I8_BN, BKB = EXPMB_I8_BK64 ? 64 : 128, STAGES = EXPMB_I8_STAGES, NSL = 4;
constexpr bool kSw64 = BKB == 64;
// UMMA shared-memory descriptor, K-major: 64B swizzle (8-row atoms of 512 B) or 128B (1024 B)
__device__ __forceinline__ uint64_t kdesc(uint32_t saddr) {
  if constexpr (!kSw64) {
    return tc::kmajor_desc(saddr);
  } else {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3fff);
    d |= (uint64_t)(16 >> 4) << 16;   // LBO (unused for swizzled K-major)
    d |= (uint64_t)(512 >> 4) << 32;  // SBO: next 8-row group
    d |= (uint64_t)1 << 46;           // descriptor version (sm100)
    d |= (uint64_t)4 << 61;           // SWIZZLE_64B
    return d;
  }
}
constexpr int A_TILE = BM * BKB;                     // 8 KB (64B swizzle)
constexpr int B_TILE = BN * BKB;                     // 4 KB (BN 64)
constexpr int STAGE_BYTES = NSL * (A_TILE + B_TILE);  // 48 KB (BN 64), 64 KB (BN 128)
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024;
// one-unit-per-CTA stage (k_i8_stage_np): EXPMB_I8_EPI_WARPS epilogue warps,
// 4 or 8; with 8, warps w and w + 4 share a TMEM lane quarter and split the
// tile's columns (the BN = 128 form runs its epilogue with the MMAs idle)
#ifndef EXPMB_I8_EPI_WARPS
#define EXPMB_I8_EPI_WARPS (EXPMB_I8_BN == 128 ? 8 : 4)
#endif
constexpr int EPI_PARTS = EXPMB_I8_EPI_WARPS / 4;
constexpr int NTHREADS_NP = 64 + 32 * EXPMB_I8_EPI_WARPS;
static_assert(EPI_PARTS == 1 || EPI_PARTS == 2, "EXPMB_I8_EPI_WARPS is 4 or 8");
constexpr uint32_t TMEM_COLS = 4 * BN;                // one int32 accumulator per level
constexpr int kNanExp = -100000;                      // row/column holds NaN/Inf
// kind::i8: D s32 (2), A s8 (1), B s8 (1), K-major both, N = 64, M = 128
static_assert(BN == 64 || BN == 128, "EXPMB_I8_BN is 64 or 128");
constexpr uint32_t kIdesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                            ((uint32_t)(BM >> 4) << 24);

struct Bufs {
  int8_t* as;  // [slot][4][n][np]  L slices, row-major (K contiguous)
  int8_t* bs;  // [slot][4][n][np]  R slices, transposed (K contiguous)
  int* er;     // [slot][n]
  int* ec;     // [slot][n]
  unsigned long long* rc;  // [slot][n] per row of L: (sum of biased exponents) << 20 | nonzero count
  unsigned long long* cc;  // [slot][n] per column of R: the same
  int* ok;     // [slot] 1 = this path handles the product (see k_i8_route)
  int np;      // padded row length (multiple of 16 bytes, TMA stride rule)
};

__device__ __forceinline__ int exp_of(float mx) {
  if (!(mx < INFINITY)) return kNanExp;  // Inf or NaN
  if (mx == 0.f) return 0;
  return ilogbf(mx) + 1;  // mx = f 2^e with f in [0.5, 1)
}

__device__ __forceinline__ void slice4(float x, int e, int8_t (&s)[4]) {
  if (e == kNanExp) {
    s[0] = s[1] = s[2] = s[3] = 0;
    return;
  }
  float y = scalbnf(x, 6 - e);  // |y| < 64, exact
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float q = rintf(y);
    s[i] = (int8_t)(int)q;
    y = (y - q) * 128.f;  // exact: |y - q| <= 1/2
  }
}

// The same four digits for four elements at once, as the four plane words
// (element u in byte u), in about a third of the instructions: the scale is a
// precomputed power of two (slice_scale), each rint is a magic-number add
// whose low mantissa byte is the digit (1.5 2^(23 - 7i) puts the mantissa's
// last place at 2^(-7i), round-to-nearest-even like rintf), and the residual
// stays unscaled.  The digits are those of slice4 (checked element by
// element on the host over six exponent ranges and the rounding ties).
__device__ __forceinline__ bool slice_scale(int e, float& sc) {  // false: use slice4 (NaN/Inf row, extreme exponent)
  sc = 0.f;
  if (e == kNanExp || e < -100 || e > 100) return false;
  sc = __int_as_float((6 - e + 127) << 23);  // 2^(6 - e)
  return true;
}
__device__ __forceinline__ void slice4x4(const float (&x)[4], float sc, uint32_t (&w)[4]) {
  float y[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) y[u] = x[u] * sc;  // |y| < 64, exact
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float M = i == 0 ? 12582912.f : i == 1 ? 98304.f : i == 2 ? 768.f : 6.f;
    uint32_t t[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const float tu = y[u] + M;
      t[u] = __float_as_uint(tu);
      y[u] -= tu - M;  // exact
    }
    w[i] = __byte_perm(__byte_perm(t[0], t[1], 0x0040), __byte_perm(t[2], t[3], 0x0040), 0x5410);
  }
}
// four elements -> plane words, by whichever path the row / column scale allows
__device__ __forceinline__ void slice_quad(const float (&x)[4], int e, bool fast, float sc, uint32_t (&w)[4]) {
  if (fast) {
    slice4x4(x, sc, w);
  } else {
    int8_t sl[4][4];
#pragma unroll
    for (int u = 0; u < 4; ++u) slice4(x[u], e, sl[u]);
#pragma unroll
    for (int j = 0; j < 4; ++j)
      w[j] = (uint32_t)(uint8_t)sl[0][j] | ((uint32_t)(uint8_t)sl[1][j] << 8) | ((uint32_t)(uint8_t)sl[2][j] << 16) |
             ((uint32_t)(uint8_t)sl[3][j] << 24);
  }
}

// Row maxima of |L| and column maxima of |R| are kept as the bit patterns of
// non-negative floats, which order like the values (NaN above Inf); for the
// routing test, the sum of the binary exponents and the count of the nonzero
// entries of every row / column travel packed in one 64-bit integer.
//
// The diagonal.  In the squaring phase X = I + (small), so a diagonal entry
// would set its row's (column's) scale and cost the off-diagonal entries
// their low bits; such a diagonal entry is SPLIT off (sliced as zero) and
// applied in the stage's epilogue: L R = Yl Yr + D_L Yr + Yl D_R + D_L D_R.
// Where the diagonal entry is no larger than the largest off-diagonal entry
// of its row of L (column of R) it is KEPT in the slices (the scale, and with
// it the routing test, is unchanged) and that row's D_L (column's D_R) is
// zero: a unit whose rows and columns all keep their diagonal skips the
// epilogue's two operand tiles.  The choice is per row / column and recorded
// in the sign bit of er / ec.
constexpr int kDiagKept = (int)0x80000000;
__device__ __forceinline__ int scale_bits(int v) { return v & 0x7fffffff; }
__device__ __forceinline__ bool diag_kept(int v) { return v < 0; }
// keep the diagonal entry (|d| as bits) of a row / column whose largest
// off-diagonal magnitude is moff (bits)?  Finite, nonzero off-diagonal mass only.
__device__ __forceinline__ bool keep_diag(int dbits, int moff) {
  return moff > 0 && moff < 0x7f800000 && dbits <= moff;  // (non-negative floats order like their bits)
}
constexpr int kExpBias = 200;
// The packed statistic of a set of entries is sum over its finite nonzero
// members of ((ilogb + kExpBias) << 20 | 1).  It is gathered in two 32-bit
// accumulators: esum collects the biased exponents (ilogb + 127), cnt the
// number of such entries; exp_pack_sum packs them.
__device__ __forceinline__ void exp_acc(float v, int& esum, int& cnt) {  // v >= 0 or NaN
  const uint32_t bits = __float_as_uint(v);
  const uint32_t e8 = bits >> 23;
  if (e8 - 1u < 254u) {  // normal, finite
    esum += (int)e8;
    ++cnt;
  } else if (e8 == 0u && bits != 0u) {  // subnormal: ilogb = 31 - clz - 149
    esum += 31 - __clz(bits) - 149 + 127;
    ++cnt;
  }
}
__device__ __forceinline__ unsigned long long exp_pack_sum(long long esum, long long cnt) {
  return ((unsigned long long)(esum + (long long)(kExpBias - 127) * cnt) << 20) | (unsigned long long)cnt;
}
// The operands of a slot's product (make_epi once per slot, not per tile).
struct I8Ops {
  const float* L;
  const float* R;
};
__device__ __forceinline__ bool i8_slot_ops(const GemmCtx<float>& g, int stage, const int* __restrict__ list,
                                            int slot, I8Ops& ops) {
  Epi<float> e;
  if (!make_epi(g, stage, list ? list[slot] : slot, e)) return false;
  ops.L = e.L;
  ops.R = e.R;
  return true;
}

// Route a product to this path only when every row of L and every column of
// R is "flat": its largest entry's binary exponent exceeds the mean exponent
// of its nonzero entries by at most 4, so typical entries keep >= 23 of the
// 28 slice bits (fp32 precision).  Graded operands, where a few large entries
// set the scale of many small ones, go to the FFMA GEMM; so do NaN / Inf.
constexpr int kFlatBits = 4;
__device__ __forceinline__ bool flat_ok(int maxbits, unsigned long long pk) {
  if (maxbits == 0) return true;                    // no off-diagonal mass
  if (maxbits >= 0x7f800000) return false;          // Inf / NaN
  const long long cnt = (long long)(pk & 0xfffffull);
  const long long esum = (long long)(pk >> 20) - (long long)kExpBias * cnt;
  const int emax = ilogbf(__int_as_float(maxbits));
  if (emax < -60 || emax > 60) return false;        // keeps the epilogue's fp32 power-of-two scales normal
  return cnt > 0 && (long long)emax * cnt - esum <= (long long)kFlatBits * cnt;
}
__global__ void __launch_bounds__(256) k_i8_route(GemmCtx<float> g, int stage, const int* __restrict__ list,
                                                   Bufs b, const int* __restrict__ dcount, int hcount) {
  const int cnt = dcount ? *dcount : hcount;
  for (int slot = blockIdx.x; slot < cnt; slot += gridDim.x) {
  const int z = list ? list[slot] : slot;
  Epi<float> e;
  const bool part = make_epi(g, stage, z, e);
  const int n = g.n;
  bool flat = true;
  if (part) {
    for (int i = threadIdx.x; i < n; i += 256) {
      const size_t o = (size_t)slot * n + i;
      flat &= flat_ok(scale_bits(b.er[o]), b.rc[o]) && flat_ok(scale_bits(b.ec[o]), b.cc[o]);
    }
  }
  flat = __syncthreads_and(flat);
  if (threadIdx.x == 0) b.ok[slot] = part && flat ? 1 : 0;
  }
}

// The prep pass: one streaming pass per operand.
//  - an L unit is 8 rows, one warp per row: the warp reads its row once for
//    the maximum |entry|, the diagonal decision and the exponent sums (no
//    atomics: the row is whole in one warp) and once more, from L1/L2, to cut
//    the four slices;
//  - an R unit is a 32-column strip: 8 warps stream its rows for the column
//    maxima (a shared-memory reduction), then re-read it in 32 x 32 tiles
//    and write the transposed slices.
#ifndef EXPMB_I8_PREP_MINB
#define EXPMB_I8_PREP_MINB 4
#endif
__device__ __forceinline__ void i8_prep_rows(const GemmCtx<float>& g, const float* __restrict__ L, const Bufs& b,
                                             int slot, int r) {
  const int n = g.n, lane = threadIdx.x & 31;
  const float* row = L + (size_t)r * n;
  int m = 0, esum = 0, ecnt = 0;  // off-diagonal maximum and statistics
  const int dgb = __float_as_int(fabsf(__ldg(row + r)));  // |diagonal entry| bits
#pragma unroll 4
  for (int c = 4 * lane; c < n; c += 128) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(row + c));
    const float x[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const float v = c + u == r ? 0.f : fabsf(x[u]);
      m = max(m, __float_as_int(v));
      exp_acc(v, esum, ecnt);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    esum += __shfl_xor_sync(0xffffffffu, esum, o);
    ecnt += __shfl_xor_sync(0xffffffffu, ecnt, o);
  }
  const bool keep = keep_diag(dgb, m);
  if (lane == 0) {
    b.er[(size_t)slot * n + r] = m | (keep ? kDiagKept : 0);
    b.rc[(size_t)slot * n + r] = exp_pack_sum(esum, ecnt);
  }
  const int ex = exp_of(__int_as_float(m));
  float sc;
  const bool fast = slice_scale(ex, sc);
  const size_t plane = (size_t)n * b.np;
  int8_t* as = b.as + (size_t)slot * NSL * plane + (size_t)r * b.np;
#pragma unroll 4
  for (int c = 4 * lane; c < n; c += 128) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(row + c));
    float x[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (!keep && c + u == r) x[u] = 0.f;
    uint32_t w[4];
    slice_quad(x, ex, fast, sc, w);
#pragma unroll
    for (int j = 0; j < NSL; ++j) *reinterpret_cast<uint32_t*>(as + j * plane + c) = w[j];
  }
}
__device__ __forceinline__ void i8_prep_cols(const GemmCtx<float>& g, const float* __restrict__ R, const Bufs& b,
                                             int slot, int c0) {
  __shared__ int pm[32][33];
  __shared__ unsigned long long ps[32][33];
  __shared__ int pex[32];
  __shared__ int pkeep[32];
  __shared__ float psc[32];
  __shared__ float tile[32][33];
  const int n = g.n;  // a multiple of 16 on this path: a float4 group is all in or all out
  // pass 1: thread (row phase ty = 0..31, column quad q4 = 0..7) streams float4s
  const int q4 = threadIdx.x & 7, ty = threadIdx.x >> 3;
  const int cq = c0 + 4 * q4;
  int m[4] = {0, 0, 0, 0}, esum[4] = {0, 0, 0, 0}, ecnt[4] = {0, 0, 0, 0};
  if (cq < n) {
#pragma unroll 4
    for (int k = ty; k < n; k += 32) {
      const float4 a = __ldg(reinterpret_cast<const float4*>(R + (size_t)k * n + cq));
      const float x[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float v = k == cq + u ? 0.f : fabsf(x[u]);
        m[u] = max(m[u], __float_as_int(v));
        exp_acc(v, esum[u], ecnt[u]);
      }
    }
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    pm[ty][4 * q4 + u] = m[u];
    ps[ty][4 * q4 + u] = exp_pack_sum(esum[u], ecnt[u]);
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    const int cl = threadIdx.x, c = c0 + cl;
    const int dd = c < n ? __float_as_int(fabsf(__ldg(R + (size_t)c * n + c))) : 0;  // |diagonal entry| bits
    int mm = 0;
    unsigned long long ss = 0;
    for (int w = 0; w < 32; ++w) {
      mm = max(mm, pm[w][cl]);
      ss += ps[w][cl];
    }
    const bool keep = keep_diag(dd, mm);
    if (c < n) {
      b.ec[(size_t)slot * n + c] = mm | (keep ? kDiagKept : 0);
      b.cc[(size_t)slot * n + c] = ss;
    }
    pkeep[cl] = keep ? 1 : 0;
    pex[cl] = exp_of(__int_as_float(mm));
    float sc;
    psc[cl] = slice_scale(pex[cl], sc) ? sc : 0.f;  // 0: slice4 path
  }
  __syncthreads();
  // pass 2: 32 x 32 tiles, one float4 per thread in, transposed slices out
  const size_t plane = (size_t)n * b.np;
  int8_t* bs = b.bs + (size_t)slot * NSL * plane;
  const int ci = threadIdx.x / 8, q = threadIdx.x % 8;
  auto ld = [&](int k) {  // this thread's float4 of tile row k (zero outside)
    return (cq < n && k < n) ? __ldg(reinterpret_cast<const float4*>(R + (size_t)k * n + cq))
                             : make_float4(0.f, 0.f, 0.f, 0.f);
  };
  const bool kept[4] = {pkeep[4 * q4] != 0, pkeep[4 * q4 + 1] != 0, pkeep[4 * q4 + 2] != 0, pkeep[4 * q4 + 3] != 0};
  // software pipelined in groups of four tiles: the next group's four loads
  // per thread are in flight while this group is sliced (one load in flight
  // per thread left the strip latency-bound: 4 KB per CTA per DRAM round trip)
  float4 nxt[4];
#pragma unroll
  for (int t = 0; t < 4; ++t) nxt[t] = ld(32 * t + ty);
  for (int k0 = 0; k0 < n; k0 += 128) {
    float4 cur[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) cur[t] = nxt[t];
    if (k0 + 128 < n) {
#pragma unroll
      for (int t = 0; t < 4; ++t) nxt[t] = ld(k0 + 128 + 32 * t + ty);
    }
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int kt = k0 + 32 * t;
      if (kt >= n) break;  // uniform
      {
        const int k = kt + ty;
        const float x[4] = {cur[t].x, cur[t].y, cur[t].z, cur[t].w};
#pragma unroll
        for (int u = 0; u < 4; ++u) tile[ty][4 * q4 + u] = (k == cq + u && !kept[u]) ? 0.f : x[u];
      }
      __syncthreads();
      const int cc = c0 + ci, k = kt + 4 * q;
      if (cc < n && k < n) {
        const float x[4] = {tile[4 * q][ci], tile[4 * q + 1][ci], tile[4 * q + 2][ci], tile[4 * q + 3][ci]};
        const float sc = psc[ci];
        uint32_t w[4];
        slice_quad(x, pex[ci], sc != 0.f, sc, w);
#pragma unroll
        for (int jj = 0; jj < NSL; ++jj) *reinterpret_cast<uint32_t*>(bs + jj * plane + (size_t)cc * b.np + k) = w[jj];
      }
      __syncthreads();
    }
  }
}
// Units of the first *dcount slots: per slot n / 8 row units, then n / 32 column strips.
__global__ void __launch_bounds__(256, EXPMB_I8_PREP_MINB) k_i8_prep(GemmCtx<float> g, int stage, const int* __restrict__ list, Bufs b,
                                                 const int* __restrict__ dcount, int hcount) {
  const int cnt = dcount ? *dcount : hcount;
  const int n = g.n;
  const int ru = (n + 7) / 8, cu = (n + 31) / 32, per_slot = ru + cu;
  const long long total = (long long)cnt * per_slot;
  int cur = -1;
  bool valid = false;
  I8Ops ops{};
  for (long long w = blockIdx.x; w < total; w += gridDim.x) {
    const int slot = (int)(w / per_slot), u = (int)(w - (long long)slot * per_slot);
    if (slot != cur) {
      cur = slot;
      valid = i8_slot_ops(g, stage, list, slot, ops);
    }
    if (!valid) continue;
    if (u < ru) {
      const int r = 8 * u + (threadIdx.x >> 5);
      if (r < n) i8_prep_rows(g, ops.L, b, slot, r);
    } else {
      __syncthreads();  // the column strip's shared arrays of the previous unit
      i8_prep_cols(g, ops.R, b, slot, 32 * (u - ru));
    }
  }
}

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t ad, uint64_t bd, uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(ad), "l"(bd), "r"(kIdesc), "r"(accumulate));
}

__device__ __forceinline__ void tmem_ld32i(uint32_t taddr, int (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = (int)r[j];
}

__device__ __forceinline__ void tmem_ld16i(uint32_t taddr, int (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int j = 0; j < 16; ++j) v[j] = (int)r[j];
}

__device__ __forceinline__ void tmem_ldw(uint32_t taddr, int (&v)[16]) { tmem_ld16i(taddr, v); }
__device__ __forceinline__ void tmem_ldw(uint32_t taddr, int (&v)[32]) { tmem_ld32i(taddr, v); }

struct Maps {
  CUtensorMap a, b;
};

// Instruction descriptors for the concatenated-slice MMAs: slice i of L times
// the R slices 0..3-i stacked along N (one operand of (4-i)*BN rows) lands in
// the level accumulators i..3, which sit side by side in TMEM.
__device__ __forceinline__ uint32_t idesc_n(int nrows) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(nrows >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}
__device__ __forceinline__ void mma_i8_d(uint32_t tmem_d, uint64_t ad, uint64_t bd, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(ad), "l"(bd), "r"(idesc), "r"(accumulate));
}
// The MMAs of one 32-byte k-step: for each L slice i, the stacked R slices
// 0..3-i in pieces of at most 256 rows (the kind::i8 N limit), piece j0 into
// the accumulators of levels i+j0 ...  first: the unit's first k-step (the
// i = 0 MMAs, issued first, initialise every level).
__device__ __forceinline__ void issue_kstep(uint32_t tmem, uint64_t ad0, uint64_t bd0, int k, bool first) {
  constexpr int PER = 256 / BN;  // R slices per MMA
#pragma unroll
  for (int i = 0; i < NSL; ++i) {
    const uint64_t a = ad0 + (uint64_t)((i * A_TILE + k * 32) >> 4);
#pragma unroll
    for (int j0 = 0; j0 < NSL - i; j0 += PER) {
      const int nr = (NSL - i - j0 < PER ? NSL - i - j0 : PER) * BN;
      const uint64_t bd = bd0 + (uint64_t)((j0 * B_TILE + k * 32) >> 4);
      mma_i8_d(tmem + (uint32_t)((i + j0) * BN), a, bd, idesc_n(nr), (first && i == 0) ? 0u : 1u);
    }
  }
}

// tcgen05.ld without the wait: issue the four level loads of a chunk, wait once
__device__ __forceinline__ void tmem_ld16_nowait(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// Persistent, warp-specialised int8-slice GEMM stage (the default).  One CTA
// per SM walks the work units (slot, 128-row block, BN-column block) of the
// first *dcount slots; warp 0 streams k-tiles through the TMA ring, warp 1
// issues the MMAs into the TMEM level accumulators, the epilogue warps drain
// them.  The four level accumulators fill all 512 TMEM columns at BN = 128,
// so there is no second accumulator set to compute into while the first is
// drained; instead the epilogue is split:
//   drain:  TMEM -> registers, the level sum as one exact 64-bit integer,
//           one rounding to fp32 and the exact power-of-two row / column
//           scales (64 values per thread), then TMEM goes back to the MMA
//           warp (~1.5 us per unit);
//   finish: the diagonal terms, the stage's fused linear combination, the
//           column-norm partials and all global traffic, overlapped with the
//           next unit's MMAs.
// The one-unit-per-CTA form (k_i8_stage_np) spent a third of each unit in its
// epilogue with the tensor pipe idle (ncu: IMMA 55% active, 14 of 40 us).
// Rounding: y0 = fl(T) 2^(er + ec - 33) is the correctly rounded product of
// the off-diagonal parts; the diagonal terms are added with two fp32 FMAs
// (k_i8_stage_np sums them in binary64 and rounds once), so results differ
// from that form in the last place.  k_i8_route keeps every row / column
// exponent within +-60, so the two scale factors and their products with
// fl(T) < 2^49 stay in the normal range whenever the result does.
__global__ void __launch_bounds__(NTHREADS_NP, (STAGE_BYTES * STAGES <= 100 * 1024 ? 2 : 1))
k_i8_stage(const __grid_constant__ Maps maps, GemmCtx<float> g, int stage, const int* __restrict__ list, Bufs bf,
           const int* __restrict__ dcount, int hcount) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ uint64_t full_bar[STAGES], empty_bar[STAGES], tfull_bar, tempty_bar;
  __shared__ uint32_t tmem_base_sh;
  constexpr int TLD = 20;        // floats per row of a warp's transpose tile (16-byte aligned rows)
  __shared__ float cf_sh[BN];    // 2^(ec - 6) per column (NaN when the column holds NaN/Inf)
  __shared__ __align__(16) float dr_sh[BN];  // diagonal of R for this unit's columns
  __shared__ float rf_sh[BM];    // 2^(er - 27) per row
  __shared__ float dl_sh[BM];    // diagonal of L for this unit's rows
  __shared__ __align__(16) float xp_sh[EXPMB_I8_EPI_WARPS][32 * TLD];  // per-warp transpose tile of a chunk
  __shared__ double red_sh[EXPMB_I8_EPI_WARPS][BN / EPI_PARTS];  // colnorm partials: one per epilogue warp and column
  // the unit's stage program, read by every epilogue thread with dynamic
  // indices: shared memory, not a per-thread local-memory copy (the ~28 KB of
  // L1 left beside the ring is swept by the epilogue's streaming loads)
  __shared__ float ec_sh[3][4], ed_sh[3];
  __shared__ float* eout_sh[3];
  __shared__ const float* ein_sh[4];
  unsigned char* sm = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int n = g.n;
  const int KT = (n + BKB - 1) / BKB;
  const int cnt = dcount ? *dcount : hcount;
  const int tn = (n + BN - 1) / BN, tm = (n + BM - 1) / BM, tiles = tn * tm;
  const int total = cnt * tiles;  // < 2^31: slots x tiles of a chunk
  if ((int)blockIdx.x >= total) return;  // uniform: no unit for this CTA

  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      tc::mbar_init(&full_bar[i], 1);
      tc::mbar_init(&empty_bar[i], 1);
    }
    tc::mbar_init(&tfull_bar, 1);
    tc::mbar_init(&tempty_bar, EXPMB_I8_EPI_WARPS);  // one arrival per epilogue warp
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     tc::smem_u32(&tmem_base_sh)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base_sh;

  // every role walks the same unit sequence and skips the same units: the
  // producer and the MMA issuer use the light test (a slot of a stage list
  // always needs its stage; the power stages run on every matrix that asked
  // for that power), the epilogue builds the full stage program (make_epi).
  // Consecutive units of a CTA's walk are gridDim.x apart, so at any time the
  // CTAs work on neighbouring tiles of one matrix (operand panels shared in L2).
  const int pw = stage == STAGE_W2 ? 2 : stage == STAGE_W3 ? 3 : stage == STAGE_W4 ? 4 : 0;
  auto unit_light = [&](int w, int& slot, int& bx, int& by) -> bool {
    slot = w / tiles;
    const int t = w - slot * tiles;
    bx = t % tn;
    by = t / tn;
    if (!bf.ok[slot]) return false;  // routed to the FFMA GEMM
    return pw == 0 || g.need[list ? list[slot] : slot] == pw;
  };
  auto unit = [&](int w, int& slot, int& z, int& bx, int& by, Epi<float>& e) -> bool {
    slot = w / tiles;
    const int t = w - slot * tiles;
    bx = t % tn;
    by = t / tn;
    if (!bf.ok[slot]) return false;  // routed to the FFMA GEMM
    z = list ? list[slot] : slot;
    return make_epi(g, stage, z, e);
  };

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer: 4 L slices + 4 R slices per k-tile ----------------
    uint32_t it = 0;
    for (int w = blockIdx.x; w < total; w += gridDim.x) {
      int slot, bx, by;
      if (!unit_light(w, slot, bx, by)) continue;
      const int m0 = by * BM, n0 = bx * BN;
      for (int kt = 0; kt < KT; ++kt, ++it) {
        const int st = it % STAGES;
        tc::mbar_wait(&empty_bar[st], ((it / STAGES) & 1) ^ 1);
        unsigned char* b = sm + st * STAGE_BYTES;
        tc::mbar_expect_tx(&full_bar[st], STAGE_BYTES);
#pragma unroll
        for (int i = 0; i < NSL; ++i) {
          tc::tma_load_3d(b + i * A_TILE, &maps.a, &full_bar[st], kt * BKB, m0, slot * NSL + i);
          tc::tma_load_3d(b + NSL * A_TILE + i * B_TILE, &maps.b, &full_bar[st], kt * BKB, n0, slot * NSL + i);
        }
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer: the concatenated-slice MMAs of every 32-byte k-step ----------------
    uint32_t it = 0, u = 0;
    for (int w = blockIdx.x; w < total; w += gridDim.x) {
      int slot, bx, by;
      if (!unit_light(w, slot, bx, by)) continue;
      tc::mbar_wait(&tempty_bar, (u & 1) ^ 1);  // the epilogue has drained the accumulators
      asm volatile("tcgen05.fence::after_thread_sync;");
      for (int kt = 0; kt < KT; ++kt, ++it) {
        const int st = it % STAGES;
        tc::mbar_wait(&full_bar[st], (it / STAGES) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t base = tc::smem_u32(sm + st * STAGE_BYTES);
        // descriptors built once per stage; slice / k-step offsets go into the
        // 16-byte-unit address field (smem < 256 KB: no carry out of it)
        const uint64_t ad0 = kdesc(base), bd0 = kdesc(base + NSL * A_TILE);
#pragma unroll
        for (int k = 0; k < BKB / 32; ++k) {
#if EXPMB_I8_CAT
          issue_kstep(tmem, ad0, bd0, k, kt == 0 && k == 0);
#else
#pragma unroll
          for (int lv = 0; lv < 4; ++lv) {
#pragma unroll
            for (int i = 0; i <= lv; ++i) {
              const int j = lv - i;
              const uint64_t a = ad0 + (uint64_t)((i * A_TILE + k * 32) >> 4);
              const uint64_t bd = bd0 + (uint64_t)((j * B_TILE + k * 32) >> 4);
              mma_i8(tmem + (uint32_t)(lv * BN), a, bd, (kt > 0 || k > 0 || i > 0) ? 1u : 0u);
            }
          }
#endif
        }
        tc::mma_commit(&empty_bar[st]);
      }
      tc::mma_commit(&tfull_bar);
      ++u;
    }
  } else if (warp >= 2) {
    // ---------------- epilogue ----------------
    constexpr int CW = 16;                  // columns per chunk
    constexpr int CPART = BN / EPI_PARTS;   // columns per epilogue warp
    constexpr int NCH = CPART / CW;
    constexpr int ETHREADS = 32 * EXPMB_I8_EPI_WARPS;
    static_assert(CPART % CW == 0 && CPART <= 64, "the drained tile part lives in registers");
    static_assert(ETHREADS >= BM && ETHREADS >= BN, "one thread per tile row / column sets up the scales");
    const int q = warp & 3;           // TMEM lane quarter of this warp
    const int hh = (warp - 2) >> 2;   // column part of this warp
    const int rl = q * 32 + lane;     // drain: this thread's row of the tile (its TMEM lane)
    const int et = threadIdx.x - 64;  // 0 .. ETHREADS - 1
    // finish: lane -> rows lr + 8 i (i = 0..3) of the warp's 32, columns 4 c4 .. 4 c4 + 3 of the chunk
    const int lr = lane >> 2, c4 = lane & 3;
    float* tile = &xp_sh[warp - 2][0];
    uint32_t u = 0;
    for (int w = blockIdx.x; w < total; w += gridDim.x) {
      int slot, z, bx, by;
      Epi<float> e;
      if (!unit(w, slot, z, bx, by, e)) continue;
      const int m0 = by * BM, n0 = bx * BN;
      asm volatile("bar.sync 1, %0;" ::"n"(ETHREADS) : "memory");  // the previous unit's readers of the scale arrays are done
      int mine = 0;  // this thread set a nonzero split diagonal entry
      if (et < BN) {
        const int c = n0 + et;
        const int ecb = (c < n) ? bf.ec[(size_t)slot * n + c] : kDiagKept;
        const int ec = exp_of(__int_as_float(scale_bits(ecb)));
        cf_sh[et] = ec == kNanExp ? NAN : scalbnf(1.f, ec - 6);
        const float dr = diag_kept(ecb) ? 0.f : e.R[(size_t)c * n + c];  // D_R: split diagonal entries only
        dr_sh[et] = dr;
        mine |= dr != 0.f;
      }
      if (et == 0) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          ed_sh[k] = e.d[k];
          eout_sh[k] = e.out[k];
#pragma unroll
          for (int qq = 0; qq < 4; ++qq) ec_sh[k][qq] = e.c[k][qq];
        }
#pragma unroll
        for (int qq = 0; qq < 4; ++qq) ein_sh[qq] = e.in[qq];
      }
      if (et < BM) {
        const int r = m0 + et;
        const int erb = (r < n) ? bf.er[(size_t)slot * n + r] : kDiagKept;
        const int er = exp_of(__int_as_float(scale_bits(erb)));
        rf_sh[et] = er == kNanExp ? NAN : scalbnf(1.f, er - 6 - 21);  // row scale / 2^21
        const float dl = diag_kept(erb) ? 0.f : e.L[(size_t)r * n + r];  // D_L: split diagonal entries only
        dl_sh[et] = dl;
        mine |= dl != 0.f;
      }
      // barrier + OR: does any row / column of this unit carry a split diagonal
      // entry?  If none does, the finish phase skips the two operand tiles.
      int need_lr;
      asm volatile(
          "{\n .reg .pred p, q;\n setp.ne.b32 q, %1, 0;\n barrier.cta.red.or.pred p, 1, %2, q;\n"
          " selp.b32 %0, 1, 0, p;\n}\n"
          : "=r"(need_lr)
          : "r"(mine), "n"(ETHREADS)
          : "memory");
      const float rf = rf_sh[rl];
      const float* const eL = e.L;
      const float* const eR = e.R;
      const float ealpha = e.alpha;
      const int enin = e.nin, enout = e.nout;
      const bool ecolnorm = e.colnorm;
      tc::mbar_wait(&tfull_bar, u & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      // ---- drain: the unit's accumulators -> y (registers), then TMEM goes back ----
      float y[CPART];
#pragma unroll
      for (int cb = 0; cb < NCH; ++cb) {
        uint32_t a0[CW], a1[CW], a2[CW], a3[CW];
        const int cl0 = hh * CPART + cb * CW;  // first column of the chunk within the tile
        const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)cl0;
        tmem_ld16_nowait(ta, a0);
        tmem_ld16_nowait(ta + BN, a1);
        tmem_ld16_nowait(ta + 2 * BN, a2);
        tmem_ld16_nowait(ta + 3 * BN, a3);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < CW; ++j) {
          // the level sum as one exact 64-bit integer (|acc| < 2^27, so < 2^49),
          // rounded once to fp32; the scales are powers of two
          const long long T = ((long long)(int)a0[j] << 21) + ((long long)(int)a1[j] << 14) +
                              ((long long)(int)a2[j] << 7) + (long long)(int)a3[j];
          y[cb * CW + j] = __ll2float_rn(T) * rf * cf_sh[cl0 + j];
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(&tempty_bar)) : "memory");
      // ---- finish: overlapped with the next unit's MMAs ----
      // L R = Yl Yr + D_L Y_R + Y_L D_R + D_L D_R with D = diagonal, Y = the rest:
      // the int8 GEMM carried Yl Yr (each row / column scaled without its
      // diagonal, which in the squaring phase dominates); the rest is
      // elementwise.  Each chunk goes through a per-warp transpose tile so that
      // a lane owns 4 consecutive columns of 4 rows: every global access is a
      // float4 and a warp instruction covers 8 rows x 64 contiguous bytes (one
      // thread per row, 16 bytes at a time, read every sector twice and the
      // evaluation stages' epilogues ran longer than their MMAs).
#pragma unroll
      for (int cb = 0; cb < NCH; ++cb) {
        const int cl0 = hh * CPART + cb * CW;
        const int c0 = n0 + cl0;
        __syncwarp();  // the previous chunk's readers of the tile are done
#pragma unroll
        for (int j = 0; j < CW; j += 4)
          *reinterpret_cast<float4*>(tile + lane * TLD + j) =
              make_float4(y[cb * CW + j], y[cb * CW + j + 1], y[cb * CW + j + 2], y[cb * CW + j + 3]);
        __syncwarp();
        const int c = c0 + 4 * c4;
        const bool colok = c < n;  // n % 16 == 0 on this path: a column quad is all in or all out
        const float4 dr4 = *reinterpret_cast<const float4*>(dr_sh + cl0 + 4 * c4);
        const float drv[4] = {dr4.x, dr4.y, dr4.z, dr4.w};
        double cs[4] = {0.0, 0.0, 0.0, 0.0};  // column abs-sums over this lane's rows
        const bool same = eR == eL;
        // two rows at a time, straight-line: every load of the pair is issued
        // before the first use (read-only loads, out-of-range rows clamped to a
        // valid address and only their stores predicated), so a chunk costs two
        // memory round trips, not one per row
#pragma unroll
        for (int ip = 0; ip < 4; ip += 2) {
          bool ok[2];
          size_t off[2];
          float4 yv4[2], lv4[2], rv4[2], xin[2][4];
          int rr[2];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int rw = lr + 8 * (ip + h);
            rr[h] = m0 + q * 32 + rw;
            ok[h] = colok && rr[h] < n;
            off[h] = ok[h] ? (size_t)rr[h] * n + c : 0;
            yv4[h] = *reinterpret_cast<const float4*>(tile + rw * TLD + 4 * c4);
            lv4[h] = need_lr ? __ldcs(reinterpret_cast<const float4*>(eL + off[h])) : make_float4(0.f, 0.f, 0.f, 0.f);
            rv4[h] = (same || !need_lr) ? lv4[h] : __ldcs(reinterpret_cast<const float4*>(eR + off[h]));
#pragma unroll
            for (int qq = 0; qq < 4; ++qq)
              xin[h][qq] = qq < enin ? __ldcs(reinterpret_cast<const float4*>(ein_sh[qq] + off[h]))
                                     : make_float4(0.f, 0.f, 0.f, 0.f);
          }
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int r = rr[h];
            const float dl = dl_sh[q * 32 + lr + 8 * (ip + h)];
            const float yv[4] = {yv4[h].x, yv4[h].y, yv4[h].z, yv4[h].w}, lv[4] = {lv4[h].x, lv4[h].y, lv4[h].z, lv4[h].w},
                        rv[4] = {rv4[h].x, rv4[h].y, rv4[h].z, rv4[h].w};
            float base[4];  // out[0]; out[k > 0] adds its own combination and identity shift to it
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              // y + D_L Yr + Yl D_R + D_L D_R at (r, c): Yr(r, r) = R(r, r) - D_R(r), Yl likewise
              const float yr = rv[j] - ((c + j == r) ? drv[j] : 0.f);
              const float v = fmaf(dl, yr, fmaf(lv[j], drv[j], yv[j]));
              base[j] = ealpha * v;
            }
#pragma unroll
            for (int k = 0; k < 3; ++k) {
              float o[4] = {base[0], base[1], base[2], base[3]};
#pragma unroll
              for (int qq = 0; qq < 4; ++qq) {
                const float cq = ec_sh[k][qq];
                const float xv[4] = {xin[h][qq].x, xin[h][qq].y, xin[h][qq].z, xin[h][qq].w};
#pragma unroll
                for (int j = 0; j < 4; ++j) o[j] = cq != 0.f ? fmaf(cq, xv[j], o[j]) : o[j];  // (0 * Inf stays out)
              }
#pragma unroll
              const float dk = ed_sh[k];
#pragma unroll
              for (int j = 0; j < 4; ++j) o[j] = (dk != 0.f && c + j == r) ? fmaf(dk, 1.f, o[j]) : o[j];
              if (ok[h] && k < enout) __stcs(reinterpret_cast<float4*>(eout_sh[k] + off[h]), make_float4(o[0], o[1], o[2], o[3]));
              if (k == 0) {
#pragma unroll
                for (int j = 0; j < 4; ++j) base[j] = o[j];
                if (ecolnorm && ok[h]) {  // (binary64 conversions: only the power stages pay for them)
#pragma unroll
                  for (int j = 0; j < 4; ++j) cs[j] += fabs((double)o[j]);
                }
              }
            }
          }
        }
        if (ecolnorm) {
          // deterministic column abs-sums of this 128-row tile (select.py:193):
          // the lane's 4 rows, then a fixed shuffle tree over the 8 lanes
          // sharing a column quad; the warps' partials meet once per unit below
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            double v = cs[j];
            v += __shfl_xor_sync(0xffffffffu, v, 4);
            v += __shfl_xor_sync(0xffffffffu, v, 8);
            v += __shfl_xor_sync(0xffffffffu, v, 16);
            if (lr == 0) red_sh[hh * 4 + q][cb * CW + 4 * c4 + j] = v;
          }
        }
      }
      if (ecolnorm) {
        // the 4 warps of this column part in lane-quarter order (one barrier
        // pair per unit: a pair per chunk kept the warps in lockstep and
        // serialised their memory round trips)
        asm volatile("bar.sync %0, 128;" ::"r"(2 + hh) : "memory");
        if (rl < CPART && n0 + hh * CPART + rl < n) {
          const double a = ((red_sh[hh * 4][rl] + red_sh[hh * 4 + 1][rl]) + red_sh[hh * 4 + 2][rl]) +
                           red_sh[hh * 4 + 3][rl];
          g.part[((size_t)z * g.tiles_m + by) * n + n0 + hh * CPART + rl] = a;
        }
        asm volatile("bar.sync %0, 128;" ::"r"(2 + hh) : "memory");
      }
      ++u;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
}

// Multicast TMA / commit helpers for the 2-CTA cluster form below.
__device__ __forceinline__ void tma_load_3d_mc(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2,
                                               uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(tc::smem_u32(dst)),
      "l"(map), "r"(tc::smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void mma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          tc::smem_u32(bar)),
      "h"(mask)
      : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// One-unit-per-CTA form of the stage (grid: column blocks x row blocks x
// slots, slots beyond the device count exit at once); A/B against the
// persistent k_i8_stage (EXPMB_I8_PERSIST).
//
// MC: launched as 2-CTA clusters along the column blocks.  The pair shares
// its 128-row L block, so each CTA loads two of the four L slices with
// .multicast::cluster into both CTAs' rings (and its own four R slices), and
// each MMA warp releases a ring stage to both producers (multicast commit;
// the empty barriers count two arrivals).  The stage was bound by the L2 ->
// SM operand stream (768 MB per 2048^2 product at 128 x 64 tiles); sharing
// the L panel cuts it to 512 MB.
template <bool MC>
__global__ void __launch_bounds__(NTHREADS_NP, (STAGE_BYTES * STAGES <= 100 * 1024 ? 2 : 1))
k_i8_stage_np(const __grid_constant__ Maps maps, GemmCtx<float> g, int stage, const int* __restrict__ list, Bufs bf,
              const int* __restrict__ dcount) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ uint64_t full_bar[STAGES], empty_bar[STAGES], tmem_bar;
  __shared__ uint32_t tmem_base_sh;
  __shared__ double cs_sh[BN];  // 2^(ec - 6) per column (NaN when the column holds NaN/Inf)
  __shared__ float dr_sh[BN];   // diagonal of R for this CTA's columns
  const int slot = blockIdx.z;
  if (dcount != nullptr && slot >= *dcount) return;  // beyond the device-resident bucket size
  if (!bf.ok[slot]) return;  // routed to the FFMA GEMM
  const int z = list ? list[slot] : slot;
  Epi<float> e;
  if (!make_epi(g, stage, z, e)) return;  // uniform per CTA

  unsigned char* sm = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int n = g.n;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int KT = (n + BKB - 1) / BKB;

  if (threadIdx.x < BN) {
    const int c = n0 + threadIdx.x;
    const int ecb = (c < n) ? bf.ec[(size_t)slot * n + c] : kDiagKept;
    const int ec = exp_of(__int_as_float(scale_bits(ecb)));
    cs_sh[threadIdx.x] = ec == kNanExp ? (double)NAN : ldexp(1.0, ec - 6);
    dr_sh[threadIdx.x] = diag_kept(ecb) ? 0.f : e.R[(size_t)c * n + c];  // D_R: split diagonal entries only
  }
  const int rank = MC ? (int)(blockIdx.x & 1) : 0;  // cluster dims (2, 1, 1): the rank is blockIdx.x % 2
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      tc::mbar_init(&full_bar[i], 1);
      tc::mbar_init(&empty_bar[i], MC ? 2 : 1);  // MC: both CTAs' MMAs release the stage
    }
    tc::mbar_init(&tmem_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     tc::smem_u32(&tmem_base_sh)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  if constexpr (MC) cluster_sync_all();  // the peer's barriers are initialised before any multicast lands
  else __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base_sh;

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer: 4 L slices + 4 R slices per k-tile ----------------
    for (int kt = 0; kt < KT; ++kt) {
      const int st = kt % STAGES;
      tc::mbar_wait(&empty_bar[st], ((kt / STAGES) & 1) ^ 1);
      unsigned char* b = sm + st * STAGE_BYTES;
      // (MC, odd column-block count: the pad CTA of the last pair has no
      // columns; it still takes its share of the L multicast, loads no R)
      const bool rvalid = !MC || n0 < n;
      tc::mbar_expect_tx(&full_bar[st], rvalid ? STAGE_BYTES : NSL * A_TILE);
#pragma unroll
      for (int i = 0; i < NSL; ++i) {
        if constexpr (MC) {
          if ((i >> 1) == rank)  // L slices 2 rank, 2 rank + 1 into both CTAs of the pair
            tma_load_3d_mc(b + i * A_TILE, &maps.a, &full_bar[st], kt * BKB, m0, slot * NSL + i, (uint16_t)3);
        } else {
          tc::tma_load_3d(b + i * A_TILE, &maps.a, &full_bar[st], kt * BKB, m0, slot * NSL + i);
        }
        if (rvalid) tc::tma_load_3d(b + NSL * A_TILE + i * B_TILE, &maps.b, &full_bar[st], kt * BKB, n0, slot * NSL + i);
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer: ten slice pairs per 32-byte k-step ----------------
    for (int kt = 0; kt < KT; ++kt) {
      const int st = kt % STAGES;
      tc::mbar_wait(&full_bar[st], (kt / STAGES) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t base = tc::smem_u32(sm + st * STAGE_BYTES);
      // descriptors built once per stage; the slice / k-step offsets go into
      // the 16-byte-unit address field (smem < 256 KB: no carry out of it)
      const uint64_t ad0 = kdesc(base), bd0 = kdesc(base + NSL * A_TILE);
#pragma unroll
      for (int k = 0; k < BKB / 32; ++k) {
        issue_kstep(tmem, ad0, bd0, k, kt == 0 && k == 0);
      }
      if constexpr (MC) mma_commit_mc(&empty_bar[st], (uint16_t)3);
      else tc::mma_commit(&empty_bar[st]);
    }
    tc::mma_commit(&tmem_bar);
  } else if (warp >= 2) {
    // ---------------- epilogue ----------------
    // 16-column chunks keep the live arrays small enough for 2 CTAs/SM
    // without spills (EXPMB_I8_CW: 32 for the one-CTA-per-SM BN = 128 form).
    constexpr int CW = EXPMB_I8_CW;
    constexpr int CPART = BN / EPI_PARTS;  // columns per epilogue warp
    static_assert(CPART % CW == 0, "chunk width");
    const int q = warp & 3;
    const int hh = (warp - 2) >> 2;  // column part of this warp
    const int rl = q * 32 + lane;
    const int r = m0 + rl;
    const bool rowok = r < n;
    // L R = Yl Yr + D_L Y_R + Y_L D_R + D_L D_R with D = diagonal, Y = the rest:
    // the int8 GEMM carries Yl Yr (each row / column scaled without its
    // diagonal, which in the squaring phase dominates), the rest is exact
    // elementwise work here, all summed in binary64 and rounded once.  The
    // operand rows of the first chunk are fetched while the MMAs still run.
    float lrow[CW], rrow[CW];
#define I8_LOAD_ROWS(C0)                                                                       \
  do {                                                                                         \
    const int c0_ = (C0);                                                                      \
    if (rowok && c0_ + CW <= n) {                                                              \
      const float4* lp = reinterpret_cast<const float4*>(e.L + (size_t)r * n + c0_);           \
      const float4* rp = reinterpret_cast<const float4*>(e.R + (size_t)r * n + c0_);           \
      _Pragma("unroll") for (int j = 0; j < CW / 4; ++j) {                                     \
        const float4 a = __ldg(lp + j);                                                        \
        lrow[4 * j] = a.x; lrow[4 * j + 1] = a.y; lrow[4 * j + 2] = a.z; lrow[4 * j + 3] = a.w; \
        const float4 bb = (e.R == e.L) ? a : __ldg(rp + j);                                    \
        rrow[4 * j] = bb.x; rrow[4 * j + 1] = bb.y; rrow[4 * j + 2] = bb.z; rrow[4 * j + 3] = bb.w; \
      }                                                                                        \
    } else {                                                                                   \
      _Pragma("unroll") for (int j = 0; j < CW; ++j) {                                         \
        const bool ok_ = rowok && c0_ + j < n;                                                 \
        lrow[j] = ok_ ? e.L[(size_t)r * n + c0_ + j] : 0.f;                                     \
        rrow[j] = ok_ ? e.R[(size_t)r * n + c0_ + j] : 0.f;                                     \
      }                                                                                        \
    }                                                                                          \
  } while (0)
    I8_LOAD_ROWS(n0 + hh * CPART);
    const int erb = rowok ? bf.er[(size_t)slot * n + r] : kDiagKept;
    const int er = exp_of(__int_as_float(scale_bits(erb)));
    const double rs21 = er == kNanExp ? (double)NAN : ldexp(1.0, er - 6 - 21);  // row scale / 2^21
    const double dl = diag_kept(erb) ? 0.0 : (double)e.L[(size_t)r * n + r];  // D_L: the split diagonal entry of this row
    tc::mbar_wait(&tmem_bar, 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    double* red = reinterpret_cast<double*>(sm) + hh * (CW * BM);  // the smem ring is idle now
#pragma unroll 1
    for (int cb = 0; cb < CPART / CW; ++cb) {
      int a0[CW], a1[CW], a2[CW], a3[CW];
      const int cl0 = hh * CPART + cb * CW;  // first column of the chunk within the tile
      const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + cl0;
      tmem_ldw(ta, a0);
      tmem_ldw(ta + BN, a1);
      tmem_ldw(ta + 2 * BN, a2);
      tmem_ldw(ta + 3 * BN, a3);
      const int c0 = n0 + cl0;
      const bool full = rowok && c0 + CW <= n;
      if (cb > 0) I8_LOAD_ROWS(c0);
      float o0[CW];
#pragma unroll
      for (int j = 0; j < CW; ++j) {
        const int c = c0 + j;
        // the level sum as one exact 64-bit integer (|acc| < 2^27, so < 2^49) and a
        // single int -> binary64 conversion (the conversion unit was the hot pipe)
        const long long T = ((long long)a0[j] << 21) + ((long long)a1[j] << 14) + ((long long)a2[j] << 7) +
                            (long long)a3[j];
        double y = (double)T * rs21 * cs_sh[cl0 + j];
        const double dr = (double)dr_sh[cl0 + j];
        // D_L Yr + Yl D_R + D_L D_R at (r, c): Yr(r, r) = R(r, r) - D_R(r), Yl likewise
        y += dl * ((double)rrow[j] - ((c == r) ? dr : 0.0)) + (double)lrow[j] * dr;
        o0[j] = e.alpha * (float)y;
      }
      for (int qq = 0; qq < e.nin; ++qq) {
        const float cq = e.c[0][qq];
        if (cq == 0.f || !rowok) continue;
        const float* ip = e.in[qq] + (size_t)r * n + c0;
        if (full) {
#pragma unroll
          for (int j = 0; j < CW; j += 4) {
            const float4 x = __ldg(reinterpret_cast<const float4*>(ip + j));
            o0[j] = fmaf(cq, x.x, o0[j]); o0[j + 1] = fmaf(cq, x.y, o0[j + 1]);
            o0[j + 2] = fmaf(cq, x.z, o0[j + 2]); o0[j + 3] = fmaf(cq, x.w, o0[j + 3]);
          }
        } else {
#pragma unroll
          for (int j = 0; j < CW; ++j)
            if (c0 + j < n) o0[j] = fmaf(cq, ip[j], o0[j]);
        }
      }
      if (e.d[0] != 0.f && r >= c0 && r < c0 + CW) {
#pragma unroll
        for (int j = 0; j < CW; ++j)
          if (c0 + j == r) o0[j] = fmaf(e.d[0], 1.f, o0[j]);
      }
      if (rowok) {
        float* op = e.out[0] + (size_t)r * n + c0;
        if (full) {
#pragma unroll
          for (int j = 0; j < CW; j += 4)
            *reinterpret_cast<float4*>(op + j) = make_float4(o0[j], o0[j + 1], o0[j + 2], o0[j + 3]);
        } else {
#pragma unroll
          for (int j = 0; j < CW; ++j)
            if (c0 + j < n) op[j] = o0[j];
        }
      }
      for (int k = 1; k < e.nout; ++k) {
        float ok[CW];
#pragma unroll
        for (int j = 0; j < CW; ++j) ok[j] = o0[j];
        for (int qq = 0; qq < e.nin; ++qq) {
          const float cq = e.c[k][qq];
          if (cq == 0.f || !rowok) continue;
          const float* ip = e.in[qq] + (size_t)r * n + c0;
          if (full) {
#pragma unroll
            for (int j = 0; j < CW; j += 4) {
              const float4 x = __ldg(reinterpret_cast<const float4*>(ip + j));
              ok[j] = fmaf(cq, x.x, ok[j]); ok[j + 1] = fmaf(cq, x.y, ok[j + 1]);
              ok[j + 2] = fmaf(cq, x.z, ok[j + 2]); ok[j + 3] = fmaf(cq, x.w, ok[j + 3]);
            }
          } else {
#pragma unroll
            for (int j = 0; j < CW; ++j)
              if (c0 + j < n) ok[j] = fmaf(cq, ip[j], ok[j]);
          }
        }
        if (e.d[k] != 0.f && r >= c0 && r < c0 + CW) {
#pragma unroll
          for (int j = 0; j < CW; ++j)
            if (c0 + j == r) ok[j] = fmaf(e.d[k], 1.f, ok[j]);
        }
        if (rowok) {
          float* op = e.out[k] + (size_t)r * n + c0;
          if (full) {
#pragma unroll
            for (int j = 0; j < CW; j += 4)
              *reinterpret_cast<float4*>(op + j) = make_float4(ok[j], ok[j + 1], ok[j + 2], ok[j + 3]);
          } else {
#pragma unroll
            for (int j = 0; j < CW; ++j)
              if (c0 + j < n) op[j] = ok[j];
          }
        }
      }
      if (e.colnorm) {
        // deterministic column abs-sums of this 128-row tile (select.py:193)
#pragma unroll
        for (int j = 0; j < CW; ++j) red[j * BM + rl] = rowok ? fabs((double)o0[j]) : 0.0;
        asm volatile("bar.sync %0, 128;" ::"r"(1 + hh) : "memory");
        if (rl < CW && c0 + rl < n) {
          double a = 0.0;
          for (int rr = 0; rr < BM; ++rr) a += red[rl * BM + rr];
          g.part[((size_t)z * g.tiles_m + blockIdx.y) * n + c0 + rl] = a;
        }
        asm volatile("bar.sync %0, 128;" ::"r"(1 + hh) : "memory");
      }
    }
#undef I8_LOAD_ROWS
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  // MC: the peer's last multicast commits target this CTA's barriers, so
  // neither CTA leaves before both are done
  if constexpr (MC) cluster_sync_all();
  else __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
}


}  // namespace i8
}  // namespace expmb
