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

#ifndef EXPMB_HM_SPLIT2
#define EXPMB_HM_SPLIT2 1  // tf32 hi/lo splits in pairs (one FADD2 per two lo parts)
#endif
#ifndef EXPMB_HM_RL
#define EXPMB_HM_RL 1  // HM products take the left operand from registers
#endif
#ifndef EXPMB_HM_ASCALAR
#define EXPMB_HM_ASCALAR 1  // A-fragment tf32 splits scalar (no pair moves; measured 80.5 -> 79.7 us on C2 with the two below)
#endif
#ifndef EXPMB_HM_NV
#define EXPMB_HM_NV 1  // HMMA asm not volatile
#endif
#ifndef EXPMB_HM_ILV
#define EXPMB_HM_ILV 1  // interleave the two column tiles' HMMA chains
#endif

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
  int plan_only;  // 1: select only (select.py:223-234) -- form the ladder's powers, write the plan, no e^W
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

// Packed fp32x2 FMA (sm_100: FFMA2, 64 FMAs per warp instruction).  The
// kernels are issue-bound, so halving the FMA instruction count is the win.
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  unsigned long long ua = *reinterpret_cast<unsigned long long*>(&a), ub = *reinterpret_cast<unsigned long long*>(&b),
                     uc = *reinterpret_cast<unsigned long long*>(&c), d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(ua), "l"(ub), "l"(uc));
  return *reinterpret_cast<float2*>(&d);
}

__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  unsigned long long ua = *reinterpret_cast<unsigned long long*>(&a), ub = *reinterpret_cast<unsigned long long*>(&b), d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(ua), "l"(ub));
  return *reinterpret_cast<float2*>(&d);
}
__device__ __forceinline__ float2 fsub2(float2 a, float2 b) {
  unsigned long long ua = *reinterpret_cast<unsigned long long*>(&a), ub = *reinterpret_cast<unsigned long long*>(&b), d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(ua), "l"(ub));
  return *reinterpret_cast<float2*>(&d);
}
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) {
  unsigned long long ua = *reinterpret_cast<unsigned long long*>(&a), ub = *reinterpret_cast<unsigned long long*>(&b), d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(ua), "l"(ub));
  return *reinterpret_cast<float2*>(&d);
}

// Column pairs of a tile row for the elementwise formula work: packed
// FFMA2/FADD2/FMUL2 for fp32 (half the instructions), two scalar ops for fp64.
template <typename T>
struct Pr {
  T x, y;
};
template <typename T>
__device__ __forceinline__ Pr<T> pfma(Pr<T> a, T c, Pr<T> b) {  // a*c + b
  if constexpr (sizeof(T) == 4) {
    const float2 r = ffma2(make_float2(a.x, a.y), make_float2(c, c), make_float2(b.x, b.y));
    return Pr<T>{r.x, r.y};
  } else {
    return Pr<T>{fma(a.x, c, b.x), fma(a.y, c, b.y)};
  }
}
template <typename T>
__device__ __forceinline__ Pr<T> padd(Pr<T> a, Pr<T> b) {
  if constexpr (sizeof(T) == 4) {
    const float2 r = fadd2(make_float2(a.x, a.y), make_float2(b.x, b.y));
    return Pr<T>{r.x, r.y};
  } else {
    return Pr<T>{a.x + b.x, a.y + b.y};
  }
}
template <typename T>
__device__ __forceinline__ Pr<T> pmul(Pr<T> a, T c) {
  if constexpr (sizeof(T) == 4) {
    const float2 r = fmul2(make_float2(a.x, a.y), make_float2(c, c));
    return Pr<T>{r.x, r.y};
  } else {
    return Pr<T>{a.x * c, a.y * c};
  }
}

__device__ __forceinline__ bool is_finite_t(float x) { return isfinite(x); }
__device__ __forceinline__ bool is_finite_t(double x) { return isfinite(x); }

// max that propagates NaN (a NaN norm must not be hidden by fmax).
__device__ __forceinline__ double nanmax(double a, double b) { return (a > b || a != a) ? a : b; }

// HM: fp32 n <= 16 products on the tensor cores with mma.sync.m16n8k8.tf32
// in 3xTF32 form (x = hi + lo, hi = x with the low 13 mantissa bits cleared,
// L R ~= Lhi Rhi + Lhi Rlo + Llo Rhi).  The FFMA2 version was bound by the
// L1/shared-memory data path (l1tex 87-90% busy: 128-bit operand loads cost 4
// wavefronts each); fragment loads are 32-bit, one wavefront, 6x fewer.
// The state tiles then use the mma accumulator layout: lane (g, t) holds rows
// {g, g+8} x columns {2t, 2t+1, 8+2t, 9+2t}.
template <typename T, int NPAD, int TM, int GROUPS, int SCHEME, bool HM = false>
struct Fused {
  static_assert(!HM || (sizeof(T) == 4 && NPAD == 16 && TM == 2), "HM is the fp32 n<=16 warp kernel");
  static constexpr int LDL = 20, LDR = 24;  // HM: A-fragment / B-fragment conflict-free strides
  static constexpr int LDR2 = 20;            // HM, register left operand: B rows 2t, 2t+1 conflict-free
  static constexpr bool HMODE = HM;
  static constexpr int TC = NPAD / 4;            // column quads
  static constexpr int TR = NPAD / TM;           // row phases
  static constexpr int TPG = TC * TR;            // threads per group
  static constexpr int NT = TPG * GROUPS;        // threads per CTA
  static constexpr int KV = Vec<T>::KV;          // k-steps per 128-bit load
  // fp32 n <= 16: unpadded rows with the 16-byte chunks XOR-swizzled by
  // (row/2)%4, so tile stores (two rows per quarter-warp) and the 8-row
  // operand loads are both conflict-free -- the padded layout made every
  // store 2-way conflicted and l1tex throughput was the C2 limiter (90%).
  static constexpr bool SWZ = (sizeof(T) == 4 && NPAD == 16 && !HM);
  static constexpr int LD = SWZ ? NPAD : NPAD + KV;  // smem row stride (elements)
  __device__ __forceinline__ static int sidx(int r, int c) {  // element offset of (row r, column c), c % 4 == 0
    if constexpr (SWZ) return r * LD + ((((c >> 2) ^ (r >> 1)) & 3) << 2);
    else return r * LD + c;
  }
  static constexpr int WARPS_PG = (TPG + 31) / 32;
  static constexpr int BUF = NPAD * (HM ? LDR : LD);  // one operand buffer (elements)
  // dynamic smem per CTA: two operand buffers per group + reduction scratch
  static constexpr size_t kSmemGroup = 2 * BUF * sizeof(T) + (WARPS_PG > 1 ? WARPS_PG * NPAD * sizeof(double) + 64 : 0);
  static_assert(BUF * sizeof(T) % 16 == 0, "operand buffers must stay 16-byte aligned");
  static constexpr size_t kSmem = GROUPS * kSmemGroup;
  static constexpr size_t kStageBytes = (size_t)NPAD * NPAD * sizeof(T);

  using Tile = T[TM][4];

  int tr, tc, g, t;
  int soff;  // shared-memory offset (elements) of this thread's first row/column in a buffer
  T* stage;  // next-matrix staging (lean variant only)
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
  // Column of register j.  fp32: 4 consecutive columns (one 16-byte vector).
  // fp64: two 16-byte pairs, one in each half of the row, so the 16 lanes of
  // a row read/write 256 contiguous bytes per instruction (a 4-column double
  // quad per lane strided the lanes 32 B apart: 2x shared-memory wavefronts).
  __device__ __forceinline__ int col(int j) const {
    if constexpr (HM) return (j < 2) ? 2 * tc + j : 8 + 2 * tc + (j - 2);
    else if constexpr (sizeof(T) == 4) return 4 * tc + j;
    else return (j >> 1) * (NPAD / 2) + 2 * tc + (j & 1);
  }

  __device__ __forceinline__ void store(T* buf, const Tile& v) const {
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      T* p = buf + (SWZ ? sidx(tr + i * TR, 4 * tc) : soff + i * TR * LD);
      if constexpr (sizeof(T) == 4) {
        *reinterpret_cast<float4*>(p) = make_float4(v[i][0], v[i][1], v[i][2], v[i][3]);
      } else {
        *reinterpret_cast<double2*>(p) = make_double2(v[i][0], v[i][1]);
        *reinterpret_cast<double2*>(p + NPAD / 2) = make_double2(v[i][2], v[i][3]);
      }
    }
  }

  // acc = L * R with L, R row-major NPAD x NPAD in shared memory.  The
  // operands of k-chunk kb+KV are loaded into registers while chunk kb is
  // multiplied (the kernel was shared-load latency bound: short_scoreboard).
  __device__ __forceinline__ void ld_chunk(const T* __restrict__ L, const T* __restrict__ R, int kb, T (&a)[TM][KV],
                                           T (&b)[KV][4]) const {
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      const T* p = L + (SWZ ? sidx(tr + i * TR, kb) : (tr + i * TR) * LD + kb);
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
      const T* q = R + (SWZ ? sidx(kb + kk, 4 * tc) : (kb + kk) * LD + (soff - tr * LD));  // row kb+kk, own columns
      if constexpr (sizeof(T) == 4) {
        float4 v = *reinterpret_cast<const float4*>(q);
        b[kk][0] = v.x; b[kk][1] = v.y; b[kk][2] = v.z; b[kk][3] = v.w;
      } else {
        double2 v0 = *reinterpret_cast<const double2*>(q);
        double2 v1 = *reinterpret_cast<const double2*>(q + NPAD / 2);
        b[kk][0] = v0.x; b[kk][1] = v0.y; b[kk][2] = v1.x; b[kk][3] = v1.y;
      }
    }
  }

  template <bool DB = true>
  __device__ __forceinline__ void mm(const T* __restrict__ L, const T* __restrict__ R, Tile& acc) const {
    if constexpr (sizeof(T) == 4 && !DB) {
      // register-lean variant (3 CTAs/SM): operands loaded right before use
      float2 acc2[TM][2];
#pragma unroll
      for (int i = 0; i < TM; ++i) acc2[i][0] = acc2[i][1] = make_float2(0.f, 0.f);
#pragma unroll(NPAD <= 16 ? NPAD / KV : 4)
      for (int kb = 0; kb < NPAD; kb += KV) {
        float a[TM][KV];
#pragma unroll
        for (int i = 0; i < TM; ++i) {
          const float4 v = *reinterpret_cast<const float4*>(L + (SWZ ? sidx(tr + i * TR, kb) : (tr + i * TR) * LD + kb));
          a[i][0] = v.x; a[i][1] = v.y; a[i][2] = v.z; a[i][3] = v.w;
        }
#pragma unroll
        for (int kk = 0; kk < KV; ++kk) {
          const float4 v = *reinterpret_cast<const float4*>(R + (SWZ ? sidx(kb + kk, 4 * tc) : (kb + kk) * LD + (soff - tr * LD)));
#pragma unroll
          for (int i = 0; i < TM; ++i) {
            const float2 ai = make_float2(a[i][kk], a[i][kk]);
            acc2[i][0] = ffma2(make_float2(v.x, v.y), ai, acc2[i][0]);
            acc2[i][1] = ffma2(make_float2(v.z, v.w), ai, acc2[i][1]);
          }
        }
      }
#pragma unroll
      for (int i = 0; i < TM; ++i) {
        acc[i][0] = acc2[i][0].x; acc[i][1] = acc2[i][0].y;
        acc[i][2] = acc2[i][1].x; acc[i][3] = acc2[i][1].y;
      }
      return;
    }
    T a[2][TM][KV], b[2][KV][4];
    ld_chunk(L, R, 0, a[0], b[0]);
    if constexpr (sizeof(T) == 4) {
      float2 acc2[TM][2];
#pragma unroll
      for (int i = 0; i < TM; ++i) acc2[i][0] = acc2[i][1] = make_float2(0.f, 0.f);
#pragma unroll(NPAD <= 16 ? NPAD / KV : 4)
      for (int kb = 0; kb < NPAD; kb += KV) {
        const int cur = (kb / KV) & 1;
        if (kb + KV < NPAD) ld_chunk(L, R, kb + KV, a[cur ^ 1], b[cur ^ 1]);
#pragma unroll
        for (int kk = 0; kk < KV; ++kk)
#pragma unroll
          for (int i = 0; i < TM; ++i) {
            const float2 ai = make_float2(a[cur][i][kk], a[cur][i][kk]);
            acc2[i][0] = ffma2(make_float2(b[cur][kk][0], b[cur][kk][1]), ai, acc2[i][0]);
            acc2[i][1] = ffma2(make_float2(b[cur][kk][2], b[cur][kk][3]), ai, acc2[i][1]);
          }
      }
#pragma unroll
      for (int i = 0; i < TM; ++i) {
        acc[i][0] = acc2[i][0].x; acc[i][1] = acc2[i][0].y;
        acc[i][2] = acc2[i][1].x; acc[i][3] = acc2[i][1].y;
      }
    } else {
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = T(0);
#pragma unroll(NPAD <= 16 ? NPAD / KV : 4)
      for (int kb = 0; kb < NPAD; kb += KV) {
        const int cur = (kb / KV) & 1;
        if (kb + KV < NPAD) ld_chunk(L, R, kb + KV, a[cur ^ 1], b[cur ^ 1]);
#pragma unroll
        for (int kk = 0; kk < KV; ++kk)
#pragma unroll
          for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[cur][i][kk], b[cur][kk][j], acc[i][j]);
      }
    }
  }

  // ---- HM (3xTF32 mma.sync) path ----
  template <int LDX>
  __device__ __forceinline__ void store_hm(T* buf, const Tile& v) const {
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      T* p = buf + (tr + 8 * i) * LDX + 2 * tc;
      *reinterpret_cast<float2*>(p) = make_float2(v[i][0], v[i][1]);
      *reinterpret_cast<float2*>(p + 8) = make_float2(v[i][2], v[i][3]);
    }
  }
  __device__ __forceinline__ static void split_tf32(float x, uint32_t& hi, uint32_t& lo) {
    const uint32_t u = __float_as_uint(x) & 0xffffe000u;
    hi = u;
    lo = __float_as_uint(x - __uint_as_float(u));
  }
  // two splits with one packed subtraction (FADD2) for the lo parts
  __device__ __forceinline__ static void split_tf32_2(float x0, float x1, uint32_t& h0, uint32_t& l0, uint32_t& h1,
                                                      uint32_t& l1) {
    h0 = __float_as_uint(x0) & 0xffffe000u;
    h1 = __float_as_uint(x1) & 0xffffe000u;
    const float2 lo = fsub2(make_float2(x0, x1), make_float2(__uint_as_float(h0), __uint_as_float(h1)));
    l0 = __float_as_uint(lo.x);
    l1 = __float_as_uint(lo.y);
  }
  __device__ __forceinline__ static void hmma(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
#if EXPMB_HM_NV
    asm(  // pure function of its operands: the compiler may schedule it
#else
    asm volatile(
#endif
        "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  }
  __device__ __forceinline__ void mm_hm(const T* __restrict__ L, const T* __restrict__ R, Tile& out) const {
    float acc[2][4];
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[nt][q] = 0.f;
    const int g8 = tr, t4 = tc;  // mma groupID / threadID_in_group
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      const int k0 = 8 * ks;
      uint32_t ah[4], al[4];
      split_tf32(L[g8 * LDL + k0 + t4], ah[0], al[0]);
      split_tf32(L[(g8 + 8) * LDL + k0 + t4], ah[1], al[1]);
      split_tf32(L[g8 * LDL + k0 + t4 + 4], ah[2], al[2]);
      split_tf32(L[(g8 + 8) * LDL + k0 + t4 + 4], ah[3], al[3]);
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        uint32_t bh0, bl0, bh1, bl1;
        split_tf32(R[(k0 + t4) * LDR + 8 * nt + g8], bh0, bl0);
        split_tf32(R[(k0 + t4 + 4) * LDR + 8 * nt + g8], bh1, bl1);
        hmma(acc[nt], al, bh0, bh1);  // small terms first
        hmma(acc[nt], ah, bl0, bl1);
        hmma(acc[nt], ah, bh0, bh1);
      }
    }
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      out[0][2 * nt] = acc[nt][0];
      out[0][2 * nt + 1] = acc[nt][1];
      out[1][2 * nt] = acc[nt][2];
      out[1][2 * nt + 1] = acc[nt][3];
    }
  }

  // HM with the left operand straight from registers: the accumulator
  // fragment a lane holds (rows g, g+8; columns 2t, 2t+1 of each 8-column
  // half) IS an A fragment once the k index is permuted (k = t -> column
  // 2t, k = t+4 -> column 2t+1 of the half); the B fragment then reads rows
  // 2t, 2t+1 of the right operand instead of t, t+4.  Saves the left
  // operand's shared-memory round trip (4 stores + 8 loads per product).
  __device__ __forceinline__ void mm_hm_rl(const Tile& Lt, const T* __restrict__ R, Tile& out) const {
    float acc[2][4];
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[nt][q] = 0.f;
    const int g8 = tr, t4 = tc;
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      uint32_t ah[4], al[4];
#if EXPMB_HM_ASCALAR
      // scalar splits: the A fragment needs four consecutive registers in the
      // order (row g, row g+8) x (k, k+4); packed (FADD2) residuals come out
      // paired along columns and cost a register move each
      split_tf32(Lt[0][2 * ks], ah[0], al[0]);
      split_tf32(Lt[1][2 * ks], ah[1], al[1]);
      split_tf32(Lt[0][2 * ks + 1], ah[2], al[2]);
      split_tf32(Lt[1][2 * ks + 1], ah[3], al[3]);
#elif EXPMB_HM_SPLIT2
      split_tf32_2(Lt[0][2 * ks], Lt[0][2 * ks + 1], ah[0], al[0], ah[2], al[2]);
      split_tf32_2(Lt[1][2 * ks], Lt[1][2 * ks + 1], ah[1], al[1], ah[3], al[3]);
#else
      split_tf32(Lt[0][2 * ks], ah[0], al[0]);
      split_tf32(Lt[1][2 * ks], ah[1], al[1]);
      split_tf32(Lt[0][2 * ks + 1], ah[2], al[2]);
      split_tf32(Lt[1][2 * ks + 1], ah[3], al[3]);
#endif
      uint32_t bh[2][2], bl[2][2];
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
#if EXPMB_HM_SPLIT2
        split_tf32_2(R[(8 * ks + 2 * t4) * LDR2 + 8 * nt + g8], R[(8 * ks + 2 * t4 + 1) * LDR2 + 8 * nt + g8],
                     bh[nt][0], bl[nt][0], bh[nt][1], bl[nt][1]);
#else
        split_tf32(R[(8 * ks + 2 * t4) * LDR2 + 8 * nt + g8], bh[nt][0], bl[nt][0]);
        split_tf32(R[(8 * ks + 2 * t4 + 1) * LDR2 + 8 * nt + g8], bh[nt][1], bl[nt][1]);
#endif
      }
#if EXPMB_HM_ILV
      // the two column tiles' chains interleaved: consecutive HMMAs are
      // independent (the 'wait' stall on the accumulator dependency)
      hmma(acc[0], al, bh[0][0], bh[0][1]);  // small terms first
      hmma(acc[1], al, bh[1][0], bh[1][1]);
      hmma(acc[0], ah, bl[0][0], bl[0][1]);
      hmma(acc[1], ah, bl[1][0], bl[1][1]);
      hmma(acc[0], ah, bh[0][0], bh[0][1]);
      hmma(acc[1], ah, bh[1][0], bh[1][1]);
#else
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        hmma(acc[nt], al, bh[nt][0], bh[nt][1]);  // small terms first
        hmma(acc[nt], ah, bl[nt][0], bl[nt][1]);
        hmma(acc[nt], ah, bh[nt][0], bh[nt][1]);
      }
#endif
    }
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      out[0][2 * nt] = acc[nt][0];
      out[0][2 * nt + 1] = acc[nt][1];
      out[1][2 * nt] = acc[nt][2];
      out[1][2 * nt + 1] = acc[nt][3];
    }
  }

  // out = L * R where L, R are register tiles (stages through smem).
  __device__ __forceinline__ void product(const Tile& Lt, const Tile& Rt, Tile& out) const {
    if constexpr (HM && EXPMB_HM_RL) {
      store_hm<LDR2>(buf1, Rt);
      sync();
      mm_hm_rl(Lt, buf1, out);
      sync();
    } else if constexpr (HM) {
      store_hm<LDL>(buf0, Lt);
      store_hm<LDR>(buf1, Rt);
      sync();
      mm_hm(buf0, buf1, out);
      sync();
    } else {
      store(buf0, Lt);
      store(buf1, Rt);
      sync();
      mm(buf0, buf1, out);
      sync();
    }
  }
  __device__ __forceinline__ void square(const Tile& Xt, Tile& out) const {
    if constexpr (HM && EXPMB_HM_RL) {
      store_hm<LDR2>(buf1, Xt);
      sync();
      mm_hm_rl(Xt, buf1, out);
      sync();
    } else if constexpr (HM) {
      store_hm<LDL>(buf0, Xt);
      store_hm<LDR>(buf1, Xt);
      sync();
      mm_hm(buf0, buf1, out);
      sync();
    } else {
      store(buf0, Xt);
      sync();
      mm(buf0, buf0, out);
      sync();
    }
  }

  // ||.||_1 of the group's matrix: column abs-sums in binary64, then max.
  // ||.||_1 of the group's matrix: column abs-sums, then max.  Sums are
  // accumulated in the working precision (fp32 sums of fp32 values carry a
  // relative error ~n u, far inside the 1e-4 log2 exemption margin; fp64
  // matches the reference's binary64 sums to rounding).
  __device__ __forceinline__ double norm1(const Tile& v) const {
    T cs[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      T a = T(0);
#pragma unroll
      for (int i = 0; i < TM; ++i) a += fabs(v[i][j]);
      cs[j] = a;
    }
    // reduce over the thread rows that share this column quad inside the warp
#pragma unroll
    for (int off = TC; off < 32 && off < TPG; off *= 2)
#pragma unroll
      for (int j = 0; j < 4; ++j) cs[j] += __shfl_xor_sync(0xffffffffu, cs[j], off);
    if constexpr (WARPS_PG == 1) {
      // max in the working precision (a double max + 64-bit shuffles was 6%
      // of the C2 kernel); NaN still propagates
      auto nmax = [](T a, T b) { return (a > b || a != a) ? a : b; };
      T mx = nmax(nmax(cs[0], cs[1]), nmax(cs[2], cs[3]));
#pragma unroll
      for (int off = 1; off < TC; off *= 2) mx = nmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
      return (double)mx;
    } else {
      const int w = t / 32, lane = t % 32;
      if (lane < TC) {  // lanes 0..TC-1 hold tr = first row phase of this warp, tc = lane
#pragma unroll
        for (int j = 0; j < 4; ++j) red[w * NPAD + col(j)] = (double)cs[j];
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
        const T* p = src + r * NPAD;
        if constexpr (HM) {
          const float2 q0 = __ldg(reinterpret_cast<const float2*>(p + col(0)));
          const float2 q1 = __ldg(reinterpret_cast<const float2*>(p + col(2)));
          v[i][0] = q0.x; v[i][1] = q0.y; v[i][2] = q1.x; v[i][3] = q1.y;
        } else if constexpr (sizeof(T) == 4) {
          float4 q = __ldg(reinterpret_cast<const float4*>(p + col(0)));
          v[i][0] = q.x; v[i][1] = q.y; v[i][2] = q.z; v[i][3] = q.w;
        } else {
          double2 q0 = __ldg(reinterpret_cast<const double2*>(p + col(0)));
          double2 q1 = __ldg(reinterpret_cast<const double2*>(p + col(2)));
          v[i][0] = q0.x; v[i][1] = q0.y; v[i][2] = q1.x; v[i][3] = q1.y;
        }
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int c = col(j);
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
        T* p = dst + r * NPAD;
        if constexpr (HM) {
          __stcs(reinterpret_cast<float2*>(p + col(0)), make_float2(v[i][0], v[i][1]));
          __stcs(reinterpret_cast<float2*>(p + col(2)), make_float2(v[i][2], v[i][3]));
        } else if constexpr (sizeof(T) == 4) {
          __stcs(reinterpret_cast<float4*>(p + col(0)), make_float4(v[i][0], v[i][1], v[i][2], v[i][3]));
        } else {
          __stcs(reinterpret_cast<double2*>(p + col(0)), make_double2(v[i][0], v[i][1]));
          __stcs(reinterpret_cast<double2*>(p + col(2)), make_double2(v[i][2], v[i][3]));
        }
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int c = col(j);
          if (r < n && c < n) dst[(size_t)r * n + c] = v[i][j];
        }
      }
    }
  }

  __device__ __forceinline__ bool is_diag(int i, int j) const { return row(i) == col(j); }

  // Next matrix of this group: static stride, or (with a work counter) the
  // next unclaimed index after the first wave -- matrices cost 0..11
  // products, so dynamic claiming removes the tail of unlucky groups.
  __device__ __forceinline__ int64_t next_index(int64_t idx, int* ctr, int64_t first_wave) const {
    if (ctr == nullptr) return idx + first_wave;
    int64_t v = 0;
    if (t == 0) v = first_wave + atomicAdd(ctr, 1);
    if constexpr (TPG == 32) {
      return __shfl_sync(0xffffffffu, v, 0);
    } else {
      int64_t* slot = reinterpret_cast<int64_t*>(red + WARPS_PG * NPAD) + 2;
      if (t == 0) *slot = v;
      sync();
      v = *slot;
      sync();
      return v;
    }
  }
};

// Steps of the per-matrix program.  Every step is "build the two operands in
// shared memory -> one product -> consume the product", so the kernel has a
// single inlined product loop (the unrolled code of five call sites thrashed
// the instruction cache: `no_instructions` was the top stall).
enum FusedStep : int {
  ST_W2 = 0,   // W^2 = W W                         (select.py:192)
  ST_W3,       // W^3 = W^2 W (PS ladder)            (select.py:192)
  ST_W4,       // W^4 = W^3 W (PS ladder)
  ST_T4,       // T4: inner * A^2                    (poly.py:198-199)
  ST_Y02,      // y02 = A^2 (c1 A^2 + c2 A)          (poly.py:209, :221)
  ST_P2,       // (y02 + c3 A^2 + c4 A)(y02 + c5 A^2) (poly.py:210, :222)
  ST_P3,       // (y12 + c8 A^2 + c9 A)(y12 + c10 y02 + c11 A)  (poly.py:224)
  ST_HORNER,   // PS: q <- q A^j (+ block)           (poly.py:179-181)
  ST_SQ,       // X <- X X                           (engine.py:80-87)
  ST_DONE
};

template <typename T, int NPAD, int TM, int GROUPS, int SCHEME, int MINB = ((NPAD == 16 && sizeof(T) == 4) ? 2 : 1),
          int VARIANT = 0>
__global__ void __launch_bounds__(Fused<T, NPAD, TM, GROUPS, SCHEME>::NT, MINB)
expm_fused_kernel(const T* __restrict__ W, T* __restrict__ X, int64_t batch, int n, double log_eps, double eps,
                  PlanOut po, int* __restrict__ ctr) {
  using F = Fused<T, NPAD, TM, GROUPS, SCHEME, (VARIANT == 2)>;
  using Tile = typename F::Tile;
  // next-matrix prefetch: registers (default), or -- in the register-lean
  // 3-CTA/SM variant -- cp.async into a per-group staging buffer
  constexpr bool kLean = (MINB >= 3);
  constexpr bool kPrefetch = !kLean && !(NPAD == 64 && sizeof(T) == 8);  // register budget
  extern __shared__ __align__(16) unsigned char smem_raw[];
  F f;
  f.g = threadIdx.x / F::TPG;
  f.t = threadIdx.x % F::TPG;
  f.tr = f.t / F::TC;
  f.tc = f.t % F::TC;
  f.soff = f.tr * F::LD + f.col(0);
  unsigned char* gbase = smem_raw + f.g * F::kSmemGroup;
  f.buf0 = reinterpret_cast<T*>(gbase);
  f.buf1 = f.buf0 + F::BUF;
  f.red = reinterpret_cast<double*>(f.buf1 + F::BUF);
  f.stage = reinterpret_cast<T*>(smem_raw + GROUPS * F::kSmemGroup + f.g * F::kStageBytes);

  const bool vec = (n == NPAD);
  const size_t nn = (size_t)n * n;
  const int64_t stride = (int64_t)gridDim.x * GROUPS;
  const double rung0_thr = rung0_threshold(log_eps);
  int64_t idx = (int64_t)blockIdx.x * GROUPS + f.g;
  if (idx >= batch) return;  // whole group exits together

#define EW(expr)                     \
  _Pragma("unroll") for (int i = 0; i < TM; ++i) \
  _Pragma("unroll") for (int j = 0; j < 4; ++j) { expr; }
#define DG(i, j) (f.is_diag(i, j) ? T(1) : T(0))
  // pairwise elementwise loops: X(i,q) is column pair q (0, 1) of row i
#define EW2(expr)                                  \
  _Pragma("unroll") for (int i = 0; i < TM; ++i)  \
  _Pragma("unroll") for (int q = 0; q < 2; ++q) { expr; }
#define GP(t) (Pr<T>{t[i][2 * q], t[i][2 * q + 1]})
#define SP(t, v)                              \
  {                                           \
    const Pr<T> _v = (v);                     \
    t[i][2 * q] = _v.x;                       \
    t[i][2 * q + 1] = _v.y;                   \
  }
#define DGP (Pr<T>{DG(i, 2 * q), DG(i, 2 * q + 1)})

  Tile B;  // W, later 2^-s W
  Tile nxt;
  f.load(W + idx * nn, n, vec, B);
  for (int64_t nidx; idx < batch; idx = nidx) {
    nidx = f.next_index(idx, ctr, stride);
    if constexpr (kPrefetch) {
      if (nidx < batch) f.load(W + nidx * nn, n, vec, nxt);
    }
    if constexpr (kLean) {
      if (vec && nidx < batch) {  // each lane stages exactly the elements it will read back
        const T* src = W + nidx * nn;
#pragma unroll
        for (int i = 0; i < TM; ++i) {
          if constexpr (F::HMODE) {  // two 8-byte column pairs per row
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int off = f.row(i) * NPAD + f.col(2 * h);
              const uint32_t d = (uint32_t)__cvta_generic_to_shared(f.stage + off);
              asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src + off) : "memory");
            }
          } else {
            const int off = f.row(i) * NPAD + f.col(0);
            const uint32_t d = (uint32_t)__cvta_generic_to_shared(f.stage + off);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src + off) : "memory");
          }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
      }
    }
    bool bad = false;
    // (a NaN/Inf input shows up in ||W||_1: the abs-sums propagate it)

    // ---- ||W||_1 and the first rung (select.py:169-188) -------------------
    double nrm[4], lw[4];
    nrm[0] = f.norm1(B);
    nrm[1] = nrm[2] = nrm[3] = NAN;
    Plan p{0, 0, 0.0, 0.0};
    Tile A2, Y0, Y1, P;  // A^2 (PS: also q), y02 (PS: A^3), y12 (PS: A^4), product
    int mults = 0;
    if constexpr (SCHEME == 2) {
      // ---- Alg. 1 term accumulation (engine.py:90-116) --------------------
      // s: smallest s >= 0 with ||W||_1 2^-s < 1/2 (engine.py:102-104)
      int s = 0;
      if (nrm[0] >= 0.5) {
        int e;
        frexp(nrm[0], &e);                // ||W||_1 = f 2^e, f in [1/2, 1)
        s = (nrm[0] <= 1e300) ? e + 1 : 1100;
      }
      const T sc = s <= 126 ? pow2_neg<T>(s) : T(0);
      EW(B[i][j] *= sc);                  // B = 2^-s W (exact)
      EW(P[i][j] = DG(i, j));             // X = I
      EW(Y0[i][j] = B[i][j]);             // Y = B
      f.store(f.buf0, B);                 // B is the left factor of every term product
      int k = 2;
      double ny = f.norm1(Y0);
      while (ny > eps && k < 400) {       // engine.py:109-112
        EW(P[i][j] += Y0[i][j]);
        f.store(f.buf1, Y0);
        f.sync();
        f.template mm<!kLean>(f.buf0, f.buf1, Y1);
        f.sync();
        const T rk = T(1) / T(k);
        EW(Y0[i][j] = Y1[i][j] * rk);     // Y = B Y / k (x/k taken as x * fl(1/k))
        ++k;
        ny = f.norm1(Y0);
      }
      for (int q = 0; q < s && q < 1100; ++q) {  // engine.py:113
        Tile Q;
        f.square(P, Q);
        EW(P[i][j] = Q[i][j]);
      }
      p.m = k - 2;
      p.s = s;
      p.e1 = ny;
      p.e2 = 0.0;
      mults = (k - 2) + s;
    } else if constexpr (SCHEME == 0 && (VARIANT == 1 || VARIANT == 2)) {
      // ---- Sastre as straight-line code per order (no step machine) ---------
      bool small = nrm[0] == 0.0;
      int need = 2;
      if (!small && !(nrm[0] > rung0_thr)) {  // rung 0 (m = 1) can only pass for tiny norms
        need = select_sastre_fast(nrm[0], 0.0, 1, log_eps, &p);
        if (need < 0) {
          lw[0] = log2_or_ninf(nrm[0]);
          need = select_walk_lw(lw, 1, log_eps, 0, &p);
        }
      }
      if (small) {
        EW(P[i][j] = DG(i, j));                         // m = 0 (engine.py:141-142)
      } else if (need < 2) {
        EW(P[i][j] = B[i][j] + DG(i, j));               // m = 1 (poly.py:192)
      } else {
        f.square(B, A2);                                // W^2 (select.py:192)
        nrm[1] = f.norm1(A2);
        bad |= !(nrm[1] < INFINITY);
        need = select_sastre_fast2(nrm[0], nrm[1], log_eps, &p);
        if (need < 0) {
          lw[0] = log2_or_ninf(nrm[0]);
          lw[1] = log2_or_ninf(nrm[1]);
          select_walk_lw(lw, 2, log_eps, 0, &p);
        }
        {
          const T sc = pow2_neg<T>(p.s), sc2 = pow2_neg<T>(2 * p.s);
          EW2(SP(B, pmul(GP(B), sc)); SP(A2, pmul(GP(A2), sc2)));
        }
        if (p.m == 2) {                                 // poly.py:196
          EW2(SP(P, padd(pfma(GP(A2), T(0.5), GP(B)), DGP)));
        } else if (p.m == 4) {                          // poly.py:198-199
          Tile L;
          EW2(SP(L, padd(pmul(pfma(GP(A2), T(0.25), GP(B)), T(1.0 / 3.0)), DGP)));
          f.product(L, A2, P);
          EW2(SP(P, padd(pfma(GP(P), T(0.5), GP(B)), DGP)));
        } else {
          const double* c = (p.m == 8) ? kT8 : kT15;
          Tile L, R;
          {
            const T c0 = (T)c[0], c1 = (T)c[1];
            EW2(SP(R, pfma(GP(A2), c0, pmul(GP(B), c1))));
          }
          f.product(A2, R, Y0);                         // y02 (poly.py:209 / :221)
          {
            const T c2 = (T)c[2], c3 = (T)c[3], c4 = (T)c[4];
            EW2(SP(L, pfma(GP(B), c3, pfma(GP(A2), c2, GP(Y0)))); SP(R, pfma(GP(A2), c4, GP(Y0))));
          }
          f.product(L, R, P);
          if (p.m == 8) {                               // poly.py:211
            const T c5 = (T)c[5];
            EW2(SP(P, padd(padd(pfma(GP(A2), T(0.5), pfma(GP(Y0), c5, GP(P))), GP(B)), DGP)));
          } else {                                      // poly.py:222-229
            {
              const T c5 = (T)c[5], c6 = (T)c[6], c7 = (T)c[7], c8 = (T)c[8], c9 = (T)c[9], c10 = (T)c[10];
              EW2(SP(Y1, pfma(GP(A2), c6, pfma(GP(Y0), c5, GP(P))));
                  SP(L, pfma(GP(B), c8, pfma(GP(A2), c7, GP(Y1))));
                  SP(R, pfma(GP(B), c10, pfma(GP(Y0), c9, GP(Y1)))));
            }
            f.product(L, R, P);
            {
              const T c11 = (T)kT15[11], c12 = (T)kT15[12], c13 = (T)kT15[13], c14 = (T)kT15[14],
                      c15 = (T)kT15[15];
              EW2(SP(P, padd(pfma(GP(B), c14, pfma(GP(A2), c13, pfma(GP(Y0), c12, pfma(GP(Y1), c11, GP(P))))),
                             pmul(DGP, c15))));
            }
            for (int q = 0; q < p.s; ++q) {             // engine.py:80-87
              f.square(P, Y1);
              EW(P[i][j] = Y1[i][j]);
            }
          }
        }
      }
      mults = budget(p.m, 0) + p.s;
    } else {
    int have = 1, step = ST_DONE, q = 0, hz = 0;
    if (nrm[0] != 0.0) {
      int need = SCHEME == 0 ? select_sastre_fast(nrm[0], 0.0, 1, log_eps, &p) : -1;
      if (need < 0) {
        lw[0] = log2_or_ninf(nrm[0]);
        need = select_walk_lw(lw, 1, log_eps, SCHEME, &p);
      }
      if (need >= 2) step = ST_W2;
    }
    T sc = T(1), sc2 = T(1);
    auto decided = [&]() {
      // exact 2^-s rescaling of W and the cached powers (engine.py:139-140)
      sc = pow2_neg<T>(p.s);
      sc2 = pow2_neg<T>(2 * p.s);
      EW2(SP(B, pmul(GP(B), sc)); SP(A2, pmul(GP(A2), sc2)));
    };
    // ---- the per-matrix program ------------------------------------------
    while (step != ST_DONE) {
      // (1) operands -> shared memory
      const T* Lb = f.buf0;
      const T* Rb = f.buf1;
      if (step == ST_W2) {
        f.store(f.buf0, B);
        Rb = f.buf0;
      } else if (step == ST_SQ) {
        f.store(f.buf0, P);
        Rb = f.buf0;
      } else if (SCHEME == 1 && (step == ST_W3 || step == ST_W4)) {
        f.store(f.buf0, step == ST_W3 ? A2 : Y0);
        f.store(f.buf1, B);
      } else if (SCHEME == 1 && step == ST_HORNER) {
        f.store(f.buf0, P);
        const int jj = ps_j_of(p.m);
        if (jj == 2) f.store(f.buf1, A2);
        else if (jj == 3) f.store(f.buf1, Y0);
        else f.store(f.buf1, Y1);
      } else if (SCHEME == 0) {
        const double* c = (p.m == 8) ? kT8 : kT15;
        if (step == ST_T4) {
          Tile L;
          // (A2/4 + A)/3 + I; x/3 taken as x * fl(1/3) (<= 1 ulp from the division)
          EW2(SP(L, padd(pmul(pfma(GP(A2), T(0.25), GP(B)), T(1.0 / 3.0)), DGP)));
          f.store(f.buf0, L);
          f.store(f.buf1, A2);
        } else if (step == ST_Y02) {
          const T c0 = (T)c[0], c1 = (T)c[1];
          Tile R;
          EW2(SP(R, pfma(GP(A2), c0, pmul(GP(B), c1))));
          f.store(f.buf0, A2);
          f.store(f.buf1, R);
        } else if (step == ST_P2) {
          const T c2 = (T)c[2], c3 = (T)c[3], c4 = (T)c[4];
          Tile L, R;
          EW2(SP(L, pfma(GP(B), c3, pfma(GP(A2), c2, GP(Y0)))); SP(R, pfma(GP(A2), c4, GP(Y0))));
          f.store(f.buf0, L);
          f.store(f.buf1, R);
        } else {  // ST_P3
          const T c7 = (T)c[7], c8 = (T)c[8], c9 = (T)c[9], c10 = (T)c[10];
          Tile L, R;
          EW2(SP(L, pfma(GP(B), c8, pfma(GP(A2), c7, GP(Y1))));
              SP(R, pfma(GP(B), c10, pfma(GP(Y0), c9, GP(Y1)))));         f.store(f.buf0, L);
          f.store(f.buf1, R);
        }
      }
      // (2) the product
      f.sync();
      f.template mm<!kLean>(Lb, Rb, P);
      f.sync();
      // (3) consume it, choose the next step
      if (step == ST_SQ) {
        step = (++q < p.s) ? ST_SQ : ST_DONE;
      } else if (step == ST_W2 || (SCHEME == 1 && (step == ST_W3 || step == ST_W4))) {
        const int pw = step == ST_W2 ? 2 : step == ST_W3 ? 3 : 4;
        if (pw == 2) { EW(A2[i][j] = P[i][j]); }
        else if (pw == 3) { EW(Y0[i][j] = P[i][j]); }
        else { EW(Y1[i][j] = P[i][j]); }
        nrm[pw - 1] = f.norm1(P);
        bad |= !(nrm[pw - 1] < INFINITY);  // a power overflowed or is NaN (matrix.py:97-98)
        have = pw;
        int need = SCHEME == 0 ? select_sastre_fast(nrm[0], nrm[1], 2, log_eps, &p) : -1;
        if (need < 0) {
          for (int q = 0; q < pw; ++q) lw[q] = log2_or_ninf(nrm[q]);
          need = select_walk_lw(lw, have, log_eps, SCHEME, &p);
        }
        if (need > 0) {
          step = need == 3 ? ST_W3 : ST_W4;
          continue;
        }
        if (po.plan_only) {  // select_sastre / select_ps: the plan is all the caller wants
          step = ST_DONE;
          break;
        }
        decided();
        if constexpr (SCHEME == 1) {
          const T sc3 = pow2_neg<T>(3 * p.s), sc4 = pow2_neg<T>(4 * p.s);
          if (have >= 3) { EW(Y0[i][j] *= sc3); }
          if (have >= 4) { EW(Y1[i][j] *= sc4); }
          // q = block((k-1) j, m)   (poly.py:179)
          const int jj = ps_j_of(p.m), kk = ps_k_of(p.m), lo = (kk - 1) * jj, cnt = p.m - lo;
          const T c0 = (T)kInvFact[lo];
          EW(P[i][j] = f.is_diag(i, j) ? c0 : T(0));
          if (cnt >= 1) { const T ct = (T)kInvFact[lo + 1]; EW(P[i][j] = P[i][j] + ct * B[i][j]); }
          if (cnt >= 2) { const T ct = (T)kInvFact[lo + 2]; EW(P[i][j] = P[i][j] + ct * A2[i][j]); }
          if (cnt >= 3) { const T ct = (T)kInvFact[lo + 3]; EW(P[i][j] = P[i][j] + ct * Y0[i][j]); }
          if (cnt >= 4) { const T ct = (T)kInvFact[lo + 4]; EW(P[i][j] = P[i][j] + ct * Y1[i][j]); }
          hz = kk - 2;  // next Horner block index r
          step = kk >= 2 ? ST_HORNER : (p.s > 0 ? ST_SQ : ST_DONE);
        } else {
          if (p.m == 2) {  // poly.py:196
            EW2(SP(P, padd(pfma(GP(A2), T(0.5), GP(B)), DGP)));
            step = ST_DONE;
          } else {
            step = p.m == 4 ? ST_T4 : ST_Y02;
          }
        }
      } else if (SCHEME == 1 && step == ST_HORNER) {
        // q <- q A^j + block(r j, r j + j - 1)
        const int jj = ps_j_of(p.m), lo = hz * jj, cnt = jj - 1;
        const T c0 = (T)kInvFact[lo];
        EW(P[i][j] = P[i][j] + (f.is_diag(i, j) ? c0 : T(0)));
        if (cnt >= 1) { const T ct = (T)kInvFact[lo + 1]; EW(P[i][j] = P[i][j] + ct * B[i][j]); }
        if (cnt >= 2) { const T ct = (T)kInvFact[lo + 2]; EW(P[i][j] = P[i][j] + ct * A2[i][j]); }
        if (cnt >= 3) { const T ct = (T)kInvFact[lo + 3]; EW(P[i][j] = P[i][j] + ct * Y0[i][j]); }
        step = (--hz >= 0) ? ST_HORNER : (p.s > 0 ? ST_SQ : ST_DONE);
      } else if (SCHEME == 0) {
        if (step == ST_T4) {  // poly.py:199
          EW2(SP(P, padd(pfma(GP(P), T(0.5), GP(B)), DGP)));
          step = ST_DONE;  // m = 4 implies s = 0
        } else if (step == ST_Y02) {
          EW(Y0[i][j] = P[i][j]);
          step = ST_P2;
        } else if (step == ST_P2) {
          const double* c = (p.m == 8) ? kT8 : kT15;
          if (p.m == 8) {  // poly.py:211
            const T c5 = (T)c[5];
            EW2(SP(P, padd(padd(pfma(GP(A2), T(0.5), pfma(GP(Y0), c5, GP(P))), GP(B)), DGP)));
            step = ST_DONE;  // m = 8 implies s = 0
          } else {  // poly.py:222-223
            const T c5 = (T)c[5], c6 = (T)c[6];
            EW2(SP(Y1, pfma(GP(A2), c6, pfma(GP(Y0), c5, GP(P)))));
            step = ST_P3;
          }
        } else {  // ST_P3 -> y22 (poly.py:224-229)
          const T c11 = (T)kT15[11], c12 = (T)kT15[12], c13 = (T)kT15[13], c14 = (T)kT15[14], c15 = (T)kT15[15];
          EW2(SP(P, padd(pfma(GP(B), c14, pfma(GP(A2), c13, pfma(GP(Y0), c12, pfma(GP(Y1), c11, GP(P))))),
                         pmul(DGP, c15))));
          step = p.s > 0 ? ST_SQ : ST_DONE;
        }
      }
    }
    // m = 0 / 1 finish without a product (poly.py:192, engine.py:141-142)
    if (nrm[0] == 0.0) {
      EW(P[i][j] = DG(i, j));
    } else if (have == 1) {
      if constexpr (SCHEME == 1) {  // PS m = 1: block(0, 1) = I + A
        EW(P[i][j] = (f.is_diag(i, j) ? (T)kInvFact[0] : T(0)) + (T)kInvFact[1] * B[i][j]);
      } else {
        EW(P[i][j] = B[i][j] + DG(i, j));
      }
    }

    mults = budget(p.m, SCHEME) + p.s;
    }  // SCHEME != 2

    if (!po.plan_only) {  // x * 0 is NaN exactly when x is Inf/NaN: one check per lane instead of eight
      Pr<T> z{T(0), T(0)};
      EW2(z = pfma(GP(P), T(0), z));
      bad |= !(z.x == T(0) && z.y == T(0));
    }
    bad = f.any_group(bad);
    if (!po.plan_only) f.save(X + idx * nn, n, vec, P);
    if (f.t == 0) {
      if (po.m) po.m[idx] = (int8_t)(p.m < 127 ? p.m : 127);  // Alg. 1 may exceed int8: saturate
      if (po.s) po.s[idx] = (int8_t)(p.s < 127 ? p.s : 127);
      if (po.e1) po.e1[idx] = p.e1;
      if (po.e2) po.e2[idx] = p.e2;
      if (po.norms) {
        po.norms[2 * idx] = nrm[0];
        po.norms[2 * idx + 1] = nrm[1];
      }
      if (po.mults) po.mults[idx] = mults;
      if (po.nonfinite) po.nonfinite[idx] = (uint8_t)(bad || !(nrm[0] < INFINITY));
    }
    if constexpr (kPrefetch) {
      EW(B[i][j] = nxt[i][j]);
    } else if constexpr (kLean) {
      if (nidx < batch) {
        if (vec) {
          asm volatile("cp.async.wait_all;" ::: "memory");
#pragma unroll
          for (int i = 0; i < TM; ++i) {
            if constexpr (F::HMODE) {
              const float2 v0 = *reinterpret_cast<const float2*>(f.stage + f.row(i) * NPAD + f.col(0));
              const float2 v1 = *reinterpret_cast<const float2*>(f.stage + f.row(i) * NPAD + f.col(2));
              B[i][0] = v0.x; B[i][1] = v0.y; B[i][2] = v1.x; B[i][3] = v1.y;
            } else {
              const float4 v = *reinterpret_cast<const float4*>(f.stage + f.row(i) * NPAD + f.col(0));
              B[i][0] = v.x; B[i][1] = v.y; B[i][2] = v.z; B[i][3] = v.w;
            }
          }
        } else {
          f.load(W + nidx * nn, n, vec, B);
        }
      }
    } else {
      if (nidx < batch) f.load(W + nidx * nn, n, vec, B);
    }
  }
#undef EW
#undef DG
#undef EW2
#undef GP
#undef SP
#undef DGP
}

}  // namespace expmb
