// select.cuh -- order/scaling selector shared by host and device.
//
// One __host__ __device__ restatement of the reference ladder
// (/root/reference/pkg/src/expmkit/select.py:164-220, select_sastre :228-234,
// select_ps :223-225) operating on the 1-norms of the powers of W that the
// kernels form in-register.  The arithmetic mirrors Python's evaluation order
// exactly (explicit round-to-nearest intrinsics on the device so nvcc cannot
// contract a*b+c into an FMA), and np.logaddexp2 is restated from NumPy's
// npymath (`npy_logaddexp2`), so the only possible differences from the
// reference are the last-ulp behaviour of log2/exp2/log1p in CUDA's libdevice.
#pragma once

#include <math.h>
#include <stdint.h>

#if defined(__CUDACC__)
#define EXPMB_HD __host__ __device__ __forceinline__
#else
#define EXPMB_HD inline
#endif

namespace expmb {

// select.py:55-56
constexpr double kUnitRoundoff = 0x1p-53;
constexpr int kMaxScaling = 20;

// log2 of the tail weights (select.py:109 computes them with math.log2);
// the hex literals are exactly the binary64 values Python produces
// (generated from oracle/expm_oracle.py, which the golden tests pin).
// SASTRE_TABLES (select.py:130-141): orders 1,2,4,8,15.
struct SastreTab {
  static constexpr int n = 5;
};
// PS_TABLES (select.py:112-125): orders 1,2,4,6,9,12,16.

EXPMB_HD double sastre_log_tail(int i) {
  switch (i) {
    case 0: return -0x1.0000000000000p+0;
    case 1: return -0x1.4ae00d1cfdeb4p+1;
    case 2: return -0x1.4ae00d1cfdeb4p+1;
    case 3: return -0x1.2570068e7ef5ap+2;
    case 4: return -0x1.ba0a7eda4c113p+2;
    case 5: return -0x1.2fbd42b465836p+3;
    case 6: return -0x1.278191a01a44ep+4;
    case 7: return -0x1.5ca82fb30d8bcp+4;
    case 8: return -0x1.6b1bc6161c270p+5;   // log2 |1/16! - b16|
    default: return -0x1.82b3695d62b2fp+5;  // log2 1/17!
  }
}
EXPMB_HD int sastre_order(int i) { return i == 0 ? 1 : i == 1 ? 2 : i == 2 ? 4 : i == 3 ? 8 : 15; }
EXPMB_HD int sastre_kcount(int i) { return i == 0 ? 1 : i == 1 ? 1 : i == 2 ? 2 : i == 3 ? 4 : 8; }

EXPMB_HD double ps_log_tail(int i) {
  switch (i) {
    case 0: return -0x1.0000000000000p+0;
    case 1: return -0x1.4ae00d1cfdeb4p+1;
    case 2: return -0x1.4ae00d1cfdeb4p+1;
    case 3: return -0x1.2570068e7ef5ap+2;
    case 4: return -0x1.ba0a7eda4c113p+2;
    case 5: return -0x1.2fbd42b465836p+3;
    case 6: return -0x1.89931cb1b5942p+3;
    case 7: return -0x1.e9931cb1b5942p+3;
    case 8: return -0x1.5ca82fb30d8bcp+4;
    case 9: return -0x1.940204ab1a464p+4;
    case 10: return -0x1.0449834aeee41p+5;
    case 11: return -0x1.22bef9ca42e83p+5;
    case 12: return -0x1.82b3695d62b2fp+5;
    default: return -0x1.a40f6b0102706p+5;
  }
}
EXPMB_HD int ps_order(int i) {
  return i == 0 ? 1 : i == 1 ? 2 : i == 2 ? 4 : i == 3 ? 6 : i == 4 ? 9 : i == 5 ? 12 : 16;
}
EXPMB_HD int ps_jpow(int i) { return i == 0 ? 1 : i <= 2 ? 2 : i <= 4 ? 3 : 4; }
EXPMB_HD int ps_kcount(int i) { return i <= 1 ? 1 : i <= 3 ? 2 : i <= 5 ? 3 : 4; }

// poly.py:136-146 ps_shape -> budget (j-1)+(k-1); poly.py:233-241 sastre budget.
EXPMB_HD int ps_j_of(int m) {
  int j = 1;
  while (j * j < m) ++j;
  return j;
}
EXPMB_HD int ps_k_of(int m) {
  int j = ps_j_of(m);
  return (m + j - 1) / j;
}
EXPMB_HD int budget(int m, int scheme /*0 sastre, 1 ps*/) {
  if (m <= 1) return 0;
  if (scheme == 1) return (ps_j_of(m) - 1) + (ps_k_of(m) - 1);
  return m == 2 ? 1 : m == 4 ? 2 : m == 8 ? 3 : 4;
}

// Round-to-nearest arithmetic that the compiler may not fuse.
#if defined(__CUDA_ARCH__)
EXPMB_HD double rn_add(double a, double b) { return __dadd_rn(a, b); }
EXPMB_HD double rn_sub(double a, double b) { return __dsub_rn(a, b); }
EXPMB_HD double rn_mul(double a, double b) { return __dmul_rn(a, b); }
EXPMB_HD double rn_div(double a, double b) { return __ddiv_rn(a, b); }
#else
EXPMB_HD double rn_add(double a, double b) { volatile double r = a + b; return r; }
EXPMB_HD double rn_sub(double a, double b) { volatile double r = a - b; return r; }
EXPMB_HD double rn_mul(double a, double b) { volatile double r = a * b; return r; }
EXPMB_HD double rn_div(double a, double b) { volatile double r = a / b; return r; }
#endif

// select.py:82-83 (out of line on the device: the libdevice log2 expansion is
// large and the kernels call it from several sites)
#if defined(__CUDACC__)
__host__ __device__ __noinline__
#else
inline
#endif
double log2_or_ninf(double x) { return x > 0.0 ? log2(x) : -INFINITY; }

// 2^-k exactly, for 0 <= k <= 126 (float) / 1022 (double): the scaling factors
// of engine.py:139-140 (ldexp), built from the exponent bits.
template <typename T>
EXPMB_HD T pow2_neg(int k);
template <>
EXPMB_HD float pow2_neg<float>(int k) {
#if defined(__CUDA_ARCH__)
  return __int_as_float((127 - k) << 23);
#else
  return ldexpf(1.0f, -k);
#endif
}
template <>
EXPMB_HD double pow2_neg<double>(int k) {
#if defined(__CUDA_ARCH__)
  return __longlong_as_double((long long)(1023 - k) << 52);
#else
  return ldexp(1.0, -k);
#endif
}

// NumPy npymath npy_logaddexp2 (np.logaddexp2 at select.py:206).
#if defined(__CUDACC__)
__host__ __device__ __noinline__
#else
inline
#endif
double logaddexp2(double x, double y) {
  const double kLog2e = 1.442695040888963407359924681001892137;
  if (x == y) return rn_add(x, 1.0);
  const double tmp = rn_sub(x, y);
  if (tmp > 0) return rn_add(x, rn_mul(kLog2e, log1p(exp2(-tmp))));
  if (tmp <= 0) return rn_add(y, rn_mul(kLog2e, log1p(exp2(tmp))));
  return tmp;  // NaN
}

struct Plan {
  int m;
  int s;
  double e1;
  double e2;
};

// Walk the ladder with the power norms known so far.  nrm[p-1] = ||W^p||_1
// for p <= have.  Returns 0 when the plan is decided (written to *out), or the
// power p > have the next rung needs (the caller forms W^p = W^(p-1) W, as
// select.py:190-194 does, and calls again; restarting the walk is exact
// because earlier rungs depend only on norms that do not change).
// Tail of the walk (select.py:210-220): scaling rule + reported bounds.
// Out of line: ceil/div/exp2 expand to a lot of code and run once per matrix.
#if defined(__CUDACC__)
__host__ __device__ __noinline__
#else
inline
#endif
void plan_tail(double l1, double l2, int m, bool finished, double log_eps, Plan* out) {
  int s = 0;
  if (!finished) {
    const double ls[2] = {l1, l2};
    for (int t = 1; t <= 2; ++t) {
      const double l = ls[t - 1];
      if (l == -INFINITY) continue;
      const double q = ceil(rn_div(rn_sub(l, log_eps), (double)(m + t)));
      // q may be +inf/NaN when a norm overflowed; the cap bounds it (the
      // reference raises NonFiniteError earlier in that case).
      if (!(q <= (double)kMaxScaling)) { s = kMaxScaling; continue; }
      const int s1 = (int)q;
      if (s1 > s) s = s1;
    }
    if (s > kMaxScaling) s = kMaxScaling;
  }
  out->m = m;
  out->s = s;
  out->e1 = exp2(l1);
  out->e2 = exp2(l2);
}

// Core walk on log2 power norms: lwp[p-1] = log2 ||W^p||_1 (select.py:176,194),
// log_eps = log2(eps) (select.py:175).  The caller handles ||W||_1 == 0.
// Fully unrolled (the rung constants fold into immediates); the exact
// logaddexp2 runs only for a rung whose [max, max+1] bracket straddles log_eps.
EXPMB_HD int select_walk_lw(const double* lwp, int have, double log_eps, int scheme, Plan* out) {
  const double lw1 = lwp[0];
  const double lw2 = have >= 2 ? lwp[1] : 0.0;
  const double lw3 = have >= 3 ? lwp[2] : 0.0;
  const double lw4 = have >= 4 ? lwp[3] : 0.0;
  double l1 = INFINITY, l2 = INFINITY;
  const int nord = scheme == 1 ? 7 : 5;
  int m = scheme == 1 ? 16 : 15;
  bool finished = false;
#pragma unroll
  for (int i = 0; i < 7; ++i) {
    if (i >= nord) break;
    const int mi = scheme == 1 ? ps_order(i) : sastre_order(i);
    const int j = scheme == 1 ? ps_jpow(i) : (i == 0 ? 1 : 2);
    const int k = scheme == 1 ? ps_kcount(i) : sastre_kcount(i);
    const double lc1 = scheme == 1 ? ps_log_tail(2 * i) : sastre_log_tail(2 * i);
    const double lc2 = scheme == 1 ? ps_log_tail(2 * i + 1) : sastre_log_tail(2 * i + 1);
    m = mi;
    if (mi == 1) {
      l1 = rn_add(lc1, rn_mul(2.0, lw1));
      l2 = rn_add(lc2, rn_mul(3.0, lw1));
    } else {
      if (j > have) return j;  // need W^j (select.py:190-194)
      const double lwj = j == 2 ? lw2 : (j == 3 ? lw3 : lw4);
      const double kl = rn_mul((double)k, lwj);
      if (scheme == 1) {
        l1 = rn_add(rn_add(lc1, kl), lw1);
        l2 = rn_add(rn_add(lc2, kl), lw2);
      } else {
        l1 = rn_add(lc1, kl);
        l2 = rn_add(lc2, kl);
        if (j * k == mi) {
          l1 = rn_add(l1, lw1);
          l2 = rn_add(l2, lw2);
        } else {
          l2 = rn_add(l2, lw1);
        }
      }
    }
    // logaddexp2(l1, l2) lies in [max, max + 1]; only a rung whose bracket
    // straddles log_eps needs the exact (transcendental) evaluation.
    const double hi = l1 > l2 ? l1 : l2;
    bool pass;
    if (rn_add(hi, 1.0) < log_eps - 1e-9) pass = true;
    else if (hi > log_eps + 1e-9) pass = false;
    else pass = logaddexp2(l1, l2) <= log_eps;
    if (pass) {
      finished = true;
      break;
    }
  }
  plan_tail(l1, l2, m, finished, log_eps, out);
  return 0;
}

// ---------------------------------------------------------------------------
// Fast Sastre selector for the fused kernels.
//
// The exact walk needs binary64 log2 of the norms and exp2 for the reported
// bounds -- ~300 instructions per matrix, 16% of the n=16 kernel.  The fast
// path evaluates the same ladder with a cheap log2 (exponent bits + fp32
// log2f of the mantissa, |error| < 4e-7) and accepts a decision only when
// every comparison it makes clears the error by a wide margin (1e-5 in log2
// units for the rung tests, 1e-5 on the fractional part for each ceil of the
// scaling rule).  Any closer call returns -1 and the caller runs the exact
// walk, so the chosen (m, s) is always the exact walk's.  e1/e2 are formed
// as tail * ||W^2||^k * ||W|| products (equal to exp2 of the log-domain sum to
// ~1e-14 relative), valid because both norms are restricted to [2^-100, 2^100].
// ---------------------------------------------------------------------------
EXPMB_HD double sastre_tail(int i) {
  switch (i) {
    case 0: return 0x1.0000000000000p-1;
    case 1: return 0x1.5555555555555p-3;
    case 2: return 0x1.5555555555555p-3;
    case 3: return 0x1.5555555555555p-5;
    case 4: return 0x1.1111111111111p-7;
    case 5: return 0x1.6c16c16c16c17p-10;
    case 6: return 0x1.71de3a556c734p-19;
    case 7: return 0x1.27e4fb7789f5cp-22;
    case 8: return 0x1.871cb69cf3722p-46;   // |1/16! - b16|
    default: return 0x1.952c77030ad4ap-49;  // 1/17!
  }
}

// log2 for the fast path: exponent bits + fp32 log2f of the mantissa in [1,2)
// (|error| < 5e-7 absolute, independent of the magnitude).
EXPMB_HD float fast_log2f(double x) {
#if defined(__CUDA_ARCH__)
  const int hi = __double2hiint(x);
  const int e = ((hi >> 20) & 0x7ff) - 1023;
  const float mant = (float)__hiloint2double((hi & 0x800fffff) | 0x3ff00000, __double2loint(x));
  return (float)e + __log2f(mant);  // MUFU.LG2: |error| ~2^-22 on [1, 2)
#else
  int e;
  const double mant = frexp(x, &e) * 2.0;
  return (float)(e - 1) + log2f((float)mant);
#endif
}

// log2(1 + 2^-d), d >= 0: the logaddexp2 correction term (|error| < 1e-6).
EXPMB_HD float fast_l2p(float d) {
#if defined(__CUDA_ARCH__)
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(-d));
  return __log2f(1.0f + y);
#else
  return log2f(1.0f + exp2f(-d));
#endif
}

// Returns 0 (decided, *out written), 2 (needs W^2 first), or -1 (too close to
// call: run select_walk_lw).  have = 1 or 2; n2 ignored when have == 1.
// All ladder arithmetic is fp32 (|l| <= ~250 so |error| < 4e-5); every
// comparison needs a margin of 2e-4 (log2 units) or it defers to the exact walk.
EXPMB_HD int select_sastre_fast(double n1, double n2, int have, double log_eps_d, Plan* out) {
  const double lo = 0x1p-100, hi = 0x1p100;
  if (!(n1 >= lo && n1 <= hi)) return -1;
  if (have >= 2 && !(n2 >= lo && n2 <= hi)) return -1;
  const float M = 2e-4f;
  const float log_eps = (float)log_eps_d;
  const float lw1 = fast_log2f(n1);
  // rung 0 (m = 1): l1 = log2(1/2!) + 2 lw1, l2 = log2(1/3!) + 3 lw1
  {
    const float l1 = -1.0f + 2.0f * lw1, l2 = -2.5849625f + 3.0f * lw1;
    const float h = fmaxf(l1, l2);
    bool pass = false, known = true;
    if (h + 1.0f < log_eps - M) pass = true;
    else if (h > log_eps + M) pass = false;
    else {
      const float lae = h + fast_l2p(fabsf(l1 - l2));
      if (lae < log_eps - M) pass = true;
      else if (!(lae > log_eps + M)) known = false;
    }
    if (!known) return -1;
    if (pass) {
      out->m = 1; out->s = 0;
      out->e1 = 0x1.0000000000000p-1 * (n1 * n1);
      out->e2 = 0x1.5555555555555p-3 * (n1 * n1 * n1);
      return 0;
    }
    if (have < 2) return 2;
  }
  const float lw2 = fast_log2f(n2);
  float l1 = 0.f, l2 = 0.f;
  int mi = 15, ri = 4;
  bool finished = false;
#pragma unroll
  for (int i = 1; i < 5; ++i) {
    mi = sastre_order(i);
    ri = i;
    const int k = sastre_kcount(i);
    l1 = (float)sastre_log_tail(2 * i) + (float)k * lw2;
    l2 = (float)sastre_log_tail(2 * i + 1) + (float)k * lw2;
    if (2 * k == mi) { l1 += lw1; l2 += lw2; } else { l2 += lw1; }
    const float h = fmaxf(l1, l2);
    if (h + 1.0f < log_eps - M) { finished = true; break; }  // certainly passes
    if (h > log_eps + M) continue;                           // certainly fails
    const float lae = h + fast_l2p(fabsf(l1 - l2));
    if (lae < log_eps - M) { finished = true; break; }
    if (!(lae > log_eps + M)) return -1;                     // too close: exact walk
  }
  int s = 0;
  if (!finished) {
    // s = clamp(max(ceil(v1), ceil(v2)), 0, 20) (select.py:210-219)
    const float v1 = (l1 - log_eps) * (1.0f / 16.0f);
    const float v2 = (l2 - log_eps) * (1.0f / 17.0f);
    const float va = fmaxf(v1, v2);
    float c_lo = ceilf(va - M), c_hi = ceilf(va + M);
    c_lo = fminf(fmaxf(c_lo, 0.f), (float)kMaxScaling);
    c_hi = fminf(fmaxf(c_hi, 0.f), (float)kMaxScaling);
    if (c_lo != c_hi) return -1;
    s = (int)c_lo;
  }
  // reported bounds exp2(l1), exp2(l2) as products (select.py:220)
  const int k = sastre_kcount(ri);
  double pk = n2;
#pragma unroll
  for (int q = 1; q < 8; ++q)
    if (q < k) pk *= n2;
  double e1 = sastre_tail(2 * ri) * pk, e2 = sastre_tail(2 * ri + 1) * pk;
  if (2 * k == mi) { e1 *= n1; e2 *= n2; } else { e2 *= n1; }
  out->m = mi;
  out->s = s;
  out->e1 = e1;
  out->e2 = e2;
  return 0;
}

// Leaner fast path for the fused kernels (same margins / same decisions as
// select_sastre_fast).  Rung 0 needs only ||W||_1 and fails certainly above
// rung0_threshold(log_eps), so the kernels skip it for all but tiny norms;
// rungs 1..4 are straight-line fp32 with lw = __log2f((float)norm); e1/e2
// use n2^k by repeated squaring (k is a power of two).
EXPMB_HD double rung0_threshold(double log_eps) {
  // rung 0 fails iff max(l1, l2) > log_eps + margin; l1 = -1 + 2 lw1 suffices
  return exp2((log_eps + 1.0 + 1e-3) * 0.5);
}

EXPMB_HD float lg2_fast(double x) {
#if defined(__CUDA_ARCH__)
  return __log2f((float)x);  // x in [2^-100, 2^100]: |error| < 5e-7
#else
  return log2f((float)x);
#endif
}

// 0: decided (*out written); -1: too close to call (run select_walk_lw).
EXPMB_HD int select_sastre_fast2(double n1, double n2, double log_eps_d, Plan* out) {
  const double lo = 0x1p-100, hi = 0x1p100;
  if (!(n1 >= lo && n1 <= hi && n2 >= lo && n2 <= hi)) return -1;
  const float M = 2e-4f;
  const float le = (float)log_eps_d;
  const float lw1 = lg2_fast(n1), lw2 = lg2_fast(n2);
  // verdict of one rung: +1 pass, 0 fail, -1 unsure
  auto verdict = [&](float l1, float l2) -> int {
    const float h = fmaxf(l1, l2);
    if (h + 1.0f < le - M) return 1;
    if (h > le + M) return 0;
    const float lae = h + fast_l2p(fabsf(l1 - l2));
    if (lae < le - M) return 1;
    if (lae > le + M) return 0;
    return -1;
  };
  // sastre_log_tail(2..9) as fp32 constants
  const float T2 = (float)-0x1.4ae00d1cfdeb4p+1, T3 = (float)-0x1.2570068e7ef5ap+2;
  const float T4 = (float)-0x1.ba0a7eda4c113p+2, T5 = (float)-0x1.2fbd42b465836p+3;
  const float T6 = (float)-0x1.278191a01a44ep+4, T7 = (float)-0x1.5ca82fb30d8bcp+4;
  const float T8 = (float)-0x1.6b1bc6161c270p+5, T9 = (float)-0x1.82b3695d62b2fp+5;
  int ri, v;
  float l1, l2;
  l1 = T2 + lw2 + lw1; l2 = T3 + lw2 + lw2;                          // m = 2, k = 1
  if ((v = verdict(l1, l2)) != 0) { ri = 1; goto done; }
  l1 = T4 + 2.0f * lw2 + lw1; l2 = T5 + 2.0f * lw2 + lw2;            // m = 4, k = 2
  if ((v = verdict(l1, l2)) != 0) { ri = 2; goto done; }
  l1 = T6 + 4.0f * lw2 + lw1; l2 = T7 + 4.0f * lw2 + lw2;            // m = 8, k = 4
  if ((v = verdict(l1, l2)) != 0) { ri = 3; goto done; }
  l1 = T8 + 8.0f * lw2; l2 = T9 + 8.0f * lw2 + lw1;                   // m = 15, k = 8
  if ((v = verdict(l1, l2)) != 0) { ri = 4; goto done; }
  ri = 4; v = 0;                                                      // no rung passed: scale
done:
  if (v < 0) return -1;
  int s = 0;
  if (v == 0) {
    const float va = fmaxf((l1 - le) * (1.0f / 16.0f), (l2 - le) * (1.0f / 17.0f));
    float c_lo = ceilf(va - M), c_hi = ceilf(va + M);
    c_lo = fminf(fmaxf(c_lo, 0.f), (float)kMaxScaling);
    c_hi = fminf(fmaxf(c_hi, 0.f), (float)kMaxScaling);
    if (c_lo != c_hi) return -1;
    s = (int)c_lo;
  }
  // reported bounds exp2(l1), exp2(l2) (select.py:220) as products
  double pk = n2;
  if (ri >= 2) pk *= pk;
  if (ri >= 3) pk *= pk;
  if (ri >= 4) pk *= pk;
  const double t1 = sastre_tail(2 * ri), t2 = sastre_tail(2 * ri + 1);
  out->m = ri == 1 ? 2 : ri == 2 ? 4 : ri == 3 ? 8 : 15;
  out->s = s;
  if (ri < 4) {
    out->e1 = t1 * pk * n1;
    out->e2 = t2 * pk * n2;
  } else {
    out->e1 = t1 * pk;
    out->e2 = t2 * pk * n1;
  }
  return 0;
}

// Branch-free form of select_sastre_fast2 for the warp-batched kernel, whose
// lanes 0..Q-1 each select for a different matrix: divergent early exits made
// the SIMT walk cost the union of every lane's path.  All four rungs are
// evaluated (two MUFU ops each) and the first one that does not certainly fail
// is picked with selects.  A rung passes if max(l1, l2) + 1 or the fast
// logaddexp2 clears log_eps - M, fails if max(l1, l2) or the fast logaddexp2
// exceeds log_eps + M, else it is too close to call (-1: exact walk).  The
// fast logaddexp2 is within 1e-6 of the exact one, which lies in
// [max, max + 1], so no decided rung can disagree with the exact walk; the
// e1/e2 products are select_sastre_fast2's.
EXPMB_HD int select_sastre_bf(double n1, double n2, double log_eps_d, Plan* out) {
  const double lo = 0x1p-100, hi = 0x1p100;
  if (!(n1 >= lo && n1 <= hi && n2 >= lo && n2 <= hi)) return -1;
  const float M = 2e-4f;
  const float le = (float)log_eps_d;
  const float lw1 = lg2_fast(n1), lw2 = lg2_fast(n2);
  const float T[8] = {(float)-0x1.4ae00d1cfdeb4p+1, (float)-0x1.2570068e7ef5ap+2, (float)-0x1.ba0a7eda4c113p+2,
                      (float)-0x1.2fbd42b465836p+3, (float)-0x1.278191a01a44ep+4, (float)-0x1.5ca82fb30d8bcp+4,
                      (float)-0x1.6b1bc6161c270p+5, (float)-0x1.82b3695d62b2fp+5};
  int ri = 4, v = 0;
  float L1 = 0.f, L2 = 0.f;
#pragma unroll
  for (int i = 4; i >= 1; --i) {  // reverse: the first rung that does not fail wins
    const float kf = (float)(1 << (i - 1));
    float l1, l2;
    if (i < 4) {  // m = 2, 4, 8: J K = m, both tails gain lw1 / lw2
      l1 = T[2 * i - 2] + kf * lw2 + lw1;
      l2 = T[2 * i - 1] + kf * lw2 + lw2;
    } else {      // m = 15
      l1 = T[6] + 8.0f * lw2;
      l2 = T[7] + 8.0f * lw2 + lw1;
    }
    const float h = fmaxf(l1, l2);
    const float lae = h + fast_l2p(fabsf(l1 - l2));
    const bool pass = (h + 1.0f < le - M) || (lae < le - M);
    const bool fail = (h > le + M) || (lae > le + M);
    const int vi = pass ? 1 : (fail ? 0 : -1);
    if (i == 4) { L1 = l1; L2 = l2; }
    if (vi != 0) { ri = i; v = vi; L1 = l1; L2 = l2; }
  }
  if (v < 0) return -1;
  int s = 0;
  if (v == 0) {
    const float va = fmaxf((L1 - le) * (1.0f / 16.0f), (L2 - le) * (1.0f / 17.0f));
    float c_lo = ceilf(va - M), c_hi = ceilf(va + M);
    c_lo = fminf(fmaxf(c_lo, 0.f), (float)kMaxScaling);
    c_hi = fminf(fmaxf(c_hi, 0.f), (float)kMaxScaling);
    if (c_lo != c_hi) return -1;
    s = (int)c_lo;
  }
  double pk = n2;
  if (ri >= 2) pk *= pk;
  if (ri >= 3) pk *= pk;
  if (ri >= 4) pk *= pk;
  const double t1 = sastre_tail(2 * ri), t2 = sastre_tail(2 * ri + 1);
  out->m = ri == 1 ? 2 : ri == 2 ? 4 : ri == 3 ? 8 : 15;
  out->s = s;
  if (ri < 4) {
    out->e1 = t1 * pk * n1;
    out->e2 = t2 * pk * n2;
  } else {
    out->e1 = t1 * pk;
    out->e2 = t2 * pk * n1;
  }
  return 0;
}

// Same walk from the norms themselves (host tests, large-n select kernels).
EXPMB_HD int select_walk(const double* nrm, int have, double eps, int scheme, Plan* out) {
  if (nrm[0] == 0.0) {  // select.py:172-173
    out->m = 0; out->s = 0; out->e1 = 0.0; out->e2 = 0.0;
    return 0;
  }
  double lw[4];
  for (int p = 1; p <= have && p <= 4; ++p) lw[p - 1] = log2_or_ninf(nrm[p - 1]);
  return select_walk_lw(lw, have, log2(eps), scheme, out);
}

}  // namespace expmb
