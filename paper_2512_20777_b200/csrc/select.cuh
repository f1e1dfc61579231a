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

// select.py:82-83
EXPMB_HD double log2_or_ninf(double x) { return x > 0.0 ? log2(x) : -INFINITY; }

// NumPy npymath npy_logaddexp2 (np.logaddexp2 at select.py:206).
EXPMB_HD double logaddexp2(double x, double y) {
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
EXPMB_HD int select_walk(const double* nrm, int have, double eps, int scheme, Plan* out) {
  const double norm1 = nrm[0];
  if (norm1 == 0.0) {  // select.py:172-173
    out->m = 0; out->s = 0; out->e1 = 0.0; out->e2 = 0.0;
    return 0;
  }
  const double log_eps = log2(eps);
  double lw[5];
  lw[1] = log2_or_ninf(norm1);
  for (int p = 2; p <= have && p <= 4; ++p) lw[p] = log2_or_ninf(nrm[p - 1]);
  double l1 = INFINITY, l2 = INFINITY;
  const int nord = scheme == 1 ? 7 : 5;
  int m = scheme == 1 ? 16 : 15;
  bool finished = false;
  for (int i = 0; i < nord; ++i) {
    const int mi = scheme == 1 ? ps_order(i) : sastre_order(i);
    const int j = scheme == 1 ? ps_jpow(i) : (i == 0 ? 1 : 2);
    const int k = scheme == 1 ? ps_kcount(i) : sastre_kcount(i);
    const double lc1 = scheme == 1 ? ps_log_tail(2 * i) : sastre_log_tail(2 * i);
    const double lc2 = scheme == 1 ? ps_log_tail(2 * i + 1) : sastre_log_tail(2 * i + 1);
    m = mi;
    if (mi == 1) {
      l1 = rn_add(lc1, rn_mul(2.0, lw[1]));
      l2 = rn_add(lc2, rn_mul(3.0, lw[1]));
    } else {
      if (j > have) return j;  // need W^j (select.py:190-194)
      const double kl = rn_mul((double)k, lw[j]);
      if (scheme == 1) {
        l1 = rn_add(rn_add(lc1, kl), lw[1]);
        l2 = rn_add(rn_add(lc2, kl), lw[2]);
      } else {
        l1 = rn_add(lc1, kl);
        l2 = rn_add(lc2, kl);
        if (j * k == mi) {
          l1 = rn_add(l1, lw[1]);
          l2 = rn_add(l2, lw[2]);
        } else {
          l2 = rn_add(l2, lw[1]);
        }
      }
    }
    if (logaddexp2(l1, l2) <= log_eps) {
      finished = true;
      break;
    }
  }
  int s = 0;
  if (!finished) {  // select.py:210-219
    const double ls[2] = {l1, l2};
    for (int t = 1; t <= 2; ++t) {
      const double l = ls[t - 1];
      if (l == -INFINITY) continue;
      const double q = ceil(rn_div(rn_sub(l, log_eps), (double)(m + t)));
      // q may be +inf/NaN when a norm overflowed; the cap below bounds it
      // (the reference raises NonFiniteError earlier in that case).
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
  return 0;
}

}  // namespace expmb
