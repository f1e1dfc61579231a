/*
 * expmb.h -- C ABI of libexpmb.so, the B200 (sm_100a) batched matrix
 * exponential behind `paper_2512_20777_b200.expm`.
 *
 * Drop-in boundary for the reference hot path
 *   expmkit.expm(W: Matrix, eps: float, scheme: str = "sastre") -> ExpmResult
 *   (/root/reference/pkg/src/expmkit/engine.py:119-152,
 *    re-exported at __init__.py:61-70)
 * batched: one call exponentiates B independent n x n matrices.
 *
 * Conventions
 *  - Every pointer argument of expmb_expm is DEVICE memory owned by the caller
 *    (the library never allocates; scratch comes from `workspace`).
 *  - Matrices are row-major, contiguous, [batch][n][n], dtype fp32 or fp64.
 *  - All work is enqueued on `stream` (a cudaStream_t passed as void*); no
 *    call synchronises the host or the device (every path, every n: the
 *    large-n pipeline buckets matrices by their (m, s) on the device and
 *    every stage reads its slot count from device memory), so the calls are
 *    capturable in CUDA graphs.
 *  - Errors in arguments are returned synchronously as negative codes
 *    (mapped by the Python layer to ToleranceError / MatrixError, exactly
 *    like select.py:72-79, matrix.py:52-55, engine.py:137).  Numerical
 *    failure is reported per matrix in `nonfinite[]` (NonFiniteError,
 *    matrix.py:56-57,95-102).
 *  - Stateless and re-entrant; constant tables live in __constant__ memory.
 */
#ifndef EXPMB_H_
#define EXPMB_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* dtype codes */
#define EXPMB_F32 0
#define EXPMB_F64 1
/* scheme codes: select.py:58-61 SCHEME_SASTRE / SCHEME_PS */
#define EXPMB_SASTRE 0
#define EXPMB_PS 1
/* Alg. 1 term accumulation, the paper's comparator: engine.py:90-116
 * (expm_baseline); any n.  m = terms added, s may exceed int8 (the
 * m/s outputs saturate at 127; mults = m + s is exact). */
#define EXPMB_BASELINE 2

/* return codes */
#define EXPMB_OK 0
#define EXPMB_ERR_TOLERANCE (-1)   /* ToleranceError  (select.py:72-79)            */
#define EXPMB_ERR_SHAPE (-2)       /* MatrixError: n < 1 / batch < 0 (matrix.py:52-55) */
#define EXPMB_ERR_SCHEME (-3)      /* MatrixError: unknown scheme (engine.py:137)  */
#define EXPMB_ERR_DTYPE (-4)       /* MatrixError: dtype not fp32/fp64             */
#define EXPMB_ERR_WORKSPACE (-5)   /* workspace missing or too small               */
#define EXPMB_ERR_CUDA (-6)        /* a CUDA launch/copy failed                    */
#define EXPMB_ERR_ALIGN (-7)       /* W/X not 16-byte aligned                      */
#define EXPMB_ERR_UNSUPPORTED (-8) /* valid but unsupported combination            */

/* Library version (major*10000 + minor*100 + patch). */
int expmb_version(void);

/* Human-readable text for a return code. */
const char* expmb_strerror(int code);

/* Smallest admissible tolerance for a dtype: 2^-53 for fp64 (select.py:55),
 * 2^-24 for fp32 (the same rule at the working precision). */
double expmb_unit_roundoff(int dtype);

/* Scratch bytes expmb_expm needs for this problem: 256 for n <= 64 (the
 * persistent kernels' work counter; optional there), the bucketed pipeline's
 * buffers for n > 64 (plus the int8-slice planes for fp32 n >= 320 unless
 * EXPMB_I8=0).  Replaces nothing in the reference (numpy allocates per op). */
size_t expmb_workspace_bytes(int64_t batch, int32_t n, int dtype, int scheme);

/*
 * Batched expm.  Replaces engine.py:119-152 (expm), which the reference
 * calls once per matrix (bench.py:266-269, cli.py:40-43).
 *
 *   W          [batch,n,n] input (read only)
 *   X          [batch,n,n] output e^W (may not alias W)
 *   eps        tolerance (>= expmb_unit_roundoff(dtype), not NaN)
 *   scheme     EXPMB_SASTRE (orders 1,2,4,8,15+) or EXPMB_PS (1..16)
 *   m, s       [batch] selected order / scaling          (EvalPlan.m/.s)
 *   e1, e2     [batch] two-term remainder bounds         (EvalPlan.e1/.e2)
 *   norms      [batch,2] ||W||_1 and ||W^2||_1 (NaN if W^2 never formed)
 *   mults      [batch] n x n products charged (ExpmResult.mults)
 *   nonfinite  [batch] 1 where the input or any produced value was NaN/Inf
 *   Any of m..nonfinite may be NULL (not written).
 */
int expmb_expm(const void* W, void* X, int64_t batch, int32_t n, int dtype,
               double eps, int scheme,
               int8_t* m, int8_t* s, double* e1, double* e2, double* norms,
               int32_t* mults, uint8_t* nonfinite,
               void* workspace, size_t workspace_bytes, void* stream);

/*
 * Plan only: select_sastre / select_ps (select.py:223-234), batched.  Forms
 * exactly the powers the ladder needs (W^2; W^3, W^4 on the PS ladder) and
 * writes the plan -- no exponential, no X.  Arguments as expmb_expm (scheme
 * EXPMB_SASTRE or EXPMB_PS; workspace expmb_workspace_bytes(batch, n, dtype,
 * scheme)).  nonfinite[] flags an input or formed power that is not finite
 * (the reference raises NonFiniteError there, matrix.py:56-57, 95-102).
 */
int expmb_select(const void* W, int64_t batch, int32_t n, int dtype, double eps, int scheme,
                 int8_t* m, int8_t* s, double* e1, double* e2, double* norms,
                 int32_t* mults, uint8_t* nonfinite, void* workspace, size_t workspace_bytes, void* stream);

/*
 * Host-side evaluation of the SAME selector the kernels run (one
 * __host__ __device__ function), for testing without a GPU.  Replaces
 * select.py:164-220 given the power norms: norms[p-1] = ||W^p||_1 for
 * p = 1..4 (entries beyond what the ladder touches are ignored).
 * Returns the highest power the ladder needed (1..4) and writes the plan.
 */
int expmb_select_host(const double* norms, double eps, int scheme,
                      int* m, int* s, double* e1, double* e2);

/*
 * Host buffers in, host buffers out (the reference's calling convention,
 * engine.py:119-152), pipelined: the batch is cut into `chunks` pieces (on
 * multiples of 4 matrices); every host->device copy is queued on `s_in`, each
 * chunk's expmb_expm runs on `s_comp` after its copy, and its result is
 * copied back on `s_out` while later chunks compute.  W_host / X_host should
 * be pinned (cudaHostAlloc) for the copies to overlap; W_dev / X_dev are
 * [batch,n,n] device staging buffers; the plan outputs are device arrays as
 * in expmb_expm.  Returns after queuing; synchronise `s_out` (after
 * `s_comp`) before reading X_host.
 */
int expmb_expm_pipelined(const void* W_host, void* X_host, void* W_dev, void* X_dev, int64_t batch, int32_t n,
                         int dtype, double eps, int scheme, int8_t* m, int8_t* s, double* e1, double* e2,
                         double* norms, int32_t* mults, uint8_t* nonfinite, int chunks, void* workspace,
                         size_t workspace_bytes, void* s_in, void* s_comp, void* s_out);

/*
 * Batched low-rank exponential.  Replaces engine.py:198-257 (expm_lowrank)
 * with the LowRankPair checks of engine.py:166-181: for W = A1 A2 returns
 * e^W = I + A1 psi(V) A2, V = A2 A1, psi(x) = sum_{i<=m} x^i/(i+1)!, the
 * order m chosen on LOWRANK_ORDERS = (1,2,4,8,15,16,20,25,30) (no scaling).
 *
 *   A1         [batch,n,t] device, row-major     (LowRankPair.a1)
 *   A2         [batch,t,n] device, row-major     (LowRankPair.a2)
 *   X          [batch,n,n] output e^(A1 A2)
 *   1 <= t <= n (MatrixError otherwise)
 *   m, e1, e2  [batch] plan (EvalPlan.m/.e1/.e2; s is always 0)
 *   norms      [batch,2] ||V||_1, ||V^2||_1 (NaN if V^2 never formed)
 *   mults      [batch] t x t products (ExpmResult.mults; rect_mults is 3)
 *   flags      [batch] EXPMB_LR_* bits; a flagged matrix's X is NaN
 *   workspace  expmb_lowrank_workspace_bytes(batch, n, t, dtype) bytes: 0
 *              (NULL allowed) for t <= 32, where every t x t operand lives
 *              in shared memory; for t > 32 the t x t operands live here
 * Any of m..flags may be NULL.  No host synchronisation.
 */
#define EXPMB_LR_BAD_INPUT 1 /* non-finite factor entry: MatrixError (engine.py:179-180)  */
#define EXPMB_LR_NONFINITE 2 /* V, a power, psi or e^W not finite: NonFiniteError        */
#define EXPMB_LR_NO_ORDER 4  /* no admissible order: LowRankOrderError (engine.py:236-240) */
size_t expmb_lowrank_workspace_bytes(int64_t batch, int32_t n, int32_t t, int dtype);
int expmb_expm_lowrank(const void* A1, const void* A2, void* X, int64_t batch, int32_t n, int32_t t,
                       int dtype, double eps, int8_t* m, double* e1, double* e2, double* norms,
                       int32_t* mults, uint8_t* flags, void* workspace, size_t workspace_bytes, void* stream);

/*
 * Host evaluation of the low-rank ladder the kernel runs (engine.py:224-244):
 * norms[0] = ||V||_1, norms[1] = ||V^2||_1 (read only when have_v2).
 * Returns 0 (plan written), 1 (||V^2||_1 needed: call again with have_v2 = 1)
 * or -1 (no admissible order).
 */
int expmb_select_lowrank_host(const double* norms, int have_v2, double eps, int* m, double* e1, double* e2);

/*
 * Time grid: X[k] = e^(t_k A) for one n x n matrix A and K times t_k, the
 * generative-flow case (BASELINE config C3).  Each
 * X[k] is what expmb_expm returns for the materialised t_k A (engine.py:
 * 119-152 per time point): the same plan (up to the last-bit difference
 * between |t_k| ||A||_1 and ||fl(t_k A)||_1), the same outputs.  For n > 64
 * the powers A^1..A^16 are formed once in binary64 and each time point costs
 * only its s_k squarings plus one fused linear combination.
 *
 *   A          [n,n] device; t [K] device (same dtype); X [K,n,n] device
 *   m..nonfinite, scheme, eps: as expmb_expm (per time point)
 *   workspace  expmb_timegrid_workspace_bytes(K, n, dtype) bytes
 * No host synchronisation (the squaring buckets are formed on the device).
 */
size_t expmb_timegrid_workspace_bytes(int64_t K, int32_t n, int dtype);
int expmb_expm_timegrid(const void* A, const void* t, void* X, int64_t K, int32_t n, int dtype, double eps,
                        int scheme, int8_t* m, int8_t* s, double* e1, double* e2, double* norms,
                        int32_t* mults, uint8_t* nonfinite, void* workspace, size_t workspace_bytes,
                        void* stream);

#ifdef __cplusplus
}
#endif

#endif /* EXPMB_H_ */
