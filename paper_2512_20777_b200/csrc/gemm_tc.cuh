// gemm_tc.cuh -- large-n fp32 products on the 5th-generation tensor cores.
//
// Each product P = L R of the evaluation formulas (poly.py:204-230), of the
// W^2 selection product (select.py:192) and of the squaring phase
// (engine.py:80-87) runs as one tcgen05 GEMM stage over a bucket of matrices:
//   * TMA (cp.async.bulk.tensor, 128B swizzle) streams 128x32 fp32 k-tiles of
//     L (K-major, row-major L) and of R^T (K-major, so the producers store every
//     right-hand operand transposed) into a 3-stage shared-memory ring;
//   * one thread issues tcgen05.mma.kind::tf32 (M=128, N=128, K=8) with the
//     accumulators in TMEM: split-TF32 ("3xTF32"): L R ~= L R + L R_lo + L_lo R,
//     where x_lo = x - tf32(x).  The hardware truncates fp32 inputs to tf32
//     (measured, tools/tc_probe.cu), so the raw fp32 array is the "hi" part
//     and the producers store x_lo = x - trunc_tf32(x) beside it;
//   * k-tiles accumulate round-robin into NACC = 4 TMEM accumulators (the
//     tensor core's fp32 accumulation truncates: the bias grows with the
//     chain length, so shorter chains, summed with round-to-nearest in the
//     epilogue, shrink it);
//   * four epilogue warps read the accumulators (tcgen05.ld 32x32b), apply
//     the stage's linear combination for the CTA's matrix, and write each
//     result in the layouts its consumers need: row-major value (+ lo) for a
//     left operand or an epilogue input, transposed value (+ lo) for a right
//     operand.  The transposed store is coalesced: the 32 lanes of a warp hold
//     32 consecutive rows.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "fused_small.cuh"
#include "gemm_simt.cuh"
#include "select.cuh"

namespace expmb {
namespace tc {

constexpr int BM = 128, BN = 128, BK = 32, STAGES = 3;
constexpr int TILE_BYTES = BM * BK * 4;           // 16 KB per operand tile
constexpr int STAGE_BYTES = 4 * TILE_BYTES;       // A, A_lo, B, B_lo
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024;
constexpr int NTHREADS = 192;                      // w0 TMA, w1 MMA/TMEM, w2..w5 epilogue
#ifndef EXPMB_TC_NACC
#define EXPMB_TC_NACC 4
#endif
constexpr int NACC = EXPMB_TC_NACC;                // k-tiles round-robin over NACC accumulators
constexpr uint32_t TMEM_COLS = NACC * 128;         // NACC 128-column fp32 accumulators

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "TC_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra TC_WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
// UMMA shared-memory descriptor: K-major, 128B swizzle, 8-row atoms 1024 B apart.
__device__ __forceinline__ uint64_t kmajor_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3fff);
  d |= (uint64_t)(16 >> 4) << 16;     // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;   // SBO: next 8-row group
  d |= (uint64_t)1 << 46;             // descriptor version (sm100)
  d |= (uint64_t)2 << 61;             // SWIZZLE_128B
  return d;
}
// kind::tf32, D fp32, A/B K-major, N = 128, M = 128
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t ad, uint64_t bd, uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(ad), "l"(bd), "r"(kIdesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
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
  for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
}

// x - tf32(x) with the hardware's truncating conversion: exact in fp32.
__device__ __forceinline__ float tf32_lo(float x) { return x - __uint_as_float(__float_as_uint(x) & 0xffffe000u); }

// ---------------------------------------------------------------------------
// stage context
// ---------------------------------------------------------------------------
enum Map : int { M_W = 0, M_WLO, M_WT, M_WTLO, M_W2, M_W2LO, M_LA, M_LALO, M_RA, M_RALO, M_LB, M_LBLO, M_RB, M_RBLO, M_COUNT };

struct Maps {
  CUtensorMap m[M_COUNT];
};

struct Ctx {
  int n;
  int tiles_m;
  int sq_step;
  int64_t ms;   // elements between matrices of a workspace buffer
  int64_t ws;   // elements between matrices of W / X
  const float* W;
  float* X;
  float *Wlo, *Wt, *Wtlo, *W2, *W2lo, *W2t, *Y0, *Y1, *La, *Lalo, *Ra, *Ralo, *Lb, *Lblo, *Rb, *Rblo;
  const int8_t* m;
  const int8_t* s;
  const int* need;
  double* part;
};

struct Out {
  float* rm;    // row-major value
  float* rmlo;  // row-major lo part
  float* t;     // transposed value
  float* tlo;   // transposed lo part
};

struct Epi {
  int mapA, mapB;
  float alpha;
  int nin, nout;
  bool colnorm;
  const float* in[4];
  float c[3][4];
  float d[3];
  Out out[3];
};

__device__ __forceinline__ Out out_rm(float* p) { return Out{p, nullptr, nullptr, nullptr}; }

// The per-matrix stage program (Sastre): same formulas as gemm_simt.cuh's make_epi.
__device__ __forceinline__ bool make_tc_epi(const Ctx& g, int stage, int z, Epi& e) {
  const int64_t o = (int64_t)z * g.ms;
  const float* Wz = g.W + (int64_t)z * g.ws;
  float* Xz = g.X + (int64_t)z * g.ws;
  e.nin = 0; e.nout = 1; e.colnorm = false; e.alpha = 1.f;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    e.d[k] = 0.f;
    e.out[k] = Out{nullptr, nullptr, nullptr, nullptr};
#pragma unroll
    for (int q = 0; q < 4; ++q) e.c[k][q] = 0.f;
  }
  e.in[0] = Wz; e.in[1] = g.W2 + o; e.in[2] = g.Y0 + o; e.in[3] = g.Y1 + o;
  if (stage == STAGE_W2) {
    if (g.need[z] != 2) return false;
    e.mapA = M_W; e.mapB = M_WT;
    e.out[0] = Out{g.W2 + o, g.W2lo + o, g.W2t + o, nullptr};
    e.colnorm = true;
    return true;
  }
  const int m = g.m[z], s = g.s[z];
  const double sg = pow2_neg<double>(s), sg2 = pow2_neg<double>(2 * s);
  const Out slot0 = Out{g.Lb + o, g.Lblo + o, g.Rb + o, g.Rblo + o};
  const Out slot1 = Out{g.La + o, g.Lalo + o, g.Ra + o, g.Ralo + o};
  if (stage == STAGE_SQ) {
    const int q = g.sq_step;
    if (s <= q) return false;
    e.mapA = (q % 2 == 0) ? M_LB : M_LA;
    e.mapB = (q % 2 == 0) ? M_RB : M_RA;
    e.out[0] = (q == s - 1) ? out_rm(Xz) : ((q % 2 == 0) ? slot1 : slot0);
    return true;
  }
  const double* c = (m == 8) ? kT8 : kT15;
  if (stage == STAGE_E1) {
    if (m == 4) {  // poly.py:199 with inner*A^2 = A^2*inner (both polynomials in W); s = 0
      e.mapA = M_W2; e.mapB = M_RA;
      e.alpha = 0.5f;
      e.nin = 1; e.c[0][0] = 1.f; e.d[0] = 1.f;
      e.out[0] = out_rm(Xz);
      return true;
    }
    if (m < 8) return false;
    e.mapA = M_W2; e.mapB = M_RA;
    e.alpha = (float)sg2;
    e.nin = 2; e.nout = 3;
    e.out[0] = out_rm(g.Y0 + o);
    e.out[1] = Out{g.Lb + o, g.Lblo + o, nullptr, nullptr};
    e.out[2] = Out{nullptr, nullptr, g.Rb + o, g.Rblo + o};
    e.c[1][1] = (float)(c[2] * sg2); e.c[1][0] = (float)(c[3] * sg);
    e.c[2][1] = (float)(c[4] * sg2);
    return true;
  }
  if (stage == STAGE_E2) {
    if (m < 8) return false;
    e.mapA = M_LB; e.mapB = M_RB;
    if (m == 8) {  // poly.py:211 (s = 0)
      e.nin = 3;
      e.c[0][2] = (float)c[5]; e.c[0][1] = 0.5f; e.c[0][0] = 1.f; e.d[0] = 1.f;
      e.out[0] = out_rm(Xz);
      return true;
    }
    e.nin = 3; e.nout = 3;
    e.out[0] = out_rm(g.Y1 + o);
    e.out[1] = Out{g.La + o, g.Lalo + o, nullptr, nullptr};
    e.out[2] = Out{nullptr, nullptr, g.Ra + o, g.Ralo + o};
    e.c[0][2] = (float)c[5]; e.c[0][1] = (float)(c[6] * sg2);
    e.c[1][1] = (float)(c[7] * sg2); e.c[1][0] = (float)(c[8] * sg);
    e.c[2][2] = (float)c[9]; e.c[2][0] = (float)(c[10] * sg);
    return true;
  }
  // STAGE_E3 (poly.py:224-229)
  if (m < 15) return false;
  e.mapA = M_LA; e.mapB = M_RA;
  e.nin = 4;
  e.c[0][3] = (float)c[11]; e.c[0][2] = (float)c[12]; e.c[0][1] = (float)(c[13] * sg2); e.c[0][0] = (float)(c[14] * sg);
  e.d[0] = (float)c[15];
  e.out[0] = (s == 0) ? out_rm(Xz) : slot0;
  return true;
}

__device__ __forceinline__ void store_out(const Out& ot, int n, int r, int c0, const float (&v)[32], bool rowok) {
  if (ot.rm) {
    if (rowok) {
#pragma unroll
      for (int j = 0; j < 32; j += 4)
        if (c0 + j + 3 < n) *reinterpret_cast<float4*>(ot.rm + (size_t)r * n + c0 + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
    }
  }
  if (ot.rmlo) {
    if (rowok) {
#pragma unroll
      for (int j = 0; j < 32; j += 4)
        if (c0 + j + 3 < n)
          *reinterpret_cast<float4*>(ot.rmlo + (size_t)r * n + c0 + j) =
              make_float4(tf32_lo(v[j]), tf32_lo(v[j + 1]), tf32_lo(v[j + 2]), tf32_lo(v[j + 3]));
    }
  }
  if (ot.t) {
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (rowok && c0 + j < n) ot.t[(size_t)(c0 + j) * n + r] = v[j];
  }
  if (ot.tlo) {
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (rowok && c0 + j < n) ot.tlo[(size_t)(c0 + j) * n + r] = tf32_lo(v[j]);
  }
}

__global__ void __launch_bounds__(NTHREADS, 1) tc_stage_kernel(const __grid_constant__ Maps maps, Ctx g, int stage,
                                                                const int* __restrict__ list) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ uint64_t full_bar[STAGES], empty_bar[STAGES], tmem_bar;
  __shared__ uint32_t tmem_base_sh;
  const int z = list ? list[blockIdx.z] : (int)blockIdx.z;
  Epi e;
  if (!make_tc_epi(g, stage, z, e)) return;  // uniform per CTA

  unsigned char* sm = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int n = g.n;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int KT = (n + BK - 1) / BK;

  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full_bar[i], 1);
      mbar_init(&empty_bar[i], 1);
    }
    mbar_init(&tmem_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base_sh;

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer ----------------
    const CUtensorMap* mA = &maps.m[e.mapA];
    const CUtensorMap* mAlo = &maps.m[e.mapA + 1];
    const CUtensorMap* mB = &maps.m[e.mapB];
    const CUtensorMap* mBlo = &maps.m[e.mapB + 1];
    for (int kt = 0; kt < KT; ++kt) {
      const int st = kt % STAGES;
      mbar_wait(&empty_bar[st], ((kt / STAGES) & 1) ^ 1);
      unsigned char* b = sm + st * STAGE_BYTES;
      mbar_expect_tx(&full_bar[st], STAGE_BYTES);
      tma_load_3d(b, mA, &full_bar[st], kt * BK, m0, z);
      tma_load_3d(b + TILE_BYTES, mAlo, &full_bar[st], kt * BK, m0, z);
      tma_load_3d(b + 2 * TILE_BYTES, mB, &full_bar[st], kt * BK, n0, z);
      tma_load_3d(b + 3 * TILE_BYTES, mBlo, &full_bar[st], kt * BK, n0, z);
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer ----------------
    for (int kt = 0; kt < KT; ++kt) {
      const int st = kt % STAGES;
      mbar_wait(&full_bar[st], (kt / STAGES) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t base = smem_u32(sm + st * STAGE_BYTES);
      const uint32_t acc = tmem + (uint32_t)((kt % NACC) * BN);
#pragma unroll
      for (int k = 0; k < BK / 8; ++k) {
        const uint64_t a = kmajor_desc(base + k * 32);
        const uint64_t alo = kmajor_desc(base + TILE_BYTES + k * 32);
        const uint64_t b = kmajor_desc(base + 2 * TILE_BYTES + k * 32);
        const uint64_t blo = kmajor_desc(base + 3 * TILE_BYTES + k * 32);
        mma_tf32(acc, a, b, (kt >= NACC || k > 0) ? 1u : 0u);
        mma_tf32(acc, a, blo, 1u);
        mma_tf32(acc, alo, b, 1u);
      }
      mma_commit(&empty_bar[st]);  // frees this smem stage when the MMAs are done
    }
    mma_commit(&tmem_bar);
  } else if (warp >= 2) {
    // ---------------- epilogue ----------------
    mbar_wait(&tmem_bar, 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    const int q = warp & 3;                  // TMEM lane quarter this warp may access
    const int rl = q * 32 + lane;            // row within the tile
    const int r = m0 + rl;
    const bool rowok = r < n;
    double* red = reinterpret_cast<double*>(sm);  // smem ring is idle now
    for (int cb = 0; cb < BN / 32; ++cb) {
      float v[32], v1[32];
      const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + cb * 32;
      tmem_ld32(ta, v);
      // pairwise sum of the accumulators that were written (KT may be < NACC)
      if (NACC == 4 && KT >= 4) {
        float v2[32], v3[32];
        tmem_ld32(ta + BN, v1);
        tmem_ld32(ta + 2 * BN, v2);
        tmem_ld32(ta + 3 * BN, v3);
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = (v[j] + v1[j]) + (v2[j] + v3[j]);
      } else {
        for (int a = 1; a < NACC && a < KT; ++a) {
          tmem_ld32(ta + a * BN, v1);
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] += v1[j];
        }
      }
      const int c0 = n0 + cb * 32;
      float o0[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) o0[j] = e.alpha * v[j];
      for (int qq = 0; qq < e.nin; ++qq) {
        const float cq = e.c[0][qq];
        if (cq == 0.f || !rowok) continue;
        const float* ip = e.in[qq] + (size_t)r * n + c0;
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          if (c0 + j + 3 < n) {
            const float4 x = __ldg(reinterpret_cast<const float4*>(ip + j));
            o0[j] = fmaf(cq, x.x, o0[j]); o0[j + 1] = fmaf(cq, x.y, o0[j + 1]);
            o0[j + 2] = fmaf(cq, x.z, o0[j + 2]); o0[j + 3] = fmaf(cq, x.w, o0[j + 3]);
          }
        }
      }
      if (e.d[0] != 0.f && r >= c0 && r < c0 + 32) {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (c0 + j == r) o0[j] += e.d[0];
      }
      store_out(e.out[0], n, r, c0, o0, rowok);
      for (int k = 1; k < e.nout; ++k) {
        float ok[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) ok[j] = o0[j];
        for (int qq = 0; qq < e.nin; ++qq) {
          const float cq = e.c[k][qq];
          if (cq == 0.f || !rowok) continue;
          const float* ip = e.in[qq] + (size_t)r * n + c0;
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            if (c0 + j + 3 < n) {
              const float4 x = __ldg(reinterpret_cast<const float4*>(ip + j));
              ok[j] = fmaf(cq, x.x, ok[j]); ok[j + 1] = fmaf(cq, x.y, ok[j + 1]);
              ok[j + 2] = fmaf(cq, x.z, ok[j + 2]); ok[j + 3] = fmaf(cq, x.w, ok[j + 3]);
            }
          }
        }
        store_out(e.out[k], n, r, c0, ok, rowok);
      }
      if (e.colnorm) {
        // deterministic column abs-sums of this 128-row tile (select.py:193)
#pragma unroll
        for (int j = 0; j < 32; ++j) red[j * BM + rl] = rowok ? fabs((double)o0[j]) : 0.0;
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (rl < 32 && c0 + rl < n) {
          double a = 0.0;
          for (int rr = 0; rr < BM; ++rr) a += red[rl * BM + rr];
          g.part[((size_t)z * g.tiles_m + blockIdx.y) * n + c0 + rl] = a;
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
}

// W -> W_lo (row-major), W^T, W^T_lo via 32x32 shared-memory tiles.
__global__ void __launch_bounds__(256) tc_prep_kernel(Ctx g, int cnt) {
  __shared__ float t[32][33];
  const int z = blockIdx.z;
  const int n = g.n;
  const float* Wz = g.W + (int64_t)z * g.ws;
  const int64_t o = (int64_t)z * g.ms;
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  const int tx = threadIdx.x % 32, ty = threadIdx.x / 32;
  for (int k = ty; k < 32; k += 8) {
    const int r = by + k, c = bx + tx;
    float v = (r < n && c < n) ? Wz[(size_t)r * n + c] : 0.f;
    if (r < n && c < n) g.Wlo[o + (size_t)r * n + c] = tf32_lo(v);
    t[k][tx] = v;
  }
  __syncthreads();
  for (int k = ty; k < 32; k += 8) {
    const int r = bx + k, c = by + tx;  // transposed coordinates
    if (r < n && c < n) {
      const float v = t[tx][k];
      g.Wt[o + (size_t)r * n + c] = v;
      g.Wtlo[o + (size_t)r * n + c] = tf32_lo(v);
    }
  }
}

// First evaluation step for the tensor-core path: finals for m <= 2, and the
// transposed right operand of the first product (inner^T for m = 4, R1^T for
// m >= 8) with its lo part (poly.py:192-199, :209, :221).
__global__ void __launch_bounds__(256) tc_elem_kernel(Ctx g, const int* __restrict__ list) {
  const int z = list[blockIdx.y];
  const int m = g.m[z], s = g.s[z];
  const int n = g.n;
  const size_t nn = (size_t)n * n;
  const int64_t o = (int64_t)z * g.ms;
  const float* Wz = g.W + (int64_t)z * g.ws;
  float* Xz = g.X + (int64_t)z * g.ws;
  const float sg = pow2_neg<float>(s), sg2 = pow2_neg<float>(2 * s);
  const double* cc = (m == 8) ? kT8 : kT15;
  const float c0 = (float)(cc[0] * (double)sg2), c1 = (float)(cc[1] * (double)sg);
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < nn; i += (size_t)gridDim.x * blockDim.x) {
    const int r = (int)(i / n), c = (int)(i % n);
    const float dg = (r == c) ? 1.f : 0.f;
    if (m == 0) {
      Xz[i] = dg;
    } else if (m == 1) {
      Xz[i] = Wz[i] + dg;
    } else if (m == 2) {
      Xz[i] = (g.W2[o + i] * 0.5f + Wz[i]) + dg;
    } else if (m == 4) {
      const float v = (g.W2t[o + i] * 0.25f + g.Wt[o + i]) * (1.0f / 3.0f) + dg;
      g.Ra[o + i] = v;
      g.Ralo[o + i] = tf32_lo(v);
    } else {
      const float v = c0 * g.W2t[o + i] + c1 * g.Wt[o + i];
      g.Ra[o + i] = v;
      g.Ralo[o + i] = tf32_lo(v);
    }
  }
}

}  // namespace tc
}  // namespace expmb
