// K2 (tensor-core form) -- expert synthesis on tcgen05 + switch telemetry +
// equaliser, persistent and software-pipelined: one CTA of 16 warps per SM
// loops over work items (unit, 128-subcarrier tile).  Iteration i:
//   * thread 0 issues the cp.async.bulk (TMA) copies of item i+1's y / tx rows
//     into the other shared-memory stage (double buffer), so HBM streams while
//     item i is equalised;
//   * every thread pulls its share of item i+1's coefficients (L2) early;
//   * thread (subcarrier j = TMEM lane, expert = warp/4 & 1, symbol half =
//     warp/8) reads item i's synthesised taps from TMEM (tcgen05.ld), stores
//     the expert outputs + |H| telemetry (half 0), and equalises its half of the
//     symbols from the stage (compile-time weights for the NR 0/5/10 pattern);
//   * then B(i+1) -- both experts' taps rotated to the tile origin, real
//     embedding, hi | lo -- is written to shared memory, one __syncthreads, and
//     thread 0 issues D(i+1) = S_hi B_hi + S_lo B_hi + S_hi B_lo
//     (tcgen05.mma kind::tf32, A = twiddles S in TMEM, 3xTF32) into the other
//     TMEM accumulator; it completes while item i+1's data lands.
// Per-tile partial sums are reduced in a fixed order (fp32 per thread, fp64
// across threads); the last tile of a unit finalises its telemetry.
#pragma once
#include <cuda.h>

#include "common.cuh"
#include "k_synth_eq.cuh"

#define TC_THREADS 512                   // epilogue threads: 128 subcarriers x 2 experts x 2 symbol halves
#define TC_BLOCK (TC_THREADS + 32)       // + the producer / MMA warp (single-group plans)

__device__ __forceinline__ uint64_t umma_desc_kmajor(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  // SWIZZLE_NONE K-major canonical layout: core matrices of 8 rows x 16 B,
  // LBO = byte distance between the two 16-B K chunks, SBO = between 8-row groups
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version 1 (sm_100)
  return d;
}

__device__ __forceinline__ void umma_tf32(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                          uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accum));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
// the same rounding (nearest, ties away from zero) in two integer ops for finite
// inputs -- cvt.rna.tf32 is emulated by a longer sequence on sm_100
__device__ __forceinline__ float tf32_rna_fast(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}


// byte offset of element (row, kappa) of a K-major SWIZZLE_NONE operand with
// `groups` 8-row groups per 8-wide K block
__device__ __forceinline__ uint32_t kmaj_off(int row, int kappa, int groups) {
  return (uint32_t)((kappa >> 3) * groups * 256 + (row >> 3) * 256 + ((kappa >> 2) & 1) * 128 +
                    (row & 7) * 16 + (kappa & 3) * 4);
}


// _time_interp_weights for the NR default (14 symbols, DMRS 0/5/10), rounded
// exactly like the plan's runtime table (fp64 weight, then float)
__host__ __device__ constexpr float std_tw(int t, int d) {
  return t <= 0    ? (d == 0 ? 1.f : 0.f)
         : t >= 10 ? (d == 2 ? 1.f : 0.f)
         : t < 5   ? (d == 0 ? (float)(1.0 - (double)t / 5.0) : d == 1 ? (float)((double)t / 5.0) : 0.f)
         : t == 5  ? (d == 1 ? 1.f : 0.f)
                   : (d == 1 ? (float)(1.0 - (double)(t - 5) / 5.0)
                             : d == 2 ? (float)((double)(t - 5) / 5.0) : 0.f);
}

template <int N>
__device__ __forceinline__ void tmem_ld_n(uint32_t taddr, float* v) {
  if constexpr (N >= 16) {
    tmem_ld16(taddr, v);
    tmem_ld_n<N - 16>(taddr + 16, v + 16);
  } else if constexpr (N >= 8) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                   "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
    tmem_ld_n<N - 8>(taddr + 8, v + 8);
  } else if constexpr (N >= 4) {
    uint32_t r[4];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(taddr));
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = __uint_as_float(r[i]);
    tmem_ld_n<N - 4>(taddr + 4, v + 4);
  } else if constexpr (N >= 2) {
    uint32_t r[2];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];"
                 : "=r"(r[0]), "=r"(r[1])
                 : "r"(taddr));
    v[0] = __uint_as_float(r[0]);
    v[1] = __uint_as_float(r[1]);
    tmem_ld_n<N - 2>(taddr + 2, v + 2);
  }
}

// one RE of one expert: interpolate, MRC, accumulate the SINR sums (fp32
// per-thread partials over <= 14 symbols, reduced in fp64 across threads)
template <int NA, int ND>
__device__ __forceinline__ void eq_re(const float2 (&h)[NA][ND], const float* wt, const float2* yv,
                                      float2 x, float m, float nv, float& sre, float& sim,
                                      float& syy) {
  float2 num = make_float2(0.f, 0.f);
  float den = 0.f;
#pragma unroll
  for (int a = 0; a < NA; ++a) {
    float2 hn = make_float2(0.f, 0.f);
#pragma unroll
    for (int d = 0; d < ND; ++d) {
      if (wt[d] == 1.f) {  // a held symbol: the DMRS estimate itself (compile-time weights)
        hn = h[a][d];
      } else if (wt[d] != 0.f) {  // folds away for compile-time weights
        hn.x = fmaf(wt[d], h[a][d].x, hn.x);
        hn.y = fmaf(wt[d], h[a][d].y, hn.y);
      }
    }
    num.x = fmaf(hn.x, yv[a].x, fmaf(hn.y, yv[a].y, num.x));
    num.y = fmaf(hn.x, yv[a].y, fmaf(-hn.y, yv[a].x, num.y));
    den = fmaf(hn.x, hn.x, fmaf(hn.y, hn.y, den));
  }
  float inv;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(inv) : "f"(den + nv));
  inv *= m;  // m = 0 on pilot REs
  const float hr = num.x * inv, hi = num.y * inv;
  sre = fmaf(x.x, hr, fmaf(x.y, hi, sre));
  sim = fmaf(x.x, hi, fmaf(-x.y, hr, sim));
  syy = fmaf(hr, hr, fmaf(hi, hi, syy));
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16};" ::"r"(taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
      "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
      "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])),
      "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
      "r"(__float_as_uint(v[15]))
      : "memory");
}

__device__ __forceinline__ void umma_tf32_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b,
                                             uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(accum));
}

// one RE of the NR 0/5/10 pattern with the MRC denominator given:
// den = sum_a |w0 h_d0 + w1 h_d1|^2 from the DMRS Gram entries (eq_std_half)
template <int NA, int ND>
__device__ __forceinline__ void eq_re_den(const float2 (&h)[NA][ND], const float* wt,
                                          const float2* yv, float2 x, float m, float den_nv,
                                          float& sre, float& sim, float& syy) {
  float2 num = make_float2(0.f, 0.f);
#pragma unroll
  for (int a = 0; a < NA; ++a) {
    float2 hn = make_float2(0.f, 0.f);
#pragma unroll
    for (int d = 0; d < ND; ++d) {
      if (wt[d] == 1.f) {
        hn = h[a][d];
      } else if (wt[d] != 0.f) {
        hn.x = fmaf(wt[d], h[a][d].x, hn.x);
        hn.y = fmaf(wt[d], h[a][d].y, hn.y);
      }
    }
    num.x = fmaf(hn.x, yv[a].x, fmaf(hn.y, yv[a].y, num.x));
    num.y = fmaf(hn.x, yv[a].y, fmaf(-hn.y, yv[a].x, num.y));
  }
  float inv;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(inv) : "f"(den_nv));
  inv *= m;  // m = 0 on pilot REs
  const float hr = num.x * inv, hi = num.y * inv;
  sre = fmaf(x.x, hr, fmaf(x.y, hi, sre));
  sim = fmaf(x.x, hi, fmaf(-x.y, hr, sim));
  syy = fmaf(hr, hr, fmaf(hi, hi, syy));
}

// one symbol half (H) of the NR 0/5/10 pattern for one expert thread; SXX:
// this thread also accumulates |x|^2 (expert-0 threads).  The MRC denominators
// come from the DMRS Gram entries G_dd = sum_a |h_ad|^2 and R = sum_a Re(h_ad^*
// h_a,d+1) of the half's DMRS pair: a held symbol's is G_dd (the same fma chain
// as the direct sum), an interpolated one's w0^2 G00 + w1^2 G11 + 2 w0 w1 R.
// PK: tx from the packed QPSK wire format (xb = this subcarrier's code byte of
// symbol 0, codes of later symbols ARCHES_TXB_ROW apart, jsh = its bit offset)
template <int NA, int ND, int H, bool SXX, bool PK = false>
__device__ __forceinline__ void eq_std_half(const float2 (&h)[NA][ND], const float2* yrow,
                                            const float2* xrow, const unsigned char* xb, int jsh,
                                            float modd, float nv, float& sre, float& sim,
                                            float& syy, float& sxx) {
  // balanced halves: 4 interpolated + 3 held symbols each
  constexpr int kSym[2][7] = {{0, 1, 2, 3, 4, 5, 10}, {6, 7, 8, 9, 11, 12, 13}};
  static_assert(ND == 3, "NR 0/5/10 pattern");
  float g[ND];
#pragma unroll
  for (int d = 0; d < ND; ++d) {
    g[d] = 0.f;
    if (H == 0 || d > 0) {
#pragma unroll
      for (int a = 0; a < NA; ++a) g[d] = fmaf(h[a][d].x, h[a][d].x, fmaf(h[a][d].y, h[a][d].y, g[d]));
    }
  }
  constexpr int d0 = H == 0 ? 0 : 1;  // the half's interpolated DMRS pair (d0, d0 + 1)
  float r = 0.f;
#pragma unroll
  for (int a = 0; a < NA; ++a)
    r = fmaf(h[a][d0].x, h[a][d0 + 1].x, fmaf(h[a][d0].y, h[a][d0 + 1].y, r));
#pragma unroll
  for (int tt = 0; tt < 7; ++tt) {
    const int t = kSym[H][tt];
    float wt[ND];
#pragma unroll
    for (int d = 0; d < ND; ++d) wt[d] = std_tw(t, d);
    float2 yv[NA];
#pragma unroll
    for (int a = 0; a < NA; ++a) yv[a] = yrow[(size_t)(a * 14 + t) * ARCHES_TILE];
    float2 x;
    if constexpr (PK) x = qpsk_code_to_x((unsigned int)xb[t * ARCHES_TXB_ROW] >> jsh);
    else x = xrow[(size_t)t * ARCHES_TILE];
    const bool dm = (t == 0 || t == 5 || t == 10);
    const float m = dm ? modd : 1.f;
    float den;
    if (wt[0] == 1.f) den = g[0];
    else if (wt[1] == 1.f) den = g[1];
    else if (wt[2] == 1.f) den = g[2];
    else {
      const float w0 = wt[d0], w1 = wt[d0 + 1];
      den = fmaf(w0 * w0, g[d0], fmaf(w1 * w1, g[d0 + 1], (2.f * w0 * w1) * r));
    }
    eq_re_den<NA, ND>(h, wt, yv, x, m, den + nv, sre, sim, syy);
    if (SXX) {
      if (dm) sxx = fmaf(m * x.x, x.x, fmaf(m * x.y, x.y, sxx));
      else sxx = fmaf(x.x, x.x, fmaf(x.y, x.y, sxx));
    }
  }
}

// 3-D tensor TMA: box {256 floats, rows, 1} of a [units][rows][2N floats] array
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      ".L2::cache_hint [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)),
      "l"(policy)
      : "memory");
}

// antenna-group form of eq_std_half (massive-MIMO plans, 4 antennas per
// group): MRC numerator / denominator per symbol accumulate in shared memory
// (g[0..6] = Re num, g[7..13] = Im num, g[14..20] = den, stride TC_THREADS)
// across the groups of one tile; the last group forms x_hat and the SINR sums.
template <int NA, int ND, int H, bool SXX>
__device__ __forceinline__ void eq_grp_half(const float2 (&h)[NA][ND], const float2* yrow,
                                            const float2* xrow, float modd, float nv, float* g,
                                            bool first, bool last, float& sre, float& sim,
                                            float& syy, float& sxx) {
  constexpr int kSym[2][7] = {{0, 1, 2, 3, 4, 5, 10}, {6, 7, 8, 9, 11, 12, 13}};
#pragma unroll
  for (int tt = 0; tt < 7; ++tt) {
    const int t = kSym[H][tt];
    float wt[ND];
#pragma unroll
    for (int d = 0; d < ND; ++d) wt[d] = std_tw(t, d);
    float2 num = first ? make_float2(0.f, 0.f) : make_float2(g[tt * TC_THREADS], g[(7 + tt) * TC_THREADS]);
    float den = first ? 0.f : g[(14 + tt) * TC_THREADS];
#pragma unroll
    for (int a = 0; a < NA; ++a) {
      const float2 yv = yrow[(size_t)(a * 14 + t) * ARCHES_TILE];
      float2 hn = make_float2(0.f, 0.f);
#pragma unroll
      for (int d = 0; d < ND; ++d) {
        if (wt[d] == 1.f) {
          hn = h[a][d];
        } else if (wt[d] != 0.f) {
          hn.x = fmaf(wt[d], h[a][d].x, hn.x);
          hn.y = fmaf(wt[d], h[a][d].y, hn.y);
        }
      }
      num.x = fmaf(hn.x, yv.x, fmaf(hn.y, yv.y, num.x));
      num.y = fmaf(hn.x, yv.y, fmaf(-hn.y, yv.x, num.y));
      den = fmaf(hn.x, hn.x, fmaf(hn.y, hn.y, den));
    }
    if (!last) {
      g[tt * TC_THREADS] = num.x;
      g[(7 + tt) * TC_THREADS] = num.y;
      g[(14 + tt) * TC_THREADS] = den;
      continue;
    }
    const float2 x = xrow[(size_t)t * ARCHES_TILE];
    const bool dm = (t == 0 || t == 5 || t == 10);
    const float m = dm ? modd : 1.f;
    float inv;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(inv) : "f"(den + nv));
    inv *= m;
    const float hr = num.x * inv, hi = num.y * inv;
    sre = fmaf(x.x, hr, fmaf(x.y, hi, sre));
    sim = fmaf(x.x, hi, fmaf(-x.y, hr, sim));
    syy = fmaf(hr, hr, fmaf(hi, hi, syy));
    if (SXX) sxx = fmaf(m * x.x, x.x, fmaf(m * x.y, x.y, sxx));
  }
}

template <int NA, int ND, bool kStd, bool kTmap, bool kGrp = false, bool kPk = false>
__global__ void __launch_bounds__(kGrp ? TC_THREADS : TC_BLOCK, 1)
    k2_tc(const PlanDev P, const K2Args args, const int n_items,
          const __grid_constant__ CUtensorMap tm_y, const __grid_constant__ CUtensorMap tm_x) {
  constexpr int R = 2 * NA * ND;                    // complex outputs: AI then MMSE
  constexpr int NCOL = ((2 * R + 15) / 16) * 16;    // MMA N (real columns)
  constexpr int NG = NCOL / 8;
  constexpr int CPE = 2 * NA * ND;                  // D columns per expert
  // B operands / TMEM accumulators in flight: item i's MMA is issued as soon as
  // the epilogue of item i - LEAD is done, so its latency hides behind a whole
  // epilogue
  constexpr int LEAD = 2;
  constexpr int NBUF = LEAD + 1;
  // single-group plans: a producer warp issues the MMAs and stage refills.
  // Antenna-group plans (longer epilogue, 96 registers would spill under a 17th
  // warp): the last epilogue warp to complete a B operand issues them itself
  constexpr bool kProd = !kGrp;
  constexpr int NST = kPk ? 3 : 2;  // y / tx stages (packed tx leaves room for a third)
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t s_full[3];       // stage landed
  __shared__ __align__(8) uint64_t s_mma[NBUF];     // accumulator ready
  __shared__ __align__(8) uint64_t s_bready[NBUF];  // B(i) written (512 thread / 16 warp arrivals)
  __shared__ uint32_t s_bcount[NBUF];               // warps arrived on B(i) (!kProd: elects the issuer)
  __shared__ uint32_t s_tmem;
  __shared__ double s_red[2][11][8];
  const int KB = P.tc_kb, L4 = 4 * KB;
  const int T = P.T;
  const int TH = (T + 1) >> 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q4 = warp & 3;                          // TMEM lane quarter
  const int ex = (warp >> 2) & 1;                   // expert: 0 = AI, 1 = MMSE
  const int half = warp >> 3;                       // symbol half
  const int j = q4 * 32 + lane;                     // subcarrier within the tile = TMEM lane
  const int AD = P.A * ND;
  const int n_tiles = P.n_tiles;
  const int G = gridDim.x;
  // antenna groups (massive MIMO): a work item is (unit, tile, group of NA
  // antennas); CTA ranges are whole tiles so the MRC sums stay on one CTA
  const int ngrp = kGrp ? P.A / NA : 1;
  const int AS = kGrp ? NA : P.A;  // antennas per shared-memory stage
  const int n_titems = n_items / ngrp;
  const int lo = (int)((long long)blockIdx.x * n_titems / G) * ngrp;
  const int hi = (int)((long long)(blockIdx.x + 1) * n_titems / G) * ngrp;
  const uint32_t b_bytes = (uint32_t)KB * NG * 256;
  // a stage holds the item's y rows and (one antenna group per item: massive
  // MIMO) the tile's tx rows live in ONE buffer next to the stages: only a tile's
  // last group reads them, and the load of the next tile's tx is issued after
  // that item's equaliser finished (the stage refill rule below)
  static_assert(!kPk || (kStd && kTmap && !kGrp), "packed tx: single-group NR-pattern plans");
  // packed tx (kPk): the tile's 2-bit codes (T x 32 B) after the y rows, padded to 512 B
  const size_t stage_elems = kPk ? (size_t)AS * T * ARCHES_TILE + 64
                                 : (size_t)(AS + (kGrp ? 0 : 1)) * T * ARCHES_TILE;
  const size_t coef_stride = coef_floats2(P);
  float2* sYX = reinterpret_cast<float2*>(sm);                               // [NST][stage]
  float2* sX = sYX + NST * stage_elems;                                       // [T][TILE] (kGrp)
  unsigned char* sB = sm + (NST * stage_elems + (kGrp ? (size_t)T * ARCHES_TILE : 0)) * sizeof(float2);
  float* gacc = reinterpret_cast<float*>(sB + 2 * NBUF * (size_t)KB * NG * 256) + threadIdx.x;  // [21][512] (kGrp)
  float2* srot = reinterpret_cast<float2*>(sB + 2 * NBUF * (size_t)KB * NG * 256 +
                                           (kGrp ? (size_t)21 * TC_THREADS * sizeof(float) : 0));  // [n_tiles][L4+8]
  const int n_all = (NCOL / 2) * L4;                                         // B entries
  const uint32_t ACC0 = 128;                                                 // TMEM columns
  // this thread's <= 2 B entries (output column pair r, tap l): source offsets
  // inside a unit's coefficients, rotation index, shared-memory offsets
  int boff[2], roff[2], gstr[2];
  bool bmm[2];
  uint32_t o0[2], o1[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int e = threadIdx.x + q * TC_THREADS;
    boff[q] = -1; roff[q] = 0; bmm[q] = false; o0[q] = o1[q] = 0; gstr[q] = 0;
    if (e < n_all) {
      const int r = e / L4, l = e - r * L4;
      o0[q] = kmaj_off(2 * r, 2 * l, NG);
      o1[q] = kmaj_off(2 * r + 1, 2 * l, NG);
      if (r < NA * ND) {
        if (r < AD && l < P.trunc) {
          boff[q] = AD * P.n_blocks * 8 + r * P.trunc + l; roff[q] = l; gstr[q] = NA * ND * P.trunc;
        }
      } else if (r < R) {
        const int ad = r - NA * ND;
        if (ad < AD && l < 8) {
          boff[q] = ad * P.n_blocks * 8 + l; roff[q] = L4 + l; bmm[q] = true; gstr[q] = NA * ND * P.n_blocks * 8;
        }
      }
    }
  }

  if (threadIdx.x == 0) {
    for (int k = 0; k < NST; ++k) mbar_init(&s_full[k], 1);
    for (int b = 0; b < NBUF; ++b) {
      mbar_init(&s_mma[b], 1);
      mbar_init(&s_bready[b], kProd ? TC_THREADS : TC_THREADS / 32);
      s_bcount[b] = 0;
    }
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        smem_u32(&s_tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  const uint32_t lane_base = tmem + ((uint32_t)(q4 * 32) << 16);

  auto issue_tma = [&](int u, int tile, int gr, int stage) {  // producer warp (all lanes)
    const uint64_t pol = l2_evict_first_policy();
    float2* dst = sYX + (size_t)stage * stage_elems;
    const bool with_x = gr == ngrp - 1;  // tx rows: needed by the last group only
    float2* xdst = kGrp ? sX : dst + (size_t)AS * T * ARCHES_TILE;
    if constexpr (kTmap) {  // lane 0: two tensor copies (y rows of the group, tx rows)
      if (lane == 0) {
        const size_t ybytes = (size_t)AS * T * ARCHES_TILE * sizeof(float2);
        const size_t xbytes = kPk ? (size_t)T * ARCHES_TXB_ROW : (size_t)T * ARCHES_TILE * sizeof(float2);
        mbar_arrive_expect_tx(&s_full[stage], (uint32_t)(with_x ? ybytes + xbytes : ybytes));
        tma_load_3d(dst, &tm_y, tile * 2 * ARCHES_TILE, gr * AS * T, u, &s_full[stage], pol);
        if constexpr (kPk)
          bulk_g2s(xdst, reinterpret_cast<const unsigned char*>(args.tx) + ((size_t)u * n_tiles + tile) * xbytes,
                   (uint32_t)xbytes, &s_full[stage], pol);
        else if (with_x)
          tma_load_3d(xdst, &tm_x, tile * 2 * ARCHES_TILE, 0, u, &s_full[stage], pol);
      }
    } else {  // one 1-D bulk copy per row, rows spread over the lanes
      const int k0 = tile * ARCHES_TILE;
      const uint32_t rowb = (uint32_t)min(ARCHES_TILE, P.N - k0) * sizeof(float2);
      const int rows = AS * T + (with_x ? T : 0);
      if (lane == 0) mbar_arrive_expect_tx(&s_full[stage], rowb * (uint32_t)rows);
      __syncwarp();
      for (int r = lane; r < rows; r += 32) {
        if (r < AS * T)
          bulk_g2s(dst + (size_t)r * ARCHES_TILE,
                   args.y + ((size_t)u * P.A * T + (size_t)gr * AS * T + r) * P.N + k0, rowb,
                   &s_full[stage], pol);
        else
          bulk_g2s(xdst + (size_t)(r - AS * T) * ARCHES_TILE,
                   args.tx + ((size_t)u * T + (r - AS * T)) * P.N + k0, rowb, &s_full[stage], pol);
      }
    }
  };
  // coefficients and the tile's phase rotation; the loads are issued one item
  // ahead and only multiplied in write_b, so their latency hides behind the
  // current item's epilogue
  auto load_b = [&](int u, int tile, int gr, float2 (&cv)[4]) {
    const float2* cu = args.coef + (size_t)u * coef_stride;
    const bool rs = P.k2_rot_smem;
    const float2* rot = (rs ? srot : P.tc_rot) + (size_t)tile * (L4 + 8);
    const int bo = P.n_blocks == 1 ? 0 : min(tile * ARCHES_TILE / P.block, P.n_blocks - 1) * 8;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      cv[2 * q] = boff[q] >= 0 ? __ldg(&cu[boff[q] + (bmm[q] ? bo : 0) + gr * gstr[q]]) : make_float2(0.f, 0.f);
      cv[2 * q + 1] = boff[q] < 0 ? make_float2(0.f, 0.f) : rs ? rot[roff[q]] : __ldg(&rot[roff[q]]);
    }
  };
  auto write_b = [&](int buf, const float2 (&cv)[4]) {
    unsigned char* bhi = sB + (size_t)buf * 2 * b_bytes;
    unsigned char* blo = bhi + b_bytes;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      if (q * TC_THREADS + (int)threadIdx.x >= n_all) break;
      const float2 c = cmul(cv[2 * q], cv[2 * q + 1]);
      const float rh = tf32_rna_fast(c.x), rl = tf32_rna_fast(c.x - rh);
      const float ih = tf32_rna_fast(c.y), il = tf32_rna_fast(c.y - ih);
      *reinterpret_cast<float2*>(bhi + o0[q]) = make_float2(rh, -ih);
      *reinterpret_cast<float2*>(bhi + o1[q]) = make_float2(ih, rh);
      *reinterpret_cast<float2*>(blo + o0[q]) = make_float2(rl, -il);
      *reinterpret_cast<float2*>(blo + o1[q]) = make_float2(il, rl);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  };
  auto issue_mma = [&](int buf) {  // lane 0 of the producer (or completing) warp, once B(buf) is written
    tc_fence_after();
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(NCOL >> 3) << 17) |
                           ((uint32_t)(ARCHES_TILE >> 4) << 24);
    const uint32_t b_hi = smem_u32(sB + (size_t)buf * 2 * b_bytes), b_lo = b_hi + b_bytes;
    const uint32_t dcol = tmem + ACC0 + 64u * buf;
    for (int kb = 0; kb < KB; ++kb) {
      const uint64_t dbh = umma_desc_kmajor(b_hi + kb * NG * 256, 128, 256);
      const uint64_t dbl = umma_desc_kmajor(b_lo + kb * NG * 256, 128, 256);
      const uint32_t ah = tmem + 8u * kb, al = tmem + 8u * KB + 8u * kb;
      umma_tf32_ts(dcol, ah, dbh, idesc, kb > 0 ? 1u : 0u);
      umma_tf32_ts(dcol, al, dbh, idesc, 1u);
      umma_tf32_ts(dcol, ah, dbl, idesc, 1u);
    }
    umma_commit(&s_mma[buf]);
  };

  // next work item after (u, tile, gr)
  auto advance = [&](int& au, int& at, int& ag) {
    if (++ag == ngrp) {
      ag = 0;
      if (++at == n_tiles) {
        at = 0;
        ++au;
      }
    }
  };
  int u = (lo / ngrp) / n_tiles, tile = (lo / ngrp) - u * n_tiles, gr = 0;
  const int count = hi - lo;
  // ---- prologue: A operand (twiddle rows) -> TMEM
  if (lo < hi) {
    if (warp < 4) {
      const float4* arow = reinterpret_cast<const float4*>(P.tc_a) + (size_t)j * (KB * 4);
      for (int c = 0; c < KB; ++c) {
        float v[16];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float4 f = __ldg(&arow[c * 4 + i]);
          v[4 * i] = f.x; v[4 * i + 1] = f.y; v[4 * i + 2] = f.z; v[4 * i + 3] = f.w;
        }
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(
                         lane_base + 8 * c),
                     "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
                     "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
                     "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7]))
                     : "memory");
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(
                         lane_base + 8 * KB + 8 * c),
                     "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])),
                     "r"(__float_as_uint(v[11])), "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])),
                     "r"(__float_as_uint(v[14])), "r"(__float_as_uint(v[15]))
                     : "memory");
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
  }
  if (P.k2_rot_smem && threadIdx.x < TC_THREADS)
    for (int i = threadIdx.x; i < n_tiles * (L4 + 8); i += TC_THREADS) srot[i] = __ldg(&P.tc_rot[i]);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  if (kProd && warp == TC_THREADS / 32) {
    // ---------------- producer / MMA warp.  B(j) written means the epilogue of
    // item j - LEAD is finished: MMA(j) goes out (its accumulator was read by
    // item j - NBUF), and the stage item j - LEAD used is refilled with item
    // j - LEAD + 2.  The epilogue warps never meet at a CTA barrier for this.
    int tu = u, tt = tile, tg = gr;  // next item to load
    for (int k = 0; k < NST && k < count; ++k) {
      issue_tma(tu, tt, tg, k);
      advance(tu, tt, tg);
    }
    for (int jj = 0; jj < count; ++jj) {
      mbar_wait(&s_bready[jj % NBUF], (jj / NBUF) & 1);
      if (lane == 0) issue_mma(jj % NBUF);
      __syncwarp();
      const int nx = jj - LEAD + NST;
      if (nx >= NST && nx < count) {
        issue_tma(tu, tt, tg, nx % NST);
        advance(tu, tt, tg);
      }
    }
  } else {
  if (!kProd && warp == 0) {  // the first two items' y / tx rows
    int tu = u, tt = tile, tg = gr;
    for (int k = 0; k < 2 && k < count; ++k) {
      issue_tma(tu, tt, tg, k);
      advance(tu, tt, tg);
    }
  }
  // B(jj) of item (bu, bt, bg) written by this thread.  !kProd: each warp arrives
  // on the buffer's mbarrier (release) and bumps a relaxed counter that elects
  // the 16th warp, which waits for the phase (acquire, completes at once) and
  // issues MMA(jj) (its accumulator was read by item jj - NBUF, whose readers
  // have all arrived) and the refill of the stage item jj - LEAD used
  auto arrive_b = [&](int jj, int bu, int bt, int bg) {
    tc_fence_before();
    if constexpr (kProd) {
      mbar_arrive(&s_bready[jj % NBUF]);
    } else {
      __syncwarp();
      uint32_t old = 0;
      if (lane == 0) {
        mbar_arrive(&s_bready[jj % NBUF]);
        old = atomicAdd(&s_bcount[jj % NBUF], 1u);
      }
      old = __shfl_sync(0xffffffffu, old, 0);
      if ((old & (TC_THREADS / 32 - 1)) == TC_THREADS / 32 - 1) {
        mbar_wait_spin(&s_bready[jj % NBUF], (jj / NBUF) & 1);
        if (lane == 0) issue_mma(jj % NBUF);
        __syncwarp();
        if (jj >= 2 && jj < count) issue_tma(bu, bt, bg, jj & 1);
      }
    }
  };
  // programmatic dependent launch behind the K1 finalize: the prologue above (TMEM,
  // twiddle operand, phase table) and the producer's y / tx loads overlap its tail;
  // the coefficients it writes are read only after its grid completed
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (lo < hi) {  // B of the first LEAD items
    int bu = u, bt = tile, bg = gr;
    for (int k = 0; k < LEAD && k < count; ++k) {
      float2 cv[4];
      load_b(bu, bt, bg, cv);
      write_b(k, cv);
      arrive_b(k, bu, bt, bg);
      advance(bu, bt, bg);
    }
  }
  // the item LEAD ahead of the current one (its B operand is written this iteration)
  int lu = u, lt = tile, lg = gr;
  for (int k = 0; k < LEAD; ++k) advance(lu, lt, lg);

  // per-thread telemetry sums, kept across the tiles of one unit
  float sa = 0.f, sp = 0.f, sre = 0.f, sim = 0.f, syy = 0.f, sxx = 0.f;
  int seg_t0 = tile;  // first tile of the current (CTA, unit) segment
  float nv = lo < hi ? (float)__ldg(&args.nv[u]) : 0.f;
  for (int item = lo, i = 0; item < hi; ++item, ++i) {
    const int buf = i % NST, ph = (i / NST) & 1;    // y / tx stage
    const int mb = i % NBUF, mph = (i / NBUF) & 1;  // B operand + TMEM accumulator
    const bool has_next = item + 1 < hi;
    const bool has_lead = item + LEAD < hi;
    const bool last_grp = gr + 1 == ngrp;
    const bool last_tile = tile + 1 == n_tiles && last_grp;  // last item of the unit
    const int gn = last_grp ? 0 : gr + 1;
    const int tn = last_grp ? (tile + 1 == n_tiles ? 0 : tile + 1) : tile;
    const int un = last_tile ? u + 1 : u;
    const bool flush = last_tile || !has_next;
    const int k0 = tile * ARCHES_TILE;
    const int kk = k0 + j;
    const bool valid = kk < P.N;
    // ---- next item's data + coefficients in flight during this item's work
    float2 cv[4];
    if (has_lead) load_b(lu, lt, lg, cv);
    // ---- this expert's synthesised taps
    mbar_wait(&s_mma[mb], mph);
    tc_fence_after();
    float vals[CPE];
    tmem_ld_n<CPE>(lane_base + ACC0 + 64u * mb + (uint32_t)(ex * CPE), vals);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    float2 h[NA][ND];
#pragma unroll
    for (int a = 0; a < NA; ++a)
#pragma unroll
      for (int d = 0; d < ND; ++d)
        h[a][d] = make_float2(vals[2 * (a * ND + d)], vals[2 * (a * ND + d) + 1]);
    float2* hout = ex ? args.h_mmse : args.h_ai;
    // expert outputs: streaming stores (written once, never re-read by this
    // step -- keeps them from evicting the y / tx lines still in flight)
    if (valid && half == 0 && hout) {  // half 0 stores the expert output ...
      float2* o = hout + ((size_t)u * AD + (size_t)gr * NA * ND) * P.N + kk;
#pragma unroll
      for (int a = 0; a < NA; ++a)
        if (kStd || a < P.A)
#pragma unroll
          for (int d = 0; d < ND; ++d) __stcs(&o[(size_t)(a * ND + d) * P.N], h[a][d]);
    }
    if (valid && half == 1) {  // ... half 1 forms its |H| telemetry
#pragma unroll
      for (int a = 0; a < NA; ++a)
#pragma unroll
        for (int d = 0; d < ND; ++d) {
          const float p2 = fmaf(h[a][d].x, h[a][d].x, h[a][d].y * h[a][d].y);
          float r;
          asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(p2));
          sa += r;
          sp += p2;
        }
    }
    // ---- equaliser over this thread's symbol half
    mbar_wait(&s_full[buf], ph);
    if (valid) {
      const float modd = (kk & 1) ? 1.f : 0.f;  // pilot REs: even k on DMRS symbols
      const float2* yrow = sYX + (size_t)buf * stage_elems + j;
      const float2* xrow = kGrp ? sX + j : yrow + (size_t)AS * T * ARCHES_TILE;
      if constexpr (kGrp) {  // antenna groups: MRC sums across the tile's groups, finalised at the last
        const bool first = gr == 0, last = gr + 1 == ngrp;
        // |x|^2 is accumulated by both experts' threads (only expert 0's is reduced):
        // one instantiation per half keeps the loop body in the instruction cache
        if (half == 0) eq_grp_half<NA, ND, 0, true>(h, yrow, xrow, modd, nv, gacc, first, last, sre, sim, syy, sxx);
        else           eq_grp_half<NA, ND, 1, true>(h, yrow, xrow, modd, nv, gacc, first, last, sre, sim, syy, sxx);
      } else if constexpr (kStd) {  // compile-time symbol half and expert: weights and pilot symbols fold
        const unsigned char* xb = reinterpret_cast<const unsigned char*>(xrow - j) + (j >> 2);
        const int jsh = (j & 3) * 2;
        if (half == 0) eq_std_half<NA, ND, 0, true, kPk>(h, yrow, xrow, xb, jsh, modd, nv, sre, sim, syy, sxx);
        else           eq_std_half<NA, ND, 1, true, kPk>(h, yrow, xrow, xb, jsh, modd, nv, sre, sim, syy, sxx);
      } else {
        const int t0 = half ? TH : 0, t1 = half ? T : TH;
        for (int t = t0; t < t1; ++t) {
          float wt[ND];
#pragma unroll
          for (int d = 0; d < ND; ++d) wt[d] = P.tw[t][d];
          float2 yv[NA];
#pragma unroll
          for (int a = 0; a < NA; ++a)
            yv[a] = (a < P.A) ? yrow[(size_t)(a * T + t) * ARCHES_TILE] : make_float2(0.f, 0.f);
          const float2 x = xrow[(size_t)t * ARCHES_TILE];
          const float m = (P.is_dmrs[t] >= 0) ? modd : 1.f;
          eq_re<NA, ND>(h, wt, yv, x, m, nv, sre, sim, syy);
          if (ex == 0) sxx = fmaf(m * x.x, x.x, fmaf(m * x.y, x.y, sxx));
        }
      }
    }
    // ---- end of a (CTA, unit) segment: per-warp partials -> s_red[i & 1] (item parity)
    if (flush) {
      const int col = half * 4 + q4;
      const double r2 = warp_sum((double)sre), r3 = warp_sum((double)sim);
      const double r4 = warp_sum((double)syy);
      double r0 = 0.0, r1 = 0.0, r5 = 0.0;
      if (half == 1) {
        r0 = warp_sum((double)sa);
        r1 = warp_sum((double)sp);
      }
      if (ex == 0) r5 = warp_sum((double)sxx);
      if (lane == 0) {
        if (half == 1) {
          s_red[i & 1][0 + ex][q4] = r0;
          s_red[i & 1][2 + ex][q4] = r1;
        }
        if (ex == 0) s_red[i & 1][4][col] = r5;
        s_red[i & 1][5 + ex][col] = r2;
        s_red[i & 1][7 + ex][col] = r3;
        s_red[i & 1][9 + ex][col] = r4;
      }
      sa = sp = sre = sim = syy = sxx = 0.f;
      named_bar(1, TC_THREADS);  // every warp's partials in s_red[i & 1]
    }
    // ---- B(i + LEAD) -> shared memory; signals the producer / MMA warp
    if (has_lead) {
      write_b((i + LEAD) % NBUF, cv);
      arrive_b(i + LEAD, lu, lt, lg);
    }
    // ---- segment partial (fixed order); per-unit finalisation runs in K3
    if (flush && warp == 1 && lane < 11) {
      double acc;
      if (lane < 4) {  // abs / pow: half 1 only
        acc = ((s_red[i & 1][lane][0] + s_red[i & 1][lane][1]) + s_red[i & 1][lane][2]) + s_red[i & 1][lane][3];
      } else {
        acc = 0.0;
        for (int w = 0; w < 8; ++w) acc += s_red[i & 1][lane][w];
      }
      reinterpret_cast<double*>(args.parts + (size_t)u * n_tiles + seg_t0)[lane] = acc;
    }
    if (last_tile) {
      seg_t0 = 0;
      if (has_next) nv = (float)__ldg(&args.nv[un]);
    }
    u = un;
    tile = tn;
    gr = gn;
    advance(lu, lt, lg);
  }
  }  // epilogue warps
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// K3 -- per-unit finalisation for the tensor-core K2, one warp per unit: lanes
// fetch the (CTA, unit) segment partials in parallel, the sum runs in tile
// order (segments only -- the other tiles hold no partial), then lanes 0 / 1
// derive the AI / MMSE candidate (link adaptation, TB, CRC, MAC split).
#define K3_THREADS 128
__global__ void __launch_bounds__(K3_THREADS) k3_finalize(const PlanDev P, const K2Args args,
                                                          int n_units, int n_items, int G) {
  const int u = (int)((blockIdx.x * (unsigned)K3_THREADS + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (u >= n_units) return;  // warp-uniform
  double acc[11];
#pragma unroll
  for (int i = 0; i < 11; ++i) acc[i] = 0.0;
  for (int t0 = 0; t0 < P.n_tiles; t0 += 32) {
    const int t = t0 + lane;
    const bool seg = t < P.n_tiles && k2_segment_start(u * P.n_tiles + t, P.n_tiles, n_items, G);
    double v[11];
    const double* p = reinterpret_cast<const double*>(args.parts + (size_t)u * P.n_tiles + t);
#pragma unroll
    for (int i = 0; i < 11; ++i) v[i] = seg ? p[i] : 0.0;
    unsigned int m = __ballot_sync(0xffffffffu, seg);
    while (m) {  // ascending tile order, identical on every lane
      const int src = __ffs(m) - 1;
      m &= m - 1;
#pragma unroll
      for (int i = 0; i < 11; ++i) acc[i] += __shfl_sync(0xffffffffu, v[i], src);
    }
  }
  if (lane >= 2) return;
  const int e = lane;  // 0 = AI, 1 = MMSE
  const int stream = u / args.n_slots;
  const double* rng = args.rng ? args.rng + 2 * u : nullptr;
  double u_crc, frac;
  if (rng) {
    u_crc = rng[0];
    frac = rng[1];
  } else {
    const long long base = args.first_slot >= 0
        ? args.first_slot
        : (long long)*reinterpret_cast<const int64_t*>(args.state + (size_t)stream * args.state_stride);
    const long long slot = base + (u - stream * args.n_slots);
    u_crc = arches_rng::stream_first_uniform(args.seeds ? args.seeds[stream] : 0ull, P.crc_key,
                                             (uint64_t)slot);
    frac = lcid4_frac(P, slot);
  }
  const double cnt = (double)P.A * P.D * P.N;
  arches_telemetry* tel = args.tel + u;
  if (e == 0) tel->sigma2_hat = args.sigma2 ? args.sigma2[u] : 0.0;
  tel->abs_mean[e] = acc[0 + e] / cnt;
  tel->rsrp[e] = acc[2 + e] / cnt;
  const double sinr = sinr_from_sums(acc[4], acc[5 + e], acc[7 + e], acc[9 + e], P.sinr_cap_db);
  tel->sinr_db[e] = sinr;
  int mcs, tb, ncb, crc, mac_rx, l4_rx;
  kpm_candidate(P, sinr, u_crc, frac, mcs, tb, ncb, crc, mac_rx, l4_rx);
  tel->mcs[e] = mcs;
  tel->tb_bytes[e] = tb;
  tel->num_cb[e] = ncb;
  tel->crc[e] = crc;
  tel->mac_rx[e] = mac_rx;
  tel->lcid4_rx[e] = l4_rx;
}
