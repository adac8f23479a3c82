// K2 (tensor-core form) -- expert synthesis on tcgen05 + switch telemetry +
// equaliser.  One CTA (8 warps) per (unit, 128-subcarrier tile):
//   * warp 0 issues cp.async.bulk (TMA) copies of the tile's y (A*T rows) and
//     tx (T rows) into shared memory at entry; they land while the synthesis runs;
//   * warps 0..3 write their TMEM lanes' rows of the twiddle operand
//     S[j][2l] = cos(-2 pi l j/N), S[j][2l+1] = sin(-2 pi l j/N) (hi | lo split,
//     from a pre-split plan table) with tcgen05.st -- A operand in TMEM;
//   * all threads build B, the real embedding of both experts' complex taps
//     rotated to the tile origin (hi | lo), in shared memory (UMMA K-major);
//   * one thread issues D[128 x 4AD] = S_hi B_hi + S_lo B_hi + S_hi B_lo
//     (tcgen05.mma kind::tf32, A from TMEM, fp32-accurate 3xTF32) and commits;
//   * thread = (subcarrier j = TMEM lane, expert = warp / 4): tcgen05.ld of its
//     expert's taps, output stores, |H| telemetry, time interpolation + MRC
//     equaliser (compile-time weights for the NR 0/5/10 pattern), fp32
//     per-thread SINR partial sums reduced in fp64, last-CTA finalisation.
#pragma once
#include "common.cuh"
#include "k_synth_eq.cuh"

#define TC_THREADS 256

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

__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
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
      if (wt[d] != 0.f) {  // folds away for compile-time weights
        hn.x = fmaf(wt[d], h[a][d].x, hn.x);
        hn.y = fmaf(wt[d], h[a][d].y, hn.y);
      }
    }
    num.x = fmaf(hn.x, yv[a].x, fmaf(hn.y, yv[a].y, num.x));
    num.y = fmaf(hn.x, yv[a].y, fmaf(-hn.y, yv[a].x, num.y));
    den = fmaf(hn.x, hn.x, fmaf(hn.y, hn.y, den));
  }
  const float inv = __frcp_rn(den + nv) * m;  // m = 0 on pilot REs
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

// TMEM columns: [0, 4KB) S_hi, [4KB, 8KB) S_lo ... rounded: A_hi at 0, A_lo at 64 - 8KB? keep simple:
//   S_hi  cols [0, 8*KB)      S_lo cols [8*KB, 16*KB)      D cols [16*KB, 16*KB + NCOL)
template <int NA, int ND, bool kStd>
__global__ void __launch_bounds__(TC_THREADS)
    k2_tc(const PlanDev P, const K2Args args, const int n_items) {
  constexpr int R = 2 * NA * ND;                    // complex outputs: AI then MMSE
  constexpr int NCOL = ((2 * R + 15) / 16) * 16;    // MMA N (real columns)
  constexpr int NG = NCOL / 8;
  constexpr int CPE = 2 * NA * ND;                  // D columns per expert
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t s_bar[2];        // [0] y/tx landed, [1] MMA done
  __shared__ uint32_t s_tmem;
  __shared__ double s_red[11][8];
  __shared__ int s_flag;
  const int KB = P.tc_kb;
  const int T = P.T;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ex = warp >> 2;                         // expert of this warp: 0 = AI, 1 = MMSE
  const int q4 = warp & 3;                          // TMEM lane quarter
  const int j = q4 * 32 + lane;                     // subcarrier within the tile = TMEM lane
  const int u = blockIdx.y, tile = blockIdx.x;
  const int k0 = tile * ARCHES_TILE;
  const int kk = k0 + j;
  const bool valid = kk < P.N;
  const int ncol = min(ARCHES_TILE, P.N - k0);
  const int AD = P.A * ND;
  const uint32_t b_bytes = (uint32_t)KB * NG * 256;
  float2* sYX = reinterpret_cast<float2*>(sm);                      // [(A+1)*T][TILE]
  unsigned char* sB = sm + (size_t)(P.A + 1) * T * ARCHES_TILE * sizeof(float2);  // [hi | lo]

  if (threadIdx.x == 0) {
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(
        smem_u32(&s_tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  // ---- y / tx tile -> shared memory (TMA), in flight during the synthesis
  if (warp == 0) {
    const uint32_t rowb = (uint32_t)ncol * sizeof(float2);
    const int rows = (P.A + 1) * T;
    if (lane == 0) mbar_arrive_expect_tx(&s_bar[0], rowb * rows);
    __syncwarp();
    const uint64_t pol = l2_evict_first_policy();
    for (int r = lane; r < rows; r += 32) {
      const float2* src = (r < P.A * T) ? args.y + ((size_t)u * P.A * T + r) * P.N + k0
                                        : args.tx + ((size_t)u * T + (r - P.A * T)) * P.N + k0;
      bulk_g2s(sYX + (size_t)r * ARCHES_TILE, src, rowb, &s_bar[0], pol);
    }
  }
  // ---- A operand rows (this lane's subcarrier) -> TMEM, from the pre-split table
  if (ex == 0) {
    const float4* arow = reinterpret_cast<const float4*>(P.tc_a) + (size_t)j * (KB * 4);  // 16*KB floats
    const uint32_t lane_base = tmem + ((uint32_t)(q4 * 32) << 16);
    for (int c = 0; c < KB; ++c) {  // 16 floats per step: 8 hi (cols 8c..) + 8 lo
      float v[16];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float4 f = __ldg(&arow[c * 4 + i]);
        v[4 * i] = f.x; v[4 * i + 1] = f.y; v[4 * i + 2] = f.z; v[4 * i + 3] = f.w;
      }
      // v[0..7] = S_hi[j][8c .. 8c+7], v[8..15] = S_lo[j][8c .. 8c+7]
      float hi8[16], lo8[16];
#pragma unroll
      for (int i = 0; i < 8; ++i) { hi8[i] = v[i]; lo8[i] = v[8 + i]; }
#pragma unroll
      for (int i = 8; i < 16; ++i) { hi8[i] = 0.f; lo8[i] = 0.f; }
      (void)hi8; (void)lo8;
      // store as two x8 groups: hi at column 8c, lo at column 8KB + 8c
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
  // ---- B operand: both experts' taps rotated to the tile origin (hi | lo)
  {
    for (uint32_t i = threadIdx.x; i < 2 * b_bytes / 4; i += blockDim.x)
      reinterpret_cast<float*>(sB)[i] = 0.f;
    __syncthreads();
    const float2* cm = args.coef + (size_t)u * coef_floats2(P);
    const float2* ca = cm + (size_t)AD * P.n_blocks * 8;
    const int rstride = 4 * KB + 8;
    const float2* rot = P.tc_rot + (size_t)tile * rstride;
    const int b = min(k0 / P.block, P.n_blocks - 1);
    unsigned char* bhi = sB;
    unsigned char* blo = sB + b_bytes;
    const int n_ai = AD * P.trunc, n_all = n_ai + AD * 8;
    for (int e = threadIdx.x; e < n_all; e += blockDim.x) {
      int r, l;
      float2 c, w;
      if (e < n_ai) {
        const int ad = e / P.trunc;
        l = e - ad * P.trunc;
        r = ad;
        c = __ldg(&ca[e]);
        w = __ldg(&rot[l]);
      } else {
        const int e2 = e - n_ai, ad = e2 >> 3;
        l = e2 & 7;
        r = NA * ND + ad;
        c = __ldg(&cm[((size_t)ad * P.n_blocks + b) * 8 + l]);
        w = __ldg(&rot[4 * KB + l]);
      }
      c = cmul(c, w);
      const float rh = tf32_rna(c.x), rl = tf32_rna(c.x - rh);
      const float ih = tf32_rna(c.y), il = tf32_rna(c.y - ih);
      const uint32_t o0 = kmaj_off(2 * r, 2 * l, NG), o1 = kmaj_off(2 * r + 1, 2 * l, NG);
      *reinterpret_cast<float2*>(bhi + o0) = make_float2(rh, -ih);
      *reinterpret_cast<float2*>(bhi + o1) = make_float2(ih, rh);
      *reinterpret_cast<float2*>(blo + o0) = make_float2(rl, -il);
      *reinterpret_cast<float2*>(blo + o1) = make_float2(il, rl);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  // ---- MMA: D = S_hi B_hi + S_lo B_hi + S_hi B_lo
  const uint32_t d_col = 16u * KB;
  if (threadIdx.x == 0) {
    tc_fence_after();
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(NCOL >> 3) << 17) |
                           ((uint32_t)(ARCHES_TILE >> 4) << 24);
    const uint32_t b_hi = smem_u32(sB), b_lo = b_hi + b_bytes;
    for (int kb = 0; kb < KB; ++kb) {
      const uint64_t dbh = umma_desc_kmajor(b_hi + kb * NG * 256, 128, 256);
      const uint64_t dbl = umma_desc_kmajor(b_lo + kb * NG * 256, 128, 256);
      const uint32_t ah = tmem + 8u * kb, al = tmem + 8u * KB + 8u * kb;
      umma_tf32_ts(tmem + d_col, ah, dbh, idesc, kb > 0 ? 1u : 0u);
      umma_tf32_ts(tmem + d_col, al, dbh, idesc, 1u);
      umma_tf32_ts(tmem + d_col, ah, dbl, idesc, 1u);
    }
    umma_commit(&s_bar[1]);
  }
  // ---- this thread's expert taps
  mbar_wait(&s_bar[1], 0);
  tc_fence_after();
  float vals[CPE];
  tmem_ld_n<CPE>(tmem + ((uint32_t)(q4 * 32) << 16) + d_col + (uint32_t)(ex * CPE), vals);
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  float2 h[NA][ND];
#pragma unroll
  for (int a = 0; a < NA; ++a)
#pragma unroll
    for (int d = 0; d < ND; ++d)
      h[a][d] = make_float2(vals[2 * (a * ND + d)], vals[2 * (a * ND + d) + 1]);
  float sa = 0.f, sp = 0.f, sre = 0.f, sim = 0.f, syy = 0.f, sxx = 0.f;
  float2* hout = ex ? args.h_mmse : args.h_ai;
  if (valid) {
    if (hout) {
      const size_t ob = (size_t)u * AD * P.N + kk;
#pragma unroll
      for (int a = 0; a < NA; ++a)
        if (a < P.A)
#pragma unroll
          for (int d = 0; d < ND; ++d) hout[ob + (size_t)(a * ND + d) * P.N] = h[a][d];
    }
#pragma unroll
    for (int a = 0; a < NA; ++a)
#pragma unroll
      for (int d = 0; d < ND; ++d) {
        const float p2 = fmaf(h[a][d].x, h[a][d].x, h[a][d].y * h[a][d].y);
        sa += sqrtf(p2);
        sp += p2;
      }
  }
  // ---- equaliser from the staged tile
  mbar_wait(&s_bar[0], 0);
  if (valid) {
    const float nv = (float)__ldg(&args.nv[u]);
    const float modd = (kk & 1) ? 1.f : 0.f;  // pilot REs: even k on DMRS symbols
    const float2* yrow = sYX + j;
    const float2* xrow = sYX + (size_t)P.A * T * ARCHES_TILE + j;
    if (kStd) {
#pragma unroll
      for (int t = 0; t < 14; ++t) {
        float wt[ND];
#pragma unroll
        for (int d = 0; d < ND; ++d) wt[d] = std_tw(t, d);
        float2 yv[NA];
#pragma unroll
        for (int a = 0; a < NA; ++a)
          yv[a] = (a < P.A) ? yrow[(size_t)(a * 14 + t) * ARCHES_TILE] : make_float2(0.f, 0.f);
        const float2 x = xrow[(size_t)t * ARCHES_TILE];
        const float m = (t == 0 || t == 5 || t == 10) ? modd : 1.f;
        eq_re<NA, ND>(h, wt, yv, x, m, nv, sre, sim, syy);
        if (ex == 0) sxx = fmaf(m * x.x, x.x, fmaf(m * x.y, x.y, sxx));
      }
    } else {
      for (int t = 0; t < T; ++t) {
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
  // ---- tile partials (fixed order) + last-CTA finalisation
  {
    const double r0 = warp_sum((double)sa), r1 = warp_sum((double)sp);
    const double r2 = warp_sum((double)sre), r3 = warp_sum((double)sim);
    const double r4 = warp_sum((double)syy), r5 = warp_sum((double)sxx);
    if (lane == 0) {
      for (int i = 0; i < 11; ++i) s_red[i][warp] = 0.0;
      s_red[0 + ex][warp] = r0;
      s_red[2 + ex][warp] = r1;
      s_red[4][warp] = r5;
      s_red[5 + ex][warp] = r2;
      s_red[7 + ex][warp] = r3;
      s_red[9 + ex][warp] = r4;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 11) {
    double acc = 0.0;
    for (int w = 0; w < 8; ++w) acc += s_red[threadIdx.x][w];
    reinterpret_cast<double*>(args.parts + (size_t)u * gridDim.x + tile)[threadIdx.x] = acc;
  }
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
  }
  if (last_block_arrive(args.counters + u, gridDim.x, &s_flag) && threadIdx.x == 0) {
    const int stream = u / args.n_slots;
    const long long base = args.first_slot >= 0
        ? args.first_slot
        : (long long)*reinterpret_cast<const int64_t*>(args.state + (size_t)stream * args.state_stride);
    const long long slot = base + (u - stream * args.n_slots);
    arches_telemetry tel;
    finalize_unit(P, args.parts + (size_t)u * gridDim.x, gridDim.x,
                  args.sigma2 ? args.sigma2 + u : nullptr, args.seeds ? args.seeds[stream] : 0ull,
                  slot, 2, &tel, args.rng ? args.rng + 2 * u : nullptr);
    args.tel[u] = tel;
  }
  (void)n_items;
}
