// K1 (tensor-core form) -- the 20-bin comb analysis of every (unit, antenna,
// DMRS symbol) row as a tcgen05 contraction, for single-block plans.
//
// Replaces the analysis half of ls_estimate / estimate_noise_var /
// mmse_estimate / denoiser_estimate (expert_bank.py:96-214):
//   B[u,a,d][l] = sum_m h[u,a,d][m] e^{+2 pi i l m / M},  h = y[.., 2m, dmrs_d] conj(p) / |p|^2
// written as  D[row][n] = sum_kappa A[row][kappa] W[kappa][n]  with
//   row   = u*A + a (128 rows per tile = 128/A units),
//   kappa = real embedding of the subcarriers (odd subcarriers meet zero
//           twiddles, so the raw grid rows are the operand, no gather),
//   n     = 2l + re/im (N = 2L padded to 16).
// Work item = (row tile g, DMRS symbol d, subcarrier part q); a CTA walks its
// items in chunks of 16 subcarriers (8 comb points starting at m0 = 8c):
//   D_c[row][l] = e^{2 pi i l m0/M} sum_{k<8} h[m0+k] e^{2 pi i l k/M}
// so the MMA operand W (k < 8, real-embedded, tf32 hi | lo) is the same for
// every chunk and stays in shared memory; the chunk's phase is applied to the
// 2L outputs in the epilogue.
//   * producer warp: one 2-D tensor TMA per chunk lands the raw DMRS row
//     segments of 128 rows (128 B each) in the UMMA K-major SWIZZLE_128B layout
//     (16-byte group g of row r at r*128 + (g ^ (r & 7))*16) in an 8-deep ring;
//   * converter warps (thread = row = TMEM lane): h = y conj(p)/|p|^2 on the
//     comb subcarriers, zero on the odd ones, tf32 hi | lo split into one of two
//     MMA operand buffers (the raw stage is released right away);
//   * MMA warp: D_c = A_hi W_hi + A_lo W_hi + A_hi W_lo (kind::tf32, 3xTF32)
//     into a ring of TMEM accumulators;
//   * converter warps, two chunks behind: tcgen05.ld of the row's 2L columns,
//     the chunk phase, fp32 sums over 4 chunks folded into fp64 (short fp32
//     chains keep the Parseval noise estimate precise); at the item end the
//     partial bins (fp64) and the row energy go to global memory.
#pragma once
#include "k_analyze.cuh"
#include "k_synth_tc.cuh"

#define K1T_CONV_WARPS 4                         // converters: warps 0-3, drains: warps 4-7
#define K1T_THREADS (32 * (2 * K1T_CONV_WARPS + 2))  // + producer + MMA warp
#define K1T_MAX_CHUNKS 112                       // phase table in shared memory (N <= 3584)
#define K1T_STAGES 4                             // raw grid stages
#define K1T_MBUF 2                               // MMA operand buffers
#define K1T_CSC 32                               // subcarriers per chunk (2 x 128-B TMA boxes)
#define K1T_CP (K1T_CSC / 2)                     // comb points per chunk (one 128-B operand row)
#define K1T_ACC 4                                // TMEM accumulator ring

struct K1TArgs {
  const float2* pil;       // [stream][M][D]
  const float* wimg;       // [hi | lo][NB rows][128 B, SWIZZLE_128B] twiddle operand, chunk-invariant
  const float2* rot;       // [n_chunks][L] chunk phases e^{2 pi i l 8c / M}
  double* dpart;           // [item][128][2L] partial bins (fp64)
  double* epart;           // [item][128] row energies
  int n_slots, n_rows;     // rows = units * A
  int n_g, parts, cpp;     // row tiles, subcarrier parts, chunks per part
  int n_chunks, nb;        // chunks per row, MMA N
};

// RNG side products of each unit (Philox CRC uniform of rng.stream(seed, "crc",
// slot), LCID4 split of _lcid4_jitter(slot); rng.py:24-34, phy_pipeline.py:
// 217-222,347-350): one thread per unit.  Independent of the grid, so
// arches_run_batch runs it on a forked stream next to K1.
__global__ void k_rng_units(const PlanDev P, double* rng, const uint64_t* seeds,
                            const unsigned char* state, size_t state_stride, long long first_slot,
                            int n_slots, int n_units) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= n_units) return;
  const int stream = u / n_slots;
  const long long base = first_slot >= 0
      ? first_slot
      : (long long)*reinterpret_cast<const int64_t*>(state + (size_t)stream * state_stride);
  const long long slot = base + (u - stream * n_slots);
  rng[2 * u] = arches_rng::stream_first_uniform(seeds[stream], P.crc_key, (uint64_t)slot);
  const double jit = arches_rng::lcid4_jitter((uint64_t)slot);
  const double f = __dadd_rn(P.lcid4_fraction, __dmul_rn(P.lcid4_jitter, jit));
  rng[2 * u + 1] = fmin(fmax(f, 0.0), 1.0);
}

constexpr uint32_t K1T_ATOM = 128 * 128;           // 128 rows x 128 B (one SWIZZLE_128B K block)
constexpr uint32_t K1T_RAW_BYTES = 2 * K1T_ATOM;    // raw chunk: 32 subcarriers of 128 rows
constexpr uint32_t K1T_OP_BYTES = K1T_ATOM;         // compacted operand: 16 comb points of 128 rows

// K-major SWIZZLE_128B shared-memory descriptor (8-row atoms of 128 B, 1024-B aligned)
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1 << 16;            // LBO: unused for swizzled K-major
  d |= (uint64_t)(1024 >> 4) << 32;  // SBO: 8-row atom stride
  d |= (uint64_t)1 << 46;            // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;            // SWIZZLE_128B
  return d;
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      ".L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

__host__ __device__ inline size_t k1t_smem_bytes(int nb) {
  return (size_t)K1T_STAGES * K1T_RAW_BYTES + (size_t)K1T_MBUF * 2 * K1T_OP_BYTES +
         (size_t)nb * 128 * 2 + (size_t)K1T_MAX_CHUNKS * 20 * sizeof(float2);
}

template <int NB, int LC>
__global__ void __launch_bounds__(K1T_THREADS, 1)
    k1_tc(const PlanDev P, const K1TArgs a, const int n_items,
          const __grid_constant__ CUtensorMap tm0, const __grid_constant__ CUtensorMap tm1,
          const __grid_constant__ CUtensorMap tm2, const __grid_constant__ CUtensorMap tm3) {
  extern __shared__ __align__(1024) unsigned char sm1k[];
  __shared__ __align__(8) uint64_t s_full[K1T_STAGES], s_empty[K1T_STAGES];
  __shared__ __align__(8) uint64_t s_conv[K1T_MBUF], s_mfree[K1T_MBUF], s_w;
  __shared__ __align__(8) uint64_t s_accf[K1T_ACC], s_acce[K1T_ACC];
  __shared__ uint32_t s_tmem;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int nb = NB;
  constexpr uint32_t w_bytes = (uint32_t)nb * 128;
  const int NT = 32 * K1T_CONV_WARPS;
  const int G = gridDim.x;
  const int cpp = a.cpp;
  unsigned char* raw = sm1k;                                            // [STAGES][2 atoms]
  unsigned char* mbuf = sm1k + (size_t)K1T_STAGES * K1T_RAW_BYTES;      // [MBUF][hi | lo]
  unsigned char* wbuf = mbuf + (size_t)K1T_MBUF * 2 * K1T_OP_BYTES;   // [hi | lo]
  float2* rotsm = reinterpret_cast<float2*>(wbuf + 2 * w_bytes);      // [n_chunks][L] chunk phases

  if (threadIdx.x == 0) {
    if (smem_u32(sm1k) & 1023u) __trap();  // SWIZZLE_128B atoms need 1024-byte alignment
    for (int s = 0; s < K1T_STAGES; ++s) {
      mbar_init(&s_full[s], 1);
      mbar_init(&s_empty[s], NT);
    }
    for (int b = 0; b < K1T_MBUF; ++b) {
      mbar_init(&s_conv[b], NT);
      mbar_init(&s_mfree[b], 1);
    }
    mbar_init(&s_w, 1);
    for (int r = 0; r < K1T_ACC; ++r) {
      mbar_init(&s_accf[r], 1);
      mbar_init(&s_acce[r], NT);
    }
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
        smem_u32(&s_tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // the finalize (programmatic dependent launch) may be scheduled onto SMs as
  // they free up; it waits for this grid's completion before reading anything
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;

  auto item_chunks = [&](int item, int& g, int& d, int& c0, int& c1) {
    g = item % a.n_g;
    const int r = item / a.n_g;
    d = r % P.D;
    const int q = r / P.D;
    c0 = q * cpp;
    c1 = min(c0 + cpp, a.n_chunks);
  };

  if (warp == 2 * K1T_CONV_WARPS) {
    // ---------------- producer: the twiddle operand once, then raw chunks
    if (lane == 0) {
      const uint64_t pol_y = l2_evict_first_policy(), pol_w = l2_evict_last_policy();
      const uint32_t rot_bytes = (uint32_t)(a.n_chunks * P.L * sizeof(float2) + 15) & ~15u;
      mbar_arrive_expect_tx(&s_w, 2 * w_bytes + rot_bytes);
      bulk_g2s(wbuf, a.wimg, 2 * w_bytes, &s_w, pol_w);
      bulk_g2s(rotsm, a.rot, rot_bytes, &s_w, pol_w);
      int j = 0;
      for (int item = blockIdx.x; item < n_items; item += G) {
        int g, d, c0, c1;
        item_chunks(item, g, d, c0, c1);
        const CUtensorMap* tm = d == 0 ? &tm0 : d == 1 ? &tm1 : d == 2 ? &tm2 : &tm3;
        for (int c = c0; c < c1; ++c, ++j) {
          const int s = j % K1T_STAGES;
          if (j >= K1T_STAGES) {
            mbar_wait_spin(&s_empty[s], ((j / K1T_STAGES) - 1) & 1);
          }
          mbar_arrive_expect_tx(&s_full[s], K1T_RAW_BYTES);
          unsigned char* dst = raw + (size_t)s * K1T_RAW_BYTES;
          tma_load_2d(dst, tm, 2 * K1T_CSC * c, g * 128, &s_full[s], pol_y);
          tma_load_2d(dst + K1T_ATOM, tm, 2 * K1T_CSC * c + 32, g * 128, &s_full[s], pol_y);
        }
      }
    }
    return;
  }
  if (warp == 2 * K1T_CONV_WARPS + 1) {
    // ---------------- MMA issuer: chunk j -> TMEM accumulator j % K1T_ACC
    if (lane == 0) {
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(nb >> 3) << 17) |
                             ((uint32_t)(128 >> 4) << 24);
      const uint32_t wh = smem_u32(wbuf), wl = wh + w_bytes;
      mbar_wait_spin(&s_w, 0);
      int j = 0;
      for (int item = blockIdx.x; item < n_items; item += G) {
        int g, d, c0, c1;
        item_chunks(item, g, d, c0, c1);
        for (int c = c0; c < c1; ++c, ++j) {
          const int b = j % K1T_MBUF, r = j % K1T_ACC;
          {
            if (j >= K1T_ACC) mbar_wait_spin(&s_acce[r], ((j / K1T_ACC) - 1) & 1);
          }
          {
            mbar_wait_spin(&s_conv[b], (j / K1T_MBUF) & 1);
          }
          tc_fence_after();
          const uint32_t dcol = tmem + (uint32_t)(r * nb);
          const uint32_t ah = smem_u32(mbuf + (size_t)b * 2 * K1T_OP_BYTES), al = ah + K1T_OP_BYTES;
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) {  // 8 tf32 (32 B) per K step inside the atom
            const uint64_t dah = umma_desc_sw128(ah + 32 * ks), dal = umma_desc_sw128(al + 32 * ks);
            const uint64_t dwh = umma_desc_sw128(wh + 32 * ks), dwl = umma_desc_sw128(wl + 32 * ks);
            umma_tf32(dcol, dah, dwh, idesc, ks > 0 ? 1u : 0u);
            umma_tf32(dcol, dal, dwh, idesc, 1u);
            umma_tf32(dcol, dah, dwl, idesc, 1u);
          }
          umma_commit(&s_mfree[b]);  // operand buffer free once these MMAs completed
          umma_commit(&s_accf[r]);   // chunk result ready
        }
      }
    }
    return;
  }

  const int L = P.L, ncol = 2 * L;
  if (warp >= K1T_CONV_WARPS) {
    // ---------------- drain warps: thread = row = TMEM lane. Phase-rotated
    // chunk sums are added in fp32 over K1T_FGRP chunks, then folded into fp64
    // (every fp32 chain stays short, so the Parseval noise estimate keeps its
    // precision); the item's partial bins go to global memory.
    constexpr int K1T_FGRP = 4;
    static_assert(LC <= NB && LC % 2 == 0, "2L output columns within the MMA N");
    const int t = threadIdx.x - 32 * K1T_CONV_WARPS;
    const uint32_t lane_base = tmem + ((uint32_t)((warp - K1T_CONV_WARPS) * 32) << 16);
    mbar_wait_spin(&s_w, 0);  // phase table landed
    int j = 0;
    for (int item = blockIdx.x; item < n_items; item += G) {
      int g, d, c0, c1;
      item_chunks(item, g, d, c0, c1);
      const int row = g * 128 + t;
      float acc[LC];
      double acc64[LC];
#pragma unroll
      for (int q = 0; q < LC; ++q) acc[q] = 0.f, acc64[q] = 0.0;
      for (int c = c0; c < c1; ++c, ++j) {
        const int r = j % K1T_ACC;
        {
          mbar_wait_spin(&s_accf[r], (j / K1T_ACC) & 1);
        }
        tc_fence_after();
        float vals[NB];
        tmem_ld_n<NB>(lane_base + (uint32_t)(r * nb), vals);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        tc_fence_before();
        mbar_arrive(&s_acce[r]);
        const float2* ph = rotsm + (size_t)c * (LC / 2);
#pragma unroll
        for (int l = 0; l < LC / 2; ++l) {
          const float2 v = cmul(make_float2(vals[2 * l], vals[2 * l + 1]), ph[l]);
          acc[2 * l] += v.x;
          acc[2 * l + 1] += v.y;
        }
        if ((c - c0) % K1T_FGRP == K1T_FGRP - 1 || c + 1 == c1) {
#pragma unroll
          for (int q = 0; q < LC; ++q) {
            acc64[q] += (double)acc[q];
            acc[q] = 0.f;
          }
        }
      }
      if (row < a.n_rows) {
        double2* dst = reinterpret_cast<double2*>(a.dpart + ((size_t)item * 128 + t) * ncol);
#pragma unroll
        for (int q = 0; q < LC; q += 2) dst[q >> 1] = make_double2(acc64[q], acc64[q + 1]);
      }
    }
    tc_fence_before();
    asm volatile("bar.arrive 2, %0;" ::"r"(2 * NT) : "memory");  // TMEM reads done
    return;
  }

  // ---------------- converter warps: thread = row
  const int t = threadIdx.x;
  const int pD = P.D;
  // this row's SWIZZLE_128B positions of the 8 16-byte groups (byte offsets)
  const uint32_t sw = (uint32_t)(t & 7);
  uint32_t swz[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) swz[k] = ((uint32_t)k ^ sw) * 16u;
  int j = 0;
  for (int item = blockIdx.x; item < n_items; item += G) {
    int g, d, c0, c1;
    item_chunks(item, g, d, c0, c1);
    const int row = g * 128 + t;
    const bool live = row < a.n_rows;
    const int stream = live ? (row / P.A) / a.n_slots : 0;
    const float2* pl = a.pil + (size_t)stream * P.M * P.D + d;
    double e64 = 0.0;
    // comb pilots, one chunk ahead of the conversion
    float2 qn[K1T_CP];
    auto load_pilots = [&](int c) {
      const int mlim = (live && c < c1) ? min(K1T_CP, P.M - c * K1T_CP) : 0;
      const float2* pc = pl + (size_t)c * K1T_CP * pD;  // this chunk's first comb point
#pragma unroll
      for (int k = 0; k < K1T_CP; ++k) {
        qn[k] = k < mlim ? __ldg(pc) : make_float2(0.f, 0.f);
        pc += pD;
      }
    };
    load_pilots(c0);
    for (int c = c0; c < c1; ++c, ++j) {
      const int s = j % K1T_STAGES, b = j % K1T_MBUF;
      float2 qv[K1T_CP];
#pragma unroll
      for (int k = 0; k < K1T_CP; ++k) qv[k] = qn[k];
      load_pilots(c + 1);
      {
        mbar_wait_spin(&s_full[s], (j / K1T_STAGES) & 1);
      }
      {
        if (j >= K1T_MBUF) mbar_wait_spin(&s_mfree[b], ((j / K1T_MBUF) - 1) & 1);
      }
      // row t, 16-byte group k of atom a at a*16K + t*128 + (k ^ (t & 7))*16
      // (SWIZZLE_128B); group = (y[2m].re, .im, y[2m+1].re, .im), m = 16c + 8a + k
      const unsigned char* src = raw + (size_t)s * K1T_RAW_BYTES + t * 128;
      unsigned char* ah = mbuf + (size_t)b * 2 * K1T_OP_BYTES + t * 128;
      unsigned char* al = ah + K1T_OP_BYTES;
      float2 hv[K1T_CP];
      float e32 = 0.f;
#pragma unroll
      for (int k = 0; k < K1T_CP; ++k) {
        const float4 v = *reinterpret_cast<const float4*>(src + (k >> 3) * K1T_ATOM + swz[k & 7]);
        const float2 p = qv[k];
        const float n2 = p.x * p.x + p.y * p.y;
        float inv;  // 1/|p|^2 within 1 ulp (exact for the unit-modulus QPSK pilots); 0 for padding
        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(inv) : "f"(n2));
        inv = n2 > 0.f ? inv : 0.f;
        hv[k] = make_float2((p.x * v.x + p.y * v.y) * inv, (p.x * v.y - p.y * v.x) * inv);
        e32 = fmaf(hv[k].x, hv[k].x, fmaf(hv[k].y, hv[k].y, e32));
      }
      // compacted operand: group k' holds comb points 2k', 2k'+1 (tf32 hi | lo)
#pragma unroll
      for (int k = 0; k < K1T_CP / 2; ++k) {
        const float2 h0 = hv[2 * k], h1 = hv[2 * k + 1];
        const float4 hi = make_float4(tf32_rna_fast(h0.x), tf32_rna_fast(h0.y), tf32_rna_fast(h1.x),
                                      tf32_rna_fast(h1.y));
        *reinterpret_cast<float4*>(ah + swz[k]) = hi;
        // lo = h - hi is exact in fp32 (<= 14 significant bits); the MMA reads its
        // top 11, so the dropped tail is < 2^-22 |h| -- no explicit rounding needed
        *reinterpret_cast<float4*>(al + swz[k]) = make_float4(h0.x - hi.x, h0.y - hi.y, h1.x - hi.z, h1.y - hi.w);
      }
      // raw stage consumed: every loaded value has been used above, so the
      // TMA refill cannot race the shared-memory reads
      mbar_arrive(&s_empty[s]);
      e64 += (double)e32;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(&s_conv[b]);
    }
    if (live) a.epart[(size_t)item * 128 + t] = e64;
  }
  // TMEM is released once the drain warps have read their last accumulator
  named_bar(2, 2 * NT);
  tc_fence_after();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

// One CTA per unit: thread o sums output o (= (a, d, component)) over the parts
// in part order (fp64, loads in flight together); warp 0 forms sigma2
// (Parseval), then the MMSE and AI taps.
#define K1T_FIN_THREADS 512
__global__ void __launch_bounds__(K1T_FIN_THREADS) k1_tc_finalize(const PlanDev P, const K1TArgs a,
                                                                 int n_units, K1Out o) {
  __shared__ double s_bins[4096];
  __shared__ double s_e[K1T_FIN_THREADS / 32], s_g[K1T_FIN_THREADS / 32];
  // launched programmatically behind K1: wait for its grid (and its writes); K2
  // may then be scheduled as this grid drains
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int u = blockIdx.x;
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const int L = P.L, ncol = 2 * L, AD = P.A * P.D, nout = AD * ncol;
  double* acc = nout <= 4096 ? s_bins : o.parts + (size_t)u * (2 * (size_t)AD * L + 2);
  const int np = a.parts;
  const size_t pstride = (size_t)P.D * a.n_g * 128 * ncol;  // next part, same (d, g, row)
  double sg = 0.0;  // this thread's share of sum_{a,d,l<guard} |B_l|^2
  for (int o2 = tid; o2 < nout; o2 += K1T_FIN_THREADS) {
    const int ad = o2 / ncol, cc = o2 - ad * ncol;
    const int aa = ad / P.D, d = ad - aa * P.D;
    const int row = u * P.A + aa, g = row / 128, r = row - g * 128;
    const double* src = a.dpart + ((size_t)(d * a.n_g + g) * 128 + r) * ncol + cc;
    double sum = 0.0;
    for (int q0 = 0; q0 < np; q0 += 8) {
      double v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = q0 + k < np ? __ldcg(src + (size_t)(q0 + k) * pstride) : 0.0;
#pragma unroll
      for (int k = 0; k < 8; ++k) sum += v[k];
    }
    acc[o2] = sum;
    if (cc < 2 * P.guard) sg += sum * sum;
  }
  // row energies: thread = (a, d, part), every load in flight at once (a per-thread
  // loop over the parts serialises one L2 round trip per part)
  double e = 0.0;
  for (int o2 = tid; o2 < AD * np; o2 += K1T_FIN_THREADS) {
    const int ad = o2 / np, q = o2 - ad * np;
    const int aa = ad / P.D, d = ad - aa * P.D;
    const int row = u * P.A + aa, g = row / 128, r = row - g * 128;
    e += __ldcg(a.epart + (size_t)((q * P.D + d) * a.n_g + g) * 128 + r);
  }
  e = warp_sum(e);
  sg = warp_sum(sg);
  if (lane == 0) {
    s_e[w] = e;
    s_g[w] = sg;
  }
  __syncthreads();
  // sigma2 (Parseval): every thread sums the warp partials in the same order
  double et = 0.0, gt = 0.0;
#pragma unroll
  for (int k = 0; k < K1T_FIN_THREADS / 32; ++k) {
    et += s_e[k];
    gt += s_g[k];
  }
  const double nvhat = (et - gt / (double)P.M) / ((double)AD * (P.M - P.guard));
  if (tid == 0) o.sigma2[u] = nvhat;
  const double s_sg = nvhat + P.ridge;
  const double sgm = s_sg;
  const int M = P.M;
  float2* cm = o.coef + (size_t)u * coef_floats2(P);
  float2* ca = cm + (size_t)AD * 8;
  for (int o2 = tid; o2 < AD * 8; o2 += K1T_FIN_THREADS) {
    const int ad = o2 >> 3, l = o2 & 7;
    const double wl = P.pdp[l] / ((double)M * P.pdp[l] + sgm);
    cm[o2] = make_float2((float)(wl * acc[ad * ncol + 2 * l]), (float)(wl * acc[ad * ncol + 2 * l + 1]));
  }
  for (int o2 = tid; o2 < AD * P.trunc; o2 += K1T_FIN_THREADS) {
    const int ad = o2 / P.trunc, l = o2 - ad * P.trunc;
    const double2 bb = make_double2(acc[ad * ncol + 2 * l], acc[ad * ncol + 2 * l + 1]);
    const double2 c = zmul(P.ai_fac[l], bb);
    ca[o2] = make_float2((float)c.x, (float)c.y);
  }
}

// Many-antenna plans (A*D*2L bins > the 4096 the per-unit finalize stages in
// shared memory): the same arithmetic in two programmatically chained grids of
// (unit, K1T_FIN_ROWS (a, d) rows) CTAs, so a handful of units still fill the
// SMs.  Rows: each CTA sums its rows' parts into the unit's bins (global
// scratch) and its share of the row energy / guard power.  Taps: each CTA sums
// the unit's shares in chunk order (every CTA of a unit forms the same sigma2)
// and writes its rows' MMSE / AI taps.
#define K1T_FIN_ROWS 16
__global__ void __launch_bounds__(K1T_FIN_THREADS) k1_tc_finalize_rows(const PlanDev P, const K1TArgs a,
                                                                      int nchunk, K1Out o,
                                                                      double* share /*[u][nchunk][2]*/) {
  __shared__ double s_e[K1T_FIN_THREADS / 32], s_g[K1T_FIN_THREADS / 32];
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int u = blockIdx.x / nchunk, c = blockIdx.x - u * nchunk;
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const int L = P.L, ncol = 2 * L, AD = P.A * P.D;
  const int r0 = c * K1T_FIN_ROWS, r1 = min(AD, r0 + K1T_FIN_ROWS);
  double* acc = o.parts + (size_t)u * (2 * (size_t)AD * L + 2);
  const int np = a.parts;
  const size_t pstride = (size_t)P.D * a.n_g * 128 * ncol;
  double sg = 0.0;
  for (int o2 = r0 * ncol + tid; o2 < r1 * ncol; o2 += K1T_FIN_THREADS) {
    const int ad = o2 / ncol, cc = o2 - ad * ncol;
    const int aa = ad / P.D, d = ad - aa * P.D;
    const int row = u * P.A + aa, g = row / 128, r = row - g * 128;
    const double* src = a.dpart + ((size_t)(d * a.n_g + g) * 128 + r) * ncol + cc;
    double sum = 0.0;
    for (int q0 = 0; q0 < np; q0 += 8) {
      double v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = q0 + k < np ? __ldcg(src + (size_t)(q0 + k) * pstride) : 0.0;
#pragma unroll
      for (int k = 0; k < 8; ++k) sum += v[k];
    }
    __stcg(&acc[o2], sum);
    if (cc < 2 * P.guard) sg += sum * sum;
  }
  double e = 0.0;
  for (int o2 = tid; o2 < (r1 - r0) * np; o2 += K1T_FIN_THREADS) {
    const int ad = r0 + o2 / np, q = o2 % np;
    const int aa = ad / P.D, d = ad - aa * P.D;
    const int row = u * P.A + aa, g = row / 128, r = row - g * 128;
    e += __ldcg(a.epart + (size_t)((q * P.D + d) * a.n_g + g) * 128 + r);
  }
  e = warp_sum(e);
  sg = warp_sum(sg);
  if (lane == 0) {
    s_e[w] = e;
    s_g[w] = sg;
  }
  __syncthreads();
  if (tid == 0) {
    double et = 0.0, gt = 0.0;
#pragma unroll
    for (int k = 0; k < K1T_FIN_THREADS / 32; ++k) {
      et += s_e[k];
      gt += s_g[k];
    }
    __stcg(&share[((size_t)u * nchunk + c) * 2], et);
    __stcg(&share[((size_t)u * nchunk + c) * 2 + 1], gt);
  }
}

__global__ void __launch_bounds__(K1T_FIN_ROWS * 32) k1_tc_finalize_taps(const PlanDev P, int nchunk,
                                                                        K1Out o, const double* share) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int u = blockIdx.x / nchunk, c = blockIdx.x - u * nchunk;
  const int tid = threadIdx.x;
  const int L = P.L, ncol = 2 * L, AD = P.A * P.D;
  const int r0 = c * K1T_FIN_ROWS, r1 = min(AD, r0 + K1T_FIN_ROWS);
  const double* acc = o.parts + (size_t)u * (2 * (size_t)AD * L + 2);
  // the unit's shares: 32 in flight per warp (one per lane), summed in chunk
  // order through shuffles -- every warp of every CTA of the unit gets the same
  double et = 0.0, gt = 0.0;
  const int lane = tid & 31;
  for (int k0 = 0; k0 < nchunk; k0 += 32) {
    const bool have = k0 + lane < nchunk;
    const double ve = have ? __ldcg(&share[((size_t)u * nchunk + k0 + lane) * 2]) : 0.0;
    const double vg = have ? __ldcg(&share[((size_t)u * nchunk + k0 + lane) * 2 + 1]) : 0.0;
    for (int k = 0; k < 32 && k0 + k < nchunk; ++k) {
      et += __shfl_sync(0xffffffffu, ve, k);
      gt += __shfl_sync(0xffffffffu, vg, k);
    }
  }
  const double nvhat = (et - gt / (double)P.M) / ((double)AD * (P.M - P.guard));
  if (c == 0 && tid == 0 && o.sigma2) o.sigma2[u] = nvhat;
  const double sgm = nvhat + P.ridge;
  const int M = P.M;
  float2* cm = o.coef + (size_t)u * coef_floats2(P);
  float2* ca = cm + (size_t)AD * 8;
  for (int o2 = r0 * 8 + tid; o2 < r1 * 8; o2 += K1T_FIN_ROWS * 32) {
    const int ad = o2 >> 3, l = o2 & 7;
    const double wl = P.pdp[l] / ((double)M * P.pdp[l] + sgm);
    cm[o2] = make_float2((float)(wl * __ldcg(&acc[ad * ncol + 2 * l])),
                         (float)(wl * __ldcg(&acc[ad * ncol + 2 * l + 1])));
  }
  for (int o2 = r0 * P.trunc + tid; o2 < r1 * P.trunc; o2 += K1T_FIN_ROWS * 32) {
    const int ad = o2 / P.trunc, l = o2 - ad * P.trunc;
    const double2 bb = make_double2(__ldcg(&acc[ad * ncol + 2 * l]), __ldcg(&acc[ad * ncol + 2 * l + 1]));
    const double2 cz = zmul(P.ai_fac[l], bb);
    ca[o2] = make_float2((float)cz.x, (float)cz.y);
  }
}
