// K1 (tensor-core form) -- the 20-bin comb analysis of every (unit, antenna,
// DMRS symbol) row as a tcgen05 contraction, for single-block plans.
//
// Replaces the analysis half of ls_estimate / estimate_noise_var /
// mmse_estimate / denoiser_estimate (expert_bank.py:96-214):
//   B[u,a,d][l] = sum_m h[u,a,d][m] e^{+2 pi i l m / M},  h = y[.., 2m, dmrs_d] conj(p) / |p|^2
// written as  D[t][n] = sum_kappa A[t][kappa] W[kappa][n]  per chunk, with
//   t     = MMA row = (data row rr, sub-chunk c): 16 data rows (row = u*A + a, one
//           stream per tile) x 8 sub-chunks of 16 comb points, so one chunk
//           spans 256 contiguous subcarriers (2 KB) of each of 16 rows,
//   kappa = real embedding of the sub-chunk's 16 comb points,
//   n     = 2l + re/im (N = 2L padded to 16).
// Sub-chunk cc (comb points m0 = 16 cc .. m0 + 15) contributes
//   e^{2 pi i l m0/M} sum_{k<16} h[m0+k] e^{2 pi i l k/M}
// so the MMA operand W (k < 16, real-embedded, tf32 hi | lo) is the same for
// every chunk and stays in shared memory; each MMA row's sub-chunk phase is
// applied to its 2L outputs in the epilogue and the 8 sub-chunks of a data row
// are summed across lanes when its segment ends.
//   * producer warp: per chunk, 16 lanes each issue one 1-D bulk copy of a
//     row's 2 KB into a 16-byte-padded row of the stage (long row requests --
//     the old 128-B swizzled tensor boxes made K1 TMA-request bound -- and the
//     padding makes the converters' natural-order reads bank-conflict free);
//   * converter warps: the 128 pilot inverses conj(p)/|p|^2 of the chunk, one per
//     thread, into shared memory; then thread tau converts MMA row (rr, c) with
//     rr = (tau/8 + c) mod 16, c = tau mod 8 (a quarter warp reads 8 rows at 8
//     bank offsets and writes 8 SWIZZLE_128B groups): h = y q, tf32 hi | lo into
//     one of two MMA operand buffers (the raw stage is released right away);
//   * MMA warp (owns the TMEM allocation): D = A_hi W_hi + A_lo W_hi + A_hi W_lo
//     (kind::tf32, 3xTF32) into a ring of TMEM accumulators;
//   * drain warps, two groups of 4 (columns [0, 24) and [24, 2L); thread = TMEM
//     lane = MMA row): tcgen05.ld, the sub-chunk phase, fp32 sums over 4 chunks
//     folded into fp64 (short fp32 chains keep the Parseval noise estimate
//     precise); at a segment end (row tile change or the CTA's last chunk) a
//     reduce-scatter over the data row's 8 sub-chunk lanes (fp64 shuffles) and
//     the segment's partial bins go to global memory (the converters sum the
//     row energies through shared memory).
// Work split: the (row tile, DMRS symbol, chunk) items in that order, cut into
// one contiguous range per CTA (balanced to one chunk); the finalize sums a
// row's segments in chunk order, a segment starting at chunk 0 or at a CTA's
// first item (k1t_row_sum).
#pragma once
#include "k_analyze.cuh"
#include "k_synth_tc.cuh"

#define K1T_CONV_WARPS 4                         // converters: warps 0-3
#define K1T_DRAIN_WARPS 8                        // drains: warps 4-11 (two column halves)
#define K1T_THREADS (32 * (K1T_CONV_WARPS + K1T_DRAIN_WARPS + 2))  // + producer + MMA warp
#define K1T_NB 48                                // MMA N (2L = 40 padded to 16)
#define K1T_MAX_SUB 112                          // sub-chunk phases in shared memory (N <= 3584)
#define K1T_STAGES 4                             // raw grid stages
#define K1T_MBUF 2                               // MMA operand buffers
#define K1T_RR 16                                // data rows per item
#define K1T_SUBS 8                               // sub-chunks per item (MMA rows = K1T_RR x K1T_SUBS)
#define K1T_CP 16                                // comb points per sub-chunk (one 128-B operand row)
#define K1T_CSC (2 * K1T_CP * K1T_SUBS)          // subcarriers per chunk (256 = one 2-KB row copy)
#define K1T_ACC 4                                // TMEM accumulator ring
#define K1T_LP 21                                // phase-table row stride (float2): conflict-free per-lane rows
#define K1T_QP 18                                // pilot-inverse row stride per sub-chunk (float2)

struct K1TArgs {
  const float2* y;         // [u][A][T][N] grid
  const float2* pil;       // [stream][M][D]
  const float* wimg;       // [hi | lo][NB rows][128 B, SWIZZLE_128B] twiddle operand, chunk-invariant
  const float2* rot;       // [n_chunks * 8][K1T_LP] sub-chunk phases e^{2 pi i l 16cc / M}
  double* dpart;           // [item][16][2L] segment partial bins (fp64), written at segment starts
  double* epart;           // [item][16] segment row energies
  int n_slots, srows;      // slots per stream, rows per stream (= n_slots * A)
  int n_rows;              // rows of the grid (= units * A)
  int gps;                 // 16-row tiles per stream (a tile never straddles streams)
  int n_g, n_chunks;       // 16-row tiles, 256-subcarrier chunks per row
  int n_items, grid;       // items = n_g * D * n_chunks, cut into `grid` contiguous ranges
  int nb;                  // MMA N
};

// CTA b's items are [k1t_first(b), k1t_first(b + 1)); 32-bit products
// (n_items * grid < 2^31 is checked at launch)
__host__ __device__ __forceinline__ int k1t_first(int b, int n_items, int grid) {
  return (int)(((unsigned)b * (unsigned)n_items) / (unsigned)grid);
}
// the CTA whose range holds item i
__device__ __forceinline__ int k1t_owner(int i, int n_items, int grid) {
  return (int)(((unsigned)(i + 1) * (unsigned)grid - 1u) / (unsigned)n_items);
}

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

#ifdef K1T_TRACE  // timing-analysis builds only (tools/k1_trace.py), never the shipped library
__device__ unsigned long long g_k1t_trace[8][64][8];
__device__ unsigned long long g_k1t_span[256][5];  // per CTA: entry, first copy, drain done, zeroed, synced
#define K1TS(slot, cond)                                         \
  do {                                                           \
    if ((cond) && blockIdx.x < 256) {                            \
      unsigned long long t_;                                     \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));     \
      g_k1t_span[blockIdx.x][(slot)] = t_;                       \
    }                                                            \
  } while (0)
#define K1TR(slot, jj, cond)                                                          \
  do {                                                                                \
    if ((cond) && blockIdx.x < 8 && (jj) < 64) {                                      \
      unsigned long long t_;                                                          \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                          \
      g_k1t_trace[blockIdx.x][(jj)][(slot)] = t_;                                     \
    }                                                                                 \
  } while (0)
#else
#define K1TR(slot, jj, cond) \
  do {                       \
  } while (0)
#define K1TS(slot, cond) \
  do {                   \
  } while (0)
#endif

constexpr uint32_t K1T_ATOM = 128 * 128;                        // 128 MMA rows x 128 B (one SWIZZLE_128B K block)
constexpr uint32_t K1T_ROWB = K1T_CSC * 8;                       // 2 KB: one row of a chunk (complex64)
constexpr uint32_t K1T_ROWP = K1T_ROWB + 16;                     // padded row stride in the stage
constexpr uint32_t K1T_RAW_BYTES = K1T_RR * K1T_ROWP;            // raw chunk: 16 rows x 256 subcarriers
constexpr uint32_t K1T_OP_BYTES = K1T_ATOM;                      // compacted operand: 16 comb points of 128 rows
static_assert(K1T_STAGES * K1T_RAW_BYTES % 1024 == 0, "operand buffers stay 1024-byte aligned");

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

__host__ __device__ inline size_t k1t_smem_bytes(int nb, int n_chunks) {
  return (size_t)K1T_STAGES * K1T_RAW_BYTES + (size_t)K1T_MBUF * 2 * K1T_OP_BYTES +
         (size_t)nb * 128 * 2 + (size_t)n_chunks * K1T_SUBS * K1T_LP * sizeof(float2);
}

// item = (row tile g, DMRS symbol d, chunk ch), chunk fastest; walked incrementally
struct K1TItem {
  int g, d, ch;
  __device__ __forceinline__ void init(int item, int nc, int D) {
    ch = item % nc;
    const int gd = item / nc;
    d = gd % D;
    g = gd / D;
  }
  __device__ __forceinline__ void next(int nc, int D) {
    if (++ch == nc) {
      ch = 0;
      if (++d == D) d = 0, ++g;
    }
  }
};

// Drain of columns [C0, C0 + NC) of every chunk's accumulator: thread = MMA
// row t = TMEM lane = (rr, c).  Phase-rotated chunk sums are added in fp32 over
// K1T_FGRP chunks, then folded into fp64 (every fp32 chain stays short, so the
// Parseval noise estimate keeps its precision); at a segment end the 8
// sub-chunk lanes of a data row are summed by xor shuffles and the segment's
// partial bins go to global memory.
template <int NC, int C0>
__device__ __forceinline__ void k1t_drain(const K1TArgs& a, int L, int t, uint32_t lane_base,
                                          const float2* rotsm, uint64_t* s_accf, uint64_t* s_acce,
                                          int i_begin, int i_end, int nc, int D) {
  constexpr int K1T_FGRP = 4;
  constexpr int NW = NC / K1T_SUBS;  // columns each lane of a data row writes
  static_assert(NC % 2 == 0 && NC % K1T_SUBS == 0, "column split");
  const int rr = t >> 3, c = t & 7, ncol = 2 * L;
  float acc[NC];
  double acc64[NC];
#pragma unroll
  for (int q = 0; q < NC; ++q) acc[q] = 0.f, acc64[q] = 0.0;
  int seg = i_begin, nf = 0;
  K1TItem it;
  it.init(i_begin, nc, D);
  for (int item = i_begin, j = 0; item < i_end; ++item, ++j, it.next(nc, D)) {
    const int r = j % K1T_ACC;
    mbar_wait_spin(&s_accf[r], (j / K1T_ACC) & 1);
    K1TR(5 + (C0 > 0), j, t == 0);
    tc_fence_after();
    float vals[NC];
    tmem_ld_n<NC>(lane_base + (uint32_t)(r * K1T_NB + C0), vals);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    tc_fence_before();
    mbar_arrive(&s_acce[r]);
    const float2* ph = rotsm + (size_t)(it.ch * K1T_SUBS + c) * K1T_LP + C0 / 2;
#pragma unroll
    for (int l = 0; l < NC / 2; ++l) {
      const float2 v = cmul(make_float2(vals[2 * l], vals[2 * l + 1]), ph[l]);
      acc[2 * l] += v.x;
      acc[2 * l + 1] += v.y;
    }
    const bool seg_end = item + 1 == i_end || it.ch + 1 == nc;
    if (++nf == K1T_FGRP || seg_end) {
      nf = 0;
#pragma unroll
      for (int q = 0; q < NC; ++q) {
        acc64[q] += (double)acc[q];
        acc[q] = 0.f;
      }
    }
    K1TR(7, j, t == 0 && C0 == 0);
    if (seg_end) {
      // reduce-scatter over the row's 8 lanes: at xor distance 4, 2, 1 a lane
      // keeps the half of its remaining columns whose owner shares its bit and
      // sends the other half, ending with its own NW columns [NW c, NW c + NW)
      // summed over the 8 sub-chunks (fixed order: deterministic)
      double r4[NC / 2], r2[NC / 4], r1[NW];
      {
        const bool hi = c & 4;
#pragma unroll
        for (int q = 0; q < NC / 2; ++q) {
          const double mine = hi ? acc64[NC / 2 + q] : acc64[q];
          const double send = hi ? acc64[q] : acc64[NC / 2 + q];
          r4[q] = mine + __shfl_xor_sync(0xffffffffu, send, 4);
        }
      }
      {
        const bool hi = c & 2;
#pragma unroll
        for (int q = 0; q < NC / 4; ++q) {
          const double mine = hi ? r4[NC / 4 + q] : r4[q];
          const double send = hi ? r4[q] : r4[NC / 4 + q];
          r2[q] = mine + __shfl_xor_sync(0xffffffffu, send, 2);
        }
      }
      {
        const bool hi = c & 1;
#pragma unroll
        for (int q = 0; q < NW; ++q) {
          const double mine = hi ? r2[NW + q] : r2[q];
          const double send = hi ? r2[q] : r2[NW + q];
          r1[q] = mine + __shfl_xor_sync(0xffffffffu, send, 1);
        }
      }
      const int stream = it.g / a.gps, lrow = (it.g - stream * a.gps) * K1T_RR + rr;
      if (lrow < a.srows) {
        double* dst = a.dpart + ((size_t)seg * K1T_RR + rr) * ncol + C0 + NW * c;
#pragma unroll
        for (int q = 0; q < NW; ++q) dst[q] = r1[q];
      }
#pragma unroll
      for (int q = 0; q < NC; ++q) acc64[q] = 0.0;
      seg = item + 1;
    }
  }
}

template <int NB, int LC>
__global__ void __launch_bounds__(K1T_THREADS, 1) k1_tc(const PlanDev P, const K1TArgs a) {
  extern __shared__ __align__(1024) unsigned char sm1k[];
  __shared__ __align__(8) uint64_t s_full[K1T_STAGES], s_empty[K1T_STAGES];
  __shared__ __align__(8) uint64_t s_conv[K1T_MBUF], s_mfree[K1T_MBUF], s_w;
  __shared__ __align__(8) uint64_t s_accf[K1T_ACC], s_acce[K1T_ACC];
  __shared__ __align__(16) float2 s_q[2][K1T_SUBS * K1T_QP];  // pilot inverses of a chunk, per sub-chunk row
  __shared__ double s_e[128];                                 // segment energies per MMA row
  __shared__ uint32_t s_tmem;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int nb = NB;
  constexpr uint32_t w_bytes = (uint32_t)nb * 128;
  const int NT = 32 * K1T_CONV_WARPS;
  const int nc = a.n_chunks, D = P.D;
  const int i_begin = k1t_first(blockIdx.x, a.n_items, a.grid);
  const int i_end = k1t_first(blockIdx.x + 1, a.n_items, a.grid);
  unsigned char* raw = sm1k;                                            // [STAGES][16 padded rows]
  unsigned char* mbuf = sm1k + (size_t)K1T_STAGES * K1T_RAW_BYTES;      // [MBUF][hi | lo]
  unsigned char* wbuf = mbuf + (size_t)K1T_MBUF * 2 * K1T_OP_BYTES;   // [hi | lo]
  float2* rotsm = reinterpret_cast<float2*>(wbuf + 2 * w_bytes);      // [sub-chunk][K1T_LP] phases

  K1TS(0, threadIdx.x == 0);
  {
    // barriers initialised one per thread (SWIZZLE_128B atoms need a 1024-byte-aligned base)
    const int k = threadIdx.x;
    if (k == 0 && (smem_u32(sm1k) & 1023u)) __trap();
    if (k < K1T_STAGES) mbar_init(&s_full[k], 1);
    else if (k < 2 * K1T_STAGES) mbar_init(&s_empty[k - K1T_STAGES], NT);
    else if (k < 2 * K1T_STAGES + K1T_MBUF) mbar_init(&s_conv[k - 2 * K1T_STAGES], NT);
    else if (k < 2 * K1T_STAGES + 2 * K1T_MBUF) mbar_init(&s_mfree[k - 2 * K1T_STAGES - K1T_MBUF], 1);
    else if (k < 2 * K1T_STAGES + 2 * K1T_MBUF + K1T_ACC) mbar_init(&s_accf[k - 2 * K1T_STAGES - 2 * K1T_MBUF], 1);
    else if (k < 2 * K1T_STAGES + 2 * K1T_MBUF + 2 * K1T_ACC)
      mbar_init(&s_acce[k - 2 * K1T_STAGES - 2 * K1T_MBUF - K1T_ACC], 32 * K1T_DRAIN_WARPS);
    else if (k == 2 * K1T_STAGES + 2 * K1T_MBUF + 2 * K1T_ACC) mbar_init(&s_w, 1);
  }
  // the finalize (programmatic dependent launch) may be scheduled onto SMs as
  // they free up; it waits for this grid's completion before reading anything
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  __syncthreads();  // barriers initialised; the TMEM allocation is off this path (MMA warp)
  constexpr int NTMEM = 32 + 32 * K1T_DRAIN_WARPS;  // MMA warp + drains: barriers 1 (alloc), 2 (release)

  static_assert(NB == K1T_NB, "MMA N");
  if (warp == K1T_CONV_WARPS + K1T_DRAIN_WARPS) {
    // ---------------- producer: the twiddle operand once, then raw chunks (lane = row)
    const uint64_t pol_y = l2_evict_first_policy();
    K1TS(3, lane == 0);
    if (lane == 0) {
      const uint64_t pol_w = l2_evict_last_policy();
      const uint32_t rot_bytes = (uint32_t)(nc * K1T_SUBS * K1T_LP * sizeof(float2) + 15) & ~15u;
      mbar_arrive_expect_tx(&s_w, 2 * w_bytes + rot_bytes);
      bulk_g2s(wbuf, a.wimg, 2 * w_bytes, &s_w, pol_w);
      bulk_g2s(rotsm, a.rot, rot_bytes, &s_w, pol_w);
    }
    const size_t rowstride = (size_t)P.T * P.N;  // float2 between consecutive (unit, antenna) rows
    K1TItem it;
    it.init(i_begin, nc, D);
    for (int item = i_begin, j = 0; item < i_end; ++item, ++j, it.next(nc, D)) {
      const int s = j % K1T_STAGES;
      const int stream = it.g / a.gps, lrow0 = (it.g - stream * a.gps) * K1T_RR;
      const int nrows = min(K1T_RR, a.srows - lrow0);
      // every copied row is a full 2 KB: a row's last chunk runs on into the next
      // OFDM symbol's subcarriers (finite grid values, met by zero pilot
      // inverses), except past the end of the grid (a DMRS symbol last in the
      // slot, on the grid's last row), where the stage row's tail is zeroed
      const uint32_t bytes = K1T_ROWB;
      const int last = stream * a.srows + lrow0 + nrows;  // one past the tile's last row
      const bool clamp = it.ch == nc - 1 && P.dsym[it.d] == P.T - 1 && last == a.n_rows;
      const uint32_t tail = (uint32_t)(P.N - it.ch * K1T_CSC) * 8;
      if (j >= K1T_STAGES) mbar_wait_spin(&s_empty[s], ((j / K1T_STAGES) - 1) & 1);
      K1TR(0, j, lane == 0);
      K1TS(1, lane == 0 && j == 0);
      if (lane == 0) mbar_arrive_expect_tx(&s_full[s], (uint32_t)nrows * bytes - (clamp ? bytes - tail : 0u));
      __syncwarp();
      if (lane < nrows) {
        const size_t grow = (size_t)(stream * a.srows + lrow0 + lane);
        const float2* src = a.y + grow * rowstride + (size_t)P.dsym[it.d] * P.N + (size_t)it.ch * K1T_CSC;
        unsigned char* dst = raw + (size_t)s * K1T_RAW_BYTES + lane * K1T_ROWP;
        uint32_t nb_copy = bytes;
        if (clamp && lane == nrows - 1) {
          nb_copy = tail;
          for (uint32_t o = tail; o < K1T_ROWB; o += 16)
            *reinterpret_cast<float4*>(dst + o) = make_float4(0.f, 0.f, 0.f, 0.f);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
        bulk_g2s(dst, src, nb_copy, &s_full[s], pol_y);
      }
    }
    return;
  }
  if (warp == K1T_CONV_WARPS + K1T_DRAIN_WARPS + 1) {
    // ---------------- MMA issuer: chunk j -> TMEM accumulator j % K1T_ACC; owns the TMEM
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
        smem_u32(&s_tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    tc_fence_before();
    named_bar(1, NTMEM);
    tc_fence_after();
    const uint32_t tmem = s_tmem;
    if (lane == 0) {
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(nb >> 3) << 17) |
                             ((uint32_t)(128 >> 4) << 24);
      const uint32_t wh = smem_u32(wbuf), wl = wh + w_bytes;
      mbar_wait_spin(&s_w, 0);
      for (int item = i_begin, j = 0; item < i_end; ++item, ++j) {
        const int b = j % K1T_MBUF, r = j % K1T_ACC;
        if (j >= K1T_ACC) mbar_wait_spin(&s_acce[r], ((j / K1T_ACC) - 1) & 1);
        mbar_wait_spin(&s_conv[b], (j / K1T_MBUF) & 1);
        K1TR(4, j, true);
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
    __syncwarp();
    named_bar(2, NTMEM);  // the drains have read their last accumulator
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
    return;
  }

  if (warp >= K1T_CONV_WARPS) {
    // ---------------- drain warps: warps 4-7 columns [0, 24), warps 8-11 [24, 2L)
    static_assert(LC <= NB && LC % 2 == 0 && LC > 24, "2L output columns within the MMA N");
    const int t = (warp & 3) * 32 + lane;  // MMA row = TMEM lane
    named_bar(1, NTMEM);                   // the MMA warp's TMEM allocation
    tc_fence_after();
    const uint32_t tmem = s_tmem;
    K1TS(4, warp == K1T_CONV_WARPS && lane == 0);
    const uint32_t lane_base = tmem + ((uint32_t)((warp & 3) * 32) << 16);
    mbar_wait_spin(&s_w, 0);  // phase table landed
    if (warp < K1T_CONV_WARPS + 4)
      k1t_drain<24, 0>(a, P.L, t, lane_base, rotsm, s_accf, s_acce, i_begin, i_end, nc, D);
    else
      k1t_drain<LC - 24, 24>(a, P.L, t, lane_base, rotsm, s_accf, s_acce, i_begin, i_end, nc, D);
    K1TS(2, warp == K1T_CONV_WARPS && lane == 0);
    tc_fence_before();
    asm volatile("bar.arrive 2, %0;" ::"r"(NTMEM) : "memory");  // TMEM reads done
    return;
  }

  // ---------------- converter warps
  const int tau = threadIdx.x;
  const int c = tau & 7, rr = ((tau >> 3) + c) & (K1T_RR - 1);
  const int t = rr * K1T_SUBS + c;  // the MMA row this thread converts
  const int M = P.M;
  double e64 = 0.0;
  int seg = i_begin;
  K1TItem it;
  it.init(i_begin, nc, D);
  // this thread's pilot of the next chunk: comb point tau of it
  auto load_pilot = [&](const K1TItem& x, bool in_range) {
    const int stream = x.g / a.gps;
    const int m = x.ch * (K1T_CP * K1T_SUBS) + tau;
    return in_range && m < M ? __ldg(a.pil + ((size_t)stream * M + m) * D + x.d) : make_float2(0.f, 0.f);
  };
  float2 pn = load_pilot(it, i_begin < i_end);
  for (int item = i_begin, j = 0; item < i_end; ++item, ++j) {
    const int s = j % K1T_STAGES, b = j % K1T_MBUF;
    {
      // pilot inverse conj(p)/|p|^2 of comb point tau (1/|p|^2 within 1 ulp,
      // exact for the unit-modulus QPSK pilots; 0 past M)
      const float2 p = pn;
      const float n2 = p.x * p.x + p.y * p.y;
      float inv;
      asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(inv) : "f"(n2));
      inv = n2 > 0.f ? inv : 0.f;
      s_q[j & 1][(tau >> 4) * K1T_QP + (tau & 15)] = make_float2(p.x * inv, -p.y * inv);
    }
    K1TItem nx = it;
    nx.next(nc, D);
    pn = load_pilot(nx, item + 1 < i_end);
    named_bar(3, NT);  // the chunk's pilot inverses are visible
    mbar_wait_spin(&s_full[s], (j / K1T_STAGES) & 1);
    K1TR(1, j, tau == 0);
    if (j >= K1T_MBUF) mbar_wait_spin(&s_mfree[b], ((j / K1T_MBUF) - 1) & 1);
    K1TR(2, j, tau == 0);
    // 16-byte group k of the sub-chunk = (y[2m].re, .im, y[2m+1].re, .im), m = 16c + k;
    // only the comb half (.x, .y) is read
    const unsigned char* src = raw + (size_t)s * K1T_RAW_BYTES + rr * K1T_ROWP + c * (2 * K1T_CP * 8);
    const float4* qs = reinterpret_cast<const float4*>(&s_q[j & 1][c * K1T_QP]);
    unsigned char* ah = mbuf + (size_t)b * 2 * K1T_OP_BYTES + t * 128;
    unsigned char* al = ah + K1T_OP_BYTES;
    float e32 = 0.f;
#pragma unroll
    for (int k = 0; k < K1T_CP / 2; ++k) {
      const float2 y0 = *reinterpret_cast<const float2*>(src + (2 * k) * 16);
      const float2 y1 = *reinterpret_cast<const float2*>(src + (2 * k + 1) * 16);
      const float4 q = qs[k];
      const float2 h0 = make_float2(fmaf(y0.x, q.x, -y0.y * q.y), fmaf(y0.x, q.y, y0.y * q.x));
      const float2 h1 = make_float2(fmaf(y1.x, q.z, -y1.y * q.w), fmaf(y1.x, q.w, y1.y * q.z));
      e32 = fmaf(h0.x, h0.x, fmaf(h0.y, h0.y, e32));
      e32 = fmaf(h1.x, h1.x, fmaf(h1.y, h1.y, e32));
      const float4 hi = make_float4(tf32_rna_fast(h0.x), tf32_rna_fast(h0.y), tf32_rna_fast(h1.x),
                                    tf32_rna_fast(h1.y));
      const uint32_t o = (uint32_t)((k ^ c) * 16);  // SWIZZLE_128B: group k of row t at (k ^ (t & 7))
      *reinterpret_cast<float4*>(ah + o) = hi;
      // lo = h - hi is exact in fp32 (<= 14 significant bits); the MMA reads its
      // top 11, so the dropped tail is < 2^-22 |h| -- no explicit rounding needed
      *reinterpret_cast<float4*>(al + o) = make_float4(h0.x - hi.x, h0.y - hi.y, h1.x - hi.z, h1.y - hi.w);
    }
    // raw stage consumed: every loaded value has been used above, so the
    // copy refill cannot race the shared-memory reads
    mbar_arrive(&s_empty[s]);
    e64 += (double)e32;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_arrive(&s_conv[b]);
    K1TR(3, j, tau == 0);
    if (item + 1 == i_end || it.ch + 1 == nc) {
      // segment end: the data row's 8 sub-chunk energies, summed in sub-chunk order
      s_e[t] = e64;
      named_bar(3, NT);
      if (tau < K1T_RR) {
        const int stream = it.g / a.gps, lrow = (it.g - stream * a.gps) * K1T_RR + tau;
        double v = 0.0;
#pragma unroll
        for (int k = 0; k < K1T_SUBS; ++k) v += s_e[tau * K1T_SUBS + k];
        if (lrow < a.srows) a.epart[(size_t)seg * K1T_RR + tau] = v;
      }
      e64 = 0.0;
      seg = item + 1;
    }
    it = nx;
  }
}

// Row `row`'s DMRS-symbol-d value (column cc of `ncol`) summed over its
// segments in chunk order (K1's partials, written at segment starts: the row
// tile's first chunk and every CTA range start inside the tile)
__device__ __forceinline__ double k1t_row_sum(const K1TArgs& a, const double* part, int ncol, int row,
                                              int d, int D, int cc) {
  const int stream = row / a.srows, lrow = row - stream * a.srows;
  const int g = stream * a.gps + lrow / K1T_RR, r = lrow % K1T_RR;
  const int i0 = (g * D + d) * a.n_chunks, i1 = i0 + a.n_chunks;
  double sum = __ldcg(part + ((size_t)i0 * K1T_RR + r) * ncol + cc);
  for (int b = k1t_owner(i0, a.n_items, a.grid) + 1;; ++b) {
    const int i = k1t_first(b, a.n_items, a.grid);
    if (i >= i1) break;
    sum += __ldcg(part + ((size_t)i * K1T_RR + r) * ncol + cc);
  }
  return sum;
}

// One CTA per unit: thread o sums output o (= (a, d, component)) over its row's
// segments in chunk order (fp64); every thread forms sigma2
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
  double sg = 0.0;  // this thread's share of sum_{a,d,l<guard} |B_l|^2
  for (int o2 = tid; o2 < nout; o2 += K1T_FIN_THREADS) {
    const int ad = o2 / ncol, cc = o2 - ad * ncol;
    const int aa = ad / P.D, d = ad - aa * P.D;
    const double sum = k1t_row_sum(a, a.dpart, ncol, u * P.A + aa, d, P.D, cc);
    acc[o2] = sum;
    if (cc < 2 * P.guard) sg += sum * sum;
  }
  // row energies: thread = (a, d)
  double e = 0.0;
  for (int ad = tid; ad < AD; ad += K1T_FIN_THREADS) {
    const int aa = ad / P.D, d = ad - aa * P.D;
    e += k1t_row_sum(a, a.epart, 1, u * P.A + aa, d, P.D, 0);
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
  double sg = 0.0;
  for (int o2 = r0 * ncol + tid; o2 < r1 * ncol; o2 += K1T_FIN_THREADS) {
    const int ad = o2 / ncol, cc = o2 - ad * ncol;
    const int aa = ad / P.D, d = ad - aa * P.D;
    const double sum = k1t_row_sum(a, a.dpart, ncol, u * P.A + aa, d, P.D, cc);
    __stcg(&acc[o2], sum);
    if (cc < 2 * P.guard) sg += sum * sum;
  }
  double e = 0.0;
  for (int ad = r0 + tid; ad < r1; ad += K1T_FIN_THREADS) {
    const int aa = ad / P.D, d = ad - aa * P.D;
    e += k1t_row_sum(a, a.epart, 1, u * P.A + aa, d, P.D, 0);
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
