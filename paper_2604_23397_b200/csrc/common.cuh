// Shared device-side definitions of the ARCHES B200 hot path.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/arches.h"

#define ARCHES_TILE 128        // K2 subcarriers per CTA (one per thread)
#define ARCHES_K1_THREADS 256  // K1 CTA size
#define ARCHES_RA 4            // K1 register tile: (a,d) rows per thread
#define ARCHES_RL 5            // K1 register tile: delay bins per thread
#define ARCHES_MAX_AD (ARCHES_MAX_ANT * ARCHES_MAX_DMRS)
#define ARCHES_FEATURES 10
#define ARCHES_QPSK_AMP 0x3F3504F3u  // float(1/sqrt(2)): the complex64 of qpsk() (rng.py:50-55)
#define ARCHES_TXB_ROW 32            // packed tx bytes per (tile, symbol): 128 REs x 2 bits

// Plan constants passed by value to every kernel (tables live in device memory).
struct PlanDev {
  int A, N, M, T, D, L;         // antennas, subcarriers, comb, symbols, dmrs, analysis bins
  int trunc, guard;             // denoiser taps, noise guard
  int n_blocks, block, diag;    // MMSE blocks, subcarriers per block, closed-form weights
  int n_tiles;                  // K2 tiles per unit
  int nbt_max;                  // max MMSE blocks overlapping one K2 tile
  int dsym[ARCHES_MAX_DMRS];    // DMRS symbol indices
  int is_dmrs[ARCHES_MAX_SYM];  // symbol -> dmrs slot or -1
  int tw_d0[ARCHES_MAX_SYM], tw_d1[ARCHES_MAX_SYM];  // time interpolation taps
  float tw_w0[ARCHES_MAX_SYM], tw_w1[ARCHES_MAX_SYM];
  double ridge;
  double pdp[8];                // MMSE prior powers p_l
  float tw[ARCHES_MAX_SYM][ARCHES_MAX_DMRS];  // _time_interp_weights (phy_pipeline.py:227-242)
  double2 ai_fac[ARCHES_MAX_BINS];  // (1 + e^{2 pi i l/N}) / N
  const float2* wM;             // [M] e^{+2 pi i j / M}
  const float2* wN;             // [N] e^{+2 pi i j / N}
  const float2* syn;            // [L][TILE] e^{-2 pi i l j / N}
  const double2* gram;          // [8][8] F^H F of one MMSE block
  const float* tc_a;            // K2 tensor-core synthesis operand (UMMA layout, hi | lo)
  int tc_kb;                    // its 8-wide K blocks (Lsyn / 4)
  const float2* tc_rot;         // [n_tiles][4*tc_kb + 8]: e^{-2 pi i l k0/N} (AI), e^{-2 pi i l (k0-b*block)/N} (MMSE)
  int num_sms;
  int k2_rot_smem;              // tensor-core K2 stages tc_rot in shared memory
  int tx_packed;                // ARCHES_FLAG_TX_PACKED: tx is the packed QPSK wire format
  // KPM layer
  double sinr_cap_db, lcid4_fraction, lcid4_jitter, crc_margin_db, crc_scale_db;
  double slot_us, slot_s;
  int64_t slot_ns;
  int n_prb, mac_header_bytes, window_length, n_mcs;
  double mcs_thr[ARCHES_MAX_MCS];
  double mcs_rate[ARCHES_MAX_MCS];
  int mcs_qam[ARCHES_MAX_MCS];
  // control plane
  int exec_mode, policy, fixed_mode, decision_period, dapp_window;
  int64_t decision_delay_ns, failsafe_timeout_ns;
  uint64_t crc_key;
};

// Per-unit coefficient record written by K1, read by K2 (workspace).
//   cm[ad][b][8]  MMSE synthesis taps per block (float2)
//   ca[ad][T]     AI synthesis taps (float2)
__host__ __device__ inline size_t coef_floats2(const PlanDev& P) {
  const size_t n = (size_t)P.A * P.D * (P.n_blocks * 8 + P.trunc);
  return (n + 1) & ~(size_t)1;  // 16-byte multiple (bulk-copy granule)
}

// K2 per-tile partial sums (fp64), reduced in tile order by the last CTA.
struct TilePartial {
  double abs_sum[2];
  double pow_sum[2];
  double sxx;
  double sxy_re[2];
  double sxy_im[2];
  double syy[2];
  double pad;
};

// Per-stream control state header (followed by rings, see state_layout).
struct PendingMsg {
  int64_t at_ns;
  int32_t mode;
  int32_t trigger;
};

struct StreamState {
  int64_t next_slot;
  int64_t cum_phy_bytes;
  int64_t mac_total, l4_total;
  int64_t last_delivery_ns;
  int32_t mode, ndi;
  int32_t prev_msg_mode, reserved2;   // oracle source: last_msg_mode one slot earlier
  int32_t n_pending, n_forced;
  int32_t since_decision, reserved3, reserved4, tripped;
  int32_t last_msg_mode, pad;
  PendingMsg pending[ARCHES_MAX_PENDING];
  PendingMsg forced[ARCHES_MAX_PENDING];
};

__host__ __device__ inline size_t state_stride_bytes(int window, int dapp_window) {
  size_t b = sizeof(StreamState) + (size_t)2 * window * sizeof(int32_t) +
             (size_t)dapp_window * ARCHES_FEATURES * sizeof(double);
  return (b + 255) & ~(size_t)255;
}

// ---------------------------------------------------------------- complex
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {  // conj(a) * b
  return make_float2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
__device__ __forceinline__ void cfma(float2& acc, float2 a, float2 b) {  // acc += a*b
  acc.x = fmaf(a.x, b.x, acc.x);
  acc.x = fmaf(-a.y, b.y, acc.x);
  acc.y = fmaf(a.x, b.y, acc.y);
  acc.y = fmaf(a.y, b.x, acc.y);
}
__device__ __forceinline__ double2 zmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---------------------------------------------------------------- async copy
// 1-D bulk copies global -> shared (TMA engine, cp.async.bulk) completing on an
// mbarrier; used to stage whole subcarrier tiles of y / tx per CTA.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  // try_wait with a suspend-time hint: the waiting warp sleeps instead of
  // spinning on issue slots the compute warps need
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(phase), "r"(0x10000u)
      : "memory");
}
__device__ __forceinline__ void mbar_wait_spin(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAITS_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAITS_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t l2_evict_last_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// Work split: CTA b owns the contiguous item range [b*n/G, (b+1)*n/G), so a
// CTA walks the tiles of one unit in order and its threads keep their
// telemetry sums in registers across them; a unit's sums are flushed once per
// (CTA, unit) segment, at the segment's first tile.  K3 adds the segments.
__host__ __device__ inline bool k2_segment_start(int item, int n_tiles, int n_items, int G) {
  if (item % n_tiles == 0) return true;
  if ((long long)n_items * G < 0x7fffffffLL) {  // 32-bit division is enough (and much cheaper)
    const unsigned b = ((unsigned)item * (unsigned)G + (unsigned)n_items - 1u) / (unsigned)n_items;
    return b < (unsigned)G && (b * (unsigned)n_items) / (unsigned)G == (unsigned)item;
  }
  const long long b = ((long long)item * G + n_items - 1) / n_items;  // ceil
  return b < G && (b * n_items) / G == item;
}

// ---------------------------------------------------------------- packed tx
// a 2-bit code of the QPSK wire format (bit 0: Re > 0, bit 1: Im > 0) as the
// complex64 of qpsk() (rng.py:50-55); k_pack_qpsk / k_unpack_qpsk define it
__device__ __forceinline__ float2 qpsk_code_to_x(unsigned int c) {
  const float q = __uint_as_float(ARCHES_QPSK_AMP);
  return make_float2((c & 1u) ? q : -q, (c & 2u) ? q : -q);
}
// RE (u, t, k) of a packed tx grid [u][n_tiles][T][32 B]
__device__ __forceinline__ float2 tx_packed_at(const PlanDev& P, const unsigned char* bits, size_t u,
                                               int t, int k) {
  const int tile = k / ARCHES_TILE, j = k - tile * ARCHES_TILE;
  const unsigned int b = bits[((u * P.n_tiles + tile) * P.T + t) * ARCHES_TXB_ROW + (j >> 2)];
  return qpsk_code_to_x(b >> ((j & 3) * 2));
}
