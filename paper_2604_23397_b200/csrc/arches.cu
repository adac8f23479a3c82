// C ABI of the ARCHES B200 hot path: plan construction, launch wrappers and
// host helpers.  See include/arches.h for the contract of every entry point.
#include <cuda.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <complex>
#include <vector>

#include "common.cuh"
#include "k_analyze.cuh"
#include "k_analyze_tc.cuh"
#include "k_control.cuh"
#include "k_control_warp.cuh"
#include "k_control_block.cuh"
#include "k_downstream.cuh"
#include "k_tree_train.cuh"
#include "k_scene.cuh"
#include "k_synth_eq.cuh"
#include "k_synth_tc.cuh"
#include "rng.cuh"

#define ARCHES_VERSION "arches-b200 0.1 (sm_100a)"

static thread_local char g_err[512];

static int set_err(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

#define CUDA_TRY(expr)                                                                  \
  do {                                                                                  \
    cudaError_t e_ = (expr);                                                            \
    if (e_ != cudaSuccess)                                                              \
      return set_err(ARCHES_E_CUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_),   \
                     __FILE__, __LINE__);                                               \
  } while (0)

#define LAUNCH_CHECK()                                                                  \
  do {                                                                                  \
    cudaError_t e_ = cudaGetLastError();                                                \
    if (e_ != cudaSuccess)                                                              \
      return set_err(ARCHES_E_CUDA, "launch: %s (%s:%d)", cudaGetErrorString(e_),       \
                     __FILE__, __LINE__);                                               \
  } while (0)

struct arches_plan {
  arches_geom g;
  arches_params p;
  PlanDev dev;
  int k1_chunk;        // K1 points per CTA (comb analysis)
  int k1_parts;        // K1 CTAs per unit (comb analysis)
  size_t k1_smem;
  int k1t_nb;          // tensor-core K1: MMA N (0 = not applicable)
  int k1t_nchunks;     // 256-subcarrier chunks per row
  float* k1t_wimg;     // twiddle operand [hi|lo][kg][nb][4] (chunk-invariant)
  float2* k1t_rot;     // sub-chunk phases [chunk * 8][K1T_LP]
  int k1_full_chunk;   // N-point (denoiser compat) variant
  int k1_full_parts;
  size_t k1_full_smem;
  size_t k2_smem;
  size_t k2_tc_smem;  // 0: tensor-core K2 not applicable to this plan
  int k2_groups;      // > 1: tensor-core K2 over antenna groups of 4 (massive MIMO)
  void* dev_tables;
  int device;          // the CUDA device the plan (tables, streams) lives on
  // Executor streams / events, created with the plan on its device (so no entry
  // point creates one under graph capture).  `side`: run_batch's RNG fork.
  // `tail`: the pipelined form (arches_run_batch_async) runs the control tail of
  // batch n (RNG, K3, K4) there next to batch n+1's K1.
  cudaStream_t side = nullptr, tail = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaEvent_t ev_start = nullptr, ev_k2 = nullptr, ev_k3 = nullptr, ev_end = nullptr;
  // mutable: execution state of a const plan (one thread at a time per plan)
  mutable bool tail_pending = false;  // ev_k3 / ev_end refer to a batch not yet joined
};

// Set by arches_run_batch_async for the duration of one call: the K1 finalize
// waits for the previous batch's K3 (it overwrites sigma2, which K3 reads) and
// K3 is launched onto the tail stream once K2 is done.
struct TailHook {
  cudaEvent_t before_fin = nullptr;
  cudaStream_t k3_stream = nullptr;
  cudaEvent_t k2_done = nullptr;
  bool k3_on_tail = false;
};
static thread_local TailHook g_hook;

static inline size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

// cudaFuncSetAttribute is a synchronous host call: do it once per (device,
// kernel) (to the largest value requested so far) so eager launches stay
// back-to-back.
template <typename K>
static cudaError_t ensure_smem(K kern, size_t smem) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> set_to;  // per device and kernel
  if (smem <= 48 * 1024) return cudaSuccess;
  int dev = 0;
  cudaError_t e0 = cudaGetDevice(&dev);
  if (e0 != cudaSuccess) return e0;
  std::lock_guard<std::mutex> lk(mu);
  size_t& cur = set_to[{dev, reinterpret_cast<const void*>(kern)}];
  if (smem <= cur) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess) cur = smem;
  return e;
}

// SMs the persistent K1 / K2 grids use.  In the cross-batch pipeline a tree
// (dApp) policy's control walk of the previous batch (K4 on the plan's tail
// stream, tens of microseconds on one SM per stream) would otherwise hold an SM
// that one of K2's statically partitioned CTAs waits for, stretching the whole
// step: one SM is left to it (config A 4.83 -> 7.29 M slots/s; the same reserve
// costs config B, whose K4 is short, 1%, so other plans keep every SM).
static int persistent_sms(const PlanDev& d) {
  const bool long_tail = g_hook.k3_stream != nullptr && d.policy == ARCHES_POLICY_TREE;
  return std::max(1, d.num_sms - (long_tail ? 1 : 0));
}

// ------------------------------------------------------------ workspace
struct WsLayout {
  size_t coef, parts, counters, k1parts, k1counters, sigma2, rng, k1t_d, k1t_e, k1t_share, total;
};

// tensor-core K1 work split: (16-row tile, DMRS symbol, 256-subcarrier chunk)
// items cut into one contiguous range per CTA (at most one wave of SMs); a
// tile never straddles streams (gps tiles per stream)
struct K1TGeom {
  int gps, n_g, n_items, grid;
};
static K1TGeom k1t_geom(const arches_plan* P, int n_streams, int n_slots);
// workspace bound over every (streams, slots) split of n_units:
// streams * ceil(slots * A / 16) <= units * ceil(A / 16)
static int k1t_max_items(const arches_plan* P, int n_units) {
  const PlanDev& d = P->dev;
  return n_units * ((d.A + K1T_RR - 1) / K1T_RR) * d.D * P->k1t_nchunks;
}

// row chunks of the tensor-core K1 finalize: 1 (one CTA per unit, bins staged in
// shared memory) unless a unit's bins exceed that stage
static int k1t_fin_chunks(const PlanDev& d) {
  const int AD = d.A * d.D;
  return AD * 2 * d.L <= 4096 ? 1 : (AD + K1T_FIN_ROWS - 1) / K1T_FIN_ROWS;
}

static WsLayout ws_layout(const arches_plan* P, int n_units) {
  const PlanDev& d = P->dev;
  WsLayout w;
  size_t off = 0;
  w.coef = off;
  off += align256((size_t)n_units * coef_floats2(d) * sizeof(float2));
  w.parts = off;
  off += align256((size_t)n_units * d.n_tiles * sizeof(TilePartial));
  w.counters = off;
  off += align256((size_t)n_units * sizeof(unsigned int));
  w.k1parts = off;
  {
    const int np = std::max(P->k1_parts, P->k1_full_parts);
    off += align256((size_t)n_units * np * (2 * (size_t)d.A * d.D * d.L + 2) * sizeof(double));
  }
  w.k1counters = off;
  off += align256((size_t)n_units * sizeof(unsigned int));
  w.sigma2 = off;
  off += align256((size_t)n_units * sizeof(double));
  w.rng = off;
  off += align256((size_t)n_units * 2 * sizeof(double));
  w.k1t_d = w.k1t_e = w.k1t_share = off;
  if (P->k1t_nb) {
    const size_t items = (size_t)k1t_max_items(P, n_units);
    w.k1t_d = off;
    off += align256(items * K1T_RR * 2 * d.L * sizeof(double));
    w.k1t_e = off;
    off += align256(items * K1T_RR * sizeof(double));
    w.k1t_share = off;  // row-chunked finalize: per-CTA energy / guard shares
    off += align256((size_t)n_units * k1t_fin_chunks(d) * 2 * sizeof(double));
  }
  w.total = off;
  return w;
}

template <class T>
static T* ws_at(void* ws, size_t off) {
  return reinterpret_cast<T*>(reinterpret_cast<unsigned char*>(ws) + off);
}

// ------------------------------------------------------------ plan
static void time_interp(const arches_geom& g, PlanDev& d) {
  // _time_interp_weights (phy_pipeline.py:227-242)
  const int D = g.n_dmrs;
  for (int s = 0; s < ARCHES_MAX_SYM; ++s) {
    for (int j = 0; j < ARCHES_MAX_DMRS; ++j) d.tw[s][j] = 0.f;
    d.tw_d0[s] = d.tw_d1[s] = -1;
    d.tw_w0[s] = d.tw_w1[s] = 0.f;
    d.is_dmrs[s] = -1;
  }
  for (int j = 0; j < D; ++j) d.is_dmrs[g.dmrs_symbols[j]] = j;
  for (int s = 0; s < g.n_sym; ++s) {
    const double xs = s;
    if (xs <= g.dmrs_symbols[0]) {
      d.tw_d0[s] = 0;
      d.tw_w0[s] = 1.f;
    } else if (xs >= g.dmrs_symbols[D - 1]) {
      d.tw_d0[s] = D - 1;
      d.tw_w0[s] = 1.f;
    } else {
      int k = 0;
      while (k + 1 < D && g.dmrs_symbols[k + 1] <= s) ++k;
      const double w = (xs - g.dmrs_symbols[k]) / (double)(g.dmrs_symbols[k + 1] - g.dmrs_symbols[k]);
      d.tw_d0[s] = k;
      d.tw_w0[s] = (float)(1.0 - w);
      d.tw_d1[s] = k + 1;
      d.tw_w1[s] = (float)w;
    }
    if (d.tw_d0[s] >= 0) d.tw[s][d.tw_d0[s]] = d.tw_w0[s];
    if (d.tw_d1[s] >= 0) d.tw[s][d.tw_d1[s]] = d.tw_w1[s];
  }
}

extern "C" int arches_plan_create(const arches_geom* geom, const arches_params* params,
                                  arches_plan** out) {
  if (!geom || !params || !out) return set_err(ARCHES_E_CONTRACT, "null argument");
  const arches_geom& g = *geom;
  const arches_params& p = *params;
  if (g.n_ant < 1 || g.n_prb < 1 || g.n_sym < 1 || g.n_dmrs < 1)
    return set_err(ARCHES_E_CONFIG, "geometry dimensions must be positive");
  if (g.n_ant > ARCHES_MAX_ANT) return set_err(ARCHES_E_CONFIG, "n_ant > %d", ARCHES_MAX_ANT);
  if (g.n_sym > ARCHES_MAX_SYM || g.n_dmrs > ARCHES_MAX_DMRS)
    return set_err(ARCHES_E_CONFIG, "n_sym <= %d and n_dmrs <= %d required", ARCHES_MAX_SYM,
                   ARCHES_MAX_DMRS);
  for (int j = 0; j < g.n_dmrs; ++j) {
    if (g.dmrs_symbols[j] < 0 || g.dmrs_symbols[j] >= g.n_sym ||
        (j && g.dmrs_symbols[j] <= g.dmrs_symbols[j - 1]))
      return set_err(ARCHES_E_CONFIG, "dmrs_symbols must be strictly increasing and < n_sym");
  }
  if (!(g.slot_duration_us > 0)) return set_err(ARCHES_E_CONFIG, "slot_duration_us must be > 0");
  const int N = 12 * g.n_prb, M = 6 * g.n_prb;
  if (p.noise_guard < 1 || p.noise_guard >= M)
    return set_err(ARCHES_E_CONFIG, "guard %d outside 1..%d", p.noise_guard, M - 1);
  if (p.truncation < 1 || p.truncation > N)
    return set_err(ARCHES_E_CONFIG, "truncation %d outside 1..%d", p.truncation, N);
  if (p.truncation > ARCHES_MAX_BINS || p.noise_guard > ARCHES_MAX_BINS)
    return set_err(ARCHES_E_CONFIG, "device path supports truncation and noise_guard <= %d",
                   ARCHES_MAX_BINS);
  if (p.mmse_block_prbs < 1) return set_err(ARCHES_E_CONFIG, "mmse_block_prbs must be >= 1");
  if (p.n_mcs < 1 || p.n_mcs > ARCHES_MAX_MCS) return set_err(ARCHES_E_CONFIG, "n_mcs outside 1..%d", ARCHES_MAX_MCS);
  if (p.window_length < 1 || p.dapp_window_slots < 1 || p.decision_period_slots < 1)
    return set_err(ARCHES_E_CONFIG, "window lengths and periods must be positive");
  if (p.assumed_delay_spread < 0) return set_err(ARCHES_E_CONFIG, "delay_spread must be >= 0");
  if (p.flags & ~(ARCHES_FLAG_NO_TC_K1 | ARCHES_FLAG_NO_TC_K2 | ARCHES_FLAG_TX_PACKED))
    return set_err(ARCHES_E_CONFIG, "unknown flags 0x%x", (unsigned)p.flags);
  {
    // The device keeps in-flight control messages in fixed queues of
    // ARCHES_MAX_PENDING (the reference list is unbounded, phy_pipeline.py:
    // 114-117).  A message emitted at the end of slot n is applied at
    // n + 1 + ceil(delay / slot) (+1 selected-only); one is emitted per
    // decision period, so at most ceil(delay / (period * slot)) + 2 are in
    // flight.  Reject the configurations that could exceed the queue.
    const double slot_ns = g.slot_duration_us * 1000.0;
    const double per = (double)p.decision_period_slots * slot_ns;
    const double need = ceil((double)std::max<int64_t>(p.decision_delay_ns, 0) / per) + 2.0;
    if (p.policy == ARCHES_POLICY_TREE && need > ARCHES_MAX_PENDING)
      return set_err(ARCHES_E_CONFIG,
                     "decision delay %lld ns over a %d-slot period keeps up to %.0f control "
                     "messages in flight; the device queue holds %d",
                     (long long)p.decision_delay_ns, p.decision_period_slots, need,
                     ARCHES_MAX_PENDING);
  }

  arches_plan* P = new arches_plan();
  memset(P, 0, sizeof(*P));
  P->g = g;
  P->p = p;
  PlanDev& d = P->dev;
  d.A = g.n_ant;
  d.N = N;
  d.M = M;
  d.T = g.n_sym;
  d.D = g.n_dmrs;
  d.trunc = p.truncation;
  d.guard = p.noise_guard;
  int block = std::min(N, 12 * p.mmse_block_prbs);
  if (N % block) block = N;  // expert_bank.py:166-168
  d.block = block;
  d.n_blocks = N / block;
  const int pil_per_block = block / 2;
  d.diag = (d.n_blocks == 1 && M >= 8) ? 1 : 0;
  d.L = std::max(std::max(p.truncation, p.noise_guard), 8);
  d.n_tiles = (N + ARCHES_TILE - 1) / ARCHES_TILE;
  d.nbt_max = 1;
  for (int t = 0; t < d.n_tiles; ++t) {
    const int k0 = t * ARCHES_TILE, k1 = std::min(N, k0 + ARCHES_TILE) - 1;
    d.nbt_max = std::max(d.nbt_max, std::min(d.n_blocks - 1, k1 / block) - k0 / block + 1);
  }
  for (int j = 0; j < g.n_dmrs; ++j) d.dsym[j] = g.dmrs_symbols[j];
  time_interp(g, d);
  d.ridge = p.ridge;
  // pdp_powers (radio_scene.py:130-137), numpy pairwise order for 8 terms
  double e[8];
  if (p.assumed_delay_spread <= 0) {
    for (int l = 0; l < 8; ++l) d.pdp[l] = l == 0 ? 1.0 : 0.0;
  } else {
    for (int l = 0; l < 8; ++l) e[l] = exp(-(double)l / p.assumed_delay_spread);
    const double sum = ((e[0] + e[1]) + (e[2] + e[3])) + ((e[4] + e[5]) + (e[6] + e[7]));
    for (int l = 0; l < 8; ++l) d.pdp[l] = e[l] / sum;
  }
  for (int l = 0; l < ARCHES_MAX_BINS; ++l) {
    const double ang = 2.0 * M_PI * (double)(l % N) / (double)N;
    d.ai_fac[l] = make_double2((1.0 + cos(ang)) / N, sin(ang) / N);
  }
  // KPM / control
  d.sinr_cap_db = p.sinr_cap_db;
  d.lcid4_fraction = p.lcid4_fraction;
  d.lcid4_jitter = p.lcid4_jitter;
  d.crc_margin_db = p.crc_margin_db;
  d.crc_scale_db = p.crc_scale_db;
  d.slot_us = g.slot_duration_us;
  {
    volatile double us = g.slot_duration_us;
    volatile double s = us * 1e-6;
    d.slot_s = s;
  }
  d.slot_ns = (int64_t)llround(g.slot_duration_us * 1000.0);
  d.n_prb = g.n_prb;
  d.mac_header_bytes = p.mac_header_bytes;
  d.window_length = p.window_length;
  d.n_mcs = p.n_mcs;
  for (int i = 0; i < p.n_mcs; ++i) {
    d.mcs_thr[i] = p.mcs_threshold_db[i];
    d.mcs_rate[i] = p.mcs_rate[i];
    d.mcs_qam[i] = p.mcs_qam[i];
  }
  d.exec_mode = p.exec_mode;
  d.policy = p.policy;
  d.fixed_mode = p.fixed_mode;
  d.decision_period = p.decision_period_slots;
  d.dapp_window = p.dapp_window_slots;
  d.decision_delay_ns = p.decision_delay_ns;
  d.failsafe_timeout_ns = p.failsafe_timeout_ns;
  d.crc_key = p.crc_purpose_key;

  // ---- device tables
  std::vector<float2> wM(M), wN(N), syn((size_t)d.L * ARCHES_TILE);
  for (int j = 0; j < M; ++j) {
    const double a = 2.0 * M_PI * (double)j / (double)M;
    wM[j] = make_float2((float)cos(a), (float)sin(a));
  }
  for (int j = 0; j < N; ++j) {
    const double a = 2.0 * M_PI * (double)j / (double)N;
    wN[j] = make_float2((float)cos(a), (float)sin(a));
  }
  for (int l = 0; l < d.L; ++l)
    for (int j = 0; j < ARCHES_TILE; ++j) {
      const long long idx = ((long long)l * j) % N;
      const double a = -2.0 * M_PI * (double)idx / (double)N;
      syn[(size_t)l * ARCHES_TILE + j] = make_float2((float)cos(a), (float)sin(a));
    }
  std::vector<double2> gram(64);
  for (int l = 0; l < 8; ++l)
    for (int lp = 0; lp < 8; ++lp) {
      double re = 0, im = 0;
      for (int q = 0; q < pil_per_block; ++q) {
        const long long idx = (((long long)(l - lp) * 2 * q) % N + N) % N;
        const double a = 2.0 * M_PI * (double)idx / (double)N;
        re += cos(a);
        im += sin(a);
      }
      gram[l * 8 + lp] = make_double2(re, im);
    }
  // K2 tensor-core operand S[j][kappa] (j < 128, kappa = 2l + c): per row j,
  // per 8-wide K block c: 8 tf32 "hi" values then the 8 matching "lo" values
  // (round-to-nearest split), ready for tcgen05.st into the row's TMEM lane.
  const int lsyn = ((std::max(p.truncation, 8) + 3) / 4) * 4;
  d.tc_kb = lsyn / 4;
  const size_t row_words = (size_t)d.tc_kb * 16;
  std::vector<float> atab((size_t)ARCHES_TILE * row_words, 0.f);
  auto tf32 = [](float x) {
    uint32_t b;
    memcpy(&b, &x, 4);
    b = (b + 0x1000u) & 0xFFFFE000u;  // round to nearest (ties away), 10-bit mantissa
    float r;
    memcpy(&r, &b, 4);
    return r;
  };
  for (int j = 0; j < ARCHES_TILE; ++j)
    for (int kap = 0; kap < 2 * lsyn; ++kap) {
      const int l = kap >> 1;
      const long long idx = ((long long)l * j) % N;
      const double ang = -2.0 * M_PI * (double)idx / (double)N;
      const float x = (float)((kap & 1) ? sin(ang) : cos(ang));
      const float hi = tf32(x), lo = tf32(x - hi);
      const size_t o = (size_t)j * row_words + (size_t)(kap >> 3) * 16 + (kap & 7);
      atab[o] = hi;
      atab[o + 8] = lo;
    }
  // per-tile synthesis rotations (fp64 -> fp32): AI e^{-2 pi i l k0/N} (l < Lsyn),
  // MMSE e^{-2 pi i l (k0 - b block)/N} (l < 8)
  const int rstride = lsyn + 8;
  std::vector<float2> rot((size_t)d.n_tiles * rstride);
  for (int t = 0; t < d.n_tiles; ++t) {
    const int k0 = t * ARCHES_TILE;
    const int b = std::min(k0 / block, d.n_blocks - 1);
    for (int l = 0; l < rstride; ++l) {
      const long long off = l < lsyn ? (long long)l * k0 : (long long)(l - lsyn) * (k0 - b * block);
      const long long idx = ((off % N) + N) % N;
      const double a = -2.0 * M_PI * (double)idx / (double)N;
      rot[(size_t)t * rstride + l] = make_float2((float)cos(a), (float)sin(a));
    }
  }
  const size_t off_wN = align256(M * sizeof(float2));
  const size_t off_syn = off_wN + align256(N * sizeof(float2));
  const size_t off_gram = off_syn + align256(syn.size() * sizeof(float2));
  const size_t off_tca = off_gram + align256(64 * sizeof(double2));
  const size_t off_rot = off_tca + align256(atab.size() * sizeof(float));
  const size_t total = off_rot + align256(rot.size() * sizeof(float2));
  unsigned char* buf = nullptr;
  cudaError_t err = cudaMalloc(&buf, total);
  if (err != cudaSuccess) {
    delete P;
    return set_err(ARCHES_E_CUDA, "cudaMalloc(plan tables): %s", cudaGetErrorString(err));
  }
  cudaMemcpy(buf, wM.data(), M * sizeof(float2), cudaMemcpyHostToDevice);
  cudaMemcpy(buf + off_wN, wN.data(), N * sizeof(float2), cudaMemcpyHostToDevice);
  cudaMemcpy(buf + off_syn, syn.data(), syn.size() * sizeof(float2), cudaMemcpyHostToDevice);
  cudaMemcpy(buf + off_tca, atab.data(), atab.size() * sizeof(float), cudaMemcpyHostToDevice);
  cudaMemcpy(buf + off_rot, rot.data(), rot.size() * sizeof(float2), cudaMemcpyHostToDevice);
  err = cudaMemcpy(buf + off_gram, gram.data(), 64 * sizeof(double2), cudaMemcpyHostToDevice);
  if (err != cudaSuccess) {
    cudaFree(buf);
    delete P;
    return set_err(ARCHES_E_CUDA, "plan table upload: %s", cudaGetErrorString(err));
  }
  P->dev_tables = buf;
  d.wM = reinterpret_cast<const float2*>(buf);
  d.wN = reinterpret_cast<const float2*>(buf + off_wN);
  d.syn = reinterpret_cast<const float2*>(buf + off_syn);
  d.gram = reinterpret_cast<const double2*>(buf + off_gram);
  d.tc_a = reinterpret_cast<const float*>(buf + off_tca);
  d.tc_rot = reinterpret_cast<const float2*>(buf + off_rot);
  {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    d.num_sms = sms > 0 ? sms : 148;
    P->device = dev;
  }

  // ---- K1 launch geometry
  const int AD = d.A * d.D;
  int chunk = std::max(32, std::min(256, (8192 / AD) / 32 * 32));
  if (d.n_blocks > 1) chunk = pil_per_block;  // one CTA per MMSE block
  P->k1_chunk = chunk;
  P->k1_parts = (M + chunk - 1) / chunk;
  auto k1_smem = [&](int ch) {
    const size_t stage = std::max((size_t)AD * ch, (size_t)ARCHES_K1_THREADS * ARCHES_RA * ARCHES_RL);
    return stage * sizeof(float2) + (size_t)AD * d.L * sizeof(double2) + 64 * sizeof(double2);
  };
  P->k1_smem = k1_smem(chunk);
  {
    // tensor-core K1: one MMSE block (closed-form taps), <= 4 DMRS symbols, 2L <= 128
    P->k1t_nb = 0;
    P->k1t_wimg = nullptr;
    P->k1t_nchunks = (N + K1T_CSC - 1) / K1T_CSC;
    const int nb = ((2 * d.L + 15) / 16) * 16;
    if (d.diag && d.D <= 4 && d.L == 20 && P->k1t_nchunks * K1T_SUBS <= K1T_MAX_SUB &&
        !(p.flags & ARCHES_FLAG_NO_TC_K1)) {  // k1_tc<48, 40>
      // chunk-invariant operand W[p][l] = e^{2 pi i l p / M} (p < 16 comb points),
      // real-embedded: kappa = 2p + (0: Re h, 1: Im h), row n = 2l + (0: Re, 1: Im);
      // [n][32 floats] in the SWIZZLE_128B layout, tf32 hi then lo
      const size_t half = (size_t)nb * 32;  // floats of one of hi | lo
      std::vector<float> img(2 * half, 0.f);
      auto tf32 = [](float x) {
        uint32_t b;
        memcpy(&b, &x, 4);
        b = (b + 0x1000u) & 0xFFFFE000u;
        float r;
        memcpy(&r, &b, 4);
        return r;
      };
      for (int pp = 0; pp < K1T_CP; ++pp)
        for (int n = 0; n < 2 * d.L; ++n) {
          const int l = n >> 1;
          const long long idx = ((long long)l * pp) % M;
          const double ang = 2.0 * M_PI * (double)idx / (double)M;
          const float wr = (float)cos(ang), wi = (float)sin(ang);
          const float bv[2] = {(n & 1) ? wi : wr, (n & 1) ? wr : -wi};
          for (int cc = 0; cc < 2; ++cc) {
            const int kap = 2 * pp + cc, grp = kap >> 2;
            const float hi = tf32(bv[cc]), lo = tf32(bv[cc] - hi);
            const size_t o = (size_t)n * 32 + (size_t)((grp ^ (n & 7)) * 4) + (kap & 3);
            img[o] = hi;
            img[half + o] = lo;
          }
        }
      // sub-chunk phases e^{2 pi i l 16c / M}, rows padded to K1T_LP
      std::vector<float2> rot((size_t)P->k1t_nchunks * K1T_SUBS * K1T_LP, make_float2(0.f, 0.f));
      for (int c = 0; c < P->k1t_nchunks * K1T_SUBS; ++c)
        for (int l = 0; l < d.L; ++l) {
          const long long idx = ((long long)l * K1T_CP * c) % M;
          const double ang = 2.0 * M_PI * (double)idx / (double)M;
          rot[(size_t)c * K1T_LP + l] = make_float2((float)cos(ang), (float)sin(ang));
        }
      const size_t rot_off = (img.size() * sizeof(float) + 255) & ~(size_t)255;
      unsigned char* dimg = nullptr;
      const size_t bytes = rot_off + rot.size() * sizeof(float2);
      if (cudaMalloc(&dimg, bytes) == cudaSuccess &&
          cudaMemcpy(dimg, img.data(), img.size() * sizeof(float), cudaMemcpyHostToDevice) == cudaSuccess &&
          cudaMemcpy(dimg + rot_off, rot.data(), rot.size() * sizeof(float2), cudaMemcpyHostToDevice) ==
              cudaSuccess) {
        P->k1t_wimg = reinterpret_cast<float*>(dimg);
        P->k1t_rot = reinterpret_cast<float2*>(dimg + rot_off);
        P->k1t_nb = nb;
      } else if (dimg) {
        cudaFree(dimg);
      }
    }
  }
  P->k1_full_chunk = std::max(32, std::min(256, (8192 / AD) / 32 * 32));
  P->k1_full_parts = (N + P->k1_full_chunk - 1) / P->k1_full_chunk;
  P->k1_full_smem = k1_smem(P->k1_full_chunk);
  P->k2_smem = ((size_t)(d.A + 1) * d.T * ARCHES_TILE + (size_t)d.nbt_max * AD * 8 +
                (size_t)AD * d.trunc) * sizeof(float2);
  {
    // tcgen05 K2: n_ant in {1,2,4} (padded), tiles inside one MMSE block; more
    // antennas (a multiple of 4, NR 0/5/10 DMRS pattern) run in groups of 4
    const bool std_pat = d.T == 14 && d.D == 3 && d.dsym[0] == 0 && d.dsym[1] == 5 && d.dsym[2] == 10;
    const bool grp = d.A > 4 && d.A % 4 == 0 && std_pat;
    const int na = d.A <= 1 ? 1 : d.A <= 2 ? 2 : d.A <= 4 ? 4 : grp ? 4 : 0;
    const bool tile_ok = d.n_blocks == 1 || (d.block % ARCHES_TILE) == 0;
    size_t sm = 0;
    if (na && tile_ok && 16 * d.tc_kb <= 128 && !(p.flags & ARCHES_FLAG_NO_TC_K2)) {
      const int R = 2 * na * d.D, ncol = ((2 * R + 15) / 16) * 16, ng = ncol / 8;
      const int n_b = (ncol / 2) * 4 * d.tc_kb;  // B entries: <= 2 per thread of 512
      const int as = grp ? 4 : d.A;               // antennas per stage
      const int nbuf = 3;  // B operands in flight (k2_tc NBUF = LEAD + 1)
      // two y (+ tx) stages; antenna groups keep the tile's tx rows in one extra buffer;
      // packed tx: the tile's 2-bit codes (padded to 512 B) instead of its tx rows
      sm = (p.flags & ARCHES_FLAG_TX_PACKED)
               ? 3 * ((size_t)as * d.T * ARCHES_TILE * sizeof(float2) + 512)  // k2_tc NST = 3
               : (2 * (size_t)(as + (grp ? 0 : 1)) + (grp ? 1 : 0)) * d.T * ARCHES_TILE * sizeof(float2);
      sm += 2 * nbuf * (size_t)d.tc_kb * ng * 256;
      if (grp) sm += (size_t)21 * TC_THREADS * sizeof(float);  // MRC sums across groups
      if (sm > 227 * 1024 || n_b > 2 * TC_THREADS || ncol > 64) sm = 0;
      // the per-tile phase rotations in shared memory when they fit
      const size_t rot_bytes = (size_t)d.n_tiles * (4 * d.tc_kb + 8) * sizeof(float2);
      d.k2_rot_smem = 0;
      if (sm && sm + rot_bytes <= 227 * 1024) {
        sm += rot_bytes;
        d.k2_rot_smem = 1;
      }
    }
    P->k2_tc_smem = sm;
    P->k2_groups = grp && sm ? d.A / 4 : 1;
    d.tx_packed = (p.flags & ARCHES_FLAG_TX_PACKED) ? 1 : 0;
    if (d.tx_packed && !(sm && !grp && std_pat && na == d.A && d.T * ARCHES_TXB_ROW <= 512)) {
      cudaFree(buf);
      if (P->k1t_wimg) cudaFree(P->k1t_wimg);
      delete P;
      return set_err(ARCHES_E_CONFIG,
                     "ARCHES_FLAG_TX_PACKED needs the tensor-core K2 over one antenna group "
                     "(n_ant 1, 2 or 4, DMRS symbols 0/5/10)");
    }
  }
  if (P->k2_smem > 200 * 1024 && !(P->k2_tc_smem && P->k2_groups > 1)) {
    cudaFree(buf);
    if (P->k1t_wimg) cudaFree(P->k1t_wimg);
    delete P;
    return set_err(ARCHES_E_CONFIG, "K2 tile does not fit shared memory (n_ant too large)");
  }
  if (cudaStreamCreateWithFlags(&P->side, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&P->tail, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&P->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&P->ev_join, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&P->ev_start, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&P->ev_k2, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&P->ev_k3, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&P->ev_end, cudaEventDisableTiming) != cudaSuccess) {
    const cudaError_t e = cudaGetLastError();
    arches_plan_destroy(P);
    return set_err(ARCHES_E_CUDA, "plan streams/events: %s", cudaGetErrorString(e));
  }
  *out = P;
  return ARCHES_OK;
}

extern "C" int arches_plan_destroy(arches_plan* plan) {
  if (!plan) return ARCHES_OK;
  int cur = -1;
  cudaGetDevice(&cur);
  if (cur != plan->device) cudaSetDevice(plan->device);
  for (cudaStream_t st : {plan->tail, plan->side})
    if (st) {
      cudaStreamSynchronize(st);
      cudaStreamDestroy(st);
    }
  for (cudaEvent_t ev : {plan->ev_fork, plan->ev_join, plan->ev_start, plan->ev_k2, plan->ev_k3,
                         plan->ev_end})
    if (ev) cudaEventDestroy(ev);
  if (plan->dev_tables) cudaFree(plan->dev_tables);
  if (plan->k1t_wimg) cudaFree(plan->k1t_wimg);
  if (cur >= 0 && cur != plan->device) cudaSetDevice(cur);
  delete plan;
  return ARCHES_OK;
}

extern "C" int32_t arches_plan_bins(const arches_plan* plan) { return plan ? plan->dev.L : 0; }

extern "C" size_t arches_state_bytes(const arches_plan* plan, int32_t n_streams) {
  return (size_t)n_streams * state_stride_bytes(plan->dev.window_length, plan->dev.dapp_window);
}

extern "C" size_t arches_workspace_bytes(const arches_plan* plan, int32_t n_units) {
  return ws_layout(plan, n_units).total;
}

extern "C" int arches_state_init(const arches_plan* plan, void* state, int32_t n_streams,
                                 arches_stream_t stream) {
  if (!plan || !state || n_streams < 1) return set_err(ARCHES_E_CONTRACT, "bad state_init args");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  CUDA_TRY(cudaMemsetAsync(state, 0, arches_state_bytes(plan, n_streams), s));
  k4_state_init<<<(n_streams + 127) / 128, 128, 0, s>>>(plan->dev, state, n_streams);
  LAUNCH_CHECK();
  return ARCHES_OK;
}

// ------------------------------------------------------------ K1
template <class Src>
static int launch_k1(const arches_plan* P, int n_units, const Src& src, const K1Out& o, int npts,
                     int chunk, size_t smem, cudaStream_t s) {
  auto kern = k1_analyze<Src>;
  CUDA_TRY(ensure_smem(kern, smem));
  dim3 grid((npts + chunk - 1) / chunk, n_units);
  kern<<<grid, ARCHES_K1_THREADS, smem, s>>>(P->dev, src, o, npts, chunk);
  LAUNCH_CHECK();
  return ARCHES_OK;
}

static K1TGeom k1t_geom(const arches_plan* P, int n_streams, int n_slots) {
  const PlanDev& d = P->dev;
  K1TGeom g;
  g.gps = (n_slots * d.A + K1T_RR - 1) / K1T_RR;
  g.n_g = n_streams * g.gps;
  g.n_items = g.n_g * d.D * P->k1t_nchunks;
  g.grid = std::max(1, std::min(g.n_items, persistent_sms(d)));
  return g;
}


typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_tiled();

// launch with programmatic stream serialization: the kernel may start while the
// previous kernel of the stream drains and synchronises with griddepcontrol.wait
template <typename K, typename... Args>
static cudaError_t launch_pdl(K kern, dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args... args) {
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

static int launch_k1t(const arches_plan* P, int n_units, const GridCombSrc& src, const K1Out& o,
                      const WsLayout& w, void* ws, cudaStream_t s) {
  const PlanDev& d = P->dev;
  const K1TGeom kg = k1t_geom(P, n_units / src.n_slots, src.n_slots);
  if ((long long)kg.n_items * kg.grid >= (1LL << 31)) return set_err(ARCHES_E_CONFIG, "K1: batch too large");
  K1TArgs a;
  a.y = src.y;
  a.pil = src.pil;
  a.wimg = P->k1t_wimg;
  a.rot = P->k1t_rot;
  a.dpart = ws_at<double>(ws, w.k1t_d);
  a.epart = ws_at<double>(ws, w.k1t_e);
  a.n_slots = src.n_slots;
  a.srows = src.n_slots * d.A;
  a.n_rows = n_units * d.A;
  a.gps = kg.gps;
  a.n_g = kg.n_g;
  a.n_chunks = P->k1t_nchunks;
  a.n_items = kg.n_items;
  a.grid = kg.grid;
  a.nb = P->k1t_nb;
  if ((reinterpret_cast<uintptr_t>(src.y) & 15) || (d.N & 1))
    return set_err(ARCHES_E_CONTRACT, "K1: grid rows must be 16-byte aligned");
  const int grid = kg.grid;
  const size_t smem = k1t_smem_bytes(a.nb, a.n_chunks);
  const int nchunk = k1t_fin_chunks(d);
  CUDA_TRY(ensure_smem(k1_tc<48, 40>, smem));
  // (a programmatic launch behind the previous batch's K2 measured 2.4% slower
  // per step: its waiting CTAs take SMs from the tail stream's K3 / K4)
  k1_tc<48, 40><<<grid, K1T_THREADS, smem, s>>>(d, a);
  LAUNCH_CHECK();
  if (g_hook.before_fin) CUDA_TRY(cudaStreamWaitEvent(s, g_hook.before_fin, 0));
  {
    // programmatic dependent launch: the finalize's CTAs are scheduled while K1's
    // last CTAs drain (launch latency off the critical path) and wait in-kernel
    cudaLaunchConfig_t cfg;
    memset(&cfg, 0, sizeof(cfg));
    cfg.gridDim = dim3(n_units * nchunk);
    cfg.blockDim = dim3(K1T_FIN_THREADS);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (nchunk > 1) {
      CUDA_TRY(cudaLaunchKernelEx(&cfg, k1_tc_finalize_rows, d, a, nchunk, o,
                                  ws_at<double>(ws, w.k1t_share)));
      LAUNCH_CHECK();
      cfg.blockDim = dim3(K1T_FIN_ROWS * 32);
      CUDA_TRY(cudaLaunchKernelEx(&cfg, k1_tc_finalize_taps, d, nchunk, o,
                                  static_cast<const double*>(ws_at<double>(ws, w.k1t_share))));
    } else
      CUDA_TRY(cudaLaunchKernelEx(&cfg, k1_tc_finalize, d, a, n_units, o));
  }
  LAUNCH_CHECK();
  return ARCHES_OK;
}

static int launch_rng(const arches_plan* plan, int n_streams, int n_slots, const uint64_t* seeds,
                      int64_t first_slot, const void* state, void* ws, cudaStream_t s) {
  const int n_units = n_streams * n_slots;
  const WsLayout w = ws_layout(plan, n_units);
  k_rng_units<<<(n_units + 127) / 128, 128, 0, s>>>(
      plan->dev, ws_at<double>(ws, w.rng), seeds, reinterpret_cast<const unsigned char*>(state),
      state_stride_bytes(plan->dev.window_length, plan->dev.dapp_window), first_slot, n_slots,
      n_units);
  LAUNCH_CHECK();
  return ARCHES_OK;
}

static int ls_analyze_impl(const arches_plan* plan, int32_t n_streams, int32_t n_slots,
                           const void* y, const void* pilots, const uint64_t* seeds,
                           int64_t first_slot, const void* state, double* sigma2_hat, void* ws,
                           arches_stream_t stream, bool with_rng);

extern "C" int arches_ls_analyze(const arches_plan* plan, int32_t n_streams, int32_t n_slots,
                                 const void* y, const void* pilots, const uint64_t* seeds,
                                 int64_t first_slot, const void* state, double* sigma2_hat,
                                 void* ws, arches_stream_t stream) {
  return ls_analyze_impl(plan, n_streams, n_slots, y, pilots, seeds, first_slot, state, sigma2_hat,
                         ws, stream, true);
}

static int ls_analyze_impl(const arches_plan* plan, int32_t n_streams, int32_t n_slots,
                           const void* y, const void* pilots, const uint64_t* seeds,
                           int64_t first_slot, const void* state, double* sigma2_hat, void* ws,
                           arches_stream_t stream, bool with_rng) {
  if (!plan || !y || !pilots || !ws || n_streams < 1 || n_slots < 1)
    return set_err(ARCHES_E_CONTRACT, "bad ls_analyze args");
  const int n_units = n_streams * n_slots;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const WsLayout w = ws_layout(plan, n_units);
  GridCombSrc src{reinterpret_cast<const float2*>(y), reinterpret_cast<const float2*>(pilots), n_slots};
  if (!plan->k1t_nb)  // last-CTA counters of the CUDA-core K1 (the tensor-core K1 has none)
    CUDA_TRY(cudaMemsetAsync(ws_at<void>(ws, w.k1counters), 0, n_units * sizeof(unsigned int), s));
  if (seeds && first_slot < 0 && !state)
    return set_err(ARCHES_E_CONTRACT, "first_slot < 0 needs the stream state (slot source)");
  if (seeds && with_rng) {  // RNG side products for K3 (run_batch forks them onto a side stream)
    const int rc = launch_rng(plan, n_streams, n_slots, seeds, first_slot, state, ws, s);
    if (rc) return rc;
  }
  K1Out o{ws_at<double>(ws, w.sigma2), nullptr, ws_at<float2>(ws, w.coef),
          ws_at<double>(ws, w.k1parts), ws_at<unsigned int>(ws, w.k1counters),
          K1_NOISE | K1_MMSE | K1_AI, nullptr, seeds,
          reinterpret_cast<const unsigned char*>(state),
          state_stride_bytes(plan->dev.window_length, plan->dev.dapp_window), first_slot, n_slots};
  if (!plan->k1t_nb && g_hook.before_fin)  // the CUDA-core K1 finalises in line
    CUDA_TRY(cudaStreamWaitEvent(s, g_hook.before_fin, 0));
  int rc = plan->k1t_nb ? launch_k1t(plan, n_units, src, o, w, ws, s)
                        : launch_k1(plan, n_units, src, o, plan->dev.M, plan->k1_chunk, plan->k1_smem, s);
  if (rc) return rc;
  if (sigma2_hat)
    CUDA_TRY(cudaMemcpyAsync(sigma2_hat, ws_at<double>(ws, w.sigma2), n_units * sizeof(double),
                             cudaMemcpyDeviceToDevice, s));
  return ARCHES_OK;
}

// ------------------------------------------------------------ K2
template <int NE>
static int launch_k2(const arches_plan* P, int n_units, const K2Args& a, cudaStream_t s) {
  const PlanDev& d = P->dev;
  dim3 grid(d.n_tiles, n_units);
  const size_t smem = P->k2_smem;
  int na = d.A <= 1 ? 1 : d.A <= 2 ? 2 : d.A <= 4 ? 4 : d.A <= 8 ? 8 : 0;
  if (!na) return set_err(ARCHES_E_CONFIG, "device equaliser path supports n_ant <= 8 (got %d)", d.A);
#define K2_CASE(NA_, ND_)                                                                   \
  if (na == NA_ && d.D == ND_) {                                                            \
    auto kern = k2_synth_equalize<NA_, ND_, NE>;                                            \
    CUDA_TRY(ensure_smem(kern, smem)); \
    kern<<<grid, ARCHES_TILE, smem, s>>>(d, a);                                             \
    LAUNCH_CHECK();                                                                         \
    return ARCHES_OK;                                                                       \
  }
  K2_CASE(1, 1) K2_CASE(1, 2) K2_CASE(1, 3) K2_CASE(1, 4)
  K2_CASE(2, 1) K2_CASE(2, 2) K2_CASE(2, 3) K2_CASE(2, 4)
  K2_CASE(4, 1) K2_CASE(4, 2) K2_CASE(4, 3) K2_CASE(4, 4)
  K2_CASE(8, 1) K2_CASE(8, 2) K2_CASE(8, 3) K2_CASE(8, 4)
#undef K2_CASE
  return set_err(ARCHES_E_CONFIG, "unsupported (n_ant, n_dmrs) = (%d, %d)", d.A, d.D);
}

static int experts_equalize_impl(const arches_plan* plan, int32_t n_streams, int32_t n_slots,
                                 const void* y, const void* tx, const double* noise_var,
                                 const uint64_t* seeds, int64_t first_slot, const void* state,
                                 void* h_mmse, void* h_ai, arches_telemetry* tel, void* ws,
                                 arches_stream_t stream, bool rng_from_k1);

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
static EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
    cudaGetLastError();
  });
  return fn;
}

// [units][rows][N] complex64 viewed as fp32 [units][rows][2N]; box = one
// 128-subcarrier tile of all rows of one unit
static bool make_row_tmap(CUtensorMap* m, const void* base, int N, int rows, int units,
                          int box_rows = 0) {
  EncodeTiledFn enc = encode_tiled();
  if (box_rows <= 0) box_rows = rows;
  if (!enc || (N & 1) || box_rows > 256 || (reinterpret_cast<uintptr_t>(base) & 15)) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)2 * N, (cuuint64_t)rows, (cuuint64_t)units};
  const cuuint64_t strides[2] = {(cuuint64_t)8 * N, (cuuint64_t)8 * N * rows};
  const cuuint32_t box[3] = {2 * ARCHES_TILE, (cuuint32_t)box_rows, 1};
  const cuuint32_t es[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static int launch_k2_tc(const arches_plan* P, int n_units, const K2Args& a, cudaStream_t s) {
  const PlanDev& d = P->dev;
  const int ngrp = P->k2_groups;
  const int n_items = n_units * d.n_tiles * ngrp;
  const int grid = std::min(n_units * d.n_tiles, persistent_sms(d));  // persistent: one CTA per SM
  const size_t smem = P->k2_tc_smem;
  const int na = d.A <= 1 ? 1 : d.A <= 2 ? 2 : 4;
  const bool std_pat = d.T == 14 && d.D == 3 && d.dsym[0] == 0 && d.dsym[1] == 5 && d.dsym[2] == 10;
  CUtensorMap tm_y, tm_x;
  memset(&tm_y, 0, sizeof(tm_y));
  memset(&tm_x, 0, sizeof(tm_x));
  // tensor maps need 16-byte aligned bases; otherwise the CUDA-core loads
  const bool tmap = make_row_tmap(&tm_y, a.y, d.N, d.A * d.T, n_units, ngrp > 1 ? 4 * d.T : 0) &&
                    (d.tx_packed || make_row_tmap(&tm_x, a.tx, d.N, d.T, n_units));
  if (d.tx_packed) {  // packed tx: y through the tensor map, the tile's codes by one bulk copy
    if (!tmap || (reinterpret_cast<uintptr_t>(a.tx) & 15))
      return set_err(ARCHES_E_CONTRACT, "packed tx needs 16-byte aligned y and tx");
#define K2TC_PK(NA_)                                                                        \
    if (d.A == NA_) {                                                                       \
      auto kern = k2_tc<NA_, 3, true, true, false, true>;                                   \
      CUDA_TRY(ensure_smem(kern, smem));                                                    \
      CUDA_TRY(launch_pdl(kern, dim3(grid), dim3(TC_BLOCK), smem, s, d, a, n_items, tm_y, tm_x)); \
      LAUNCH_CHECK();                                                                       \
    }
    K2TC_PK(4) else K2TC_PK(2) else K2TC_PK(1) else return set_err(ARCHES_E_CONFIG, "packed tx: n_ant");
#undef K2TC_PK
    cudaStream_t s3 = s;
    if (g_hook.k3_stream) {
      CUDA_TRY(cudaEventRecord(g_hook.k2_done, s));
      CUDA_TRY(cudaStreamWaitEvent(g_hook.k3_stream, g_hook.k2_done, 0));
      s3 = g_hook.k3_stream;
      g_hook.k3_on_tail = true;
    }
    k3_finalize<<<(n_units * 32 + K3_THREADS - 1) / K3_THREADS, K3_THREADS, 0, s3>>>(d, a, n_units,
                                                                                     n_items, grid);
    LAUNCH_CHECK();
    return ARCHES_OK;
  }
#define K2TC_LAUNCH_G(NA_, ND_, STD_, GRP_)                                                  \
  {                                                                                          \
    auto kern = tmap ? k2_tc<NA_, ND_, STD_, true, GRP_> : k2_tc<NA_, ND_, STD_, false, GRP_>; \
    CUDA_TRY(ensure_smem(kern, smem));                                                       \
    CUDA_TRY(launch_pdl(kern, dim3(grid), dim3(GRP_ ? TC_THREADS : TC_BLOCK), smem, s, d, a, n_items, tm_y, tm_x)); \
    LAUNCH_CHECK();                                                                          \
    /* K3 locates the (CTA, unit) segments in tile units */                                  \
    cudaStream_t s3 = s;                                                                     \
    if (g_hook.k3_stream) {                                                                  \
      CUDA_TRY(cudaEventRecord(g_hook.k2_done, s));                                          \
      CUDA_TRY(cudaStreamWaitEvent(g_hook.k3_stream, g_hook.k2_done, 0));                    \
      s3 = g_hook.k3_stream;                                                                 \
      g_hook.k3_on_tail = true;                                                              \
    }                                                                                        \
    k3_finalize<<<(n_units * 32 + K3_THREADS - 1) / K3_THREADS, K3_THREADS, 0, s3>>>(        \
        d, a, n_units, n_items / ngrp, grid);                                                \
    LAUNCH_CHECK();                                                                          \
    return ARCHES_OK;                                                                        \
  }
#define K2TC_LAUNCH(NA_, ND_, STD_) K2TC_LAUNCH_G(NA_, ND_, STD_, false)
  if (ngrp > 1) K2TC_LAUNCH_G(4, 3, true, true)  /* massive MIMO: groups of 4 antennas */
#define K2TC_CASE(NA_, ND_)                                                                  \
  if (na == NA_ && d.D == ND_) K2TC_LAUNCH(NA_, ND_, false)
  if (std_pat && d.A == 4) K2TC_LAUNCH(4, 3, true)  /* kStd: exact n_ant, NR 0/5/10 pattern */
  if (std_pat && d.A == 2) K2TC_LAUNCH(2, 3, true)
  if (std_pat && d.A == 1) K2TC_LAUNCH(1, 3, true)
  K2TC_CASE(1, 1) K2TC_CASE(1, 2) K2TC_CASE(1, 3) K2TC_CASE(1, 4)
  K2TC_CASE(2, 1) K2TC_CASE(2, 2) K2TC_CASE(2, 3) K2TC_CASE(2, 4)
  K2TC_CASE(4, 1) K2TC_CASE(4, 2) K2TC_CASE(4, 3) K2TC_CASE(4, 4)
#undef K2TC_CASE
#undef K2TC_LAUNCH
#undef K2TC_LAUNCH_G
  return launch_k2<2>(P, n_units, a, s);
}

extern "C" int arches_experts_equalize(const arches_plan* plan, int32_t n_streams, int32_t n_slots,
                                       const void* y, const void* tx, const double* noise_var,
                                       const uint64_t* seeds, int64_t first_slot,
                                       const void* state, void* h_mmse, void* h_ai,
                                       arches_telemetry* tel, void* ws, arches_stream_t stream) {
  return experts_equalize_impl(plan, n_streams, n_slots, y, tx, noise_var, seeds, first_slot,
                               state, h_mmse, h_ai, tel, ws, stream, false);
}

static int experts_equalize_impl(const arches_plan* plan, int32_t n_streams, int32_t n_slots,
                                 const void* y, const void* tx, const double* noise_var,
                                 const uint64_t* seeds, int64_t first_slot, const void* state,
                                 void* h_mmse, void* h_ai, arches_telemetry* tel, void* ws,
                                 arches_stream_t stream, bool rng_from_k1) {
  if (!plan || !y || !tx || !noise_var || !seeds || !ws || !tel || n_streams < 1 || n_slots < 1)
    return set_err(ARCHES_E_CONTRACT, "bad experts_equalize args");
  if (first_slot < 0 && !state)
    return set_err(ARCHES_E_CONTRACT, "first_slot < 0 needs the stream state (slot source)");
  const int n_units = n_streams * n_slots;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const WsLayout w = ws_layout(plan, n_units);
  if (!plan->k2_tc_smem)  // the FFMA form's last-CTA counters (the tensor-core form uses K3)
    CUDA_TRY(cudaMemsetAsync(ws_at<void>(ws, w.counters), 0, n_units * sizeof(unsigned int), s));
  K2Args a;
  memset(&a, 0, sizeof(a));
  a.y = reinterpret_cast<const float2*>(y);
  a.tx = reinterpret_cast<const float2*>(tx);
  a.coef = ws_at<float2>(ws, w.coef);
  a.nv = noise_var;
  a.sigma2 = ws_at<double>(ws, w.sigma2);
  a.seeds = seeds;
  a.h_mmse = reinterpret_cast<float2*>(h_mmse);
  a.h_ai = reinterpret_cast<float2*>(h_ai);
  a.parts = ws_at<TilePartial>(ws, w.parts);
  a.counters = ws_at<unsigned int>(ws, w.counters);
  a.tel = tel;
  a.state = reinterpret_cast<const unsigned char*>(state);
  a.state_stride = state_stride_bytes(plan->dev.window_length, plan->dev.dapp_window);
  a.first_slot = first_slot;
  a.n_slots = n_slots;
  a.rng = rng_from_k1 ? ws_at<double>(ws, w.rng) : nullptr;
  if (plan->k2_tc_smem) return launch_k2_tc(plan, n_units, a, s);
  return launch_k2<2>(plan, n_units, a, s);
}

extern "C" int32_t arches_batch_kernels(const arches_plan* plan) {
  if (!plan) return 0;
  const int k1 = plan->k1t_nb ? 1 + (k1t_fin_chunks(plan->dev) > 1 ? 2 : 1) : 1;
  const int k2 = plan->k2_tc_smem ? 2 : 1;  // tensor-core K2 + K3, or the FFMA form
  return 1 + k1 + k2 + 1;                    // + RNG, K4
}

// ------------------------------------------------------------ K4 / K5
extern "C" int arches_kpm_scan(const arches_plan* plan, int32_t n_streams, int32_t n_slots,
                               const arches_telemetry* tel, const int8_t* regime,
                               const arches_tree* tree, void* state, arches_kpm* kpm,
                               arches_message* msg_log, int32_t* msg_count, int32_t msg_cap,
                               arches_stream_t stream) {
  if (!plan || !tel || !state || !kpm || n_streams < 1 || n_slots < 1)
    return set_err(ARCHES_E_CONTRACT, "bad kpm_scan args");
  if (plan->dev.policy == ARCHES_POLICY_TREE && !tree)
    return set_err(ARCHES_E_CONTRACT, "tree policy needs a tree");
  if (plan->dev.policy == ARCHES_POLICY_ORACLE && !regime)
    return set_err(ARCHES_E_CONTRACT, "oracle policy needs the regime timeline");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  K4Args a{tel, regime, tree, state, kpm, msg_log, msg_count, msg_cap, n_streams, n_slots};
  k4_kpm_scan_block<<<n_streams, K4B_THREADS, 0, s>>>(plan->dev, a);
  LAUNCH_CHECK();
  return ARCHES_OK;
}

extern "C" int arches_kpm_scan_sequential(const arches_plan* plan, int32_t n_streams,
                                          int32_t n_slots, const arches_telemetry* tel,
                                          const int8_t* regime, const arches_tree* tree,
                                          void* state, arches_kpm* kpm, arches_message* msg_log,
                                          int32_t* msg_count, int32_t msg_cap,
                                          arches_stream_t stream) {
  if (!plan || !tel || !state || !kpm || n_streams < 1 || n_slots < 1)
    return set_err(ARCHES_E_CONTRACT, "bad kpm_scan args");
  if (plan->dev.policy == ARCHES_POLICY_TREE && !tree)
    return set_err(ARCHES_E_CONTRACT, "tree policy needs a tree");
  if (plan->dev.policy == ARCHES_POLICY_ORACLE && !regime)
    return set_err(ARCHES_E_CONTRACT, "oracle policy needs the regime timeline");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  K4Args a{tel, regime, tree, state, kpm, msg_log, msg_count, msg_cap, n_streams, n_slots};
  k4_kpm_scan<<<(n_streams + 31) / 32, 32, 0, s>>>(plan->dev, a);
  LAUNCH_CHECK();
  return ARCHES_OK;
}

extern "C" int arches_run_batch(const arches_plan* plan, int32_t n_streams, int32_t n_slots,
                                int64_t first_slot, const void* y, const void* tx,
                                const void* pilots, const double* noise_var, const uint64_t* seeds,
                                const int8_t* regime, const arches_tree* tree, void* state,
                                void* h_mmse, void* h_ai, arches_telemetry* tel, arches_kpm* kpm,
                                arches_message* msg_log, int32_t* msg_count, int32_t msg_cap,
                                void* ws, arches_stream_t stream) {
  if (!plan || !seeds) return set_err(ARCHES_E_CONTRACT, "bad run_batch args");
  if (first_slot < 0 && !state)
    return set_err(ARCHES_E_CONTRACT, "first_slot < 0 needs the stream state (slot source)");
  if (plan->tail_pending) {  // a pipelined batch is still in flight: order after it
    const int rc = arches_join(plan, stream);
    if (rc) return rc;
  }
  // fork: the RNG side products (independent of the grid) on the plan's side
  // stream next to K1; join before K2 / K3 consume them (a fork-join node pair
  // when the caller captures this into a CUDA graph)
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  cudaStream_t side = plan->side;
  cudaEvent_t ev_fork = plan->ev_fork, ev_join = plan->ev_join;
  CUDA_TRY(cudaEventRecord(ev_fork, s));
  CUDA_TRY(cudaStreamWaitEvent(side, ev_fork, 0));
  int rc = launch_rng(plan, n_streams, n_slots, seeds, first_slot, state, ws, side);
  if (rc) return rc;
  CUDA_TRY(cudaEventRecord(ev_join, side));
  rc = ls_analyze_impl(plan, n_streams, n_slots, y, pilots, seeds, first_slot, state, nullptr, ws,
                       stream, false);
  if (rc) return rc;
  CUDA_TRY(cudaStreamWaitEvent(s, ev_join, 0));
  rc = experts_equalize_impl(plan, n_streams, n_slots, y, tx, noise_var, seeds, first_slot,
                             state, h_mmse, h_ai, tel, ws, stream, /* RNG side products */ true);
  if (rc) return rc;
  return arches_kpm_scan(plan, n_streams, n_slots, tel, regime, tree, state, kpm, msg_log,
                         msg_count, msg_cap, stream);
}

extern "C" int arches_join(const arches_plan* plan, arches_stream_t stream) {
  if (!plan) return set_err(ARCHES_E_CONTRACT, "bad join args");
  const arches_plan* P = plan;
  if (!P->tail_pending) return ARCHES_OK;
  CUDA_TRY(cudaStreamWaitEvent(reinterpret_cast<cudaStream_t>(stream), P->ev_end, 0));
  P->tail_pending = false;
  return ARCHES_OK;
}

// Cross-batch pipeline.  Per call (batch n), with T the plan's tail stream:
//   T:      RNG(n)                         (after K4(n-1): the slot counter)
//   stream: K1(n) -> [K3(n-1) done] -> K1 finalize(n) -> K2(n)
//   T:      [K2(n) done] -> K3(n) -> K4(n)
// Buffer hazards: K1 finalize(n) overwrites sigma2 (read by K3(n-1)) and K2(n)
// the segment partials (read by K3(n-1)) -- both wait for K3(n-1); RNG(n) /
// K3(n) overwrite rng / tel read by K3(n-1) / K4(n-1), ordered on T.  The
// K3 / K4 of batch n thus overlap K1 of batch n+1.
extern "C" int arches_run_batch_async(const arches_plan* plan, int32_t n_streams, int32_t n_slots,
                                      int64_t first_slot, const void* y, const void* tx,
                                      const void* pilots, const double* noise_var,
                                      const uint64_t* seeds, const int8_t* regime,
                                      const arches_tree* tree, void* state, void* h_mmse,
                                      void* h_ai, arches_telemetry* tel, arches_kpm* kpm,
                                      arches_message* msg_log, int32_t* msg_count,
                                      int32_t msg_cap, void* ws, arches_stream_t stream) {
  if (!plan || !seeds) return set_err(ARCHES_E_CONTRACT, "bad run_batch_async args");
  if (first_slot < 0 && !state)
    return set_err(ARCHES_E_CONTRACT, "first_slot < 0 needs the stream state (slot source)");
  const arches_plan* P = plan;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (!P->k2_tc_smem) {
    // The FFMA K2 finalises its units in its last CTA on `stream`: it reads the
    // RNG side products and writes tel, both owned by the tail stream in the
    // pipelined form.  Such plans (tiles straddling MMSE blocks, n_ant 3 / 5-7)
    // run the ordered single-stream form instead -- same results.
    return arches_run_batch(plan, n_streams, n_slots, first_slot, y, tx, pilots, noise_var, seeds,
                            regime, tree, state, h_mmse, h_ai, tel, kpm, msg_log, msg_count,
                            msg_cap, ws, stream);
  }
  struct HookGuard {
    ~HookGuard() { g_hook = TailHook(); }
  } guard;
  CUDA_TRY(cudaEventRecord(P->ev_start, s));  // T follows what the caller queued so far
  CUDA_TRY(cudaStreamWaitEvent(P->tail, P->ev_start, 0));
  int rc = launch_rng(plan, n_streams, n_slots, seeds, first_slot, state, ws, P->tail);
  if (rc) return rc;
  g_hook.before_fin = P->tail_pending ? P->ev_k3 : nullptr;
  g_hook.k3_stream = P->tail;
  g_hook.k2_done = P->ev_k2;
  rc = ls_analyze_impl(plan, n_streams, n_slots, y, pilots, seeds, first_slot, state, nullptr, ws,
                       stream, false);
  if (rc) return rc;
  rc = experts_equalize_impl(plan, n_streams, n_slots, y, tx, noise_var, seeds, first_slot,
                             state, h_mmse, h_ai, tel, ws, stream, true);
  if (rc) return rc;
  if (!g_hook.k3_on_tail) return set_err(ARCHES_E_STATE, "pipelined K3 was not placed on the tail");
  CUDA_TRY(cudaEventRecord(P->ev_k3, P->tail));
  rc = arches_kpm_scan(plan, n_streams, n_slots, tel, regime, tree, state, kpm, msg_log,
                       msg_count, msg_cap, reinterpret_cast<arches_stream_t>(P->tail));
  if (rc) return rc;
  CUDA_TRY(cudaEventRecord(P->ev_end, P->tail));
  P->tail_pending = true;
  return ARCHES_OK;
}

extern "C" int arches_switch_copy(const arches_plan* plan, int32_t n_units, const arches_kpm* kpm,
                                  const void* h_mmse, void* h_ai, arches_stream_t stream) {
  if (!plan || !kpm || !h_mmse || !h_ai || n_units < 1)
    return set_err(ARCHES_E_CONTRACT, "bad switch_copy args");
  const size_t per_unit = (size_t)plan->dev.A * plan->dev.D * plan->dev.N;  // complex values
  if (per_unit % 2) return set_err(ARCHES_E_CONTRACT, "unit size must be even");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const size_t f4 = per_unit / 2;
  const size_t blocks = std::min<size_t>((f4 * (size_t)n_units + 255) / 256,
                                         (size_t)plan->dev.num_sms * 16);
  k5_switch_copy<<<(unsigned)std::max<size_t>(blocks, 1), 256, 0, s>>>(kpm, reinterpret_cast<const float4*>(h_mmse),
                                      reinterpret_cast<float4*>(h_ai), f4, n_units);
  LAUNCH_CHECK();
  return ARCHES_OK;
}

extern "C" int arches_switch_copy_one(const int32_t* mode, const void* src, void* dst, size_t n,
                                      arches_stream_t stream) {
  if (!mode || !src || !dst) return set_err(ARCHES_E_CONTRACT, "bad switch_copy_one args");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const unsigned blocks = (unsigned)std::max<size_t>(1, std::min<size_t>((n + 255) / 256, 1184));
  k5_switch_copy_one<<<blocks, 256, 0, s>>>(mode, reinterpret_cast<const float2*>(src),
                                            reinterpret_cast<float2*>(dst), n);
  LAUNCH_CHECK();
  return ARCHES_OK;
}

// ------------------------------------------------------------ K6 / K7
extern "C" int arches_downstream(const arches_plan* plan, int32_t n_units, const arches_kpm* kpm,
                                 const void* h_mmse, const void* h_ai, const void* y,
                                 const double* noise_var, void* x_hat, float* llr,
                                 arches_stream_t stream) {
  if (!plan || !kpm || !h_mmse || !h_ai || !y || !noise_var || n_units < 1)
    return set_err(ARCHES_E_CONTRACT, "bad downstream args");
  if (!x_hat && !llr) return ARCHES_OK;
  dim3 grid((plan->dev.N + K6_THREADS - 1) / K6_THREADS, n_units);
  if (n_units > 65535) return set_err(ARCHES_E_CONTRACT, "downstream: at most 65535 units per call");
  k6_xhat_demap<<<grid, K6_THREADS, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      plan->dev, kpm, reinterpret_cast<const float2*>(h_mmse), reinterpret_cast<const float2*>(h_ai),
      reinterpret_cast<const float2*>(y), noise_var, reinterpret_cast<float2*>(x_hat), llr, n_units);
  LAUNCH_CHECK();
  return ARCHES_OK;
}

extern "C" int arches_perturb_mmse(const arches_plan* plan, int32_t n_streams, int32_t n_slots,
                                   int64_t first_slot, const double* rho, const uint64_t* seeds,
                                   const void* state, const void* y, const void* tx,
                                   const double* noise_var, void* h_mmse, arches_telemetry* tel,
                                   void* ws, arches_stream_t stream) {
  if (!plan || !rho || !seeds || !y || !tx || !noise_var || !h_mmse || !tel || !ws ||
      n_streams < 1 || n_slots < 1)
    return set_err(ARCHES_E_CONTRACT, "bad perturb_mmse args");
  if (first_slot < 0 && !state)
    return set_err(ARCHES_E_CONTRACT, "first_slot < 0 needs the stream state (slot source)");
  const int n_units = n_streams * n_slots;
  if (n_units > 65535) return set_err(ARCHES_E_CONTRACT, "perturb_mmse: at most 65535 units per call");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const WsLayout w = ws_layout(plan, n_units);
  CUDA_TRY(cudaMemsetAsync(ws_at<void>(ws, w.counters), 0, n_units * sizeof(unsigned int), s));
  static const uint64_t inject_key =
      arches_rng::blake2b64(reinterpret_cast<const uint8_t*>("inject"), 6);
  K7Args a;
  a.rho = rho;
  a.seeds = seeds;
  a.inject_key = inject_key;
  a.state = reinterpret_cast<const unsigned char*>(state);
  a.state_stride = state_stride_bytes(plan->dev.window_length, plan->dev.dapp_window);
  a.first_slot = first_slot;
  a.n_slots = n_slots;
  a.y = reinterpret_cast<const float2*>(y);
  a.tx = reinterpret_cast<const float2*>(tx);
  a.nv = noise_var;
  a.h_mmse = reinterpret_cast<float2*>(h_mmse);
  a.tel = tel;
  a.parts = ws_at<TilePartial>(ws, w.parts);
  a.counters = ws_at<unsigned int>(ws, w.counters);
  dim3 grid((plan->dev.N + K6_THREADS - 1) / K6_THREADS, n_units);
  k_perturb_mmse<<<grid, K6_THREADS, 0, s>>>(plan->dev, a);
  LAUNCH_CHECK();
  return ARCHES_OK;
}

// ------------------------------------------------------------ scene synthesis
static uint64_t purpose_key64(const char* p) {
  return arches_rng::blake2b64(reinterpret_cast<const uint8_t*>(p), (int)strlen(p));
}

extern "C" size_t arches_scene_state_bytes(const arches_plan* plan, int32_t n_streams) {
  return plan && n_streams > 0 ? (size_t)n_streams * scene_state_stride(plan->dev.A) : 0;
}

extern "C" size_t arches_scene_workspace_bytes(const arches_plan* plan, int32_t n_units) {
  return plan && n_units > 0 ? (size_t)n_units * 2 * plan->dev.A * SCENE_TAPS * sizeof(double2) : 0;
}

extern "C" int arches_scene_pilots(const arches_plan* plan, int32_t n_streams, const uint64_t* seeds,
                                   void* pilots, arches_stream_t stream) {
  if (!plan || !seeds || !pilots || n_streams < 1) return set_err(ARCHES_E_CONTRACT, "bad scene_pilots args");
  const int MD = plan->dev.M * plan->dev.D;
  dim3 grid((MD + 127) / 128, n_streams);
  k_scene_pilots<<<grid, 128, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      plan->dev, seeds, purpose_key64("pilot"), reinterpret_cast<float2*>(pilots), n_streams);
  LAUNCH_CHECK();
  return ARCHES_OK;
}

extern "C" int arches_synthesize(const arches_plan* plan, int32_t n_streams, int32_t n_slots,
                                 const uint64_t* seeds, const arches_scene_regime* regimes,
                                 const uint8_t* prb_mask, const double* sqrt_pdp,
                                 int32_t excess_delay, const int8_t* regime, const double* shadow_z,
                                 const void* pilots, void* scene_state, void* scene_ws, void* y,
                                 void* tx, double* noise_var, arches_stream_t stream) {
  if (!plan || !seeds || !regimes || !prb_mask || !sqrt_pdp || !regime || !shadow_z || !pilots ||
      !scene_state || !scene_ws || !y || !tx || !noise_var || n_streams < 1 || n_slots < 1)
    return set_err(ARCHES_E_CONTRACT, "bad synthesize args");
  const PlanDev& d = plan->dev;
  if (d.A * SCENE_TAPS > 1024) return set_err(ARCHES_E_CONFIG, "synthesize: n_ant > 128");
  const int n_units = n_streams * n_slots;
  if (n_units > 65535) return set_err(ARCHES_E_CONTRACT, "synthesize: at most 65535 units per call");
  if (excess_delay < 0 || excess_delay + SCENE_TAPS > d.M)
    return set_err(ARCHES_E_CONFIG, "interference_excess_delay does not fit the comb span");
  SceneArgs a;
  memset(&a, 0, sizeof(a));
  a.seeds = seeds;
  for (int r = 0; r < 2; ++r) {
    a.reg[r].noise_var = regimes[r].noise_var;
    a.reg[r].interference_var = regimes[r].interference_var;
    a.reg[r].temporal_correlation = regimes[r].temporal_correlation;
    a.reg[r].shadow_sigma_db = regimes[r].shadow_sigma_db;
    a.reg[r].shadow_correlation = regimes[r].shadow_correlation;
  }
  a.prb_mask = prb_mask;
  for (int l = 0; l < SCENE_TAPS; ++l) a.sqrt_p[l] = sqrt_pdp[l];
  a.excess_delay = excess_delay;
  a.shadowed = 1;
  a.regime = regime;
  a.shadow_z = shadow_z;
  a.state = reinterpret_cast<unsigned char*>(scene_state);
  a.taps_u = reinterpret_cast<double2*>(scene_ws);
  a.y = reinterpret_cast<float2*>(y);
  a.tx = reinterpret_cast<float2*>(tx);
  a.noise_var = noise_var;
  a.n_slots = n_slots;
  a.key_channel = purpose_key64("channel");
  a.key_interferer = purpose_key64("interferer");
  a.key_awgn = purpose_key64("awgn");
  a.key_data = purpose_key64("data");
  a.key_idata = purpose_key64("interferer-data");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int th = ((d.A * SCENE_TAPS + 31) / 32) * 32;
  k_scene_taps<<<n_streams, th, 0, s>>>(d, a);
  LAUNCH_CHECK();
  dim3 grid((d.N + 127) / 128, n_units);
  k_scene_grid<<<grid, 128, 0, s>>>(d, a, reinterpret_cast<const float2*>(pilots), n_units);
  LAUNCH_CHECK();
  return ARCHES_OK;
}

// ------------------------------------------------------------ tree training
extern "C" int arches_tree_eval_splits(const double* xT, const int32_t* order, const uint8_t* y,
                                       int32_t n, int32_t n_features, const int32_t* root_feature,
                                       const double* root_threshold, int32_t n_roots,
                                       arches_split_eval* out, arches_stream_t stream) {
  if (!xT || !order || !y || !root_feature || !root_threshold || !out || n < 1 ||
      n_features < 1 || n_roots < 1)
    return set_err(ARCHES_E_CONTRACT, "bad tree_eval_splits args");
  const unsigned blocks = (unsigned)((n_roots + TT_WARPS - 1) / TT_WARPS);
  k_tree_eval_splits<<<blocks, 32 * TT_WARPS, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      xT, order, y, n, n_features, root_feature, root_threshold, n_roots, out);
  LAUNCH_CHECK();
  return ARCHES_OK;
}

// ------------------------------------------------------------ packed QPSK tx
extern "C" size_t arches_tx_bits_bytes(const arches_plan* plan, int32_t n_units) {
  if (!plan || n_units < 1) return 0;
  return (size_t)n_units * plan->dev.n_tiles * plan->dev.T * ARCHES_TXB_ROW;
}

static unsigned qpsk_blocks(const arches_plan* plan, size_t n_bytes) {
  return (unsigned)std::max<size_t>(1, std::min<size_t>((n_bytes + 255) / 256,
                                                        (size_t)plan->dev.num_sms * 8));
}

extern "C" int arches_pack_qpsk(const arches_plan* plan, int32_t n_units, const void* tx,
                                void* tx_bits, int32_t* bad, arches_stream_t stream) {
  if (!plan || !tx || !tx_bits || !bad || n_units < 1)
    return set_err(ARCHES_E_CONTRACT, "bad pack_qpsk args");
  const size_t n_bytes = arches_tx_bits_bytes(plan, n_units);
  k_pack_qpsk<<<qpsk_blocks(plan, n_bytes), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      plan->dev, reinterpret_cast<const float2*>(tx), reinterpret_cast<unsigned char*>(tx_bits),
      bad, n_bytes);
  LAUNCH_CHECK();
  return ARCHES_OK;
}

extern "C" int arches_unpack_qpsk(const arches_plan* plan, int32_t n_units, const void* tx_bits,
                                  void* tx, arches_stream_t stream) {
  if (!plan || !tx || !tx_bits || n_units < 1)
    return set_err(ARCHES_E_CONTRACT, "bad unpack_qpsk args");
  const size_t n_bytes = arches_tx_bits_bytes(plan, n_units);
  if (n_bytes >= (1ull << 32)) return set_err(ARCHES_E_CONTRACT, "unpack_qpsk: batch too large");
  k_unpack_qpsk<<<qpsk_blocks(plan, n_bytes), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      plan->dev, reinterpret_cast<const unsigned char*>(tx_bits), reinterpret_cast<float2*>(tx),
      n_bytes);
  LAUNCH_CHECK();
  return ARCHES_OK;
}

// ------------------------------------------------------------ compat forms
extern "C" int arches_ls_materialize(const arches_plan* plan, int32_t n_units, const void* y,
                                     const void* pilots, void* ls, arches_stream_t stream) {
  if (!plan || !y || !pilots || !ls || n_units < 1) return set_err(ARCHES_E_CONTRACT, "bad ls args");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  GridCombSrc src{reinterpret_cast<const float2*>(y), reinterpret_cast<const float2*>(pilots), 1};
  k_ls_materialize<<<592, 256, 0, s>>>(plan->dev, src, reinterpret_cast<float2*>(ls), n_units);
  LAUNCH_CHECK();
  return ARCHES_OK;
}

extern "C" int arches_expert_from_ls(const arches_plan* plan, int32_t n_units, int32_t which,
                                     const void* ls, const double* noise_var_in, double* sigma2_hat,
                                     void* out, void* ws, arches_stream_t stream) {
  const bool c128 = (which & ARCHES_EXPERT_OUT_C128) != 0;
  which &= ~ARCHES_EXPERT_OUT_C128;
  if (!plan || !ls || !ws || n_units < 1 || which < 0 || which > 2)
    return set_err(ARCHES_E_CONTRACT, "bad expert_from_ls args");
  if ((which == 1 || which == 2) && !out) return set_err(ARCHES_E_CONTRACT, "missing output");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const WsLayout w = ws_layout(plan, n_units);
  const float2* l = reinterpret_cast<const float2*>(ls);
  int rc;
  CUDA_TRY(cudaMemsetAsync(ws_at<void>(ws, w.k1counters), 0, n_units * sizeof(unsigned int), s));
  if (which == 2) {
    LsFullSrc src{l};
    K1Out o{nullptr, nullptr, ws_at<float2>(ws, w.coef), ws_at<double>(ws, w.k1parts),
            ws_at<unsigned int>(ws, w.k1counters), K1_AI, nullptr, nullptr, nullptr, 0, 0, 1};
    rc = launch_k1(plan, n_units, src, o, plan->dev.N, plan->k1_full_chunk, plan->k1_full_smem, s);
  } else {
    LsCombSrc src{l};
    K1Out o{sigma2_hat ? sigma2_hat : ws_at<double>(ws, w.sigma2), noise_var_in,
            which == 1 ? ws_at<float2>(ws, w.coef) : nullptr, ws_at<double>(ws, w.k1parts),
            ws_at<unsigned int>(ws, w.k1counters), which == 1 ? (K1_NOISE | K1_MMSE) : K1_NOISE,
            nullptr, nullptr, nullptr, 0, 0, 1};
    rc = launch_k1(plan, n_units, src, o, plan->dev.M, plan->k1_chunk, plan->k1_smem, s);
  }
  if (rc || which == 0) return rc;
  dim3 grid((plan->dev.N + 127) / 128, n_units);
  if (c128)
    k_synth_one_f64<<<grid, 128, 0, s>>>(plan->dev, ws_at<float2>(ws, w.coef), which,
                                         reinterpret_cast<double2*>(out));
  else
    k_synth_one<<<grid, 128, 0, s>>>(plan->dev, ws_at<float2>(ws, w.coef), which,
                                     reinterpret_cast<float2*>(out));
  LAUNCH_CHECK();
  return ARCHES_OK;
}

extern "C" int arches_equalize(const arches_plan* plan, int32_t n_units, const void* y,
                               const void* est, const void* tx, const double* noise_var,
                               double* sinr_db, double* abs_mean, double* rsrp, void* x_hat,
                               void* ws, arches_stream_t stream) {
  if (!plan || !y || !est || !tx || !noise_var || !ws || n_units < 1)
    return set_err(ARCHES_E_CONTRACT, "bad equalize args");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const WsLayout w = ws_layout(plan, n_units);
  CUDA_TRY(cudaMemsetAsync(ws_at<void>(ws, w.counters), 0, n_units * sizeof(unsigned int), s));
  K2Args a;
  memset(&a, 0, sizeof(a));
  a.y = reinterpret_cast<const float2*>(y);
  a.tx = reinterpret_cast<const float2*>(tx);
  a.est = reinterpret_cast<const float2*>(est);
  a.nv = noise_var;
  a.x_hat = reinterpret_cast<float2*>(x_hat);
  a.parts = ws_at<TilePartial>(ws, w.parts);
  a.counters = ws_at<unsigned int>(ws, w.counters);
  a.sinr_out = sinr_db;
  a.abs_out = abs_mean;
  a.rsrp_out = rsrp;
  a.n_slots = 1;
  return launch_k2<1>(plan, n_units, a, s);
}

extern "C" int arches_window_features(const double* rows, int32_t n_rows, double* out,
                                      arches_stream_t stream) {
  if (!rows || !out) return set_err(ARCHES_E_CONTRACT, "bad window_features args");
  if (n_rows < 1) return set_err(ARCHES_E_CONTRACT, "empty KPM window");
  k_window_features<<<1, 32, 0, reinterpret_cast<cudaStream_t>(stream)>>>(rows, n_rows, out);
  LAUNCH_CHECK();
  return ARCHES_OK;
}

extern "C" int arches_tree_predict(const arches_tree* tree, const double* x, int32_t n,
                                   int32_t n_features, int32_t* labels, arches_stream_t stream) {
  if (!tree || !x || !labels || n < 1) return set_err(ARCHES_E_CONTRACT, "bad predict args");
  k_tree_predict<<<(n + 127) / 128, 128, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      tree, x, n, n_features, labels);
  LAUNCH_CHECK();
  return ARCHES_OK;
}

// ------------------------------------------------------------ host helpers
extern "C" const char* arches_last_error(void) { return g_err; }
extern "C" const char* arches_version(void) { return ARCHES_VERSION; }

extern "C" double arches_host_crc_uniform(uint64_t seed, uint64_t purpose_key, uint64_t slot) {
  return arches_rng::stream_first_uniform(seed, purpose_key, slot);
}

extern "C" double arches_host_lcid4_jitter(uint64_t slot) { return arches_rng::lcid4_jitter(slot); }

extern "C" uint64_t arches_host_blake2b64(const void* data, size_t len) {
  if (len > 128) return 0;
  return arches_rng::blake2b64(reinterpret_cast<const uint8_t*>(data), (int)len);
}

extern "C" int32_t arches_device_available(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n > 0 ? 1 : 0;
}

#ifdef K1T_TRACE
extern "C" int arches_k1t_trace(void* host) {
  return cudaMemcpyFromSymbol(host, g_k1t_trace, sizeof(g_k1t_trace)) == cudaSuccess ? 0 : 1;
}
extern "C" int arches_k1t_span(void* host) {
  return cudaMemcpyFromSymbol(host, g_k1t_span, sizeof(g_k1t_span)) == cudaSuccess ? 0 : 1;
}
#endif
