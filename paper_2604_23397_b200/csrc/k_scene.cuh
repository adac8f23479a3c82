// Device-side slot synthesis (input generation for the hot path):
// restates rng.py:24-55 and radio_scene.py:140-306 as the reference's Pipeline
// drives them (phy_pipeline.py:430-433,459; `CellScene` in scene.py is the host
// form the tests pin against the reference).
//
//   K-scene-taps (one CTA per stream, thread = (antenna, tap), slots in order):
//     AR(1) TDL taps  taps = phi taps + sqrt(1 - phi^2) (CN(0,1) * sqrt(p))
//     (`ChannelProcess.step_taps`, radio_scene.py:170-192) for the serving
//     channel (purpose "channel", log-normal shadow 10^(s/20), AR(1) in dB) and
//     the interferer (purpose "interferer", unshadowed);
//   K-scene-grid (thread = subcarrier, all antennas x symbols of one unit):
//     H = FFT_N of the 8 taps (a direct 8-term DFT), interferer H_i with the
//     excess-delay phase, QPSK data grids (Lemire bits of the Philox uint32
//     stream: numpy Generator.integers(0, 2)) with the pilots on the DMRS comb,
//     Y = H X + sqrt(nv) W + sqrt(iv) H_i X_i on the interfered PRBs, W =
//     complex_normal(stream(seed, "awgn", slot)) -- every stream keyed and
//     indexed as numpy does, so every random bit is the reference's; the fp64
//     transcendental (log1p, sincos, pow) and DFT rounding differs from glibc /
//     pocketfft by ulps (tests state the tolerance).
// The shadow's standard normal (numpy's 256-box ziggurat, one draw per slot
// per cell) is supplied by the host.
#pragma once
#include "common.cuh"
#include "k_synth_eq.cuh"
#include "rng.cuh"

#define SCENE_TAPS 8

// one regime's scenario (ScenarioConfig, radio_scene.py:66-120)
struct SceneRegime {
  double noise_var;             // scen.noise_var(n_ant)
  double interference_var;      // scen.interference_var() (0: none)
  double temporal_correlation;  // phi
  double shadow_sigma_db, shadow_correlation;
};

struct SceneArgs {
  const uint64_t* seeds;        // [stream]
  SceneRegime reg[2];           // 0 = poor, 1 = good (regime codes of the engine)
  const uint8_t* prb_mask;      // [2][n_prb] interference PRB mask per regime
  double sqrt_p[SCENE_TAPS];    // sqrt(pdp_powers(delay_spread)) of the first regime
  int excess_delay;             // interferer excess delay (first regime)
  int shadowed;                 // 1: the serving channel carries the log-normal shadow
  const int8_t* regime;         // [u]
  const double* shadow_z;       // [u] stream(seed, "shadow", slot).standard_normal()
  unsigned char* state;         // [stream] SceneState + taps
  double2* taps_u;              // [u][2][A][8] per-unit channel / interferer taps (workspace)
  float2* y;                    // [u][A][T][N]
  float2* tx;                   // [u][T][N]
  double* noise_var;            // [u]
  int n_slots;
  uint64_t key_channel, key_interferer, key_awgn, key_data, key_idata, key_pilot;
};

struct SceneState {
  int64_t next_slot;
  double shadow_db;
};

__host__ __device__ inline size_t scene_state_stride(int A) {
  return (sizeof(SceneState) + 2 * (size_t)A * SCENE_TAPS * sizeof(double2) + 255) & ~(size_t)255;
}

// complex multiply without FMA contraction (numpy: (ac - bd) + (ad + bc) i)
__device__ __forceinline__ double2 zmul_rn(double2 a, double2 b) {
  return make_double2(__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)),
                      __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
}
__device__ __forceinline__ double2 zscale(double s, double2 a) {
  return make_double2(__dmul_rn(s, a.x), __dmul_rn(s, a.y));
}
__device__ __forceinline__ double2 zadd(double2 a, double2 b) {
  return make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y));
}

// qpsk() bit #i of stream(seed, purpose, slot): Generator.integers(0, 2) = the top
// bit of successive 32-bit draws (low half, then high half of each 64-bit output)
__device__ __forceinline__ int qpsk_bit(uint64_t seed, uint64_t key, uint64_t slot, uint64_t i) {
  const uint64_t j = i >> 1;
  uint64_t c[4] = {1ull + (j >> 2), slot, 0ull, 0ull};
  arches_rng::philox4x64_10(c, seed, key);
  const uint64_t w = c[j & 3];
  return (int)((i & 1) ? (w >> 63) : ((w >> 31) & 1ull));
}

// qpsk symbol (+-1 +-1j) / sqrt(2) from its two bits (rng.py:50-55: (2b - 1) / sqrt(2.0))
__device__ __forceinline__ double2 qpsk_sym(int b_re, int b_im) {
  const double s = 0.7071067811865475;  // 1 / np.sqrt(2.0)
  return make_double2(b_re ? s : -s, b_im ? s : -s);
}

// pilot_sequence (radio_scene.py:233-237): qpsk(stream(seed, "pilot"), (M, D))
__global__ void k_scene_pilots(const PlanDev P, const uint64_t* seeds, uint64_t key_pilot,
                               float2* pilots, int n_streams) {
  const int s = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;  // m * D + d
  const int MD = P.M * P.D;
  if (s >= n_streams || i >= MD) return;
  const int br = qpsk_bit(seeds[s], key_pilot, 0, (uint64_t)i);
  const int bi = qpsk_bit(seeds[s], key_pilot, 0, (uint64_t)MD + i);
  const double2 v = qpsk_sym(br, bi);
  pilots[(size_t)s * MD + i] = make_float2((float)v.x, (float)v.y);
}

// AR(1) tap recursion of every stream over the batch's slots
__global__ void k_scene_taps(const PlanDev P, const SceneArgs a) {
  const int stream = blockIdx.x;
  const int th = threadIdx.x;  // antenna * 8 + tap
  const int A = P.A;
  const bool act = th < A * SCENE_TAPS;
  unsigned char* st = a.state + (size_t)stream * scene_state_stride(A);
  SceneState* hs = reinterpret_cast<SceneState*>(st);
  double2* taps = reinterpret_cast<double2*>(st + sizeof(SceneState));   // [2][A][8]
  __shared__ double s_shadow;
  const uint64_t seed = a.seeds[stream];
  const int64_t n0 = hs->next_slot;
  double2 tc = act ? taps[th] : make_double2(0.0, 0.0);
  double2 ti = act ? taps[A * SCENE_TAPS + th] : make_double2(0.0, 0.0);
  if (th == 0) s_shadow = hs->shadow_db;
  __syncthreads();
  const uint64_t ncn = (uint64_t)A * SCENE_TAPS;
  for (int s = 0; s < a.n_slots; ++s) {
    const int u = stream * a.n_slots + s;
    const int64_t n = n0 + s;
    const SceneRegime& R = a.reg[a.regime[u] ? 1 : 0];
    const double phi = R.temporal_correlation;
    const double q = sqrt(__dsub_rn(1.0, __dmul_rn(phi, phi)));
    if (act) {
      const double sp = a.sqrt_p[th & (SCENE_TAPS - 1)];
      // _innovation: complex_normal(stream(seed, purpose, slot), (A, 1, 8)) * sqrt_p
      const double2 zc = zscale(sp, arches_rng::complex_normal_at(seed, a.key_channel, (uint64_t)n, ncn, th));
      const double2 zi = zscale(sp, arches_rng::complex_normal_at(seed, a.key_interferer, (uint64_t)n, ncn, th));
      tc = n == 0 ? zc : zadd(zscale(phi, tc), zscale(q, zc));
      ti = n == 0 ? zi : zadd(zscale(phi, ti), zscale(q, zi));
    }
    __syncthreads();
    if (th == 0 && a.shadowed && R.shadow_sigma_db != 0.0) {
      const double g = __dmul_rn(R.shadow_sigma_db, a.shadow_z[u]);
      const double ps = R.shadow_correlation;
      s_shadow = n == 0 ? g
                        : __dadd_rn(__dmul_rn(ps, s_shadow),
                                    __dmul_rn(sqrt(__dsub_rn(1.0, __dmul_rn(ps, ps))), g));
    }
    __syncthreads();
    if (act) {
      double2 out = tc;
      if (a.shadowed && R.shadow_sigma_db != 0.0) out = zscale(pow(10.0, s_shadow / 20.0), tc);
      a.taps_u[((size_t)u * 2 + 0) * A * SCENE_TAPS + th] = out;
      a.taps_u[((size_t)u * 2 + 1) * A * SCENE_TAPS + th] = ti;
    }
    __syncthreads();
  }
  if (act) {
    taps[th] = tc;
    taps[A * SCENE_TAPS + th] = ti;
  }
  if (th == 0) {
    hs->shadow_db = s_shadow;
    hs->next_slot = n0 + a.n_slots;
  }
}

// Y = H X + sqrt(nv) W + sqrt(iv) H_i X_i for one subcarrier of one unit
__global__ void __launch_bounds__(128) k_scene_grid(const PlanDev P, const SceneArgs a,
                                                     const float2* pilots, int n_units) {
  const int u = blockIdx.y;
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= n_units || k >= P.N) return;
  const int stream = u / a.n_slots;
  const int A = P.A, T = P.T, N = P.N, D = P.D;
  const uint64_t seed = a.seeds[stream];
  const SceneRegime& R = a.reg[a.regime[u] ? 1 : 0];
  // slot index of the unit: the taps kernel already advanced the state by n_slots
  const unsigned char* st = a.state + (size_t)stream * scene_state_stride(A);
  const int64_t n = reinterpret_cast<const SceneState*>(st)->next_slot - a.n_slots +
                    (u - stream * a.n_slots);
  const bool interf = R.interference_var > 0.0 && a.prb_mask[(a.regime[u] ? 1 : 0) * P.n_prb + k / 12];
  // transmit grid column k (data QPSK, pilots on the comb of the DMRS symbols)
  double2 x[ARCHES_MAX_SYM], xi[ARCHES_MAX_SYM];
  const uint64_t NT = (uint64_t)N * T;
  for (int t = 0; t < T; ++t) {
    const int dj = P.is_dmrs[t];
    if (dj >= 0 && (k & 1) == 0) {
      const float2 pv = pilots[((size_t)stream * P.M + (k >> 1)) * D + dj];
      x[t] = xi[t] = make_double2((double)pv.x, (double)pv.y);
    } else {
      const uint64_t i = (uint64_t)k * T + t;
      x[t] = qpsk_sym(qpsk_bit(seed, a.key_data, (uint64_t)n, i),
                      qpsk_bit(seed, a.key_data, (uint64_t)n, NT + i));
      xi[t] = interf ? qpsk_sym(qpsk_bit(seed, a.key_idata, (uint64_t)n, i),
                                qpsk_bit(seed, a.key_idata, (uint64_t)n, NT + i))
                     : make_double2(0.0, 0.0);
    }
    a.tx[((size_t)u * T + t) * N + k] = make_float2((float)x[t].x, (float)x[t].y);
  }
  const double snv = R.noise_var > 0.0 ? sqrt(R.noise_var) : 0.0;
  const double siv = interf ? sqrt(R.interference_var) : 0.0;
  // interferer excess-delay phase exp(-2j pi e k / N): numpy evaluates
  // ((-2j * pi) * e) * k / N, then cexp of (+-0, y)
  double2 ph = make_double2(1.0, 0.0);
  if (interf && a.excess_delay) {
    const double y = __ddiv_rn(__dmul_rn(__dmul_rn(-6.283185307179586, (double)a.excess_delay), (double)k),
                               (double)N);
    double sn, cs;
    sincos(y, &sn, &cs);
    ph = make_double2(cs, sn);
  }
  const uint64_t nw = (uint64_t)A * N * T;
  const double2* tu = a.taps_u + (size_t)u * 2 * A * SCENE_TAPS;
  for (int ant = 0; ant < A; ++ant) {
    // H[k] = sum_l taps[l] e^{-2 pi i l k / N} (np.fft.fft(taps, n=N)[k])
    double2 h = make_double2(0.0, 0.0), hi = make_double2(0.0, 0.0);
    for (int l = 0; l < SCENE_TAPS; ++l) {
      double sn, cs;
      sincospi(__ddiv_rn(2.0 * (double)(((long long)l * k) % N), (double)N), &sn, &cs);
      const double2 w = make_double2(cs, -sn);
      h = zadd(h, zmul_rn(tu[ant * SCENE_TAPS + l], w));
      if (interf) hi = zadd(hi, zmul_rn(tu[(A + ant) * SCENE_TAPS + l], w));
    }
    if (interf && a.excess_delay) hi = zmul_rn(hi, ph);
    const double2 hs = interf ? zscale(siv, hi) : make_double2(0.0, 0.0);
    for (int t = 0; t < T; ++t) {
      double2 yv = zmul_rn(h, x[t]);
      if (snv > 0.0) {
        const uint64_t e = ((uint64_t)ant * N + k) * T + t;
        yv = zadd(yv, zscale(snv, arches_rng::complex_normal_at(seed, a.key_awgn, (uint64_t)n, nw, e)));
      }
      if (interf) yv = zadd(yv, zmul_rn(hs, xi[t]));
      a.y[(((size_t)u * A + ant) * T + t) * N + k] = make_float2((float)yv.x, (float)yv.y);
    }
  }
  if (k == 0) a.noise_var[u] = R.noise_var;
}
