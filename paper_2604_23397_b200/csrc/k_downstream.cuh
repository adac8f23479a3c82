// Downstream of the zero-gap switch, after K4 has fixed each slot's mode:
//
// K6 `k6_xhat_demap` -- the equalised-symbol data path: x_hat of the SELECTED
//   expert (the buffer switch_select leaves downstream, phy_pipeline.py:81-91,
//   451-452) exactly as equalize() forms it (phy_pipeline.py:258-266: time
//   interpolation, MRC num / (sum |h|^2 + noise_var), every RE), plus a
//   max-log demapper for the slot's scheduled modulation (kpm.qam_order;
//   Gray QPSK / 16QAM / 64QAM of TS 38.211 s5.1.3-5.1.5) on the data REs.
//
// K7 `k_perturb_mmse` -- Eq. 3 perturbation (perturbation_lab.py:92-98, the
//   Pipeline.perturb hook at phy_pipeline.py:444-445): the MMSE output gets
//   rho * mean|H_mmse| * CN(0,1) with CN from stream(seed, "inject", slot) over
//   the reference's (A, 1, N, D) element order, is written back (the MMSE
//   buffer holds the perturbed values), re-equalised, and the MMSE candidate
//   of the unit's telemetry (rsrp, SINR, link adaptation, TB, CRC, MAC) is
//   re-derived; abs_mean stays the pre-injection mean (the hook's
//   est_abs_mean).  rho == 0 leaves everything bit-identical (no-op).
#pragma once
#include "common.cuh"
#include "k_synth_eq.cuh"
#include "rng.cuh"

#define K6_THREADS 128

// one RE of one expert estimate h[a][d] (global, [A][D][N] of the unit):
// equalize()'s x_hat, and den = sum_a |h_interp|^2
__device__ __forceinline__ float2 xhat_re(const PlanDev& P, const float2* h, const float2* y,
                                          int k, int t, float nv, float& den_out) {
  float2 num = make_float2(0.f, 0.f);
  float den = 0.f;
  for (int a = 0; a < P.A; ++a) {
    float2 hn = make_float2(0.f, 0.f);
    for (int d = 0; d < P.D; ++d) {
      const float w = P.tw[t][d];
      const float2 hv = h[((size_t)a * P.D + d) * P.N + k];
      hn.x = fmaf(w, hv.x, hn.x);
      hn.y = fmaf(w, hv.y, hn.y);
    }
    const float2 yv = y[((size_t)a * P.T + t) * P.N + k];
    num.x = fmaf(hn.x, yv.x, fmaf(hn.y, yv.y, num.x));
    num.y = fmaf(hn.x, yv.y, fmaf(-hn.y, yv.x, num.y));
    den = fmaf(hn.x, hn.x, fmaf(hn.y, hn.y, den));
  }
  den_out = den;
  const float inv = 1.0f / (den + nv);
  return make_float2(num.x * inv, num.y * inv);
}

// max-log LLRs (log P(b=0) / P(b=1)) of one PAM dimension of a Gray QAM:
// levels of bits (b_i, b_{i+2}, b_{i+4}) per TS 38.211 s5.1; z = unbiased
// component, s2 = its noise variance.  qm = 2 (QPSK), 4, 6.
__device__ __forceinline__ void pam_llr(float z, float s2, int qm, float* out /*stride 2*/) {
  const int nb = qm >> 1;  // bits per dimension
  const float scale = qm == 2 ? 0.70710678118654752f : qm == 4 ? 0.31622776601683794f
                                                               : 0.15430334996209191f;
  float best0[3] = {3.4e38f, 3.4e38f, 3.4e38f}, best1[3] = {3.4e38f, 3.4e38f, 3.4e38f};
  for (int lab = 0; lab < (1 << nb); ++lab) {  // bits b_i = lab bit 0, b_{i+2} = bit 1, ...
    const int c0 = 1 - 2 * (lab & 1), c1 = 1 - 2 * ((lab >> 1) & 1), c2 = 1 - 2 * ((lab >> 2) & 1);
    const float lev = (float)(nb == 1 ? c0 : nb == 2 ? c0 * (2 - c1) : c0 * (4 - c1 * (2 - c2))) * scale;
    const float dd = (z - lev) * (z - lev);
    for (int i = 0; i < nb; ++i) {
      if ((lab >> i) & 1) best1[i] = fminf(best1[i], dd);
      else best0[i] = fminf(best0[i], dd);
    }
  }
  for (int i = 0; i < nb; ++i) out[2 * i] = (best1[i] - best0[i]) / s2;
}

__global__ void __launch_bounds__(K6_THREADS)
    k6_xhat_demap(const PlanDev P, const arches_kpm* kpm, const float2* h_mmse, const float2* h_ai,
                  const float2* y, const double* noise_var, float2* x_hat, float* llr, int n_units) {
  const int u = blockIdx.y;
  const int k = blockIdx.x * K6_THREADS + threadIdx.x;
  if (u >= n_units || k >= P.N) return;
  const int mode = kpm[u].mode;
  const int qm = kpm[u].qam_order;
  const size_t hoff = (size_t)u * P.A * P.D * P.N;
  const float2* h = (mode == 1 ? h_mmse : h_ai) + hoff;  // the switch predicate
  const float2* yu = y + (size_t)u * P.A * P.T * P.N;
  const float nv = (float)noise_var[u];
  for (int t = 0; t < P.T; ++t) {
    float den;
    const float2 xh = xhat_re(P, h, yu, k, t, nv, den);
    const size_t re = ((size_t)u * P.T + t) * P.N + k;
    if (x_hat) x_hat[re] = xh;
    if (llr) {
      float* o = llr + re * ARCHES_LLR_STRIDE;
      for (int i = 0; i < ARCHES_LLR_STRIDE; ++i) o[i] = 0.f;
      const bool pilot = (k & 1) == 0 && P.is_dmrs[t] >= 0;  // data_re_mask (phy_pipeline.py:245-250)
      if (!pilot && (qm == 2 || qm == 4 || qm == 6) && den > 0.f) {
        // x_hat = beta x + e, beta = den / (den + nv): unbiased z = x_hat / beta, var nv / den
        const float beta = den / (den + nv);
        const float s2 = nv > 0.f ? nv / den : 1e-30f;
        pam_llr(xh.x / beta, s2, qm, o);      // b0, b2, b4 from Re
        pam_llr(xh.y / beta, s2, qm, o + 1);  // b1, b3, b5 from Im
      }
    }
  }
}

// ---- K7: Eq. 3 injection into the MMSE output + re-equalisation
struct K7Args {
  const double* rho;        // [stream]
  const uint64_t* seeds;    // [stream] scenario seeds (stream(seed, "inject", slot))
  uint64_t inject_key;      // blake2b64("inject")
  const unsigned char* state;
  size_t state_stride;
  long long first_slot;     // < 0: the stream's device next_slot
  int n_slots;
  const float2* y;
  const float2* tx;
  const double* nv;
  float2* h_mmse;
  arches_telemetry* tel;
  TilePartial* parts;       // [u][n_tiles]
  unsigned int* counters;   // [u]
};

__global__ void __launch_bounds__(K6_THREADS) k_perturb_mmse(const PlanDev P, const K7Args a) {
  __shared__ double s_scr[11 * (K6_THREADS / 32)];
  __shared__ int s_flag;
  const int u = blockIdx.y, tile = blockIdx.x;
  const int stream = u / a.n_slots;
  const double rho = a.rho[stream];
  if (rho == 0.0) return;  // _inject_values: rho = 0 is the identity (uniform per CTA)
  const int k = tile * K6_THREADS + threadIdx.x;
  const bool valid = k < P.N;
  const long long base = a.first_slot >= 0
      ? a.first_slot
      : (long long)*reinterpret_cast<const int64_t*>(a.state + (size_t)stream * a.state_stride);
  const long long slot = base + (u - stream * a.n_slots);
  const double m = a.tel[u].abs_mean[1];  // mean |H_mmse| before the injection (K3)
  const double g = rho * m;
  const uint64_t seed = a.seeds[stream];
  const uint64_t n_el = (uint64_t)P.A * P.N * P.D;
  float2* h = a.h_mmse + (size_t)u * P.A * P.D * P.N;
  double v[11];
  for (int i = 0; i < 11; ++i) v[i] = 0.0;
  if (valid) {
    float sp = 0.f;
    for (int aa = 0; aa < P.A; ++aa)
      for (int d = 0; d < P.D; ++d) {
        float2* hp = &h[((size_t)aa * P.D + d) * P.N + k];
        const float2 h0 = *hp;
        // reference element order of (A, 1, N, D): e = (a * N + k) * D + d
        const uint64_t e = ((uint64_t)aa * P.N + k) * P.D + d;
        const double2 z = arches_rng::complex_normal_at(seed, a.inject_key, (uint64_t)slot, n_el, e);
        const float2 h1 = make_float2((float)((double)h0.x + g * z.x), (float)((double)h0.y + g * z.y));
        *hp = h1;
        sp = fmaf(h1.x, h1.x, fmaf(h1.y, h1.y, sp));
      }
    v[3] = sp;  // pow_sum of the MMSE candidate
    const float2* yu = a.y + (size_t)u * P.A * P.T * P.N;
    const float nv = (float)a.nv[u];
    const bool even = (k & 1) == 0;
    for (int t = 0; t < P.T; ++t) {
      float den;
      const float2 xh = xhat_re(P, h, yu, k, t, nv, den);
      if (even && P.is_dmrs[t] >= 0) continue;  // pilot RE
      const float2 x = P.tx_packed
                           ? tx_packed_at(P, reinterpret_cast<const unsigned char*>(a.tx), u, t, k)
                           : a.tx[((size_t)u * P.T + t) * P.N + k];
      const double xr = x.x, xi = x.y, hr = xh.x, hi = xh.y;
      v[4] += xr * xr + xi * xi;
      v[6] += xr * hr + xi * hi;
      v[8] += xr * hi - xi * hr;
      v[10] += hr * hr + hi * hi;
    }
  }
  TilePartial* mine = a.parts + (size_t)u * gridDim.x + tile;
  reduce_tile(v, s_scr, mine);
  if (last_block_arrive(a.counters + u, gridDim.x, &s_flag) && threadIdx.x == 0) {
    double acc[11];
    for (int i = 0; i < 11; ++i) acc[i] = 0.0;
    for (int t = 0; t < (int)gridDim.x; ++t) {
      const double* p = reinterpret_cast<const double*>(&a.parts[(size_t)u * gridDim.x + t]);
      for (int i = 0; i < 11; ++i) acc[i] += p[i];
    }
    const double cnt = (double)P.A * P.D * P.N;
    arches_telemetry& tl = a.tel[u];
    tl.rsrp[1] = acc[3] / cnt;
    tl.sinr_db[1] = sinr_from_sums(acc[4], acc[6], acc[8], acc[10], P.sinr_cap_db);
    const double u_crc = arches_rng::stream_first_uniform(seed, P.crc_key, (uint64_t)slot);
    kpm_candidate(P, tl.sinr_db[1], u_crc, lcid4_frac(P, slot), tl.mcs[1], tl.tb_bytes[1],
                  tl.num_cb[1], tl.crc[1], tl.mac_rx[1], tl.lcid4_rx[1]);
  }
}
