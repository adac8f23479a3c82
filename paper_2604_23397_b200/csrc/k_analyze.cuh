// K1 -- LS front end + delay-domain analysis (one CTA per unit).
//
// Replaces ls_estimate (expert_bank.py:96-116), estimate_noise_var (:199-214)
// and the noise-dependent half of mmse_estimate/_wiener_matrix (:139-177) and
// denoiser_estimate (:182-196).
//
// Exact factorisation used (derived in DESIGN.md s3):
//   bins   B[ad][l]  = sum_m h[ad][m] e^{+2 pi i l m / M}          (l < L)
//   sigma2 = (sum |h|^2 - sum_{ad, l<guard} |B|^2 / M) / (AD (M - guard))   (Parseval)
//   MMSE   out[k] = sum_{l<8} c_l e^{-2 pi i l k / N},  c = P (Gamma P + s I)^-1 B
//          (Gamma = M I for one block with M >= 8 -> c_l = p_l B_l / (M p_l + s))
//   AI     out[k] = sum_{l<T} c_l e^{-2 pi i l k / N},  c_l = (1 + e^{2 pi i l/N}) B_l / N
// The analysis is a (AD x npts) x (npts x L) complex contraction; each thread
// owns a 4 (ad) x 5 (l) register tile over a K-slice of points, twiddles come
// from an exactly rounded table plus a <= 4-step recurrence.
#pragma once
#include "common.cuh"
#include "rng.cuh"

// --- point sources -------------------------------------------------------
// pipeline: comb REs of the received grid divided by the pilots
struct GridCombSrc {
  const float2* y;    // [u][A][T][N]
  const float2* pil;  // [stream][M][D]
  int n_slots;
  static constexpr bool kComb = true;
  static constexpr bool kGrid = true;
  __device__ __forceinline__ float2 load(const PlanDev& P, int u, int ad, int m) const {
    const int a = ad / P.D, d = ad - a * P.D;
    const float2 v = __ldg(&y[(((size_t)u * P.A + a) * P.T + P.dsym[d]) * P.N + 2 * m]);
    const float2 p = __ldg(&pil[((size_t)(u / n_slots) * P.M + m) * P.D + d]);
    const float inv = 1.0f / (p.x * p.x + p.y * p.y);
    const float2 q = cmulc(p, v);  // conj(p) * v
    return make_float2(q.x * inv, q.y * inv);
  }
};
// compat: comb positions of a materialised LS grid ls[u][A][D][N]
struct LsCombSrc {
  const float2* ls;
  static constexpr bool kComb = true;
  static constexpr bool kGrid = false;
  __device__ __forceinline__ float2 load(const PlanDev& P, int u, int ad, int m) const {
    return __ldg(&ls[((size_t)u * P.A * P.D + ad) * P.N + 2 * m]);
  }
};
// compat: every subcarrier of an LS grid (general denoiser input)
struct LsFullSrc {
  const float2* ls;
  static constexpr bool kComb = false;
  static constexpr bool kGrid = false;
  __device__ __forceinline__ float2 load(const PlanDev& P, int u, int ad, int k) const {
    return __ldg(&ls[((size_t)u * P.A * P.D + ad) * P.N + k]);
  }
};

// what K1 produces
enum { K1_NOISE = 1, K1_MMSE = 2, K1_AI = 4 };

struct K1Out {
  double* sigma2;           // [u] (may be null)
  const double* nv_in;      // [u] override (>= 0) or null
  float2* coef;             // [u][coef_floats2]
  double* parts;            // [u][n_parts][2*AD*L + 2] partial bins + energy (fp64)
  unsigned int* counters;   // [u] arrival counters (self re-arming)
  int what;
  // per-unit RNG side products for K2 (Philox CRC uniform, LCID4 split)
  double* rng;              // [u][2] or null
  const uint64_t* seeds;    // [stream]
  const unsigned char* state;
  size_t state_stride;
  long long first_slot;     // < 0: stream next_slot from state
  int n_slots;
};

__device__ inline void solve8_gram(const PlanDev& P, double s, double2* K /*[8][8]*/) {
  // K = Pd (Gamma Pd + s I)^-1, Gauss-Jordan with partial pivoting on
  // X^T: rows of K are solutions of (Gamma Pd + s I)^T z = Pd_row.
  double2 a[8][16];
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 8; ++j) {
      double2 g = P.gram[j * 8 + i];
      a[i][j] = make_double2(g.x * P.pdp[i] + (i == j ? s : 0.0), g.y * P.pdp[i]);
      a[i][8 + j] = make_double2(i == j ? P.pdp[i] : 0.0, 0.0);
    }
  for (int c = 0; c < 8; ++c) {
    int piv = c;
    double best = a[c][c].x * a[c][c].x + a[c][c].y * a[c][c].y;
    for (int r = c + 1; r < 8; ++r) {
      double v = a[r][c].x * a[r][c].x + a[r][c].y * a[r][c].y;
      if (v > best) best = v, piv = r;
    }
    if (piv != c)
      for (int j = 0; j < 16; ++j) {
        double2 t = a[c][j];
        a[c][j] = a[piv][j];
        a[piv][j] = t;
      }
    const double den = a[c][c].x * a[c][c].x + a[c][c].y * a[c][c].y;
    const double2 inv = make_double2(a[c][c].x / den, -a[c][c].y / den);
    for (int j = 0; j < 16; ++j) a[c][j] = zmul(a[c][j], inv);
    for (int r = 0; r < 8; ++r) {
      if (r == c) continue;
      const double2 f = a[r][c];
      for (int j = 0; j < 16; ++j) {
        const double2 t = zmul(f, a[c][j]);
        a[r][j].x -= t.x;
        a[r][j].y -= t.y;
      }
    }
  }
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 8; ++j) K[j * 8 + i] = a[i][8 + j];
}

// One CTA per (part, unit): part p covers points [p*chunk, (p+1)*chunk).
// In blocked-MMSE plans chunk == pilots per MMSE block, so a part's l < 8
// partial bins are that block's bins (up to the block-origin phase).
template <class Src>
__global__ void __launch_bounds__(ARCHES_K1_THREADS, 3)
    k1_analyze(const PlanDev P, const Src src, const K1Out out, const int npts, const int chunk) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ double s_e[ARCHES_K1_THREADS / 32];
  __shared__ int s_flag;
  __shared__ double s_sc;
  const int part = blockIdx.x, n_parts = gridDim.x;
  const int u = blockIdx.y;
  const int tid = threadIdx.x;
  const int AD = P.A * P.D;
  const int L = P.L;
  const int n_l_t = (L + ARCHES_RL - 1) / ARCHES_RL;
  const int n_tiles = ((AD + ARCHES_RA - 1) / ARCHES_RA) * n_l_t;
  const int KS = max(1, ARCHES_K1_THREADS / n_tiles);
  const int tile = tid / KS, ks = tid - tile * KS;
  const bool active = tile < n_tiles;
  const int ad0 = (tile / n_l_t) * ARCHES_RA, l0 = (tile % n_l_t) * ARCHES_RL;
  const float2* wtab = Src::kComb ? P.wM : P.wN;
  const size_t rec = 2 * (size_t)AD * L + 2;  // doubles per partial record

  // smem: [hs: AD*chunk float2 | red: 256*RA*RL float2 (aliased)] [bins: AD*L double2]
  float2* hs = reinterpret_cast<float2*>(smem_raw);
  float2* red = hs;
  const size_t stage = max((size_t)AD * chunk, (size_t)ARCHES_K1_THREADS * ARCHES_RA * ARCHES_RL);
  double2* bins = reinterpret_cast<double2*>(hs + stage);
  double2* Kmat = bins + (size_t)AD * L;

  const int base = part * chunk;
  const int len = min(chunk, npts - base);
  // ---- LS of this part into smem (loads batched for memory-level parallelism)
  float e32 = 0.f;
  if constexpr (Src::kGrid) {
    if (chunk == ARCHES_K1_THREADS && AD <= 16) {
      // one comb point per thread: pilots of its D symbols loaded once, the
      // A*D received samples issued back to back
      const int m = base + tid;
      const bool okp = tid < len;
      const float2* gsrc = reinterpret_cast<const GridCombSrc*>(&src)->y;
      const float2* psrc = reinterpret_cast<const GridCombSrc*>(&src)->pil;
      const int nsl = reinterpret_cast<const GridCombSrc*>(&src)->n_slots;
      float2 pc[ARCHES_MAX_DMRS];
      float pinv[ARCHES_MAX_DMRS];
#pragma unroll
      for (int d = 0; d < ARCHES_MAX_DMRS; ++d) {
        pc[d] = (okp && d < P.D) ? __ldg(&psrc[((size_t)(u / nsl) * P.M + m) * P.D + d])
                                 : make_float2(1.f, 0.f);
        pinv[d] = 1.0f / (pc[d].x * pc[d].x + pc[d].y * pc[d].y);
      }
      float2 v[16];
      const float2* yu = gsrc + (size_t)u * P.A * P.T * P.N + 2 * (size_t)m;
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        if (q < AD && okp) {
          const int a = q / P.D, d = q - a * P.D;
          v[q] = __ldg(&yu[((size_t)a * P.T + P.dsym[d]) * P.N]);
        } else {
          v[q] = make_float2(0.f, 0.f);
        }
      }
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        if (q < AD) {
          const int d = q % P.D;
          float2 pd = pc[0];
          float pi = pinv[0];
#pragma unroll
          for (int dd = 1; dd < ARCHES_MAX_DMRS; ++dd)
            if (d == dd) pd = pc[dd], pi = pinv[dd];
          const float2 qv = cmulc(pd, v[q]);
          const float2 h = make_float2(qv.x * pi, qv.y * pi);
          hs[(size_t)q * chunk + tid] = h;
          e32 = fmaf(h.x, h.x, fmaf(h.y, h.y, e32));
        }
      }
      goto ls_done;
    }
  }
  {
    int ad = tid / chunk, jj = tid - ad * chunk;
    const int step_ad = ARCHES_K1_THREADS / chunk, step_j = ARCHES_K1_THREADS - step_ad * chunk;
    for (int e = tid; e < AD * chunk; e += 8 * ARCHES_K1_THREADS) {
      float2 v[8];
      int aa[8], jv[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        aa[q] = ad;
        jv[q] = jj;
        const bool ok = (ad < AD) && (jj < len);
        v[q] = ok ? src.load(P, u, ad, base + jj) : make_float2(0.f, 0.f);
        ad += step_ad;
        jj += step_j;
        if (jj >= chunk) {
          jj -= chunk;
          ++ad;
        }
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        if (aa[q] < AD) {
          hs[(size_t)aa[q] * chunk + jv[q]] = v[q];
          e32 = fmaf(v[q].x, v[q].x, fmaf(v[q].y, v[q].y, e32));
        }
      }
    }
  }
ls_done:
  __syncthreads();
  // ---- partial analysis bins: register tile RA x RL over a K-slice of points
  float2 acc[ARCHES_RA][ARCHES_RL];
#pragma unroll
  for (int i = 0; i < ARCHES_RA; ++i)
#pragma unroll
    for (int q = 0; q < ARCHES_RL; ++q) acc[i][q] = make_float2(0.f, 0.f);
  if (active && ks < len) {
    int pt = base + ks;
    int idx = (int)(((long long)l0 * pt) % npts);
    const int step = (int)(((long long)l0 * KS) % npts);
    for (int j = ks; j < len; j += KS) {
      const float2 w1 = __ldg(&wtab[pt]);
      float2 w = __ldg(&wtab[idx]);
      float2 hv[ARCHES_RA];
#pragma unroll
      for (int i = 0; i < ARCHES_RA; ++i)
        hv[i] = (ad0 + i < AD) ? hs[(ad0 + i) * chunk + j] : make_float2(0.f, 0.f);
#pragma unroll
      for (int q = 0; q < ARCHES_RL; ++q) {
#pragma unroll
        for (int i = 0; i < ARCHES_RA; ++i) cfma(acc[i][q], hv[i], w);
        w = cmul(w, w1);
      }
      pt += KS;
      idx += step;
      if (idx >= npts) idx -= npts;
    }
  }
  __syncthreads();  // red aliases hs
#pragma unroll
  for (int i = 0; i < ARCHES_RA; ++i)
#pragma unroll
    for (int q = 0; q < ARCHES_RL; ++q)
      red[(size_t)tid * ARCHES_RA * ARCHES_RL + i * ARCHES_RL + q] = acc[i][q];
  double en = warp_sum((double)e32);
  if ((tid & 31) == 0) s_e[tid >> 5] = en;
  __syncthreads();
  double* my = out.parts + ((size_t)u * n_parts + part) * rec;
  for (int o = tid; o < AD * L; o += blockDim.x) {
    const int ad = o / L, l = o - ad * L;
    const int t = (ad / ARCHES_RA) * n_l_t + l / ARCHES_RL;
    const int slot = (ad % ARCHES_RA) * ARCHES_RL + (l % ARCHES_RL);
    double sx = 0.0, sy = 0.0;
    for (int kk = 0; kk < KS; ++kk) {
      const float2 v = red[(size_t)(t * KS + kk) * ARCHES_RA * ARCHES_RL + slot];
      sx += (double)v.x;
      sy += (double)v.y;
    }
    my[2 * o] = sx;
    my[2 * o + 1] = sy;
  }
  if (tid == 0) {
    double e = 0.0;
    for (int w = 0; w < ARCHES_K1_THREADS / 32; ++w) e += s_e[w];
    my[rec - 2] = e;
  }
  // ---- the last CTA of the unit reduces the parts (part order) and finalises
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    const unsigned int prev = atomicAdd(out.counters + u, 1u);
    s_flag = (prev == (unsigned int)n_parts - 1);
    if (s_flag) out.counters[u] = 0u;
  }
  __syncthreads();
  if (!s_flag) return;
  __threadfence();
  const double* all = out.parts + (size_t)u * n_parts * rec;
  for (int o = tid; o < AD * L; o += blockDim.x) {
    double sx = 0.0, sy = 0.0;
    for (int p = 0; p < n_parts; ++p) {
      sx += all[p * rec + 2 * o];
      sy += all[p * rec + 2 * o + 1];
    }
    bins[o] = make_double2(sx, sy);
  }
  __syncthreads();
  if (tid == 32 && out.rng) {  // RNG side products (independent of the bins: other warp)
    const int stream = u / out.n_slots;
    const long long base = out.first_slot >= 0
        ? out.first_slot
        : (long long)*reinterpret_cast<const int64_t*>(out.state + (size_t)stream * out.state_stride);
    const long long slot = base + (u - stream * out.n_slots);
    out.rng[2 * u] = arches_rng::stream_first_uniform(out.seeds[stream], P.crc_key, (uint64_t)slot);
    const double j = arches_rng::lcid4_jitter((uint64_t)slot);
    const double f = __dadd_rn(P.lcid4_fraction, __dmul_rn(P.lcid4_jitter, j));
    out.rng[2 * u + 1] = fmin(fmax(f, 0.0), 1.0);
  }
  if (tid == 0) {
    double e = 0.0;
    for (int p = 0; p < n_parts; ++p) e += all[p * rec + rec - 2];
    double sg = 0.0;
    if (Src::kComb) {
      for (int ad = 0; ad < AD; ++ad)
        for (int l = 0; l < P.guard; ++l) {
          const double2 b = bins[ad * L + l];
          sg += b.x * b.x + b.y * b.y;
        }
    }
    const double nvhat = Src::kComb ? (e - sg / (double)P.M) / ((double)AD * (P.M - P.guard)) : 0.0;
    if (out.sigma2) out.sigma2[u] = nvhat;
    double s = nvhat;
    if (out.nv_in && out.nv_in[u] >= 0.0) s = out.nv_in[u];
    s_sc = s + P.ridge;
    if ((out.what & K1_MMSE) && !P.diag) solve8_gram(P, s + P.ridge, Kmat);
  }
  __syncthreads();
  if (!out.coef) return;
  const double s = s_sc;
  float2* cm = out.coef + (size_t)u * coef_floats2(P);
  float2* ca = cm + (size_t)AD * P.n_blocks * 8;
  if (out.what & K1_MMSE) {
    if (P.diag) {
      for (int o = tid; o < AD * 8; o += blockDim.x) {
        const int ad = o >> 3, l = o & 7;
        const double w = P.pdp[l] / ((double)P.M * P.pdp[l] + s);
        const double2 b = bins[ad * L + l];
        cm[o] = make_float2((float)(w * b.x), (float)(w * b.y));
      }
    } else {
      const int nb = P.n_blocks;
      for (int o = tid; o < AD * nb * 8; o += blockDim.x) {
        const int ad = o / (nb * 8), r = o - ad * nb * 8, b = r >> 3, l = r & 7;
        double2 acc2 = make_double2(0.0, 0.0);
        for (int lp = 0; lp < 8; ++lp) {
          double2 bb;
          if (nb == 1) {
            bb = bins[ad * L + lp];
          } else {
            // block-local bins: part b's partial with the block-origin phase removed
            const double* pr = all + (size_t)b * rec + 2 * (ad * L + lp);
            double sn, cs;
            sincospi(-2.0 * (double)(((long long)lp * b * chunk) % npts) / (double)npts, &sn, &cs);
            bb = make_double2(pr[0] * cs - pr[1] * sn, pr[0] * sn + pr[1] * cs);
          }
          const double2 t = zmul(Kmat[l * 8 + lp], bb);
          acc2.x += t.x;
          acc2.y += t.y;
        }
        cm[o] = make_float2((float)acc2.x, (float)acc2.y);
      }
    }
  }
  if (out.what & K1_AI) {
    for (int o = tid; o < AD * P.trunc; o += blockDim.x) {
      const int ad = o / P.trunc, l = o - ad * P.trunc;
      const double2 b = bins[ad * L + l];
      double2 v;
      if (Src::kComb) {
        v = zmul(P.ai_fac[l], b);
      } else {
        v = make_double2(b.x / (double)P.N, b.y / (double)P.N);
      }
      ca[o] = make_float2((float)v.x, (float)v.y);
    }
  }
}

// ls_estimate materialised: ls[u][A][D][N], odd subcarriers copy the even one
__global__ void k_ls_materialize(const PlanDev P, const GridCombSrc src, float2* ls, int n_units) {
  const size_t total = (size_t)n_units * P.A * P.D * P.N;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const int k = (int)(i % P.N);
    const size_t r = i / P.N;
    const int ad = (int)(r % (P.A * P.D));
    const int u = (int)(r / (P.A * P.D));
    ls[i] = src.load(P, u, ad, k >> 1);
  }
}
