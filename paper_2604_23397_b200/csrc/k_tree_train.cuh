// Exhaustive depth-2 Gini tree training on the GPU (switch_policy.py:173-234).
//
// The reference scores every root split (feature f, midpoint t between
// consecutive distinct sorted values of f) by the total leaf impurity of the
// best depth-1 tree on each side (`_best_depth1`, :141-162, over every
// feature and every midpoint of the SUBSET), keeping the first minimum in
// (feature, threshold) order -- O(F^2 n^2) work in a Python loop.  Here one
// warp evaluates one root candidate: a ballot pass counts the two subsets,
// then for every child feature g the warp walks g's pre-sorted row order in
// chunks of 32, forms both subsets' running label counts with ballots /
// popc, finds each member's next member in the subset (shuffle; carried
// across chunks), and scores every cut exactly as `_split_candidates`
// (:116-132) does -- the same fp64 operations in the same order, so totals,
// thresholds and every tie (first cut in a feature, strictly better feature,
// strictly better root) match the reference bit for bit.
#pragma once
#include "common.cuh"
#include "k_synth_eq.cuh"

#define TT_WARPS 4

// _leaf_total: n - (c0^2 + c1^2) / n (CPython: exact int numerator, correctly rounded /)
__device__ __forceinline__ double tt_leaf_total(long long n, long long c0) {
  if (n == 0) return 0.0;
  const long long c1 = n - c0;
  return xsub((double)n, xdiv((double)(c0 * c0 + c1 * c1), (double)n));
}

// _split_candidates totals[k] for a cut after n_l members (c0 of label 0) of a
// subset of n members, t0 of label 0 (numpy float64 element-wise, same order)
__device__ __forceinline__ double tt_split_total(double n_l, double c0, double n, double t0) {
  const double c1 = xsub(n_l, c0);
  const double t1 = xsub(n, t0);
  const double r0 = xsub(t0, c0), r1 = xsub(t1, c1);
  const double n_r = xsub(n, n_l);
  const double a = xsub(n_l, xdiv(xadd(xmul(c0, c0), xmul(c1, c1)), n_l));
  const double b = xsub(n_r, xdiv(xadd(xmul(r0, r0), xmul(r1, r1)), n_r));
  return xadd(a, b);
}

struct TTBest {     // running best of one subset
  double total;     // best total so far
  double thr;
  int feat;         // -1: leaf
};

__global__ void __launch_bounds__(32 * TT_WARPS)
    k_tree_eval_splits(const double* xT, const int32_t* order, const uint8_t* y, int n, int F,
                       const int32_t* root_feat, const double* root_thr, int n_roots,
                       arches_split_eval* out) {
  const int c = blockIdx.x * TT_WARPS + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (c >= n_roots) return;  // warp-uniform
  const int f = root_feat[c];
  const double t = root_thr[c];
  const unsigned FULL = 0xffffffffu;
  const unsigned lt_mask = (1u << lane) - 1u, le_mask = lt_mask | (1u << lane);
  // ---- subset sizes (left = x[:, f] <= t; f < 0: the whole set is "left")
  int nl = 0, nl0 = 0, n0 = 0;
  for (int i = lane; i < n; i += 32) {
    const bool in_l = f < 0 || xT[(size_t)f * n + i] <= t;
    const bool lab0 = y[i] == 0;
    nl += in_l;
    nl0 += in_l && lab0;
    n0 += lab0;
  }
  for (int o = 16; o; o >>= 1) {
    nl += __shfl_xor_sync(FULL, nl, o);
    nl0 += __shfl_xor_sync(FULL, nl0, o);
    n0 += __shfl_xor_sync(FULL, n0, o);
  }
  const int nr = n - nl, nr0 = n0 - nl0;
  const int ns[2] = {nl, nr}, ns0[2] = {nl0, nr0};
  TTBest best[2];
  bool active[2];
  for (int s = 0; s < 2; ++s) {
    best[s].total = tt_leaf_total(ns[s], ns0[s]);
    best[s].thr = 0.0;
    best[s].feat = -1;
    active[s] = ns0[s] != 0 && ns0[s] != ns[s];  // a pure subset stays a leaf (:151-152)
  }
  for (int g = 0; g < F && (active[0] || active[1]); ++g) {
    const int32_t* og = order + (size_t)g * n;
    const double* xg = xT + (size_t)g * n;
    double fb_tot[2] = {INFINITY, INFINITY}, fb_thr[2] = {0.0, 0.0};
    int cnt[2] = {0, 0}, cnt0[2] = {0, 0};           // members / label-0 members so far
    bool pend[2] = {false, false};                   // last member of the previous chunk
    double pend_v[2] = {0.0, 0.0};
    int pend_n[2] = {0, 0}, pend_c0[2] = {0, 0};
    const double nsd[2] = {(double)nl, (double)nr}, ns0d[2] = {(double)nl0, (double)nr0};
    for (int i0 = 0; i0 < n; i0 += 32) {
      const int i = i0 + lane;
      const bool valid = i < n;
      const int r = valid ? og[i] : 0;
      const double v = valid ? xg[r] : 0.0;
      const bool in_l = valid && (f < 0 || xT[(size_t)f * n + r] <= t);
      const bool lab0 = valid && y[r] == 0;
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        if (!active[s]) continue;  // warp-uniform
        const bool mem = valid && (s == 0 ? in_l : !in_l);
        const unsigned mask = __ballot_sync(FULL, mem);
        const unsigned mask0 = __ballot_sync(FULL, mem && lab0);
        if (!mask) continue;
        const int first = __ffs(mask) - 1;
        const double v_first = __shfl_sync(FULL, v, first);
        if (pend[s] && pend_v[s] < v_first) {  // cut after the previous chunk's last member
          const double tot = tt_split_total((double)pend_n[s], (double)pend_c0[s], nsd[s], ns0d[s]);
          if (tot < fb_tot[s]) {
            fb_tot[s] = tot;
            fb_thr[s] = xmul(0.5, xadd(pend_v[s], v_first));
          }
        }
        // this member's inclusive counts and its next member inside the chunk
        const int my_n = cnt[s] + __popc(mask & le_mask);
        const int my_c0 = cnt0[s] + __popc(mask0 & le_mask);
        const unsigned above = mask & ~le_mask;
        const int nxt = above ? __ffs(above) - 1 : lane;
        const double v_next = __shfl_sync(FULL, v, nxt);
        const bool cut = mem && above && v < v_next;
        double tot = cut ? tt_split_total((double)my_n, (double)my_c0, nsd[s], ns0d[s]) : INFINITY;
        // first (lowest-position) minimum of the chunk
        int arg = lane;
        for (int o = 16; o; o >>= 1) {
          const double ot = __shfl_xor_sync(FULL, tot, o);
          const int oa = __shfl_xor_sync(FULL, arg, o);
          if (ot < tot || (ot == tot && oa < arg)) {
            tot = ot;
            arg = oa;
          }
        }
        const double va = __shfl_sync(FULL, v, arg), vn = __shfl_sync(FULL, v_next, arg);
        if (tot < fb_tot[s]) {  // warp-uniform; earlier chunks win ties
          fb_tot[s] = tot;
          fb_thr[s] = xmul(0.5, xadd(va, vn));
        }
        const int last = 31 - __clz(mask);
        pend[s] = true;
        pend_v[s] = __shfl_sync(FULL, v, last);
        pend_n[s] = __shfl_sync(FULL, my_n, last);
        pend_c0[s] = __shfl_sync(FULL, my_c0, last);
        cnt[s] += __popc(mask);
        cnt0[s] += __popc(mask0);
      }
    }
    for (int s = 0; s < 2; ++s)  // _best_depth1: a strictly better feature replaces (:156-160)
      if (active[s] && fb_tot[s] < best[s].total) {
        best[s].total = fb_tot[s];
        best[s].thr = fb_thr[s];
        best[s].feat = g;
      }
  }
  if (lane == 0) {
    arches_split_eval e;
    e.left_total = best[0].total;
    e.right_total = best[1].total;
    e.total = xadd(best[0].total, best[1].total);
    e.left_threshold = best[0].thr;
    e.right_threshold = best[1].thr;
    e.left_feature = best[0].feat;
    e.right_feature = best[1].feat;
    out[c] = e;
  }
}
