// K4 (block form) -- one CTA per stream; slot-parallel KPM derivation over
// chunks of blockDim slots.
//
// Same semantics and bit-exact records as the sequential k4_kpm_scan
// (k_control.cuh, cross-checked in tests/test_kpm_scan_gpu.py) -- the order-dependent tail of
// Pipeline.run_slot (phy_pipeline.py:462-488), SwitchController (:94-144),
// ThroughputWindow (:325-344), Dapp.on_indication / window_features /
// predict (dapp_control.py:85-120, switch_policy.py:237-248), FailsafeMonitor
// (dapp_control.py:123-149) -- with the chunk widened from a warp to the whole
// CTA, so a 256-slot batch of one stream takes one pass of loads, block-wide
// prefix scans and stores instead of eight dependent warp passes:
//   1. control walk: the oracle source in closed form (slot-parallel), the
//      other sources walked by thread 0 up to the next dApp decision slot;
//   2. thread = slot: candidate select, cumulative PHY bytes / NDI parity /
//      MAC + LCID4 window totals as block prefix scans, CPython-order fp64;
//   3. at a decision slot threads 0..9 form the window means (sequential fp64
//      column sums in slot order), thread 0 runs the tree.
#pragma once
#include <limits.h>

#include "k_control_warp.cuh"

#define K4B_THREADS 256
#define K4B_WIN_ROWS 128  // dApp window rows staged per pass (10 KB of fp64)

// block-wide inclusive scan (blockDim == K4B_THREADS); `tmp` holds one entry per warp
template <typename T>
__device__ __forceinline__ T block_incl_scan(T v, T* tmp) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  v = warp_incl_scan(v, lane);
  if (lane == 31) tmp[w] = v;
  __syncthreads();
  if (w == 0) {
    T x = lane < K4B_THREADS / 32 ? tmp[lane] : T(0);
    x = warp_incl_scan(x, lane);
    if (lane < K4B_THREADS / 32) tmp[lane] = x;
  }
  __syncthreads();
  const T off = w > 0 ? tmp[w - 1] : T(0);
  __syncthreads();  // tmp reusable by the next scan
  return v + off;
}

__global__ void __launch_bounds__(K4B_THREADS) k4_kpm_scan_block(const PlanDev P, const K4Args a) {
  const int stream = blockIdx.x;
  const int tid = threadIdx.x;
  __shared__ int s_mode[K4B_THREADS];
  __shared__ int s_g[K4B_THREADS];
  __shared__ int32_t s_mac[K4B_THREADS], s_l4[K4B_THREADS];
  __shared__ long long s_tmp[K4B_THREADS / 32];
  __shared__ int s_len, s_decide;
  __shared__ StreamState s_st;
  __shared__ double s_feat[ARCHES_FEATURES];
  __shared__ double s_win[K4B_WIN_ROWS * ARCHES_FEATURES];
  StateView sv = state_view(a.state, stream, P.window_length, P.dapp_window);
  if (tid == 0) s_st = *sv.h;
  __syncthreads();
  const int W = P.window_length, WD = P.dapp_window;
  const int64_t slot_ns = P.slot_ns;
  int s0 = 0;
  while (s0 < a.n_slots) {
    // ---------------- 1. control walk
    const int lim = min(K4B_THREADS, a.n_slots - s0);
    if (P.policy == ARCHES_POLICY_ORACLE) {
      const int uu = stream * a.n_slots + s0 + tid;
      s_g[tid] = (tid < lim && a.regime && a.regime[uu]) ? 1 : 0;
    }
    __syncthreads();
    if (P.policy == ARCHES_POLICY_ORACLE && s_st.n_forced == 0) {
      // closed form (every slot is independent given the regimes): L(n) = regime(n), a message iff
      // regime(n) != L(n-1), applied at the next (concurrent) or the one after
      // (selected-only) boundary
      const bool act0 = tid < lim;
      const int g = s_g[tid];
      const int lm1 = tid >= 1 ? s_g[tid - 1] : s_st.last_msg_mode;
      const int lm2 = tid >= 2 ? s_g[tid - 2] : tid == 1 ? s_st.last_msg_mode : s_st.prev_msg_mode;
      const bool sel = P.exec_mode == ARCHES_EXEC_SELECTED_ONLY;
      const int mode = sel ? lm2 : lm1;
      const int msg = (act0 && g != lm1) ? 1 : 0;
      if (act0) s_mode[tid] = mode;
      const int cnt0 = a.msg_count ? a.msg_count[stream] : 0;
      const long long before = block_incl_scan((long long)msg, s_tmp) - msg;
      const int64_t n = s_st.next_slot + tid;
      const int64_t end_ns = (n + 1) * slot_ns;
      if (msg && a.msg_log) {
        const long long idx = cnt0 + before;
        if (idx < a.msg_cap) {
          arches_message m;
          m.decided_at_ns = end_ns;
          m.deliverable_at_ns = end_ns;
          m.mode = g;
          m.trigger = ARCHES_TRIGGER_ORACLE;
          a.msg_log[(size_t)stream * a.msg_cap + idx] = m;
        }
      }
      const int last = lim - 1;
      if (tid == last) {
        s_tmp[0] = before + msg;  // messages in this chunk
        StreamState& st = s_st;
        const int g_last = g, lm1_last = lm1, mode_last = mode, msg_l1 = msg;
        const int g_l2 = last > 0 ? s_g[last - 1] : 0;
        const int lml2 = last > 1 ? s_g[last - 2] : last == 1 ? st.last_msg_mode : 0;
        const int msg_l2 = last > 0 ? ((g_l2 != lml2) ? 1 : 0) : 0;
        const int64_t n_last = st.next_slot + last;
        const int64_t cut = sel ? (n_last - 1) * slot_ns : n_last * slot_ns;  // begin_slot(n_last)
        RegQueue pq;
        pq.load(st.pending, st.n_pending);
        RegQueue nq;
        nq.load(st.pending, 0);
#pragma unroll
        for (int i = 0; i < ARCHES_MAX_PENDING; ++i) nq.at[i] = 0, nq.mode[i] = 0, nq.trig[i] = 0;
        for (int i = 0; i < ARCHES_MAX_PENDING; ++i) {
          if (i >= pq.n) break;
          if (pq.at[0] > cut) nq.insert(pq.at[0], pq.mode[0], pq.trig[0]);
          pq.pop();
        }
        if (last > 0 && msg_l2 && n_last * slot_ns > cut)
          nq.insert(n_last * slot_ns, g_l2, ARCHES_TRIGGER_ORACLE);
        if (msg_l1 && (n_last + 1) * slot_ns > cut)
          nq.insert((n_last + 1) * slot_ns, g_last, ARCHES_TRIGGER_ORACLE);
        nq.store(st.pending, st.n_pending);
        st.mode = mode_last;
        st.prev_msg_mode = lm1_last;
        st.last_msg_mode = g_last;
        s_len = lim;
        s_decide = 0;
      }
      __syncthreads();
      if (tid == 0 && a.msg_count) a.msg_count[stream] = cnt0 + (int)s_tmp[0];
    } else if (P.policy != ARCHES_POLICY_ORACLE && lim > 8) {
      // tree / fixed sources, slot-parallel: between two dApp decisions the queues
      // only drain (plus at most one fail-safe trip), so every slot's mode is the
      // latest queued event applied by then -- key (apply slot, pending < forced,
      // queue order) -- and the trip is the first slot whose predicate holds
      // (SwitchController.begin_slot, phy_pipeline.py:123-139; FailsafeMonitor,
      // dapp_control.py:123-149).  Same states and logs as the sequential walk,
      // which still serves short chunks (a decision every slot: fewer barriers).
      const StreamState& st = s_st;
      const int64_t nbase = st.next_slot;
      const bool sel = P.exec_mode == ARCHES_EXEC_SELECTED_ONLY;
      int len = lim, decide = 0;
      if (P.policy == ARCHES_POLICY_TREE) {
        const int jd = max(0, P.decision_period - st.since_decision - 1);  // the decision slot
        if (jd < lim) {
          len = jd + 1;
          decide = 1;
        }
      }
      const int np = st.n_pending, nf = st.n_forced;
      const int64_t n = nbase + tid;
      // apply slot of a message: first slot whose begin time passes it
      auto ceil_slot = [&](int64_t at) { return at <= 0 ? (int64_t)0 : (at + slot_ns - 1) / slot_ns; };
      int best_s = -1, best_k = -1, best_i = -1, mode = st.mode;
      auto consider = [&](int64_t as, int kind, int i, int m) {
        if (as > n) return;
        const int asi = (int)(as - nbase);
        if (asi > best_s || (asi == best_s && (kind > best_k || (kind == best_k && i > best_i)))) {
          best_s = asi;
          best_k = kind;
          best_i = i;
          mode = m;
        }
      };
      if (tid < len) {
        for (int i = 0; i < np; ++i)
          consider(ceil_slot(st.pending[i].at_ns) + (sel ? 1 : 0), 0, i, st.pending[i].mode);
        for (int i = 0; i < nf; ++i) consider(ceil_slot(st.forced[i].at_ns), 1, i, st.forced[i].mode);
      }
      if (tid == 0) s_decide = INT_MAX;  // first fail-safe trip slot (scratch)
      __syncthreads();
      if (P.policy == ARCHES_POLICY_TREE && tid < len && !(decide && tid == len - 1) && !st.tripped &&
          (n + 1) * slot_ns - st.last_delivery_ns > P.failsafe_timeout_ns && mode != 1)
        atomicMin(&s_decide, tid);
      __syncthreads();
      const int trip = s_decide;  // INT_MAX: none
      if (tid < len) {
        if (trip != INT_MAX && tid > trip) consider(nbase + trip + 1, 1, ARCHES_MAX_PENDING, 1);
        s_mode[tid] = mode;
      }
      __syncthreads();
      if (tid == 0) {
        StreamState& sw = s_st;
        const int64_t last = nbase + len - 1;
        RegQueue pq, fq;
        pq.load(sw.pending, sw.n_pending);
        fq.load(sw.forced, sw.n_forced);
        while (pq.n > 0 && ceil_slot(pq.at[0]) + (sel ? 1 : 0) <= last) pq.pop();
        while (fq.n > 0 && ceil_slot(fq.at[0]) <= last) fq.pop();
        int cnt = a.msg_count ? a.msg_count[stream] : 0;
        if (trip != INT_MAX) {
          const int64_t end_ns = (nbase + trip + 1) * slot_ns;
          if (nbase + trip + 1 > last) fq.insert(end_ns, 1, ARCHES_TRIGGER_FAILSAFE);  // applies next chunk
          sw.tripped = 1;
          log_msg_fast(a.msg_log, a.msg_cap, stream, cnt, 1, end_ns, end_ns, ARCHES_TRIGGER_FAILSAFE);
        }
        pq.store(sw.pending, sw.n_pending);
        fq.store(sw.forced, sw.n_forced);
        sw.mode = s_mode[len - 1];
        if (P.policy == ARCHES_POLICY_TREE) sw.since_decision += len;
        if (a.msg_count) a.msg_count[stream] = cnt;
        s_len = len;
        s_decide = decide;
      }
    } else if (tid == 0) {
      StreamState& st = s_st;
      RegQueue pq, fq;
      pq.load(st.pending, st.n_pending);
      fq.load(st.forced, st.n_forced);
      int mode = st.mode, last_msg = st.last_msg_mode, prev_msg = st.prev_msg_mode;
      int since = st.since_decision;
      int tripped = st.tripped;
      int64_t last_del = st.last_delivery_ns;
      int cnt = a.msg_count ? a.msg_count[stream] : 0;
      const int64_t nbase = st.next_slot;
      int j = 0, decide = 0;
      for (; j < lim; ++j) {
        const int64_t n = nbase + j;
        const int64_t t0 = n * slot_ns;
        const int64_t cut = (P.exec_mode == ARCHES_EXEC_SELECTED_ONLY) ? t0 - slot_ns : t0;
        while (pq.n > 0 && pq.at[0] <= cut) {
          mode = pq.mode[0];
          pq.pop();
        }
        while (fq.n > 0 && fq.at[0] <= t0) {
          mode = fq.mode[0];
          fq.pop();
        }
        s_mode[j] = mode;
        const int64_t end_ns = t0 + slot_ns;
        if (P.policy == ARCHES_POLICY_ORACLE) {
          const int want = s_g[j];
          prev_msg = last_msg;
          if (want != last_msg) {
            pq.insert(end_ns, want, ARCHES_TRIGGER_ORACLE);
            last_msg = want;
            log_msg_fast(a.msg_log, a.msg_cap, stream, cnt, want, end_ns, end_ns, ARCHES_TRIGGER_ORACLE);
          }
        } else if (P.policy == ARCHES_POLICY_TREE) {
          if (++since >= P.decision_period) {
            decide = 1;  // features of slots <= n needed: stop the walk here
            ++j;
            break;
          }
          if (!tripped && end_ns - last_del > P.failsafe_timeout_ns && mode != 1) {
            tripped = 1;
            fq.insert(end_ns, 1, ARCHES_TRIGGER_FAILSAFE);
            log_msg_fast(a.msg_log, a.msg_cap, stream, cnt, 1, end_ns, end_ns, ARCHES_TRIGGER_FAILSAFE);
          }
        }
      }
      pq.store(st.pending, st.n_pending);
      fq.store(st.forced, st.n_forced);
      st.mode = mode;
      st.last_msg_mode = last_msg;
      st.prev_msg_mode = prev_msg;
      st.since_decision = since;
      st.tripped = tripped;
      st.last_delivery_ns = last_del;
      if (a.msg_count) a.msg_count[stream] = cnt;
      s_len = j;
      s_decide = decide;
    }
    __syncthreads();
    const int len = s_len;
    const int decide = s_decide;
    const int64_t n0 = s_st.next_slot;
    // ---------------- 2. slot-parallel KPM derivation
    const bool act = tid < len;
    const int64_t n = n0 + tid;
    const int u = stream * a.n_slots + s0 + tid;
    int e = 0, mcs = 0, tb = 0, crc = 0, mac_rx = 0, l4_rx = 0, ncb = 1;
    double rsrp = 0.0, snr = 0.0, absm = 0.0;
    if (act) {
      e = s_mode[tid];
      const arches_telemetry& tl = a.tel[u];
      mcs = tl.mcs[e];
      tb = tl.tb_bytes[e];
      crc = tl.crc[e];
      mac_rx = tl.mac_rx[e];
      l4_rx = tl.lcid4_rx[e];
      ncb = tl.num_cb[e];
      rsrp = tl.rsrp[e];
      snr = tl.sinr_db[e];
      absm = tl.abs_mean[e];
    }
    s_mac[tid] = mac_rx;
    s_l4[tid] = l4_rx;
    // chunk-start totals, read before any thread carries the new ones below
    const long long mac0 = s_st.mac_total, l40 = s_st.l4_total, cum0 = s_st.cum_phy_bytes;
    const int ndi0 = s_st.ndi;
    __syncthreads();
    // evicted window values (pushed W slots earlier), ring indexed by n % W
    int32_t ev_mac = 0, ev_l4 = 0;
    if (act && n >= W) {
      if (tid >= W) {
        ev_mac = s_mac[tid - W];
        ev_l4 = s_l4[tid - W];
      } else {
        ev_mac = sv.mac_ring[n % W];
        ev_l4 = sv.l4_ring[n % W];
      }
    }
    const long long d_mac = act ? (long long)mac_rx - ev_mac : 0;
    const long long d_l4 = act ? (long long)l4_rx - ev_l4 : 0;
    const long long d_phy = (act && crc) ? (long long)tb : 0;
    const long long c_crc = (act && crc) ? 1 : 0;
    const long long mac_tot = mac0 + block_incl_scan(d_mac, s_tmp);
    const long long l4_tot = l40 + block_incl_scan(d_l4, s_tmp);
    const long long cum = cum0 + block_incl_scan(d_phy, s_tmp);
    const long long crc_incl = block_incl_scan(c_crc, s_tmp);
    const int ndi = ndi0 ^ (int)((crc_incl - c_crc) & 1);
    if (act) {
      const int filled = (int)min((long long)W, (long long)n + 1);
      const double denom = xmul((double)filled, P.slot_s);
      const double mac_t = xdiv(xdiv(xmul((double)mac_tot, 8.0), 1e6), denom);
      const double l4_t = xdiv(xdiv(xmul((double)l4_tot, 8.0), 1e6), denom);
      const double elapsed = xmul(xmul((double)(n + 1), P.slot_us), 1e-6);
      const double phy_t = xdiv(xdiv(xmul((double)cum, 8.0), 1e6), elapsed);
      const int pdu = max(tb - P.mac_header_bytes, 0);
      arches_kpm r;
      r.slot_index = n;
      r.phy_throughput = phy_t;
      r.rsrp = rsrp;
      r.code_rate = P.mcs_rate[mcs];
      r.snr_db = snr;
      r.mac_throughput = mac_t;
      r.lcid4_throughput = l4_t;
      r.est_abs_mean = absm;
      r.mcs_index = mcs;
      r.pdu_length = pdu;
      r.ndi = ndi;
      r.qam_order = P.mcs_qam[mcs];
      r.num_cb = ncb;
      r.tb_size = tb;
      r.mac_rx_bytes = mac_rx;
      r.lcid4_rx_bytes = l4_rx;
      r.mode = e;
      r.crc_pass = crc;
      a.kpm[u] = r;
      // ring updates: the last slot mapping to a ring entry wins
      if (tid + W >= len) {
        sv.mac_ring[n % W] = mac_rx;
        sv.l4_ring[n % W] = l4_rx;
      }
      if (P.policy == ARCHES_POLICY_TREE && tid + WD >= len) {
        double* row = sv.feat + (size_t)(n % WD) * ARCHES_FEATURES;
        row[0] = phy_t;
        row[1] = (double)mcs;
        row[2] = (double)pdu;
        row[3] = (double)ndi;
        row[4] = rsrp;
        row[5] = snr;
        row[6] = mac_t;
        row[7] = l4_t;
        row[8] = (double)mac_rx;
        row[9] = (double)l4_rx;
      }
      if (tid == len - 1) {  // carry the chunk totals
        s_st.mac_total = mac_tot;
        s_st.l4_total = l4_tot;
        s_st.cum_phy_bytes = cum;
        s_st.ndi = ndi ^ (int)c_crc;
        s_st.next_slot = n0 + len;
      }
    }
    __syncthreads();
    // ---------------- 3. dApp decision at the chunk's last slot
    if (decide) {
      const int64_t nd = n0 + len - 1;
      const int rows = (int)min((long long)WD, (long long)nd + 1);
      // the window rows are staged into shared memory by the whole CTA (coalesced,
      // all loads in flight at once), then threads 0..9 add them in slot order
      double acc = 0.0;
      for (int r0 = 0; r0 < rows; r0 += K4B_WIN_ROWS) {
        const int nr = min(K4B_WIN_ROWS, rows - r0);
        for (int i = tid; i < nr * ARCHES_FEATURES; i += K4B_THREADS) {
          const int r = i / ARCHES_FEATURES, f = i - r * ARCHES_FEATURES;
          const int64_t p = nd - rows + 1 + r0 + r;  // oldest first
          s_win[i] = sv.feat[(size_t)(p % WD) * ARCHES_FEATURES + f];
        }
        __syncthreads();
        if (tid < ARCHES_FEATURES)
          for (int r = 0; r < nr; ++r) acc = xadd(acc, s_win[r * ARCHES_FEATURES + tid]);
        __syncthreads();
      }
      if (tid < ARCHES_FEATURES) s_feat[tid] = xdiv(acc, (double)rows);
      __syncthreads();
      if (tid == 0) {
        StreamState& st = s_st;
        st.since_decision = 0;
        const int64_t end_ns = (nd + 1) * slot_ns;
        const int mode = tree_descend(a.tree, s_feat);
        const int64_t decided = end_ns + P.decision_delay_ns;
        PendingMsg m = {decided, mode, ARCHES_TRIGGER_POLICY};
        queue_insert(st.pending, st.n_pending, m);
        st.last_delivery_ns = max(st.last_delivery_ns, decided);
        st.tripped = 0;
        log_message(a.msg_log, a.msg_count, a.msg_cap, stream, mode, decided, decided,
                    ARCHES_TRIGGER_POLICY);
        if (!st.tripped && end_ns - st.last_delivery_ns > P.failsafe_timeout_ns && st.mode != 1) {
          st.tripped = 1;
          PendingMsg f = {end_ns, 1, ARCHES_TRIGGER_FAILSAFE};
          queue_insert(st.forced, st.n_forced, f);
          log_message(a.msg_log, a.msg_count, a.msg_cap, stream, 1, end_ns, end_ns,
                      ARCHES_TRIGGER_FAILSAFE);
        }
      }
      __syncthreads();
    }
    s0 += len;
  }
  if (tid == 0) *sv.h = s_st;
}
