// K4 (warp form) -- one warp per stream; slot-parallel KPM derivation.
//
// Same semantics as k4_kpm_scan (k_control.cuh), restructured so only the
// control plane stays sequential:
//   1. lane 0 walks up to 32 slots applying SwitchController.begin_slot, the
//      oracle message source and the fail-safe (integer ns, cheap) and stops
//      early at a dApp decision slot -- the only event that needs KPMs;
//   2. all lanes derive their slot's KPM record in parallel: cumulative PHY
//      bytes / NDI parity / MAC + LCID4 window totals are warp prefix scans,
//      the throughput divisions are per-lane fp64 with CPython rounding;
//   3. at a decision slot lanes 0..9 form the window-mean features (sequential
//      fp64 column sums in slot order, as numpy's axis-0 mean), lane 0 runs the
//      tree and queues the ControlMessage.
// Rings are indexed by push count: mac/l4 values at [n % W], features at
// [n % WD] (n = slot index since stream start == pushes so far).
#pragma once
#include "k_control.cuh"

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

// register-resident copy of a PendingMsg queue (static indexing only)
struct RegQueue {
  int64_t at[ARCHES_MAX_PENDING];
  int32_t mode[ARCHES_MAX_PENDING];
  int32_t trig[ARCHES_MAX_PENDING];
  int32_t n;
  __device__ __forceinline__ void load(const PendingMsg* q, int32_t cnt) {
    n = cnt;
#pragma unroll
    for (int i = 0; i < ARCHES_MAX_PENDING; ++i) {
      at[i] = q[i].at_ns;
      mode[i] = q[i].mode;
      trig[i] = q[i].trigger;
    }
  }
  __device__ __forceinline__ void store(PendingMsg* q, int32_t& cnt) const {
    cnt = n;
#pragma unroll
    for (int i = 0; i < ARCHES_MAX_PENDING; ++i) {
      q[i].at_ns = at[i];
      q[i].mode = mode[i];
      q[i].trigger = trig[i];
    }
  }
  __device__ __forceinline__ void pop() {
#pragma unroll
    for (int i = 0; i < ARCHES_MAX_PENDING - 1; ++i) {
      at[i] = at[i + 1];
      mode[i] = mode[i + 1];
      trig[i] = trig[i + 1];
    }
    at[ARCHES_MAX_PENDING - 1] = 0;
    mode[ARCHES_MAX_PENDING - 1] = 0;
    trig[ARCHES_MAX_PENDING - 1] = 0;
    --n;
  }
  // stable insert by time (same semantics as queue_insert)
  __device__ __forceinline__ void insert(int64_t t, int32_t m, int32_t tr) {
    if (n >= ARCHES_MAX_PENDING) pop();
    int pos = n;
#pragma unroll
    for (int i = ARCHES_MAX_PENDING - 1; i >= 0; --i)
      if (i < n && at[i] > t) pos = i;
#pragma unroll
    for (int i = ARCHES_MAX_PENDING - 1; i > 0; --i)
      if (i > pos && i <= n) {
        at[i] = at[i - 1];
        mode[i] = mode[i - 1];
        trig[i] = trig[i - 1];
      }
#pragma unroll
    for (int i = 0; i < ARCHES_MAX_PENDING; ++i)
      if (i == pos) {
        at[i] = t;
        mode[i] = m;
        trig[i] = tr;
      }
    ++n;
  }
};

__device__ __forceinline__ void log_msg_fast(arches_message* log, int cap, int stream, int& cnt,
                                             int mode, int64_t decided, int64_t deliverable,
                                             int trigger) {
  if (log && cnt < cap) {
    arches_message m;
    m.decided_at_ns = decided;
    m.deliverable_at_ns = deliverable;
    m.mode = mode;
    m.trigger = trigger;
    log[(size_t)stream * cap + cnt] = m;
  }
  ++cnt;
}

__global__ void __launch_bounds__(32) k4_kpm_scan_warp(const PlanDev P, const K4Args a) {
  const int stream = blockIdx.x;
  const int lane = threadIdx.x;
  if (stream >= a.n_streams) return;
  __shared__ int s_mode[32];
  __shared__ int s_len, s_decide;
  __shared__ StreamState s_st;
  StateView sv = state_view(a.state, stream, P.window_length, P.dapp_window);
  if (lane == 0) s_st = *sv.h;
  __syncwarp();
  const int W = P.window_length, WD = P.dapp_window;
  const int64_t slot_ns = P.slot_ns;
  int s0 = 0;
  while (s0 < a.n_slots) {
    // ---------------- 1. sequential control walk (lane 0, registers only)
    unsigned int good_mask = 0u;
    if (P.policy == ARCHES_POLICY_ORACLE) {
      const int uu = stream * a.n_slots + s0 + lane;
      const int g = (s0 + lane < a.n_slots && a.regime && a.regime[uu]) ? 1 : 0;
      good_mask = __ballot_sync(0xffffffffu, g);
    }
    if (P.policy == ARCHES_POLICY_ORACLE && s_st.n_forced == 0) {
      // Oracle source in closed form (every slot is independent given the
      // regimes): after slot n the last message mode is L(n) = regime(n); a
      // message is emitted iff regime(n) != L(n-1); it is applied at the next
      // boundary (concurrent) or the one after (selected-only), so
      // mode(n) = L(n-1) resp. L(n-2).  Identical to the sequential walk.
      const int lim = min(32, a.n_slots - s0);
      const bool act0 = lane < lim;
      const int g = (good_mask >> lane) & 1;
      int lm1 = __shfl_up_sync(0xffffffffu, g, 1);
      int lm2 = __shfl_up_sync(0xffffffffu, g, 2);
      if (lane == 0) lm1 = s_st.last_msg_mode;
      if (lane == 0) lm2 = s_st.prev_msg_mode;
      if (lane == 1) lm2 = s_st.last_msg_mode;
      const bool sel = P.exec_mode == ARCHES_EXEC_SELECTED_ONLY;
      const int mode = sel ? lm2 : lm1;
      const int msg = (act0 && g != lm1) ? 1 : 0;
      if (act0) s_mode[lane] = mode;
      const unsigned int mm = __ballot_sync(0xffffffffu, msg);
      const int cnt0 = a.msg_count ? a.msg_count[stream] : 0;
      const int64_t n = s_st.next_slot + lane;
      const int64_t end_ns = (n + 1) * slot_ns;
      if (msg && a.msg_log) {
        const int idx = cnt0 + __popc(mm & ((1u << lane) - 1u));
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
      const int g_last = __shfl_sync(0xffffffffu, g, last);
      const int lm1_last = __shfl_sync(0xffffffffu, lm1, last);
      const int mode_last = __shfl_sync(0xffffffffu, mode, last);
      const int msg_l1 = __shfl_sync(0xffffffffu, msg, last);
      const int msg_l2 = __shfl_sync(0xffffffffu, msg, last > 0 ? last - 1 : 0);
      const int g_l2 = __shfl_sync(0xffffffffu, g, last > 0 ? last - 1 : 0);
      if (lane == 0) {
        StreamState& st = s_st;
        const int64_t n_last = st.next_slot + last;
        const int64_t cut = sel ? (n_last - 1) * slot_ns : n_last * slot_ns;  // begin_slot(n_last)
        RegQueue pq;
        pq.load(st.pending, st.n_pending);
        RegQueue nq;
        nq.load(st.pending, 0);  // empty, canonical zeros
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
        if (a.msg_count) a.msg_count[stream] = cnt0 + __popc(mm);
        s_len = lim;
        s_decide = 0;
      }
    } else if (lane == 0) {
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
      const int lim = min(32, a.n_slots - s0);
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
          const int want = (good_mask >> j) & 1;
          prev_msg = last_msg;
          if (want != last_msg) {
            pq.insert(end_ns, want, ARCHES_TRIGGER_ORACLE);
            last_msg = want;
            log_msg_fast(a.msg_log, a.msg_cap, stream, cnt, want, end_ns, end_ns,
                         ARCHES_TRIGGER_ORACLE);
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
            log_msg_fast(a.msg_log, a.msg_cap, stream, cnt, 1, end_ns, end_ns,
                         ARCHES_TRIGGER_FAILSAFE);
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
    __syncwarp();
    const int len = s_len;
    const int decide = s_decide;
    const int64_t n0 = s_st.next_slot;
    // ---------------- 2. slot-parallel KPM derivation
    const bool act = lane < len;
    const int64_t n = n0 + lane;
    const int u = stream * a.n_slots + s0 + lane;
    int e = 0, mcs = 0, tb = 0, crc = 0, mac_rx = 0, l4_rx = 0, ncb = 1;
    double rsrp = 0.0, snr = 0.0, absm = 0.0;
    if (act) {
      e = s_mode[lane];
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
    // evicted window values (pushed W slots earlier), ring indexed by n % W
    int32_t sh_mac = 0, sh_l4 = 0;
    if (W < 32) {  // warp-uniform: the evicted value may come from this chunk
      sh_mac = __shfl_sync(0xffffffffu, mac_rx, (lane - W) & 31);
      sh_l4 = __shfl_sync(0xffffffffu, l4_rx, (lane - W) & 31);
    }
    int32_t ev_mac = 0, ev_l4 = 0;
    if (act && n >= W) {
      if (lane >= W) {
        ev_mac = sh_mac;
        ev_l4 = sh_l4;
      } else {
        ev_mac = sv.mac_ring[n % W];
        ev_l4 = sv.l4_ring[n % W];
      }
    }
    const long long d_mac = act ? (long long)mac_rx - ev_mac : 0;
    const long long d_l4 = act ? (long long)l4_rx - ev_l4 : 0;
    const long long d_phy = (act && crc) ? (long long)tb : 0;
    const int c_crc = (act && crc) ? 1 : 0;
    const long long mac_tot = s_st.mac_total + warp_incl_scan(d_mac, lane);
    const long long l4_tot = s_st.l4_total + warp_incl_scan(d_l4, lane);
    const long long cum = s_st.cum_phy_bytes + warp_incl_scan(d_phy, lane);
    const int crc_incl = warp_incl_scan(c_crc, lane);
    const int ndi = s_st.ndi ^ ((crc_incl - c_crc) & 1);
    __syncwarp();
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
      // ring updates: the last lane mapping to a slot wins (only matters for W < 32)
      if (lane + W >= len) {
        sv.mac_ring[n % W] = mac_rx;
        sv.l4_ring[n % W] = l4_rx;
      }
      if (P.policy == ARCHES_POLICY_TREE && lane + WD >= len) {
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
    }
    // carry the chunk totals (last active lane)
    const int last = len - 1;
    const long long mac_c = __shfl_sync(0xffffffffu, mac_tot, last);
    const long long l4_c = __shfl_sync(0xffffffffu, l4_tot, last);
    const long long cum_c = __shfl_sync(0xffffffffu, cum, last);
    const int ndi_next = __shfl_sync(0xffffffffu, ndi ^ c_crc, last);
    __syncwarp();
    __threadfence_block();
    if (lane == 0) {
      s_st.mac_total = mac_c;
      s_st.l4_total = l4_c;
      s_st.cum_phy_bytes = cum_c;
      s_st.ndi = ndi_next;
      s_st.next_slot = n0 + len;
    }
    __syncwarp();
    // ---------------- 3. dApp decision at the chunk's last slot
    if (decide) {
      __shared__ double s_feat[ARCHES_FEATURES];
      const int64_t nd = n0 + len - 1;
      const int rows = (int)min((long long)WD, (long long)nd + 1);
      if (lane < ARCHES_FEATURES) {
        double acc = 0.0;
        for (int i = 0; i < rows; ++i) {
          const int64_t p = nd - rows + 1 + i;  // oldest first
          acc = xadd(acc, sv.feat[(size_t)(p % WD) * ARCHES_FEATURES + lane]);
        }
        s_feat[lane] = xdiv(acc, (double)rows);
      }
      __syncwarp();
      if (lane == 0) {
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
      __syncwarp();
    }
    s0 += len;
  }
  if (lane == 0) *sv.h = s_st;
}
