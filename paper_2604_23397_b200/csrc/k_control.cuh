// K4 -- per-stream slot-ordered KPM derivation and control plane; K5 switch.
//
// K4 replaces the order-dependent tail of Pipeline.run_slot (phy_pipeline.py:
// 427,462-488), SwitchController.begin_slot/deliver/force_mode (:114-139),
// ThroughputWindow (:325-344), Dapp.on_indication + window_features
// (dapp_control.py:85-120), predict (switch_policy.py:237-248),
// FailsafeMonitor (dapp_control.py:123-144) and the message sources of
// harness.execute_run (harness.py:186-226).  Everything mode-independent was
// already computed for both candidate experts by K2; K4 selects the active
// candidate per slot and advances the small sequential state.  All fp64
// arithmetic is explicitly rounded in CPython's operation order.
#pragma once
#include "common.cuh"
#include "k_synth_eq.cuh"

struct StateView {
  StreamState* h;
  int32_t* mac_ring;
  int32_t* l4_ring;
  double* feat;  // [dapp_window][10]
};

__device__ __host__ inline StateView state_view(void* base, int stream, int window, int dapp_window) {
  unsigned char* p = reinterpret_cast<unsigned char*>(base) + (size_t)stream * state_stride_bytes(window, dapp_window);
  StateView v;
  v.h = reinterpret_cast<StreamState*>(p);
  v.mac_ring = reinterpret_cast<int32_t*>(p + sizeof(StreamState));
  v.l4_ring = v.mac_ring + window;
  v.feat = reinterpret_cast<double*>(v.l4_ring + window);
  return v;
}

// queues are kept canonical: entries at index >= n are zero (so the
// sequential and warp-parallel scans leave byte-identical state)
__device__ inline void queue_pop_front(PendingMsg* q, int32_t& n) {
  for (int i = 1; i < n; ++i) q[i - 1] = q[i];
  q[n - 1] = PendingMsg{0, 0, 0};
  --n;
}

__device__ inline void queue_insert(PendingMsg* q, int32_t& n, PendingMsg m) {
  // stable insertion by time (list.sort(key=...) keeps arrival order on ties)
  if (n >= ARCHES_MAX_PENDING) queue_pop_front(q, n);  // overflow: drop the earliest entry
  int pos = n;
  while (pos > 0 && q[pos - 1].at_ns > m.at_ns) {
    q[pos] = q[pos - 1];
    --pos;
  }
  q[pos] = m;
  ++n;
}



// ThroughputWindow.push (phy_pipeline.py:334-340) with the ring indexed by push
// count n (ring[n % W] holds the value pushed W slots ago until overwritten)
__device__ inline double window_push(int32_t* ring, int64_t& total, int64_t n, int window,
                                     int32_t nbytes, double slot_s) {
  total += nbytes;
  if (n >= window) total -= ring[n % window];
  ring[n % window] = nbytes;
  const int filled = (int)min((int64_t)window, n + 1);
  return xdiv(xdiv(xmul((double)total, 8.0), 1e6), xmul((double)filled, slot_s));
}

__device__ inline void log_message(arches_message* log, int32_t* count, int cap, int stream,
                                   int mode, int64_t decided, int64_t deliverable, int trigger) {
  if (!count) return;
  const int idx = count[stream];
  if (log && idx < cap) {
    arches_message m;
    m.decided_at_ns = decided;
    m.deliverable_at_ns = deliverable;
    m.mode = mode;
    m.trigger = trigger;
    log[(size_t)stream * cap + idx] = m;
  }
  count[stream] = idx + 1;
}

__device__ inline int tree_descend(const arches_tree* tree, const double* x) {
  int node = 0;
  for (int guard = 0; guard < ARCHES_MAX_TREE_NODES; ++guard) {
    const arches_tree_node& nd = tree->nodes[node];
    if (nd.feature < 0) return nd.label;
    node = (x[nd.feature] <= nd.threshold) ? nd.left : nd.right;
  }
  return 1;
}

struct K4Args {
  const arches_telemetry* tel;  // [u]
  const int8_t* regime;         // [u] 1 = good (oracle policy)
  const arches_tree* tree;
  void* state;
  arches_kpm* kpm;              // [u]
  arches_message* msg_log;
  int32_t* msg_count;
  int32_t msg_cap;
  int n_streams, n_slots;
};

__global__ void k4_kpm_scan(const PlanDev P, const K4Args a) {
  const int stream = blockIdx.x * blockDim.x + threadIdx.x;
  if (stream >= a.n_streams) return;
  StateView sv = state_view(a.state, stream, P.window_length, P.dapp_window);
  StreamState st = *sv.h;
  const int W = P.window_length, WD = P.dapp_window;
  const int64_t slot_ns = P.slot_ns;
  for (int s = 0; s < a.n_slots; ++s) {
    const int u = stream * a.n_slots + s;
    const int64_t n = st.next_slot;
    // ---- SwitchController.begin_slot
    const int64_t t0 = n * slot_ns;
    const int64_t cut = (P.exec_mode == ARCHES_EXEC_SELECTED_ONLY) ? t0 - slot_ns : t0;
    while (st.n_pending > 0 && st.pending[0].at_ns <= cut) {
      st.mode = st.pending[0].mode;
      queue_pop_front(st.pending, st.n_pending);
    }
    while (st.n_forced > 0 && st.forced[0].at_ns <= t0) {
      st.mode = st.forced[0].mode;
      queue_pop_front(st.forced, st.n_forced);
    }
    const int e = st.mode;  // 1 = MMSE, 0 = AI (telemetry index == expert id)
    const arches_telemetry& tl = a.tel[u];
    // ---- KPM derivation (run_slot :462-488)
    const int mcs = tl.mcs[e], tb = tl.tb_bytes[e], crc = tl.crc[e];
    const int pdu = max(tb - P.mac_header_bytes, 0);
    const int mac_rx = tl.mac_rx[e], l4_rx = tl.lcid4_rx[e];
    if (crc) st.cum_phy_bytes += tb;
    const double mac_t = window_push(sv.mac_ring, st.mac_total, n, W, mac_rx, P.slot_s);
    const double l4_t = window_push(sv.l4_ring, st.l4_total, n, W, l4_rx, P.slot_s);
    const double elapsed = xmul(xmul((double)(n + 1), P.slot_us), 1e-6);
    const double phy_t = xdiv(xdiv(xmul((double)st.cum_phy_bytes, 8.0), 1e6), elapsed);
    const int ndi = st.ndi;
    if (crc) st.ndi = 1 - st.ndi;
    arches_kpm r;
    r.slot_index = n;
    r.phy_throughput = phy_t;
    r.rsrp = tl.rsrp[e];
    r.code_rate = P.mcs_rate[mcs];
    r.snr_db = tl.sinr_db[e];
    r.mac_throughput = mac_t;
    r.lcid4_throughput = l4_t;
    r.est_abs_mean = tl.abs_mean[e];
    r.mcs_index = mcs;
    r.pdu_length = pdu;
    r.ndi = ndi;
    r.qam_order = P.mcs_qam[mcs];
    r.num_cb = tl.num_cb[e];
    r.tb_size = tb;
    r.mac_rx_bytes = mac_rx;
    r.lcid4_rx_bytes = l4_rx;
    r.mode = e;
    r.crc_pass = crc;
    a.kpm[u] = r;
    // ---- control traffic produced at the end of this slot (harness.py:203-226)
    const int64_t end_ns = (n + 1) * slot_ns;
    if (P.policy == ARCHES_POLICY_ORACLE) {
      const int want = (a.regime && a.regime[u]) ? 1 : 0;
      st.prev_msg_mode = st.last_msg_mode;
      if (want != st.last_msg_mode) {
        PendingMsg m = {end_ns, want, ARCHES_TRIGGER_ORACLE};
        queue_insert(st.pending, st.n_pending, m);
        st.last_msg_mode = want;
        log_message(a.msg_log, a.msg_count, a.msg_cap, stream, want, end_ns, end_ns, ARCHES_TRIGGER_ORACLE);
      }
    } else if (P.policy == ARCHES_POLICY_TREE) {
      // Dapp.on_indication: append the record's features to the window
      double* row = sv.feat + (size_t)(n % WD) * ARCHES_FEATURES;
      row[0] = phy_t;
      row[1] = (double)mcs;
      row[2] = (double)pdu;
      row[3] = (double)ndi;
      row[4] = r.rsrp;
      row[5] = r.snr_db;
      row[6] = mac_t;
      row[7] = l4_t;
      row[8] = (double)mac_rx;
      row[9] = (double)l4_rx;
      if (++st.since_decision >= P.decision_period) {
        st.since_decision = 0;
        double feat[ARCHES_FEATURES];
        const int rows = (int)min((int64_t)WD, n + 1);
        for (int f = 0; f < ARCHES_FEATURES; ++f) feat[f] = 0.0;
        for (int i = 0; i < rows; ++i) {
          const double* rw = sv.feat + (size_t)((n - rows + 1 + i) % WD) * ARCHES_FEATURES;
          for (int f = 0; f < ARCHES_FEATURES; ++f) feat[f] = xadd(feat[f], rw[f]);
        }
        for (int f = 0; f < ARCHES_FEATURES; ++f) feat[f] = xdiv(feat[f], (double)rows);
        const int mode = tree_descend(a.tree, feat);
        const int64_t decided = end_ns + P.decision_delay_ns;
        PendingMsg m = {decided, mode, ARCHES_TRIGGER_POLICY};
        queue_insert(st.pending, st.n_pending, m);
        st.last_delivery_ns = max(st.last_delivery_ns, decided);
        st.tripped = 0;
        log_message(a.msg_log, a.msg_count, a.msg_cap, stream, mode, decided, decided, ARCHES_TRIGGER_POLICY);
      }
      // FailsafeMonitor.check(end_ns, current mode)
      if (!st.tripped && end_ns - st.last_delivery_ns > P.failsafe_timeout_ns && st.mode != 1) {
        st.tripped = 1;
        PendingMsg f = {end_ns, 1, ARCHES_TRIGGER_FAILSAFE};
        queue_insert(st.forced, st.n_forced, f);
        log_message(a.msg_log, a.msg_count, a.msg_cap, stream, 1, end_ns, end_ns, ARCHES_TRIGGER_FAILSAFE);
      }
    }
    st.next_slot = n + 1;
  }
  *sv.h = st;
}

__global__ void k4_state_init(const PlanDev P, void* state, int n_streams) {
  const int stream = blockIdx.x * blockDim.x + threadIdx.x;
  if (stream >= n_streams) return;
  StateView sv = state_view(state, stream, P.window_length, P.dapp_window);
  StreamState st;
  memset(&st, 0, sizeof(st));
  st.mode = 1;
  st.last_msg_mode = 1;
  st.prev_msg_mode = 1;
  if (P.policy == ARCHES_POLICY_FIXED) {
    PendingMsg f = {0, P.fixed_mode, ARCHES_TRIGGER_FIXED};
    queue_insert(st.forced, st.n_forced, f);
  }
  *sv.h = st;
}

// K5: mode-predicated coalesced copy of the MMSE output into the AI buffer;
// grid-stride over every (unit, float4) of the batch (any number of units)
__global__ void k5_switch_copy(const arches_kpm* kpm, const float4* src, float4* dst,
                               size_t per_unit_f4, int n_units) {
  const size_t total = per_unit_f4 * (size_t)n_units;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const size_t u = i / per_unit_f4;
    if (__ldg(&kpm[u].mode) == 1) dst[i] = src[i];  // mode 0: no-op
  }
}

__global__ void k5_switch_copy_one(const int32_t* mode, const float2* src, float2* dst, size_t n) {
  if (*mode != 1) return;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

// window_features: sequential fp64 column sums in row order, then / n
__global__ void k_window_features(const double* rows, int n_rows, double* out) {
  const int f = threadIdx.x;
  if (f >= ARCHES_FEATURES) return;
  double s = 0.0;
  for (int i = 0; i < n_rows; ++i) s = xadd(s, rows[(size_t)i * ARCHES_FEATURES + f]);
  out[f] = xdiv(s, (double)n_rows);
}

__global__ void k_tree_predict(const arches_tree* tree, const double* x, int n, int nf,
                               int32_t* labels) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) labels[i] = tree_descend(tree, x + (size_t)i * nf);
}

// tx[u][T][N] complex64 -> packed QPSK codes [u][n_tiles][T][32] (ARCHES_FLAG_TX_PACKED);
// one thread per code byte (4 REs); any RE that is not exactly a qpsk() symbol
// raises *bad
__global__ void k_pack_qpsk(const PlanDev P, const float2* tx, unsigned char* bits, int32_t* bad,
                            size_t n_bytes) {
  const float q = __uint_as_float(ARCHES_QPSK_AMP);
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_bytes;
       i += (size_t)gridDim.x * blockDim.x) {
    const size_t row = i / ARCHES_TXB_ROW;  // (u, tile, t)
    const int jb = (int)(i - row * ARCHES_TXB_ROW);
    const int t = (int)(row % P.T);
    const size_t ut = row / P.T;
    const int tile = (int)(ut % P.n_tiles);
    const size_t u = ut / P.n_tiles;
    unsigned int code = 0;
    bool ok = true;
    for (int r = 0; r < 4; ++r) {
      const int k = tile * ARCHES_TILE + jb * 4 + r;
      if (k >= P.N) break;
      const float2 x = tx[(u * P.T + t) * (size_t)P.N + k];
      ok = ok && (x.x == q || x.x == -q) && (x.y == q || x.y == -q);
      code |= ((x.x > 0.f ? 1u : 0u) | (x.y > 0.f ? 2u : 0u)) << (2 * r);
    }
    bits[i] = (unsigned char)code;
    if (!ok) *bad = 1;
  }
}

// packed QPSK codes -> the complex64 grid tx[u][T][N]; one thread per code byte
__global__ void k_unpack_qpsk(const PlanDev P, const unsigned char* bits, float2* tx, size_t n_bytes) {
  const float q = __uint_as_float(ARCHES_QPSK_AMP);
  // 32-bit index arithmetic (callers stay below 2^32 code bytes: 1.4e6 units at 273 PRB)
  for (unsigned int i = blockIdx.x * blockDim.x + threadIdx.x; i < (unsigned int)n_bytes;
       i += gridDim.x * blockDim.x) {
    const unsigned int row = i / ARCHES_TXB_ROW;  // (u, tile, t)
    const int jb = (int)(i - row * ARCHES_TXB_ROW);
    const int t = (int)(row % (unsigned)P.T);
    const unsigned int ut = row / (unsigned)P.T;
    const int tile = (int)(ut % (unsigned)P.n_tiles);
    const size_t u = ut / (unsigned)P.n_tiles;
    const unsigned int code = bits[i];
    float2* dst = tx + (u * P.T + t) * (size_t)P.N;
    for (int r = 0; r < 4; ++r) {
      const int k = tile * ARCHES_TILE + jb * 4 + r;
      if (k >= P.N) break;
      const unsigned int c = code >> (2 * r);
      dst[k] = make_float2((c & 1u) ? q : -q, (c & 2u) ? q : -q);
    }
  }
}
