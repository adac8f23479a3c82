// K4 helpers shared by the block form (k_control_block.cuh): warp scans and a
// register-resident pending-message queue.  The parallel K4 has the same
// semantics as k4_kpm_scan (k_control.cuh), restructured so only the control
// plane stays sequential:
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
