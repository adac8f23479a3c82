/*
 * arches.h -- C ABI of the B200-native ARCHES uplink channel-estimation hot path.
 *
 * The reference (`/root/reference/pkg/src/ranswitch`, pure Python) has no FFI;
 * its drop-in boundary is the Python call surface that `Pipeline.run_slot`
 * (phy_pipeline.py:422-493) and `harness.execute_run` (harness.py:174-231)
 * bind by name.  Each entry point below names the reference
 * function(s) it replaces.  All pointers are DEVICE pointers unless a
 * parameter says "host".  Complex values are interleaved float2 (complex64);
 * scalars, features and accumulators are fp64.  No entry point allocates on
 * the hot path: callers own every buffer (sizes via arches_*_bytes).  Every
 * call returns an ARCHES_* status; arches_last_error() gives the thread-local
 * message.  A plan lives on the device that was current at arches_plan_create
 * (its tables, and the internal streams of the executors) and must be used
 * with that device current.  Threading: the per-call entry points (K1, K2, K4,
 * K5, compat forms) only read the plan and may be called from several threads;
 * the executors (arches_run_batch, arches_run_batch_async, arches_join) also
 * use the plan's internal streams / pipeline state, so one thread at a time
 * per plan for those.  Work is enqueued on the caller's cudaStream_t
 * (NULL = legacy).
 *
 * Device layouts (unit u = stream * n_slots + slot; a stream is one
 * single-layer DMRS port of one cell; A antennas, T symbols, D DMRS symbols,
 * N = 12*n_prb subcarriers, M = N/2 comb positions):
 *   y        [u][A][T][N]   received grid, frequency-contiguous rows
 *   tx       [u][T][N]      known transmitted grid (genie, equaliser SINR)
 *   pilots   [stream][M][D] unit-magnitude DMRS pilots
 *   h_mmse   [u][A][D][N]   MMSE expert output
 *   h_ai     [u][A][D][N]   AI-expert (delay-truncation denoiser) output
 */
#ifndef ARCHES_H_
#define ARCHES_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* arches_stream_t; /* == cudaStream_t */

/* status codes: 1:1 with validation.py:9-26 plus CUDA failures */
#define ARCHES_OK 0
#define ARCHES_E_CONFIG 1    /* ConfigurationError */
#define ARCHES_E_CONTRACT 2  /* ContractViolation */
#define ARCHES_E_ESTIMATOR 3 /* EstimatorError */
#define ARCHES_E_STATE 4     /* PipelineStateError */
#define ARCHES_E_CUDA 5      /* CUDA runtime error */

#define ARCHES_MAX_ANT 64
#define ARCHES_MAX_DMRS 4
#define ARCHES_MAX_SYM 14
#define ARCHES_MAX_BINS 64 /* analysis bins: max(truncation, noise_guard, 8) */
#define ARCHES_MAX_MCS 32
#define ARCHES_MAX_TREE_NODES 64
#define ARCHES_MAX_PENDING 8

/* arches_params.flags: force the CUDA-core forms (same results; used by the
 * parity tests to cover the fallback kernels on geometries that would pick the
 * tensor-core ones) */
#define ARCHES_FLAG_NO_TC_K1 0x1 /* K1: CUDA-core comb analysis instead of tcgen05 */
#define ARCHES_FLAG_NO_TC_K2 0x2 /* K2: FFMA synthesis/equaliser instead of tcgen05 */
/* the `tx` argument of arches_run_batch / arches_run_batch_async /
 * arches_experts_equalize / arches_perturb_mmse is the packed QPSK wire format
 * ([u][n_tiles][T][32] bytes, arches_pack_qpsk) instead of the complex64 grid:
 * K2 reads 2 bits per RE (results identical).  Requires the tensor-core K2 over
 * one antenna group with the NR 0/5/10 DMRS pattern (n_ant 1, 2 or 4). */
#define ARCHES_FLAG_TX_PACKED 0x4

enum { ARCHES_EXEC_CONCURRENT = 0, ARCHES_EXEC_SELECTED_ONLY = 1 };
enum { ARCHES_POLICY_ORACLE = 0, ARCHES_POLICY_FIXED = 1, ARCHES_POLICY_TREE = 2 };
enum { ARCHES_TRIGGER_POLICY = 0, ARCHES_TRIGGER_FAILSAFE = 1, ARCHES_TRIGGER_ORACLE = 2,
       ARCHES_TRIGGER_FIXED = 3 };

/* SlotGeometry (radio_scene.py:30-63) */
typedef struct arches_geom {
  int32_t n_ant;
  int32_t n_prb;
  int32_t n_sym;
  int32_t n_dmrs;
  int32_t dmrs_symbols[ARCHES_MAX_DMRS];
  double slot_duration_us;
} arches_geom;

/* PipelineConfig (phy_pipeline.py:353-374) + MMSE prior (ScenarioConfig.
 * assumed_delay_spread) + Dapp/LatencyModel (dapp_control.py:26-68) */
typedef struct arches_params {
  int32_t noise_guard;          /* estimate_noise_var guard (expert_bank.py:199) */
  int32_t truncation;           /* denoiser taps (expert_bank.py:182) */
  int32_t mmse_block_prbs;      /* mmse_estimate block (expert_bank.py:154,166) */
  int32_t window_length;        /* MAC/LCID4 throughput windows */
  double assumed_delay_spread;  /* MMSE PDP prior */
  double ridge;                 /* RIDGE, expert_bank.py:19 */
  double sinr_cap_db;
  double lcid4_fraction;
  double lcid4_jitter;
  double crc_margin_db;
  double crc_scale_db;
  int32_t mac_header_bytes;
  int32_t n_mcs;
  double mcs_threshold_db[ARCHES_MAX_MCS];
  int32_t mcs_qam[ARCHES_MAX_MCS];
  double mcs_rate[ARCHES_MAX_MCS];
  int32_t exec_mode;            /* ARCHES_EXEC_* */
  int32_t policy;               /* ARCHES_POLICY_* */
  int32_t fixed_mode;           /* policy == FIXED */
  int32_t decision_period_slots;
  int32_t dapp_window_slots;
  int32_t flags;                /* ARCHES_FLAG_* (0 = fastest applicable kernels) */
  int64_t decision_delay_ns;    /* LatencyModel.decision_delay_ns() */
  int64_t failsafe_timeout_ns;  /* DappConfig.timeout_ns() */
  uint64_t crc_purpose_key;     /* blake2b-64("crc"), rng.py:17-21 */
} arches_params;

/* depth-limited tree node (switch_policy.py:63-98); feature < 0 = leaf */
typedef struct arches_tree_node {
  int32_t feature;
  int32_t left;
  int32_t right;
  int32_t label;
  double threshold;
} arches_tree_node;

typedef struct arches_tree {
  int32_t n_nodes;
  int32_t reserved;
  arches_tree_node nodes[ARCHES_MAX_TREE_NODES];
} arches_tree;

/* per unit telemetry of BOTH experts; index 0 = AI (ExpertId.AI), 1 = MMSE */
typedef struct arches_telemetry {
  double sigma2_hat;            /* estimate_noise_var */
  double abs_mean[2];           /* mean |H| (run_slot :454) */
  double rsrp[2];               /* mean |H|^2 (run_slot :455) */
  double sinr_db[2];            /* equalize (phy_pipeline.py:253-279) */
  int32_t mcs[2];
  int32_t tb_bytes[2];
  int32_t num_cb[2];
  int32_t crc[2];
  int32_t mac_rx[2];
  int32_t lcid4_rx[2];
} arches_telemetry;

/* KpmRecord (phy_pipeline.py:291-310) + the slot outcome extras */
typedef struct arches_kpm {
  int64_t slot_index;
  double phy_throughput;
  double rsrp;
  double code_rate;
  double snr_db;
  double mac_throughput;
  double lcid4_throughput;
  double est_abs_mean;
  int32_t mcs_index;
  int32_t pdu_length;
  int32_t ndi;
  int32_t qam_order;
  int32_t num_cb;
  int32_t tb_size;
  int32_t mac_rx_bytes;
  int32_t lcid4_rx_bytes;
  int32_t mode;                 /* active expert of the slot (1 MMSE, 0 AI) */
  int32_t crc_pass;
} arches_kpm;

/* control message log entry (ControlMessage, phy_pipeline.py:43-52) */
typedef struct arches_message {
  int64_t decided_at_ns;
  int64_t deliverable_at_ns;
  int32_t mode;
  int32_t trigger;              /* ARCHES_TRIGGER_* */
} arches_message;

typedef struct arches_plan arches_plan;

/* ---- plan ---------------------------------------------------------- */
int arches_plan_create(const arches_geom* geom, const arches_params* params,
                       arches_plan** out);
int arches_plan_destroy(arches_plan* plan);
/* bytes of the caller-owned per-stream control state (windows, queues) */
size_t arches_state_bytes(const arches_plan* plan, int32_t n_streams);
/* scratch bytes for a batch of n_units stream-slots */
size_t arches_workspace_bytes(const arches_plan* plan, int32_t n_units);
/* reset control state of n_streams streams (ModeVar default 1, fixed-policy
 * force at t=0 as harness.py:186-189).  Replaces Pipeline.__init__ state. */
int arches_state_init(const arches_plan* plan, void* state, int32_t n_streams,
                      arches_stream_t stream);

/* ---- K1: LS front end + delay-domain analysis -----------------------
 * Replaces ls_estimate (expert_bank.py:96-116), estimate_noise_var (:199-214)
 * and the noise-dependent half of mmse_estimate/_wiener_matrix (:139-177) and
 * denoiser_estimate (:182-196): comb Y/X, 20-bin comb DFT, Parseval tail
 * power -> sigma2_hat, per-unit Wiener taps and AI taps (written to ws).
 * When seeds != NULL the last CTA of each unit also draws the unit's Philox
 * CRC uniform and LCID4 split (rng.py:24-34, phy_pipeline.py:221,347-350) for
 * run_batch's K2; slot numbering as in arches_experts_equalize. */
int arches_ls_analyze(const arches_plan* plan, int32_t n_streams, int32_t n_slots,
                      const void* y, const void* pilots, const uint64_t* seeds,
                      int64_t first_slot, const void* state, double* sigma2_hat, void* ws,
                      arches_stream_t stream);

/* ---- K2: expert synthesis + switch telemetry + equaliser ------------
 * Replaces the synthesis of mmse_estimate/denoiser_estimate, the |H| and
 * |H|^2 reductions of run_slot (:453-455) and equalize (:253-279) for BOTH
 * experts in one pass over y/tx, then (last CTA per unit) link adaptation,
 * transport block, Philox CRC and LCID4 split for both candidates
 * (phy_pipeline.py:192-222,462-470).  Writes h_mmse, h_ai, tel.  Slot index of
 * unit (stream, s) = first_slot + s, or, when first_slot < 0, the stream's
 * device-resident next_slot (from `state`) + s -- graph-replayable. */
int arches_experts_equalize(const arches_plan* plan, int32_t n_streams, int32_t n_slots,
                            const void* y, const void* tx, const double* noise_var,
                            const uint64_t* seeds, int64_t first_slot, const void* state,
                            void* h_mmse, void* h_ai, arches_telemetry* tel, void* ws,
                            arches_stream_t stream);

/* ---- K4: per-stream sequential KPM windows + control plane ----------
 * Replaces the order-dependent tail of run_slot (:471-488: windows, NDI,
 * cumulative PHY rate), SwitchController.begin_slot (:123-139),
 * Dapp.on_indication + window_features + predict (dapp_control.py:85-120,
 * switch_policy.py:237-248), FailsafeMonitor (dapp_control.py:123-144) and
 * the oracle/fixed message sources of execute_run (harness.py:186-226).
 * regime may be NULL unless policy == ORACLE (1 = good).  Writes kpm (which
 * carries the switch predicate `mode` of every slot) and appends to msg_log
 * (capacity msg_cap per stream; msg_count[stream] is advanced). */
int arches_kpm_scan(const arches_plan* plan, int32_t n_streams, int32_t n_slots,
                    const arches_telemetry* tel, const int8_t* regime, const arches_tree* tree,
                    void* state, arches_kpm* kpm, arches_message* msg_log,
                    int32_t* msg_count, int32_t msg_cap, arches_stream_t stream);

/* Same contract and results as arches_kpm_scan, one thread walking every slot
 * of a stream (the literal restatement; the default scan is block-parallel).
 * Kept exported so parity tests can cross-check the two forms. */
int arches_kpm_scan_sequential(const arches_plan* plan, int32_t n_streams, int32_t n_slots,
                               const arches_telemetry* tel, const int8_t* regime,
                               const arches_tree* tree, void* state, arches_kpm* kpm,
                               arches_message* msg_log, int32_t* msg_count, int32_t msg_cap,
                               arches_stream_t stream);

/* The per-step hot path for one batch: RNG side products || K1 (+ finalize) ->
 * K2 -> K3 -> K4; first_slot < 0 takes the slot numbering from the device state
 * (CUDA-graph friendly).  The RNG kernel runs on an internal stream forked from
 * and joined back into `stream` (event fork/join, so it captures into a graph);
 * when the call returns, all work is ordered on `stream` as for the other
 * entry points.  seeds is required. */
int arches_run_batch(const arches_plan* plan, int32_t n_streams, int32_t n_slots,
                     int64_t first_slot, const void* y, const void* tx, const void* pilots,
                     const double* noise_var, const uint64_t* seeds, const int8_t* regime,
                     const arches_tree* tree, void* state, void* h_mmse, void* h_ai,
                     arches_telemetry* tel, arches_kpm* kpm, arches_message* msg_log,
                     int32_t* msg_count, int32_t msg_cap, void* ws, arches_stream_t stream);

/* Pipelined form of arches_run_batch for a sequence of batches (the slots of
 * consecutive steps).  The control tail of the batch -- RNG side products, K3
 * (per-unit telemetry + KPM candidates) and K4 (KPM scan / decision policy) --
 * runs on an internal stream of the plan and overlaps the next call's K1; the
 * heavy kernels (K1, K1 finalize, K2) stay on `stream`.  Results are identical
 * to arches_run_batch.  Ordering contract:
 *  - the outputs of the tail (tel, kpm, msg_log, msg_count, state) and the
 *    inputs it reads (regime, tree, seeds) belong to the library until
 *    arches_join(plan, stream) -- do not read or overwrite them before;
 *  - h_mmse / h_ai / y / tx / noise_var follow `stream` order as usual;
 *  - one thread at a time per plan; arches_run_batch joins a pending tail first;
 *  - a CUDA-graph capture must contain its arches_join;
 *  - plans whose K2 is the FFMA form (tiles straddling MMSE blocks, n_ant 3 or
 *    5-7, ARCHES_FLAG_NO_TC_K2) run the single-stream arches_run_batch order
 *    (that K2 finalises on `stream` and reads the tail's RNG products).
 * Same arguments as arches_run_batch. */
int arches_run_batch_async(const arches_plan* plan, int32_t n_streams, int32_t n_slots,
                           int64_t first_slot, const void* y, const void* tx, const void* pilots,
                           const double* noise_var, const uint64_t* seeds, const int8_t* regime,
                           const arches_tree* tree, void* state, void* h_mmse, void* h_ai,
                           arches_telemetry* tel, arches_kpm* kpm, arches_message* msg_log,
                           int32_t* msg_count, int32_t msg_cap, void* ws, arches_stream_t stream);
/* Order `stream` after every pending arches_run_batch_async tail of the plan
 * (no-op when none is pending). */
int arches_join(const arches_plan* plan, arches_stream_t stream);

/* Number of kernels one arches_run_batch / arches_run_batch_async call launches
 * for this plan (RNG, K1, the K1 finalize grid(s), K2, K3, K4; memsets and
 * event records not counted).  Benchmarks report it; no reference counterpart. */
int32_t arches_batch_kernels(const arches_plan* plan);

/* ---- K5: zero-gap switch, reference aliasing semantics ---------------
 * switch_select (phy_pipeline.py:81-91): for every unit whose kpm.mode == 1
 * copy the MMSE output into the AI (downstream) buffer; mode 0 is a no-op. */
int arches_switch_copy(const arches_plan* plan, int32_t n_units, const arches_kpm* kpm,
                       const void* h_mmse, void* h_ai, arches_stream_t stream);
/* single-buffer form: copy n complex values when *mode == 1 (device int) */
int arches_switch_copy_one(const int32_t* mode, const void* src, void* dst, size_t n,
                           arches_stream_t stream);

/* ---- downstream of the switch (after K4 fixed each slot's mode) ------
 * K6: x_hat of the SELECTED expert per unit (kpm.mode: 1 = h_mmse, 0 = h_ai --
 * the buffer switch_select leaves downstream), formed exactly like equalize()
 * (phy_pipeline.py:258-266: time interpolation, MRC num / (sum |h|^2 +
 * noise_var), every RE): x_hat[u][T][N] complex64 (NULL = skip); and max-log
 * LLRs log P(b=0)/P(b=1) for the slot's scheduled modulation (kpm.qam_order:
 * Gray QPSK / 16QAM / 64QAM, TS 38.211 s5.1.3-5.1.5) of the unbiased symbol
 * x_hat / beta, beta = den / (den + noise_var), noise variance noise_var / den:
 * llr[u][T][N][ARCHES_LLR_STRIDE] floats, bit i of the RE at [i], zero on pilot
 * REs and beyond qam_order (NULL = skip). */
#define ARCHES_LLR_STRIDE 6
int arches_downstream(const arches_plan* plan, int32_t n_units, const arches_kpm* kpm,
                      const void* h_mmse, const void* h_ai, const void* y,
                      const double* noise_var, void* x_hat, float* llr, arches_stream_t stream);

/* ---- Eq. 3 perturbation of the MMSE expert (perturbation_lab.py:92-98 +
 * the Pipeline.perturb hook, phy_pipeline.py:401,444-445) --------------
 * Run between arches_experts_equalize (K2 + K3) and arches_kpm_scan (K4) of a
 * batch: for every stream with rho[stream] != 0 the MMSE output gets
 * rho * mean|H_mmse| * CN(0,1) (CN from stream(seeds[stream], "inject", slot)
 * in the reference's (A, 1, N, D) element order), is written back into h_mmse,
 * re-equalised, and the MMSE candidate of tel (rsrp, SINR, MCS, TB, CRC, MAC
 * bytes) is re-derived; abs_mean[1] stays the pre-injection mean (the hook's
 * est_abs_mean).  rho == 0 streams are untouched.  tx complex64; slot
 * numbering as arches_experts_equalize. */
int arches_perturb_mmse(const arches_plan* plan, int32_t n_streams, int32_t n_slots,
                        int64_t first_slot, const double* rho, const uint64_t* seeds,
                        const void* state, const void* y, const void* tx, const double* noise_var,
                        void* h_mmse, arches_telemetry* tel, void* ws, arches_stream_t stream);

/* ---- exhaustive depth-2 tree training (switch_policy.py:173-234) ------
 * Scores root split candidates of a labelled dataset the way `train` does:
 * for candidate c (feature root_feature[c], threshold root_threshold[c];
 * feature -1 = no root split, the whole set is the "left" subset) the best
 * depth-1 tree of each side (`_best_depth1`: every feature, every midpoint
 * between consecutive distinct values of the SUBSET, first minimum per
 * feature, strictly better feature wins) and its total leaf impurity
 * (sum n * gini), fp64 in the reference's operation order.  The host picks
 * the first minimum over candidates in (feature, threshold) order.
 * xT[F][n] feature-major values; order[F][n] each column's stable ascending
 * argsort; y[n] labels 0/1. */
typedef struct arches_split_eval {
  double total;            /* left_total + right_total */
  double left_total, right_total;
  double left_threshold, right_threshold;
  int32_t left_feature, right_feature; /* -1: that side stays a leaf */
} arches_split_eval;
int arches_tree_eval_splits(const double* xT, const int32_t* order, const uint8_t* y, int32_t n,
                            int32_t n_features, const int32_t* root_feature,
                            const double* root_threshold, int32_t n_roots,
                            arches_split_eval* out, arches_stream_t stream);

/* ---- device-side slot synthesis (input generation) -----
 * The reference scene (rng.py:24-55, radio_scene.py:140-306, driven as
 * Pipeline.run_slot does, phy_pipeline.py:430-433,459) for n_streams cells x
 * n_slots consecutive slots: AR(1) TDL channel + log-normal shadow, delayed
 * interferer, pilots, QPSK data, Y = H X + sqrt(nv) W + sqrt(iv) H_i X_i -- every
 * Philox stream keyed and indexed as numpy does (bits exact; fp64 libm / DFT
 * rounding within ulps).  Per-stream AR(1) state lives in scene_state (zeroed =
 * slot 0).  regimes[2]: 0 = poor, 1 = good (the engine's regime codes); the
 * unit's regime[u] picks one.  shadow_z[u] = stream(seed, "shadow", slot).
 * standard_normal() (numpy's ziggurat; host-drawn, one per cell-slot).
 * Outputs y[u][A][T][N], tx[u][T][N] complex64, noise_var[u]. */
typedef struct arches_scene_regime {
  double noise_var;             /* ScenarioConfig.noise_var(n_ant) */
  double interference_var;      /* ScenarioConfig.interference_var() */
  double temporal_correlation;
  double shadow_sigma_db;
  double shadow_correlation;
} arches_scene_regime;
size_t arches_scene_state_bytes(const arches_plan* plan, int32_t n_streams);
size_t arches_scene_workspace_bytes(const arches_plan* plan, int32_t n_units);
/* pilot_sequence (radio_scene.py:233-237) of every stream: pilots[stream][M][D] */
int arches_scene_pilots(const arches_plan* plan, int32_t n_streams, const uint64_t* seeds,
                        void* pilots, arches_stream_t stream);
int arches_synthesize(const arches_plan* plan, int32_t n_streams, int32_t n_slots,
                      const uint64_t* seeds, const arches_scene_regime* regimes /* host [2] */,
                      const uint8_t* prb_mask /* device [2][n_prb] */,
                      const double* sqrt_pdp /* host [8] */, int32_t excess_delay,
                      const int8_t* regime, const double* shadow_z, const void* pilots,
                      void* scene_state, void* scene_ws, void* y, void* tx, double* noise_var,
                      arches_stream_t stream);

/* ---- packed QPSK transmit grids (host <-> device wire format) -------
 * The genie transmit grid the equaliser scores against is QPSK everywhere
 * (qpsk(), rng.py:50-55, pilots included: radio_scene.py:240-249), so it
 * crosses PCIe as 2-bit codes: tx_bits[u][n_tiles][T][32] bytes, n_tiles =
 * ceil(N / 128); the RE (symbol t, subcarrier k = 128 tile + j) is byte j / 4
 * of row t, bits 2 (j % 4) .. +1: bit 0 set = Re > 0, bit 1 set = Im > 0, value
 * ((2 b0 - 1) + i (2 b1 - 1)) * float(1/sqrt(2)) -- exactly the complex64 of
 * qpsk().  Pad codes (k >= N) are ignored.  K2 reads the complex64 grid
 * (decoding 2-bit codes in its issue-bound epilogue measured slower than the
 * 94 MB per 256 slots it would save), so unpack once per batch after the H2D.
 * arches_pack_qpsk sets *bad (device int, caller-zeroed) to 1 when any RE is
 * not exactly a qpsk() symbol. */
size_t arches_tx_bits_bytes(const arches_plan* plan, int32_t n_units);
int arches_pack_qpsk(const arches_plan* plan, int32_t n_units, const void* tx, void* tx_bits,
                     int32_t* bad, arches_stream_t stream);
int arches_unpack_qpsk(const arches_plan* plan, int32_t n_units, const void* tx_bits, void* tx,
                       arches_stream_t stream);

/* ---- per-call drop-in forms (compat layer) -------------------------- */
/* ls_estimate: materialise the comb-filled LS grid ls[u][A][D][N] */
int arches_ls_materialize(const arches_plan* plan, int32_t n_units, const void* y,
                          const void* pilots, void* ls, arches_stream_t stream);
/* estimate_noise_var / mmse_estimate / denoiser_estimate from an LS grid
 * ls[u][A][D][N]; which: 0 = noise var only, 1 = MMSE (noise_var_in[u] >= 0
 * overrides sigma2_hat), 2 = denoiser (general N-point analysis); OR-ing
 * ARCHES_EXPERT_OUT_C128 makes `out` complex128 (fp64 synthesis, the
 * reference's output dtype) instead of complex64 */
#define ARCHES_EXPERT_OUT_C128 0x100
int arches_expert_from_ls(const arches_plan* plan, int32_t n_units, int32_t which,
                          const void* ls, const double* noise_var_in, double* sigma2_hat,
                          void* out, void* ws, arches_stream_t stream);
/* equalize(rx, est, noise_var, tx): est[u][A][D][N]; writes sinr_db[u] and,
 * when x_hat != NULL, x_hat[u][T][N] */
int arches_equalize(const arches_plan* plan, int32_t n_units, const void* y, const void* est,
                    const void* tx, const double* noise_var, double* sinr_db,
                    double* abs_mean, double* rsrp, void* x_hat, void* ws,
                    arches_stream_t stream);
/* window_features: column means of rows[n_rows][10] (sequential fp64 sum) */
int arches_window_features(const double* rows, int32_t n_rows, double* out,
                           arches_stream_t stream);
/* predict: labels[i] for x[n][n_features] */
int arches_tree_predict(const arches_tree* tree, const double* x, int32_t n, int32_t n_features,
                        int32_t* labels, arches_stream_t stream);

/* ---- host helpers (no GPU required) ---------------------------------- */
const char* arches_last_error(void);
const char* arches_version(void);
/* stream(seed, "crc", slot).random() (rng.py:24-34, phy_pipeline.py:221) */
double arches_host_crc_uniform(uint64_t seed, uint64_t purpose_key, uint64_t slot);
/* _lcid4_jitter(slot) (phy_pipeline.py:347-350) */
double arches_host_lcid4_jitter(uint64_t slot);
/* blake2b-64 of an arbitrary byte string (rng.py:17-21) */
uint64_t arches_host_blake2b64(const void* data, size_t len);
/* analysis bins the plan computes per (a, d) */
int32_t arches_plan_bins(const arches_plan* plan);
/* 1 if a CUDA device is usable from this process */
int32_t arches_device_available(void);

#ifdef __cplusplus
}
#endif
#endif /* ARCHES_H_ */
