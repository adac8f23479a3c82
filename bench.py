#!/usr/bin/env python
"""Benchmark: UL channel-estimation slots/s (273 PRB, 4 RX) on B200.

BASELINE.json metric "UL ch-est slots/sec (273 PRB, 4 RX) at 1/2/4/8 B200; p99
per-slot latency", workload configs[1] (config B): one cell per GPU, 273 PRB,
4 RX, 1 layer, good/poor regimes alternating every slot so the oracle policy
flips the expert every slot (concurrent execution, mode applied at the next
boundary).

A step = one pass of the hot path (K1 LS + delay-domain analysis on tcgen05 ->
K1 finalize (sigma2, taps) -> K2 experts + switch telemetry + equaliser on
tcgen05 -> K3 KPM candidates -> K4 KPM windows / control plane; RNG side
products on a side stream) over a batch of S consecutive slots of each of the
rank's streams.  A stream is one single-layer DMRS port of one cell.

Multi-GPU: one process per GPU.  `--gpus N` without a torchrun
environment re-launches itself under `torch.distributed.run` with N ranks.  The
job's cells are sharded contiguously over ranks (`dist.shard_cells`), every
(cell, layer) stream seeded `dist.cell_seed(1000, cell * layers + layer)`; no
collective on the data path, one `dist.reduce_metrics` (max time, summed units)
at the end: weak scaling.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--slots S]
                  [--cells C] [--layers L] [--n-prb P] [--n-ant A]
                  [--policy oracle|tree] [--mode pipeline|policy-stress]
                  [--impl ours|reference]

Workloads (BASELINE.json configs):
  B (default)  one cell per rank, 273 PRB, 4 RX
  A            --n-prb 52 --policy tree       (depth-2 tree, default dApp 100/100)
  C            --cells 8 --layers 2 --slots 16 per GPU (64 cells over 8 GPUs: --cells 64)
  D            --mode policy-stress           (K4 only: 1024 cells per slot boundary)
  E            --n-ant 64 --layers 4 --slots 8
Prints ONE JSON line (rank 0).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "UL ch-est slots/sec (273 PRB, 4 RX)"
UNIT = "slots/s"
DEFAULT_TREE = os.path.join(ROOT, "tests", "golden", "tree_52prb.txt")  # trained by the reference
CLOCK_REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
                 0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
                 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
                 0x100: "display_clock_setting"}


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--slots", type=int, default=256, help="slots per step per stream")
    ap.add_argument("--n-prb", type=int, default=273)
    ap.add_argument("--n-ant", type=int, default=4)
    ap.add_argument("--cells", type=int, default=0, help="cells in the job (default: 1 per rank)")
    ap.add_argument("--layers", type=int, default=1, help="layer ports per cell (independent streams)")
    ap.add_argument("--policy", default="oracle", choices=["oracle", "tree"])
    ap.add_argument("--tree", default=DEFAULT_TREE)
    ap.add_argument("--mode", default="pipeline", choices=["pipeline", "policy-stress"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--latency-slots", type=int, default=400)
    ap.add_argument("--tx", default="packed", choices=["packed", "complex"],
                    help="resident genie-tx format: 2-bit QPSK codes read by K2 "
                         "(ARCHES_FLAG_TX_PACKED, n_ant 1/2/4; other plans fall back to the grid), "
                         "or the complex64 grid")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--sequential", action="store_true",
                    help="one CUDA graph per step, no cross-batch pipeline (arches_run_batch)")
    a = ap.parse_args(argv)
    if a.mode == "policy-stress" and a.cells == 0:
        a.cells = 1024
    return a


# ------------------------------------------------------------------ workload
def job_cells(a, world):
    return a.cells or world


def workload(a, world):
    """The `config` dict -- identical in both arms (it names the workload only)."""
    cells = job_cells(a, world)
    if a.mode == "policy-stress":
        name = (f"D: telemetry + policy stress, {cells} cells per slot boundary (K4 only: KPM "
                "windows, dApp window features over 100 slots, depth-2 tree, decision every slot)")
        return {"workload": name, "cells": cells, "window_slots": 100, "decision_period_slots": 1,
                "policy": "tree", "parallelism": f"dp{world} (cells sharded by rank)"}
    tag = ("A" if a.n_prb == 52 and a.policy == "tree" else
           "E" if a.n_ant > 4 else "C" if a.layers > 1 or cells > world else "B")
    name = (f"{tag}: {cells} cell(s) x {a.layers} layer(s) over {world} GPU(s), {a.n_prb} PRB, "
            f"{a.n_ant} RX, good/poor alternating every slot, {a.policy} policy, concurrent experts")
    return {"workload": name, "n_prb": a.n_prb, "n_ant": a.n_ant, "cells": cells,
            "layers": a.layers, "slots_per_step": a.slots, "policy": a.policy,
            "exec_mode": "concurrent", "parallelism": f"dp{world} (cells sharded by rank)"}


def metric_name(a) -> str:
    if a.mode == "policy-stress":
        return "policy decisions/sec (1024 cells per slot boundary)"
    if a.n_prb == 273 and a.n_ant == 4:
        return METRIC
    return f"UL ch-est slots/sec ({a.n_prb} PRB, {a.n_ant} RX, per single-layer stream)"


# ------------------------------------------------------------------ launcher
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def relaunch(argv, n):
    """`--gpus N` outside torchrun: one process per GPU via torch.distributed.run."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}",
           os.path.abspath(__file__), *argv]
    return subprocess.run(cmd, cwd=ROOT).returncode


# ------------------------------------------------------------------ CPU (oracle)
def _ref_module():
    """The reference's own code when staged (baseline/_ref, tools/fetch_ref.py): kind
    "reference"; otherwise the pinned oracle port (oracle/cpu_bench.py): kind "port"."""
    from oracle.ref_bench import staged
    return ("oracle.ref_bench", "reference") if staged() else ("oracle.cpu_bench", "port")


def _cpu_run(procs: int, slots: int, threads: int, extra):
    """Run `procs` CPU-baseline processes concurrently; returns list of per-proc JSON."""
    env = dict(os.environ)
    for k in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
        env[k] = str(threads)
    env["CUDA_VISIBLE_DEVICES"] = ""
    ps = [subprocess.Popen([sys.executable, "-m", _ref_module()[0], "--slots", str(slots),
                            "--seed", str(i), *extra], cwd=ROOT, env=env,
                           stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)
          for i in range(procs)]
    out = []
    for p in ps:
        o, e = p.communicate()
        if p.returncode != 0:
            raise RuntimeError(f"{_ref_module()[0]} failed: {e[-2000:]}")
        out.append(json.loads(o.strip().splitlines()[-1]))
    return out


def cpu_reference_rate(a, warm, timed):
    """Best of (i) one process using every core for BLAS and (ii) one single-
    threaded process per core on independent cells.  Returns
    ((slots/s, cores, sample text, seconds per step), alternatives)."""
    cores = os.cpu_count() or 1
    procs = min(cores, 64)
    extra = ["--n-prb", str(a.n_prb), "--n-ant", str(a.n_ant), "--policy", a.policy]
    what = ("the reference's own Pipeline.run_slot loop (staged ranswitch)"
            if _ref_module()[1] == "reference" else "the pinned oracle port")
    if a.policy == "tree":
        extra += ["--tree", a.tree]
    res = {}
    r = _cpu_run(procs, warm + timed, 1, extra)
    t = max(sum(x["per_slot_s"][warm:]) for x in r)
    res["multiproc"] = (procs * timed / t, procs, f"{what}: {procs} procs x 1 BLAS thread x {timed} "
                        f"timed slots each (+{warm} warm-up); a step = one slot per process",
                        t / timed)
    r = _cpu_run(1, warm + timed, cores, extra)
    t = sum(r[0]["per_slot_s"][warm:])
    res["blas"] = (timed / t, cores, f"{what}: 1 proc x {cores} BLAS threads x {timed} timed slots "
                   f"(+{warm} warm-up); a step = one slot", t / timed)
    best = max(res.values(), key=lambda v: v[0])
    return best, res


def cpu_policy_rate(a, warm, timed):
    """Config D on the host: Dapp.on_indication for a sample of cells per boundary,
    one process per core; decisions/s for the whole job's cells."""
    cores = os.cpu_count() or 1
    sample = 16
    r = _cpu_run(cores, warm + timed, 1, ["--policy-stress", "--cells", str(sample),
                                          "--tree", a.tree])
    t = max(sum(x["per_boundary_s"][warm:]) for x in r)
    rate = cores * sample * timed / t           # cell-decisions per second
    return rate, cores, (f"{_ref_module()[0]}: {cores} procs x {sample} cells x {timed} boundaries "
                         f"(+{warm} warm-up); a step = one boundary of {sample} cells per process"), \
        t / timed


def run_reference_arm(a, rank, world):
    """The reference's CPU path (the pinned oracle port, oracle/cpu_bench.py) on
    the host cores, rank 0 only.  A step is a bounded sample of the workload:
    one slot (one boundary in policy-stress mode) per worker process; exactly
    `--steps` steps are timed after `--warmup` (at most 3) untimed ones."""
    if rank != 0:
        return
    K, W = a.steps, a.warmup
    wu = min(W, 3)
    if a.mode == "policy-stress":
        rate, cores, sample, s_per_step = cpu_policy_rate(a, wu, K)
        alts = None
    else:
        (rate, cores, sample, s_per_step), allres = cpu_reference_rate(a, wu, K)
        alts = {k: v[0] for k, v in allres.items()}
    line = {"metric": metric_name(a), "value": rate, "unit": UNIT if a.mode != "policy-stress"
            else "decisions/s", "n_gpus": world, "steps": K, "warmup": wu,
            "ms_per_step": 1000.0 * s_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "c128/f64", "data": "synthetic", "impl": "reference",
            "config": workload(a, world),
            "cpu_baseline": {"value": rate, "unit": UNIT, "cores": cores, "kind": _ref_module()[1],
                             "sample": sample, "alternatives": alts},
            "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ clocks
class ClockSampler:
    def __init__(self, gpu_index: int):
        self.samples, self.proc, self.gpu = [], None, gpu_index

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), "--query-gpu=clocks.sm,clocks.max.sm,"
                 "clocks_event_reasons.active,power.draw", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            try:
                self.samples.append((float(parts[0]), float(parts[1]), int(parts[2], 16),
                                     float(parts[3])))
            except (ValueError, IndexError):
                pass

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [s[0] for s in self.samples]
        mask = 0
        for s in self.samples:
            mask |= s[2]
        reasons = [n for b, n in CLOCK_REASONS.items() if mask & b and b != 0x1] or ["none"]
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(s[1] for s in self.samples),
                "reasons": reasons, "samples": len(sm),
                "power_w_max": max(s[3] for s in self.samples)}


def physical_gpu(torch):
    dev = torch.cuda.current_device()
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    return int(vis.split(",")[dev]) if vis else dev


# ------------------------------------------------------------------ host placement
def gpu_numa_bind(dev_index: int):
    """Bind this process to the CPUs of the GPU's NUMA node; returns the previous
    affinity (None if the topology is not visible)."""
    try:
        import torch
        pr = torch.cuda.get_device_properties(dev_index)
        bus = f"{pr.pci_domain_id:04x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
        node = int(open(f"/sys/bus/pci/devices/{bus}/numa_node").read().strip())
        if node < 0:
            return None
        cpus = set()
        for part in open(f"/sys/devices/system/node/node{node}/cpulist").read().strip().split(","):
            lo, _, hi = part.partition("-")
            cpus.update(range(int(lo), int(hi or lo) + 1))
        old = os.sched_getaffinity(0)
        cpus &= old
        if not cpus:
            return None
        os.sched_setaffinity(0, cpus)
        return old
    except Exception:
        return None


# ------------------------------------------------------------------ inputs
def make_inputs(n_prb, n_ant, S, seed):
    """One stream's S slots from the reference scene (bit-exact synthesis)."""
    from paper_2604_23397_b200.geometry import SlotGeometry, default_scenarios
    from paper_2604_23397_b200.scene import CellScene
    geo = SlotGeometry(n_ant=n_ant, n_prb=n_prb)
    scens = default_scenarios(seed, geo)
    regimes = ["good" if i % 2 == 0 else "poor" for i in range(S)]
    cs = CellScene(geo, scens, regimes[0])
    N, T, A = geo.n_sc, geo.n_sym, n_ant
    y = np.empty((S, A, T, N), np.complex64)
    tx = np.empty((S, T, N), np.complex64)
    nv = np.empty(S)
    for i, r in enumerate(regimes):
        s = cs.next_slot(r)
        y[i] = np.transpose(s.y, (0, 2, 1))
        tx[i] = s.tx.T
        nv[i] = s.noise_var
    reg = np.array([1 if r == "good" else 0 for r in regimes], np.int8)
    return geo, scens, cs.pilots, y, tx, nv, reg


def make_stream_inputs(n_prb, n_ant, S, seeds):
    """One scene per stream; stream-major unit order."""
    outs = [make_inputs(n_prb, n_ant, S, sd) for sd in seeds]
    geo, scens = outs[0][0], outs[0][1]
    pil = np.stack([o[2] for o in outs])
    cat = lambda i: np.concatenate([o[i] for o in outs])  # noqa: E731
    return geo, scens, pil, cat(3), cat(4), cat(5), cat(6)


def rank_streams(a, rank, world):
    """(cell, layer) streams of this rank and their seeds."""
    from paper_2604_23397_b200.dist import cell_seed, shard_cells
    cells = shard_cells(job_cells(a, world), rank, world)
    return [cell_seed(1000, c * a.layers + l) for c in cells for l in range(a.layers)]


# ------------------------------------------------------------------ ours
def run_ours(a, rank, world, backend):
    import torch
    from paper_2604_23397_b200 import _lib
    from paper_2604_23397_b200.config import ExecutionMode, PipelineConfig
    from paper_2604_23397_b200.dist import reduce_metrics
    from paper_2604_23397_b200.engine import ArchesPlan, SlotEngine
    from paper_2604_23397_b200.policy import from_text
    from paper_2604_23397_b200.scene import pack_qpsk

    dev = torch.device("cuda", torch.cuda.current_device())
    red_dev = dev if backend == "nccl" else None
    S, K, W = a.slots, a.steps, max(3, a.warmup)
    seeds = rank_streams(a, rank, world)
    C = len(seeds)
    geo, scens, pil, y, tx, nv, reg = make_stream_inputs(a.n_prb, a.n_ant, S, seeds)
    A, T, N, D = geo.n_ant, geo.n_sym, geo.n_sc, geo.n_dmrs
    tree = from_text(open(a.tree).read()) if a.policy == "tree" else None
    # --tx packed: tx resident as the packed QPSK wire format K2 reads (n_ant 1, 2, 4)
    packed = a.tx == "packed" and A in (1, 2, 4)
    plan = ArchesPlan(geo, scens["good"].assumed_delay_spread, PipelineConfig(),
                      ExecutionMode.CONCURRENT, a.policy, flags=_lib.FLAG_TX_PACKED if packed else 0)
    eng = SlotEngine(plan, C, S, tree=tree)
    eng.set_streams(pil, seeds)
    eng.load(y=y, tx=tx, noise_var=nv, regime=reg)
    U = C * S  # units (stream-slots) per step on this rank
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()

    # ---- warm-up (eager), then capture the step as a CUDA graph
    for _ in range(W):
        eng.run()
    eng.capture_graph()
    for _ in range(W):
        eng.run()
    clocks = ClockSampler(physical_gpu(torch))
    clocks.start()
    t_end = time.time() + 1.0   # sustained load so the sampler sees the clocks under load
    while time.time() < t_end:
        for _ in range(20):
            eng.run()
        torch.cuda.synchronize()

    # ---- timed region: exactly K steps.  Default: cross-batch pipeline (the
    # control tail of step n -- RNG, K3, K4 -- overlaps step n+1's K1 on the
    # plan's second stream, arches_run_batch_async), the K steps and the final
    # join captured as one CUDA graph.  --sequential: one CUDA graph per step.
    # Both are measured; the other one is reported as value_alt.
    def timed(pipelined):
        if pipelined:
            g = eng.capture_pipeline(K)
            eng.run_pipeline(g, K)  # warm replay (K >= W untimed steps)
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        if pipelined:
            eng.run_pipeline(g, K)
        else:
            for _ in range(K):
                eng.run()
        e1.record()
        barrier()
        return e0.elapsed_time(e1)

    pipelined = not a.sequential
    t_ms = timed(pipelined)
    clk = clocks.stop()
    t_alt = timed(not pipelined)
    t_max, units = reduce_metrics(t_ms, K * U, red_dev)
    t_alt_max, _ = reduce_metrics(t_alt, K * U, red_dev)
    value = units / (t_max / 1000.0)

    # ---- per-kernel times (eager, events around each stage on the launch stream)
    L = _lib.lib()
    st = torch.cuda.current_stream().cuda_stream
    ws = eng.ws
    reps = 10
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4 * reps)]
    for r in range(reps):
        ev[4 * r].record()
        _lib.check(L.arches_ls_analyze(plan.handle, C, S, _lib.ptr(eng.y), _lib.ptr(eng.pilots),
                                       None, -1, _lib.ptr(eng.state), None, _lib.ptr(ws), st))
        ev[4 * r + 1].record()
        _lib.check(L.arches_experts_equalize(plan.handle, C, S, _lib.ptr(eng.y), _lib.ptr(eng.tx),
                                             _lib.ptr(eng.noise_var), _lib.ptr(eng.seeds), -1,
                                             _lib.ptr(eng.state), _lib.ptr(eng.h_mmse),
                                             _lib.ptr(eng.h_ai), _lib.ptr(eng.tel), _lib.ptr(ws), st))
        ev[4 * r + 2].record()
        _lib.check(L.arches_kpm_scan(plan.handle, C, S, _lib.ptr(eng.tel), _lib.ptr(eng.regime),
                                     _lib.ptr(eng.tree), _lib.ptr(eng.state), _lib.ptr(eng.kpm),
                                     _lib.ptr(eng.msg_log), _lib.ptr(eng.msg_count), eng.msg_cap, st))
        ev[4 * r + 3].record()
    torch.cuda.synchronize()
    k1 = np.mean([ev[4 * r].elapsed_time(ev[4 * r + 1]) for r in range(reps)])
    k2 = np.mean([ev[4 * r + 1].elapsed_time(ev[4 * r + 2]) for r in range(reps)])
    k4 = np.mean([ev[4 * r + 2].elapsed_time(ev[4 * r + 3]) for r in range(reps)])
    # algorithmic bytes per unit: y read once (8 A T N), both experts written
    # (2 x 8 A D N), the genie tx read once: 2-bit codes (n_tiles T 32 B) when
    # packed, else the complex64 grid (8 T N) = 8 N (20 A + 14)
    tx_bytes = -(-N // 128) * T * 32 if packed else 8 * T * N
    unit_bytes = 8 * N * A * (T + 2 * D) + tx_bytes
    pk_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    peaks = json.load(open(pk_path)) if os.path.exists(pk_path) else {"hbm_gbs": 6650.0}
    peak = float(peaks["hbm_gbs"])
    k2_gbs = U * unit_bytes / (k2 * 1e-3) / 1e9
    step_gbs = U * unit_bytes / (t_ms / K * 1e-3) / 1e9
    k1_bytes = 8 * N * A * D  # K1 reads the DMRS rows of y (both parities of each 32-byte sector)
    k1_gbs = U * k1_bytes / (k1 * 1e-3) / 1e9
    traffic, traffic_src = None, None
    tpath = os.path.join(ROOT, "profiles", "k2_dram_traffic.json")
    if os.path.exists(tpath):  # dram__bytes_read + write per K2 launch, from a committed ncu capture
        entries = json.load(open(tpath))
        for tj in entries if isinstance(entries, list) else [entries]:
            if (tj.get("n_prb") == a.n_prb and tj.get("n_ant") == A and tj.get("units") == U
                    and tj.get("tx", "complex") == ("packed" if packed else "complex")):
                traffic = tj["bytes_per_launch"]
                traffic_src = (f"committed ncu capture ({os.path.relpath(tpath, ROOT)}, "
                               f"{tj.get('captured', 'this config')}), not measured in this run")

    # ---- e2e through the public engine API: pinned host inputs -> H2D -> run -> D2H KPMs.
    # Pinned buffers are placed on the GPU's NUMA node (first touch by a thread
    # bound to it), as a PHY host process would run; affinity restored after.
    aff0 = gpu_numa_bind(torch.cuda.current_device())
    y_h = torch.from_numpy(y).pin_memory()
    # the transmit grids cross PCIe in the packed QPSK wire format (2 bits per RE,
    # expanded on the device by arches_unpack_qpsk inside load())
    tx_host = pack_qpsk(tx)
    tx_h = torch.from_numpy(tx_host).pin_memory()
    nv_h = torch.from_numpy(nv).pin_memory()
    reg_h = torch.from_numpy(reg).pin_memory()
    kpm_h = torch.empty(eng.kpm.numel(), dtype=torch.uint8).pin_memory()
    # double-buffered: stage() copies step n+1's inputs into the engine's idle input
    # set on its copy stream while step n runs (run_staged); every step's inputs
    # still cross PCIe inside the timed region
    for _ in range(2):
        eng.stage(y_h, tx_h, nv_h, reg_h)
        eng.run_staged()
        kpm_h.copy_(eng.kpm, non_blocking=True)
    torch.cuda.synchronize()
    barrier()
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record()
    eng._copy_stream.wait_stream(torch.cuda.current_stream())  # step 0's copy starts after e2
    eng.stage(y_h, tx_h, nv_h, reg_h)
    for k in range(K):
        eng.run_staged()
        kpm_h.copy_(eng.kpm, non_blocking=True)
        if k + 1 < K:
            eng.stage(y_h, tx_h, nv_h, reg_h)
    e3.record()
    barrier()
    te, e2e_units = reduce_metrics(e2.elapsed_time(e3), K * U, red_dev)
    recs = kpm_h.numpy().view(_lib.KPM_DTYPE)
    assert recs["slot_index"][-1] > 0 and set(np.unique(recs["mode"])) <= {0, 1}
    h2d = y.nbytes + tx_host.nbytes + nv.nbytes + reg.nbytes
    d2h = kpm_h.numel()
    if aff0 is not None:
        os.sched_setaffinity(0, aff0)

    # ---- per-slot latency: one slot per launch (graph), inputs resident
    lat = None
    if a.latency_slots > 0:
        eng1 = SlotEngine(plan, 1, 1, tree=tree)
        eng1.set_streams(pil[:1], seeds[:1])
        eng1.load(y=y[:1], tx=tx[:1], noise_var=nv[:1], regime=reg[:1])
        for _ in range(5):
            eng1.run()
        eng1.capture_graph()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(a.latency_slots)]
        torch.cuda.synchronize()
        for i, (b, e) in enumerate(evs):
            j = i % S
            eng1.y.copy_(eng.y[j:j + 1])   # next slot's grid (not timed)
            eng1.tx.copy_(eng.tx[j:j + 1])
            b.record()
            eng1.run()
            e.record()
        torch.cuda.synchronize()
        us = np.array([b.elapsed_time(e) * 1000.0 for b, e in evs])
        lat = {"p50_us": float(np.percentile(us, 50)), "p99_us": float(np.percentile(us, 99)),
               "max_us": float(us.max()), "slots": int(len(us)),
               "how": "1 slot of one stream per CUDA-graph launch (K1, K1 finalize, K2, K3, K4), "
                      "CUDA events, inputs in HBM"}
        # host-to-host: the slot's pinned y + packed tx -> H2D -> unpack + graph ->
        # D2H KPM record -> host holds the decision (wall clock, one slot at a time)
        y1 = [torch.from_numpy(y[j:j + 1]).pin_memory() for j in range(min(S, 16))]
        t1 = [torch.from_numpy(pack_qpsk(tx[j:j + 1])).pin_memory() for j in range(min(S, 16))]
        k1h = torch.empty(eng1.kpm.numel(), dtype=torch.uint8).pin_memory()
        h2h = []
        for i in range(a.latency_slots):
            j = i % len(y1)
            t0 = time.perf_counter()
            eng1.load(y=y1[j], tx=t1[j], non_blocking=True)
            eng1.run()
            k1h.copy_(eng1.kpm, non_blocking=True)
            torch.cuda.current_stream().synchronize()
            h2h.append((time.perf_counter() - t0) * 1e6)
        h2h = np.array(h2h[min(5, len(h2h) // 2):])   # first few: warm-up
        lat["host_to_host"] = {
            "p50_us": float(np.percentile(h2h, 50)), "p99_us": float(np.percentile(h2h, 99)),
            "max_us": float(h2h.max()), "slots": int(len(h2h)),
            "how": "wall clock per slot: pinned y (1 slot, complex64) + packed tx -> H2D -> "
                   "unpack + CUDA-graph step -> D2H KPM record -> stream sync"}

    line = None
    if rank == 0:
        cpu = None
        if world == 1 and not a.no_cpu_baseline:
            (rate, cores, sample, _), allres = cpu_reference_rate(a, 1, 2)
            cpu = {"value": rate, "unit": UNIT, "cores": cores, "kind": _ref_module()[1],
                   "sample": sample, "alternatives": {k: v[0] for k, v in allres.items()}}
        line = {
            "metric": metric_name(a), "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
            "warmup": W, "ms_per_step": t_max / K, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "c64/f64",
            "data": "synthetic (reference TDL scene, bit-exact; S-slot pool per stream replayed each step)",
            "config": workload(a, world),
            "units_per_step": units // K, "streams_per_rank": C,
            "tx_format": ("packed QPSK codes (2 bits/RE) read by K2" if packed
                          else "complex64 grid"),
            "l2": f"inputs {U * unit_bytes / 1e6:.0f} MB per step per GPU vs 126 MB L2 "
                  f"({'> L2, no flush' if U * unit_bytes > 126e6 else '< L2: NOT L2-cold'})",
            "executor": ("cross-batch pipeline: step n's RNG/K3/K4 overlap step n+1's K1 "
                         "(arches_run_batch_async; the K steps as one CUDA graph)") if pipelined else
                        "one CUDA graph per step (arches_run_batch)",
            "value_alt": {"value": units / (t_alt_max / 1000.0),
                          "executor": "one CUDA graph per step" if pipelined else "cross-batch pipeline"},
            "roofline": {"bound": "hbm", "achieved": k2_gbs, "peak": peak, "unit": "GB/s",
                         "frac": k2_gbs / peak, "traffic": traffic, "traffic_source": traffic_src,
                         "kernel": "k2_tc (+k3_finalize): expert synthesis on tcgen05 + switch "
                                   "telemetry + equaliser",
                         "algorithmic_bytes_per_unit": unit_bytes, "units_per_launch": U,
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst copy)",
                         "kernel_ms": {"k1_tc+finalize": k1, "k2_tc+k3": k2, "k4_kpm_scan_block": k4},
                         "k1": {"achieved": k1_gbs, "frac": k1_gbs / peak,
                                "algorithmic_bytes_per_unit": k1_bytes},
                         "step_gbs": step_gbs, "step_frac": step_gbs / peak},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_units / (te / 1000.0), "unit": UNIT,
                    "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                    "how": "pinned host y (complex64) + tx (packed QPSK wire format, 2 bits/RE) + "
                           "noise_var + regime -> H2D -> " + ("" if packed else "unpack + ") +
                           "run (eager, ordered executor) -> D2H KPM records, every step; "
                           "double-buffered: step n+1's H2D on a copy stream overlaps step n"},
            "latency": lat,
            "gpu_launches": plan.batch_kernels() * K,  # RNG, K1, K1 finalize(s), K2, K3, K4 per step
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    return line


def run_policy_stress(a, rank, world, backend):
    """Config D: K4 only for the job's cells (sharded by rank), one decision per
    cell per slot boundary over a 100-slot dApp window, depth-2 tree.  A step =
    one boundary (one arches_kpm_scan launch with n_slots = 1); the K steps are
    captured as one CUDA graph.  Telemetry = synthetic K3 records."""
    import torch
    from paper_2604_23397_b200 import _lib
    from paper_2604_23397_b200.config import DappConfig, ExecutionMode, PipelineConfig
    from paper_2604_23397_b200.dist import reduce_metrics, shard_cells
    from paper_2604_23397_b200.engine import ArchesPlan
    from paper_2604_23397_b200.geometry import SlotGeometry
    from paper_2604_23397_b200.policy import from_text, to_device_struct

    dev = torch.device("cuda", torch.cuda.current_device())
    red_dev = dev if backend == "nccl" else None
    C = len(shard_cells(job_cells(a, world), rank, world))
    K, W = a.steps, max(3, a.warmup)
    pcfg = PipelineConfig()
    plan = ArchesPlan(SlotGeometry(n_ant=4, n_prb=52), 1.25, pcfg, ExecutionMode.CONCURRENT,
                      "tree", DappConfig(decision_period_slots=1, window_length_slots=100))
    L = _lib.lib()
    tree = torch.frombuffer(bytearray(bytes(to_device_struct(from_text(open(a.tree).read())))),
                            dtype=torch.uint8).to(dev)
    rng = np.random.default_rng(rank)
    n_b = K + W + 100
    tel = np.zeros((n_b, C), dtype=_lib.TELEMETRY_DTYPE)     # one record per cell per boundary
    for e in (0, 1):
        tel["rsrp"][..., e] = rng.random((n_b, C)) + 0.5
        tel["abs_mean"][..., e] = rng.random((n_b, C))
        tel["sinr_db"][..., e] = rng.normal(10, 8, (n_b, C))
        tel["mcs"][..., e] = rng.integers(0, pcfg.mcs_table.n_mcs, (n_b, C))
        tel["tb_bytes"][..., e] = rng.integers(0, 3000, (n_b, C))
        tel["num_cb"][..., e] = 1
        tel["crc"][..., e] = rng.random((n_b, C)) < 0.7
        tel["mac_rx"][..., e] = np.where(tel["crc"][..., e], tel["tb_bytes"][..., e] - 3, 0)
        tel["lcid4_rx"][..., e] = (tel["mac_rx"][..., e] * 0.85).astype(np.int32)
    tel_d = torch.from_numpy(tel.view(np.uint8).copy()).to(dev).view(n_b, -1)
    state = torch.zeros(plan.state_bytes(C), dtype=torch.uint8, device=dev)
    kpm = torch.zeros(C * 104, dtype=torch.uint8, device=dev)
    cap = 8
    log = torch.zeros(C * cap * 24, dtype=torch.uint8, device=dev)
    cnt = torch.zeros(C, dtype=torch.int32, device=dev)
    _lib.check(L.arches_state_init(plan.handle, _lib.ptr(state), C, None))
    st = torch.cuda.current_stream()

    def boundary(b):
        _lib.check(L.arches_kpm_scan(plan.handle, C, 1, _lib.ptr(tel_d[b]), None, _lib.ptr(tree),
                                     _lib.ptr(state), _lib.ptr(kpm), _lib.ptr(log), _lib.ptr(cnt),
                                     cap, st.cuda_stream))

    for b in range(100 + W):              # fill the 100-slot windows, then warm up
        boundary(b)
    torch.cuda.synchronize()
    s2 = torch.cuda.Stream()
    s2.wait_stream(st)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s2):
        with torch.cuda.graph(g, stream=s2):
            for k in range(K):
                _lib.check(L.arches_kpm_scan(plan.handle, C, 1, _lib.ptr(tel_d[100 + W + k]), None,
                                             _lib.ptr(tree), _lib.ptr(state), _lib.ptr(kpm),
                                             _lib.ptr(log), _lib.ptr(cnt), cap, s2.cuda_stream))
    st.wait_stream(s2)
    g.replay()
    torch.cuda.synchronize()
    clocks = ClockSampler(physical_gpu(torch))
    clocks.start()
    t_end = time.time() + 1.0   # sustained load so the sampler sees the clocks under load
    while time.time() < t_end:
        for _ in range(20):
            g.replay()
        torch.cuda.synchronize()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    clk = clocks.stop()
    t_max, units = reduce_metrics(e0.elapsed_time(e1), K * C, red_dev)
    # e2e: each boundary's telemetry from pinned host memory, decisions (KPM mode) back
    tel_h = torch.from_numpy(tel.view(np.uint8).copy()).view(n_b, -1).pin_memory()
    kpm_h = torch.empty(C * 104, dtype=torch.uint8).pin_memory()
    stage = torch.empty_like(tel_d[0])
    torch.cuda.synchronize()
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record()
    for k in range(K):
        stage.copy_(tel_h[100 + W + k], non_blocking=True)
        _lib.check(L.arches_kpm_scan(plan.handle, C, 1, _lib.ptr(stage), None, _lib.ptr(tree),
                                     _lib.ptr(state), _lib.ptr(kpm), _lib.ptr(log), _lib.ptr(cnt),
                                     cap, st.cuda_stream))
        kpm_h.copy_(kpm, non_blocking=True)
    e3.record()
    torch.cuda.synchronize()
    te, _ = reduce_metrics(e2.elapsed_time(e3), K * C, red_dev)
    if rank == 0:
        cpu = None
        if world == 1 and not a.no_cpu_baseline:
            rate, cores, sample, _ = cpu_policy_rate(a, 1, 3)
            cpu = {"value": rate, "unit": "decisions/s", "cores": cores, "kind": _ref_module()[1],
                   "sample": sample}
        us_b = t_max / K * 1000.0
        line = {"metric": metric_name(a), "value": units / (t_max / 1000.0), "unit": "decisions/s",
                "n_gpus": world, "steps": K, "warmup": W, "ms_per_step": t_max / K,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic K3 telemetry records", "config": workload(a, world),
                "us_per_boundary": us_b,
                "roofline": {"bound": "latency", "achieved": None, "peak": None, "unit": "us",
                             "frac": None, "traffic": None,
                             "kernel": "k4_kpm_scan_block (one CTA per cell)",
                             "note": f"{us_b:.2f} us per boundary for {C} cells/GPU; the 100x10 "
                                     "fp64 window (8 KB per cell) is L2-resident"},
                "cpu_baseline": cpu,
                "e2e": {"value": units / (te / 1000.0), "unit": "decisions/s",
                        "h2d_bytes_per_step": C * 104, "d2h_bytes_per_step": C * 104},
                "gpu_launches": K, "clocks": clk}
        print(json.dumps(line), flush=True)


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    a = parse(argv)
    if "WORLD_SIZE" not in os.environ and a.gpus > 1:
        sys.exit(relaunch(argv, a.gpus))
    from paper_2604_23397_b200.dist import rank_world
    rank, world = rank_world()
    if a.impl == "reference":
        run_reference_arm(a, rank, world)
        return
    import torch
    backend = None
    if world > 1:
        import torch.distributed as dist
        local = int(os.environ.get("LOCAL_RANK", "0"))
        # one process per GPU; ARCHES_DIST_BACKEND=gloo is a test hook that lets
        # several ranks share one GPU (the reduction then goes via the host)
        backend = os.environ.get("ARCHES_DIST_BACKEND", "nccl")
        torch.cuda.set_device(local % torch.cuda.device_count())
        if backend == "nccl":
            os.environ.setdefault("NCCL_DEBUG", "INFO")          # init lines: ranks / transport
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
        else:
            dist.init_process_group(backend)
    if a.mode == "policy-stress":
        run_policy_stress(a, rank, world, backend)
    else:
        run_ours(a, rank, world, backend)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
