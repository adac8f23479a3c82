"""bench.py's JSON-line contract (the driver parses it): the reference arm on
CPU (one rank and the self-launched two-rank form), our arm on the GPU at a
reduced size, one rank and two ranks sharing the GPU over gloo."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout, env=None):
    e = dict(os.environ)
    e.pop("WORLD_SIZE", None)
    e.update(env or {})
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                         capture_output=True, text=True, timeout=timeout, env=e)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0]), out


BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config", "e2e", "cpu_baseline"}


def test_reference_arm_line():
    d, _ = _run(["--impl", "reference", "--steps", "2", "--warmup", "1", "--n-prb", "12"], 600)
    assert BASE_KEYS <= set(d), BASE_KEYS - set(d)
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "slots/s"
    assert d["cpu_baseline"]["kind"] in ("port", "reference") and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["steps"] == 2 and "a step = one slot" in d["cpu_baseline"]["sample"]
    assert d["config"]["n_prb"] == 12 and "workload" in d["config"]


def test_reference_arm_self_launches_two_ranks():
    """`--gpus 2` outside torchrun re-launches under torch.distributed.run; rank 0
    alone prints, describing the 2-rank job (the config names 2 cells)."""
    d, _ = _run(["--gpus", "2", "--impl", "reference", "--steps", "1", "--warmup", "1",
                 "--n-prb", "12", "--n-ant", "2"], 600)
    assert d["n_gpus"] == 2 and d["config"]["cells"] == 2
    assert d["config"]["parallelism"].startswith("dp2")


def test_config_dicts_identical_in_both_arms():
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    a = bench.parse([])
    assert bench.workload(a, 1)["workload"].startswith("B:")
    assert bench.workload(bench.parse(["--n-prb", "52", "--policy", "tree"]), 1)["workload"].startswith("A:")
    assert bench.workload(bench.parse(["--cells", "64", "--layers", "2"]), 8)["workload"].startswith("C:")
    assert bench.workload(bench.parse(["--mode", "policy-stress"]), 1)["workload"].startswith("D:")
    assert bench.workload(bench.parse(["--n-ant", "64", "--layers", "4"]), 1)["workload"].startswith("E:")
    # sharding: 64 cells x 2 layers over 8 ranks -> 16 streams per rank, seeds disjoint
    a = bench.parse(["--cells", "64", "--layers", "2"])
    seeds = [bench.rank_streams(a, r, 8) for r in range(8)]
    assert all(len(s) == 16 for s in seeds)
    assert len(set(x for s in seeds for x in s)) == 128


@pytest.mark.gpu
def test_our_arm_line():
    d, _ = _run(["--steps", "4", "--warmup", "3", "--slots", "32", "--no-cpu-baseline",
                 "--latency-slots", "5"], 900)
    assert BASE_KEYS | {"roofline", "gpu_launches", "clocks"} <= set(d)
    assert d["value"] > 0 and d["higher_is_better"] is True and d["scaling"] == "weak"
    r = d["roofline"]
    assert r["bound"] == "hbm" and 0 < r["frac"] < 1 and r["peak"] > 0
    assert d["gpu_launches"] == 6 * d["steps"]
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["clocks"]["sm_mhz"] > 0


@pytest.mark.gpu
def test_our_arm_two_ranks_on_one_gpu():
    """The multi-GPU command form (--gpus 2 -> torchrun, cells sharded, one
    reduction) with both ranks on the one GPU through the gloo backend."""
    d, _ = _run(["--gpus", "2", "--steps", "3", "--warmup", "3", "--slots", "16", "--n-prb", "52",
                 "--latency-slots", "0"], 900, env={"ARCHES_DIST_BACKEND": "gloo"})
    assert d["n_gpus"] == 2 and d["config"]["cells"] == 2
    assert d["units_per_step"] == 2 * 16 and d["streams_per_rank"] == 1
    assert d["value"] > 0 and d["cpu_baseline"] is None


@pytest.mark.gpu
def test_policy_stress_line():
    d, _ = _run(["--mode", "policy-stress", "--steps", "20", "--warmup", "3",
                 "--no-cpu-baseline"], 600)
    assert d["config"]["cells"] == 1024 and d["unit"] == "decisions/s"
    assert d["us_per_boundary"] > 0 and d["value"] == pytest.approx(1024 / (d["us_per_boundary"] * 1e-6),
                                                                   rel=1e-6)


@pytest.mark.gpu
def test_config_a_tree_line():
    d, _ = _run(["--n-prb", "52", "--policy", "tree", "--steps", "3", "--warmup", "3",
                 "--slots", "64", "--no-cpu-baseline", "--latency-slots", "5"], 900)
    assert d["config"]["workload"].startswith("A:") and d["value"] > 0
