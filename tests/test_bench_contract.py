"""bench.py's JSON line keeps the driver's contract: the B200 arm on a GPU,
the reference arm (oracle/_ref, CPU) anywhere the reference was built."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def _run(*args, timeout=600):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, r.stdout  # exactly one JSON line on stdout
    return json.loads(lines[0])


def test_reference_arm_line(ref):
    d = _run("--impl", "reference", "--workload", "c1_planted_plp", "--steps", "1", "--warmup", "0")
    assert d["impl"] == "reference" and d["unit"] == "edges/s" and d["value"] > 0
    for k in ("metric", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling", "config"):
        assert k in d
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert set(d["config"]) == CONFIG_KEYS


CONFIG_KEYS = {"workload", "desc", "algo", "seed", "n", "m", "entries"}


def test_default_workload_is_c3():
    """The headline is the largest single-GPU config (BASELINE.json configs[2])."""
    sys.path.insert(0, ROOT)
    import bench
    assert bench.parse.__code__ and "c3_rmat24_plp" in bench.WORKLOADS
    import argparse
    old = sys.argv
    try:
        sys.argv = ["bench.py"]
        assert bench.parse().workload == "c3_rmat24_plp"
    finally:
        sys.argv = old


def test_gpus_n_spawns_ranks(ref):
    """--gpus 2 outside torchrun re-launches itself with 2 ranks; rank 0 alone
    prints (the reference arm: other ranks exit without work)."""
    d = _run("--impl", "reference", "--gpus", "2", "--workload", "t0_planted_plp", "--steps", "1", "--warmup", "0")
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["config"]["workload"] == "t0_planted_plp"


@pytest.mark.gpu
def test_b200_arm_line():
    d = _run("--workload", "c1_planted_plp", "--steps", "3", "--warmup", "3", "--no-cpu-baseline")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches", "roofline", "cpu_baseline", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["value"] > 0
    assert d["config"]["workload"] == "c1_planted_plp" and set(d["config"]) == CONFIG_KEYS
    ref_line = _run("--impl", "reference", "--workload", "c1_planted_plp", "--steps", "1", "--warmup", "0")
    assert ref_line["config"] == d["config"]  # same workload, same keys and values in both arms
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r, k
    assert r["bound"] == "hbm" and 0 < r["frac"] < 1 and r["kernels"]
    assert r["share_of_step"] <= 1.0  # the family is timed as it runs in the step: never longer than it
    c = d["clocks"]
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(c)
