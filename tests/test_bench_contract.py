"""bench.py host logic (CPU): the algorithmic work counts behind every reported
TFLOP/s and MUFU figure, and the reference arm's JSON line (the fp64 oracle timed
on the host, the one arm that runs without a GPU)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def _brute_pairs(S, causal, wl, wr):
    i = np.arange(S)[:, None]
    j = np.arange(S)[None, :]
    ok = np.ones((S, S), bool)
    if causal:
        ok &= j <= i
    if wl >= 0:
        ok &= i - j <= wl
    if wr >= 0:
        ok &= j - i <= wr
    return int(ok.sum())


@pytest.mark.parametrize("S,var", [
    (257, dict()), (257, dict(causal=True)), (300, dict(causal=True, window=(63, 0))),
    (300, dict(window=(10, 20))), (128, dict(window=(0, 0))), (1, dict(causal=True)),
])
def test_allowed_pairs_matches_brute_force(S, var):
    wl, wr = var.get("window", (-1, -1))
    assert bench.allowed_pairs(S, var) == _brute_pairs(S, var.get("causal", False), wl, wr)


def test_baseline_workload_flops():
    # C2a 1.0995 TFLOP, C2b 0.5499, C3 1.6494, C4 (i) 137.4 GFLOP, (ii)/(iii) 68.75
    def flops(name):
        _, B, Hq, _, S, D, var = bench.WORKLOADS[name]
        return 4.0 * D * bench.allowed_pairs(S, var) * B * Hq
    assert flops("mha") == pytest.approx(1.0995e12, rel=1e-4)
    assert flops("mha_causal") == pytest.approx(0.5499e12, rel=1e-3)
    assert flops("gqa_window") == pytest.approx(1.6494e12, rel=1e-4)
    assert flops("var_scaled_dot") == pytest.approx(137.4e9, rel=1e-3)
    assert flops("var_alibi_causal") == pytest.approx(68.75e9, rel=1e-3)


@pytest.mark.timeout(300)
def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "3"], capture_output=True, text=True, timeout=280, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["metric"] == bench.METRIC
    assert line["warmup"] >= 3 and line["value"] > 0 and line["higher_is_better"] is True
    cb = line["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["sample"] and cb["value"] == line["value"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    assert line["config"]["workload"].startswith("mha")
