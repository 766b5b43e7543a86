"""bench.py's contract on the CPU: the reference arm (the CPU oracle, BASELINE has no code to
install) prints one JSON line with the driver's keys; our arm refuses to run without a GPU
(no CPU fallback)."""
import json
import os
import subprocess
import sys

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
        "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "impl",
        "cpu_baseline", "e2e"}


def _bench(*argv, timeout=300):
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *argv], cwd=ROOT,
                          capture_output=True, text=True, timeout=timeout)


@pytest.mark.parametrize("workload", ["8192f32", "2048f64"])
def test_reference_arm_prints_one_line(workload):
    p = _bench("--impl", "reference", "--workload", workload, "--steps", "3", "--warmup", "3",
               "--reference-seconds", "3")
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert KEYS <= set(d), KEYS - set(d)
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["config"]["workload"]


def test_warmup_floor():
    p = _bench("--impl", "reference", "--steps", "3", "--warmup", "2")
    assert p.returncode != 0 and "warmup" in (p.stderr + p.stdout)


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_our_arm_needs_a_gpu():
    p = _bench("--steps", "3", "--warmup", "3", "--no-oracle", "--no-e2e", timeout=120)
    assert p.returncode != 0
    assert not [ln for ln in p.stdout.splitlines() if ln.startswith("{")]


def test_context_measurements_run_after_the_parity_check():
    """The same-bytes copy / graph-replay context writes into the timed output buffers, so
    it must run after the parity check of ours_arm (an r02 ordering bug made every R = 1
    workload report MISMATCH although the kernels were exact)."""
    import inspect
    import bench
    src = inspect.getsource(bench.ours_arm)
    assert src.index('parity = ("bit-exact vs oracle"') < src.index("live_ceiling_context(")
