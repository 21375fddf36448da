"""bench.py contract on CPU: the reference arm (the reference's own stepper from
oracle/_ref with the CPU physics) prints one JSON line with the keys the
driver reads, on the same metric/unit as the GPU arm.  The GPU arm itself is
exercised by the GPU round (it needs a B200)."""
import json
import os
import subprocess
import sys

import pytest

import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_reference_arm_json_line():
    out = subprocess.run(
        [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "C1",
         "--steps", "1", "--warmup", "0", "--sample-n", "6"],
        capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["unit"] == "cell-updates/s" and line["higher_is_better"] is True
    assert line["value"] > 0 and line["e2e"]["value"] == line["value"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    cb = line["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and cb["value"] == line["value"]
    assert "workload" in line["config"]


def test_gpus_n_without_gpus_fails_loudly():
    """--gpus N > 1 outside a launcher starts N ranks itself, and refuses when
    fewer than N GPUs are visible (no silent one-GPU run)."""
    import torch
    if torch.cuda.device_count() >= 2:
        pytest.skip("GPUs visible")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1",
                          "--warmup", "1"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode != 0
    assert "--gpus 2 but only" in out.stderr


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_reference_arm_relaunches_ranks():
    """The reference arm with --gpus 2: bench.py starts two ranks under
    torch.distributed.run; rank 0 alone measures and prints, with n_gpus 2."""
    out = subprocess.run(
        [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
         "--config", "C1", "--steps", "1", "--warmup", "0", "--sample-n", "6"],
        capture_output=True, text=True, timeout=600, cwd=ROOT,
        env=dict(os.environ, MASTER_ADDR="127.0.0.1"))
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    line = json.loads(lines[0])
    assert line["impl"] == "reference" and line["n_gpus"] == 2
