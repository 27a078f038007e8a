"""bench.py's contract: the reference arm runs on the CPU and prints one
JSON line whose config object is the one our arm prints (CPU test); our
arm runs end to end on a small configuration with its parity check against
the oracle (GPU test)."""

import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT


def _run(args, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                         capture_output=True, text=True, timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_line_and_config():
    d = _run(["--impl", "reference", "--config", "0", "--steps", "2", "--warmup", "1"])
    assert d["impl"] == "reference" and d["unit"] == "queries/s" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "port"
    sys.path.insert(0, ROOT)
    import bench

    class A:
        config, scaling = 0, "weak"
    assert d["config"] == bench.config_block(A, 1)
    # config 3 defaults to strong scaling (one global batch split across GPUs)
    class B:
        config, scaling = 3, "strong"
    assert bench.config_block(B, 8)["spheres_per_job"] == 64 << 20


@pytest.mark.gpu
def test_our_arm_small_config_with_parity():
    d = _run(["--config", "0", "--steps", "5", "--warmup", "3", "--e2e-steps", "1",
              "--no-cpu-baseline"])
    assert d["parity"]["mismatches"] == 0 and d["parity"]["spheres"] == 1 << 20
    assert d["parity"]["boundary"] == d["parity"]["boundary_device_counter_rank_sum"]
    assert d["parity"]["tree"]["mismatches"] == 0
    assert d["gpu_launches"] > 0 and d["roofline"]["bound"] == "hbm"
    assert d["e2e"]["h2d_bytes_per_step"] == 16 << 20
