"""bench.py's driver contract on the CPU: --gpus N never silently runs fewer
GPUs, the CPU sample windows cover the whole index range, and the reference
arm prints its JSON line."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_gpus_more_than_visible_fails_loudly():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                        "--steps", "1", "--warmup", "3"], capture_output=True, text=True,
                       timeout=300, env={**os.environ, "CUDA_VISIBLE_DEVICES": ""})
    assert r.returncode == 2, r.stdout + r.stderr
    assert "only 0 CUDA device" in r.stdout


def test_world_size_mismatch_is_an_error():
    env = {**os.environ, "WORLD_SIZE": "1", "RANK": "0", "LOCAL_RANK": "0"}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4"],
                       capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode != 0
    assert "WORLD_SIZE=1" in r.stderr


def test_cpu_windows_span_the_range():
    import bench

    w = bench.windows(1 << 28, 1 << 20)
    assert len(w) == bench.CPU_WINDOWS
    assert w[0][0] == 0 and w[-1][0] >= (1 << 28) * (bench.CPU_WINDOWS - 1) // bench.CPU_WINDOWS
    assert all(c == (1 << 20) // bench.CPU_WINDOWS for _, c in w)
    assert all(a + c <= 1 << 28 for a, c in w)
    small = bench.windows(1 << 24, 1 << 24)
    assert sum(c for _, c in small) == 1 << 24  # the whole C1 range


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libqmcref.so")),
                    reason="reference build absent")
def test_reference_arm_prints_its_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--steps", "1", "--warmup", "0"], capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "reference"
    assert line["e2e"]["h2d_bytes_per_step"] == 0
