"""The qmc::-shaped C++ wrapper (include/qmcgpu.hpp) compiles against the
C-ABI and, on a GPU, reproduces the reference's golden checksums."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2307_15584_b200")


def _build(tmp_path):
    exe = str(tmp_path / "wrapper_test")
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "wrapper_test.cpp"), "-L", PKG, "-lqmcgpu",
                    "-Wl,-rpath," + PKG, "-o", exe], check=True)
    return exe


def test_wrapper_compiles(tmp_path):
    assert os.path.exists(_build(tmp_path))


def test_wrapper_host_calls(tmp_path):
    """Host-side wrapper calls (tables, loaders, enumerations, errors) run
    without a GPU."""
    r = subprocess.run([_build(tmp_path), "--host"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_wrapper_runs_on_gpu(tmp_path, golden):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    exe = _build(tmp_path)
    r = subprocess.run([exe, golden["sobol_f32_65536x32_fnv"],
                        golden["render64_spp16_fnv"]["pixel-shifted-lattice/kahan"],
                        str(torch.cuda.device_count())],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
