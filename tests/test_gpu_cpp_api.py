"""Runs the C++ conformance cases (tests/cpp/test_gpu_api.cpp, reference-test style) against
the C++ host API include/sparsefusion_gpu.hpp on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_cpp_api_conformance(gpu):
    exe = os.path.join(ROOT, "tests", "cpp", "_build", "test_gpu_api")
    # incremental: rebuilds the binary when sf_gpu.h / the wrapper / the library changed
    subprocess.run(["make", "-C", ROOT, "cpptests"], check=True, capture_output=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout
