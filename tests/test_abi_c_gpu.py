"""The C ABI from plain C++ (Option C): tests/abi_c/abi_caller.cpp includes only
include/cce_b200.h, links libcce_b200.so, runs the forward + merge on host-made bf16 inputs and
checks them against a double-precision log-sum-exp; then the error channel."""
import os
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
PKG = ROOT / "paper_2411_09009_b200"
SRC = ROOT / "tests" / "abi_c" / "abi_caller.cpp"


def _build(tmp_path):
    exe = tmp_path / "abi_caller"
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    cmd = [nvcc, "-O2", "-std=c++17", "-I", str(ROOT / "include"), str(SRC), "-o", str(exe),
           "-L", str(PKG), "-lcce_b200", f"-Xlinker=-rpath={PKG}"]
    subprocess.run(cmd, check=True, capture_output=True, text=True, timeout=300)
    return exe


def test_c_caller_builds_against_header(tmp_path):
    """CPU: the program compiles and links against the header and the library alone."""
    if not (PKG / "libcce_b200.so").exists():
        pytest.skip("libcce_b200.so not built")
    assert _build(tmp_path).exists()


@pytest.mark.gpu
def test_c_caller_runs(cuda_device, tmp_path):
    exe = _build(tmp_path)
    res = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "abi caller ok" in res.stdout
