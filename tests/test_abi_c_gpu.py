"""The C ABI from plain C++ (Option C): the programs in tests/abi_c/ include only
include/cce_b200.h and link libcce_b200.so.  abi_caller: forward + merge against a
double-precision log-sum-exp, and the error channel.  abi_train: the memory="fast" training path
(compaction, vocabulary order, sorted copy, tile-recording forward, kept backward) against
double-precision loss, dE and dC.  abi_train_stream: the default bounded path (per-group forward,
streamed backward) against the same."""
import os
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
PKG = ROOT / "paper_2411_09009_b200"


PROGRAMS = {"abi_caller": "abi caller ok", "abi_train": "abi training path ok",
            "abi_train_stream": "abi bounded training path ok"}


def _build(tmp_path, name):
    exe = tmp_path / name
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    cmd = [nvcc, "-O2", "-std=c++17", "-Wno-deprecated-gpu-targets", "-I", str(ROOT / "include"), str(ROOT / "tests" / "abi_c" / f"{name}.cpp"),
           "-o", str(exe), "-L", str(PKG), "-lcce_b200", f"-Xlinker=-rpath={PKG}"]
    subprocess.run(cmd, check=True, capture_output=True, text=True, timeout=300)
    return exe


@pytest.mark.parametrize("name", sorted(PROGRAMS))
def test_c_caller_builds_against_header(tmp_path, name):
    """CPU: each program compiles and links against the header and the library alone."""
    if not (PKG / "libcce_b200.so").exists():
        pytest.skip("libcce_b200.so not built")
    assert _build(tmp_path, name).exists()


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(PROGRAMS))
def test_c_caller_runs(cuda_device, tmp_path, name):
    exe = _build(tmp_path, name)
    res = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stdout + res.stderr
    assert PROGRAMS[name] in res.stdout
