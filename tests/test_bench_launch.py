"""bench.py's multi-rank entry point: `--gpus N` outside torchrun launches N ranks itself, and a
run whose WORLD_SIZE disagrees with --gpus refuses to report a number."""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def test_gpus_n_relaunches_under_torchrun(monkeypatch):
    import bench

    calls = []
    monkeypatch.setattr(bench.subprocess, "call", lambda cmd: calls.append(cmd) or 0)
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "5", "--warmup", "3"])
    bench.main()
    assert len(calls) == 1
    cmd = calls[0]
    assert cmd[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"]
    assert "--nproc-per-node=4" in cmd and "127.0.0.1" in cmd
    assert cmd[-6:] == ["--gpus", "4", "--steps", "5", "--warmup", "3"]


def test_reference_arm_needs_no_launcher(monkeypatch, capsys):
    import bench

    monkeypatch.setattr(bench.subprocess, "call", lambda cmd: pytest.fail("relaunched"))
    monkeypatch.setenv("RANK", "1")  # a non-zero rank of the reference arm exits without work
    monkeypatch.setattr(sys, "argv", ["bench.py", "--impl", "reference", "--gpus", "2"])
    bench.main()
    assert capsys.readouterr().out == ""


@pytest.mark.gpu
def test_two_rank_bench_on_one_gpu(cuda_device):
    """The N-rank path end to end on one device (gloo, a functional check, not a number):
    one JSON line, n_gpus 2, vocab-parallel."""
    env = dict(os.environ, CCE_BENCH_BACKEND="gloo", CCE_BENCH_SAME_DEVICE="1")
    env.pop("WORLD_SIZE", None)
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--steps", "2", "--warmup", "3",
                          "--config", "gpt2", "--no-cpu-baseline", "--no-e2e"],
                         capture_output=True, text=True, env=env, timeout=600, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, res.stdout
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["config"]["parallelism"] == "vocab2"
    assert line["value"] > 0
    assert "comm_nranks=2" in res.stderr
