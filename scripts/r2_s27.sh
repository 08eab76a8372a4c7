#!/bin/bash
out=gpurun_out/r2s27; mkdir -p $out
python -m paper_2411_09009_b200._build > $out/build.log 2>&1 || { tail $out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --deselect tests/test_baseline_parity_gpu.py > $out/pytest_gpu.log 2>&1; echo "exit $?" >> $out/pytest_gpu.log
grep -E "FAILED|passed|failed|exit" $out/pytest_gpu.log | tail -25
