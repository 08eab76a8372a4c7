#!/bin/bash
out=gpurun_out/r2s25; mkdir -p $out
python -m paper_2411_09009_b200._build > $out/build.log 2>&1 || { tail $out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --deselect tests/test_baseline_parity_gpu.py -x > $out/pytest_gpu.log 2>&1; echo "exit $?" >> $out/pytest_gpu.log
grep -E "FAILED|Error|passed|failed|exit" $out/pytest_gpu.log | tail -15
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $out/bench.log 2>&1; echo "exit $?" >> $out/bench.log
tail -c 1500 $out/bench.log
