#!/bin/bash
out=gpurun_out/full1; mkdir -p $out
python -m paper_2411_09009_b200._build > $out/build.log 2>&1 || exit 1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $out/pytest_gpu.log 2>&1; echo "exit $?" >> $out/pytest_gpu.log
grep -E "^FAILED|passed|failed|exit" $out/pytest_gpu.log | tail -8
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke exit $?"; tail -2 $out/smoke.log
timeout 600 python bench.py > $out/bench.log 2>&1; tail -c 600 $out/bench.log
