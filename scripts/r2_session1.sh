#!/bin/bash
# round-2 first GPU session: new tests, full suite, bench, large-config forward profiles
out=gpurun_out/r2s1; mkdir -p $out
python -m paper_2411_09009_b200._build > $out/build.log 2>&1
timeout 1500 python -m pytest tests/test_advice_fixes_gpu.py tests/test_bench_launch.py tests/test_baseline_parity_gpu.py -m gpu -q -s -p no:cacheprovider > $out/pytest_new.log 2>&1; echo "exit $?" >> $out/pytest_new.log
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --deselect tests/test_baseline_parity_gpu.py > $out/pytest_gpu.log 2>&1; echo "exit $?" >> $out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $out/bench.log 2>&1; echo "exit $?" >> $out/bench.log
for cfg in gemma2-9b nemo-12b; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"cce_lse_kernel" -c 1 -o $out/fwd_$cfg \
    python bench.py --config $cfg --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $out/ncu_$cfg.log 2>&1; echo "exit $?" >> $out/ncu_$cfg.log
done
tail -n 5 $out/*.log
