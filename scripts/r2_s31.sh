#!/bin/bash
out=gpurun_out/r2s31; mkdir -p $out
python -m paper_2411_09009_b200._build > $out/build.log 2>&1 || { tail $out/build.log; exit 1; }
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv \
   python bench.py --steps 1 --warmup 2 --no-cpu-baseline --no-e2e > $out/launches.log 2>&1
python scripts/launch_summary.py $out/launches.csv > $out/launches_summary.txt 2>&1; head -40 $out/launches_summary.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=25 > $out/pytest_gpu.log 2>&1; echo "exit $?" >> $out/pytest_gpu.log
grep -E "FAILED|passed|failed|exit" $out/pytest_gpu.log | tail -25
grep -A30 "slowest" $out/pytest_gpu.log | head -30
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $out/bench.log 2>&1; echo "exit $?" >> $out/bench.log
tail -c 2500 $out/bench.log
