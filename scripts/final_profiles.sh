#!/bin/bash
# launch list + default bench of the final build (profiles/r2)
out=gpurun_out/final_prof; mkdir -p $out
python -m paper_2411_09009_b200._build > /dev/null 2>&1 || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv \
   python bench.py --steps 1 --warmup 2 --no-cpu-baseline --no-e2e > $out/launches.log 2>&1
python scripts/launch_summary.py $out/launches.csv > $out/launches_summary.txt 2>&1; head -12 $out/launches_summary.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"cce_stream3_kernel" -s 1 -c 1 -o $out/stream3 \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $out/ncu_stream.log 2>&1
python scripts/ncu_summary.py $out/stream3.ncu-rep $out/stream3.json 2>&1 | tail -1
