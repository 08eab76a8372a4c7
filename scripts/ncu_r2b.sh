#!/bin/bash
# final build: launch list of the default bench + ncu --set full of one forward group launch (37 tiles)
out=gpurun_out/ncu_r2b; mkdir -p $out
python -m paper_2411_09009_b200._build > /dev/null 2>&1 || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv \
   python bench.py --steps 1 --warmup 2 --no-cpu-baseline --no-e2e > $out/launches.log 2>&1
python scripts/launch_summary.py $out/launches.csv > $out/launches_summary.txt 2>&1; head -24 $out/launches_summary.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"cce_lse_kernel" -s 30 -c 1 -o $out/fwd_g2b \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $out/ncu_fwd.log 2>&1; echo "fwd exit $?"
python scripts/ncu_summary.py $out/fwd_g2b.ncu-rep $out/fwd_g2b.json 2>&1 | tail -1
