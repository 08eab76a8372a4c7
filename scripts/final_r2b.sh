#!/bin/bash
# final build: round-end check (GPU suite, smoke, bench, reference arm, 2-rank functional), launch
# list, ncu of one forward group launch, every head and variant
bash scripts/final_check.sh
out=gpurun_out/ncu_r2c; mkdir -p $out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv \
   python bench.py --steps 1 --warmup 2 --no-cpu-baseline --no-e2e > $out/launches.log 2>&1
python scripts/launch_summary.py $out/launches.csv > $out/launches_summary.txt 2>&1; head -14 $out/launches_summary.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"cce_lse_kernel" -s 25 -c 1 -o $out/fwd_g2b \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $out/ncu_fwd.log 2>&1; echo "fwd exit $?"
python scripts/ncu_summary.py $out/fwd_g2b.ncu-rep $out/fwd_g2b.json 2>&1 | tail -1
bash scripts/configs_r2.sh
