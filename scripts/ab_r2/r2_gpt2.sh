#!/bin/bash
python -m paper_2411_09009_b200._build > /dev/null 2>&1 || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/l.csv \
   python bench.py --config gpt2 --steps 1 --warmup 2 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python scripts/launch_summary.py /tmp/l.csv 2>&1 | head -14
for pq in "32 54" "40 50" "48 50" "32 44" "24 60"; do set -- $pq; echo "P=$1 QC=$2: $(CCE_STREAM_P=$1 CCE_STREAM_QC=$2 REPS=5 timeout 200 python scripts/stream_pass_probe.py gpt2 both:1 2>&1 | grep gpt2 | awk '{print $4, $5}')"; done
