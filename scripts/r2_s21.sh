#!/bin/bash
python -m paper_2411_09009_b200._build > /dev/null 2>&1
for pq in "50 50" "56 56" "60 50" "50 60" "64 56" "44 56" "56 64" "70 50"; do
  set -- $pq
  echo "== P=$1 QC=$2: $(CCE_STREAM_P=$1 CCE_STREAM_QC=$2 REPS=5 timeout 100 python scripts/stream_pass_probe.py gemma2-2b both:0,de:0,dc:0 2>&1 | grep 'gemma' | awk '{print $3, $4}' | tr '\n' ' ')"
done
