#!/bin/bash
python -m paper_2411_09009_b200._build > /dev/null 2>&1
for p in 50 74 100; do
  echo "== P=$p: $(CCE_STREAM_P=$p REPS=5 timeout 100 python scripts/stream_pass_probe.py gemma2-2b de:0,dc:0 2>&1 | grep 'gemma' | awk '{print $3, $4, $5, $6, $7}' | tr '\n' ' ')"
done
for pq in "44 56" "40 50" "36 44" "50 50"; do
  set -- $pq
  echo "== P=$1 QC=$2: $(CCE_STREAM_P=$1 CCE_STREAM_QC=$2 REPS=5 timeout 100 python scripts/stream_pass_probe.py gemma2-2b both:0,both:1 2>&1 | grep 'gemma' | awk '{print $2, $4, $6, $8}' | tr '\n' ' ')"
done
