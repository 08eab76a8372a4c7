#!/bin/bash
python -m paper_2411_09009_b200._build > /dev/null 2>&1
for p in 30 50 74 100 118; do
  echo "== P=$p: $(CCE_STREAM_P=$p REPS=5 timeout 100 python scripts/stream_pass_probe.py gemma2-2b de:0,dc:0 2>&1 | grep 'gemma' | awk '{print $3, $4, $5}' | tr '\n' ' ')"
done
