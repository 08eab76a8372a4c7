#!/bin/bash
python -m paper_2411_09009_b200._build > /dev/null 2>&1 || exit 1
for e in "X=1" "CCE_STREAM_DEBUG_DE=1" "CCE_STREAM_DEBUG_DE=2" "CCE_STREAM_DEBUG_DE=3" "CCE_STREAM_DEBUG_DE=15"; do
  echo "$e: $(env CCE_STREAM_P=74 $e REPS=5 timeout 200 python scripts/stream_pass_probe.py gemma2-2b de:1 2>&1 | grep gemma | awk '{print $4, $5, $6}')  both: $(env $e REPS=5 timeout 200 python scripts/stream_pass_probe.py gemma2-2b both:1 2>&1 | grep gemma | awk '{print $4, $5}')"
done
