#!/bin/bash
python -m paper_2411_09009_b200._build > /dev/null 2>&1 || exit 1
for p in 36 50 74; do
  echo "P=$p: $(CCE_STREAM_P=$p REPS=5 timeout 200 python scripts/stream_pass_probe.py gemma2-2b de:1,dc:1 2>&1 | grep gemma | awk '{print $3,$4,$5}' | tr '\n' ' ')"
done
echo "default both: $(REPS=5 timeout 200 python scripts/stream_pass_probe.py gemma2-2b both:1 2>&1 | grep gemma)"
