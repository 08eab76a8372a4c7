#!/bin/bash
python -m paper_2411_09009_b200._build > /dev/null 2>&1
for env in "CCE_STREAM_RING=4096" "CCE_STREAM_RING=512"; do
  echo "== $env"
  env $env REPS=3 timeout 60 python scripts/stream_pass_probe.py small de:0,de:0,both:0,both:1,dc:1 2>&1 | grep "small\|timed" | head -8
done
