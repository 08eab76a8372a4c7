#!/bin/bash
python -m paper_2411_09009_b200._build > /dev/null 2>&1
for env in "CCE_STREAM_NOPDL=1" "CCE_STREAM_NOPDL=2" "CCE_STREAM_NOPDL=3"; do
  echo "== $env"
  env $env CCE_STREAM_RING=4096 REPS=2 timeout 60 python scripts/stream_pass_probe.py small de:0,de:0,de:0 2>&1 | grep "small\|timed" | head -4
done
