#!/bin/bash
python -m paper_2411_09009_b200._build > /dev/null 2>&1
for env in "CCE_STREAM_RING=512" "CCE_STREAM_RING=1024" "CCE_STREAM_RING=2048" \
           "CCE_STREAM_RING=1024 CCE_STREAM_P=44 CCE_STREAM_QC=40" "CCE_STREAM_RING=1024 CCE_STREAM_P=40 CCE_STREAM_QC=36" \
           "CCE_STREAM_RING=1024 CCE_STREAM_P=50 CCE_STREAM_QC=36" "CCE_STREAM_RING=1024 CCE_STREAM_P=56 CCE_STREAM_QC=40"; do
  echo "== $env: $(env $env REPS=5 timeout 100 python scripts/stream_pass_probe.py gemma2-2b both:0,both:1 2>&1 | grep 'gemma' | awk '{print $2, $4}' | tr '\n' ' ')"
done
