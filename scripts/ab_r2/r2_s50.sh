#!/bin/bash
python -m paper_2411_09009_b200._build > /dev/null 2>&1 || exit 1
for cfg in "X=1" "CCE_STREAM_DE=2" "CCE_STREAM_DE=2 CCE_STREAM_P=36 CCE_STREAM_QC=56" "CCE_STREAM_DE=2 CCE_STREAM_P=40 CCE_STREAM_QC=56" "CCE_STREAM_DE=2 CCE_STREAM_P=40 CCE_STREAM_QC=60" "X=1"; do
  echo "$cfg: $(env $cfg REPS=5 timeout 200 python scripts/stream_pass_probe.py gemma2-2b both:1 2>&1 | grep gemma | awk '{print $4, $5}')"
done
