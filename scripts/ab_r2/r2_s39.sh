#!/bin/bash
python -m paper_2411_09009_b200._build > /dev/null 2>&1 || exit 1
for cfg in "CCE_STREAM_P=74" "CCE_STREAM_P=74 CCE_STREAM_DYN=1" "CCE_STREAM_P=50" "CCE_STREAM_P=50 CCE_STREAM_DYN=1" "CCE_STREAM_P=36 CCE_STREAM_DYN=1"; do
  echo "$cfg: $(env $cfg REPS=5 timeout 200 python scripts/stream_pass_probe.py gemma2-2b de:1 2>&1 | grep gemma | awk '{print $4, $5, $6, $7, $8}')"
done
for cfg in "CCE_STREAM_DYN=1 CCE_STREAM_P=36 CCE_STREAM_QC=56" "CCE_STREAM_DYN=1 CCE_STREAM_P=32 CCE_STREAM_QC=50" "CCE_STREAM_DYN=1 CCE_STREAM_P=36 CCE_STREAM_QC=44" "CCE_STREAM_DYN=1"; do
  echo "both $cfg: $(env $cfg REPS=5 timeout 200 python scripts/stream_pass_probe.py gemma2-2b both:1 2>&1 | grep gemma | awk '{print $4, $5}')"
done
