#!/bin/bash
python -m paper_2411_09009_b200._build > /dev/null 2>&1 || exit 1
for pq in "32 54" "36 52" "40 50" "44 48"; do set -- $pq; echo "gemma2b-cap P=$1 QC=$2: $(CCE_STREAM_P=$1 CCE_STREAM_QC=$2 REPS=5 timeout 200 python scripts/stream_pass_probe.py gemma2b-cap both:1 2>&1 | grep gemma | awk '{print $4, $5}')"; done
for pq in "32 54" "36 52" "40 50"; do set -- $pq; echo "gemma9b P=$1 QC=$2: $(CCE_STREAM_P=$1 CCE_STREAM_QC=$2 REPS=3 timeout 600 python scripts/stream_pass_probe.py gemma9b both:1 2>&1 | grep gemma | awk '{print $4, $5}')"; done
