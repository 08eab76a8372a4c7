#!/bin/bash
python -m paper_2411_09009_b200._build > /dev/null 2>&1 || exit 1
REPS=5 timeout 200 python scripts/stream_pass_probe.py gemma2-2b both:1,both:0,both:1,both:0,dc:0,dc:1,de:1 2>&1 | grep gemma
for pq in "36 56" "32 56" "40 60"; do set -- $pq; echo "alias0 P=$1 QC=$2: $(CCE_STREAM_P=$1 CCE_STREAM_QC=$2 REPS=5 timeout 200 python scripts/stream_pass_probe.py gemma2-2b both:0 2>&1 | grep gemma | awk '{print $4,$5}')"; done
