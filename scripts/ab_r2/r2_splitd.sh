#!/bin/bash
python -m paper_2411_09009_b200._build > /dev/null 2>&1 || exit 1
for pq in "48 46" "56 42" "64 38" "72 34"; do set -- $pq; echo "gpt2 P=$1 QC=$2: $(CCE_STREAM_P=$1 CCE_STREAM_QC=$2 REPS=5 timeout 200 python scripts/stream_pass_probe.py gpt2 both:1 2>&1 | grep gpt2 | awk '{print $4, $5}')"; done
for pq in "40 50" "36 52" "32 54" "28 56" "24 58"; do set -- $pq; echo "d1536 P=$1 QC=$2: $(CCE_STREAM_P=$1 CCE_STREAM_QC=$2 REPS=5 timeout 200 python scripts/stream_pass_probe.py d1536 both:1 2>&1 | grep d1536 | awk '{print $4, $5}')"; done
for pq in "36 52" "32 54" "28 56" "24 58"; do set -- $pq; echo "llama P=$1 QC=$2: $(CCE_STREAM_P=$1 CCE_STREAM_QC=$2 REPS=5 timeout 200 python scripts/stream_pass_probe.py llama both:1 2>&1 | grep llama | awk '{print $4, $5}')"; done
