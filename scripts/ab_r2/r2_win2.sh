#!/bin/bash
python -m paper_2411_09009_b200._build > /dev/null 2>&1 || exit 1
for e in "X=1" "CCE_STREAM_WINDOW=128" "CCE_STREAM_WINDOW=192" "CCE_STREAM_WINDOW=320" "CCE_STREAM_RING=640" "X=1"; do echo "$e: $(env $e REPS=5 timeout 200 python scripts/stream_pass_probe.py gemma2-2b both:1 2>&1 | grep gemma | awk '{print $4, $5}')"; done
