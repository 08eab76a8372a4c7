#!/bin/bash
python -m paper_2411_09009_b200._build > /dev/null 2>&1
for r in 512 1024 2048; do
  echo "== R=$r dE-only P=100: $(CCE_STREAM_RING=$r CCE_STREAM_P=100 REPS=5 timeout 100 python scripts/stream_pass_probe.py gemma2-2b de:0 2>&1 | grep 'gemma' | awk '{print $5}' | tr '\n' ' ')"
  echo "== R=$r both P=40 QC=50: $(CCE_STREAM_RING=$r CCE_STREAM_P=40 CCE_STREAM_QC=50 REPS=5 timeout 100 python scripts/stream_pass_probe.py gemma2-2b both:0 2>&1 | grep 'gemma' | awk '{print $4}' | tr '\n' ' ')"
done
