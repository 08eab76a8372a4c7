#!/bin/bash
python -m paper_2411_09009_b200._build > /dev/null 2>&1
CCE_LIB=libcce_b200_prof.so timeout 120 python scripts/stream_prof.py de 2>&1 | tail -30 | head -12
REPS=5 timeout 200 python scripts/stream_pass_probe.py gemma2-2b 2>&1 | grep "gemma\|timed"
