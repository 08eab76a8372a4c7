#!/bin/bash
python -m paper_2411_09009_b200._build > /dev/null 2>&1 || exit 1
python -m paper_2411_09009_b200._build --variant prof CCE_STREAM_PROF=1 > /dev/null 2>&1 || exit 1
CCE_LIB=libcce_b200_prof.so timeout 300 python scripts/stream_prof.py both 2>&1 | head -12
