#!/bin/bash
python -m paper_2411_09009_b200._build > /dev/null 2>&1
CCE_LIB=libcce_b200_prof.so timeout 120 python scripts/stream_prof.py de 2>&1 | tail -30
