#!/bin/bash
python -m paper_2411_09009_b200._build > /dev/null 2>&1 || exit 1
python -m paper_2411_09009_b200._build --variant prof CCE_STREAM_PROF=1 > /dev/null 2>&1 || exit 1
echo "== dE only, P=50"; CCE_LIB=libcce_b200_prof.so CCE_STREAM_P=50 timeout 200 python scripts/stream_prof.py de 2>&1 | tail -16
echo "== dE only, P=36"; CCE_LIB=libcce_b200_prof.so CCE_STREAM_P=36 timeout 200 python scripts/stream_prof.py de 2>&1 | tail -16
echo "== both default"; CCE_LIB=libcce_b200_prof.so timeout 200 python scripts/stream_prof.py both 2>&1 | tail -16
