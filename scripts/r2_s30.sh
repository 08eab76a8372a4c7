#!/bin/bash
python -m paper_2411_09009_b200._build > /dev/null 2>&1
CCE_STREAM_P=36 CCE_STREAM_QC=44 timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e 2>&1 | grep -v "^ \|^frame" | tail -8
timeout 300 compute-sanitizer --tool memcheck --print-limit 3 python -m pytest tests/test_stream_gpu.py -m gpu -q -p no:cacheprovider -x -k "matches_stored and 300-64" 2>&1 | grep -E "Invalid|Device Frame|at 0x|passed|failed|Error" | head -12
