#!/bin/bash
python -m paper_2411_09009_b200._build > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests/test_stream_gpu.py -m gpu -q -p no:cacheprovider 2>&1 | tail -1
for i in 1 2; do for e in "X=1" "CCE_LIB=libcce_b200_nored.so"; do echo "$e: $(env $e REPS=5 timeout 200 python scripts/stream_pass_probe.py gemma2-2b both:1 2>&1 | grep gemma | awk '{print $4, $5}' | tr '\n' ' ')"; done; done
