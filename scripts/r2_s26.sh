#!/bin/bash
python -m paper_2411_09009_b200._build > /dev/null 2>&1
timeout 600 compute-sanitizer --tool memcheck --print-limit 5 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "adapts_operands and False-64-dtype0" 2>&1 | grep -v "^    \|^=========     at\|Host Frame" | head -40
