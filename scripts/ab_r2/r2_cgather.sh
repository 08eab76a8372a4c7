#!/bin/bash
python -m paper_2411_09009_b200._build > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests/test_stream_gpu.py tests/test_memory_gpu.py -m gpu -q -p no:cacheprovider -x 2>&1 | grep -E "^E  |^FAILED|passed|failed" | head -5
for i in 1 2; do for e in "X=1" "CCE_STREAM_CGATHER=0"; do echo "$e: $(env $e REPS=5 timeout 200 python scripts/stream_pass_probe.py gemma2-2b both:1 2>&1 | grep gemma | awk '{print $4, $5, $6, $7}')"; done; done
for i in 1 2; do for e in "X=1" "CCE_STREAM_CGATHER=0"; do echo "bench $e: $(env $e timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python3 -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); k=d['kernel_ms']; print(f\"{d['ms_per_step']:.2f} ms  fwd {k['fwd']:.2f} bwd {k['bwd']:.2f} clk {d['clocks']['sm_mhz']}\")
")"; done; done
