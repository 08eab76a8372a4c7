#!/bin/bash
python -m paper_2411_09009_b200._build > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests/test_stream_gpu.py tests/test_memory_gpu.py tests/test_baseline_parity_gpu.py -m gpu -q -p no:cacheprovider 2>&1 | grep -E "^E  |^FAILED|passed|failed" | head -20
run() { timeout 900 python bench.py --config $1 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e ${@:2} 2>/dev/null | python3 -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); k=d['kernel_ms']; print(f\"{d['ms_per_step']:.2f} ms  fwd {k['fwd']:.2f} bwd {k['bwd']:.2f} peak {d['memory']['step_peak_transient_bytes']/2**20:.0f} MiB\")
"; }
echo "gemma2b bounded: $(run gemma2-2b)"
echo "gemma2b fast: $(run gemma2-2b --memory fast)"
echo "gemma2b sigma2 bounded: $(run gemma2-2b --sigma 2)"
echo "gemma2b zipf bounded: $(run gemma2-2b --dist zipf)"
echo "llama bounded: $(run llama3-8b)"
echo "gemma9b bounded: $(run gemma2-9b)"
