#!/bin/bash
python -m paper_2411_09009_b200._build > /dev/null 2>&1 || exit 1
for env in "X=1"; do
echo "$env: $(env $env timeout 600 python -m pytest tests/test_stream_gpu.py -m gpu -q -p no:cacheprovider -k "unpermute" 2>&1 | grep -E "^FAILED|passed|failed" | tr '\n' ' ')"
done
timeout 600 python -m pytest tests/test_stream_gpu.py tests/test_memory_gpu.py tests/test_vocab_parallel_gpu.py tests/test_full_size_gpu.py -m gpu -q -p no:cacheprovider -x -s 2>&1 | grep -E "kept tiles|passed|failed|Error|error|assert" | head
run() { env "$@" timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python3 -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); k=d['kernel_ms']; print(f\"{d['ms_per_step']:.2f} ms  fwd {k['fwd']:.2f} fwdk {k.get('fwd_kernel',0):.2f} bwd {k['bwd']:.2f} peak {d['memory']['step_peak_transient_bytes']/2**20:.0f} MiB\")
"; }
echo "base: $(run)"
echo "base: $(run)"
