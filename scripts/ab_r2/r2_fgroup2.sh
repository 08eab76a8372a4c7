#!/bin/bash
# fitted forward groups (default) vs the plain 48 MB budget (CCE_FWD_GROUP_FIT=0)
python -m paper_2411_09009_b200._build > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests/test_stream_gpu.py tests/test_memory_gpu.py tests/test_baseline_parity_gpu.py -m gpu -q -p no:cacheprovider -x 2>&1 | grep -E "^E  |^FAILED|passed|failed" | head -5
for i in 1 2 3; do for e in "CCE_FWD_GROUP_FIT=1" "CCE_FWD_GROUP_FIT=0"; do echo "bench $e: $(env $e timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python3 -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); k=d['kernel_ms']; m=d['memory']; print(f\"{d['ms_per_step']:.2f} ms  fwd {k['fwd']:.3f} fwdk {k.get('fwd_kernel',0):.3f} bwd {k['bwd']:.2f} clk {d['clocks']['sm_mhz']} fwdpeak {m['fwd_peak_transient_bytes']>>20} MiB step {m['step_peak_transient_bytes']>>20} MiB\")
")"; done; done
for c in gpt2 llama3-8b; do for e in "CCE_FWD_GROUP_FIT=1" "CCE_FWD_GROUP_FIT=0"; do echo "$c $e: $(env $e timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python3 -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); k=d['kernel_ms']; print(f\"{d['ms_per_step']:.2f} ms  fwd {k['fwd']:.3f} fwdk {k.get('fwd_kernel',0):.3f} bwd {k['bwd']:.2f} clk {d['clocks']['sm_mhz']}\")
")"; done; done
