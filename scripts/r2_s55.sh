#!/bin/bash
python -m paper_2411_09009_b200._build > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests/test_stream_gpu.py tests/test_memory_gpu.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x 2>&1 | grep -E "^E  |^FAILED|passed|failed" | head -10
run() { env $1 timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python3 -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); k=d['kernel_ms']; print(f\"{d['ms_per_step']:.2f} ms  fwd {k['fwd']:.2f} fwdk {k.get('fwd_kernel',0):.2f} bwd {k['bwd']:.2f} peak {d['memory']['step_peak_transient_bytes']/2**20:.0f} fwdpk {d['memory']['fwd_peak_transient_bytes']/2**20:.0f} MiB clk {d['clocks']['sm_mhz']}\")
"; }
for i in 1 2; do echo "side: $(run X=1)"; echo "inline: $(run CCE_STREAM_SIDE=0)"; done
