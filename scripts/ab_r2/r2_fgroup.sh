#!/bin/bash
# forward group sizes: 40 tiles (48 MB, default) vs 37 tiles (42 MB: 32 token pairs x 37 = 16 waves of 74 pairs)
python -m paper_2411_09009_b200._build > /dev/null 2>&1 || exit 1
for i in 1 2 3; do for e in "CCE_FWD_GROUP_MB=48" "CCE_FWD_GROUP_MB=42" "CCE_FWD_GROUP_MB=39"; do echo "bench $e: $(env $e timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python3 -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); k=d['kernel_ms']; print(f\"{d['ms_per_step']:.2f} ms  fwd {k['fwd']:.3f} fwdk {k.get('fwd_kernel',0):.3f} bwd {k['bwd']:.2f} clk {d['clocks']['sm_mhz']} mem {d['memory']}\")
")"; done; done
