#!/bin/bash
# chain vs events: 5 alternations of 20-step benches
python -m paper_2411_09009_b200._build > /dev/null 2>&1 || exit 1
run() { env "$@" timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>&1 | python3 -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); k=d['kernel_ms']; print(f\"{d['ms_per_step']:.3f} ms  fwd {k['fwd']:.3f} bwd {k['bwd']:.3f} clk {d['clocks']['sm_mhz']}\")
"; }
for i in 1 2 3 4 5; do
  echo "chain:  $(run CCE_FWD_CHAIN=1)"
  echo "events: $(run CCE_FWD_CHAIN=0)"
done
