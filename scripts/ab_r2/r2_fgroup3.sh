#!/bin/bash
# forward groups: 37 tiles (48 MB budget, default) vs 46 tiles (52 MB budget) with folds every 4 / 8 groups
python -m paper_2411_09009_b200._build > /dev/null 2>&1 || exit 1
run() { env "$@" timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python3 -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); k=d['kernel_ms']; m=d['memory']; print(f\"{d['ms_per_step']:.2f} ms  fwd {k['fwd']:.3f} fwdk {k.get('fwd_kernel',0):.3f} bwd {k['bwd']:.3f} clk {d['clocks']['sm_mhz']} fwdpk {m['fwd_peak_transient_bytes']/2**20:.1f} step {m['step_peak_transient_bytes']/2**20:.1f} MiB\")
"; }
for i in 1 2 3; do
  echo "37/8:  $(run X=1)"
  echo "46/4:  $(run CCE_FWD_GROUP_MB=52 CCE_FWD_FOLD=4)"
  echo "46/8:  $(run CCE_FWD_GROUP_MB=52 CCE_FWD_FOLD=8)"
done
