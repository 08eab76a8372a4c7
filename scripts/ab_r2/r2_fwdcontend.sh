#!/bin/bash
# forward sweep time (fwd_kernel: the group launches alone) with the gathers overlapped (default)
# vs in line (CCE_FWD_OVERLAP=0), and the fast path's single sweep over the sorted copy
python -m paper_2411_09009_b200._build > /dev/null 2>&1 || exit 1
run() { env "$@" timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e $EXTRA 2>/dev/null | python3 -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); k=d['kernel_ms']; print(f\"{d['ms_per_step']:.2f} ms  fwd {k['fwd']:.3f} fwdk {k.get('fwd_kernel',0):.3f} bwd {k['bwd']:.3f} clk {d['clocks']['sm_mhz']}\")
"; }
for i in 1 2; do
  echo "overlap:   $(run X=1)"
  echo "inline:    $(run CCE_FWD_OVERLAP=0)"
  echo "fast:      $(EXTRA='--memory fast' run X=1)"
done
