#!/bin/bash
for i in 1 2; do for e in "X=1" "CCE_LIB=libcce_b200_fh.so"; do echo "$e: $(env $e timeout 300 python scripts/fwd_variants.py gemma2-2b stream:48 2>&1 | tail -1)"; done; done
for i in 1 2; do for e in "X=1" "CCE_LIB=libcce_b200_fh.so"; do echo "bench $e: $(env $e timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python3 -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); k=d['kernel_ms']; print(f\"{d['ms_per_step']:.2f} ms  fwd {k['fwd']:.2f} fwdk {k['fwd_kernel']:.2f} bwd {k['bwd']:.2f} clk {d['clocks']['sm_mhz']}\")
")"; done; done
