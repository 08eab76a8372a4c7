#!/bin/bash
python -m paper_2411_09009_b200._build > /dev/null 2>&1 || exit 1
run() { env $2 timeout 900 python bench.py --config $1 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null | python3 -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); k=d['kernel_ms']; print(f\"{d['ms_per_step']:.2f} ms  fwd {k['fwd']:.2f} bwd {k['bwd']:.2f} peak {d['memory']['step_peak_transient_bytes']/2**20:.0f} MiB clk {d['clocks']['sm_mhz']}\")
"; }
for e in "X=1" "CCE_STREAM_CHUNK_TILES=512 CCE_STREAM_RING=4096" "CCE_STREAM_CHUNK_TILES=512 CCE_STREAM_RING=2048" "X=1"; do echo "nemo $e: $(run nemo-12b "$e")"; done
