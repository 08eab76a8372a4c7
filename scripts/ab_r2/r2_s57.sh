#!/bin/bash
python -m paper_2411_09009_b200._build > /dev/null 2>&1 || exit 1
run() { env $2 timeout 900 python bench.py --config $1 --steps 4 --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null | python3 -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); k=d['kernel_ms']; print(f\"{d['ms_per_step']:.2f} ms  fwd {k['fwd']:.2f} bwd {k['bwd']:.2f} peak {d['memory']['step_peak_transient_bytes']/2**20:.0f} MiB clk {d['clocks']['sm_mhz']}\")
"; }
for cfg in gemma2-9b nemo-12b; do
for e in "CCE_STREAM_CHUNK_TILES=128 CCE_STREAM_RING=1024" "CCE_STREAM_CHUNK_TILES=256 CCE_STREAM_RING=2048" "CCE_STREAM_CHUNK_TILES=128 CCE_STREAM_RING=2048" "CCE_STREAM_CHUNK_TILES=128 CCE_STREAM_RING=1024"; do
  echo "$cfg $e: $(run $cfg "$e")"
done; done
