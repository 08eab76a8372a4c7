#!/bin/bash
# forward group launches as one flag-synchronised PDL chain (default) vs per-group stream waits
python -m paper_2411_09009_b200._build > /dev/null 2>&1 || exit 1
timeout 600 python -m pytest tests/test_stream_gpu.py tests/test_api_gpu.py -m gpu -q -p no:cacheprovider -x 2>&1 | grep -E "^E  |^FAILED|passed|failed|timed out|rror" | head -8
run() { env "$@" timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | python3 -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); k=d['kernel_ms']; m=d['memory']; print(f\"{d['ms_per_step']:.2f} ms  fwd {k['fwd']:.3f} fwdk {k.get('fwd_kernel',0):.3f} bwd {k['bwd']:.3f} clk {d['clocks']['sm_mhz']} fwdpk {m['fwd_peak_transient_bytes']/2**20:.1f} MiB\")
    elif 'rror' in l or 'timed out' in l: print(l.strip()[:300])
"; }
for i in 1 2 3; do
  echo "chain:  $(run CCE_FWD_CHAIN=1)"
  echo "events: $(run CCE_FWD_CHAIN=0)"
done
