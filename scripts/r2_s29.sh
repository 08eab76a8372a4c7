#!/bin/bash
python -m paper_2411_09009_b200._build > /dev/null 2>&1
run() { env "$@" timeout 300 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python3 -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(f\"{d['ms_per_step']:.2f} ms  fwd {d['kernel_ms']['fwd']:.2f} bwd {d['kernel_ms']['bwd']:.2f} peak {d['memory']['step_peak_transient_bytes']/2**20:.0f} MiB\")
"; }
for pq in "40 50" "36 44" "32 44" "36 40" "30 40"; do set -- $pq; echo "DE2 P=$1 QC=$2: $(run CCE_STREAM_P=$1 CCE_STREAM_QC=$2)"; done
echo "DE1 P=36 QC=50: $(run CCE_STREAM_DE=1 CCE_STREAM_P=36 CCE_STREAM_QC=50)"
timeout 600 python -m pytest tests/test_stream_gpu.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k stream 2>&1 | tail -2
