#!/bin/bash
python -m paper_2411_09009_b200._build > /dev/null 2>&1
run() { env "$@" timeout 300 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python3 -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(f\"{d['ms_per_step']:.2f} ms  fwd {d['kernel_ms']['fwd']:.2f} bwd {d['kernel_ms']['bwd']:.2f} peak {d['memory']['step_peak_transient_bytes']/2**20:.0f} MiB fwdpk {d['memory']['fwd_peak_transient_bytes']/2**20:.0f}\")
"; }
for g in 12 24 48 96; do echo "FWD_GROUP_MB=$g: $(run CCE_FWD_GROUP_MB=$g)"; done
for pq in "40 50" "36 50" "40 56" "44 50"; do set -- $pq; echo "P=$1 QC=$2: $(run CCE_STREAM_P=$1 CCE_STREAM_QC=$2)"; done
echo "R=1024 P=40 QC=50: $(run CCE_STREAM_RING=1024 CCE_STREAM_P=40 CCE_STREAM_QC=50)"
echo "fast: $(run CCE_MEMORY=fast)"
