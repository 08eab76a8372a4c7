#!/bin/bash
out=gpurun_out/r2s32; mkdir -p $out
python -m paper_2411_09009_b200._build > $out/build.log 2>&1 || { tail $out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_stream_gpu.py tests/test_memory_gpu.py -m gpu -q -p no:cacheprovider -x 2>&1 | tail -5
run() { env "$@" timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python3 -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); k=d['kernel_ms']; print(f\"{d['ms_per_step']:.2f} ms  fwd {k['fwd']:.2f} fwdk {k.get('fwd_kernel',0):.2f} bwd {k['bwd']:.2f} peak {d['memory']['step_peak_transient_bytes']/2**20:.0f} MiB\")
"; }
echo "base: $(run)"
echo "gather: $(run CCE_STREAM_GATHER=1)"
echo "base: $(run)"
echo "gather: $(run CCE_STREAM_GATHER=1)"
for pq in "44 50" "50 50" "30 50"; do set -- $pq; echo "gather P=$1 QC=$2: $(run CCE_STREAM_GATHER=1 CCE_STREAM_P=$1 CCE_STREAM_QC=$2)"; done
