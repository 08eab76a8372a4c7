#!/bin/bash
out=gpurun_out/r2s54; mkdir -p $out
python -m paper_2411_09009_b200._build > /dev/null 2>&1 || exit 1
run() { env $1 timeout 900 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python3 -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); k=d['kernel_ms']; print(f\"{d['ms_per_step']:.2f} ms  fwd {k['fwd']:.2f} fwdk {k.get('fwd_kernel',0):.2f} bwd {k['bwd']:.2f} fwdpk {d['memory']['fwd_peak_transient_bytes']/2**20:.0f} MiB clk {d['clocks']['sm_mhz']}\")
"; }
for i in 1 2; do for g in 24 48 96; do echo "group $g MB: $(run CCE_FWD_GROUP_MB=$g)"; done; done
sel="stream and (matches_stored or chunks or unpermute or gather_mode) and not 256000"
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 10 python -m pytest tests/test_stream_gpu.py -x -q -m gpu -k "$sel" -p no:cacheprovider > $out/sanitize_$tool.log 2>&1; echo "$tool exit $?"; grep -E "ERROR SUMMARY|passed|failed" $out/sanitize_$tool.log | tail -3
done
