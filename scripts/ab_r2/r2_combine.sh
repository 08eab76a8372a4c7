#!/bin/bash
# slot-parallel combine of the forward partials: tests + bench (kernel time in the launch list)
python -m paper_2411_09009_b200._build > /dev/null 2>&1 || exit 1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | grep -E "^E  |^FAILED|passed|failed" | head -5
for i in 1 2 3; do echo "bench: $(timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python3 -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); k=d['kernel_ms']; m=d['memory']; print(f\"{d['ms_per_step']:.2f} ms  fwd {k['fwd']:.3f} fwdk {k.get('fwd_kernel',0):.3f} bwd {k['bwd']:.3f} clk {d['clocks']['sm_mhz']} step {m['step_peak_transient_bytes']>>20} MiB\")
")"; done
out=gpurun_out/combine; mkdir -p $out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv \
   python bench.py --steps 1 --warmup 2 --no-cpu-baseline --no-e2e > $out/launches.log 2>&1
python scripts/launch_summary.py $out/launches.csv > $out/launches_summary.txt 2>&1; head -16 $out/launches_summary.txt
